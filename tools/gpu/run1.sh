set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests/test_gpu_jacobi.py -x -q -m "gpu and not slow" 2>&1 | tail -5
python tools/time2d.py 4 5 6 7 8 2>&1
FTN_WF_OLD=1 python tools/time2d.py 5 2>&1
