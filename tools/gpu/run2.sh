python tools/time2d.py 4 5 6 7 8 2>&1
python -m pytest tests/test_gpu_virtual_ranks.py -x -q 2>&1 | tail -15
python -m pytest tests/test_gpu_jacobi.py tests/test_gpu_dist.py -x -q -m "gpu and not slow" 2>&1 | tail -3
