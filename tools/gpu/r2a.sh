set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/pytest_r2a.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_r2a.log
timeout 300 python tools/time2d.py 4 5 6 7 8 2>&1
FTN_WF_OLD=1 timeout 120 python tools/time2d.py 5 2>&1
timeout 600 python bench.py > gpurun_out/bench_r2a.json 2> gpurun_out/bench_r2a.err; echo "bench rc=$?"; head -c 1500 gpurun_out/bench_r2a.json
