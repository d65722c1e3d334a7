mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m "gpu and not slow" -x > gpurun_out/pytest_r2g.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_r2g.log
timeout 600 python -m pytest tests/test_gpu_jacobi.py -q -m slow -k c2_full > gpurun_out/pytest_slow_r2g.log 2>&1; echo "slow c2 rc=$?"; tail -2 gpurun_out/pytest_slow_r2g.log
timeout 900 python bench.py > gpurun_out/bench_r2g.json 2> gpurun_out/bench_r2g.err; echo "bench rc=$?"
python bench.py --steps 2 --warmup 1 --rows none --no-cpu > gpurun_out/bench_small_r2g.json 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r2g.csv \
  python bench.py --steps 2 --warmup 1 --rows none --no-cpu > gpurun_out/ncu_launch_r2g.log 2>&1; echo "ncu launches rc=$?"
python tools/time2d.py --reps 1 8 > gpurun_out/plain_wq8_r2g.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:jacobi2d_wq -s 2 -c 1 \
    -o gpurun_out/wq8_r2g -f python tools/time2d.py --reps 1 8 > gpurun_out/ncu_wq8_r2g.log 2>&1; echo "ncu full rc=$?"
