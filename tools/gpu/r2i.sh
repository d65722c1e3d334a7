mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m "gpu and not slow" > gpurun_out/pytest_r2i.log 2>&1; echo "pytest rc=$?"; grep -E "FAILED|passed|failed" gpurun_out/pytest_r2i.log | tail -8
timeout 900 python bench.py --no-cpu > gpurun_out/bench_r2i.json 2> gpurun_out/bench_r2i.err; echo "bench rc=$?"; tail -2 gpurun_out/bench_r2i.err
