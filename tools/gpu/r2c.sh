mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m "gpu and not slow" > gpurun_out/pytest_r2c.log 2>&1; echo "pytest rc=$?"; grep -E "FAILED|ERROR|passed|failed" gpurun_out/pytest_r2c.log | tail -25
