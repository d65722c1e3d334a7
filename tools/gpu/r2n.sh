mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m "gpu and not slow" -x > gpurun_out/pytest_r2n.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_r2n.log
timeout 900 python -m pytest tests/test_gpu_jacobi.py -q -m slow > gpurun_out/pytest_slow_r2n.log 2>&1; echo "slow jacobi rc=$?"; tail -2 gpurun_out/pytest_slow_r2n.log
timeout 600 python bench.py --rows c5 --no-cpu --steps 4 > gpurun_out/bench_c5_r2n.json 2>gpurun_out/bench_c5_r2n.err; echo "c5 rc=$?"
timeout 600 python bench.py --rows c5 --no-cpu --steps 4 --dist > gpurun_out/bench_c5d_r2n.json 2>>gpurun_out/bench_c5_r2n.err; echo "c5 dist rc=$?"
python - <<'PY'
import json
for f in ("gpurun_out/bench_c5_r2n.json","gpurun_out/bench_c5d_r2n.json"):
    d=json.loads(open(f).read().strip().splitlines()[-1]); print(f, d["rows"]["c5_jacobi3d_2048"])
PY
