set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_solve.py tests/test_gpu_virtual_ranks.py tests/test_gpu_advection.py tests/test_gpu_elemental.py tests/test_gpu_jacobi.py tests/test_gpu_nccl.py tests/test_gpu_dist.py -x -q -m "gpu and not slow" > gpurun_out/pytest_r2b.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_r2b.log
timeout 600 python bench.py --rows c5 --no-cpu --steps 4 --warmup 3 > gpurun_out/bench_c5_r2b.json 2> gpurun_out/bench_c5_r2b.err; echo "c5 rc=$?"
timeout 600 python bench.py --rows c5 --no-cpu --steps 4 --warmup 3 --dist > gpurun_out/bench_c5dist_r2b.json 2> gpurun_out/bench_c5dist_r2b.err; echo "c5 dist rc=$?"
python - <<'PY'
import json
for f in ("gpurun_out/bench_c5_r2b.json", "gpurun_out/bench_c5dist_r2b.json"):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d["value"], d["rows"].get("c5_jacobi3d_2048"))
    except Exception as e:
        print(f, "ERR", e)
PY
tail -3 gpurun_out/bench_c5_r2b.err gpurun_out/bench_c5dist_r2b.err
