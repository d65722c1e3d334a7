mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tra_adv.py -q -x > gpurun_out/pytest_tra.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_tra.log
timeout 600 python bench.py --rows f4 --no-cpu --steps 4 > gpurun_out/bench_f4.json 2> gpurun_out/bench_f4.err; echo "bench rc=$?"; tail -2 gpurun_out/bench_f4.err
python - <<'PY'
import json
d=json.loads(open("gpurun_out/bench_f4.json").read().strip().splitlines()[-1]); print(json.dumps(d["rows"], indent=1))
PY
