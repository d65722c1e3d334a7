mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tra_adv.py -q -x > gpurun_out/pytest_tra2.log 2>&1; echo "pytest fused rc=$?"; tail -3 gpurun_out/pytest_tra2.log
FTN_TA_PASSES=8 timeout 900 python -m pytest tests/test_gpu_tra_adv.py -q -x -m "not slow" 2>&1 | tail -1
timeout 600 python bench.py --rows f4 --no-cpu --steps 4 > gpurun_out/bench_f4b.json 2> gpurun_out/bench_f4b.err; echo "bench rc=$?"
python - <<'PY'
import json
d=json.loads(open("gpurun_out/bench_f4b.json").read().strip().splitlines()[-1]); print(json.dumps(d["rows"]["f4_tra_adv_1024x512x512_x20"], indent=1))
PY
