mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_matmul_streamk.py tests/test_gpu_transpose_matmul.py tests/test_gpu_matmul_f3.py tests/test_gpu_virtual_ranks.py -q -m "gpu and not slow" -x > gpurun_out/pytest_r2o.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_r2o.log
timeout 600 python - <<'PY'
import torch, sys, os
sys.path.insert(0, os.getcwd())
from paper_2409_18824_b200 import ftn
for (m, n, k) in ((8192, 1024, 8192), (8192, 8192, 8192), (8192, 2048, 8192), (4096, 4096, 4096)):
    A, B, C = ftn.FArray.empty((m, k)), ftn.FArray.empty((k, n)), ftn.FArray.empty((m, n))
    ftn.gen_fill(A, 1, 1, ftn.GEN_U11); ftn.gen_fill(B, 1, 2, ftn.GEN_U11)
    for env in ("1", "0"):
        os.environ["FTN_MATMUL_SK"] = env
        ftn.matmul(C, A, B); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5): ftn.matmul(C, A, B)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        print(m, n, k, "SK env", env, f"{ms:.3f} ms {2*m*n*k/ms/1e9:.2f} TFLOP/s", flush=True)
PY
