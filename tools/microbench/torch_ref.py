# In-run library comparators (context only): cuBLAS DGEMM and torch copy/sum on B200.
import torch, time
def t(f, reps=5):
    f(); torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): f()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
for n in (4096, 8192):
    A = torch.rand(n, n, dtype=torch.float64, device="cuda"); B = torch.rand(n, n, dtype=torch.float64, device="cuda")
    ms = t(lambda: A @ B)
    print(f"cublas_dgemm_{n} {2*n**3/ms/1e9:.2f} TFLOP/s")
x = torch.rand(1 << 30, dtype=torch.float64, device="cuda")
ms = t(lambda: x.sum()); print(f"torch_sum_2^30 {x.numel()*8/ms/1e6:.1f} GB/s")
y = torch.empty_like(x); ms = t(lambda: y.copy_(x)); print(f"torch_copy_2^30 {x.numel()*16/ms/1e6:.1f} GB/s")
