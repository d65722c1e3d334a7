"""Time ftn_jacobi_solve (fused residual, one host read per block) against plain ftn_jacobi on
the headline grid: GLUPS for several check intervals.

    python tools/time_solve.py [n] [sweeps]
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2409_18824_b200 import ftn  # noqa: E402


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
    sweeps = int(sys.argv[2]) if len(sys.argv) > 2 else 100
    torch.cuda.set_device(0)
    U, W = ftn.FArray.empty((n, n)), ftn.FArray.empty((n, n))
    ftn.gen_fill(U, 18824, 0, ftn.GEN_U01)
    ftn.assign(W, U)
    lups = (n - 2) ** 2 * sweeps
    ms = timeit(lambda: ftn.jacobi(U, W, sweeps))
    print(f"plain jacobi {sweeps}: {ms:.3f} ms {lups / ms / 1e6:.0f} GLUPS", flush=True)
    for every in (sweeps, 50, 20, 10):
        ms = timeit(lambda: ftn.jacobi_solve(U, W, sweeps, every, 0.0))
        print(f"solve check_every {every}: {ms:.3f} ms {lups / ms / 1e6:.0f} GLUPS", flush=True)
    for every in (50, 20):
        def blocks():
            for _ in range(sweeps // every):
                ftn.jacobi(U, W, every)
        ms = timeit(blocks)
        print(f"plain jacobi in blocks of {every}: {ms:.3f} ms {lups / ms / 1e6:.0f} GLUPS", flush=True)


if __name__ == "__main__":
    main()
