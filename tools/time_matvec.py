"""Time the rank-1 MATMUL forms (f3): y = MATMUL(a, x) and y = MATMUL(x, b), 8192^2 real(8),
GB/s of the matrix stream (8 B per element).

    python tools/time_matvec.py [n]
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2409_18824_b200 import ftn  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
    torch.cuda.set_device(0)
    A = ftn.FArray.empty((n, n))
    ftn.gen_fill(A, 18824, 1, ftn.GEN_U11)
    x = ftn.FArray.empty((n,))
    ftn.gen_fill(x, 18824, 2, ftn.GEN_U11)
    y = ftn.FArray.empty((n,))
    for name, fn in (("matvec", lambda: ftn.matmul(y, A, x)), ("vecmat", lambda: ftn.matmul(y, x, A))):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        reps = 20
        ev[0].record()
        for _ in range(reps):
            fn()
        ev[1].record()
        torch.cuda.synchronize()
        ms = ev[0].elapsed_time(ev[1]) / reps
        print(f"{name} {n}^2: {ms * 1e3:.1f} us {8 * n * n / ms / 1e6:.0f} GB/s", flush=True)


if __name__ == "__main__":
    main()
