"""Time the 3-D Jacobi (jacobi3d_wr<T>) at several fusion factors: GLUPS of `sweeps` sweeps.
The rank-3 fusion is capped at FTN_J3_T (default 3): set FTN_J3_T=4 to time T = 4; the line
prints the T actually used.

    python tools/time3d_T.py [--sweeps S] [--reps K] n [n ...]
"""
import argparse
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2409_18824_b200 import ftn  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sweeps", type=int, default=100)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--T", default="2,3,4")
    ap.add_argument("n", type=int, nargs="*", default=[2048])
    a = ap.parse_args()
    torch.cuda.set_device(0)
    for n in a.n:
        U, W = ftn.FArray.empty((n, n, n)), ftn.FArray.empty((n, n, n))
        ftn.gen_fill(U, 18824, 7, ftn.GEN_U01)
        ftn.assign(W, U)
        for T in [int(x) for x in a.T.split(",")]:
            ftn.jacobi_set_fusion(T)
            ftn.jacobi(U, W, a.sweeps)
            torch.cuda.synchronize()
            ts = []
            for _ in range(a.reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                ftn.jacobi(U, W, a.sweeps)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            ms = min(ts)
            Ta = ftn.jacobi_fusion(U)          # the sweeps per launch actually used (rank 3: <= FTN_J3_T)
            nl = len(ftn.jacobi_plan(a.sweeps, Ta))
            gl = (n - 2) ** 3 * a.sweeps / ms / 1e6
            print(f"n={n} T={Ta} launches={nl} {ms:.2f} ms {gl:.1f} GLUPS per-launch HBM "
                  f"{16 * (n - 2) ** 3 * nl / ms / 1e6:.0f} GB/s", flush=True)
        ftn.jacobi_set_fusion(0)
        del U, W
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
