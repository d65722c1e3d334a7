"""Time the 3-D Jacobi paths (single-sweep jacobi3d_tma vs two-sweep jacobi3d_tb2) per sweep.

    python tools/time3d.py [n ...]
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2409_18824_b200 import ftn  # noqa: E402


def main(shapes):
    torch.cuda.set_device(0)
    for shape in shapes:
        U, W = ftn.FArray.empty(shape), ftn.FArray.empty(shape)
        ftn.gen_fill(U, 18824, 0, ftn.GEN_U01)
        ftn.assign(W, U)
        for T in (1, 2):
            ftn.jacobi_set_fusion(T)
            sweeps = 10
            ftn.jacobi(U, W, sweeps)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 3
            e0.record()
            for _ in range(reps):
                ftn.jacobi(U, W, sweeps)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps / sweeps
            gl = (shape[0] - 2) * (shape[1] - 2) * (shape[2] - 2) / ms / 1e6
            print(f"{shape} T={T}: {ms:.3f} ms/sweep  {gl:.1f} GLUPS  ({gl * 16:.0f} GB/s-equiv)")
        ftn.jacobi_set_fusion(4)
        del U, W
        torch.cuda.empty_cache()


if __name__ == "__main__":
    # arguments: n (an n^3 cube) or n1xn2xn3
    main([tuple(int(v) for v in a.split("x")) if "x" in a else (int(a),) * 3 for a in sys.argv[1:]]
         or [(n,) * 3 for n in (512, 1024, 2048)])
