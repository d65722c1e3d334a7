"""Time the 3-D Jacobi paths (single-sweep jacobi3d_tma vs two-sweep jacobi3d_tb2) per sweep.

    python tools/time3d.py [n ...]
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2409_18824_b200 import ftn  # noqa: E402
DEFAULT_FUSION = 5   # ftn_jacobi_get_fusion() default (FTN_JACOBI_FUSE unset)


def main(shapes, pad=0):
    torch.cuda.set_device(0)
    for shape in shapes:
        if pad:   # leading dimension padded by `pad` elements: sections of a larger array
            BU, BW = ftn.FArray.empty((shape[0] + pad,) + shape[1:]), ftn.FArray.empty((shape[0] + pad,) + shape[1:])
            sec = [(1, shape[0])] + [(1, e) for e in shape[1:]]
            U, W = BU.section(*sec), BW.section(*sec)
        else:
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
        ftn.jacobi_set_fusion(DEFAULT_FUSION)
        del U, W
        if pad:
            del BU, BW
        torch.cuda.empty_cache()


if __name__ == "__main__":
    # arguments: [--pad P] n (an n^3 cube) or n1xn2xn3 ...
    args = sys.argv[1:]
    pad = 0
    if args[:1] == ["--pad"]:
        pad, args = int(args[1]), args[2:]
    main([tuple(int(v) for v in a.split("x")) if "x" in a else (int(a),) * 3 for a in args]
         or [(n,) * 3 for n in (512, 1024, 2048)], pad)
