"""Jacobi on arrays the TMA kernels cannot address (odd leading dimension, strided section):
padded fused path vs the generic kernel.  python tools/time_odd.py"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2409_18824_b200 import ftn  # noqa: E402


def t(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


for shape, sec in [((8191, 8192), None), ((16384, 8192), ((1, 16384, 2), (1, 8192)))]:
    U, W = ftn.FArray.empty(shape), ftn.FArray.empty(shape)
    ftn.gen_fill(U, 1, 0, ftn.GEN_U01)
    ftn.assign(W, U)
    su, sw = (U, W) if sec is None else (U.section(*sec), W.section(*sec))
    n = su.shape
    ms = t(lambda: ftn.jacobi(su, sw, 100))
    print(f"{shape} section={sec is not None}: 100 sweeps {ms:.1f} ms = {(n[0]-2)*(n[1]-2)*100/ms/1e6:.0f} GLUPS")
