"""One jacobi3d_wr<T> launch (T sweeps) on an n^3 grid, for ncu.

    python tools/prof3d_wr.py n T
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2409_18824_b200 import ftn  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
T = int(sys.argv[2]) if len(sys.argv) > 2 else 3
torch.cuda.set_device(0)
U, W = ftn.FArray.empty((n, n, n)), ftn.FArray.empty((n, n, n))
ftn.gen_fill(U, 18824, 0, ftn.GEN_U01)
ftn.assign(W, U)
ftn.jacobi_set_fusion(T)
ftn.jacobi(U, W, T)   # one jacobi3d_wr<T> launch
torch.cuda.synchronize()
print("ok", ftn.launch_count())
