"""One jacobi3d_tb2 launch (plus one single sweep) on an n^3 grid, for ncu.

    python tools/prof3d.py n
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2409_18824_b200 import ftn  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
torch.cuda.set_device(0)
U, W = ftn.FArray.empty((n, n, n)), ftn.FArray.empty((n, n, n))
ftn.gen_fill(U, 18824, 0, ftn.GEN_U01)
ftn.assign(W, U)
ftn.jacobi(U, W, 4)   # two jacobi3d_tb2 launches
torch.cuda.synchronize()
print("ok", ftn.launch_count())
