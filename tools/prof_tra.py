"""tra-adv launches for timing / ncu: python tools/prof_tra.py [ni nj nk] [iters]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_18824_b200 import ftn  # noqa: E402

ni, nj, nk = (int(v) for v in sys.argv[1:4]) if len(sys.argv) >= 4 else (1024, 512, 512)
iters = int(sys.argv[4]) if len(sys.argv) >= 5 else 1
D = [ftn.FArray.empty((ni, nj, nk)) for _ in range(8)]
for q, d in enumerate(D):
    ftn.gen_fill(d, 18824, 70 + q, ftn.GEN_U11 if q < 5 else ftn.GEN_U01)
D2 = [ftn.FArray.empty((ni, nj)) for _ in range(3)]
for q, d in enumerate(D2):
    ftn.gen_fill(d, 18824, 90 + q, ftn.GEN_U01)
RZ = ftn.FArray.empty((nk,))
ftn.gen_fill(RZ, 18824, 95, ftn.GEN_U01)
ftn.tra_adv(*D, *D2, RZ, iters)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
ftn.tra_adv(*D, *D2, RZ, iters)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
print(f"{ni}x{nj}x{nk} x{iters}: {ms:.2f} ms, {ni * nj * nk * iters / ms / 1e6:.2f} Gcell-it/s", flush=True)
