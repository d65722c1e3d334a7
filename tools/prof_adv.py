"""pw-advection launches for timing / ncu: python tools/prof_adv.py [nz ny nx] [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_18824_b200 import ftn  # noqa: E402

nz, ny, nx = (int(v) for v in sys.argv[1:4]) if len(sys.argv) >= 4 else (2048, 1024, 1024)
reps = int(sys.argv[4]) if len(sys.argv) >= 5 else 5
F = [ftn.FArray.empty((nz, ny, nx)) for _ in range(3)]
O = [ftn.FArray.empty((nz, ny, nx)) for _ in range(3)]
Z = [ftn.FArray.empty((nz,)) for _ in range(4)]
for q, f in enumerate(F):
    ftn.gen_fill(f, 18824, 50 + q, ftn.GEN_U11)
for q, z in enumerate(Z):
    ftn.gen_fill(z, 18824, 60 + q, ftn.GEN_U11)
ftn.pw_advection(*O, *F, *Z, 0.1, 0.2)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    ftn.pw_advection(*O, *F, *Z, 0.1, 0.2)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
cells = (nz - 2) * (ny - 2) * (nx - 2)
print(f"{nz}x{ny}x{nx}: {ms:.3f} ms  {cells / ms / 1e6:.1f} Gcells/s  {48 * cells / ms / 1e6:.0f} GB/s", flush=True)
