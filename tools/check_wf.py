"""Parity of the 2-D fused Jacobi for one fusion T under the current FTN_WF_CFG (tuning aid):
python tools/check_wf.py T"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import synth  # noqa: E402
from oracle import FArray as OA  # noqa: E402
from paper_2409_18824_b200 import ftn  # noqa: E402

T = int(sys.argv[1])
ftn.jacobi_set_fusion(T)
bad = 0
for shape in [(3, 3), (5, 40), (40, 5), (129, 31), (200, 301), (257, 77), (1000, 130), (3000, 2000)]:
    for sweeps in (1, 2, T, T + 1, 2 * T, 3 * T + 1, 12):
        u0 = synth.jacobi_init(shape, array_id=sum(shape) + sweeps)
        U, W = ftn.FArray.from_numpy(u0), ftn.FArray.from_numpy(u0)
        new = ftn.jacobi(U, W, sweeps)
        uo, wo = u0.copy(order="F"), u0.copy(order="F")
        newo = oracle.jacobi(OA(uo), OA(wo), sweeps, 0.25)
        ok = new == newo and np.array_equal((W if new else U).to_numpy(), wo if newo else uo)
        bad += not ok
        if not ok:
            print("MISMATCH", shape, sweeps)
print("check_wf T=%d cfg=%s: %s" % (T, os.environ.get("FTN_WF_CFG", "default"), "ok" if not bad else f"{bad} bad"))
