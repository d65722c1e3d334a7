"""Time the 2-D Jacobi plan (ftn_jacobi) at several fusion factors T.

    python tools/time2d.py [--n N] [--sweeps S] [--reps K] T [T ...]

Prints one line per T: ms per step of S sweeps, GLUPS, and the per-launch HBM fraction
(16 B per interior point per launch / launch time, MEASURED_PEAKS hbm_gbs if present).
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2409_18824_b200 import ftn  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=8192)
    ap.add_argument("--sweeps", type=int, default=100)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("T", type=int, nargs="*", default=[5])
    a = ap.parse_args()
    torch.cuda.set_device(0)
    peak = 6556.2
    try:
        peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:
        pass
    n = a.n
    U, W = ftn.FArray.empty((n, n)), ftn.FArray.empty((n, n))
    ftn.gen_fill(U, 18824, 0, ftn.GEN_U01)
    ftn.assign(W, U)
    for T in a.T:
        ftn.jacobi_set_fusion(T)
        plan = ftn.jacobi_plan(a.sweeps, T)
        ftn.jacobi(U, W, a.sweeps)
        torch.cuda.synchronize()
        times = []
        for _ in range(a.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            ftn.jacobi(U, W, a.sweeps)
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
        ms = min(times)
        glups = (n - 2) ** 2 * a.sweeps / ms / 1e6
        per_launch = ms / len(plan)
        frac = 16 * (n - 2) ** 2 / (per_launch * 1e-3) / 1e9 / peak
        print(json.dumps({"T": T, "n": n, "sweeps": a.sweeps, "launches": len(plan), "ms_min": round(ms, 3),
                          "ms_all": [round(t, 3) for t in times], "glups": round(glups, 1),
                          "per_launch_hbm_frac": round(frac, 3)}), flush=True)


if __name__ == "__main__":
    main()
