"""L2-resident Jacobi (the paper's 1024^2 shape): GLUPS per sweeps-per-launch T, plain stream
launches vs the same launch sequence captured once in a CUDA graph and replayed.
Usage: python tools/time_small.py [n] [sweeps]  -> one line per configuration."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_18824_b200 import ftn  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    sweeps = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
    U, W = ftn.FArray.empty((n, n)), ftn.FArray.empty((n, n))
    ftn.gen_fill(U, 18824, 0, ftn.GEN_U01)
    ftn.assign(W, U)
    lups = (n - 2) ** 2 * sweeps
    for T in (1, 2, 3, 4, 5, 6):
        ftn.jacobi_set_fusion(T)
        for _ in range(2):
            ftn.jacobi(U, W, sweeps)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5):
            ftn.jacobi(U, W, sweeps)
        b.record()
        torch.cuda.synchronize()
        t_stream = a.elapsed_time(b) / 5 / 1e3
        s = torch.cuda.Stream()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            ftn.jacobi(U, W, sweeps, stream=s)
            s.synchronize()
            with torch.cuda.graph(g, stream=s):
                ftn.jacobi(U, W, sweeps, stream=s)
        g.replay()
        torch.cuda.synchronize()
        a.record()
        for _ in range(5):
            g.replay()
        b.record()
        torch.cuda.synchronize()
        t_graph = a.elapsed_time(b) / 5 / 1e3
        nl = len(ftn.jacobi_plan(sweeps, T))
        print(f"n={n} T={T} launches={nl} stream {lups / t_stream / 1e9:.1f} GLUPS ({t_stream / nl * 1e6:.2f} us/launch)"
              f"  graph {lups / t_graph / 1e9:.1f} GLUPS ({t_graph / nl * 1e6:.2f} us/launch)", flush=True)
    ftn.jacobi_set_fusion(5)


if __name__ == "__main__":
    main()
