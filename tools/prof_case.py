"""Small, ncu-friendly invocations of each hot kernel (one call each after a warm-up call).

    python tools/prof_case.py [jacobi2d,jacobi3d,muladd,sum,transpose,matmul,matvec,advection|all]

Working sets are larger than L2 but small enough for ncu's replay save/restore.
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2409_18824_b200 import ftn  # noqa: E402
DEFAULT_FUSION = 0   # ftn_jacobi_set_fusion(0): back to the size-dependent default

SEED = 18824


def main(which):
    torch.cuda.set_device(0)
    if "jacobi2d" in which:
        n = 8192
        U, W = ftn.FArray.empty((n, n)), ftn.FArray.empty((n, n))
        ftn.gen_fill(U, SEED, 0, ftn.GEN_U01)
        ftn.assign(W, U)
        ftn.jacobi(U, W, 16)     # two fused launches (8 sweeps each, jacobi2d_wq<8>), the default
        ftn.jacobi(U, W, 14)     # two launches of jacobi2d_wq<7>
        ftn.jacobi_set_fusion(5)
        ftn.jacobi(U, W, 10)     # two launches of jacobi2d_wf<5> (grids <= 2^23 points use it)
        ftn.jacobi_set_fusion(1)
        ftn.jacobi(U, W, 1)      # the single-sweep kernel (jacobi2d_tma)
        ftn.jacobi_set_fusion(DEFAULT_FUSION)
        del U, W
    if "jacobi3d" in which:
        n = 512
        U, W = ftn.FArray.empty((n, n, n)), ftn.FArray.empty((n, n, n))
        ftn.gen_fill(U, SEED, 0, ftn.GEN_U01)
        ftn.assign(W, U)
        ftn.jacobi(U, W, 6)      # two launches of jacobi3d_wr<3> (the default)
        ftn.jacobi(U, W, 4)      # two launches of jacobi3d_tb2 (2 sweeps each)
        ftn.jacobi_set_fusion(1)
        ftn.jacobi(U, W, 1)      # the single-sweep kernel (jacobi3d_tma)
        ftn.jacobi_set_fusion(DEFAULT_FUSION)
        del U, W
    if "muladd" in which:
        n = 1 << 27
        b, c, d, r = (ftn.FArray.empty((n,)) for _ in range(4))
        for k, a in enumerate((b, c, d)):
            ftn.gen_fill(a, SEED, k, ftn.GEN_U01)
        ftn.muladd(r, b, c, d)
        ftn.muladd(r, b, c, d)
        del b, c, d, r
    if "sum" in which:
        x = ftn.FArray.empty((1 << 28,))
        ftn.gen_fill(x, SEED, 0, ftn.GEN_U01)
        ftn.sum(x)
        ftn.sum(x)
        del x
    if "transpose" in which:
        n = 16384
        a = ftn.FArray.empty((n, n), dtype=torch.int32)
        r = ftn.FArray.empty((n, n), dtype=torch.int32)
        ftn.gen_fill(a, SEED, 0, ftn.GEN_LINEAR)
        ftn.transpose(r, a)
        ftn.transpose(r, a)
        del a, r
    if "matmul" in which:
        n = 4096
        A, B, C = (ftn.FArray.empty((n, n)) for _ in range(3))
        ftn.gen_fill(A, SEED, 1, ftn.GEN_U11)
        ftn.gen_fill(B, SEED, 2, ftn.GEN_U11)
        ftn.matmul(C, A, B)
        ftn.matmul(C, A, B)
    if "matvec" in which:
        n = 8192
        A = ftn.FArray.empty((n, n))
        x, y = ftn.FArray.empty((n,)), ftn.FArray.empty((n,))
        ftn.gen_fill(A, SEED, 1, ftn.GEN_U11)
        ftn.gen_fill(x, SEED, 2, ftn.GEN_U11)
        for _ in range(2):
            ftn.matmul(y, A, x)   # matvec_v4_kernel + matvec_combine
            ftn.matmul(y, x, A)   # vecmat_v4_kernel
    if "advection" in which:
        nz, ny, nx = 1024, 512, 256
        F = [ftn.FArray.empty((nz, ny, nx)) for _ in range(6)]
        Z = [ftn.FArray.empty((nz,)) for _ in range(4)]
        for q, f in enumerate(F[:3] + Z):
            ftn.gen_fill(f, SEED, q, ftn.GEN_U11)
        ftn.pw_advection(*F[3:], *F[:3], *Z, 0.1, 0.2)
        ftn.pw_advection(*F[3:], *F[:3], *Z, 0.1, 0.2)
        del F, Z
    torch.cuda.synchronize()
    print("ok", ftn.launch_count())


if __name__ == "__main__":
    arg = sys.argv[1] if len(sys.argv) > 1 else "all"
    main(["jacobi2d", "jacobi3d", "muladd", "sum", "transpose", "matmul", "matvec", "advection"] if arg == "all" else arg.split(","))
