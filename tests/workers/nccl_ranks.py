"""One rank of the real NCCL multi-GPU path (launched by tests/test_gpu_nccl.py under
torchrun, one process per GPU).  Each rank runs the library's distributed calls on its slab
-- ftn_jacobi_dist, ftn_jacobi_solve_dist, ftn_{sum,maxval,dot_product}_global, ftn_bcast +
ftn_matmul_colsharded -- and compares its owned part with the ORACLE on the undivided array;
rank 0 prints "NCCL-RANKS OK" when every rank passed."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
from oracle import FArray as OA  # noqa: E402
from paper_2409_18824_b200 import dist as D  # noqa: E402
from paper_2409_18824_b200 import ftn  # noqa: E402


def slab_of(ftn, u0, p, r, halo):
    g0, nl = D.jacobi_slab(u0.shape[-1], p, r, halo)
    part = np.full(u0.shape[:-1] + (nl,), 7.0e300, order="F")
    for k in range(nl):
        if 0 <= g0 + k < u0.shape[-1]:
            part[..., k] = u0[..., g0 + k]
    return g0, nl, ftn.FArray.from_numpy(part), ftn.FArray.from_numpy(part)


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    comm = ftn.Comm.from_torch_distributed(local)
    ok = True
    try:
        # Jacobi (2-D deep halo with overlap, 3-D two-sweep slabs)
        for shape, halo, sweeps in (((300, 203), 5, 23), ((70, 40, 61), 2, 9)):
            coeff = 0.25 if len(shape) == 2 else 1.0 / 6.0
            u0 = synth.jacobi_init(shape, array_id=3)
            a, b = u0.copy(order="F"), u0.copy(order="F")
            new_o = oracle.jacobi(OA(a), OA(b), sweeps, coeff)
            ref = b if new_o else a
            g0, nl, U, W = slab_of(ftn, u0, world, rank, halo)
            new = comm.jacobi(U, W, sweeps, coeff, halo=halo)
            got = (W if new else U).to_numpy()[..., halo:nl - halo]
            ok &= new == new_o and np.array_equal(got, ref[..., g0 + halo:g0 + nl - halo])
            # to convergence
            a, b = u0.copy(order="F"), u0.copy(order="F")
            d_o, r_o, n_o = oracle.jacobi_solve(OA(a), OA(b), 30, 7, 1e-3, coeff)
            ref = b if n_o else a
            g0, nl, U, W = slab_of(ftn, u0, world, rank, halo)
            d, r_, n = comm.jacobi_solve(U, W, 30, 7, 1e-3, coeff, halo=halo)
            got = (W if n else U).to_numpy()[..., halo:nl - halo]
            ok &= (d, r_, n) == (d_o, r_o, n_o) and np.array_equal(got, ref[..., g0 + halo:g0 + nl - halo])
        # global reductions on chunk-aligned slabs: bit-identical to the oracle's order R
        n_local = 65536 * 4
        xs = synth.values(n_local * world, array_id=21, mode=synth.U11)
        ys = synth.values(n_local * world, array_id=22, mode=synth.U11)
        X = ftn.FArray.from_numpy(np.asfortranarray(xs[rank * n_local:(rank + 1) * n_local]))
        Y = ftn.FArray.from_numpy(np.asfortranarray(ys[rank * n_local:(rank + 1) * n_local]))
        XO, YO = OA(np.asfortranarray(xs)), OA(np.asfortranarray(ys))
        ok &= comm.sum(X).item() == oracle.reduce_orderR(XO, oracle.SUM)
        ok &= comm.maxval(X).item() == oracle.maxval(XO)
        ok &= comm.dot_product(X, Y).item() == oracle.dot_orderR(XO, YO)
        # bcast + column-sharded MATMUL
        m, k, n = 96, 64, 32 * world
        a_h = synth.farray((m, k), array_id=11, mode=synth.U11)
        b_h = synth.farray((k, n), array_id=12, mode=synth.U11)
        A = ftn.FArray.from_numpy(a_h if rank == 0 else np.zeros((m, k), order="F"))
        nb = n // world
        B = ftn.FArray.from_numpy(np.asfortranarray(b_h[:, rank * nb:(rank + 1) * nb]))
        C = ftn.FArray.empty((m, nb))
        comm.bcast(A, 0)
        comm.matmul(C, A, B)
        co, ab = np.zeros((m, n), order="F"), np.zeros((m, n), order="F")
        oracle.matmul(OA(co), OA(a_h), OA(b_h), OA(ab))
        sl = slice(rank * nb, (rank + 1) * nb)
        ok &= np.array_equal(A.to_numpy(), a_h)
        ok &= bool(np.all(np.abs(C.to_numpy() - co[:, sl]) <= 4 * k * 2.0 ** -53 * ab[:, sl]))
    finally:
        torch.cuda.synchronize()
        flag = torch.tensor([1 if ok else 0], device="cuda")
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        comm.destroy()
        dist.destroy_process_group()
    if rank == 0:
        print("NCCL-RANKS OK" if int(flag.item()) == 1 else "NCCL-RANKS FAILED", flush=True)
    return 0 if int(flag.item()) == 1 else 1


if __name__ == "__main__":
    sys.exit(main())
