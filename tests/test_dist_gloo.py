"""CPU (gloo, world size 2 and 4) tests of the multi-GPU plan.

The NCCL exchange itself lives in libftn (ftn_jacobi_dist, ftn_*_global) and needs GPUs;
here the same protocol -- last-dimension slabs with one halo plane per side, owned
boundary planes sent to r-1 / r+1 every sweep, rank partials all-gathered and combined
by the fixed tree -- is run with torch.distributed over gloo, the per-rank compute done
by the oracle, and the gathered result compared bit for bit with the undivided oracle.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_2409_18824_b200 import dist as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_slab_partition():
    for n in (1, 2, 7, 64, 2048):
        for p in (1, 2, 3, 4, 8):
            if p > n:
                continue
            slabs = [D.slab(n, p, r) for r in range(p)]
            assert slabs[0].lo == 0 and slabs[-1].hi == n
            for a, b in zip(slabs, slabs[1:]):
                assert a.hi == b.lo
            sizes = [s.owned for s in slabs]
            assert max(sizes) - min(sizes) <= 1
    g0, nl = D.jacobi_slab(2048, 8, 3)
    assert nl == 2046 // 8 + (1 if 3 < 2046 % 8 else 0) + 2 and g0 == 3 * (2046 // 8) + min(3, 2046 % 8)
    assert D.reduction_slab_aligned(1 << 30, 1 << 20, 8)
    assert not D.reduction_slab_aligned(1 << 30, 1 << 20, 3)


def _worker(rank, world, port, q, shape2, shape3, sweeps):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = {}
        for shape, coeff in ((shape2, 0.25), (shape3, 1.0 / 6.0)):
            full = synth.jacobi_init(shape)
            nlast = shape[-1]
            g0, nl = D.jacobi_slab(nlast, world, rank)
            # local arrays hold global planes [g0, g0 + nl)
            sl = [slice(None)] * (len(shape) - 1)
            u = np.asfortranarray(full[tuple(sl + [slice(g0, g0 + nl)])].copy())
            w = u.copy(order="F")
            cur, nxt = u, w
            for _ in range(sweeps):
                # halo exchange of the source (the protocol of ftn_jacobi_dist)
                reqs = []
                recv_lo = torch.empty(cur[..., 0].size, dtype=torch.float64)
                recv_hi = torch.empty(cur[..., 0].size, dtype=torch.float64)
                if rank > 0:
                    reqs.append(dist.isend(torch.from_numpy(cur[..., 1].ravel(order="F").copy()), rank - 1))
                    reqs.append(dist.irecv(recv_lo, rank - 1))
                if rank < world - 1:
                    reqs.append(dist.isend(torch.from_numpy(cur[..., nl - 2].ravel(order="F").copy()), rank + 1))
                    reqs.append(dist.irecv(recv_hi, rank + 1))
                for r in reqs:
                    r.wait()
                if rank > 0:
                    cur[..., 0] = recv_lo.numpy().reshape(cur[..., 0].shape, order="F")
                if rank < world - 1:
                    cur[..., nl - 1] = recv_hi.numpy().reshape(cur[..., 0].shape, order="F")
                oracle.jacobi(oracle.FArray(cur), oracle.FArray(nxt), 1, coeff)  # local interior
                cur, nxt = nxt, cur
            owned = cur[..., 1:nl - 1]
            parts = [None] * world
            dist.all_gather_object(parts, (g0 + 1, owned))
            out[len(shape)] = parts
        # global SUM: local order-R value of a chunk-aligned slab, all-gather, fixed tree
        n = 4 * 65536 * world
        v = synth.values(n, mode=synth.U11)
        per = n // world
        local = oracle.reduce_orderR(oracle.FArray(v[rank * per:(rank + 1) * per].copy()), oracle.SUM)
        t = torch.tensor([local], dtype=torch.float64)
        gathered = [torch.empty(1, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(gathered, t)
        out["sum"] = oracle.tree_combine([g.item() for g in gathered], oracle.SUM)
        if rank == 0:
            q.put(out)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_distributed_protocol_matches_undivided(world):
    shape2, shape3, sweeps = (37, 46), (19, 13, 26), 5
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, shape2, shape3, sweeps)) for r in range(world)]
    for p in procs:
        p.start()
    out = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for shape, coeff in ((shape2, 0.25), (shape3, 1.0 / 6.0)):
        full = synth.jacobi_init(shape)
        a, b = full.copy(order="F"), full.copy(order="F")
        new = oracle.jacobi(oracle.FArray(a), oracle.FArray(b), sweeps, coeff)
        ref = b if new else a
        for first, owned in out[len(shape)]:
            np.testing.assert_array_equal(owned, ref[..., first:first + owned.shape[-1]])
    n = 4 * 65536 * world
    v = synth.values(n, mode=synth.U11)
    assert out["sum"] == oracle.reduce_orderR(oracle.FArray(v), oracle.SUM)   # decomposition independent
