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
        for shape, coeff, halo in ((shape2, 0.25, 1), (shape2, 0.25, 3), (shape3, 1.0 / 6.0, 1)):
            full = synth.jacobi_init(shape)
            nlast = shape[-1]
            sl = D.slab(nlast - 2, world, rank)          # owned global planes [sl.lo+1, sl.hi+1)
            g0 = sl.lo + 1 - halo                       # global plane of local plane 0
            nl = sl.owned + 2 * halo
            cur = np.full(shape[:-1] + (nl,), np.nan, order="F")
            for k in range(nl):
                if 0 <= g0 + k < nlast:
                    cur[..., k] = full[..., g0 + k]
            nxt = cur.copy(order="F")
            k_sweeps = halo                              # sweeps per exchange (ftn_jacobi_dist's T)
            steps = [k_sweeps] * (sweeps // k_sweeps) + [1] * (sweeps % k_sweeps)
            for k in steps:
                # exchange the k owned planes next to each neighbour into its k innermost halo planes
                reqs = []
                plane_sz = int(np.prod(shape[:-1]))
                recv_lo = torch.empty(plane_sz * k, dtype=torch.float64)
                recv_hi = torch.empty(plane_sz * k, dtype=torch.float64)
                if rank > 0:
                    reqs.append(dist.isend(torch.from_numpy(cur[..., halo:halo + k].ravel(order="F").copy()), rank - 1))
                    reqs.append(dist.irecv(recv_lo, rank - 1))
                if rank < world - 1:
                    reqs.append(dist.isend(torch.from_numpy(cur[..., nl - halo - k:nl - halo].ravel(order="F").copy()),
                                           rank + 1))
                    reqs.append(dist.irecv(recv_hi, rank + 1))
                for r in reqs:
                    r.wait()
                if rank > 0:
                    cur[..., halo - k:halo] = recv_lo.numpy().reshape(shape[:-1] + (k,), order="F")
                if rank < world - 1:
                    cur[..., nl - halo:nl - halo + k] = recv_hi.numpy().reshape(shape[:-1] + (k,), order="F")
                # k local sweeps on the window [halo - k, nl - halo + k): its outer planes are held
                # fixed by the oracle (the global boundary on the first / last rank), and errors
                # from holding a halo plane fixed travel one plane per sweep, never reaching the
                # owned planes.  Only the owned planes are kept.
                lo = max(halo - k, halo - 1 if rank == 0 else 0)
                hi = min(nl - halo + k, nl - halo + 1 if rank == world - 1 else nl)
                a = np.asfortranarray(cur[..., lo:hi])
                b = a.copy(order="F")
                new = oracle.jacobi(oracle.FArray(a), oracle.FArray(b), k, coeff)
                res = b if new else a
                nxt[..., halo:nl - halo] = res[..., halo - lo:nl - halo - lo]
                cur, nxt = nxt, cur
            owned = cur[..., halo:nl - halo]
            parts = [None] * world
            dist.all_gather_object(parts, (g0 + halo, owned))
            out[(len(shape), halo)] = parts
        # global SUM: local order-R value of a chunk-aligned slab, all-gather, fixed tree
        n = 4 * 65536 * world
        v = synth.values(n, mode=synth.U11)
        per = n // world
        local = oracle.reduce_orderR(oracle.FArray(v[rank * per:(rank + 1) * per].copy()), oracle.SUM)
        t = torch.tensor([local], dtype=torch.float64)
        gathered = [torch.empty(1, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(gathered, t)
        out["sum"] = oracle.tree_combine([g.item() for g in gathered], oracle.SUM)
        # global MAXVAL: local value, all-reduce MAX (order-free)
        tm = torch.tensor([oracle.reduce_orderR(oracle.FArray(v[rank * per:(rank + 1) * per].copy()), oracle.MAX)],
                          dtype=torch.float64)
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
        out["max"] = tm.item()
        # column-sharded MATMUL (ftn_matmul_colsharded's plan): A broadcast from rank 0, rank r
        # owns the column block J_r of b and c; blocks gathered in rank order
        m, k, n = 23, 17, 4 * world + 3
        a_full = synth.farray((m, k), array_id=31, mode=synth.U11) if rank == 0 else np.zeros((m, k), order="F")
        ta = torch.from_numpy(np.ascontiguousarray(a_full.ravel(order="F")))
        dist.broadcast(ta, 0)
        a_loc = np.asfortranarray(ta.numpy().reshape((m, k), order="F"))
        b_full = synth.farray((k, n), array_id=32, mode=synth.U11)
        cols = D.slab(n, world, rank)
        c_loc = np.zeros((m, cols.owned), order="F")
        oracle.matmul(oracle.FArray(c_loc), oracle.FArray(a_loc),
                      oracle.FArray(np.asfortranarray(b_full[:, cols.lo:cols.hi])))
        blocks = [None] * world
        dist.all_gather_object(blocks, (cols.lo, c_loc))
        out["matmul"] = blocks
        if rank == 0:
            q.put(out)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_distributed_protocol_matches_undivided(world):
    shape2, shape3, sweeps = (37, 46), (19, 13, 26), 7
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
    for shape, coeff, halo in ((shape2, 0.25, 1), (shape2, 0.25, 3), (shape3, 1.0 / 6.0, 1)):
        full = synth.jacobi_init(shape)
        a, b = full.copy(order="F"), full.copy(order="F")
        new = oracle.jacobi(oracle.FArray(a), oracle.FArray(b), sweeps, coeff)
        ref = b if new else a
        for first, owned in out[(len(shape), halo)]:
            np.testing.assert_array_equal(owned, ref[..., first:first + owned.shape[-1]])
    n = 4 * 65536 * world
    v = synth.values(n, mode=synth.U11)
    assert out["sum"] == oracle.reduce_orderR(oracle.FArray(v), oracle.SUM)   # decomposition independent
    assert out["max"] == oracle.reduce_orderR(oracle.FArray(v), oracle.MAX)
    m, k, n = 23, 17, 4 * world + 3
    a = synth.farray((m, k), array_id=31, mode=synth.U11)
    b = synth.farray((k, n), array_id=32, mode=synth.U11)
    c = np.zeros((m, n), order="F")
    oracle.matmul(oracle.FArray(c), oracle.FArray(a), oracle.FArray(b))
    got = np.zeros((m, n), order="F")
    for lo, blk in out["matmul"]:
        got[:, lo:lo + blk.shape[1]] = blk
    np.testing.assert_array_equal(got, c)      # every element's fold is local to one rank


def _solve_worker(rank, world, port, q, shape, max_sweeps, check, tol):
    """ftn_jacobi_solve_dist's protocol with the oracle as the local compute: halo-1 slabs, one
    sweep per exchange, and after every block of `check` sweeps the residual over each rank's
    owned interior, all-gathered; the maximum decides the stop (R#25)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        coeff = 0.25 if len(shape) == 2 else 1.0 / 6.0
        full = synth.jacobi_init(shape, array_id=5)
        nlast = shape[-1]
        sl = D.slab(nlast - 2, world, rank)
        g0, nl = sl.lo, sl.owned + 2                  # halo 1: local plane 0 = global plane sl.lo
        cur = np.asfortranarray(full[..., g0:g0 + nl].copy())
        prev = cur.copy(order="F")
        plane_sz = int(np.prod(shape[:-1]))
        inner = (slice(1, -1),) * (len(shape) - 1)
        done, res = 0, 0.0
        while done < max_sweeps:
            k = min(check, max_sweeps - done)
            for _ in range(k):
                reqs = []
                lo_buf = torch.empty(plane_sz, dtype=torch.float64)
                hi_buf = torch.empty(plane_sz, dtype=torch.float64)
                if rank > 0:
                    reqs.append(dist.isend(torch.from_numpy(cur[..., 1].ravel(order="F").copy()), rank - 1))
                    reqs.append(dist.irecv(lo_buf, rank - 1))
                if rank < world - 1:
                    reqs.append(dist.isend(torch.from_numpy(cur[..., nl - 2].ravel(order="F").copy()), rank + 1))
                    reqs.append(dist.irecv(hi_buf, rank + 1))
                for r in reqs:
                    r.wait()
                if rank > 0:
                    cur[..., 0] = lo_buf.numpy().reshape(shape[:-1], order="F")
                if rank < world - 1:
                    cur[..., nl - 1] = hi_buf.numpy().reshape(shape[:-1], order="F")
                prev = cur.copy(order="F")
                a, b = cur.copy(order="F"), cur.copy(order="F")
                new = oracle.jacobi(oracle.FArray(a), oracle.FArray(b), 1, coeff)
                cur = np.asfortranarray(b if new else a)
            done += k
            local = oracle.maxabsdiff(oracle.FArray(np.asfortranarray(cur[inner + (slice(1, nl - 1),)])),
                                      oracle.FArray(np.asfortranarray(prev[inner + (slice(1, nl - 1),)])))
            vals = [torch.empty(1, dtype=torch.float64) for _ in range(world)]
            dist.all_gather(vals, torch.tensor([local], dtype=torch.float64))
            res = max(v.item() for v in vals)
            if res <= tol:
                break
        parts = [None] * world
        dist.all_gather_object(parts, (g0 + 1, cur[..., 1:nl - 1].copy(order="F")))
        if rank == 0:
            q.put((done, res, parts))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("shape,check,tol", [((23, 31), 4, 1e-2), ((11, 9, 14), 3, -1.0)])
def test_distributed_solve_protocol_matches_undivided(world, shape, check, tol):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_solve_worker, args=(r, world, port, q, shape, 17, check, tol)) for r in range(world)]
    for p in procs:
        p.start()
    done, res, parts = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    coeff = 0.25 if len(shape) == 2 else 1.0 / 6.0
    full = synth.jacobi_init(shape, array_id=5)
    a, b = full.copy(order="F"), full.copy(order="F")
    d_o, r_o, n_o = oracle.jacobi_solve(oracle.FArray(a), oracle.FArray(b), 17, check, tol, coeff)
    ref = b if n_o else a
    assert (done, res) == (d_o, r_o)
    for first, owned in parts:
        np.testing.assert_array_equal(owned, ref[..., first:first + owned.shape[-1]])
