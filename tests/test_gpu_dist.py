"""GPU tests of the multi-GPU layer that fit on one GPU:
* the NCCL entry points at nranks = 1 equal their single-GPU counterparts bit for bit;
* decomposition independence: p slabs with halo planes, the halo exchange emulated with
  device copies between the slabs and the local sweeps run by the same kernels, give the
  undivided result bit for bit; chunk-aligned slab partials combined by the fixed tree give
  the undivided SUM bit for bit (p = 2, 4, 8)."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ftn():
    from paper_2409_18824_b200 import ftn
    return ftn


@pytest.fixture(scope="module")
def comm(ftn):
    c = ftn.Comm(1, 0, ftn.Comm.unique_id(), 0)
    yield c
    c.destroy()


def test_nccl_single_rank_entry_points(ftn, comm):
    x = ftn.FArray.empty((300, 200, 7))
    ftn.gen_fill(x, synth.SEED, 1, ftn.GEN_U11)
    assert comm.sum(x).item() == ftn.sum(x).item()
    assert comm.maxval(x).item() == ftn.maxval(x).item()
    assert comm.minval(x).item() == ftn.minval(x).item()
    v = ftn.FArray.empty((100003,))
    w = ftn.FArray.empty((100003,))
    ftn.gen_fill(v, synth.SEED, 2, ftn.GEN_U11)
    ftn.gen_fill(w, synth.SEED, 3, ftn.GEN_U11)
    assert comm.dot_product(v, w).item() == ftn.dot_product(v, w).item()
    a, b = ftn.FArray.empty((200, 150)), ftn.FArray.empty((150, 90))
    ftn.gen_fill(a, synth.SEED, 4, ftn.GEN_U11)
    ftn.gen_fill(b, synth.SEED, 5, ftn.GEN_U11)
    c1, c2 = ftn.FArray.empty((200, 90)), ftn.FArray.empty((200, 90))
    comm.matmul(c1, a, b)
    ftn.matmul(c2, a, b)
    assert torch.equal(c1.tensor, c2.tensor)
    comm.bcast(a, 0)
    u0 = synth.jacobi_init((77, 50))
    U1, W1 = ftn.FArray.from_numpy(u0), ftn.FArray.from_numpy(u0)
    U2, W2 = ftn.FArray.from_numpy(u0), ftn.FArray.from_numpy(u0)
    n1 = comm.jacobi(U1, W1, 7, halo=1)
    n2 = ftn.jacobi(U2, W2, 7)
    assert n1 == n2
    assert torch.equal((W1 if n1 else U1).tensor, (W2 if n2 else U2).tensor)


def _slabs(u0, p, halo, rng_fill=True):
    """Local arrays of p slabs with `halo` planes per side (garbage outside the global array)."""
    from paper_2409_18824_b200 import dist as D
    nlast = u0.shape[-1]
    out = []
    for r in range(p):
        s = D.slab(nlast - 2, p, r)                 # owned global planes [s.lo+1, s.hi+1)
        g0 = s.lo + 1 - halo                        # global plane of local plane 0
        nl = s.owned + 2 * halo
        part = np.full(u0.shape[:-1] + (nl,), 7.0e300, order="F")   # garbage outside the array
        for k in range(nl):
            g = g0 + k
            if 0 <= g < nlast:
                part[..., k] = u0[..., g]
        out.append((g0, nl, s.owned))
    return out


@pytest.mark.parametrize("p", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("shape,halo", [((300, 203), 1), ((300, 203), 3), ((140, 33, 45), 1), ((130, 301), 4),
                                        ((260, 407), 5), ((200, 500), 6),
                                        ((129, 201), 2), ((70, 40, 61), 2), ((64, 33, 50), 3), ((65, 33, 50), 2),
                                        ((70, 40, 10), 1), ((90, 10), 1)])   # 1-plane slabs at p = 8
def test_jacobi_decomposition_independence(ftn, p, shape, halo):
    """p slabs with `halo` halo planes; k owned planes exchanged per step (device copies standing
    in for ncclSend/Recv), ftn_jacobi_slab advancing k sweeps; == the undivided ftn_jacobi."""
    sweeps = 10
    u0 = synth.jacobi_init(shape)
    U, W = ftn.FArray.from_numpy(u0), ftn.FArray.from_numpy(u0)
    new = ftn.jacobi(U, W, sweeps)
    ref = (W if new else U).to_numpy()
    meta = _slabs(u0, p, halo)
    arrs = []
    for (g0, nl, owned) in meta:
        part = np.full(u0.shape[:-1] + (nl,), 7.0e300, order="F")
        for k in range(nl):
            if 0 <= g0 + k < shape[-1]:
                part[..., k] = u0[..., g0 + k]
        arrs.append([ftn.FArray.from_numpy(part), ftn.FArray.from_numpy(part)])
    # TMA-able slabs: every stride beyond dim 1 a multiple of 16 B (the local slabs share them)
    tma_able = all((int(np.prod(shape[:d])) * 8) % 16 == 0 for d in range(1, len(shape)))
    fuse = ftn.jacobi_fusion() if len(shape) == 2 else min(2, ftn.jacobi_fusion())
    T = min(fuse, halo) if tma_able else 1
    steps = ftn.jacobi_plan(sweeps, T)                 # ftn_jacobi_dist's launch plan
    cur = 0
    for k in steps:
        for r in range(p):
            g0, nl, owned = meta[r]
            src = arrs[r][cur].tensor
            if r > 0:
                lnl = meta[r - 1][1]
                src[..., halo - k:halo].copy_(arrs[r - 1][cur].tensor[..., lnl - halo - k:lnl - halo])
            if r < p - 1:
                src[..., nl - halo:nl - halo + k].copy_(arrs[r + 1][cur].tensor[..., halo:halo + k])
        for r in range(p):
            ftn.jacobi_slab(arrs[r][cur], arrs[r][1 - cur], k, halo, r == 0, r == p - 1)
        cur = 1 - cur
    assert (cur == 1) == new                       # same result parity as the undivided run
    for (g0, nl, owned), a in zip(meta, arrs):
        got = a[cur].to_numpy()[..., halo:halo + owned]
        np.testing.assert_array_equal(got, ref[..., g0 + halo:g0 + halo + owned])


def test_jacobi_dist_single_rank_deep_halo(ftn, comm):
    """ftn_jacobi_dist at nranks = 1 with halo 3: the global boundary sits at local planes 2 and
    n_last-3, the planes outside it are garbage that must never be consumed."""
    u0 = synth.jacobi_init((250, 120))
    halo = 3
    part = np.full((250, 120 + 2 * (halo - 1)), 7.0e300, order="F")
    part[:, halo - 1:halo - 1 + 120] = u0
    U, W = ftn.FArray.from_numpy(part), ftn.FArray.from_numpy(part)
    n1 = comm.jacobi(U, W, 11, halo=halo)
    R, S = ftn.FArray.from_numpy(u0), ftn.FArray.from_numpy(u0)
    n2 = ftn.jacobi(R, S, 11)
    assert n1 == n2
    got = (W if n1 else U).to_numpy()[:, halo - 1:halo - 1 + 120]
    np.testing.assert_array_equal(got, (S if n2 else R).to_numpy())


@pytest.mark.parametrize("halo,sweeps", [(2, 10), (2, 7), (3, 9)])
def test_jacobi_dist_single_rank_3d_two_sweeps(ftn, comm, halo, sweeps):
    """ftn_jacobi_dist at nranks = 1 on a 3-D slab with 2-3 halo planes: two fused sweeps per
    exchange (jacobi3d_tb2 on a plane range with the global boundary planes held fixed); the
    planes outside the global array are garbage that must never be consumed."""
    u0 = synth.jacobi_init((70, 45, 40))
    part = np.full((70, 45, 40 + 2 * (halo - 1)), 7.0e300, order="F")
    part[:, :, halo - 1:halo - 1 + 40] = u0
    U, W = ftn.FArray.from_numpy(part), ftn.FArray.from_numpy(part)
    n1 = comm.jacobi(U, W, sweeps, halo=halo)
    R, S = ftn.FArray.from_numpy(u0), ftn.FArray.from_numpy(u0)
    n2 = ftn.jacobi(R, S, sweeps)
    assert n1 == n2
    got = (W if n1 else U).to_numpy()[:, :, halo - 1:halo - 1 + 40]
    np.testing.assert_array_equal(got, (S if n2 else R).to_numpy())


@pytest.mark.parametrize("shape,halo,sweeps", [((300, 200), 5, 23), ((300, 200), 3, 10), ((257, 40), 5, 12),
                                              ((70, 45, 60), 2, 9), ((70, 45, 60), 1, 5), ((100, 30, 12), 2, 6)])
def test_jacobi_dist_overlap_split(ftn, comm, shape, halo, sweeps):
    """ftn_comm_set_overlap(2) at nranks = 1: every launch is split into the interior part on
    the communicator's side stream and the two halo-adjacent parts on the caller's stream
    (the N > 1 overlap schedule); bit-identical to the unsplit run and to ftn_jacobi."""
    u0 = synth.jacobi_init(shape, array_id=sum(shape))
    ext = shape[:-1] + (shape[-1] + 2 * (halo - 1),)
    part = np.full(ext, 7.0e300, order="F")
    part[..., halo - 1:halo - 1 + shape[-1]] = u0
    R, S = ftn.FArray.from_numpy(u0), ftn.FArray.from_numpy(u0)
    n2 = ftn.jacobi(R, S, sweeps)
    ref = (S if n2 else R).to_numpy()
    try:
        for mode in (2, 0):
            comm.set_overlap(mode)
            U, W = ftn.FArray.from_numpy(part), ftn.FArray.from_numpy(part)
            n1 = comm.jacobi(U, W, sweeps, halo=halo)
            torch.cuda.synchronize()
            assert n1 == n2
            np.testing.assert_array_equal((W if n1 else U).to_numpy()[..., halo - 1:halo - 1 + shape[-1]], ref)
    finally:
        comm.set_overlap(1)


@pytest.mark.parametrize("p", [2, 4, 8])
def test_sum_decomposition_independence(ftn, p):
    n = 8 * 65536 * 4
    x = ftn.FArray.empty((n,))
    ftn.gen_fill(x, synth.SEED, 7, ftn.GEN_U11)
    whole = ftn.sum(x).item()
    per = n // p
    parts = [ftn.sum(x.section((r * per + 1, (r + 1) * per))).item() for r in range(p)]
    assert oracle.tree_combine(parts, oracle.SUM) == whole
