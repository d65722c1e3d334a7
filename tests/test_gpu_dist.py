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
    n1 = comm.jacobi(U1, W1, 7)
    n2 = ftn.jacobi(U2, W2, 7)
    assert n1 == n2
    assert torch.equal((W1 if n1 else U1).tensor, (W2 if n2 else U2).tensor)


@pytest.mark.parametrize("p", [2, 3, 4, 8])
@pytest.mark.parametrize("shape", [(300, 203), (140, 33, 45)])
def test_jacobi_decomposition_independence(ftn, p, shape):
    from paper_2409_18824_b200 import dist as D
    sweeps = 6
    u0 = synth.jacobi_init(shape)
    nlast = shape[-1]
    U, W = ftn.FArray.from_numpy(u0), ftn.FArray.from_numpy(u0)
    new = ftn.jacobi(U, W, sweeps)
    ref = (W if new else U).to_numpy()
    slabs = []
    for r in range(p):
        g0, nl = D.jacobi_slab(nlast, p, r)
        part = np.asfortranarray(u0[..., g0:g0 + nl])
        slabs.append((g0, nl, [ftn.FArray.from_numpy(part), ftn.FArray.from_numpy(part)]))
    cur = 0
    for _ in range(sweeps):
        # halo exchange of the current source arrays (ftn_jacobi_dist's protocol)
        for r in range(p):
            g0, nl, arr = slabs[r]
            src = arr[cur].tensor
            if r > 0:
                src[..., 0].copy_(slabs[r - 1][2][cur].tensor[..., slabs[r - 1][1] - 2])
            if r < p - 1:
                src[..., nl - 1].copy_(slabs[r + 1][2][cur].tensor[..., 1])
        for r in range(p):
            arr = slabs[r][2]
            ftn.jacobi(arr[cur], arr[1 - cur], 1)
        cur = 1 - cur
    for g0, nl, arr in slabs:
        got = arr[cur].to_numpy()[..., 1:nl - 1]
        np.testing.assert_array_equal(got, ref[..., g0 + 1:g0 + nl - 1])


@pytest.mark.parametrize("p", [2, 4, 8])
def test_sum_decomposition_independence(ftn, p):
    n = 8 * 65536 * 4
    x = ftn.FArray.empty((n,))
    ftn.gen_fill(x, synth.SEED, 7, ftn.GEN_U11)
    whole = ftn.sum(x).item()
    per = n // p
    parts = [ftn.sum(x.section((r * per + 1, (r + 1) * per))).item() for r in range(p)]
    assert oracle.tree_combine(parts, oracle.SUM) == whole
