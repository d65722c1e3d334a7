"""The multi-GPU code path at p > 1 on one GPU: p virtual ranks
(ftn_comm_init_virtual, one host thread per rank, each rank its own stream) run the
library's OWN distributed loops -- ftn_jacobi_dist (launch plan, deep halos, the buffer
offsets of the exchange, the interior / halo-adjacent overlap on the side stream),
ftn_jacobi_solve_dist, ftn_{sum,maxval,minval,dot_product}_global (order-R rank partials,
all-gather, fixed tree), ftn_bcast and ftn_matmul_colsharded -- with every message a device
copy ordered by CUDA events.  Results are compared with the ORACLE on the undivided array:
bit-exact for the Jacobi and MAX/MIN, bit-exact vs order R for chunk-aligned SUM/DOT and
within the R#8 bound otherwise, within the MATMUL bound for the column-sharded product."""
import threading

import numpy as np
import pytest
import torch

import oracle
import synth
from oracle import FArray as OA

pytestmark = pytest.mark.gpu
C2, C3 = 0.25, 1.0 / 6.0
GARBAGE = 7.0e300


@pytest.fixture(scope="module")
def ftn():
    from paper_2409_18824_b200 import ftn
    return ftn


def run_ranks(p, fn):
    """fn(r) in one thread per rank (the ctypes calls release the GIL); re-raise the first
    exception."""
    errs = [None] * p
    torch.cuda.synchronize()   # inputs built on the default stream are complete

    def body(r):
        try:
            fn(r)
        except BaseException as e:  # noqa: BLE001
            errs[r] = e

    ts = [threading.Thread(target=body, args=(r,)) for r in range(p)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(600)
    for e in errs:
        if e is not None:
            raise e


def slab_arrays(ftn, u0, p, halo, pad=0):
    """Per rank: (first global plane of the local array, local extent, owned planes, FArray
    pair); planes outside the global array hold garbage.  pad > 0: each local array is the
    section u(1:n1, ...) of a parent with leading dimension n1 + pad."""
    from paper_2409_18824_b200 import dist as D
    nlast = u0.shape[-1]
    out = []
    for r in range(p):
        g0, nl = D.jacobi_slab(nlast, p, r, halo)
        owned = nl - 2 * halo
        part = np.full(u0.shape[:-1] + (nl,), GARBAGE, order="F")
        for k in range(nl):
            if 0 <= g0 + k < nlast:
                part[..., k] = u0[..., g0 + k]
        pair = []
        for _ in range(2):
            if pad:
                big = np.full((u0.shape[0] + pad,) + part.shape[1:], -3.0, order="F")
                big[:u0.shape[0]] = part
                B = ftn.FArray.from_numpy(big)
                pair.append((B, B.section((1, u0.shape[0]), *[(1, e) for e in part.shape[1:]])))
            else:
                A = ftn.FArray.from_numpy(part)
                pair.append((A, A))
        out.append((g0, nl, owned, pair))
    return out


def oracle_jacobi(u0, sweeps, coeff):
    a, b = u0.copy(order="F"), u0.copy(order="F")
    new = oracle.jacobi(OA(a), OA(b), sweeps, coeff)
    return new, (b if new else a)


@pytest.mark.parametrize("p", [2, 3, 4, 8])
@pytest.mark.parametrize("shape,halo,sweeps", [
    ((300, 203), 1, 7), ((300, 203), 3, 10), ((130, 301), 4, 13), ((260, 407), 5, 12), ((200, 500), 6, 23),
    ((200, 500), 8, 17), ((129, 201), 2, 9), ((90, 10), 1, 6),                                  # 2-D
    ((140, 33, 45), 1, 5), ((70, 40, 61), 2, 9), ((64, 33, 50), 3, 8), ((65, 33, 50), 2, 7),
    ((70, 40, 10), 1, 4)])                                                                     # 3-D
@pytest.mark.parametrize("overlap", [0, 2])
def test_jacobi_dist_virtual_vs_oracle(ftn, p, shape, halo, sweeps, overlap):
    """ftn_jacobi_dist at p virtual ranks == the oracle's DO nest on the undivided array, bit for
    bit, on every owned plane; both overlap schedules; the planes beyond the global array stay
    garbage that must never be consumed."""
    coeff = C2 if len(shape) == 2 else C3
    if shape[-1] - 2 < p:
        pytest.skip("fewer interior planes than ranks")
    u0 = synth.jacobi_init(shape, array_id=sum(shape) + p)
    new_o, ref = oracle_jacobi(u0, sweeps, coeff)
    slabs = slab_arrays(ftn, u0, p, halo)
    comms = ftn.Comm.virtual(p)
    streams = [torch.cuda.Stream() for _ in range(p)]
    res = [None] * p
    try:
        for c in comms:
            c.set_overlap(overlap)

        def rank(r):
            (_, U), (_, W) = slabs[r][3]
            res[r] = comms[r].jacobi(U, W, sweeps, coeff, halo=halo, stream=streams[r])
            streams[r].synchronize()
        run_ranks(p, rank)
    finally:
        for c in comms:
            c.destroy()
    assert all(x == new_o for x in res)
    for (g0, nl, owned, pair) in slabs:
        got = pair[1 if new_o else 0][1].to_numpy()
        np.testing.assert_array_equal(got[..., halo:halo + owned], ref[..., g0 + halo:g0 + halo + owned])
        if g0 < 0:   # planes beyond the global boundary are never written
            assert np.all(got[..., :-g0] == GARBAGE)


@pytest.mark.parametrize("p,halo,sweeps", [(2, 2, 9), (4, 5, 12), (3, 3, 7)])
def test_jacobi_dist_padded_leading_dimension(ftn, p, halo, sweeps):
    """2-D slabs that are sections u(1:n1,:) of a parent with a padded leading dimension: the
    planes of a slab are not adjacent, so each halo plane travels as its own message (ADVICE r1:
    one message of k*plane elements would send the padding and write past the section); the
    padding rows of the parents stay untouched."""
    shape = (200, 301)
    u0 = synth.jacobi_init(shape, array_id=p)
    new_o, ref = oracle_jacobi(u0, sweeps, C2)
    slabs = slab_arrays(ftn, u0, p, halo, pad=6)
    comms = ftn.Comm.virtual(p)
    streams = [torch.cuda.Stream() for _ in range(p)]
    res = [None] * p
    try:
        def rank(r):
            (_, U), (_, W) = slabs[r][3]
            res[r] = comms[r].jacobi(U, W, sweeps, C2, halo=halo, stream=streams[r])
            streams[r].synchronize()
        run_ranks(p, rank)
    finally:
        for c in comms:
            c.destroy()
    assert all(x == new_o for x in res)
    for (g0, nl, owned, pair) in slabs:
        parent, sec = pair[1 if new_o else 0]
        np.testing.assert_array_equal(sec.to_numpy()[..., halo:halo + owned], ref[..., g0 + halo:g0 + halo + owned])
        for P, _ in pair:
            assert np.all(P.to_numpy()[shape[0]:] == -3.0)


def _global_case(ftn, p, n_local, mode=synth.U11):
    x = [ftn.FArray.empty((n_local,)) for _ in range(p)]
    y = [ftn.FArray.empty((n_local,)) for _ in range(p)]
    for r in range(p):
        ftn.gen_fill(x[r], synth.SEED, 100 + r, mode)
        ftn.gen_fill(y[r], synth.SEED, 200 + r, mode)
    torch.cuda.synchronize()
    xs = np.concatenate([a.to_numpy() for a in x])
    ys = np.concatenate([a.to_numpy() for a in y])
    return x, y, xs, ys


def _run_globals(ftn, p, x, y):
    comms = ftn.Comm.virtual(p)
    streams = [torch.cuda.Stream() for _ in range(p)]
    out = [None] * p
    try:
        def rank(r):
            with torch.cuda.stream(streams[r]):
                c = comms[r]
                vals = (c.sum(x[r], stream=streams[r]), c.maxval(x[r], stream=streams[r]),
                        c.minval(x[r], stream=streams[r]), c.dot_product(x[r], y[r], stream=streams[r]))
                streams[r].synchronize()
                out[r] = [v.item() for v in vals]
        run_ranks(p, rank)
    finally:
        for c in comms:
            c.destroy()
    return out


@pytest.mark.parametrize("p", [2, 4, 8])
def test_global_reductions_chunk_aligned(ftn, p):
    """Chunk-aligned slabs (each rank an equal power-of-two number of R chunks): the global SUM
    and DOT equal the oracle's order-R reduction of the undivided array bit for bit; MAXVAL /
    MINVAL exact; every rank holds the same values."""
    n_local = 65536 * 8 // p * 2
    x, y, xs, ys = _global_case(ftn, p, n_local)
    out = _run_globals(ftn, p, x, y)
    X, Y = OA(np.asfortranarray(xs)), OA(np.asfortranarray(ys))
    ref = [oracle.reduce_orderR(X, oracle.SUM), oracle.maxval(X), oracle.minval(X), oracle.dot_orderR(X, Y)]
    for r in range(p):
        assert out[r] == ref, (r, out[r], ref)
    exact = oracle.sum_exact(X)
    assert abs(out[0][0] - exact) <= 4 * xs.size * 2.0 ** -53 * oracle.sum_abs(X)


@pytest.mark.parametrize("p", [3, 5])
def test_global_reductions_unaligned(ftn, p):
    """Slabs that are not chunk aligned: SUM / DOT within the R#8 bound of the exact value, MAX
    / MIN exact, all ranks identical."""
    n_local = 100003
    x, y, xs, ys = _global_case(ftn, p, n_local)
    out = _run_globals(ftn, p, x, y)
    X, Y = OA(np.asfortranarray(xs)), OA(np.asfortranarray(ys))
    n = xs.size
    assert abs(out[0][0] - oracle.sum_exact(X)) <= 4 * n * 2.0 ** -53 * oracle.sum_abs(X)
    dex, dabs = oracle.dot_exact(X, Y)
    assert abs(out[0][3] - dex) <= 4 * n * 2.0 ** -53 * dabs
    assert out[0][1] == oracle.maxval(X) and out[0][2] == oracle.minval(X)
    assert all(o == out[0] for o in out)


@pytest.mark.parametrize("p", [2, 4])
def test_bcast_and_matmul_colsharded(ftn, p):
    """ftn_bcast of A from the root (the other ranks start with garbage) and the column-sharded
    MATMUL c(:, J_r) = MATMUL(a, b(:, J_r)): within the bound of the oracle's product."""
    m, k, n = 160, 96, 64 * p
    a_h = synth.farray((m, k), array_id=11, mode=synth.U11)
    b_h = synth.farray((k, n), array_id=12, mode=synth.U11)
    A = [ftn.FArray.from_numpy(a_h if r == 0 else np.full((m, k), GARBAGE, order="F")) for r in range(p)]
    nb = n // p
    B = [ftn.FArray.from_numpy(np.asfortranarray(b_h[:, r * nb:(r + 1) * nb])) for r in range(p)]
    C = [ftn.FArray.empty((m, nb)) for _ in range(p)]
    comms = ftn.Comm.virtual(p)
    streams = [torch.cuda.Stream() for _ in range(p)]
    try:
        def rank(r):
            comms[r].bcast(A[r], 0, stream=streams[r])
            comms[r].matmul(C[r], A[r], B[r], stream=streams[r])
            streams[r].synchronize()
        run_ranks(p, rank)
    finally:
        for c in comms:
            c.destroy()
    co, ab = np.zeros((m, n), order="F"), np.zeros((m, n), order="F")
    oracle.matmul(OA(co), OA(a_h), OA(b_h), OA(ab))
    for r in range(p):
        np.testing.assert_array_equal(A[r].to_numpy(), a_h)
        got = C[r].to_numpy()
        assert np.all(np.abs(got - co[:, r * nb:(r + 1) * nb]) <= 4 * k * 2.0 ** -53 * ab[:, r * nb:(r + 1) * nb])


def test_virtual_rank_errors(ftn):
    """A message size mismatch between sender and receiver is an error, not a hang or a
    partial copy (the two ranks' slabs have different plane sizes)."""
    comms = ftn.Comm.virtual(2)
    u = [synth.jacobi_init((60, 30), array_id=1), synth.jacobi_init((62, 30), array_id=2)]
    arrs = [(ftn.FArray.from_numpy(v), ftn.FArray.from_numpy(v)) for v in u]
    errs = [None, None]
    try:
        def rank(r):
            try:
                comms[r].jacobi(arrs[r][0], arrs[r][1], 2, C2, halo=1)
            except ftn.FtnError as e:
                errs[r] = e
        run_ranks(2, rank)
    finally:
        for c in comms:
            c.destroy()
    assert all(e is not None and e.name == "FTN_ERR_NCCL" for e in errs)


@pytest.mark.parametrize("p", [2, 3, 4])
@pytest.mark.parametrize("shape,halo,check,tol", [
    ((300, 203), 5, 10, 1e-3), ((130, 301), 3, 7, -1.0), ((200, 150), 1, 4, 2e-3), ((200, 160), 8, 9, 1e-4),
    ((70, 40, 61), 2, 5, 1e-3), ((64, 33, 50), 1, 3, -1.0)])
@pytest.mark.parametrize("overlap", [0, 2])
def test_jacobi_solve_dist_virtual_vs_oracle(ftn, p, shape, halo, check, tol, overlap):
    """ftn_jacobi_solve_dist at p virtual ranks == the oracle's solve on the undivided array:
    sweeps done, the global residual (max over the ranks' owned interiors; fused into the last
    launch of each block for 2-D slabs) and every owned plane bit for bit, the same on every
    rank."""
    coeff = C2 if len(shape) == 2 else C3
    if shape[-1] - 2 < p:
        pytest.skip("fewer interior planes than ranks")
    u0 = synth.jacobi_init(shape, array_id=7 * p + len(shape))
    a, b = u0.copy(order="F"), u0.copy(order="F")
    d_o, r_o, n_o = oracle.jacobi_solve(OA(a), OA(b), 40, check, tol, coeff)
    ref = b if n_o else a
    slabs = slab_arrays(ftn, u0, p, halo)
    comms = ftn.Comm.virtual(p)
    streams = [torch.cuda.Stream() for _ in range(p)]
    out = [None] * p
    try:
        for c in comms:
            c.set_overlap(overlap)

        def rank(r):
            (_, U), (_, W) = slabs[r][3]
            out[r] = comms[r].jacobi_solve(U, W, 40, check, tol, coeff, halo=halo, stream=streams[r])
            streams[r].synchronize()
        run_ranks(p, rank)
    finally:
        for c in comms:
            c.destroy()
    assert all(o == (d_o, r_o, n_o) for o in out), (out, (d_o, r_o, n_o))
    for (g0, nl, owned, pair) in slabs:
        got = pair[1 if n_o else 0][1].to_numpy()
        np.testing.assert_array_equal(got[..., halo:halo + owned], ref[..., g0 + halo:g0 + halo + owned])
