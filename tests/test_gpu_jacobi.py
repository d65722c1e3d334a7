"""GPU parity: Jacobi sweeps (TMA 2-D / 3-D kernels and the generic strided kernel) vs the
oracle, bit-exact (R#16, R#23)."""
import os

import numpy as np
import pytest
import torch

import oracle
import synth
from oracle import FArray as OA
DEFAULT_FUSION = 0   # ftn_jacobi_set_fusion(0): back to the default (size-dependent)

pytestmark = pytest.mark.gpu
C2, C3 = 0.25, 1.0 / 6.0


@pytest.fixture(scope="module")
def ftn():
    from paper_2409_18824_b200 import ftn
    return ftn


@pytest.fixture
def streaming(ftn):
    """The streaming (temporally blocked) kernels (the only Jacobi path since round 2)."""
    yield


def _run_both(ftn, u0, sweeps, coeff, lbs=None):
    U, W = ftn.FArray.from_numpy(u0, lbs), ftn.FArray.from_numpy(u0, lbs)
    in_new = ftn.jacobi(U, W, sweeps, coeff)
    got = (W if in_new else U).to_numpy()
    uo, wo = u0.copy(order="F"), u0.copy(order="F")
    in_new_o = oracle.jacobi(OA(uo, lbs), OA(wo, lbs), sweeps, coeff)
    assert in_new == in_new_o
    return got, (wo if in_new_o else uo)


@pytest.mark.parametrize("shape", [(3, 3), (3, 40), (40, 3), (4, 5), (129, 31), (130, 62), (131, 100),
                                   (257, 65), (300, 301), (1000, 77)])
@pytest.mark.parametrize("sweeps", [1, 2, 5])
def test_2d_vs_oracle(ftn, shape, sweeps):
    u0 = synth.jacobi_init(shape, array_id=sum(shape))
    got, ref = _run_both(ftn, u0, sweeps, C2, [0, -7])
    np.testing.assert_array_equal(got, ref)


@pytest.mark.parametrize("shape", [(3, 3, 3), (5, 4, 3), (40, 3, 9), (3, 40, 9), (130, 18, 7), (131, 19, 11),
                                   (64, 64, 64), (257, 35, 20), (100, 33, 41)])
@pytest.mark.parametrize("sweeps", [1, 3])
def test_3d_vs_oracle(ftn, shape, sweeps):
    u0 = synth.jacobi_init(shape, array_id=sum(shape))
    got, ref = _run_both(ftn, u0, sweeps, C3, [1, 1, 1])
    np.testing.assert_array_equal(got, ref)


def test_every_extent_2d(ftn):
    """Each extent in [3, 40] in each dimension (strip / chunk / halo remainders)."""
    for n in range(3, 41):
        for shape in ((n, 37), (37, n)):
            u0 = synth.jacobi_init(shape, array_id=n)
            got, ref = _run_both(ftn, u0, 2, C2)
            np.testing.assert_array_equal(got, ref, err_msg=str(shape))


def test_harmonic_fixed_points(ftn):
    i, j = np.meshgrid(np.arange(200.0), np.arange(150.0), indexing="ij")
    for f in (i + 2 * j, i * j, i * i - j * j):
        u0 = np.asfortranarray(f)
        got, _ = _run_both(ftn, u0, 4, C2)
        np.testing.assert_array_equal(got, u0)
    i, j, k = np.meshgrid(np.arange(140.0), np.arange(20.0), np.arange(12.0), indexing="ij")
    u3 = np.asfortranarray(i + 2 * j + 3 * k)
    got, _ = _run_both(ftn, u3, 3, C3)
    np.testing.assert_array_equal(got, u3)


def test_strided_generic_path(ftn):
    """Sections (dim-1 stride 16 B, reversed dim 2) take the generic kernel; same bits."""
    big = synth.jacobi_init((61, 50))
    Bu, Bw = ftn.FArray.from_numpy(big), ftn.FArray.from_numpy(big)
    su, sw = Bu.section((1, 61, 2), (50, 1, -1)), Bw.section((1, 61, 2), (50, 1, -1))
    in_new = ftn.jacobi(su, sw, 3)
    got = (sw if in_new else su).to_numpy()
    ou, ow = big.copy(order="F"), big.copy(order="F")
    so, sow = OA(ou).section((1, 61, 2), (50, 1, -1)), OA(ow).section((1, 61, 2), (50, 1, -1))
    oracle.jacobi(so, sow, 3, C2)
    np.testing.assert_array_equal(got, sow.to_numpy() if in_new else so.to_numpy())
    b3 = synth.jacobi_init((20, 9, 8))
    U3, W3 = ftn.FArray.from_numpy(b3), ftn.FArray.from_numpy(b3)
    s3u, s3w = U3.section((20, 1, -1), (1, 9), (1, 8)), W3.section((20, 1, -1), (1, 9), (1, 8))
    ftn.jacobi(s3u, s3w, 1)
    o3u, o3w = b3.copy(order="F"), b3.copy(order="F")
    oracle.jacobi(OA(o3u).section((20, 1, -1), (1, 9, 1), (1, 8, 1)), OA(o3w).section((20, 1, -1), (1, 9, 1), (1, 8, 1)),
                  1, C3)
    np.testing.assert_array_equal(s3w.to_numpy(), OA(o3w).section((20, 1, -1), (1, 9, 1), (1, 8, 1)).to_numpy())


def test_zero_sweeps_and_errors(ftn):
    u0 = synth.jacobi_init((10, 10))
    U, W = ftn.FArray.from_numpy(u0), ftn.FArray.from_numpy(u0)
    assert ftn.jacobi(U, W, 0) is False
    np.testing.assert_array_equal(U.to_numpy(), u0)
    with pytest.raises(ftn.FtnError):
        ftn.jacobi(U, ftn.FArray.empty((10, 11)), 1)
    with pytest.raises(ftn.FtnError):
        ftn.jacobi(U, U, 1)


@pytest.mark.slow
def test_c2_full_size_sampled(ftn):
    """C2 at full size (8192^2, 100 sweeps, the bench's launch configuration): every sampled
    output point is recomputed by the oracle on its dependence cone (a 203x203 window, which
    the 100 sweeps cannot see past), bit-exact; plus a full-size harmonic field."""
    n, sweeps = 8192, 100
    U, W = ftn.FArray.empty((n, n)), ftn.FArray.empty((n, n))
    ftn.gen_fill(U, synth.SEED, 0, ftn.GEN_U01)
    for face in ((1, n), (1, 1)), ((1, n), (n, n)), ((1, 1), (1, n)), ((n, n), (1, n)):
        ftn.fill(U.section(*face), 0.0)
    ftn.fill(U.section((1, n), (1, 1)), 1.0)
    ftn.assign(W, U)
    u_host = U.to_numpy()
    in_new = ftn.jacobi(U, W, sweeps)
    res = (W if in_new else U)
    rng = np.random.default_rng(0)
    pts = [(1, 1), (n - 2, n - 2), (0, 5), (4000, 1), (1, 4000)] + [tuple(int(v) for v in rng.integers(0, n, 2))
                                                                      for _ in range(10)]
    R = sweeps + 1
    for (i, j) in pts:
        i0, i1 = max(0, i - R), min(n, i + R + 1)
        j0, j1 = max(0, j - R), min(n, j + R + 1)
        win = np.asfortranarray(u_host[i0:i1, j0:j1])
        a, b = win.copy(order="F"), win.copy(order="F")
        new = oracle.jacobi(OA(a), OA(b), sweeps, C2)
        ref = (b if new else a)[i - i0, j - j0]
        got = res.section((i + 1, i + 1), (j + 1, j + 1)).to_numpy()[0, 0]
        assert got == ref, (i, j)


@pytest.mark.parametrize("T", [1, 2, 3, 4, 5, 6, 7, 8])
@pytest.mark.parametrize("shape", [(3, 3), (5, 40), (40, 5), (129, 31), (200, 301), (257, 77), (1000, 130)])
@pytest.mark.parametrize("sweeps", [1, 2, 3, 4, 7, 8, 9])
def test_2d_temporal_blocking(ftn, streaming, T, shape, sweeps):
    """Fused launches of T sweeps are bit-identical to the oracle's
    sweep-by-sweep DO nest, and the result lands where the sweep parity says."""
    ftn.jacobi_set_fusion(T)
    try:
        u0 = synth.jacobi_init(shape, array_id=sum(shape) + sweeps)
        got, ref = _run_both(ftn, u0, sweeps, C2, [1, 0])
        np.testing.assert_array_equal(got, ref)
    finally:
        ftn.jacobi_set_fusion(DEFAULT_FUSION)


def test_2d_temporal_blocking_long_strip(ftn):
    """Many units per CTA, uneven segments, 60 sweeps."""
    for T in (2, 3, 4, 5, 6, 7, 8):
        ftn.jacobi_set_fusion(T)
        u0 = synth.jacobi_init((3000, 2000), array_id=T)
        got, ref = _run_both(ftn, u0, 12, C2)
        np.testing.assert_array_equal(got, ref)
    ftn.jacobi_set_fusion(DEFAULT_FUSION)


@pytest.mark.parametrize("T", [1, 2, 3, 4])
@pytest.mark.parametrize("shape", [(3, 3, 3), (4, 5, 6), (61, 29, 5), (62, 30, 6), (63, 31, 4), (121, 57, 9),
                                   (130, 18, 7), (64, 64, 64), (200, 90, 40), (17, 100, 33), (57, 25, 8),
                                   (58, 27, 12), (113, 49, 11), (114, 52, 3)])
@pytest.mark.parametrize("sweeps", [1, 2, 3, 4, 5])
def test_3d_temporal_blocking(ftn, T, shape, sweeps):
    """Rank-3 launches of T fused sweeps (jacobi3d_wr<T>) are bit-identical to
    the oracle's DO nest; boxes of 64 x 32 with (64 - 2H) x (32 - 2T) outputs (56 x 26 at
    T = 3, 60 x 28 at T = 2), so these shapes cover one tile, exact multiples and ragged tails
    in i and j.  ftn_jacobi caps rank-3 launches at FTN_J3_T (3), so T = 4 here runs T = 3;
    wr<4> is covered by test_3d_slab_step_every_fusion."""
    ftn.jacobi_set_fusion(T)
    try:
        u0 = synth.jacobi_init(shape, array_id=sum(shape) + sweeps)
        got, ref = _run_both(ftn, u0, sweeps, C3, [0, 2, -1])
        np.testing.assert_array_equal(got, ref)
    finally:
        ftn.jacobi_set_fusion(DEFAULT_FUSION)


@pytest.mark.parametrize("sweeps", [2, 3, 4])
@pytest.mark.parametrize("shape", [(62, 31, 12), (122, 57, 20), (64, 64, 30), (200, 90, 13)])   # TMA-able: even n1
def test_3d_slab_step_every_fusion(ftn, sweeps, shape):
    """ftn_jacobi_slab on one whole-array slab runs exactly `sweeps` fused sweeps per launch
    (jacobi3d_tb2 for 2, jacobi3d_wr<3>, jacobi3d_wr<4> -- ftn_jacobi caps rank-3 launches at
    FTN_J3_T = 3, so this is the path that reaches wr<4>); the owned planes equal the oracle's
    DO nest after `sweeps` sweeps, bit for bit."""
    from paper_2409_18824_b200 import dist as D
    halo = sweeps
    n = shape[-1]
    g0, nl = D.jacobi_slab(n, 1, 0, halo)
    u0 = synth.jacobi_init(shape, array_id=sum(shape) + sweeps)
    part = np.full(shape[:-1] + (nl,), 7.0e300, order="F")
    for q in range(nl):
        if 0 <= g0 + q < n:
            part[..., q] = u0[..., g0 + q]
    U, W = ftn.FArray.from_numpy(part), ftn.FArray.from_numpy(part)
    ftn.jacobi_slab(U, W, sweeps, halo, True, True)
    a, b = u0.copy(order="F"), u0.copy(order="F")
    new = oracle.jacobi(OA(a), OA(b), sweeps, C3)
    ref = b if new else a
    owned = nl - 2 * halo
    got = W.to_numpy()
    np.testing.assert_array_equal(got[..., halo:halo + owned], ref[..., g0 + halo:g0 + halo + owned])


def test_3d_temporal_blocking_many_units(ftn):
    """More units than CTAs (several k segments per tile column), random data, 6 sweeps."""
    u0 = np.asfortranarray(synth.farray((250, 180, 150), array_id=9, mode=synth.U11))
    got, ref = _run_both(ftn, u0, 6, C3)
    np.testing.assert_array_equal(got, ref)
    i, j, k = np.meshgrid(np.arange(130.0), np.arange(60.0), np.arange(50.0), indexing="ij")
    u3 = np.asfortranarray(i - 2 * j + 3 * k)
    got, _ = _run_both(ftn, u3, 4, C3)
    np.testing.assert_array_equal(got, u3)


@pytest.mark.slow
def test_c5_full_size_sampled(ftn):
    """C5 at full size (2048^3, 10 sweeps, the bench's launch configuration): sampled points
    recomputed by the oracle on their dependence cone (a 23^3 window), bit-exact."""
    n, sweeps = 2048, 10
    U, W = ftn.FArray.empty((n, n, n)), ftn.FArray.empty((n, n, n))
    ftn.gen_fill(U, synth.SEED, 0, ftn.GEN_U01)
    ftn.assign(W, U)
    rng = np.random.default_rng(5)
    pts = [(1, 1, 1), (n - 2, n - 2, n - 2), (0, 7, 9), (1000, 1, 1000), (59, 27, 300), (60, 28, 301)] + \
          [tuple(int(v) for v in rng.integers(0, n, 3)) for _ in range(8)]
    R = sweeps + 1
    wins = []
    for p in pts:
        lo = [max(0, c - R) for c in p]
        hi = [min(n, c + R + 1) for c in p]
        sec = U.section(*[(a + 1, b) for a, b in zip(lo, hi)])
        wins.append((p, lo, np.asfortranarray(sec.to_numpy())))
    in_new = ftn.jacobi(U, W, sweeps)
    res = W if in_new else U
    for p, lo, win in wins:
        a, b = win.copy(order="F"), win.copy(order="F")
        new = oracle.jacobi(OA(a), OA(b), sweeps, C3)
        ref = (b if new else a)[tuple(c - l for c, l in zip(p, lo))]
        got = res.section(*[(c + 1, c + 1) for c in p]).to_numpy().ravel()[0]
        assert got == ref, p


@pytest.mark.parametrize("shape,sweeps", [((130, 77), 9), ((300, 301), 4), ((61, 29, 9), 5), ((3, 3), 1), ((40, 50), 0)])
def test_jacobi_host_buffers(ftn, shape, sweeps):
    """ftn_jacobi_host: host in -> device -> sweeps -> host out, same bits as the oracle; the
    result buffer may alias the input buffer."""
    u0 = synth.jacobi_init(shape, array_id=7)
    coeff = C2 if len(shape) == 2 else C3
    host_u = torch.from_numpy(u0.copy(order="F").T.copy()).permute(*range(len(shape) - 1, -1, -1))
    host_u = host_u.pin_memory() if torch.cuda.is_available() else host_u
    host_out = torch.empty(shape[::-1], dtype=torch.float64).pin_memory().permute(*range(len(shape) - 1, -1, -1))
    U, W = ftn.FArray.empty(shape), ftn.FArray.empty(shape)
    new = ftn.jacobi_host(host_u, host_out, U, W, sweeps, coeff)
    torch.cuda.synchronize()
    uo, wo = u0.copy(order="F"), u0.copy(order="F")
    new_o = oracle.jacobi(OA(uo), OA(wo), sweeps, coeff)
    assert new == new_o
    np.testing.assert_array_equal(host_out.numpy(), wo if new_o else uo)
    ftn.jacobi_host(host_u, host_u, U, W, sweeps, coeff)       # in place on the host
    torch.cuda.synchronize()
    np.testing.assert_array_equal(host_u.numpy(), wo if new_o else uo)


@pytest.mark.slow
def test_c5_bench_configuration_100_sweeps(ftn):
    """C5 exactly as bench.py runs it (2048^3, 100 sweeps = 26 launches of jacobi3d_wr: 22 of 4
    and 4 of 3 sweeps): sampled points recomputed by the oracle on their dependence cone
    (203^3 windows)."""
    n, sweeps = 2048, 100
    U, W = ftn.FArray.empty((n, n, n)), ftn.FArray.empty((n, n, n))
    ftn.gen_fill(U, synth.SEED, 7, ftn.GEN_U01)
    ftn.assign(W, U)
    assert ftn.jacobi_plan(sweeps, 4) == [4] * 22 + [3] * 4
    pts = [(1, 1, 1), (n - 2, 1000, 5), (700, 1300, 1900), (150, n - 2, 60), (56, 24, 1024), (57, 25, 2046)]
    R = sweeps + 1
    wins = []
    for p in pts:
        lo = [max(0, c - R) for c in p]
        hi = [min(n, c + R + 1) for c in p]
        wins.append((p, lo, np.asfortranarray(U.section(*[(a + 1, b) for a, b in zip(lo, hi)]).to_numpy())))
    in_new = ftn.jacobi(U, W, sweeps)
    assert not in_new
    for p, lo, win in wins:
        a, b = win.copy(order="F"), win.copy(order="F")
        new = oracle.jacobi(OA(a), OA(b), sweeps, C3)
        ref = (b if new else a)[tuple(c - l for c, l in zip(p, lo))]
        got = U.section(*[(c + 1, c + 1) for c in p]).to_numpy().ravel()[0]
        assert got == ref, p


def test_error_paths_launch_nothing(ftn):
    """Every rejected call returns its status before any launch and leaves the arrays as they
    were (host validation first, never partial output)."""
    u0 = synth.jacobi_init((20, 16))
    U, W = ftn.FArray.from_numpy(u0), ftn.FArray.from_numpy(u0)
    n0 = ftn.launch_count()
    cases = [
        lambda: ftn.jacobi(U, W, -1),                                          # negative sweeps
        lambda: ftn.jacobi(U, U.section((1, 20), (1, 16)), 1),                 # overlapping
        lambda: ftn.jacobi(ftn.FArray.empty((20, 16), dtype=torch.float32),
                           ftn.FArray.empty((20, 16), dtype=torch.float32), 1),  # real(4)
        lambda: ftn.jacobi_slab(U, W, 2, 1, True, True),                       # sweeps > halo
        lambda: ftn.jacobi_slab(U, W, 1, 8, True, True),                       # no owned plane
        lambda: ftn.jacobi_set_fusion(13),
        lambda: ftn.jacobi_set_fusion(-1),
    ]
    for f in cases:
        with pytest.raises(ftn.FtnError):
            f()
    host = torch.zeros((16, 20), dtype=torch.float64).t()
    h10 = torch.zeros((16, 10), dtype=torch.float64).t()
    with pytest.raises(ftn.FtnError):            # device arrays must be packed
        ftn.jacobi_host(h10, h10, U.section((1, 20, 2), (1, 16)), W.section((1, 20, 2), (1, 16)), 1)
    with pytest.raises(ValueError):              # host buffers must have u's shape
        ftn.jacobi_host(torch.zeros((5, 5), dtype=torch.float64), host, U, W, 1)
    assert ftn.launch_count() == n0
    np.testing.assert_array_equal(U.to_numpy(), u0)
    np.testing.assert_array_equal(W.to_numpy(), u0)


def test_random_shapes_fusions_and_sweeps(ftn, streaming):
    """Fuzz: random 2-D / 3-D shapes, lower bounds, sweep counts and fusion settings, all
    bit-identical to the oracle (covers unit / segment / strip remainders the fixed cases miss)."""
    rng = np.random.default_rng(2409)
    try:
        for it in range(40):
            T = int(rng.integers(1, 9))
            ftn.jacobi_set_fusion(T)
            if it % 4 == 3:
                shape = tuple(int(v) for v in rng.integers(3, 90, 3))
                coeff = C3
            else:
                shape = (int(rng.integers(3, 700)), int(rng.integers(3, 300)))
                coeff = C2
            sweeps = int(rng.integers(0, 14))
            lbs = [int(v) for v in rng.integers(-5, 6, len(shape))]
            u0 = synth.jacobi_init(shape, array_id=it)
            got, ref = _run_both(ftn, u0, sweeps, coeff, lbs)
            np.testing.assert_array_equal(got, ref, err_msg=f"shape {shape} sweeps {sweeps} T {T}")
    finally:
        ftn.jacobi_set_fusion(DEFAULT_FUSION)


@pytest.mark.parametrize("case", ["odd_ld_2d", "section_2d", "odd_ld_3d", "section_3d"])
@pytest.mark.parametrize("sweeps", [8, 9, 23])
def test_non_tma_arrays_take_padded_fused_path(ftn, case, sweeps):
    """Arrays the TMA kernels cannot address (odd leading dimension, strided / reversed
    sections) run the fused kernels on padded packed copies for >= 8 sweeps: same bits as the
    oracle on the same (section) arrays, the rest of the parent untouched."""
    if case.endswith("2d"):
        parent_shape, sec = (301, 120), ((1, 301, 2), (120, 1, -1))
        coeff = C2
    else:
        parent_shape, sec = (45, 30, 21), ((45, 1, -1), (1, 30), (1, 21, 2))
        coeff = C3
    if case.startswith("odd_ld"):
        sec = tuple((1, n) for n in parent_shape)
    big = synth.jacobi_init(parent_shape, array_id=sweeps)
    Bu, Bw = ftn.FArray.from_numpy(big), ftn.FArray.from_numpy(big)
    su, sw = Bu.section(*sec), Bw.section(*sec)
    new = ftn.jacobi(su, sw, sweeps, coeff)
    ou, ow = big.copy(order="F"), big.copy(order="F")
    osec = tuple(t if len(t) == 3 else (t[0], t[1], 1) for t in sec)
    onew = oracle.jacobi(OA(ou).section(*osec), OA(ow).section(*osec), sweeps, coeff)
    assert new == onew
    # the result array matches the oracle's everywhere (inside the section: the sweeps;
    # outside: untouched); the other array holds an earlier iterate inside the section and is
    # untouched outside it
    res_parent, ref_parent = (Bw, ow) if new else (Bu, ou)
    np.testing.assert_array_equal(res_parent.to_numpy(), ref_parent)
    other = (Bu if new else Bw).to_numpy()
    inside = np.zeros(parent_shape, bool)
    idx = []
    for t, n in zip(osec, parent_shape):
        lo, hi, st = t
        idx.append(np.arange(lo - 1, hi - 1 + (1 if st > 0 else -1), st))
    inside[np.ix_(*idx)] = True
    np.testing.assert_array_equal(other[~inside], big[~inside])
    res = (sw if new else su).to_numpy()
    ref = (OA(ow) if onew else OA(ou)).section(*osec).to_numpy()
    np.testing.assert_array_equal(res, ref)


def test_subnormal_values_are_not_flushed(ftn):
    """Neither side flushes subnormals (SURVEY §7 hard part 3): a field scaled into the
    subnormal range gives the same bits on the fused GPU kernels and in the oracle."""
    for shape, coeff, sweeps in (((130, 70), C2, 7), ((40, 30, 20), C3, 4)):
        u0 = np.asfortranarray(synth.jacobi_init(shape, array_id=3) * 2.0 ** -1060)
        assert np.count_nonzero((np.abs(u0) < 2.0 ** -1022) & (u0 != 0)) > 0
        got, ref = _run_both(ftn, u0, sweeps, coeff)
        np.testing.assert_array_equal(got, ref)
        assert np.count_nonzero((np.abs(got) < 2.0 ** -1022) & (got != 0)) > 0


def test_fusion_above_the_build_limit_is_capped(ftn):
    """ftn_jacobi_set_fusion accepts 1..12, the default build fuses at most 8 rank-2 sweeps per
    launch: a setting of 10 runs launches of <= 8 (ftn_jacobi_fusion_for reports 8), results
    bit-identical to the oracle."""
    ftn.jacobi_set_fusion(10)
    try:
        U = ftn.FArray.empty((300, 200))
        assert ftn.jacobi_fusion(U) == 8
        u0 = synth.jacobi_init((300, 200), array_id=10)
        got, ref = _run_both(ftn, u0, 23, C2, [1, 1])
        np.testing.assert_array_equal(got, ref)
    finally:
        ftn.jacobi_set_fusion(DEFAULT_FUSION)


def test_3d_banded_cells_dynamic_and_captured(tmp_path):
    """The (tile, band) cell orders of jacobi3d_wr forced on a small grid
    (FTN_W3_RR=16 in a fresh process): dynamic cells from the ticket counter in a plain call,
    the static round-robin deal inside a CUDA-graph capture (replayed twice); both bit-identical
    to the oracle's DO nest."""
    import subprocess
    import sys
    import textwrap
    script = textwrap.dedent("""
        import sys
        import numpy as np
        import torch
        sys.path.insert(0, %r)
        import oracle, synth
        from oracle import FArray as OA
        from paper_2409_18824_b200 import ftn
        C3 = 1.0 / 6.0
        shape, sweeps = (130, 90, 70), 6
        u0 = synth.jacobi_init(shape, array_id=77)
        a, b = u0.copy(order="F"), u0.copy(order="F")
        new = oracle.jacobi(OA(a), OA(b), sweeps, C3)
        ref = b if new else a
        U, W = ftn.FArray.from_numpy(u0), ftn.FArray.from_numpy(u0)
        got_new = ftn.jacobi(U, W, sweeps, C3)
        assert got_new == new
        np.testing.assert_array_equal((W if new else U).to_numpy(), ref)
        U, W, U0 = ftn.FArray.from_numpy(u0), ftn.FArray.from_numpy(u0), ftn.FArray.from_numpy(u0)
        s = torch.cuda.Stream()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            ftn.jacobi(U, W, 1, C3, stream=s)     # warm-up (attributes, tensor maps) outside the capture
            s.synchronize()
            ftn.assign(U, U0, stream=s)
            ftn.assign(W, U0, stream=s)
            s.synchronize()
            with torch.cuda.graph(g, stream=s):
                ftn.jacobi(U, W, sweeps, C3, stream=s)
        for rep in range(2):   # replay twice from the initial state
            ftn.assign(U, U0)
            ftn.assign(W, U0)
            torch.cuda.synchronize()
            g.replay()
            torch.cuda.synchronize()
            np.testing.assert_array_equal((W if new else U).to_numpy(), ref)
        print("ok")
    """) % os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, FTN_W3_RR="16")
    r = subprocess.run([sys.executable, "-c", script], capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-3000:]
