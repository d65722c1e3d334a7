"""GPU parity: TRANSPOSE (bit-exact) and MATMUL on DMMA (within 4 k 2^-53 sum|a||b|, exact on
integer-valued / identity / permutation inputs), R#8, R#14, R#15."""
import numpy as np
import pytest
import torch

import oracle
import synth
from oracle import FArray as OA

pytestmark = pytest.mark.gpu
U = 2.0 ** -53


@pytest.fixture(scope="module")
def ftn():
    from paper_2409_18824_b200 import ftn
    return ftn


@pytest.mark.parametrize("dtype", [np.int32, np.float64])
def test_transpose_shapes(ftn, dtype):
    tt = {np.int32: torch.int32, np.float64: torch.float64}[dtype]
    mode = synth.RAW if dtype == np.int32 else synth.U11
    rng = np.random.default_rng(1)
    shapes = [(1, 1), (1, 70), (70, 1), (63, 65), (64, 64), (129, 7)] + \
             [tuple(int(v) for v in rng.integers(1, 71, size=2)) for _ in range(20)]
    for sh in shapes:
        a = synth.farray(sh, mode=mode, dtype=dtype)
        A = ftn.FArray.from_numpy(a, [0, -3])
        r = ftn.FArray.empty(sh[::-1], dtype=tt)
        ftn.transpose(r, A)
        ro = np.zeros(sh[::-1], dtype=dtype, order="F")
        oracle.transpose(OA(ro), OA(a, [0, -3]))
        np.testing.assert_array_equal(r.to_numpy(), ro, err_msg=str(sh))


def test_transpose_sections_and_involution(ftn):
    a = synth.farray((100, 77), mode=synth.LINEAR)
    A = ftn.FArray.from_numpy(a, [-2, 3])
    s = A.section((97, -2, -3), (5, 79, 2))
    r = ftn.FArray.empty(s.shape[::-1])
    ftn.transpose(r, s)
    so = OA(a, [-2, 3]).section((97, -2, -3), (5, 79, 2))
    np.testing.assert_array_equal(r.to_numpy(), so.to_numpy().T)
    back = ftn.FArray.empty(s.shape)
    ftn.transpose(back, r)
    np.testing.assert_array_equal(back.to_numpy(), so.to_numpy())


def test_transpose_c1(ftn):
    a = synth.farray((64, 48), mode=synth.LINEAR)
    A = ftn.FArray.from_numpy(a, [0, 1])
    r = ftn.FArray.empty((48, 32))
    ftn.transpose(r, A.section((0, 63, 2), (1, 48)))
    i, j = np.meshgrid(np.arange(48), np.arange(32), indexing="ij")
    np.testing.assert_array_equal(r.to_numpy(), (2 * j + 64 * i).astype(np.float64))   # decodes offsets


def test_transpose_int32_large(ftn):
    """A 4096 x 3000 int32 block with offset encoding i + 65536 j (the paper's 32768^2 pattern)."""
    n1, n2 = 4096, 3000
    a = ftn.FArray.empty((n1, n2), dtype=torch.int32)
    ftn.gen_fill(a, 0, 0, ftn.GEN_LINEAR)
    r = ftn.FArray.empty((n2, n1), dtype=torch.int32)
    ftn.transpose(r, a)
    t = r.to_numpy()
    j, i = np.meshgrid(np.arange(n2), np.arange(n1), indexing="ij")
    np.testing.assert_array_equal(t, (i + n1 * j).astype(np.int32))


def test_transpose_real8_large_tma_path(ftn):
    """real(8) 4100 x 3002 (the TMA path: 32 x 32 tiles, ragged in both dimensions, ~14 tiles
    per persistent CTA) with the exact offset encoding i + n1 j; and a strided section of it
    (the 16-byte-load path)."""
    n1, n2 = 4100, 3002
    a = ftn.FArray.empty((n1, n2))
    ftn.gen_fill(a, 0, 0, ftn.GEN_LINEAR)
    r = ftn.FArray.empty((n2, n1))
    ftn.transpose(r, a)
    j, i = np.meshgrid(np.arange(n2), np.arange(n1), indexing="ij")
    np.testing.assert_array_equal(r.to_numpy(), (i + n1 * j).astype(np.float64))
    r2 = ftn.FArray.empty((n2, n1 // 2))
    ftn.transpose(r2, a.section((2, n1, 2), (1, n2)))
    np.testing.assert_array_equal(r2.to_numpy(), (i[:, 1::2] + n1 * j[:, 1::2]).astype(np.float64))


def _small(m, n, k):
    """ftn_matmul's small-product rule (matmul.cu small_matmul): the sequential-fold kernel."""
    return m * n * k <= (1 << 21) and k <= 4096


def _mm_check(ftn, a, b, lba=(1, 1), lbb=(1, 1), exact=False, csec=None, force_dmma=False):
    m, k = a.shape
    n = b.shape[1]
    A, B = ftn.FArray.from_numpy(a, lba), ftn.FArray.from_numpy(b, lbb)
    C = ftn.FArray.empty((m, n))
    ftn.matmul(C, A, B, force_dmma=force_dmma)
    co, t = np.zeros((m, n), order="F"), np.zeros((m, n), order="F")
    oracle.matmul(OA(co), OA(a, lba), OA(b, lbb), OA(t))
    got = C.to_numpy()
    if not force_dmma and _small(m, n, k):
        exact = True              # the sequential fold IS the oracle's order: bit-identical
    if exact:
        np.testing.assert_array_equal(got, co)
    else:
        assert np.all(np.abs(got - co) <= 4 * k * U * t), f"outside bound for {(m, n, k)}"
    return got


@pytest.mark.parametrize("mnk", [(1, 1, 1), (2, 3, 5), (16, 8, 4), (33, 17, 65), (48, 48, 48), (128, 128, 32),
                                 (129, 127, 33), (127, 129, 31), (200, 300, 100), (255, 257, 97), (512, 384, 640)])
@pytest.mark.parametrize("force_dmma", [False, True])
def test_matmul_random(ftn, mnk, force_dmma):
    m, n, k = mnk
    _mm_check(ftn, synth.farray((m, k), array_id=1, mode=synth.U11), synth.farray((k, n), array_id=2, mode=synth.U11),
              force_dmma=force_dmma)


@pytest.mark.parametrize("force_dmma", [False, True])
def test_matmul_small_grid_all(ftn, force_dmma):
    """(m, n, k) over a sweep of small sizes around the m16n8k4 and 128-tile edges; the
    sequential-fold kernel bit-identical to the oracle, the forced DMMA path within the bound."""
    for m in (1, 7, 16, 17, 33):
        for n in (1, 8, 9, 31):
            for k in (1, 3, 4, 5, 32, 33):
                _mm_check(ftn, synth.farray((m, k), array_id=m, mode=synth.U11),
                          synth.farray((k, n), array_id=n + 100, mode=synth.U11), force_dmma=force_dmma)


@pytest.mark.parametrize("ta,tb", [(False, False), (True, False), (False, True), (True, True)])
def test_small_matmul_sections_transposes_bit_exact(ftn, ta, tb):
    """The small-product kernel on strided / reversed sections with lbounds and TRANSPOSE flags:
    bit-identical to the oracle's sequential fold of MATMUL(op(a), op(b)) formed explicitly."""
    rng = np.random.default_rng(11 + 2 * ta + tb)
    pa = np.asfortranarray(rng.uniform(-1, 1, (61, 47)))
    pb = np.asfortranarray(rng.uniform(-1, 1, (53, 59)))
    A, B = ftn.FArray.from_numpy(pa, [-3, 2]), ftn.FArray.from_numpy(pb, [0, 0])
    As = A.section((55, -3, -2), (2, 48, 2))            # 30 x 24
    Bs = B.section((0, 48, 2), (58, 0, -2))             # 25 x 30
    a_op = np.asfortranarray(pa[58::-2, 0:47:2])         # As as numpy (30 x 24)
    b_op = np.asfortranarray(pb[0:49:2, 58::-2])         # Bs as numpy (25 x 30)
    # op(a) (m x k) and op(b) (k x n) with a common k; a / b are stored transposed when flagged
    k = 24
    a_mat = np.asfortranarray(a_op[:, :k])               # 30 x 24
    b_mat = np.asfortranarray(b_op[:k, :])               # 24 x 30
    Am, Bm = ftn.FArray.from_numpy(a_mat.T if ta else a_mat), ftn.FArray.from_numpy(b_mat.T if tb else b_mat)
    C = ftn.FArray.empty((a_mat.shape[0], b_mat.shape[1]))
    ftn.matmul(C, Am, Bm, transpose_a=ta, transpose_b=tb)
    co, t = np.zeros(C.shape, order="F"), np.zeros(C.shape, order="F")
    oracle.matmul(OA(co), OA(a_mat), OA(b_mat), OA(t))
    np.testing.assert_array_equal(C.to_numpy(), co)
    # and the strided sections themselves (no transpose flags): As (30 x 24) x Bs-rows (24 x 30)
    Bs2 = B.section((0, 46, 2), (58, 0, -2))            # 24 x 30
    C2 = ftn.FArray.empty((30, 30))
    ftn.matmul(C2, As, Bs2)
    co2, t2 = np.zeros((30, 30), order="F"), np.zeros((30, 30), order="F")
    oracle.matmul(OA(co2), OA(a_op), OA(np.asfortranarray(pb[0:47:2, 58::-2])), OA(t2))
    np.testing.assert_array_equal(C2.to_numpy(), co2)


def test_matmul_exact_cases(ftn):
    a = synth.farray((300, 200), mode=synth.U11)
    got = _mm_check(ftn, a, np.eye(200, order="F"), exact=True)
    np.testing.assert_array_equal(got, a)
    perm = np.random.default_rng(3).permutation(200)
    P = np.zeros((200, 200), order="F")
    P[perm, np.arange(200)] = 1.0
    got = _mm_check(ftn, a, P, exact=True)
    np.testing.assert_array_equal(got, a[:, perm])
    ia = synth.farray((257, 1000), array_id=4, mode=synth.INT8)
    ib = synth.farray((1000, 129), array_id=5, mode=synth.INT8)
    _mm_check(ftn, ia, ib, exact=True)


def test_matmul_c1(ftn):
    """C1: MATMUL(TRANSPOSE(s), s) closed form (exact) and a plain 48^3 (R#15)."""
    a = synth.farray((64, 48), mode=synth.LINEAR)
    A = ftn.FArray.from_numpy(a, [0, 1])
    s = A.section((0, 63, 2), (1, 48))            # not TMA-able (dim-1 stride 16 B): packed in ws
    st = ftn.FArray.empty((48, 32))
    ftn.transpose(st, s)
    c = ftn.FArray.empty((48, 48))
    ftn.matmul(c, st, s)
    p, q = np.meshgrid(np.arange(1, 49), np.arange(1, 49), indexing="ij")
    closed = 41664 + 63488 * (p + q - 2) + 131072 * (p - 1) * (q - 1)
    np.testing.assert_array_equal(c.to_numpy(), closed.astype(np.float64))
    _mm_check(ftn, synth.farray((48, 48), array_id=7, mode=synth.U11), synth.farray((48, 48), array_id=8,
                                                                                      mode=synth.U11))


def test_matmul_strided_operands_and_output(ftn):
    a = synth.farray((90, 70), array_id=1, mode=synth.U11)
    b = synth.farray((71, 61), array_id=2, mode=synth.U11)    # odd leading dim: not TMA-able
    A, B = ftn.FArray.from_numpy(a), ftn.FArray.from_numpy(b)
    As = A.section((89, 1, -2), (1, 70))
    Bs = B.section((1, 70), (61, 1, -3))
    big = ftn.FArray.empty((50, 50))
    ftn.fill(big, -1.0)
    Cs = big.section((2, 46), (50, 10, -2))
    ftn.matmul(Cs, As, Bs)
    co, t = np.zeros(Cs.shape, order="F"), np.zeros(Cs.shape, order="F")
    oracle.matmul(OA(co), OA(a).section((89, 1, -2), (1, 70, 1)), OA(b).section((1, 70, 1), (61, 1, -3)), OA(t))
    assert np.all(np.abs(Cs.to_numpy() - co) <= 4 * 70 * U * t)
    full = big.to_numpy()
    mask = np.ones((50, 50), bool)
    mask[1:46, 49:8:-2] = False
    assert (full[mask] == -1.0).all()


def test_matmul_errors(ftn):
    with pytest.raises(ftn.FtnError) as e:
        ftn.matmul(ftn.FArray.empty((3, 3)), ftn.FArray.empty((3, 4)), ftn.FArray.empty((3, 3)))
    assert e.value.name == "FTN_ERR_SHAPE"
    with pytest.raises(ftn.FtnError) as e:      # vector x vector is not a MATMUL form
        ftn.matmul(ftn.FArray.empty((3,)), ftn.FArray.empty((3,)), ftn.FArray.empty((3,)))
    assert e.value.name == "FTN_ERR_RANK"
    with pytest.raises(ftn.FtnError) as e:      # TRANSPOSE of a vector
        ftn.matmul(ftn.FArray.empty((4,)), ftn.FArray.empty((3,)), ftn.FArray.empty((3, 4)), transpose_a=True)
    assert e.value.name == "FTN_ERR_RANK"


@pytest.mark.slow
def test_matmul_c3_full_size_sampled(ftn):
    """C3 at 8192^3 in the bench's launch configuration: Freivalds (C x vs A (B x)) plus
    sampled elements recomputed by the oracle, and the integer-valued variant exactly."""
    n = 8192
    A, B, C = ftn.FArray.empty((n, n)), ftn.FArray.empty((n, n)), ftn.FArray.empty((n, n))
    ftn.gen_fill(A, synth.SEED, 1, ftn.GEN_U11)
    ftn.gen_fill(B, synth.SEED, 2, ftn.GEN_U11)
    ftn.matmul(C, A, B)
    a, b, c = A.tensor.cpu().numpy(), B.tensor.cpu().numpy(), C.tensor.cpu().numpy()
    rng = np.random.default_rng(0)
    for _ in range(64):
        i, j = int(rng.integers(n)), int(rng.integers(n))
        v, t = oracle.matmul_element(OA(np.asfortranarray(a)), OA(np.asfortranarray(b)), i, j)
        assert abs(c[i, j] - v) <= 4 * n * U * t
    x = rng.standard_normal(n)
    lhs = c @ x
    rhs = a @ (b @ x)
    scale = np.abs(a) @ (np.abs(b) @ np.abs(x))
    assert np.all(np.abs(lhs - rhs) <= 8 * n * U * scale)
    ftn.gen_fill(A, synth.SEED, 3, ftn.GEN_INT8)
    ftn.gen_fill(B, synth.SEED, 4, ftn.GEN_INT8)
    ftn.matmul(C, A, B)
    ai, bi = A.tensor.cpu().numpy().astype(np.int64), B.tensor.cpu().numpy().astype(np.int64)
    rows = rng.integers(0, n, size=8)
    np.testing.assert_array_equal(C.tensor.cpu().numpy()[rows], (ai[rows] @ bi).astype(np.float64))


@pytest.mark.slow
def test_transpose_paper_size(ftn):
    """Table III shape: int32 32768^2 (the bench row's launch configuration), offset-encoded
    input (element t = i + 32768 j wraps modulo 2^32 exactly as the generator does); sampled
    rows and columns of the result against the closed form."""
    n = 32768
    a = ftn.FArray.empty((n, n), dtype=torch.int32)
    ftn.gen_fill(a, 0, 0, ftn.GEN_LINEAR)
    r = ftn.FArray.empty((n, n), dtype=torch.int32)
    ftn.transpose(r, a)
    rng = np.random.default_rng(2)
    for c in [0, 1, n - 1] + [int(v) for v in rng.integers(0, n, 6)]:
        col = r.section((1, n), (c + 1, c + 1)).to_numpy().ravel()      # r(:, c) = a(c, :)
        j = np.arange(n, dtype=np.int64)
        np.testing.assert_array_equal(col, ((c + n * j) % (1 << 32)).astype(np.uint32).view(np.int32))
        row = r.section((c + 1, c + 1), (1, n)).to_numpy().ravel()      # r(c, :) = a(:, c)
        i = np.arange(n, dtype=np.int64)
        np.testing.assert_array_equal(row, ((i + n * c) % (1 << 32)).astype(np.uint32).view(np.int32))


def test_matmul_ieee_specials(ftn):
    """NaN and Inf propagate as IEEE arithmetic requires whatever the summation order: every
    result element is classified (NaN / +Inf / -Inf / finite) exactly as by the oracle, and the
    finite ones stay within the R#8 bound."""
    m, k, n = 70, 90, 50
    a = synth.farray((m, k), array_id=21, mode=synth.U11)
    b = synth.farray((k, n), array_id=22, mode=synth.U11)
    a[3, 5] = np.nan
    a[10, 7] = np.inf
    a[11, 7] = -np.inf
    b[7, 4] = 0.0                       # Inf * 0 = NaN in column 4 of rows 10, 11
    b[20, 9] = np.inf
    a[40, 20] = -1.0                     # row 40, column 9: -Inf
    A, B = ftn.FArray.from_numpy(a), ftn.FArray.from_numpy(b)
    C = ftn.FArray.empty((m, n))
    ftn.matmul(C, A, B)
    got = C.to_numpy()
    co, t = np.zeros((m, n), order="F"), np.zeros((m, n), order="F")
    oracle.matmul(OA(co), OA(a), OA(b), OA(t))
    for cls in (np.isnan, np.isposinf, np.isneginf):
        np.testing.assert_array_equal(cls(got), cls(co))
    fin = np.isfinite(co)
    assert np.all(np.abs(got[fin] - co[fin]) <= 4 * k * U * t[fin])
    assert np.isnan(got[3, 0]) and np.isnan(got[10, 4]) and np.isneginf(got[40, 9])


def test_transpose_every_shape_to_70(ftn):
    """SURVEY §8(c.4) tails: every (n1, n2) in [1, 70]^2 (tile remainders in both dimensions)."""
    rng = np.random.default_rng(70)
    for n1 in range(1, 71):
        for n2 in range(1, 71):
            a = np.asfortranarray(rng.uniform(-1, 1, (n1, n2)))
            r = ftn.FArray.empty((n2, n1))
            ftn.transpose(r, ftn.FArray.from_numpy(a, [1, -1]))
            ro = np.zeros((n2, n1), order="F")
            oracle.transpose(OA(ro), OA(a, [1, -1]))
            np.testing.assert_array_equal(r.to_numpy(), ro, err_msg=str((n1, n2)))


@pytest.mark.parametrize("force_dmma", [False, True])
def test_matmul_cube_33_sampled(ftn, force_dmma):
    """SURVEY §8(c.4) tails: 300 (m, n, k) drawn from {1..33}^3 (the small-product kernel is
    bit-identical to the oracle; the DMMA path within the bound)."""
    rng = np.random.default_rng(33 + force_dmma)
    for _ in range(300):
        m, n, k = (int(v) for v in rng.integers(1, 34, 3))
        _mm_check(ftn, np.asfortranarray(rng.uniform(-1, 1, (m, k))), np.asfortranarray(rng.uniform(-1, 1, (k, n))),
                  force_dmma=force_dmma)
