"""Pins for the oracle's TRANSPOSE and MATMUL (R#8, R#14, R#15).

Independent references: numpy's transpose and BLAS matmul (within the bound),
identity / permutation products (exact), integer-valued products (exact in any order),
the C1 closed form of MATMUL(TRANSPOSE(s), s), and SPEC's 1e-12 triple-loop criterion.
"""
import json
import os

import numpy as np
import pytest

import oracle
import synth
from oracle import FArray

U = 2.0 ** -53
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.mark.parametrize("dtype", [np.float64, np.int32, np.float32, np.int64])
@pytest.mark.parametrize("shape", [(1, 1), (1, 9), (33, 17), (64, 48)])
def test_transpose_vs_numpy(orc, dtype, shape):
    mode = synth.U11 if np.dtype(dtype).kind == "f" else synth.RAW
    a = synth.farray(shape, mode=mode, dtype=dtype)
    r = np.zeros(shape[::-1], dtype=dtype, order="F")
    orc.transpose(FArray(r, [1, 1]), FArray(a, [0, 5]))
    np.testing.assert_array_equal(r, a.T)
    back = np.zeros(shape, dtype=dtype, order="F")
    orc.transpose(FArray(back), FArray(r))
    np.testing.assert_array_equal(back, a)                   # involution


def test_transpose_of_section(orc):
    """TRANSPOSE(a(sec1, sec2)) == TRANSPOSE(a)(sec2, sec1)."""
    a = synth.farray((20, 30), mode=synth.LINEAR)
    A = FArray(a, [-2, 3])
    s = A.section((16, -2, -3), (5, 32, 2))
    r1 = np.zeros(s.shape[::-1], order="F")
    orc.transpose(FArray(r1), s)
    at = np.zeros((30, 20), order="F")
    orc.transpose(FArray(at, [3, -2]), A)
    s2 = FArray(at, [3, -2]).section((5, 32, 2), (16, -2, -3))
    np.testing.assert_array_equal(r1, s2.to_numpy())


def _mm(orc, a, b, lbs=((1, 1), (1, 1))):
    m, k = a.shape
    n = b.shape[1]
    c = np.zeros((m, n), order="F")
    t = np.zeros((m, n), order="F")
    orc.matmul(FArray(c), FArray(a, lbs[0]), FArray(b, lbs[1]), FArray(t))
    return c, t


@pytest.mark.parametrize("mnk", [(1, 1, 1), (5, 7, 3), (33, 17, 65), (48, 48, 48), (16, 16, 16)])
def test_matmul_vs_blas_within_bound(orc, mnk):
    m, n, k = mnk
    a = synth.farray((m, k), array_id=1, mode=synth.U11)
    b = synth.farray((k, n), array_id=2, mode=synth.U11)
    c, t = _mm(orc, a, b)
    ref = a @ b
    assert np.all(np.abs(c - ref) <= 2 * 4 * k * U * t)      # both within 4kU of exact
    if m == n == k == 16:
        assert np.max(np.abs(c - ref) / np.abs(ref)) < 1e-12  # SPEC S:469 triple-loop criterion


def test_matmul_identity_and_permutation_exact(orc):
    a = synth.farray((37, 29), mode=synth.U11)
    c, _ = _mm(orc, a, np.eye(29, order="F"))
    np.testing.assert_array_equal(c, a)
    perm = np.random.default_rng(2).permutation(29)
    P = np.zeros((29, 29), order="F")
    P[perm, np.arange(29)] = 1.0                               # column q of a@P is column perm[q] of a
    c, _ = _mm(orc, a, P)
    np.testing.assert_array_equal(c, a[:, perm])
    c, _ = _mm(orc, np.asfortranarray(P.T[:, :]), np.asfortranarray(a[:29, :]))
    np.testing.assert_array_equal(c, a[:29, :][perm, :])


def test_matmul_integer_valued_exact(orc):
    a = synth.farray((40, 300), array_id=3, mode=synth.INT8)
    b = synth.farray((300, 24), array_id=4, mode=synth.INT8)
    c, _ = _mm(orc, a, b)
    np.testing.assert_array_equal(c, (a.astype(np.int64) @ b.astype(np.int64)).astype(np.float64))


def test_c1_matmul_transpose_closed_form(orc):
    g = json.load(open(os.path.join(GOLDEN, "c1_closed_forms.json")))
    assert "41664" in g["MATMUL(TRANSPOSE(s),s)(p,q)"]
    a = synth.farray((64, 48), mode=synth.LINEAR)
    s = FArray(a, [0, 1]).section((0, 63, 2), (1, 48, 1))
    st = np.zeros((48, 32), order="F")
    orc.transpose(FArray(st), s)
    c, _ = _mm(orc, st, s.to_numpy())
    p, q = np.meshgrid(np.arange(1, 49), np.arange(1, 49), indexing="ij")
    closed = 41664 + 63488 * (p + q - 2) + 131072 * (p - 1) * (q - 1)
    np.testing.assert_array_equal(c, closed.astype(np.float64))


def test_matmul_element_matches_full(orc):
    a = synth.farray((19, 23), array_id=5, mode=synth.U11)
    b = synth.farray((23, 11), array_id=6, mode=synth.U11)
    c, t = _mm(orc, a, b)
    for i, j in [(0, 0), (18, 10), (7, 3)]:
        v, ab = orc.matmul_element(FArray(a), FArray(b), i, j)
        assert v == c[i, j] and ab == t[i, j]


def test_matmul_shape_errors(orc):
    with pytest.raises(oracle.OracleError) as e:
        orc.matmul(FArray(np.zeros((3, 3), order="F")), FArray(np.zeros((3, 4), order="F")),
                   FArray(np.zeros((3, 3), order="F")))
    assert e.value.code == 4


# ---- rank-1 forms ---------------------------------------------------------

@pytest.mark.parametrize("mk", [(1, 1), (7, 3), (65, 130), (300, 17)])
def test_matvec_vecmat_vs_blas_and_exact(orc, mk):
    m, k = mk
    a = synth.farray((m, k), array_id=1, mode=synth.U11)
    x = synth.values(k, array_id=2, mode=synth.U11)
    y, t = orc.matvec(FArray(a, [0, 3]), FArray(x, [-2]))
    assert np.all(np.abs(y - a @ x) <= 2 * 4 * k * U * t)
    b = synth.farray((k, m), array_id=3, mode=synth.U11)
    z, s = orc.vecmat(FArray(x), FArray(b))
    assert np.all(np.abs(z - x @ b) <= 2 * 4 * k * U * s)
    ia = synth.farray((m, k), array_id=4, mode=synth.INT8)
    ix = synth.values(k, array_id=5, mode=synth.INT8)
    yi, _ = orc.matvec(FArray(ia), FArray(ix))
    np.testing.assert_array_equal(yi, (ia.astype(np.int64) @ ix.astype(np.int64)).astype(np.float64))
    ib = synth.farray((k, m), array_id=6, mode=synth.INT8)
    zi, _ = orc.vecmat(FArray(ix), FArray(ib))
    np.testing.assert_array_equal(zi, (ix.astype(np.int64) @ ib.astype(np.int64)).astype(np.float64))


def test_matvec_identity_and_sections(orc):
    x = synth.values(40, mode=synth.U11)
    y, _ = orc.matvec(FArray(np.eye(40, order="F")), FArray(x))
    np.testing.assert_array_equal(y, x)
    a = synth.farray((50, 30), mode=synth.U11)
    s = FArray(a).section((49, 1, -2), (2, 30, 2))        # 25 x 15 strided, reversed
    xs = synth.values(15, array_id=9, mode=synth.U11)
    y, t = orc.matvec(s, FArray(xs))
    assert np.all(np.abs(y - s.to_numpy() @ xs) <= 2 * 4 * 15 * U * t)
