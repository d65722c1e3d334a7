"""GPU parity for SURVEY §8(f) f3: MATMUL rank-1 forms and MATMUL with TRANSPOSE'd operands
(no materialised transpose), within 4 k 2^-53 sum|a||b| of the oracle and exact on
integer-valued / identity data (R#8, R#14)."""
import numpy as np
import pytest

import oracle
import synth
from oracle import FArray as OA

pytestmark = pytest.mark.gpu
U = 2.0 ** -53


@pytest.fixture(scope="module")
def ftn():
    from paper_2409_18824_b200 import ftn
    return ftn


def _oracle_mm(a, b):
    m, k = a.shape
    n = b.shape[1]
    c, t = np.zeros((m, n), order="F"), np.zeros((m, n), order="F")
    oracle.matmul(OA(c), OA(np.asfortranarray(a)), OA(np.asfortranarray(b)), OA(t))
    return c, t


@pytest.mark.parametrize("ta,tb", [(True, False), (False, True), (True, True)])
@pytest.mark.parametrize("mnk", [(1, 1, 1), (7, 9, 5), (33, 17, 65), (128, 128, 32), (129, 257, 100), (300, 200, 513)])
def test_matmul_transposed_operands(ftn, ta, tb, mnk):
    m, n, k = mnk
    a = synth.farray((k, m) if ta else (m, k), array_id=1, mode=synth.U11)
    b = synth.farray((n, k) if tb else (k, n), array_id=2, mode=synth.U11)
    A, B = ftn.FArray.from_numpy(a), ftn.FArray.from_numpy(b)
    C = ftn.FArray.empty((m, n))
    ftn.matmul(C, A, B, transpose_a=ta, transpose_b=tb)
    # the oracle composes the definitions: TRANSPOSE then MATMUL
    opa = np.asfortranarray(a.T) if ta else a
    opb = np.asfortranarray(b.T) if tb else b
    co, t = _oracle_mm(opa, opb)
    assert np.all(np.abs(C.to_numpy() - co) <= 4 * k * U * t), (ta, tb, mnk)


def test_matmul_transpose_c1_closed_form(ftn):
    """MATMUL(TRANSPOSE(s), s) of the C1 section without forming TRANSPOSE(s): exact."""
    a = synth.farray((64, 48), mode=synth.LINEAR)
    A = ftn.FArray.from_numpy(a, [0, 1])
    s = A.section((0, 63, 2), (1, 48))
    c = ftn.FArray.empty((48, 48))
    ftn.matmul(c, s, s, transpose_a=True)
    p, q = np.meshgrid(np.arange(1, 49), np.arange(1, 49), indexing="ij")
    closed = 41664 + 63488 * (p + q - 2) + 131072 * (p - 1) * (q - 1)
    np.testing.assert_array_equal(c.to_numpy(), closed.astype(np.float64))


def test_matmul_transposed_integer_exact(ftn):
    a = synth.farray((700, 300), array_id=3, mode=synth.INT8)     # (k, m) -> TRANSPOSE gives (300, 700)
    b = synth.farray((200, 700), array_id=4, mode=synth.INT8)     # (n, k)
    C = ftn.FArray.empty((300, 200))
    ftn.matmul(C, ftn.FArray.from_numpy(a), ftn.FArray.from_numpy(b), transpose_a=True, transpose_b=True)
    ref = (a.T.astype(np.int64) @ b.T.astype(np.int64)).astype(np.float64)
    np.testing.assert_array_equal(C.to_numpy(), ref)


@pytest.mark.parametrize("mk", [(1, 1), (5, 3), (257, 129), (1000, 2000), (4096, 777), (3, 10000)])
def test_matvec_and_vecmat(ftn, mk):
    m, k = mk
    a = synth.farray((m, k), array_id=5, mode=synth.U11)
    x = synth.values(k, array_id=6, mode=synth.U11)
    A, X = ftn.FArray.from_numpy(a), ftn.FArray.from_numpy(x)
    y = ftn.FArray.empty((m,))
    ftn.matmul(y, A, X)
    yo, t = oracle.matvec(OA(a), OA(x))
    assert np.all(np.abs(y.to_numpy() - yo) <= 4 * k * U * t)
    b = synth.farray((k, m), array_id=7, mode=synth.U11)
    z = ftn.FArray.empty((m,))
    ftn.matmul(z, X, ftn.FArray.from_numpy(b))
    zo, s = oracle.vecmat(OA(x), OA(b))
    assert np.all(np.abs(z.to_numpy() - zo) <= 4 * k * U * s)
    ia = synth.farray((m, k), array_id=8, mode=synth.INT8)
    ix = synth.values(k, array_id=9, mode=synth.INT8)
    yi = ftn.FArray.empty((m,))
    ftn.matmul(yi, ftn.FArray.from_numpy(ia), ftn.FArray.from_numpy(ix))
    np.testing.assert_array_equal(yi.to_numpy(), (ia.astype(np.int64) @ ix.astype(np.int64)).astype(np.float64))
    ib = synth.farray((k, m), array_id=10, mode=synth.INT8)
    zi = ftn.FArray.empty((m,))
    ftn.matmul(zi, ftn.FArray.from_numpy(ix), ftn.FArray.from_numpy(ib))     # vector x matrix, exact
    np.testing.assert_array_equal(zi.to_numpy(), (ix.astype(np.int64) @ ib.astype(np.int64)).astype(np.float64))


def test_matvec_sections(ftn):
    a = synth.farray((300, 200), mode=synth.U11)
    x = synth.values(400, array_id=3, mode=synth.U11)
    A, X = ftn.FArray.from_numpy(a), ftn.FArray.from_numpy(x)
    As = A.section((299, 1, -3), (1, 200, 2))            # 100 x 100 strided/reversed
    Xs = X.section((400, 1, -4))                         # 100, reversed
    y = ftn.FArray.empty((200,))
    ys = y.section((1, 200, 2))
    ftn.matmul(ys, As, Xs)
    yo, t = oracle.matvec(OA(a).section((299, 1, -3), (1, 200, 2)), OA(x).section((400, 1, -4)))
    assert np.all(np.abs(ys.to_numpy() - yo) <= 4 * 100 * U * t)
