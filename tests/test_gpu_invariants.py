"""GPU invariants: results do not depend on the lower bounds of the
descriptors (index-origin correctness), and identical runs give identical bits
(determinism: fixed combine orders, no atomics in any floating-point result)."""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ftn():
    from paper_2409_18824_b200 import ftn
    return ftn


def _ops(ftn, lb2, lb3):
    a = synth.farray((300, 217), array_id=1, mode=synth.U11)
    b = synth.farray((300, 217), array_id=2, mode=synth.U11)
    m = synth.farray((217, 130), array_id=3, mode=synth.U11)
    c3 = synth.farray((70, 33, 12), array_id=4, mode=synth.U11)
    A, B = ftn.FArray.from_numpy(a, lb2), ftn.FArray.from_numpy(b, lb2)
    M = ftn.FArray.from_numpy(m, lb2)
    C3 = ftn.FArray.from_numpy(c3, lb3)
    out = {}
    R = ftn.FArray.empty((300, 217), lbounds=lb2)
    ftn.muladd(R, A, B, A)
    out["muladd"] = R.to_numpy()
    out["sum"] = ftn.sum(A).item()
    out["maxval"] = ftn.maxval(C3).item()
    out["product"] = ftn.product(C3.section((1 + lb3[0], 5 + lb3[0]), (lb3[1], lb3[1] + 2), (lb3[2], lb3[2]))).item()
    out["sum_dim2"] = ftn.sum_dim(C3, 2).to_numpy()
    flat_a = ftn.FArray.from_numpy(a.reshape(-1, order="F").copy(), [lb2[0]])
    flat_b = ftn.FArray.from_numpy(b.reshape(-1, order="F").copy(), [lb2[1]])
    out["dot"] = ftn.dot_product(flat_a, flat_b).item()
    T = ftn.FArray.empty((217, 300), lbounds=lb2[::-1])
    ftn.transpose(T, A)
    out["transpose"] = T.to_numpy()
    P = ftn.FArray.empty((300, 130), lbounds=lb2)
    ftn.matmul(P, A, M)
    out["matmul"] = P.to_numpy()
    u0 = synth.jacobi_init((150, 90))
    U, W = ftn.FArray.from_numpy(u0, lb2), ftn.FArray.from_numpy(u0, lb2)
    new = ftn.jacobi(U, W, 11)
    out["jacobi"] = (W if new else U).to_numpy()
    f = [ftn.FArray.from_numpy(synth.farray((66, 20, 7), array_id=10 + q, mode=synth.U11), lb3) for q in range(3)]
    z = [ftn.FArray.from_numpy(synth.values(66, array_id=20 + q, mode=synth.U11), [lb3[0]]) for q in range(4)]
    o = [ftn.FArray.empty((66, 20, 7), lbounds=lb3) for _ in range(3)]
    for x in o:
        ftn.fill(x, 0.0)
    ftn.pw_advection(*o, *f, *z, 0.1, 0.2)
    out["advection"] = [x.to_numpy() for x in o]
    return out


def _same(a, b):
    for k in a:
        x, y = a[k], b[k]
        if isinstance(x, list):
            for p, q in zip(x, y):
                np.testing.assert_array_equal(p, q, err_msg=k)
        elif isinstance(x, np.ndarray):
            np.testing.assert_array_equal(x, y, err_msg=k)
        else:
            assert x == y or (np.isnan(x) and np.isnan(y)), k


def test_lower_bounds_do_not_change_results(ftn):
    _same(_ops(ftn, [1, 1], [1, 1, 1]), _ops(ftn, [-7, 13], [0, -511, 1024]))


def test_reruns_are_bit_identical(ftn):
    first = _ops(ftn, [1, 1], [1, 1, 1])
    for _ in range(2):
        _same(first, _ops(ftn, [1, 1], [1, 1, 1]))
