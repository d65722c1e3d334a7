"""GPU parity for SURVEY §8(f) f2: MAXVAL(ABS(x-y)) and Jacobi to convergence (R#25) vs the
oracle -- sweeps done, residual and result bit-exact, for every temporal-blocking factor."""
import numpy as np
import pytest

import oracle
import synth
from oracle import FArray as OA
DEFAULT_FUSION = 0   # ftn_jacobi_set_fusion(0): back to the default (size-dependent)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ftn():
    from paper_2409_18824_b200 import ftn
    return ftn


def test_maxval_absdiff(ftn):
    for shape in ((1,), (1000,), (65537,), (300, 301), (40, 30, 20)):
        a = synth.farray(shape, array_id=1, mode=synth.U11)
        b = synth.farray(shape, array_id=2, mode=synth.U11)
        got = ftn.maxval_absdiff(ftn.FArray.from_numpy(a), ftn.FArray.from_numpy(b)).item()
        assert got == oracle.maxabsdiff(OA(a), OA(b)) == np.max(np.abs(a - b))
    a = synth.farray((90, 80), array_id=3, mode=synth.U11)
    b = synth.farray((90, 80), array_id=4, mode=synth.U11)
    A, B = ftn.FArray.from_numpy(a), ftn.FArray.from_numpy(b)
    got = ftn.maxval_absdiff(A.section((89, 1, -2), (1, 80, 3)), B.section((1, 89, 2), (80, 1, -3))).item()
    assert got == np.max(np.abs(a[88::-2, ::3] - b[0:89:2, ::-3]))


@pytest.mark.parametrize("T", [1, 2, 3, 4, 5, 6, 7, 8])
@pytest.mark.parametrize("shape,check,tol", [((130, 97), 5, 1e-3), ((130, 97), 7, -1.0), ((300, 200), 10, 1e-4),
                                             ((60, 50, 40), 4, 1e-3)])
def test_jacobi_solve(ftn, T, shape, check, tol):
    ftn.jacobi_set_fusion(T)
    try:
        u0 = synth.jacobi_init(shape)
        U, W = ftn.FArray.from_numpy(u0), ftn.FArray.from_numpy(u0)
        coeff = 0.25 if len(shape) == 2 else 1.0 / 6.0
        done, res, new = ftn.jacobi_solve(U, W, 60, check, tol, coeff)
        a, b = u0.copy(order="F"), u0.copy(order="F")
        d2, r2, n2 = oracle.jacobi_solve(OA(a), OA(b), 60, check, tol, coeff)
        assert (done, res, new) == (d2, r2, n2)
        np.testing.assert_array_equal((W if new else U).to_numpy(), b if n2 else a)
    finally:
        ftn.jacobi_set_fusion(DEFAULT_FUSION)


@pytest.mark.parametrize("shape,sec", [((131, 97), None), ((200, 150), ((1, 200, 2), (150, 1, -1))),
                                       ((45, 30, 21), ((45, 1, -1), (1, 30), (1, 21, 2)))])
def test_jacobi_solve_non_tma_arrays(ftn, shape, sec):
    """Solve on arrays the TMA kernels cannot address (padded temporaries): same sweeps,
    residual and result as the oracle's solve on the same (section) arrays."""
    big = synth.jacobi_init(shape)
    coeff = 0.25 if len(shape) == 2 else 1.0 / 6.0
    Bu, Bw = ftn.FArray.from_numpy(big), ftn.FArray.from_numpy(big)
    osec = tuple((1, n, 1) for n in shape) if sec is None else tuple(t if len(t) == 3 else (t[0], t[1], 1) for t in sec)
    su, sw = Bu.section(*osec), Bw.section(*osec)
    done, res, new = ftn.jacobi_solve(su, sw, 40, 7, 1e-3, coeff)
    ou, ow = big.copy(order="F"), big.copy(order="F")
    d2, r2, n2 = oracle.jacobi_solve(OA(ou).section(*osec), OA(ow).section(*osec), 40, 7, 1e-3, coeff)
    assert (done, res, new) == (d2, r2, n2)
    np.testing.assert_array_equal((sw if new else su).to_numpy(), (OA(ow) if n2 else OA(ou)).section(*osec).to_numpy())


@pytest.mark.parametrize("T", [2, 5])
@pytest.mark.parametrize("shape", [(2, 40), (40, 2), (3, 2, 9), (3, 3)])
def test_jacobi_solve_degenerate_interiors(ftn, T, shape):
    """R#25 / R#10: no interior point (or a single one): every block runs, the residual of an
    empty interior is -inf (never <= tol = -1, so all max_sweeps run), equal to the oracle."""
    ftn.jacobi_set_fusion(T)
    try:
        u0 = synth.jacobi_init(shape)
        coeff = 0.25 if len(shape) == 2 else 1.0 / 6.0
        U, W = ftn.FArray.from_numpy(u0), ftn.FArray.from_numpy(u0)
        got = ftn.jacobi_solve(U, W, 9, 4, -1.0, coeff)
        a, b = u0.copy(order="F"), u0.copy(order="F")
        ref = oracle.jacobi_solve(OA(a), OA(b), 9, 4, -1.0, coeff)
        assert got == ref
        np.testing.assert_array_equal(U.to_numpy(), a)
        np.testing.assert_array_equal(W.to_numpy(), b)
    finally:
        ftn.jacobi_set_fusion(DEFAULT_FUSION)


def test_jacobi_ws_allocates_nothing_without_workspace(ftn):
    """ftn_jacobi on arrays the TMA kernels cannot address runs the generic kernel (no
    temporaries); ftn_jacobi_ws with ftn_jacobi_workspace_size bytes runs the padded path;
    both equal the oracle."""
    import ctypes
    u0 = synth.jacobi_init((131, 97))
    coeff = 0.25
    a, b = u0.copy(order="F"), u0.copy(order="F")
    new_o = oracle.jacobi(OA(a), OA(b), 12, coeff)
    ref = b if new_o else a
    for use_ws in (False, True):
        U, W = ftn.FArray.from_numpy(u0), ftn.FArray.from_numpy(u0)
        n = ctypes.c_size_t()
        ftn._call("ftn_jacobi_workspace_size", U.ref(), W.ref(), 12, ctypes.byref(n))
        assert n.value > 0
        r = ctypes.c_int32()
        if use_ws:
            ws = ftn.workspace(n.value, slot="test_ws")
            ftn._call("ftn_jacobi_ws", U.ref(), W.ref(), 12, coeff, ctypes.c_void_p(ws.data_ptr()), ws.numel(),
                      ctypes.byref(r), None)
        else:
            ftn._call("ftn_jacobi", U.ref(), W.ref(), 12, coeff, ctypes.byref(r), None)
        assert bool(r.value) == new_o
        np.testing.assert_array_equal((W if r.value else U).to_numpy(), ref)
