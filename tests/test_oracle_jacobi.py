"""Pins for the oracle's Jacobi sweeps (R#16, R#17, R#23).

Independent references: discrete-harmonic fields (exact fixed points), the delta
impulse response, a hand-worked 3x3 grid whose value depends on the neighbour-sum
order, mirror symmetry, and the maximum principle.
"""
import numpy as np
import pytest

import oracle
import synth
from oracle import FArray

C2, C3 = 0.25, 1.0 / 6.0


def _grid2(n1, n2, f):
    i, j = np.meshgrid(np.arange(n1, dtype=np.float64), np.arange(n2, dtype=np.float64), indexing="ij")
    return np.asfortranarray(f(i, j))


def _run(orc, u, sweeps, c, lbs=None):
    w = u.copy(order="F")
    U_, W_ = FArray(u, lbs), FArray(w, lbs)
    in_new = orc.jacobi(U_, W_, sweeps, c)
    return (w if in_new else u), in_new


@pytest.mark.parametrize("f", [lambda i, j: i + 2 * j, lambda i, j: i * j, lambda i, j: i * i - j * j])
@pytest.mark.parametrize("sweeps", [1, 2, 7])
def test_2d_harmonic_fixed_points(orc, f, sweeps):
    u0 = _grid2(13, 9, f)
    res, in_new = _run(orc, u0.copy(order="F"), sweeps, C2, [0, -4])
    assert in_new == (sweeps % 2 == 1)
    np.testing.assert_array_equal(res, u0)


def test_3d_harmonic_fixed_point(orc):
    """R#23: c = fl(1/6); (6u) * fl(1/6) == u for integer u < 2^20, so i + 2j + 3k is fixed."""
    i, j, k = np.meshgrid(np.arange(9.0), np.arange(7.0), np.arange(6.0), indexing="ij")
    u0 = np.asfortranarray(i + 2 * j + 3 * k)
    for sweeps in (1, 4):
        res, _ = _run(orc, u0.copy(order="F"), sweeps, C3, [1, 1, 1])
        np.testing.assert_array_equal(res, u0)
    assert float.hex(C3) == "0x1.5555555555555p-3"


def test_2d_delta_impulse(orc):
    u = np.zeros((7, 6), order="F")
    u[3, 2] = 1.0
    res, _ = _run(orc, u, 1, C2)
    expect = np.zeros((7, 6))
    for di, dj in ((-1, 0), (1, 0), (0, -1), (0, 1)):
        expect[3 + di, 2 + dj] = 0.25
    np.testing.assert_array_equal(res, expect)


def test_3d_delta_impulse(orc):
    u = np.zeros((5, 5, 5), order="F")
    u[2, 2, 2] = 1.0
    res, _ = _run(orc, u, 1, C3)
    expect = np.zeros((5, 5, 5))
    for d in range(3):
        for s in (-1, 1):
            idx = [2, 2, 2]
            idx[d] += s
            expect[tuple(idx)] = C3
    np.testing.assert_array_equal(res, expect)


def test_3x3_neighbour_order(orc):
    """One interior point: c * (((u(1,2) + u(3,2)) + u(2,1)) + u(2,3)).  With u(1,2) = 1,
    u(3,2) = u(2,1) = 2^-53, u(2,3) = 0 the prescribed order gives 1 * 0.25 = 0.25 (both tiny
    additions tie to even), while adding the two tiny terms first would give 0.25 + 2^-54."""
    u = np.zeros((3, 3), order="F")
    u[0, 1], u[2, 1], u[1, 0], u[1, 2] = 1.0, 2.0 ** -53, 2.0 ** -53, 0.0
    res, _ = _run(orc, u, 1, C2)
    assert res[1, 1] == 0.25
    u2 = np.zeros((3, 3), order="F")
    u2[0, 1], u2[2, 1], u2[1, 0], u2[1, 2] = 2.0 ** -53, 2.0 ** -53, 1.0, 0.0
    res2, _ = _run(orc, u2, 1, C2)
    assert res2[1, 1] == 0.25 + 2.0 ** -54          # (u + u) + 1 = 1 + 2^-52


def test_3d_neighbour_order(orc):
    # pairs are added (i), then j-1, j+1, k-1, k+1: ((((1e-16... ) chosen so order matters
    u = np.zeros((3, 3, 3), order="F")
    u[0, 1, 1], u[2, 1, 1] = 2.0 ** -53, 2.0 ** -53    # i pair first: 2^-52
    u[1, 0, 1] = 1.0                                   # then 1 -> 1 + 2^-52
    res, _ = _run(orc, u, 1, 1.0)
    assert res[1, 1, 1] == 1.0 + 2.0 ** -52
    v = np.zeros((3, 3, 3), order="F")
    v[0, 1, 1], v[1, 0, 1], v[1, 1, 2] = 1.0, 2.0 ** -53, 2.0 ** -53   # 1 + u -> 1, + u -> 1
    res, _ = _run(orc, v, 1, 1.0)
    assert res[1, 1, 1] == 1.0


def test_mirror_commutes(orc):
    """Reversing dim 1 commutes bit-exactly (the first pair is the i pair, + is commutative)."""
    u = synth.jacobi_init((17, 11))
    a, _ = _run(orc, u.copy(order="F"), 5, C2)
    m = np.asfortranarray(u[::-1, :])
    b, _ = _run(orc, m, 5, C2)
    np.testing.assert_array_equal(a[::-1, :], b)
    u3 = synth.jacobi_init((9, 8, 7))
    a3, _ = _run(orc, u3.copy(order="F"), 3, C3)
    b3, _ = _run(orc, np.asfortranarray(u3[::-1, :, :]), 3, C3)
    np.testing.assert_array_equal(a3[::-1], b3)


def test_maximum_principle(orc):
    u = synth.jacobi_init((33, 21))
    lo, hi = u.min(), u.max()
    res, _ = _run(orc, u.copy(order="F"), 25, C2)
    assert res.min() >= lo and res.max() <= hi
    iv = np.asfortranarray(synth.farray((15, 14, 13), mode=synth.INT8) * 6.0)
    res3, _ = _run(orc, iv.copy(order="F"), 1, C3)
    assert res3.min() >= iv.min() and res3.max() <= iv.max()


def test_boundary_untouched_and_degenerate(orc):
    u = synth.jacobi_init((12, 10))
    w = np.full((12, 10), -9.0, order="F")
    in_new = orc.jacobi(FArray(u), FArray(w), 1, C2)
    assert in_new
    assert (w[0, :] == -9).all() and (w[-1, :] == -9).all() and (w[:, 0] == -9).all() and (w[:, -1] == -9).all()
    for shape in ((2, 10), (10, 2), (1, 1)):           # no interior: nothing changes
        a = synth.farray(shape)
        b = a.copy(order="F")
        orc.jacobi(FArray(a), FArray(b), 3, C2)
        np.testing.assert_array_equal(a, b)
    a = synth.farray((6, 6))
    b = a.copy(order="F")
    assert orc.jacobi(FArray(a), FArray(b), 0, C2) is False
    np.testing.assert_array_equal(a, b)


def test_strided_descriptors(orc):
    """The DO nest over a section gives the same values as over its packed copy."""
    big = synth.jacobi_init((30, 24))
    B = FArray(big)
    s = B.section((2, 28, 2), (24, 1, -1))
    packed = s.to_numpy()
    w_big = big.copy(order="F")
    orc.jacobi(s, FArray(w_big).section((2, 28, 2), (24, 1, -1)), 4, C2)
    res_sec = s.to_numpy()
    res_p, _ = _run(orc, packed, 4, C2)
    np.testing.assert_array_equal(res_sec, res_p)


# ---- convergence (R#25) ------------------------------------------

def test_maxabsdiff_vs_numpy(orc):
    a = synth.farray((40, 30), array_id=1, mode=synth.U11)
    b = synth.farray((40, 30), array_id=2, mode=synth.U11)
    assert orc.maxabsdiff(FArray(a), FArray(b)) == np.max(np.abs(a - b))
    assert orc.maxabsdiff(FArray(a), FArray(a)) == 0.0
    assert orc.maxabsdiff(FArray(np.zeros(0)), FArray(np.zeros(0))) == -np.inf


def test_solve_equals_fixed_sweeps_when_not_converging(orc):
    u = synth.jacobi_init((37, 29))
    a, b = u.copy(order="F"), u.copy(order="F")
    done, res, new = orc.jacobi_solve(FArray(a), FArray(b), 13, 4, -1.0, C2)
    assert done == 13 and new
    c, d = u.copy(order="F"), u.copy(order="F")
    orc.jacobi(FArray(c), FArray(d), 13, C2)
    np.testing.assert_array_equal(b, d)
    assert res == np.max(np.abs(b[1:-1, 1:-1] - a[1:-1, 1:-1]))   # last two iterates, interior (R#25)


def test_solve_harmonic_stops_at_first_check(orc):
    i, j = np.meshgrid(np.arange(20.0), np.arange(15.0), indexing="ij")
    u = np.asfortranarray(i + 2 * j)
    done, res, _ = orc.jacobi_solve(FArray(u.copy(order="F")), FArray(u.copy(order="F")), 100, 5, 0.0, C2)
    assert done == 5 and res == 0.0


def test_solve_residual_monotone_on_dyadic_data(orc):
    """||u_{s+1} - u_s||_inf <= ||u_s - u_{s-1}||_inf (Jacobi is an averaging map); dyadic data keep
    every sum exact for the first sweeps, so the inequality holds bit for bit."""
    u = np.asfortranarray(synth.farray((16, 16), mode=synth.INT8) * 2.0 ** -4)
    res = []
    for s in range(1, 12):
        a, b = u.copy(order="F"), u.copy(order="F")
        _, r, _ = orc.jacobi_solve(FArray(a), FArray(b), s, s, -1.0, C2)
        res.append(r)
    assert all(x >= y for x, y in zip(res, res[1:]))


def test_solve_residual_is_over_the_interior(orc):
    """R#25: the residual compares the last two iterates on the points a sweep updates.  With
    different boundary rings in u and unew (each array keeps its own ring under the swap) the
    ring differences do not enter; the iterates themselves come from the plain DO nest."""
    u = synth.jacobi_init((23, 19))
    w = u.copy(order="F")
    w[0, :] += 100.0          # unew's ring differs from u's by 100 on one face
    for s in (1, 2, 5, 6):
        a, b = u.copy(order="F"), w.copy(order="F")
        done, res, new = orc.jacobi_solve(FArray(a), FArray(b), s, s, -1.0, C2)
        assert done == s and new == (s % 2 == 1)
        c, d = u.copy(order="F"), w.copy(order="F")          # iterates s-1 and s by the DO nest
        orc.jacobi(FArray(c), FArray(d), s, C2)
        assert res == np.max(np.abs(d[1:-1, 1:-1] - c[1:-1, 1:-1])) < 100.0
    e = np.zeros((2, 9), order="F")                           # no interior: -inf (R#10)
    _, res, _ = orc.jacobi_solve(FArray(e.copy(order="F")), FArray(e.copy(order="F")), 3, 3, -1.0, C2)
    assert res == -np.inf
