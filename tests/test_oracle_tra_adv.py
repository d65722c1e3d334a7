"""Pins for the oracle's tra-adv DO nests (R#28).

The kernel body is the NEMO tracer-advection benchmark (not in the paper), recalled in
DESIGN.md R#28.  The pins are special cases worked out by hand from the advection scheme,
not a retyped copy of the oracle:
  * no velocity: every flux is a zero, so after the vertical step (md = -zbtr*(zwx -
    zwx(jk+1))) every updated point is an exact zero (its sign follows the tracer's signs) and
    every other point keeps its value;
  * a constant tracer C > 0 carried by constant velocities: every flux is velocity * C, so
    away from the first interior row / column (whose upstream flux is the boundary gradient
    umask * (md(2) - md(1)) = 0 of step 2) every flux difference is +0 and every updated
    point becomes exactly -0.0;
  * a tracer linear in jk with a constant vertical velocity W and zind = 1: the slope limiter
    gives -b in the interior, -0 next to the top (the sign of a 0 * (-b) product), and the
    upwind flux with its slope correction is worked out plane by plane below, for W > 0 and
    W < 0;
  * zind = 0 makes the scheme linear in the tracer: doubling md doubles the result exactly
    (dyadic data);
  * boundary points (ji, jj at the edges, the top jk plane) are never written.
"""
import numpy as np
import pytest

import oracle
import synth
from oracle import FArray


def _f(shape, val):
    return np.full(shape, val, dtype=np.float64, order="F")


def _run(md, tsn, pun, pvn, pwn, umask, vmask, tmask, ztfreez, rnfmsk, upsmsk, rz, iters=1):
    out = md.copy(order="F")
    oracle.tra_adv(FArray(out), FArray(tsn), FArray(pun), FArray(pvn), FArray(pwn), FArray(umask), FArray(vmask),
                   FArray(tmask), FArray(ztfreez), FArray(rnfmsk), FArray(upsmsk), rz, iters)
    return out


def _interior(shape):
    ni, nj, nk = shape
    m = np.zeros(shape, dtype=bool, order="F")
    m[1:ni - 1, 1:nj - 1, 0:nk - 1] = True
    return m


def _negzero(x):
    return (x == 0) & np.signbit(x)


@pytest.mark.parametrize("iters", [1, 3])
def test_zero_velocity_gives_negative_zero_interior(iters):
    shape = (9, 7, 6)
    md = synth.farray(shape, array_id=1, mode=synth.U11)
    z = _f(shape, 0.0)
    r = synth.farray(shape[:2], array_id=2)
    out = _run(md, synth.farray(shape, array_id=3), z, z, z, _f(shape, 1.0), _f(shape, 1.0),
               synth.farray(shape, array_id=4), r, r, r, np.linspace(0, 1, shape[2]), iters)
    inner = _interior(shape)
    assert np.all(out[inner] == 0.0)
    np.testing.assert_array_equal(out[~inner], md[~inner])


def test_constant_tracer_constant_velocities():
    """One iteration with md = C and pun, pvn, pwn constant: every flux is velocity * C, so
    every difference of fluxes away from the first interior row / column is +0 and the
    updated points become -0.0 (a second iteration no longer starts from a constant field)."""
    shape = (8, 9, 7)
    md = _f(shape, 0.75)
    out = _run(md, _f(shape, 0.5), _f(shape, 0.25), _f(shape, -0.5), _f(shape, 0.125), _f(shape, 1.0),
               _f(shape, 0.5), _f(shape, 1.0), _f(shape[:2], 0.0), _f(shape[:2], 0.3), _f(shape[:2], 0.2),
               np.full(shape[2], 0.5), 1)
    assert np.all(_negzero(out[2:-1, 2:-1, :-1]))
    assert np.all(out[1:-1, 1:-1, :-1] != 0.75)        # every updated point was written
    np.testing.assert_array_equal(out[~_interior(shape)], md[~_interior(shape)])


def _vertical_case(W):
    """md = 1 + jk/8 (jk = 0..5), pun = pvn = 0, pwn = W, zind = 1 (tmask = 1, rnfmsk = upsmsk
    = 0, tsn = 1 > ztfreez + 0.1 = 0.1)."""
    shape = (5, 4, 6)
    k = np.arange(6, dtype=np.float64)
    md = np.asfortranarray(np.broadcast_to(1.0 + k / 8.0, shape).copy())
    out = _run(md, _f(shape, 1.0), _f(shape, 0.0), _f(shape, 0.0), _f(shape, W), _f(shape, 1.0), _f(shape, 1.0),
               _f(shape, 1.0), _f(shape[:2], 0.0), _f(shape[:2], 0.0), _f(shape[:2], 0.0), np.full(6, 0.7))
    return md, out


def test_vertical_upwind_positive_w():
    """W = 0.5 (zalpha = 1, zw = 0.5 - 0.25 = 0.25).  Gradients zwx(jk) = md(jk-1) - md(jk) =
    -1/8 for jk = 1..4, 0 at jk = 0 and 5; limited slopes -1/8 for jk = 1..3 and -0 at jk = 4
    ((-1/8 + 0) * (0.25 + SIGN(0.25, -0)) = -0); fluxes zwx(0) = W md(0) = 0.5 and
    zwx(jk+1) = W (md(jk+1) + 0.25 slope(jk+1)) = 0.546875, 0.609375, 0.671875, 0.75, 0.8125;
    md(jk) = -(zwx(jk) - zwx(jk+1))."""
    md, out = _vertical_case(0.5)
    expect = [0.046875, 0.0625, 0.0625, 0.078125, 0.0625]
    for kk, e in enumerate(expect):
        assert np.all(out[1:-1, 1:-1, kk] == e), (kk, out[1:-1, 1:-1, kk])
    np.testing.assert_array_equal(out[:, :, 5], md[:, :, 5])
    np.testing.assert_array_equal(out[0], md[0])
    np.testing.assert_array_equal(out[:, -1], md[:, -1])


def test_vertical_upwind_negative_w():
    """W = -0.5 (zalpha = 0, zw = -0.5 + 0.25 = -0.25): fluxes zwx(0) = W md(0) = -0.5 and
    zwx(jk+1) = W (md(jk) - 0.25 slope(jk)) = -0.5, -0.578125, -0.640625, -0.703125, -0.75;
    md(0) = -(-0.5 - (-0.5)) = -0.0."""
    md, out = _vertical_case(-0.5)
    assert np.all(_negzero(out[1:-1, 1:-1, 0]))
    expect = [-0.078125, -0.0625, -0.0625, -0.046875]
    for kk, e in enumerate(expect, start=1):
        assert np.all(out[1:-1, 1:-1, kk] == e), (kk, out[1:-1, 1:-1, kk])


def test_linear_in_the_tracer_when_zind_is_zero():
    """zind = 0 (upsmsk = 1, tmask = 1) removes the slope terms: every flux is a velocity
    times a tracer value, so md -> 2 md doubles every updated point exactly (dyadic data)."""
    shape = (10, 8, 7)
    ints = lambda i: synth.farray(shape, array_id=i, mode=synth.INT8) / 8.0  # noqa: E731
    args = [ints(11), ints(12), ints(13), ints(14), _f(shape, 1.0), _f(shape, 1.0), _f(shape, 1.0),
            _f(shape[:2], 0.0), _f(shape[:2], 0.0), _f(shape[:2], 1.0), np.zeros(7)]
    md = ints(10)
    a = _run(md, *args)
    b = _run(np.asfortranarray(2 * md), *args)
    np.testing.assert_array_equal(b, 2 * a)


def test_horizontal_upwind_seen_through_the_vertical_step():
    """md = ji/8 (0-based ji, constant in jj, jk), pun = U = 0.5, pvn = 0, pwn = W = 1, zind = 0.
    Step 2: zwx = 1/8; step 5 (U > 0: zalpha = 0): zwx(ji) = U md(ji); step 6:
    md6(ji) = md - U (md(ji) - md(ji-1)) = ji/8 - 1/16 for ji >= 2, and 1/4 - 1/16 = 3/16 at
    ji = 1 (its upstream flux is step 2's 1/8).  Vertical (W > 0, zind = 0): zwx(jk+1) =
    W md6(jk+1), the top plane keeping md = ji/8, so md(jk) = -(md6(jk) - md6(jk+1)) = -0.0
    below the last updated plane and, on it, -(md6 - ji/8) = 1/16 (ji >= 2), -1/16 (ji = 1)."""
    shape = (8, 5, 5)
    i = np.arange(8, dtype=np.float64)
    md = np.asfortranarray(np.broadcast_to((i / 8.0)[:, None, None], shape).copy())
    out = _run(md, _f(shape, 1.0), _f(shape, 0.5), _f(shape, 0.0), _f(shape, 1.0), _f(shape, 1.0),
               _f(shape, 1.0), _f(shape, 1.0), _f(shape[:2], 0.0), _f(shape[:2], 0.0), _f(shape[:2], 1.0),
               np.zeros(5))
    assert np.all(_negzero(out[1:-1, 1:-1, :3]))
    assert np.all(out[2:-1, 1:-1, 3] == 1.0 / 16)
    assert np.all(out[1, 1:-1, 3] == -1.0 / 16)
    np.testing.assert_array_equal(out[:, :, 4], md[:, :, 4])
