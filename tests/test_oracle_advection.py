"""Pins for the oracle's pw-advection DO nest (R#26).

The kernel body is the public pw-advection benchmark (not in the paper), reproduced in
DESIGN.md R#26.  The pins below are derived by hand from the advection form, not by retyping
the oracle: constant fields (the self-advection flux differences cancel exactly and only the
tz coefficient differences survive), single-point impulses in each field (which output points
move, with which coefficient and sign), a constant field crossed with an impulse (the
transverse interpolation stencils), quadratic homogeneity (x -> -x leaves every output
unchanged, x -> 2x scales it by 4, both exactly), untouched boundaries, and a strided section
equal to its packed copy.
"""
import numpy as np
import pytest

import oracle
import synth
from oracle import FArray

TCX, TCY = 0.25, 0.125


def _coeffs(nz, seed=3):
    r = np.random.default_rng(seed)
    # dyadic values keep products of dyadic fields exact
    return [np.asarray(r.integers(-8, 9, nz), dtype=np.float64) / 16.0 for _ in range(4)]


def _run(u, v, w, z, fill=0.0, tcx=TCX, tcy=TCY):
    outs = [np.full(u.shape, fill, order="F") for _ in range(3)]
    oracle.pw_advection(*[FArray(o) for o in outs], FArray(u), FArray(v), FArray(w), *z, tcx, tcy)
    return outs


def _field(shape, val=0.0):
    return np.full(shape, val, dtype=np.float64, order="F")


def test_constant_fields():
    nz, ny, nx = 9, 7, 6
    c = 0.5                                    # power of two: every product is exact
    z = _coeffs(nz)
    su, sv, sw = _run(_field((nz, ny, nx), c), _field((nz, ny, nx), c), _field((nz, ny, nx), c), z)
    tzc1, tzc2, tzd1, tzd2 = z
    k = np.arange(nz)[:, None, None]
    inner = (slice(1, -1),) * 3
    # x and y fluxes cancel: c*(2c) - c*(2c) = 0; the z flux leaves 2c^2 (tz1(k) - tz2(k))
    np.testing.assert_array_equal(su[inner], np.broadcast_to(2 * c * c * (tzc1 - tzc2)[k], su.shape)[inner])
    np.testing.assert_array_equal(sv[inner], np.broadcast_to(2 * c * c * (tzc1 - tzc2)[k], sv.shape)[inner])
    np.testing.assert_array_equal(sw[inner], np.broadcast_to(2 * c * c * (tzd1 - tzd2)[k], sw.shape)[inner])


@pytest.mark.parametrize("field", ["u", "v", "w"])
def test_single_impulse_self_advection(field):
    """A single value a in one field (others 0): only that field's self-advection term is
    nonzero, +coef a^2 one point downstream and -coef a^2 one point upstream."""
    shape = (9, 8, 7)
    k0, j0, i0, a = 4, 3, 3, 1.5
    f = {n: _field(shape) for n in "uvw"}
    f[field][k0, j0, i0] = a
    z = _coeffs(shape[0], seed=5)
    su, sv, sw = _run(f["u"], f["v"], f["w"], z)
    out = {"u": su, "v": sv, "w": sw}[field]
    expect = np.zeros(shape)
    if field == "u":            # x-flux tcx*(u(i-1)(u+u(i-1)) - u(i+1)(u+u(i+1)))
        expect[k0, j0, i0 + 1] = TCX * a * a
        expect[k0, j0, i0 - 1] = -TCX * a * a
    elif field == "v":          # y-flux
        expect[k0, j0 + 1, i0] = TCY * a * a
        expect[k0, j0 - 1, i0] = -TCY * a * a
    else:                       # z-flux with the level coefficients tzd1(k), tzd2(k)
        expect[k0 + 1, j0, i0] = z[2][k0 + 1] * a * a
        expect[k0 - 1, j0, i0] = -z[3][k0 - 1] * a * a
    np.testing.assert_array_equal(out, expect)
    for other in "uvw":
        if other != field:
            np.testing.assert_array_equal({"u": su, "v": sv, "w": sw}[other], np.zeros(shape))


def test_constant_u_crossed_with_v_impulse():
    """u = c everywhere, v = a at one point, w = 0.  su's y-flux interpolates v to the u point:
    tcy*c*(v(j-1,i) + v(j-1,i+1) - v(j,i) - v(j,i+1)); sv's x-flux carries u = c:
    tcx*(2c v(i-1) - 2c v(i+1)), plus its own y self-advection; sw stays 0."""
    shape = (6, 9, 9)
    k0, j0, i0, a, c = 2, 4, 4, 0.75, 0.5
    u, v, w = _field(shape, c), _field(shape), _field(shape)
    v[k0, j0, i0] = a
    z = _coeffs(shape[0], seed=7)
    su, sv, sw = _run(u, v, w, z)
    tzc1, tzc2 = z[0], z[1]
    e_su = np.zeros(shape)                       # (u's x and z fluxes vanish: u const, w = 0)
    e_su[k0, j0 + 1, i0] += TCY * (c * a)        # v(j-1, i) term
    e_su[k0, j0 + 1, i0 - 1] += TCY * (c * a)    # v(j-1, i+1) term
    e_su[k0, j0, i0] += -TCY * (c * a)           # v(j, i) term
    e_su[k0, j0, i0 - 1] += -TCY * (c * a)       # v(j, i+1) term
    inner = (slice(1, -1),) * 3
    np.testing.assert_array_equal(su[inner], e_su[inner])
    e_sv = np.zeros(shape)
    e_sv[k0, j0 + 1, i0] += TCY * a * a          # y self-advection
    e_sv[k0, j0 - 1, i0] += -TCY * a * a
    e_sv[k0, j0, i0 + 1] += TCX * (a * (2 * c))  # x flux: v(i-1) (u(j,i-1) + u(j+1,i-1))
    e_sv[k0, j0, i0 - 1] += -TCX * (a * (2 * c))
    np.testing.assert_array_equal(sv[inner], e_sv[inner])
    np.testing.assert_array_equal(sw, np.zeros(shape))
    assert tzc1.shape == tzc2.shape


@pytest.mark.parametrize("carrier", ["u", "v"])
def test_constant_carrier_crossed_with_w_impulse(carrier):
    """u (or v) = c everywhere, w = a at one point.  The carrier's z flux interpolates w to its
    point with the level coefficients: tzc1(k) c (w(k-1) + w(k-1, +1)) - tzc2(k) c (w(k) + w(k, +1))
    where +1 is i+1 for su and j+1 for sv; sw gets the carrier's transverse flux 2c a (tcx for u,
    tcy for v) and its own z self-advection tzd1(k+1) a^2 / -tzd2(k-1) a^2."""
    shape = (8, 9, 9)
    k0, j0, i0, a, c = 3, 4, 4, 0.75, 0.5
    f = {n: _field(shape) for n in "uvw"}
    f[carrier][:] = c
    f["w"][k0, j0, i0] = a
    z = _coeffs(shape[0], seed=11)
    tzc1, tzc2, tzd1, tzd2 = z
    su, sv, sw = _run(f["u"], f["v"], f["w"], z)
    inner = (slice(1, -1),) * 3
    e_s = np.zeros(shape)
    if carrier == "u":
        up = (k0 + 1, j0, i0 - 1)   # w(k-1, i+1) feeds the point one level up, one column left
        lo = (k0, j0, i0 - 1)
    else:
        up = (k0 + 1, j0 - 1, i0)
        lo = (k0, j0 - 1, i0)
    e_s[k0 + 1, j0, i0] += (tzc1[k0 + 1] * c) * a
    e_s[up] += (tzc1[k0 + 1] * c) * a
    e_s[k0, j0, i0] += -((tzc2[k0] * c) * a)
    e_s[lo] += -((tzc2[k0] * c) * a)
    got = su if carrier == "u" else sv
    np.testing.assert_array_equal(got[inner], e_s[inner])
    np.testing.assert_array_equal((sv if carrier == "u" else su), np.zeros(shape))
    e_sw = np.zeros(shape)
    e_sw[k0 + 1, j0, i0] += (tzd1[k0 + 1] * a) * a
    e_sw[k0 - 1, j0, i0] += -((tzd2[k0 - 1] * a) * a)
    t = TCX if carrier == "u" else TCY
    if carrier == "u":
        e_sw[k0, j0, i0 + 1] += t * (a * (2 * c))
        e_sw[k0, j0, i0 - 1] += -t * (a * (2 * c))
    else:
        e_sw[k0, j0 + 1, i0] += t * (a * (2 * c))
        e_sw[k0, j0 - 1, i0] += -t * (a * (2 * c))
    np.testing.assert_array_equal(sw[inner], e_sw[inner])


def test_homogeneity_and_boundary():
    shape = (10, 9, 8)
    u = synth.farray(shape, array_id=1, mode=synth.U11)
    v = synth.farray(shape, array_id=2, mode=synth.U11)
    w = synth.farray(shape, array_id=3, mode=synth.U11)
    z = _coeffs(shape[0])
    ref = _run(u, v, w, z, fill=-7.0)
    neg = _run(np.asfortranarray(-u), np.asfortranarray(-v), np.asfortranarray(-w), z, fill=-7.0)
    dbl = _run(np.asfortranarray(2 * u), np.asfortranarray(2 * v), np.asfortranarray(2 * w), z, fill=-7.0)
    inner = (slice(1, -1),) * 3
    for r, n, d in zip(ref, neg, dbl):
        np.testing.assert_array_equal(n, r)
        np.testing.assert_array_equal(d[inner], 4 * r[inner])
        m = np.ones(shape, bool)
        m[inner] = False
        assert (r[m] == -7.0).all()


def test_section_equals_packed():
    big = [synth.farray((14, 12, 10), array_id=q, mode=synth.U11) for q in range(3)]
    secs = [FArray(b).section((13, 2, -1), (1, 12, 2), (2, 9)) for b in big]
    packed = [s.to_numpy() for s in secs]
    z = _coeffs(12)
    outs_sec_owner = [np.zeros((14, 12, 10), order="F") for _ in range(3)]
    outs_sec = [FArray(o).section((13, 2, -1), (1, 12, 2), (2, 9)) for o in outs_sec_owner]
    oracle.pw_advection(*outs_sec, *secs, *z, TCX, TCY)
    outs_p = _run(*packed, z)
    for s, p in zip(outs_sec, outs_p):
        np.testing.assert_array_equal(s.to_numpy()[1:-1, 1:-1, 1:-1], p[1:-1, 1:-1, 1:-1])


def _order_case(field):
    """Fields for which the Fortran statement order of R#26 decides the rounded result of one
    output point (k0, j0, i0) of `field`; returns (fields, coefficients, tcx, tcy, expected).

    Each tendency is x term, then y term, then the parenthesised vertical term
    (tz1*flux_in - tz2*flux_out).  The cases put 2^53 into the vertical fluxes, where adding 1
    is a round-half-even tie:
      su, sv: x term = 1, y term = 0, both vertical fluxes = 2^53  ->  1 + (2^53 - 2^53) = 1
              ((1 + 2^53) - 2^53 would give 0);
      sw:     x term = 1, y term = 1, vertical term = 2^53 - 0     ->  (1 + 1) + 2^53 = 2^53 + 2
              (2^53 first, then + 1 + 1, would give 2^53)."""
    shape = (7, 7, 7)
    nz = shape[0]
    u, v, w = _field(shape), _field(shape), _field(shape)
    tz = [np.zeros(nz), np.zeros(nz), np.zeros(nz), np.zeros(nz)]
    i0 = j0 = k0 = 3
    if field == "su":
        # x: tcx*(u(i-1)*(u(i)+u(i-1)) - u(i+1)*(u(i)+u(i+1))) = 0.5*(1*2 - 0) = 1
        u[:, :, i0 - 1] = 1.0
        u[:, :, i0] = 1.0
        w[:] = 1.0                          # y: v = 0 -> 0
        tz[0][:] = tz[1][:] = 2.0 ** 52     # z: 2^52*u(k-1)*(1+1) = 2^52*u(k+1)*(1+1) = 2^53
        return (u, v, w), tz, 0.5, 0.5, 1.0
    if field == "sv":
        # x: tcx*(v(i-1)*(u(i-1)+u(j+1,i-1)) - v(i+1)*(u(i)+u(j+1,i))) = 0.5*(1*2 - 1*0) = 1
        u[:, :, i0 - 1] = 1.0
        v[:] = 1.0                          # y: tcy*(1*(1+1) - 1*(1+1)) = 0
        w[:] = 1.0
        tz[0][:] = tz[1][:] = 2.0 ** 52     # z: 2^52*1*2 - 2^52*1*2
        return (u, v, w), tz, 0.5, 0.5, 1.0
    # sw
    w[:] = 1.0
    u[:, :, i0 - 1] = 1.0                   # x: 0.5*(1*(1+1) - 1*(0+0)) = 1
    v[:, j0 - 1, :] = 1.0                   # y: 0.5*(1*(1+1) - 1*(0+0)) = 1
    tz[2][:] = 2.0 ** 52                    # z: 2^52*1*(1+1) - 0 = 2^53
    return (u, v, w), tz, 0.5, 0.5, 2.0 ** 53 + 2.0


@pytest.mark.parametrize("field", ["su", "sv", "sw"])
def test_statement_order_and_vertical_parenthesis(field):
    (u, v, w), tz, tcx, tcy, expected = _order_case(field)
    outs = _run(u, v, w, tz, tcx=tcx, tcy=tcy)
    got = outs["su sv sw".split().index(field)][3, 3, 3]
    assert got == expected, (field, got, expected)
