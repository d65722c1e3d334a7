"""GPU parity for pw-advection (R#26): the TMA-tiled kernel and the
generic strided kernel vs the oracle, bit-exact (one rounding per operation in Fortran order on
both sides), over shapes spanning several 64 x 16 tiles with ragged tails, sections, and the
full-size configuration on sampled points."""
import numpy as np
import pytest
import torch

import oracle
import synth
from oracle import FArray as OA

pytestmark = pytest.mark.gpu
TCX, TCY = 0.1, 0.2


@pytest.fixture(scope="module")
def ftn():
    from paper_2409_18824_b200 import ftn
    return ftn


def _coeffs(nz, seed=1):
    return [synth.values(nz, array_id=40 + q, mode=synth.U11) for q in range(4)]


def _fields(shape, seed=0):
    return [synth.farray(shape, array_id=seed + q, mode=synth.U11) for q in range(3)]


def _check(ftn, shape, lbs=None, fill=-3.0):
    u, v, w = _fields(shape, seed=sum(shape))
    z = _coeffs(shape[0])
    U, V, W = (ftn.FArray.from_numpy(a, lbs) for a in (u, v, w))
    outs = [ftn.FArray.from_numpy(np.full(shape, fill, order="F"), lbs) for _ in range(3)]
    Z = [ftn.FArray.from_numpy(c) for c in z]
    ftn.pw_advection(*outs, U, V, W, *Z, TCX, TCY)
    ref = [np.full(shape, fill, order="F") for _ in range(3)]
    oracle.pw_advection(*[OA(r) for r in ref], OA(u), OA(v), OA(w), *z, TCX, TCY)
    for o, r, name in zip(outs, ref, ("su", "sv", "sw")):
        np.testing.assert_array_equal(o.to_numpy(), r, err_msg=f"{name} {shape}")


@pytest.mark.parametrize("shape", [(3, 3, 3), (4, 5, 6), (66, 18, 5), (67, 19, 4), (130, 34, 9), (64, 16, 3),
                                   (200, 50, 12), (17, 100, 7), (129, 17, 33)])
def test_tma_path_vs_oracle(ftn, shape):
    _check(ftn, shape, lbs=[0, -2, 5])


def test_many_units(ftn):
    """More units than CTAs: several i-segments per tile column and tiles per CTA."""
    _check(ftn, (258, 70, 300))


def test_generic_path_sections(ftn):
    """Strided / reversed sections take the generic kernel; same bits as the oracle on the
    same sections."""
    shape = (40, 30, 20)
    big = _fields(shape, seed=7)
    sec = ((39, 2, -1), (1, 30, 2), (3, 18))
    ins = [ftn.FArray.from_numpy(b).section(*sec) for b in big]
    outs_host = [np.full(shape, 9.0, order="F") for _ in range(3)]
    outs = [ftn.FArray.from_numpy(o).section(*sec) for o in outs_host]
    nz = ins[0].shape[0]
    z = _coeffs(nz)
    ftn.pw_advection(*outs, *ins, *[ftn.FArray.from_numpy(c) for c in z], TCX, TCY)
    ref_host = [np.full(shape, 9.0, order="F") for _ in range(3)]
    ref = [OA(r).section(*sec) for r in ref_host]
    oracle.pw_advection(*ref, *[OA(b).section(*sec) for b in big], *z, TCX, TCY)
    for o, r in zip(outs, ref):
        np.testing.assert_array_equal(o.to_numpy(), r.to_numpy())


def test_errors(ftn):
    a = [ftn.FArray.empty((8, 8, 8)) for _ in range(6)]
    z = [ftn.FArray.empty((8,)) for _ in range(4)]
    with pytest.raises(ftn.FtnError):
        ftn.pw_advection(a[0], a[1], a[2], a[0], a[4], a[5], *z, 1.0, 1.0)     # output aliases input
    with pytest.raises(ftn.FtnError):
        ftn.pw_advection(a[0], a[1], a[2], a[3], a[4], ftn.FArray.empty((8, 8, 9)), *z, 1.0, 1.0)
    with pytest.raises(ftn.FtnError):
        ftn.pw_advection(*a, *z[:3], ftn.FArray.empty((7,)), 1.0, 1.0)


@pytest.mark.slow
def test_f4_full_size_sampled(ftn):
    """The bench configuration (2048 x 1024 x 1024, three fields): sampled output points are
    recomputed by the oracle on their 3x3x3 window, bit-exact."""
    nz, ny, nx = 2048, 1024, 1024
    F = [ftn.FArray.empty((nz, ny, nx)) for _ in range(3)]
    for q, f in enumerate(F):
        ftn.gen_fill(f, synth.SEED, 50 + q, ftn.GEN_U11)
    O = [ftn.FArray.empty((nz, ny, nx)) for _ in range(3)]
    z = _coeffs(nz)
    ftn.pw_advection(*O, *F, *[ftn.FArray.from_numpy(c) for c in z], TCX, TCY)
    rng = np.random.default_rng(3)
    pts = [(1, 1, 1), (nz - 2, ny - 2, nx - 2), (64, 16, 500), (65, 17, 1)] + \
          [tuple(int(rng.integers(1, n - 1)) for n in (nz, ny, nx)) for _ in range(12)]
    for (k, j, i) in pts:
        win = [np.asfortranarray(f.section((k, k + 2), (j, j + 2), (i, i + 2)).to_numpy()) for f in F]
        ref = [np.zeros((3, 3, 3), order="F") for _ in range(3)]
        zz = [c[k - 1:k + 2] for c in z]
        oracle.pw_advection(*[OA(r) for r in ref], *[OA(a) for a in win], *zz, TCX, TCY)
        for o, r in zip(O, ref):
            got = o.section((k + 1, k + 1), (j + 1, j + 1), (i + 1, i + 1)).to_numpy().ravel()[0]
            assert got == r[1, 1, 1], (k, j, i)


def test_random_shapes(ftn):
    """Fuzz: random shapes (tile remainders in k and j, short i), lower bounds, bit-exact."""
    rng = np.random.default_rng(18824)
    for it in range(12):
        shape = (int(rng.integers(3, 300)), int(rng.integers(3, 40)), int(rng.integers(3, 20)))
        _check(ftn, shape, lbs=[int(v) for v in rng.integers(-3, 4, 3)])
