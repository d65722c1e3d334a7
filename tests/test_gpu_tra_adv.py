"""GPU parity for tra-adv (R#28): ftn_tra_adv against the oracle's
DO nests, bit for bit, on ragged shapes, several iteration counts, strided sections, and
sampled points of the bench configuration (1024 x 512 x 512, 20 iterations) recomputed by the
oracle on their dependence windows."""
import numpy as np
import pytest

import oracle
import synth
from oracle import FArray as OA

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ftn():
    from paper_2409_18824_b200 import ftn
    return ftn


def _inputs(shape, seed_base=0):
    ni, nj, nk = shape
    f3 = [synth.farray(shape, array_id=70 + seed_base + q, mode=synth.U11) for q in range(5)]   # md tsn pun pvn pwn
    m3 = [synth.farray(shape, array_id=80 + seed_base + q, mode=synth.U01) for q in range(3)]   # umask vmask tmask
    f2 = [synth.farray((ni, nj), array_id=90 + seed_base + q, mode=synth.U01) for q in range(3)]
    f2[0] = f2[0] - 1.0     # ztfreez in [-1, 0): some tsn <= ztfreez + 0.1, some not
    rz = synth.values(nk, array_id=95 + seed_base, mode=synth.U01)
    return f3, m3, f2, rz


def _oracle(f3, m3, f2, rz, iters):
    md = f3[0].copy(order="F")
    oracle.tra_adv(OA(md), OA(f3[1]), OA(f3[2]), OA(f3[3]), OA(f3[4]), OA(m3[0]), OA(m3[1]), OA(m3[2]),
                   OA(np.asfortranarray(f2[0])), OA(np.asfortranarray(f2[1])), OA(np.asfortranarray(f2[2])), rz, iters)
    return md


def _gpu(ftn, f3, m3, f2, rz, iters):
    d3 = [ftn.FArray.from_numpy(a) for a in f3 + m3]
    d2 = [ftn.FArray.from_numpy(np.asfortranarray(a)) for a in f2]
    ftn.tra_adv(*d3, *d2, ftn.FArray.from_numpy(rz), iters)
    return d3[0].to_numpy()


@pytest.mark.parametrize("shape", [(5, 4, 3), (3, 3, 3), (37, 29, 11), (64, 33, 17), (130, 20, 9), (257, 6, 5)])
@pytest.mark.parametrize("iters", [1, 2, 3])
def test_tra_adv_vs_oracle(ftn, shape, iters):
    f3, m3, f2, rz = _inputs(shape, seed_base=sum(shape) % 7)
    np.testing.assert_array_equal(_gpu(ftn, f3, m3, f2, rz, iters), _oracle(f3, m3, f2, rz, iters))


def test_tra_adv_sections(ftn):
    """Every field a strided / reversed section of a larger parent (generic addressing)."""
    shape = (40, 21, 9)
    f3, m3, f2, rz = _inputs(shape, seed_base=3)
    big = [np.full((2 * shape[0] + 1, shape[1] + 2, shape[2]), 9.0, order="F") for _ in range(8)]
    d3 = []
    for b, a in zip(big, f3 + m3):
        b[1::2][:shape[0], 1:shape[1] + 1, ::-1] = a
        B = ftn.FArray.from_numpy(b)
        d3.append((B, B.section((2, 2 * shape[0], 2), (2, shape[1] + 1), (shape[2], 1, -1))))
    d2 = [ftn.FArray.from_numpy(np.asfortranarray(a)) for a in f2]
    ftn.tra_adv(*[s for _, s in d3], *d2, ftn.FArray.from_numpy(rz), 2)
    np.testing.assert_array_equal(d3[0][1].to_numpy(), _oracle(f3, m3, f2, rz, 2))
    for (B, _), b in zip(d3[1:], big[1:]):        # inputs untouched, parents' gaps untouched
        np.testing.assert_array_equal(B.to_numpy(), b)


def test_tra_adv_errors(ftn):
    shape = (10, 8, 6)
    f3, m3, f2, rz = _inputs(shape)
    d3 = [ftn.FArray.from_numpy(a) for a in f3 + m3]
    d2 = [ftn.FArray.from_numpy(np.asfortranarray(a)) for a in f2]
    R = ftn.FArray.from_numpy(rz)
    with pytest.raises(ftn.FtnError):             # md overlapping an input
        ftn.tra_adv(d3[0], d3[0], *d3[2:], *d2, R, 1)
    with pytest.raises(ftn.FtnError):             # rnfmsk_z of the wrong extent
        ftn.tra_adv(*d3, *d2, ftn.FArray.from_numpy(rz[:-1].copy()), 1)
    with pytest.raises(ftn.FtnError):             # negative iteration count
        ftn.tra_adv(*d3, *d2, R, -1)
    np.testing.assert_array_equal(d3[0].to_numpy(), f3[0])


@pytest.mark.slow
def test_tra_adv_bench_configuration_sampled(ftn):
    """The bench's configuration (1024 x 512 x 512, 20 iterations, same generator): sampled points
    recomputed by the oracle on a window of radius 3 * 20 + 2 around them (a point depends on
    md within 2 cells in ji / jj and 3 in jk per iteration), bit-exact."""
    shape, iters = (1024, 512, 512), 20
    ni, nj, nk = shape
    D = [ftn.FArray.empty(shape) for _ in range(8)]
    for q, d in enumerate(D[:5]):
        ftn.gen_fill(d, synth.SEED, 70 + q, ftn.GEN_U11)
    for q, d in enumerate(D[5:]):
        ftn.gen_fill(d, synth.SEED, 80 + q, ftn.GEN_U01)
    D2 = [ftn.FArray.empty((ni, nj)) for _ in range(3)]
    for q, d in enumerate(D2):
        ftn.gen_fill(d, synth.SEED, 90 + q, ftn.GEN_U01)
    RZ = ftn.FArray.empty((nk,))
    ftn.gen_fill(RZ, synth.SEED, 95, ftn.GEN_U01)
    host3 = [d.to_numpy() for d in D]
    host2 = [d.to_numpy() for d in D2]
    rz = RZ.to_numpy()
    ftn.tra_adv(*D, *D2, RZ, iters)
    got = D[0].to_numpy()
    R = 3 * iters + 2
    rng = np.random.default_rng(9)
    pts = [(1, 1, 0), (ni - 2, nj - 2, nk - 2), (500, 1, 255), (3, 300, nk - 1), (1023, 200, 100)] + \
          [tuple(int(rng.integers(0, e)) for e in shape) for _ in range(4)]
    for p in pts:
        lo = [max(0, c - R) for c in p]
        hi = [min(e, c + R + 1) for c, e in zip(p, shape)]
        sl = tuple(slice(a, b) for a, b in zip(lo, hi))
        w3 = [np.asfortranarray(h[sl]) for h in host3]
        w2 = [np.asfortranarray(h[sl[:2]]) for h in host2]
        ref = _oracle(w3[:5], w3[5:], w2, np.ascontiguousarray(rz[sl[2]]), iters)
        assert got[p] == ref[tuple(c - l for c, l in zip(p, lo))], p
