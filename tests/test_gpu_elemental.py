"""GPU parity: element-wise expressions, assignment, fill and the generator vs the oracle
(bit-exact, R#5, R#6, R#9).  Calls go through the C ABI (ctypes binding)."""
import numpy as np
import pytest
import torch

import oracle
import synth
from oracle import FArray as OA

pytestmark = pytest.mark.gpu

TORCH = {np.float64: torch.float64, np.float32: torch.float32, np.int32: torch.int32, np.int64: torch.int64}


@pytest.fixture(scope="module")
def ftn():
    from paper_2409_18824_b200 import ftn
    return ftn


def _pair(ftn, a_host, lbounds=None):
    return ftn.FArray.from_numpy(a_host, lbounds), OA(a_host.copy(order="F"), lbounds)


def _random_section(rng, shape_parent):
    trip = []
    for n in shape_parent:
        st = int(rng.choice([-2, -1, 1, 2, 3]))
        cnt = int(rng.integers(1, (n - 1) // abs(st) + 2))
        if st > 0:
            lo = int(rng.integers(1, n - (cnt - 1) * st + 1))
            trip.append((lo, lo + (cnt - 1) * st, st))
        else:
            hi_first = int(rng.integers((cnt - 1) * (-st) + 1, n + 1))
            trip.append((hi_first, hi_first + (cnt - 1) * st, st))
    return trip


@pytest.mark.parametrize("mode", [synth.U01, synth.U11, synth.INT8, synth.LINEAR, synth.MOD1024])
def test_generator_matches_synth(ftn, mode):
    x = ftn.FArray.empty((37, 41, 3))
    ftn.gen_fill(x, synth.SEED, 5, mode)
    np.testing.assert_array_equal(x.to_numpy(), synth.farray((37, 41, 3), array_id=5, mode=mode))
    big = ftn.FArray.empty((1 << 20,))
    ftn.gen_fill(big, 7, 3, mode)
    np.testing.assert_array_equal(big.to_numpy(), synth.values(1 << 20, seed=7, array_id=3, mode=mode))
    # a slab of a larger array generated where it lives (ftn_gen_fill_at): sequence offset t0
    sl = ftn.FArray.empty((37, 41, 5))
    t0 = 37 * 41 * 11
    ftn.gen_fill(sl, synth.SEED, 5, mode, t0=t0)
    np.testing.assert_array_equal(sl.to_numpy(), synth.values(37 * 41 * 5, array_id=5, mode=mode, start=t0)
                                  .reshape((37, 41, 5), order="F"))


@pytest.mark.parametrize("dtype", [np.int32, np.int64])
def test_generator_integer_modes(ftn, dtype):
    for mode in (synth.RAW, synth.INT8, synth.LINEAR):
        x = ftn.FArray.empty((1000, 3), dtype=TORCH[dtype])
        ftn.gen_fill(x, synth.SEED, 9, mode)
        np.testing.assert_array_equal(x.to_numpy(), synth.farray((1000, 3), array_id=9, mode=mode, dtype=dtype))


def test_c1_muladd_and_aliasing(ftn):
    """BASELINE configs[0]: r = b*c + d with b = a(::2,:), c = a(1::2,:), d = e(-5:26,10:57)."""
    a = synth.farray((64, 48), mode=synth.U11, array_id=1)
    e = synth.farray((32, 48), mode=synth.U11, array_id=2)
    A, Ao = _pair(ftn, a, [0, 1])
    E, Eo = _pair(ftn, e, [-5, 10])
    for contract in (False, True):
        r, ro = ftn.FArray.empty((32, 48)), OA(np.zeros((32, 48), order="F"))
        ftn.muladd(r, A.section((0, 63, 2), (1, 48)), A.section((1, 63, 2), (1, 48)), E, contract=contract)
        oracle.elemental(oracle.MULADD, ro, Ao.section((0, 63, 2), (1, 48, 1)), Ao.section((1, 63, 2), (1, 48, 1)),
                         Eo, contract)
        np.testing.assert_array_equal(r.to_numpy(), ro.arr)
    # a(::2,:) = a(::2,:)*c + d  (identical mapping: in place)
    ftn.muladd(A.section((0, 63, 2), (1, 48)), A.section((0, 63, 2), (1, 48)), A.section((1, 63, 2), (1, 48)), E)
    oracle.elemental(oracle.MULADD, Ao.section((0, 63, 2), (1, 48, 1)), Ao.section((0, 63, 2), (1, 48, 1)),
                     Ao.section((1, 63, 2), (1, 48, 1)), Eo)
    np.testing.assert_array_equal(A.to_numpy(), Ao.arr)
    # a(2:63,:) = a(1:62,:)*2 + 0  (overlap: RHS first through a temporary)
    ftn.muladd(A.section((2, 63), (1, 48)), A.section((1, 62), (1, 48)), 2.0, 0.0)
    oracle.elemental(oracle.MULADD, Ao.section((2, 63, 1), (1, 48, 1)), Ao.section((1, 62, 1), (1, 48, 1)),
                     OA(np.array(2.0)), OA(np.array(0.0)))
    np.testing.assert_array_equal(A.to_numpy(), Ao.arr)


@pytest.mark.parametrize("seed", range(12))
def test_random_sections_all_ops(ftn, seed):
    rng = np.random.default_rng(100 + seed)
    dtype = [np.float64, np.float32, np.int32, np.int64][seed % 4]
    r = 1 + seed % 3
    pshape = tuple(int(rng.integers(3, 40)) for _ in range(r))
    mode = synth.U11 if np.dtype(dtype).kind == "f" else synth.RAW
    ops = []
    for k in range(3):
        trip = _random_section(rng, pshape)
        ops.append(trip)
    # make the three sections conformable: same counts per dim
    counts = [min(len(range(t[0], t[1] + (1 if t[2] > 0 else -1), t[2])) for t in col) for col in zip(*ops)]
    fixed = []
    for trip in ops:
        fixed.append([(t[0], t[0] + (c - 1) * t[2], t[2]) for t, c in zip(trip, counts)])
    arrs = [synth.farray(pshape, array_id=10 + k, mode=mode, dtype=dtype) for k in range(3)]
    lbs = [[int(v) for v in rng.integers(-3, 4, size=r)] for _ in range(3)]
    G = [ftn.FArray.from_numpy(a, lb) for a, lb in zip(arrs, lbs)]
    O = [OA(a.copy(order="F"), lb) for a, lb in zip(arrs, lbs)]
    gsec = [g.section(*[(t[0] + lb[d] - 1, t[1] + lb[d] - 1, t[2]) for d, t in enumerate(tr)])
            for g, tr, lb in zip(G, fixed, lbs)]
    osec = [o.section(*[(t[0] + lb[d] - 1, t[1] + lb[d] - 1, t[2]) for d, t in enumerate(tr)])
            for o, tr, lb in zip(O, fixed, lbs)]
    shape = tuple(counts)
    for op in (oracle.ADD, oracle.SUB, oracle.MUL, oracle.MULADD) + ((oracle.DIV,) if np.dtype(dtype).kind == "f" else ()):
        dst = ftn.FArray.empty(shape, dtype=TORCH[dtype], lbounds=[2] * r)
        do = OA(np.zeros(shape, dtype=dtype, order="F"), [2] * r)
        ftn.elemental(op, dst, gsec[0], gsec[1], gsec[2])
        oracle.elemental(op, do, osec[0], osec[1], osec[2])
        np.testing.assert_array_equal(dst.to_numpy(), do.arr, err_msg=f"op {op} dtype {dtype} shape {shape}")
    # assignment into a strided destination section of a fresh array
    ftn.assign(gsec[0], gsec[1])
    oracle.assign(osec[0], osec[1])
    np.testing.assert_array_equal(G[0].to_numpy(), O[0].arr)


@pytest.mark.parametrize("n", [0, 1, 3, 4, 5, 1023, 2047, 2048, 2049, 4096 + 3, 100001])
def test_ragged_lengths_vector_path(ftn, n):
    b, c, d = (synth.values(n, array_id=k, mode=synth.U11) for k in range(3))
    B, C, D = (ftn.FArray.from_numpy(v) for v in (b, c, d))
    r = ftn.FArray.empty((n,))
    ftn.muladd(r, B, C, D)
    np.testing.assert_array_equal(r.to_numpy(), np.add(np.multiply(b, c), d))


def test_rank3_lbounds_and_section_variant(ftn):
    """C4 shapes scaled down: x(-7:8, 0:15, 1:16) whole arrays and p(:,:,1:32:2) sections."""
    shape = (16, 16, 16)
    lbs = [-7, 0, 1]
    b, c, d = (synth.farray(shape, array_id=k, mode=synth.U01) for k in range(3))
    G = [ftn.FArray.from_numpy(v, lbs) for v in (b, c, d)]
    r = ftn.FArray.empty(shape, lbounds=lbs)
    ftn.muladd(r, *G)
    np.testing.assert_array_equal(r.to_numpy(), np.add(np.multiply(b, c), d))
    parents = [synth.farray((16, 16, 32), array_id=20 + k, mode=synth.U01) for k in range(4)]
    P = [ftn.FArray.from_numpy(v) for v in parents]
    S = [p.section((1, 16), (1, 16), (1, 32, 2)) for p in P]
    ftn.muladd(S[3], S[0], S[1], S[2])
    ref = parents[3].copy(order="F")
    ref[:, :, ::2] = np.add(np.multiply(parents[0][:, :, ::2], parents[1][:, :, ::2]), parents[2][:, :, ::2])
    np.testing.assert_array_equal(P[3].to_numpy(), ref)
    # dim-1 strided variant (0:2n-1:2, :, :)
    Q = ftn.FArray.from_numpy(synth.farray((32, 16, 16), array_id=30, mode=synth.U01))
    qo = synth.farray((32, 16, 16), array_id=30, mode=synth.U01)
    out = ftn.FArray.empty((16, 16, 16))
    ftn.elemental(ftn.ADD, out, Q.section((1, 31, 2), (1, 16), (1, 16)), 1.5)
    np.testing.assert_array_equal(out.to_numpy(), qo[::2] + 1.5)


def test_fill_and_reversal(ftn):
    x = ftn.FArray.empty((7, 5))
    ftn.fill(x, -2.25)
    assert (x.to_numpy() == -2.25).all()
    v = synth.values(1001, mode=synth.LINEAR)
    V = ftn.FArray.from_numpy(v)
    ftn.assign(V, V.section((1001, 1, -1)))                       # x = x(n:1:-1)
    np.testing.assert_array_equal(V.to_numpy(), v[::-1])
    iv = ftn.FArray.empty((9,), dtype=torch.int32)
    ftn.fill(iv, 7)
    assert (iv.to_numpy() == 7).all()


def test_errors_launch_nothing(ftn):
    a = ftn.FArray.empty((4, 5))
    b = ftn.FArray.empty((5, 4))
    with pytest.raises(ftn.FtnError) as e:
        ftn.assign(a, b)
    assert e.value.name == "FTN_ERR_SHAPE"
    with pytest.raises(ftn.FtnError) as e:
        a.section((0, 4), (1, 5))
    assert e.value.name == "FTN_ERR_BOUNDS"
    with pytest.raises(ftn.FtnError) as e:
        ftn.assign(a, ftn.FArray.empty((4, 5), dtype=torch.float32))
    assert e.value.name == "FTN_ERR_TYPE"


def test_interleaved_disjoint_sections_need_no_temporary(ftn):
    """a(2::2,:) = a(1::2,:)*2 + 1 (even leading extent): the sections interleave but share no
    element, so the alias test (ftn_desc_may_overlap) lets the kernel write in place -- one
    launch, no temporary -- and the result equals the oracle's.  With an odd leading extent the
    test cannot prove it and the temporary path runs; the result is the same either way."""
    for lead, launches in ((64, 1), (63, None)):
        a = synth.farray((lead, 9), mode=synth.U11, array_id=11)
        A, Ao = _pair(ftn, a)
        hi = lead - (lead % 2 == 1)
        dst, src = A.section((2, hi, 2), (1, 9)), A.section((1, hi - 1, 2), (1, 9))
        torch.cuda.synchronize()
        n0 = ftn.launch_count()
        ftn.muladd(dst, src, 2.0, 1.0)
        torch.cuda.synchronize()
        if launches is not None:
            assert ftn.launch_count() - n0 == launches
        oracle.elemental(oracle.MULADD, Ao.section((2, hi, 2), (1, 9, 1)), Ao.section((1, hi - 1, 2), (1, 9, 1)),
                         OA(np.array(2.0)), OA(np.array(1.0)))
        np.testing.assert_array_equal(A.to_numpy(), Ao.arr)
