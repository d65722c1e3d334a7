"""Pins for the oracle's element-wise expressions and assignment (R#5, R#6, R#9).

Independent references: numpy ufuncs (np.multiply then np.add: two roundings, no
contraction; numpy guarantees no-overlap semantics for overlapping operands),
hand-computed fma cases, integer-valued exactness, identities.
"""
import numpy as np
import pytest

import oracle
import synth
from oracle import FArray


def _sec_pair(rng, shape, dtype=np.float64, mode=synth.U11, array_id=0):
    """A parent with random lbounds and a random strided (possibly reversed) section of it."""
    parent = synth.farray(tuple(s * 2 + 1 for s in shape), seed=int(rng.integers(1 << 30)),
                          array_id=array_id, mode=mode, dtype=dtype)
    lbs = [int(rng.integers(-4, 5)) for _ in shape]
    P = FArray(parent, lbs)
    trip, sl = [], []
    for d, n in enumerate(shape):
        st = int(rng.choice([-2, -1, 1, 2]))
        if st > 0:
            lo = lbs[d] + int(rng.integers(0, parent.shape[d] - (n - 1) * st))
            trip.append((lo, lo + (n - 1) * st, st))
        else:
            lo = lbs[d] + (n - 1) * (-st) + int(rng.integers(0, parent.shape[d] - (n - 1) * (-st)))
            trip.append((lo, lo + (n - 1) * st, st))
    S = P.section(*trip)
    return S


@pytest.mark.parametrize("seed", range(8))
def test_muladd_vs_numpy(orc, seed):
    rng = np.random.default_rng(seed)
    shape = (7, 5, 3)[: int(rng.integers(1, 4))]
    b, c, d = (_sec_pair(rng, shape, array_id=i) for i in range(3))
    dst = FArray(np.zeros(shape, order="F"), [3] * len(shape))
    orc.elemental(orc.MULADD, dst, b, c, d)
    ref = np.add(np.multiply(b.to_numpy(), c.to_numpy()), d.to_numpy())
    np.testing.assert_array_equal(dst.arr, ref)


@pytest.mark.parametrize("op,fn", [(oracle.ADD, np.add), (oracle.SUB, np.subtract),
                                   (oracle.MUL, np.multiply), (oracle.DIV, np.divide)])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_binary_ops_vs_numpy(orc, op, fn, dtype):
    rng = np.random.default_rng(op)
    a = _sec_pair(rng, (9, 4), dtype=dtype, array_id=1)
    b = _sec_pair(rng, (9, 4), dtype=dtype, array_id=2)
    dst = FArray(np.zeros((9, 4), dtype=dtype, order="F"))
    orc.elemental(op, dst, a, b)
    np.testing.assert_array_equal(dst.arr, fn(a.to_numpy(), b.to_numpy()))


@pytest.mark.parametrize("dtype", [np.int32, np.int64])
def test_integer_wraparound_vs_numpy(orc, dtype):
    """integer arithmetic wraps modulo 2^w (numpy integer ufuncs wrap too)."""
    rng = np.random.default_rng(3)
    a = _sec_pair(rng, (11, 3), dtype=dtype, mode=synth.RAW, array_id=4)
    b = _sec_pair(rng, (11, 3), dtype=dtype, mode=synth.RAW, array_id=5)
    c = _sec_pair(rng, (11, 3), dtype=dtype, mode=synth.RAW, array_id=6)
    dst = FArray(np.zeros((11, 3), dtype=dtype, order="F"))
    with np.errstate(over="ignore"):
        for op, fn in ((oracle.ADD, np.add), (oracle.SUB, np.subtract), (oracle.MUL, np.multiply)):
            orc.elemental(op, dst, a, b)
            np.testing.assert_array_equal(dst.arr, fn(a.to_numpy(), b.to_numpy()))
        orc.elemental(oracle.MULADD, dst, a, b, c)
        np.testing.assert_array_equal(dst.arr, a.to_numpy() * b.to_numpy() + c.to_numpy())


def test_integer_division_truncates(orc):
    a = FArray(np.array([7, -7, 7, -7, 0], dtype=np.int32))
    b = FArray(np.array([2, 2, -2, -2, 5], dtype=np.int32))
    dst = FArray(np.zeros(5, dtype=np.int32))
    orc.elemental(oracle.DIV, dst, a, b)
    assert list(dst.arr) == [3, -3, -3, 3, 0]   # Fortran: truncation toward zero


def test_contraction_hand_case(orc):
    """R#6: b = 1+2^-52, c = 1-2^-52, d = -1: b*c = 1 - 2^-104 rounds to 1, so the unfused
    result is 0 while the single-rounding fma keeps -2^-104."""
    b = FArray(np.array([1 + 2.0 ** -52]))
    c = FArray(np.array([1 - 2.0 ** -52]))
    d = FArray(np.array([-1.0]))
    dst = FArray(np.zeros(1))
    orc.elemental(oracle.MULADD, dst, b, c, d, contract=False)
    assert dst.arr[0] == 0.0
    orc.elemental(oracle.MULADD, dst, b, c, d, contract=True)
    assert dst.arr[0] == -(2.0 ** -104)


def test_contraction_agrees_on_integer_valued(orc):
    """b*c exact for small integers, so fused and unfused agree bit for bit."""
    b, c, d = (FArray(synth.farray((13, 6), array_id=i, mode=synth.INT8)) for i in range(3))
    r1 = FArray(np.zeros((13, 6), order="F"))
    r2 = FArray(np.zeros((13, 6), order="F"))
    orc.elemental(oracle.MULADD, r1, b, c, d, contract=False)
    orc.elemental(oracle.MULADD, r2, b, c, d, contract=True)
    np.testing.assert_array_equal(r1.arr, r2.arr)
    np.testing.assert_array_equal(r1.arr, b.arr * c.arr + d.arr)


def test_identity_expression(orc):
    x = FArray(synth.farray((17, 3), mode=synth.U11))
    one = FArray(np.array(1.0))
    zero = FArray(np.array(0.0))
    r = FArray(np.zeros((17, 3), order="F"))
    orc.elemental(oracle.MULADD, r, x, one, zero)
    np.testing.assert_array_equal(r.arr, x.arr)


def test_overlapping_assignment_uses_rhs_first(orc):
    """C1 aliasing case a(2:63,:) = a(1:62,:)*2 + 0: the RHS is evaluated before the store
    (numpy ufuncs buffer overlapping operands, giving the same semantics)."""
    a = synth.farray((64, 48), mode=synth.LINEAR)
    ref = a.copy(order="F")
    A = FArray(a, [0, 1])
    two = FArray(np.array(2.0))
    zero = FArray(np.array(0.0))
    orc.elemental(oracle.MULADD, A.section((2, 63, 1), (1, 48, 1)), A.section((1, 62, 1), (1, 48, 1)), two, zero)
    ref[2:64, :] = np.add(np.multiply(ref[1:63, :], 2.0), 0.0)
    np.testing.assert_array_equal(a, ref)


def test_reversal_assignment(orc):
    """x(1:n) = x(n:1:-1): every element overlaps another; Fortran gives the reversal."""
    x = synth.farray((37,), mode=synth.LINEAR)
    X = FArray(x)
    orc.assign(X, X.section((37, 1, -1)))
    np.testing.assert_array_equal(x, np.arange(36, -1, -1, dtype=np.float64))


def test_identical_mapping_in_place(orc):
    """C1 aliasing case a(::2,:) = a(::2,:)*c + d (identical mapping)."""
    a = synth.farray((64, 48), mode=synth.U11, array_id=1)
    e = synth.farray((32, 48), mode=synth.U11, array_id=2)
    A = FArray(a, [0, 1])
    s = A.section((0, 63, 2), (1, 48, 1))
    c = A.section((1, 63, 2), (1, 48, 1))
    d = FArray(e, [-5, 10])
    ref = np.add(np.multiply(a[::2], a[1::2]), e)
    orc.elemental(oracle.MULADD, s, s, c, d)
    np.testing.assert_array_equal(a[::2], ref)


def test_fill_and_shape_errors(orc):
    x = FArray(np.zeros((4, 5), order="F"))
    orc.assign(x, FArray(np.array(2.5)))
    assert (x.arr == 2.5).all()
    with pytest.raises(oracle.OracleError) as e:
        orc.assign(x, FArray(np.zeros((5, 4), order="F")))
    assert e.value.code == 4
    with pytest.raises(oracle.OracleError) as e:
        orc.assign(x, FArray(np.zeros((4, 5), dtype=np.float32, order="F")))
    assert e.value.code == 3
