"""Pins for the oracle's reductions: SUM (sequential fold, exact, order R), MAXVAL/MINVAL,
integer SUM, DOT_PRODUCT (R#7-R#12, section 4.2).

Independent references: math.fsum (Shewchuk, correctly rounded), fractions.Fraction
(exact rationals, float() rounds correctly), np.cumsum (a sequential fold), numpy
max/min/fmax, closed forms, and hand-worked order-R examples whose value depends
on the exact pairing the order prescribes.
"""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synth
from oracle import FArray

U = 2.0 ** -53
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _wide(n, seed):
    """Random values over a wide dynamic range, mixed signs, with cancellation."""
    rng = np.random.default_rng(seed)
    v = rng.standard_normal(n) * np.exp2(rng.integers(-60, 61, size=n))
    k = n // 4
    v[:k] = -v[k:2 * k] * (1 + 2.0 ** -40)  # near-cancelling pairs
    return v


@pytest.mark.parametrize("seed", range(6))
def test_exact_sum_vs_fsum(orc, seed):
    v = _wide(5000 + seed * 777, seed)
    assert orc.sum_exact(FArray(v)) == math.fsum(v)
    assert orc.fsum(v) == math.fsum(v)


def test_exact_sum_special_ranges(orc):
    tiny = np.array([5e-324, 5e-324, -1e-310, 2.2250738585072014e-308, 3e-320])
    assert orc.sum_exact(FArray(tiny)) == math.fsum(tiny)
    big = np.array([1e300, -1e300, 1e-300, 3.5, 1e300, 2.0 ** 1000])
    assert orc.sum_exact(FArray(big)) == math.fsum(big)
    ties = np.array([1.0, U, U * U])          # 1 + 2^-53 + 2^-106: above the tie -> rounds up
    assert orc.sum_exact(FArray(ties)) == 1.0 + 2 * U == math.fsum(ties)
    tie = np.array([1.0, U])                  # exact tie -> even (1.0)
    assert orc.sum_exact(FArray(tie)) == 1.0
    odd = np.array([1.0 + 2 * U, U])          # tie with odd last bit -> up
    assert orc.sum_exact(FArray(odd)) == 1.0 + 4 * U
    assert orc.sum_exact(FArray(np.array([-1.0, -U]))) == -1.0
    assert orc.sum_exact(FArray(np.zeros(0))) == 0.0


def test_exact_sum_vs_fraction(orc):
    rng = np.random.default_rng(11)
    for _ in range(30):
        v = rng.standard_normal(40) * np.exp2(rng.integers(-30, 30, size=40))
        exact = float(sum((Fraction(x) for x in v), Fraction(0)))
        assert orc.sum_exact(FArray(v)) == exact
        assert orc.sum_abs(FArray(v)) == float(sum((abs(Fraction(x)) for x in v), Fraction(0)))


def test_sequential_fold_vs_cumsum(orc):
    """P:243's linalg.reduce loop is a left fold: np.cumsum is one too."""
    v = _wide(20001, 3)
    assert orc.sum_seq(FArray(v)) == np.cumsum(v)[-1]
    a = np.asfortranarray(_wide(35 * 21, 4).reshape(35, 21, order="F"))
    sec = FArray(a, [0, -3]).section((33, 1, -2), (-3, 17, 3))
    assert orc.sum_seq(sec) == np.cumsum(sec.to_numpy().ravel(order="F"))[-1]


def test_closed_forms(orc):
    n = 1 << 24
    x = FArray(synth.values(n, mode=synth.MOD1024))
    s_closed = (n // 1024) * (1023 * 1024 // 2)
    for s in (orc.sum_seq(x), orc.sum_exact(x), orc.reduce_orderR(x, oracle.SUM)):
        assert s == s_closed
    d_closed = (n // 1024) * (1023 * 1024 * 2047 // 6)
    assert orc.dot_orderR(x, x) == d_closed
    assert orc.dot_exact(x, x)[0] == d_closed
    lin = FArray(synth.values(1 << 20, mode=synth.LINEAR))          # t = 0..n-1
    m = 1 << 20
    assert orc.reduce_orderR(lin, oracle.SUM) == m * (m - 1) // 2 == orc.sum_seq(lin)


def test_c1_closed_forms_derivation(orc):
    g = json.load(open(os.path.join(GOLDEN, "c1_closed_forms.json")))
    # independent derivation of the closed forms with integer arithmetic
    vals = [i + 64 * (j - 1) for j in range(1, 49) for i in range(0, 64, 2)]
    assert sum(vals) == g["SUM(s)"] and max(vals) == g["MAXVAL(s)"] and min(vals) == g["MINVAL(s)"]
    a = synth.farray((64, 48), mode=synth.LINEAR)
    s = FArray(a, [0, 1]).section((0, 63, 2), (1, 48, 1))
    assert orc.sum_seq(s) == orc.sum_exact(s) == orc.reduce_orderR(s, oracle.SUM) == g["SUM(s)"]
    assert orc.maxval(s) == g["MAXVAL(s)"] and orc.minval(s) == g["MINVAL(s)"]


# ---- order R: hand-worked cases ------------------------------------------

def _orderR_of(n, entries):
    v = np.zeros(n)
    for k, val in entries.items():
        v[k] = val
    return oracle.reduce_orderR(FArray(v), oracle.SUM), np.cumsum(v)[-1]


def test_orderR_group_of_four(orc):
    # thread 0 holds x0..x3 in acc_0..acc_3 -> (x0 + x1) + (x2 + x3) = 1 + 2^-52;
    # the sequential fold gives 1 (both 2^-53 additions tie to even).
    r, seq = _orderR_of(4, {0: 1.0, 2: U, 3: U})
    assert r == 1.0 + 2 * U and seq == 1.0


def test_orderR_m_ascending(orc):
    # acc_0 of thread 0 adds x0, x1024, x2048 in that order: (1 + u) + u = 1
    r, _ = _orderR_of(2049, {0: 1.0, 1024: U, 2048: U})
    assert r == 1.0


def test_orderR_butterfly(orc):
    # lanes 0 and 16 (x0, x64) combine first (mask 16) -> 2^-52, then lane 1 (x4 = 1) at mask 1
    r, seq = _orderR_of(68, {0: U, 4: 1.0, 64: U})
    assert r == 1.0 + 2 * U and seq == 1.0


def test_orderR_warp_combine(orc):
    # warps 0, 4, 6 (x0, x512, x768): ((w0+w1)+(w2+w3)) + ((w4+w5)+(w6+w7)) = 1 + 2^-52
    r, seq = _orderR_of(769, {0: 1.0, 512: U, 768: U})
    assert r == 1.0 + 2 * U and seq == 1.0


def test_orderR_chunk_tree(orc):
    # chunk partials 1, 0, u, u -> (1 + 0) + (u + u) = 1 + 2^-52
    r, seq = _orderR_of(3 * 65536 + 1, {0: 1.0, 2 * 65536: U, 3 * 65536: U})
    assert r == 1.0 + 2 * U and seq == 1.0
    # three partials padded with +0: (1 + u) + (u + 0) = 1
    r, _ = _orderR_of(2 * 65536 + 1, {0: 1.0, 65536: U, 2 * 65536: U})
    assert r == 1.0


def test_tree_combine_small(orc):
    assert orc.tree_combine([]) == 0.0
    assert orc.tree_combine([3.5]) == 3.5
    assert orc.tree_combine([1.0, U, U]) == 1.0                 # (1+u) + (u+0)
    assert orc.tree_combine([U, U, 1.0]) == 1.0 + 2 * U         # (u+u) + (1+0)
    assert orc.tree_combine([1.0, -5.0, 7.0], oracle.MAX) == 7.0
    assert orc.tree_combine([], oracle.MIN) == math.inf


def test_orderR_edges(orc):
    assert orc.reduce_orderR(FArray(np.zeros(0)), oracle.SUM) == 0.0
    assert orc.reduce_orderR(FArray(np.array([-2.5])), oracle.SUM) == -2.5
    neg0 = orc.reduce_orderR(FArray(np.array([-0.0, -0.0])), oracle.SUM)
    assert neg0 == 0.0 and math.copysign(1, neg0) == 1.0            # +0 initialised output


@pytest.mark.parametrize("n", [1, 5, 1023, 1025, 65535, 65536, 65537, 3 * 65536 + 17, 300001])
def test_orderR_within_bound(orc, n):
    """R#8: |R - exact| <= 4 n 2^-53 sum|x| (any order is within gamma_n)."""
    v = _wide(n, n)
    x = FArray(v)
    r = orc.reduce_orderR(x, oracle.SUM)
    exact = math.fsum(v)
    bound = 4 * n * U * orc.sum_abs(x)
    assert abs(r - exact) <= bound
    iv = FArray(np.rint(v % 1000.0))                                 # integer-valued: exact in any order
    assert orc.reduce_orderR(iv, oracle.SUM) == math.fsum(iv.arr)


@pytest.mark.parametrize("n", [0, 1, 7, 1024, 65537, 200003])
def test_orderR_maxmin_vs_numpy(orc, n):
    v = _wide(max(n, 1), n + 1)[:n]
    x = FArray(v)
    assert orc.reduce_orderR(x, oracle.MAX) == (v.max() if n else -math.inf)
    assert orc.reduce_orderR(x, oracle.MIN) == (v.min() if n else math.inf)


# ---- MAXVAL / MINVAL -----------------------------------------------------------------------

@pytest.mark.parametrize("pos", [0, 65535, 65536, 131071, 150000, 150001 - 1])
def test_maxval_minval_planted(orc, pos):
    n = 150001
    v = synth.values(n, mode=synth.U11)
    v[pos] = 7.0
    x = FArray(v)
    assert orc.maxval(x) == 7.0 == v.max()
    v[pos] = -7.0
    assert orc.minval(x) == -7.0 == v.min()


def test_maxval_empty_nan_and_int(orc):
    assert orc.maxval(FArray(np.zeros(0))) == -math.inf
    assert orc.minval(FArray(np.zeros(0))) == math.inf
    assert orc.maxval(FArray(np.zeros(0, dtype=np.int32))) == np.iinfo(np.int32).min
    assert orc.minval(FArray(np.zeros(0, dtype=np.int64))) == np.iinfo(np.int64).max
    v = np.array([np.nan, 1.0, np.nan, -3.0, 2.0])
    assert orc.maxval(FArray(v)) == np.fmax.reduce(v) == 2.0
    assert orc.minval(FArray(v)) == np.fmin.reduce(v) == -3.0
    assert math.isnan(orc.maxval(FArray(np.array([np.nan, np.nan]))))
    iv = synth.farray((33, 7), mode=synth.RAW, dtype=np.int64)
    assert orc.maxval(FArray(iv)) == iv.max() and orc.minval(FArray(iv)) == iv.min()


@pytest.mark.parametrize("dtype", [np.int32, np.int64])
def test_integer_sum_wraps(orc, dtype):
    iv = synth.farray((129, 65), mode=synth.RAW, dtype=dtype)
    sec = FArray(iv, [-1, 2]).section((127, -1, -3), (2, 66, 2))
    with np.errstate(over="ignore"):
        assert orc.sum_int(sec) == np.sum(sec.to_numpy(), dtype=dtype)


# ---- DOT_PRODUCT ---------------------------------------------------------------------------

def test_dot_products_vs_numpy(orc):
    x = synth.values(1000, array_id=1, mode=synth.U11)
    y = synth.values(2000, array_id=2, mode=synth.U11)
    X, Y = FArray(x), FArray(y).section((2000, 1, -2))
    np.testing.assert_array_equal(orc.dot_products(X, Y), np.multiply(x, y[::-2]))


def test_dot_exact_vs_fraction(orc):
    rng = np.random.default_rng(5)
    for _ in range(20):
        x = rng.standard_normal(64) * np.exp2(rng.integers(-20, 20, size=64))
        y = rng.standard_normal(64)
        exact = float(sum((Fraction(a) * Fraction(b) for a, b in zip(x, y)), Fraction(0)))
        absum = float(sum((abs(Fraction(a) * Fraction(b)) for a, b in zip(x, y)), Fraction(0)))
        e, a = orc.dot_exact(FArray(x), FArray(y))
        assert e == exact and a == absum


@pytest.mark.parametrize("n", [3, 4096, 70001])
def test_dot_orderR_within_bound(orc, n):
    x = synth.values(n, array_id=3, mode=synth.U11)
    y = synth.values(n, array_id=4, mode=synth.U11)
    X, Y = FArray(x), FArray(y)
    e, a = orc.dot_exact(X, Y)
    assert abs(orc.dot_orderR(X, Y) - e) <= 4 * n * U * a
    assert orc.dot_orderR(X, FArray(np.ones(n))) == orc.reduce_orderR(X, oracle.SUM)  # x.1 = SUM(x)
