"""Pins for the oracle's PRODUCT and DIM= reductions ("dimensions",
"product ... also implemented"; R#24).

Independent references: np.cumsum / np.cumprod along an axis (sequential folds in
ascending index order), np.fmax / np.fmin reductions (NaN-ignoring), fractions.Fraction
(exact products), closed forms."""
import math
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synth
from oracle import FArray

U = 2.0 ** -53


def _sec(a, lbs, trip):
    return FArray(a, lbs).section(*trip)


@pytest.mark.parametrize("shape", [(7,), (5, 9), (6, 4, 3), (1, 8), (8, 1, 5)])
@pytest.mark.parametrize("kind", [oracle.SUM, oracle.PROD])
def test_dim_fold_vs_cumulative(orc, shape, kind):
    a = synth.farray(shape, mode=synth.U11) + (1.5 if kind == oracle.PROD else 0.0)
    for dim in range(1, len(shape) + 1):
        got = orc.reduce_dim(FArray(a, [3] * len(shape)), dim, kind)
        cum = np.cumsum(a, axis=dim - 1) if kind == oracle.SUM else np.cumprod(a, axis=dim - 1)
        ref = np.take(cum, -1, axis=dim - 1)
        np.testing.assert_array_equal(got, ref)


def test_dim_on_sections(orc):
    a = synth.farray((20, 15, 6), mode=synth.U11)
    trip = ((19, 2, -3), (1, 15, 2), (6, 1, -1))
    S = _sec(a, [1, 1, 1], trip)
    view = S.to_numpy()
    for dim in (1, 2, 3):
        got = orc.reduce_dim(S, dim, oracle.SUM)
        np.testing.assert_array_equal(got, np.take(np.cumsum(view, axis=dim - 1), -1, axis=dim - 1))
        np.testing.assert_array_equal(orc.reduce_dim(S, dim, oracle.MAX), np.fmax.reduce(view, axis=dim - 1))
        np.testing.assert_array_equal(orc.reduce_dim(S, dim, oracle.MIN), np.fmin.reduce(view, axis=dim - 1))


def test_dim_maxmin_nan_and_empty(orc):
    a = np.array([[np.nan, 1.0, np.nan], [np.nan, np.nan, np.nan]], order="F").T.copy(order="F")  # (3, 2)
    mx = orc.reduce_dim(FArray(a), 1, oracle.MAX)
    assert mx[0] == 1.0 and math.isnan(mx[1])
    e = np.zeros((0, 4), order="F")
    assert (orc.reduce_dim(FArray(e), 1, oracle.MAX) == -math.inf).all()
    assert (orc.reduce_dim(FArray(e), 1, oracle.MIN) == math.inf).all()
    assert (orc.reduce_dim(FArray(e), 1, oracle.SUM) == 0.0).all()
    assert (orc.reduce_dim(FArray(e), 1, oracle.PROD) == 1.0).all()
    assert orc.reduce_dim(FArray(e), 2, oracle.SUM).shape == (0,)


@pytest.mark.parametrize("dtype", [np.int32, np.int64])
def test_dim_integer_wraps(orc, dtype):
    a = synth.farray((9, 7, 4), mode=synth.RAW, dtype=dtype)
    with np.errstate(over="ignore"):
        for dim in (1, 2, 3):
            np.testing.assert_array_equal(orc.reduce_dim(FArray(a), dim, oracle.SUM), np.sum(a, axis=dim - 1, dtype=dtype))
            np.testing.assert_array_equal(orc.reduce_dim(FArray(a), dim, oracle.PROD),
                                          np.prod(a, axis=dim - 1, dtype=dtype))
            np.testing.assert_array_equal(orc.reduce_dim(FArray(a), dim, oracle.MAX), a.max(axis=dim - 1))
            np.testing.assert_array_equal(orc.reduce_dim(FArray(a), dim, oracle.MIN), a.min(axis=dim - 1))


def test_product_full(orc):
    v = 1.0 + synth.values(3000, mode=synth.U11) * 2.0 ** -8
    x = FArray(v)
    assert orc.product_seq(x) == np.cumprod(v)[-1]
    exact = Fraction(1)
    for t in v:
        exact *= Fraction(t)
    r = orc.reduce_orderR(x, oracle.PROD)
    n = v.size
    assert abs(Fraction(r) - exact) <= Fraction(2 * n) * Fraction(U) * abs(exact)
    p2 = np.exp2(synth.values(5000, mode=synth.INT8))                # powers of two: exact
    assert orc.reduce_orderR(FArray(p2), oracle.PROD) == 2.0 ** float(np.sum(np.log2(p2)))
    iv = np.array([3.0, -2.0, 5.0, 7.0, -1.0, 11.0, 2.0, 13.0])        # exact integer product
    assert orc.reduce_orderR(FArray(iv), oracle.PROD) == 3 * -2 * 5 * 7 * -1 * 11 * 2 * 13
    assert orc.reduce_orderR(FArray(np.zeros(0)), oracle.PROD) == 1.0
    assert orc.tree_combine([2.0, 3.0, 5.0], oracle.PROD) == 30.0
    ia = synth.farray((40, 3), mode=synth.RAW, dtype=np.int64)
    with np.errstate(over="ignore"):
        assert orc.product_int(FArray(ia)) == np.prod(ia, dtype=np.int64)
