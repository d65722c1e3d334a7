"""GPU parity: PRODUCT (order R) and SUM/PRODUCT/MAXVAL/MINVAL(x, DIM=d) (sequential fold,
DESIGN.md R#24) vs the oracle -- bit-exact."""
from fractions import Fraction

import numpy as np
import pytest
import torch

import oracle
import synth
from oracle import FArray as OA

pytestmark = pytest.mark.gpu
TT = {np.float64: torch.float64, np.int32: torch.int32, np.int64: torch.int64}
KINDS = [(oracle.SUM, "sum_dim"), (oracle.PROD, "product_dim"), (oracle.MAX, "maxval_dim"),
         (oracle.MIN, "minval_dim")]


@pytest.fixture(scope="module")
def ftn():
    from paper_2409_18824_b200 import ftn
    return ftn


@pytest.mark.parametrize("shape", [(1,), (37,), (5, 9), (64, 33), (1, 70), (70, 1), (33, 40, 7), (3, 1, 130),
                                   (257, 3, 2), (1000, 300)])
@pytest.mark.parametrize("dtype", [np.float64, np.int64, np.int32])
def test_dim_reductions_vs_oracle(ftn, shape, dtype):
    mode = synth.U11 if dtype == np.float64 else synth.RAW
    a = synth.farray(shape, mode=mode, dtype=dtype)
    if dtype == np.float64:
        a = a + 1.0                                          # products stay in range
    G, O = ftn.FArray.from_numpy(a, [2] * len(shape)), OA(a, [2] * len(shape))
    for dim in range(1, len(shape) + 1):
        for kind, name in KINDS:
            got = getattr(ftn, name)(G, dim)
            ref = oracle.reduce_dim(O, dim, kind)
            np.testing.assert_array_equal(got.to_numpy() if got.rank else got.tensor.cpu().numpy(), ref,
                                          err_msg=f"{name} dim={dim} shape={shape}")


def test_dim_reductions_on_sections_into_sections(ftn):
    a = synth.farray((90, 41, 12), mode=synth.U11)
    G, O = ftn.FArray.from_numpy(a), OA(a)
    trip = ((89, 2, -3), (1, 41, 2), (12, 1, -1))
    gs, os_ = G.section(*trip), O.section(*trip)
    for dim in (1, 2, 3):
        shape = tuple(e for d, e in enumerate(gs.shape) if d != dim - 1)
        big = ftn.FArray.empty(tuple(2 * e for e in shape))
        ftn.fill(big, -5.0)
        dst = big.section(*[(2 * e, 1, -2) for e in shape])       # reversed, strided result
        ftn.sum_dim(gs, dim, dst)
        np.testing.assert_array_equal(dst.to_numpy(), oracle.reduce_dim(os_, dim, oracle.SUM))
        ftn.maxval_dim(gs, dim, dst)
        np.testing.assert_array_equal(dst.to_numpy(), oracle.reduce_dim(os_, dim, oracle.MAX))


def test_dim_nan_empty(ftn):
    a = np.array([[np.nan, 1.0], [np.nan, np.nan], [np.nan, 3.0]], order="F")   # (3, 2)
    r = ftn.maxval_dim(ftn.FArray.from_numpy(a), 1).to_numpy()
    assert r[0] == np.nan or np.isnan(r[0]) and r[1] == 3.0
    e = ftn.FArray.empty((0, 6))
    assert (ftn.maxval_dim(e, 1).to_numpy() == -np.inf).all()
    assert (ftn.sum_dim(e, 1).to_numpy() == 0).all() and (ftn.product_dim(e, 1).to_numpy() == 1).all()
    assert ftn.sum_dim(e, 2).shape == (0,)


@pytest.mark.parametrize("n", [0, 1, 5, 1024, 65536, 65537, 300001])
def test_product_full(ftn, n):
    v = 1.0 + synth.values(n, mode=synth.U11) * 2.0 ** -10
    G, O = ftn.FArray.from_numpy(v), OA(v)
    got = ftn.product(G).item()
    assert got == oracle.reduce_orderR(O, oracle.PROD)
    if 0 < n <= 1024:
        exact = Fraction(1)
        for t in v:
            exact *= Fraction(t)
        assert abs(Fraction(got) - exact) <= Fraction(2 * n) * Fraction(2.0 ** -53) * abs(exact)
    iv = synth.farray((70, 30), mode=synth.RAW, dtype=np.int64)
    with np.errstate(over="ignore"):
        assert ftn.product(ftn.FArray.from_numpy(iv)).item() == np.prod(iv, dtype=np.int64)


def test_c4_dim_sums_full_size(ftn):
    """C4 x(-511:512,0:1023,1:1024) reduced along each dimension; t mod 1024 pattern (exact)."""
    x = ftn.FArray.empty((1024, 1024, 256), lbounds=[-511, 0, 1])
    ftn.gen_fill(x, synth.SEED, 0, ftn.GEN_MOD1024)
    s1 = ftn.sum_dim(x, 1).to_numpy()
    assert (s1 == 523776.0).all()                       # each column holds 0..1023
    s3 = ftn.sum_dim(x, 3).to_numpy()
    i = np.arange(1024)
    assert (s3 == (i[:, None] * 256).astype(np.float64)).all()
