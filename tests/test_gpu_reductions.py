"""GPU parity: SUM / MAXVAL / MINVAL / DOT_PRODUCT vs the oracle.

fp64 SUM/DOT: bit-exact vs the oracle's emulation of order R AND within
4 n 2^-53 sum|x| of the exact sum (R#8).  MAXVAL/MINVAL and integer SUM: bit-exact."""
import math

import numpy as np
import pytest
import torch

import oracle
import synth
from oracle import FArray as OA

pytestmark = pytest.mark.gpu
U = 2.0 ** -53


@pytest.fixture(scope="module")
def ftn():
    from paper_2409_18824_b200 import ftn
    return ftn


def _check_sum(ftn, G, O):
    got = ftn.sum(G).item()
    assert got == oracle.reduce_orderR(O, oracle.SUM), "not order R"
    exact = oracle.sum_exact(O)
    n = int(np.prod(O.shape)) if O.shape else 1
    assert abs(got - exact) <= 4 * max(n, 1) * U * oracle.sum_abs(O)


SIZES = [0, 1, 2, 3, 4, 5, 7, 1023, 1024, 1025, 4095, 65535, 65536, 65537, 2 * 65536 + 1, 3 * 65536 - 1,
         5 * 65536 + 12345]


@pytest.mark.parametrize("n", SIZES)
def test_sum_max_min_sizes(ftn, n):
    v = synth.values(n, array_id=n % 7, mode=synth.U11) * np.exp2(synth.values(n, array_id=9, mode=synth.INT8) * 4)
    G, O = ftn.FArray.from_numpy(v), OA(v)
    _check_sum(ftn, G, O)
    assert ftn.maxval(G).item() == oracle.maxval(O)
    assert ftn.minval(G).item() == oracle.minval(O)


def test_every_small_n(ftn):
    """Every N in [0, 2100] (covers every warp / group-of-4 / block remainder)."""
    v = synth.values(2100, mode=synth.U11)
    big = ftn.FArray.from_numpy(v)
    for n in range(0, 2101, 7):
        G = big.section((1, n)) if n > 0 else ftn.FArray.empty((0,))
        O = OA(v[:n].copy())
        got = ftn.sum(G).item()
        assert got == oracle.reduce_orderR(O, oracle.SUM), n
        # and within the R#8 bound of the exactly rounded sum (independent of the R emulation)
        assert abs(got - oracle.sum_exact(O)) <= 4 * max(n, 1) * U * oracle.sum_abs(O), n
        assert ftn.maxval(G).item() == oracle.maxval(O), n


def test_c1_section(ftn):
    a = synth.farray((64, 48), mode=synth.LINEAR)
    A = ftn.FArray.from_numpy(a, [0, 1])
    s = A.section((0, 63, 2), (1, 48))
    assert ftn.sum(s).item() == 2357760.0
    assert ftn.maxval(s).item() == 3070.0 and ftn.minval(s).item() == 0.0
    au = synth.farray((64, 48), mode=synth.U11)
    Au, Ao = ftn.FArray.from_numpy(au, [0, 1]), OA(au, [0, 1])
    _check_sum(ftn, Au.section((0, 63, 2), (1, 48)), Ao.section((0, 63, 2), (1, 48, 1)))


@pytest.mark.parametrize("seed", range(6))
def test_sections_equal_packed_copy(ftn, seed):
    """Invariant: SUM(section) is bit-identical to SUM(packed copy) (the group width is logical)."""
    rng = np.random.default_rng(seed)
    shape = (int(rng.integers(5, 300)), int(rng.integers(3, 200)), int(rng.integers(1, 6)))
    a = synth.farray(shape, array_id=seed, mode=synth.U11)
    A = ftn.FArray.from_numpy(a, [-3, 4, 0])
    st = [int(rng.choice([-2, -1, 1, 2])) for _ in range(3)]
    trip = []
    for d in range(3):
        lb = [-3, 4, 0][d]
        ub = lb + shape[d] - 1
        trip.append((lb, ub, st[d]) if st[d] > 0 else (ub, lb, st[d]))
    S = A.section(*trip)
    packed = ftn.FArray.empty(S.shape)
    ftn.assign(packed, S)
    assert ftn.sum(S).item() == ftn.sum(packed).item()
    O = OA(a, [-3, 4, 0]).section(*trip)
    _check_sum(ftn, S, O)
    assert ftn.maxval(S).item() == oracle.maxval(O) and ftn.minval(S).item() == oracle.minval(O)


@pytest.mark.parametrize("dtype", [np.int32, np.int64])
def test_integer_reductions(ftn, dtype):
    a = synth.farray((333, 417), mode=synth.RAW, dtype=dtype)
    tt = {np.int32: torch.int32, np.int64: torch.int64}[dtype]
    G, O = ftn.FArray.from_numpy(a), OA(a)
    assert ftn.sum(G).item() == oracle.sum_int(O)
    assert ftn.maxval(G).item() == oracle.maxval(O) and ftn.minval(G).item() == oracle.minval(O)
    S = G.section((333, 1, -3), (2, 417, 2))
    So = O.section((333, 1, -3), (2, 417, 2))
    assert ftn.sum(S).item() == oracle.sum_int(So)
    e = ftn.FArray.empty((0,), dtype=tt)
    assert ftn.maxval(e).item() == np.iinfo(dtype).min and ftn.minval(e).item() == np.iinfo(dtype).max
    assert ftn.sum(e).item() == 0


def test_empty_and_nan(ftn):
    e = ftn.FArray.empty((0, 5))
    assert ftn.sum(e).item() == 0.0
    assert ftn.maxval(e).item() == -math.inf and ftn.minval(e).item() == math.inf
    v = np.array([np.nan, 1.0, np.nan, -3.0, 2.0])
    G = ftn.FArray.from_numpy(v)
    assert ftn.maxval(G).item() == 2.0 and ftn.minval(G).item() == -3.0
    assert math.isnan(ftn.maxval(ftn.FArray.from_numpy(np.array([np.nan, np.nan]))).item())


@pytest.mark.parametrize("pos", [0, 1023, 65535, 65536, 131073, 300000 - 1])
def test_planted_extrema(ftn, pos):
    v = synth.values(300000, mode=synth.U11)
    v[pos] = 9.0
    G = ftn.FArray.from_numpy(v)
    assert ftn.maxval(G).item() == 9.0
    v[pos] = -9.0
    G = ftn.FArray.from_numpy(v)
    assert ftn.minval(G).item() == -9.0


@pytest.mark.parametrize("n", [1, 4, 1000, 65536, 65537, 262147])
def test_dot_product(ftn, n):
    x = synth.values(n, array_id=1, mode=synth.U11)
    y = synth.values(2 * n, array_id=2, mode=synth.U11)
    X = ftn.FArray.from_numpy(x)
    Y = ftn.FArray.from_numpy(y).section((2 * n - 1, 1, -2))        # strided, reversed
    Xo, Yo = OA(x), OA(y).section((2 * n - 1, 1, -2))
    got = ftn.dot_product(X, Y).item()
    assert got == oracle.dot_orderR(Xo, Yo)
    e, a = oracle.dot_exact(Xo, Yo)
    assert abs(got - e) <= 4 * n * U * a
    # DOT(x, y) == SUM(x*y) bit for bit
    p = ftn.FArray.empty((n,))
    ftn.elemental(ftn.MUL, p, X, Y)
    assert ftn.sum(p).item() == got


def test_closed_form_mod1024(ftn):
    n = 1 << 24
    x = ftn.FArray.empty((n,))
    ftn.gen_fill(x, synth.SEED, 0, ftn.GEN_MOD1024)
    assert ftn.sum(x).item() == (n // 1024) * 523776
    assert ftn.dot_product(x, x).item() == (n // 1024) * 357389824


@pytest.mark.slow
def test_c4_full_size(ftn):
    """C4 at full size: x(-511:512, 0:1023, 1:1024), 2^30 elements, closed forms (exact in any order)
    and the section variant p(:,:,1:2048:2) vs the packed copy."""
    shape = (1024, 1024, 1024)
    x = ftn.FArray.empty(shape, lbounds=[-511, 0, 1])
    ftn.gen_fill(x, synth.SEED, 0, ftn.GEN_MOD1024)
    assert ftn.sum(x).item() == 549218942976.0
    flat = ftn.FArray(x.tensor.permute(2, 1, 0).reshape(-1))
    assert ftn.dot_product(flat, flat).item() == 374750392090624.0
    assert ftn.maxval(x).item() == 1023.0 and ftn.minval(x).item() == 0.0
    del x, flat
    torch.cuda.empty_cache()
    p = ftn.FArray.empty((1024, 1024, 2048))
    ftn.gen_fill(p, synth.SEED, 1, ftn.GEN_U01)
    s = p.section((1, 1024), (1, 1024), (1, 2048, 2))
    packed = ftn.FArray.empty(s.shape)
    ftn.assign(packed, s)
    assert ftn.sum(s).item() == ftn.sum(packed).item()
    # sampled check of the R-order result against the oracle on one full chunk-aligned slab
    sub = s.section((1, 1024), (1, 1024), (1, 1))
    host = sub.to_numpy()
    assert ftn.sum(sub).item() == oracle.reduce_orderR(OA(host), oracle.SUM)


@pytest.mark.slow
def test_c4_full_size_order_r_bit_exact(ftn):
    """The bench's C4 SUM / MAXVAL / MINVAL on x(-511:512, 0:1023, 1:1024) = 2^30 elements of
    U[0,1) (same generator and launch configuration as bench.py): bit-exact vs the oracle's
    order-R emulation over the whole array; and DOT_PRODUCT at the paper's 2^27 size, bit-exact
    vs order R and within the R#8 bound of the exact dot."""
    x = ftn.FArray.empty((1024, 1024, 1024), lbounds=[-511, 0, 1])
    ftn.gen_fill(x, synth.SEED, 10, ftn.GEN_U01)
    host = x.to_numpy()
    O = OA(host, [-511, 0, 1])
    got = ftn.sum(x).item()
    assert got == oracle.reduce_orderR(O, oracle.SUM)
    assert abs(got - oracle.sum_exact(O)) <= 4 * (1 << 30) * U * oracle.sum_abs(O)   # R#8, exact sum
    assert ftn.maxval(x).item() == oracle.maxval(O)
    assert ftn.minval(x).item() == oracle.minval(O)
    del x, host, O
    torch.cuda.empty_cache()
    n = 1 << 27
    X, Y = ftn.FArray.empty((n,)), ftn.FArray.empty((n,))
    ftn.gen_fill(X, synth.SEED, 20, ftn.GEN_U11)
    ftn.gen_fill(Y, synth.SEED, 21, ftn.GEN_U11)
    got = ftn.dot_product(X, Y).item()
    xo, yo = OA(X.to_numpy()), OA(Y.to_numpy())
    assert got == oracle.dot_orderR(xo, yo)
    e, a = oracle.dot_exact(xo, yo)
    assert abs(got - e) <= 4 * n * U * a


@pytest.mark.slow
def test_more_than_2_32_elements(ftn):
    """64-bit indexing end to end (SURVEY §7 hard part 6): a (2^16 + 3) x 2^16 array (2^32 +
    196608 elements, 32 GB) with the t mod 1024 pattern: SUM / MAXVAL closed forms, and an
    element-wise b*c+d into a second array checked at sampled positions past 2^32."""
    n1, n2 = 65536 + 3, 65536
    x = ftn.FArray.empty((n1, n2))
    ftn.gen_fill(x, synth.SEED, 0, ftn.GEN_MOD1024)
    n = n1 * n2
    full, rem = divmod(n, 1024)
    assert ftn.sum(x).item() == float(full * 523776 + rem * (rem - 1) // 2)
    assert ftn.maxval(x).item() == 1023.0
    r = ftn.FArray.empty((n1, n2))
    ftn.muladd(r, x, x, x)                                  # t' (t' + 1), t' = t mod 1024
    for t in [0, 1023, (1 << 32) - 1, 1 << 32, (1 << 32) + 1025, n - 1]:
        i, j = t % n1, t // n1
        v = r.section((i + 1, i + 1), (j + 1, j + 1)).to_numpy().ravel()[0]
        m = t % 1024
        assert v == float(m * m + m), t


def test_concurrent_streams_do_not_share_workspaces(ftn):
    """Reductions issued on several streams at once get separate workspaces (the binding keys
    them by stream): every result equals the serial one."""
    xs = [ftn.FArray.empty((3 * 65536 + 77,)) for _ in range(4)]
    for q, x in enumerate(xs):
        ftn.gen_fill(x, synth.SEED, 30 + q, ftn.GEN_U11)
    serial = [ftn.sum(x).item() for x in xs]
    streams = [torch.cuda.Stream() for _ in xs]
    for _ in range(3):
        outs = [ftn.sum(x, stream=s) for x, s in zip(xs, streams)]
        torch.cuda.synchronize()
        assert [o.item() for o in outs] == serial


@pytest.mark.parametrize("kind", ["sum", "maxval", "absdiff"])
def test_chunk_contiguous_sections(ftn, kind):
    """Sections whose collapsed rows are whole multiples of the 65536-element chunk (every
    other plane of a stack) take the 256-bit chunk path, one- and two-operand: bit-exact vs
    order R on the oracle / exact max |x - y|."""
    shape = (256, 512, 6)                                 # plane = 131072 elements = 2 chunks
    a = synth.farray(shape, array_id=11, mode=synth.U11)
    b = synth.farray(shape, array_id=12, mode=synth.U11)
    A, B = ftn.FArray.from_numpy(a), ftn.FArray.from_numpy(b)
    sec = ((1, 256), (1, 512), (1, 6, 2))
    G = A.section(*sec)
    O = OA(a).section((1, 256, 1), (1, 512, 1), (1, 6, 2))
    if kind == "sum":
        assert ftn.sum(G).item() == oracle.reduce_orderR(O, oracle.SUM)
        packed = ftn.FArray.empty(G.shape)
        ftn.assign(packed, G)
        assert ftn.sum(G).item() == ftn.sum(packed).item()
    elif kind == "maxval":
        assert ftn.maxval(G).item() == oracle.maxval(O)
    else:
        got = ftn.maxval_absdiff(G, B.section(*sec)).item()
        assert got == np.max(np.abs(a[:, :, ::2] - b[:, :, ::2]))
