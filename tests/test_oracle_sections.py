"""Pins for the oracle's descriptor / section logic (R#1-R#4).

Every expected value here comes from outside the oracle: the paper's and SPEC's
worked examples (tests/golden/*.json, cited), Python's range() enumeration of a
DO loop, numpy's basic slicing, or closed-form strides.
"""
import json
import os

import numpy as np
import pytest

import oracle
from oracle import FArray, OracleError

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _range_of(lo, hi, step):
    """Fortran DO / triplet enumeration via Python's range (independent library routine)."""
    return list(range(lo, hi + (1 if step > 0 else -1), step))


def test_golden_do_loops(orc):
    g = json.load(open(os.path.join(GOLDEN, "triplets.json")))
    for c in g["cases"]:
        idx = orc.triplet_indices(c["lo"], c["hi"], c["step"])
        assert idx == c["indices"]
        assert sum(idx) == c["acc"]


def test_exhaustive_triplets_vs_range(orc):
    """S:539 / S:565: l,u in [-6,6], s in [-3,-1] U [1,3] vs brute-force enumeration."""
    for lo in range(-6, 7):
        for hi in range(-6, 7):
            for st in (-3, -2, -1, 1, 2, 3):
                expect = _range_of(lo, hi, st)
                assert orc.triplet_indices(lo, hi, st) == expect
                # the section extent formula max(0, (hi-lo+st) div st) gives the same count
                parent = FArray(np.arange(13, dtype=np.int32), [-6])
                sec = parent.section((lo, hi, st))
                assert sec.shape == (len(expect),)
                assert sec.lbounds == [1]


def test_exhaustive_triplets_values(orc):
    vals = np.arange(-6, 7, dtype=np.int64)          # parent(-6:6) with parent(i) = i
    parent = FArray(vals, [-6])
    for lo in range(-6, 7):
        for hi in range(-6, 7):
            for st in (-3, -2, -1, 1, 2, 3):
                sec = parent.section((lo, hi, st))
                assert list(sec.to_numpy()) == _range_of(lo, hi, st)


def test_zero_step_and_out_of_bounds(orc):
    a = FArray(np.zeros(10, dtype=np.float64), [1])
    with pytest.raises(OracleError) as e:
        a.section((1, 10, 0))
    assert e.value.code == 6
    with pytest.raises(OracleError) as e:
        a.section((0, 10, 1))
    assert e.value.code == 5
    with pytest.raises(OracleError) as e:
        a.section((1, 11, 1))
    assert e.value.code == 5
    # empty sections never check bounds (extent 0): a(20:5) is legal
    assert a.section((20, 5, 1)).shape == (0,)
    # the selected elements, not hi, must be in bounds: a(1:14:4) selects 1,5,9,13 -> 13 is out,
    # while a(1:12:4) selects 1,5,9 and hi = 12 itself is never referenced
    with pytest.raises(OracleError):
        a.section((1, 14, 4))
    assert a.section((1, 12, 4)).shape == (3,)
    assert a.section((10, -1, -4)).shape == (3,)   # 10, 6, 2 (hi = -1 is never referenced)


def test_paper_worked_example(orc):
    """allocate(data(10)); data(2)=100 -> memref index 1 (origin subtraction)."""
    g = json.load(open(os.path.join(GOLDEN, "worked_examples.json")))
    ex = g["allocatable"]
    buf = np.zeros(ex["extent"], dtype=np.int32)
    data = FArray(buf, [ex["lbound"]])
    off = orc.element_offset(data, ex["subscript"])
    assert off == ex["memref_index"] * ex["elem_len"]
    one = FArray(np.array(ex["value"], dtype=np.int32))
    tgt = data.section((ex["subscript"], ex["subscript"], 1))
    orc.assign(tgt, one)
    assert buf[ex["memref_index"]] == ex["value"] and buf.sum() == ex["value"]
    ex0 = g["origin_zero"]
    d0 = FArray(np.zeros(ex0["extent"], dtype=np.int32), [ex0["lbound"]])
    assert orc.element_offset(d0, ex0["subscript"]) == ex0["memref_index"] * 4


def test_c1_descriptors(orc):
    """BASELINE configs[0]: a(0:63,1:48) -> a(::2,:) = {1,32,16},{1,48,512}; a(1::2,:) at base+8."""
    a = np.zeros((64, 48), dtype=np.float64, order="F")
    A = FArray(a, [0, 1])
    s = A.section((0, 63, 2), (1, 48, 1))
    assert s.shape == (32, 48) and s.strides == (16, 512) and s.lbounds == [1, 1]
    assert s.base_offset() == 0
    c = A.section((1, 63, 2), (1, 48, 1))
    assert c.shape == (32, 48) and c.base_offset() == 8


def test_c4_descriptors(orc):
    """C4: x(-511:512,0:1023,1:1024) has sm = (8, 8192, 8 MiB); p(:,:,1:2048:2) has sm3 = 16 MiB.
    (numpy's own stride computation is the independent check; no data is allocated.)"""
    shape = (1024, 1024, 1024)
    strides = np.lib.stride_tricks.as_strided(np.zeros(1), shape=shape, strides=(8, 8192, 8 << 20)).strides
    assert strides == (8, 8192, 8 << 20)
    x = np.lib.stride_tricks.as_strided(np.zeros(1), shape=(2, 2, 2048), strides=(8, 8192, 8 << 20))
    P = FArray(x, [1, 1, 1])
    sec = P.section((1, 2, 1), (1, 2, 1), (1, 2048, 2))
    assert sec.strides[2] == 16 << 20 and sec.shape == (2, 2, 1024)


@pytest.mark.parametrize("seed", range(20))
def test_sections_vs_numpy_slicing(orc, seed):
    """Random rank-1..3 sections (mixed lbounds, negative steps) select the same elements
    as numpy basic slicing."""
    rng = np.random.default_rng(seed)
    r = int(rng.integers(1, 4))
    shape = tuple(int(rng.integers(1, 9)) for _ in range(r))
    lbs = [int(rng.integers(-5, 6)) for _ in range(r)]
    arr = np.asfortranarray(rng.standard_normal(shape))
    A = FArray(arr, lbs)
    trip, sl = [], []
    for d in range(r):
        n, lb = shape[d], lbs[d]
        st = int(rng.choice([-3, -2, -1, 1, 2, 3]))
        i0, i1 = sorted(int(v) for v in rng.integers(0, n, size=2))
        lo, hi = (lb + i0, lb + i1) if st > 0 else (lb + i1, lb + i0)
        trip.append((lo, hi, st))
        stop = (hi - lb + 1) if st > 0 else (hi - lb - 1)
        sl.append(slice(lo - lb, stop if stop >= 0 else None, st))
    S = A.section(*trip)
    ref = arr[tuple(sl)]
    assert S.shape == ref.shape
    np.testing.assert_array_equal(S.to_numpy(), ref)


def test_section_aliasing(orc):
    """S:326 / P:237: writes through a section are visible in the parent."""
    rng = np.random.default_rng(7)
    a = np.asfortranarray(rng.standard_normal((10, 7)))
    expect = a.copy()
    A = FArray(a, [1, 1])
    sec = A.section((2, 9, 3), (7, 1, -2))
    src = np.asfortranarray(rng.standard_normal(sec.shape))
    oracle.assign(sec, FArray(src))
    expect[1:9:3, 6::-2] = src
    np.testing.assert_array_equal(a, expect)
