"""CPU checks of the C-ABI library: it loads without a GPU, exports every symbol
include/ftn.h declares, and its host-only descriptor logic (sections, inquiry) agrees
with the oracle's independently written section logic.  No compute calls."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle
from oracle import FArray as OA

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def ftn():
    from paper_2409_18824_b200 import build
    build.build()
    from paper_2409_18824_b200 import ftn
    return ftn


def test_exports_every_declared_symbol(ftn):
    hdr = open(os.path.join(ROOT, "include", "ftn.h")).read()
    names = set(re.findall(r"^(?:ftn_status_t|u?int(?:32|64)_t|const char\s*\*)\s*(ftn_\w+)\s*\(", hdr, re.M))
    assert len(names) >= 50
    for n in sorted(names):
        assert hasattr(ftn.lib, n), f"libftn.so does not export {n}"


def _desc(ftn, lb, ext, type_=4):
    d = ftn.Desc()
    r = len(ext)
    rc = ftn.lib.ftn_desc_contiguous(ctypes.byref(d), ctypes.c_void_p(1 << 20), type_, r,
                                     (ctypes.c_int64 * r)(*lb), (ctypes.c_int64 * r)(*ext))
    assert rc == 0
    return d


def _section(ftn, d, trip):
    r = d.rank
    out = ftn.Desc()
    rc = ftn.lib.ftn_desc_section(ctypes.byref(out), ctypes.byref(d), (ctypes.c_int64 * r)(*[t[0] for t in trip]),
                                  (ctypes.c_int64 * r)(*[t[1] for t in trip]),
                                  (ctypes.c_int64 * r)(*[t[2] for t in trip]))
    return rc, out


def test_sections_agree_with_oracle_exhaustively(ftn):
    """ftn_desc_section vs orc_section on every triplet with l,u in [-6,6], s in +-[1,3]."""
    buf = np.zeros(13, dtype=np.float64)
    par_o = OA(buf, [-6])
    par_g = _desc(ftn, [-6], [13])
    for lo in range(-6, 7):
        for hi in range(-6, 7):
            for st in (-3, -2, -1, 1, 2, 3):
                rc, g = _section(ftn, par_g, [(lo, hi, st)])
                assert rc == 0
                o = par_o.section((lo, hi, st))
                assert g.dim[0].extent == o.shape[0] and g.dim[0].sm == o.strides[0]
                assert g.dim[0].lower_bound == 1
                if o.shape[0]:
                    assert g.base_addr - (1 << 20) == o.base_offset()
    rc, _ = _section(ftn, par_g, [(1, 3, 0)])
    assert rc == 5                                          # FTN_ERR_BOUNDS: zero step
    rc, _ = _section(ftn, par_g, [(-7, 3, 1)])
    assert rc == 5


def test_rank3_sections_and_inquiry(ftn):
    d = _desc(ftn, [-511, 0, 1], [1024, 1024, 1024])
    assert [d.dim[k].sm for k in range(3)] == [8, 8192, 8 << 20]
    rc, s = _section(ftn, d, [(-511, 512, 1), (0, 1023, 1), (1, 1024, 2)])
    assert rc == 0 and s.dim[2].sm == 16 << 20 and s.dim[2].extent == 512
    out = ctypes.c_int64()
    assert ftn.lib.ftn_lbound(ctypes.byref(d), 1, ctypes.byref(out)) == 0 and out.value == -511
    assert ftn.lib.ftn_ubound(ctypes.byref(d), 1, ctypes.byref(out)) == 0 and out.value == 512
    assert ftn.lib.ftn_size(ctypes.byref(d), 0, ctypes.byref(out)) == 0 and out.value == 1 << 30
    assert ftn.lib.ftn_size(ctypes.byref(d), 4, ctypes.byref(out)) == 6          # FTN_ERR_DIM
    shp = (ctypes.c_int64 * 3)()
    assert ftn.lib.ftn_shape(ctypes.byref(s), shp) == 0 and list(shp) == [1024, 1024, 512]
    # C1 and the paper's worked example: data(2) at byte offset 4
    c1 = _desc(ftn, [0, 1], [64, 48])
    rc, s = _section(ftn, c1, [(0, 63, 2), (1, 48, 1)])
    assert (s.dim[0].extent, s.dim[0].sm, s.dim[1].extent, s.dim[1].sm) == (32, 16, 48, 512)
    data = _desc(ftn, [1], [10], type_=1)
    rc, e2 = _section(ftn, data, [(2, 2, 1)])
    assert rc == 0 and e2.base_addr - (1 << 20) == 4


def test_compute_calls_validate_before_device(ftn):
    """Argument errors are reported before any device work (works without a GPU)."""
    a = _desc(ftn, [1, 1], [4, 5])
    b = _desc(ftn, [1, 1], [5, 4])
    rc = ftn.lib.ftn_assign(ctypes.byref(a), ctypes.byref(b), None)
    assert rc == 4                                                              # FTN_ERR_SHAPE
    assert b"not conformable" in ftn.lib.ftn_last_error()
    assert ftn.lib.ftn_status_string(8) == b"FTN_ERR_UNSUPPORTED"


def test_jacobi_launch_plan(ftn):
    """ftn_jacobi_plan (host logic): sweep counts sum to S, each in 1..T, the launch count has
    the parity of S (the result lands in unew iff S is odd) and is the smallest such count
    >= ceil(S/T), and the sweeps are spread evenly (sizes differ by at most one)."""
    for S in range(0, 120):
        for T in range(1, 13):
            p = ftn.jacobi_plan(S, T)
            assert sum(p) == S and len(p) % 2 == S % 2 and all(1 <= k <= T for k in p), (S, T, p)
            n = -(-S // T)
            assert len(p) == (n if n % 2 == S % 2 else n + 1), (S, T, p)
            assert not p or max(p) - min(p) <= 1, (S, T, p)
    assert ftn.jacobi_plan(100, 4) == [4] * 22 + [3] * 4
    assert ftn.jacobi_plan(100, 8) == [8] * 2 + [7] * 12   # 14 launches, none short
    assert ftn.jacobi_plan(100, 5) == [5] * 20          # no short launch
    assert ftn.jacobi_plan(100, 2) == [2] * 50          # C5's plan


def _bytes(d):
    """Brute force: the set of byte addresses a descriptor's elements occupy."""
    import itertools
    out = set()
    exts = [d.dim[k].extent for k in range(d.rank)]
    for idx in itertools.product(*[range(e) for e in exts]):
        a = d.base_addr + sum(i * d.dim[k].sm for k, i in enumerate(idx))
        out.update(range(a, a + d.elem_len))
    return out


def test_may_overlap_is_sound_and_sees_interleaved_sections(ftn):
    """ftn_desc_may_overlap (R#5's alias test) against brute-force byte sets: never 0 when two
    sections share a byte; 0 for the interleaved disjoint pairs a(1::2,:) / a(2::2,:) of an
    array with an even leading extent, and for disjoint byte ranges."""
    rng = np.random.default_rng(5)
    out = ctypes.c_int32()
    for type_, lead in ((4, 6), (4, 5), (3, 8)):
        par = _desc(ftn, [1, 1], [lead, 5], type_=type_)
        secs = []
        for _ in range(60):
            lo = [int(rng.integers(1, lead + 1)), int(rng.integers(1, 6))]
            hi = [int(rng.integers(lo[0], lead + 1)), int(rng.integers(lo[1], 6))]
            st = [int(rng.choice([1, 2, 3])), int(rng.choice([1, 2]))]
            rc, s = _section(ftn, par, list(zip(lo, hi, st)))
            assert rc == 0
            secs.append((s, _bytes(s)))
        for a, ba in secs:
            for b, bb in secs[:20]:
                assert ftn.lib.ftn_desc_may_overlap(ctypes.byref(a), ctypes.byref(b), ctypes.byref(out)) == 0
                if ba & bb:
                    assert out.value == 1
    par = _desc(ftn, [1, 1], [8, 4], type_=4)
    rc, odd = _section(ftn, par, [(1, 8, 2), (1, 4, 1)])
    rc, even = _section(ftn, par, [(2, 8, 2), (1, 4, 1)])
    assert ftn.lib.ftn_desc_may_overlap(ctypes.byref(odd), ctypes.byref(even), ctypes.byref(out)) == 0
    assert out.value == 0 and not (_bytes(odd) & _bytes(even))
    assert ftn.lib.ftn_desc_may_overlap(ctypes.byref(odd), ctypes.byref(odd), ctypes.byref(out)) == 0
    assert out.value == 1
    par7 = _desc(ftn, [1, 1], [7, 4], type_=4)   # odd leading extent: the residue test cannot tell
    rc, odd7 = _section(ftn, par7, [(1, 7, 2), (1, 4, 1)])
    rc, even7 = _section(ftn, par7, [(2, 7, 2), (1, 4, 1)])
    assert ftn.lib.ftn_desc_may_overlap(ctypes.byref(odd7), ctypes.byref(even7), ctypes.byref(out)) == 0
    assert out.value == 1
