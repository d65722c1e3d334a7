"""MATMUL's stream-K tail (matmul.cu): when whole 128 x 128 tiles would leave
the last one-CTA-per-SM wave less than ~93 % full, all but one full wave stay whole tiles and
the remaining tiles' k-steps are split evenly over one persistent wave; a tile's partial sums
are combined in k order by the CTA that completes it.  The result must stay within R#8's bound
of the oracle (and bit-exact where every partial sum is an exact integer), and be the same
bits on every run (the combine order does not depend on which CTA finishes last)."""
import numpy as np
import pytest
import torch

import oracle
import synth
from oracle import FArray as OA

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ftn():
    from paper_2409_18824_b200 import ftn
    return ftn


def _sms():
    return torch.cuda.get_device_properties(0).multi_processor_count


# (M, N, K): tiles = ceil(M/128) * ceil(N/128) with a ragged last wave on 148 SMs
#   2048 x 1280: 160 tiles (all stream-K), 2048 x 2560: 320 tiles (148 whole + 172 stream-K),
#   1000 x 2600 ragged edges: 8 x 21 = 168 tiles, K not a multiple of 32
CASES = [(2048, 1280, 256), (2048, 2560, 256), (1000, 2600, 300), (1152, 2176, 4096)]


@pytest.mark.parametrize("mnk", CASES)
def test_stream_k_within_bound_and_deterministic(ftn, mnk):
    m, n, k = mnk
    a_h = synth.farray((m, k), array_id=31, mode=synth.U11)
    b_h = synth.farray((k, n), array_id=32, mode=synth.U11)
    A, B = ftn.FArray.from_numpy(a_h), ftn.FArray.from_numpy(b_h)
    C1, C2 = ftn.FArray.empty((m, n)), ftn.FArray.empty((m, n))
    ftn.matmul(C1, A, B)
    ftn.matmul(C2, A, B)
    got = C1.to_numpy()
    np.testing.assert_array_equal(got, C2.to_numpy())          # same bits run to run
    co, ab = np.zeros((m, n), order="F"), np.zeros((m, n), order="F")
    oracle.matmul(OA(co), OA(a_h), OA(b_h), OA(ab))
    assert np.all(np.abs(got - co) <= 4 * k * 2.0 ** -53 * ab)


def test_stream_k_integer_exact(ftn):
    """Integer-valued entries in [-8, 8]: every partial sum is exact, so the split k range
    changes nothing and the product equals the oracle bit for bit."""
    m, n, k = 2048, 2560, 512
    a_h = synth.farray((m, k), array_id=33, mode=synth.INT8)
    b_h = synth.farray((k, n), array_id=34, mode=synth.INT8)
    C = ftn.FArray.empty((m, n))
    ftn.matmul(C, ftn.FArray.from_numpy(a_h), ftn.FArray.from_numpy(b_h))
    co = np.zeros((m, n), order="F")
    oracle.matmul(OA(co), OA(a_h), OA(b_h))
    np.testing.assert_array_equal(C.to_numpy(), co)


def test_stream_k_transposed_operands(ftn):
    """MATMUL(TRANSPOSE(a), b) and MATMUL(a, TRANSPOSE(b)) through the same tail."""
    m, n, k = 2048, 1280, 256
    at = synth.farray((k, m), array_id=35, mode=synth.U11)
    b_h = synth.farray((k, n), array_id=36, mode=synth.U11)
    C = ftn.FArray.empty((m, n))
    ftn.matmul(C, ftn.FArray.from_numpy(at), ftn.FArray.from_numpy(b_h), transpose_a=True)
    a_h = np.asfortranarray(at.T)
    co, ab = np.zeros((m, n), order="F"), np.zeros((m, n), order="F")
    oracle.matmul(OA(co), OA(a_h), OA(b_h), OA(ab))
    assert np.all(np.abs(C.to_numpy() - co) <= 4 * k * 2.0 ** -53 * ab)
    bt = np.asfortranarray(b_h.T)
    ftn.matmul(C, ftn.FArray.from_numpy(a_h), ftn.FArray.from_numpy(bt), transpose_b=True)
    assert np.all(np.abs(C.to_numpy() - co) <= 4 * k * 2.0 ** -53 * ab)


def test_stream_k_with_packed_operands(ftn):
    """Operands the TMA boxes cannot address (a leading dimension of 2049 doubles: rows not
    16-byte aligned) are packed into the workspace first; the stream-K slots follow the packed
    copies in the same workspace."""
    m, n, k = 2048, 1280, 256
    a_big = synth.farray((m + 1, k), array_id=41, mode=synth.U11)
    b_big = synth.farray((k + 1, n), array_id=42, mode=synth.U11)
    A = ftn.FArray.from_numpy(a_big).section((1, m), (1, k))
    B = ftn.FArray.from_numpy(b_big).section((1, k), (1, n))
    C = ftn.FArray.empty((m, n))
    ftn.matmul(C, A, B)
    a_h, b_h = np.asfortranarray(a_big[:m]), np.asfortranarray(b_big[:k])
    co, ab = np.zeros((m, n), order="F"), np.zeros((m, n), order="F")
    oracle.matmul(OA(co), OA(a_h), OA(b_h), OA(ab))
    assert np.all(np.abs(C.to_numpy() - co) <= 4 * k * 2.0 ** -53 * ab)
