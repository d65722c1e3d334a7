"""GPU: zero-extent operands through the C ABI -- every call succeeds, launches nothing it does
not need, and leaves the Fortran results (R#5, R#7): TRANSPOSE of an empty array is empty,
MATMUL with a zero inner extent is all zeros (the empty sum, as the oracle computes it), an
element-wise expression on an empty section touches nothing, SUM of nothing is 0."""
import numpy as np
import pytest
import torch

import oracle
from oracle import FArray as OA

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ftn():
    from paper_2409_18824_b200 import ftn
    return ftn


@pytest.mark.parametrize("dtype", [torch.int32, torch.float64])
@pytest.mark.parametrize("shape", [(0, 5), (5, 0), (0, 0)])
def test_transpose_empty(ftn, dtype, shape):
    a = ftn.FArray.empty(shape, dtype=dtype)
    r = ftn.FArray.empty(shape[::-1], dtype=dtype)
    ftn.transpose(r, a)
    torch.cuda.synchronize()


@pytest.mark.parametrize("force_dmma", [False, True])
@pytest.mark.parametrize("m,n", [(7, 5), (130, 129)])
def test_matmul_zero_inner_extent(ftn, m, n, force_dmma):
    a = ftn.FArray.empty((m, 0))
    b = ftn.FArray.empty((0, n))
    c = ftn.FArray.from_numpy(np.full((m, n), 3.5, order="F"))
    ftn.matmul(c, a, b, force_dmma=force_dmma)
    co = OA(np.full((m, n), 3.5, order="F"))
    oracle.matmul(co, OA(np.zeros((m, 0), order="F")), OA(np.zeros((0, n), order="F")))
    np.testing.assert_array_equal(c.to_numpy(), co.arr)
    assert (co.arr == 0).all()


def test_matmul_empty_result(ftn):
    for m, k, n in ((0, 4, 3), (4, 3, 0), (0, 0, 0)):
        c = ftn.FArray.empty((m, n))
        ftn.matmul(c, ftn.FArray.empty((m, k)), ftn.FArray.empty((k, n)))
    torch.cuda.synchronize()


def test_elemental_and_sum_on_empty_sections(ftn):
    a = ftn.FArray.from_numpy(np.arange(20.0).reshape(4, 5, order="F"))
    before = a.to_numpy().copy()
    e = a.section((3, 2), (1, 5))                 # a(3:2, :): no elements
    ftn.muladd(e, e, 2.0, 1.0)
    ftn.fill(e, 7.0)
    np.testing.assert_array_equal(a.to_numpy(), before)
    assert float(ftn.sum(e).item()) == 0.0
    assert float(ftn.sum(a.section((1, 4), (5, 4))).item()) == 0.0
