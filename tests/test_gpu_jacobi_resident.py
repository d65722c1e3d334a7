"""GPU parity: the SMEM-resident 2-D Jacobi (one cooperative launch for all sweeps, neighbour
flags instead of a grid barrier) vs the oracle's DO nest with swapped arrays,
bit-exact on BOTH arrays: the result array holds iterate S, the other iterate S-1, and each
array keeps its own boundary values (u and unew may carry different boundaries)."""
import numpy as np
import pytest
import torch

import oracle
import synth
from oracle import FArray as OA

pytestmark = pytest.mark.gpu
C2 = 0.25


@pytest.fixture(scope="module")
def ftn():
    from paper_2409_18824_b200 import ftn
    yield ftn
    ftn.jacobi_set_resident(0, 0)


def _fits(shape, K):
    """The resident planner's rule (stencil_res.cu resident_plan): the register slab (n1 <= 1024,
    owned + 2K rows <= 16) or both iterates of the largest row slab plus K halo rows per side in
    227 KB of shared memory; every CTA owning >= K rows."""
    n1, n2 = shape
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    pitch = (n1 + 1) & ~1
    for reg in (True, False):
        if reg and n1 > 1024:
            continue
        for k in ([K] if K else [4, 3, 2, 1]):
            g = min(sms, (n2 - 2) // k)
            if g < 1:
                continue
            rows = -(-(n2 - 2) // g) + 2 * k
            if reg and rows <= 16:
                return True
            if not reg and 2 * rows * pitch * 8 <= 227 * 1024:
                return True
    return False


def _both(ftn, u0, w0, sweeps, lbs=None, resident=True):
    """Both arrays vs the oracle when the resident path runs; else the result array only (the
    streaming kernels leave an earlier iterate, not necessarily S-1, in the other array)."""
    U, W = ftn.FArray.from_numpy(u0, lbs), ftn.FArray.from_numpy(w0, lbs)
    n0 = ftn.launch_count()
    in_new = ftn.jacobi(U, W, sweeps, C2)
    launches = ftn.launch_count() - n0
    uo, wo = u0.copy(order="F"), w0.copy(order="F")
    in_new_o = oracle.jacobi(OA(uo, lbs), OA(wo, lbs), sweeps, C2)
    assert in_new == in_new_o
    if resident:
        np.testing.assert_array_equal(U.to_numpy(), uo)
        np.testing.assert_array_equal(W.to_numpy(), wo)
    else:
        np.testing.assert_array_equal((W if in_new else U).to_numpy(), wo if in_new else uo)
    return launches


def _w0(u0, seed, own_boundary=True):
    """unew: garbage interior and, for the resident path, its own boundary ring (the DO nest
    with swapped arrays reads each array's boundary; the streaming kernels assume the caller
    preset equal rings, R#16, so they get u0's ring)."""
    rng = np.random.default_rng(seed)
    w0 = np.asfortranarray(rng.uniform(-3.0, 3.0, u0.shape))
    if not own_boundary:
        w0 = u0.copy(order="F")
        w0[1:-1, 1:-1] = rng.uniform(-3.0, 3.0, (u0.shape[0] - 2, u0.shape[1] - 2))
    return w0


@pytest.mark.parametrize("K", [0, 1, 2, 3, 4])
@pytest.mark.parametrize("shape", [(3, 3), (4, 5), (5, 40), (40, 5), (129, 31), (200, 301), (257, 77),
                                   (1000, 130), (1024, 1024), (1025, 1023)])
@pytest.mark.parametrize("sweeps", [4, 5, 8, 13])
def test_resident_vs_oracle(ftn, K, shape, sweeps):
    ftn.jacobi_set_resident(1, K)
    u0 = synth.jacobi_init(shape, array_id=sum(shape) + sweeps)
    fits = _fits(shape, K)
    launches = _both(ftn, u0, _w0(u0, sum(shape) + K, fits), sweeps, [0, -3], resident=fits)
    if K == 0:                    # every one of these grids fits with the automatic K: one launch
        assert fits and launches == 1


@pytest.mark.parametrize("sweeps", [1, 2, 3, 41, 200])
def test_resident_sweep_counts(ftn, sweeps):
    ftn.jacobi_set_resident(1, 0)
    u0 = synth.jacobi_init((301, 700), array_id=sweeps)
    assert _both(ftn, u0, u0.copy(order="F"), sweeps) == 1


def test_resident_many_ctas_few_rows(ftn):
    """interior rows < num_SMs * K: fewer CTAs, every one owning >= K rows."""
    for n2 in (6, 9, 20, 150, 300, 445):
        for K in (1, 2, 3, 4):
            ftn.jacobi_set_resident(1, K)
            u0 = synth.jacobi_init((70, n2), array_id=n2 + K)
            fits = _fits((70, n2), K)
            _both(ftn, u0, _w0(u0, n2, fits), 9, resident=fits)


def test_resident_strided_sections(ftn):
    """Generic strides: sections of larger parents (odd leading dims, every other column)."""
    ftn.jacobi_set_resident(1, 0)
    P = synth.jacobi_init((301, 420), array_id=7)
    Q = _w0(P, 8)
    PU, PW = ftn.FArray.from_numpy(P), ftn.FArray.from_numpy(Q)
    U, W = PU.section((1, 301, 2), (11, 410)), PW.section((1, 301, 2), (11, 410))
    in_new = ftn.jacobi(U, W, 9, C2)
    pu, pw = P.copy(order="F"), Q.copy(order="F")
    ou, ow = OA(pu).section((1, 301, 2), (11, 410)), OA(pw).section((1, 301, 2), (11, 410))
    assert in_new == oracle.jacobi(ou, ow, 9, C2)
    np.testing.assert_array_equal(PU.to_numpy(), pu)
    np.testing.assert_array_equal(PW.to_numpy(), pw)


def test_resident_matches_streaming_kernels(ftn):
    """The resident and the streaming paths give the same result array bit for bit."""
    u0 = synth.jacobi_init((1024, 1024), array_id=99)
    out = []
    for mode in (1, 0):
        ftn.jacobi_set_resident(mode, 0)
        U, W = ftn.FArray.from_numpy(u0), ftn.FArray.from_numpy(u0)
        in_new = ftn.jacobi(U, W, 100)
        out.append(((W if in_new else U).to_numpy(), in_new))
    ftn.jacobi_set_resident(0, 0)
    assert out[0][1] == out[1][1]
    np.testing.assert_array_equal(out[0][0], out[1][0])


def test_resident_paper_shape_sampled(ftn):
    """The paper's jacobi grid 1024^2 for 2000 sweeps (10^5 in the bench): the discrete-harmonic
    field i*j is a bit-exact fixed point of the DO nest."""
    i, j = np.meshgrid(np.arange(1024.0), np.arange(1024.0), indexing="ij")
    h = np.asfortranarray(i * j)                    # discrete harmonic: a bit-exact fixed point
    ftn.jacobi_set_resident(1, 0)
    U, W = ftn.FArray.from_numpy(h), ftn.FArray.from_numpy(h)
    in_new = ftn.jacobi(U, W, 2000)
    np.testing.assert_array_equal((W if in_new else U).to_numpy(), h)


def test_resident_set_errors(ftn):
    for args in ((-1, 0), (4, -1), (4, 9)):
        with pytest.raises(ftn.FtnError):
            ftn.jacobi_set_resident(*args)
    ftn.jacobi_set_resident(0, 0)


def test_resident_on_side_stream_and_graph(ftn):
    """Stream-ordered (flags workspace from the stream's pool) and capturable in a CUDA graph."""
    ftn.jacobi_set_resident(1, 0)
    u0 = synth.jacobi_init((500, 600), array_id=5)
    U, W = ftn.FArray.from_numpy(u0), ftn.FArray.from_numpy(u0)
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        ftn.jacobi(U, W, 6, stream=s)                 # warm-up (attributes, pool)
        s.synchronize()
        with torch.cuda.graph(g, stream=s):
            ftn.jacobi(U, W, 6, stream=s)
    U2, W2 = ftn.FArray.from_numpy(u0), ftn.FArray.from_numpy(u0)
    U.tensor.copy_(U2.tensor)
    W.tensor.copy_(W2.tensor)
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    ftn.jacobi(U2, W2, 6)
    np.testing.assert_array_equal(U.to_numpy(), U2.to_numpy())
    np.testing.assert_array_equal(W.to_numpy(), W2.to_numpy())


def test_resident_fuzz(ftn):
    """Random shapes (both the register and the shared-memory slab), halo depths, sweep counts
    and lower bounds; both arrays bit-exact vs the oracle whenever the resident path runs."""
    rng = np.random.default_rng(1824)
    ran = 0
    try:
        for it in range(120):
            shape = (int(rng.integers(3, 1200)), int(rng.integers(3, 700)))
            K = int(rng.integers(0, 5))
            sweeps = int(rng.integers(1, 40))
            lbs = [int(v) for v in rng.integers(-4, 5, 2)]
            ftn.jacobi_set_resident(1, K)
            u0 = synth.jacobi_init(shape, array_id=it)
            fits = _fits(shape, K)
            _both(ftn, u0, _w0(u0, it, fits), sweeps, lbs, resident=fits)
            ran += fits
    finally:
        ftn.jacobi_set_resident(0, 0)
    assert ran > 60
