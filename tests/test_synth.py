"""The seeded generator (synth) -- DESIGN.md section 5.  Not method arithmetic."""
import numpy as np

import synth


def test_splitmix64_reference_vector():
    """Vigna's splitmix64 from state 0: outputs of states gamma and 2*gamma
    (published reference sequence e220a8397b1dcdaf, 6e789e6aa1b965f4)."""
    g = 0x9E3779B97F4A7C15
    out = synth.splitmix64(np.array([0, g], dtype=np.uint64))
    assert [int(v) for v in out] == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4]


def test_modes_ranges_and_determinism():
    n = 100000
    u = synth.values(n, mode=synth.U01)
    assert u.min() >= 0.0 and u.max() < 1.0 and abs(u.mean() - 0.5) < 0.01
    v = synth.values(n, mode=synth.U11)
    np.testing.assert_array_equal(v, 2.0 * u - 1.0)
    k = synth.values(n, mode=synth.INT8)
    assert k.min() == -8 and k.max() == 8 and np.all(k == np.rint(k))
    np.testing.assert_array_equal(synth.values(n, mode=synth.U01), u)
    assert not np.array_equal(synth.values(n, array_id=1), u)
    np.testing.assert_array_equal(synth.values(10, start=5), u[5:15])
    a = synth.farray((4, 3), mode=synth.LINEAR)
    assert a[1, 2] == 1 + 4 * 2                      # element order is column-major


def test_jacobi_init_faces():
    u = synth.jacobi_init((6, 5))
    assert (u[:, 0] == 1.0).all() and (u[0, 1:] == 0).all() and (u[-1, 1:] == 0).all() and (u[:, -1] == 0).all()
    assert (u[1:-1, 1:-1] > 0).all() or (u[1:-1, 1:-1] >= 0).all()
