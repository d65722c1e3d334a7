"""The C ABI from plain C (examples/c_api_demo.c, no Python in the loop): compiled with gcc
against include/ftn.h and libftn.so, run, and its output compared with the oracle."""
import os
import subprocess

import numpy as np
import pytest

import oracle
import synth
from oracle import FArray as OA

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_c_program_matches_oracle(tmp_path):
    exe = tmp_path / "c_api_demo"
    lib = os.path.join(ROOT, "paper_2409_18824_b200")
    cuda = os.environ.get("CUDA_HOME", "/usr/local/cuda")
    subprocess.run(["gcc", "-O2", os.path.join(ROOT, "examples", "c_api_demo.c"), "-I", os.path.join(ROOT, "include"),
                    "-I", os.path.join(cuda, "include"), "-L", lib, "-lftn", "-L", os.path.join(cuda, "lib64"),
                    "-lcudart", f"-Wl,-rpath,{lib}", f"-Wl,-rpath,{os.path.join(cuda, 'lib64')}", "-o", str(exe)],
                   check=True)
    out = tmp_path / "out.bin"
    r = subprocess.run([str(exe), str(out)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    raw = out.read_bytes()
    total = np.frombuffer(raw[:8], dtype=np.float64)[0]
    in_unew = bool(np.frombuffer(raw[8:12], dtype=np.int32)[0])
    n1, n2 = 300, 200
    got = np.frombuffer(raw[12:], dtype=np.float64).reshape((n1, n2), order="F")
    u0 = synth.jacobi_init((n1, n2))           # the same recipe as the C program
    uo, wo = u0.copy(order="F"), u0.copy(order="F")
    new = oracle.jacobi(OA(uo, [0, -5]), OA(wo, [0, -5]), 10, 0.25)
    ref = wo if new else uo
    assert in_unew == new
    np.testing.assert_array_equal(got, ref)
    assert total == oracle.reduce_orderR(OA(ref, [0, -5]).section((0, n1 - 1, 2), (-5, n2 - 6, 1)), oracle.SUM)


def test_c1_latency_program(tmp_path):
    """examples/c1_latency.c (the bench's C-ABI latency leg) builds, runs and finds the C1
    closed form SUM(a(::2,:)) = 2357760 through plain C calls."""
    import json
    exe = tmp_path / "c1_latency"
    lib = os.path.join(ROOT, "paper_2409_18824_b200")
    cuda = os.environ.get("CUDA_HOME", "/usr/local/cuda")
    subprocess.run(["gcc", "-O2", os.path.join(ROOT, "examples", "c1_latency.c"), "-I", os.path.join(ROOT, "include"),
                    "-I", os.path.join(cuda, "include"), "-L", lib, "-lftn", "-L", os.path.join(cuda, "lib64"),
                    "-lcudart", f"-Wl,-rpath,{lib}", f"-Wl,-rpath,{os.path.join(cuda, 'lib64')}", "-o", str(exe)],
                   check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert d["sum_closed_form_ok"] is True
    assert set(d["sync_median_us"]) == set(d["back_to_back_mean_us"]) and len(d["sync_median_us"]) == 6


def test_c_linalg_program_matches_oracle(tmp_path):
    """examples/c_api_linalg.c: MATMUL (within the R#8 bound of the oracle), TRANSPOSE (exact) and
    ftn_jacobi_solve (sweeps, residual, result-in-unew and the result array, exact) from plain C."""
    exe = tmp_path / "c_api_linalg"
    lib = os.path.join(ROOT, "paper_2409_18824_b200")
    cuda = os.environ.get("CUDA_HOME", "/usr/local/cuda")
    subprocess.run(["gcc", "-O2", "-Wall", "-Werror", os.path.join(ROOT, "examples", "c_api_linalg.c"), "-I",
                    os.path.join(ROOT, "include"), "-I", os.path.join(cuda, "include"), "-L", lib, "-lftn", "-L",
                    os.path.join(cuda, "lib64"), "-lcudart", f"-Wl,-rpath,{lib}",
                    f"-Wl,-rpath,{os.path.join(cuda, 'lib64')}", "-o", str(exe)], check=True)
    out = tmp_path / "out.bin"
    r = subprocess.run([str(exe), str(out)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    raw = out.read_bytes()
    sweeps = int(np.frombuffer(raw[:8], dtype=np.int64)[0])
    residual = float(np.frombuffer(raw[8:16], dtype=np.float64)[0])
    in_unew = bool(np.frombuffer(raw[16:20], dtype=np.int32)[0])
    m, k, n, n1, n2 = 64, 80, 48, 130, 90
    vals = np.frombuffer(raw[20:], dtype=np.float64)
    c = vals[:m * n].reshape((m, n), order="F")
    at = vals[m * n:m * n + k * m].reshape((k, m), order="F")
    res = vals[m * n + k * m:].reshape((n1, n2), order="F")
    a = synth.farray((m, k), array_id=1, mode=synth.U11)
    b = synth.farray((k, n), array_id=2, mode=synth.U11)
    co, absum = np.zeros((m, n), order="F"), np.zeros((m, n), order="F")
    oracle.matmul(OA(co), OA(a), OA(b), OA(absum))
    assert np.all(np.abs(c - co) <= 4 * k * 2.0 ** -53 * absum)
    np.testing.assert_array_equal(at, a.T)
    u0 = synth.jacobi_init((n1, n2))
    uo, wo = u0.copy(order="F"), u0.copy(order="F")
    d, rr, new = oracle.jacobi_solve(OA(uo), OA(wo), 3000, 10, 1e-6, 0.25)
    assert (sweeps, residual, in_unew) == (d, rr, new)
    np.testing.assert_array_equal(res, wo if new else uo)
