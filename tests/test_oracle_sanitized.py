"""The oracle's own pins re-run against an AddressSanitizer + UndefinedBehaviorSanitizer build
of oracle/ftn_oracle.c (sanitizers on the oracle build).  Any out-of-bounds access,
use-after-free or undefined behaviour inside the oracle aborts the child run."""
import os
import subprocess
import sys

import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _runtime(name):
    r = subprocess.run(["gcc", f"-print-file-name={name}"], capture_output=True, text=True)
    path = r.stdout.strip()
    return path if os.path.isabs(path) and os.path.exists(path) else None


@pytest.mark.slow
def test_oracle_pins_under_asan_ubsan():
    asan = _runtime("libasan.so")
    if asan is None:
        pytest.skip("libasan not available")
    san = oracle.build(sanitize=True)
    env = dict(os.environ, LD_PRELOAD=asan, FTN_ORACLE_LIB=san, ASAN_OPTIONS="detect_leaks=0:abort_on_error=1",
               UBSAN_OPTIONS="halt_on_error=1:print_stacktrace=1")
    files = [os.path.join("tests", f) for f in sorted(os.listdir(os.path.join(ROOT, "tests")))
             if f.startswith("test_oracle_") and f != "test_oracle_sanitized.py"]
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider", *files], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, (r.stdout[-3000:] + r.stderr[-3000:])
