"""CPU: bench.py's command line and the reference arm's JSON line (the driver
contract): --impl reference runs the oracle on the headline's config, honours --sweeps /
--seed / --mode, and bad --config values are rejected before any work."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                          timeout=600, cwd=ROOT)


def test_reference_line_follows_the_cli():
    r = _run("--impl", "reference", "--steps", "1", "--warmup", "0", "--sweeps", "1", "--seed", "7",
             "--mode", "closed")
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["metric"].endswith("1 sweeps per step)")
    assert line["config"]["seed"] == 7 and line["config"]["input_mode"] == "closed"
    assert line["config"]["global_grid"] == "8192x8192" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "oracle"


def test_bad_config_is_rejected():
    r = _run("--config", "C9", "--impl", "reference")
    assert r.returncode == 2 and "unknown" in r.stderr
