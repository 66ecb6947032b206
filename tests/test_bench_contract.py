"""bench.py keeps the driver's JSON contract (CPU: the reference arm; GPU: the b200 arm)."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def run(args, timeout=600):
    r = subprocess.run([sys.executable, "bench.py", *args], cwd=ROOT, capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_contract():
    d = run(["--impl", "reference", "--workload", "c1", "--steps", "2", "--warmup", "1"])
    assert d["impl"] == "reference" and d["unit"] == "Gmulmod/s" and d["value"] > 0
    for k in ("metric", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "config", "cpu_baseline", "e2e"):
        assert k in d
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "oracle"


@pytest.mark.gpu
def test_b200_arm_contract():
    d = run(["--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--soak", "0", "--e2e-steps", "1"])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "clocks", "e2e", "gpu_launches", "kernels"):
        assert k in d, k
    assert d["steps"] == 3 and d["n_gpus"] == 1 and d["value"] > 0 and d["gpu_launches"] == 21
    assert all(d["parity"]["checks"].values())
    assert d["roofline"]["bound"] in ("hbm", "alu") and 0 < d["roofline"]["frac"] < 1.5
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    import oracle
    import synth
    want = []
    for P in synth.CONFIG_PRIMES:   # the step's configs[1] checksums, computed by the oracle
        a, b = synth.c2_inputs(P, 0, 1 << 26)
        want.append(oracle.checksum(P, oracle.mont_mul(P, a, b)))
    assert d["parity"]["box_checksums"] == want
