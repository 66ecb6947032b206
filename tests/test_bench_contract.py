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
    assert d["steps"] == 3 and d["n_gpus"] == 1 and d["value"] > 0 and d["gpu_launches"] % 3 == 0 and 6 <= d["gpu_launches"] <= 21
    assert all(d["parity"]["checks"].values())
    assert d["roofline"]["bound"] in ("hbm", "alu") and 0 < d["roofline"]["frac"] < 1.5
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    # configs[4] and configs[0] ride along: box checksum = the oracle's (tests/golden/c5_checksum.json)
    assert d["c5"]["checksum_ok"] and d["c5"]["identity_all_elements"] and d["c5"]["n_total"] == 1 << 31
    assert d["c1"]["checksum_ok"] and d["c1"]["latency_us"]["host_call_to_completion"] > 0
    assert all(d["parity"]["timed_graph_outputs"].values())
    import oracle
    import synth
    want = []
    for P in synth.CONFIG_PRIMES:   # the step's configs[1] checksums, computed by the oracle
        a, b = synth.c2_inputs(P, 0, 1 << 26)
        want.append(oracle.checksum(P, oracle.mont_mul(P, a, b)))
    assert d["parity"]["box_checksums"] == want


def test_gpus_flag_spawns_ranks():
    """`bench.py --gpus 2` with no launcher starts 2 ranks itself (torch.distributed.run on
    127.0.0.1); exactly one JSON line comes back, from rank 0, with n_gpus = 2 (CPU: the
    reference arm, which needs no GPU)."""
    d = run(["--impl", "reference", "--workload", "c1", "--steps", "1", "--warmup", "0", "--gpus", "2"])
    assert d["impl"] == "reference" and d["n_gpus"] == 2


def test_gpus_flag_must_match_launcher():
    import os
    env = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--workload", "c1", "--gpus", "1"],
                       cwd=ROOT, capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 2 and "disagrees with WORLD_SIZE" in r.stdout


@pytest.mark.gpu
def test_b200_arm_two_ranks_on_one_gpu():
    """`--gpus 2` launches two ranks itself; on the single gpurun GPU they share it in the
    orchestration dry-run mode (gloo collectives on the CPU, kernels of different ranks never wait
    on each other).  Two ranks report n_gpus 2, slice configs[4] in halves, and the box checksum
    is still the oracle's."""
    import os
    env = dict(os.environ, MONT_SHARE_GPU="1", MONT_DIST_BACKEND="gloo")
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--steps", "3", "--warmup", "3", "--soak", "0",
                        "--no-cpu-baseline", "--no-e2e"], cwd=ROOT, capture_output=True, text=True, timeout=900,
                       env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["c5"]["ranks"] == 2 and d["c5"]["n_rank"] == 1 << 30
    assert d["c5"]["checksum_ok"] and all(d["parity"]["checks"].values())


@pytest.mark.gpu
@pytest.mark.parametrize("workload", ["c1", "c2", "c3", "c4", "c5", "ntt"])
def test_b200_arm_each_workload(workload):
    """Every --workload prints one line whose parity checks (before timing and on the timed
    graph's outputs) all hold."""
    d = run(["--workload", workload, "--steps", "3", "--warmup", "3", "--soak", "0", "--no-cpu-baseline", "--no-e2e"])
    assert d["value"] > 0 and all(d["parity"]["checks"].values())
    assert all(d["parity"].get("timed_graph_outputs", {}).values())
