"""Writes tests/golden/c5_checksum.json: the configs[4] box checksum (sum over all n = 2^31
elements of REDC(a_i, b_i), mod P = 2013265921) computed by the ORACLE ONLY (oracle/, plain
naive-% definitions) on the shared seeded inputs (synth/), streamed in chunks on the host cores.
Also the checksum of every 1/W slice for W in {1, 2, 4, 8}, so a sharded run can be checked
rank by rank.  bench.py compares its box checksum (and tests/test_gpu_fullsize.py its C5 run)
against this file; nothing in it comes from the CUDA path.

    python scripts/golden_c5.py        (about a minute on 8 cores)
"""
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import oracle  # noqa: E402
import synth  # noqa: E402

P = 2013265921
N = 1 << 31
CHUNK = 1 << 25


def main():
    t0 = time.time()
    raw = []   # uint64 raw sums per chunk
    for lo in range(0, N, CHUNK):
        a, b = synth.c5_inputs(P, lo, CHUNK)
        raw.append(oracle.raw_sum(oracle.mont_mul(P, a, b)))
    slices = {}
    for W in (1, 2, 4, 8):
        per = N // W // CHUNK
        slices[str(W)] = [sum(raw[r * per:(r + 1) * per]) % P for r in range(W)]
    box = sum(raw) % P
    assert all(sum(v) % P == box for v in slices.values())
    out = {"_source": "scripts/golden_c5.py: oracle.mont_mul + oracle.raw_sum over synth.c5_inputs, chunked "
                      "(oracle/ only; SURVEY.md §8(c) sharding pin: the checksum is identical for W = 1, 2, 4, 8)",
           "P": P, "n": N, "seed": synth.DEFAULT_SEED, "box_checksum_mod_P": box,
           "rank_checksums_mod_P": slices, "seconds": round(time.time() - t0, 1), "host_cores": os.cpu_count()}
    (ROOT / "tests" / "golden" / "c5_checksum.json").write_text(json.dumps(out, indent=1) + "\n")
    print(json.dumps(out))


if __name__ == "__main__":
    main()
