"""Sweep of the two-lane step's launch shapes (bench.py's graph-replayed step): the pow lane's
variant / CTAs per SM and the HBM lane's launch configurations.  One JSON object per shape;
outputs are re-verified after each timing (bench.verify on the graph's buffers).  Not part of the
product; picks bench.py's defaults.

    python scripts/step_sweep.py [--shapes NAME,...]
"""
import itertools
import json
import os
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import bench  # noqa: E402


def main():
    torch.cuda.set_device(0)
    bench.POW_CTAS, bench.POW_VARIANT = 2, 11
    wl = bench.Workload("step", 0, 1)
    m = wl.m
    assert all(bench.verify(wl).values())
    L = m.Launch
    # (variant, ctas_per_sm, reserved smem bytes): ctas 0 = flat grid
    pows = [tuple(int(x) for x in (v.split(":") + ["256"])[:4]) for v in
            os.environ.get("SWEEP_POWS", "10:1:0,11:1:0,10:2:0").split(",")]   # variant:ctas:smem[:threads]
    prios = [None if v == "none" else v for v in os.environ.get("SWEEP_PRIOS", "imad").split(",")]
    hstreams = [int(v) for v in os.environ.get("SWEEP_HBM_STREAMS", "1").split(",")]
    modes = os.environ.get("SWEEP_HBM_MODES", "streams").split(",")
    shapes = [tuple(int(x) for x in v.split("x")) for v in os.environ.get("SWEEP_RUN_SHAPES", "256x2").split(",")]
    if os.environ.get("SWEEP_WIDE"):
        pows = [(11, 0, 0), (11, 0, 200 * 1024), (11, 0, 110 * 1024), (11, 0, 72 * 1024), (11, 0, 54 * 1024),
                (11, 1, 0), (11, 2, 0), (10, 2, 0)]
        prios = [None, "hbm", "imad"]
    hbms = {
        "default": {},   # mul+checksum 512 x 2, to/from 512 x 2, twiddle flat 512 x 4
        "u2": {"mul": L(threads=256, unroll=2), "conv": L(threads=512, unroll=2), "tw": None},
        "m256u1": {"mul": L(threads=256, unroll=1)},
        "m256u4": {"mul": L(threads=256, unroll=4)},
        "m1024u1": {"mul": L(threads=1024, unroll=1)},
        "c256u2": {"conv": L(threads=256, unroll=2)},
        "c256u4": {"conv": L(threads=256, unroll=4)},
        "t256u4": {"tw": L(threads=256, unroll=4, variant=2)},
        "t512u2": {"tw": L(threads=512, unroll=2, variant=2)},
        "t256u8": {"tw": L(threads=256, unroll=8, variant=2)},
        "all256u4": {"mul": L(threads=256, unroll=4), "conv": L(threads=256, unroll=4),
                     "tw": L(threads=256, unroll=4, variant=2)},
        "u2c4": {"mul": L(threads=256, unroll=2), "conv": L(threads=256, unroll=4)},
        "u2c4tma": {"mul": L(threads=256, unroll=2), "conv": L(threads=256, unroll=4), "tw": L(variant=4)},
        "u2c4tma4k": {"mul": L(threads=256, unroll=2), "conv": L(threads=256, unroll=4), "tw": L(variant=4, chunk=4096)},
        "m256u1tma": {"mul": L(threads=256, unroll=1), "tw": L(variant=4)},
        "m256u4tma": {"mul": L(threads=256, unroll=4), "tw": L(variant=4)},
        "m512u2tma": {"mul": L(threads=512, unroll=2), "tw": L(variant=4)},
        "m128u4tma": {"mul": L(threads=128, unroll=4), "tw": L(variant=4)},
        "m512u1tma": {"mul": L(threads=512, unroll=1), "tw": L(variant=4)},
        "fp64mul": {"mul": L(threads=256, unroll=2, variant=4), "conv": L(threads=256, unroll=4)},
        "fp64mul512": {"mul": L(threads=512, unroll=2, variant=4), "conv": L(threads=256, unroll=4)},
    }
    only = os.environ.get("SWEEP_HBM")
    rebuilds = int(os.environ.get("SWEEP_REBUILDS", "2"))
    pdls = [v == "1" for v in os.environ.get("SWEEP_PDL", "0").split(",")]
    for (pv, pc, sm, pt), (hname, hcfg), prio, hs, mode, shape, pdl in itertools.product(
            pows, hbms.items(), prios, hstreams, modes, shapes, pdls):
        if only and hname not in only.split(","):
            continue
        if mode == "run" and (hs != 1 or hname != "default"):
            continue   # the run has its own launch shape and one launch
        if mode == "streams" and shape != shapes[0]:
            continue
        bench.HBM_STREAMS, bench.HBM_MODE, bench.RUN_SHAPE = hs, mode, shape
        for attr in ("_run_launch", "_pair_launch", "_pair_mode"):
            if hasattr(wl, attr):
                delattr(wl, attr)
        wl.pow_cfg_lane = L(ctas_per_sm=pc, variant=pv, chunk=sm, threads=pt)
        wl.hbm_cfg_lane = {k: v for k, v in hcfg.items() if v is not None}
        bench.PDL = pdl
        wl.hbm_cfg_lane_pdl = {k: L(threads=v.threads, ctas_per_sm=v.ctas_per_sm, unroll=v.unroll, variant=v.variant,
                                    chunk=v.chunk, flags=1) for k, v in wl.hbm_cfg_lane.items()}
        wl.hbm_cfg_lane_pdl.setdefault("tw", L(flags=1))
        # lane streams: torch priority -1 = high, 0 = low (graph kernel nodes inherit it)
        wl._lanes = {"hbm": torch.cuda.Stream(priority=-1 if prio == "hbm" else 0),
                     "imad": torch.cuda.Stream(priority=-1 if prio == "imad" else 0)}
        wl._hbm_extra = []
        for rb in range(rebuilds):
            try:
                g = bench.capture_step_graph(wl)
            except Exception as ex:  # noqa: BLE001
                print(json.dumps({"pow": [pv, pc, sm, pt], "hbm": hname, "error": str(ex)}), flush=True)
                break
            for _ in range(3):
                g.replay()
            torch.cuda.synchronize()
            ts = [bench.time_steps_graph(wl, g, 20) / 20 for _ in range(3)]
            ok = all(bench.verify(wl, run=False).values())
            print(json.dumps({"pow": [pv, pc, sm, pt], "hbm": hname, "prio": prio, "hbm_streams": hs, "mode": mode,
                              "pdl": pdl,
                              "run_shape": list(shape) if mode != "streams" else None,
                              "rebuild": rb,
                              "ms_per_step": round(statistics.median(ts), 4), "ms_best": round(min(ts), 4),
                              "outputs_ok": ok}), flush=True)
            del g


if __name__ == "__main__":
    main()
