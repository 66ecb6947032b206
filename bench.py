#!/usr/bin/env python
"""bench.py -- the driver's benchmark contract for the batched 32-bit Montgomery path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl {b200,reference}]
                    [--workload {step,c1,c2,c3,c4,c5,ntt}]

One "step" (default workload) is one pass of the whole hot path of
SURVEY.md §8(a) (rows A1-A11) over one batch of synthetic input, per rank:

  A1   mont_ctx_init for the three config primes (host)
  A7   mont_mul_vec_checksum  configs[1]: n = 2^26 pairs with 1 % specials, for
                      each of P in {2013265921, 469762049, 998244353}, with the
                      A11 checksum partial fused into the same pass (3 launches)
  A2   to_mont        the P0 operand a (2^26)                      (1 launch)
  A10  from_mont      back again (2^26)                            (1 launch)
  A8   mont_mul_twiddle configs[2]: 4096 x 2^14 against tw[j] = to_mont(w^j)
  A9   mont_pow_vec   configs[3]: 2^24 bases/exponents, P = 469762049
  A11  the cross-rank NCCL all-reduce of the checksum partials runs once,
                      after timing

metric/unit are BASELINE.json's: useful Montgomery products per second
(Gmulmod/s) of the whole job: C2 3*2^26 + to/from 2*2^26 + C3 2^26 + C4
sum_i(31 + popcount(exp_i)) ladder products.  Inputs are generated in HBM by
the device generator (synth_fill) from the GLOBAL element index, so rank r of
N processes slice r of an N-times larger job (weak scaling, no data-path
collective).  The step's working set (~3.3 GiB) is far larger than the
126 MB L2, so no L2 flush is needed between steps (configs[0], 768 KiB, is
timed step by step after an L2 flush instead).  The other workloads time one
config each (c1..c5 = BASELINE configs[0..4]; ntt = SURVEY §8(f) NEXT #1).

Besides `value`, the line carries `roofline` (the dominant kernel against the
measured HBM copy rate, the nominal 8 TB/s and an in-run triad), `kernels`
(every launch), `e2e` (the same step through the host-buffer executor
mont_host_run, copies inside the timed region), `cpu_baseline` (the oracle on
all host cores and on one), `clocks` and `parity`.

--impl reference times the CPU oracle (oracle/, the slow plain-definition
program) on a bounded sample of the same workload on the host cores; there
is no reference GPU implementation (the paper ships no code).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

P0, P1, P2 = 2013265921, 469762049, 998244353
PRIMES = (P0, P1, P2)
N_C2 = 1 << 26
TW_BATCH, TW_LEN = 4096, 1 << 14
N_C4 = 1 << 24
N_C5 = 1 << 31
SEED = 42
METRIC = json.loads((ROOT / "BASELINE.json").read_text())["metric"]
G11_GENERATOR = 31
POW_CTAS = 0   # set from --pow-ctas
POW_VARIANT = 0  # set from --pow-variant
LANE_ORDER = tuple(os.environ.get("MONT_LANE_ORDER", "imad,hbm").split(","))
# the lane whose stream gets the higher priority in the two-lane step (graph kernel nodes inherit
# it): the persistent pow grid is placed first, one CTA per SM, and the HBM-bound launches fill
# the rest of every SM (scripts/step_sweep.py, profiles/r02_step_sweep*.jsonl)
LANE_PRIO = os.environ.get("MONT_LANE_PRIO", "imad")
# the HBM lane of the step: "pair" (default) = the individual launches on HBM_STREAMS streams except
# to_mont -> from_mont, which run as ONE fused mont_run launch (0.599-0.601 ms per step);
# "streams" = all individual (0.630); "run" = one mont_run launch over all HBM jobs (fastest alone,
# 546 vs 598 us, but slower next to the pow lane: 0.64-0.65 ms) -- profiles/r02_step_sweep.jsonl
HBM_MODE = os.environ.get("MONT_HBM_MODE", "pair")
# tile shape of that mont_run launch inside the step (threads, uint4 per thread): 256-thread tiles
# leave the co-running pow grid the room 512-thread ones take (profiles/r02_step_sweep.jsonl)
RUN_SHAPE = tuple(int(v) for v in os.environ.get("MONT_RUN_SHAPE", "512,2").split(","))
# programmatic dependent launch inside the HBM lane: every HBM launch after the lane's first may
# start while the previous one drains (MONT_LAUNCH_OVERLAP_PREV; the lane's launches are independent)
PDL = os.environ.get("MONT_PDL", "1") == "1"
# streams the HBM-bound launches are spread over inside the step (independent launches only)
HBM_STREAMS = int(os.environ.get("MONT_HBM_STREAMS", "1"))


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="step", choices=["step", "c1", "c2", "c3", "c4", "c5", "ntt"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--soak", type=float, default=1.0, help="seconds of untimed steps before timing (clocks)")
    ap.add_argument("--serial", action="store_true", help="report the serial (one-stream) step instead")
    ap.add_argument("--no-graph", dest="graph", action="store_false",
                    help="issue the two-lane step launch by launch instead of replaying it as one CUDA graph")
    ap.add_argument("--pow-ctas", type=int, default=1, help="CTAs per SM of the persistent pow grid (0 = flat)")
    ap.add_argument("--pow-variant", type=int, default=10, help="mont_pow_vec_ex variant used in the lane schedule")
    ap.add_argument("--no-subruns", action="store_true", help="skip the configs[4] / configs[0] sub-objects")
    return ap.parse_args()


def launch_ranks(args):
    """`--gpus N` launches N ranks itself when no launcher did (one process per GPU under
    torch.distributed.run, rendezvous on 127.0.0.1); under a launcher, --gpus must equal
    WORLD_SIZE.  Returns the exit code of the child launcher, or None to run in this process."""
    ws = os.environ.get("WORLD_SIZE")
    if ws is not None:
        if int(ws) != args.gpus:
            print(json.dumps({"error": f"--gpus {args.gpus} disagrees with WORLD_SIZE={ws}"}), flush=True)
            return 2
        return None
    if args.gpus <= 1:
        return None
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(ROOT / "bench.py"), *sys.argv[1:]]
    return subprocess.call(cmd)


def dist_timeout():
    import datetime
    return datetime.timedelta(seconds=int(os.environ.get("MONT_DIST_TIMEOUT_S", "900")))


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured", float(d.get("sm_max_mhz", 1965.0))
    return 6650.0, "fallback", 1965.0


# ----------------------------------------------------------------- clocks

class ClockSampler:
    """nvidia-smi clock / throttle sampling during the timed region (B200_PROFILING.md)."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_id: str):
        self.gpu_id = gpu_id
        self.proc = None
        self.lines = []
        self.t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", self.gpu_id, f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, smax, reasons, n = [], None, set(), 0
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                cur, mx = float(f[0]), float(f[1])
            except ValueError:
                continue
            n += 1
            smax = mx
            if cur > 0.5 * mx:  # under load (idle samples read ~120-900 MHz)
                sm.append(cur)
            for nm, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": n, "samples_under_load": len(sm)}


# ----------------------------------------------------------------- workload

class Workload:
    """Device buffers + the list of launches that make one step on this rank."""

    def __init__(self, kind: str, rank: int, world: int):
        import torch

        import paper_1609_00999_b200 as m
        self.m, self.torch = m, torch
        self.kind, self.rank, self.world = kind, rank, world
        dev = torch.device("cuda", torch.cuda.current_device())
        self.dev = dev
        u32 = dict(dtype=torch.uint32, device=dev)
        self.ctx = {P: m.ctx_init(P) for P in PRIMES}          # A1
        self.launches = []     # (name, fn, algorithmic bytes, useful mulmods, bound)
        self.inputs, self.outputs = [], []                     # tensors copied in / out by e2e
        self.acc = torch.zeros(len(PRIMES), dtype=torch.int64, device=dev)
        self.config = {}
        # launch configurations of the HBM-bound launches in the two-lane step: mul_vec+checksum
        # 256 threads x 2 uint4, to/from 256 x 4 (the shapes that leave the co-running pow grid
        # most room, profiles/r02_step_sweep4.jsonl); the twiddle multiply keeps the library
        # default.  The serial pass uses the library defaults.
        self.hbm_cfg_lane = {"mul": m.Launch(threads=256, unroll=2), "conv": m.Launch(threads=256, unroll=4)}
        if os.environ.get("MONT_HBM_DEFAULTS") == "1":
            self.hbm_cfg_lane = {}
        ov = m.OVERLAP_PREV
        self.hbm_cfg_lane_pdl = {k: m.Launch(threads=v.threads, unroll=v.unroll, flags=ov)
                                 for k, v in self.hbm_cfg_lane.items()}
        self.hbm_cfg_lane_pdl.setdefault("tw", m.Launch(flags=ov))
        # one HBM lane alone (c2): the library-default shapes, flagged
        self.hbm_cfg_pdl_alone = {k: m.Launch(flags=ov) for k in ("mul", "conv", "tw")}
        self.run_flags = 0   # flags of the mont_run launches (set per launch by step_concurrent)
        self.hbm_cfg = {}    # the serial step: library defaults (each kernel's best standalone shape)
        self.lane_events = None
        L = self.launches
        if kind in ("step", "c2"):
            off = rank * N_C2
            self.c2 = {}
            for si, P in enumerate(PRIMES):
                a = torch.empty(N_C2, **u32)
                b = torch.empty(N_C2, **u32)
                c = torch.empty(N_C2, **u32)
                m.synth_fill(a, SEED, 1, off, P, 0, True)
                m.synth_fill(b, SEED, 2, off, P, 0, True)
                self.c2[P] = (a, b, c)
                self.inputs += [a, b]
                self.outputs.append(c)
                # A7 + A11 fused: c = REDC(a, b) and the checksum partial in one pass
                L.append((f"mont_mul_vec_checksum[P={P}]",
                          (lambda ctx=self.ctx[P], a=a, b=b, c=c, si=si:
                           m.mul_vec_checksum(ctx, a, b, out=c, acc=self.acc[si:si + 1],
                                              cfg=self.hbm_cfg.get("mul"))),
                          12 * N_C2, N_C2, "hbm"))
            self.config.update({"c2_n": N_C2, "c2_primes": list(PRIMES)})
        if kind == "step":
            a0 = self.c2[P0][0]
            abar = torch.empty(N_C2, **u32)
            back = torch.empty(N_C2, **u32)
            self.outputs.append(back)
            self.abar, self.back = abar, back
            L.append(("to_mont", lambda a0=a0, abar=abar: m.to_mont(self.ctx[P0], a0, out=abar,
                                                                     cfg=self.hbm_cfg.get("conv")), 8 * N_C2, N_C2, "hbm"))
            L.append(("from_mont", lambda abar=abar, back=back: m.from_mont(self.ctx[P0], abar, out=back,
                                                                            cfg=self.hbm_cfg.get("conv")),
                      8 * N_C2, N_C2, "hbm"))
        if kind in ("step", "c3"):
            x = torch.empty(TW_BATCH * TW_LEN, **u32)
            m.synth_fill(x, SEED, 5, rank * TW_BATCH * TW_LEN, P0, 0, False)
            x = x.view(TW_BATCH, TW_LEN)
            w = pow(G11_GENERATOR, (P0 - 1) // TW_LEN, P0)   # the config's root of unity (an input)
            tw = m.twiddle_table(self.ctx[P0], w, TW_LEN, device=dev)
            o = torch.empty_like(x)
            self.tw_x, self.tw, self.tw_out, self.w = x, tw, o, w
            self.inputs += [x]
            self.outputs.append(o)
            L.append(("mont_mul_twiddle", lambda x=x, tw=tw, o=o: m.mul_twiddle(self.ctx[P0], x, tw, out=o,
                                                                                 cfg=self.hbm_cfg.get("tw")),
                      8 * TW_BATCH * TW_LEN, TW_BATCH * TW_LEN, "hbm"))
            self.config.update({"c3_batch": TW_BATCH, "c3_len": TW_LEN})
        if kind in ("step", "c4"):
            base = torch.empty(N_C4, **u32)
            e = torch.empty(N_C4, **u32)
            o = torch.empty(N_C4, **u32)
            m.synth_fill(base, SEED, 3, rank * N_C4, P1, 1, False)
            m.synth_fill(e, SEED, 4, rank * N_C4, P1, 2, False)
            torch.cuda.synchronize()
            ladder = 31 * N_C4 + int(_popcount_sum(e))
            self.pow_bufs = (base, e, o)
            self.inputs += [base, e]
            self.outputs.append(o)
            # in the two-lane schedule pow runs as a persistent grid of POW_CTAS CTAs per SM so it
            # co-resides with the HBM-bound kernels instead of filling every SM first
            self.pow_cfg_lane = m.Launch(ctas_per_sm=POW_CTAS, variant=POW_VARIANT) if POW_CTAS > 0 else None
            self.pow_cfg = None   # flat grid (best standalone) unless a lane schedule is running
            L.append(("mont_pow_vec", lambda base=base, e=e, o=o:
                      m.pow_vec(self.ctx[P1], base, e, out=o, cfg=self.pow_cfg), 12 * N_C4, ladder, "imad"))
            self.config.update({"c4_n": N_C4, "c4_ladder_mulmods": ladder})
        if kind == "c1":
            # configs[0]: n = 65536 with the fixed-index edge values (G12); launch-latency bound
            import numpy as np

            import synth as _synth  # the shared input generator (no method arithmetic)
            ha, hb = _synth.c1_inputs(P0)
            a = torch.from_numpy(ha).to(dev)
            b = torch.from_numpy(hb).to(dev)
            c = torch.empty_like(a)
            self.c1 = (a, b, c)
            self.inputs += [a, b]
            self.outputs.append(c)
            L.append(("mont_mul_vec_checksum[c1]",
                      lambda a=a, b=b, c=c: m.mul_vec_checksum(self.ctx[P0], a, b, out=c, acc=self.acc[0:1]),
                      12 * a.numel(), a.numel(), "hbm"))
            self.config.update({"c1_n": a.numel()})
        if kind == "ntt":
            # forward NTT of the configs[2] batch (4096 rows of 2^14) over P0
            x = torch.empty(TW_BATCH * TW_LEN, **u32)
            m.synth_fill(x, SEED, 5, rank * TW_BATCH * TW_LEN, P0, 0, False)
            x = x.view(TW_BATCH, TW_LEN)
            w = pow(G11_GENERATOR, (P0 - 1) // TW_LEN, P0)
            tw = m.ntt_twiddles(self.ctx[P0], w, 14, device=dev)
            self.ntt_x, self.ntt_x0, self.ntt_w, self.ntt_tw = x, x.clone(), w, tw
            self.inputs += [x]
            self.outputs.append(x)
            redc = TW_BATCH * (TW_LEN // 2) * 14
            L.append(("mont_ntt", lambda x=x, tw=tw: m.ntt(self.ctx[P0], x, tw), 8 * TW_BATCH * TW_LEN, redc, "imad"))
            self.config.update({"ntt_batch": TW_BATCH, "ntt_n": TW_LEN, "ntt_redc_per_pass": redc})
        if kind == "c5":
            n = N_C5 // world
            lo = (rank * N_C5) // world
            a = torch.empty(n, **u32)
            b = torch.empty(n, **u32)
            c = torch.empty(n, **u32)
            m.synth_fill(a, SEED, 1, lo, P0, 0, False)
            m.synth_fill(b, SEED, 2, lo, P0, 0, False)
            self.c5 = (a, b, c)
            self.inputs += [a, b]
            self.outputs.append(c)
            L.append(("mont_mul_vec_checksum[c5]",
                      lambda a=a, b=b, c=c: m.mul_vec_checksum(self.ctx[P0], a, b, out=c, acc=self.acc[0:1]),
                      12 * n, n, "hbm"))
            self.config.update({"c5_n_total": N_C5, "c5_n_rank": n})
        torch.cuda.synchronize()

    @property
    def mulmods(self):
        return sum(x[3] for x in self.launches)

    @property
    def step_launches(self):
        """The launches of the two-lane step: the HBM-bound ones as ONE mont_run (include/
        mont_run.h: one flat grid over all their tiles, to_mont -> from_mont fused) when
        HBM_MODE == "run", else individually; the IMAD-bound ones as they are."""
        hbm = [x for x in self.launches if x[4] == "hbm"]
        if HBM_MODE in ("pair", "pairtw") and hasattr(self, "abar"):
            # the to_mont -> from_mont pair (pairtw: and the twiddle multiply) as one fused mont_run
            # launch, the rest individual
            with_tw = HBM_MODE == "pairtw" and hasattr(self, "tw_x")
            if getattr(self, "_pair_mode", None) != HBM_MODE:
                m = self.m
                self.pair_jobs = [m.run_job("to_mont", self.ctx[P0], self.abar, self.c2[P0][0]),
                                  m.run_job("from_mont", self.ctx[P0], self.back, self.abar)]
                if with_tw:
                    self.pair_jobs.append(m.run_job("twiddle", self.ctx[P0], self.tw_out.view(-1),
                                                    self.tw_x.view(-1), self.tw))
                self._pair_launch = ("mont_run[to_mont -> from_mont fused" + (", twiddle" if with_tw else "") + "]",
                                     lambda: m.run(self.pair_jobs, cfg=m.Launch(threads=RUN_SHAPE[0],
                                                                                unroll=RUN_SHAPE[1],
                                                                                flags=self.run_flags)),
                                     m.run_bytes(self.pair_jobs),
                                     2 * N_C2 + (TW_BATCH * TW_LEN if with_tw else 0), "hbm")
                self._pair_mode = HBM_MODE
            out = []
            for x in self.launches:
                if x[0] == "to_mont":
                    out.append(self._pair_launch)
                elif x[0] == "from_mont" or (with_tw and x[0] == "mont_mul_twiddle"):
                    continue
                else:
                    out.append(x)
            return out
        if HBM_MODE != "run" or len(hbm) < 2:
            return self.launches
        if not hasattr(self, "_run_launch"):
            m = self.m
            jobs = []
            for name, *_ in hbm:
                if name.startswith("mont_mul_vec_checksum[P="):
                    P = int(name.split("=")[1].rstrip("]"))
                    a, b, c = self.c2[P]
                    si = PRIMES.index(P)
                    jobs.append(m.run_job("mul_vec", self.ctx[P], c, a, b, acc=self.acc[si:si + 1]))
                elif name == "to_mont":
                    jobs.append(m.run_job("to_mont", self.ctx[P0], self.abar, self.c2[P0][0]))
                elif name == "from_mont":
                    jobs.append(m.run_job("from_mont", self.ctx[P0], self.back, self.abar))
                elif name == "mont_mul_twiddle":
                    jobs.append(m.run_job("twiddle", self.ctx[P0], self.tw_out.view(-1), self.tw_x.view(-1), self.tw))
                else:
                    raise RuntimeError(f"no mont_run job for {name}")
            self.run_jobs = jobs
            self.run_bytes = m.run_bytes(jobs)
            self._run_launch = ("mont_run[hbm lane: " + ", ".join(x[0] for x in hbm) + "]",
                                lambda: m.run(self.run_jobs, cfg=m.Launch(threads=RUN_SHAPE[0], unroll=RUN_SHAPE[1],
                                                                          flags=self.run_flags)),
                                self.run_bytes, sum(x[3] for x in hbm), "hbm")
        return [self._run_launch] + [x for x in self.launches if x[4] != "hbm"]

    def step(self):
        """Serial step: every launch in order on the current stream."""
        for _, fn, *_ in self.launches:
            fn()

    def step_concurrent(self):
        """The step as the runtime schedules it: the HBM-bound launches (mul_vec x3,
        to_mont -> from_mont, twiddle) in order on one stream and the FMAHeavy-bound
        pow ladder on a second stream, so the integer-multiply pipes and HBM work at
        the same time.  Both lanes are joined back into the current stream; the
        launches are independent (disjoint outputs), so results are identical."""
        torch = self.torch
        cur = torch.cuda.current_stream()
        # the persistent pow grid only pays when HBM-bound launches co-run with it
        launches = self.step_launches
        both = {b for *_, b in launches} >= {"hbm", "imad"}
        self.pow_cfg = getattr(self, "pow_cfg_lane", None) if both else None
        self.hbm_cfg = self.hbm_cfg_lane if both else {}   # lane shapes only next to a pow lane
        if not hasattr(self, "_lanes"):
            self._lanes = {ln: torch.cuda.Stream(priority=-1 if ln == LANE_PRIO else 0) for ln in ("hbm", "imad")}
        nh = max(1, HBM_STREAMS)
        if not hasattr(self, "_hbm_extra") or len(self._hbm_extra) != nh - 1:
            self._hbm_extra = [torch.cuda.Stream(priority=-1 if LANE_PRIO == "hbm" else 0) for _ in range(nh - 1)]
        hbm_streams = [self._lanes["hbm"]] + self._hbm_extra
        # HBM launches that do not depend on each other go to different streams (graph branches), so
        # one kernel's tail overlaps the next one's ramp; to_mont -> from_mont stay in order
        groups = []
        for name, *_rest in launches:
            g = "conv" if name in ("to_mont", "from_mont") else name
            if _rest[-1] == "hbm" and g not in groups:
                groups.append(g)
        m_ov = self.m.OVERLAP_PREV
        ev = torch.cuda.Event()
        ev.record(cur)
        for st in list(self._lanes.values()) + self._hbm_extra:
            st.wait_event(ev)
        started = set()   # streams that already carry an HBM launch of this step
        for lane in LANE_ORDER:
            for i, (name, fn, _, _, bound) in enumerate(launches):
                if bound != lane:
                    continue
                if lane == "hbm":
                    g = "conv" if name in ("to_mont", "from_mont") else name
                    st = hbm_streams[groups.index(g) % nh]
                    # PDL: a launch whose predecessor on its stream is another (independent) HBM launch
                    # of this step may overlap that one's tail; never with external events in between
                    pdl = PDL and st in started and self.lane_events is None
                    self.hbm_cfg = ((self.hbm_cfg_lane_pdl if both else self.hbm_cfg_pdl_alone) if pdl
                                    else self.hbm_cfg_lane if both else {})
                    self.run_flags = m_ov if pdl else 0
                    started.add(st)
                else:
                    st = self._lanes[lane]
                with torch.cuda.stream(st):
                    if self.lane_events is not None:   # external events: graph event-record nodes
                        self.lane_events[i][0].record(st)
                    fn()
                    if self.lane_events is not None:
                        self.lane_events[i][1].record(st)
        for st in list(self._lanes.values()) + self._hbm_extra:
            cur.wait_stream(st)
        self.pow_cfg = None
        self.hbm_cfg = {}
        self.run_flags = 0

    def h2d_bytes(self):
        return sum(t.numel() * 4 for t in self.inputs)

    def d2h_bytes(self):
        return sum(t.numel() * 4 for t in self.outputs)


def _popcount_sum(t):
    import numpy as np
    x = t.cpu().numpy()
    return int(np.unpackbits(x.view(np.uint8)).sum())


# ----------------------------------------------------------- verification

def verify(wl: Workload, run: bool = True) -> dict:
    """Independent correctness checks of this rank's outputs before any timing is
    reported (a benchmark that computes wrong answers must fail), and again
    (run=False) on the buffers the timed CUDA graph wrote.  Uses torch int64 arithmetic and
    Python's built-in pow -- never the product kernels' own helpers and never the oracle."""
    torch = wl.torch
    if run:
        wl.step()
    torch.cuda.synchronize()
    checks = {}

    def i64(t):  # uint32 bit pattern -> int64 value, through int32 (torch uint32 has few ops)
        return t.view(torch.int32).to(torch.int64) & 0xFFFFFFFF

    def identity(P, a, b, c):  # c * 2^32 == a*b (mod P) and c < P, elementwise, on the GPU
        ok = True
        for s in range(0, a.numel(), 1 << 24):
            aa = i64(a[s:s + (1 << 24)])
            bb = i64(b[s:s + (1 << 24)])
            cc = i64(c[s:s + (1 << 24)])
            ok &= bool(((cc << 32) % P == (aa * bb) % P).all()) and bool((cc < P).all())
        return ok

    if hasattr(wl, "c2"):
        for P, (a, b, c) in wl.c2.items():
            checks[f"c2_identity_P{P}"] = identity(P, a, b, c)
    if hasattr(wl, "abar"):
        a0 = wl.c2[P0][0]
        checks["to_from_roundtrip"] = bool((wl.back.view(torch.int32) == a0.view(torch.int32)).all())
        one = torch.ones(a0.numel(), dtype=torch.int32, device=a0.device).view(torch.uint32)
        checks["to_mont_identity"] = identity(P0, wl.abar, one, a0)
    if hasattr(wl, "tw_x"):
        x, o = wl.tw_x, wl.tw_out
        ok = True
        for r in range(0, TW_BATCH, 512):
            xr = x[r:r + 512]
            tw = wl.tw.view(torch.int32).view(1, -1).expand(xr.shape[0], -1).contiguous().view(torch.uint32)
            ok &= identity(P0, xr.reshape(-1), tw.reshape(-1), o[r:r + 512].reshape(-1))
        checks["c3_identity"] = ok
        js = [0, 1, 2, 3, 777, 8192, 16383]
        twh = [int(v) for v in wl.tw.cpu().numpy()]
        checks["c3_table"] = all(twh[j] == (pow(wl.w, j, P0) << 32) % P0 for j in js)
    if hasattr(wl, "pow_bufs"):
        base, e, o = (t.cpu().numpy() for t in wl.pow_bufs)
        idx = list(range(0, base.size, max(1, base.size // 4096)))
        checks["c4_sampled_pow"] = all(int(o[i]) == pow(int(base[i]), int(e[i]), P1) for i in idx)
    if hasattr(wl, "c5"):
        a, b, c = wl.c5
        checks["c5_identity"] = identity(P0, a, b, c)
    if hasattr(wl, "c1"):
        a, b, c = wl.c1
        checks["c1_identity"] = identity(P0, a, b, c)
    if hasattr(wl, "ntt_x"):
        x0 = wl.ntt_x0[7].cpu().numpy()
        X = wl.ntt_x[7].cpu().numpy()
        ok = True
        for k in (0, 1, 4097, TW_LEN - 1):
            wk, acc, pw = pow(wl.ntt_w, k, P0), 0, 1
            for v in x0:
                acc = (acc + int(v) * pw) % P0
                pw = pw * wk % P0
            ok &= int(X[k]) == acc
        checks["ntt_sampled_dft"] = ok
        wl.ntt_x.copy_(wl.ntt_x0)
    return checks


# ------------------------------------------------ configs[4] and configs[0] sub-runs

GOLDEN = ROOT / "tests" / "golden"


def run_c5(m, torch, rank: int, world: int, reps: int = 5) -> dict:
    """configs[4] inside every line: n = 2^31 uint32 pairs in total, rank r owns the contiguous
    global-index slice [r n / W, (r+1) n / W) (generated on its GPU from the global index), the
    fused mul_vec + checksum kernel per rank, box time = MAX over ranks of each rank's median
    (CUDA events, barrier + synchronize around every rep), then ONE all-reduce SUM of the
    checksum partials.  The box checksum must equal the oracle's (tests/golden/c5_checksum.json,
    written by scripts/golden_c5.py from oracle/ only) for every W."""
    from paper_1609_00999_b200 import shard
    lo, hi = shard.slice_bounds(N_C5, world, rank)
    n = hi - lo
    ctx = m.ctx_init(P0)
    u32 = dict(dtype=torch.uint32, device=torch.device("cuda", torch.cuda.current_device()))
    a, b, c = torch.empty(n, **u32), torch.empty(n, **u32), torch.empty(n, **u32)
    m.synth_fill(a, SEED, 1, lo, P0, 0, False)
    m.synth_fill(b, SEED, 2, lo, P0, 0, False)
    acc = torch.zeros(1, dtype=torch.int64, device=a.device)
    fn = lambda: m.mul_vec_checksum(ctx, a, b, out=c, acc=acc)
    for _ in range(2):
        fn()
    st = torch.cuda.current_stream()
    ts = []
    for _ in range(reps):
        shard.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        fn()
        e1.record(st)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    local = statistics.median(ts)
    box_ms = shard.max_over_ranks(local)
    fastest = -shard.max_over_ranks(-local)
    acc.zero_()
    fn()
    torch.cuda.synchronize()
    part = int(acc.item())
    box = shard.combine_checksums(part, P0)
    ok = True   # Montgomery identity c 2^32 = a b (mod P), 0 <= c < P, on every element
    for s0 in range(0, n, 1 << 25):
        aa, bb, cc = (t[s0:s0 + (1 << 25)].view(torch.int32).to(torch.int64) & 0xFFFFFFFF for t in (a, b, c))
        ok &= bool(((cc << 32) % P0 == (aa * bb) % P0).all()) and bool((cc < P0).all())
        del aa, bb, cc
    ok_all = shard.max_over_ranks(0.0 if ok else 1.0) == 0.0
    want = None
    gp = GOLDEN / "c5_checksum.json"
    if gp.exists():
        g = json.loads(gp.read_text())
        want = g["box_checksum_mod_P"]
        rank_want = g["rank_checksums_mod_P"].get(str(world))
        rank_ok = rank_want is None or rank_want[rank] == part % P0
        ok_all &= shard.max_over_ranks(0.0 if rank_ok else 1.0) == 0.0
    del a, b, c
    torch.cuda.empty_cache()
    return {"config": "configs[4]: n = 2^31 uint32 pairs, P = 2013265921, contiguous global-index slices, "
                      "fused mul_vec + checksum, one NCCL all-reduce SUM of the partials after timing",
            "n_total": N_C5, "n_rank": n, "ranks": world, "reps": reps,
            "ms_box": round(box_ms, 4), "ms_fastest_rank": round(fastest, 4),
            "rank_skew": round((box_ms - fastest) / box_ms, 4) if box_ms else None,
            "gmulmod_s_box": round(N_C5 / (box_ms * 1e-3) / 1e9, 2),
            "gbs_aggregate": round(12 * N_C5 / (box_ms * 1e-3) / 1e9, 1),
            "box_checksum": box, "checksum_oracle": want,
            "checksum_ok": (want is None or box == want) and ok_all, "identity_all_elements": ok_all,
            "scaling": "strong (fixed total n)"}


def run_c1(m, torch) -> dict:
    """configs[0] inside every line (single GPU, launch-latency bound): one
    mont_mul_vec_checksum call on n = 65536 with the G12 edge values.  Reports the latency of one
    call (host call to completion, and between CUDA events after an L2 flush) and the throughput
    of the call replayed back to back from a CUDA graph."""
    import numpy as np  # noqa: F401

    import synth as _synth  # the shared input generator (no method arithmetic)
    dev = torch.device("cuda", torch.cuda.current_device())
    ha, hb = _synth.c1_inputs(P0)
    a, b = torch.from_numpy(ha).to(dev), torch.from_numpy(hb).to(dev)
    c = torch.empty_like(a)
    acc = torch.zeros(1, dtype=torch.int64, device=dev)
    ctx = m.ctx_init(P0)
    fn = lambda: m.mul_vec_checksum(ctx, a, b, out=c, acc=acc)
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    flush = torch.empty(128 << 20, dtype=torch.int32, device=dev)
    host, devt = [], []
    for k in range(50):   # one call from an idle GPU: host call to completion (L2 flushed first)
        flush.fill_(k)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        host.append((time.perf_counter() - t0) * 1e6)
    for k in range(50):   # the call's device time: queued behind the flush, so no host gap in it
        flush.fill_(k)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        devt.append(e0.elapsed_time(e1) * 1e3)
    del flush
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    reps = 200
    with torch.cuda.graph(g, stream=s):
        for _ in range(reps):
            fn()
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        g.replay()
    e1.record()
    e1.synchronize()
    per_call_us = e0.elapsed_time(e1) * 1e3 / (5 * reps)
    acc.zero_()
    fn()
    torch.cuda.synchronize()
    checksum = int(acc.item()) % P0
    ka = GOLDEN / "survey_known_answers.json"
    want = json.loads(ka.read_text())["c1"]["checksum_mod_P"] if ka.exists() else None
    hc = c.cpu()
    return {"config": "configs[0]: mont_mul_vec (fused checksum) n = 65536, P = 2013265921, G12 edge values",
            "latency_us": {"host_call_to_completion": round(statistics.median(host), 2),
                           "device_events_after_l2_flush": round(statistics.median(devt), 2)},
            "graph_replay_us_per_call": round(per_call_us, 3),
            "graph_replay_gmulmod_s": round(65536 / (per_call_us * 1e-6) / 1e9, 2),
            "checksum": checksum, "checksum_survey_known_answer": want,
            "checksum_ok": want is None or checksum == want,
            "identity_ok": bool((((hc.view(torch.int32).to(torch.int64) & 0xFFFFFFFF) << 32) % P0 ==
                                 ((a.cpu().view(torch.int32).to(torch.int64) & 0xFFFFFFFF) *
                                  (b.cpu().view(torch.int32).to(torch.int64) & 0xFFFFFFFF)) % P0).all())}


# ----------------------------------------------------------- device timing

def time_steps_concurrent(wl: Workload, K: int):
    """K concurrent-schedule steps between CUDA events on the current stream (the
    lanes are joined into it, so the events bracket all of each step's work)."""
    torch = wl.torch
    s = torch.cuda.current_stream()
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    start.record(s)
    for _ in range(K):
        wl.step_concurrent()
    end.record(s)
    end.synchronize()
    return start.elapsed_time(end)


def capture_step_graph(wl: Workload):
    """Capture one two-lane step (both lanes, forked from and joined into the capture stream)
    into a CUDA graph; replaying it issues the step's launches with one graph launch."""
    torch = wl.torch
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        wl.step_concurrent()            # warm the lanes on this stream
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s):
        wl.step_concurrent()
    torch.cuda.synchronize()
    return g


def imad_launch_clock_mhz(wl: Workload, K: int):
    """The SM clock the IMAD-bound launch (pow) runs at in the serial step: K more serial steps, in
    each of which mb_sm_clock (one warp timing clock64 against %globaltimer) runs on a high-priority
    side stream DURING the pow launch -- it is released by an event recorded just before pow and
    spins for ~2/3 of pow's duration, taking the first slot a finishing pow CTA frees.  Median MHz
    over the K steps (not a timed pass)."""
    torch, m = wl.torch, wl.m
    s = torch.cuda.current_stream()
    side = torch.cuda.Stream(priority=-1)
    buf = torch.zeros(K, 2, dtype=torch.int64, device=wl.dev)
    got = False
    for k in range(K):
        for name, fn, _, _, bound in wl.launches:
            if bound == "imad":
                ev = torch.cuda.Event()
                ev.record(s)
                side.wait_event(ev)
                fn()
                m.lib().mb_sm_clock(buf[k].data_ptr(), 300000, side.cuda_stream)   # ~160 us at 1.9 GHz
                got = True
            else:
                fn()
        s.wait_stream(side)
    torch.cuda.synchronize()
    if not got:
        return None
    v = [c / ns * 1e3 for c, ns in buf.tolist() if ns > 0]
    return statistics.median(v) if v else None


def in_step_kernel_times(wl: Workload, K: int, hbm_mode: str, hbm_streams: int):
    """Each launch's duration INSIDE the two-lane step: a second capture of the step graph with
    external CUDA events (graph event-record nodes) on each launch's own stream around it, replayed
    K times; median per launch over the replays (a synchronize between replays to read the events,
    outside any timed region).  hbm_mode / hbm_streams select how the HBM lane is issued: "streams"
    with 1 stream gives each individual HBM kernel the memory system to itself (only the pow lane
    co-runs); the timed configuration gives the lane as timed.  Returns (the step's launch list,
    per-launch ms, {lane: wall ms from its first launch's start to its last launch's end})."""
    global HBM_STREAMS, HBM_MODE
    torch = wl.torch
    saved = HBM_STREAMS, HBM_MODE
    HBM_STREAMS, HBM_MODE = hbm_streams, hbm_mode
    launches = wl.step_launches
    wl.lane_events = [(torch.cuda.Event(enable_timing=True, external=True),
                       torch.cuda.Event(enable_timing=True, external=True)) for _ in launches]
    try:
        g = capture_step_graph(wl)
        per = [[] for _ in launches]
        span = {}
        for _ in range(max(3, K)):
            g.replay()
            torch.cuda.synchronize()
            for i, (e0, e1) in enumerate(wl.lane_events):
                per[i].append(e0.elapsed_time(e1))
            for lane in {b for *_, b in launches}:
                idx = [i for i, (*_, b) in enumerate(launches) if b == lane]
                ref = wl.lane_events[idx[0]][0]
                t0 = min(ref.elapsed_time(wl.lane_events[i][0]) for i in idx)
                t1 = max(ref.elapsed_time(wl.lane_events[i][1]) for i in idx)
                span.setdefault(lane, []).append(t1 - t0)
        del g
        return launches, [statistics.median(v) for v in per], {k: statistics.median(v) for k, v in span.items()}
    finally:
        wl.lane_events = None
        HBM_STREAMS, HBM_MODE = saved


def time_steps_graph(wl: Workload, g, K: int):
    torch = wl.torch
    s = torch.cuda.current_stream()
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    start.record(s)
    for _ in range(K):
        g.replay()
    end.record(s)
    end.synchronize()
    return start.elapsed_time(end)


def time_steps_flushed(wl: Workload, K: int):
    """configs[0] fits in L2 (768 KiB): each of the K steps is timed alone between CUDA events,
    after a 512 MiB write that evicts the 126 MB L2.  The flush (~80 us of GPU time) is queued
    before the start event, so the GPU is still busy while the host enqueues the step and the
    interval holds only the step."""
    torch = wl.torch
    s = torch.cuda.current_stream()
    flush = torch.empty(128 << 20, dtype=torch.int32, device=s.device)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    for k, (e0, e1) in enumerate(evs):
        flush.fill_(k)
        e0.record(s)
        wl.step()
        e1.record(s)
    torch.cuda.synchronize()
    return sum(e0.elapsed_time(e1) for e0, e1 in evs)


def time_steps(wl: Workload, K: int):
    """K serial steps between CUDA events on the launching stream; per-launch events too."""
    torch = wl.torch
    s = torch.cuda.current_stream()
    nl = len(wl.launches)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(nl + 1)] for _ in range(K)]
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    start.record(s)
    for k in range(K):
        e = evs[k]
        e[0].record(s)
        for i, (_, fn, *_rest) in enumerate(wl.launches):
            fn()
            e[i + 1].record(s)
    end.record(s)
    end.synchronize()
    total_ms = start.elapsed_time(end)
    # per launch: the median over the K steps (one late host enqueue inflates a single
    # event interval with GPU idle time; the step total above is unaffected by the choice)
    per = [statistics.median(evs[k][i].elapsed_time(evs[k][i + 1]) for k in range(K)) for i in range(nl)]
    return total_ms, per


def time_e2e(wl: Workload, steps: int):
    """The same step through the library's HOST-buffer C ABI (include/mont_host.h,
    mont_host_run): every input starts in pinned host memory and every output lands in pinned
    host memory, inside the timed region.  All operations of the step are jobs of one run,
    whose chunks stream through one ring: one H2D stream, one compute stream, one D2H stream."""
    torch, m = wl.torch, wl.m
    pin = lambda t: torch.empty(t.shape, dtype=t.dtype, pin_memory=True).copy_(t)
    empty = lambda t: torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    jobs, keep = [], []
    if hasattr(wl, "c2"):
        for si, P in enumerate(PRIMES):
            a, b, c = wl.c2[P]
            ha, hb, hc = pin(a), pin(b), empty(c)
            acc = torch.zeros(1, dtype=torch.int64, pin_memory=True)
            jobs.append(m.host_job("mul_vec", wl.ctx[P], hc, ha, hb, acc=acc))
            keep += [ha, hb, hc, acc]
            if P == P0 and hasattr(wl, "abar"):
                # to_mont(a0) and from_mont(to_mont's result) right after the P0 product: the three
                # jobs form one fusion group (a0 is uploaded once, abar comes back to the host but
                # from_mont reads it on the device)
                h_bar, h_back = empty(a), empty(a)
                jobs.append(m.host_job("to_mont", wl.ctx[P0], h_bar, ha))
                jobs.append(m.host_job("from_mont", wl.ctx[P0], h_back, h_bar))
                keep += [h_bar, h_back]
    if hasattr(wl, "tw_x"):
        hx, htw, ho = pin(wl.tw_x), pin(wl.tw), empty(wl.tw_x)
        jobs.append(m.host_job("twiddle", wl.ctx[P0], ho, hx, htw))
        keep += [hx, htw, ho]
    if hasattr(wl, "pow_bufs"):
        base, e, o = wl.pow_bufs
        hb, he, ho2 = pin(base), pin(e), empty(o)
        jobs.append(m.host_job("pow_vec", wl.ctx[P1], ho2, hb, he))
        keep += [hb, he, ho2]
    if hasattr(wl, "c1"):
        a, b, c = wl.c1
        ha, hb, hc = pin(a), pin(b), empty(c)
        acc = torch.zeros(1, dtype=torch.int64, pin_memory=True)
        jobs.append(m.host_job("mul_vec", wl.ctx[P0], hc, ha, hb, acc=acc))
        keep += [ha, hb, hc, acc]
    if hasattr(wl, "c5"):
        a, b, c = wl.c5
        ha, hb, hc = pin(a), pin(b), empty(c)
        acc = torch.zeros(1, dtype=torch.int64, pin_memory=True)
        jobs.append(m.host_job("mul_vec", wl.ctx[P0], hc, ha, hb, acc=acc))
        keep += [ha, hb, hc, acc]
    if hasattr(wl, "ntt_x"):
        # the forward transform of host rows (mont_host_run NTT jobs: rows streamed through the ring
        # and transformed in place in the slot), the table copied once per run
        hx, ho = pin(wl.ntt_x0), empty(wl.ntt_x0)
        htw = pin(wl.ntt_tw)
        jobs.append(m.host_job("ntt", wl.ctx[P0], ho, hx, htw))
        keep += [hx, ho, htw]
    # bytes actually copied per step, as the library plans them (after fusion)
    wl.e2e_h2d, wl.e2e_d2h = m.host_run_bytes(jobs)
    ws = m.host_workspace("twiddle", TW_LEN, min_bytes=512 << 20)
    cur = torch.cuda.current_stream()
    m.host_run(jobs, ws)
    torch.cuda.synchronize()
    from paper_1609_00999_b200 import shard
    shard.barrier()  # all ranks share the host's memory system: start the timed region together
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(cur)
    for _ in range(steps):
        m.host_run(jobs, ws)
    e1.record(cur)
    e1.synchronize()
    return e0.elapsed_time(e1) / steps


# ----------------------------------------------------------- CPU baseline

def cpu_model() -> str:
    """/proc/cpuinfo model name of the host the oracle ran on."""
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline(kind: str, target_s: float = 1.5, nsteps: int = 1, threads: int = 0):
    """The oracle (oracle/, plain naive-% definitions, all host cores) on a bounded
    sample of the same workload.  Returns (Gmulmod/s, cores, sample text, seconds)."""
    import numpy as np

    import oracle
    import synth
    cores = threads or os.cpu_count() or 1
    memo = {}

    def gen(fn, *a, **kw):  # inputs are generated once per sample size, outside the timed region
        key = (fn.__name__, a, tuple(sorted(kw.items())))
        if key not in memo:
            memo[key] = fn(*a, **kw)
        return memo[key]

    def run(frac):
        t_total, mm = 0.0, 0
        n2 = max(4, int(N_C2 * frac))
        n4 = max(4, int(N_C4 * frac))
        rows = max(1, int(TW_BATCH * frac))
        parts = []
        if kind == "c1":
            a, b = gen(synth.c1_inputs, P0)
            t0 = time.perf_counter()
            for _ in range(max(1, int(frac * 1024))):
                oracle.mont_mul(P0, a, b, nthreads=cores)
            t_total += time.perf_counter() - t0
            mm += a.size * max(1, int(frac * 1024))
            parts.append(f"c1 {a.size} x {max(1, int(frac * 1024))} repetitions")
        if kind in ("step", "c2", "c5"):
            for P in (PRIMES if kind != "c5" else (P0,)):
                a, b = gen(synth.c2_inputs, P, 0, n2) if kind != "c5" else gen(synth.c5_inputs, P, 0, n2)
                t0 = time.perf_counter()
                c = oracle.mont_mul(P, a, b, nthreads=cores)
                oracle.checksum(P, c, nthreads=cores)
                t_total += time.perf_counter() - t0
                mm += n2
            parts.append(f"c2 {n2}x{3 if kind != 'c5' else 1}")
        if kind == "step":
            a, _ = gen(synth.c2_inputs, P0, 0, n2)
            t0 = time.perf_counter()
            ab = oracle.to_mont(P0, a, nthreads=cores)
            oracle.from_mont(P0, ab, nthreads=cores)
            t_total += time.perf_counter() - t0
            mm += 2 * n2
            parts.append(f"to/from {n2}")
        if kind in ("step", "c3"):
            x = gen(synth.c3_x, P0, batch=rows, length=TW_LEN)
            w = oracle.root_of_unity(P0, G11_GENERATOR, TW_LEN)
            tw = oracle.twiddle_table(P0, w, TW_LEN)
            t0 = time.perf_counter()
            oracle.twiddle(P0, x, tw, nthreads=cores)
            t_total += time.perf_counter() - t0
            mm += rows * TW_LEN
            parts.append(f"c3 {rows}x{TW_LEN}")
        if kind in ("step", "c4"):
            base, e = gen(synth.c4_inputs, P1, 0, n4)
            t0 = time.perf_counter()
            oracle.power(P1, base, e, nthreads=cores)
            t_total += time.perf_counter() - t0
            mm += 31 * n4 + int(np.unpackbits(e.view(np.uint8)).sum())
            parts.append(f"c4 {n4}")
        if kind == "ntt":
            # the oracle evaluates the DFT by definition (O(N^2)) for one row; the metric counts the
            # (N/2) log N butterfly products of the transform it replaces
            x = synth.c3_x(P0, batch=1, length=TW_LEN)
            w = oracle.root_of_unity(P0, G11_GENERATOR, TW_LEN)
            t0 = time.perf_counter()
            oracle.dft(P0, w, x)
            t_total += time.perf_counter() - t0
            mm += (TW_LEN // 2) * 14
            parts.append(f"ntt 1 row of {TW_LEN} (definition DFT, single thread)")
        return t_total, mm, ", ".join(parts)

    frac = 1.0 / 1024
    t, mm, desc = run(frac)
    while t < target_s / 4 and frac < 1.0:  # rescale until one sample pass is a measurable fraction
        frac = min(1.0, frac * target_s / max(t, 1e-3))
        t, mm, desc = run(frac)
    # repeat the sample until about target_s of wall time (target_s x cores of CPU work) is timed
    t_sum, mm_sum, reps = 0.0, 0, 0
    while reps < nsteps or t_sum < target_s:
        t, mm, desc = run(frac)
        t_sum, mm_sum, reps = t_sum + t, mm_sum + mm, reps + 1
    return (mm_sum / t_sum / 1e9, cores,
            f"{frac:.4g} of the {kind} workload ({desc}) x {reps} passes, {t_sum:.1f} s timed; generation excluded",
            t_sum / reps, frac)


# ----------------------------------------------------------------- main

def nvsmi_id(torch, local_rank: int) -> str:
    """nvidia-smi id (UUID) of this rank's CUDA device, robust to CUDA_VISIBLE_DEVICES."""
    try:
        uuid = str(torch.cuda.get_device_properties(local_rank).uuid)
        out = subprocess.run(["nvidia-smi", "--query-gpu=uuid", "--format=csv,noheader"], capture_output=True,
                             text=True, timeout=20).stdout.split()
        for u in out:
            if u.replace("GPU-", "") == uuid.replace("GPU-", ""):
                return u
    except Exception:
        pass
    vis = os.environ.get("CUDA_VISIBLE_DEVICES")
    if vis:
        ids = vis.split(",")
        if local_rank < len(ids):
            return ids[local_rank]
    return str(local_rank)


def ncu_traffic(name: str, nbytes: int = 0):
    """DRAM bytes per launch of this kernel kind from the committed ncu capture (2^26-element
    launches); None when this launch's algorithmic bytes are not that capture's (other sizes)."""
    p = ROOT / "profiles" / "ncu_summary.json"
    if not p.exists():
        return None
    try:
        d = json.loads(p.read_text())
        v = d.get("traffic_bytes_per_launch", {}).get(name.split("[")[0])
        if v is None or (nbytes and not 0.5 <= float(v) / nbytes <= 1.5):
            return None
        return int(v)
    except Exception:
        return None


def main():
    args = parse()
    rc = launch_ranks(args)
    if rc is not None:
        sys.exit(rc)
    global POW_CTAS, POW_VARIANT
    POW_CTAS = 0 if args.serial else args.pow_ctas
    POW_VARIANT = args.pow_variant
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "reference":
        return main_reference(args, rank, world)

    import torch
    import torch.distributed as dist

    from paper_1609_00999_b200 import shard
    # MONT_DIST_BACKEND=gloo + MONT_SHARE_GPU=1: orchestration dry run with all ranks on one GPU
    # (the kernels of different ranks never wait on each other; only CPU-side gloo collectives)
    backend = os.environ.get("MONT_DIST_BACKEND", "nccl")
    dev_index = 0 if os.environ.get("MONT_SHARE_GPU") == "1" else local_rank
    if os.environ.get("MONT_SHARE_GPU") != "1" and torch.cuda.device_count() < world:
        if rank == 0:
            print(json.dumps({"error": f"{world} ranks but {torch.cuda.device_count()} visible GPUs"}), flush=True)
        sys.exit(2)
    torch.cuda.set_device(dev_index)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev_index), timeout=dist_timeout())
        else:
            dist.init_process_group(backend, timeout=dist_timeout())
    wl = Workload(args.workload, rank, world)
    checks = verify(wl)
    ok = all(checks.values())
    ok_all = shard.max_over_ranks(0.0 if ok else 1.0) == 0.0
    if not ok_all:
        if rank == 0:
            print(json.dumps({"error": "parity check failed", "checks": checks}), flush=True)
        sys.exit(1)
    sampler = ClockSampler(nvsmi_id(torch, dev_index))
    sampler.start()
    for _ in range(max(3, args.warmup)):
        wl.step()
    torch.cuda.synchronize()
    # per-kernel durations (`kernels`): a serial pass with events around each launch on the warm GPU,
    # then the clock the IMAD-bound launch ran at (its roofline is clock-normalised)
    _, per_ms = time_steps(wl, args.steps)
    imad_mhz = imad_launch_clock_mhz(wl, max(3, args.steps))
    t_end = time.perf_counter() + args.soak
    while time.perf_counter() < t_end:
        wl.step_concurrent()
        torch.cuda.synchronize()
    shard.barrier()
    torch.cuda.synchronize()
    # the serial step after the soak (ms_per_step_serial; it also lets the clock settle before the
    # timed two-lane step: the overlapped step draws more power than the serial one)
    serial_ms, _ = time_steps(wl, args.steps)
    for _ in range(3):
        wl.step_concurrent()
    torch.cuda.synchronize()
    shard.barrier()
    torch.cuda.synchronize()
    # the reported number: K steps with the runtime's two-lane schedule
    graph = None
    if wl.kind == "c1":
        total_ms = time_steps_flushed(wl, args.steps)
    elif args.graph and not args.serial:
        graph = capture_step_graph(wl)
        for _ in range(3):
            graph.replay()
        torch.cuda.synchronize()
        shard.barrier()
        torch.cuda.synchronize()
        total_ms = time_steps_graph(wl, graph, args.steps)
    else:
        total_ms = time_steps_concurrent(wl, args.steps) if not args.serial else serial_ms
    torch.cuda.synchronize()
    shard.barrier()
    clocks = sampler.stop()
    # the timed graph's own outputs, checked again (no re-run): what was timed is what was verified.
    # The NTT transforms in place, so its input is restored and the graph replayed once first.
    if graph is not None and hasattr(wl, "ntt_x"):
        wl.ntt_x.copy_(wl.ntt_x0)
        graph.replay()
        torch.cuda.synchronize()
    post = verify(wl, run=False) if graph is not None else {}
    # per-kernel in-step durations: HBM launches one after another (each alone on the memory
    # system, co-running with pow); lane wall times: the timed configuration
    in_step_ms = timed_launches = timed_ms = lane_wall = None
    if graph is not None:
        _, in_step_ms, _ = in_step_kernel_times(wl, args.steps, "streams", 1)
        timed_launches, timed_ms, lane_wall = in_step_kernel_times(wl, args.steps, HBM_MODE, HBM_STREAMS)
    # the HBM lane's one mont_run launch alone (its standalone rate), when the step uses it
    run_alone_ms = None
    if graph is not None and HBM_MODE == "run" and hasattr(wl, "_run_launch"):
        fn = wl._run_launch[1]
        for _ in range(3):
            fn()
        evr = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(10)]
        for e0, e1 in evr:
            e0.record()
            fn()
            e1.record()
        torch.cuda.synchronize()
        run_alone_ms = statistics.median(e0.elapsed_time(e1) for e0, e1 in evr)
    post_ok = shard.max_over_ranks(0.0 if all(post.values()) else 1.0) == 0.0
    if not post_ok:
        if rank == 0:
            print(json.dumps({"error": "parity check of the timed graph's outputs failed", "checks": post}), flush=True)
        sys.exit(1)
    total_ms = shard.max_over_ranks(total_ms)
    serial_ms = shard.max_over_ranks(serial_ms)
    ms_per_step = total_ms / args.steps
    # checksum partials -> one NCCL all-reduce SUM (A11), outside the timed region
    if wl.kind in ("step", "c1", "c2", "c5"):
        wl.acc.zero_()
        for name, fn, *_ in wl.launches:
            if name.startswith("mont_mul_vec_checksum"):
                fn()
        torch.cuda.synchronize()
        local = [int(v) for v in wl.acc.tolist()]
        prim = list(PRIMES) if wl.kind not in ("c5", "c1") else [P0]
        box_checksums = shard.combine_checksums(local[:len(prim)], prim)
    else:
        box_checksums = None
    # SURVEY §8(d)'s third HBM denominator: a triad (c = a ^ b, 12 B per element, the mul_vec
    # launch shape, no modular arithmetic) over 2^26 words, measured in this run
    triad_gbs = None
    if wl.kind in ("step", "c2", "c5"):
        import ctypes as _C
        n_t = 1 << 26
        ta, tb, tc = (torch.empty(n_t, dtype=torch.uint32, device="cuda") for _ in range(3))
        st = torch.cuda.current_stream()
        launch = lambda: wl.m.lib().mb_triad(tc.data_ptr(), ta.data_ptr(), tb.data_ptr(), n_t, None, st.cuda_stream)
        for _ in range(3):
            launch()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(10)]
        for e0, e1 in ev:
            e0.record(st)
            launch()
            e1.record(st)
        torch.cuda.synchronize()
        triad_gbs = 12 * n_t / (statistics.median(e0.elapsed_time(e1) for e0, e1 in ev) * 1e-3) / 1e9
        del ta, tb, tc
    # the integer-multiply denominator measured in this run: the K8 microbenchmark's chain of the
    # library's signed REDC (mb_imad kind 3: 8 independent chains per thread, 8 CTAs/SM)
    redc_peak = None
    if wl.kind in ("step", "c4", "ntt"):
        import ctypes as _C
        sms = torch.cuda.get_device_properties(0).multi_processor_count
        sink = torch.empty(sms * 8 * 256, dtype=torch.uint32, device="cuda")
        nthr = _C.c_ulonglong(0)
        cfg = wl.m.Launch(ctas_per_sm=8)
        st = torch.cuda.current_stream()
        run = lambda: wl.m.lib().mb_imad(sink.data_ptr(), 3, 400, _C.byref(cfg), st.cuda_stream, _C.byref(nthr))
        run()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(5)]
        for e0, e1 in ev:
            e0.record(st)
            run()
            e1.record(st)
        torch.cuda.synchronize()
        med = statistics.median(e0.elapsed_time(e1) for e0, e1 in ev) * 1e-3
        redc_peak = nthr.value * 400 * 64 / med / 1e12  # REDCs per second, in T/s
        del sink
    latency_us = None
    if wl.kind == "c1":  # configs[0] is launch-latency bound -- report one call's latency
        lat = []
        for _ in range(50):
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0 = time.perf_counter()
            ev0.record()
            wl.step()
            ev1.record()
            ev1.synchronize()
            lat.append(((time.perf_counter() - t0) * 1e6, ev0.elapsed_time(ev1) * 1e3))
        latency_us = {"host_call_to_completion": round(statistics.median(h for h, _ in lat), 2),
                      "device_events": round(statistics.median(d for _, d in lat), 2)}
    e2e_ms = None
    if not args.no_e2e and world >= 1:
        e2e_ms = time_e2e(wl, max(1, args.e2e_steps))
        e2e_ms = None if e2e_ms is None else shard.max_over_ranks(e2e_ms)
    # configs[4] (sharded n = 2^31, strong scaling) and configs[0] (latency) ride along in the
    # default line, after the step's own timing: the driver runs only the default workload
    c5 = c1 = None
    if wl.kind == "step" and not args.no_subruns:   # 24 GiB / W more on top of the step's 3.3 GiB
        c5 = run_c5(wl.m, torch, rank, world)
        if rank == 0:
            c1 = run_c1(wl.m, torch)
    if rank != 0:
        if dist.is_initialized():
            dist.destroy_process_group()
        return
    mulmods_job = wl.mulmods * world
    value = mulmods_job / (ms_per_step * 1e-3) / 1e9
    hbm_peak, peak_kind, sm_max = peaks()
    sms = torch.cuda.get_device_properties(0).multi_processor_count

    def kernel_rows(times, imad_clk_mhz, launches=None):
        clk = (imad_clk_mhz or clocks.get("sm_mhz") or sm_max) * 1e6
        rows = []
        for (name, _, nbytes, mm, bound), t in zip(launches or wl.launches, times):
            r = {"kernel": name, "ms": round(t, 4), "share": round(t / max(sum(times), 1e-9), 4),
                 "gmulmod_s": round(mm / (t * 1e-3) / 1e9, 2) if mm else None, "lane": bound}
            if bound == "hbm":
                gbs = nbytes / (t * 1e-3) / 1e9
                r.update({"bound": "hbm", "achieved": round(gbs, 1), "peak": hbm_peak, "unit": "GB/s",
                          "frac": round(gbs / hbm_peak, 4), "bytes_per_launch": nbytes,
                          "frac_nominal_8tbs": round(gbs / 8000.0, 4)})
            else:
                # integer-multiply (FMAHeavy) pipe: the measured REDC floor is 5 FMAHeavy issue
                # slots per product (profiles/r02_pipes.jsonl) -> 64/5 per clk per SM
                peak = sms * 64 / 5 * clk / 1e12
                ach = mm / (t * 1e-3) / 1e12
                r.update({"bound": "alu", "achieved": round(ach, 4), "peak": round(peak, 4), "unit": "Tmulmod/s",
                          "frac": round(ach / peak, 4),
                          "peak_basis": f"{sms} SMs x 64 FMAHeavy lanes/clk / 5 issue slots per REDC x "
                                        f"{clk/1e6:.0f} MHz" + (" (SM clock measured during the launch by a "
                                                                "co-running one-warp mb_sm_clock)" if imad_clk_mhz else
                                                                " (median nvidia-smi clock of the timed region)"),
                          # SURVEY §8(d)'s other denominator: 4 multiplies per REDC at the full IMAD rate
                          # (IMAD.WIDE measured half rate on B200, so this one is not reachable)
                          "frac_imad_div4": round(ach / (sms * 64 / 4 * clk / 1e12), 4)})
                if redc_peak:
                    r.update({"redc_chain_peak_measured": round(redc_peak, 4),
                              "frac_redc_measured": round(ach / redc_peak, 4)})
            r["traffic"] = ncu_traffic(name, nbytes)
            rows.append(r)
        return rows

    rooflines = kernel_rows(per_ms, imad_mhz)   # standalone, serial pass, library-default shapes
    in_step = kernel_rows(in_step_ms, None) if in_step_ms else None
    timed_rows = kernel_rows(timed_ms, None, timed_launches) if timed_ms else None
    # dominant kernel: in the timed step (its own launches), the longest lane (the critical path)
    # and within it the kernel kind with the largest share; without a lane schedule, the serial pass
    src = timed_rows if timed_rows else rooflines
    lanes = {}
    for r in src:
        lanes[r["lane"]] = lanes.get(r["lane"], 0.0) + r["ms"]
    crit = max(lanes, key=lanes.get) if in_step else None
    kinds = {}
    for r in src:
        if crit is None or r["lane"] == crit:
            k = r["kernel"].split("[")[0]
            kinds[k] = kinds.get(k, 0.0) + r["ms"]
    dom_kind = max(kinds, key=kinds.get)
    dom_r = max((r for r in src if r["kernel"].split("[")[0] == dom_kind and (crit is None or r["lane"] == crit)),
                key=lambda r: r["ms"])
    roof = {k: dom_r[k] for k in ("bound", "achieved", "peak", "unit", "frac", "traffic")}
    roof["kernel"] = dom_r["kernel"]
    roof["traffic_source"] = ("cited, not measured in this run: dram__bytes_read.sum + dram__bytes_write.sum per "
                              "launch from the committed ncu --set full capture, profiles/ncu_summary.json")
    roof["peak_kind"] = peak_kind if dom_r["bound"] == "hbm" else "derived (DESIGN.md §6)"
    if triad_gbs is not None and dom_r["bound"] == "hbm":
        roof["triad_gbs"] = round(triad_gbs, 1)
        roof["frac_triad"] = round(dom_r["achieved"] / triad_gbs, 4)
    standalone = next((r for r in rooflines if r["kernel"] == dom_r["kernel"]), None)
    if standalone is not None:
        roof["frac_standalone"] = standalone["frac"]
    elif run_alone_ms and dom_r["kernel"].startswith("mont_run"):
        roof["frac_standalone"] = round(wl.run_bytes / (run_alone_ms * 1e-3) / 1e9 / hbm_peak, 4)
        roof["ms_standalone"] = round(run_alone_ms, 4)
    if dom_r["kernel"].startswith("mont_run"):
        roof["bytes_per_launch"] = wl.run_bytes
        roof["bytes_note"] = ("algorithmic bytes of the run by plan (mont_run_bytes): every job's reads and writes, "
                              "the fused to_mont -> from_mont pair reading its input once (12 B per element)")
    if timed_rows:
        roof["duration"] = ("inside the timed two-lane step: median over K replays of a capture of the step graph "
                            "with external CUDA events around each launch on its own stream, co-running with the "
                            "pow lane as timed")
        roof["lanes_ms_in_step"] = {k: round(v, 4) for k, v in lanes.items()}
        roof["critical_lane"] = crit
        if lane_wall and "hbm" in lane_wall:
            hb = sum(nb for _, _, nb, _, b in timed_launches if b == "hbm")
            w = lane_wall["hbm"]
            roof["hbm_lane"] = {"mode": HBM_MODE, "streams": HBM_STREAMS if HBM_MODE != "run" else 1,
                                "wall_ms": round(w, 4), "bytes": hb,
                                "achieved_gbs": round(hb / (w * 1e-3) / 1e9, 1),
                                "frac": round(hb / (w * 1e-3) / 1e9 / hbm_peak, 4),
                                "what": "all HBM launches of the step as timed (first start to last end, external "
                                        "graph events), algorithmic bytes / wall time"}
            # the same bytes over the timed step itself (no events between the launches, so with the
            # programmatic-dependent-launch overlap): the HBM lane is the critical path, so this is a
            # lower bound on the lane's bandwidth as timed
            roof["hbm_lane"]["achieved_gbs_timed_step"] = round(hb / (ms_per_step * 1e-3) / 1e9, 1)
            roof["hbm_lane"]["frac_timed_step"] = round(hb / (ms_per_step * 1e-3) / 1e9 / hbm_peak, 4)
    else:
        roof["duration"] = "median over the K timed steps of a serial pass with CUDA events around each launch"
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "Gmulmod/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 5),
        "higher_is_better": True, "scaling": "weak" if wl.kind != "c5" else "strong",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic (seeded SplitMix64 counter generator, device-side)",
        "config": {"workload": {"step": "one pass of SURVEY §8(a) A1-A11: configs[1] mul_vec x3 primes + to/from_mont + "
                                         "configs[2] twiddle + configs[3] pow (checksum fused into mul_vec)",
                                "c2": "configs[1] mul_vec x3 primes + checksums", "c3": "configs[2] twiddle",
                                "c4": "configs[3] pow", "c5": "configs[4] sharded mul_vec n=2^31 + checksum",
                                "c1": "configs[0] mul_vec n=65536 with fixed edge values (launch-latency bound)",
                                "ntt": "SURVEY 8(f) NEXT #1: in-place forward NTT of the configs[2] batch, 4096 x 2^14"}[wl.kind],
                   "parallelism": f"dp{world} (contiguous global-index slices, no data-path collective)",
                   "l2": ("L2 flushed before every timed step (512 MiB write; the 768 KiB inputs fit in L2)"
                          if wl.kind == "c1" else
                          "inputs larger than L2 (working set per step: " +
                          {"step": "~3.3 GiB", "c2": "2.3 GiB", "c3": "512 MiB", "c4": "192 MiB",
                           "c5": f"{12 * (N_C5 // world) / 2**30:.0f} GiB", "ntt": "256 MiB"}[wl.kind] +
                          " vs 126 MB L2)"),
                   "mulmods_per_step_per_rank": wl.mulmods, **wl.config},
        "gpu_launches": (len(wl.step_launches) if graph is not None else len(wl.launches)) * args.steps,
        "schedule": ("each step alone between CUDA events after an L2 flush" if wl.kind == "c1" else
                     "serial, one stream" if args.serial else
                     ("one lane: " + ", ".join(x[0] for x in wl.launches) + " in order on one stream" +
                      (", each after the first chained by programmatic dependent launch (MONT_LAUNCH_OVERLAP_PREV)"
                       if PDL and len(wl.launches) > 1 else "") +
                      (", replayed as one CUDA graph" if args.graph else ""))
                     if len({x[4] for x in wl.launches}) < 2 else
                     ("two lanes: the HBM-bound operations as ONE mont_run launch (one flat grid over all their "
                      "tiles, to_mont -> from_mont fused)" if HBM_MODE == "run" else
                      "two lanes: the HBM-bound launches in order on one stream (mul_vec+checksum 256 threads x 2 "
                      "uint4 x 3, to_mont -> from_mont as one fused mont_run launch, twiddle default" +
                      (", each after the first launched with MONT_LAUNCH_OVERLAP_PREV: programmatic dependent "
                       "launch, its CTAs start in the previous one's tail)" if PDL else ")")
                      if HBM_MODE == "pair" else
                      f"two lanes: the HBM-bound launches on {HBM_STREAMS} stream(s) (mul_vec+checksum 256 threads x 2 "
                      "uint4, to/from_mont 256 x 4, twiddle default)") +
                     ", the IMAD-bound pow on another, higher-priority "
                     f"stream as a persistent grid of {POW_CTAS} CTA(s) per SM (mont_pow_vec_ex variant {POW_VARIANT})" +
                     (", replayed as one CUDA graph" if args.graph else "")),
        "ms_per_step_serial": round(serial_ms / args.steps, 5),
        "roofline": roof,
        "kernels": rooflines,
        "kernels_note": ("'kernels': each launch alone (serial pass, library-default launch shapes); "
                         "'kernels_in_step': the same individual launches inside the two-lane step (HBM ones one "
                         "after another next to the pow lane); 'kernels_timed_step': the launches of the timed "
                         "step itself (its HBM lane as timed: the to_mont -> from_mont pair as one fused mont_run "
                         "launch in the default 'pair' mode), with external events between them, so without the "
                         "programmatic-dependent-launch overlap of the timed graph"),
        "clocks": {k: clocks.get(k) for k in ("sm_mhz", "sm_max_mhz", "reasons", "samples", "samples_under_load")},
        "parity": {"checks": checks, "box_checksums": box_checksums},
    }
    if in_step:
        line["kernels_in_step"] = in_step
    if timed_rows and timed_launches is not wl.launches:
        line["kernels_timed_step"] = timed_rows
    if latency_us is not None:
        line["latency_us"] = latency_us
    if c5 is not None:
        line["c5"] = c5
        line["parity"]["c5_checksum_ok"] = c5["checksum_ok"]
    if c1 is not None:
        line["c1"] = c1
        line["parity"]["c1_checksum_ok"] = c1["checksum_ok"]
    if post:
        line["parity"]["timed_graph_outputs"] = post
    if e2e_ms is not None:
        line["e2e"] = {"value": round(mulmods_job / (e2e_ms * 1e-3) / 1e9, 3), "unit": "Gmulmod/s",
                       "ms_per_step": round(e2e_ms, 3), "h2d_bytes_per_step": wl.e2e_h2d,
                       "d2h_bytes_per_step": wl.e2e_d2h,
                       "h2d_gbs": round(wl.e2e_h2d / (e2e_ms * 1e-3) / 1e9, 2),
                       "path": "host-buffer C ABI (include/mont_host.h mont_host_run): every input H2D from "
                               "pinned host and every output D2H to pinned host inside the timed region; all "
                               "operations as jobs of one H2D / kernel / D2H ring"}
    if world == 1 and not args.no_cpu_baseline:
        v, cores, sample, secs, frac = cpu_baseline(wl.kind)
        line["cpu_baseline"] = {"value": float(f"{v:.4g}"), "unit": "Gmulmod/s", "cores": cores, "kind": "oracle",
                                "sample": sample, "seconds": round(secs, 3), "cpu_model": cpu_model()}
        if cores > 1:  # the oracle on one thread too (a smaller sample)
            v1, _, sample1, _, _ = cpu_baseline(wl.kind, target_s=1.0, threads=1)
            line["cpu_baseline"]["single_thread"] = {"value": float(f"{v1:.4g}"), "unit": "Gmulmod/s",
                                                     "sample": sample1}
    print(json.dumps(line), flush=True)
    if dist.is_initialized():
        dist.destroy_process_group()


def main_reference(args, rank, world):
    """--impl reference: the CPU oracle, as it stands, on the host cores (rank 0 only)."""
    if rank != 0:
        return
    kind = args.workload
    v0, cores, sample, secs, frac = cpu_baseline(kind, target_s=1.0)
    plan, cores = _ref_plan(kind, frac)
    sample = f"{frac:.4g} of the {kind} workload (inputs generated once, outside the timed calls)"
    times = []
    for i in range(max(0, args.warmup) + args.steps):
        v, secs = _ref_step(plan)
        if i >= args.warmup:
            times.append((secs, v))
    tot_s = sum(s for s, _ in times)
    value = statistics.median(v for _, v in times)
    line = {"impl": "reference", "metric": METRIC, "value": float(f"{value:.4g}"), "unit": "Gmulmod/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * tot_s / max(1, len(times)), 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
            "data": "synthetic (seeded SplitMix64 counter generator, host-side synth/)",
            "config": {"workload": f"bounded sample of the '{kind}' workload (oracle/ on host cores)",
                       "sample_fraction": frac},
            "cpu_baseline": {"value": float(f"{value:.4g}"), "unit": "Gmulmod/s", "cores": cores, "kind": "oracle",
                             "sample": sample, "cpu_model": cpu_model()},
            "e2e": {"value": round(value, 4), "unit": "Gmulmod/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _ref_plan(kind, frac):
    """The reference arm's bounded sample, generated ONCE (host-side synth/, untimed): a list of
    (oracle call, mulmods) that every reference step then runs and times."""
    import numpy as np

    import oracle
    import synth
    cores = os.cpu_count() or 1
    n2 = max(4, int(N_C2 * frac))
    n4 = max(4, int(N_C4 * frac))
    rows = max(1, int(TW_BATCH * frac))
    plan = []
    if kind == "c1":
        a, b = synth.c1_inputs(P0)
        reps = max(1, int(frac * 1024))

        def c1_calls(a=a, b=b, reps=reps):
            for _ in range(reps):
                oracle.mont_mul(P0, a, b, nthreads=cores)
        plan.append((c1_calls, a.size * reps))
    if kind in ("step", "c2", "c5"):
        for P in (PRIMES if kind != "c5" else (P0,)):
            a, b = synth.c2_inputs(P, 0, n2)
            plan.append((lambda P=P, a=a, b=b: oracle.checksum(P, oracle.mont_mul(P, a, b, nthreads=cores),
                                                               nthreads=cores), n2))
    if kind == "step":
        a, _ = synth.c2_inputs(P0, 0, n2)
        plan.append((lambda a=a: oracle.from_mont(P0, oracle.to_mont(P0, a, nthreads=cores), nthreads=cores), 2 * n2))
    if kind in ("step", "c3"):
        x = synth.c3_x(P0, batch=rows, length=TW_LEN)
        tw = oracle.twiddle_table(P0, oracle.root_of_unity(P0, G11_GENERATOR, TW_LEN), TW_LEN)
        plan.append((lambda x=x, tw=tw: oracle.twiddle(P0, x, tw, nthreads=cores), rows * TW_LEN))
    if kind in ("step", "c4"):
        base, e = synth.c4_inputs(P1, 0, n4)
        plan.append((lambda base=base, e=e: oracle.power(P1, base, e, nthreads=cores),
                     31 * n4 + int(np.unpackbits(e.view(np.uint8)).sum())))
    if kind == "ntt":
        x = synth.c3_x(P0, batch=1, length=TW_LEN)
        w = oracle.root_of_unity(P0, G11_GENERATOR, TW_LEN)
        plan.append((lambda x=x, w=w: oracle.dft(P0, w, x), (TW_LEN // 2) * 14))
    return plan, cores


def _ref_step(plan):
    """One reference step = the oracle over the fixed bounded sample (inputs already generated)."""
    t_total, mm = 0.0, 0
    for fn, mulmods in plan:
        t0 = time.perf_counter()
        fn()
        t_total += time.perf_counter() - t0
        mm += mulmods
    return mm / t_total / 1e9, t_total


if __name__ == "__main__":
    main()
