"""Quick on-GPU sweep: microbenchmarks (IMAD kinds, triad/copy) and kernel launch-config
sweeps.  Prints one JSON object per measurement.  Used to pick library defaults
(DESIGN.md §6); not part of the product."""
import argparse
import json
import os
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1609_00999_b200 as m  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--what", default="all")
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--logn", type=int, default=0)
args = ap.parse_args()

dev = torch.device("cuda:0")
s = torch.cuda.current_stream()
sms = m.sm_count()


def timeit(fn, reps=args.reps, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for e0, e1 in ev:
        e0.record()
        fn()
        e1.record()
    torch.cuda.synchronize()
    t = sorted(e0.elapsed_time(e1) for e0, e1 in ev)
    return t[len(t) // 2] * 1e-3, t[0] * 1e-3


def out(**kw):
    print(json.dumps(kw), flush=True)


def lib():
    return m.lib()


if args.what in ("all", "imad"):
    import ctypes as C
    sink = torch.empty(sms * 32 * 256, dtype=torch.uint32, device=dev)
    names = {0: "IMAD", 1: "IMAD.HI", 2: "IMAD.WIDE(hoisted)", 3: "sredc", 4: "redc", 5: "sredc_mulhi",
             6: "sredc_hiadd", 7: "DFMA", 8: "fmulmod", 9: "IADD", 10: "LOP3", 11: "mix3:1", 12: "mix1:1",
             13: "VIMNMX(fused 3-in)", 14: "SHF", 15: "fredc_p1(Alg.3 shifts)", 16: "mix7:1 sredc:fredc_p1",
             17: "mix3:1 sredc:fredc_p1"}
    kinds = [int(k) for k in os.environ.get("PROBE_KINDS", "").split(",") if k] or list(range(18))
    for kind in kinds:
        for ctas in (4, 8):
            iters = 2000
            nthr = C.c_ulonglong(0)
            cfg = m.Launch(ctas_per_sm=ctas)

            def f():
                st = lib().mb_imad(sink.data_ptr(), kind, iters, C.byref(cfg), s.cuda_stream, C.byref(nthr))
                assert st == 0

            med, best = timeit(f, reps=5)
            ops = nthr.value * iters * 64
            out(what="imad", kind=names[kind], ctas_per_sm=ctas, ops=ops, sec=med,
                gops=ops / med / 1e9, per_sm_per_clk_at_1965=ops / med / sms / 1.965e9)

if args.what == "pipes":
    # mb_pipe (csrc/k_pipes.cu): per-instruction rates from dependent chains nothing can hoist.
    # Reports lanes/clk/SM at the SM clock nvidia-smi shows right after each kind (the kernel runs
    # ~50-100 ms so the clock settles), and at the max clock.
    import ctypes as C
    import subprocess
    names = {0: "IMAD R,R,R", 1: "IMAD R,R,imm", 2: "IMAD R,R,UR", 3: "IMAD.HI R,R,R", 4: "IMAD.HI R,R,imm",
             5: "IMAD.WIDE R,R,R", 6: "IMAD.WIDE+IMAD.HI 1:1", 7: "IMAD.WIDE+IMAD 1:1",
             8: "add.u32 (IADD3 / IMAD.IADD split)", 9: "LOP3", 10: "SEL", 11: "VIMNMX", 12: "SHF",
             13: "FFMA R,R,R", 14: "FFMA R,R,imm", 15: "DFMA", 16: "IMAD.WIDE+FFMA 1:1",
             17: "IMAD.WIDE+IADD3 1:1", 18: "IMAD.WIDE+DFMA 1:1", 19: "IMAD.WIDE+IMAD imm 1:1",
             20: "IMAD+FFMA 1:1", 21: "IMAD+IADD3 1:1", 22: "IMAD.WIDE+LOP3 1:1", 23: "IMAD+IMAD imm 1:1",
             24: "IMAD+DFMA 1:1", 25: "IMAD.WIDE+DMUL 1:1", 26: "IMAD.WIDE+DADD 1:1", 27: "sredc (products)",
             28: "fmulmod (products)", 29: "sredc+fmulmod 1:1 (products)", 30: "sredc+fmulmod 3:1 (products)",
             31: "DMUL", 32: "DADD", 33: "IMAD+DMUL 1:1", 34: "warp-specialised 1/2 fmulmod (products)",
             35: "warp-specialised 2/5 fmulmod (products)", 36: "warp-specialised 1/3 fmulmod (products)",
             37: "warp-specialised 1/4 fmulmod (products)", 38: "warps IMAD.WIDE | DFMA",
             39: "warps IMAD.WIDE | DMUL", 40: "warps sredc | DFMA (ops)", 41: "warps IMAD.WIDE | fmulmod (ops)",
             43: "in-warp 1 sredc : 1 fmulmod chains", 44: "in-warp 3:1", 45: "in-warp 6:2", 46: "2 sredc chains",
             47: "2 fmulmod chains", 48: "4 sredc chains", 49: "IMAD.HI R,R,R,RZ (mul.hi)"}
    sink = torch.empty(sms * 32 * 256, dtype=torch.uint32, device=dev)
    clkbuf = torch.zeros(2, dtype=torch.int64, device=dev)

    def smi_clock():
        try:
            o = subprocess.run(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm", "--format=csv,noheader,nounits"],
                               capture_output=True, text=True, timeout=10).stdout.strip()
            return float(o.split()[0])
        except Exception:
            return None

    kinds = [int(k) for k in os.environ.get("PROBE_KINDS", "").split(",") if k] or list(range(42)) + list(range(43, 50))
    if os.environ.get("PROBE_SLOTS"):
        nthr = C.c_ulonglong(0)
        lib().mb_pipe(sink.data_ptr(), 42, 1, C.byref(m.Launch(ctas_per_sm=8)), s.cuda_stream, C.byref(nthr), None)
        torch.cuda.synchronize()
        sl = sink[:nthr.value].view(-1, 256)[:, ::32].cpu().numpy().tolist()
        out(what="warp_slots", first_ctas=sl[:6], note="per CTA: %warpid of warps 0..7")
    for kind in kinds:
        for ctas in (4, 8):
            iters = int(os.environ.get("PROBE_ITERS", "3000"))
            nthr = C.c_ulonglong(0)
            cfg = m.Launch(ctas_per_sm=ctas)

            def f():
                st = lib().mb_pipe(sink.data_ptr(), kind, iters, C.byref(cfg), s.cuda_stream, C.byref(nthr),
                                   clkbuf.data_ptr())
                assert st == 0

            med, best = timeit(f, reps=7)
            cyc, ns = (int(v) for v in clkbuf.tolist())
            mhz = cyc / ns * 1e3 if ns else None   # CTA 0's clock64 / globaltimer over its lifetime
            ops = nthr.value * iters * lib().mb_pipe_ops_per_iter(kind)
            if kind in (35, 36, 37):  # the FP64 half of the warps runs fewer trips
                fi = {35: iters * 2 // 3, 36: iters // 2, 37: iters // 3}[kind]
                ops = nthr.value * (iters + fi) // 2 * lib().mb_pipe_ops_per_iter(kind)
            out(what="pipe", kind=kind, name=names[kind], ctas_per_sm=ctas, ops=ops, sec=med,
                gops=ops / med / 1e9, sm_mhz_in_kernel=mhz, smi_mhz_after=smi_clock(),
                lanes_per_sm_clk=(ops / med / sms / (mhz * 1e6)) if mhz else None,
                lanes_per_sm_clk_at_1965=ops / med / sms / 1.965e9)

if args.what in ("all", "hbm"):
    import ctypes as C
    n = 1 << 26
    a = torch.empty(n, dtype=torch.uint32, device=dev)
    b = torch.empty(n, dtype=torch.uint32, device=dev)
    c = torch.empty(n, dtype=torch.uint32, device=dev)
    m.synth_fill(a, 42, 1, 0, 2013265921)
    m.synth_fill(b, 42, 2, 0, 2013265921)
    ctx = m.ctx_init(2013265921)
    for threads in (128, 256, 512):
        for ctas in (4, 8):
            for unroll in (1, 2, 4):
                for variant in (0, 1):
                    if variant == 0 and ctas != 4:
                        continue
                    cfg = m.Launch(threads=threads, ctas_per_sm=ctas, unroll=unroll, variant=variant)
                    med, best = timeit(lambda: lib().mb_triad(c.data_ptr(), a.data_ptr(), b.data_ptr(), n,
                                                              C.byref(cfg), s.cuda_stream))
                    out(what="triad", threads=threads, ctas=ctas, unroll=unroll, variant=variant,
                        us=med * 1e6, gbs=12 * n / med / 1e9, gbs_best=12 * n / best / 1e9)
                    med, best = timeit(lambda: m.mul_vec(ctx, a, b, out=c, cfg=cfg))
                    out(what="mul_vec", threads=threads, ctas=ctas, unroll=unroll, variant=variant,
                        us=med * 1e6, gbs=12 * n / med / 1e9, gbs_best=12 * n / best / 1e9,
                        gmulmod=n / med / 1e9)
    acc = torch.zeros(1, dtype=torch.int64, device=dev)
    for threads in (256, 512):
        for unroll in (1, 2, 4, 8):
            cfg = m.Launch(threads=threads, unroll=unroll)
            med, best = timeit(lambda: m.mul_vec_checksum(ctx, a, b, out=c, acc=acc, cfg=cfg))
            out(what="mul_vec_checksum", threads=threads, unroll=unroll, us=med * 1e6, gbs=12 * n / med / 1e9)
            med, best = timeit(lambda: m.to_mont(ctx, a, out=c, cfg=cfg))
            out(what="to_mont_cfg", threads=threads, unroll=unroll, us=med * 1e6, gbs=8 * n / med / 1e9)
            med, best = timeit(lambda: lib().mb_copy(c.data_ptr(), a.data_ptr(), n, C.byref(cfg), s.cuda_stream))
            out(what="copy_cfg", threads=threads, unroll=unroll, us=med * 1e6, gbs=8 * n / med / 1e9)
    cfg = m.Launch()
    med, best = timeit(lambda: lib().mb_copy(c.data_ptr(), a.data_ptr(), n, C.byref(cfg), s.cuda_stream))
    out(what="copy", us=med * 1e6, gbs=8 * n / med / 1e9)
    med, best = timeit(lambda: c.copy_(a))
    out(what="torch_copy", us=med * 1e6, gbs=8 * n / med / 1e9)
    med, best = timeit(lambda: m.to_mont(ctx, a, out=c))
    out(what="to_mont", us=med * 1e6, gbs=8 * n / med / 1e9)
    med, best = timeit(lambda: m.from_mont(ctx, a, out=c))
    out(what="from_mont", us=med * 1e6, gbs=8 * n / med / 1e9)
    acc = torch.zeros(1, dtype=torch.int64, device=dev)
    med, best = timeit(lambda: m.checksum(ctx, a, acc=acc))
    out(what="checksum", us=med * 1e6, gbs=4 * n / med / 1e9)

if args.what in ("all", "tw"):
    P = 2013265921
    ctx = m.ctx_init(P)
    batch, L = 4096, 1 << 14
    x = torch.empty(batch * L, dtype=torch.uint32, device=dev)
    m.synth_fill(x, 42, 5, 0, P)
    x = x.view(batch, L)
    o = torch.empty_like(x)
    tw = m.twiddle_table(ctx, 1657000625, L)
    for variant in (4, 1):  # 4 = bulk-copy staged table chunk per CTA, 1 = table through L1/L2
        for ctas in (3, 8, 16, 32, 64):
            for unroll in (1, 2, 4):
                for chunk in (2048, 4096, 16384):
                    for threads in (256, 512):
                        cfg = m.Launch(threads=threads, ctas_per_sm=ctas, unroll=unroll, variant=variant,
                                       chunk=chunk)
                        try:
                            med, best = timeit(lambda: m.mul_twiddle(ctx, x, tw, out=o, cfg=cfg))
                        except m.MontError as e:
                            out(what="twiddle", err=str(e), ctas=ctas, chunk=chunk)
                            continue
                        out(what="twiddle", variant=variant, ctas=ctas, unroll=unroll, chunk=chunk,
                            threads=threads, us=med * 1e6, gbs=8 * batch * L / med / 1e9,
                            gmulmod=batch * L / med / 1e9)

if args.what in ("all", "pow"):
    P = 469762049
    ctx = m.ctx_init(P)
    n = 1 << 24
    base = torch.empty(n, dtype=torch.uint32, device=dev)
    e = torch.empty(n, dtype=torch.uint32, device=dev)
    o = torch.empty(n, dtype=torch.uint32, device=dev)
    m.synth_fill(base, 42, 3, 0, P, mode=1)
    m.synth_fill(e, 42, 4, 0, P, mode=2)
    pc = e.cpu().numpy()
    import numpy as np
    useful = int(31 * n + np.unpackbits(pc.view(np.uint8)).sum())
    variants = [int(v) for v in os.environ.get("PROBE_POW_VARIANTS", "0,10,2,5,6,7,8,9").split(",")]
    ctas_list = [int(v) for v in os.environ.get("PROBE_POW_CTAS", "0").split(",")]
    threads_list = [int(v) for v in os.environ.get("PROBE_POW_THREADS", "256").split(",")]
    primes = [int(v) for v in os.environ.get("PROBE_POW_PRIMES", str(P)).split(",")]
    for Pp in primes:
        ctx = m.ctx_init(Pp)
        if Pp != P:
            m.synth_fill(base, 42, 3, 0, Pp, mode=1)
        ref = m.pow_vec(ctx, base, e, cfg=m.Launch(variant=0))
        for variant in variants:
            for ctas in ctas_list:
                for thr in threads_list:
                    cfg = m.Launch(variant=variant, ctas_per_sm=ctas, threads=thr)
                    try:
                        med, best = timeit(lambda: m.pow_vec(ctx, base, e, out=o, cfg=cfg), reps=10)
                    except m.MontError as ex:
                        out(what="pow", P=Pp, variant=variant, ctas=ctas, threads=thr, err=str(ex))
                        continue
                    same = bool((o.view(torch.int32) == ref.view(torch.int32)).all())
                    out(what="pow", P=Pp, variant=variant, ctas=ctas, threads=thr, us=med * 1e6, us_best=best * 1e6,
                        useful_mulmods=useful, tmulmod=useful / med / 1e12, equal_to_variant0=same)

if args.what == "powctx":
    # pow (default launch) timed: back to back; after a 512 MiB L2 flush; after the twiddle kernel;
    # each followed by mb_sm_clock for the clock it ran at
    import numpy as np
    P = 469762049
    ctx = m.ctx_init(P)
    n = 1 << 24
    base = torch.empty(n, dtype=torch.uint32, device=dev)
    e = torch.empty(n, dtype=torch.uint32, device=dev)
    o = torch.empty(n, dtype=torch.uint32, device=dev)
    m.synth_fill(base, 42, 3, 0, P, mode=1)
    m.synth_fill(e, 42, 4, 0, P, mode=2)
    useful = int(31 * n + np.unpackbits(e.cpu().numpy().view(np.uint8)).sum())
    flush = torch.empty(128 << 20, dtype=torch.int32, device=dev)
    clk = torch.zeros(2, dtype=torch.int64, device=dev)
    for ctxname in ("back_to_back", "after_flush", "after_flush_sync"):
        for variant in (11, 10, 17):
            cfg = m.Launch(variant=variant)
            ts, mhz = [], []
            for k in range(20):
                if ctxname != "back_to_back":
                    flush.fill_(k)
                if ctxname == "after_flush_sync":
                    torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                m.pow_vec(ctx, base, e, out=o, cfg=cfg)
                e1.record()
                lib().mb_sm_clock(clk.data_ptr(), 40000, s.cuda_stream)
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1) * 1e3)
                c, ns = clk.tolist()
                mhz.append(c / ns * 1e3)
            tm, cm = sorted(ts)[len(ts) // 2], sorted(mhz)[len(mhz) // 2]
            floor_us = n / 32 * 478 / (sms * 4) / (cm * 1e6) * 1e6   # 478 FMAHeavy cycles per warp-ladder
            out(what="powctx", ctx=ctxname, variant=variant, us=tm, mhz_after=cm, floor_us_at_that_clock=floor_us,
                frac_floor=floor_us / tm, tmulmod=useful / tm / 1e6)

if args.what == "run":
    # the step's HBM lane alone: individual launches (library defaults / the lane's shapes) vs ONE
    # mont_run launch (to_mont -> from_mont fused), CUDA events, no pow lane
    sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
    import bench
    wl = bench.Workload("step", 0, 1)
    hbm = [x for x in wl.launches if x[4] == "hbm"]
    nbytes = sum(x[2] for x in hbm)

    def serial(cfgs):
        wl.hbm_cfg = cfgs
        for _, fn, *_ in hbm:
            fn()
        wl.hbm_cfg = {}

    bench.HBM_MODE = "run"
    run_l = wl.step_launches[0]
    L = m.Launch
    for name, fn in (("individual, library defaults", lambda: serial({})),
                     ("individual, lane shapes 256x2 / 256x4",
                      lambda: serial({"mul": L(threads=256, unroll=2), "conv": L(threads=256, unroll=4)})),
                     ("one mont_run (to/from fused)", run_l[1]),
                     ("mont_run 256 x 2", lambda: m.run(wl.run_jobs, cfg=L(threads=256, unroll=2))),
                     ("mont_run 256 x 4", lambda: m.run(wl.run_jobs, cfg=L(threads=256, unroll=4))),
                     ("mont_run 512 x 1", lambda: m.run(wl.run_jobs, cfg=L(threads=512, unroll=1))),
                     ("mont_run 512 x 4", lambda: m.run(wl.run_jobs, cfg=L(threads=512, unroll=4)))):
        med, best = timeit(fn, reps=20)
        out(what="run", how=name, us=med * 1e6, us_best=best * 1e6, bytes_individual=nbytes, bytes_run=wl.run_bytes,
            gbs_algorithmic=(wl.run_bytes if "run" in name else nbytes) / med / 1e9)

if args.what in ("pcie",):
    n = 1 << 26   # 256 MiB
    hs = [torch.empty(n, dtype=torch.uint32, pin_memory=True) for _ in range(2)]
    ds = [torch.empty(n, dtype=torch.uint32, device=dev) for _ in range(2)]
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    med, _ = timeit(lambda: ds[0].copy_(hs[0], non_blocking=True), reps=5)
    out(what="h2d", gbs=4 * n / med / 1e9)
    med, _ = timeit(lambda: hs[1].copy_(ds[1], non_blocking=True), reps=5)
    out(what="d2h", gbs=4 * n / med / 1e9)

    def both():
        ev = torch.cuda.Event()
        ev.record()
        s1.wait_event(ev)
        s2.wait_event(ev)
        with torch.cuda.stream(s1):
            ds[0].copy_(hs[0], non_blocking=True)
        with torch.cuda.stream(s2):
            hs[1].copy_(ds[1], non_blocking=True)
        torch.cuda.current_stream().wait_stream(s1)
        torch.cuda.current_stream().wait_stream(s2)
    med, _ = timeit(both, reps=5)
    out(what="h2d+d2h concurrent", gbs_each=4 * n / med / 1e9, gbs_total=8 * n / med / 1e9)
    import subprocess
    out(what="nvidia-smi topo", txt=subprocess.run(["nvidia-smi", "-q", "-d", "PCIE"], capture_output=True, text=True).stdout[-1500:])

if args.what in ("ntt",):
    P = int(os.environ.get("PROBE_P", "2013265921"))
    G = {2013265921: 31, 469762049: 3, 998244353: 3}[P]
    ctx = m.ctx_init(P)
    import numpy as np
    for log_n in ((args.logn,) if args.logn else (10, 12, 13, 14, 15)):
        N = 1 << log_n
        batch = (1 << 26) // N
        w = pow(G, (P - 1) // N, P)
        tw = m.ntt_twiddles(ctx, w, log_n)
        d = torch.empty(batch * N, dtype=torch.uint32, device=dev)
        m.synth_fill(d, 42, 5, 0, P)
        d = d.view(batch, N)
        tw2 = m.ntt_twiddles_pq(ctx, w, log_n)
        for variant in [int(v) for v in os.environ.get("PROBE_NTT_VARIANTS", "0,1,3,4,5,6,7").split(",")]:
            med, best = timeit(lambda: m.ntt(ctx, d, tw2 if variant in (3, 5, 7) else tw, variant=variant), reps=10)
            redc = batch * (N // 2) * log_n
            out(what="ntt", variant={0: "dif", 1: "dit", 3: "dif_pq", 4: "dif_swizzled", 5: "dif_pq_swizzled", 6: "dif_persistent",
                         7: "dif_pq_persistent"}[variant],
                log_n=log_n, batch=batch, us=med * 1e6,
                gbs=8 * batch * N / med / 1e9, tredc=redc / med / 1e12,
                frac_imad_floor=redc / med / (148 * 64 / 5 * 1.965e9))

if args.what in ("barrett",):
    import numpy as np
    P = 469762049
    n = 1 << 24
    base = torch.empty(n, dtype=torch.uint32, device=dev)
    e = torch.empty(n, dtype=torch.uint32, device=dev)
    o = torch.empty(n, dtype=torch.uint32, device=dev)
    m.synth_fill(base, 42, 3, 0, P, mode=1)
    m.synth_fill(e, 42, 4, 0, P, mode=2)
    useful = int(31 * n + np.unpackbits(e.cpu().numpy().view(np.uint8)).sum())
    bctx = m.barrett_ctx_init(P)
    ctx = m.ctx_init(P)
    med, _ = timeit(lambda: m.barrett_pow_vec(bctx, base, e, out=o), reps=10)
    out(what="pow_barrett", us=med * 1e6, tmulmod=useful / med / 1e12)
    med, _ = timeit(lambda: m.pow_vec(ctx, base, e, out=o), reps=10)
    out(what="pow_montgomery", us=med * 1e6, tmulmod=useful / med / 1e12)
    nn = 1 << 26
    a = torch.empty(nn, dtype=torch.uint32, device=dev)
    b = torch.empty(nn, dtype=torch.uint32, device=dev)
    c = torch.empty(nn, dtype=torch.uint32, device=dev)
    m.synth_fill(a, 42, 1, 0, P)
    m.synth_fill(b, 42, 2, 0, P)
    med, _ = timeit(lambda: m.barrett_mul_vec(bctx, a, b, out=c))
    out(what="mul_vec_barrett", us=med * 1e6, gbs=12 * nn / med / 1e9)
    med, _ = timeit(lambda: m.mul_vec(ctx, a, b, out=c))
    out(what="mul_vec_montgomery", us=med * 1e6, gbs=12 * nn / med / 1e9)
    sink = torch.empty(sms * 8 * 256, dtype=torch.uint32, device=dev)

if args.what in ("dot",):
    P = 2013265921
    ctx = m.ctx_init(P)
    batch, L = 4096, 1 << 14
    A = torch.empty(batch * L, dtype=torch.uint32, device=dev)
    m.synth_fill(A, 42, 31, 0, P)
    A = A.view(batch, L)
    x = torch.empty(L, dtype=torch.uint32, device=dev)
    m.synth_fill(x, 42, 32, 0, P)
    o = torch.empty(batch, dtype=torch.uint32, device=dev)
    ref = m.dot(ctx, A, x, cfg=m.Launch(variant=1))
    for name, cfg in (("default", None), ("one CTA per row, 4 uint4 (variant 1)", m.Launch(variant=1)),
                      ("8 uint4 (variant 2)", m.Launch(variant=2)), ("4 uint4 prefetched (variant 3)", m.Launch(variant=3)),
                      ("8 uint4 prefetched (variant 4)", m.Launch(variant=4)),
                      ("split 4096 (variant 5)", m.Launch(variant=5)), ("split 8192", m.Launch(variant=5, chunk=8192)),
                      ("2 rows per CTA (variant 6)", m.Launch(variant=6)), ("4 rows per CTA (variant 7)", m.Launch(variant=7)),
                      *[(f"bulk-copy ring (variant 8) stages={st} ctas/SM={k} tile={ch}",
                         m.Launch(variant=8, unroll=st, ctas_per_sm=k, chunk=ch))
                        for st, k, ch in ((2, 2, 4096), (4, 1, 4096), (2, 1, 8192), (2, 3, 4096), (4, 2, 2048),
                                          (2, 4, 2048), (8, 1, 2048))]):
        med, _ = timeit(lambda: m.dot(ctx, A, x, out=o, cfg=cfg))
        same = bool((o.view(torch.int32) == ref.view(torch.int32)).all())
        out(what="dot", launch=name, us=med * 1e6, gbs=4 * batch * L / med / 1e9, gmulmod=batch * L / med / 1e9,
            equal_to_one_cta_per_row=same)

if args.what in ("tma",):
    import ctypes as C
    n = 1 << 26
    a = torch.empty(n, dtype=torch.uint32, device=dev)
    b = torch.empty(n, dtype=torch.uint32, device=dev)
    c = torch.empty(n, dtype=torch.uint32, device=dev)
    m.synth_fill(a, 42, 1, 0, 2013265921)
    m.synth_fill(b, 42, 2, 0, 2013265921)
    ctx = m.ctx_init(2013265921)
    acc = torch.zeros(1, dtype=torch.int64, device=dev)
    for chunk in (0, 2048, 4096, 8192, 12288, 16384, 24576):
        for variant in ((2,) if chunk else (0, 2)):
            cfg = m.Launch(variant=variant, chunk=chunk)
            med, best = timeit(lambda: m.mul_vec(ctx, a, b, out=c, cfg=cfg))
            out(what="mul_vec", variant=variant, chunk=chunk, us=med * 1e6, gbs=12 * n / med / 1e9)
            med, best = timeit(lambda: lib().mb_triad(c.data_ptr(), a.data_ptr(), b.data_ptr(), n, C.byref(cfg),
                                                      s.cuda_stream))
            out(what="triad", variant=variant, chunk=chunk, us=med * 1e6, gbs=12 * n / med / 1e9)
            med, best = timeit(lambda: m.mul_vec_checksum(ctx, a, b, out=c, acc=acc, cfg=cfg))
            out(what="mul_vec_checksum", variant=variant, chunk=chunk, us=med * 1e6, gbs=12 * n / med / 1e9)

if args.what in ("hostrun",):
    import numpy as np
    P = 2013265921
    ctx = m.ctx_init(P)
    n = 1 << 26
    ha = torch.empty(n, dtype=torch.uint32, pin_memory=True)
    hb = torch.empty(n, dtype=torch.uint32, pin_memory=True)
    hcs = [torch.empty(n, dtype=torch.uint32, pin_memory=True) for _ in range(3)]
    d = torch.empty(n, dtype=torch.uint32, device=dev)
    m.synth_fill(d, 42, 1, 0, P)
    ha.copy_(d)
    m.synth_fill(d, 42, 2, 0, P)
    hb.copy_(d)
    for ws_mb in (96, 192, 512, 1024):
        ws = m.host_workspace("mul_vec", min_bytes=ws_mb << 20)
        jobs = [m.host_job("mul_vec", ctx, hc, ha, hb) for hc in hcs]
        med, _ = timeit(lambda: m.host_run(jobs, ws), reps=3, warm=1)
        out(what="host_run 3x mul_vec", ws_mb=ws_mb, ms=med * 1e3, h2d_gbs=3 * 8 * n / med / 1e9,
            d2h_gbs=3 * 4 * n / med / 1e9)
    # raw: the same bytes as two big concurrent copies
    dbig = torch.empty(6 * n, dtype=torch.uint32, device=dev)
    hbig = torch.empty(6 * n, dtype=torch.uint32, pin_memory=True)
    dout = torch.empty(3 * n, dtype=torch.uint32, device=dev)
    hout = torch.empty(3 * n, dtype=torch.uint32, pin_memory=True)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def raw():
        ev = torch.cuda.Event()
        ev.record()
        s1.wait_event(ev)
        s2.wait_event(ev)
        with torch.cuda.stream(s1):
            dbig.copy_(hbig, non_blocking=True)
        with torch.cuda.stream(s2):
            hout.copy_(dout, non_blocking=True)
        torch.cuda.current_stream().wait_stream(s1)
        torch.cuda.current_stream().wait_stream(s2)
    med, _ = timeit(raw, reps=3, warm=1)
    out(what="raw 1.5GB h2d || 0.75GB d2h", ms=med * 1e3, h2d_gbs=24 * n / med / 1e9)
    med, _ = timeit(lambda: dbig.copy_(hbig, non_blocking=True), reps=3, warm=1)
    out(what="raw 1.5GB h2d alone", ms=med * 1e3, gbs=24 * n / med / 1e9)

if args.what in ("nttlarge",):
    P = int(os.environ.get("PROBE_P", "2013265921"))
    G = {2013265921: 31, 469762049: 3, 998244353: 3}[P]
    ctx = m.ctx_init(P)
    for log_n in ((args.logn,) if args.logn else tuple(k for k in (20, 22, 23, 24, 25, 26, 27) if (P - 1) % (1 << k) == 0)):
        N = 1 << log_n
        w = pow(G, (P - 1) // N, P)
        plan = m.ntt_plan(ctx, w, log_n)
        x = torch.empty(N, dtype=torch.uint32, device=dev)
        m.synth_fill(x, 42, 5, 0, P)
        o = torch.empty_like(x)
        med, _ = timeit(lambda: m.ntt_large(ctx, x, plan, out=o), reps=10)
        out(what="ntt_large", log_n=log_n, us=med * 1e6, gbs_5pass=40 * N / med / 1e9,
            tbutterfly=(N // 2) * log_n / med / 1e12)

if args.what in ("tw2",):
    P = 2013265921
    ctx = m.ctx_init(P)
    batch, L = 4096, 1 << 14
    x = torch.empty(batch * L, dtype=torch.uint32, device=dev)
    m.synth_fill(x, 42, 5, 0, P)
    x = x.view(batch, L)
    o = torch.empty_like(x)
    tw = m.twiddle_table(ctx, 1657000625, L)
    med, _ = timeit(lambda: m.mul_twiddle(ctx, x, tw, out=o))
    out(what="twiddle default", us=med * 1e6, gbs=8 * batch * L / med / 1e9)
    cfg = m.Launch(variant=3)
    med, _ = timeit(lambda: m.mul_twiddle(ctx, x, tw, out=o, cfg=cfg))
    out(what="twiddle TMA-staged once + CLC work stealing (variant 3)", us=med * 1e6, gbs=8 * batch * L / med / 1e9)
    for threads, ctas, unroll, chunk in [(256, 64, 4, 4096), (256, 32, 4, 4096), (256, 64, 2, 4096),
                                         (512, 32, 4, 4096), (256, 16, 4, 16384), (512, 8, 4, 16384),
                                         (256, 64, 4, 2048), (128, 64, 4, 4096)]:
        cfg = m.Launch(variant=4, threads=threads, ctas_per_sm=ctas, unroll=unroll, chunk=chunk)
        med, _ = timeit(lambda: m.mul_twiddle(ctx, x, tw, out=o, cfg=cfg))
        out(what="twiddle TMA-staged per CTA (variant 4)", threads=threads, ctas=ctas, unroll=unroll, chunk=chunk,
            us=med * 1e6, gbs=8 * batch * L / med / 1e9)
    for threads in (256, 512):
        for unroll in (1, 2, 4):
            cfg = m.Launch(threads=threads, unroll=unroll, variant=2)
            med, _ = timeit(lambda: m.mul_twiddle(ctx, x, tw, out=o, cfg=cfg))
            out(what="twiddle flat", threads=threads, unroll=unroll, us=med * 1e6, gbs=8 * batch * L / med / 1e9)
    cfg = m.Launch(threads=512, unroll=2)
    med, _ = timeit(lambda: m.to_mont(ctx, x.view(-1), out=o.view(-1), cfg=cfg))
    out(what="to_mont 512x2", us=med * 1e6, gbs=8 * batch * L / med / 1e9)

if args.what in ("pipe",):
    # variant 3 (persistent bulk-copy pipeline) vs the flat default, standalone
    P = 2013265921
    ctx = m.ctx_init(P)
    n = 1 << 26
    a = torch.empty(n, dtype=torch.uint32, device=dev)
    b = torch.empty(n, dtype=torch.uint32, device=dev)
    m.synth_fill(a, 42, 1, 0, P)
    m.synth_fill(b, 42, 2, 0, P)
    c = torch.empty_like(a)
    acc = torch.zeros(1, dtype=torch.int64, device=dev)
    cfgs = [None] + [m.Launch(threads=t, ctas_per_sm=k, unroll=1, variant=3, chunk=ch)
                     for t in (128, 256) for k in (1, 2) for ch in (1024, 2048, 4096)]
    for cfg in cfgs:
        try:
            med, best = timeit(lambda: m.mul_vec_checksum(ctx, a, b, out=c, acc=acc, cfg=cfg))
        except Exception as ex:  # noqa: BLE001
            out(what="pipe_mulvec", cfg=str(cfg and (cfg.threads, cfg.ctas_per_sm, cfg.chunk)), err=str(ex))
            continue
        out(what="pipe_mulvec", cfg=None if cfg is None else (cfg.threads, cfg.ctas_per_sm, cfg.chunk),
            us=med * 1e6, gbs=12 * n / med / 1e9)
    for cfg in [None] + [m.Launch(threads=t, ctas_per_sm=k, unroll=1, variant=3, chunk=ch)
                         for t in (128, 256) for k in (1, 2) for ch in (2048, 4096)]:
        med, best = timeit(lambda: m.to_mont(ctx, a, out=c, cfg=cfg))
        out(what="pipe_tomont", cfg=None if cfg is None else (cfg.threads, cfg.ctas_per_sm, cfg.chunk),
            us=med * 1e6, gbs=8 * n / med / 1e9)
