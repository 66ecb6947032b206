"""Summarise the ncu artefacts of one profiling pass (scripts/profile.sh) into profiles/.

    python scripts/ncu_summary.py --round r01 [--src gpurun_out]

Writes profiles/<round>_launches.csv (per-launch durations of the bench command, our kernels and
torch's), profiles/<round>_ncu_summary.md (key --set full metrics per kernel) and
profiles/ncu_summary.json (DRAM traffic per launch, read by bench.py for `roofline.traffic`).
Runs on the CPU box: `ncu -i <report> --page raw --csv`.
"""
import argparse
import collections
import csv
import io
import json
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed", "FMAHeavy (IMAD) pipe % of peak"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed", "FP64 pipe % of peak"),
    ("smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio", "stall: math pipe throttle / issue"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall: long scoreboard / issue"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU inst % of peak"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "stall: barrier / issue"),
    ("smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio", "stall: not selected / issue"),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "stall: wait / issue"),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "stall: short scoreboard / issue"),
    ("smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio", "stall: MIO throttle / issue"),
    ("sm__inst_executed_pipe_fmaheavy.sum", "FMAHeavy warp instructions"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("lts__t_bytes.sum", "L2 bytes"),
]

KIND = {  # ncu kernel name prefix -> bench.py kernel label prefix
    "k_map2": "mont_mul_vec_checksum",
    "k_map1": "to_mont",
    "k_twiddle": "mont_mul_twiddle",
    "k_pow": "mont_pow_vec",
    "k_pow2": "mont_pow_vec",
    "k_pow8": "mont_pow_vec[lane launch, variant 10]",
    "k_sum": "mont_checksum",
    "k_ntt_r32": "mont_ntt",
    "k_ntt_dif": "mont_ntt",
    "k_ntt_dif_pq": "mont_ntt[variant 3]",
    "k_ntt_col": "mont_ntt_large[column pass]",
}


def raw(rep: Path):
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return None
    hdr, units = rows[0], rows[1]
    recs = []
    for vals in rows[2:]:
        recs.append({h: (v, u) for h, v, u in zip(hdr, vals, units)})
    return recs


def to_bytes(v, u):
    f = float(v.replace(",", ""))
    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", default="r01")
    ap.add_argument("--src", default=str(ROOT / "gpurun_out"))
    args = ap.parse_args()
    src = Path(args.src)
    prof = ROOT / "profiles"
    prof.mkdir(exist_ok=True)
    md = [f"# ncu summary, round {args.round}", "",
          "Source: `scripts/profile.sh` on one B200 (`ncu --set full --clock-control none --import-source on`, one",
          "launch per kernel after warm-up, from `python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e",
          "--soak 0`). ncu replays each kernel serialised with caches flushed, so durations are cold-cache;",
          "the bench's CUDA-event numbers are the reported ones.", ""]
    traffic = {}
    for rep in sorted(src.glob("prof_*.ncu-rep")):
        recs = raw(rep)
        if not recs:
            continue
        r = recs[0]
        name = r.get("Kernel Name", ("?", ""))[0]
        md.append(f"## `{name}`")
        md.append("")
        md.append("| metric | value |")
        md.append("|---|---|")
        for key, label in METRICS:
            if key in r:
                v, u = r[key]
                md.append(f"| {label} (`{key}`) | {v} {u} |")
        md.append("")
        if "dram__bytes_read.sum" in r and "dram__bytes_write.sum" in r:
            tb = to_bytes(*r["dram__bytes_read.sum"]) + to_bytes(*r["dram__bytes_write.sum"])
            short = rep.stem.replace("prof_", "")
            label = KIND.get(short, short)
            traffic[label] = tb
            if short == "k_map1":
                traffic["from_mont"] = tb
            if short == "k_map2":
                traffic["mont_mul_vec"] = tb
    # launch list
    lc = src / "launches.csv"
    if lc.exists():
        rows = list(csv.reader(open(lc)))
        hdr = None
        data = []
        for rr in rows:
            if rr and rr[0] == "ID":
                hdr = rr
                continue
            if hdr and len(rr) == len(hdr):
                data.append(dict(zip(hdr, rr)))
        with open(prof / f"{args.round}_launches.csv", "w", newline="") as f:
            w = csv.writer(f)
            w.writerow(["id", "kernel", "grid", "block", "duration_ns"])
            for d in data:
                if d["Metric Name"] == "gpu__time_duration.sum":
                    w.writerow([d["ID"], d["Kernel Name"][:120], d["Grid Size"], d["Block Size"], d["Metric Value"]])
        agg = collections.OrderedDict()
        for d in data:
            if d["Metric Name"] != "gpu__time_duration.sum":
                continue
            k = d["Kernel Name"].split("(")[0][:70]
            agg.setdefault(k, []).append(float(d["Metric Value"]))
        ours = {k: v for k, v in agg.items() if "mont::" in k or k.startswith("void mont::")}
        # the step's kernels (the microbenchmarks that give roofline denominators, the input generator
        # and the twiddle-table builder are excluded); share = each kind's total serialised time over
        # the command / the total of the step's kinds -- every pass of the command (verify, warm-up,
        # serial pass, graph replays) runs each step kernel in the same proportion
        skip = ("k_synth", "twiddle_table", "k_imad", "k_pipe", "k_sm_clock", "OpXor", "OpCopy")
        hot = {k: v for k, v in ours.items() if not any(x in k for x in skip)}
        tot = sum(sum(v) for v in hot.values())
        md += ["## Launch list (same bench command, `--metrics gpu__time_duration.sum`)", "",
               "ncu serialises every launch, so the two lanes of the timed step do not overlap here: the shares "
               "are of the serialised kernel time (the step's own overlap is in the bench line's "
               "`kernels_timed_step`).", "",
               "| kernel | launches | mean µs | share of the step kernels' serialised time |", "|---|---|---|---|"]
        for k, v in agg.items():
            mean = sum(v) / len(v) / 1e3
            share = (sum(v) / tot) if k in hot and tot else None
            md.append(f"| `{k}` | {len(v)} | {mean:.1f} | {'' if share is None else f'{share:.3f}'} |")
        md.append("")
    (prof / f"{args.round}_ncu_summary.md").write_text("\n".join(md) + "\n")
    js = {"round": args.round, "traffic_bytes_per_launch": traffic,
          "note": "dram__bytes_read.sum + dram__bytes_write.sum of one --set full launch; keys are bench.py kernel "
                  "labels without the [..] suffix"}
    (prof / "ncu_summary.json").write_text(json.dumps(js, indent=1) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()
