#!/bin/bash
# One bench line per workload (configs[0..4], the NTT row) into gpurun_out/bench_<w>.json (run under gpurun).
set -u
mkdir -p gpurun_out
for w in c1 c2 c3 c4 c5 ntt step; do
  timeout 900 python bench.py --workload $w > gpurun_out/bench_$w.log 2>&1
  echo "$w rc=$?"
  tail -1 gpurun_out/bench_$w.log > gpurun_out/bench_$w.json
done
