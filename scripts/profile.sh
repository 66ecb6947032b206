#!/bin/bash
# On-GPU measurement pass (run under gpurun):
#   1. the default bench line (the number), 2. the bench command under ncu: per-launch
#   durations, 3. ncu --set full captures of the top kernels (each after its own plain run).
set -u
OUT=${OUT:-gpurun_out}
ROUND=${ROUND:-r02}
mkdir -p $OUT
timeout 900 python bench.py > $OUT/bench_final.log 2>&1; echo "bench rc=$?"
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --soak 0 --no-subruns"
$CMD > $OUT/plain_small.log 2>&1 || { echo "plain small bench failed"; tail -20 $OUT/plain_small.log; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launches.log 2>&1
echo "launch list rc=$?"
for K in k_map2 k_pow2 k_pow8 k_twiddle k_map1; do
  ncu --set full --clock-control none --import-source on -k regex:"^${K}" -s 3 -c 1 -o $OUT/prof_${K} $CMD > $OUT/ncu_${K}.log 2>&1
  echo "ncu full ${K} rc=$?"
done
CMD2="python bench.py --workload ntt --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --soak 0"
$CMD2 > $OUT/plain_ntt.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"^k_ntt_dif" -s 3 -c 1 -o $OUT/prof_k_ntt_dif $CMD2 > $OUT/ncu_k_ntt.log 2>&1
echo "ncu full k_ntt rc=$?"
# NEXT-row kernels from the probe (after a plain run of the same probe): the precomputed-quotient
# DIF rows at 2^14 (the probe times REDC DIF x13, DIT x13, then the PQ DIF) and the 3-pass large transform's column kernel at 2^26
python scripts/probe.py --what ntt --logn 14 > $OUT/plain_probe_ntt.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"^k_ntt_dif" -s 13 -c 1 \
      -o $OUT/prof_k_ntt_dif_pq python scripts/probe.py --what ntt --logn 14 > $OUT/ncu_k_ntt_pq.log 2>&1
echo "ncu full k_ntt_dif pq rc=$?"
python scripts/probe.py --what nttlarge --logn 26 > $OUT/plain_probe_nttlarge.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"k_ntt_col" -s 3 -c 1 \
      -o $OUT/prof_k_ntt_col python scripts/probe.py --what nttlarge --logn 26 > $OUT/ncu_k_ntt_col.log 2>&1
echo "ncu full k_ntt_col rc=$?"
# summarise on the box (the .ncu-rep files are too large to bring back): profiles/ summaries into
# $OUT/prof_out/, then drop the reports
python scripts/ncu_summary.py --round $ROUND --src $OUT > $OUT/summary.log 2>&1; echo "summary rc=$?"
mkdir -p $OUT/prof_out
cp profiles/${ROUND}_ncu_summary.md profiles/${ROUND}_launches.csv profiles/ncu_summary.json $OUT/prof_out/
tail -1 $OUT/bench_final.log > $OUT/prof_out/${ROUND}_bench_step.json
rm -f $OUT/*.ncu-rep
