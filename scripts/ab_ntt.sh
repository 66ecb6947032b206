#!/bin/bash
# A/B of NTT row kernels on one box: alternates the in-tree library and build_ab/libmont_<tag>.so
# for each tag (scripts/ab_build.sh), twice each, printing one line per (lib, variant, log_n).
# usage: TAGS="a b" scripts/ab_ntt.sh [log_n ...]   (env PROBE_NTT_VARIANTS as in scripts/probe.py)
SIZES=${@:-12 13 14 15}
for rep in 1 2; do
  for lib in main $TAGS; do
    for L in $SIZES; do
      if [ $lib = main ]; then unset MONT_LIB_AB; else export MONT_LIB_AB=$lib; fi
      timeout 300 python scripts/probe.py --what ntt --logn $L | sed "s/^{/{\"lib\": \"$lib\", \"rep\": $rep, /"
    done
  done
done
