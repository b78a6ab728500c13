#!/bin/bash
# A/B timing of variant builds (build.py TACSNN_LIB_NAME / TACSNN_DEFS) on one layer:
#   scripts/ab_layer.sh <layer> <B> lib_a lib_b ...   (names under paper_2603_13810_b200/)
# Runs the variants round-robin twice so clock / thermal drift shows up as spread.
L=$1; B=$2; shift 2
for rep in 1 2; do
  for v in "$@"; do
    t=$(TACSNN_LIB=paper_2603_13810_b200/$v timeout 120 python scripts/profile_layer.py --config C5 --layer $L --B $B --iters 5 2>&1 | grep " ms " | tail -2 | awk '{print $1}' | tr '\n' ' ')
    echo "rep $rep layer $L $v: $t"
  done
done
