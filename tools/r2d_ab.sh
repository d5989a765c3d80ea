#!/bin/bash
# A/B: CFD_LIB_VARIANT=$1 vs the default library, interleaved, at bench shapes
mkdir -p gpurun_out; o=gpurun_out/r2d_ab_${1}.txt; : > $o
for rep in 1 2; do for v in $1 ""; do echo "lib ${v:-current}" >> $o; for l in 400x128 700x128 1600x8; do
  CFD_LIB_VARIANT=$v timeout 120 python tools/attn_bench.py --lens $l >> $o 2>&1; done; done; done
echo ab_done >> $o
