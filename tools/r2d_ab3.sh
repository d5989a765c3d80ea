#!/bin/bash
mkdir -p gpurun_out; o=gpurun_out/r2d_ab3.txt; : > $o
for v in base nozero qvalid ""; do echo "lib ${v:-current}" >> $o; for l in 400x128 700x128; do
  CFD_LIB_VARIANT=$v timeout 120 python tools/attn_bench.py --lens $l >> $o 2>&1; done; done
echo ab_done >> $o
