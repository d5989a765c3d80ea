#!/bin/bash
# attention v7 ablations (timing only, wrong results): no exponentials / no PV MMAs / neither
mkdir -p gpurun_out; o=gpurun_out/r2e_ablate.txt; : > $o
for v in "" noexp nopv noboth; do echo "lib ${v:-default}" >> $o; for l in 700x128 400x128; do
  CFD_LIB_VARIANT=$v timeout 120 python tools/attn_bench.py --lens $l >> $o 2>&1; done; done
echo ablate_done >> $o
