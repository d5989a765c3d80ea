#!/bin/bash
# attention v7 ablations (timing only): S TMEM loads replaced by registers / P stores dropped / no exps / all three
mkdir -p gpurun_out; o=gpurun_out/r2f_ablate2.txt; : > $o
for v in "" sld pst noexp all3; do echo "lib ${v:-default}" >> $o; for l in 700x128 400x128; do
  CFD_LIB_VARIANT=$v timeout 120 python tools/attn_bench.py --lens $l >> $o 2>&1; done; done
echo ablate_done >> $o
