#!/bin/bash
mkdir -p gpurun_out; o=gpurun_out/r2h_pst32.txt; : > $o
for l in 400,400,400 700,60,1600,16,129,400; do CFD_LIB_VARIANT=pst32 timeout 60 python tools/attn_check.py 7 2 $l >> $o 2>&1; done
for rep in 1 2; do for v in pst32 ""; do echo "lib ${v:-current}" >> $o; for l in 700x128 400x128; do
  CFD_LIB_VARIANT=$v timeout 120 python tools/attn_bench.py --lens $l >> $o 2>&1; done; done; done
echo done >> $o
