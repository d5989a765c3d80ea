#!/bin/bash
mkdir -p gpurun_out; o=gpurun_out/r2d_sleep.txt; : > $o
for opt in "" "--opt 21=1" "--opt 21=2" "--opt 21=8" "--opt 21=0" "--opt 24=0" "--opt 24=64"; do for l in 400x128 700x128; do
  timeout 120 python tools/attn_bench.py $opt --lens $l >> $o 2>&1; done; done
echo sleep_done >> $o
