#!/bin/bash
# v7 switches at the 128-frame bench shapes: NPP (key 1), start stagger (key 5), warpgroups (key 22)
mkdir -p gpurun_out; o=gpurun_out/r2h_sweep.txt; : > $o
for opt in "" "--opt 1=0" "--opt 1=4" "--opt 5=0" "--opt 5=350" "--opt 5=1400" "--opt 22=3" "--opt 16=0"; do for l in 700x128 400x128; do
  timeout 120 python tools/attn_bench.py $opt --lens $l >> $o 2>&1; done; done
echo sweep_done >> $o
