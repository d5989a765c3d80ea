#!/bin/bash
# tail-mix item order (option 25): correctness on ragged / coarse batches, timing at bench shapes
mkdir -p gpurun_out; o=gpurun_out/r2d_mix.txt; : > $o
for l in 400,400,400 700,60,1600,16,129,400; do CFD_OPTS="25=1" timeout 120 python tools/attn_check.py 7 2 $l >> $o 2>&1; done
for opt in "" "--opt 25=1"; do for l in 400x128 700x128 1600x8 700x32; do
  timeout 120 python tools/attn_bench.py $opt --lens $l >> $o 2>&1; done; done
echo mix_done >> $o
