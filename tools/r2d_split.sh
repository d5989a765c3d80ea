#!/bin/bash
# attention v7 split tail tiles: correctness + timing at bench shapes
mkdir -p gpurun_out; o=gpurun_out/r2d_split.txt; : > $o
for l in 400,400,400 700,60,1600,16,129,400 64,65,1,127,128,129 160,161,33,32,31,2 16 400; do timeout 120 python tools/attn_check.py 7 2 $l >> $o 2>&1; done
for l in 400x128 700x128 1600x8 700x32 400x32; do timeout 120 python tools/attn_bench.py --lens $l >> $o 2>&1; done
timeout 600 python -m pytest tests -m gpu -q -x >> $o 2>&1
echo split_done >> $o
