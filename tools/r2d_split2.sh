#!/bin/bash
mkdir -p gpurun_out; o=gpurun_out/r2d_split2.txt; : > $o
timeout 600 python -m pytest tests -m gpu -q -x >> $o 2>&1
for l in 400,400,400 700,60,1600,16,129,400 160,161,33,32,31,2 16; do timeout 120 python tools/attn_check.py 7 2 $l >> $o 2>&1; done
bash tools/r2d_ab.sh base
echo split_done >> $o
