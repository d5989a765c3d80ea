#!/bin/bash
# attention v7 with S released as soon as it is in registers: correctness + timing at bench shapes
mkdir -p gpurun_out; o=gpurun_out/r2d_spec.txt; : > $o
for l in 400,400,400 700,60,1600,16,129,400 64,65,1,127,128,129; do timeout 120 python tools/attn_check.py 7 2 $l >> $o 2>&1; done
for l in 400x128 700x128 1600x8 700x32; do timeout 120 python tools/attn_bench.py --lens $l >> $o 2>&1; done
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "attention or attn" >> $o 2>&1
echo spec_done >> $o
