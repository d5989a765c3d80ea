#!/bin/bash
# v4 split MMA accumulator chains (option 10): correctness + timing
for lens in 400 700 28 1 32 33 64 65 257 400,640,880,1120,1360,1600 16,700,3,1600; do
  CFD_SPLIT=1 timeout 60 python tools/attn_check.py 4 4 $lens | head -2
done
CFD_SPLIT=1 CFD_SPIKE=1 timeout 60 python tools/attn_check.py 4 4 400,640,880,1120,1360,1600 | head -2
for sp in 0 1; do
  for lens in 700x32 400x32 1600x8; do
    timeout 60 python tools/attn_bench.py --variant 4 --npp 4 --split $sp --lens $lens --reps 50
  done
done
