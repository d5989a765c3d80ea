#!/bin/bash
# v4 K/V ring depth: correctness + timing at 4 / 6 / 8 stages
for st in 6 8; do
  for lens in 400 700 65 16,700,3,1600 400,640,880,1120,1360,1600; do
    CFD_STAGES=$st timeout 60 python tools/attn_check.py 4 4 $lens | head -1
  done
done
for st in 4 6 8; do
  for lens in 700x32 400x32 1600x8 400x1,640x1,880x1,1120x1,1360x1,1600x1; do
    timeout 60 python tools/attn_bench.py --variant 4 --npp 4 --stages $st --lens $lens --reps 50
  done
done
