#!/bin/bash
# v4 exp-phase token ring (option 9): correctness + timing
for lens in 400 700 28 65 257 400,640,880,1120,1360,1600 16,700,3,1600; do
  CFD_TOKEN=1 timeout 60 python tools/attn_check.py 4 4 $lens | head -2
done
CFD_TOKEN=1 CFD_SPIKE=1 timeout 60 python tools/attn_check.py 4 4 400,640,880,1120,1360,1600 | head -2
for tok in 0 1; do
  for npp in 4 6 0; do
    for lens in 700x32 400x32 1600x8; do
      timeout 60 python tools/attn_bench.py --variant 4 --npp $npp --token $tok --lens $lens --reps 50
    done
  done
done
