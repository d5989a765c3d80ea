#!/bin/bash
# attention v6 correctness (vs torch fp32) incl. spiky logits, then timing vs v4
for v in 6 4; do
  for lens in 400 700 28 1 64 65 129 257 400,640,880,1120,1360,1600 16,700,3,1600; do
    timeout 60 python tools/attn_check.py $v 4 $lens | head -3
  done
  for lens in 700 400,640,880,1120,1360,1600 1600; do
    CFD_SPIKE=1 timeout 60 python tools/attn_check.py $v 4 $lens | head -3
  done
done
for v in 4 6; do
  for npp in 4 6; do
    for lens in 700x32 400x32 1600x8; do
      timeout 60 python tools/attn_bench.py --variant $v --npp $npp --lens $lens --reps 50
    done
  done
done
