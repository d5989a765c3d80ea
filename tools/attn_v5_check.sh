#!/bin/bash
# attention v5 correctness (vs torch fp32) over ragged length mixes, then timing vs v4
for lens in 400 700 28 1 64 65 129 255 256 257 400,640,880,1120,1360,1600 400,400,700,880,1120,1600 1600,1600,1600 16,700,3,1600; do
  timeout 60 python tools/attn_check.py 5 4 $lens || echo "FAIL $lens"
done
for v in 4 5; do
  for lens in 700x32 400x32 1600x8 400x1,640x1,880x1,1120x1,1360x1,1600x1; do
    timeout 60 python tools/attn_bench.py --variant $v --npp 4 --lens $lens --reps 50
  done
done
