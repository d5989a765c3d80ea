#!/bin/bash
# attention v4: warpgroup start stagger (cycles) sweep at the bench's shapes
for st in 0 300 600 900; do
  for lens in 700x32 400x32; do
    timeout 60 python tools/attn_bench.py --variant 4 --npp 4 --lens $lens --reps 50 --stagger $st
  done
done
