#!/bin/bash
# exp2 MUFU/polynomial split sweep of the default attention kernel at the bench's shapes
for npp in 0 2 4 6 8 10 12; do
  for lens in 700x32 400x32; do
    timeout 60 python tools/attn_bench.py --variant 4 --npp $npp --lens $lens --reps 50
  done
done
