#!/bin/bash
# A/B timing of attention variants at the bench's shapes: tools/attn_ab.sh "4 5"
for v in ${1:-4 5}; do
  for lens in 700x32 400x32 1600x8 400x1,640x1,880x1,1120x1,1360x1,1600x1; do
    timeout 60 python tools/attn_bench.py --variant $v --npp ${NPP:-4} --lens $lens --reps 50
  done
done
