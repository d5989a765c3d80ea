#!/bin/bash
# attention with spiky logits (rows far below / above the running max) for every variant
for v in 2 3 4 5 6; do
  for lens in 700 400,640,880,1120,1360,1600 1600; do
    CFD_SPIKE=1 timeout 60 python tools/attn_check.py $v 4 $lens | head -2
  done
done
