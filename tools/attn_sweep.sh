#!/bin/bash
# correctness of each attention variant on ragged cases (debug lib: hangs trap)
export CFD_LIB_DEBUG=${CFD_LIB_DEBUG:-1}
DEFAULT_CASES="16 64 65 128 129 400 700,1 400,640,880,1120,1360,1600 129,255,257,3 1600,1600,1600,1600,1600,1600,1600,1600 700,700,700,700,700,700,700,700,700,700,700,700,700,700,700,700,700,700,700,700,700,700,700,700,700,700,700,700,700,700,700,700"
CASES=${CASES:-$DEFAULT_CASES}
for v in ${VARIANTS:-3}; do for npp in ${NPPS:-0}; do
  for lens in $CASES; do
    timeout 60 python tools/attn_check.py $v $npp $lens 2>&1 | grep -vE "^\s*$" | head -${LINES_PER:-40}
  done
done; done
