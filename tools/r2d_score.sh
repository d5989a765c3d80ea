#!/bin/bash
mkdir -p gpurun_out; o=gpurun_out/r2d_score_npp.txt; : > $o
for v in np0 np2 "" np6 np8; do echo "variant ${v:-default(np4)}" >> $o; for a in "64 400" "128 400"; do CFD_LIB_VARIANT=$v timeout 120 python tools/score_bench.py $a >> $o 2>&1; done; done
echo score_done >> $o
