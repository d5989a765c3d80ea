#!/bin/bash
mkdir -p gpurun_out; o=gpurun_out/r2i_o11.txt; : > $o
run() { timeout 120 python bench.py --no-cpu-baseline --no-e2e --no-check --steps 3 --warmup 3 "$@" > gpurun_out/ab_tmp.json 2>/dev/null; echo "$* rc=$? $(python -c "import json; d=json.load(open('gpurun_out/ab_tmp.json')); print(d['value'])" 2>/dev/null)" >> $o; }
CFD_LIB_VARIANT=old39 run --option 11=0
run --option 11=0 --frames 32
run --option 11=0 --frames 32 --streams 2
CFD_LIB_VARIANT=old39 run --option 11=0 --frames 32
echo done >> $o
