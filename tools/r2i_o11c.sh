#!/bin/bash
mkdir -p gpurun_out; o=gpurun_out/r2i_o11c.txt; : > $o
run() { timeout 120 python bench.py --no-cpu-baseline --no-e2e --steps 3 --warmup 3 "$@" > gpurun_out/ab_tmp.json 2>gpurun_out/ab_tmp.err; echo "$* rc=$? $(python -c "import json; d=json.load(open('gpurun_out/ab_tmp.json')); print(d['value'], d['check']['pass'])" 2>/dev/null)" >> $o; }
run --option 11=0 --option 4=0
run --option 11=0 --frames 64
run --option 11=0 --frames 48
echo done >> $o
