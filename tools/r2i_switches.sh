#!/bin/bash
# every tuning switch at the bench size (128 c640 frames, one lane), one at a time: runs, checks against the oracle
mkdir -p gpurun_out; o=gpurun_out/r2i_switches.txt; : > $o
run() { timeout 150 python bench.py --no-cpu-baseline --no-e2e --steps 3 --warmup 3 "$@" > gpurun_out/ab_tmp.json 2>gpurun_out/ab_tmp.err; echo "$* rc=$? $(python -c "import json; d=json.load(open('gpurun_out/ab_tmp.json')); print(d['value'], d['check']['pass'])" 2>/dev/null)" >> $o; }
for opt in "0=1" "1=0" "1=8" "2=0" "3=0" "5=0" "7=0" "13=0" "14=0" "15=0" "16=0" "17=74" "18=1" "21=1" "21=2" "22=3" "23=0" "24=0" "25=0"; do
  run --option $opt
done
echo done >> $o
