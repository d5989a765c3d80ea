#!/bin/bash
mkdir -p gpurun_out; o=gpurun_out/r2i_o11b.txt; : > $o
run() { timeout 120 python bench.py --no-cpu-baseline --no-e2e --steps 3 --warmup 3 "$@" > gpurun_out/ab_tmp.json 2>gpurun_out/ab_tmp.err; echo "$* rc=$? $(python -c "import json; d=json.load(open('gpurun_out/ab_tmp.json')); print(d['value'], d['check']['pass'])" 2>/dev/null)" >> $o; }
run --option 11=0
run
run --option 4=0 --option 20=1 --frames 32
run --option 4=0 --option 20=1
tail -3 gpurun_out/ab_tmp.err >> $o
timeout 300 python -m pytest tests -m gpu -q -x > gpurun_out/r2i_o11b_pytest.log 2>&1; echo "suite rc=$?" >> $o; tail -1 gpurun_out/r2i_o11b_pytest.log >> $o
echo done >> $o
