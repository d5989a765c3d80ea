#!/bin/bash
mkdir -p gpurun_out; o=gpurun_out/r2i_o11d.txt; : > $o
timeout 400 python -m pytest tests -m gpu -q > gpurun_out/r2i_o11d_pytest.log 2>&1; echo "suite rc=$?" >> $o; tail -1 gpurun_out/r2i_o11d_pytest.log >> $o
run() { timeout 120 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3 "$@" > gpurun_out/ab_tmp.json 2>gpurun_out/ab_tmp.err; echo "$* rc=$? $(python -c "import json; d=json.load(open('gpurun_out/ab_tmp.json')); print(d['value'], d['check']['pass'])" 2>/dev/null)" >> $o; }
run --option 11=0
run
run --option 4=0
run --option 19=0
echo done >> $o
