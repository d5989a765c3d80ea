#!/bin/bash
mkdir -p gpurun_out; o=gpurun_out/r2h_score2.txt; : > $o
for a in "64 400" "128 400" "2 180" "1 16" "4 1024"; do timeout 60 python tools/score_bench.py $a >> $o 2>&1; done
timeout 300 python -m pytest tests -m gpu -q -x > gpurun_out/r2h_score2_pytest.log 2>&1; echo "suite rc=$?" >> $o; tail -2 gpurun_out/r2h_score2_pytest.log >> $o
timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 10 > gpurun_out/ab_tmp.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/ab_tmp.json')); k=d['kernels']
print('bench', d['value'], d['ms_per_step'], 'score', k['score']['us_per_launch_alone'], 'check', d['check']['pass'])" >> $o
echo done >> $o
