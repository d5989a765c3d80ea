#!/bin/bash
mkdir -p gpurun_out; o=gpurun_out/r2h_embf.txt; : > $o
timeout 100 python tools/step_once.py 16 1 >> $o 2>&1; echo "step rc=$?" >> $o
if grep -q "ok 16 1" $o; then
  timeout 300 python -m pytest tests -m gpu -q -x > gpurun_out/r2h_embf_pytest.log 2>&1; echo "suite rc=$?" >> $o; tail -2 gpurun_out/r2h_embf_pytest.log >> $o
  for rep in 1 2; do for opt in "--option 25=0" ""; do
    timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 10 $opt > gpurun_out/ab_tmp.json 2>/dev/null
    python - "$opt" >> $o <<'PY'
import json, sys
d = json.load(open("gpurun_out/ab_tmp.json")); k = d["kernels"]
print(f"{sys.argv[1] or 'default':14s} {d['value']:9.0f} frames/s  embed_c {k['gemm_embed_c']['us_per_launch_alone']:.1f}  embed_f {k['gemm_embed_f']['us_per_launch_alone']:.1f} us  check {d['check']['pass']}")
PY
  done; done
fi
echo done >> $o
