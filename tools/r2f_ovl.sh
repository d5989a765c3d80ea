#!/bin/bash
mkdir -p gpurun_out; o=gpurun_out/r2f_ovl.txt; : > $o
CFD_LIB_DEBUG=1 timeout 100 python tools/step_once.py 64 1 >> $o 2>&1; echo "debug step rc=$?" >> $o
if grep -q "ok 64 1" $o; then
  CFD_LIB_VARIANT=ovl timeout 300 python -m pytest tests -m gpu -q -x > gpurun_out/r2f_pytest_ovl.log 2>&1; echo "ovl suite rc=$?" >> $o; tail -2 gpurun_out/r2f_pytest_ovl.log >> $o
  for rep in 1 2; do for opt in "" "--option 26=1"; do
    timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 10 $opt > gpurun_out/ab_tmp.json 2>/dev/null
    python - "$opt" >> $o <<'PY'
import json, sys
d = json.load(open("gpurun_out/ab_tmp.json"))
k = d["kernels"]
print(f"{sys.argv[1] or 'default':14s} {d['value']:9.0f} frames/s  step {d['ms_per_step']:.4f} ms  " +
      "  ".join(f"{n} {k[n]['us_per_launch_alone']:.1f}" for n in ("attention", "mlp_fused", "gemm_qkv", "gemm_embed_c", "score")))
PY
  done; done
fi
echo ovl_done >> $o
