#!/bin/bash
# embed pair (option 25, default on) and the MLP MMA_o overlap (option 26 / variant "ovl"): GPU suite on both
# libraries, then bench A/B through options
mkdir -p gpurun_out; o=gpurun_out/r2f_ab.txt; : > $o
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r2f_pytest_default.log 2>&1; echo "default suite rc=$?" >> $o; tail -2 gpurun_out/r2f_pytest_default.log >> $o
CFD_LIB_VARIANT=ovl timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r2f_pytest_ovl.log 2>&1; echo "ovl suite rc=$?" >> $o; tail -2 gpurun_out/r2f_pytest_ovl.log >> $o
for rep in 1 2; do for opt in "--option 25=0" "" "--option 26=1"; do
  timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 10 $opt > gpurun_out/ab_tmp.json 2>/dev/null
  python - "$opt" >> $o <<'PY'
import json, sys
d = json.load(open("gpurun_out/ab_tmp.json"))
k = d["kernels"]
print(f"{sys.argv[1] or 'default':14s} {d['value']:9.0f} frames/s  step {d['ms_per_step']:.4f} ms  " +
      "  ".join(f"{n} {k[n]['us_per_launch_alone']:.1f}" for n in ("attention", "mlp_fused", "gemm_qkv", "gemm_embed_c", "score")))
PY
done; done
echo ab_done >> $o
