#!/bin/bash
# A/B of a library variant through the whole bench step: CFD_LIB_VARIANT=$1 vs the default, twice
mkdir -p gpurun_out; o=gpurun_out/r2e_ab_$1.txt; : > $o
for rep in 1 2; do for v in $1 ""; do
  CFD_LIB_VARIANT=$v timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 10 > gpurun_out/ab_tmp.json 2>/dev/null
  python - "$v" >> $o <<'PY'
import json, sys
d = json.load(open("gpurun_out/ab_tmp.json"))
k = d["kernels"]
print(f"lib {sys.argv[1] or 'current':8s} {d['value']:9.0f} frames/s  step {d['ms_per_step']:.4f} ms  " +
      "  ".join(f"{n} {k[n]['us_per_launch_alone']:.1f}" for n in ("attention", "mlp_fused", "gemm_qkv", "score")))
PY
done; done
echo ab_done >> $o
