#!/bin/bash
mkdir -p gpurun_out; o=gpurun_out/r2h_embst.txt; : > $o
for rep in 1 2; do for v in st6 st8 ""; do
  CFD_LIB_VARIANT=$v timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 10 > gpurun_out/ab_tmp.json 2>/dev/null
  python - "$v" >> $o <<'PY'
import json, sys
d = json.load(open("gpurun_out/ab_tmp.json")); k = d["kernels"]
print(f"{sys.argv[1] or 'st12':6s} {d['value']:9.0f} frames/s  embed_c {k['gemm_embed_c']['us_per_launch_alone']:.1f} us  embed_f {k['gemm_embed_f']['us_per_launch_alone']:.1f}  qkv {k['gemm_qkv']['us_per_launch_alone']:.1f}")
PY
done; done
echo done >> $o
