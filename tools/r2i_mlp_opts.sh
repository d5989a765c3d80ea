#!/bin/bash
mkdir -p gpurun_out; o=gpurun_out/r2i_mlp_opts.txt; : > $o
for opt in "" "--option 4=0" "--option 4=0 --option 20=1" "--option 11=0" "--option 23=0" "--option 16=0"; do
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-check --steps 10 $opt > gpurun_out/ab_tmp.json 2>/dev/null
  python - "$opt" >> $o <<'PY'
import json, sys
d = json.load(open("gpurun_out/ab_tmp.json")); k = d["kernels"]
print(f"{sys.argv[1] or 'default':28s} {d['value']:9.0f} frames/s  mlp {k['mlp_fused']['us_per_launch_alone']:.1f}  qkv {k['gemm_qkv']['us_per_launch_alone']:.1f}  attn {k['attention']['us_per_launch_alone']:.1f}")
PY
done
echo done >> $o
