#!/bin/bash
mkdir -p gpurun_out; o=gpurun_out/r2h_gather.txt; : > $o
for rep in 1 2; do for v in gu4 gu2 gu1; do
  CFD_LIB_VARIANT=$v timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 10 > gpurun_out/ab_tmp.json 2>/dev/null
  python - "$v" >> $o <<'PY'
import json, sys
d = json.load(open("gpurun_out/ab_tmp.json")); k = d["kernels"]
print(f"{sys.argv[1] or 'GU8':6s} {d['value']:9.0f} frames/s  gather {k['gather']['us_per_launch_alone']:.1f} us ({k['gather']['gbs']:.0f} GB/s) check {d['check']['pass']}")
PY
done; done
echo done >> $o
