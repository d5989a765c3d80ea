#!/bin/bash
# lanes per GPU: c640 with e2e, multi48 (balanced and S:348)
mkdir -p gpurun_out; o=gpurun_out/r2g_streams2.txt; : > $o
for w in "--workload c640" "--workload multi48" "--workload multi48 --mix s348"; do for st in 1 2; do
  timeout 300 python bench.py --no-cpu-baseline --no-check --steps 10 --streams $st $w > gpurun_out/ab_tmp.json 2>/dev/null
  python - "$st" "$w" >> $o <<'PY'
import json, sys
d = json.load(open("gpurun_out/ab_tmp.json"))
print(f"{sys.argv[2]:32s} streams {sys.argv[1]}: {d['value']:9.0f} frames/s  step {d['ms_per_step']:.4f} ms  e2e {d['e2e']['value']:9.0f}")
PY
done; done
echo done >> $o
