#!/bin/bash
mkdir -p gpurun_out; o=gpurun_out/r2g_streams.txt; : > $o
for st in 1 2 3; do
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-check --steps 10 --streams $st > gpurun_out/ab_tmp.json 2>/dev/null
  python - "$st" >> $o <<'PY'
import json, sys
d = json.load(open("gpurun_out/ab_tmp.json"))
print(f"streams {sys.argv[1]}: {d['value']:9.0f} frames/s  step {d['ms_per_step']:.4f} ms  frames {d['config']['frames_per_step_per_gpu']}")
PY
done
echo done >> $o
