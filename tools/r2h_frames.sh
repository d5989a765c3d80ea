#!/bin/bash
# frames in flight per GPU (one lane): persistent-kernel round quantisation (items / 592 warpgroups, tiles / 74 pairs)
mkdir -p gpurun_out; o=gpurun_out/r2h_frames.txt; : > $o
for f in 128 148 160 192 222 256; do
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-check --steps 10 --frames $f > gpurun_out/ab_tmp.json 2>/dev/null
  python - "$f" >> $o <<'PY'
import json, sys
d = json.load(open("gpurun_out/ab_tmp.json")); k = d["kernels"]
print(f"frames {sys.argv[1]:>4s}: {d['value']:9.0f} frames/s  step {d['ms_per_step']:.4f} ms  attn {k['attention']['us_per_launch_alone']:.1f} us "
      f"({k['attention']['frac_tensor_burst']:.3f})  mlp {k['mlp_fused']['us_per_launch_alone']:.1f} ({k['mlp_fused']['frac_tensor_burst']:.3f})")
PY
done
echo done >> $o
