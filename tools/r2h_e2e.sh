#!/bin/bash
mkdir -p gpurun_out; o=gpurun_out/r2h_e2e.txt; : > $o
for sk in "" h2d d2h "h2d,d2h"; do
  CFD_E2E_SKIP=$sk timeout 300 python bench.py --no-cpu-baseline --no-check --steps 10 > gpurun_out/ab_tmp.json 2>/dev/null
  python - "$sk" >> $o <<'PY'
import json, sys
d = json.load(open("gpurun_out/ab_tmp.json"))
print(f"skip {sys.argv[1] or '-':8s} value {d['value']:8.0f}  e2e {d['e2e']['value']:8.0f}  e2e_bf16 {d.get('e2e_bf16_input', {}).get('value', 0):8.0f}")
PY
done
echo done >> $o
