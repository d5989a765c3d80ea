#!/bin/bash
mkdir -p gpurun_out; o=gpurun_out/r2h_e2e2.txt; : > $o
for st in 10 40 80; do for sk in "" "h2d,d2h"; do
  CFD_E2E_SKIP=$sk timeout 300 python bench.py --no-cpu-baseline --no-check --steps $st > gpurun_out/ab_tmp.json 2>/dev/null
  python - "$sk" "$st" >> $o <<'PY'
import json, sys
d = json.load(open("gpurun_out/ab_tmp.json"))
print(f"steps {sys.argv[2]:>3s} skip {sys.argv[1] or '-':8s} value {d['value']:8.0f}  e2e {d['e2e']['value']:8.0f}")
PY
done; done
echo done >> $o
