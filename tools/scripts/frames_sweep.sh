for f in 32 48 64; do for s in 1 2 3; do python bench.py --frames $f --streams $s --no-cpu-baseline --no-check --no-e2e --steps 10 > gpurun_out/b.json 2>/dev/null; python -c "
import json;j=json.load(open('gpurun_out/b.json'));print('frames $f streams $s', j['value'], j['ms_per_step'])"; done; done
