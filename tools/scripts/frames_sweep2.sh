for f in 96 128; do for s in 2 4; do python bench.py --frames $f --streams $s --no-cpu-baseline --no-check --no-e2e --steps 10 > gpurun_out/b.json 2>/dev/null; python -c "
import json;j=json.load(open('gpurun_out/b.json'));print('frames $f streams $s', j['value'], j['ms_per_step'])"; done; done
