for o in "" "--option 22=3" "--option 1=0" "--option 1=4" "--option 5=0" "--option 0=4"; do python bench.py --no-cpu-baseline --no-check --no-e2e --steps 10 $o > gpurun_out/b.json 2>/dev/null; python -c "
import json;j=json.load(open('gpurun_out/b.json'));k=j['kernels']
print('$o', j['value'], j['ms_per_step'], 'attn', k['attention']['us_per_launch_alone'], k['attention']['frac_tensor_burst'], k['attention']['share_of_step'])"; done
