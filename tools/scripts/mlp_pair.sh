python -m pytest tests/test_gpu_parity.py -m gpu -q -k "pair or fused" > gpurun_out/pair_test.log 2>&1; tail -3 gpurun_out/pair_test.log
for o in "" "--option 4=1"; do python bench.py --no-cpu-baseline --no-check --no-e2e $o > gpurun_out/b.json 2>/dev/null; python -c "
import json;j=json.load(open('gpurun_out/b.json'));k=j['kernels']
print('$o', j['value'], j['ms_per_step'], 'mlp', k['mlp_fused']['us_per_launch_alone'], k['mlp_fused'].get('share_of_step'), j['roofline']['kernel'], j['roofline']['frac'])"; done
