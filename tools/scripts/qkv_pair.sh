python -m pytest tests -m gpu -q -x > gpurun_out/t.log 2>&1; tail -2 gpurun_out/t.log
for f in 32 128; do for o in "" "--option 23=0"; do python bench.py --frames $f --no-cpu-baseline --no-check --no-e2e --steps 10 $o > gpurun_out/b.json 2>/dev/null; python -c "
import json;j=json.load(open('gpurun_out/b.json'));k=j['kernels']
print('frames $f $o', j['value'], j['ms_per_step'], 'qkv', k['gemm_qkv']['us_per_launch_alone'], k['gemm_qkv']['frac_tensor_burst'], k['gemm_qkv']['share_of_step'])"; done; done
