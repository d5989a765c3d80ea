#!/bin/bash
# end-of-round evidence: GPU tests, the default bench line, the ncu launch list of a bench step
# (single stream, so launches serialise cleanly) and --set full captures of one step's fused
# O-projection+MLP and attention launches (traffic), CUPTI timelines
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/final_pytest.log 2>&1; echo rc=$? >> gpurun_out/final_pytest.log
timeout 900 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
  --log-file gpurun_out/final_launches.csv python bench.py --steps 2 --warmup 3 --streams 1 --no-cpu-baseline --no-check \
  > gpurun_out/final_launches.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:mlp_tc_kernel --launch-skip 12 -c 12 \
  -o gpurun_out/final_mlp_full -f python bench.py --steps 2 --warmup 3 --streams 1 --no-cpu-baseline --no-check \
  > gpurun_out/final_mlp_full.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:attn7_tc_kernel --launch-skip 12 -c 12 \
  -o gpurun_out/final_attn_full -f python bench.py --steps 2 --warmup 3 --streams 1 --no-cpu-baseline --no-check \
  > gpurun_out/final_attn_full.log 2>&1
for k in mlp attn; do
  ncu -i gpurun_out/final_${k}_full.ncu-rep --page raw --csv \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active > gpurun_out/final_${k}_traffic.csv 2>&1
done
for k in mlp attn; do
  python tools/ncu_summary.py full gpurun_out/final_${k}_full.ncu-rep > gpurun_out/final_${k}_full.txt 2>&1
  rm -f gpurun_out/final_${k}_full.ncu-rep   # gpurun copies back <= 64 MiB
done
timeout 300 python tools/stream_timeline.py 2 > gpurun_out/final_timeline_s2.txt 2>&1
timeout 300 python tools/gap_profile.py > gpurun_out/final_timeline_s1.txt 2>&1
echo final_done
