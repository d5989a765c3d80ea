#!/bin/bash
# ncu --set full of one bench step's 12 attention launches (6 coarse N=400, 6 refine N=700):
# DRAM bytes per launch for bench.py's roofline "traffic" (profiles/traffic.json)
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none -k regex:attn7_tc_kernel --launch-skip 12 -c 12 \
  -o gpurun_out/attn_step_full -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-check \
  > gpurun_out/attn_step_full.log 2>&1
ncu -i gpurun_out/attn_step_full.ncu-rep --page raw --csv \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size > gpurun_out/attn_step_traffic.csv 2>&1
echo traffic_done
