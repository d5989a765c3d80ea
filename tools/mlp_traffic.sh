#!/bin/bash
# ncu --set full of one bench step's 12 fused-MLP launches (6 coarse, 6 refine): DRAM bytes per
# launch for bench.py's roofline "traffic" (profiles/traffic.json, key mlp_fused)
mkdir -p gpurun_out
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:mlp_tc_kernel --launch-skip 12 -c 12 \
  -o gpurun_out/mlp_step_full -f python bench.py --steps 2 --warmup 3 --streams 1 --no-cpu-baseline --no-check \
  > gpurun_out/mlp_step_full.log 2>&1
ncu -i gpurun_out/mlp_step_full.ncu-rep --page raw --csv \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active > gpurun_out/mlp_step_traffic.csv 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
  --log-file gpurun_out/launches_r1f.csv python bench.py --steps 2 --warmup 3 --streams 1 --no-cpu-baseline --no-check \
  > gpurun_out/launches_r1f.log 2>&1
echo traffic_done
