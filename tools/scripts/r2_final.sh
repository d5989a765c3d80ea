set -x
python bench.py > gpurun_out/bench_c640.json 2> gpurun_out/bench_c640.err
for w in c640b1 batch6 fine8 multi48; do python bench.py --workload $w --cpu-seconds 8 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; done
python bench.py --workload multi48 --mix s348 --cpu-seconds 8 > gpurun_out/bench_multi48_s348.json 2> gpurun_out/bench_multi48_s348.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-check --no-e2e > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"attn7|mlp_tc|gemm_tc|score|gather|select" --csv --log-file gpurun_out/step_traffic.csv python tools/step_once.py 128 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:attn7 -s 6 -c 2 -o gpurun_out/attn7_full python tools/step_once.py 128 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:mlp_tc -s 6 -c 2 -o gpurun_out/mlp_full python tools/step_once.py 128 1 > /dev/null 2>&1
ls -la gpurun_out
