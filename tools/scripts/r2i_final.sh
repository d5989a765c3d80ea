# end-of-session evidence (round 2, session i (final)): GPU suite, bench lines of every workload + the oracle arm,
# ncu launch list of the bench step, per-launch DRAM traffic of one 128-frame step, full captures of the
# attention, fused MLP and score kernels
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/i_pytest.log 2>&1; echo rc=$? >> gpurun_out/i_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/i_smoke.log 2>&1; echo rc=$? >> gpurun_out/i_smoke.log
timeout 900 python bench.py > gpurun_out/i_bench_c640.json 2> gpurun_out/i_bench_c640.err
for w in c640b1 batch6 fine8 multi48; do timeout 900 python bench.py --workload $w --cpu-seconds 8 > gpurun_out/i_bench_$w.json 2> gpurun_out/i_bench_$w.err; done
timeout 900 python bench.py --workload multi48 --mix s348 --cpu-seconds 8 > gpurun_out/i_bench_multi48_s348.json 2> gpurun_out/i_bench_multi48_s348.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/i_bench_reference.json 2> gpurun_out/i_bench_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/i_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-check --no-e2e > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"attn7|mlp_tc|gemm_tc|score|gather|select" --csv --log-file gpurun_out/i_step_traffic.csv python tools/step_once.py 128 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn7 -s 6 -c 2 -o gpurun_out/i_attn7_full python tools/step_once.py 128 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mlp_tc -s 6 -c 2 -o gpurun_out/i_mlp_full python tools/step_once.py 128 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:score -c 1 -o gpurun_out/i_score_full python tools/step_once.py 128 1 > /dev/null 2>&1
ls -la gpurun_out
CFD_DIST_BACKEND=gloo timeout 600 python bench.py --gpus 2 --workload multi48 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/i_multi48_2rank_shared_gpu.json 2> gpurun_out/i_multi48_2rank.err
