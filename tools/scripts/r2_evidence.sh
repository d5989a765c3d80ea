set -x
python -m pytest tests -m gpu -q > gpurun_out/gputest.log 2>&1; tail -3 gpurun_out/gputest.log
python bench.py > gpurun_out/bench_c640.json 2> gpurun_out/bench_c640.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-check --no-e2e > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:attn7 -s 12 -c 2 -o gpurun_out/attn7_full python tools/step_once.py 16 2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:mlp_tc -s 12 -c 2 -o gpurun_out/mlp_full python tools/step_once.py 16 2 > /dev/null 2>&1
ls -la gpurun_out
