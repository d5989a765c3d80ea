for ms in 100 1000; do
  for i in 1 2 3 4 5; do
    CFD_BENCH_CLOCK_MS=$ms python bench.py --no-cpu-baseline --no-check > gpurun_out/st.json 2>/dev/null
    python -c "import json,sys; d=json.load(open('gpurun_out/st.json')); print('clock_ms=$ms', d['value'], d['ms_per_step'], d['step_ms_min'], d['step_ms_max'], d['clocks']['samples'])"
  done
done
