for o in 0 1; do
  for st in 2 1; do
    python bench.py --no-cpu-baseline --no-check --streams $st --option 16=$o > gpurun_out/dyn_${o}_${st}.json 2>/dev/null
    python -c "import json,sys; d=json.load(open(sys.argv[1])); print(sys.argv[1], d['value'], d['ms_per_step'], d['kernels']['attention']['ms_per_step'])" gpurun_out/dyn_${o}_${st}.json
  done
done
