#!/bin/bash
# re-entry check of HEAD: GPU suite, smoke, default bench line, attention micro-bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r2d_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2d_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2d_smoke.log 2>&1; echo rc=$? >> gpurun_out/r2d_smoke.log
timeout 900 python bench.py > gpurun_out/r2d_bench_c640.json 2> gpurun_out/r2d_bench_c640.err
for l in 700x128 400x128 1600x8 700x32; do timeout 120 python tools/attn_bench.py --lens $l >> gpurun_out/r2d_attn_bench.txt 2>&1; done
echo check_done
