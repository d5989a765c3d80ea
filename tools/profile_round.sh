#!/bin/bash
# ncu evidence for profiles/: the launch list of a short bench run (single-pass metric, clocks
# not locked) and one `--set full` capture per hot kernel.  Run on the GPU box via gpurun.
#   tools/profile_round.sh <tag> [list|full|both]
set -u
TAG=${1:-r1}
WHAT=${2:-both}
OUT=gpurun_out
mkdir -p $OUT
BENCH="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-check"
if [ "$WHAT" != full ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
    --log-file $OUT/launches_$TAG.csv $BENCH > $OUT/launches_$TAG.log 2>&1
fi
if [ "$WHAT" != list ]; then
  # name  demangled-name regex  launches to skip (warm-up first)
  while read -r name rx skip; do
    if [ -n "${ONLY:-}" ] && ! echo " $ONLY " | grep -q " $name "; then continue; fi
    timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
      -k "regex:$rx" --launch-skip "$skip" -c 1 -o "$OUT/full_${TAG}_$name" -f $BENCH \
      > "$OUT/full_${TAG}_$name.log" 2>&1
  done <<LIST
mlp mlp_tc_kernel 20
attn attn7_tc_kernel 20
oproj gemm_tc_kernel<.int.256,..int.2,..int.5 20
qkv gemm_tc_kernel<.int.256,..int.[34],..int.0 20
score score_tc_kernel 2
gather gather_kernel 2
LIST
fi
echo profile_done
