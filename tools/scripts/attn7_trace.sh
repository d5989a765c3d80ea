# v7 pipeline traces with the trace-only debug library: B = 4 (one or two warpgroups per SM)
# and B = 32 (four per SM)
python -m paper_2505_23317_b200.build --trace > /dev/null
for B in 4 32; do echo "=== B=$B"; CFD_LIB_DEBUG=1 timeout 120 python tools/attn_trace.py $B; done
