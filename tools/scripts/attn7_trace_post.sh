python -m paper_2505_23317_b200.build --trace --force > /dev/null
for B in 32; do echo "=== B=$B (MMA events after issue)"; CFD_LIB_DEBUG=1 timeout 120 python tools/attn_trace.py $B; done
