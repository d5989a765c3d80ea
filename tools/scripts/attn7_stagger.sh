for st in 0 300 600 900 1300 2000; do timeout 60 python tools/attn_bench.py --opt 0=7 --opt 5=$st --lens 700x32; done
for st in 0 900; do timeout 60 python tools/attn_bench.py --opt 0=7 --opt 5=$st --lens 400x32; done
CFD_OPTS="0=7 5=900" timeout 120 python tools/attn_trace.py 32 | head -40
