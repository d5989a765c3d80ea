for sl in 0 32 128; do timeout 60 python tools/attn_bench.py --opt 0=7 --opt 21=$sl --lens 700x32; done
CFD_OPTS="0=7" timeout 120 python tools/attn_trace.py 32
