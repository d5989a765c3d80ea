for L in 28 400 700 400,640,880,1120,1360,1600 16,700,3,1600 129,255,257,3; do timeout 60 python tools/attn_check.py 7 4 $L; done
for sl in 0 32; do for st in 0 900; do timeout 60 python tools/attn_bench.py --opt 0=7 --opt 21=$sl --opt 5=$st --lens 700x32; done; done
timeout 60 python tools/attn_bench.py --opt 0=4 --lens 700x32
CFD_OPTS="0=7" timeout 120 python tools/attn_trace.py 32 | head -30
