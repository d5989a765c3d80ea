for L in 28 400 700 400,640,880,1120,1360,1600 16,700,3,1600 129,255,257,3; do timeout 60 python tools/attn_check.py 7 4 $L; done
for nwg in 3 4; do for L in 700x32 400x32 1600x8; do timeout 60 python tools/attn_bench.py --opt 0=7 --opt 22=$nwg --lens $L; done; done
timeout 60 python tools/attn_bench.py --opt 0=7 --opt 21=0 --lens 700x32
timeout 60 python tools/attn_bench.py --opt 0=4 --lens 700x32
CFD_OPTS="0=7 22=3" timeout 120 python tools/attn_trace.py 32 | head -16
CFD_OPTS="0=7 22=4" timeout 120 python tools/attn_trace.py 32 | head -16
