for st in 0 350 700 1000; do for nwg in 3 4; do timeout 20 python tools/attn_bench.py --opt 0=7 --opt 22=$nwg --opt 5=$st --lens 700x32; done; done
for st in 0 700; do timeout 20 python tools/attn_bench.py --opt 0=7 --opt 22=4 --opt 5=$st --lens 400x32; timeout 20 python tools/attn_bench.py --opt 0=7 --opt 22=4 --opt 5=$st --lens 1600x8; done
CFD_OPTS="0=7 22=4 5=700" timeout 120 python tools/attn_trace.py 32 2>&1 | head -48
