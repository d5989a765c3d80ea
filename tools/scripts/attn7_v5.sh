timeout 20 python tools/attn_check.py 7 4 700
timeout 20 python tools/attn_check.py 7 4 400,640,880,1120,1360,1600
for L in 700x32 400x32 1600x8; do timeout 20 python tools/attn_bench.py --opt 0=7 --opt 22=4 --lens $L; done
