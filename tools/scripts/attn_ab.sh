set -x
for L in 16 28 65 128 257 400 700 400,640,880,1120,1360,1600 16,700,3,1600 129,255,257,3; do timeout 60 python tools/attn_check.py 7 4 $L; done
CFD_SPIKE=1 timeout 60 python tools/attn_check.py 7 4 400,640,880,1120,1360,1600
for L in 700x32 400x32 1600x8 400x16,640x16; do for v in 4 7; do timeout 60 python tools/attn_bench.py --opt 0=$v --lens $L; done; done
