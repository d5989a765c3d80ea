for sl in 32 0 1 2 8; do for L in 700x8 700x32 400x32 700x128; do timeout 30 python tools/attn_bench.py --opt 21=$sl --lens $L; done; done
