for ps in 32 256 1024; do for L in 700x32 400x32 1600x8 700x128; do timeout 30 python tools/attn_bench.py --opt 24=$ps --lens $L; done; done
