for T in 4 8 12 16 20 24 28 32 36 40 48 56 64 96 128; do timeout 30 python tools/attn_bench.py --lens 700x$T; done
for T in 8 16 32 64; do timeout 30 python tools/attn_bench.py --lens 640x$T; done
