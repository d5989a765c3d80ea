for L in 700x32 400x32 1600x8; do for npp in 0 2 4; do timeout 20 python tools/attn_bench.py --opt 1=$npp --lens $L; done; done
