for npp in 2 4 6 8; do timeout 20 python tools/attn_bench.py --opt 1=$npp --lens 700x32; done
for sl in 0 128; do timeout 20 python tools/attn_bench.py --opt 21=$sl --lens 700x32; done
for st in 400 1000; do timeout 20 python tools/attn_bench.py --opt 5=$st --lens 700x32; done
timeout 20 python tools/attn_bench.py --opt 16=0 --lens 700x32
