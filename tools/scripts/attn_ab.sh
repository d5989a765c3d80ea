# attention A/B: kernel times at the bench shapes, then the attention tests
for L in 700x8 700x32 400x32 1600x8 700x128 400x128; do timeout 30 python tools/attn_bench.py --lens $L; done
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -k "attn or attention" 2>&1 | tail -3
