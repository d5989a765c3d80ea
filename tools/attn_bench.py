"""Time the attention kernel alone at bench shapes (for ncu captures and variant sweeps).
python tools/attn_bench.py --variant 2 --npp 0 --lens 700x32 --reps 20"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_2505_23317_b200 import _lib as L  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--variant", type=int, default=2)
ap.add_argument("--npp", type=int, default=0)
ap.add_argument("--lens", default="700x32")
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--stagger", type=int, default=0)
ap.add_argument("--stages", type=int, default=4)
ap.add_argument("--token", type=int, default=0)
ap.add_argument("--split", type=int, default=0)
a = ap.parse_args()
lib = L.load()
assert lib.cfdx_set_option(0, a.variant) == 0 and lib.cfdx_set_option(1, a.npp) == 0
assert lib.cfdx_set_option(5, a.stagger) == 0
assert lib.cfdx_set_option(6, a.stages) == 0
assert lib.cfdx_set_option(9, a.token) == 0
assert lib.cfdx_set_option(10, a.split) == 0
lens = []
for part in a.lens.split(","):
    n, c = part.split("x")
    lens += [int(n)] * int(c)
d, nh = 256, 8
cu_l = [0]
for n in lens:
    cu_l.append(cu_l[-1] + n)
cap = cu_l[-1] + 256
qkv = torch.randn(cap, 3 * d, device="cuda").to(torch.bfloat16)
cu = torch.tensor(cu_l, dtype=torch.int32, device="cuda")
out = torch.zeros(cap, d, device="cuda", dtype=torch.bfloat16)
s = torch.cuda.current_stream().cuda_stream
run = lambda: lib.cfdx_attention(len(lens), cu.data_ptr(), max(lens), cap, d, nh, qkv.data_ptr(), out.data_ptr(),
                                 None, 0, s)
for _ in range(3):
    run()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.reps):
    run()
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) / a.reps * 1e3
fl = sum(4 * n * n * d for n in lens)
print(f"variant {a.variant} npp {a.npp} stages {a.stages} token {a.token} split {a.split} lens {a.lens}: {us:.1f} us  {fl / us / 1e6:.1f} TFLOP/s")
