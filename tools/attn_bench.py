"""Time the attention kernel alone at bench shapes (for ncu captures and variant sweeps): reps
back-to-back launches replayed from one CUDA graph, CUDA events around the replay.
python tools/attn_bench.py --opt 0=1 --opt 1=4 --lens 700x32 --reps 20   (--opt K=V: cfdx_set_option)"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_2505_23317_b200 import _lib as L  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--opt", action="append", default=[])
ap.add_argument("--lens", default="700x32")
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
lib = L.load()
for kv in a.opt:
    k_, v_ = (int(t) for t in kv.split("="))
    assert lib.cfdx_set_option(None, k_, v_) == 0, kv
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
work = torch.zeros(2, dtype=torch.int32, device="cuda")
run = lambda: lib.cfdx_attention(len(lens), cu.data_ptr(), max(lens), cap, d, nh, qkv.data_ptr(), out.data_ptr(),
                                 None, 0, work.data_ptr(), torch.cuda.current_stream().cuda_stream)
for _ in range(3):
    run()
torch.cuda.synchronize()
# replay the launches from a CUDA graph: eager ctypes launches are host-bound below ~25 us
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    for _ in range(a.reps):
        run()
g.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
g.replay()
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) / a.reps * 1e3
fl = sum(4 * n * n * d for n in lens)
print(f"opts {' '.join(a.opt) or 'default'} lens {a.lens}: {us:.1f} us  {fl / us / 1e6:.1f} TFLOP/s")
