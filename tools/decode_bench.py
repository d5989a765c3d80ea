"""NEXT f3 measurement: the decoder block (cfd_decode: LN + projections, cross-attention of
128 learned queries over each task's packed encoder tokens, O-projection, detection heads)
on the bench's refine batch (32 c640 tasks, 700 tokens each), CUDA graph + CUDA events, with
the fp64 oracle timed on a bounded sample beside it.  python tools/decode_bench.py"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import cfd_inputs as ci  # noqa: E402
import oracle as O  # noqa: E402
from paper_2505_23317_b200.api import CFDetrEncoder, bf16_tensor  # noqa: E402

cfg = ci.CONFIGS["c640"]
T, Q = 32, 128
k = 100
enc = CFDetrEncoder(cfg, ci.make_weights(cfg, seed=0), max_tasks=T)
wd = ci.make_decoder_weights(cfg, Q, seed=4)
enc.set_decoder(wd)
imgs = bf16_tensor(ci.make_frames(cfg, T), "cuda")
co = enc.coarse_encode(imgs)
sel = enc.select_regions(co["scores"], k=[k] * T)
ro = enc.batch_refine(imgs, co["x0"], sel["sel_idx"], sel["sel_count"])
torch.cuda.synchronize()
cu = ro["cu_seqlens"]
n = int(cu[-1])
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    out = enc.decode(ro["y"], cu, T, n, stream=s)
s.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    with torch.cuda.graph(g, stream=s):
        out2 = enc.decode(ro["y"], cu, T, n, stream=s)
s.synchronize()
for _ in range(5):
    g.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with torch.cuda.stream(s):
    e0.record(s)
    for _ in range(50):
        g.replay()
    e1.record(s)
torch.cuda.synchronize()
us = e0.elapsed_time(e1) / 50 * 1e3
d = cfg.d_model
N = n // T
flops = T * (2 * N * d * 2 * d + 4 * Q * N * d + 2 * Q * d * d + 2 * Q * d * 5) + 2 * Q * d * d
print(f"decode: {T} tasks x {N} tokens, {Q} queries: {us:.1f} us per call ({T / us * 1e6:.0f} frames/s), "
      f"{flops / us / 1e6:.1f} TFLOP/s algorithmic")
# oracle on a bounded sample (shared input: the GPU's encoder output)
y0 = ro["y"][:int(cu[1])].double().cpu().numpy()
t0 = time.perf_counter()
reps = 0
while time.perf_counter() - t0 < 5.0:
    O.decode(wd, y0, cfg.n_heads, cfg.ln_eps)
    reps += 1
ms = (time.perf_counter() - t0) / reps * 1e3
print(f"oracle (fp64 numpy, {os.cpu_count()} host cores): {ms:.1f} ms per task ({1e3 / ms:.1f} frames/s)")
z, box, conf = O.decode(wd, y0, cfg.n_heads, cfg.ln_eps)
print(f"task 0 parity: z rel-L2 {np.linalg.norm(out2['z'][0].double().cpu().numpy() - z) / np.linalg.norm(z):.2e}, "
      f"box max-abs {np.abs(out2['boxes'][0].double().cpu().numpy() - box).max():.2e}, "
      f"conf max-abs {np.abs(out2['conf'][0].double().cpu().numpy() - conf).max():.2e}")
