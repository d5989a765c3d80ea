"""A3 multi-level batching: varlen (block-diagonal, no padding; this build) against the
paper's pad-to-max batch (P:466 draft) on the batch6 workload (6 tasks, k = 0..400,
N = 400..1600).  Padding every task to the longest (1600 tokens) costs what refining every
task fully costs, so the padded figure is timed as the same refine launch with k = 400 for
all six tasks (identical kernels, 9600 instead of 6000 tokens).  CUDA graphs, CUDA events.
python tools/padded_vs_varlen.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import cfd_inputs as ci  # noqa: E402
from paper_2505_23317_b200.api import CFDetrEncoder, bf16_tensor  # noqa: E402

cfg = ci.CONFIGS["batch6"]
ks_var = list(ci.WORKLOADS["batch6"].ks)
ks_pad = [cfg.n_coarse] * len(ks_var)
enc = CFDetrEncoder(cfg, ci.make_weights(cfg, seed=0), max_tasks=8)
imgs = bf16_tensor(ci.make_frames(cfg, len(ks_var)), "cuda")
s = torch.cuda.Stream()
res = {}
for name, ks in (("varlen", ks_var), ("padded-to-max", ks_pad)):
    counts = [cfg.n_coarse + 3 * k for k in ks]
    with torch.cuda.stream(s):
        co = enc.coarse_encode(imgs, stream=s)
        sel = enc.select_regions(co["scores"], k=ks, stream=s)
        ro = enc.batch_refine(imgs, co["x0"], sel["sel_idx"], sel["sel_count"], token_counts=counts, stream=s)
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            enc.batch_refine(imgs, co["x0"], sel["sel_idx"], sel["sel_count"], token_counts=counts, out=ro, stream=s)
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
    res[name] = (e0.elapsed_time(e1) / 50, sum(counts))
    print(f"{name:14s}: refine batch of 6 tasks, {sum(counts):5d} tokens: {res[name][0] * 1e3:8.1f} us")
print(f"varlen saves {100 * (1 - res['varlen'][0] / res['padded-to-max'][0]):.1f} % of the padded refine time "
      f"({res['padded-to-max'][1] / res['varlen'][1]:.2f}x the tokens)")
