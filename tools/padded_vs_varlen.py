"""A3 multi-level batching: varlen (block-diagonal, no padding; cfd_batch_refine) against the
paper's pad-to-max batch (P:466 draft; cfd_batch_refine_padded: every task padded to the
longest task's token count, pad keys masked) on the batch6 workload (6 tasks, k = 0..400,
N = 400..1600).  The two produce the same per-task rows bit for bit (tests/test_gpu_parity.py);
this times them: CUDA graphs of the refine call alone, CUDA events, L2 not flushed (both fit).
python tools/padded_vs_varlen.py [--multi48]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import cfd_inputs as ci  # noqa: E402
from paper_2505_23317_b200.api import CFDetrEncoder, bf16_tensor  # noqa: E402

cfg = ci.CONFIGS["batch6"]
if "--multi48" in sys.argv:
    ks = [k for g in range(8) for k in ci.multi48_group_ks(g)]
    name = "multi48 (48 streams)"
else:
    ks = list(ci.WORKLOADS["batch6"].ks)
    name = "batch6"
T = len(ks)
counts = [cfg.n_coarse + 3 * k for k in ks]
pad = max(counts)
enc = CFDetrEncoder(cfg, ci.make_weights(cfg, seed=0), max_tasks=max(8, T))
imgs = bf16_tensor(ci.make_frames(cfg, T), "cuda")
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    co = enc.coarse_encode(imgs, stream=s)
    sel = enc.select_regions(co["scores"], k=ks, stream=s)
    ro = enc.batch_refine(imgs, co["x0"], sel["sel_idx"], sel["sel_count"], token_counts=counts, stream=s)
    po = enc.batch_refine_padded(imgs, co["x0"], sel["sel_idx"], sel["sel_count"], pad, stream=s)
s.synchronize()
cu = ro["cu_seqlens"].cpu().tolist()
same = all(torch.equal(po["y"][t * pad:t * pad + counts[t]], ro["y"][cu[t]:cu[t + 1]]) for t in range(T))
res = {}
for mode in ("varlen", "padded-to-max"):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            if mode == "varlen":
                enc.batch_refine(imgs, co["x0"], sel["sel_idx"], sel["sel_count"], token_counts=counts, out=ro, stream=s)
            else:
                enc.batch_refine_padded(imgs, co["x0"], sel["sel_idx"], sel["sel_count"], pad, out=po, stream=s)
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
    toks = sum(counts) if mode == "varlen" else T * pad
    res[mode] = (e0.elapsed_time(e1) / 50, toks)
    print(f"{name} {mode:14s}: refine batch of {T} tasks, {toks:6d} token rows: {res[mode][0] * 1e3:8.1f} us")
print(f"padded rows equal the varlen rows bit for bit: {same}")
print(f"varlen saves {100 * (1 - res['varlen'][0] / res['padded-to-max'][0]):.1f} % of the padded refine time "
      f"({res['padded-to-max'][1] / res['varlen'][1]:.2f}x the token rows)")
