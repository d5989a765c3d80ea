"""The encoder step (coarse -> select -> refine, one 32-frame CUDA graph) on bf16 frames vs
on 8-bit frames converted on the device by cfd_frames_from_u8: selection counts, finite
outputs and step time (the work is fixed by k, so the times must match).
python tools/ingest_timing.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import cfd_inputs as ci
from paper_2505_23317_b200.api import CFDetrEncoder, bf16_tensor
cfg = ci.CONFIGS["c640"]; B = 32; k = 100
enc = CFDetrEncoder(cfg, ci.make_weights(cfg, seed=0), max_tasks=B)
ks = [k]*B; counts = [cfg.n_coarse + 3*k]*B
sc, sh = ci.u8_affine()
u8 = torch.from_numpy(ci.make_frames_u8(cfg, B)).cuda()
fb = bf16_tensor(ci.make_frames(cfg, B), "cuda")
fu = enc.frames_from_u8(u8, sc, sh)
s = torch.cuda.Stream()
for name, im in (("bf16", fb), ("u8conv", fu)):
    with torch.cuda.stream(s):
        co = enc.coarse_encode(im, stream=s)
        sel = enc.select_regions(co["scores"], k=ks, stream=s)
        ro = enc.batch_refine(im, co["x0"], sel["sel_idx"], sel["sel_count"], token_counts=counts, stream=s)
    s.synchronize()
    print(name, "sel_count", sel["sel_count"][:4].tolist(), "cu", ro["cu_seqlens"][-1].item(), "finite", torch.isfinite(ro["y"][:int(ro["cu_seqlens"][-1])]).all().item(),
          "scores", co["scores"][0,:5].tolist(), "img", im.float().abs().mean().item())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            enc.coarse_encode(im, out=co, stream=s)
            enc.select_regions(co["scores"], k=ks, out=sel, stream=s)
            enc.batch_refine(im, co["x0"], sel["sel_idx"], sel["sel_count"], token_counts=counts, out=ro, stream=s)
    for _ in range(3): g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); 
    for _ in range(20): g.replay()
    e1.record(); torch.cuda.synchronize()
    print(name, "ms/step", e0.elapsed_time(e1)/20)
