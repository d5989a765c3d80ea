"""One eager c640 step (coarse_encode -> select_regions(top-k) -> batch_refine) of B frames,
repeated R times -- a short command for ncu captures of the step's kernels.
python tools/step_once.py [B=16] [R=2] [K=V option ...]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import cfd_inputs as ci  # noqa: E402
from paper_2505_23317_b200.api import CFDetrEncoder, bf16_tensor  # noqa: E402

args = [a for a in sys.argv[1:] if "=" not in a]
B = int(args[0]) if args else 16
R = int(args[1]) if len(args) > 1 else 2
cfg = ci.CONFIGS["c640"]
enc = CFDetrEncoder(cfg, ci.make_weights(cfg, seed=0), max_tasks=max(B, 8))
for kv in (a for a in sys.argv[1:] if "=" in a):
    enc.set_option(*(int(t) for t in kv.split("=")))
imgs = bf16_tensor(ci.make_frames(cfg, B), "cuda")
ks = [100] * B
for _ in range(R):
    co = enc.coarse_encode(imgs)
    sel = enc.select_regions(co["scores"], k=ks)
    ro = enc.batch_refine(imgs, co["x0"], sel["sel_idx"], sel["sel_count"], token_counts=[400 + 3 * k for k in ks])
torch.cuda.synchronize()
enc.check()
print("ok", B, R)
