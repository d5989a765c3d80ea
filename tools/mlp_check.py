"""Fused-MLP vs two-GEMM path: determinism and oracle error per variant."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import cfd_inputs as ci, oracle as O
from paper_2505_23317_b200 import _lib as L
from paper_2505_23317_b200.api import CFDetrEncoder, bf16_tensor
lib = L.load()
cfg = ci.CONFIGS["c640"]
w = ci.make_weights(cfg, seed=0)
enc = CFDetrEncoder(cfg, w, max_tasks=64)
imgs_np = ci.make_frames(cfg, 3, task0=7)
imgs = bf16_tensor(imgs_np, "cuda")
oc = O.coarse_encode(cfg, w, [imgs_np[1]])[0]
res = []
for fused in (1, 0, 1, 0):
    enc.set_option(2, fused)
    co = enc.coarse_encode(imgs, want_layers=True)
    torch.cuda.synchronize()
    y = co["layer_out"][:, 1].double().cpu().numpy()
    errs = [float(np.linalg.norm(y[l] - oc["layers"][l]) / np.linalg.norm(oc["layers"][l])) for l in range(6)]
    res.append(co["y"].clone())
    print("fused", fused, "per-layer rel vs oracle (frame 1):", ["%.2e" % e for e in errs])
print("fused run-to-run equal:", torch.equal(res[0], res[2]), " unfused run-to-run equal:", torch.equal(res[1], res[3]))
print("fused vs unfused rel:", ((res[0] - res[1]).norm() / res[1].norm()).item())
