"""Run one c640 coarse+refine step with the debug library and print the fused-MLP pipeline
trace (cfdx_mlp_trace) of the last MLP launch: per-event median over CTAs, in cycles
relative to each CTA's kernel start.   CFD_LIB_DEBUG=1 python tools/mlp_trace.py"""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["CFD_LIB_DEBUG"] = "1"
import torch  # noqa: E402

import cfd_inputs as ci  # noqa: E402
from paper_2505_23317_b200 import _lib as L  # noqa: E402
from paper_2505_23317_b200.api import CFDetrEncoder, bf16_tensor  # noqa: E402

OPTS = [tuple(int(t) for t in kv.split("=")) for kv in os.environ.get("CFD_OPTS", "").split()]
cfg = ci.CONFIGS["c640"]
B = int(sys.argv[1]) if len(sys.argv) > 1 else 32
enc = CFDetrEncoder(cfg, ci.make_weights(cfg, seed=0), max_tasks=B)
for k_, v_ in OPTS:
    enc.set_option(k_, v_)
imgs = bf16_tensor(ci.make_frames(cfg, B), "cuda")
ks = [100] * B
co = enc.coarse_encode(imgs)
sel = enc.select_regions(co["scores"], k=ks)
ro = enc.batch_refine(imgs, co["x0"], sel["sel_idx"], sel["sel_count"])
torch.cuda.synchronize()
buf = (C.c_uint64 * (148 * 96))()
assert L.load().cfdx_mlp_trace(buf, 148 * 96) == 0
t = np.frombuffer(buf, dtype=np.uint64).reshape(148, 2, 48).astype(np.int64)
t0 = t[:, 0, 47:48]
names = {0: "prod: first h piece", 1: "epi: h landed", 2: "epi: h in TMEM", 3: "mma: ht_full seen"}
for j in range(8):
    names[4 + j] = f"mma: MMA1({j}) issue"
    names[12 + j] = f"mma: MMA2({j}) issue"
    names[20 + j] = f"epi: a1_full({j})"
    names[28 + j] = f"epi: GELU({j}) done"
names[36] = "epi: final epi start"
names[37] = "epi: tile done"
names[38] = "epi: OPJ resid start"
names[39] = "epi: OPJ resid done"
names[40] = "mma: MMA_o start"
names[41] = "mma: MMA_o committed"
names[42] = "mma: MMA_o kb1 start"
for it in range(2):
    valid = t[:, it, 37] > 0 if it else np.ones(148, bool)
    if it and not valid.any():
        break
    print(f"--- tile {it} ({valid.sum()} CTAs), cycles since kernel start (median / max)")
    rel = t[valid, it, :] - t0[valid]
    order = sorted(names, key=lambda e: np.median(rel[:, e]))
    for e in order:
        print(f"  {names[e]:24s} {int(np.median(rel[:, e])):8d} {int(rel[:, e].max()):8d}")
