"""Run one c640 coarse+refine step with the debug library and print the attention (v4)
pipeline trace (cfdx_attn_trace) of the last attention launch (refine, N = 700): per
sub-tile, the median over CTAs of each event in cycles relative to the warpgroup's s_full
of sub-tile 0, plus per-phase durations.   python tools/attn_trace.py [frames]"""
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
co = enc.coarse_encode(imgs)
sel = enc.select_regions(co["scores"], k=[100] * B)
ro = enc.batch_refine(imgs, co["x0"], sel["sel_idx"], sel["sel_count"])
torch.cuda.synchronize()
NW = 148 * 4 * 2 * 12 * 8 + 148
buf = (C.c_uint64 * NW)()
assert L.load().cfdx_attn_trace(buf, NW) == 0
a = np.frombuffer(buf, dtype=np.uint64).astype(np.int64)
t0 = a[148 * 4 * 2 * 12 * 8:]
t = a[:148 * 4 * 2 * 12 * 8].reshape(148, 4, 2, 12, 8)
names = ["s_full", "S in regs", "max", "exps", "o_full(+resc)", "p_full arr", "MMA QK(u)", "MMA PV(u)"]
# v5: event 5 = second named barrier passed (P stored); QK/PV are issued by the traced thread itself
ctl = os.environ.get("CFD_TRACE_CTL")  # v7: slot 3 = warpgroup 0's control thread
for it in range(2):
    for w in range(4):
        if ctl and w == 3:
            ok = t[:, 3, it, 0, 0] > 0
            ref = t[ok, 0, it, 0, 0][:, None]
            cn = ["top", "pumped", "kv_full", "s_free", "QK issued", "p_full seen", "PV issued"]
            print(f"--- item {it}, control thread of warpgroup 0 (cycles since warpgroup 0's s_full of sub-tile 0)")
            print("  u  " + " ".join(f"{n:>12s}" for n in cn))
            for u in range(12):
                if (t[ok, 3, it, u, 0] == 0).all():
                    break
                print(f" {u:2d}  " + " ".join(f"{int(np.median(t[ok, 3, it, u, e] - ref[:, 0])):12d}" for e in range(7)))
            continue
        ok = (t[:, w, it, 0, 0] > 0) & (t[:, w, it, 0, 5] > 0)
        if not ok.any():
            continue
        ref = t[ok, w, it, 0, 0][:, None, None]
        rel = t[ok, w, it] - ref
        print(f"--- item {it}, warpgroup {w}: {ok.sum()} CTAs; start at {int(np.median(t[ok, w, it, 0, 0] - t0[ok]))} cycles "
              "after kernel start; medians (cycles since s_full of sub-tile 0)")
        print("  u  " + " ".join(f"{n:>13s}" for n in names))
        for u in range(12):
            if (t[ok, w, it, u, 5] == 0).all():
                break
            print(f" {u:2d}  " + " ".join(f"{int(np.median(rel[:, u, e])):13d}" for e in range(8)))
        d = np.diff(t[ok, w, it, :11, :6], axis=2)
        per = np.median(np.diff(t[ok, w, it, :11, 0], axis=1))
        print("  phase medians over u<11: " + ", ".join(f"{names[e]}->{names[e + 1]} {int(np.median(d[:, :, e]))}"
                                                         for e in range(5)) + f"; period {int(per)}")
