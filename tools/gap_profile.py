"""Kernel timeline of the bench step (CUDA-graph replays) from torch.profiler (CUPTI):
per-kernel device durations and the idle gaps between consecutive kernels of a step.
python tools/gap_profile.py [--option K=V ...]"""
import argparse
import os
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import cfd_inputs as ci  # noqa: E402
from paper_2505_23317_b200 import _lib as L  # noqa: E402
from paper_2505_23317_b200.api import CFDetrEncoder, bf16_tensor  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--option", action="append", default=[])
ap.add_argument("--frames", type=int, default=32)
a = ap.parse_args()
OPTS = [tuple(int(t) for t in kv.split("=")) for kv in a.option]
cfg = ci.CONFIGS["c640"]
B = a.frames
ks = [25 * cfg.n_coarse // 100] * B
counts = [cfg.n_coarse + (cfg.m ** 2 - 1) * ks[0]] * B
enc = CFDetrEncoder(cfg, ci.make_weights(cfg, seed=0), max_tasks=B)
for k_, v_ in OPTS:
    enc.set_option(k_, v_)
imgs = bf16_tensor(ci.make_frames(cfg, B), "cuda")
s = torch.cuda.Stream()
co, sel, ro = {}, {}, {}
with torch.cuda.stream(s):
    co.update(enc.coarse_encode(imgs, stream=s))
    sel.update(enc.select_regions(co["scores"], k=ks, stream=s))
    ro.update(enc.batch_refine(imgs, co["x0"], sel["sel_idx"], sel["sel_count"], token_counts=counts, stream=s))
s.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    with torch.cuda.graph(g, stream=s):
        enc.coarse_encode(imgs, out=co, stream=s)
        enc.select_regions(co["scores"], k=ks, out=sel, stream=s)
        enc.batch_refine(imgs, co["x0"], sel["sel_idx"], sel["sel_count"], token_counts=counts, out=ro, stream=s)
s.synchronize()
for _ in range(5):
    g.replay()
torch.cuda.synchronize()
REPS = 5
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    for _ in range(REPS):
        g.replay()
        torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda e: e.time_range.start)
# split into steps at gaps > 50 us
steps, cur = [], []
for e in evs:
    if cur and e.time_range.start - cur[-1].time_range.end > 50:
        steps.append(cur)
        cur = []
    cur.append(e)
steps.append(cur)
dur = defaultdict(float)
gap_after = defaultdict(float)
cnt = defaultdict(int)
spans, busy = [], []
for st in steps[1:]:  # first replay after profiler start may include setup
    spans.append(st[-1].time_range.end - st[0].time_range.start)
    busy.append(sum(e.time_range.end - e.time_range.start for e in st))
    for i, e in enumerate(st):
        nm = e.name[:60]
        dur[nm] += e.time_range.end - e.time_range.start
        cnt[nm] += 1
        if i + 1 < len(st):
            gap_after[nm] += st[i + 1].time_range.start - e.time_range.end
n = len(steps) - 1
print(f"steps {n}: span {sum(spans)/n:.1f} us, kernels busy {sum(busy)/n:.1f} us, idle {sum(spans)/n - sum(busy)/n:.1f} us, "
      f"{len(steps[-1])} kernels/step")
print(f"{'kernel':60s} {'n/step':>6s} {'us/step':>9s} {'us/launch':>9s} {'gap after (us/launch)':>22s}")
for nm in sorted(dur, key=lambda x: -dur[x]):
    print(f"{nm:60s} {cnt[nm]/n:6.1f} {dur[nm]/n:9.1f} {dur[nm]/cnt[nm]:9.2f} {gap_after[nm]/cnt[nm]:22.2f}")
