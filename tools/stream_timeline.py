"""CUPTI timeline of the bench step as S concurrent sub-batch pipelines (torch.profiler):
per stream busy time, time with both / one / no pipeline running a kernel, and the kernels
that run alone.   python tools/stream_timeline.py [streams]"""
import os
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import cfd_inputs as ci  # noqa: E402
from paper_2505_23317_b200.api import CFDetrEncoder, bf16_tensor  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 2
cfg = ci.CONFIGS["c640"]
B = 32
k = 25 * cfg.n_coarse // 100
w = ci.make_weights(cfg, seed=0)
imgs_all = bf16_tensor(ci.make_frames(cfg, B), "cuda")
bounds = [round(B * i / S) for i in range(S + 1)]
pipes = []
for i in range(S):
    f0, f1 = bounds[i], bounds[i + 1]
    enc = CFDetrEncoder(cfg, w, max_tasks=max(f1 - f0, 8))
    im = imgs_all[f0:f1]
    ks = [k] * (f1 - f0)
    cnt = [cfg.n_coarse + 3 * k] * (f1 - f0)
    s = torch.cuda.Stream()
    co, sel, ro = {}, {}, {}
    with torch.cuda.stream(s):
        co.update(enc.coarse_encode(im, stream=s))
        sel.update(enc.select_regions(co["scores"], k=ks, stream=s))
        ro.update(enc.batch_refine(im, co["x0"], sel["sel_idx"], sel["sel_count"], token_counts=cnt, stream=s))
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            enc.coarse_encode(im, out=co, stream=s)
            enc.select_regions(co["scores"], k=ks, out=sel, stream=s)
            enc.batch_refine(im, co["x0"], sel["sel_idx"], sel["sel_count"], token_counts=cnt, out=ro, stream=s)
    s.synchronize()
    pipes.append((enc, s, g, (co, sel, ro, im)))


def step():
    main = torch.cuda.current_stream()
    fork = torch.cuda.Event()
    fork.record(main)
    for _, s, g, _ in pipes:
        s.wait_event(fork)
        with torch.cuda.stream(s):
            g.replay()
        ev = torch.cuda.Event()
        ev.record(s)
        main.wait_event(ev)


for _ in range(5):
    step()
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    for _ in range(4):
        step()
        torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA and "cfd::" in e.name]
evs.sort(key=lambda e: e.time_range.start)
# split into steps at gaps > 50 us; keep the last complete step
steps, cur = [], []
for e in evs:
    if cur and e.time_range.start - max(x.time_range.end for x in cur) > 50:
        steps.append(cur)
        cur = []
    cur.append(e)
steps.append(cur)
st = steps[-2] if len(steps) > 1 else steps[-1]
t0 = min(e.time_range.start for e in st)
t1 = max(e.time_range.end for e in st)
# sweep: number of kernels running at each instant
pts = sorted([(e.time_range.start, 1) for e in st] + [(e.time_range.end, -1) for e in st])
occ = defaultdict(float)
n, last = 0, t0
for t, dv in pts:
    occ[n] += t - last
    n += dv
    last = t
print(f"streams {S}: step span {t1 - t0:.1f} us, {len(st)} kernels; time with 0/1/2+ kernels running: "
      f"{occ[0]:.1f} / {occ[1]:.1f} / {sum(v for kk, v in occ.items() if kk >= 2):.1f} us")
alone = defaultdict(float)
for e in st:
    a, b = e.time_range.start, e.time_range.end
    others = [(x.time_range.start, x.time_range.end) for x in st if x is not e]
    # time of e not overlapped by any other kernel
    segs = [(a, b)]
    for oa, ob in others:
        nxt = []
        for sa, sb in segs:
            if ob <= sa or oa >= sb:
                nxt.append((sa, sb))
            else:
                if oa > sa:
                    nxt.append((sa, oa))
                if ob < sb:
                    nxt.append((ob, sb))
        segs = nxt
    alone[e.name[:60]] += sum(sb - sa for sa, sb in segs)
print("kernel time running alone (us per step):")
for nm, v in sorted(alone.items(), key=lambda x: -x[1])[:12]:
    print(f"  {nm:60s} {v:8.1f}")
