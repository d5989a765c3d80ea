"""NEXT f4: measured batch WCET tables in SPEC.md's BatchWcetTables form for the
out-of-scope DBA scheduler, from this build's kernels on one B200.

  coarse[n]    = C_{B^S}(n): coarse_encode + select_regions of n c640 frames (one image-level
                 batch, A3 level 1)
  fine[w][n]   = C_batch(w, n): batch_refine of n tasks all at workload level w (patch-level
                 batch, A3 level 2)

Workload levels (reading R25): the paper's S < 3000 <= M <= 4800 < L fine
patches are counts for its own backbone resolution; on the c640 geometry
(400 regions, m = 2) the levels are refine ratios, each measured at its upper bound:
S = 25 % (k = 100), M = 60 % (k = 240), L = 100 % (k = 400) -- the multi48 ratio mix grouped.

Each entry: R runs, each one CUDA-graph replay timed alone with CUDA events, L2 flushed
before it (outside the events), enqueued behind a spin kernel (no host-side gaps).

Published WCET ("wcet_ms", the Duration of the table): the 99th percentile of the runs, raised
to the running maximum over smaller levels and batch sizes (a monotone envelope: a WCET bound
may always be raised, and S:55 requires fine(., n) non-decreasing in level and n).  The
observed maximum ("max_ms", measurement-based as the paper's 1000-run WCETs)
is reported beside it: it carries isolated ~2 ms device stalls (about 1 run in 1000, present
with the host decoupled), which is why it is not the published bound.  The S:52-55 invariants
are asserted on wcet_ms exactly (tests/test_batch_wcet_tables.py).
python tools/batch_wcet_tables.py [runs] [n_max] > table.json"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import cfd_inputs as ci  # noqa: E402
from paper_2505_23317_b200.api import CFDetrEncoder, bf16_tensor  # noqa: E402

R = int(sys.argv[1]) if len(sys.argv) > 1 else 300
NMAX = int(sys.argv[2]) if len(sys.argv) > 2 else 8
LEVELS = {"S": 100, "M": 240, "L": 400}

cfg = ci.CONFIGS["c640"]
enc = CFDetrEncoder(cfg, ci.make_weights(cfg, seed=0), max_tasks=NMAX)
imgs = bf16_tensor(ci.make_frames(cfg, NMAX), "cuda")
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
s = torch.cuda.Stream()


def timed(fn_capture):
    """Capture fn_capture() in a graph; R replays, each timed alone after an L2 flush."""
    with torch.cuda.stream(s):
        fn_capture()
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            fn_capture()
    s.synchronize()
    for _ in range(5):
        with torch.cuda.stream(s):
            g.replay()
    s.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(R)]
    # the GPU is held by a spin kernel while the host enqueues each chunk of 50 runs, so a
    # host-side stall can never open a gap between a start event and its replay
    with torch.cuda.stream(s):
        for c0 in range(0, R, 50):
            torch.cuda._sleep(20_000_000)
            for a, b in ev[c0:c0 + 50]:
                flush.zero_()
                a.record(s)
                g.replay()
                b.record(s)
    s.synchronize()
    t = sorted(a.elapsed_time(b) for a, b in ev)
    return {"mean_ms": round(sum(t) / len(t), 4), "max_ms": round(t[-1], 4),
            "p99_ms": round(t[min(len(t) - 1, int(0.99 * len(t)))], 4), "runs": R}


coarse = {}
co_out, sel_out = {}, {}
for n in range(1, NMAX + 1):
    im = imgs[:n]
    o_c, o_s = {}, {}

    def run(im=im, o_c=o_c, o_s=o_s, n=n):
        o_c.update(enc.coarse_encode(im, out=o_c if o_c else None, stream=s))
        o_s.update(enc.select_regions(o_c["scores"], k=[LEVELS["L"]] * n, out=o_s if o_s else None, stream=s))
    coarse[n] = timed(run)
    co_out[n], sel_out[n] = o_c, o_s

fine = {}
for w, k in LEVELS.items():
    fine[w] = {}
    for n in range(1, NMAX + 1):
        im = imgs[:n]
        o_c = co_out[n]
        sel = enc.select_regions(o_c["scores"], k=[k] * n)
        torch.cuda.synchronize()
        counts = [cfg.n_coarse + 3 * k] * n
        o_r = {}

        def run(im=im, o_c=o_c, sel=sel, counts=counts, o_r=o_r):
            o_r.update(enc.batch_refine(im, o_c["x0"], sel["sel_idx"], sel["sel_count"], token_counts=counts,
                                        out=o_r if o_r else None, stream=s))
        fine[w][n] = timed(run)

def envelope(coarse, fine, levels, n_max):
    """wcet_ms: p99 raised to the running maximum over smaller sizes (coarse) and smaller levels
    and sizes (fine) -- the monotone envelope of the measured 99th percentiles."""
    run = 0.0
    for n in range(1, n_max + 1):
        run = max(run, coarse[n]["p99_ms"])
        coarse[n]["wcet_ms"] = round(run, 4)
    for i, w in enumerate(levels):
        for n in range(1, n_max + 1):
            v = fine[w][n]["p99_ms"]
            if n > 1:
                v = max(v, fine[w][n - 1]["wcet_ms"])
            if i > 0:
                v = max(v, fine[levels[i - 1]][n]["wcet_ms"])
            fine[w][n]["wcet_ms"] = round(v, 4)


def invariants(coarse, fine, levels, n_max):
    """SPEC.md S:52-55 on the published wcet_ms (batching property; fine monotone in level and n)."""
    c1 = coarse[1]["wcet_ms"]
    checks = [("coarse(n) <= n coarse(1)", all(coarse[n]["wcet_ms"] <= n * c1 for n in coarse))]
    for w in levels:
        f1 = fine[w][1]["wcet_ms"]
        checks.append((f"fine({w},n) <= n fine({w},1)", all(fine[w][n]["wcet_ms"] <= n * f1 for n in fine[w])))
    checks.append(("fine monotone in level", all(fine[levels[i]][n]["wcet_ms"] <= fine[levels[i + 1]][n]["wcet_ms"]
                                               for i in range(len(levels) - 1) for n in range(1, n_max + 1))))
    checks.append(("fine monotone in n", all(fine[w][n]["wcet_ms"] <= fine[w][n + 1]["wcet_ms"]
                                           for w in levels for n in range(1, n_max))))
    return checks


lv = list(LEVELS)
envelope(coarse, fine, lv, NMAX)
checks = invariants(coarse, fine, lv, NMAX)
out = {"form": "BatchWcetTables (SPEC.md S:50-56)", "device": torch.cuda.get_device_name(),
       "workload": "c640 (640x640, Pc 32, Pf 16, d256/h8/L6)",
       "levels": {w: {"k": k, "refine_pct": 100 * k // cfg.n_coarse, "tokens_per_task": cfg.n_coarse + 3 * k}
                  for w, k in LEVELS.items()},
       "coarse": coarse, "fine": fine, "invariants": {name: ok for name, ok in checks}}
print(json.dumps(out, indent=1))
