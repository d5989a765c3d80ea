"""Is the step faster as S concurrent sub-batches on S streams (each sub-batch its own
encoder / workspace / CUDA graph) than as one 32-frame batch?  Concurrent graphs fill each
other's kernel tails (persistent kernels leave SMs idle in their last wave).
python tools/dual_stream.py [frames] [splits...]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import cfd_inputs as ci  # noqa: E402
from paper_2505_23317_b200.api import CFDetrEncoder, bf16_tensor  # noqa: E402

cfg = ci.CONFIGS["c640"]
B = int(sys.argv[1]) if len(sys.argv) > 1 else 32
splits = [int(x) for x in sys.argv[2:]] or [1, 2, 4]
w = ci.make_weights(cfg, seed=0)
k = 25 * cfg.n_coarse // 100
imgs_all = bf16_tensor(ci.make_frames(cfg, B), "cuda")
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")


def build(nsplit):
    per = B // nsplit
    parts = []
    for i in range(nsplit):
        enc = CFDetrEncoder(cfg, w, max_tasks=max(per, 8))
        imgs = imgs_all[i * per:(i + 1) * per].contiguous()
        ks = [k] * per
        counts = [cfg.n_coarse + 3 * k] * per
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
        parts.append((enc, s, g, ro, (co, sel, imgs)))  # keep every buffer the graph uses alive
    return parts


def run(parts, reps=int(os.environ.get("REPS", "20"))):
    main = torch.cuda.current_stream()
    times = []
    warm = 3 if reps > 1 else 0
    for rep in range(reps + warm):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(main)
        for _, s, g, _, _ in parts:
            s.wait_event(e0)
            with torch.cuda.stream(s):
                g.replay()
            if os.environ.get("SERIAL"):
                ev = torch.cuda.Event()
                ev.record(s)
                ev.synchronize()
        for _, s, _, _, _ in parts:
            ev = torch.cuda.Event()
            ev.record(s)
            main.wait_event(ev)
        e1.record(main)
        torch.cuda.synchronize()
        if rep >= warm:
            times.append(e0.elapsed_time(e1))
    return sum(times) / len(times)


ref = None
for n in splits:
    parts = build(n)
    ms = run(parts)
    y = torch.cat([p[3]["y"][:(B // n) * (cfg.n_coarse + 3 * k)] for p in parts])
    if ref is None:
        ref = y.clone()
    same = torch.equal(y, ref)
    print(f"{n} stream(s) x {B // n} frames: {ms:.4f} ms/step  {B / ms * 1e3:.0f} frames/s  outputs bit-identical to first: {same}")
    for e, _, _, _, _ in parts:
        e.close()
