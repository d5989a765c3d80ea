#!/usr/bin/env python
"""Benchmark of the CF-DETR coarse-to-fine encoder hot path on B200.

One step = one pass of the whole hot path over one batch of synthetic camera frames:
cfd_coarse_encode(frames) -> cfd_select_regions(top-k per frame) -> cfd_batch_refine(tasks),
captured in CUDA graphs and replayed.  A rank's tasks run as --streams S concurrent lanes
(contiguous sub-batches, each with its own encoder context, workspace, stream and graph):
one lane's kernels fill the SMs the other's leave idle in their last wave.  The lane outputs
are checked to equal the single-launch batch bit for bit before timing.

Workloads (BASELINE.json configs):
  c640     (default) 640x640 frames, Pc 32 / Pf 16, d256/h8/L6, k = 100 (25 %), --frames 128
           in flight per GPU as two 64-frame lanes (weak scaling: every rank its own frames);
           frames/s rises with the frames in flight (32: 24.7k, 64: 29.3k, 128: 33.7k, 256:
           35.5k on one B200, profiles/r2_frames_sweep.txt) -- per-launch tails shrink
           as launches carry more tiles; c640b1 is the one-frame latency line
  c640b1   the same model, one frame per step (latency)
  batch6   6 tasks, k = (0, 80, 160, 240, 320, 400): one varlen launch per op
  fine8    8 frames, every region refined (1600 fine tokens each): the dense-attention case
  multi48  48 camera streams in groups of 6 at ratios {0,0,25,40,60,100} % (permuted per
           group); --scaling strong (default): the 48 streams shard over the N GPUs by whole
           groups; weak: 48 streams per GPU.  --mix s348: i.i.d. S:348 ratio mix, sharded by
           LPT on the predicted per-task cost

Launch: `python bench.py --gpus N ...` re-executes itself under torch.distributed.run with
N ranks when WORLD_SIZE is unset (one process per GPU, NCCL); under torchrun --gpus must equal
WORLD_SIZE.  Timing: W warm-up replays, K timed steps between a barrier + synchronize, CUDA
events on the main stream (fork / join to the lane streams), L2 flushed between timed steps
(256 MiB memset outside the events), max over ranks.  Rank 0 prints ONE JSON line.
`--impl reference` times the fp64 CPU oracle on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import cfd_inputs as ci  # noqa: E402

METRIC = "encoder frames/s"
UNIT = "frames/s"
WORKLOADS = ("c640", "c640b1", "batch6", "fine8", "multi48")


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c640", choices=WORKLOADS)
    ap.add_argument("--scaling", default=None, choices=["weak", "strong"],
                    help="multi48 only: strong (48 streams over N GPUs, default) or weak (48 per GPU)")
    ap.add_argument("--mix", default="balanced", choices=["balanced", "s348"], help="multi48 ratio mix")
    ap.add_argument("--frames", type=int, default=128, help="c640: frames in flight per GPU per step")
    ap.add_argument("--ratio", type=int, default=25, help="c640: refine percentage per frame")
    ap.add_argument("--streams", type=int, default=None,
                    help="concurrent lanes per GPU (own encoder / stream / CUDA graph each); default 2 for "
                         "multi48 (its e2e overlaps the lanes' copies), 1 otherwise")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-check", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--option", action="append", default=[],
                    help="library tuning switch KEY=VAL (cfdx_set_option, include/cfdetr_debug.h) on every "
                         "encoder context; repeatable")
    return ap.parse_args(argv)


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def respawn_under_torchrun(args) -> int:
    """`bench.py --gpus N` without a torchrun environment: run N ranks (one per GPU) under
    torch.distributed.run on this node and return its exit code."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


# ============================================================================ workloads
class Work:
    """One rank's share of a workload: the global task ids it owns (frame seed = (task, 0)),
    the refine count k of each, and the config description for the JSON line."""

    def __init__(self, args, rank, world):
        self.name = args.workload
        self.cfg = cfg = ci.CONFIGS["c640"]
        Nc = cfg.n_coarse
        self.scaling = "weak"
        note = {}
        if self.name == "c640":
            k = args.ratio * Nc // 100
            B = args.frames
            self.all_ids = list(range(B * world))
            self.all_ks = [k] * (B * world)
            self.assign = [list(range(r * B, (r + 1) * B)) for r in range(world)]
            note = {"frames_per_step_per_gpu": B, "refine_ratio_pct": args.ratio, "k_per_frame": k,
                    "tokens_per_frame": Nc + 3 * k}
        elif self.name == "c640b1":
            self.all_ids = list(range(world))
            self.all_ks = [100] * world
            self.assign = [[r] for r in range(world)]
            note = {"frames_per_step_per_gpu": 1, "refine_ratio_pct": 25, "k_per_frame": 100, "latency": True}
        elif self.name == "batch6":
            ks = list(ci.WORKLOADS["batch6"].ks)
            self.all_ids = list(range(6 * world))
            self.all_ks = ks * world
            self.assign = [list(range(r * 6, (r + 1) * 6)) for r in range(world)]
            note = {"tasks_per_step_per_gpu": 6, "ks": ks, "tokens": [Nc + 3 * k for k in ks],
                    "refine": "one varlen launch per op over the 6 ragged tasks"}
        elif self.name == "fine8":
            self.all_ids = list(range(8 * world))
            self.all_ks = [Nc] * (8 * world)
            self.assign = [list(range(r * 8, (r + 1) * 8)) for r in range(world)]
            note = {"frames_per_step_per_gpu": 8, "k_per_frame": Nc, "tokens_per_frame": 4 * Nc,
                    "note": "every region refined: the refine pass is the full fine pass"}
        else:  # multi48
            from paper_2505_23317_b200 import shard
            self.scaling = args.scaling or "strong"
            n_streams = 48 if self.scaling == "strong" else 48 * world
            if self.scaling == "strong" and 48 % world:
                raise SystemExit(f"bench: multi48 strong scaling needs N | 48 (N = {world})")
            self.all_ids = list(range(n_streams))
            if args.mix == "balanced":
                self.all_ks = [k for g in range(n_streams // 6) for k in ci.multi48_group_ks(g)]
                per = n_streams // world
                self.assign = [list(range(r * per, (r + 1) * per)) for r in range(world)]
                imb = 1.0
            else:
                # S:348 stress mix: easy with p = 0.5, else S / M / L with (0.4, 0.35, 0.25) -> 25/40/60 %
                rng = np.random.default_rng(348)
                ks = []
                for _ in range(n_streams):
                    if rng.random() < 0.5:
                        ks.append(0)
                    else:
                        ks.append(ci.ks_for_ratios(Nc, (int(rng.choice([25, 40, 60], p=[0.4, 0.35, 0.25])),))[0])
                self.all_ks = ks
                costs = [shard.task_cost(Nc + 3 * k, cfg.d_model, cfg.n_layers) for k in ks]
                self.assign = shard.lpt_assign(costs, world)
                imb = shard.imbalance(costs, self.assign)
            note = {"streams_total": n_streams, "streams_per_gpu": n_streams // world, "mix": args.mix,
                    "ratios_pct": "{0,0,25,40,60,100} per group of 6, permuted per group" if args.mix == "balanced"
                    else "S:348 i.i.d. (p_hard 0.5; S/M/L 0.4/0.35/0.25 -> 25/40/60 %)",
                    "sharding": "contiguous whole groups" if args.mix == "balanced" else "LPT on L(24d^2N + 4dN^2)",
                    "imbalance_max_over_mean": round(imb, 4)}
        self.ids = self.assign[rank]
        self.ks = [self.all_ks[i] for i in self.ids]
        self.counts = [Nc + (cfg.m ** 2 - 1) * k for k in self.ks]
        self.frames_total = len(self.all_ids)  # frames per step over all ranks
        self.note = note

    def config(self, args, world, l2_note, streams):
        cfg = self.cfg
        return {"workload": self.name, "img": f"{cfg.img_h}x{cfg.img_w}", "patch_coarse": cfg.patch_coarse,
                "patch_fine": cfg.patch_fine, "encoder": f"d{cfg.d_model}/h{cfg.n_heads}/L{cfg.n_layers}",
                **self.note, "global_batch_frames": self.frames_total,
                "parallelism": f"task-sharded x{world} (no collective on the hot path)",
                "l2": l2_note, "streams_per_gpu": streams,
                **({"options": list(args.option)} if args.option else {})}


# ============================================================================ CPU oracle
def run_oracle_task(cfg, w, img, k):
    import oracle as O
    c = O.coarse_encode(cfg, w, [img])[0]
    sel = O.select_topk(c["scores"].astype(np.float32), k)
    O.refine_encode(cfg, w, img, c["x0"], sel)


def oracle_threads():
    try:
        from threadpoolctl import threadpool_info
        return int(max((i.get("num_threads", 1) for i in threadpool_info()), default=1))
    except Exception:
        return os.cpu_count() or 1


def time_oracle(work, seconds, max_tasks, threads=None):
    """The oracle as it stands on this host: whole tasks of the workload (cycling through the
    rank's tasks) until `seconds` or `max_tasks`; threads=1 limits numpy's BLAS pool."""
    import contextlib
    cfg = work.cfg
    w = ci.make_weights(cfg, seed=0)
    if threads is not None:
        from threadpoolctl import threadpool_limits
        limit = threadpool_limits(limits=threads)
    else:
        limit = contextlib.nullcontext()
    with limit:
        used = oracle_threads()
        n, t0 = 0, time.perf_counter()
        while True:
            i = n % len(work.ids)
            img = ci.make_frame(cfg.img_h, cfg.img_w, ci.frame_seed(work.ids[i], 0))
            run_oracle_task(cfg, w, img, work.ks[i])
            n += 1
            el = time.perf_counter() - t0
            if el >= seconds or n >= max_tasks:
                break
    ks = sorted(set(work.ks[j % len(work.ks)] for j in range(n)))
    return {"value": n / el, "unit": UNIT, "cores": used, "kind": "oracle",
            "sample": f"{n} {work.name} frames (coarse + top-k select (k in {ks}) + refine, fp64 numpy), "
                      f"{el:.1f} s on {used} thread(s); host has {len(os.sched_getaffinity(0))} usable cores"}


def reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    work = Work(args, 0, world)
    cfg = work.cfg
    w = ci.make_weights(cfg, seed=0)
    imgs = [ci.make_frame(cfg.img_h, cfg.img_w, ci.frame_seed(work.ids[i % len(work.ids)], 0)) for i in range(4)]
    ks = [work.ks[i % len(work.ks)] for i in range(4)]
    for i in range(args.warmup):
        run_oracle_task(cfg, w, imgs[i % 4], ks[i % 4])
    t0 = time.perf_counter()
    for i in range(args.steps):
        run_oracle_task(cfg, w, imgs[i % 4], ks[i % 4])
    el = time.perf_counter() - t0
    v = args.steps / el
    sample = (f"1 {work.name} frame per step (coarse + top-k select + refine, fp64 numpy oracle), cycling "
              f"through 4 of the workload's frames")
    out = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": el / args.steps * 1e3, "higher_is_better": True, "scaling": work.scaling,
           "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
           "config": work.config(args, world, "n/a (CPU)", 1),
           "cpu_baseline": {"value": v, "unit": UNIT, "cores": oracle_threads(), "kind": "oracle", "sample": sample},
           "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# ============================================================================ clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", os.environ.get("CFD_BENCH_CLOCK_MS", "100")], stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        rows = [r for r in self.rows if len(r) >= 8]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        sm = [num(r[0]) for r in rows if num(r[0])]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i].lower().startswith("active")})
        loaded = [s for s in sm if s >= 0.5 * max(sm)] if sm else []
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": num(rows[0][1]), "reasons": reasons, "samples": len(rows)}


# ============================================================================ algorithmic work
def algorithmic_flops(cfg, ks):
    """Per-step algorithmic FLOPs by kernel class for frames with refine counts ks
    (linear 24d^2 per token-layer, attention 4N^2d per sequence-layer)."""
    d, F, L, Nc = cfg.d_model, cfg.d_ff, cfg.n_layers, cfg.n_coarse
    m2 = cfg.m ** 2
    Nts = [Nc + (m2 - 1) * k for k in ks]
    B = len(ks)
    rows = B * Nc + sum(Nts)
    return {
        "attention": L * sum(4 * Nc * Nc * d + 4 * n * n * d for n in Nts),
        "score": B * 2 * Nc * Nc * d,
        "gemm_qkv": L * 2 * rows * d * 3 * d,
        "gemm_oproj": L * 2 * rows * d * d,
        "gemm_mlp1": L * 2 * rows * d * F,
        "gemm_mlp2": L * 2 * rows * F * d,
        "gemm_embed_c": 2 * B * Nc * cfg.k_coarse * d,
        "gemm_embed_f": 2 * sum(m2 * k for k in ks) * cfg.k_fine * d,
    }


def algorithmic_bytes(cfg, ks):
    """Per-step algorithmic HBM bytes of the memory-bound kernels.  gather:
    read + write the unselected x0 rows, read + write the selected fine pixels, mixed_src and
    frow / fidx."""
    d, Nc = cfg.d_model, cfg.n_coarse
    m2 = cfg.m ** 2
    B = len(ks)
    return {
        "select": sum(4 * Nc + 4 * Nc + 4 for _ in ks),
        "gather": sum((Nc - k) * d * 4 * 2 + m2 * k * cfg.k_fine * 2 * 2 + 4 * (Nc + (m2 - 1) * k) + m2 * k * 8
                      for k in ks),
        "im2col": B * cfg.img_h * cfg.img_w * 3 * 2 * 2,
        # standalone LN only for layer 0 of the refine pass; later LNs are fused into epilogues
        "layernorm": sum((Nc + (m2 - 1) * k) * d * (4 + 2) for k in ks),
    }


def n_exps(cfg, ks):
    Nc = cfg.n_coarse
    return cfg.n_layers * cfg.n_heads * sum(Nc * Nc + (Nc + (cfg.m ** 2 - 1) * k) ** 2 for k in ks)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        j = json.load(open(p))
        return {"hbm": j["hbm_gbs"], "tensor_burst": j["bf16_tflops"],
                "tensor_sustained": j.get("bf16_tflops_sustained", j["bf16_tflops"]), "src": "measured"}
    return {"hbm": 6650.0, "tensor_burst": 1590.0, "tensor_sustained": 1400.0, "src": "fallback"}


# ============================================================================ GPU arm
class Lane:
    """One encoder context + stream + CUDA graph over a contiguous slice of the rank's tasks."""

    def __init__(self, work, imgs, f0, f1, dev, options, streams_cls):
        from paper_2505_23317_b200.api import CFDetrEncoder
        self.f0, self.f1 = f0, f1
        self.ks = work.ks[f0:f1]
        self.counts = work.counts[f0:f1]
        self.enc = CFDetrEncoder(work.cfg, work.weights, max_tasks=max(f1 - f0, 8), device=str(dev))
        for k_, v_ in options:
            self.enc.set_option(k_, v_)
        self.stream = streams_cls(device=dev)
        self.imgs = imgs[f0:f1]
        self.co, self.sel, self.ro = {}, {}, {}

    def step(self, s, eager=False):
        e = self.enc
        if eager:
            self.co.update(e.coarse_encode(self.imgs, stream=s))
            self.sel.update(e.select_regions(self.co["scores"], k=self.ks, stream=s))
            self.ro.update(e.batch_refine(self.imgs, self.co["x0"], self.sel["sel_idx"], self.sel["sel_count"],
                                          token_counts=self.counts, stream=s))
            return
        e.coarse_encode(self.imgs, out=self.co, stream=s)
        e.select_regions(self.co["scores"], k=self.ks, out=self.sel, stream=s)
        e.batch_refine(self.imgs, self.co["x0"], self.sel["sel_idx"], self.sel["sel_count"],
                       token_counts=self.counts, out=self.ro, stream=s)

    def capture(self):
        import torch
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(self.stream):
            with torch.cuda.graph(g, stream=self.stream):
                self.step(self.stream)
        self.stream.synchronize()
        return g


def replay(lanes, graphs, main):
    """One step: every lane's graph on its own stream, forked from and joined to `main`."""
    import torch
    if len(lanes) == 1:
        with torch.cuda.stream(main):
            graphs[0].replay()
        return
    fork = torch.cuda.Event()
    fork.record(main)
    for ln, g in zip(lanes, graphs):
        ln.stream.wait_event(fork)
        with torch.cuda.stream(ln.stream):
            g.replay()
        done = torch.cuda.Event()
        done.record(ln.stream)
        main.wait_event(done)


def probe_kernels(L, lanes, main, reps, flush):
    """Per-kernel-class device time of the step as it runs: CUDA event pairs around every
    launch (cudaEventRecordExternal nodes on the launching lane stream) captured into
    instrumented copies of the lane graphs, replayed `reps` times exactly like the timed step
    (lanes concurrent, L2 flushed before each).  Returns {class: (ms per step, launches per
    step)}.  With several lanes a kernel's span includes time it waits for SMs the other lane
    holds, so the class times add up to about lanes x the step time."""
    import torch
    lib = L.load()
    cap = 96
    evs = {}
    for name, kid in L.PROBE_KINDS.items():
        st = [torch.cuda.Event(enable_timing=True) for _ in range(cap)]
        en = [torch.cuda.Event(enable_timing=True) for _ in range(cap)]
        for e in st + en:
            e.record(main)  # torch creates the cudaEvent_t lazily on first record
        evs[name] = (st, en)
    main.synchronize()
    for name, kid in L.PROBE_KINDS.items():
        st, en = evs[name]
        L.check("probe", lib.cfdx_probe_install(kid, (L.P * cap)(*[e.cuda_event for e in st]),
                                                (L.P * cap)(*[e.cuda_event for e in en]), cap))
    try:
        graphs = [ln.capture() for ln in lanes]
        counts = {name: lib.cfdx_probe_count(kid) for name, kid in L.PROBE_KINDS.items()}
    finally:
        for kid in L.PROBE_KINDS.values():
            lib.cfdx_probe_install(kid, None, None, 0)
    tot = {n: 0.0 for n in counts}
    for _ in range(reps):
        with torch.cuda.stream(main):
            flush.zero_()
        replay(lanes, graphs, main)
        torch.cuda.synchronize()
        for name, n in counts.items():
            st, en = evs[name]
            tot[name] += sum(st[i].elapsed_time(en[i]) for i in range(min(n, cap)))
    return {n: (tot[n] / reps, counts[n]) for n in counts if counts[n] > 0}


def gpu_arm(args):
    import torch
    import torch.distributed as dist
    from paper_2505_23317_b200 import _lib as L
    from paper_2505_23317_b200 import shard
    from paper_2505_23317_b200.api import bf16_tensor

    rank, world, local = dist_env()
    # CFD_DIST_BACKEND=gloo (with ranks sharing GPUs: local rank mod device count) exercises the
    # multi-rank path on a one-GPU box -- timing is then not a scaling measurement
    backend = os.environ.get("CFD_DIST_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    cdev = dev if backend == "nccl" else torch.device("cpu")  # collective tensors
    work = Work(args, rank, world)
    cfg = work.cfg
    work.weights = ci.make_weights(cfg, seed=0)
    options = [tuple(int(t) for t in kv.split("=")) for kv in args.option]
    B = len(work.ids)
    imgs_np = np.stack([ci.make_frame(cfg.img_h, cfg.img_w, ci.frame_seed(t, 0)) for t in work.ids])
    imgs = bf16_tensor(imgs_np, dev)
    # lanes: one 128-frame lane beats two 64-frame lanes for c640 since the round-2 kernels
    # (36.1k vs 35.2k frames/s, e2e 31.5k vs 31.2k; profiles/r2g_streams.txt); multi48 keeps two
    # (device 22.0k vs 21.6k but e2e 20.1k vs 20.5k with one)
    S = args.streams if args.streams is not None else (2 if work.name == "multi48" else 1)
    S = max(1, min(S, B))
    main = torch.cuda.Stream(device=dev)

    # the whole batch as one lane (the reference for the lanes' outputs, and the kernel-alone probes)
    full = Lane(work, imgs, 0, B, dev, options, torch.cuda.Stream)
    with torch.cuda.stream(full.stream):
        full.step(full.stream, eager=True)
    full.stream.synchronize()
    full.enc.check(full.stream)
    g_full = full.capture()
    if S == 1:
        lanes, graphs = [full], [g_full]
    else:
        bounds = [round(B * si / S) for si in range(S + 1)]
        lanes = [Lane(work, imgs, bounds[si], bounds[si + 1], dev, options, torch.cuda.Stream) for si in range(S)]
        for ln in lanes:
            with torch.cuda.stream(ln.stream):
                ln.step(ln.stream, eager=True)
            ln.stream.synchronize()
        graphs = [ln.capture() for ln in lanes]
        replay(lanes, graphs, main)
        torch.cuda.synchronize()
        for ln in lanes:  # the lanes' packed outputs are the full batch's, bit for bit
            t0, t1 = sum(work.counts[:ln.f0]), sum(work.counts[:ln.f1])
            if not torch.equal(ln.ro["y"][:t1 - t0], full.ro["y"][t0:t1]):
                raise SystemExit("bench: lane outputs differ from the single-launch batch outputs")
    n0 = L.load().cfdx_launch_count()
    for ln in lanes:
        with torch.cuda.stream(ln.stream):
            ln.step(ln.stream)
    torch.cuda.synchronize()
    launches_per_step = int(L.load().cfdx_launch_count() - n0)

    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    for _ in range(max(args.warmup, 3)):
        replay(lanes, graphs, main)
    torch.cuda.synchronize()

    # ---------------------------------------------------------------- timed region
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with torch.cuda.stream(main):
        # hold the GPU (outside the timed steps) while the host enqueues all K steps, so a
        # host-side hiccup can never open an idle gap inside a step's events
        torch.cuda._sleep(int(1e6) * max(20, min(args.steps, 500)))
        for i in range(args.steps):
            flush.zero_()
            starts[i].record(main)
            replay(lanes, graphs, main)
            ends[i].record(main)
    main.synchronize()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    step_ms = [starts[i].elapsed_time(ends[i]) for i in range(args.steps)]
    total_ms = sum(step_ms)
    clk = clocks.stop()
    total_ms_max = shard.max_over_ranks(total_ms, cdev)
    value = work.frames_total * args.steps / (total_ms_max / 1e3)

    # ---------------------------------------------------------------- per-kernel probes
    peaks = load_peaks()
    probe_reps = max(2, min(args.steps, 10))
    alone = probe_kernels(L, [full], full.stream, probe_reps, flush)       # kernels one at a time
    in_step = alone if S == 1 else probe_kernels(L, lanes, main, probe_reps, flush)
    flops = algorithmic_flops(cfg, work.ks)
    bytes_ = algorithmic_bytes(cfg, work.ks)

    def merge_mlp(dct):
        # the fused MLP kernel (probe class MLP1) also does MLP2 and the O-projection
        if "gemm_mlp1" in dct and "gemm_mlp2" not in dct:
            dct["mlp_fused"] = dct.pop("gemm_mlp1")
        return dct
    alone, in_step = merge_mlp(dict(alone)), merge_mlp(dict(in_step))
    if "mlp_fused" in alone:
        flops["mlp_fused"] = flops["gemm_mlp1"] + flops["gemm_mlp2"] + (
            flops["gemm_oproj"] if "gemm_oproj" not in alone else 0)
    step_sum = sum(v[0] for v in in_step.values())
    kernels = {}
    for n, (ms, cnt) in alone.items():
        e = {"ms_per_step_alone": round(ms, 4), "launches_per_step": cnt, "us_per_launch_alone": round(ms / cnt * 1e3, 2)}
        if n in in_step:
            e["ms_per_step_in_step"] = round(in_step[n][0], 4)
            e["share_of_step"] = round(in_step[n][0] / step_sum, 4) if step_sum else None
        if n in flops and ms > 0:
            tf = flops[n] / (ms / 1e3) / 1e12
            e["tflops"] = round(tf, 1)
            e["frac_tensor_burst"] = round(tf / peaks["tensor_burst"], 4)
        if n in bytes_ and ms > 0:
            gbs = bytes_[n] / (ms / 1e3) / 1e9
            e["gbs"] = round(gbs, 1)
            e["frac_hbm"] = round(gbs / peaks["hbm"], 4)
        kernels[n] = e
    dom = max((n for n in in_step), key=lambda n: in_step[n][0])

    def roofline_for(n):
        ms, cnt = alone[n]
        avg_s = ms / cnt / 1e3
        if n in flops:
            per_launch = flops[n] / cnt
            ach = per_launch / avg_s / 1e12
            return {"kernel": n, "bound": "tensor", "achieved": round(ach, 2), "peak": peaks["tensor_burst"],
                    "unit": "TFLOP/s", "frac": round(ach / peaks["tensor_burst"], 4), "traffic": None,
                    "algorithmic_per_launch": per_launch, "avg_launch_us": round(avg_s * 1e6, 2),
                    "peak_src": f"{peaks['src']} bf16 burst (MEASURED_PEAKS bf16_tflops)"}
        per_launch = bytes_.get(n, 0) / cnt
        ach = per_launch / avg_s / 1e9 if avg_s > 0 else 0.0
        return {"kernel": n, "bound": "hbm", "achieved": round(ach, 1), "peak": peaks["hbm"], "unit": "GB/s",
                "frac": round(ach / peaks["hbm"], 4), "traffic": None, "algorithmic_per_launch": per_launch,
                "avg_launch_us": round(avg_s * 1e6, 2), "peak_src": f"{peaks['src']} copy"}

    roofline = roofline_for(dom)
    roofline["timing"] = ("CUDA events around each launch inside replays of the rank's whole batch as one CUDA "
                          "graph (kernels one at a time, all SMs), L2 flushed before each replay")
    attn_roof = roofline_for("attention")
    traffic_path = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(traffic_path):
        try:
            tr = json.load(open(traffic_path)).get(work.name, {})
            for r_ in (roofline, attn_roof):
                if r_["kernel"] in tr:
                    r_["traffic"] = tr[r_["kernel"]]
        except Exception:
            pass
    # At dh = 32 a score element carries 128 tensor FLOPs but one exp2: the
    # exp-unit roofline beside the tensor one, MUFU ex2 at 16 per clock per SM x SMs x max clock
    # (part of the exps run as an FMA-pipe polynomial, so > 100 % is possible)
    n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
    sm_mhz = (clk or {}).get("sm_max_mhz") or 1965.0
    exp_peak = 16 * n_sm * sm_mhz * 1e6 / 1e9
    attn_ms = alone["attention"][0]
    exp_ach = n_exps(cfg, work.ks) / (attn_ms / 1e3) / 1e9
    attn_exp_roof = {"kernel": "attention", "bound": "alu", "unit": "Gexp/s", "achieved": round(exp_ach, 1),
                     "peak": round(exp_peak, 1), "frac": round(exp_ach / exp_peak, 4),
                     "peak_src": f"MUFU ex2 16/clk/SM x {n_sm} SMs x {sm_mhz:.0f} MHz"}

    # ---------------------------------------------------------------- e2e through the public API
    e2e = None if args.no_e2e else e2e_measure(args, work, lanes, imgs, imgs_np, dev, main, world, u8=True, cdev=cdev)
    if e2e:
        e2e["input"] = "8-bit HWC camera frames, converted on the device (cfd_frames_from_u8, inside the graph)"
        e2e["note"] = ("pinned host frames -> device and packed refined tokens -> host every step, per lane "
                       "double-buffered, uploads and downloads on their own streams overlapped with compute")
    e2e_bf16 = None
    if e2e and work.name == "c640":
        e2e_bf16 = e2e_measure(args, work, lanes, imgs, imgs_np, dev, main, world, u8=False, cdev=cdev)
        e2e_bf16["input"] = "bf16 HWC frames (the device-resident value's input), PCIe-bound"
        e2e_bf16["outputs_equal_device_step"] = e2e_bf16.pop("_same", None)

    # ---------------------------------------------------------------- outputs gathered over NCCL, checked
    check = None if args.no_check else gather_and_check(args, work, full, rank, world, cdev)
    cpu = cpu1 = None
    if rank == 0 and not args.no_cpu_baseline and world == 1:
        cpu = time_oracle(work, args.cpu_seconds, 64)
        cpu1 = time_oracle(work, max(4.0, args.cpu_seconds / 3), 3, threads=1)

    if rank == 0:
        out = {"metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": round(total_ms_max / args.steps, 4), "higher_is_better": True,
               "scaling": work.scaling, "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
               "config": work.config(args, world, "flushed between timed steps (256 MiB memset outside events)", S),
               "roofline": roofline, "attention_roofline": attn_roof, "attention_exp_roofline": attn_exp_roof,
               "cpu_baseline": cpu, "cpu_baseline_1thread": cpu1, "e2e": e2e,
               **({"e2e_bf16_input": e2e_bf16} if e2e_bf16 else {}),
               "gpu_launches": launches_per_step * args.steps, "clocks": clk, "kernels": kernels,
               "kernel_timing": {"alone": "one replay of the whole batch as a single graph (kernels serialised)",
                                 "in_step": f"{S} lane(s) replayed concurrently as in the timed step; class "
                                            "times sum to ~lanes x step time", "probe_sum_in_step_ms":
                                            round(step_sum, 4), "lanes_x_step_ms": round(S * total_ms / args.steps, 4)},
               "step_ms_min": round(min(step_ms), 4), "step_ms_max": round(max(step_ms), 4), "check": check,
               "dist": {"backend": backend if world > 1 else None, "world_size": world,
                        "nccl_version": ".".join(map(str, torch.cuda.nccl.version())) if world > 1 else None,
                        "collectives": "max-over-ranks time, all_gather of sampled task outputs (outside timing)"},
               "impl": "ours", "library": L.load().cfd_version().decode()}
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    for ln in {id(x): x for x in [full, *lanes]}.values():
        ln.enc.close()


def e2e_measure(args, work, lanes, imgs, imgs_np, dev, main, world, u8, cdev=None):
    """Serving loop through the public API: every step uploads its frames from pinned host
    memory (8-bit camera frames converted on the device by cfd_frames_from_u8, or the bf16
    frames) and downloads the packed refined tokens + cu_seqlens to pinned host memory.  Each
    lane double-buffers: while its batch i computes, its upload stream brings batch i+1 and its
    download stream returns batch i-1.  Timed with CUDA events on `main` (fork / join to every
    lane stream), max over ranks."""
    import torch
    from paper_2505_23317_b200 import shard
    cfg = work.cfg
    u8_scale, u8_shift = ci.u8_affine()
    if u8:
        h_all = torch.from_numpy(np.stack([ci.make_frame_u8(cfg.img_h, cfg.img_w, ci.frame_seed(t, 0))
                                           for t in work.ids])).pin_memory()
    else:
        h_all = torch.from_numpy(imgs_np.view(np.int16)).pin_memory()
    ls = []
    for ln in lanes:
        e_l, s_l, f0, f1 = ln.enc, ln.stream, ln.f0, ln.f1
        h_in = h_all[f0:f1]
        ks_l, cnt_l = work.ks[f0:f1], work.counts[f0:f1]
        n_out_l = sum(cnt_l)
        sets = []
        for _ in range(2):
            d_in = torch.empty(h_in.shape, dtype=h_in.dtype, device=dev)
            d_im = torch.empty((f1 - f0, *imgs.shape[1:]), dtype=imgs.dtype, device=dev)
            o_co, o_sel, o_ro = {}, {}, {}

            def run_step(e_l=e_l, s_l=s_l, o_co=o_co, o_sel=o_sel, o_ro=o_ro, d_in=d_in, d_im=d_im, ks_l=ks_l,
                         cnt_l=cnt_l):
                if u8:
                    e_l.frames_from_u8(d_in, u8_scale, u8_shift, out=d_im, stream=s_l)
                    src = d_im
                else:
                    src = d_in.view(imgs.dtype)
                o_co.update(e_l.coarse_encode(src, out=o_co if o_co else None, stream=s_l))
                o_sel.update(e_l.select_regions(o_co["scores"], k=ks_l, out=o_sel if o_sel else None, stream=s_l))
                o_ro.update(e_l.batch_refine(src, o_co["x0"], o_sel["sel_idx"], o_sel["sel_count"],
                                             token_counts=cnt_l, out=o_ro if o_ro else None, stream=s_l))
            with torch.cuda.stream(s_l):
                d_in.copy_(h_in)
                run_step()
            s_l.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.stream(s_l):
                with torch.cuda.graph(g, stream=s_l):
                    run_step()
            s_l.synchronize()
            sets.append(dict(inp=d_in, ro=o_ro, graph=g, keep=(d_im, o_co, o_sel),
                             h_y=torch.empty(n_out_l, cfg.d_model, dtype=torch.float32).pin_memory(),
                             h_cu=torch.empty(f1 - f0 + 1, dtype=torch.int32).pin_memory(),
                             up=torch.cuda.Event(), done=torch.cuda.Event(), down=torch.cuda.Event()))
        ls.append(dict(h_in=h_in, sets=sets, s=s_l, n_out=n_out_l, copy_s=torch.cuda.Stream(device=dev),
                       down_s=torch.cuda.Stream(device=dev)))
    # at least 40 timed steps: the loop's fill (first upload) and drain (last download) are not
    # overlapped with compute, which a continuously running serving loop does not pay per step
    # (c640, 128 frames: 10 steps 31.4k, 40 steps 33.6k, 80 steps 33.6k frames/s;
    # profiles/r2h_e2e_window.txt)
    n_steps_t = max(40, args.steps)

    def run(n_steps):
        fork = torch.cuda.Event()
        fork.record(main)
        for ln in ls:
            sets, s_l, copy_s, down_s = ln["sets"], ln["s"], ln["copy_s"], ln["down_s"]
            for st_ in (s_l, copy_s, down_s):
                st_.wait_event(fork)
            with torch.cuda.stream(copy_s):
                sets[0]["inp"].copy_(ln["h_in"], non_blocking=True)
                sets[0]["up"].record(copy_s)
        for i in range(n_steps):
            for ln in ls:
                sets, s_l, copy_s, down_s = ln["sets"], ln["s"], ln["copy_s"], ln["down_s"]
                cur, nxt = sets[i % 2], sets[(i + 1) % 2]
                s_l.wait_event(cur["up"])
                if i >= 2:
                    s_l.wait_event(cur["down"])       # results of step i-2 read out of this set
                with torch.cuda.stream(s_l):
                    cur["graph"].replay()
                cur["done"].record(s_l)
                with torch.cuda.stream(copy_s):
                    if i + 1 < n_steps:
                        if i >= 1:
                            copy_s.wait_event(nxt["done"])  # step i-1 finished with the other set
                        nxt["inp"].copy_(ln["h_in"], non_blocking=True)
                        nxt["up"].record(copy_s)
                with torch.cuda.stream(down_s):
                    down_s.wait_event(cur["done"])
                    cur["h_y"].copy_(cur["ro"]["y"][:ln["n_out"]], non_blocking=True)
                    cur["h_cu"].copy_(cur["ro"]["cu_seqlens"], non_blocking=True)
                    cur["down"].record(down_s)
        for ln in ls:
            for st_ in (ln["s"], ln["copy_s"], ln["down_s"]):
                ev = torch.cuda.Event()
                ev.record(st_)
                main.wait_event(ev)

    run(2)
    torch.cuda.synchronize()
    e_s, e_e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    e_s.record(main)
    run(n_steps_t)
    e_e.record(main)
    torch.cuda.synchronize()
    e2e_ms = shard.max_over_ranks(e_s.elapsed_time(e_e), cdev if cdev is not None else dev)
    out = {"value": work.frames_total * n_steps_t / (e2e_ms / 1e3), "unit": UNIT,
           "h2d_bytes_per_step": int(h_all.numel() * h_all.element_size()),
           "d2h_bytes_per_step": int(sum(ln["sets"][0]["h_y"].numel() * 4 + ln["sets"][0]["h_cu"].numel() * 4
                                         for ln in ls)), "lanes": len(ls)}
    if not u8:
        full_y = torch.cat([ln["sets"][0]["ro"]["y"][:ln["n_out"]] for ln in ls])
        ref = torch.cat([ln_.ro["y"][:sum(ln_.counts)] for ln_ in lanes])
        out["_same"] = bool(torch.equal(full_y, ref))
    return out


def check_sample(work):
    """Local task indices whose outputs are gathered and checked: the first refined task and
    the last task of the rank."""
    idx = [i for i, k in enumerate(work.ks) if k > 0][:1] + [len(work.ks) - 1]
    return sorted(set(idx))


def gather_and_check(args, work, full, rank, world, dev):
    """Outside timing: every rank packs its sampled tasks' refined outputs, scores, token
    counts and global ids into fixed-capacity tensors; NCCL all_gather brings them to every
    rank; rank 0 checks each against the oracle on the same seeded frame (shared-score
    protocol: the oracle selects from the GPU's scores; north_star tolerance rel-L2 <= 2e-2,
    max-abs <= 5e-2) and counts the oracle-own-score selection flips."""
    import torch
    import torch.distributed
    from paper_2505_23317_b200 import shard
    cfg = work.cfg
    Nc, Nf, d = cfg.n_coarse, cfg.n_fine, cfg.d_model
    sample = check_sample(work)
    n_s = 2
    y = torch.zeros(n_s, Nf, d, dtype=torch.float32, device=dev)
    sc = torch.zeros(n_s, Nc, dtype=torch.float32, device=dev)
    meta = torch.full((n_s, 3), -1, dtype=torch.int64, device=dev)  # global id, k, tokens
    cu = full.ro["cu_seqlens"].cpu().numpy()
    for j, i in enumerate(sample[:n_s]):
        n = int(cu[i + 1] - cu[i])
        y[j, :n] = full.ro["y"][cu[i]:cu[i + 1]].to(dev)
        sc[j] = full.co["scores"][i].to(dev)
        meta[j] = torch.tensor([work.ids[i], work.ks[i], n])
    ys, scs, metas = shard.gather_outputs(y), shard.gather_outputs(sc), shard.gather_outputs(meta)
    if rank != 0:
        return None
    import oracle as O
    w = work.weights
    worst_rel = worst_abs = 0.0
    flips = 0
    checked = []
    for r in range(world):
        for j in range(n_s):
            gid, k, n = (int(v) for v in metas[r, j].tolist())
            if gid < 0:
                continue
            img = ci.make_frame(cfg.img_h, cfg.img_w, ci.frame_seed(gid, 0))
            oc = O.coarse_encode(cfg, w, [img])[0]
            s_gpu = scs[r, j].cpu().numpy()
            sel_shared = O.select_topk(s_gpu, k)
            rr = O.refine_encode(cfg, w, img, oc["x0"], sel_shared)
            yg = ys[r, j, :n].double().cpu().numpy()
            if yg.shape != rr["y"].shape:
                worst_rel = float("inf")
                continue
            worst_rel = max(worst_rel, float(np.linalg.norm(yg - rr["y"]) / np.linalg.norm(rr["y"])))
            worst_abs = max(worst_abs, float(np.abs(yg - rr["y"]).max()))
            flips += len(set(O.select_topk(oc["scores"], k).tolist()) - set(sel_shared.tolist()))
            checked.append([r, gid, k])
    return {"tasks_checked": len(checked), "ranks_checked": sorted({c[0] for c in checked}),
            "tasks": checked, "max_rel_l2": worst_rel, "max_abs": worst_abs,
            "own_score_selection_flips": flips,
            "pass": worst_rel <= 2e-2 and worst_abs <= 5e-2,
            "gathered_via": f"{torch.distributed.get_backend()} all_gather" if world > 1 else "local",
            "tasks_per_rank_gathered": n_s}


def main():
    args = parse()
    if args.impl == "reference":
        reference_arm(args)
        return
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(respawn_under_torchrun(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        raise SystemExit(f"bench: --gpus {args.gpus} but WORLD_SIZE={world}: launch with matching values")
    gpu_arm(args)


if __name__ == "__main__":
    main()
