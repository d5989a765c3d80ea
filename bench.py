#!/usr/bin/env python
"""Benchmark of the CF-DETR coarse-to-fine encoder hot path on B200.

One step = one pass of the whole hot path over one batch of synthetic frames:
cfd_coarse_encode(B frames) -> cfd_select_regions(top-k per frame) ->
cfd_batch_refine(B tasks), captured in CUDA graphs and replayed.  The B frames run as
--streams S concurrent sub-batches of B/S frames (default 2), each with its own encoder
context, stream and graph, so one sub-batch's kernels fill the SMs the other's leave
idle in their last wave; the sub-batch outputs are checked to equal the full-batch
outputs bit for bit before timing.

Workload (N=1 and per rank for N>1, weak scaling): BASELINE.json configs[1]
"c640" frames — 640x640, Pc=32/Pf=16, d=256, 8 heads, 6 layers, 25 % of the
400 regions refined (k=100) — with B=32 frames in flight per GPU.  Each rank
draws its frames from the global task ids [rank*B, rank*B+B) (seeded).  L2 is
flushed (256 MiB memset) between timed steps, outside the timed events.

Prints ONE JSON line (rank 0).  `--impl reference` times the fp64 CPU oracle on
a bounded sample of the same workload instead (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
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


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--frames", type=int, default=32, help="frames in flight per GPU per step")
    ap.add_argument("--ratio", type=int, default=25, help="refine percentage per frame")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-check", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--streams", type=int, default=2,
                    help="concurrent sub-batches per GPU (own encoder / stream / CUDA graph each): their kernels "
                         "fill each other's idle SMs (persistent kernels leave SMs idle in their last wave)")
    ap.add_argument("--option", action="append", default=[],
                    help="library tuning switch KEY=VAL (cfdx_set_option, include/cfdetr_debug.h); repeatable")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def workload_config(args, n_gpus, l2_note):
    cfg = ci.CONFIGS["c640"]
    k = args.ratio * cfg.n_coarse // 100
    return {"workload": "c640", "frames_per_step_per_gpu": args.frames, "img": f"{cfg.img_h}x{cfg.img_w}",
            "patch_coarse": cfg.patch_coarse, "patch_fine": cfg.patch_fine, "refine_ratio_pct": args.ratio,
            "k_per_frame": k, "tokens_per_frame": cfg.n_coarse + 3 * k, "encoder": "d256/h8/L6",
            "parallelism": f"task-sharded x{n_gpus} (no collective on the hot path)", "l2": l2_note,
            "global_batch_frames": args.frames * n_gpus,
            "streams_per_gpu": getattr(args, "streams", 1),
            "frames_per_stream": round(args.frames / max(1, getattr(args, "streams", 1)), 2),
            **({"options": list(args.option)} if getattr(args, "option", None) else {})}


# ============================================================================ CPU oracle
def run_oracle_frames(cfg, w, imgs, k):
    import oracle as O
    for img in imgs:
        c = O.coarse_encode(cfg, w, [img])[0]
        sel = O.select_topk(c["scores"].astype(np.float32), k)
        O.refine_encode(cfg, w, img, c["x0"], sel)


def oracle_cores():
    try:
        from threadpoolctl import threadpool_info
        n = max((i.get("num_threads", 1) for i in threadpool_info()), default=1)
        return int(n)
    except Exception:
        return os.cpu_count() or 1


def cpu_baseline(args, seconds, gathered=None):
    """Oracle, as it stands, on the host cores: whole frames of the workload until `seconds`.
    Before timing (untimed), the GPU outputs gathered from the ranks (`gathered`: each rank's
    first task) are checked against the oracle on the same frames (shared-score protocol):
    the bench's only other use of oracle/ is here, in this leg."""
    cfg = ci.CONFIGS["c640"]
    w = ci.make_weights(cfg, seed=0)
    k = args.ratio * cfg.n_coarse // 100
    check = None
    if gathered is not None:
        import oracle as O
        ys, scs = gathered
        worst = 0.0
        for r in range(len(ys)):
            img = ci.make_frame(cfg.img_h, cfg.img_w, ci.frame_seed(r * args.frames, 0))
            oc = O.coarse_encode(cfg, w, [img])[0]
            selo = O.select_topk(scs[r].cpu().numpy(), k)
            rr = O.refine_encode(cfg, w, img, oc["x0"], selo)
            yg = ys[r].double().cpu().numpy()
            worst = max(worst, float(np.linalg.norm(yg - rr["y"]) / np.linalg.norm(rr["y"])))
        check = {"tasks_checked": len(ys), "max_rel_l2": worst, "pass": worst <= 2e-2}
    n = 0
    t0 = time.perf_counter()
    while True:
        img = ci.make_frame(cfg.img_h, cfg.img_w, ci.frame_seed(n, 0))
        run_oracle_frames(cfg, w, [img], k)
        n += 1
        el = time.perf_counter() - t0
        if el >= seconds or n >= 64:
            break
    return {"value": n / el, "unit": UNIT, "cores": oracle_cores(), "kind": "oracle",
            "sample": f"{n} c640 frames (coarse + top-{k} select + refine, fp64 numpy), {el:.1f} s"}, check


def reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    cfg = ci.CONFIGS["c640"]
    w = ci.make_weights(cfg, seed=0)
    k = args.ratio * cfg.n_coarse // 100
    imgs = [ci.make_frame(cfg.img_h, cfg.img_w, ci.frame_seed(i, 0)) for i in range(4)]
    for i in range(args.warmup):
        run_oracle_frames(cfg, w, [imgs[i % 4]], k)
    t0 = time.perf_counter()
    for i in range(args.steps):
        run_oracle_frames(cfg, w, [imgs[i % 4]], k)
    el = time.perf_counter() - t0
    v = args.steps / el
    cores = oracle_cores()
    sample = f"1 c640 frame per step (coarse + top-{k} select + refine, fp64 numpy oracle)"
    out = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": el / args.steps * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
           "dtype": "f64", "data": "synthetic", "impl": "reference",
           "config": workload_config(args, world, "n/a (CPU)"),
           "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
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


# ============================================================================ GPU arm
def algorithmic_flops(cfg, B, k):
    """Per-step algorithmic FLOPs by kernel class."""
    d, F, L, Nc = cfg.d_model, cfg.d_ff, cfg.n_layers, cfg.n_coarse
    m2 = cfg.m ** 2
    Nt = Nc + (m2 - 1) * k
    Mc, Mr = B * Nc, B * Nt
    Rf = B * m2 * k
    return {
        "attention": L * B * (4 * Nc * Nc * d + 4 * Nt * Nt * d),
        "score": B * 2 * Nc * Nc * d,
        "gemm_qkv": L * 2 * (Mc + Mr) * d * 3 * d,
        "gemm_oproj": L * 2 * (Mc + Mr) * d * d,
        "gemm_mlp1": L * 2 * (Mc + Mr) * d * F,
        "gemm_mlp2": L * 2 * (Mc + Mr) * F * d,
        "gemm_embed_c": 2 * Mc * cfg.k_coarse * d,
        "gemm_embed_f": 2 * Rf * cfg.k_fine * d,
    }


def algorithmic_bytes(cfg, B, k):
    """Per-step algorithmic HBM bytes of the memory-bound kernels."""
    d, Nc = cfg.d_model, cfg.n_coarse
    m2 = cfg.m ** 2
    Nt = Nc + (m2 - 1) * k
    return {
        "select": B * (4 * Nc + 4 * Nc + 4),
        "gather": B * ((Nc - k) * d * 4 * 2 + m2 * k * cfg.k_fine * 2 * 2 + 4 * Nt + m2 * k * 8),
        "im2col": B * cfg.img_h * cfg.img_w * 3 * 2 * 2,
        # standalone LN only for layer 0 of each pass; later LN1/LN2 are fused into GEMM epilogues
        "layernorm": B * (Nc + Nt) * d * (4 + 2),
    }


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        j = json.load(open(p))
        return {"hbm": j["hbm_gbs"], "tensor_burst": j["bf16_tflops"],
                "tensor_sustained": j.get("bf16_tflops_sustained", j["bf16_tflops"]), "src": "measured"}
    return {"hbm": 6650.0, "tensor_burst": 1590.0, "tensor_sustained": 1400.0, "src": "fallback"}


def gpu_arm(args):
    import torch
    import torch.distributed as dist
    from paper_2505_23317_b200 import _lib as L
    from paper_2505_23317_b200 import shard
    from paper_2505_23317_b200.api import CFDetrEncoder, bf16_tensor

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    cfg = ci.CONFIGS["c640"]
    B = args.frames
    k = args.ratio * cfg.n_coarse // 100
    ks = [k] * B
    counts = [cfg.n_coarse + (cfg.m ** 2 - 1) * k] * B
    w = ci.make_weights(cfg, seed=0)
    for kv in args.option:
        k_, v_ = (int(t) for t in kv.split("="))
        if L.load().cfdx_set_option(k_, v_) != 0:
            raise SystemExit(f"bench: invalid --option {kv}")
    enc = CFDetrEncoder(cfg, w, max_tasks=max(B, 8), device=str(dev))
    my_tasks = shard.rank_tasks(rank, world, B)  # weak scaling: B camera frames per GPU
    imgs_np = ci.make_frames(cfg, B, task0=my_tasks[0])
    imgs = bf16_tensor(imgs_np, dev)
    stream = torch.cuda.Stream(device=dev)
    co, sel, ro = {}, {}, {}

    def step(s):  # outputs were allocated by the eager warm-up below
        enc.coarse_encode(imgs, out=co, stream=s)
        enc.select_regions(co["scores"], k=ks, out=sel, stream=s)
        enc.batch_refine(imgs, co["x0"], sel["sel_idx"], sel["sel_count"], token_counts=counts, out=ro, stream=s)

    # eager warm-up (allocates outputs, sets kernel attributes), then capture
    with torch.cuda.stream(stream):
        o1 = enc.coarse_encode(imgs, stream=stream)
        co.update(o1)
        sel.update(enc.select_regions(co["scores"], k=ks, stream=stream))
        ro.update(enc.batch_refine(imgs, co["x0"], sel["sel_idx"], sel["sel_count"], token_counts=counts,
                                   stream=stream))
    stream.synchronize()
    enc.check(stream)
    n0 = L.load().cfdx_launch_count()
    with torch.cuda.stream(stream):
        step(stream)
    stream.synchronize()
    launches_per_step = int(L.load().cfdx_launch_count() - n0)

    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(stream):
        with torch.cuda.graph(graph, stream=stream):
            step(stream)
    stream.synchronize()

    # sub-batch pipelines for the timed step: S encoders (own ctx / workspace), each on its own
    # stream with its own CUDA graph over B / S frames; a step replays them concurrently
    S = max(1, min(args.streams, B))
    bounds = [round(B * si / S) for si in range(S + 1)]  # sub-batch si = frames [bounds[si], bounds[si+1])
    subs = []
    sub_launches = 0
    if S > 1:
        for si in range(S):
            f0, f1 = bounds[si], bounds[si + 1]
            e_i = CFDetrEncoder(cfg, w, max_tasks=max(f1 - f0, 8), device=str(dev))
            im_i = imgs[f0:f1]
            s_i = torch.cuda.Stream(device=dev)
            c_i, sl_i, r_i = {}, {}, {}
            ks_i, cnt_i = ks[f0:f1], counts[f0:f1]
            with torch.cuda.stream(s_i):
                c_i.update(e_i.coarse_encode(im_i, stream=s_i))
                sl_i.update(e_i.select_regions(c_i["scores"], k=ks_i, stream=s_i))
                r_i.update(e_i.batch_refine(im_i, c_i["x0"], sl_i["sel_idx"], sl_i["sel_count"], token_counts=cnt_i,
                                            stream=s_i))
            s_i.synchronize()
            n1 = L.load().cfdx_launch_count()
            g_i = torch.cuda.CUDAGraph()
            with torch.cuda.stream(s_i):
                with torch.cuda.graph(g_i, stream=s_i):
                    e_i.coarse_encode(im_i, out=c_i, stream=s_i)
                    e_i.select_regions(c_i["scores"], k=ks_i, out=sl_i, stream=s_i)
                    e_i.batch_refine(im_i, c_i["x0"], sl_i["sel_idx"], sl_i["sel_count"], token_counts=cnt_i,
                                     out=r_i, stream=s_i)
            s_i.synchronize()
            sub_launches += int(L.load().cfdx_launch_count() - n1)
            subs.append(dict(enc=e_i, stream=s_i, graph=g_i, keep=(im_i, c_i, sl_i, r_i)))
        # the sub-batch outputs are the full batch's, bit for bit (checked once here)
        for si, sb in enumerate(subs):
            sb["graph"].replay()
        torch.cuda.synchronize()
        for si, sb in enumerate(subs):
            t0, t1 = sum(counts[:bounds[si]]), sum(counts[:bounds[si + 1]])
            if not torch.equal(sb["keep"][3]["y"][:t1 - t0], ro["y"][t0:t1]):
                raise SystemExit("bench: sub-batch outputs differ from the full-batch outputs")
        launches_per_step = sub_launches

    def replay_step(main):
        if S == 1:
            graph.replay()
            return
        fork = torch.cuda.Event()
        fork.record(main)
        for sb in subs:
            sb["stream"].wait_event(fork)
            with torch.cuda.stream(sb["stream"]):
                sb["graph"].replay()
            done = torch.cuda.Event()
            done.record(sb["stream"])
            main.wait_event(done)

    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    with torch.cuda.stream(stream):
        for _ in range(max(args.warmup, 3)):
            replay_step(stream)
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
    with torch.cuda.stream(stream):
        # hold the GPU (outside the timed steps) while the host enqueues all K steps, so a
        # host-side hiccup (GC, the clock-sampler thread) can never open an idle gap inside
        # a step's events: the device time measured is the device's alone
        torch.cuda._sleep(int(1e6) * max(20, min(args.steps, 500)))
        for i in range(args.steps):
            flush.zero_()
            starts[i].record(stream)
            replay_step(stream)
            ends[i].record(stream)
    stream.synchronize()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    step_ms = [starts[i].elapsed_time(ends[i]) for i in range(args.steps)]
    total_ms = sum(step_ms)
    clk = clocks.stop()
    total_ms_max = shard.max_over_ranks(total_ms, dev)
    frames_total = B * world * args.steps
    value = frames_total / (total_ms_max / 1e3)

    # ---------------------------------------------------------------- per-kernel probes (live, eager steps)
    lib = L.load()
    kinds = L.PROBE_KINDS
    cap = 64
    evs = {}
    for name, kid in kinds.items():
        st = [torch.cuda.Event(enable_timing=True) for _ in range(cap)]
        en = [torch.cuda.Event(enable_timing=True) for _ in range(cap)]
        for e in st + en:
            e.record(stream)  # torch creates the cudaEvent_t lazily on first record
        evs[name] = (st, en)
    stream.synchronize()
    kern_ms = {n: 0.0 for n in kinds}
    kern_cnt = {n: 0 for n in kinds}
    probe_steps = max(1, min(args.steps, 5))
    for _ in range(probe_steps):
        for name, kid in kinds.items():
            st, en = evs[name]
            arr_s = (L.P * cap)(*[e.cuda_event for e in st])
            arr_e = (L.P * cap)(*[e.cuda_event for e in en])
            L.check("probe", lib.cfdx_probe_install(kid, arr_s, arr_e, cap))
        with torch.cuda.stream(stream):
            flush.zero_()
            step(stream)
        stream.synchronize()
        for name, kid in kinds.items():
            n = lib.cfdx_probe_count(kid)
            st, en = evs[name]
            kern_ms[name] += sum(st[i].elapsed_time(en[i]) for i in range(n))
            kern_cnt[name] += n
    for name, kid in kinds.items():
        lib.cfdx_probe_install(kid, None, None, 0)
    kern_ms = {n: v / probe_steps for n, v in kern_ms.items()}
    kern_cnt = {n: v // probe_steps for n, v in kern_cnt.items()}
    probed_total = sum(kern_ms.values())

    peaks = load_peaks()
    flops = algorithmic_flops(cfg, B, k)
    bytes_ = algorithmic_bytes(cfg, B, k)
    # the fused MLP kernel (probe class MLP1) also does MLP2 and, with the fused O-projection,
    # the O-projection: its algorithmic work is theirs too, reported as "mlp_fused"
    if kern_cnt.get("gemm_mlp1", 0) and not kern_cnt.get("gemm_mlp2", 0):
        f = flops["gemm_mlp1"] + flops["gemm_mlp2"]
        if not kern_cnt.get("gemm_oproj", 0):
            f += flops["gemm_oproj"]
        flops["mlp_fused"] = f
        for dct in (kern_ms, kern_cnt):
            dct["mlp_fused"] = dct.pop("gemm_mlp1")
        kinds = {("mlp_fused" if n == "gemm_mlp1" else n): v for n, v in kinds.items()}
    kernels = {}
    for n in kinds:
        if kern_cnt[n] == 0:
            continue
        e = {"ms_per_step": round(kern_ms[n], 4), "launches_per_step": kern_cnt[n],
             "share": round(kern_ms[n] / probed_total, 4) if probed_total else None}
        if n in flops and kern_ms[n] > 0:
            tf = flops[n] / (kern_ms[n] / 1e3) / 1e12
            e["tflops"] = round(tf, 1)
            e["frac_tensor"] = round(tf / peaks["tensor_sustained"], 4)
        if n in bytes_ and kern_ms[n] > 0:
            gbs = bytes_[n] / (kern_ms[n] / 1e3) / 1e9
            e["gbs"] = round(gbs, 1)
            e["frac_hbm"] = round(gbs / peaks["hbm"], 4)
        kernels[n] = e
    dom = max(kernels, key=lambda n: kern_ms[n])

    def roofline_for(n):
        if n in flops:
            per_launch = flops[n] / max(kern_cnt[n], 1)
            avg_s = kern_ms[n] / max(kern_cnt[n], 1) / 1e3
            ach = per_launch / avg_s / 1e12
            return {"kernel": n, "bound": "tensor", "achieved": round(ach, 2), "peak": peaks["tensor_sustained"],
                    "unit": "TFLOP/s", "frac": round(ach / peaks["tensor_sustained"], 4), "traffic": None,
                    "algorithmic_per_launch": per_launch, "avg_launch_us": round(avg_s * 1e6, 2),
                    "peak_src": f"{peaks['src']} bf16 sustained"}
        per_launch = bytes_.get(n, 0) / max(kern_cnt[n], 1)
        avg_s = kern_ms[n] / max(kern_cnt[n], 1) / 1e3
        ach = per_launch / avg_s / 1e9 if avg_s > 0 else 0.0
        return {"kernel": n, "bound": "hbm", "achieved": round(ach, 1), "peak": peaks["hbm"], "unit": "GB/s",
                "frac": round(ach / peaks["hbm"], 4), "traffic": None, "algorithmic_per_launch": per_launch,
                "avg_launch_us": round(avg_s * 1e6, 2), "peak_src": f"{peaks['src']} copy"}

    roofline = roofline_for(dom)
    attn_roof = roofline_for("attention")
    traffic_path = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(traffic_path):
        try:
            tr = json.load(open(traffic_path))
            for r_ in (roofline, attn_roof):
                if r_["kernel"] in tr:
                    r_["traffic"] = tr[r_["kernel"]]
        except Exception:
            pass
    # At dh = 32 a score element carries 4*dh = 128 tensor FLOPs but one exp2 (SURVEY.md §8(d)
    # "per-element ceilings"): the kernel is bounded by the exp / FMA issue, not the tensor
    # pipe.  Exp-unit roofline beside the tensor one: exps per step / attention time against
    # MUFU ex2 at 16 per clock per SM (profiles/r1_mufu_micro.txt) x SMs x max SM clock.
    # (A quarter of the exps run as an FMA-pipe polynomial, so > 100 % is possible.)
    n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
    sm_mhz = (clk or {}).get("sm_max_mhz") or 1965.0
    exps = cfg.n_layers * B * cfg.n_heads * (cfg.n_coarse ** 2 + (cfg.n_coarse + (cfg.m ** 2 - 1) * k) ** 2)
    exp_peak = 16 * n_sm * sm_mhz * 1e6 / 1e9  # Gexp/s
    exp_ach = exps / (kern_ms["attention"] / 1e3) / 1e9 if kern_ms.get("attention") else 0.0
    attn_exp_roof = {"kernel": "attention", "bound": "alu", "unit": "Gexp/s", "achieved": round(exp_ach, 1),
                     "peak": round(exp_peak, 1), "frac": round(exp_ach / exp_peak, 4),
                     "peak_src": f"MUFU ex2 16/clk/SM x {n_sm} SMs x {sm_mhz:.0f} MHz"}

    # ---------------------------------------------------------------- e2e through the public API, host buffers
    # Serving-style loop: frames arrive in pinned host memory, results return to pinned host
    # memory.  The step's frames are served by the same S sub-batch lanes as the timed step
    # (one encoder / compute stream per lane), each lane a double-buffered loop: while its
    # batch i computes (graph replay on the lane's stream) its upload stream brings batch i+1
    # and its download stream returns batch i-1's refined tokens (both PCIe directions at
    # once).  The headline e2e takes 8-bit HWC camera frames (1 B per value over PCIe) and
    # converts them on the device (cfd_frames_from_u8, inside each graph); `e2e_bf16_input`
    # uploads the bf16 frames the device-resident `value` uses (2 B per value, PCIe-bound).
    u8_scale, u8_shift = ci.u8_affine()
    h_u8 = torch.from_numpy(ci.make_frames_u8(cfg, B, task0=my_tasks[0])).pin_memory()
    h_bf = torch.from_numpy(imgs_np.view(np.int16)).pin_memory()
    if S > 1:
        lane_defs = [(sb["enc"], sb["stream"], bounds[si], bounds[si + 1]) for si, sb in enumerate(subs)]
    else:
        lane_defs = [(enc, stream, 0, B)]

    def e2e_measure(u8_input):
        h_all = h_u8 if u8_input else h_bf
        lanes = []
        for (e_l, s_l, f0, f1) in lane_defs:
            h_in = h_all[f0:f1]
            ks_l, cnt_l = ks[f0:f1], counts[f0:f1]
            n_out_l = sum(cnt_l)
            sets = []
            for _bset in range(2):
                d_in = torch.empty(h_in.shape, dtype=h_in.dtype, device=dev)
                d_im = torch.empty((f1 - f0, *imgs.shape[1:]), dtype=imgs.dtype, device=dev)
                o_co, o_sel, o_ro = {}, {}, {}

                def run_step(e_l=e_l, s_l=s_l, o_co=o_co, o_sel=o_sel, o_ro=o_ro, d_in=d_in, d_im=d_im,
                             ks_l=ks_l, cnt_l=cnt_l):
                    if u8_input:
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
            lanes.append(dict(h_in=h_in, sets=sets, s=s_l, n_out=n_out_l, copy_s=torch.cuda.Stream(device=dev),
                              down_s=torch.cuda.Stream(device=dev)))
        n_steps_t = max(8, args.steps)

        def e2e_run(n_steps, main):
            fork = torch.cuda.Event()
            fork.record(main)
            for ln in lanes:
                sets, s_l, copy_s, down_s = ln["sets"], ln["s"], ln["copy_s"], ln["down_s"]
                for st_ in (s_l, copy_s, down_s):
                    st_.wait_event(fork)
                with torch.cuda.stream(copy_s):
                    sets[0]["inp"].copy_(ln["h_in"], non_blocking=True)
                    sets[0]["up"].record(copy_s)
            for i in range(n_steps):
                for ln in lanes:
                    sets, s_l, copy_s, down_s = ln["sets"], ln["s"], ln["copy_s"], ln["down_s"]
                    cur, nxt = sets[i % 2], sets[(i + 1) % 2]
                    s_l.wait_event(cur["up"])
                    if i >= 2:
                        s_l.wait_event(cur["down"])       # results of step i-2 read out of this set
                    with torch.cuda.stream(s_l):        # replay() launches on the current stream
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
            for ln in lanes:  # join every lane's compute and copies
                for st_ in (ln["s"], ln["copy_s"], ln["down_s"]):
                    ev = torch.cuda.Event()
                    ev.record(st_)
                    main.wait_event(ev)

        e2e_run(2, stream)
        torch.cuda.synchronize()
        e_s = torch.cuda.Event(enable_timing=True)
        e_e = torch.cuda.Event(enable_timing=True)
        if world > 1:
            dist.barrier()
        e_s.record(stream)
        e2e_run(n_steps_t, stream)
        e_e.record(stream)
        torch.cuda.synchronize()
        e2e_ms = shard.max_over_ranks(e_s.elapsed_time(e_e), dev)
        # the served outputs are the device-resident step's (checked once, outside the timing)
        y_served = torch.cat([ln["sets"][0]["ro"]["y"][:ln["n_out"]] for ln in lanes])
        same = bool(torch.equal(y_served, ro["y"][:sum(counts)])) if not u8_input else None
        return {"value": B * world * n_steps_t / (e2e_ms / 1e3), "unit": UNIT,
                "h2d_bytes_per_step": int(h_all.numel() * h_all.element_size()),
                "d2h_bytes_per_step": int(sum(ln["sets"][0]["h_y"].numel() * 4 + ln["sets"][0]["h_cu"].numel() * 4
                                              for ln in lanes)),
                "lanes": len(lanes), **({"outputs_equal_device_step": same} if same is not None else {})}

    e2e = e2e_measure(True)
    e2e["input"] = "8-bit HWC camera frames, converted on the device (cfd_frames_from_u8, inside the graph)"
    e2e["note"] = ("pinned host frames -> device and packed refined tokens -> host every step, per sub-batch "
                   "lane double-buffered, uploads and downloads on their own streams overlapped with compute")
    e2e_bf16 = e2e_measure(False)
    e2e_bf16["input"] = "bf16 HWC frames (the device-resident value's input), PCIe-bound"

    # ---------------------------------------------------------------- NCCL gather of outputs for checking
    gathered = None if args.no_check else gather_outputs(rank, cfg, co, ro, k)
    cpu, check = None, None
    if rank == 0 and not args.no_cpu_baseline and world == 1:
        cpu, check = cpu_baseline(args, args.cpu_seconds, gathered)
    if check is not None:
        check["gathered_via"] = "nccl all_gather" if world > 1 else "local"
    elif rank == 0 and gathered is not None:
        ys, _ = gathered
        check = {"tasks_checked": 0, "gathered_via": "nccl all_gather" if world > 1 else "local",
                 "all_finite": bool(all(torch.isfinite(y).all() for y in ys)),
                 "note": "oracle check runs in the cpu_baseline leg (rank 0, N=1)"}

    if rank == 0:
        out = {"metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": round(total_ms_max / args.steps, 4), "higher_is_better": True,
               "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
               "config": workload_config(args, world, "flushed between timed steps (256 MiB memset outside events)"),
               "roofline": roofline, "attention_roofline": attn_roof, "attention_exp_roofline": attn_exp_roof,
               "cpu_baseline": cpu, "e2e": e2e, "e2e_bf16_input": e2e_bf16,
               "gpu_launches": launches_per_step * args.steps, "clocks": clk, "kernels": kernels,
               "step_ms_min": round(min(step_ms), 4), "step_ms_max": round(max(step_ms), 4), "check": check,
               "impl": "ours", "library": lib.cfd_version().decode()}
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()
    enc.close()


def gather_outputs(rank, cfg, co, ro, k):
    """Outside timing: all-gather (NCCL) each rank's first task (packed refined rows, coarse
    scores); rank 0 gets the lists, the others None."""
    from paper_2505_23317_b200 import shard
    Nt = cfg.n_coarse + 3 * k
    ys = shard.gather_outputs(ro["y"][:Nt].contiguous())
    scs = shard.gather_outputs(co["scores"][0].contiguous())
    return (ys, scs) if rank == 0 else None


def main():
    args = parse()
    if args.impl == "reference":
        reference_arm(args)
        return
    gpu_arm(args)


if __name__ == "__main__":
    main()
