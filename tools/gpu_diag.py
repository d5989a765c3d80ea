"""Kernel-by-kernel diagnostics on the GPU (one subprocess per probe so a fault
in one kernel does not hide the others).  Usage: python tools/gpu_diag.py [probe ...]"""
import json
import os
import subprocess
import sys
import traceback

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _setup():
    import torch
    from paper_2505_23317_b200 import _lib as L
    return torch, L.load()


def probe_gemm():
    torch, lib = _setup()
    res = {}
    torch.manual_seed(0)
    for (M, N, K, epi) in [(128, 64, 64, 2), (128, 256, 256, 2), (300, 768, 256, 0), (1000, 1024, 256, 1),
                           (777, 256, 1024, 2), (400, 256, 3072, 2), (33, 128, 768, 0)]:
        A = (torch.randn(M, K, device="cuda") * 0.5).to(torch.bfloat16)
        W = (torch.randn(N, K, device="cuda") * 0.05).to(torch.bfloat16)
        bias = torch.randn(N, device="cuda") * 0.1
        ref = A.float() @ W.float().T + bias
        s = torch.cuda.current_stream().cuda_stream
        if epi == 2:
            base = torch.randn(M, N, device="cuda")
            out = base.clone()
            st = lib.cfdx_gemm(M, N, K, A.data_ptr(), W.data_ptr(), bias.data_ptr(), epi, None, out.data_ptr(), s)
            ref = ref + base
            got = out
        else:
            out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
            st = lib.cfdx_gemm(M, N, K, A.data_ptr(), W.data_ptr(), bias.data_ptr(), epi, out.data_ptr(), None, s)
            if epi == 1:
                ref = torch.nn.functional.gelu(ref)
            got = out.float()
        torch.cuda.synchronize()
        err = (got - ref).abs().max().item()
        rel = ((got - ref).norm() / ref.norm()).item()
        res[f"{M}x{N}x{K}/e{epi}"] = dict(status=st, maxabs=err, rel=rel)
    return res


def _attn_ref(qkv, cu, d, nh):
    import torch
    out = torch.zeros(qkv.shape[0], d, device=qkv.device)
    lse = torch.zeros(nh, qkv.shape[0], device=qkv.device)
    q, k, v = qkv[:, :d].float(), qkv[:, d:2 * d].float(), qkv[:, 2 * d:].float()
    for t in range(len(cu) - 1):
        a, b = cu[t], cu[t + 1]
        for h in range(nh):
            c = slice(h * 32, (h + 1) * 32)
            S = q[a:b, c] @ k[a:b, c].T / (32 ** 0.5)
            lse[h, a:b] = torch.logsumexp(S, dim=1)
            out[a:b, c] = torch.softmax(S, dim=1) @ v[a:b, c]
    return out, lse


def probe_attention():
    torch, lib = _setup()
    res = {}
    torch.manual_seed(1)
    for lens, d in [([128], 64), ([16], 64), ([400], 256), ([400, 640, 1600, 28], 256), ([700, 1], 256)]:
        nh = d // 32
        cu_l = [0]
        for n in lens:
            cu_l.append(cu_l[-1] + n)
        rows = cu_l[-1]
        cap = rows + 256
        qkv = (torch.randn(cap, 3 * d, device="cuda") * 1.0).to(torch.bfloat16)
        cu = torch.tensor(cu_l, dtype=torch.int32, device="cuda")
        out = torch.zeros(cap, d, device="cuda", dtype=torch.bfloat16)
        lse = torch.zeros(nh, cap, device="cuda")
        s = torch.cuda.current_stream().cuda_stream
        st = lib.cfdx_attention(len(lens), cu.data_ptr(), max(lens), cap, d, nh, qkv.data_ptr(), out.data_ptr(),
                                lse.data_ptr(), cap, s)
        torch.cuda.synchronize()
        ref, rlse = _attn_ref(qkv, cu_l, d, nh)
        got = out.float()[:rows]
        res[f"{lens}/d{d}"] = dict(status=st, maxabs=(got - ref[:rows]).abs().max().item(),
                                   rel=((got - ref[:rows]).norm() / ref[:rows].norm()).item(),
                                   lse_maxabs=(lse[:, :rows] - rlse[:, :rows]).abs().max().item())
    return res


def probe_layernorm():
    torch, lib = _setup()
    res = {}
    for M, d in [(5, 64), (300, 256)]:
        x = torch.randn(M, d, device="cuda") * 2 + 0.5
        g = torch.randn(d, device="cuda")
        b = torch.randn(d, device="cuda")
        y = torch.empty(M, d, device="cuda", dtype=torch.bfloat16)
        st = lib.cfdx_layernorm(M, d, x.data_ptr(), g.data_ptr(), b.data_ptr(), 1e-6, y.data_ptr(),
                                torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        ref = torch.nn.functional.layer_norm(x, (d,), g, b, 1e-6)
        res[f"{M}x{d}"] = dict(status=st, maxabs=(y.float() - ref).abs().max().item())
    return res


def probe_score():
    torch, lib = _setup()
    res = {}
    torch.manual_seed(2)
    for B, Nc, d in [(1, 16, 64), (3, 400, 256)]:
        nh = d // 32
        cap = B * Nc + 256
        qkv = torch.randn(cap, 3 * d, device="cuda").to(torch.bfloat16)
        cu_l = [i * Nc for i in range(B + 1)]
        _, rlse = _attn_ref(qkv, cu_l, d, nh)
        lse = rlse.contiguous()
        scores = torch.zeros(B, Nc, device="cuda")
        st = lib.cfdx_score(B, Nc, d, nh, qkv.data_ptr(), cap, lse.data_ptr(), cap, scores.data_ptr(),
                            torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        q, k = qkv[:, :d].float(), qkv[:, d:2 * d].float()
        ref = torch.zeros(B, Nc, device="cuda")
        for b in range(B):
            for h in range(nh):
                c = slice(h * 32, (h + 1) * 32)
                S = q[b * Nc:(b + 1) * Nc, c] @ k[b * Nc:(b + 1) * Nc, c].T / (32 ** 0.5)
                ref[b] += torch.softmax(S, dim=1).sum(0)
            ref[b] /= nh * Nc
        res[f"B{B}/Nc{Nc}"] = dict(status=st, maxabs=(scores - ref).abs().max().item(),
                                   rel=((scores - ref).norm() / ref.norm()).item(), sum=scores.sum(1).tolist())
    return res


def probe_pipeline():
    torch, lib = _setup()
    import numpy as np
    import cfd_inputs as ci
    import oracle as O
    from paper_2505_23317_b200.api import CFDetrEncoder, bf16_tensor
    res = {}
    for name in ("tiny", "c640"):
        cfg = ci.CONFIGS[name]
        w = ci.make_weights(cfg, seed=0)
        enc = CFDetrEncoder(cfg, w, max_tasks=8)
        nf = 2
        imgs = ci.make_frames(cfg, nf)
        dimg = bf16_tensor(imgs, "cuda")
        co = enc.coarse_encode(dimg, want_layers=True)
        k = [ci.WORKLOADS[name].ks[0]] * nf
        sel = enc.select_regions(co["scores"], k=k)
        counts = [enc.Nc + 3 * kk for kk in k]
        ro = enc.batch_refine(dimg, co["x0"], sel["sel_idx"], sel["sel_count"], token_counts=counts)
        torch.cuda.synchronize()
        enc.check()
        oc = O.coarse_encode(cfg, w, list(imgs))
        r = {}
        for f in range(nf):
            y_ref = oc[f]["y"]
            y_gpu = co["y"][f].double().cpu().numpy()
            r[f"coarse{f}_rel"] = float(np.linalg.norm(y_gpu - y_ref) / np.linalg.norm(y_ref))
            r[f"coarse{f}_maxabs"] = float(np.abs(y_gpu - y_ref).max())
            r[f"x0_{f}_maxabs"] = float(np.abs(co["x0"][f].double().cpu().numpy() - oc[f]["x0"]).max())
            s_gpu = co["scores"][f].cpu().numpy()
            r[f"score{f}_rel"] = float(np.linalg.norm(s_gpu - oc[f]["scores"]) / np.linalg.norm(oc[f]["scores"]))
            sel_gpu = sel["sel_idx"][f, :k[f]].cpu().numpy()
            sel_o = O.select_topk(s_gpu, k[f])
            r[f"sel{f}_exact"] = bool(np.array_equal(sel_gpu, sel_o))
            rr = O.refine_encode(cfg, w, imgs[f], oc[f]["x0"], sel_o)
            cu = ro["cu_seqlens"].cpu().numpy()
            yr = ro["y"][cu[f]:cu[f + 1]].double().cpu().numpy()
            r[f"refine{f}_rel"] = float(np.linalg.norm(yr - rr["y"]) / np.linalg.norm(rr["y"]))
            r[f"refine{f}_maxabs"] = float(np.abs(yr - rr["y"]).max())
            r[f"msrc{f}_exact"] = bool(np.array_equal(ro["mixed_src"][cu[f]:cu[f + 1]].cpu().numpy(), rr["mixed_src"]))
        res[name] = r
        enc.close()
    return res


def probe_attn_variants():
    torch, lib = _setup()
    res = {}
    d, nh = 256, 8
    cases = [[16], [128], [400], [700, 1], [400, 640, 880, 1120, 1360, 1600], [129, 255, 257, 3]]
    for var, npp in [(1, 4), (2, 0), (3, 0), (3, 2), (3, 4), (3, 6), (3, 8)]:
        assert lib.cfdx_set_option(0, var) == 0 and lib.cfdx_set_option(1, npp) == 0
        key = f"v{var}_npp{npp}"
        r = {}
        worst = 0.0
        for lens in cases:
            cu_l = [0]
            for n in lens:
                cu_l.append(cu_l[-1] + n)
            rows = cu_l[-1]
            cap = rows + 256
            g = torch.Generator(device="cuda").manual_seed(rows)
            qkv = (torch.randn(cap, 3 * d, device="cuda", generator=g) * 1.5).to(torch.bfloat16)
            cu = torch.tensor(cu_l, dtype=torch.int32, device="cuda")
            out = torch.zeros(cap, d, device="cuda", dtype=torch.bfloat16)
            lse = torch.zeros(nh, cap, device="cuda")
            st = lib.cfdx_attention(len(lens), cu.data_ptr(), max(lens), cap, d, nh, qkv.data_ptr(), out.data_ptr(),
                                    lse.data_ptr(), cap, torch.cuda.current_stream().cuda_stream)
            torch.cuda.synchronize()
            ref, rlse = _attn_ref(qkv, cu_l, d, nh)
            rel = ((out.float()[:rows] - ref[:rows]).norm() / ref[:rows].norm()).item()
            le = (lse[:, :rows] - rlse[:, :rows]).abs().max().item()
            worst = max(worst, rel)
            r[str(lens)] = dict(st=st, rel=rel, lse=le)
        # timing at bench shapes
        for lens in ([400] * 32, [700] * 32, [1600] * 8):
            cu_l = [0]
            for n in lens:
                cu_l.append(cu_l[-1] + n)
            cap = cu_l[-1] + 256
            qkv = torch.randn(cap, 3 * d, device="cuda").to(torch.bfloat16)
            cu = torch.tensor(cu_l, dtype=torch.int32, device="cuda")
            out = torch.zeros(cap, d, device="cuda", dtype=torch.bfloat16)
            s = torch.cuda.current_stream().cuda_stream
            for _ in range(3):
                lib.cfdx_attention(len(lens), cu.data_ptr(), max(lens), cap, d, nh, qkv.data_ptr(), out.data_ptr(), None, 0, s)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(20):
                lib.cfdx_attention(len(lens), cu.data_ptr(), max(lens), cap, d, nh, qkv.data_ptr(), out.data_ptr(), None, 0, s)
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) / 20 * 1e3
            fl = sum(4 * n * n * d for n in lens)
            r[f"time_{lens[0]}x{len(lens)}"] = dict(us=us, tflops=fl / us / 1e6)
        r["worst_rel"] = worst
        res[key] = r
    return res



PROBES = {k[6:]: v for k, v in globals().items() if k.startswith("probe_")}

if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "--one":
        name = sys.argv[2]
        try:
            out = PROBES[name]()
            print("RESULT " + json.dumps(out))
        except Exception:
            traceback.print_exc()
            sys.exit(3)
        sys.exit(0)
    names = sys.argv[1:] or list(PROBES)
    for n in names:
        r = subprocess.run(["timeout", "240", sys.executable, __file__, "--one", n], capture_output=True, text=True)
        line = [l for l in r.stdout.splitlines() if l.startswith("RESULT ")]
        print(f"=== {n}: rc={r.returncode}")
        if line:
            print(json.dumps(json.loads(line[0][7:]), indent=1))
        else:
            print(r.stdout[-3000:], r.stderr[-3000:])
        sys.stdout.flush()

