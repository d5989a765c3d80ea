"""Saturation sweep of the HBM-bound kernels: select (B7) and
gather/split/merge (B8) over T in {48, 512, 4096} c640 tasks (k = 100 each), so a
launch moves enough bytes for GB/s to be meaningful.  Prints one JSON line.

Algorithmic bytes per task (same formula as bench.py):
  select: read scores 4*Nc, write sel_idx 4*Nc + sel_count 4
  gather: x0 rows (Nc-k)*d*4 read + write, fine pixels m^2*k*3*Pf^2*2 read + write,
          mixed_src 4*N_t, frow/fidx 8*m^2*k
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import cfd_inputs as ci  # noqa: E402
from paper_2505_23317_b200 import _lib as L  # noqa: E402
from paper_2505_23317_b200.api import CFDetrEncoder  # noqa: E402


def timed(fn, reps=10):
    for _ in range(2):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps / 1e3  # seconds


def main():
    cfg = ci.CONFIGS["c640"]
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6650.0}
    hbm = peaks["hbm_gbs"]
    lib = L.load()
    enc = CFDetrEncoder(cfg, ci.make_weights(cfg, seed=0), max_tasks=4096)
    Nc, d, k, m2 = cfg.n_coarse, cfg.d_model, 100, cfg.m ** 2
    Nt = Nc + (m2 - 1) * k
    out = {"kernel_sweep": "select+gather", "k_per_task": k, "peak_hbm_gbs": hbm, "rows": []}
    s = torch.cuda.current_stream().cuda_stream
    for T in (48, 512, 4096):
        scores = torch.rand(T, Nc, device="cuda")
        sel_idx = torch.empty(T, Nc, dtype=torch.int32, device="cuda")
        sel_cnt = torch.empty(T, dtype=torch.int32, device="cuda")
        hk = (L.I32 * T)(*([k] * T))
        t_sel = timed(lambda: lib.cfd_select_regions(enc.ctx, T, scores.data_ptr(), 0, hk, 0.0, sel_idx.data_ptr(),
                                                     sel_cnt.data_ptr(), s))
        b_sel = T * (4 * Nc + 4 * Nc + 4)
        imgs = torch.randn(T, cfg.img_h, cfg.img_w, 3, device="cuda").to(torch.bfloat16)
        x0 = torch.randn(T, Nc, d, device="cuda")
        cap = T * cfg.n_fine
        X = torch.empty(cap, d, device="cuda")
        cu = torch.empty(T + 1, dtype=torch.int32, device="cuda")
        msrc = torch.empty(cap, dtype=torch.int32, device="cuda")
        A_f = torch.empty(T * m2 * k, cfg.k_fine, dtype=torch.bfloat16, device="cuda")
        frow = torch.empty(T * m2 * k, dtype=torch.int32, device="cuda")
        fidx = torch.empty(T * m2 * k, dtype=torch.int32, device="cuda")
        meta = torch.empty(4, dtype=torch.int32, device="cuda")
        t_g = timed(lambda: lib.cfdx_gather(enc.ctx, T, imgs.data_ptr(), x0.data_ptr(), sel_idx.data_ptr(),
                                            sel_cnt.data_ptr(), X.data_ptr(), cu.data_ptr(), msrc.data_ptr(),
                                            A_f.data_ptr(), frow.data_ptr(), fidx.data_ptr(), meta.data_ptr(), s))
        b_g = T * ((Nc - k) * d * 4 * 2 + m2 * k * cfg.k_fine * 2 * 2 + 4 * Nt + m2 * k * 8)
        out["rows"].append({"T": T, "select_us": t_sel * 1e6, "select_gbs": b_sel / t_sel / 1e9,
                            "select_frac": b_sel / t_sel / 1e9 / hbm, "gather_us": t_g * 1e6,
                            "gather_bytes": b_g, "gather_gbs": b_g / t_g / 1e9, "gather_frac": b_g / t_g / 1e9 / hbm})
        del imgs, x0, X, A_f
        torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
