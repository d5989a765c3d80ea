"""Thin Python binding over libcfdetr.so: the same four calls as include/cfdetr.h.

Argument marshalling only (torch owns device memory, streams supply the queue);
every step of the path runs in the library's sm_100a kernels.
"""
from __future__ import annotations

import ctypes as C
from typing import Dict, List, Optional, Sequence

import numpy as np
import torch

from . import _lib as L

_BF16 = torch.bfloat16


def _ptr(t: Optional[torch.Tensor]) -> Optional[int]:
    return None if t is None else t.data_ptr()


def _stream(stream: Optional[torch.cuda.Stream]) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def bf16_tensor(x, device) -> torch.Tensor:
    """numpy float32 (exact bf16 values) or uint16 bf16 bits -> torch bf16 on device."""
    a = np.asarray(x)
    if a.dtype == np.uint16:
        return torch.from_numpy(a.view(np.int16).copy()).view(_BF16).to(device)
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(device).to(_BF16)


def f32_tensor(x, device) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(device)


class CFDetrEncoder:
    """B200 coarse-to-fine encoder (one library ctx).

    cfg: object with img_h, img_w, patch_coarse, patch_fine, d_model, n_heads,
    n_layers, d_ff, score_layer, ln_eps (e.g. cfd_inputs.ModelConfig).
    weights: dict of numpy arrays in the layout of cfd_inputs.make_weights.
    """

    def __init__(self, cfg, weights: dict, max_tasks: int = 64, device: str = "cuda",
                 stream: Optional[torch.cuda.Stream] = None):
        self.lib = L.load()
        self.device = torch.device(device)
        self.cfg = cfg
        self.max_tasks = int(max_tasks)
        c = L.cfd_config(cfg.img_h, cfg.img_w, cfg.patch_coarse, cfg.patch_fine, cfg.d_model, cfg.n_heads,
                         cfg.n_layers, cfg.d_ff, cfg.score_layer, self.max_tasks, cfg.ln_eps)
        dev = self.device
        # keep device copies alive until cfd_create's repack has run on the stream
        self._w = {k: (bf16_tensor(v, dev) if k.startswith("w_") else f32_tensor(v, dev))
                   for k, v in weights.items() if k != "layers"}
        self._lw: List[Dict[str, torch.Tensor]] = []
        arr = (L.cfd_layer_weights * cfg.n_layers)()
        for i, lw in enumerate(weights["layers"]):
            t = {k: (bf16_tensor(v, dev) if k.startswith("w_") else f32_tensor(v, dev)) for k, v in lw.items()}
            self._lw.append(t)
            arr[i] = L.cfd_layer_weights(*[t[k].data_ptr() for k in (
                "w_qkv", "w_o", "w_1", "w_2", "b_qkv", "b_o", "b_1", "b_2", "ln1_g", "ln1_b", "ln2_g", "ln2_b")])
        w = L.cfd_weights(self._w["w_embed_c"].data_ptr(), self._w["w_embed_f"].data_ptr(),
                          self._w["b_embed_c"].data_ptr(), self._w["b_embed_f"].data_ptr(),
                          self._w["pe_c"].data_ptr(), self._w["pe_f"].data_ptr(), arr)
        ctx = C.c_void_p()
        s = _stream(stream)
        L.check("cfd_create", self.lib.cfd_create(C.byref(c), C.byref(w), s, C.byref(ctx)))
        torch.cuda.current_stream().synchronize() if stream is None else stream.synchronize()
        self.ctx = ctx
        self._w = None
        self._lw = None
        nc, nf, mt, ws = C.c_int32(), C.c_int32(), C.c_int32(), C.c_size_t()
        L.check("cfd_query", self.lib.cfd_query(ctx, 1, C.byref(nc), C.byref(nf), C.byref(mt), C.byref(ws)))
        self.Nc, self.Nf = nc.value, nf.value
        self._ws: Dict[int, torch.Tensor] = {}

    # ------------------------------------------------------------------ helpers
    def workspace(self, n: int) -> torch.Tensor:
        if n not in self._ws:
            ws = C.c_size_t()
            L.check("cfd_query", self.lib.cfd_query(self.ctx, n, None, None, None, C.byref(ws)))
            self._ws[n] = torch.empty(ws.value, dtype=torch.uint8, device=self.device)
        return self._ws[n]

    def close(self):
        if getattr(self, "ctx", None):
            self.lib.cfd_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_option(self, key: int, value: int) -> None:
        """Tuning switch of this context (cfdx_set_option, include/cfdetr_debug.h)."""
        L.check("cfdx_set_option", self.lib.cfdx_set_option(self.ctx, int(key), int(value)))

    def check(self, stream=None):
        L.check("cfd_check", self.lib.cfd_check(self.ctx, _stream(stream)))

    # ------------------------------------------------------------------ the four calls
    def coarse_encode(self, images: torch.Tensor, want_scores: bool = True, want_layers: bool = False,
                      out: Optional[dict] = None, stream=None) -> dict:
        """images [B, H, W, 3] bf16 (device) -> dict(x0, y, scores, layer_out)."""
        B = images.shape[0]
        d = self.cfg.d_model
        o = out if out is not None else {}
        dev = self.device
        if "x0" not in o:
            o["x0"] = torch.empty(B, self.Nc, d, dtype=torch.float32, device=dev)
            o["y"] = torch.empty(B, self.Nc, d, dtype=torch.float32, device=dev)
            o["scores"] = torch.empty(B, self.Nc, dtype=torch.float32, device=dev) if want_scores else None
            o["layer_out"] = (torch.empty(self.cfg.n_layers, B, self.Nc, d, dtype=torch.float32, device=dev)
                              if want_layers else None)
        ws = self.workspace(B)
        L.check("cfd_coarse_encode", self.lib.cfd_coarse_encode(
            self.ctx, B, images.data_ptr(), o["x0"].data_ptr(), o["y"].data_ptr(), _ptr(o["scores"]),
            _ptr(o["layer_out"]), ws.data_ptr(), ws.numel(), _stream(stream)))
        return o

    def select_regions(self, scores: torch.Tensor, k: Optional[Sequence[int]] = None,
                       threshold: Optional[float] = None, out: Optional[dict] = None, stream=None) -> dict:
        """Top-k (k per task) or threshold selection -> dict(sel_idx [T, Nc], sel_count [T])."""
        T = scores.shape[0]
        o = out if out is not None else {}
        if "sel_idx" not in o:
            o["sel_idx"] = torch.empty(T, self.Nc, dtype=torch.int32, device=self.device)
            o["sel_count"] = torch.empty(T, dtype=torch.int32, device=self.device)
        if k is not None:
            hk = (C.c_int32 * T)(*[int(v) for v in k])
            st = self.lib.cfd_select_regions(self.ctx, T, scores.data_ptr(), 0, hk, 0.0, o["sel_idx"].data_ptr(),
                                             o["sel_count"].data_ptr(), _stream(stream))
        else:
            st = self.lib.cfd_select_regions(self.ctx, T, scores.data_ptr(), 1, None, float(threshold),
                                             o["sel_idx"].data_ptr(), o["sel_count"].data_ptr(), _stream(stream))
        L.check("cfd_select_regions", st)
        return o

    def batch_refine(self, images: torch.Tensor, x0: torch.Tensor, sel_idx: torch.Tensor, sel_count: torch.Tensor,
                     token_counts: Optional[Sequence[int]] = None, want_layers: bool = False,
                     out: Optional[dict] = None, stream=None) -> dict:
        """Patch-level batch refine of T tasks -> dict(y [cap, d], cu_seqlens [T+1], mixed_src [cap], layer_out)."""
        T = images.shape[0]
        cap = T * self.Nf
        d = self.cfg.d_model
        o = out if out is not None else {}
        dev = self.device
        if "y" not in o:
            o["y"] = torch.empty(cap, d, dtype=torch.float32, device=dev)
            o["cu_seqlens"] = torch.empty(T + 1, dtype=torch.int32, device=dev)
            o["mixed_src"] = torch.empty(cap, dtype=torch.int32, device=dev)
            o["layer_out"] = (torch.empty(self.cfg.n_layers, cap, d, dtype=torch.float32, device=dev)
                              if want_layers else None)
        ws = self.workspace(T)
        hint = (C.c_int32 * T)(*[int(v) for v in token_counts]) if token_counts is not None else None
        L.check("cfd_batch_refine", self.lib.cfd_batch_refine(
            self.ctx, T, images.data_ptr(), x0.data_ptr(), sel_idx.data_ptr(), sel_count.data_ptr(), hint,
            o["y"].data_ptr(), o["cu_seqlens"].data_ptr(), o["mixed_src"].data_ptr(), _ptr(o["layer_out"]),
            ws.data_ptr(), ws.numel(), _stream(stream)))
        return o

    def batch_refine_padded(self, images: torch.Tensor, x0: torch.Tensor, sel_idx: torch.Tensor,
                            sel_count: torch.Tensor, max_tokens: int, want_layers: bool = False,
                            out: Optional[dict] = None, stream=None) -> dict:
        """The paper's pad-to-max batch (NEXT f4, cfd_batch_refine_padded): every task spans
        max_tokens rows, pad keys masked -> dict(y [T*max_tokens, d], cu_seqlens, kv_len [T],
        mixed_src, layer_out)."""
        T = images.shape[0]
        rows = T * int(max_tokens)
        d = self.cfg.d_model
        o = out if out is not None else {}
        dev = self.device
        if "y" not in o:
            o["y"] = torch.empty(rows, d, dtype=torch.float32, device=dev)
            o["cu_seqlens"] = torch.empty(T + 1, dtype=torch.int32, device=dev)
            o["kv_len"] = torch.empty(T, dtype=torch.int32, device=dev)
            o["mixed_src"] = torch.empty(rows, dtype=torch.int32, device=dev)
            o["layer_out"] = (torch.empty(self.cfg.n_layers, rows, d, dtype=torch.float32, device=dev)
                              if want_layers else None)
        ws = self.workspace(T)
        L.check("cfd_batch_refine_padded", self.lib.cfd_batch_refine_padded(
            self.ctx, T, images.data_ptr(), x0.data_ptr(), sel_idx.data_ptr(), sel_count.data_ptr(), int(max_tokens),
            o["y"].data_ptr(), o["cu_seqlens"].data_ptr(), o["kv_len"].data_ptr(), o["mixed_src"].data_ptr(),
            _ptr(o["layer_out"]), ws.data_ptr(), ws.numel(), _stream(stream)))
        return o

    def refine_encode(self, image: torch.Tensor, x0: torch.Tensor, sel_idx: torch.Tensor, sel_count: torch.Tensor,
                      want_layers: bool = False, stream=None) -> dict:
        """Single-task refine (image [H, W, 3] or [1, H, W, 3])."""
        d = self.cfg.d_model
        dev = self.device
        o = {"y": torch.empty(self.Nf, d, dtype=torch.float32, device=dev),
             "mixed_src": torch.empty(self.Nf, dtype=torch.int32, device=dev),
             "cu_seqlens": torch.empty(2, dtype=torch.int32, device=dev),
             "layer_out": (torch.empty(self.cfg.n_layers, self.Nf, d, dtype=torch.float32, device=dev)
                           if want_layers else None)}
        ws = self.workspace(1)
        L.check("cfd_refine_encode", self.lib.cfd_refine_encode(
            self.ctx, image.data_ptr(), x0.data_ptr(), sel_idx.data_ptr(), sel_count.data_ptr(), o["y"].data_ptr(),
            o["mixed_src"].data_ptr(), o["cu_seqlens"].data_ptr(), _ptr(o["layer_out"]), ws.data_ptr(), ws.numel(),
            _stream(stream)))
        return o


def _hardness(self, conf: torch.Tensor, c_hi: float = 0.8, tau_easy: float = 0.05, stream=None) -> torch.Tensor:
    """A1 hardness gate (NEXT f2): conf [B, Q] fp32 -> hard [B] int32 (1 = refine, 0 = easy)."""
    B, Q = conf.shape
    hard = torch.empty(B, dtype=torch.int32, device=self.device)
    L.check("cfd_hardness", self.lib.cfd_hardness(self.ctx, B, Q, conf.data_ptr(), c_hi, tau_easy, hard.data_ptr(),
                                                  _stream(stream)))
    return hard


def _box_scores(self, boxes: torch.Tensor, conf: torch.Tensor, c_lo: float = 0.05, c_hi: float = 0.8,
                stream=None) -> torch.Tensor:
    """Box-driven region scores (NEXT f1): boxes [B, Q, 4], conf [B, Q] -> scores [B, Nc]."""
    B, Q = conf.shape
    scores = torch.empty(B, self.Nc, dtype=torch.float32, device=self.device)
    L.check("cfd_box_scores", self.lib.cfd_box_scores(self.ctx, B, Q, boxes.data_ptr(), conf.data_ptr(), c_lo, c_hi,
                                                      scores.data_ptr(), _stream(stream)))
    return scores


def _set_decoder(self, wdec: dict, stream=None) -> None:
    """Load the NEXT-f3 decoder block (cfd_set_decoder): dict from cfd_inputs.make_decoder_weights."""
    dev = self.device
    t = {k: (bf16_tensor(v, dev) if k in ("w_q", "w_kv", "w_o") else f32_tensor(v, dev)) for k, v in wdec.items()}
    dw = L.cfd_decoder_weights(int(wdec["queries"].shape[0]), *[t[k].data_ptr() for k in (
        "queries", "ln_q_g", "ln_q_b", "ln_m_g", "ln_m_b", "w_q", "w_kv", "w_o", "b_q", "b_kv", "b_o", "w_head",
        "b_head")])
    L.check("cfd_set_decoder", self.lib.cfd_set_decoder(self.ctx, C.byref(dw), _stream(stream)))
    (stream or torch.cuda.current_stream()).synchronize()
    self.n_queries = int(wdec["queries"].shape[0])
    self._ws = {}  # the workspace size depends on the query count (cfd_query after cfd_set_decoder)


def _decode(self, y: torch.Tensor, cu_seqlens: torch.Tensor, n_tasks: int, max_tokens: int, stream=None) -> dict:
    """Decoder cross-attention + heads (NEXT f3) over packed encoder outputs:
    -> z [T, Q, d] fp32, boxes [T, Q, 4] (cx, cy, w, h), conf [T, Q]."""
    T, Q, d = int(n_tasks), self.n_queries, self.cfg.d_model
    z = torch.empty(T, Q, d, dtype=torch.float32, device=self.device)
    boxes = torch.empty(T, Q, 4, dtype=torch.float32, device=self.device)
    conf = torch.empty(T, Q, dtype=torch.float32, device=self.device)
    ws = self.workspace(T)
    L.check("cfd_decode", self.lib.cfd_decode(self.ctx, T, y.data_ptr(), cu_seqlens.data_ptr(), int(max_tokens),
                                              z.data_ptr(), boxes.data_ptr(), conf.data_ptr(), ws.data_ptr(),
                                              ws.numel(), _stream(stream)))
    return {"z": z, "boxes": boxes, "conf": conf}



def _f3(v) -> "C.Array":
    a = [float(x) for x in v]
    if len(a) != 3:
        raise ValueError("expected 3 per-channel values")
    return (L.F32 * 3)(*a)


def frames_from_u8_flat(src: torch.Tensor, scale, shift, out: Optional[torch.Tensor] = None,
                        stream=None) -> torch.Tensor:
    """cfdx_frames_u8 on a flat uint8 device tensor (any length; element i is channel i mod 3)."""
    n = src.numel()
    o = out if out is not None else torch.empty(n, dtype=_BF16, device=src.device)
    L.check("cfdx_frames_u8", L.load().cfdx_frames_u8(n, src.data_ptr(), _f3(scale), _f3(shift), o.data_ptr(),
                                                      _stream(stream)))
    return o


def _frames_from_u8(self, src: torch.Tensor, scale, shift, out: Optional[torch.Tensor] = None,
                    stream=None) -> torch.Tensor:
    """8-bit HWC frames [B, H, W, 3] uint8 (device) -> bf16 frames for the encode calls
    (cfd_frames_from_u8: bf16_rn(fma_f32(p, scale[c], shift[c])))."""
    if src.dtype != torch.uint8 or not src.is_contiguous():
        raise ValueError("frames_from_u8: src must be a contiguous uint8 tensor")
    B = src.shape[0]
    o = out if out is not None else torch.empty(B, self.cfg.img_h, self.cfg.img_w, 3, dtype=_BF16,
                                                device=self.device)
    L.check("cfd_frames_from_u8", self.lib.cfd_frames_from_u8(self.ctx, B, src.data_ptr(), _f3(scale), _f3(shift),
                                                              o.data_ptr(), _stream(stream)))
    return o

CFDetrEncoder.set_decoder = _set_decoder
CFDetrEncoder.decode = _decode
CFDetrEncoder.hardness = _hardness
CFDetrEncoder.box_scores = _box_scores
CFDetrEncoder.frames_from_u8 = _frames_from_u8


def launch_count() -> int:
    return int(L.load().cfdx_launch_count())
