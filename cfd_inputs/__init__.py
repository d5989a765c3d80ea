"""Seeded synthetic inputs shared by the oracle, the tests and the bench.

This module holds NONE of the method's arithmetic (no patchify, embedding,
attention, scoring, selection or merge).  It only produces the *inputs* both
sides consume, so that oracle-vs-GPU differences measure arithmetic only:

* model geometry for the five BASELINE.json configs,
* camera frames (bf16, HWC) shaped like the paper's multi-camera AV workloads
  (KITTI-like urban scenes, §V-A; several cameras, PAPER.md:117
  §II-A; critical-object size 16384 px^2, §II-B),
* random-init model parameters (bf16 matrices, fp32 vectors) and the fixed
  sin-cos positional tables, which this build treats as model parameters
  (reading R3: the paper is silent on positional encoding),
* per-task refine counts k_t.

Recipe; all randomness is numpy PCG64 with explicit seeds.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Dict, List, Sequence

import numpy as np

__all__ = [
    "ModelConfig", "Workload", "CONFIGS", "WORKLOADS", "bf16_round", "bf16_bits", "make_decoder_weights",
    "bf16_from_bits", "make_frame", "make_frames", "make_weights", "frame_seed",
    "pe_table", "ks_for_ratios", "multi48_group_ks", "make_queries",
]


# ----------------------------------------------------------------------------
# geometry
# ----------------------------------------------------------------------------
@dataclasses.dataclass(frozen=True)
class ModelConfig:
    img_h: int
    img_w: int
    patch_coarse: int   # Pc
    patch_fine: int     # Pf
    d_model: int        # d
    n_heads: int        # nh
    n_layers: int       # L
    d_ff: int           # F = 4d
    score_layer: int    # layer whose attention map scores regions (default L-1)
    ln_eps: float = 1e-6

    @property
    def m(self) -> int:
        return self.patch_coarse // self.patch_fine

    @property
    def gc_h(self) -> int:
        return self.img_h // self.patch_coarse

    @property
    def gc_w(self) -> int:
        return self.img_w // self.patch_coarse

    @property
    def gf_w(self) -> int:
        return self.img_w // self.patch_fine

    @property
    def n_coarse(self) -> int:
        return self.gc_h * self.gc_w

    @property
    def n_fine(self) -> int:
        return self.n_coarse * self.m * self.m

    @property
    def d_head(self) -> int:
        return self.d_model // self.n_heads

    @property
    def k_coarse(self) -> int:
        return 3 * self.patch_coarse * self.patch_coarse

    @property
    def k_fine(self) -> int:
        return 3 * self.patch_fine * self.patch_fine


TINY = ModelConfig(128, 128, 32, 16, 64, 2, 1, 256, 0)
C640 = ModelConfig(640, 640, 32, 16, 256, 8, 6, 1024, 5)

CONFIGS: Dict[str, ModelConfig] = {
    "tiny": TINY,
    "c640": C640,
    "batch6": C640,
    "fine8": C640,
    "multi48": C640,
}


@dataclasses.dataclass(frozen=True)
class Workload:
    """One BASELINE.json config: frames per coarse batch and k per refine task."""
    name: str
    model: ModelConfig
    ks: tuple  # refine count per task (== per frame)

    @property
    def n_tasks(self) -> int:
        return len(self.ks)


def ks_for_ratios(n_coarse: int, pcts: Sequence[int]) -> tuple:
    """k from a refine percentage: integer pct*Nc/100 (exact for every config)."""
    out = []
    for p in pcts:
        assert (p * n_coarse) % 100 == 0, (p, n_coarse)
        out.append(p * n_coarse // 100)
    return tuple(out)


def multi48_group_ks(group: int, frame: int = 0) -> tuple:
    """Ratios {0,0,25,40,60,100}% per group of 6, assignment permuted per (group, frame)."""
    base = ks_for_ratios(400, (0, 0, 25, 40, 60, 100))
    rng = np.random.default_rng(4800 + 97 * group + frame)
    perm = rng.permutation(6)
    return tuple(base[i] for i in perm)


WORKLOADS: Dict[str, Workload] = {
    "tiny": Workload("tiny", TINY, (4,)),
    "c640": Workload("c640", C640, (100,)),
    "batch6": Workload("batch6", C640, ks_for_ratios(400, (0, 20, 40, 60, 80, 100))),
    "fine8": Workload("fine8", C640, (400,) * 8),
    "multi48": Workload("multi48", C640, multi48_group_ks(0)),
}


# ----------------------------------------------------------------------------
# bf16 helpers (input quantisation only)
# ----------------------------------------------------------------------------
def bf16_bits(x: np.ndarray) -> np.ndarray:
    """float -> bf16 bit pattern (uint16), round-to-nearest-even."""
    f = np.ascontiguousarray(x, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    rnd = ((u >> 16) & 1) + 0x7FFF
    return ((u + rnd) >> 16).astype(np.uint16)


def bf16_from_bits(b: np.ndarray) -> np.ndarray:
    """bf16 bit pattern (uint16) -> exact float32 values."""
    return (np.asarray(b, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


def bf16_round(x: np.ndarray) -> np.ndarray:
    return bf16_from_bits(bf16_bits(x))


# ----------------------------------------------------------------------------
# frames
# ----------------------------------------------------------------------------
def frame_seed(task: int, frame: int) -> int:
    return 2505233 + 1000 * task + frame


def _scene(h: int, w: int, seed: int) -> np.ndarray:
    """fp64 [H, W, 3] scene in ~[0, 1] before normalisation (see make_frame)."""
    rng = np.random.default_rng(seed)
    t = np.linspace(0.0, 1.0, h, dtype=np.float64)[:, None]
    sky = np.array([0.55, 0.70, 0.95])
    road = np.array([0.35, 0.33, 0.30])
    img = np.empty((h, w, 3), dtype=np.float64)
    horizon = 0.45 + 0.1 * rng.random()
    for c in range(3):
        above = sky[c] * (1.0 - 0.4 * t / horizon)
        below = road[c] + 0.15 * (t - horizon)
        img[:, :, c] = np.where(t < horizon, above, below)
    n_obj = rng.poisson(8)
    for _ in range(n_obj):
        sw = int(round(math.exp(rng.uniform(math.log(8), math.log(192)))))
        sh = int(round(math.exp(rng.uniform(math.log(8), math.log(192)))))
        x0 = int(rng.integers(0, max(1, w - sw + 1)))
        y0 = int(rng.integers(0, max(1, h - sh + 1)))
        img[y0:y0 + sh, x0:x0 + sw, :] = rng.random(3)
    img += rng.normal(0.0, 0.05, size=img.shape)
    return img


def make_frame(h: int, w: int, seed: int, constant: bool = False) -> np.ndarray:
    """One synthetic camera frame, returned as bf16 bits [H, W, 3] (HWC, uint16).

    Sky-to-road vertical gradient + Poisson(8) axis-aligned rectangles of random
    colour with log-uniform side in [8, 192] px (some above the 16384 px^2
    critical size; many small, O2 PAPER.md:156), Gaussian noise
    sigma=0.05, per-channel normalisation to mean 0 / std 1, then bf16.
    `constant=True` returns an all-0.5 frame (used by the equal-score pin).
    """
    if constant:
        return bf16_bits(np.full((h, w, 3), 0.5, dtype=np.float32))
    img = _scene(h, w, seed)
    mu = img.mean(axis=(0, 1), keepdims=True)
    sd = img.std(axis=(0, 1), keepdims=True)
    img = (img - mu) / np.maximum(sd, 1e-6)
    return bf16_bits(img.astype(np.float32))


def make_frame_u8(h: int, w: int, seed: int) -> np.ndarray:
    """The same scene as make_frame(seed) as an 8-bit camera frame [H, W, 3] uint8
    (clip to [0, 1], x 255, round) -- the serving-path input of cfd_frames_from_u8."""
    return np.clip(np.rint(_scene(h, w, seed) * 255.0), 0, 255).astype(np.uint8)


def make_frames_u8(cfg: "ModelConfig", n: int, task0: int = 0, frame: int = 0) -> np.ndarray:
    """[n, H, W, 3] uint8; frame i uses seed(task0 + i, frame)."""
    return np.stack([make_frame_u8(cfg.img_h, cfg.img_w, frame_seed(task0 + i, frame)) for i in range(n)])


# per-channel ingest constants for 8-bit frames: (p/255 - mean_c) / std_c as one fp32 FMA,
# scale_c = 1 / (255 std_c), shift_c = -mean_c / std_c (ImageNet statistics, the usual DETR
# input normalisation), rounded once to fp32
U8_MEAN = (0.485, 0.456, 0.406)
U8_STD = (0.229, 0.224, 0.225)


def u8_affine(mean=U8_MEAN, std=U8_STD):
    """-> (scale[3], shift[3]) as float32 arrays."""
    m = np.asarray(mean, dtype=np.float64)
    s = np.asarray(std, dtype=np.float64)
    return (1.0 / (255.0 * s)).astype(np.float32), (-m / s).astype(np.float32)


def make_frames(cfg: ModelConfig, n: int, task0: int = 0, frame: int = 0) -> np.ndarray:
    """[n, H, W, 3] bf16 bits; frame i uses seed(task0 + i, frame)."""
    return np.stack([make_frame(cfg.img_h, cfg.img_w, frame_seed(task0 + i, frame))
                     for i in range(n)])


# ----------------------------------------------------------------------------
# parameters
# ----------------------------------------------------------------------------
def pe_table(n_rows: int, n_cols: int, patch: int, img_h: int, img_w: int, d: int) -> np.ndarray:
    """Fixed 2-D sin-cos table of patch centres, computed in fp64, stored fp32.

    Row r = (gy, gx) raster; centre (x, y) = (patch*gx + patch/2, patch*gy + patch/2);
    u = 2*pi*x/W, v = 2*pi*y/H, w_i = 10000^(-i/(d/4)), i < d/4;
    PE = [sin(u w) | cos(u w) | sin(v w) | cos(v w)].  (Reading R3.)
    """
    q = d // 4
    omega = 10000.0 ** (-np.arange(q, dtype=np.float64) / q)
    gy, gx = np.divmod(np.arange(n_rows * n_cols), n_cols)
    x = patch * gx + patch / 2.0
    y = patch * gy + patch / 2.0
    u = (2.0 * np.pi * x / img_w)[:, None] * omega[None, :]
    v = (2.0 * np.pi * y / img_h)[:, None] * omega[None, :]
    return np.concatenate([np.sin(u), np.cos(u), np.sin(v), np.cos(v)], axis=1).astype(np.float32)


def _xavier(rng, fan_in: int, fan_out: int, scale: float = 1.0) -> np.ndarray:
    bound = math.sqrt(6.0 / (fan_in + fan_out))
    w = rng.uniform(-bound, bound, size=(fan_in, fan_out)) * scale
    return bf16_round(w.astype(np.float32))


def make_decoder_weights(cfg: ModelConfig, n_queries: int = 128, seed: int = 1) -> dict:
    """Random-init NEXT-f3 decoder block (reading R24), layout (in, out): learned queries
    U(-1, 1) fp32 [Q, d]; LN gammas 1 + U(+-0.1), betas U(+-0.1); W_q [d, d], W_kv [d, 2d],
    W_o [d, d] (x0.5) xavier-uniform bf16-rounded; W_head [d, 5] xavier bf16-rounded (stored
    fp32); biases U(+-0.02)."""
    rng = np.random.default_rng(seed)
    d = cfg.d_model
    g = lambda: (1.0 + rng.uniform(-0.1, 0.1, size=d)).astype(np.float32)
    b = lambda n: rng.uniform(-0.02, 0.02, size=n).astype(np.float32)
    return {
        "queries": rng.uniform(-1.0, 1.0, size=(n_queries, d)).astype(np.float32),
        "ln_q_g": g(), "ln_q_b": rng.uniform(-0.1, 0.1, size=d).astype(np.float32),
        "ln_m_g": g(), "ln_m_b": rng.uniform(-0.1, 0.1, size=d).astype(np.float32),
        "w_q": _xavier(rng, d, d), "w_kv": _xavier(rng, d, 2 * d), "w_o": _xavier(rng, d, d, 0.5),
        "b_q": b(d), "b_kv": b(2 * d), "b_o": b(d),
        "w_head": _xavier(rng, d, 5), "b_head": b(5),
    }


def make_weights(cfg: ModelConfig, seed: int = 0, tied: bool = False, pe: bool = True) -> dict:
    """Random-init parameters, layout (in, out) for every matrix.

    Matrices are xavier-uniform and bf16-rounded (returned as exact float32
    values; `bf16_bits` gives the bytes the GPU receives); W_o and W_2 are
    scaled x0.5.  Biases U(-0.02, 0.02); LN gamma = 1 + U(-0.1, 0.1),
    beta = U(-0.1, 0.1).  `tied=True` sets W_c[(py,px,ch)] = W_f[(py%Pf,px%Pf,ch)]/m^2
    and b_c = b_f (reading R1: the paper's pooled coarse tokens); /m^2 is exact
    in bf16 for m a power of two.  `pe=False` zeroes both PE tables.
    """
    rng = np.random.default_rng(seed)
    d, F = cfg.d_model, cfg.d_ff
    w = {}
    w["w_embed_f"] = _xavier(rng, cfg.k_fine, d)
    w["b_embed_f"] = rng.uniform(-0.02, 0.02, size=d).astype(np.float32)
    if tied:
        Pc, Pf, m = cfg.patch_coarse, cfg.patch_fine, cfg.m
        py, px, ch = np.meshgrid(np.arange(Pc), np.arange(Pc), np.arange(3), indexing="ij")
        src = ((py % Pf) * Pf + (px % Pf)) * 3 + ch
        w["w_embed_c"] = (w["w_embed_f"][src.reshape(-1)] / float(m * m)).astype(np.float32)
        w["b_embed_c"] = w["b_embed_f"].copy()
        assert np.array_equal(bf16_round(w["w_embed_c"]), w["w_embed_c"])
    else:
        w["w_embed_c"] = _xavier(rng, cfg.k_coarse, d)
        w["b_embed_c"] = rng.uniform(-0.02, 0.02, size=d).astype(np.float32)
    if pe:
        w["pe_c"] = pe_table(cfg.gc_h, cfg.gc_w, cfg.patch_coarse, cfg.img_h, cfg.img_w, d)
        w["pe_f"] = pe_table(cfg.gc_h * cfg.m, cfg.gc_w * cfg.m, cfg.patch_fine, cfg.img_h, cfg.img_w, d)
    else:
        w["pe_c"] = np.zeros((cfg.n_coarse, d), np.float32)
        w["pe_f"] = np.zeros((cfg.n_fine, d), np.float32)
    layers: List[dict] = []
    for _ in range(cfg.n_layers):
        lw = {
            "w_qkv": _xavier(rng, d, 3 * d),
            "w_o": _xavier(rng, d, d, 0.5),
            "w_1": _xavier(rng, d, F),
            "w_2": _xavier(rng, F, d, 0.5),
            "b_qkv": rng.uniform(-0.02, 0.02, size=3 * d).astype(np.float32),
            "b_o": rng.uniform(-0.02, 0.02, size=d).astype(np.float32),
            "b_1": rng.uniform(-0.02, 0.02, size=F).astype(np.float32),
            "b_2": rng.uniform(-0.02, 0.02, size=d).astype(np.float32),
            "ln1_g": (1.0 + rng.uniform(-0.1, 0.1, size=d)).astype(np.float32),
            "ln1_b": rng.uniform(-0.1, 0.1, size=d).astype(np.float32),
            "ln2_g": (1.0 + rng.uniform(-0.1, 0.1, size=d)).astype(np.float32),
            "ln2_b": rng.uniform(-0.1, 0.1, size=d).astype(np.float32),
        }
        layers.append(lw)
    w["layers"] = layers
    return w


# ----------------------------------------------------------------------------
# coarse-stage detections (inputs of the NEXT rows f1/f2; no trained decoder here)
# ----------------------------------------------------------------------------
def make_queries(seed: int, n_queries: int = 128, hard: bool = True):
    """Synthetic per-query detections (cx, cy, w, h, c), boxes normalised, shaped like
    PAPER.md:225-227: a few high-confidence (c > 0.8) queries, intermediate ones
    (0.05 < c <= 0.8: ~20 on a hard frame, ~3 on an easy one) and background (c <= 0.05).
    Box sides log-uniform in [8, 192] px of a 640 px frame.  Returns (boxes [Q,4] fp32,
    conf [Q] fp32)."""
    rng = np.random.default_rng(seed)
    n_hi = 5
    n_mid = 20 if hard else 3
    conf = np.concatenate([rng.uniform(0.8001, 1.0, n_hi), rng.uniform(0.0501, 0.8, n_mid),
                           rng.uniform(0.0, 0.05, n_queries - n_hi - n_mid)])
    rng.shuffle(conf)
    side = np.exp(rng.uniform(np.log(8 / 640), np.log(192 / 640), size=(n_queries, 2)))
    ctr = rng.uniform(0.0, 1.0, size=(n_queries, 2))
    boxes = np.concatenate([ctr, side], axis=1)
    return boxes.astype(np.float32), conf.astype(np.float32)
