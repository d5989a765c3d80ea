"""Pins of the fp64 oracle against things other than itself (CPU only).

Each test names the oracle function it pins and what fixes the expected value:
an independent library implementation (torch), a closed form, an invariant the
paper implies, or brute force on tiny inputs.  See DESIGN.md §4.
"""
import itertools
import math

import numpy as np
import pytest
import torch

import cfd_inputs as ci
import oracle as O

TINY = ci.CONFIGS["tiny"]


def _rng(s=0):
    return np.random.default_rng(s)


# --------------------------------------------------------------------------- patchify
@pytest.mark.parametrize("P", [32, 16])
def test_patchify_matches_reshape_formulation(P):
    """patchify == an independent reshape/transpose formulation of the same tiling."""
    img = ci.make_frame(128, 96, 7)
    H, W, _ = img.shape
    ref = img.reshape(H // P, P, W // P, P, 3).transpose(0, 2, 1, 3, 4).reshape((H // P) * (W // P), -1)
    assert np.array_equal(O.patchify(img, P), ref)


def test_patchify_bijection_and_fine_tiles_cover_coarse():
    """Every pixel appears in exactly one coarse and one fine patch, and the m^2
    fine patches of region c cover exactly coarse patch c's pixels."""
    cfg = ci.ModelConfig(96, 160, 32, 16, 64, 2, 1, 256, 0)
    H, W = cfg.img_h, cfg.img_w
    coord = np.arange(H * W, dtype=np.int64).reshape(H, W)
    cimg = np.repeat(coord[:, :, None], 3, axis=2)
    pc = O.patchify(cimg, 32)
    pf = O.patchify(cimg, 16)
    assert sorted(np.unique(pc)) == list(range(H * W))
    assert np.bincount(pc.reshape(-1)).tolist() == [3] * (H * W)
    assert np.bincount(pf.reshape(-1)).tolist() == [3] * (H * W)
    for c in range(cfg.n_coarse):
        kids = [O.cfdetr_oracle._fine_index(cfg, c, dy, dx) for dy in range(2) for dx in range(2)]
        assert set(pc[c].tolist()) == set(np.concatenate([pf[f] for f in kids]).tolist())


def test_patch_vector_order_is_py_px_ch():
    img = ci.make_frame(64, 64, 3)
    p = O.patchify(img, 32)
    c = 1 * 2 + 1  # cy=1, cx=1
    py, px, ch = 5, 17, 2
    assert p[c, (py * 32 + px) * 3 + ch] == img[32 + py, 32 + px, ch]


# --------------------------------------------------------------------------- embedding
def test_tied_embedding_is_pooling_closed_form():
    """Tied mode (reading R1): coarse token (PE off) == mean of its m^2 fine tokens."""
    w = ci.make_weights(TINY, seed=3, tied=True, pe=False)
    img = O.as_f64_image(ci.make_frame(128, 128, 11))
    xc = O.patch_embed(O.patchify(img, 32), w["w_embed_c"], w["b_embed_c"], w["pe_c"])
    xf = O.patch_embed(O.patchify(img, 16), w["w_embed_f"], w["b_embed_f"], w["pe_f"])
    for c in range(TINY.n_coarse):
        kids = [O.cfdetr_oracle._fine_index(TINY, c, dy, dx) for dy in range(2) for dx in range(2)]
        np.testing.assert_allclose(xc[c], xf[kids].mean(axis=0), rtol=0, atol=1e-12)


def test_embed_matches_torch_linear():
    w = ci.make_weights(TINY, seed=1)
    img = O.as_f64_image(ci.make_frame(128, 128, 5))
    p = O.patchify(img, 32)
    x = O.patch_embed(p, w["w_embed_c"], w["b_embed_c"], w["pe_c"])
    ref = torch.nn.functional.linear(torch.tensor(p), torch.tensor(w["w_embed_c"], dtype=torch.float64).T,
                                     torch.tensor(w["b_embed_c"], dtype=torch.float64)) + torch.tensor(w["pe_c"], dtype=torch.float64)
    np.testing.assert_allclose(x, ref.numpy(), rtol=0, atol=1e-11)


def test_pe_table_values():
    """PE generator check (input-side): row 0 of the coarse table, column 0 = sin(2*pi*16/640)."""
    pe = ci.pe_table(20, 20, 32, 640, 640, 256)
    assert abs(pe[0, 0] - math.sin(2 * math.pi * 16 / 640)) < 1e-7
    assert abs(pe[21, 64 + 0] - math.cos(2 * math.pi * 48 / 640)) < 1e-7  # gx=1
    assert abs(pe[21, 128 + 0] - math.sin(2 * math.pi * 48 / 640)) < 1e-7  # gy=1


# --------------------------------------------------------------------------- LN / GELU
def test_layer_norm_matches_torch():
    x = _rng(1).normal(size=(7, 64)) * 3 + 1
    g, b = _rng(2).normal(size=64), _rng(3).normal(size=64)
    ref = torch.nn.functional.layer_norm(torch.tensor(x), (64,), torch.tensor(g), torch.tensor(b), eps=1e-6)
    np.testing.assert_allclose(O.layer_norm(x, g, b, 1e-6), ref.numpy(), rtol=0, atol=1e-12)


def test_gelu_matches_torch_and_closed_forms():
    z = np.linspace(-8, 8, 1001)
    ref = torch.nn.functional.gelu(torch.tensor(z), approximate="none").numpy()
    np.testing.assert_allclose(O.gelu(z), ref, rtol=0, atol=1e-14)
    assert O.gelu(np.array([0.0]))[0] == 0.0
    np.testing.assert_allclose(O.gelu(z) - O.gelu(-z), z, atol=1e-13)  # GELU(z) - GELU(-z) = z
    assert abs(O.gelu(np.array([1.0]))[0] - 0.8413447460685429) < 1e-15  # Phi(1)


# --------------------------------------------------------------------------- encoder block
def _torch_layer(lw, d, nh, F):
    layer = torch.nn.TransformerEncoderLayer(d, nh, F, dropout=0.0, activation="gelu", layer_norm_eps=1e-6,
                                             batch_first=True, norm_first=True, dtype=torch.float64)
    t = lambda a: torch.tensor(np.asarray(a, dtype=np.float64))
    with torch.no_grad():
        layer.self_attn.in_proj_weight.copy_(t(lw["w_qkv"]).T)
        layer.self_attn.in_proj_bias.copy_(t(lw["b_qkv"]))
        layer.self_attn.out_proj.weight.copy_(t(lw["w_o"]).T)
        layer.self_attn.out_proj.bias.copy_(t(lw["b_o"]))
        layer.linear1.weight.copy_(t(lw["w_1"]).T)
        layer.linear1.bias.copy_(t(lw["b_1"]))
        layer.linear2.weight.copy_(t(lw["w_2"]).T)
        layer.linear2.bias.copy_(t(lw["b_2"]))
        layer.norm1.weight.copy_(t(lw["ln1_g"]))
        layer.norm1.bias.copy_(t(lw["ln1_b"]))
        layer.norm2.weight.copy_(t(lw["ln2_g"]))
        layer.norm2.bias.copy_(t(lw["ln2_b"]))
    return layer.eval()


@pytest.mark.parametrize("d,nh,N", [(64, 2, 28), (256, 8, 57)])
def test_encoder_layer_matches_torch_transformer_layer(d, nh, N):
    """The whole pre-LN block against torch.nn.TransformerEncoderLayer(norm_first, gelu) in fp64."""
    cfg = ci.ModelConfig(64, 64, 32, 16, d, nh, 2, 4 * d, 1)
    w = ci.make_weights(cfg, seed=4)
    x = _rng(5).normal(size=(N, d))
    y = x
    for lw in w["layers"]:
        y, _ = O.encoder_layer(y, lw, nh, 1e-6)
        ref = _torch_layer(lw, d, nh, 4 * d)
    with torch.no_grad():
        r = torch.tensor(x)[None]
        for lw in w["layers"]:
            r = _torch_layer(lw, d, nh, 4 * d)(r)
    np.testing.assert_allclose(y, r[0].numpy(), rtol=0, atol=1e-10)


def test_attention_probs_and_score_match_torch_mha():
    """P_h and the head-averaged column mean (criticality score) against torch MHA weights."""
    d, nh, N = 64, 2, 16
    cfg = ci.ModelConfig(64, 64, 32, 16, d, nh, 1, 4 * d, 0)
    lw = ci.make_weights(cfg, seed=8)["layers"][0]
    x = _rng(9).normal(size=(N, d))
    _, probs = O.encoder_layer(x, lw, nh, 1e-6, want_probs=True)
    layer = _torch_layer(lw, d, nh, 4 * d)
    with torch.no_grad():
        h = layer.norm1(torch.tensor(x))[None]
        _, wts = layer.self_attn(h, h, h, need_weights=True, average_attn_weights=False)
        _, avg = layer.self_attn(h, h, h, need_weights=True, average_attn_weights=True)
    for hh in range(nh):
        np.testing.assert_allclose(probs[hh], wts[0, hh].numpy(), rtol=0, atol=1e-13)
    np.testing.assert_allclose(O.criticality_score(probs), avg[0].numpy().mean(axis=0), rtol=0, atol=1e-14)


def test_attention_closed_forms():
    rng = _rng(10)
    q, k = rng.normal(size=(9, 32)), rng.normal(size=(9, 32))
    P = O.attention_probs(q, k)
    np.testing.assert_allclose(P.sum(axis=1), 1.0, atol=1e-14)          # rows sum to 1
    P1 = O.attention_probs(q, np.repeat(k[:1], 9, axis=0))
    np.testing.assert_allclose(P1, 1.0 / 9, atol=1e-15)                 # identical keys -> uniform
    assert O.attention_probs(q[:1], k[:1])[0, 0] == 1.0                 # one token -> P = 1


def test_single_token_attention_output_is_v():
    """N=1: attention output = v, so the block = x + (v W_o + b_o) + MLP (explicit closed form)."""
    d, nh = 64, 2
    cfg = ci.ModelConfig(64, 64, 32, 16, d, nh, 1, 4 * d, 0)
    lw = ci.make_weights(cfg, seed=12)["layers"][0]
    x = _rng(13).normal(size=(1, d))
    y, _ = O.encoder_layer(x, lw, nh, 1e-6)
    mu, sd = x.mean(), x.std()
    h = (x - mu) / math.sqrt(sd * sd + 1e-6) * lw["ln1_g"] + lw["ln1_b"]
    v = h @ lw["w_qkv"][:, 2 * d:] + lw["b_qkv"][2 * d:]
    x1 = x + v @ lw["w_o"] + lw["b_o"]
    mu2, sd2 = x1.mean(), x1.std()
    h2 = (x1 - mu2) / math.sqrt(sd2 * sd2 + 1e-6) * lw["ln2_g"] + lw["ln2_b"]
    z = h2 @ lw["w_1"] + lw["b_1"]
    ref = x1 + (0.5 * z * (1 + torch.erf(torch.tensor(z) / math.sqrt(2)).numpy())) @ lw["w_2"] + lw["b_2"]
    np.testing.assert_allclose(y, ref, rtol=0, atol=1e-12)


def _torch_stack_with_hooks(layers, d, nh, score_layer):
    """torch.nn.TransformerEncoder(num_layers=L, norm_first, gelu) in fp64 with the given
    per-layer weights; returns a closure x -> (y, [per-layer outputs], score column means at
    `score_layer`) where the per-layer outputs come from forward hooks on encoder.layers[l]
    and the score from the head-averaged attention weights of encoder.layers[score_layer]
    (torch MHA need_weights on the LN1 output that layer's self-attention receives)."""
    L = len(layers)
    proto = torch.nn.TransformerEncoderLayer(d, nh, 4 * d, dropout=0.0, activation="gelu", layer_norm_eps=1e-6,
                                             batch_first=True, norm_first=True, dtype=torch.float64)
    stack = torch.nn.TransformerEncoder(proto, num_layers=L, enable_nested_tensor=False)
    for l, lw in enumerate(layers):
        src = _torch_layer(lw, d, nh, 4 * d)
        stack.layers[l].load_state_dict(src.state_dict())
    stack.eval()
    outs, attn_in = [], []
    for l in range(L):
        stack.layers[l].register_forward_hook(lambda m, a, o: outs.append(o.detach()[0].numpy().copy()))
    stack.layers[score_layer].self_attn.register_forward_pre_hook(lambda m, a: attn_in.append(a[0].detach()))

    def run(x):
        outs.clear()
        attn_in.clear()
        # grad enabled (no torch.no_grad) keeps torch off its fused inference fast path, so
        # the module hooks fire on the plain layer code
        y = stack(torch.tensor(x)[None]).detach()[0].numpy()
        h = attn_in[0]
        _, avg = stack.layers[score_layer].self_attn(h, h, h, need_weights=True, average_attn_weights=True)
        return y, list(outs), avg.detach()[0].numpy().mean(axis=0)
    return run


@pytest.mark.parametrize("d,nh,N,score_layer", [(64, 2, 21, 5), (64, 2, 21, 2), (256, 8, 40, 5)])
def test_encoder_L6_matches_torch_transformer_encoder(d, nh, N, score_layer):
    """O.encoder at L = 6 (§V-A "six encoder/decoder layers"; the stack of global
    self-attention blocks of PAPER.md:120-122 §II-A) against torch.nn.TransformerEncoder with
    the same six distinct weight sets: every per-layer output (so the layer ORDER is pinned:
    the blocks do not commute) and the criticality score taken from the attention map of layer
    `score_layer` (so probs_at is pinned: a different layer's map gives a different score)."""
    cfg = ci.ModelConfig(64, 64, 32, 16, d, nh, 6, 4 * d, score_layer)
    w = ci.make_weights(cfg, seed=17)
    x = _rng(18).normal(size=(N, d))
    y, outs, probs = O.encoder(x, w["layers"], nh, 1e-6, probs_at=score_layer)
    yr, outs_r, s_r = _torch_stack_with_hooks(w["layers"], d, nh, score_layer)(x)
    assert len(outs) == len(outs_r) == 6
    for l in range(6):
        np.testing.assert_allclose(outs[l], outs_r[l], rtol=0, atol=1e-10, err_msg=f"layer {l}")
    np.testing.assert_allclose(y, yr, rtol=0, atol=1e-10)
    assert len(probs) == nh
    np.testing.assert_allclose(O.criticality_score(probs), s_r, rtol=0, atol=1e-13)


def test_coarse_encode_L6_scores_come_from_the_configured_score_layer():
    """O.coarse_encode end to end at L = 6: its per-layer outputs and scores against the torch
    stack fed the (separately pinned) patch embedding, for score_layer = L-1 (reading R15) and
    for another layer, so a coarse_encode that ignored cfg.score_layer fails one of them."""
    for sl in (5, 1):
        cfg = ci.ModelConfig(128, 128, 32, 16, 64, 2, 6, 256, sl)
        w = ci.make_weights(cfg, seed=19)
        img = ci.make_frame(128, 128, 23)
        out = O.coarse_encode(cfg, w, [img])[0]
        x0 = O.patch_embed(O.patchify(O.as_f64_image(img), 32), w["w_embed_c"], w["b_embed_c"], w["pe_c"])
        yr, outs_r, s_r = _torch_stack_with_hooks(w["layers"], 64, 2, sl)(x0)
        for l in range(6):
            np.testing.assert_allclose(out["layers"][l], outs_r[l], rtol=0, atol=1e-10)
        np.testing.assert_allclose(out["scores"], s_r, rtol=0, atol=1e-13)


def test_encoder_permutation_equivariance():
    d, nh = 64, 2
    cfg = ci.ModelConfig(64, 64, 32, 16, d, nh, 2, 4 * d, 1)
    w = ci.make_weights(cfg, seed=14)
    x = _rng(15).normal(size=(21, d))
    perm = _rng(16).permutation(21)
    y, _, _ = O.encoder(x, w["layers"], nh, 1e-6)
    yp, _, _ = O.encoder(x[perm], w["layers"], nh, 1e-6)
    np.testing.assert_allclose(yp, y[perm], rtol=0, atol=1e-12)


# --------------------------------------------------------------------------- score
def test_score_is_a_distribution():
    w = ci.make_weights(TINY, seed=0)
    out = O.coarse_encode(TINY, w, [ci.make_frame(128, 128, 21)])[0]
    s = out["scores"]
    assert (s >= 0).all()
    assert abs(s.sum() - 1.0) < 1e-13


def test_constant_image_gives_equal_scores_and_lowest_index_topk():
    """Constant image, PE off -> all coarse tokens identical -> s_j = 1/Nc -> top-k = {0..k-1}."""
    w = ci.make_weights(TINY, seed=0, pe=False)
    img = ci.make_frame(128, 128, 0, constant=True)
    s = O.coarse_encode(TINY, w, [img])[0]["scores"]
    np.testing.assert_allclose(s, 1.0 / TINY.n_coarse, rtol=0, atol=1e-15)
    s32 = np.full(16, np.float32(1.0 / 16))
    assert O.select_topk(s32, 4).tolist() == [0, 1, 2, 3]


# --------------------------------------------------------------------------- selection
def _brute_topk(s, k):
    """Smallest (lexicographic) index set among all k-subsets whose every member
    ranks at or above every non-member (NaN ranks below everything)."""
    rank_val = lambda x: (0, 0.0) if np.isnan(x) else (1, float(x))
    best = None
    for sub in itertools.combinations(range(len(s)), k):
        inside = [rank_val(s[j]) for j in sub]
        outside = [rank_val(s[j]) for j in range(len(s)) if j not in sub]
        if not outside or not inside or min(inside) >= max(outside):
            if best is None or sub < best:
                best = sub
    return list(best)


@pytest.mark.parametrize("case", range(12))
def test_topk_brute_force(case):
    rng = _rng(100 + case)
    if case < 4:
        s = rng.random(16).astype(np.float32)
    elif case < 8:
        s = rng.choice(np.array([0.1, 0.2, 0.3], np.float32), size=16)  # many ties
    else:
        s = rng.choice(np.array([0.0, -0.0, 1.0, -1.0, np.inf, -np.inf, np.nan, 0.5], np.float32), size=16)
    for k in (0, 1, 4, 15, 16):
        assert O.select_topk(s, k).tolist() == _brute_topk(s, k), (s, k)


def test_topk_signed_zero_and_nan_rules():
    s = np.array([-0.0, 0.0, np.nan, -np.inf], np.float32)
    assert O.select_topk(s, 1).tolist() == [0]          # -0 == +0, lower index wins
    assert O.select_topk(s, 3).tolist() == [0, 1, 3]    # NaN below -inf


def test_threshold_count():
    rng = _rng(7)
    s = rng.random(400).astype(np.float32)
    for tau in (0.0, 0.25, 0.5, 0.999, 1.0):
        sel = O.select_threshold(s, np.float32(tau))
        assert len(sel) == int((s > np.float32(tau)).sum())
        assert (np.diff(sel) > 0).all()


def test_threshold_is_strict_at_ties():
    """Reading R7 ("exceeds", PAPER.md:454 [draft]): s == tau is NOT selected.  Hand-written
    expected index sets (not recomputed from a formula) on vectors that hit tau exactly,
    including -0 == +0, NaN (never selected) and +-inf."""
    f = np.float32
    s = np.array([0.1, 0.5, 0.5, 0.7, np.nan, -0.0, 0.0, np.inf, -np.inf, 0.5000001], f)
    assert O.select_threshold(s, f(0.5)).tolist() == [3, 7, 9]
    assert O.select_threshold(s, f(0.0)).tolist() == [0, 1, 2, 3, 7, 9]
    assert O.select_threshold(s, f(-0.0)).tolist() == [0, 1, 2, 3, 7, 9]
    assert O.select_threshold(s, np.nextafter(f(0.5), f(0))).tolist() == [1, 2, 3, 7, 9]
    assert O.select_threshold(s, f(np.inf)).tolist() == []
    assert O.select_threshold(s, f(-np.inf)).tolist() == [0, 1, 2, 3, 5, 6, 7, 9]
    eq = np.full(16, f(1 / 16))
    assert O.select_threshold(eq, f(1 / 16)).tolist() == []                       # all tied at tau
    assert O.select_threshold(eq, np.nextafter(f(1 / 16), f(0))).tolist() == list(range(16))


# --------------------------------------------------------------------------- merge / layout
def test_gather_layout_closed_forms():
    cfg = TINY
    rng = _rng(3)
    sels = [np.sort(rng.choice(16, size=k, replace=False)) for k in (0, 4, 16, 7)]
    imgs = [ci.make_frame(128, 128, 40 + t) for t in range(4)]
    cu, msrc, frow, fidx, af = O.gather_layout(cfg, sels, imgs)
    m2 = cfg.m * cfg.m
    assert np.diff(cu).tolist() == [cfg.n_coarse + (m2 - 1) * len(s) for s in sels]
    for t, sel in enumerate(sels):
        seq = msrc[cu[t]:cu[t + 1]]
        for c in range(cfg.n_coarse):
            off = c + (m2 - 1) * int((sel < c).sum())          # off[c] closed form
            if c in sel:
                cy, cx = divmod(c, cfg.gc_w)
                f0 = (2 * cy) * cfg.gf_w + 2 * cx
                assert seq[off] == -1 - f0
            else:
                assert seq[off] == c
    assert len(frow) == len(fidx) == af.shape[0] == m2 * sum(len(s) for s in sels)
    assert (msrc[frow] == -1 - fidx).all()


def test_gather_layout_af_rows_are_the_fine_patch_pixels():
    """A_f row r holds exactly the pixel bytes of fine patch fidx[r] of its own task's frame,
    against an independent reshape/transpose tiling of the frame (not O.patchify); frow is
    strictly increasing (fine tokens in packed order) and the m^2 rows of one selected region
    reassemble that region's coarse patch byte for byte."""
    cfg = TINY
    rng = _rng(4)
    sels = [np.sort(rng.choice(16, size=k, replace=False)) for k in (3, 0, 16, 5)]
    imgs = [ci.make_frame(128, 128, 70 + t) for t in range(4)]
    cu, msrc, frow, fidx, af = O.gather_layout(cfg, sels, imgs)
    P, H, W, m = 16, 128, 128, cfg.m

    def tiles(img, p):
        return img.reshape(H // p, p, W // p, p, 3).transpose(0, 2, 1, 3, 4).reshape((H // p) * (W // p), -1)

    assert (np.diff(frow) > 0).all()
    task = np.searchsorted(cu, frow, side="right") - 1
    for r in range(len(frow)):
        assert np.array_equal(af[r], tiles(imgs[task[r]], P)[fidx[r]]), r
    r = 0
    for t, sel in enumerate(sels):
        for c in sel:
            rows = af[r:r + m * m].reshape(m, m, P, P, 3)           # (dy, dx, py, px, ch)
            patch = rows.transpose(0, 2, 1, 3, 4).reshape(32 * 32 * 3)
            assert np.array_equal(patch, tiles(imgs[t], 32)[c])
            r += m * m
    assert r == len(frow)


def test_refine_k0_equals_coarse_pass():
    """Refining zero regions reproduces the coarse pass exactly (PAPER.md:234 reuse; A1 easy frames)."""
    w = ci.make_weights(TINY, seed=0)
    img = ci.make_frame(128, 128, 50)
    c = O.coarse_encode(TINY, w, [img])[0]
    r = O.refine_encode(TINY, w, img, c["x0"], [])
    assert np.array_equal(r["y"], c["y"])
    assert r["mixed_src"].tolist() == list(range(16))


def test_refine_all_regions_equals_fine_pass():
    """Refining every region reproduces the full fine pass up to the region-major permutation."""
    w = ci.make_weights(TINY, seed=0)
    img = ci.make_frame(128, 128, 51)
    c = O.coarse_encode(TINY, w, [img])[0]
    r = O.refine_encode(TINY, w, img, c["x0"], list(range(16)))
    f = O.fine_pass(TINY, w, img)
    order = -1 - r["mixed_src"]
    assert sorted(order.tolist()) == list(range(64))
    np.testing.assert_allclose(r["y"], f["y"][order], rtol=0, atol=1e-11)


def test_batch_refine_equals_per_task_refine():
    w = ci.make_weights(TINY, seed=0)
    imgs = [ci.make_frame(128, 128, 60 + t) for t in range(3)]
    cs = O.coarse_encode(TINY, w, imgs)
    sels = [O.select_topk(c["scores"].astype(np.float32), k) for c, k in zip(cs, (0, 4, 9))]
    b = O.batch_refine(TINY, w, imgs, [c["x0"] for c in cs], sels)
    assert np.diff(b["cu_seqlens"]).tolist() == [16, 28, 43]
    for t in range(3):
        r = O.refine_encode(TINY, w, imgs[t], cs[t]["x0"], sels[t])
        assert np.array_equal(b["y"][b["cu_seqlens"][t]:b["cu_seqlens"][t + 1]], r["y"])


def test_bf16_rounding_helper():
    x = np.array([1.0, 1.00390625, 1.005859375, -2.5, 3.0e-3], np.float32)
    # 1+2^-8 ties to even -> 1.0; 1+1.5*2^-8 rounds up to 1+2^-7
    assert ci.bf16_round(x)[:4].tolist() == [1.0, 1.0, 1.0078125, -2.5]
    assert ci.bf16_round(ci.bf16_round(x)).tolist() == ci.bf16_round(x).tolist()


# --------------------------------------------------------------------------- NEXT rows f1 / f2
def test_hardness_gate_against_vectorised_mean_and_special_cases():
    rng = _rng(31)
    for t in range(50):
        conf = rng.random(128).astype(np.float32) * (0.2 if t % 2 else 1.0)
        keep = conf[conf <= np.float32(0.8)].astype(np.float64)
        ref = 0 if keep.size == 0 else int(keep.mean() >= 0.05)
        if keep.size and abs(keep.mean() - 0.05) < 1e-12:
            continue
        assert O.hardness_gate(conf) == ref
    assert O.hardness_gate(np.full(10, 0.9, np.float32)) == 0          # only critical objects -> easy
    assert O.hardness_gate(np.array([0.95, 0.3], np.float32)) == 1      # one ambiguous query -> hard
    assert O.hardness_gate(np.array([0.01, 0.02, 0.9], np.float32)) == 0  # background only -> easy


def test_box_cell_scores_against_pixel_mask_rasterisation():
    cfg = ci.ModelConfig(128, 160, 32, 16, 64, 2, 1, 256, 0)
    boxes, conf = ci.make_queries(7, 40, hard=True)
    s = O.box_cell_scores(cfg, boxes, conf)
    mask_count = np.zeros((cfg.img_h, cfg.img_w), np.int64)
    for b, c in zip(boxes, conf):
        if 0.05 < float(c) <= 0.8:
            x0, x1, y0, y1 = O.box_pixel_rect(b, cfg.img_h, cfg.img_w)
            m = np.zeros_like(mask_count)
            m[y0:y1, x0:x1] = 1
            mask_count += m
    ref = mask_count.reshape(cfg.gc_h, 32, cfg.gc_w, 32).sum(axis=(1, 3)).reshape(-1)
    assert np.array_equal(s.astype(np.int64), ref)


def test_box_cell_scores_closed_forms():
    cfg = ci.ModelConfig(128, 128, 32, 16, 64, 2, 1, 256, 0)
    full = np.array([[0.5, 0.5, 1.0, 1.0]], np.float32)
    assert (O.box_cell_scores(cfg, full, np.array([0.5], np.float32)) == 32 * 32).all()
    assert (O.box_cell_scores(cfg, full, np.array([0.9], np.float32)) == 0).all()    # critical: not refined
    inner = np.array([[40 / 128, 40 / 128, 8 / 128, 8 / 128]], np.float32)           # pixels [36,44)^2 in cell (1,1)
    s = O.box_cell_scores(cfg, inner, np.array([0.3], np.float32))
    assert s[1 * 4 + 1] == 64 and s.sum() == 64


# ------------------------------------------------------------------ NEXT f3 decoder
def _torch_decode(wd, y, n_heads, eps):
    """Reference from library routines: torch nn.MultiheadAttention (cross-attention, fp64,
    in_proj = [W_q | W_k | W_v]^T) on F.layer_norm'd queries / memory, + residual, + heads."""
    F = torch.nn.functional
    t = lambda a: torch.as_tensor(np.asarray(a, np.float64))
    Q0, Y = t(wd["queries"]), t(y)
    d = Q0.shape[1]
    mha = torch.nn.MultiheadAttention(d, n_heads, batch_first=True, dtype=torch.float64)
    with torch.no_grad():
        wkv = t(wd["w_kv"])
        mha.in_proj_weight.copy_(torch.cat([t(wd["w_q"]), wkv[:, :d], wkv[:, d:]], dim=1).T)
        mha.in_proj_bias.copy_(torch.cat([t(wd["b_q"]), t(wd["b_kv"])]))
        mha.out_proj.weight.copy_(t(wd["w_o"]).T)
        mha.out_proj.bias.copy_(t(wd["b_o"]))
        hq = F.layer_norm(Q0, (d,), t(wd["ln_q_g"]), t(wd["ln_q_b"]), eps)
        hm = F.layer_norm(Y, (d,), t(wd["ln_m_g"]), t(wd["ln_m_b"]), eps)
        o, _ = mha(hq[None], hm[None], hm[None], need_weights=False)
        z = Q0 + o[0]
        out = torch.sigmoid(z @ t(wd["w_head"]) + t(wd["b_head"]))
    return z.numpy(), out[:, :4].numpy(), out[:, 4].numpy()


@pytest.mark.parametrize("N,Q,d,nh", [(28, 16, 64, 2), (400, 128, 256, 8), (1, 8, 64, 2)])
def test_decode_matches_torch_multihead_cross_attention(N, Q, d, nh):
    cfg = ci.ModelConfig(128, 128, 32, 16, d, nh, 1, 4 * d, 0)
    wd = ci.make_decoder_weights(cfg, Q, seed=N)
    y = np.random.default_rng(N).normal(size=(N, d))
    z, box, conf = O.decode(wd, y, nh, 1e-6)
    zr, br, cr = _torch_decode(wd, y, nh, 1e-6)
    np.testing.assert_allclose(z, zr, rtol=0, atol=1e-10)
    np.testing.assert_allclose(box, br, rtol=0, atol=1e-12)
    np.testing.assert_allclose(conf, cr, rtol=0, atol=1e-12)
    assert ((box > 0) & (box < 1)).all() and ((conf > 0) & (conf < 1)).all()


def test_decode_closed_forms():
    """One memory token: every query's attention output is that token's v, so
    z - Q0 is the same row for all queries.  Identical memory tokens: the same (uniform
    attention over equal values)."""
    cfg = ci.ModelConfig(128, 128, 32, 16, 64, 2, 1, 256, 0)
    wd = ci.make_decoder_weights(cfg, 12, seed=5)
    Q0 = wd["queries"].astype(np.float64)
    row = np.random.default_rng(1).normal(size=(1, 64))
    z1, _, _ = O.decode(wd, row, 2, 1e-6)
    zk, _, _ = O.decode(wd, np.repeat(row, 7, axis=0), 2, 1e-6)
    delta = z1 - Q0
    assert np.allclose(delta, delta[0], atol=1e-12, rtol=0)
    np.testing.assert_allclose(zk, z1, atol=1e-12, rtol=0)


# ---------------------------------------------------------------------------- frame ingest
def test_round_to_float_matches_numpy_fp32_and_torch_bf16():
    """The oracle's exact rounding helper against library conversions (RNE, subnormals)."""
    from fractions import Fraction
    import torch
    rng = np.random.default_rng(5)
    xs = np.concatenate([rng.normal(0, 1, 2000), rng.normal(0, 1, 200) * 1e-39, rng.normal(0, 1, 200) * 1e30,
                         [0.0, 1.0, -1.0, 2.0 ** -149, 3 * 2.0 ** -150]])
    for x in xs:
        assert float(O.round_to_float(Fraction(float(x)), 24)) == float(np.float32(x)), x
    f32 = rng.normal(0, 10, 3000).astype(np.float32)
    bf = torch.from_numpy(f32).bfloat16().float().numpy()
    for x, y in zip(f32, bf):
        assert float(O.round_to_float(Fraction(float(x)), 8)) == float(y), x


def test_frames_from_u8_against_library_conversions():
    """Where p*scale+shift is exact in fp64, fp64 -> fp32 -> bf16 by torch must agree."""
    from fractions import Fraction
    import torch
    sc, sh = ci.u8_affine()
    src = np.repeat(np.arange(256, dtype=np.uint8), 3).reshape(256, 3)
    v64 = src.astype(np.float64) * sc.astype(np.float64) + sh.astype(np.float64)
    for p in range(256):
        for c in range(3):
            assert Fraction(p) * Fraction(float(sc[c])) + Fraction(float(sh[c])) == Fraction(v64[p, c])
    ref = torch.from_numpy(v64).float().bfloat16().view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(O.frames_from_u8(src, sc, sh), ref)


def test_frames_from_u8_closed_forms():
    one, zero = np.ones(3, np.float32), np.zeros(3, np.float32)
    src = np.repeat(np.arange(256, dtype=np.uint8), 3).reshape(256, 3)
    # identity: integers <= 256 are exact in bf16
    ident = O.frames_from_u8(src, one, zero)
    assert np.array_equal(ident, (np.arange(256, dtype=np.float32).view(np.uint32) >> 16).astype(np.uint16)[:, None]
                          .repeat(3, 1))
    bits = lambda v: np.uint16(np.float32(v).view(np.uint32) >> 16)  # noqa: E731
    # ties to even in [256, 512) (bf16 spacing 2): 257 -> 256, 259 -> 260; channel = index mod 3
    out = O.frames_from_u8(np.array([[255, 255, 253]], np.uint8), one, np.array([2.0, 4.0, 2.0], np.float32))
    assert list(out[0]) == [bits(256.0), bits(260.0), bits(255.0)]
    # fp32 first: 257 + 2^-20 rounds to 257 in fp32 (ulp 2^-15), then ties to 256 -- a direct
    # bf16 rounding of the exact value would give 258
    out = O.frames_from_u8(np.array([[255, 0, 0]], np.uint8), one, np.array([2.0 + 2.0 ** -20, 0.0, 0.0], np.float32))
    assert out[0, 0] == bits(256.0)
    # p = 0 gives bf16(shift); a negative scale flips the sign
    out = O.frames_from_u8(np.array([[0, 10, 0]], np.uint8), np.array([1, -1, 1], np.float32),
                           np.array([-0.5, 0.0, 3.0], np.float32))
    assert list(out[0]) == [bits(-0.5), bits(-10.0), bits(3.0)]
