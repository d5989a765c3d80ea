"""NEXT rows on the GPU, bit-exact against the oracle:
f2 the A1 hardness gate and f1 box-driven region proposal."""
import numpy as np
import pytest
import torch

import cfd_inputs as ci
import oracle as O

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)

from paper_2505_23317_b200.api import CFDetrEncoder  # noqa: E402


@pytest.fixture(scope="module")
def enc():
    cfg = ci.CONFIGS["c640"]
    return CFDetrEncoder(cfg, ci.make_weights(cfg, seed=0), max_tasks=64)


def _queries(B, Q, seed):
    bx, cf = zip(*[ci.make_queries(seed + b, Q, hard=(b % 3 != 0)) for b in range(B)])
    return np.stack(bx), np.stack(cf)


def test_hardness_gate_bit_exact(enc):
    boxes, conf = _queries(48, 128, 100)
    conf[5, :] = 0.9            # only critical objects -> easy
    conf[6, :] = 0.01           # background only -> easy
    conf[7, :] = 0.01
    conf[7, 3] = 0.9
    conf[7, 4] = 0.5            # one ambiguous query -> hard
    hard = enc.hardness(torch.from_numpy(conf).cuda())
    torch.cuda.synchronize()
    ref = [O.hardness_gate(conf[b]) for b in range(48)]
    assert hard.cpu().tolist() == ref
    assert 0 in ref and 1 in ref


def test_box_scores_bit_exact_and_threshold_selection(enc):
    cfg = ci.CONFIGS["c640"]
    boxes, conf = _queries(12, 128, 200)
    boxes[0, 0] = [0.5, 0.5, 1.0, 1.0]      # full-frame box
    conf[0, 0] = 0.5
    d_boxes = torch.from_numpy(boxes).cuda()
    s = enc.box_scores(d_boxes, torch.from_numpy(conf).cuda())
    sel = enc.select_regions(s, threshold=0.0)
    torch.cuda.synchronize()
    for b in range(12):
        ref = O.box_cell_scores(cfg, boxes[b], conf[b])
        assert np.array_equal(s[b].cpu().numpy().astype(np.float64), ref), b
        rsel = O.select_threshold(ref.astype(np.float32), np.float32(0.0))
        n = int(sel["sel_count"][b])
        assert n == len(rsel) and np.array_equal(sel["sel_idx"][b, :n].cpu().numpy(), rsel)
    assert int(sel["sel_count"][0]) == cfg.n_coarse   # the full-frame box touches every cell


def test_gate_then_box_regions_then_refine(enc):
    """The NEXT rows feeding the hot path: easy frames refine nothing (k=0), hard frames
    refine the cells their intermediate boxes touch; checked against the oracle."""
    cfg = ci.CONFIGS["c640"]
    w = ci.make_weights(cfg, seed=0)
    B = 3
    boxes, conf = _queries(B, 128, 300)
    imgs = ci.make_frames(cfg, B, task0=40)
    from paper_2505_23317_b200.api import bf16_tensor
    dimg = bf16_tensor(imgs, "cuda")
    co = enc.coarse_encode(dimg)
    hard = enc.hardness(torch.from_numpy(conf).cuda())
    s = enc.box_scores(torch.from_numpy(boxes).cuda(), torch.from_numpy(conf).cuda())
    s = s * hard[:, None].float()          # easy frames: no region scores above 0
    sel = enc.select_regions(s, threshold=0.0)
    ro = enc.batch_refine(dimg, co["x0"], sel["sel_idx"], sel["sel_count"])
    torch.cuda.synchronize()
    cu = ro["cu_seqlens"].cpu().numpy()
    for b in range(B):
        hb = O.hardness_gate(conf[b])
        ref_sel = O.select_threshold((O.box_cell_scores(cfg, boxes[b], conf[b]) * hb).astype(np.float32),
                                     np.float32(0.0))
        oc = O.coarse_encode(cfg, w, [imgs[b]])[0]
        rr = O.refine_encode(cfg, w, imgs[b], oc["x0"], ref_sel)
        y = ro["y"][cu[b]:cu[b + 1]].double().cpu().numpy()
        assert y.shape == rr["y"].shape
        rel = np.linalg.norm(y - rr["y"]) / np.linalg.norm(rr["y"])
        assert rel <= 2e-2 and np.abs(y - rr["y"]).max() <= 5e-2


# ------------------------------------------------------------------ f3 decoder (reading R24)
def _check_decode(cfg, ws_seed, Q, frames, ks):
    from paper_2505_23317_b200.api import bf16_tensor
    w = ci.make_weights(cfg, seed=0)
    wd = ci.make_decoder_weights(cfg, Q, seed=ws_seed)
    e = CFDetrEncoder(cfg, w, max_tasks=max(8, len(ks)))
    e.set_decoder(wd)
    imgs = bf16_tensor(ci.make_frames(cfg, len(ks), task0=frames), "cuda")
    co = e.coarse_encode(imgs)
    sel = e.select_regions(co["scores"], k=ks)
    ro = e.batch_refine(imgs, co["x0"], sel["sel_idx"], sel["sel_count"])
    cu = ro["cu_seqlens"]
    n = int(cu[-1])
    dec = e.decode(ro["y"], cu, len(ks), n)
    # the coarse output decodes too (cu = [0, Nc, 2Nc, ...])
    ccu = torch.arange(len(ks) + 1, dtype=torch.int32, device="cuda") * e.Nc
    dec_c = e.decode(co["y"].reshape(-1, cfg.d_model), ccu, len(ks), len(ks) * e.Nc)
    torch.cuda.synchronize()
    cu_h = cu.cpu().numpy()
    for t in range(len(ks)):
        # shared-input protocol: the oracle decodes the GPU's encoder output
        for y_t, got in ((ro["y"][cu_h[t]:cu_h[t + 1]], dec), (co["y"][t], dec_c)):
            z, box, conf = O.decode(wd, y_t.double().cpu().numpy(), cfg.n_heads, cfg.ln_eps)
            zg = got["z"][t].double().cpu().numpy()
            rel = np.linalg.norm(zg - z) / np.linalg.norm(z)
            assert rel <= 2e-2 and np.abs(zg - z).max() <= 5e-2, (t, rel)
            assert np.abs(got["boxes"][t].double().cpu().numpy() - box).max() <= 1e-2
            assert np.abs(got["conf"][t].double().cpu().numpy() - conf).max() <= 1e-2
    e.close()


def test_decoder_cross_attention_tiny_ragged():
    _check_decode(ci.CONFIGS["tiny"], 3, 16, 0, [0, 4, 16, 1])


def test_decoder_tiny_128_queries_more_queries_than_tokens():
    """Q = 128 queries per task on the tiny geometry (Nf = 64 < Q, 8 tasks): the workspace
    is sized for T * Q attention-output rows once the decoder is set (obuf overflow)."""
    _check_decode(ci.CONFIGS["tiny"], 3, 128, 2, [0, 4, 16, 1, 7, 0, 16, 3])


def test_decoder_cross_attention_c640_128_queries():
    _check_decode(ci.CONFIGS["c640"], 4, 128, 5, [0, 100, 400])


def test_decoded_queries_drive_gate_box_selection_and_refine():
    """A1 -> A2 -> A3 closed on the GPU: coarse encode -> decoder (f3) ->
    hardness gate (f2) and box-driven cell scores (f1) from the DECODED confidences / boxes ->
    threshold selection -> refine.  Gate, scores and selection bit-exact against the oracle
    fed the same decoded outputs; the refine against the oracle's refine of that selection."""
    from paper_2505_23317_b200.api import bf16_tensor
    cfg = ci.CONFIGS["c640"]
    w = ci.make_weights(cfg, seed=0)
    wd = ci.make_decoder_weights(cfg, 128, seed=6)
    e = CFDetrEncoder(cfg, w, max_tasks=8)
    e.set_decoder(wd)
    B = 2
    imgs = ci.make_frames(cfg, B, task0=3)
    dimg = bf16_tensor(imgs, "cuda")
    co = e.coarse_encode(dimg)
    ccu = torch.arange(B + 1, dtype=torch.int32, device="cuda") * e.Nc
    dec = e.decode(co["y"].reshape(-1, cfg.d_model), ccu, B, B * e.Nc)
    hard = e.hardness(dec["conf"])
    sc = e.box_scores(dec["boxes"], dec["conf"])
    sel = e.select_regions(sc, threshold=0.0)
    ro = e.batch_refine(dimg, co["x0"], sel["sel_idx"], sel["sel_count"])
    torch.cuda.synchronize()
    boxes, conf = dec["boxes"].cpu().numpy(), dec["conf"].cpu().numpy()
    cu = ro["cu_seqlens"].cpu().numpy()
    for b in range(B):
        assert int(hard[b]) == O.hardness_gate(conf[b])
        s_ref = O.box_cell_scores(cfg, boxes[b], conf[b])
        assert np.array_equal(sc[b].cpu().numpy(), s_ref.astype(np.float32))
        sel_ref = O.select_threshold(s_ref.astype(np.float32), 0.0)
        k = int(sel["sel_count"][b])
        assert np.array_equal(sel["sel_idx"][b, :k].cpu().numpy(), sel_ref)
        oc = O.coarse_encode(cfg, w, [imgs[b]])[0]
        rr = O.refine_encode(cfg, w, imgs[b], oc["x0"], sel_ref)
        y = ro["y"][cu[b]:cu[b + 1]].double().cpu().numpy()
        rel = np.linalg.norm(y - rr["y"]) / np.linalg.norm(rr["y"])
        assert rel <= 2e-2 and np.abs(y - rr["y"]).max() <= 5e-2, (b, rel)
    e.close()
