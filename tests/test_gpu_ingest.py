"""Serving-path frame ingest on the GPU (cfd_frames_from_u8, include/cfdetr.h): 8-bit HWC
camera frames -> bf16 frames, bit-exact against oracle.frames_from_u8 (an exact-rational
definition of bf16_rn(fp32_fma(p, scale_c, shift_c))), and the encoder on converted frames
equal, bit for bit, to the encoder on the same frames converted on the host."""
import numpy as np
import pytest
import torch

import cfd_inputs as ci
import oracle as O

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)

from paper_2505_23317_b200.api import CFDetrEncoder, bf16_tensor, frames_from_u8_flat  # noqa: E402


def _bits(t):
    return t.view(torch.int16).cpu().numpy().view(np.uint16)


def test_frames_from_u8_c640_bit_exact():
    cfg = ci.CONFIGS["c640"]
    enc = CFDetrEncoder(cfg, ci.make_weights(cfg, seed=0), max_tasks=8)
    u8 = ci.make_frames_u8(cfg, 5, task0=11)
    sc, sh = ci.u8_affine()
    out = enc.frames_from_u8(torch.from_numpy(u8).cuda(), sc, sh)
    torch.cuda.synchronize()
    assert np.array_equal(_bits(out), O.frames_from_u8(u8, sc, sh))
    # n_frames = 0 is a no-op
    enc.frames_from_u8(torch.empty(0, cfg.img_h, cfg.img_w, 3, dtype=torch.uint8, device="cuda"), sc, sh)
    enc.close()


@pytest.mark.parametrize("n", [0, 1, 2, 15, 16, 17, 47, 48, 49, 1000003])
def test_frames_u8_flat_ragged_lengths(n):
    rng = np.random.default_rng(n)
    src = rng.integers(0, 256, size=n, dtype=np.uint8)
    sc = np.array([0.75, -1.5, 1.0 / 255.0], dtype=np.float32)
    sh = np.array([2.0 + 2.0 ** -20, -0.125, -3.0], dtype=np.float32)
    sentinel = torch.full((n + 8,), 7.0, dtype=torch.bfloat16, device="cuda")
    out = frames_from_u8_flat(torch.from_numpy(src).cuda(), sc, sh, out=sentinel)
    torch.cuda.synchronize()
    got = _bits(out)
    assert np.array_equal(got[:n], O.frames_from_u8(src, sc, sh))
    assert np.all(got[n:] == _bits(torch.tensor([7.0], dtype=torch.bfloat16))[0])  # nothing past n written


def test_encoder_on_ingested_frames_equals_host_converted():
    cfg = ci.CONFIGS["tiny"]
    enc = CFDetrEncoder(cfg, ci.make_weights(cfg, seed=1), max_tasks=8)
    u8 = ci.make_frames_u8(cfg, 3)
    sc, sh = ci.u8_affine()
    dev_frames = enc.frames_from_u8(torch.from_numpy(u8).cuda(), sc, sh)
    host_frames = bf16_tensor(O.frames_from_u8(u8, sc, sh), "cuda")
    a = enc.coarse_encode(dev_frames)
    b = enc.coarse_encode(host_frames)
    torch.cuda.synchronize()
    assert torch.equal(a["y"], b["y"]) and torch.equal(a["scores"], b["scores"])
    enc.close()
