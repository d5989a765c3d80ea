"""Time the criticality-score kernel alone (cfdx_score) at bench shapes: reps back-to-back launches
replayed from one CUDA graph, CUDA events around the replay.  python tools/score_bench.py [B] [Nc]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_2505_23317_b200 import _lib as L  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
Nc = int(sys.argv[2]) if len(sys.argv) > 2 else 400
reps = 20
d, nh = 256, 8
lib = L.load()
cap = B * Nc + 256
qkv = torch.randn(cap, 3 * d, device="cuda").to(torch.bfloat16)
q = qkv[:B * Nc, :d].float().view(B, Nc, nh, 32).transpose(1, 2)
k = qkv[:B * Nc, d:2 * d].float().view(B, Nc, nh, 32).transpose(1, 2)
S = q @ k.transpose(-1, -2) / 32 ** 0.5                       # [B, nh, Nc, Nc]
lse = torch.zeros(nh, cap, device="cuda")
lse[:, :B * Nc] = torch.logsumexp(S, dim=-1).permute(1, 0, 2).reshape(nh, B * Nc)
ref = torch.softmax(S, dim=-1).sum(dim=(1, 2)) / (nh * Nc)  # [B, Nc]
del S
scores = torch.zeros(B, Nc, device="cuda")
run = lambda: lib.cfdx_score(B, Nc, d, nh, qkv.data_ptr(), cap, lse.data_ptr(), cap, scores.data_ptr(),
                             torch.cuda.current_stream().cuda_stream)
assert run() == 0
torch.cuda.synchronize()
err = ((scores - ref).abs() / ref.abs().clamp_min(1e-12)).max().item()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    for _ in range(reps):
        run()
g.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
g.replay()
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) * 1e3 / reps
exps = B * nh * Nc * Nc
print(f"score B={B} Nc={Nc}: {us:.1f} us  {exps / us * 1e-3:.0f} Gexp/s  max rel err {err:.2e} "
      f"{'OK' if err < 1e-3 else 'BAD'}")
