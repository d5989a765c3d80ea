"""Host <-> device copy rates on this box for the e2e step's transfer sizes (pinned host memory):
H2D of 128 8-bit c640 frames (157 MB), D2H of their refined tokens (92 MB fp32), and both at once."""
import torch

h_in = torch.empty(157286400, dtype=torch.uint8).pin_memory()
d_in = torch.empty_like(h_in, device="cuda")
d_out = torch.empty(91750400 // 4, dtype=torch.float32, device="cuda")
h_out = torch.empty(d_out.shape, dtype=torch.float32).pin_memory()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def both():
    ev = torch.cuda.Event()
    ev.record()
    s1.wait_event(ev)
    s2.wait_event(ev)
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)
    for s in (s1, s2):
        e = torch.cuda.Event()
        e.record(s)
        torch.cuda.current_stream().wait_event(e)


t_h2d = timed(lambda: d_in.copy_(h_in, non_blocking=True))
t_d2h = timed(lambda: h_out.copy_(d_out, non_blocking=True))
t_both = timed(both)
print(f"H2D 157.3 MB: {t_h2d:.3f} ms ({157.3 / t_h2d:.1f} GB/s); D2H 91.8 MB: {t_d2h:.3f} ms ({91.8 / t_d2h:.1f} GB/s); "
      f"both concurrently: {t_both:.3f} ms -> e2e ceiling {128 / t_both * 1e3:.0f} frames/s at 128 frames per step")
