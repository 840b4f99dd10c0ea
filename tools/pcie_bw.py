"""Pinned host<->device copy bandwidth on this box (the e2e leg's ceiling):
H2D alone, D2H alone, and both at once on two streams (32 MiB / 16 MiB per copy,
the e2e leg's per-step sizes)."""
import torch
h_in = torch.empty(32 << 20, dtype=torch.uint8).pin_memory()
h_out = torch.empty(16 << 20, dtype=torch.uint8).pin_memory()
d_in = torch.empty(32 << 20, dtype=torch.uint8, device="cuda")
d_out = torch.empty(16 << 20, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def run(h2d, d2h, reps=200):
    for _ in range(5):
        if h2d:
            with torch.cuda.stream(s1): d_in.copy_(h_in, non_blocking=True)
        if d2h:
            with torch.cuda.stream(s2): h_out.copy_(d_out, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    s1.wait_event(e0); s2.wait_event(e0)
    for _ in range(reps):
        if h2d:
            with torch.cuda.stream(s1): d_in.copy_(h_in, non_blocking=True)
        if d2h:
            with torch.cuda.stream(s2): h_out.copy_(d_out, non_blocking=True)
    ev1, ev2 = torch.cuda.Event(), torch.cuda.Event()
    ev1.record(s1); ev2.record(s2)
    torch.cuda.current_stream().wait_event(ev1); torch.cuda.current_stream().wait_event(ev2)
    e1.record(); torch.cuda.synchronize()
    t = e0.elapsed_time(e1) * 1e-3
    return (reps * (32 << 20) / t / 1e9 if h2d else 0.0), (reps * (16 << 20) / t / 1e9 if d2h else 0.0)
print("h2d alone GB/s %.1f" % run(True, False)[0])
print("d2h alone GB/s %.1f" % run(False, True)[1])
a, b = run(True, True)
print("both: h2d %.1f d2h %.1f GB/s -> e2e ceiling at 32 MiB in + 16 MiB out per 64 frames: %.0f frames/s" % (a, b, a * 1e9 / (32 << 20) * 64))
