"""Device time per frame of multi-frame ddh_step calls (T frames per call, so
the host enqueue does not bound it).  usage: python tools/step_time.py N S [T] [flags]"""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from paper_2305_03284_b200 import DDH
n, S = int(sys.argv[1]), int(sys.argv[2])
T = int(sys.argv[3]) if len(sys.argv) > 3 else 32
flags = int(sys.argv[4]) if len(sys.argv) > 4 else 0
cfg = dict(synth.CONFIGS["c2" if n == 256 else "c1"]) if n in (64, 256) else dict(synth.CONFIGS["c3"])
cfg["n"] = n
cfg["diam"] = n
y, _ = synth.make_batch(cfg, streams=S, frames=T, want_phi=False)
yd = torch.from_numpy(y).cuda()
ctx = DDH(n, S, noise_var=synth.recon_noise_var(n, n, 5.0), flags=flags)
ctx.step(yd)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
R = 5
e0.record()
for _ in range(R):
    ctx.step(yd)
e1.record()
torch.cuda.synchronize()
print(f"N={n} S={S} flags={flags}: {e0.elapsed_time(e1) / (R * T) * 1000:.1f} us per step")
