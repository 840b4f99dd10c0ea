"""Per-kernel device times (CUDA events, serialised lanes=1) vs stream count,
to expose wave quantisation.  usage: python tools/kernel_times.py N S1 S2 ..."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from paper_2305_03284_b200 import DDH
n = int(sys.argv[1])
cfg = dict(synth.CONFIGS["c3"])
y, _ = synth.make_batch(cfg, streams=max(int(s) for s in sys.argv[2:]), frames=4, want_phi=False)
yd = torch.from_numpy(y).cuda()
nv = synth.recon_noise_var(256, 256, 5.0)
lanes = int(os.environ.get("LANES", "1"))
for S in map(int, sys.argv[2:]):
    ctx = DDH(n, S, noise_var=nv, lanes=lanes, flags=int(os.environ.get("FLAGS", "0")), chunk_streams=int(os.environ.get("CHUNK", "0")))
    ys = yd[:, :S].contiguous()
    for t in range(3):
        ctx.step(ys[t:t + 1])
    torch.cuda.synchronize()
    prof_on = os.environ.get("PROF", "1") == "1"
    ctx.profile(prof_on); ctx.profile_read()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    K = 50
    import time
    e0.record()
    h0 = time.perf_counter()
    for k in range(K):
        ctx.step(ys[k % 4:k % 4 + 1])
    h1 = time.perf_counter()
    e1.record(); torch.cuda.synchronize()
    host_us = (h1 - h0) / K * 1e6
    prof = ctx.profile_read(); ctx.profile(False)
    tot = e0.elapsed_time(e1) / K * 1000
    print(f"S={S:3d} step {tot:7.1f} us (host enqueue {host_us:6.1f} us)  " + "  ".join(f"{k} {v[0] / K * 1000:6.1f}" for k, v in prof.items()), flush=True)
    del ctx
