"""throughput of the c3 workload (256^2, 64 streams) vs the
number of EM iterations per time step N_k in {1, 2, 4, 8} (uninstrumented
CUDA-event timing, inputs resident in HBM).  Writes profiles/<round>_nk_sweep.json
(gpurun_out/ on a gpurun box, whose profiles/ is not copied back)."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2305_03284_b200 import DDH, sched  # noqa: E402

rnd = sys.argv[1] if len(sys.argv) > 1 else "r01"
cfg = dict(synth.CONFIGS["c3"])
S, F = cfg["streams"], 8
y, _ = synth.make_batch(cfg, frames=F, want_phi=False)
yd = torch.from_numpy(y).cuda()
nv = synth.recon_noise_var(256, 256, cfg["snr_db"])
res = {}
for nk in (1, 2, 4, 8):
    ctx = DDH(256, S, noise_var=nv, n_k=nk, flags=64)
    sched.run_steps(ctx, yd, 0, 3, F)
    torch.cuda.synchronize()
    K = 100 // nk
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    sched.run_steps(ctx, yd, 3, K, F)  # multi-frame calls, as bench.py
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / K
    res[nk] = {"ms_per_step": ms, "frames_per_s": S / (ms * 1e-3), "em_iterations_per_s": S * nk / (ms * 1e-3)}
    print(f"N_k={nk}: {ms * 1000:8.1f} us/step  {S / (ms * 1e-3):10.0f} frames/s  {S * nk / (ms * 1e-3):10.0f} EM-iter/s",
          flush=True)
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump({"workload": "c3: 256x256, 64 streams, synthetic", "results": res},
          open(os.path.join(ROOT, "gpurun_out" if os.environ.get("GRAFT_REPO_ROOT") else "profiles", f"{rnd}_nk_sweep.json"), "w"), indent=1)
