"""f2 at N = 64: frames/s and EM iterations/s of the on-chip chain (one CTA per
stream, all N_k iterations in shared memory) against the streaming kernels
(DDH_CHAIN=0) and the library's automatic choice, N_k in {1, 2, 4, 8}, S streams, multi-frame calls, device time
(CUDA events).  usage: python tools/chain_bench.py [round] [S...]"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2305_03284_b200 import DDH  # noqa: E402

rnd = sys.argv[1] if len(sys.argv) > 1 else "r02"
Ss = [int(x) for x in sys.argv[2:]] or [64, 296, 1024]
cfg = dict(synth.CONFIGS["c1"])
n, F = 64, 16
res = []
for S in Ss:
    y, _ = synth.make_batch(cfg, streams=S, frames=F, want_phi=False)
    yd = torch.from_numpy(y).cuda()
    nv = synth.recon_noise_var(n, n, cfg["snr_db"])
    for chain in (1, 0, "auto"):
        if chain == "auto":
            os.environ.pop("DDH_CHAIN", None)  # the library's choice (use_chain in ddh_api.cpp)
        else:
            os.environ["DDH_CHAIN"] = str(chain)
        for nk in (1, 2, 4, 8):
            ctx = DDH(n, S, noise_var=nv, n_k=nk)
            ctx.step(yd[:4])
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(4):
                ctx.step(yd)
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) * 1000 / (4 * F)
            row = {"streams": S, "chain": chain if chain == "auto" else bool(chain), "n_k": nk, "us_per_step": us, "frames_per_s": S / (us * 1e-6),
                   "em_iterations_per_s": S * nk / (us * 1e-6)}
            res.append(row)
            print(f"S={S:5d} chain={chain} N_k={nk}: {us:8.1f} us/step {row['frames_per_s']:10.0f} frames/s "
                  f"{row['em_iterations_per_s']:10.0f} EM-iter/s", flush=True)
os.environ.pop("DDH_CHAIN", None)
out = os.path.join(ROOT, "gpurun_out" if os.environ.get("GRAFT_REPO_ROOT") else "profiles", f"{rnd}_chain64.json")
os.makedirs(os.path.dirname(out), exist_ok=True)
json.dump({"workload": "64x64 (c1 recipe), S streams, multi-frame calls of 16 frames, device time", "results": res},
          open(out, "w"), indent=1)
