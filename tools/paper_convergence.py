"""Context check against the paper's own result: under its
simulation conditions (config "paper": N = 256, D/r0 = 10, |v| = 0.595
px/frame, SNR 10 dB, cold start) DDH-MBIR with N_k = 1 reaches a Strehl ratio
>= 0.8 within 150 time frames.  Runs the GPU path for N_k = 1, 2, 4, 8 over
300 frames of the synthetic stand-in sequence and reports the per-frame Strehl
(ddh_strehl).  Context only (the USAF scene and the paper's seeds are absent).
Writes profiles/<round>_paper_convergence.json."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2305_03284_b200 import DDH  # noqa: E402

rnd = sys.argv[1] if len(sys.argv) > 1 else "r01"
seeds = int(sys.argv[2]) if len(sys.argv) > 2 else 4
cfg = dict(synth.CONFIGS["paper"])
scene = sys.argv[3] if len(sys.argv) > 3 else "bars"
cfg["scene"] = scene
n, T = cfg["n"], cfg["frames"]
nv = synth.recon_noise_var(n, cfg["diam"], cfg["snr_db"])
dev = torch.device("cuda:0")
res = {}
y, ph = synth.make_batch(cfg, streams=seeds)  # independent seeds = streams of one ctx
yd, pt = torch.from_numpy(y).to(dev), torch.from_numpy(ph).to(dev)
for nk in (1, 2, 4, 8):
    ctx = DDH(n, seeds, noise_var=nv, n_k=nk)
    phi_o = torch.empty((T, seeds, n, n), device=dev)
    ctx.step(yd, phi_o)
    torch.cuda.synchronize()
    sc = DDH(n, seeds, noise_var=nv)
    st = np.array(sc.strehl(phi_o.reshape(T * seeds, n, n), pt.reshape(T * seeds, n, n))).reshape(T, seeds)
    first = [int(np.argmax(st[:, k] >= 0.8)) if (st[:, k] >= 0.8).any() else None for k in range(seeds)]
    res[nk] = {"strehl_median_per_frame": [round(float(v), 4) for v in np.median(st, 1)],
               "strehl_median_frames_150_300": float(np.median(st[150:])),
               "first_frame_ge_0.8": first}
    print(f"N_k={nk}: median Strehl frames 150-300 {np.median(st[150:]):.3f}; frame 50/100/150/299 "
          f"{np.median(st[50]):.3f} {np.median(st[100]):.3f} {np.median(st[150]):.3f} {np.median(st[299]):.3f}; "
          f"first frame >= 0.8: {first}", flush=True)
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump({"config": "paper (P:218-229): 256^2, D/r0 10, |v| 0.595 px/frame at 45 deg, SNR 10 dB, cold start, "
                     f"{seeds} seeds, scene {scene}", "paper_result": "Strehl >= 0.8 within 150 frames at N_k = 1 (P:266, 270)",
           "results": res}, open(os.path.join(ROOT, "gpurun_out" if os.environ.get("GRAFT_REPO_ROOT") else "profiles", f"{rnd}_paper_convergence_{scene}.json"), "w"), indent=1)
