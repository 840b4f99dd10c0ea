"""Exploration of the prior-constant readings (R7) under the paper's
own simulation conditions (config "paper", bar-target scene): which
(sigma_r, q, sigma_phi) make DDH-MBIR with N_k = 1 reach the paper's reported
behaviour (Strehl >= 0.8 within 150 frames)?  GPU path; per-frame
Strehl by ddh_strehl.  usage: python tools/reading_sweep.py [seeds] [frames]"""
import itertools
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2305_03284_b200 import DDH  # noqa: E402

seeds = int(sys.argv[1]) if len(sys.argv) > 1 else 4
T = int(sys.argv[2]) if len(sys.argv) > 2 else 300
cfg = dict(synth.CONFIGS["paper"])
n = cfg["n"]
nv = synth.recon_noise_var(n, cfg["diam"], cfg["snr_db"])
y, ph = synth.make_batch(cfg, streams=seeds, frames=T)
yd, pt = torch.from_numpy(y).cuda(), torch.from_numpy(ph).cuda()
sc = DDH(n, seeds, noise_var=nv)
mode = os.environ.get("SWEEP", "priors")
if mode == "priors":
    grid = [dict(r_sigma=rs, r_q=q, phi_sigma=ps, n_k=1)
            for rs in (0.1, 0.5, 2.0) for q in (1.2, 2.0) for ps in (0.25, 0.5, 2.0, 0.0)]
else:
    grid = [dict(icd_sweeps=sw, nvs=k, n_k=1) for sw in (1, 2, 4) for k in (3.0, 10.0, 30.0, 100.0)]
for kw in grid:
    kw = dict(kw)
    nvs = kw.pop("nvs", 1.0)
    ctx = DDH(n, seeds, noise_var=nv * nvs, **kw)
    kw["nvs"] = nvs
    phi_o = torch.empty((T, seeds, n, n), device="cuda")
    ctx.step(yd, phi_o)
    torch.cuda.synchronize()
    st = np.array(sc.strehl(phi_o.reshape(T * seeds, n, n), pt.reshape(T * seeds, n, n))).reshape(T, seeds)
    first = [int(np.argmax(st[:, k] >= 0.8)) if (st[:, k] >= 0.8).any() else -1 for k in range(seeds)]
    print(f"{kw}: median S[100:] {np.median(st[100:]):.3f}  S@50/100/150/{T-1} "
          f"{np.median(st[50]):.2f} {np.median(st[100]):.2f} {np.median(st[min(150, T-1)]):.2f} {np.median(st[-1]):.2f}  first>=0.8 {first}",
          flush=True)
