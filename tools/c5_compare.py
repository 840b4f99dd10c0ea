"""the BASELINE configs[4] experiment (c5: 1024^2, 1 stream,
50 frames, D/r0 = 30, flow 2 px/frame, SNR 2 dB): DDH-MBIR with N_k = 1, 5, 50
EM iterations per frame (cold start, Fig. 1) against conventional single-shot
DH-MBIR with 300 iterations on each frame (resets every 200).
Per-frame Strehl ratio against the synthetic truth (ddh_strehl) and
device time per frame.  Synthetic frozen-flow sequence stands in
for the paper's USAF-chart simulation; the paper's own Strehl values are for
its scene and are context only.  Writes profiles/<round>_c5_compare.json.

    python tools/c5_compare.py [round] [frames]
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2305_03284_b200 import DDH  # noqa: E402

rnd = sys.argv[1] if len(sys.argv) > 1 else "r01"
T = int(sys.argv[2]) if len(sys.argv) > 2 else 50
cfg = dict(synth.CONFIGS["c5"])
n = cfg["n"]
t0 = time.time()
y, ph = synth.make_batch(cfg, frames=T)
gen = time.time() - t0
nv = synth.recon_noise_var(n, cfg["diam"], cfg["snr_db"])
dev = torch.device("cuda:0")
yd = torch.from_numpy(y).to(dev)
pt = torch.from_numpy(ph).to(dev)
out = {"config": "c5: 1024x1024, 1 stream, %d frames, D/r0 30, flow 2 px/frame, SNR 2 dB" % T,
       "data": "synthetic frozen-flow Kolmogorov sequence (DESIGN.md 5)", "synth_seconds": round(gen, 1),
       "methods": {}}


def run(label, fn):
    phi_o = torch.empty((T, 1, n, n), device=dev)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn(phi_o)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    ctx = DDH(n, 1, noise_var=nv)
    st = np.array(ctx.strehl(phi_o.reshape(T, n, n), pt.reshape(T, n, n)))
    out["methods"][label] = {"strehl": [round(float(v), 4) for v in st], "strehl_mean": float(st.mean()),
                             "strehl_mean_last_half": float(st[T // 2:].mean()), "ms_per_frame": ms / T}
    print(f"{label:28s} Strehl mean {st.mean():.3f} (last half {st[T // 2:].mean():.3f})  {ms / T:8.3f} ms/frame",
          flush=True)


for nk in (1, 5, 50):
    ctx = DDH(n, 1, noise_var=nv, n_k=nk)
    run(f"DDH-MBIR N_k={nk}", lambda o, c=ctx: c.step(yd, o))
ctx = DDH(n, 1, noise_var=nv)
run("static DH-MBIR 300 iters", lambda o, c=ctx: c.static(yd, 300, o))
os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(out, open(os.path.join(ROOT, "gpurun_out" if os.environ.get("GRAFT_REPO_ROOT") else "profiles", f"{rnd}_c5_compare.json"), "w"), indent=1)
