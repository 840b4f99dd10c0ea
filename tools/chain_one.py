"""One configuration of the N = 64 chain for profiling: S streams, N_k, DDH_CHAIN
from the environment.  usage: python tools/chain_one.py S N_k [calls]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2305_03284_b200 import DDH  # noqa: E402

S, nk = int(sys.argv[1]), int(sys.argv[2])
calls = int(sys.argv[3]) if len(sys.argv) > 3 else 2
cfg = dict(synth.CONFIGS["c1"])
y, _ = synth.make_batch(cfg, streams=S, frames=4, want_phi=False)
yd = torch.from_numpy(y).cuda()
ctx = DDH(64, S, noise_var=synth.recon_noise_var(64, 64, cfg["snr_db"]), n_k=nk)
for _ in range(calls):
    ctx.step(yd)
torch.cuda.synchronize()
print("ok")
