#!/bin/bash
# chain (DDH_CHAIN=1) device time per step for the in-tree build and tools/variants/libddh_<v>.so (run under gpurun)
for v in base "$@"; do
  if [ "$v" = base ]; then L=""; else L="tools/variants/libddh_$v.so"; fi
  for S in 296 1024; do for nk in 1 8; do
    env ${L:+DDH_LIB=$L} DDH_CHAIN=1 python - $S $nk <<'PY'
import os, sys, torch
sys.path.insert(0, os.getcwd())
import synth
from paper_2305_03284_b200 import DDH
S, nk = int(sys.argv[1]), int(sys.argv[2])
cfg = dict(synth.CONFIGS["c1"]); y, _ = synth.make_batch(cfg, streams=S, frames=16, want_phi=False); yd = torch.from_numpy(y).cuda()
ctx = DDH(64, S, noise_var=synth.recon_noise_var(64, 64, cfg["snr_db"]), n_k=nk)
ctx.step(yd[:4]); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(4): ctx.step(yd)
e1.record(); torch.cuda.synchronize()
print(f"{os.environ.get('DDH_LIB') or 'base':40s} S={S} N_k={nk}: {e0.elapsed_time(e1)*1000/64:7.1f} us/step")
PY
  done; done
done
