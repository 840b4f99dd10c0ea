"""Run one c3 step with the instrumented library and average the per-phase
clock64 deltas printed by rank-0 CTAs (tools/build_timing.sh)."""
import os, subprocess, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import os, sys, torch, numpy as np
sys.path.insert(0, "%s")
import synth
from paper_2305_03284_b200 import DDH
cfg = synth.CONFIGS["c3"]
S = int(os.environ.get("S", "64"))
y, _ = synth.make_batch(cfg, streams=S, frames=3, want_phi=False)
yd = torch.from_numpy(y).cuda()
ctx = DDH(256, S, noise_var=synth.recon_noise_var(256, 256, 5.0), lanes=int(os.environ.get("LANES", "1")))
for t in range(3):
    ctx.step(yd[t:t+1]); torch.cuda.synchronize()
''' % ROOT
env = dict(os.environ, DDH_LIB=os.path.join(ROOT, "paper_2305_03284_b200/lib/timing/libddh_timing.so"))
out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
lines = [l.split() for l in out.stdout.splitlines() if l[:2] in ("KA", "KB", "KC")]
sync = {}
for l in lines:
    if l[0].endswith("sync"):
        sync.setdefault(l[0], []).append(int(l[1]))
lines = [l for l in lines if not l[0].endswith("sync")]
if not lines:
    print(out.stdout[-2000:], out.stderr[-2000:])
by = {}
for l in lines[len(lines) // 3:]:  # skip the first frame (warm-up)
    by.setdefault(l[0], []).append([int(x) for x in l[1:]])
for k, rows in by.items():
    import numpy as np
    a = np.array(rows)
    print(k, "mean cycles per phase:", " ".join(f"{v:.0f}" for v in a.mean(0)), " total", f"{a.sum(1).mean():.0f}")

for k, v in sync.items():
    print(k, "cycles in cluster barrier + halo-copy barrier (thread 0):", f"{np.mean(v[len(v)//3:]):.0f}")
