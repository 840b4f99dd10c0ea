"""Root-iteration study of the r update (DESIGN 6.5): the r-ICD inputs
(r, q, B, S) of one c3 stream captured from the oracle after a bootstrap and
7 frames, plus random cases, through the device r_update compiled for the
host (tests/tools/r_iter_host.cu), with and without the two-step Halley stop
(DDH_HALLEY_STRICT); reports mean iterations, the mean per-warp maximum and
the max relative error against the oracle's exact minimiser (ties excluded).
usage: python tests/tools/r_iter_study.py"""
import os, subprocess, sys, tempfile
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle.ddh_oracle as O  # noqa: E402
import synth  # noqa: E402

tmp = tempfile.mkdtemp()
src = os.path.join(ROOT, "tests", "tools", "r_iter_host.cu")
for exe, extra in (("strict", ["-DDDH_HALLEY_STRICT"]), ("default", [])):
    subprocess.run(["nvcc", "-x", "cu", "-O2", *extra, "-o", os.path.join(tmp, exe), src], check=True,
                   capture_output=True)

cfg = dict(synth.CONFIGS["c3"])
n = cfg["n"]
y, _ = synth.make_batch(cfg, streams=1, frames=8, workers=1)
p = O.OracleParams(n=n, aperture_diam=n, noise_var=synth.recon_noise_var(n, n, cfg["snr_db"]))
a = O.aperture_of(p)
cap, orig = [], O.r_update_pixels


def hook(r_cur, q, B, S, r_min, **kw):
    cap.append(np.stack([r_cur, q, B, S]).astype(np.float32))
    return orig(r_cur, q, B, S, r_min, **kw)


r, phi, _ = O.bootstrap(y[0, 0], p, 10, a)
for t in range(1, 8):
    cap.clear()
    O.r_update_pixels = hook
    r, phi, _ = O.ddh_step(r, phi, y[t, 0], p, a)
    O.r_update_pixels = orig
sets = {"c3": np.concatenate(cap, axis=1)}
g = np.random.default_rng(1)
m = 200000
for scale in (1.0, 0.01, 100.0):
    q = g.random(m) * 2 * scale + 1e-4
    B = g.random(m) * 4 / scale + 0.05
    S = B * g.random(m) * 3 * scale - 0.2 * B * scale
    rr = g.random(m) * 2 * scale + 1e-3
    sets[f"rand{scale:g}"] = np.stack([rr, q, B, S]).astype(np.float32)
for name, d in sets.items():
    m = d.shape[1]
    fin = os.path.join(tmp, "in.bin")
    with open(fin, "wb") as f:
        np.array([m], np.int32).tofile(f)
        d.tofile(f)
    rr, q, B, S = d.astype(float)
    ref, gap = O.r_update_pixels(rr, q, B, S, 1e-4, return_gap=True)
    for exe in ("strict", "default"):
        so = subprocess.run([os.path.join(tmp, exe), fin, os.path.join(tmp, "out.bin")], capture_output=True,
                            text=True).stdout.strip()
        out = np.fromfile(os.path.join(tmp, "out.bin"), np.float32)[:m]
        rel = np.abs(out - ref) / ref
        print(f"{name:9s} {exe:8s} {so}  max rel (non-tie) {rel[gap > 1e-6].max():.2e}")
