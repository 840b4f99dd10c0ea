"""Host check of the device r-update (tests/tools/r_update_host.cu) against the oracle."""
import subprocess, sys
import numpy as np
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__)))))
import oracle.ddh_oracle as O
_HERE = __import__("os").path.dirname(__import__("os").path.abspath(__file__))
subprocess.run(["nvcc", "-x", "cu", "-O2", "-o", "/tmp/r_update_host", __import__("os").path.join(_HERE, "r_update_host.cu")],
               check=True)
g = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
m = 200000
for scale in (1.0, 0.01, 100.0):
    q = (g.random(m) * 2 * scale + 1e-4).astype(np.float32)
    B = (g.random(m) * 4 / scale + 0.05).astype(np.float32)
    S = (B * g.random(m) * 3 * scale - 0.2 * B * scale).astype(np.float32)
    r = (g.random(m) * 2 * scale + 1e-3).astype(np.float32)
    inp = "\n".join(f"{a:.9g} {b:.9g} {c:.9g} {d:.9g} 1e-4" for a, b, c, d in zip(r, q, B, S))
    out = np.array(subprocess.run(["/tmp/r_update_host"], input=inp, capture_output=True, text=True).stdout.split(), float)
    ref, gap = O.r_update_pixels(r.astype(float), q.astype(float), B.astype(float), S.astype(float), 1e-4, return_gap=True)
    rel = np.abs(out - ref) / ref
    ok = gap > 1e-6
    print(f"scale {scale}: max rel (non-tie) {rel[ok].max():.2e}, p99.9 {np.quantile(rel[ok], 0.999):.2e}, ties {int((~ok).sum())}, 3-root-ish {int(np.isfinite(gap).sum())}")
