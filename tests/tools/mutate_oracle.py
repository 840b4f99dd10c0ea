"""Mutation run for the oracle pins.

Each mutation is a plausible mistake in ``oracle/ddh_oracle.py`` (a dropped
term, a wrong sign / factor / index, a transposed operand, a skipped step).
For each one, a scratch copy of the oracle, the synthesiser and the CPU pin
tests is made, the mutation applied, and ``tests/test_oracle_pins.py`` run.
A mutation that passes every pin is a SURVIVOR: some part of the oracle is
not pinned.  Writes a JSON report (default ``profiles/r02_oracle_mutations.json``).

    python tests/tools/mutate_oracle.py [--out FILE]
"""
import argparse
import json
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
ORACLE = "oracle/ddh_oracle.py"

# (name, description, old text, new text): old must occur exactly once; a list of
# (old, new) pairs is one mutation applied consistently in several places
MUTATIONS = [
    ("M1", "qGGMRF exponent q instead of 2-q, consistently in rho and its weight",
     ["t = np.abs(d / (T * sig)) ** (2.0 - q)\n    return d * d",
      "t = np.abs(d / (T * sig)) ** (2.0 - q)\n    return (1.0",
      "(1.0 - (2.0 - q) * t / (2.0 * (1.0 + t)))"],
     ["t = np.abs(d / (T * sig)) ** q\n    return d * d",
      "t = np.abs(d / (T * sig)) ** q\n    return (1.0",
      "(1.0 - q * t / (2.0 * (1.0 + t)))"]),
    ("M1r", "qGGMRF exponent q instead of 2-q in rho only",
     "t = np.abs(d / (T * sig)) ** (2.0 - q)\n    return d * d",
     "t = np.abs(d / (T * sig)) ** q\n    return d * d"),
    ("M1w", "qGGMRF exponent q instead of 2-q in the weight only",
     "t = np.abs(d / (T * sig)) ** (2.0 - q)\n    return (1.0",
     "t = np.abs(d / (T * sig)) ** q\n    return (1.0"),
    ("M2", "phase-correlation weight 1/s2 instead of 2/s2",
     "c = (2.0 / s2) * a", "c = (1.0 / s2) * a"),
    ("M3", "bootstrap resets only at k = 0",
     "if k % p.boot_period == 0:", "if k == 0:"),
    ("M4", "theta sign flipped (arg(conj(y) f))",
     "theta = np.angle(yhat * np.conj(f))", "theta = np.angle(np.conj(yhat) * f)"),
    ("M5", "E-step variance term dropped from q",
     "q = np.abs(mu) ** 2 + C", "q = np.abs(mu) ** 2"),
    ("M6", "Wiener gain r/(r+s2) replaced by s2/(r+s2)",
     "w = r / (r + s2)", "w = s2 / (r + s2)"),
    ("M7", "Eq. 3 weights swapped (lam <-> 1-lam)",
     "(1.0 - lam) * r + lam * alpha", "lam * r + (1.0 - lam) * alpha"),
    ("M8", "Eq. 3 without alpha",
     "lam * alpha * np.abs(u) ** 2", "lam * np.abs(u) ** 2"),
    ("M9", "Normalize without the mean subtraction",
     "return math.sqrt(y.size) * (y - mu) / d", "return math.sqrt(y.size) * y / d"),
    ("M10", "Normalize with sqrt(p) missing",
     "return math.sqrt(y.size) * (y - mu) / d", "return (y - mu) / d"),
    ("M11", "plane fit without piston",
     "return c[0] + c[1] * x + c[2] * yy", "return c[1] * x + c[2] * yy"),
    ("M12", "plane x/y coordinates transposed",
     "return c[0] + c[1] * x + c[2] * yy", "return c[0] + c[1] * yy + c[2] * x"),
    ("M13", "adjoint with e^{+j phi}",
     "return fft2c(a * np.exp(-1j * phi) * y)", "return fft2c(a * np.exp(1j * phi) * y)"),
    ("M14", "adjoint without the aperture",
     "return fft2c(a * np.exp(-1j * phi) * y)", "return fft2c(np.exp(-1j * phi) * y)"),
    ("M15", "second FFT forward instead of inverse",
     "f = ifft2c(mu)", "f = fft2c(mu)"),
    ("M16", "r surrogate with +2 S x",
     "return np.log(x) + q / x + B * x * x - 2.0 * S * x",
     "return np.log(x) + q / x + B * x * x + 2.0 * S * x"),
    ("M17", "companion matrix: linear coefficient sign flipped",
     "comp[:, 0, 1] = -1.0 / (2.0 * B)", "comp[:, 0, 1] = 1.0 / (2.0 * B)"),
    ("M18", "r candidates without r_min",
     "cand = np.concatenate([np.full((m, 1), r_min), np.maximum(roots.real, r_min)], axis=1)",
     "cand = np.maximum(roots.real, r_min)"),
    ("M19", "r prior weight uses r_j - r_i with r_i in S (S += bt * ri)",
     "S += bt * rj", "S += bt * ri"),
    ("M20", "diagonal neighbours weighted 1/6",
     "(-1, -1, 1.0 / 12.0), (-1, 1, 1.0 / 12.0)", "(-1, -1, 1.0 / 6.0), (-1, 1, 1.0 / 6.0)"),
    ("M21", "colour order (0,1) before (0,0)",
     "COLOURS = ((0, 0), (0, 1), (1, 0), (1, 1))", "COLOURS = ((0, 1), (0, 0), (1, 0), (1, 1))"),
    ("M22", "two-colour checkerboard ((0,0),(1,1) merged)",
     "COLOURS = ((0, 0), (0, 1), (1, 0), (1, 1))", "COLOURS = ((0, 0), (1, 1))"),
    ("M23", "phi ICD: periodic boundary instead of free",
     "pj, valid = _neigh(phi, ii, jj, di, dj, periodic=False)",
     "pj, valid = _neigh(phi, ii, jj, di, dj, periodic=True)"),
    ("M24", "phi ICD: s = 1 (no cosine bound curvature)",
     "num = cc * s * tt + wphi * nb", "num = cc * tt + wphi * nb"),
    ("M25", "phi prior weight 1/sigma instead of 1/sigma^2",
     "wphi = 1.0 / (p.phi_sigma * p.phi_sigma) if prior else 0.0",
     "wphi = 1.0 / p.phi_sigma if prior else 0.0"),
    ("M26", "tip/tilt removal skipped in ddh_step",
     "    if p.tiptilt:\n        phi = remove_tip_tilt(phi, a)", "    pass"),
    ("M27", "N_k loop: u not recomputed after the first iteration",
     "        if k > 0:\n            u = adjoint(phi, yhat, a)", "        pass"),
    ("M28", "Strehl denominator uses psi (ratio = 1 always)",
     "den = np.max(np.abs(ifft2c(a.astype(np.complex128))) ** 2)",
     "den = np.max(np.abs(ifft2c(a * np.exp(1j * psi))) ** 2)"),
    ("M29", "aperture includes the boundary circle (<=)",
     "return ((i * i + j * j) < (diam / 2.0) ** 2)", "return ((i * i + j * j) <= (diam / 2.0) ** 2)"),
    ("M30", "centred DFT without the output shift",
     "return np.fft.fftshift(np.fft.fft2(np.fft.ifftshift(x), norm=\"ortho\"))",
     "return np.fft.fft2(np.fft.ifftshift(x), norm=\"ortho\")"),
    ("M31", "bootstrap reset without boot_alpha",
     "r = np.maximum(p.boot_alpha * np.abs(u) ** 2, p.r_min)",
     "r = np.maximum(np.abs(u) ** 2, p.r_min)"),
    ("M32", "degenerate frame not detected",
     "    if d == 0.0:\n        return None", "    if d < 0.0:\n        return None"),
    ("M33", "qGGMRF weight: (2-q) factor dropped in the derivative term",
     "(1.0 - (2.0 - q) * t / (2.0 * (1.0 + t)))", "(1.0 - t / (2.0 * (1.0 + t)))"),
    ("M34", "tie rule: farthest candidate instead of nearest",
     "best = cand[np.arange(m), dist.argmin(axis=1)]",
     "best = cand[np.arange(m), np.where(np.isinf(dist), -1.0, dist).argmax(axis=1)]"),
]


# Mutations that cannot change any result (argued here, so a survivor is explained)
EQUIVALENT = {
    "M18": "f'(x) = g(x)/x^2 with g the cubic; every real root is clamped to r_min, so when the "
           "minimiser over [r_min, inf) is r_min there is a root <= r_min (g > 0 on (r_min, x2) "
           "means the smallest root lies below r_min) and max(root, r_min) already supplies it; "
           "when g < 0 at r_min f decreases there and r_min is not the minimiser",
}


def run_one(name, old, new):
    with tempfile.TemporaryDirectory() as tmp:
        for d in ("oracle", "synth", "tests"):
            shutil.copytree(os.path.join(ROOT, d), os.path.join(tmp, d),
                            ignore=shutil.ignore_patterns("__pycache__"))
        path = os.path.join(tmp, ORACLE)
        src = open(path).read()
        if old is not None:
            olds, news = (old, new) if isinstance(old, list) else ([old], [new])
            for o, n_ in zip(olds, news):
                k = src.count(o)
                if k != 1:
                    return {"error": f"pattern occurs {k} times"}
                src = src.replace(o, n_)
            open(path, "w").write(src)
        cmd = [sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
               "tests/test_oracle_pins.py"]
        pr = subprocess.run(cmd, cwd=tmp, capture_output=True, text=True, timeout=1800)
        failed = [l.split("::")[-1].split(" ")[0] for l in pr.stdout.splitlines() if l.startswith("FAILED")]
        return {"rc": pr.returncode, "killed_by": failed, "tail": pr.stdout.strip().splitlines()[-1:]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_oracle_mutations.json"))
    args = ap.parse_args()
    base = run_one("base", None, None)
    assert base["rc"] == 0, f"unmutated pins fail: {base}"
    rep = {"oracle": ORACLE, "pins": "tests/test_oracle_pins.py", "mutations": []}
    for name, desc, old, new in MUTATIONS:
        res = run_one(name, old, new)
        res.update(name=name, desc=desc, survived=(res.get("rc") == 0))
        if name in EQUIVALENT:
            res["equivalent"] = EQUIVALENT[name]
        rep["mutations"].append(res)
        print(f"{name:5s} {'SURVIVED' if res['survived'] else 'killed  '} {desc}  {res.get('killed_by') or res.get('error', '')}",
              flush=True)
    rep["survivors"] = [m["name"] for m in rep["mutations"] if m["survived"] and "equivalent" not in m]
    rep["equivalent_survivors"] = [m["name"] for m in rep["mutations"] if m["survived"] and "equivalent" in m]
    rep["errors"] = [m["name"] for m in rep["mutations"] if "error" in m]
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump(rep, open(args.out, "w"), indent=1)
    print("survivors:", rep["survivors"], "errors:", rep["errors"])


if __name__ == "__main__":
    main()
