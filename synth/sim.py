"""Frame-sequence synthesiser (input generation only; see synth/__init__.py).

Recipe (restated in DESIGN.md):
  1. r: iid U[0,1] on N x N, periodic Gaussian blur (sigma_b, kernel summing
     to 1), min-max rescale to [0,1], clamp >= r_min (R23).
  2. phi screen: FFT method on an M1 x M2 periodic grid, coefficients
     (z1 + j z2) sqrt(Phi(f) df1 df2), Phi(f) = 0.023 r0^{-5/3} |f|^{-11/3}
     (f in cycles/px, r0 = D_px/(D/r0)), DC = 0, phi = Re(sum) (R22).
  3. frozen flow: frame t uses the window at offset t v; integer v is an exact
     crop of a strip, non-integer v a Fourier shift of the periodic screen
     (R24).  Piston, tip and tilt are removed over the aperture.
  4. speckle g_t = sqrt(r/2)(z1 + j z2), fresh per frame (R21).
  5. noise sigma_n^2 = mean(r)/10^{SNR/10} (SNR in dB, R20).
  6. y_t = a e^{j phi_t} F_c^{-1}(g_t) + w_t, stored as complex64.
  7. RNG: numpy PCG64 keyed by (seed, stream, frame, purpose): deterministic
     and independent of worker count.
"""
from __future__ import annotations

import math
import os
from concurrent.futures import ProcessPoolExecutor
from typing import Dict, Tuple

import numpy as np

SEED0 = 20230504

# Purposes for RNG keys.
_P_SCENE, _P_SCREEN, _P_SPECKLE, _P_NOISE, _P_DIR, _P_DR0 = range(6)


def rng_for(seed: int, stream: int, frame: int, purpose: int) -> np.random.Generator:
    return np.random.default_rng([int(seed), int(stream), int(frame), int(purpose)])


# BASELINE.json configs as concrete synthetic workloads.
CONFIGS: Dict[str, dict] = {
    "c1": dict(name="c1", n=64, diam=64, streams=1, frames=16, d_r0=10.0, d_r0_range=None,
               flow=1.0, direction="cols", sigma_b=2.0, snr_db=10.0, n_k=1, k_b=50),
    "c2": dict(name="c2", n=256, diam=256, streams=1, frames=200, d_r0=15.0, d_r0_range=None,
               flow=1.0, direction="cols", sigma_b=3.0, snr_db=5.0, n_k=1, k_b=0),
    "c3": dict(name="c3", n=256, diam=256, streams=64, frames=100, d_r0=None, d_r0_range=(10.0, 20.0),
               flow=1.0, direction="random", sigma_b=3.0, snr_db=5.0, n_k=1, k_b=0),
    "c4": dict(name="c4", n=512, diam=512, streams=512, frames=100, d_r0=20.0, d_r0_range=None,
               flow=2.0, direction="cols", sigma_b=4.0, snr_db=2.0, n_k=1, k_b=0),
    "c5": dict(name="c5", n=1024, diam=1024, streams=1, frames=50, d_r0=30.0, d_r0_range=None,
               flow=2.0, direction="cols", sigma_b=4.0, snr_db=2.0, n_k=1, k_b=0),
    # the paper's own simulation conditions (not a BASELINE config): N = 256,
    # D/r0 = 10, f_g/f_s = 100 Hz / 10 kHz -> |v| = 0.595 px/frame along (1, 1)/sqrt 2
    # (v = (0.421, 0.421)), SNR 10 dB, cold start; the USAF chart is replaced by R23's field
    "paper": dict(name="paper", n=256, diam=256, streams=1, frames=300, d_r0=10.0, d_r0_range=None,
                  flow=(1.0 / 0.43) * (100.0 / 10000.0) * (256 / 10.0), direction="angle", angle=math.pi / 4,
                  sigma_b=3.0, snr_db=10.0, n_k=1, k_b=0, scene="bars"),
}


def aperture_mask(n: int, diam: float) -> np.ndarray:
    i = np.arange(n)[:, None] - n / 2
    j = np.arange(n)[None, :] - n / 2
    return ((i * i + j * j) < (diam / 2.0) ** 2).astype(np.float64)


def recon_noise_var(n: int, diam: float, snr_db: float) -> float:
    """Reconstruction sigma^2 in normalised-data units (R19):
    1/(rho_a 10^{SNR/10} + 1), rho_a = aperture fill fraction."""
    rho_a = float(aperture_mask(n, diam).mean())
    return 1.0 / (rho_a * 10.0 ** (snr_db / 10.0) + 1.0)


def flow_velocity(fg: float, fs: float, n: int, d_r0: float) -> float:
    """||v|| = (1/0.43)(f_g/f_s)(N/(D/r0)) pixels per sample."""
    return (1.0 / 0.43) * (fg / fs) * (n / d_r0)


def _ifft2c(x):
    return np.fft.fftshift(np.fft.ifft2(np.fft.ifftshift(x), norm="ortho"))


def kolmogorov_psd(m1: int, m2: int, r0_px: float) -> np.ndarray:
    """Phi(f) df1 df2 on the FFT grid (DC = 0)."""
    f1 = np.fft.fftfreq(m1)[:, None]
    f2 = np.fft.fftfreq(m2)[None, :]
    f = np.sqrt(f1 * f1 + f2 * f2)
    with np.errstate(divide="ignore"):
        phi = 0.023 * r0_px ** (-5.0 / 3.0) * f ** (-11.0 / 3.0)
    phi[0, 0] = 0.0
    return phi * (1.0 / m1) * (1.0 / m2)


def screen_coeffs(m1: int, m2: int, r0_px: float, rng: np.random.Generator) -> np.ndarray:
    """FFT-method screen coefficients (R22)."""
    z = rng.standard_normal((m1, m2)) + 1j * rng.standard_normal((m1, m2))
    return z * np.sqrt(kolmogorov_psd(m1, m2, r0_px))


def screen_from_coeffs(c: np.ndarray, shift=(0.0, 0.0)) -> np.ndarray:
    """phi(x) = Re sum_k c_k e^{2 pi i f_k . (x - shift)} on the periodic grid."""
    m1, m2 = c.shape
    if shift != (0.0, 0.0):
        f1 = np.fft.fftfreq(m1)[:, None]
        f2 = np.fft.fftfreq(m2)[None, :]
        c = c * np.exp(-2j * np.pi * (f1 * shift[0] + f2 * shift[1]))
    return np.real(np.fft.ifft2(c)) * (m1 * m2)


def structure_function_expected(m1: int, m2: int, r0_px: float, delta: Tuple[int, int]) -> float:
    """Exact discrete expectation D(Delta) = sum_k 2 Phi(f_k) df1 df2 (1 - cos 2 pi f_k . Delta) (R22)."""
    f1 = np.fft.fftfreq(m1)[:, None]
    f2 = np.fft.fftfreq(m2)[None, :]
    w = kolmogorov_psd(m1, m2, r0_px)
    return float(np.sum(2.0 * w * (1.0 - np.cos(2 * np.pi * (f1 * delta[0] + f2 * delta[1])))))


def remove_plane(phi: np.ndarray, a: np.ndarray) -> np.ndarray:
    """Remove piston, tip and tilt over the aperture, by lstsq."""
    n = phi.shape[0]
    x = np.broadcast_to(np.arange(n)[None, :] - n / 2, (n, n))
    yy = np.broadcast_to(np.arange(n)[:, None] - n / 2, (n, n))
    m = a > 0
    A = np.stack([np.ones(int(m.sum())), x[m], yy[m]], axis=1)
    coef, *_ = np.linalg.lstsq(A, phi[m], rcond=None)
    return phi - (coef[0] + coef[1] * x + coef[2] * yy)


def blurred_reflectance(n: int, sigma_b: float, rng: np.random.Generator, r_min: float = 1e-4) -> np.ndarray:
    """Blurred-uniform reflectance (configs; R23)."""
    u = rng.random((n, n))
    d = np.minimum(np.arange(n), n - np.arange(n)).astype(np.float64)
    k1 = np.exp(-d * d / (2.0 * sigma_b * sigma_b))
    k = k1[:, None] * k1[None, :]
    k /= k.sum()
    rb = np.real(np.fft.ifft2(np.fft.fft2(u) * np.fft.fft2(k)))
    rb = (rb - rb.min()) / (rb.max() - rb.min())
    return np.maximum(rb, r_min)


def bar_target(n: int, low: float = 0.02) -> np.ndarray:
    """Procedural bar-target reflectance for the paper-conditions check (a
    stand-in for a resolution chart, not a copy of one): groups of three bright
    bars, alternately horizontal and vertical, halving in size group by group,
    on a dark background (value `low`), scaled to the grid."""
    r = np.full((n, n), low)
    s = n / 256.0
    x0, y0, w = int(24 * s), int(24 * s), 16.0 * s
    k = 0
    while w >= 1.0 and y0 < n - 2:
        wi, L = max(1, int(round(w))), max(3, int(round(5 * w)))
        for b in range(3):
            if k % 2 == 0:  # horizontal bars
                r[y0 + 2 * b * wi:y0 + (2 * b + 1) * wi, x0:x0 + L] = 1.0
            else:           # vertical bars
                r[y0:y0 + L, x0 + 2 * b * wi:x0 + (2 * b + 1) * wi] = 1.0
        x0 += L + 3 * wi
        if x0 + 5 * w > n - 8 * s:
            x0, y0 = int(24 * s), y0 + L + 3 * wi
        w /= 1.41421356
        k += 1
    return r


def make_stream(cfg: dict, stream: int, frames: int = None, seed: int = SEED0,
                snr_db: float = None, d_r0: float = None, r_true: np.ndarray = None):
    """Synthesize one stream of a config.  Returns (y [T][N][N] complex64,
    phi_true [T][N][N] float32, r_true [N][N] float64)."""
    n = cfg["n"]
    diam = cfg["diam"]
    T = cfg["frames"] if frames is None else frames
    snr = cfg["snr_db"] if snr_db is None else snr_db
    sd = seed + stream
    a = aperture_mask(n, diam)
    if r_true is None:
        if cfg.get("scene") == "bars":
            r_true = bar_target(n)
        else:
            r_true = blurred_reflectance(n, cfg["sigma_b"], rng_for(sd, stream, 0, _P_SCENE))
    if d_r0 is None:
        if cfg.get("d_r0_range"):
            lo, hi = cfg["d_r0_range"]
            d_r0 = lo + (hi - lo) * rng_for(sd, stream, 0, _P_DR0).random()
        else:
            d_r0 = cfg["d_r0"]
    r0_px = diam / d_r0 if d_r0 > 0 else float("inf")
    v = cfg["flow"]
    if cfg["direction"] in ("random", "angle"):
        th = cfg["angle"] if cfg["direction"] == "angle" else 2 * np.pi * rng_for(sd, stream, 0, _P_DIR).random()
        m = 2 * n
        coeffs = screen_coeffs(m, m, r0_px, rng_for(sd, stream, 0, _P_SCREEN)) if d_r0 > 0 else None
    else:
        th = None
        m1, m2 = n, int(2 ** math.ceil(math.log2(n + v * T + 1)))
        coeffs = screen_coeffs(m1, m2, r0_px, rng_for(sd, stream, 0, _P_SCREEN)) if d_r0 > 0 else None
        strip = screen_from_coeffs(coeffs) if coeffs is not None else None
    sig_n2 = float(r_true.mean()) / 10.0 ** (snr / 10.0)
    y = np.empty((T, n, n), np.complex64)
    ph = np.empty((T, n, n), np.float32)
    for t in range(T):
        if coeffs is None:
            phi = np.zeros((n, n))
        elif th is not None:
            s = (t * v * math.sin(th), t * v * math.cos(th))
            phi = screen_from_coeffs(coeffs, s)[:n, :n]
        else:
            off = int(round(t * v))
            phi = strip[:, off:off + n]
        phi = remove_plane(phi, a)
        rs = rng_for(sd, stream, t, _P_SPECKLE)
        g = np.sqrt(r_true / 2.0) * (rs.standard_normal((n, n)) + 1j * rs.standard_normal((n, n)))
        rn = rng_for(sd, stream, t, _P_NOISE)
        w = math.sqrt(sig_n2 / 2.0) * (rn.standard_normal((n, n)) + 1j * rn.standard_normal((n, n)))
        y[t] = (a * np.exp(1j * phi) * _ifft2c(g) + w).astype(np.complex64)
        ph[t] = phi.astype(np.float32)
    return y, ph, r_true


def _stream_job(args):
    cfg, s, frames, seed = args
    y, ph, _ = make_stream(cfg, s, frames, seed)
    return s, y, ph


def make_batch(cfg: dict, streams: int = None, frames: int = None, seed: int = SEED0,
               first_stream: int = 0, workers: int = None, want_phi: bool = True):
    """Synthesize streams [first_stream, first_stream+streams) of a config as
    y [T][S][N][N] complex64 (+ phi_true [T][S][N][N] float32)."""
    S = cfg["streams"] if streams is None else streams
    T = cfg["frames"] if frames is None else frames
    n = cfg["n"]
    y = np.empty((T, S, n, n), np.complex64)
    ph = np.empty((T, S, n, n), np.float32) if want_phi else None
    jobs = [(cfg, first_stream + k, T, seed) for k in range(S)]
    if workers is None:
        workers = min(S, len(os.sched_getaffinity(0)))
    if workers <= 1 or S == 1:
        results = map(_stream_job, jobs)
    else:
        ex = ProcessPoolExecutor(max_workers=workers)
        results = ex.map(_stream_job, jobs)
    for s, ys, phs in results:
        k = s - first_stream
        y[:, k] = ys
        if want_phi:
            ph[:, k] = phs
    if workers > 1 and S > 1:
        ex.shutdown()
    return y, ph
