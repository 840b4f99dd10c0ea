"""Sequence metrics of DDH-MBIR runs (the step after the hot
path): per-frame peak Strehl series of several independent
simulations and their box-plot statistics (Fig. 3/4: "box plot over
10 simulations"), the first frame reaching a Strehl level ("Strehl >= 0.8
within 150 timeframes"), and the residual phase / PSF of a frame.
The estimator and the Strehl / residual evaluation run in libddh (ddh_step,
ddh_strehl, ddh_residual); this module only orders the calls and summarises
the per-frame scalars on the host."""
from __future__ import annotations

from typing import Dict, List, Optional

import numpy as np


def box_stats(series) -> Dict[str, np.ndarray]:
    """Per-frame box-plot statistics over simulations: series [sims][frames]
    -> min, q1, median, q3, max, mean (each [frames]); quartiles by linear
    interpolation between order statistics (numpy's default)."""
    s = np.asarray(series, dtype=np.float64)
    if s.ndim != 2 or s.shape[0] < 1:
        raise ValueError("series must be [simulations][frames]")
    q = np.percentile(s, [0, 25, 50, 75, 100], axis=0)
    return {"min": q[0], "q1": q[1], "median": q[2], "q3": q[3], "max": q[4], "mean": s.mean(axis=0)}


def first_crossing(series, level: float = 0.8) -> List[Optional[int]]:
    """Per simulation, the first frame index whose Strehl is >= level (None
    if never)."""
    out = []
    for row in np.asarray(series, dtype=np.float64):
        k = np.nonzero(row >= level)[0]
        out.append(int(k[0]) if k.size else None)
    return out


def strehl_sequence(cfg: dict, sims: int, frames: int, n_k: Optional[int] = None, k_b: int = 0, device: int = 0,
                    first_stream: int = 0, residual_at: Optional[int] = None, **params) -> Dict:
    """Run `sims` independent simulations of config `cfg` (one stream each,
    seeds by global stream id, the on-device synthesiser) for `frames` frames
    through ddh_step (after a bootstrap of k_b iterations on frame 0 when
    k_b > 0) and evaluate the peak Strehl of every frame (ddh_strehl).
    Returns the series [sims][frames], its box statistics, the first frames
    reaching 0.8 and, when residual_at is a frame index, that frame's residual
    phase and PSF (ddh_residual) as host arrays [sims][N][N]."""
    import torch

    import synth
    from . import sched
    from .ddh import DDH, DDHSynth
    n = cfg["n"]
    d_r0, vel = sched.stream_draws(cfg, first_stream, sims)
    z = DDHSynth(n, sims, d_r0=d_r0, velocity=vel, sigma_b=cfg["sigma_b"], snr_db=cfg["snr_db"], diam=cfg["diam"],
                 seed=20230504 + first_stream, device=device)
    y, phi_true = z.frames(0, frames, want_phi=True)
    params.setdefault("noise_var", synth.recon_noise_var(n, cfg["diam"], cfg["snr_db"]))
    params.setdefault("n_k", cfg.get("n_k", 1) if n_k is None else n_k)
    ctx = DDH(n, sims, device=device, aperture_diam=cfg["diam"], **params)
    t0 = 0
    if k_b > 0:
        ctx.bootstrap(y[0], k_b)
        t0 = 1
    phi_hat = torch.empty((frames, sims, n, n), dtype=torch.float32, device=y.device)
    if t0:
        phi_hat[0] = ctx.get_state()[1]
    ctx.step(y[t0:], phi_hat[t0:])
    S = np.empty((sims, frames))
    for s in range(sims):
        S[s] = ctx.strehl(phi_hat[:, s].contiguous(), phi_true[:, s].contiguous())
    out = {"strehl": S, "box": box_stats(S), "first_0_8": first_crossing(S, 0.8), "frames": frames, "sims": sims}
    if residual_at is not None:
        resid, psf, st = ctx.residual(phi_hat[residual_at].contiguous(), phi_true[residual_at].contiguous())
        out.update(residual_phase=resid.cpu().numpy(), residual_psf=psf.cpu().numpy(), residual_strehl=st)
    out["phi_hat"] = phi_hat
    out["phi_true"] = phi_true
    return out
