"""GPU parity: the CUDA path (through the C ABI) against the FP64 oracle on
the same seeded synthetic frames (-m gpu).

Tolerances (north_star):
  * per step, from identical FP32 state: max piston-removed wrapped |dphi|
    over the WHOLE grid <= 1e-3 rad; relative L2 r error <= 1e-4 and max
    pointwise relative r error <= 1e-3, over every pixel.  Where the r
    surrogate has two minima within FP32 evaluation precision of each other
    ("several results are correct") the oracle is guided to the
    minimiser the GPU chose (oracle.r_update_pixels(guide=...)): the GPU's
    choice must be one of the near-optimal candidates, and every later pixel
    of the sweep is then compared against the same history;
  * end to end: per-frame phi (piston-removed, wrapped, over the aperture)
    <= 1e-3 rad and per-frame Strehl within 0.01 absolute, on scenes where the
    estimate moves (a phi = 0 stand-in fails the same test);
  * stages (the streaming kernels' own device code): FFT relative L2 <= 3e-6
    (FP32 floor ~ eps log2 N), E-step <= 1e-6, ICDs <= 1e-5.
"""
import math
import os

import numpy as np
import pytest
import torch

import oracle.ddh_oracle as O
import synth

pytestmark = pytest.mark.gpu

DEV = torch.device("cuda:0")


@pytest.fixture(scope="module", autouse=True)
def _lib():
    from paper_2305_03284_b200 import build
    build.build()
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def DDH(*a, **k):
    from paper_2305_03284_b200 import DDH as _D
    return _D(*a, **k)


def crandn(g, *shape):
    return (g.standard_normal(shape) + 1j * g.standard_normal(shape)).astype(np.complex64)


def oracle_params(n, diam=None, **kw):
    p = O.OracleParams(n=n, aperture_diam=float(n if diam is None else diam))
    for k, v in kw.items():
        setattr(p, k, v)
    return p


PATH_FLAGS = {"stream": 0, "multipass": 2, "nochain": 0, False: 0, True: 2}


class chain_env:
    """Context manager: DDH contexts created inside use (on=True) or do not use
    (on=False) the on-chip chain at N = 64 (DDH_CHAIN, read by ddh_create)."""

    def __init__(self, on):
        self.on = on

    def __enter__(self):
        self.old = os.environ.get("DDH_CHAIN")
        os.environ["DDH_CHAIN"] = "1" if self.on else "0"

    def __exit__(self, *a):
        if self.old is None:
            os.environ.pop("DDH_CHAIN", None)
        else:
            os.environ["DDH_CHAIN"] = self.old


def gpu_kwargs(p: O.OracleParams, unfused=False):
    return dict(aperture_diam=p.aperture_diam, noise_var=p.noise_var, lam=p.lam, alpha=p.alpha, n_k=p.n_k, r_min=p.r_min, r_sigma=p.r_sigma,
                r_T=p.r_T, r_q=p.r_q, phi_sigma=p.phi_sigma, icd_sweeps=p.icd_sweeps, boot_period=p.boot_period,
                boot_alpha=p.boot_alpha, flags=(0 if p.tiptilt else 1) | PATH_FLAGS[unfused])


def phi_err(phi_g, phi_o, a, full=True):
    """max |wrap(phi_g - phi_o) - piston| over the grid (full) or the aperture;
    the piston is the circular mean of the difference over the aperture."""
    d = np.angle(np.exp(1j * (phi_g.astype(np.float64) - phi_o)))
    pist = np.angle(np.mean(np.exp(1j * d[a > 0])))
    d = np.angle(np.exp(1j * (d - pist)))
    return float(np.max(np.abs(d if full else d[a > 0])))


def r_errs(r_g, r_o):
    """(relative L2, max pointwise relative) over every pixel."""
    r_g = r_g.astype(np.float64)
    return (float(np.linalg.norm(r_g - r_o) / np.linalg.norm(r_o)),
            float(np.max(np.abs(r_g - r_o) / np.abs(r_o))))


def oracle_step_guided(r, phi, y, p, a, guides):
    """O.ddh_step (Fig. 1) with the r M-step of EM iteration k guided by
    guides[k] (the GPU's r after iteration k): the oracle's own functions in
    O.ddh_step's order, so that at a near-tie of an earlier iteration the oracle
    follows the GPU's valid choice too."""
    yhat = O.normalize(y)
    if p.tiptilt:
        phi = O.remove_tip_tilt(phi, a)
    u = O.adjoint(phi, yhat, a)
    r = O.warm_start(r, u, p.lam, p.alpha, p.r_min)
    for k in range(p.n_k):
        if k > 0:
            u = O.adjoint(phi, yhat, a)
        r, phi = O.em_update(r, phi, yhat, u, a, p, None, guides[k])
    return r, phi


def check_step(r_g, phi_g, r_in, phi_in, y, p, a, tol_phi=1e-3, tol_r=1e-4, tol_rmax=1e-3, guides=None):
    """One oracle step from (r_in, phi_in) on frame y against the GPU's
    (r_g, phi_g); near-tie pixels follow the GPU's valid choice (guided
    oracle; with N_k > 1, `guides` = the GPU's r after each iteration, from
    runs with N_k = 1, 2, ... from the same state).  Returns a dict of the
    errors and the tie / guided counts."""
    n = r_in.shape[0]
    gaps = np.full((n, n), np.inf)
    r_def, _, _ = O.ddh_step(r_in, phi_in, y, p, a, gaps)
    if guides is not None and p.n_k > 1:
        r_ref, phi_ref = oracle_step_guided(r_in, phi_in, y, p, a, [g.astype(np.float64) for g in guides])
    else:
        r_ref, phi_ref, st = O.ddh_step(r_in, phi_in, y, p, a, guide=r_g.astype(np.float64))
    ep = phi_err(phi_g, phi_ref, a)
    er, emax = r_errs(r_g, r_ref)
    res = {"phi": ep, "r_l2": er, "r_max": emax, "ties": int((gaps < 1e-6).sum()),
           "guided": int(np.sum(np.abs(r_ref - r_def) > 1e-6 * np.abs(r_def)))}
    if (p.n_k > 1 and guides is None) or p.icd_sweeps > 1:
        # the GPU's choices at near-ties of earlier sweeps (or, without per-
        # iteration guides, iterations) are not observable (only the final r
        # is), so the guide is exact for the last sweep only; a different valid
        # choice in an earlier sweep moves the pixels that later colour phases
        # reach from it.  The pointwise bound then holds for 99.9 % of the
        # pixels; the L2 bound covers every pixel.
        rel = np.abs(r_g.astype(np.float64) - r_ref) / np.abs(r_ref)
        res.update(r_max_all=emax, r_p999=float(np.quantile(rel, 0.999)))
        emax = res["r_max"] = res["r_p999"]
    assert ep <= tol_phi, res
    assert er <= tol_r and emax <= tol_rmax, res
    # validity at near-ties is by construction: the guide may only choose among
    # candidates within guide_tol of the minimum, so a GPU pixel in a worse
    # minimum differs from the guided oracle and fails the r bounds above
    return res


def frames(n, S, T, cfg="c1", **over):
    c = dict(synth.CONFIGS[cfg], n=n, diam=n, **over)
    y, ph = synth.make_batch(c, streams=S, frames=T, workers=1)
    return y, ph, c


# ------------------------------------------------------------------ stages


@pytest.mark.parametrize("flags", [pytest.param(0, id="stream"), pytest.param(2, id="multipass")])
@pytest.mark.parametrize("n", [64, 128, 256, 512, 1024])
def test_fft2c_parity(n, flags):
    g = np.random.default_rng(n)
    B = 3 if n <= 256 else 2
    x = crandn(g, B, n, n)
    ctx = DDH(n, 1, flags=flags)
    xt = torch.from_numpy(x).to(DEV)
    for inv in (False, True):
        out = ctx.test_fft2c(xt, inverse=inv).cpu().numpy()
        for b in range(B):
            ref = O.ifft2c(x[b].astype(np.complex128)) if inv else O.fft2c(x[b].astype(np.complex128))
            err = np.linalg.norm(out[b] - ref) / np.linalg.norm(ref)
            assert err < 3e-6, (n, inv, err)


@pytest.mark.parametrize("warm", [True, False])
def test_estep_stage_parity(warm):
    """S2's Eq. 3 + E-step epilogue (estep_px) against the oracle's warm_start
    and e_step on the same u, r_prev (FP32 inputs)."""
    n, B = 64, 3
    g = np.random.default_rng(17)
    u = (crandn(g, B, n, n) * 3).astype(np.complex64)
    r = (g.random((B, n, n)) * 2 + 1e-4).astype(np.float32)
    p = oracle_params(n, noise_var=0.287)
    ctx = DDH(n, 1, **gpu_kwargs(p))
    r0, mu, q = (t.cpu().numpy() for t in ctx.test_estep(torch.from_numpy(u).to(DEV), torch.from_numpy(r).to(DEV), warm))
    for b in range(B):
        ub, rb = u[b].astype(np.complex128), r[b].astype(np.float64)
        r_ref = O.warm_start(rb, ub, p.lam, p.alpha, p.r_min) if warm else rb
        mu_ref, _, q_ref = O.e_step(ub, r_ref, p.noise_var)
        assert np.max(np.abs(r0[b] - r_ref) / r_ref) < 1e-6
        assert np.max(np.abs(mu[b] - mu_ref)) < 1e-6 * np.max(np.abs(mu_ref))
        assert np.max(np.abs(q[b] - q_ref) / q_ref) < 1e-6


def _realistic_rq(n, seed):
    """(r, q) from an oracle E-step on a synthetic frame (FP32-rounded)."""
    y, _, c = frames(n, 1, 1, "c1")
    p = oracle_params(n, noise_var=synth.recon_noise_var(n, n, 10.0))
    a = O.aperture_of(p)
    g = np.random.default_rng(seed)
    r = (g.random((n, n)) * 0.5 + 0.01)
    u = O.adjoint(np.zeros((n, n)), O.normalize(y[0, 0].astype(np.complex128)), a)
    r = O.warm_start(r, u, 0.45, 0.025, 1e-4)
    _, _, q = O.e_step(u, r, p.noise_var)
    return r.astype(np.float32), q.astype(np.float32), p


@pytest.mark.parametrize("flags", [pytest.param(0, id="stream"), pytest.param(2, id="multipass")])
@pytest.mark.parametrize("n,kind,sweeps", [(64, "random", 1), (256, "random", 1), (128, "realistic", 1),
                                           (256, "realistic", 1), (128, "random", 2)])
def test_ricd_stage_parity(n, kind, sweeps, flags):
    g = np.random.default_rng(7 + n)
    B = 2
    if kind == "random":
        r = (g.random((B, n, n)) * 2 + 1e-3).astype(np.float32)
        q = (g.random((B, n, n)) * 2 + 1e-4).astype(np.float32)
        p = oracle_params(n)
    else:
        rq = [_realistic_rq(n, s) for s in range(B)]
        r = np.stack([x[0] for x in rq])
        q = np.stack([x[1] for x in rq])
        p = rq[0][2]
    p.icd_sweeps = sweeps
    ctx = DDH(n, B, **dict(gpu_kwargs(p), flags=flags))
    out = ctx.test_ricd(torch.from_numpy(r).to(DEV), torch.from_numpy(q).to(DEV)).cpu().numpy()
    outs = [out]
    if sweeps > 1:
        # every sweep's output, from a one-sweep ctx applied sweep after sweep (the
        # multi-sweep call runs exactly these launches: checked bit for bit)
        c1 = DDH(n, B, **dict(gpu_kwargs(p), flags=flags, icd_sweeps=1))
        cur, outs = torch.from_numpy(r).to(DEV), []
        for _ in range(sweeps):
            cur = c1.test_ricd(cur, torch.from_numpy(q).to(DEV))
            outs.append(cur.cpu().numpy())
        assert np.array_equal(outs[-1], out)
    p1 = O.OracleParams(**{**p.__dict__, "icd_sweeps": 1})
    for b in range(B):
        ref = r[b].astype(np.float64)
        for k in range(sweeps):  # follow the GPU at near-ties, sweep by sweep
            ref = O.r_icd(ref, q[b].astype(np.float64), p1, guide=outs[k][b].astype(np.float64))
        e, emax = r_errs(out[b], ref)
        assert e < 1e-5 and emax < 1e-3, (b, e, emax)


@pytest.mark.parametrize("n,B,sweeps", [(64, 300, 1), (256, 20, 1), (256, 20, 2), (512, 2, 1), (512, 2, 2),
                                         (1024, 1, 1)])
def test_ricd_large_launch_stage_parity(n, B, sweeps):
    """The r-ICD kernels of large launches against the oracle's colour-ordered
    sweep, every pixel of the first and last stream: the four colour passes
    (N <= 256 with >= 2 64-tiles per SM) and the two row-parity kernels
    (colours 0+1, then 2+3; N >= 512 at every launch size, 256- and
    512-thread CTAs)."""
    g = np.random.default_rng(11 + n)
    r = (g.random((B, n, n)) * 2 + 1e-3).astype(np.float32)
    q = (g.random((B, n, n)) * 2 + 1e-4).astype(np.float32)
    p = oracle_params(n)
    p.icd_sweeps = sweeps
    ctx = DDH(n, B, **gpu_kwargs(p))
    out = ctx.test_ricd(torch.from_numpy(r).to(DEV), torch.from_numpy(q).to(DEV)).cpu().numpy()
    outs = [out]
    if sweeps > 1:
        c1 = DDH(n, B, **dict(gpu_kwargs(p), icd_sweeps=1))
        cur, outs = torch.from_numpy(r).to(DEV), []
        for _ in range(sweeps):
            cur = c1.test_ricd(cur, torch.from_numpy(q).to(DEV))
            outs.append(cur.cpu().numpy())
        assert np.array_equal(outs[-1], out)
    p1 = O.OracleParams(**{**p.__dict__, "icd_sweeps": 1})
    for b in (0, B - 1):
        ref = r[b].astype(np.float64)
        for k in range(sweeps):
            ref = O.r_icd(ref, q[b].astype(np.float64), p1, guide=outs[k][b].astype(np.float64))
        e, emax = r_errs(out[b], ref)
        assert e < 1e-5 and emax < 1e-3, (b, e, emax)


def test_ricd_prior_off_is_clamp():
    n = 64
    g = np.random.default_rng(3)
    r = g.random((1, n, n)).astype(np.float32)
    q = (g.random((1, n, n)) * 1e-3).astype(np.float32)
    ctx = DDH(n, 1, r_sigma=0.0)  # streaming S3 with the prior off
    out = ctx.test_ricd(torch.from_numpy(r).to(DEV), torch.from_numpy(q).to(DEV)).cpu().numpy()
    assert np.array_equal(out[0], np.maximum(q[0], np.float32(1e-4)))


@pytest.mark.parametrize("flags", [pytest.param(0, id="stream"), pytest.param(2, id="multipass")])
@pytest.mark.parametrize("n,prior,sweeps", [(64, True, 1), (256, True, 1), (128, False, 1), (128, True, 2)])
def test_phiicd_stage_parity(n, prior, sweeps, flags):
    g = np.random.default_rng(11 + n)
    B = 2
    phi = (g.standard_normal((B, n, n)) * 2).astype(np.float32)
    c = (g.random((B, n, n)) * 5).astype(np.float32)
    c[:, :, : n // 8] = 0.0  # pixels outside an aperture: prior only
    th = g.uniform(-math.pi, math.pi, (B, n, n)).astype(np.float32)
    p = oracle_params(n, phi_sigma=0.5 if prior else 0.0, icd_sweeps=sweeps)
    ctx = DDH(n, B, **dict(gpu_kwargs(p), flags=flags))
    out = ctx.test_phiicd(*(torch.from_numpy(v).to(DEV) for v in (phi, c, th))).cpu().numpy()
    for b in range(B):
        ref = O.phi_icd(phi[b].astype(np.float64), c[b].astype(np.float64), th[b].astype(np.float64), p)
        d = np.angle(np.exp(1j * (out[b] - ref)))
        assert np.max(np.abs(d)) < 2e-4, np.max(np.abs(d))


# -------------------------------------------------------------- one step


def _step_parity(n, S, p, cfg="c1", chunk=0, pre_boot=8, seed_frames=3, unfused=False, **frame_over):
    y, ph, c = frames(n, S, seed_frames, cfg, **frame_over)
    a = O.aperture_of(p)
    # a realistic state: oracle bootstrap on frame 0, rounded to FP32
    orc = O.DDHOracle(p, S)
    st = orc.bootstrap(y[0], pre_boot)
    assert not st.any()
    r32 = orc.r.astype(np.float32)
    p32 = orc.phi.astype(np.float32)
    orc.set_state(r32, p32, 1)
    if unfused == "nochain" and n != 64:
        pytest.skip("the on-chip chain exists at N = 64 only")
    with chain_env(unfused != "nochain"):
        ctx = DDH(n, S, chunk_streams=chunk, **gpu_kwargs(p, unfused))
    ctx.set_state(torch.from_numpy(r32).to(DEV), torch.from_numpy(p32).to(DEV), 1)
    yt = torch.from_numpy(y[1:2]).to(DEV)
    phi_o = torch.empty((1, S, n, n), device=DEV)
    r_o = torch.empty_like(phi_o)
    status = torch.empty((1, S), dtype=torch.uint8, device=DEV)
    ctx.step(yt, phi_o, r_o, status)
    torch.cuda.synchronize()
    phi_g = phi_o.cpu().numpy()[0]
    r_g = r_o.cpu().numpy()[0]
    assert status.cpu().numpy().sum() == 0
    # the state matches the per-frame outputs
    r_s, phi_s, fi = ctx.get_state()
    assert fi == 2
    assert np.array_equal(r_s.cpu().numpy(), r_g) and np.array_equal(phi_s.cpu().numpy(), phi_g)
    guides = None
    if p.n_k > 1:  # the GPU's r after EM iterations 1 .. N_k - 1: the same step with fewer iterations
        guides = []
        for k in range(1, p.n_k):
            pk = O.OracleParams(**{**p.__dict__, "n_k": k})
            with chain_env(unfused != "nochain"):
                ck = DDH(n, S, chunk_streams=chunk, **gpu_kwargs(pk, unfused))
            ck.set_state(torch.from_numpy(r32).to(DEV), torch.from_numpy(p32).to(DEV), 1)
            rk = torch.empty_like(r_o)
            ck.step(yt, None, rk)
            guides.append(rk.cpu().numpy()[0])
        guides.append(r_g)
    worst = (0.0, 0.0)
    for s in range(S):
        res = check_step(r_g[s], phi_g[s], orc.r[s], orc.phi[s], y[1, s], p, a,
                         guides=None if guides is None else [g[s] for g in guides])
        worst = (max(worst[0], res["phi"]), max(worst[1], res["r_l2"]))
    return worst


# the implementations of the EM iteration: streaming (default; at N = 64 the
# on-chip chain), multi-pass, and at N = 64 the streaming kernels without the chain
PATHS = [pytest.param("stream", id="stream"), pytest.param("multipass", id="multipass"),
         pytest.param("nochain", id="nochain")]


@pytest.mark.parametrize("unfused", PATHS)
@pytest.mark.parametrize("n,S,chunk", [(64, 2, 0), (128, 3, 2), (256, 2, 0), (512, 1, 0)])
def test_step_parity_priors_on(n, S, chunk, unfused):
    p = oracle_params(n, noise_var=synth.recon_noise_var(n, n, 10.0))
    _step_parity(n, S, p, chunk=chunk, unfused=unfused, pre_boot=8 if n <= 256 else 2)


@pytest.mark.parametrize("unfused", PATHS)
def test_step_parity_priors_off(unfused):
    n = 64
    p = oracle_params(n, noise_var=synth.recon_noise_var(n, n, 10.0), r_sigma=0.0, phi_sigma=0.0)
    _step_parity(n, 2, p, unfused=unfused)


@pytest.mark.parametrize("unfused", PATHS)
def test_step_parity_nk2_two_sweeps_no_tiptilt(unfused):
    n = 128
    p = oracle_params(n, noise_var=0.2, n_k=2, icd_sweeps=2, tiptilt=False)
    _step_parity(n, 2, p, unfused=unfused)


@pytest.mark.parametrize("unfused", PATHS)
def test_step_parity_masked_aperture(unfused):
    n = 64
    p = oracle_params(n, diam=50, noise_var=0.15)
    _step_parity(n, 2, p, unfused=unfused)


@pytest.mark.parametrize("n_k,tiptilt,priors,sweeps", [(1, True, True, 1), (2, True, True, 1), (4, True, True, 1),
                                                         (8, True, True, 1), (2, False, True, 2), (2, True, False, 1)])
def test_chain_step_parity(n_k, tiptilt, priors, sweeps):
    """The on-chip chain (one CTA per stream, all N_k EM
    iterations in shared memory) against the oracle's step, every pixel."""
    n = 64
    p = oracle_params(n, noise_var=synth.recon_noise_var(n, n, 10.0), n_k=n_k, tiptilt=tiptilt, icd_sweeps=sweeps,
                      **({} if priors else dict(r_sigma=0.0, phi_sigma=0.0)))
    _step_parity(n, 3, p)


def test_chain_and_streaming_kernels_agree():
    """At N = 64 the chain and the streaming kernels compute the same steps
    (FP32 rounding order differs: parity tolerance, 4 frames, N_k = 2)."""
    n, S, T = 64, 3, 4
    y, _, _ = frames(n, S, T)
    yt = torch.from_numpy(y).to(DEV)
    outs = []
    for on in (True, False):
        with chain_env(on):
            ctx = DDH(n, S, noise_var=0.2, n_k=2)
        l0 = ctx.kernel_launches
        po = torch.empty((T, S, n, n), device=DEV)
        ro = torch.empty_like(po)
        ctx.step(yt, po, ro)
        outs.append((po.cpu().numpy(), ro.cpu().numpy(), ctx.kernel_launches - l0))
    assert outs[0][2] == T  # one chain launch per frame
    a = O.aperture(n, n)
    for t in range(T):
        for s in range(S):
            assert phi_err(outs[0][0][t, s], outs[1][0][t, s].astype(np.float64), a) < 1e-3
            assert np.linalg.norm(outs[0][1][t, s] - outs[1][1][t, s]) / np.linalg.norm(outs[1][1][t, s]) < 1e-3


def test_chain_launch_groups_bit_exact():
    """The chain over ragged launch groups (5 streams in groups of 2) equals one
    group bit for bit (one CTA per stream, no cross-stream arithmetic)."""
    n, S, T = 64, 5, 3
    y, _, _ = frames(n, S, T)
    yt = torch.from_numpy(y).to(DEV)
    outs = []
    with chain_env(True):
        for chunk in (0, 2):
            ctx = DDH(n, S, noise_var=0.1, n_k=2, chunk_streams=chunk)
            po = torch.empty((T, S, n, n), device=DEV)
            ro = torch.empty_like(po)
            ctx.step(yt, po, ro)
            outs.append((po, ro))
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])


def test_chain_selection_rule():
    """The library's automatic choice at N = 64 (use_chain, ddh_api.cpp): the
    six kernels at N_k = 1 (2 streams: far from a full wave), the chain (one
    launch per frame) at N_k >= 2."""
    n, S = 64, 2
    y, _, _ = frames(n, S, 1)
    yt = torch.from_numpy(y).to(DEV)
    old = os.environ.pop("DDH_CHAIN", None)
    try:
        for nk, per_frame in ((1, 6), (2, 1), (4, 1)):
            ctx = DDH(n, S, noise_var=0.1, n_k=nk)
            l0 = ctx.kernel_launches
            ctx.step(yt[:1])
            assert ctx.kernel_launches - l0 == per_frame, (nk, ctx.kernel_launches - l0)
    finally:
        if old is not None:
            os.environ["DDH_CHAIN"] = old


# -------------------------------------------------- bootstrap and static


def test_bootstrap_and_static_parity():
    n, S = 64, 2
    p = oracle_params(n, noise_var=synth.recon_noise_var(n, n, 10.0), boot_period=3)
    y, _, _ = frames(n, S, 2)
    a = O.aperture_of(p)
    ctx = DDH(n, S, **gpu_kwargs(p))
    ctx.bootstrap(torch.from_numpy(y[0]).to(DEV), 5)
    r_g, phi_g, fi = ctx.get_state()
    assert fi == 1
    for s in range(S):
        r_ref, phi_ref, _ = O.bootstrap(y[0, s], p, 5, a)
        # 5 chained iterations from a cold start: FP32 drift stays far inside the per-step bar
        assert phi_err(phi_g[s].cpu().numpy(), phi_ref, a) < 1e-3
        assert r_errs(r_g[s].cpu().numpy(), r_ref)[0] < 1e-3
    phi_o = torch.empty((2, S, n, n), device=DEV)
    ctx.static(torch.from_numpy(y).to(DEV), 4, phi_out=phi_o)
    for t in range(2):
        for s in range(S):
            _, phi_ref, _ = O.static_dhmbir(y[t, s], p, 4, a)
            assert phi_err(phi_o[t, s].cpu().numpy(), phi_ref, a) < 1e-3


# ---------------------------------------------------------- end to end


def _e2e(cfg, T, n_k=1, k_b=0, streams=1):
    """Both sides run free from their own state over T frames of config `cfg`
    (bootstrap on frame 0 when k_b > 0, else cold start at frame 0).  Returns
    per-frame errors and Strehl series (GPU phi, oracle phi, phi = 0)."""
    n = cfg["n"]
    y, ph = synth.make_batch(cfg, streams=streams, frames=T, workers=1)
    p = oracle_params(n, diam=cfg["diam"], noise_var=synth.recon_noise_var(n, cfg["diam"], cfg["snr_db"]), n_k=n_k)
    a = O.aperture_of(p)
    ctx = DDH(n, streams, **gpu_kwargs(p))
    t0 = 0
    if k_b > 0:
        ctx.bootstrap(torch.from_numpy(y[0]).to(DEV), k_b)
        t0 = 1
    phi_o = torch.empty((T - t0, streams, n, n), device=DEV)
    r_o = torch.empty_like(phi_o)
    ctx.step(torch.from_numpy(np.ascontiguousarray(y[t0:])).to(DEV), phi_o, r_o)
    s_api = [ctx.strehl(phi_o[:, s].contiguous(), torch.from_numpy(np.ascontiguousarray(ph[t0:, s])).to(DEV))
             for s in range(streams)]
    phi_g, r_g = phi_o.cpu().numpy(), r_o.cpu().numpy()
    out = []
    for s in range(streams):
        if k_b > 0:
            r, phi, _ = O.bootstrap(y[0, s], p, k_b, a)
        else:
            r, phi = np.full((n, n), p.r_min), np.zeros((n, n))
        for t in range(t0, T):
            r, phi, _ = O.ddh_step(r, phi, y[t, s], p, a)
            k = t - t0
            out.append(dict(t=t, s=s, phi=phi_err(phi_g[k, s], phi, a, full=False),
                            phi_zero=phi_err(np.zeros((n, n), np.float32), phi, a, full=False),
                            r=r_errs(r_g[k, s], r)[0],
                            S_ref=O.strehl(phi, ph[t, s], a), S_gpu=O.strehl(phi_g[k, s], ph[t, s], a),
                            S_zero=O.strehl(np.zeros((n, n)), ph[t, s], a), S_api=s_api[s][k]))
    return out


def _assert_e2e(rows, tol_phi=1e-3, tol_r=1e-3, discriminate_strehl=True):
    worst = {k: max(abs(r_[k]) for r_ in rows) for k in ("phi", "r")}
    dS = max(abs(r_["S_gpu"] - r_["S_ref"]) for r_ in rows)
    dS0 = max(abs(r_["S_zero"] - r_["S_ref"]) for r_ in rows)
    dapi = max(abs(r_["S_gpu"] - r_["S_api"]) for r_ in rows)
    info = dict(worst, dS=dS, dS_zero=dS0, d_api=dapi)
    assert worst["phi"] <= tol_phi and worst["r"] <= tol_r and dS <= 0.01, info
    assert dapi < 1e-5, info  # ddh_strehl vs the oracle's Strehl on the same phi-hat
    # the test discriminates: a phi-hat = 0 stand-in fails the phi bound (and,
    # where the estimate moves the Strehl, the Strehl bound too)
    assert max(r_["phi_zero"] for r_ in rows) > 10 * tol_phi, info
    if discriminate_strehl:
        assert dS0 > 0.01, info
    return info


def test_end_to_end_c1():
    """BASELINE config 1: 64x64, bootstrap (K_b = 50) then 1 EM iteration per
    frame, 16 frames; phi-hat and r-hat compared on every frame."""
    cfg = synth.CONFIGS["c1"]
    _assert_e2e(_e2e(cfg, cfg["frames"], k_b=cfg["k_b"]), discriminate_strehl=False)


def test_end_to_end_bar_scene_paper_conditions():
    """The paper's conditions (256^2, D/r0 = 10, |v| = 0.595 px per
    frame, SNR 10 dB) on a scene with support (synth bar target), cold start,
    N_k = 1, 60 frames: the estimate moves the Strehl from ~0.055 to ~0.12, so
    phi-hat = 0 misses the oracle's Strehl by > 0.01 and the test can fail."""
    _assert_e2e(_e2e(synth.CONFIGS["paper"], 60))


def test_end_to_end_c2():
    """BASELINE config 2: 256^2, 1 stream, 200 frames, SNR 5 dB, cold start,
    N_k = 1: phi-hat and r-hat on every frame."""
    cfg = synth.CONFIGS["c2"]
    _assert_e2e(_e2e(cfg, cfg["frames"]), discriminate_strehl=False)


def test_strehl_parity():
    n = 256
    a = O.aperture(n, n)
    g = np.random.default_rng(5)
    B = 3
    hat = np.stack([synth.screen_from_coeffs(synth.screen_coeffs(n, n, n / 3.0, g)) for _ in range(B)]).astype(np.float32)
    tru = (g.standard_normal((B, n, n)) * 0.1).astype(np.float32)
    ctx = DDH(n, 1)
    out = ctx.strehl(torch.from_numpy(hat).to(DEV), torch.from_numpy(tru).to(DEV))
    for b in range(B):
        assert abs(out[b] - O.strehl(hat[b], tru[b], a)) < 1e-5
    zero = torch.zeros((1, n, n), device=DEV)
    assert abs(ctx.strehl(zero, zero)[0] - 1.0) < 1e-6


# ----------------------------------------------- full BASELINE sizes, sampled


def test_c3_full_size_sampled_streams():
    """BASELINE config 3 shape (256^2, 64 streams, launch groups as bench.py):
    one cold-start step on all 64 streams; streams 0 and 63 checked against
    the oracle."""
    cfg = synth.CONFIGS["c3"]
    n, S = cfg["n"], cfg["streams"]
    y, _ = synth.make_batch(cfg, streams=S, frames=1, want_phi=False)
    p = oracle_params(n, noise_var=synth.recon_noise_var(n, n, cfg["snr_db"]))
    a = O.aperture_of(p)
    ctx = DDH(n, S, **gpu_kwargs(p))
    phi_o = torch.empty((1, S, n, n), device=DEV)
    r_o = torch.empty_like(phi_o)
    ctx.step(torch.from_numpy(y).to(DEV), phi_o, r_o)
    for s in (0, S - 1):
        check_step(r_o[0, s].cpu().numpy(), phi_o[0, s].cpu().numpy(), np.full((n, n), p.r_min),
                   np.zeros((n, n)), y[0, s], p, a)


@pytest.mark.parametrize("cfgname,S", [("c4", 6), ("c5", 1)])
def test_large_grid_sampled(cfgname, S):
    cfg = synth.CONFIGS[cfgname]
    n = cfg["n"]
    y, _ = synth.make_batch(cfg, streams=S, frames=1, want_phi=False, workers=1)
    p = oracle_params(n, noise_var=synth.recon_noise_var(n, n, cfg["snr_db"]))
    a = O.aperture_of(p)
    ctx = DDH(n, S, **gpu_kwargs(p))
    phi_o = torch.empty((1, S, n, n), device=DEV)
    r_o = torch.empty_like(phi_o)
    ctx.step(torch.from_numpy(y).to(DEV), phi_o, r_o)
    s = S - 1
    check_step(r_o[0, s].cpu().numpy(), phi_o[0, s].cpu().numpy(), np.full((n, n), p.r_min),
               np.zeros((n, n)), y[0, s], p, a)


# ------------------------------------------------ edge cases / invariants


@pytest.mark.parametrize("chain", [True, False])
def test_degenerate_frame_keeps_state(chain):
    n, S = 64, 2
    y, _, _ = frames(n, S, 2)
    with chain_env(chain):
        ctx = DDH(n, S, noise_var=0.1)
    ctx.bootstrap(torch.from_numpy(y[0]).to(DEV), 3)
    r0, phi0, _ = ctx.get_state()
    yy = y[1:2].copy()
    yy[0, 1] = 0.7 - 0.2j  # constant frame on stream 1
    status = torch.empty((1, S), dtype=torch.uint8, device=DEV)
    ctx.step(torch.from_numpy(yy).to(DEV), status=status)
    r1, phi1, fi = ctx.get_state()
    assert status.cpu().tolist() == [[0, 1]]
    assert torch.equal(r1[1], r0[1]) and torch.equal(phi1[1], phi0[1])
    assert not torch.equal(phi1[0], phi0[0])
    assert fi == 2


@pytest.mark.parametrize("chain", [True, False])
def test_state_continuity_bit_exact(chain):
    n, S = 64, 2
    y, _, _ = frames(n, S, 6)
    yt = torch.from_numpy(y).to(DEV)
    with chain_env(chain):
        a = DDH(n, S, noise_var=0.1)
        b = DDH(n, S, noise_var=0.1)
        c = DDH(n, S, noise_var=0.1)
    pa = torch.empty((6, S, n, n), device=DEV)
    pb = torch.empty_like(pa)
    a.step(yt, pa)
    b.step(yt[:2].contiguous(), pb[:2])
    b.step(yt[2:].contiguous(), pb[2:])
    assert torch.equal(pa, pb)
    # one call per frame (no S0 prefetch inside a call; RemoveTipTilt sums from
    # the previous S5) and a checkpoint / resume in the middle (sums recomputed
    # by S0): the same bits
    pc = torch.empty_like(pa)
    for t in range(6):
        c.step(yt[t:t + 1].contiguous(), pc[t:t + 1])
        if t == 2:
            r_, p_, f_ = c.get_state()
            c.set_state(r_.clone(), p_.clone(), f_)
    assert torch.equal(pa, pc)


def test_call_graphs_bit_exact():
    """Multi-frame calls replay captured chunk graphs (include/ddh.h
    DDH_F_CALL_GRAPHS): graphs captured with stand-in buffers and replayed on other
    buffers, chunks of both state parities and a direct remainder give the
    same bits as direct launches (phi-hat, r-hat, status, state), with lanes,
    the r-ICD side stream and the fused next-frame sums in play."""
    from paper_2305_03284_b200.ddh import DDH_F_CALL_GRAPHS
    n, S, T = 256, 40, 19
    y, _, _ = frames(n, S, T)
    yt = torch.from_numpy(y).to(DEV)
    res = []
    for flags in (0, DDH_F_CALL_GRAPHS):
        ctx = DDH(n, S, noise_var=0.1, flags=flags)
        po = torch.empty((T, S, n, n), device=DEV)
        ro = torch.empty_like(po)
        st = torch.empty((T, S), dtype=torch.uint8, device=DEV)
        ctx.step(yt[:9].contiguous(), po[:9], ro[:9], st[:9])          # chunk (captured) + 1 frame
        ctx.step(yt[9:].contiguous(), po[9:], ro[9:], st[9:])          # other parity: captured; then 2 frames
        po2 = torch.empty((8, S, n, n), device=DEV)
        ctx.step(yt[:8].contiguous(), po2)                             # replay on new buffers, phi only
        r_, p_, f_ = ctx.get_state()
        res.append((po, ro, st, po2, r_, p_, f_))
    for a, b in zip(res[0], res[1]):
        if isinstance(a, torch.Tensor):
            assert torch.equal(a, b)
        else:
            assert a == b


def test_adaptive_call_graphs_bit_exact(monkeypatch):
    """A long multi-frame call that finds the device waiting for the host switches
    to chunk graphs by itself (include/ddh.h DDH_F_NO_ADAPTIVE_GRAPHS).  Test mode
    (DDH_ADAPTIVE_GRAPHS=2: every check counts as starved) forces the switch at
    frame 3 of a 45-frame call: direct frames, a frame without prefetch, five chunk
    graphs and a direct tail give the bits of direct launches, with fewer host
    launches; with the feature off, or a call too short, nothing is replayed."""
    n, S, T = 128, 24, 45
    y, _, _ = frames(n, S, 5)
    yt = torch.from_numpy(y).to(DEV).repeat(9, 1, 1, 1).contiguous()
    res, launches = [], []
    for mode in ("0", "2", "1"):
        monkeypatch.setenv("DDH_ADAPTIVE_GRAPHS", mode)
        ctx = DDH(n, S, noise_var=0.1, lanes=2)
        po = torch.empty((T, S, n, n), device=DEV)
        ro = torch.empty_like(po)
        st = torch.empty((T, S), dtype=torch.uint8, device=DEV)
        l0 = ctx.kernel_launches
        ctx.step(yt, po, ro, st)
        torch.cuda.synchronize()
        launches.append(ctx.kernel_launches - l0)
        short0 = ctx.kernel_launches
        ctx.step(yt[:20], po[:20])  # too short to switch (at most four chunks left at frame 2)
        short = ctx.kernel_launches - short0
        po3 = torch.empty((T, S, n, n), device=DEV)
        ctx.step(yt, po3)  # after a switch: the next long calls start on graphs at frame 0
        r_, p_, f_ = ctx.get_state()
        res.append((po, ro, st, po3, r_, p_, f_, short))
    for other in res[1:]:
        for a, b in zip(res[0], other):
            assert torch.equal(a, b) if isinstance(a, torch.Tensor) else a == b
    assert launches[1] != launches[0]  # five chunks came from graphs (+1 descriptor launch each)


def test_sharding_and_launch_groups_bit_exact():
    """Streams are independent: the per-stream results do not depend on how
    streams are grouped into launches or split over contexts (G-GPU sharding
    emulated by two ctxs on one device)."""
    n, S = 128, 4
    y, _, _ = frames(n, S, 3)
    yt = torch.from_numpy(y).to(DEV)
    outs = []
    for chunk, lanes in ((1, 1), (4, 1), (4, 3), (4, 4)):
        ctx = DDH(n, S, noise_var=0.1, chunk_streams=chunk, lanes=lanes)
        po = torch.empty((3, S, n, n), device=DEV)
        ro = torch.empty_like(po)
        ctx.step(yt, po, ro)
        outs.append((po, ro))
    for po, ro in outs[1:]:
        assert torch.equal(outs[0][0], po) and torch.equal(outs[0][1], ro)
    outs = [o[0] for o in outs]
    halves = []
    for h in range(2):
        ctx = DDH(n, 2, noise_var=0.1)
        po = torch.empty((3, 2, n, n), device=DEV)
        ctx.step(yt[:, 2 * h:2 * h + 2].contiguous(), po)
        halves.append(po)
    assert torch.equal(torch.cat(halves, 1), outs[0])


@pytest.mark.parametrize("chain", [False, True])
def test_step_host_matches_device_path(chain):
    n, S, T = 64, 2, 3
    y, _, _ = frames(n, S, T)
    with chain_env(chain):
        a = DDH(n, S, noise_var=0.1)
        b = DDH(n, S, noise_var=0.1)
    pa = torch.empty((T, S, n, n), device=DEV)
    a.step(torch.from_numpy(y).to(DEV), pa)
    yh = torch.from_numpy(y).pin_memory()
    pb = torch.empty((T, S, n, n)).pin_memory()
    rb = torch.empty((T, S, n, n)).pin_memory()
    sb = torch.empty((T, S), dtype=torch.uint8).pin_memory()
    b.step_host(yh, pb, rb, sb)
    assert torch.equal(pa.cpu(), pb)
    assert sb.sum().item() == 0


def test_step_host_async_pipeline_matches_device_path():
    """ddh_step_host_async: consecutive calls continue one copy/compute
    pipeline; after ddh_sync the host outputs (phi-hat, r-hat, status) equal
    the device path's, frame for frame."""
    n, S, T = 64, 2, 5
    y, _, _ = frames(n, S, T)
    a = DDH(n, S, noise_var=0.1)
    b = DDH(n, S, noise_var=0.1)
    pa = torch.empty((T, S, n, n), device=DEV)
    ra = torch.empty_like(pa)
    a.step(torch.from_numpy(y).to(DEV), pa, ra)
    yh = torch.from_numpy(y).pin_memory()
    pb = torch.empty((T, S, n, n)).pin_memory()
    rb = torch.empty((T, S, n, n)).pin_memory()
    sb = torch.full((T, S), 7, dtype=torch.uint8).pin_memory()
    for t0, t1 in ((0, 2), (2, 3), (3, 5)):  # calls of 2, 1, 2 frames, one pipeline
        b.step_host(yh[t0:t1], pb[t0:t1], rb[t0:t1], sb[t0:t1], asynchronous=True)
    b.sync()
    assert torch.equal(pa.cpu(), pb) and torch.equal(ra.cpu(), rb)
    assert sb.sum().item() == 0 and b.get_state()[2] == T


def test_kernel_launch_count_and_empty_call():
    n, S = 64, 1
    with chain_env(False):
        ctx = DDH(n, S, noise_var=0.1)
    l0 = ctx.kernel_launches
    ctx.step(torch.empty((0, S, n, n), dtype=torch.complex64, device=DEV))
    assert ctx.kernel_launches == l0
    y, _, _ = frames(n, S, 1)
    ctx.step(torch.from_numpy(y).to(DEV))
    assert ctx.kernel_launches - l0 == 6  # streaming: S0 S1 S2 S3 S4 S5
    with pytest.raises(Exception, match="retired"):
        DDH(n, S, noise_var=0.1, flags=4)  # the cluster path is gone
    u = DDH(n, S, noise_var=0.1, flags=2)
    l0 = u.kernel_launches
    u.step(torch.from_numpy(y).to(DEV))
    assert u.kernel_launches - l0 == 6  # unfused: K0 K1 K2a K2b K3a K3b


def test_fused_and_unfused_paths_agree():
    """The streaming and multi-pass kernels compute the same step
    (FP32 rounding order differs: compare at the parity tolerance, 3 frames)."""
    n, S = 256, 2
    y, _, _ = frames(n, S, 3)
    yt = torch.from_numpy(y).to(DEV)
    outs = []
    for flags in (2, 0):
        ctx = DDH(n, S, noise_var=0.2, flags=flags)
        po = torch.empty((3, S, n, n), device=DEV)
        ro = torch.empty_like(po)
        ctx.step(yt, po, ro)
        outs.append((po.cpu().numpy(), ro.cpu().numpy()))
    a = O.aperture(n, n)
    for o in outs[1:]:
        for t in range(3):
            for s in range(S):
                assert phi_err(o[0][t, s], outs[0][0][t, s].astype(np.float64), a) < 1e-3
                assert np.linalg.norm(o[1][t, s] - outs[0][1][t, s]) / np.linalg.norm(outs[0][1][t, s]) < 1e-3


@pytest.mark.parametrize("n,flags", [(128, 0), (128, 1), pytest.param(64, 0, id="chain")])
def test_graph_replay_bit_exact(n, flags):
    """A recurring single-frame call (fixed frame and output buffers) is
    captured into a CUDA graph on its second occurrence and replayed; results
    equal the launch-by-launch path bit for bit (phi ping-pong included; at
    N = 64 the on-chip chain)."""
    S, T = 2, 6
    y, _, _ = frames(n, S, T)
    yt = torch.from_numpy(y).to(DEV)
    with chain_env(n == 64):
        ctxs = [DDH(n, S, noise_var=0.1, flags=flags | 32), DDH(n, S, noise_var=0.1, flags=flags)]
    bufs = [torch.empty((1, S, n, n), dtype=torch.complex64, device=DEV) for _ in ctxs]
    outs = [(torch.empty((1, S, n, n), device=DEV), torch.empty((1, S, n, n), device=DEV)) for _ in ctxs]
    for t in range(T):
        res = []
        for c, b, (po, ro) in zip(ctxs, bufs, outs):
            b.copy_(yt[t:t + 1])
            c.step(b, po, ro)
            res.append((po.clone(), ro.clone()))
        torch.cuda.synchronize()
        assert torch.equal(res[0][0], res[1][0]) and torch.equal(res[0][1], res[1][1]), t
    r0, p0, f0 = ctxs[0].get_state()
    r1, p1, f1 = ctxs[1].get_state()
    assert torch.equal(r0, r1) and torch.equal(p0, p1) and f0 == f1 == T
    assert ctxs[0].kernel_launches == ctxs[1].kernel_launches


def test_misaligned_frames_are_rejected():
    """Whole frame rows move by bulk asynchronous copies: a y pointer that is
    not 16-byte aligned is refused with DDH_E_INVAL (not a CUDA fault), and
    the ctx stays usable."""
    import ctypes
    n, S = 64, 1
    ctx = DDH(n, S, noise_var=0.1)
    y = torch.zeros((2, S, n, n), dtype=torch.complex64, device=DEV)
    rc = ctx.lib.ddh_step(ctx.h, ctypes.c_void_p(y.data_ptr() + 8), 1, None, None, None)
    assert rc == 1 and b"aligned" in ctx.lib.ddh_last_error(ctx.h)
    rc = ctx.lib.ddh_bootstrap(ctx.h, ctypes.c_void_p(y.data_ptr() + 8), 2, None)
    assert rc == 1
    y[0] = torch.from_numpy(frames(n, S, 1)[0][0]).to(DEV)
    ctx.step(y[:1])
    torch.cuda.synchronize()
    assert ctx.get_state()[2] == 1


def test_kernel_variants_bit_exact():
    """The launch-size-dependent kernel variants compute the same arithmetic:
    at 256^2 with 20 streams, launch groups of 1, 4 and 20 streams take the
    16x16, 32x32 and 64x64 ICD tiles (halo recomputation gives exactly the
    global colour-ordered sweep) and the staged / plain column kernel; the
    results agree bit for bit."""
    n, S, T = 256, 20, 2
    y, _, _ = frames(n, S, T)
    yt = torch.from_numpy(y).to(DEV)
    outs = []
    for chunk in (1, 4, 20):
        ctx = DDH(n, S, noise_var=0.1, chunk_streams=chunk)
        po = torch.empty((T, S, n, n), device=DEV)
        ro = torch.empty_like(po)
        ctx.step(yt, po, ro)
        outs.append((po, ro))
    for po, ro in outs[1:]:
        assert torch.equal(outs[0][0], po) and torch.equal(outs[0][1], ro)


def test_residual_phase_and_psf_parity():
    """ddh_residual against the oracle: residual phase (wrapped,
    tip/tilt removed) and the normalised residual PSF, plus its Strehl."""
    n, B = 256, 2
    a = O.aperture(n, n)
    g = np.random.default_rng(9)
    tru = np.stack([synth.screen_from_coeffs(synth.screen_coeffs(n, n, n / 10.0, g)) for _ in range(B)]).astype(np.float32)
    hat = (tru + g.standard_normal((B, n, n)) * 0.3).astype(np.float32)
    ctx = DDH(n, 1)
    resid, psf, st = ctx.residual(torch.from_numpy(hat).to(DEV), torch.from_numpy(tru).to(DEV))
    for b in range(B):
        r_ref = O.residual_phase(hat[b], tru[b], a)
        d = np.angle(np.exp(1j * (resid[b].cpu().numpy() - r_ref)))
        assert np.max(np.abs(d)) < 1e-4
        p_ref = O.residual_psf(hat[b], tru[b], a)
        assert np.max(np.abs(psf[b].cpu().numpy() - p_ref)) < 1e-5 * p_ref.max() + 1e-7
        assert abs(st[b] - O.strehl(hat[b], tru[b], a)) < 1e-5
        assert abs(st[b] - float(psf[b].max())) < 1e-6


def test_strehl_sequence_metrics():
    """metrics.strehl_sequence: per-frame Strehl of several simulations from
    the on-device synthesiser through ddh_step / ddh_strehl equals the
    oracle's Strehl of the same phi-hat; box statistics are those of the series."""
    from paper_2305_03284_b200 import metrics
    cfg = dict(synth.CONFIGS["c1"])
    out = metrics.strehl_sequence(cfg, sims=3, frames=6, k_b=10, residual_at=5)
    S = out["strehl"]
    a = O.aperture(cfg["n"], cfg["diam"])
    ph, pt = out["phi_hat"].cpu().numpy(), out["phi_true"].cpu().numpy()
    for s in range(3):
        for t in range(6):
            assert abs(S[s, t] - O.strehl(ph[t, s], pt[t, s], a)) < 1e-5
    assert np.allclose(out["box"]["median"], np.median(S, axis=0))
    assert out["residual_psf"].shape == (3, cfg["n"], cfg["n"])
    assert np.allclose(out["residual_strehl"], S[:, 5], atol=1e-6)


def test_run_streams_threads_match_one_context():
    """sched.run_streams in host-thread mode (two GPU units emulated on one
    device): each unit runs its contiguous block of streams with its own ctx;
    the final per-stream states equal one ctx over all streams, bit for bit."""
    from paper_2305_03284_b200 import sched
    cfg = dict(synth.CONFIGS["c1"], streams=3)
    res = sched.run_streams(cfg, steps=5, warmup=2, frames=8, scaling="weak", source="host", devices=[0, 0],
                            return_state=True)
    assert res["gpus"] == 2 and res["streams_total"] == 6 and res["frames_per_s"] > 0
    one = sched.StreamRank(cfg, 0, 6, 0, 8, source="host")
    one.steps(2 + 5)
    r1, p1, f1 = one.ctx.get_state()
    for row in res["per_gpu"]:
        r, p, f = row["state"]
        k0, k1 = row["first"], row["first"] + row["streams"]
        assert f == f1 == 7
        assert np.array_equal(r, r1[k0:k1].cpu().numpy()) and np.array_equal(p, p1[k0:k1].cpu().numpy())


def test_bench_under_torchrun_two_ranks_one_gpu():
    """bench.py's GPU arm under torchrun with 2 ranks (both on this GPU: the
    scheduler falls back to gloo for its host-side collectives): one JSON
    line, n_gpus 2, weak scaling over 2 x 64 streams."""
    import json
    import os
    import socket
    import subprocess
    import sys
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(port), "bench.py", "--gpus", "2", "--steps", "6", "--warmup", "3",
           "--frames", "8", "--no-e2e", "--no-latency", "--no-cpu-baseline", "--no-parity"]
    pr = subprocess.run(cmd, cwd=root, capture_output=True, text=True, timeout=600)
    assert pr.returncode == 0, pr.stderr[-3000:]
    lines = [l for l in pr.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, pr.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "weak" and d["value"] > 0
