"""FP64 CPU oracle for the Dynamic DH-MBIR (DDH-MBIR) hot path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/`` (incl. the developer scripts in
``tests/tools/``), ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg, its ``--impl reference`` arm and the parity sample
printed beside the number) may import this module.  The product path (``paper_2305_03284_b200``, ``include/ddh.h``,
``csrc/``) never imports, links or calls it, and the two share no code: this
file uses numpy's FFT and LAPACK (``eigvals``) as library primitives, the CUDA
path uses its own kernels.

Every function cites the passage of the paper it follows.  Citation key:
``P:<line>`` = line of ``/root/reference/PAPER.md`` (the paper's LaTeX),
``R<k>`` = reading ``k`` of SURVEY.md section 8.c.7 (repeated in DESIGN.md),
which fixes what the paper leaves silent (the paper defers the EM internals
to [pellizzari2017], which is not available).

Conventions:
  * grid N x N, row-major, index (i=row, j=col), centre (N/2, N/2), N even;
  * aperture a_ij = 1 iff (i-N/2)^2 + (j-N/2)^2 < (D/2)^2          (R28)
  * F_c = fftshift . fft2 . ifftshift, unitary ("normalized 2D DFT", R3/R4)
  * A_phi = D_a D(e^{j phi}) F_c^{-1}  (image -> pupil),  Gamma = I (R3, R5)
  * A_phi^H y = F_c(a . e^{-j phi} . y)                              (pupil -> image)

Parity status of each function is listed in DESIGN.md section "Oracle pins";
nothing here is "parity unpinned" except the paper's absolute Strehl accuracy,
which is context only (the paper's scene and seeds are absent).
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional, Tuple

import numpy as np

# ---------------------------------------------------------------------------
# Parameters
# ---------------------------------------------------------------------------


@dataclasses.dataclass
class OracleParams:
    """Algorithm parameters (mirror of ``ddh_params`` in include/ddh.h).

    lam, alpha: Eq. 3 weights, defaults 0.45 / 0.025.
    n_k: EM iterations per time step (Fig. 1).
    noise_var: sigma^2 of the reconstruction in normalised-data units (R19).
    r_min: floor on r (replaces Fig. 1's r <- 0, R14).
    r_sigma, r_T, r_q: qGGMRF prior on r (north_star; R6/R7); r_sigma <= 0 -> prior off.
    phi_sigma: GMRF prior on phi (north_star; R11); phi_sigma <= 0 -> prior off.
    icd_sweeps: 4-colour sweeps per M-step (R8).
    boot_period, boot_alpha: bootstrap reset period / back-projection weight (R15).
    tiptilt: apply RemoveTipTilt in ddh_step (Fig. 1).
    """

    n: int = 64
    aperture_diam: float = 64.0
    aperture_mask: Optional[np.ndarray] = None
    noise_var: float = 0.113
    lam: float = 0.45
    alpha: float = 0.025
    n_k: int = 1
    r_min: float = 1e-4
    r_sigma: float = 0.5
    r_T: float = 1.0
    r_q: float = 1.2
    phi_sigma: float = 0.5
    icd_sweeps: int = 1
    boot_period: int = 200
    boot_alpha: float = 1.0
    tiptilt: bool = True


# 8-neighbour stencil weights b_ij: 1/6 for the 4 nearest, 1/12 for the 4
# diagonal neighbours (R7).  Order is irrelevant (sums).
NEIGHBOURS = (
    (-1, 0, 1.0 / 6.0), (1, 0, 1.0 / 6.0), (0, -1, 1.0 / 6.0), (0, 1, 1.0 / 6.0),
    (-1, -1, 1.0 / 12.0), (-1, 1, 1.0 / 12.0), (1, -1, 1.0 / 12.0), (1, 1, 1.0 / 12.0),
)
# Colour classes (i mod 2, j mod 2), visited in this order (R8).
COLOURS = ((0, 0), (0, 1), (1, 0), (1, 1))


# ---------------------------------------------------------------------------
# Forward model (Section 2 of the paper)
# ---------------------------------------------------------------------------


def aperture(n: int, diam: float) -> np.ndarray:
    """D_a, the camera aperture: a_ij = 1 iff the pixel centre lies
    strictly inside the circle of diameter ``diam`` centred at (N/2, N/2)."""
    i = np.arange(n)[:, None] - n / 2
    j = np.arange(n)[None, :] - n / 2
    return ((i * i + j * j) < (diam / 2.0) ** 2).astype(np.float64)


def aperture_of(p: OracleParams) -> np.ndarray:
    if p.aperture_mask is not None:
        return np.asarray(p.aperture_mask, dtype=np.float64)
    return aperture(p.n, p.aperture_diam)


def fft2c(x: np.ndarray) -> np.ndarray:
    """F_c, the normalised (unitary) centred 2-D DFT ("normalized 2D
    discrete Fourier transform"; centring R4)."""
    return np.fft.fftshift(np.fft.fft2(np.fft.ifftshift(x), norm="ortho"))


def ifft2c(x: np.ndarray) -> np.ndarray:
    """F_c^{-1} (inverse of :func:`fft2c`)."""
    return np.fft.fftshift(np.fft.ifft2(np.fft.ifftshift(x), norm="ortho"))


def forward(phi: np.ndarray, g: np.ndarray, a: np.ndarray) -> np.ndarray:
    """A_phi g = D_a D(e^{j phi}) F_c^{-1} g, Gamma = I (Eq. 1, R3, R5)."""
    return a * np.exp(1j * phi) * ifft2c(g)


def adjoint(phi: np.ndarray, y: np.ndarray, a: np.ndarray) -> np.ndarray:
    """A_phi^H y = F_c(a e^{-j phi} y): the back-projection of Eq. 3
    and the first transform of one EM iteration (R13)."""
    return fft2c(a * np.exp(-1j * phi) * y)


# ---------------------------------------------------------------------------
# Streaming-loop pre-processing (Section 4)
# ---------------------------------------------------------------------------


def normalize(y: np.ndarray) -> Optional[np.ndarray]:
    """Normalize(y) = sqrt(p) (y - mu)/||y - mu|| (Eq. 4); p = N^2
    entries, taken over the whole frame (R16).  Returns None for the
    degenerate frame ||y - mu|| = 0 (the frame is skipped)."""
    y = np.asarray(y, dtype=np.complex128)
    mu = y.mean()
    d = np.linalg.norm(y - mu)
    if d == 0.0:
        return None
    return math.sqrt(y.size) * (y - mu) / d


def plane_coords(n: int) -> Tuple[np.ndarray, np.ndarray]:
    """Pixel coordinates x = j - N/2 (columns), y = i - N/2 (rows)."""
    x = np.broadcast_to(np.arange(n)[None, :] - n / 2, (n, n)).astype(np.float64)
    yy = np.broadcast_to(np.arange(n)[:, None] - n / 2, (n, n)).astype(np.float64)
    return x, yy


def plane_fit(phi: np.ndarray, a: np.ndarray) -> np.ndarray:
    """Least-squares plane c0 + c1 x + c2 y of phi over {a = 1} (RemoveTipTilt,
    P:153, 167, 195: "removes the linear component of the phase ... using
    least-squares regression"; piston included, R17).  Solved from the 3x3
    normal equations."""
    n = phi.shape[0]
    x, yy = plane_coords(n)
    m = a > 0
    basis = np.stack([np.ones(int(m.sum())), x[m], yy[m]], axis=1)
    G = basis.T @ basis
    h = basis.T @ phi[m]
    return np.linalg.solve(G, h)


def plane_eval(c: np.ndarray, n: int) -> np.ndarray:
    x, yy = plane_coords(n)
    return c[0] + c[1] * x + c[2] * yy


def remove_tip_tilt(phi: np.ndarray, a: np.ndarray) -> np.ndarray:
    """phi - plane at every pixel (Fig. 1; R17)."""
    return phi - plane_eval(plane_fit(phi, a), phi.shape[0])


def warm_start(r: np.ndarray, u: np.ndarray, lam: float, alpha: float, r_min: float) -> np.ndarray:
    """Eq. 3: r_init = (1 - lam) r_{n-1} + lam alpha |A^H y|^2,
    floored at r_min (R14)."""
    return np.maximum((1.0 - lam) * r + lam * alpha * np.abs(u) ** 2, r_min)


# ---------------------------------------------------------------------------
# EM iteration (Section 3; internals per readings R1-R12)
# ---------------------------------------------------------------------------


def e_step(u: np.ndarray, r: np.ndarray, s2: float):
    """E-step for g ~ CN(0, D(r)) given u = A_phi^H y: the diagonal
    posterior w = r/(r + s2), mean mu = w u, variance C = w s2, second moment
    q = |mu|^2 + C (R1; exact when a = 1, the masked case is R2)."""
    w = r / (r + s2)
    mu = w * u
    C = w * s2
    q = np.abs(mu) ** 2 + C
    return mu, C, q


def qggmrf_rho(d: np.ndarray, sig: float, T: float, q: float) -> np.ndarray:
    """qGGMRF potential with p = 2 (R6): rho(D) = D^2/(2 sig^2) * 1/(1 + t),
    t = |D/(T sig)|^(2 - q)."""
    t = np.abs(d / (T * sig)) ** (2.0 - q)
    return d * d / (2.0 * sig * sig) / (1.0 + t)


def qggmrf_weight(d: np.ndarray, sig: float, T: float, q: float) -> np.ndarray:
    """Symmetric-bound surrogate coefficient rho'(D)/(2D) of :func:`qggmrf_rho`
    (R6): (1/(2 sig^2)) * (1/(1+t)) * (1 - (2-q) t / (2 (1+t))); equal to
    1/(2 sig^2) at D = 0."""
    t = np.abs(d / (T * sig)) ** (2.0 - q)
    return (1.0 / (2.0 * sig * sig)) / (1.0 + t) * (1.0 - (2.0 - q) * t / (2.0 * (1.0 + t)))


def r_surrogate(x, q, B, S):
    """Per-pixel 1-D surrogate of the r M-step (R9):
    f(x) = log x + q/x + B x^2 - 2 S x."""
    return np.log(x) + q / x + B * x * x - 2.0 * S * x


def _neigh(arr: np.ndarray, ii: np.ndarray, jj: np.ndarray, di: int, dj: int, periodic: bool):
    n = arr.shape[0]
    i2 = ii + di
    j2 = jj + dj
    if periodic:
        return arr[i2 % n, j2 % n], np.ones(ii.shape, dtype=bool)
    valid = (i2 >= 0) & (i2 < n) & (j2 >= 0) & (j2 < n)
    return arr[np.clip(i2, 0, n - 1), np.clip(j2, 0, n - 1)], valid



def r_prior_coeffs(r, ii, jj, p: OracleParams):
    """B = sum_j b~_ij, S = sum_j b~_ij r_j for pixels (ii, jj), with
    b~_ij = b_ij rho'(D)/(2D) at D = r_i - r_j, 8 neighbours, periodic (R6-R8)."""
    ri = r[ii, jj]
    B = np.zeros_like(ri)
    S = np.zeros_like(ri)
    for (di, dj, b) in NEIGHBOURS:
        rj, _ = _neigh(r, ii, jj, di, dj, periodic=True)
        bt = b * qggmrf_weight(ri - rj, p.r_sigma, p.r_T, p.r_q)
        B += bt
        S += bt * rj
    return B, S


def phi_prior_coeffs(phi, ii, jj):
    """sum_j b_ij phi_j and sum_j b_ij over the existing 8 neighbours (free
    boundary, R11)."""
    nb = np.zeros(ii.shape)
    sb = np.zeros(ii.shape)
    for (di, dj, b) in NEIGHBOURS:
        pj, valid = _neigh(phi, ii, jj, di, dj, periodic=False)
        nb += np.where(valid, b * pj, 0.0)
        sb += np.where(valid, b, 0.0)
    return nb, sb

def r_update_pixels(r_cur, q, B, S, r_min, return_gap=False, guide=None, guide_tol=1e-5):
    """Exact minimiser of the surrogate over x >= r_min for a vector of pixels
    (R9).  Stationary points solve 2 B x^3 - 2 S x^2 + x - q = 0; the roots are
    the eigenvalues of the companion matrix of the monic cubic (LAPACK).
    Candidates = {r_min} U {max(Re(root), r_min)}; the minimiser of f wins, and
    among candidates within 1e-12 (1 + |f|) of the minimum the one nearest the
    current value.

    ``guide`` (parity tests only, SURVEY 8.c.9 "several results are correct"):
    values an implementation produced for these pixels; among the candidates
    within ``guide_tol`` (1 + |f|) of the minimum -- all of them minimisers
    up to the precision of an FP32 evaluation of f -- the one nearest the
    guide is taken, so a test can follow the implementation's valid choice at
    a near-tie and compare every pixel after it."""
    m = r_cur.shape[0]
    comp = np.zeros((m, 3, 3))
    comp[:, 0, 0] = S / B
    comp[:, 0, 1] = -1.0 / (2.0 * B)
    comp[:, 0, 2] = q / (2.0 * B)
    comp[:, 1, 0] = 1.0
    comp[:, 2, 1] = 1.0
    roots = np.linalg.eigvals(comp)
    cand = np.concatenate([np.full((m, 1), r_min), np.maximum(roots.real, r_min)], axis=1)
    f = r_surrogate(cand, q[:, None], B[:, None], S[:, None])
    fmin = f.min(axis=1, keepdims=True)
    if guide is None:
        near = f <= fmin + 1e-12 * (1.0 + np.abs(fmin))
        dist = np.where(near, np.abs(cand - r_cur[:, None]), np.inf)
    else:
        near = f <= fmin + guide_tol * (1.0 + np.abs(fmin))
        dist = np.where(near, np.abs(cand - np.asarray(guide)[:, None]), np.inf)
    best = cand[np.arange(m), dist.argmin(axis=1)]
    if not return_gap:
        return best
    # diagnostic for the parity protocol: cost gap to the best
    # candidate that is far (> 1e-3 relative) from the chosen one
    far = np.abs(cand - best[:, None]) > 1e-3 * np.maximum(best[:, None], r_min)
    gap = np.where(far, f - fmin, np.inf).min(axis=1) / (1.0 + np.abs(fmin[:, 0]))
    return best, gap


def r_icd(r: np.ndarray, q: np.ndarray, p: OracleParams, gaps: Optional[np.ndarray] = None,
          guide: Optional[np.ndarray] = None) -> np.ndarray:
    """r M-step: colour-ordered ICD with the qGGMRF prior (north_star; R6-R9).

    For each colour (i mod 2, j mod 2) in order (0,0),(0,1),(1,0),(1,1), every
    pixel of the colour minimises log x + q_i/x + B x^2 - 2 S x with
    b~_ij = b_ij rho'(D)/(2D) at D = r_i - r_j (8 neighbours, periodic
    boundary), B = sum b~, S = sum b~ r_j.  Pixels of one colour have no
    neighbour of the same colour, so updating a colour at once equals a raster
    sweep over it.  Prior off (r_sigma <= 0): r = max(q, r_min)."""
    if p.r_sigma <= 0:
        return np.maximum(q, p.r_min)
    r = r.copy()
    n = r.shape[0]
    for _ in range(p.icd_sweeps):
        for (ci, cj) in COLOURS:
            ii, jj = np.meshgrid(np.arange(ci, n, 2), np.arange(cj, n, 2), indexing="ij")
            ii = ii.ravel()
            jj = jj.ravel()
            B, S = r_prior_coeffs(r, ii, jj, p)
            gd = None if guide is None else guide[ii, jj]
            if gaps is None:
                r[ii, jj] = r_update_pixels(r[ii, jj], q[ii, jj], B, S, p.r_min, guide=gd)
            else:
                r[ii, jj], g = r_update_pixels(r[ii, jj], q[ii, jj], B, S, p.r_min, return_gap=True, guide=gd)
                gaps[ii, jj] = np.minimum(gaps[ii, jj], g)
    return r


def phase_correlation(yhat: np.ndarray, f: np.ndarray, a: np.ndarray, s2: float):
    """Data term of the phi M-step.  The phi-dependent part of the expected
    log-likelihood is (2/s2) Re sum conj(y_i) a_i e^{j phi_i} f_i with
    f = F_c^{-1} mu (the second FFT of P:140), i.e. sum_i c_i cos(phi_i - theta_i)
    with c = (2/s2) a |y| |f|, theta = arg(y conj(f))."""
    c = (2.0 / s2) * a * np.abs(yhat) * np.abs(f)
    theta = np.angle(yhat * np.conj(f))
    return c, theta


def wrap(x):
    """wrap(x) in (-pi, pi]."""
    return np.angle(np.exp(1j * np.asarray(x)))


def phi_icd(phi: np.ndarray, c: np.ndarray, theta: np.ndarray, p: OracleParams) -> np.ndarray:
    """phi M-step: colour-ordered ICD with the GMRF prior (north_star; R10-R11).

    Per pixel: x0 = wrap(phi_i - theta_i), s = sin(x0)/x0 (1 at 0),
    theta~ = phi_i - x0; the symmetric bound of -c cos(.) at x0 gives
    phi_i <- (c s theta~ + w sum b_ij phi_j)/(c s + w sum b_ij), w = 1/phi_sigma^2,
    8 neighbours with free boundary (missing neighbours dropped).  A zero
    denominator keeps phi_i.  Prior off: phi_i <- theta~_i where c_i > 0
    (the exact argmax)."""
    phi = phi.copy()
    n = phi.shape[0]
    prior = p.phi_sigma > 0
    wphi = 1.0 / (p.phi_sigma * p.phi_sigma) if prior else 0.0
    for _ in range(p.icd_sweeps):
        for (ci, cj) in COLOURS:
            ii, jj = np.meshgrid(np.arange(ci, n, 2), np.arange(cj, n, 2), indexing="ij")
            ii = ii.ravel()
            jj = jj.ravel()
            ph = phi[ii, jj]
            cc = c[ii, jj]
            x0 = wrap(ph - theta[ii, jj])
            tt = ph - x0
            if not prior:
                phi[ii, jj] = np.where(cc > 0, tt, ph)
                continue
            with np.errstate(invalid="ignore", divide="ignore"):
                s = np.where(x0 == 0.0, 1.0, np.sin(x0) / np.where(x0 == 0.0, 1.0, x0))
            nb, sb = phi_prior_coeffs(phi, ii, jj)
            num = cc * s * tt + wphi * nb
            den = cc * s + wphi * sb
            with np.errstate(invalid="ignore", divide="ignore"):
                phi[ii, jj] = np.where(den != 0.0, num / np.where(den != 0.0, den, 1.0), ph)
    return phi


def em_update(r, phi, yhat, u, a, p: OracleParams, gaps=None, guide=None):
    """One EM iteration EM(r, phi; y) given u = A_phi^H y:
    E-step, r M-step (uses q only) and phi M-step (uses f = F_c^{-1} mu only).
    The two M-steps read only E-step quantities, so their order is
    irrelevant (R12).  Exactly two 2-D FFTs per iteration (R13)."""
    mu, _C, q = e_step(u, r, p.noise_var)
    r_new = r_icd(r, q, p, gaps, guide)
    f = ifft2c(mu)
    c, theta = phase_correlation(yhat, f, a, p.noise_var)
    phi_new = phi_icd(phi, c, theta, p)
    return r_new, phi_new


# ---------------------------------------------------------------------------
# DDH-MBIR loop (Fig. 1), bootstrap and static DH-MBIR (Section 3)
# ---------------------------------------------------------------------------


def ddh_step(r, phi, y, p: OracleParams, a=None, gaps=None, guide=None):
    """One time step of DDH_MBIR (Fig. 1):
    y <- Normalize(y); phi <- RemoveTipTilt(phi);
    r <- (1-lam) r + lam alpha |A_phi^H y|^2 (Eq. 3); N_k x EM(r, phi; y).
    The back-projection of Eq. 3 is the first E-step's u (R13).
    Returns (r, phi, status); status 1 = degenerate frame, state unchanged."""
    if a is None:
        a = aperture_of(p)
    yhat = normalize(y)
    if yhat is None:
        return r.copy(), phi.copy(), 1
    if p.tiptilt:
        phi = remove_tip_tilt(phi, a)
    u = adjoint(phi, yhat, a)
    r = warm_start(r, u, p.lam, p.alpha, p.r_min)
    for k in range(p.n_k):
        if k > 0:
            u = adjoint(phi, yhat, a)
        r, phi = em_update(r, phi, yhat, u, a, p, gaps, guide)
    return r, phi, 0


def bootstrap(y0, p: OracleParams, k_b: int, a=None, gaps=None):
    """Bootstrap on the first frame (R15): cold start
    r = r_min, phi = 0, then K_b EM iterations; before iteration k with
    k mod P_b == 0 the reflectance is reset to the back-projection
    max(alpha_b |A_phi^H y|^2, r_min) ([pellizzari2017b] "reset to a
    backprojected estimate every 200 iterations").
    Returns (r, phi, status)."""
    if a is None:
        a = aperture_of(p)
    n = p.n
    r = np.full((n, n), p.r_min)
    phi = np.zeros((n, n))
    yhat = normalize(y0)
    if yhat is None:
        return r, phi, 1
    for k in range(k_b):
        u = adjoint(phi, yhat, a)
        if k % p.boot_period == 0:
            r = np.maximum(p.boot_alpha * np.abs(u) ** 2, p.r_min)
        r, phi = em_update(r, phi, yhat, u, a, p, gaps)
    return r, phi, 0


def static_dhmbir(y, p: OracleParams, iters: int, a=None):
    """Conventional single-shot DH-MBIR: an independent
    cold-started bootstrap run of ``iters`` EM iterations on one frame."""
    return bootstrap(y, p, iters, a)


# ---------------------------------------------------------------------------
# Metrics (Section 5.2)
# ---------------------------------------------------------------------------


def strehl(phi_hat, phi_true, a, remove_plane: bool = True) -> float:
    """Peak Strehl ratio:
    S = max|A^H_{phi^-phi} D_a|^2 / max|A^H_0 D_a|^2, evaluated as
    max_k |F_c^{-1}(a e^{j psi})|^2 / max_k |F_c^{-1}(a)|^2 with
    psi = phi^ - phi minus its LS plane over a (R25, R26)."""
    psi = np.asarray(phi_hat, np.float64) - np.asarray(phi_true, np.float64)
    if remove_plane:
        psi = remove_tip_tilt(psi, a)
    num = np.max(np.abs(ifft2c(a * np.exp(1j * psi))) ** 2)
    den = np.max(np.abs(ifft2c(a.astype(np.complex128))) ** 2)
    return float(num / den)


def residual_phase(phi_hat, phi_true, a) -> np.ndarray:
    """Residual phase error angle(e^{j(phi - phi_hat)}) (Fig. 5 caption
    P:320: tip and tilt removed): the LS plane of phi_hat - phi over the
    aperture is removed first (R26), values on the aperture in (-pi, pi],
    0 elsewhere."""
    psi = remove_tip_tilt(np.asarray(phi_hat, np.float64) - np.asarray(phi_true, np.float64), a)
    return np.where(a > 0, np.angle(np.exp(-1j * psi)), 0.0)


def residual_psf(phi_hat, phi_true, a) -> np.ndarray:
    """Residual point-spread function (Fig. 5 caption P:320): the image-plane
    intensity |F_c^{-1}(a e^{j psi})|^2 of the corrected pupil, normalised by
    the diffraction-limited peak max|F_c^{-1}(a)|^2, so that its
    maximum is the peak Strehl ratio of :func:`strehl`."""
    psi = remove_tip_tilt(np.asarray(phi_hat, np.float64) - np.asarray(phi_true, np.float64), a)
    num = np.abs(ifft2c(a * np.exp(1j * psi))) ** 2
    den = np.max(np.abs(ifft2c(a.astype(np.complex128))) ** 2)
    return num / den


def cost_J(r, phi, yhat, p: OracleParams, a=None) -> float:
    """MAP cost of Eq. 2 for a full aperture (a = 1), where A_phi
    is unitary and y ~ CN(0, A(D(r) + s2 I)A^H):
    J = sum_i [log(r_i+s2) + |u_i|^2/(r_i+s2)] + sum_pairs b rho(r_i - r_j)
        + (1/(2 sig_phi^2)) sum_pairs b (phi_i - phi_j)^2,   u = A_phi^H y.
    (periodic pairs for r, free-boundary pairs for phi, as in the ICDs.)"""
    return float(sum(cost_J_parts(r, phi, yhat, p, a)))


def cost_J_parts(r, phi, yhat, p: OracleParams, a=None):
    """(data, r-prior, phi-prior) terms of :func:`cost_J`."""
    if a is None:
        a = aperture_of(p)
    s2 = p.noise_var
    u = adjoint(phi, yhat, a)
    J = float(np.sum(np.log(r + s2) + np.abs(u) ** 2 / (r + s2)))
    Jr = 0.0
    Jp = 0.0
    n = r.shape[0]
    # each unordered pair once: offsets (0,1),(1,0),(1,1),(1,-1)
    half = ((0, 1, 1.0 / 6.0), (1, 0, 1.0 / 6.0), (1, 1, 1.0 / 12.0), (1, -1, 1.0 / 12.0))
    if p.r_sigma > 0:
        for (di, dj, b) in half:
            d = r - np.roll(np.roll(r, -di, axis=0), -dj, axis=1)
            Jr += float(np.sum(b * qggmrf_rho(d, p.r_sigma, p.r_T, p.r_q)))
    if p.phi_sigma > 0:
        wphi = 1.0 / (2.0 * p.phi_sigma ** 2)
        for (di, dj, b) in half:
            i0, i1 = max(0, -di), n - max(0, di)
            j0, j1 = max(0, -dj), n - max(0, dj)
            d = phi[i0:i1, j0:j1] - phi[i0 + di:i1 + di, j0 + dj:j1 + dj]
            Jp += float(wphi * np.sum(b * d * d))
    return J, Jr, Jp


# ---------------------------------------------------------------------------
# Multi-stream driver (mirror of the C ABI, host FP64)
# ---------------------------------------------------------------------------


class DDHOracle:
    """Host FP64 mirror of ``ddh_ctx``: S independent streams with state
    (r, phi, n) (Fig. 1: n <- 0, r <- 0 (r_min, R14), phi <- 0)."""

    def __init__(self, p: OracleParams, streams: int):
        self.p = p
        self.S = streams
        self.a = aperture_of(p)
        n = p.n
        self.r = np.full((streams, n, n), p.r_min)
        self.phi = np.zeros((streams, n, n))
        self.frame_index = 0

    def set_state(self, r, phi, frame_index=0):
        self.r = np.array(r, dtype=np.float64).reshape(self.S, self.p.n, self.p.n)
        self.phi = np.array(phi, dtype=np.float64).reshape(self.S, self.p.n, self.p.n)
        self.frame_index = int(frame_index)

    def bootstrap(self, y0, k_b: int):
        status = np.zeros(self.S, np.uint8)
        if k_b <= 0:
            return status
        for s in range(self.S):
            self.r[s], self.phi[s], status[s] = bootstrap(y0[s], self.p, k_b, self.a)
        self.frame_index += 1
        return status

    def step(self, y):
        """y: [T][S][N][N] complex.  Returns phi_out, r_out [T][S][N][N], status [T][S]."""
        y = np.asarray(y)
        T = y.shape[0]
        n = self.p.n
        phi_out = np.zeros((T, self.S, n, n))
        r_out = np.zeros((T, self.S, n, n))
        status = np.zeros((T, self.S), np.uint8)
        for t in range(T):
            for s in range(self.S):
                self.r[s], self.phi[s], status[t, s] = ddh_step(self.r[s], self.phi[s], y[t, s], self.p, self.a)
                phi_out[t, s] = self.phi[s]
                r_out[t, s] = self.r[s]
            self.frame_index += 1
        return phi_out, r_out, status
