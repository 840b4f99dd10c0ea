"""Pins of the FP64 oracle to things other than itself (-m "not gpu").

Each test names what fixes the expected value: a closed form, a textbook
construction written independently of the oracle (dense matrices, brute-force
grid searches), a value printed in the paper (tests/golden/), or an invariant
of the mathematics (EM monotonicity, equivariances).
"""
import math
import os

import numpy as np
import pytest

import oracle.ddh_oracle as O
import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def rng(k=0):
    return np.random.default_rng(1234 + k)


def crandn(g, *shape):
    return g.standard_normal(shape) + 1j * g.standard_normal(shape)


def dense_centred_dft(n):
    """Dense 2-D centred unitary DFT from its definition (not via fftshift):
    F_c[(k1,k2),(n1,n2)] = (1/N) exp(-2 pi i [(k1-N/2)(n1-N/2) + (k2-N/2)(n2-N/2)]/N)."""
    k = np.arange(n) - n / 2
    W1 = np.exp(-2j * np.pi * np.outer(k, k) / n) / math.sqrt(n)
    return np.kron(W1, W1)


# --------------------------------------------------------------------- FFT


@pytest.mark.parametrize("n", [2, 4, 8, 16])
def test_fft2c_matches_naive_dft(n):
    g = rng(n)
    x = crandn(g, n, n)
    F = dense_centred_dft(n)
    ref = (F @ x.ravel()).reshape(n, n)
    assert np.max(np.abs(O.fft2c(x) - ref)) < 1e-12 * max(1.0, np.abs(ref).max())
    refi = (F.conj().T @ x.ravel()).reshape(n, n)
    assert np.max(np.abs(O.ifft2c(x) - refi)) < 1e-12 * max(1.0, np.abs(refi).max())


@pytest.mark.parametrize("n", [6, 8, 64])
def test_fft2c_unitary_and_chi_identity(n):
    g = rng(n)
    x = crandn(g, n, n)
    assert abs(np.linalg.norm(O.fft2c(x)) - np.linalg.norm(x)) < 1e-12 * np.linalg.norm(x)
    assert np.max(np.abs(O.ifft2c(O.fft2c(x)) - x)) < 1e-12
    # F_c = chi F chi for even N in 2-D (R4; the GPU folds chi into its stages)
    i = np.arange(n)
    chi = (-1.0) ** (i[:, None] + i[None, :])
    assert np.max(np.abs(O.fft2c(x) - chi * np.fft.fft2(chi * x) / n)) < 1e-12


# ----------------------------------------------------------- forward model


def test_adjoint_identity_and_mask():
    n = 16
    g = rng(1)
    a = O.aperture(n, 12.0)
    phi = g.standard_normal((n, n))
    x = crandn(g, n, n)
    y = crandn(g, n, n)
    Ax = O.forward(phi, x, a)
    AHy = O.adjoint(phi, y, a)
    lhs = np.vdot(y, Ax)
    rhs = np.vdot(AHy, x)
    assert abs(lhs - rhs) < 1e-12 * np.linalg.norm(x) * np.linalg.norm(y)
    assert np.all(Ax[a == 0] == 0)
    # delta at the centre of the image, phi = 0 -> constant modulus 1/N inside a
    d = np.zeros((n, n), complex)
    d[n // 2, n // 2] = 1.0
    out = O.forward(np.zeros((n, n)), d, a)
    assert np.allclose(np.abs(out[a > 0]), 1.0 / n, atol=1e-14)


def test_aperture_strictly_inside():
    a = O.aperture(8, 8.0)
    # (i-4)^2 + (j-4)^2 < 16: centre row spans j = 1..7 (j=0 gives 16, excluded)
    assert a[4].tolist() == [0, 1, 1, 1, 1, 1, 1, 1]
    assert a[0].sum() == 0


# ------------------------------------------------------------- Normalize


def test_normalize_examples():
    out = O.normalize(np.array([1.0, -1.0]))
    assert np.allclose(out, [1.0, -1.0], atol=1e-15)
    assert O.normalize(np.full((4, 4), 3.0 + 2.0j)) is None  # degenerate frame
    g = rng(2)
    y = crandn(g, 32, 32) + (5 - 2j)
    yh = O.normalize(y)
    assert abs(yh.mean()) < 1e-12
    assert abs(np.sum(np.abs(yh) ** 2) - y.size) < 1e-9 * y.size


# --------------------------------------------------------------- tip/tilt


def test_plane_fit_exact_and_idempotent():
    n = 32
    a = O.aperture(n, 30.0)
    x, yy = O.plane_coords(n)
    phi = 2.0 + 3.0 * x - 1.0 * yy
    c = O.plane_fit(phi, a)
    assert np.allclose(c, [2.0, 3.0, -1.0], atol=1e-10)
    assert np.allclose(O.plane_fit(np.full((n, n), 5.0), a), [5.0, 0.0, 0.0], atol=1e-12)
    g = rng(3)
    psi = g.standard_normal((n, n))
    once = O.remove_tip_tilt(psi, a)
    twice = O.remove_tip_tilt(once, a)
    assert np.max(np.abs(once - twice)) < 1e-12
    # independent dense least squares (numpy lstsq on the design matrix)
    m = a > 0
    A = np.stack([np.ones(m.sum()), x[m], yy[m]], 1)
    coef, *_ = np.linalg.lstsq(A, psi[m], rcond=None)
    assert np.allclose(O.plane_fit(psi, a), coef, atol=1e-12)


# ------------------------------------------------------------------ Eq. 3


def test_warm_start_endpoints():
    g = rng(4)
    r = g.random((8, 8)) + 0.1
    u = crandn(g, 8, 8)
    assert np.array_equal(O.warm_start(r, u, 0.0, 0.025, 1e-4), np.maximum(r, 1e-4))
    assert np.allclose(O.warm_start(r, u, 1.0, 0.3, 1e-4), np.maximum(0.3 * np.abs(u) ** 2, 1e-4))


# ----------------------------------------------------------------- E-step


@pytest.mark.parametrize("n", [4, 8])
def test_e_step_equals_dense_gaussian_conditioning(n):
    """a = 1: mu and diag(C) equal the textbook conditional of y = A g + w,
    g ~ CN(0, D(r)), w ~ CN(0, s2 I), with A built densely from the DFT
    definition (not from the oracle's FFT)."""
    g = rng(10 + n)
    P = n * n
    a = np.ones((n, n))
    phi = g.standard_normal((n, n))
    r = g.random((n, n)) * 2 + 0.05
    s2 = 0.3
    y = crandn(g, n, n)
    Fc = dense_centred_dft(n)
    A = np.diag(np.exp(1j * phi.ravel())) @ Fc.conj().T
    Dr = np.diag(r.ravel())
    Sy = A @ Dr @ A.conj().T + s2 * np.eye(P)
    K = Dr @ A.conj().T @ np.linalg.inv(Sy)
    mu_ref = K @ y.ravel()
    C_ref = np.real(np.diag(Dr - K @ A @ Dr))
    mu, C, q = O.e_step(O.adjoint(phi, y, a), r, s2)
    assert np.max(np.abs(mu.ravel() - mu_ref)) < 1e-10 * np.abs(mu_ref).max()
    assert np.max(np.abs(C.ravel() - C_ref)) < 1e-10 * C_ref.max()
    assert np.allclose(q, np.abs(mu) ** 2 + C)


def test_e_step_limits():
    u = np.array([1.0 + 2.0j, -0.5j])
    mu, C, _ = O.e_step(u, np.full(2, 0.2), 0.2)  # r = s2 -> mu = u/2, C = s2/2
    assert np.allclose(mu, u / 2) and np.allclose(C, 0.1)
    mu, _, _ = O.e_step(u, np.full(2, 1e12 * 0.2), 0.2)
    assert np.allclose(mu, u, rtol=1e-9)


# ------------------------------------------------------------ qGGMRF / r


def test_qggmrf_weight_is_rho_prime_over_2delta():
    sig, T, q = 0.5, 1.0, 1.2
    d = np.array([1e-3, 0.05, 0.3, 1.0, 2.5, -0.7])
    h = 1e-6
    fd = (O.qggmrf_rho(d + h, sig, T, q) - O.qggmrf_rho(d - h, sig, T, q)) / (2 * h)
    assert np.allclose(O.qggmrf_weight(d, sig, T, q), fd / (2 * d), rtol=1e-6)
    assert O.qggmrf_weight(np.array([0.0]), sig, T, q)[0] == pytest.approx(1 / (2 * sig * sig))


def test_qggmrf_symmetric_bound_is_a_majoriser():
    sig, T, q = 0.5, 1.0, 1.2
    D = np.linspace(-6, 6, 2001)
    for d0 in [-3.0, -0.4, 0.0, 0.01, 0.7, 2.0, 5.0]:
        bound = O.qggmrf_rho(np.array(d0), sig, T, q) + O.qggmrf_weight(np.array(d0), sig, T, q) * (D * D - d0 * d0)
        assert np.all(O.qggmrf_rho(D, sig, T, q) <= bound + 1e-12)


def test_r_update_matches_bruteforce_grid():
    """The per-pixel minimiser equals a 1-D brute-force search of the
    surrogate over 2e5 log-spaced points in [r_min, 50]."""
    g = rng(20)
    m = 400
    r_min = 1e-4
    q = g.random(m) * 3 + 1e-3
    B = g.random(m) * 4 + 0.05
    S = B * (g.random(m) * 3)
    r_cur = g.random(m) * 2 + r_min
    x = O.r_update_pixels(r_cur, q, B, S, r_min)
    grid = np.geomspace(r_min, 50.0, 200001)
    for k in range(m):
        f = O.r_surrogate(grid, q[k], B[k], S[k])
        jbest = int(np.argmin(f))
        fx = O.r_surrogate(x[k], q[k], B[k], S[k])
        assert fx <= f[jbest] + 1e-9 * (1 + abs(f[jbest]))
        if abs(f[jbest] - np.partition(f, 1)[1]) > 1e-6:  # unambiguous minimum
            assert abs(x[k] - grid[jbest]) <= 2e-4 * max(1.0, grid[jbest]) + 1e-12


def test_r_icd_prior_off_and_consensus():
    p = O.OracleParams(n=8, r_sigma=0.0)
    g = rng(21)
    q = g.random((8, 8)) * 2
    q[0, 0] = 0.0
    out = O.r_icd(g.random((8, 8)), q, p)
    assert np.array_equal(out, np.maximum(q, 1e-4))
    # consensus: all values equal q -> r = q (prior term vanishes)
    p = O.OracleParams(n=8)
    qc = np.full((8, 8), 0.731)
    assert np.allclose(O.r_icd(qc.copy(), qc, p), qc, atol=1e-12)


def test_r_icd_each_pixel_decreases_true_cost():
    """MM property: after the ICD every updated pixel's true conditional cost
    log x + q/x + sum_j b rho(x - r_j) is <= its value before the update."""
    n = 16
    p = O.OracleParams(n=n)
    g = rng(22)
    r = g.random((n, n)) + 0.01
    q = g.random((n, n)) * 2 + 0.01
    r_work = r.copy()
    for (ci, cj) in O.COLOURS:
        ii, jj = np.meshgrid(np.arange(ci, n, 2), np.arange(cj, n, 2), indexing="ij")
        ii, jj = ii.ravel(), jj.ravel()

        def cost(x):
            tot = np.log(x) + q[ii, jj] / x
            for (di, dj, b) in O.NEIGHBOURS:
                rj = r_work[(ii + di) % n, (jj + dj) % n]
                tot = tot + b * O.qggmrf_rho(x - rj, p.r_sigma, p.r_T, p.r_q)
            return tot

        before = cost(r_work[ii, jj])
        pp = O.OracleParams(n=n)
        # one colour step through the oracle: run full ICD on a copy and read this colour
        B = np.zeros(len(ii))
        S = np.zeros(len(ii))
        for (di, dj, b) in O.NEIGHBOURS:
            rj = r_work[(ii + di) % n, (jj + dj) % n]
            bt = b * O.qggmrf_weight(r_work[ii, jj] - rj, pp.r_sigma, pp.r_T, pp.r_q)
            B += bt
            S += bt * rj
        new = O.r_update_pixels(r_work[ii, jj], q[ii, jj], B, S, pp.r_min)
        after = cost(new)
        assert np.all(after <= before + 1e-12 * (1 + np.abs(before)))
        r_work[ii, jj] = new
    assert np.allclose(r_work, O.r_icd(r, q, p), atol=1e-12)


# ------------------------------------------------------------------- phi


def test_cosine_symmetric_bound_is_a_majoriser():
    X = np.linspace(-20, 20, 8001)
    for x0 in np.linspace(-math.pi, math.pi, 41):
        s = 1.0 if x0 == 0 else math.sin(x0) / x0
        bound = -math.cos(x0) + 0.5 * s * (X * X - x0 * x0)
        assert np.all(-np.cos(X) <= bound + 1e-12)


def test_phi_update_prior_off_is_grid_argmax():
    n = 8
    p = O.OracleParams(n=n, phi_sigma=0.0)
    g = rng(30)
    c = g.random((n, n)) + 0.1
    theta = g.uniform(-math.pi, math.pi, (n, n))
    phi0 = g.standard_normal((n, n)) * 4
    out = O.phi_icd(phi0, c, theta, p)
    grid = 2 * math.pi * np.arange(4096) / 4096
    for i in range(n):
        for j in range(n):
            best = grid[np.argmax(c[i, j] * np.cos(grid - theta[i, j]))]
            d = (out[i, j] - best + math.pi) % (2 * math.pi) - math.pi
            assert abs(d) <= 2 * math.pi / 4096
            assert abs(out[i, j] - phi0[i, j]) <= math.pi + 1e-12  # nearest branch


def test_phi_recovered_exactly_from_known_g():
    """north_star pin: noise-free y = a e^{j phi} F_c^{-1} g with g known; the
    phi update with yhat := y, mu := g, prior off returns phi (mod 2pi) on a."""
    n = 32
    a = O.aperture(n, 30.0)
    g = rng(31)
    phi = g.standard_normal((n, n)) * 2
    gg = crandn(g, n, n)
    y = a * np.exp(1j * phi) * np.fft.fftshift(np.fft.ifft2(np.fft.ifftshift(gg), norm="ortho"))
    f = O.ifft2c(gg)
    c, theta = O.phase_correlation(y, f, a, 0.1)
    out = O.phi_icd(np.zeros((n, n)), c, theta, O.OracleParams(n=n, phi_sigma=0.0))
    d = np.angle(np.exp(1j * (out - phi)))
    assert np.max(np.abs(d[a > 0])) < 1e-12


def test_phi_icd_each_pixel_decreases_true_cost():
    n = 16
    p = O.OracleParams(n=n)
    g = rng(32)
    phi = g.standard_normal((n, n))
    c = g.random((n, n)) * 3
    theta = g.uniform(-math.pi, math.pi, (n, n))
    w = 1.0 / p.phi_sigma ** 2
    cur = phi.copy()
    for col in O.COLOURS:
        pp = O.OracleParams(n=n)
        ii, jj = np.meshgrid(np.arange(col[0], n, 2), np.arange(col[1], n, 2), indexing="ij")

        def cost(x):
            tot = -c[ii, jj] * np.cos(x - theta[ii, jj])
            for (di, dj, b) in O.NEIGHBOURS:
                i2, j2 = ii + di, jj + dj
                ok = (i2 >= 0) & (i2 < n) & (j2 >= 0) & (j2 < n)
                pj = cur[np.clip(i2, 0, n - 1), np.clip(j2, 0, n - 1)]
                tot = tot + np.where(ok, 0.5 * w * b * (x - pj) ** 2, 0.0)
            return tot

        before = cost(cur[ii, jj])
        # single colour step: run the ICD restricted to this colour
        saved = O.COLOURS
        try:
            O.COLOURS = (col,)
            nxt = O.phi_icd(cur, c, theta, pp)
        finally:
            O.COLOURS = saved
        after = cost(nxt[ii, jj])
        assert np.all(after <= before + 1e-12)
        cur = nxt
    assert np.allclose(cur, O.phi_icd(phi, c, theta, p), atol=1e-12)


# ------------------------------------------------------ EM as a whole


def _em_run(p, yhat, a, iters):
    n = p.n
    phi = np.zeros((n, n))
    u = O.adjoint(phi, yhat, a)
    r = np.maximum(p.boot_alpha * np.abs(u) ** 2, p.r_min)
    Js = [O.cost_J(r, phi, yhat, p, a)]
    for _ in range(iters):
        u = O.adjoint(phi, yhat, a)
        r, phi = O.em_update(r, phi, yhat, u, a, p)
        Js.append(O.cost_J(r, phi, yhat, p, a))
    return np.array(Js), r, phi


@pytest.mark.parametrize("prior", [True, False])
def test_em_cost_J_non_increasing_full_aperture(prior):
    """a = 1: the E-step is exact and both ICDs are MM steps, so (r, phi)-EM
    is a generalised EM and the MAP cost J of Eq. 2 never increases."""
    n = 16
    a = np.ones((n, n))
    p = O.OracleParams(n=n, aperture_mask=a, noise_var=0.2)
    if not prior:
        p.r_sigma = 0.0
        p.phi_sigma = 0.0
    cfg = dict(synth.CONFIGS["c1"], n=n, diam=n)
    y, _, _ = synth.make_stream(cfg, 0, frames=1)
    yhat = O.normalize(y[0].astype(np.complex128))
    Js, _, _ = _em_run(p, yhat, a, 12)
    dif = np.diff(Js)
    assert np.all(dif <= 1e-9 * np.abs(Js[:-1])), Js
    assert dif.sum() < 0


def test_em_cost_J_matches_dense_likelihood():
    """J's data term equals -log p(y|r,phi) + const from the dense covariance
    A(D(r) + s2 I)A^H (slogdet + solve), a = 1, N = 4."""
    n = 4
    P = n * n
    a = np.ones((n, n))
    p = O.OracleParams(n=n, aperture_mask=a, r_sigma=0.0, phi_sigma=0.0, noise_var=0.37)
    g = rng(40)
    r = g.random((n, n)) + 0.1
    phi = g.standard_normal((n, n))
    y = crandn(g, n, n)
    A = np.diag(np.exp(1j * phi.ravel())) @ dense_centred_dft(n).conj().T
    Sy = A @ np.diag(r.ravel()) @ A.conj().T + p.noise_var * np.eye(P)
    _, logdet = np.linalg.slogdet(Sy)
    nll = logdet + np.real(np.vdot(y.ravel(), np.linalg.solve(Sy, y.ravel())))
    assert O.cost_J(r, phi, y, p, a) == pytest.approx(nll, rel=1e-12)


def test_em_piston_equivariance_and_scale_relation():
    n = 16
    p = O.OracleParams(n=n, aperture_diam=14.0, noise_var=0.2)
    a = O.aperture_of(p)
    g = rng(41)
    r = g.random((n, n)) + 0.05
    phi = g.standard_normal((n, n))
    y = crandn(g, n, n)
    r1, p1 = O.em_update(r, phi, y, O.adjoint(phi, y, a), a, p)
    r2, p2 = O.em_update(r, phi + 0.9, y, O.adjoint(phi + 0.9, y, a), a, p)
    assert np.allclose(r1, r2, rtol=1e-10, atol=1e-12)
    assert np.allclose(p2 - p1, 0.9, atol=1e-10)
    # scale: y -> c y, s2 -> k s2, r -> k r, r_min -> k r_min, sig_r -> k sig_r, k = |c|^2
    cs = 1.7 - 0.6j
    k = abs(cs) ** 2
    ps = O.OracleParams(n=n, aperture_diam=14.0, noise_var=0.2 * k, r_min=1e-4 * k, r_sigma=0.5 * k)
    r3, p3 = O.em_update(k * r, phi, cs * y, O.adjoint(phi, cs * y, a), a, ps)
    assert np.allclose(r3, k * r1, rtol=1e-9)
    assert np.allclose(p3, p1, atol=1e-9)


# --------------------------------------------------------- loop + metrics


def test_ddh_step_degenerate_frame_keeps_state():
    p = O.OracleParams(n=8, aperture_diam=8)
    r = np.full((8, 8), 0.3)
    phi = np.ones((8, 8))
    r2, phi2, st = O.ddh_step(r, phi, np.full((8, 8), 1 + 1j), p)
    assert st == 1 and np.array_equal(r2, r) and np.array_equal(phi2, phi)


def test_ddh_step_lambda_endpoints():
    """lam = 0 -> r_init = r_prev; lam = 1 -> r_init = alpha |A^H y|^2 (Eq. 3)."""
    n = 8
    g = rng(50)
    y = crandn(g, n, n)
    a = O.aperture(n, 8)
    r = g.random((n, n)) + 0.1
    phi = g.standard_normal((n, n))
    p0 = O.OracleParams(n=n, aperture_diam=8, lam=0.0)
    yh = O.normalize(y)
    ph = O.remove_tip_tilt(phi, a)
    u = O.adjoint(ph, yh, a)
    mu, _, q = O.e_step(u, np.maximum(r, p0.r_min), p0.noise_var)
    exp_r = O.r_icd(np.maximum(r, p0.r_min), q, p0)
    r_out, _, _ = O.ddh_step(r, phi, y, p0, a)
    assert np.allclose(r_out, exp_r, atol=1e-13)
    p1 = O.OracleParams(n=n, aperture_diam=8, lam=1.0, alpha=0.3)
    r1 = np.maximum(0.3 * np.abs(u) ** 2, p1.r_min)
    mu, _, q = O.e_step(u, r1, p1.noise_var)
    r_out1, _, _ = O.ddh_step(r, phi, y, p1, a)
    assert np.allclose(r_out1, O.r_icd(r1, q, p1), atol=1e-13)


def test_bootstrap_period_larger_than_iters_is_plain_em():
    n = 16
    p = O.OracleParams(n=n, aperture_diam=16, boot_period=1000)
    g = rng(51)
    y = crandn(g, n, n)
    a = O.aperture_of(p)
    r, phi, st = O.bootstrap(y, p, 5, a)
    yh = O.normalize(y)
    phi2 = np.zeros((n, n))
    r2 = np.maximum(np.abs(O.adjoint(phi2, yh, a)) ** 2, p.r_min)
    for _ in range(5):
        r2, phi2 = O.em_update(r2, phi2, yh, O.adjoint(phi2, yh, a), a, p)
    assert st == 0 and np.allclose(r, r2) and np.allclose(phi, phi2)


def test_strehl_closed_forms():
    n = 64
    a = O.aperture(n, 64)
    g = rng(60)
    x, yy = O.plane_coords(n)
    zero = np.zeros((n, n))
    assert O.strehl(zero, zero, a) == pytest.approx(1.0, abs=1e-12)
    assert O.strehl(zero + 1.3, zero, a, remove_plane=False) == pytest.approx(1.0, abs=1e-12)
    assert O.strehl(0.3 + 0.05 * x - 0.02 * yy, zero, a) == pytest.approx(1.0, abs=1e-12)
    psi = g.standard_normal((n, n)) * 0.5
    assert O.strehl(psi, zero, a) == pytest.approx(O.strehl(-psi, zero, a), rel=1e-12)
    # uncorrected D/r0 = 10 screen -> S < 0.2
    c = synth.screen_coeffs(n, n, n / 10.0, np.random.default_rng(5))
    scr = synth.remove_plane(synth.screen_from_coeffs(c), a)
    assert O.strehl(zero, scr, a) < 0.2


def test_zero_turbulence_high_snr_recovers_flat_phase():
    """north_star pin: zero turbulence at high SNR -> Strehl ~ 1."""
    cfg = dict(synth.CONFIGS["c1"], d_r0=0.0, snr_db=40.0)
    y, ph_true, _ = synth.make_stream(cfg, 0, frames=6)
    p = O.OracleParams(n=64, aperture_diam=64, noise_var=synth.recon_noise_var(64, 64, 40.0))
    a = O.aperture_of(p)
    r, phi, _ = O.bootstrap(y[0], p, 20, a)
    for t in range(1, 6):
        r, phi, _ = O.ddh_step(r, phi, y[t], p, a)
        assert O.strehl(phi, ph_true[t], a) > 0.98


# ------------------------------------------------------------- simulator


def test_paper_velocity_golden():
    rows = [l.split() for l in open(os.path.join(GOLDEN, "paper_velocity.txt")) if not l.startswith("#")]
    n, fs, fg, dr0, vx, vy = map(float, rows[0])
    v = synth.flow_velocity(fg, fs, int(n), dr0)
    assert v == pytest.approx(0.5953, abs=5e-5)
    assert round(v / math.sqrt(2), 3) == vx == vy


def test_paper_parameters_golden():
    vals = dict(l.split() for l in open(os.path.join(GOLDEN, "paper_parameters.txt")) if not l.startswith("#"))
    p = O.OracleParams()
    assert p.alpha == float(vals["alpha"]) and p.lam == float(vals["lambda"])
    assert p.boot_period == int(vals["boot_period"])


def test_structure_function_matches_discrete_expectation():
    m, r0 = 128, 8.0
    acc = {d: 0.0 for d in (2, 4, 8, 16)}
    seeds = 20
    for s in range(seeds):
        scr = synth.screen_from_coeffs(synth.screen_coeffs(m, m, r0, np.random.default_rng(s)))
        for d in acc:
            acc[d] += 0.5 * (np.mean((np.roll(scr, -d, 0) - scr) ** 2) + np.mean((np.roll(scr, -d, 1) - scr) ** 2))
    for d in acc:
        exp = synth.structure_function_expected(m, m, r0, (d, 0))
        assert acc[d] / seeds == pytest.approx(exp, rel=0.05)


def test_speckle_and_snr_statistics():
    cfg = dict(synth.CONFIGS["c1"], d_r0=0.0)
    y, _, r = synth.make_stream(cfg, 0, frames=20, snr_db=10.0)
    a = synth.aperture_mask(64, 64)
    # E|F_c^{-1} g|^2 = mean(r) at every pixel; noise = mean(r)/10
    p_in = np.mean(np.abs(y[:, a > 0]) ** 2)
    p_out = np.mean(np.abs(y[:, a == 0]) ** 2)
    snr = (p_in - p_out) / p_out
    assert snr == pytest.approx(10.0, rel=0.05)
    assert p_in == pytest.approx(r.mean() * 1.1, rel=0.02)


def test_icd_stencils_are_tangent_to_J_pair_sums():
    """The ICD neighbour weights/sets are pinned to the pair sums of J
    (written independently as each unordered pair once): the gradient of the
    r surrogate's prior part, 2(B r_i - S), and of the phi prior,
    w (sum b phi_i - sum b phi_j), equal the finite-difference gradient of
    J's prior terms at every pixel (edges included)."""
    n = 8
    p = O.OracleParams(n=n, aperture_mask=np.ones((n, n)), noise_var=0.3)
    a = np.ones((n, n))
    g = rng(70)
    r = g.random((n, n)) + 0.2
    phi = g.standard_normal((n, n))
    y = crandn(g, n, n)
    h = 1e-6
    ii, jj = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    ii, jj = ii.ravel(), jj.ravel()
    B, S = O.r_prior_coeffs(r, ii, jj, p)
    nb, sb = O.phi_prior_coeffs(phi, ii, jj)
    w = 1.0 / p.phi_sigma ** 2
    for k in range(n * n):
        i, j = ii[k], jj[k]
        e = np.zeros((n, n))
        e[i, j] = h
        dJr = (O.cost_J_parts(r + e, phi, y, p, a)[1] - O.cost_J_parts(r - e, phi, y, p, a)[1]) / (2 * h)
        dJp = (O.cost_J_parts(r, phi + e, y, p, a)[2] - O.cost_J_parts(r, phi - e, y, p, a)[2]) / (2 * h)
        assert dJr == pytest.approx(2 * (B[k] * r[i, j] - S[k]), rel=1e-6, abs=1e-8)
        assert dJp == pytest.approx(w * (sb[k] * phi[i, j] - nb[k]), rel=1e-6, abs=1e-8)


# ------------------------------------------- pins added after the round-1 mutation run


def test_qggmrf_potential_shape_and_exponents():
    """R6 fixes the qGGMRF potential with p = 2 (north_star "qGGMRF"): near zero
    it is the Gaussian Delta^2/(2 sigma^2) (exponent p = 2), in the tail it grows
    as |Delta|^q, and the transition sits at |Delta| = T sigma where the two
    branches have equal weight (rho = T^2/4 there).  These follow from the
    definition rho = |D|^p/(p sig^p) / (1 + |D/(T sig)|^(p-q)) and are checked
    on log-log slopes measured by finite differences of log rho, so a swapped
    exponent (q for 2-q) or a misplaced T fails."""
    for sig, T, q in [(0.5, 1.0, 1.2), (0.2, 2.0, 1.5), (1.3, 0.5, 1.05)]:
        # Gaussian limit at zero
        for d in (1e-14 * T * sig, -1e-14 * T * sig):
            rho = float(O.qggmrf_rho(np.array(d), sig, T, q))
            assert rho * 2 * sig * sig / (d * d) == pytest.approx(1.0, abs=1e-6)
        # local log-log slopes
        def slope(d):
            h = 1e-4
            return (math.log(float(O.qggmrf_rho(np.array(d * math.exp(h)), sig, T, q)))
                    - math.log(float(O.qggmrf_rho(np.array(d * math.exp(-h)), sig, T, q)))) / (2 * h)
        assert slope(1e-7 * T * sig) == pytest.approx(2.0, abs=1e-3)
        assert slope(1e9 * T * sig) == pytest.approx(q, abs=1e-3)
        assert slope(-1e9 * T * sig) == pytest.approx(q, abs=1e-3)
        # transition point: the two factors are equal (t = 1)
        assert float(O.qggmrf_rho(np.array(T * sig), sig, T, q)) == pytest.approx(T * T / 4.0, rel=1e-12)
        # the slope at the transition is the mean of the two exponents
        assert slope(T * sig) == pytest.approx((2.0 + q) / 2.0, abs=1e-6)


@pytest.mark.parametrize("n", [4])
def test_phase_correlation_is_expected_complete_data_loglik(n):
    """The phi M-step data term sum_i c_i cos(phi_i - theta_i) must equal the
    phi-dependent part of Q(phi) = E[log p(y | g, phi)] = -E||y - A_phi g||^2/s2
    + const (EM; y = A g + w, w ~ CN(0, s2 I)), with the
    expectation over the posterior of g at the current (r, phi0).  Q is built
    densely here: posterior mean and covariance by textbook Gaussian
    conditioning, A_phi from the DFT definition, the trace term written out.
    a = 1 (exact E-step).  Pins the factor 2/s2 in c and the sign of theta."""
    g = rng(80)
    P = n * n
    a = np.ones((n, n))
    s2 = 0.37
    r = g.random((n, n)) * 2 + 0.05
    phi0 = g.standard_normal((n, n))
    y = crandn(g, n, n)
    Fc = dense_centred_dft(n)

    def A_of(phi):
        return np.diag(np.exp(1j * phi.ravel())) @ Fc.conj().T

    A0 = A_of(phi0)
    Dr = np.diag(r.ravel())
    Sy = A0 @ Dr @ A0.conj().T + s2 * np.eye(P)
    K = Dr @ A0.conj().T @ np.linalg.inv(Sy)
    mu = K @ y.ravel()
    Sig = Dr - K @ A0 @ Dr
    M2 = Sig + np.outer(mu, mu.conj())      # E[g g^H]

    def Q(phi):
        A = A_of(phi)
        e = (np.vdot(y.ravel(), y.ravel()) - 2 * np.real(np.vdot(y.ravel(), A @ mu))
             + np.real(np.trace(A.conj().T @ A @ M2)))
        return -np.real(e) / s2

    # the oracle's data term from its own E-step and second FFT
    mu_o, _, _ = O.e_step(O.adjoint(phi0, y, a), r, s2)
    c, theta = O.phase_correlation(y, O.ifft2c(mu_o), a, s2)

    def D(phi):
        return float(np.sum(c * np.cos(phi - theta)))

    for k in range(5):
        phi = phi0 + g.standard_normal((n, n)) * (0.3 + k)
        lhs = Q(phi) - Q(phi0)
        rhs = D(phi) - D(phi0)
        assert lhs == pytest.approx(rhs, rel=1e-10, abs=1e-10 * abs(Q(phi0)))
    # and the gradient at phi0 (finite differences of the dense Q)
    h = 1e-6
    for k in range(P):
        e = np.zeros(P)
        e[k] = h
        e = e.reshape(n, n)
        gq = (Q(phi0 + e) - Q(phi0 - e)) / (2 * h)
        gd = float((-c * np.sin(phi0 - theta)).ravel()[k])
        assert gq == pytest.approx(gd, rel=1e-6, abs=1e-8)


def test_bootstrap_resets_every_period():
    """the bootstrap resets r to a back-projected estimate every P_b
    iterations ([pellizzari2017b], "every 200 iterations").  K_b = 5, P_b = 2:
    resets happen before iterations 0, 2 and 4, written out by hand."""
    n = 16
    p = O.OracleParams(n=n, aperture_diam=14, boot_period=2, boot_alpha=0.7)
    g = rng(81)
    y = crandn(g, n, n) * 1.3
    a = O.aperture_of(p)
    r, phi, st = O.bootstrap(y, p, 5, a)
    yh = O.normalize(y)
    r2 = np.full((n, n), p.r_min)
    phi2 = np.zeros((n, n))
    for k in range(5):
        u = O.adjoint(phi2, yh, a)
        if k in (0, 2, 4):
            r2 = np.maximum(0.7 * np.abs(u) ** 2, p.r_min)
        r2, phi2 = O.em_update(r2, phi2, yh, u, a, p)
    assert st == 0
    assert np.allclose(r, r2, rtol=1e-12, atol=1e-14) and np.allclose(phi, phi2, rtol=1e-12, atol=1e-14)
    # and it differs from the run with a single reset at k = 0 (the pin discriminates)
    r3 = np.full((n, n), p.r_min)
    phi3 = np.zeros((n, n))
    for k in range(5):
        u = O.adjoint(phi3, yh, a)
        if k == 0:
            r3 = np.maximum(0.7 * np.abs(u) ** 2, p.r_min)
        r3, phi3 = O.em_update(r3, phi3, yh, u, a, p)
    assert np.max(np.abs(r3 - r)) > 1e-3


def test_remove_tip_tilt_removes_piston_and_plane():
    """R17: RemoveTipTilt (Fig. 1) removes the LS plane including piston,
    so a pure plane (any piston) maps to exactly zero at every pixel, and the
    residual of any phase has zero mean and zero x/y moments over the aperture."""
    n = 32
    a = O.aperture(n, 30.0)
    x, yy = O.plane_coords(n)
    out = O.remove_tip_tilt(2.0 + 3.0 * x - 1.0 * yy, a)
    assert np.max(np.abs(out)) < 1e-11
    res = O.remove_tip_tilt(rng(82).standard_normal((n, n)), a)
    m = a > 0
    for basis in (np.ones((n, n)), x, yy):
        assert abs(np.sum(res[m] * basis[m])) < 1e-9


def _hand_r_icd(r, q, p):
    """Pixel-by-pixel colour-ordered ICD written out with plain loops (R8):
    colours (0,0),(0,1),(1,0),(1,1); inside a colour, raster order; each pixel
    minimises the per-pixel surrogate (R9) given its current neighbours."""
    r = r.copy()
    n = r.shape[0]
    for (ci, cj) in ((0, 0), (0, 1), (1, 0), (1, 1)):
        for i in range(ci, n, 2):
            for j in range(cj, n, 2):
                B = S = 0.0
                for (di, dj, b) in ((-1, 0, 1 / 6), (1, 0, 1 / 6), (0, -1, 1 / 6), (0, 1, 1 / 6),
                                    (-1, -1, 1 / 12), (-1, 1, 1 / 12), (1, -1, 1 / 12), (1, 1, 1 / 12)):
                    rj = r[(i + di) % n, (j + dj) % n]
                    bt = b * float(O.qggmrf_weight(np.array(r[i, j] - rj), p.r_sigma, p.r_T, p.r_q))
                    B += bt
                    S += bt * rj
                r[i, j] = O.r_update_pixels(np.array([r[i, j]]), np.array([q[i, j]]),
                                            np.array([B]), np.array([S]), p.r_min)[0]
    return r


def _hand_phi_icd(phi, c, theta, p):
    """Pixel-by-pixel GMRF phi-ICD (R8, R11) with plain loops: colour order as R8,
    raster inside a colour, free boundary (neighbours off the grid dropped)."""
    phi = phi.copy()
    n = phi.shape[0]
    w = 1.0 / p.phi_sigma ** 2
    for (ci, cj) in ((0, 0), (0, 1), (1, 0), (1, 1)):
        for i in range(ci, n, 2):
            for j in range(cj, n, 2):
                x0 = math.remainder(phi[i, j] - theta[i, j], 2 * math.pi)
                if x0 == -math.pi:
                    x0 = math.pi
                s = 1.0 if x0 == 0 else math.sin(x0) / x0
                nb = sb = 0.0
                for (di, dj, b) in ((-1, 0, 1 / 6), (1, 0, 1 / 6), (0, -1, 1 / 6), (0, 1, 1 / 6),
                                    (-1, -1, 1 / 12), (-1, 1, 1 / 12), (1, -1, 1 / 12), (1, 1, 1 / 12)):
                    if 0 <= i + di < n and 0 <= j + dj < n:
                        nb += b * phi[i + di, j + dj]
                        sb += b
                num = c[i, j] * s * (phi[i, j] - x0) + w * nb
                den = c[i, j] * s + w * sb
                if den != 0:
                    phi[i, j] = num / den
    return phi


def test_icd_sweeps_equal_hand_written_sequential_sweeps():
    """R8: the vectorised colour-phase ICDs equal a pixel-by-pixel sequential
    sweep in the colour order (0,0),(0,1),(1,0),(1,1) (brute force, N = 6, with
    values spread so the colour order changes the result)."""
    n = 6
    p = O.OracleParams(n=n)
    g = rng(83)
    r = g.random((n, n)) * 2 + 0.01
    q = g.random((n, n)) * 3 + 0.01
    assert np.allclose(O.r_icd(r, q, p), _hand_r_icd(r, q, p), rtol=1e-12, atol=1e-14)
    phi = g.standard_normal((n, n)) * 2
    c = g.random((n, n)) * 4
    theta = g.uniform(-math.pi, math.pi, (n, n))
    assert np.allclose(O.phi_icd(phi, c, theta, p), _hand_phi_icd(phi, c, theta, p), rtol=1e-12, atol=1e-13)


def test_ddh_step_n_k_two_recomputes_the_back_projection():
    """Fig. 1 P:169-171 / a9: with N_k = 2 the second EM iteration runs the
    E-step on u = A^H_{phi_1} y, the back-projection through the phase the
    first iteration produced (same normalised y, no second Eq. 3)."""
    n = 16
    p2 = O.OracleParams(n=n, aperture_diam=14, n_k=2, noise_var=0.2)
    p1 = O.OracleParams(n=n, aperture_diam=14, n_k=1, noise_var=0.2)
    a = O.aperture_of(p2)
    g = rng(84)
    y = crandn(g, n, n)
    r = g.random((n, n)) + 0.05
    phi = g.standard_normal((n, n))
    r_a, phi_a, _ = O.ddh_step(r, phi, y, p2, a)
    r_b, phi_b, _ = O.ddh_step(r, phi, y, p1, a)
    yh = O.normalize(y)
    r_b, phi_b = O.em_update(r_b, phi_b, yh, O.adjoint(phi_b, yh, a), a, p1)
    assert np.allclose(r_a, r_b, rtol=1e-12, atol=1e-14) and np.allclose(phi_a, phi_b, rtol=1e-12, atol=1e-14)


def test_r_update_exact_tie_picks_candidate_nearest_current():
    """SURVEY 8.c.4 tie rule: two local minima x1 < x3 of the surrogate with
    equal cost -> the one nearest the current r.  The tie is constructed in
    closed form: the stationary points are the roots of 2B(x-x1)(x-x2)(x-x3),
    so B = 1/(2 e2), S = B e1, q = 2B e3, and x2 is solved so f(x1) = f(x3)."""
    x1, x3 = 0.3, 2.0

    def coeffs(x2):
        e1, e2, e3 = x1 + x2 + x3, x1 * x2 + x1 * x3 + x2 * x3, x1 * x2 * x3
        B = 1.0 / (2.0 * e2)
        return 2.0 * B * e3, B, B * e1

    def gap(x2):
        q, B, S = coeffs(x2)
        f = lambda x: math.log(x) + q / x + B * x * x - 2 * S * x
        return f(x1) - f(x3)

    lo, hi = x1 + 1e-6, x3 - 1e-6
    assert gap(lo) * gap(hi) < 0
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        if gap(lo) * gap(mid) <= 0:
            hi = mid
        else:
            lo = mid
    q, B, S = coeffs(0.5 * (lo + hi))
    qv, Bv, Sv = np.array([q, q]), np.array([B, B]), np.array([S, S])
    out = O.r_update_pixels(np.array([0.25, 2.4]), qv, Bv, Sv, 1e-4)
    assert out[0] == pytest.approx(x1, rel=1e-9) and out[1] == pytest.approx(x3, rel=1e-9)


def test_guided_tie_rule_only_moves_near_ties():
    """The parity tests' guided oracle: a guide changes the
    choice only among candidates within guide_tol of the minimum; a pixel with
    a unique minimiser ignores it."""
    x1, x3 = 0.3, 2.0

    def coeffs(x2):
        e1, e2, e3 = x1 + x2 + x3, x1 * x2 + x1 * x3 + x2 * x3, x1 * x2 * x3
        B = 1.0 / (2.0 * e2)
        return 2.0 * B * e3, B, B * e1

    def gap(x2):
        q, B, S = coeffs(x2)
        return (math.log(x1) + q / x1 + B * x1 * x1 - 2 * S * x1) - (math.log(x3) + q / x3 + B * x3 * x3 - 2 * S * x3)

    lo, hi = x1 + 1e-6, x3 - 1e-6
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        lo, hi = (lo, mid) if gap(lo) * gap(mid) <= 0 else (mid, hi)
    q, B, S = coeffs(0.5 * (lo + hi))
    one = lambda v: np.array([v])
    # near tie: the guide decides, whatever the current value
    assert O.r_update_pixels(one(0.25), one(q), one(B), one(S), 1e-4, guide=one(1.9))[0] == pytest.approx(x3, rel=1e-9)
    assert O.r_update_pixels(one(2.4), one(q), one(B), one(S), 1e-4, guide=one(0.31))[0] == pytest.approx(x1, rel=1e-9)
    # unique minimiser: the guide is ignored
    g = rng(85)
    m = 200
    qq = g.random(m) * 3 + 1e-3
    BB = g.random(m) * 4 + 0.05
    SS = BB * g.random(m)
    rc = g.random(m) + 1e-3
    best, gp = O.r_update_pixels(rc, qq, BB, SS, 1e-4, return_gap=True)
    uniq = gp > 1e-4
    gd = O.r_update_pixels(rc, qq, BB, SS, 1e-4, guide=g.random(m) * 10)
    assert uniq.sum() > m // 2 and np.array_equal(gd[uniq], best[uniq])


def test_residual_phase_and_psf_closed_forms():
    """Residual phase / PSF: a perfect estimate (up to piston and
    tilt) leaves zero residual and the diffraction-limited PSF whose peak is 1
    at the centre; the PSF of any residual carries the aperture's energy
    (Parseval: sum_k psf_k = N^2 / sum a, since max|F_c^{-1} a|^2 = (sum a)^2 / N^2)
    and its maximum is the Strehl ratio; the residual is -psi wrapped."""
    n = 32
    a = O.aperture(n, 30.0)
    x, yy = O.plane_coords(n)
    g = rng(90)
    phi = g.standard_normal((n, n)) * 2
    hat = phi + 0.7 + 0.1 * x - 0.05 * yy
    assert np.max(np.abs(O.residual_phase(hat, phi, a))) < 1e-12
    psf0 = O.residual_psf(hat, phi, a)
    assert psf0.max() == pytest.approx(1.0, abs=1e-12) and psf0[n // 2, n // 2] == pytest.approx(1.0, abs=1e-12)
    dense = np.abs(dense_centred_dft(n).conj().T @ a.ravel()) ** 2  # F_c^{-1} a from the definition
    assert np.allclose(psf0.ravel(), dense / dense.max(), atol=1e-12)
    err = g.standard_normal((n, n)) * 0.6
    psf = O.residual_psf(phi + err, phi, a)
    assert psf.sum() == pytest.approx(n * n / a.sum(), rel=1e-12)
    assert psf.max() == pytest.approx(O.strehl(phi + err, phi, a), rel=1e-12)
    res = O.residual_phase(phi + err, phi, a)
    ref = -O.remove_tip_tilt(err, a)
    d = np.angle(np.exp(1j * (res - ref)))
    assert np.max(np.abs(d[a > 0])) < 1e-12 and np.all(res[a == 0] == 0)
    assert np.all(np.abs(res) <= math.pi)
