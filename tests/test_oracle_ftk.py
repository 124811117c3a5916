"""Pins for oracle.ftk / oracle.brute / oracle.closed_form (no GPU).

FTK (Steps 1-3) is pinned to the brute-force definition (no Bessel/SVD/FFT), which is pinned to
the exact Gaussian inner products; plus special cases that reduce to textbook quantities.
"""
import math

import numpy as np
import pytest

from oracle import brute, closed_form, fb, ftk, kernel_svd as ks
import synth


def _plan(cfg, eps=None, shifts=None):
    sh = synth.shift_list(cfg) if shifts is None else shifts
    return ks.build_plan(cfg.n, cfg.K, synth.delta_max(cfg), sh, cfg.eps if eps is None else eps, cfg.n_k, cfg.n_psi)


@pytest.fixture(scope="module")
def tiny():
    cfg = synth.config("tiny")
    plan = _plan(cfg)
    imgs, pi = synth.draw_items(cfg, "images", range(4), plan.k, "planted")
    tpls, pt = synth.draw_items(cfg, "templates", range(4), plan.k)
    return cfg, plan, imgs, tpls, pi, pt


def test_tiny_plan_shape(tiny):
    cfg, plan, *_ = tiny
    assert plan.H == 27 and plan.H_plus == 15          # SURVEY Sec. 8 table [calc], strict Sigma > eps
    assert abs(plan.W - 0.75 * math.sqrt(2) / 2) < 1e-15


def test_ftk_vs_brute_force_tiny(tiny):
    """|X^FTK - X^bf| <= 4 eps ||A|| ||B|| per inner product (north star), full landscapes."""
    cfg, plan, imgs, tpls, *_ = tiny
    X = ftk.ftk_landscapes(fb.fb_coeffs(imgs), fb.fb_coeffs(tpls), plan)
    na, nb = fb.discrete_norm(imgs, plan.w), fb.discrete_norm(tpls, plan.w)
    for i in range(4):
        for j in range(4):
            Xb = brute.brute_landscape(imgs[i], tpls[j], plan.k, plan.w, plan.shifts)
            assert np.max(np.abs(X[i, j] - Xb)) <= 4 * cfg.eps * na[i] * nb[j]
    assert np.max(np.abs(X.imag)) < 1e-12 * np.max(np.abs(X.real))   # real images -> Im X = 0


def test_ftk_tends_to_brute_force_as_eps_shrinks(tiny):
    cfg, _, imgs, tpls, *_ = tiny
    plan = _plan(cfg, eps=1e-9)
    X = ftk.ftk_landscapes(fb.fb_coeffs(imgs[:1]), fb.fb_coeffs(tpls[:2]), plan)
    for j in range(2):
        Xb = brute.brute_landscape(imgs[0], tpls[j], plan.k, plan.w, plan.shifts)
        assert np.max(np.abs(X[0, j] - Xb)) < 1e-7 * np.max(np.abs(Xb))


def test_brute_force_vs_closed_form(tiny):
    """Brute force vs (2 pi)^2 <R T A, B> in closed form: quadrature-limited at tiny (n_k = 16)."""
    cfg, plan, imgs, tpls, pi, pt = tiny
    na, nb = fb.discrete_norm(imgs, plan.w), fb.discrete_norm(tpls, plan.w)
    for i, j in [(0, 0), (1, 3), (3, 2)]:
        Xb = brute.brute_landscape(imgs[i], tpls[j], plan.k, plan.w, plan.shifts)
        for t, r in [(0, 0), (24, 0), (13, 17), (48, 63)]:
            cf = closed_form.gaussian_ip(pi, pt, i, j, plan.shifts[t], 2 * math.pi * r / cfg.n_psi)
            assert abs(Xb[t, r] - cf) < 3e-3 * na[i] * nb[j]


@pytest.mark.parametrize("name,tol", [("c2", 1e-4), ("c3", 1e-6)])
def test_brute_force_vs_closed_form_configs(name, tol):
    cfg = synth.config(name)
    plan = _plan(cfg, shifts=synth.shift_list(cfg)[:3])
    x, px = synth.draw_items(cfg, "images", [0, 1], plan.k, noise=False)
    y, py = synth.draw_items(cfg, "templates", [0], plan.k, noise=False)
    for i in range(2):
        for t, r in [(0, 0), (2, 5)]:
            v = brute.brute_points(x[i], y[0], plan.k, plan.w, plan.shifts, [t], [r])[0]
            cf = closed_form.gaussian_ip(px, py, i, 0, plan.shifts[t], 2 * math.pi * r / cfg.n_psi)
            assert abs(v - cf) < tol * (2 * math.pi) ** 2


def test_zero_shift_is_rotational_correlation_and_plain_ip(tiny):
    """delta = 0: U(0; l != 0) = 0 so X(0, gamma) = 2 pi sum_m w_m sum_q a conj(b) e^{-i q gamma}
    (P:583-589 with L = 0); at gamma = 0 the plain discrete inner product (no transform at all)."""
    cfg, _, imgs, tpls, *_ = tiny
    plan = _plan(cfg, shifts=np.zeros((1, 2)))
    a, b = fb.fb_coeffs(imgs[:2]), fb.fb_coeffs(tpls[:2])
    X = ftk.ftk_landscapes(a, b, plan)
    n = cfg.n_psi
    q = np.arange(n)
    for i in range(2):
        for j in range(2):
            for r in (0, 7, 40):
                ref = 2 * math.pi * np.sum(plan.w[:, None] * a[i] * np.conj(b[j]) * np.exp(-2j * math.pi * q * r / n)[None, :])
                assert abs(X[i, j, 0, r] - ref) < 1.5 * cfg.eps * 40
            plain = (2 * math.pi / n) * np.sum(plan.w[:, None] * imgs[i].astype(complex) * np.conj(tpls[j].astype(complex)))
            assert abs(X[i, j, 0, 0] - plain) <= cfg.eps * 40


def test_template_rotation_is_cyclic_shift(tiny):
    """Template rotated by 2 pi j/n_psi (samples rolled by j) -> X'(t, r) = X(t, r - j), exactly."""
    cfg, plan, imgs, tpls, *_ = tiny
    a = fb.fb_coeffs(imgs[:1])
    b = fb.fb_coeffs(tpls[:1])
    b_rot = fb.fb_coeffs(np.roll(tpls[:1], 5, axis=-1))
    X = ftk.ftk_landscapes(a, b, plan)[0, 0]
    Xr = ftk.ftk_landscapes(a, b_rot, plan)[0, 0]
    assert np.max(np.abs(Xr - np.roll(X, 5, axis=-1))) < 1e-12 * np.max(np.abs(X))


def test_image_rotation_by_quarter_turn(tiny):
    """Image rotated by alpha = pi/2 (roll n/4): X'(delta, gamma) = X(R_{-alpha} delta, gamma + alpha);
    the square lattice maps to itself, so one plan serves both sides (F^SVD is rotation-covariant)."""
    cfg, plan, imgs, tpls, *_ = tiny
    n = cfg.n_psi
    a = fb.fb_coeffs(imgs[:1])
    a_rot = fb.fb_coeffs(np.roll(imgs[:1], n // 4, axis=-1))
    b = fb.fb_coeffs(tpls[1:2])
    X = ftk.ftk_landscapes(a, b, plan)[0, 0]
    Xr = ftk.ftk_landscapes(a_rot, b, plan)[0, 0]
    sh = plan.shifts
    rot = np.stack([sh[:, 1], -sh[:, 0]], 1)          # R_{-pi/2} delta
    idx = [int(np.argmin(np.hypot(*(sh - p).T))) for p in rot]
    for t in range(sh.shape[0]):
        assert np.max(np.abs(Xr[t] - np.roll(X[idx[t]], -n // 4))) < 1e-12 * np.max(np.abs(X))


def test_linearity_and_scale(tiny):
    cfg, plan, imgs, tpls, *_ = tiny
    a, b = fb.fb_coeffs(imgs[:2]), fb.fb_coeffs(tpls[:1])
    X = ftk.ftk_landscapes(a, b, plan)
    Xc = ftk.ftk_landscapes(2.0 * a[:1] - 0.5 * a[1:2], b, plan)
    assert np.max(np.abs(Xc[0] - (2.0 * X[0] - 0.5 * X[1]))) < 1e-12 * np.max(np.abs(X))
    v, j, t, r, _ = ftk.best_per_image(X)
    v2, j2, t2, r2, _ = ftk.best_per_image(3.0 * X)
    assert np.array_equal(np.stack([j, t, r]), np.stack([j2, t2, r2]))


def test_planted_recovery_noiseless(tiny):
    """P:1324 consistency check: argmax = (j0, -delta0, -gamma0) (reading R12)."""
    cfg, plan, imgs, tpls, *_ = tiny
    X = ftk.ftk_landscapes(fb.fb_coeffs(imgs), fb.fb_coeffs(tpls), plan)
    v, j, t, r, _ = ftk.best_per_image(X)
    sh = plan.shifts
    for i in range(4):
        j0, t0, r0 = synth.planted_truth(cfg, i, sh.shape[0])
        assert j[i] == j0
        assert np.allclose(sh[t[i]], -sh[t0])
        assert r[i] == (-r0) % cfg.n_psi


def test_argmax_tie_break():
    X = np.zeros((1, 2, 3, 4))
    X[0, 1, 0, 0] = 1.0
    X[0, 0, 2, 3] = 1.0
    v, j, t, r, gap = ftk.best_per_image(X)
    assert (j[0], t[0], r[0]) == (0, 2, 3) and gap[0] == 0.0


def test_ftk_best_blocked_equals_full(tiny):
    cfg, plan, imgs, tpls, *_ = tiny
    a, b = fb.fb_coeffs(imgs), fb.fb_coeffs(tpls)
    v, j, t, r, _ = ftk.best_per_image(ftk.ftk_landscapes(a, b, plan))
    bv, bi = ftk.ftk_best(a, b, plan, chunk_i=3, chunk_j=3)
    assert np.allclose(bv, v, rtol=1e-13) and np.all(bi[:, 0] == j) and np.all(bi[:, 1] == t) and np.all(bi[:, 2] == r)


def test_c2_ftk_vs_brute_sampled():
    """c2 (W=1, eps=1e-2, SNR 1), sampled inner products."""
    cfg = synth.config("c2")
    plan = _plan(cfg)
    assert plan.H == 36 and plan.H_plus == 20
    x, _ = synth.draw_items(cfg, "images", [0, 1], plan.k)
    y, _ = synth.draw_items(cfg, "templates", [0, 1], plan.k)
    X = ftk.ftk_landscapes(fb.fb_coeffs(x), fb.fb_coeffs(y), plan)
    na, nb = fb.discrete_norm(x, plan.w), fb.discrete_norm(y, plan.w)
    rng = np.random.default_rng(3)
    T = rng.integers(0, plan.shifts.shape[0], 25)
    R = rng.integers(0, cfg.n_psi, 25)
    for i in range(2):
        for j in range(2):
            v = brute.brute_points(x[i], y[j], plan.k, plan.w, plan.shifts, T, R)
            assert np.max(np.abs(X[i, j][T, R] - v)) <= 4 * cfg.eps * na[i] * nb[j]


# ---------------- more rotations than angular samples (n_gamma > n_psi, reading R21)

def _small_exact_plan():
    """n = 32 px, n_k = 32 (radial rule exact to ~1e-11 for these blobs), n_psi = 64, eps = 1e-5."""
    cfg = synth.config("tiny", n_k=32, eps=1e-5)
    sh = synth.shift_list(cfg)[[0, 24, 30]]
    plan = ks.build_plan(cfg.n, cfg.K, synth.delta_max(cfg), sh, cfg.eps, cfg.n_k, cfg.n_psi, n_nodes=96)
    return cfg, plan


def test_n_gamma_grid_subsampling_and_reality():
    """Every (n_gamma / n_psi)-th rotation reproduces the n_gamma = n_psi landscape (the zero padding
    changes no grid value), and for real images X stays real at the new angles too (only the symmetric
    Nyquist split has this property)."""
    cfg, plan = _small_exact_plan()
    cfg = synth.config("tiny", n_k=32, eps=1e-5, snr=0.5)  # white noise: energy up to the Nyquist index
    x, _ = synth.draw_items(cfg, "images", [0, 1], plan.k)
    y, _ = synth.draw_items(cfg, "templates", [0, 1, 2], plan.k)
    a, b = fb.fb_coeffs(x), fb.fb_coeffs(y)
    assert np.min(np.abs(a[..., cfg.n_psi // 2])) > 0.0
    X1 = ftk.ftk_landscapes(a, b, plan)
    X4 = ftk.ftk_landscapes(a, b, plan, n_gamma=4 * cfg.n_psi)
    scale = np.max(np.abs(X1))
    assert np.max(np.abs(X4[..., ::4] - X1)) < 1e-12 * scale
    assert np.max(np.abs(np.imag(X4))) < 1e-12 * scale


def test_n_gamma_off_grid_matches_closed_form():
    """Off-grid rotations gamma = 2 pi r / n_gamma (r odd) of noiseless Gaussian-blob images against
    the exact (2 pi)^2 <R_gamma T_delta A, B> (closed form, any gamma): the trigonometric interpolation
    of Step 2 is exact for angularly band-limited data, so the error is the FTK one (<= 4 eps) plus the
    quadrature error."""
    cfg, plan = _small_exact_plan()
    x, px = synth.draw_items(cfg, "images", [0], plan.k, noise=False)
    y, py = synth.draw_items(cfg, "templates", [0], plan.k, noise=False)
    ng = 4 * cfg.n_psi
    X = np.real(ftk.ftk_landscapes(fb.fb_coeffs(x), fb.fb_coeffs(y), plan, n_gamma=ng))[0, 0]
    na = fb.discrete_norm(x, plan.w)[0]
    nb = fb.discrete_norm(y, plan.w)[0]
    worst = 0.0
    for t in range(plan.shifts.shape[0]):
        for r in range(1, ng, 7):
            cf = closed_form.gaussian_ip(px, py, 0, 0, plan.shifts[t], 2 * math.pi * r / ng)
            worst = max(worst, abs(X[t, r] - cf) / (na * nb))
    assert worst < 4 * plan.eps + 1e-8, worst


def test_n_gamma_planted_off_grid_rotation_recovered():
    """A template rotated by an off-grid angle gamma0 (analytic blobs) peaks at gamma = -gamma0 on the
    finer rotation grid (reading R12), which the n_psi grid cannot represent."""
    cfg, plan = _small_exact_plan()
    k = plan.k
    py = synth.blob_params(cfg, "templates", [0])
    ng = 8 * cfg.n_psi
    r0 = 37                                   # gamma0 = 2 pi r0 / ng: not a multiple of ng / n_psi
    g0 = 2 * math.pi * r0 / ng
    c, s = math.cos(g0), math.sin(g0)
    px = {key: np.array(v, copy=True) for key, v in py.items()}
    px["cx"], px["cy"] = c * py["cx"] - s * py["cy"], s * py["cx"] + c * py["cy"]
    x = synth.polar_samples(px, k, cfg.n_psi)
    y = synth.polar_samples(py, k, cfg.n_psi)
    X = np.real(ftk.ftk_landscapes(fb.fb_coeffs(x), fb.fb_coeffs(y), plan, n_gamma=ng))[0, 0]
    t0 = int(np.argmin(np.sum(plan.shifts ** 2, axis=1)))     # delta = 0
    assert int(np.argmax(X[t0])) == (ng - r0) % ng


# ---------------------------------------------------------------- marginalization (NEXT-3, reading R22)
def test_log_marginal_closed_forms():
    """log sum_{t,r} exp(X / tau) against closed forms: a constant landscape gives c / tau + log(N_t n_gamma);
    a two-level landscape (k cells at c1, scattered over both axes) gives log(k e^{c1/tau} + (N - k) e^{c2/tau});
    no overflow at X / tau = 1000; Jensen / Hoeffding bounds log N + mean / tau <= L <= that + (max - min)^2 / 8 tau^2;
    and the tau -> 0 limit tau L -> max X within tau log N."""
    rng = np.random.default_rng(5)
    shape = (3, 2, 49, 64)
    N = 49 * 64
    c = rng.normal(size=(3, 2))
    X = np.broadcast_to(c[:, :, None, None], shape).copy()
    for tau in (0.01, 0.3, 7.0):
        L = ftk.log_marginal(X, tau)
        assert L.shape == (3, 2)
        assert np.allclose(L, c / tau + math.log(N), rtol=0, atol=1e-12 * (1 + np.abs(c).max() / tau))
    X2 = np.full((49, 64), -0.4)
    cells = rng.choice(N, size=37, replace=False)
    X2.reshape(-1)[cells] = 0.9
    for tau in (0.05, 1.0):
        want = math.log(37 * math.exp(0.9 / tau) + (N - 37) * math.exp(-0.4 / tau))
        assert abs(ftk.log_marginal(X2, tau) - want) < 1e-12 * abs(want)
    assert abs(ftk.log_marginal(np.full((7, 8), 1000.0), 1.0) - (1000.0 + math.log(56))) < 1e-9
    Xr = rng.normal(size=(49, 64))
    for tau in (0.5, 3.0, 40.0):
        L = ftk.log_marginal(Xr, tau)
        lo = math.log(N) + Xr.mean() / tau
        assert lo - 1e-12 <= L <= lo + (Xr.max() - Xr.min()) ** 2 / (8 * tau * tau) + 1e-12
    for tau in (1e-2, 1e-3):
        assert Xr.max() <= tau * ftk.log_marginal(Xr, tau) <= Xr.max() + tau * math.log(N) + 1e-12
    # complex input: the real part is used (Re X)
    assert abs(ftk.log_marginal(X2 + 1j, 1.0) - ftk.log_marginal(X2, 1.0)) < 1e-14


def test_log_marginal_through_ftk(tiny):
    """Through the FTK landscapes: a zero image gives log(N_t n_psi) exactly; rotating the template by a
    grid angle leaves L unchanged (X'(t, r) = X(t, r - j) permutes the grid); and L of the FTK landscape
    is within max |X_FTK - X_exact| / tau of L of the exact Gaussian landscape (closed form, Eq. planch
    P:207-212; log-sum-exp is 1-Lipschitz in the sup norm)."""
    cfg, plan, imgs, tpls, pi, pt = tiny
    b = fb.fb_coeffs(tpls[:2])
    X0 = ftk.ftk_landscapes(np.zeros_like(fb.fb_coeffs(imgs[:1])), b, plan)
    assert np.allclose(ftk.log_marginal(X0, 0.1), math.log(len(plan.shifts) * cfg.n_psi), rtol=0, atol=1e-12)
    a = fb.fb_coeffs(imgs[:1])
    b_rot = fb.fb_coeffs(np.roll(tpls[:1], 9, axis=-1))
    L1 = ftk.log_marginal(ftk.ftk_landscapes(a, b[:1], plan), 0.05)
    L2 = ftk.log_marginal(ftk.ftk_landscapes(a, b_rot, plan), 0.05)
    assert abs(L1 - L2) < 1e-10 * abs(L1)
    i, j = 1, 3
    X = np.real(ftk.ftk_landscapes(fb.fb_coeffs(imgs[i:i + 1]), fb.fb_coeffs(tpls[j:j + 1]), plan))[0, 0]
    Xc = np.array([[closed_form.gaussian_ip(pi, pt, i, j, plan.shifts[t], 2 * math.pi * r / cfg.n_psi)
                    for r in range(cfg.n_psi)] for t in range(len(plan.shifts))])
    dmax = np.max(np.abs(X - Xc))
    na, nb = fb.discrete_norm(imgs, plan.w), fb.discrete_norm(tpls, plan.w)
    assert dmax < 3e-3 * na[i] * nb[j]
    for tau in (0.02, 0.2, 2.0):
        tau_abs = tau * na[i] * nb[j]
        assert abs(ftk.log_marginal(X, tau_abs) - ftk.log_marginal(Xc, tau_abs)) <= dmax / tau_abs + 1e-12
