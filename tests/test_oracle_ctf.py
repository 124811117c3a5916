"""Pins for oracle.ctf, the CTF-parameterized factorized kernel (Sec. 6
P:1389-1403; DESIGN reading R24).  No GPU.

The brute-force CTF landscape is pinned to (a) the exact Gaussian inner products (a Gaussian filter
maps a Gaussian-blob template to wider blobs), (b) the self-adjointness of a real radial filter
(moving it from the template to the image), (c) c = 1 giving the plain brute force.  The joint
(delta, tau) factorization is pinned by the Cauchy-Schwarz bound |X^FTK - X^bf| <= max|cF - F^SVD|
||A|| ||B|| with the certificate taken from F's definition, by the singular-value invariants of the
construction (c = 1 reproduces the plain operator spectrum; identical filters scale Sigma by sqrt(n_tau);
c -> alpha c scales Sigma by |alpha|), and by eps -> 0 convergence.
"""
import math

import numpy as np
import pytest

from oracle import brute, closed_form, ctf, fb, ftk, kernel_svd as ks
import synth

DEFOCI = [8000.0, 15000.0, 22000.0, 30000.0]


@pytest.fixture(scope="module")
def tiny():
    cfg = synth.config("tiny")
    base = ks.build_plan(cfg.n, cfg.K, synth.delta_max(cfg), synth.shift_list(cfg), cfg.eps, cfg.n_k, cfg.n_psi)
    f = synth.ctf_filters(base.k, DEFOCI)
    plan = ctf.build_plan_ctf(cfg.n, cfg.K, synth.delta_max(cfg), synth.shift_list(cfg), cfg.eps, cfg.n_k,
                              cfg.n_psi, f)
    imgs, pi = synth.draw_items(cfg, "images", range(3), plan.k, "planted")
    tpls, pt = synth.draw_items(cfg, "templates", range(3), plan.k)
    return cfg, base, plan, f, imgs, tpls, pi, pt


def test_ctf_filters_are_the_weak_phase_model(tiny):
    """Input generator sanity: c(0) = -A (amplitude contrast), |c| <= 1, zero crossings move inward with
    defocus (chi grows with dF)."""
    cfg, base, plan, f, *_ = tiny
    c0 = synth.ctf_filters(np.array([0.0]), DEFOCI)
    assert np.allclose(c0, -0.07, atol=1e-15)
    assert np.all(np.abs(f) <= 1.0 + 1e-15)
    k = np.linspace(1e-3, base.k_max, 4000)
    first_zero = [k[np.argmax(np.diff(np.sign(c)) != 0)] for c in synth.ctf_filters(k, DEFOCI)]
    assert all(a > b for a, b in zip(first_zero, first_zero[1:]))


def test_brute_ctf_unit_filter_is_plain_brute_force(tiny):
    cfg, base, plan, f, imgs, tpls, *_ = tiny
    Xc = ctf.brute_landscape_ctf(imgs[0], tpls[1], base.k, base.w, base.shifts, np.ones((1, cfg.n_k)))
    Xb = brute.brute_landscape(imgs[0], tpls[1], base.k, base.w, base.shifts)
    assert np.max(np.abs(Xc[0] - Xb)) <= 1e-13 * np.max(np.abs(Xb))


def test_brute_ctf_filter_is_self_adjoint(tiny):
    """<R T A, c B> = <R T (c A), B> for a real radial c (c commutes with R and with the phase F)."""
    cfg, base, plan, f, imgs, tpls, *_ = tiny
    Xc = ctf.brute_landscape_ctf(imgs[1], tpls[2], base.k, base.w, base.shifts, f)
    for tau in range(len(DEFOCI)):
        Xm = brute.brute_landscape(f[tau][:, None] * imgs[1], tpls[2], base.k, base.w, base.shifts)
        assert np.max(np.abs(Xc[tau] - Xm)) <= 1e-13 * np.max(np.abs(Xm))


@pytest.mark.parametrize("beta", [0.7, 1.5])
def test_brute_ctf_gaussian_filter_closed_form(beta):
    """Filter c(k) = exp(-beta^2 k^2 / 2) turns each template blob (sigma, amp) into (sqrt(sigma^2 +
    beta^2), amp sigma^2 / (sigma^2 + beta^2)) (Gaussian Fourier transform), so the filtered landscape is
    the closed-form Gaussian inner product with the widened template (c3: quadrature-exact)."""
    cfg = synth.config("c3")
    sh = synth.shift_list(cfg)[:3]
    plan = ks.build_plan(cfg.n, cfg.K, synth.delta_max(cfg), sh, cfg.eps, cfg.n_k, cfg.n_psi)
    x, px = synth.draw_items(cfg, "images", [0], plan.k, noise=False)
    y, py = synth.draw_items(cfg, "templates", [0], plan.k, noise=False)
    c = np.exp(-0.5 * beta ** 2 * plan.k ** 2)[None, :]
    pw = dict(py)
    s2 = py["sigma"] ** 2 + beta ** 2
    pw["sigma"] = np.sqrt(s2)
    pw["amp"] = py["amp"] * py["sigma"] ** 2 / s2
    Xc = ctf.brute_landscape_ctf(x[0], y[0], plan.k, plan.w, sh, c)[0]
    for t, r in [(0, 0), (1, 7), (2, 100)]:
        cf = closed_form.gaussian_ip(px, pw, 0, 0, sh[t], 2 * math.pi * r / cfg.n_psi)
        assert abs(Xc[t, r] - cf) < 1e-6 * (2 * math.pi) ** 2


def test_ctf_plan_unit_filter_reproduces_plain_spectrum(tiny):
    """c = 1, n_tau = 1: the discrete-k operator has the plain operator's singular values (Eq. Jsvd)."""
    cfg, base, *_ = tiny
    p1 = ctf.build_plan_ctf(cfg.n, cfg.K, base.delta_max, base.shifts, cfg.eps, cfg.n_k, cfg.n_psi,
                            np.ones((1, cfg.n_k)))
    assert p1.H == base.H
    for ell, S in base.all_sigma.items():
        if ell in p1.all_sigma:
            m = S > cfg.eps
            assert np.allclose(p1.all_sigma[ell][:m.sum()], S[m], rtol=1e-9, atol=1e-12)


def test_ctf_plan_sigma_invariants(tiny):
    cfg, base, plan, f, *_ = tiny
    one = f[1:2]
    p1 = ctf.build_plan_ctf(cfg.n, cfg.K, base.delta_max, base.shifts, 1e-6, cfg.n_k, cfg.n_psi, one)
    p3 = ctf.build_plan_ctf(cfg.n, cfg.K, base.delta_max, base.shifts, 1e-6, cfg.n_k, cfg.n_psi,
                            np.repeat(one, 3, axis=0))
    pa = ctf.build_plan_ctf(cfg.n, cfg.K, base.delta_max, base.shifts, 1e-6, cfg.n_k, cfg.n_psi, -0.5 * one)
    for ell in (0, 1, 4):
        s1 = p1.all_sigma[ell][:6]
        assert np.allclose(p3.all_sigma[ell][:6], math.sqrt(3.0) * s1, rtol=1e-10)
        assert np.allclose(pa.all_sigma[ell][:6], 0.5 * s1, rtol=1e-10)
    # the joint factorization never needs more terms than the filters separately
    sep = sum(ctf.build_plan_ctf(cfg.n, cfg.K, base.delta_max, base.shifts, cfg.eps, cfg.n_k, cfg.n_psi,
                                 f[t:t + 1]).H for t in range(len(DEFOCI)))
    assert plan.H <= sep


def test_ctf_ftk_vs_brute_force_bound(tiny):
    """|X^FTK - X^bf| <= max_{tau,t,m,p} |c F - F^SVD| ||A|| ||B|| (Cauchy-Schwarz in the discrete
    norm), certificate from F's definition; and the north-star gate 4 eps ||A|| ||B|| (reading R16)."""
    cfg, base, plan, f, imgs, tpls, *_ = tiny
    cert = ctf.kernel_certificate_ctf(plan, f)
    assert cert < 20 * cfg.eps
    X = ftk.ftk_landscapes(fb.fb_coeffs(imgs), fb.fb_coeffs(tpls), plan)
    na, nb = fb.discrete_norm(imgs, plan.w), fb.discrete_norm(tpls, plan.w)
    N_t = base.shifts.shape[0]
    for i in range(3):
        for j in range(3):
            Xb = ctf.brute_landscape_ctf(imgs[i], tpls[j], plan.k, plan.w, base.shifts, f).reshape(-1, cfg.n_psi)
            err = np.max(np.abs(X[i, j] - Xb))
            assert err <= cert * na[i] * nb[j] * (1 + 1e-9)
            assert err <= 4 * cfg.eps * na[i] * nb[j]
    assert X.shape[2] == len(DEFOCI) * N_t
    assert np.max(np.abs(X.imag)) < 1e-12 * np.max(np.abs(X.real))


def test_ctf_ftk_tends_to_brute_force(tiny):
    cfg, base, plan, f, imgs, tpls, *_ = tiny
    p = ctf.build_plan_ctf(cfg.n, cfg.K, base.delta_max, base.shifts, 1e-9, cfg.n_k, cfg.n_psi, f[:2])
    X = ftk.ftk_landscapes(fb.fb_coeffs(imgs[:1]), fb.fb_coeffs(tpls[:1]), p)[0, 0]
    Xb = ctf.brute_landscape_ctf(imgs[0], tpls[0], p.k, p.w, base.shifts, f[:2]).reshape(-1, cfg.n_psi)
    assert np.max(np.abs(X - Xb)) < 1e-7 * np.max(np.abs(Xb))
