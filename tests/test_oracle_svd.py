"""Pins for oracle.kernel_svd and oracle.bounds (no GPU).

What pins the plan: the paper's printed ranks (golden fixture), the energy identity
sum Sigma^2 = pi^2 W^2 (from sum_l J_l^2 = 1), Sigma depending only on D K
checked with an SVD in unscaled variables, agreement of two independent discretizations,
pointwise reconstruction against mpmath Bessel values, orthonormality under an independent
quadrature, Lemma 2 / Theorem 1 bounds, and the Hilbert-Schmidt tail identity (Eq. efrob).
"""
import json
import math
import os

import mpmath
import numpy as np
import pytest

from oracle import bounds, kernel_svd as ks, quadrature

GOLD = os.path.dirname(__file__) + "/golden/"


@pytest.fixture(scope="module")
def spectra_w1():
    return ks.modal_spectra(1.0, 1e-2, "nystrom", 128)


def _H(spec, eps):
    return {l: int((m.sigma > eps).sum()) for l, m in spec.items()}


def test_paper_worked_example_ranks(spectra_w1):
    g = json.load(open(GOLD + "paper_rank_W1_eps1e-2.json"))
    Hl = _H(spectra_w1, g["eps"])
    assert Hl[0] == g["H_0"] and Hl[3] == g["H_3"]
    H = Hl[0] + 2 * sum(v for l, v in Hl.items() if l > 0)
    assert abs(H - g["H"]) <= g["H_tolerance"]


@pytest.mark.parametrize("W", [0.5, 1.0, 2.0])
def test_energy_identity(W):
    """sum_l sum_eta Sigma_eta(l)^2 = ||J_l(xy)||_HS^2 summed over l = (2 pi W)^2/4 = pi^2 W^2."""
    spec = ks.modal_spectra(W, 1e-2, "nystrom", 128)
    e = sum((m.sigma ** 2).sum() * (1 if l == 0 else 2) for l, m in spec.items())
    assert abs(e / (math.pi ** 2 * W ** 2) - 1) < 1e-10


@pytest.mark.parametrize("W", [1.0, 2.0])
def test_two_discretizations_agree(W):
    nys = ks.modal_spectra(W, 1e-3, "nystrom", 128)
    jac = ks.modal_spectra(W, 1e-3, "jacobi", 128)
    for l in nys:
        s1, s2 = nys[l].sigma[:12], jac[l].sigma[:12]
        assert np.max(np.abs(s1 - s2)) < 1e-10


def test_sigma_depends_only_on_DK():
    """SVD of J_l(delta k) on [0,D]x[0,K] (weights delta d delta, k dk) in UNSCALED variables."""
    def svals(D, K, ell, n=96):
        d, wd = quadrature.gauss_jacobi_01(n, D)
        k, wk = quadrature.gauss_jacobi_01(n, K)
        from scipy.special import jv
        M = np.sqrt(wd)[:, None] * jv(ell, d[:, None] * k[None, :]) * np.sqrt(wk)[None, :]
        return np.linalg.svd(M, compute_uv=False)[:10]
    for ell in (0, 3, 7):
        a, b = svals(2.0, math.pi, ell), svals(1.0, 2 * math.pi, ell)
        c = ks.modal_svd_nystrom(ell, 2 * math.pi, 96).sigma[:10]
        assert np.max(np.abs(a - b)) < 1e-12 and np.max(np.abs(a - c)) < 1e-12


@pytest.mark.parametrize("method", ["nystrom", "jacobi"])
def test_pointwise_reconstruction_vs_mpmath(method):
    W = 1.5
    a = 2 * math.pi * W
    rng = np.random.default_rng(1)
    for ell in (0, 2, 9):
        ms = ks.modal_svd_nystrom(ell, a, 128) if method == "nystrom" else ks.modal_svd_jacobi(ell, a, 48, 128)
        nt = int((ms.sigma > 1e-13).sum())
        for x, y in zip(rng.uniform(0, a, 6), rng.uniform(0, 1, 6)):
            approx = sum(ms.u(np.array([x]), e)[0] * ms.sigma[e] * ms.v(np.array([y]), e)[0] for e in range(nt))
            assert abs(approx - float(mpmath.besselj(ell, x * y))) < 1e-11


def test_orthonormality_independent_quadrature():
    """u orthonormal under x dx on [0,2 pi W], v under y dy on [0,1], Gauss-Legendre check."""
    W = 2.0
    a = 2 * math.pi * W
    ms = ks.modal_svd_nystrom(4, a, 128)
    x, wx = quadrature.gauss_legendre_k(80, a)
    y, wy = quadrature.gauss_legendre_k(80, 1.0)
    U = np.stack([ms.u(x, e) for e in range(5)])
    V = np.stack([ms.v(y, e) for e in range(5)])
    assert np.max(np.abs((U * wx) @ U.T - np.eye(5))) < 1e-10
    assert np.max(np.abs((V * wy) @ V.T - np.eye(5))) < 1e-10


@pytest.mark.parametrize("W", [1.0, 2.0, 3.0])
@pytest.mark.parametrize("eps", [1e-2, 1e-3, 1e-4])
def test_lemma2_theorem1_and_fit(W, eps):
    spec = ks.modal_spectra(W, eps, "nystrom", 128)
    Hl = _H(spec, eps)
    for l, h in Hl.items():
        assert h <= bounds.lemma2(l, W, eps)                       # Lemma 2
        fit = bounds.empirical_fit(l, W, eps)                      # P:1144, an approximate fit:
        if fit > 1:                                                # tolerance 3 terms (reading R19)
            assert abs(h - fit) <= 3.0
    H = Hl[0] + 2 * sum(v for l, v in Hl.items() if l > 0)
    assert H <= bounds.theorem1_total(W, eps)                      # Theorem 1
    assert all(Hl[l] >= Hl[l + 1] for l in range(len(Hl) - 1))    # triangular support (Fig. 3 caption)


def test_spec_bound_values():
    g = json.load(open(GOLD + "spec_examples.json"))
    assert math.ceil(bounds.lemma2(0, 1.0, 1e-2)) == g["lemma2_ell0_W1_eps1e-2_ceil"]
    assert 2 * math.ceil(bounds.theorem1_calH(1.0, 1e-2)) ** 2 == g["theorem1_W1_eps1e-2_ceil_form"]


def test_rank_grows_with_W_and_digits():
    """H grows with W at fixed eps and with log(1/eps) at fixed W."""
    Hs = []
    for W in (0.5, 1.0, 1.5, 2.0):
        spec = ks.modal_spectra(W, 1e-2, "nystrom", 96)
        h = _H(spec, 1e-2)
        Hs.append(h[0] + 2 * sum(v for l, v in h.items() if l > 0))
    assert all(b > a for a, b in zip(Hs, Hs[1:]))
    spec = ks.modal_spectra(1.0, 1e-4, "nystrom", 96)
    Hd = [(lambda h: h[0] + 2 * sum(v for l, v in h.items() if l > 0))(_H(spec, e)) for e in (1e-2, 1e-3, 1e-4)]
    assert Hd[0] < Hd[1] < Hd[2]


def test_kernel_factorization_hs_tail_and_pointwise():
    """Assembled F^SVD (incl. Y/G phases and the +-ell mirror):
    (1/(2 pi)^2) int_{Omega_D} int_{Omega_K} |F - F^SVD|^2 = sum_{zeta > H} Sigma_zeta^2  (Eq. efrob; reading R18
    for the (2 pi)^2 from the two angular integrals), and the pointwise error is O(eps)."""
    W, eps, kmax = 1.0, 1e-2, math.pi
    D = 2 * math.pi * W / kmax
    plan = ks.build_plan(64, 32, D, [[0.0, 0.0]], eps, 32, 128)
    nd, na = 40, 80
    dr, dw = quadrature.gauss_legendre_k(nd, D)
    kr, kw = quadrature.gauss_legendre_k(nd, kmax)
    ang = 2 * math.pi * np.arange(na) / na
    tot = 0.0
    worst = 0.0
    for i in range(nd):
        dxy = np.stack([dr[i] * np.cos(ang), dr[i] * np.sin(ang)], 1)
        Fs = ks.f_svd(plan, dxy, kr, ang)
        F = np.exp(-1j * kr[None, :, None] * (dxy[:, 0, None, None] * np.cos(ang)[None, None, :]
                                               + dxy[:, 1, None, None] * np.sin(ang)[None, None, :]))
        e = np.abs(F - Fs) ** 2
        worst = max(worst, float(np.sqrt(e.max())))
        tot += dw[i] * (2 * math.pi / na) ** 2 * np.einsum("k,ikp->", kw, e)
    tail = sum((s[s <= eps] ** 2).sum() * (1 if l == 0 else 2) for l, s in plan.all_sigma.items())
    assert abs(tot / (2 * math.pi) ** 2 / tail - 1) < 1e-6
    assert worst < 12 * eps


def test_fsvd_converges_to_F_for_tiny_eps():
    plan = ks.build_plan(32, 16, 1.0, [[0.3, -0.7], [1.0, 0.0]], 1e-10, 16, 64)
    psi = np.linspace(0, 2 * math.pi, 17)
    k = np.linspace(0, math.pi, 9)
    Fs = ks.f_svd(plan, plan.shifts, k, psi)
    F = np.exp(-1j * k[None, :, None] * (plan.shifts[:, 0, None, None] * np.cos(psi) + plan.shifts[:, 1, None, None] * np.sin(psi)))
    assert np.max(np.abs(F - Fs)) < 1e-8
