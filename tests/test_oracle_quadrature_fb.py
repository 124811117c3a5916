"""Pins for oracle.quadrature and oracle.fb against closed forms (no GPU)."""
import json
import math
import os

import mpmath
import numpy as np
import pytest

from oracle import fb, quadrature
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")


@pytest.mark.parametrize("rule,exact_deg", [("gl", lambda n: 2 * n - 2), ("gj", lambda n: 2 * n - 1)])
@pytest.mark.parametrize("n_k,K", [(1, 1.0), (8, 1.0), (16, math.pi), (64, math.pi)])
def test_radial_rule_exactness(rule, exact_deg, n_k, K):
    """int_0^K k^j k dk = K^(j+2)/(j+2) exactly up to the rule's degree."""
    k, w = quadrature.radial_rule(n_k, K, rule)
    assert np.all(np.diff(k) > 0) and np.all((k > 0) & (k < K)) and np.all(w > 0)
    assert abs(w.sum() - K * K / 2) < 1e-13 * K * K
    for j in range(0, max(exact_deg(n_k), 0) + 1):
        exact = K ** (j + 2) / (j + 2)
        assert abs((w * k ** j).sum() - exact) <= 1e-12 * exact


def test_spec_gauss_jacobi_examples():
    g = json.load(open(GOLD))
    k, w = quadrature.gauss_jacobi_01(1, 1.0)
    assert abs(k[0] - g["gj_1_on_unit"]["node"]) < 1e-15 and abs(w[0] - g["gj_1_on_unit"]["weight"]) < 1e-15
    k, w = quadrature.gauss_jacobi_01(8, 1.0)
    assert abs((w * k ** 9).sum() - g["gj_8_moment_k9"]) < 1e-14


def test_scipy_bessel_against_mpmath():
    """The oracle's J_ell (scipy library primitive) vs an independent arbitrary-precision evaluation."""
    from scipy.special import jv
    g = json.load(open(GOLD))
    assert abs(jv(0, g["J0_first_root"])) < 1e-12
    rng = np.random.default_rng(0)
    for ell in range(0, 30, 3):
        for z in rng.uniform(0, 4 * math.pi, 5):
            assert abs(jv(ell, z) - float(mpmath.besselj(ell, z))) < 1e-14
            assert abs(jv(-ell, z) - (-1) ** ell * jv(ell, z)) < 1e-15
    z = 7.3
    assert abs(sum(jv(l, z) ** 2 for l in range(-60, 61)) - 1.0) < 1e-13


def test_fb_coeffs_closed_form_single_blob():
    """Single isotropic blob at c: a(k;q) = alpha 2 pi s^2 e^{-s^2 k^2/2} J_q(k|c|) e^{-i q (theta_c + pi/2)}
    (Jacobi-Anger, applied to Eq. aqk)."""
    n_psi = 64
    k = np.array([0.3, 1.1, 2.0, 3.0])
    p = {"cx": np.array([[3.0]]), "cy": np.array([[-4.0]]), "sigma": np.array([[2.0]]), "amp": np.array([[0.7]])}
    s = synth.polar_samples(p, k, n_psi)[0].astype(np.complex128)
    a = fb.fb_coeffs(s)
    r, th = 5.0, math.atan2(-4.0, 3.0)
    for m, km in enumerate(k):
        for q in range(-20, 21):
            ref = 0.7 * 2 * math.pi * 4.0 * math.exp(-2.0 * km * km) * complex(mpmath.besselj(q, km * r)) \
                * complex(mpmath.exp(-1j * q * (th + math.pi / 2)))
            # complex64 input rounding ~6e-8 relative to the ring maximum
            assert abs(a[m, q % n_psi] - ref) < 2e-7 * 0.7 * 2 * math.pi * 4.0


def test_fb_reality_and_norm():
    """Real images: a(k;-q) = (-1)^q conj a(k;q); ||A|| is the discrete bandlimited norm."""
    cfg = synth.config("c2")
    k, w = quadrature.radial_rule(cfg.n_k, cfg.k_max)
    x, _ = synth.draw_items(cfg, "templates", [0, 1], k)
    a = fb.fb_coeffs(x)
    q = np.arange(cfg.n_psi)
    lhs = a[..., (-q) % cfg.n_psi]
    rhs = ((-1.0) ** q) * np.conj(a)
    assert np.max(np.abs(lhs - rhs)) < 1e-12 * np.max(np.abs(a))
    nrm = fb.discrete_norm(x, w)
    # unit L2 images + Plancherel: ||A||_disc ~ 2 pi * sqrt(1 + 1/SNR) in expectation
    assert np.all(np.abs(nrm / (2 * math.pi * math.sqrt(1 + 1 / cfg.snr)) - 1) < 0.05)
    # Parseval on each ring: (1/n) sum_p |Ahat|^2 = sum_q |a|^2
    assert np.allclose(np.mean(np.abs(x.astype(np.complex128)) ** 2, -1), np.sum(np.abs(a) ** 2, -1), rtol=1e-12)
