"""Pins for oracle.pixels (Eq. Ahattrap; reading R23), no GPU.

The trapezoid sum is pinned to the exact Fourier transform of a Gaussian (closed form, well sampled and
far from the border, so aliasing and truncation are below 1e-8), to the DC sum, to the shift theorem,
to Hermitian symmetry, and to the analytic polar samples the rest of the oracle uses (same blobs)."""
import math

import numpy as np

import synth
from oracle import pixels


def _blob_image(n, cx, cy, sig):
    x = np.arange(n) - n / 2.0
    return np.exp(-((x[:, None] - cx) ** 2 + (x[None, :] - cy) ** 2) / (2 * sig * sig))


def test_gaussian_closed_form():
    n, cx, cy, sig = 32, 1.3, -0.7, 2.0
    A = _blob_image(n, cx, cy, sig)
    rng = np.random.default_rng(0)
    kk = rng.uniform(0, math.pi, 200)
    th = rng.uniform(0, 2 * math.pi, 200)
    kx, ky = kk * np.cos(th), kk * np.sin(th)
    got = pixels.ft_points(A, kx, ky)
    want = 2 * math.pi * sig ** 2 * np.exp(-sig ** 2 * kk ** 2 / 2) * np.exp(-1j * (kx * cx + ky * cy))
    assert np.max(np.abs(got - want)) < 1e-8 * 2 * math.pi * sig ** 2


def test_dc_shift_and_hermitian():
    rng = np.random.default_rng(1)
    n = 16
    A = np.zeros((n, n))
    A[2:-2, 2:-2] = rng.standard_normal((n - 4, n - 4))
    assert abs(pixels.ft_points(A, [0.0], [0.0])[0] - A.sum()) < 1e-12 * np.abs(A).sum()
    kx, ky = rng.uniform(-math.pi, math.pi, 50), rng.uniform(-math.pi, math.pi, 50)
    F = pixels.ft_points(A, kx, ky)
    Fx = pixels.ft_points(np.roll(A, 1, axis=0), kx, ky)       # shift by +1 px in x (index i)
    Fy = pixels.ft_points(np.roll(A, -1, axis=1), kx, ky)      # shift by -1 px in y (index j)
    assert np.max(np.abs(Fx - np.exp(-1j * kx) * F)) < 1e-12 * np.abs(A).sum()
    assert np.max(np.abs(Fy - np.exp(1j * ky) * F)) < 1e-12 * np.abs(A).sum()
    assert np.max(np.abs(pixels.ft_points(A, -kx, -ky) - np.conj(F))) < 1e-12 * np.abs(A).sum()


def test_polar_layout_and_analytic_samples():
    """polar_from_pixels is [n_k][n_psi] with psi_p = 2 pi p / n_psi; for noiseless blob items it agrees
    with the analytic polar samples of the same blobs (synth.polar_samples, P:196-200 convention) to the
    aliasing level of sigma >= 1.5 px blobs at the Nyquist ring (exp(-sigma^2 pi^2 / 2) ~ 1.5e-5)."""
    cfg = synth.config("c2")
    k = np.linspace(0.05, cfg.k_max, 9)
    pix, par = synth.draw_pixel_items(cfg, "templates", [0, 3], noise=False)
    P = pixels.polar_from_pixels(pix, k, cfg.n_psi)
    assert P.shape == (2, 9, cfg.n_psi)
    m, p = 4, 37
    psi = 2 * math.pi * p / cfg.n_psi
    one = pixels.ft_points(pix[1].astype(np.float64), [k[m] * math.cos(psi)], [k[m] * math.sin(psi)])[0]
    assert abs(P[1, m, p] - one) < 1e-12 * np.abs(P[1]).max()
    ana = synth.polar_samples(par, k, cfg.n_psi).astype(np.complex128)
    scale = np.abs(ana).max()
    assert np.max(np.abs(P - ana)) < 5e-5 * scale       # float32 pixels + aliasing
    assert np.max(np.abs(P[:, :4] - ana[:, :4])) < 2e-6 * scale   # low rings: float32 rounding only
