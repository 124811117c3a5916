"""Fourier-Bessel coefficients and the discrete bandlimited norm (TEST INFRASTRUCTURE ONLY).

Eq. (aqkcalc): on each ring,
    a(k_m; q) = (1/2Q) sum_p Ahat(k_m, psi_p) exp(-i q psi_p),  psi_p uniform,
with 2Q -> n_psi and psi_p = 2 pi p / n_psi (reading R3).  q is kept
cyclic, q in Z/n_psi (reading R5).  numpy's FFT is the library DFT step.
"""
from __future__ import annotations

import numpy as np


def fb_coeffs(samples):
    """samples [..., n_k, n_psi] (complex) -> a [..., n_k, n_psi] complex128, a[..., m, q]."""
    s = np.asarray(samples).astype(np.complex128)
    return np.fft.fft(s, axis=-1) / s.shape[-1]


def discrete_norm(samples, w):
    """||A|| := sqrt((2 pi / n_psi) sum_m w_m sum_p |Ahat(k_m, psi_p)|^2)  (= sqrt(X^bf_AA(0,0)))."""
    s = np.asarray(samples).astype(np.complex128)
    n_psi = s.shape[-1]
    return np.sqrt((2.0 * np.pi / n_psi) * np.einsum("m,...mp->...", np.asarray(w), np.abs(s) ** 2))
