"""Direct brute-force evaluation of the bandlimited inner product (TEST INFRASTRUCTURE ONLY).

Eq. (Xdg) P:293-298 (second form, with the conjugate on Bhat restored; reading R10):
  X(delta, gamma) = int_{Omega_K} F(delta, k) Ahat(k) conj(R_{-gamma} Bhat(k)) dk,
F(delta, k) = exp(-i delta.k) (Eq. Fdk), R_gamma Ahat(k, psi) = Ahat(k, psi - gamma)
(P:255-263).  Discretized with the radial rule and the periodic trapezoid rule in psi:
  X^bf(t, r) = (2 pi / n_psi) sum_m w_m sum_p F(delta_t; k_m, psi_p) Ahat(m, p) conj Bhat(m, (p + r) mod n_psi).
No Bessel function, no SVD, no FFT: the plain definition written out.
"""
from __future__ import annotations

import math

import numpy as np


def _phase(delta_xy, k, n_psi):
    psi = 2.0 * math.pi * np.arange(n_psi) / n_psi
    d = np.asarray(delta_xy, dtype=np.float64).reshape(-1, 2)
    proj = d[:, 0, None] * np.cos(psi)[None, :] + d[:, 1, None] * np.sin(psi)[None, :]   # [T, P]
    return np.exp(-1j * np.asarray(k)[None, :, None] * proj[:, None, :])                   # [T, M, P]


def brute_landscape(A, B, k, w, shifts):
    """Full landscape X^bf [N_t, n_psi] (complex) for one (image A, template B) polar-sample pair."""
    A = np.asarray(A, dtype=np.complex128)
    B = np.asarray(B, dtype=np.complex128)
    n_psi = A.shape[-1]
    FA = _phase(shifts, k, n_psi) * A[None]                                 # [T, M, P]
    Brot = np.stack([np.roll(B, -r, axis=-1) for r in range(n_psi)])        # Brot[r, m, p] = B[m, (p + r) mod n]
    return (2.0 * math.pi / n_psi) * np.einsum("m,tmp,rmp->tr", np.asarray(w), FA, np.conj(Brot))


def brute_points(A, B, k, w, shifts, t_idx, r_idx):
    """X^bf at selected (t, r) points (same definition, for large configs)."""
    A = np.asarray(A, dtype=np.complex128)
    B = np.asarray(B, dtype=np.complex128)
    n_psi = A.shape[-1]
    out = np.empty(len(t_idx), dtype=np.complex128)
    for n, (t, r) in enumerate(zip(t_idx, r_idx)):
        FA = _phase(np.asarray(shifts)[t], k, n_psi)[0] * A
        out[n] = (2.0 * math.pi / n_psi) * np.einsum("m,mp,mp->", np.asarray(w), FA, np.conj(np.roll(B, -int(r), axis=-1)))
    return out
