"""FTK Steps 1-3, written as PAPER.md Eq. (fbk3) reads (TEST INFRASTRUCTURE ONLY).

Eq. (fbk3), for every retained term zeta = (ell, eta) (both signs of ell):
  Step 1  Zhat_zeta(q) = 2 pi sum_m w_m conj(b(k_m; q)) a(k_m; q - ell) G_zeta(k_m)
  Step 2  Z_zeta(gamma) = sum_q exp(-i q gamma) Zhat_zeta(q)
  Step 3  X(delta, gamma) = sum_zeta Y_zeta(delta) Z_zeta(gamma)
with q cyclic mod n_psi (reading R5), gamma_r = 2 pi r / n_psi (reading R3/R4), so
Step 2 is numpy's forward DFT over q (exp(-2 pi i q r / n_psi)).  X is complex; its
imaginary part is kept as a diagnostic (it vanishes for real images).

More rotations than angular samples (n_gamma > n_psi; "by zero-padding and using a larger
FFT in the second step"): Step 2 is evaluated at gamma_r = 2 pi r / n_gamma as the trigonometric
sum over the signed frequencies q in [-n_psi/2, n_psi/2] with the Nyquist coefficient split equally
between -n_psi/2 and +n_psi/2 (reading R21: the paper's sum over q = -Q..Q counts the aliased
Nyquist index twice; the symmetric split keeps X real for real images and reproduces the n_psi-grid
values exactly).
"""
from __future__ import annotations

import math

import numpy as np

from .kernel_svd import OraclePlan


def step2_rotations(Zhat, n_gamma=None):
    """Step 2 (Eq. 1dfft): Z(gamma_r) = sum_q exp(-i q gamma_r) Zhat(q),
    gamma_r = 2 pi r / n_gamma.  Zhat [..., n_psi] over cyclic q; n_gamma = n_psi is numpy's FFT,
    n_gamma > n_psi the direct sum over signed q with the Nyquist term split (reading R21)."""
    n_psi = Zhat.shape[-1]
    if n_gamma is None or n_gamma == n_psi:
        return np.fft.fft(Zhat, axis=-1)
    Q = n_psi // 2
    q = np.arange(n_psi)
    qs = np.where(q < Q, q, q - n_psi).astype(np.float64)        # signed frequency of cyclic index q
    gam = 2.0 * math.pi * np.arange(n_gamma) / n_gamma
    E = np.exp(-1j * qs[:, None] * gam[None, :])                  # [q, r]
    E[Q, :] = np.cos(Q * gam)                                     # Nyquist: (e^{-iQg} + e^{iQg}) / 2
    return np.einsum("...q,qr->...r", Zhat, E)


def ftk_landscapes(a, b, plan: OraclePlan, n_gamma=None):
    """a: FB coeffs of images [I, n_k, n_psi]; b: templates [J, n_k, n_psi] (complex).
    Returns X [I, J, N_t, n_gamma] complex128 (n_gamma defaults to n_psi).  The two contractions are
    plain matrix products per pair (np.matmul, a library primitive), summed over m and zeta exactly as
    Eq. fbk3 states."""
    a = np.asarray(a, dtype=np.complex128)
    b = np.asarray(b, dtype=np.complex128)
    I, J = a.shape[0], b.shape[0]
    n_psi = a.shape[-1]
    H = plan.H
    Zhat = np.empty((I, J, H, n_psi), dtype=np.complex128)
    bc = np.conj(b)
    ells = sorted({t.ell for t in plan.terms})
    for ell in ells:
        zs = [z for z, t in enumerate(plan.terms) if t.ell == ell]
        a_shift = np.roll(a, ell, axis=-1)                      # a_shift[..., q] = a[..., (q - ell) mod n]
        P = a_shift[:, None, :, :] * bc[None, :, :, :]          # [I, J, m, q]
        Gw = 2.0 * math.pi * plan.w[None, :] * plan.G[zs]       # [h, m]
        Zhat[:, :, zs, :] = np.matmul(Gw, P)                    # Step 1: sum_m Gw[h, m] P[i, j, m, q]
    Z = step2_rotations(Zhat, n_gamma)                          # Step 2
    return np.matmul(plan.Y, Z)                                 # Step 3: sum_h Y[t, h] Z[i, j, h, r]


def best_per_image(X):
    """Per image: max over (j, t, r) of Re X; ties -> smallest (j, t, r) (reading R9).
    X [I, J, N_t, n_psi] (complex or real).  Returns (value, j, t, r, gap) arrays, gap = top-2 margin."""
    R = np.real(X)
    I = R.shape[0]
    flat = R.reshape(I, -1)
    idx = np.argmax(flat, axis=1)
    val = flat[np.arange(I), idx]
    j, t, r = np.unravel_index(idx, R.shape[1:])
    srt = np.sort(flat, axis=1)
    gap = srt[:, -1] - srt[:, -2] if flat.shape[1] > 1 else np.full(I, np.inf)
    return val, j, t, r, gap


def ftk_best(a, b, plan: OraclePlan, chunk_i: int = 4, chunk_j: int = 16, n_gamma=None):
    """Per-image bests over all templates, blocked over pairs (same arithmetic as ftk_landscapes)."""
    I, J = a.shape[0], b.shape[0]
    best_v = np.full(I, -np.inf)
    best_idx = np.zeros((I, 3), dtype=np.int64)
    for i0 in range(0, I, chunk_i):
        for j0 in range(0, J, chunk_j):
            X = np.real(ftk_landscapes(a[i0:i0 + chunk_i], b[j0:j0 + chunk_j], plan, n_gamma))
            v, j, t, r, _ = best_per_image(X)
            for ii in range(v.size):
                if v[ii] > best_v[i0 + ii]:     # strict: earlier j wins ties
                    best_v[i0 + ii] = v[ii]
                    best_idx[i0 + ii] = (j[ii] + j0, t[ii], r[ii])
    return best_v, best_idx


def log_marginal(X, tau):
    """Marginalization over the alignment grid ("sampling this
    entire landscape is necessary in a Bayesian framework, where an integral of a probability
    distribution over shifts and angles is used to marginalize the likelihood").  Uniform weights on
    the shift list and the rotation grid (reading R22):
        L = log sum_{t, r} exp(Re X(delta_t, gamma_r) / tau)        per (image, template) pair.
    X [..., N_t, n_gamma] (complex or real); tau > 0.  Evaluated as the textbook log-sum-exp
    m + log sum exp(X / tau - m) with m the maximum of X / tau (no overflow)."""
    if not tau > 0:
        raise ValueError("tau must be positive")
    R = np.real(np.asarray(X, dtype=np.complex128 if np.iscomplexobj(X) else np.float64)) / tau
    m = R.max(axis=(-2, -1), keepdims=True)
    s = np.exp(R - m).sum(axis=(-2, -1), keepdims=True)
    return (m + np.log(s))[..., 0, 0]
