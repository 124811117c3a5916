"""Pixel images -> Fourier samples by the trapezoid rule (TEST INFRASTRUCTURE ONLY).

PAPER.md Sec. "Conversion of discrete input images to the Fourier domain", Eq. (Ahattrap):
    Ahat(k) = (dx)^2 sum_{i,j} A_ij exp(-i k . x_ij),   x_ij = (i dx - 1, j dx - 1),  i, j in {0..n-1},
written in pixel units (dx = 1 px, the box [-1, 1]^2 -> [-n/2, n/2)^2; reading R23):
    Ahat(k) = sum_{i,j} A_ij exp(-i (k_x x_i + k_y y_j)),   x_i = i - n/2,  y_j = j - n/2,
evaluated directly (no NUFFT: the plain definition; the CUDA path uses a type-2 NUFFT).
The polar grid is (k_m, psi_p), psi_p = 2 pi p / n_psi (reading R3), k = k_m (cos psi_p, sin psi_p).
"""
from __future__ import annotations

import numpy as np


def ft_points(A, kx, ky):
    """Eq. (Ahattrap) at arbitrary frequencies.  A [n, n] real (i = x index, j = y index); kx, ky [P]
    (rad/px).  The phase separates, exp(-i(k_x x_i + k_y y_j)) = exp(-i k_x x_i) exp(-i k_y y_j), so
    Ahat(k_p) = sum_i exp(-i k_x x_i) sum_j A_ij exp(-i k_y y_j) (a matrix product per point)."""
    A = np.asarray(A, dtype=np.float64)
    n = A.shape[0]
    x = np.arange(n, dtype=np.float64) - n / 2.0
    kx = np.asarray(kx, dtype=np.float64)
    ky = np.asarray(ky, dtype=np.float64)
    ex = np.exp(-1j * kx[:, None] * x[None, :])     # [P, n] over i
    ey = np.exp(-1j * ky[:, None] * x[None, :])     # [P, n] over j
    inner = ey @ A.T                                 # [P, n]: sum_j A_ij exp(-i k_y y_j), indexed by i
    return np.einsum("pi,pi->p", ex, inner)


def polar_from_pixels(A, k, n_psi: int, chunk: int = 4096):
    """A [N, n, n] (or [n, n]) -> Ahat [N, n_k, n_psi] complex128 on the polar grid (k_m, psi_p)."""
    A = np.asarray(A, dtype=np.float64)
    single = A.ndim == 2
    if single:
        A = A[None]
    k = np.asarray(k, dtype=np.float64)
    psi = 2.0 * np.pi * np.arange(n_psi) / n_psi
    kx = (k[:, None] * np.cos(psi)[None, :]).reshape(-1)
    ky = (k[:, None] * np.sin(psi)[None, :]).reshape(-1)
    out = np.empty((A.shape[0], k.size * n_psi), dtype=np.complex128)
    for a in range(A.shape[0]):
        for s in range(0, kx.size, chunk):
            out[a, s:s + chunk] = ft_points(A[a], kx[s:s + chunk], ky[s:s + chunk])
    out = out.reshape(A.shape[0], k.size, n_psi)
    return out[0] if single else out
