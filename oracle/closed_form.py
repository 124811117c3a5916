"""Exact inner products of Gaussian-blob images (TEST INFRASTRUCTURE ONLY).

For A = sum_b alpha_b exp(-|x - c_b|^2 / 2 s_b^2) and B likewise (beta, c', s'):
  R_gamma T_delta A has blob centres R_gamma (c_b + delta),
  int exp(-|x-u|^2/2s^2) exp(-|x-v|^2/2t^2) dx = 2 pi s^2 t^2 / (s^2 + t^2) exp(-|u-v|^2 / 2(s^2+t^2)),
and by Plancherel (Eq. planch) the (untruncated) Fourier-domain inner product is
  (2 pi)^2 <R_gamma T_delta A, B>.  Truncation to Omega_K (Eq. Xdg) changes it by the Gaussian tail
  beyond K, < 1e-9 relative for s, t >= 1.5 px at K = pi rad/px.
"""
from __future__ import annotations

import math

import numpy as np


def gaussian_ip(pa, pb, ia: int, ib: int, delta_xy, gamma) -> float:
    """(2 pi)^2 <R_gamma T_delta A_ia, B_ib> for blob parameter dicts pa, pb (see synth.blob_params)."""
    cx, cy, sa, aa = pa["cx"][ia], pa["cy"][ia], pa["sigma"][ia], pa["amp"][ia]
    dx, dy, sb, ab = pb["cx"][ib], pb["cy"][ib], pb["sigma"][ib], pb["amp"][ib]
    ux, uy = cx + delta_xy[0], cy + delta_xy[1]
    c, s = math.cos(gamma), math.sin(gamma)
    ux, uy = c * ux - s * uy, s * ux + c * uy
    s2 = sa[:, None] ** 2 + sb[None, :] ** 2
    d2 = (ux[:, None] - dx[None, :]) ** 2 + (uy[:, None] - dy[None, :]) ** 2
    ov = 2.0 * math.pi * (sa[:, None] ** 2) * (sb[None, :] ** 2) / s2 * np.exp(-d2 / (2.0 * s2))
    return (2.0 * math.pi) ** 2 * float(aa @ ov @ ab)
