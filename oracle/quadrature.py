"""Radial quadrature rules for int_0^K g(k) k dk (TEST INFRASTRUCTURE ONLY).

PAPER.md Sec. 3.1 "Discretization and truncation": nodes k_m in [0,K],
weights w_m with  int_0^K g(k) k dk ~ sum_m g(k_m) w_m.  The paper prefers
Gauss-Jacobi (alpha=0, beta=1); BASELINE.json's configs name Gauss-Legendre
nodes on [0,K] with weight k dk (reading R2): w_m = omega_m (K/2) k_m.
"""
from __future__ import annotations

import numpy as np
from scipy.special import roots_jacobi


def gauss_legendre_k(n_k: int, k_max: float):
    """Gauss-Legendre on [0,K] times the area element k: exact for k^j k dk, j <= 2 n_k - 2."""
    t, om = np.polynomial.legendre.leggauss(n_k)
    k = 0.5 * k_max * (1.0 + t)
    w = om * 0.5 * k_max * k
    return k, w


def gauss_jacobi_01(n_k: int, k_max: float):
    """Gauss-Jacobi (alpha=0, beta=1) mapped to [0,K]: k dk = (K^2/4)(1+t) dt."""
    t, om = roots_jacobi(n_k, 0.0, 1.0)
    k = 0.5 * k_max * (1.0 + t)
    w = om * 0.25 * k_max * k_max
    return k, w


def radial_rule(n_k: int, k_max: float, rule: str = "gl"):
    if rule == "gl":
        return gauss_legendre_k(n_k, k_max)
    if rule == "gj":
        return gauss_jacobi_01(n_k, k_max)
    raise ValueError(rule)
