"""CTF-parameterized factorized kernel (TEST INFRASTRUCTURE ONLY).

PAPER.md Sec. 6 "Other 2D kernels": images are filtered by a contrast transfer function
parametrized by defocus tau; "translating by delta and filtering by a CTF with defocus
parameters tau corresponds to pointwise multiplication by a function dependent on delta and tau" and
the approach extends by "factorizing this function into terms of the form Y_zeta(delta, tau) G_zeta(k)"
(P:1401-1403).  The paper gives no formula beyond this sketch; reading R24:

  * the filters are real and radial, c_tau(|k|), given by the caller on the radial nodes k_m (any CTF
    model; astigmatism, which would make c depend on psi, is out of scope);
  * the filter acts on the template:  X(delta, gamma, tau) = <R_gamma T_delta A, c_tau B>, i.e. the
    brute-force sum of oracle.brute with the extra factor c_tau(k_m);
  * F(delta, k) c_tau(|k|) is factorized per Bessel order ell (the ell-th angular mode of F is
    J_ell(|delta| |k|), Eq. (Fexp) / (Jsvd) P:786-797; c_tau only rescales it radially), exactly as the
    paper does for c = 1, by an SVD of J_ell(x y) c_tau(y K) over rows (x, tau)
    (x = K |delta| in [0, 2 pi W] with weight x dx, every tau weight 1) and columns y_m = k_m / K (weight
    w_m / K^2 -- the radial rule itself, since c is known only on k_m); Sigma > eps kept, global relabel
    as P:858-873 (reading R6/R8); Y_zeta(delta, tau) = U_zeta(|delta|, tau) e^{-i ell (omega + pi/2)},
    G_zeta(k_m) = Sigma_zeta V_zeta(k_m) (Eq. svdtrunc P:828-831 with U extended in x by Nystrom).
    With weight 1 per tau the discarded tail bounds every filter's error: sum_tau ||E_tau||^2 =
    sum over dropped Sigma^2.

Results index the virtual shift v = tau * N_t + t (tau-major), so oracle.ftk.ftk_landscapes runs the
unchanged Steps 1-3 on the returned plan.
"""
from __future__ import annotations

import math

import numpy as np
from scipy.special import jv

from . import bounds as _bounds
from .brute import _phase
from .kernel_svd import OraclePlan, Term, _gj_nodes, order_terms
from .quadrature import radial_rule


def brute_landscape_ctf(A, B, k, w, shifts, filters):
    """X^bf[tau, t, r] = (2 pi / n_psi) sum_m w_m c_tau(k_m) sum_p F(delta_t; k_m, psi_p) Ahat(m, p)
    conj Bhat(m, (p + r) mod n_psi): Eq. (Xdg) (reading R10) with the template filtered by the
    real radial c_tau.  Plain definition, no Bessel function / SVD / FFT."""
    A = np.asarray(A, dtype=np.complex128)
    B = np.asarray(B, dtype=np.complex128)
    c = np.atleast_2d(np.asarray(filters, dtype=np.float64))
    n_psi = A.shape[-1]
    FA = _phase(shifts, k, n_psi) * A[None]                                  # [T, M, P]
    Brot = np.stack([np.roll(B, -r, axis=-1) for r in range(n_psi)])         # [R, M, P]
    return (2.0 * math.pi / n_psi) * np.einsum("m,cm,tmp,rmp->ctr", np.asarray(w), c, FA, np.conj(Brot))


def modal_svd_ctf(ell, a, y, wy, filters, n_nodes=128):
    """SVD of M[(tau, i), m] = sqrt(wx_i) J_ell(x_i y_m) c_tau(m) sqrt(wy_m) (reading R24).
    Returns (S, QT, x, wx): singular values (non-increasing), right vectors QT[e, m] (sign: largest
    |v(y_m)| = |QT[e, m]| / sqrt(wy_m) positive), and the x nodes / weights."""
    x, wx, _ = _gj_nodes(n_nodes, a)
    c = np.atleast_2d(np.asarray(filters, dtype=np.float64))
    J = jv(ell, x[:, None] * y[None, :])                                      # [i, m]
    M = (np.sqrt(wx)[None, :, None] * J[None] * c[:, None, :] * np.sqrt(wy)[None, None, :]).reshape(-1, y.size)
    _, S, QT = np.linalg.svd(M, full_matrices=False)
    for e in range(S.size):
        v = QT[e] / np.sqrt(wy)
        if v[int(np.argmax(np.abs(v)))] < 0:
            QT[e] = -QT[e]
    return S, QT, x, wx


def build_plan_ctf(n, K_cycles, delta_max, shifts, eps, n_k, n_psi, filters, rule="gl", n_nodes=128):
    """The CTF-parameterized FTK plan: radial rule, per-ell joint (delta, tau) SVDs, eps truncation,
    G_zeta(k_m) and Y_zeta(delta_t, tau) on the virtual shift list (tau-major)."""
    k_max = 2.0 * math.pi * K_cycles / n                  # reading R1
    W = delta_max * k_max / (2.0 * math.pi)
    a = 2.0 * math.pi * W
    k, w = radial_rule(n_k, k_max, rule)
    c = np.atleast_2d(np.asarray(filters, dtype=np.float64))
    n_tau = c.shape[0]
    shifts = np.asarray(shifts, dtype=np.float64).reshape(-1, 2)
    y = k / k_max
    wy = w / k_max ** 2
    ell_cap = int(math.ceil(2.0 * _bounds.theorem1_calH(W, eps)))
    modal, kept = {}, []
    for ell in range(ell_cap + 1):
        S, QT, _, _ = modal_svd_ctf(ell, a, y, wy, c, n_nodes)
        modal[ell] = (S, QT)
        for eta, s in enumerate(S):
            if s > eps:
                kept.append(Term(ell, eta, float(s)))
                if ell > 0:
                    kept.append(Term(-ell, eta, float(s)))
    terms = order_terms(kept)
    d = np.hypot(shifts[:, 0], shifts[:, 1])
    om = np.arctan2(shifts[:, 1], shifts[:, 0])
    N_t = shifts.shape[0]
    G = np.empty((len(terms), n_k))
    Y = np.empty((n_tau * N_t, len(terms)), dtype=np.complex128)
    for z, t in enumerate(terms):
        S, QT = modal[abs(t.ell)]
        par = (-1.0) ** abs(t.ell) if t.ell < 0 else 1.0      # J_{-l} = (-1)^l J_l (reading R7)
        G[z] = t.sigma * par * (QT[t.eta] / np.sqrt(wy)) / k_max          # Sigma V(k_m), V = v(k/K)/K
        Jt = jv(abs(t.ell), k_max * d[:, None] * y[None, :])               # [t, m]
        u = (Jt[None] * c[:, None, :]) @ (np.sqrt(wy) * QT[t.eta]) / t.sigma   # [tau, t]: Nystrom in x
        Y[:, z] = (k_max * u).reshape(-1) * np.tile(np.exp(-1j * t.ell * (om + 0.5 * math.pi)), n_tau)
    return OraclePlan(n, K_cycles, k_max, delta_max, W, eps, n_k, n_psi, k, w, np.tile(shifts, (n_tau, 1)),
                      terms, G, Y, {}, {l: m[0] for l, m in modal.items()})


def kernel_certificate_ctf(plan: OraclePlan, filters, n_psi=None):
    """max over (tau, t, m, p) of |c_tau(k_m) F(delta_t, k_m, psi_p) - sum_zeta Y G e^{i ell psi}|, F from
    its definition exp(-i k.delta) (Eq. Fdk)."""
    n_psi = plan.n_psi if n_psi is None else n_psi
    c = np.atleast_2d(np.asarray(filters, dtype=np.float64))
    n_tau = c.shape[0]
    N_t = plan.shifts.shape[0] // n_tau
    psi = 2.0 * math.pi * np.arange(n_psi) / n_psi
    ells = np.array([t.ell for t in plan.terms])
    E = np.exp(1j * ells[:, None] * psi[None, :])                            # [z, p]
    Fs = np.einsum("vz,zm,zp->vmp", plan.Y, plan.G, E)
    sh = plan.shifts
    F = np.exp(-1j * plan.k[None, :, None] * (sh[:, 0, None, None] * np.cos(psi)[None, None, :]
                                              + sh[:, 1, None, None] * np.sin(psi)[None, None, :]))
    cf = np.repeat(c, N_t, axis=0)[:, :, None]                               # [v, m, 1]
    return float(np.max(np.abs(cf * F - Fs)))
