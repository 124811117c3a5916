"""Operator SVD of the Bessel translation kernel and the FTK plan (TEST INFRASTRUCTURE ONLY).

PAPER.md Sec. 4.5:
  * Eq. (Jsvd): J_ell(delta k) = sum_eta U_eta(delta; ell) Sigma_eta(ell) V_eta(k; ell)
    on delta in [0,D], k in [0,K], with U orthonormal under delta d delta and V under k dk;
    Sigma depends only on D K = 2 pi W.  We work in the rescaled variables of the Lemma 2
    proof: x = K delta in [0, 2 pi W], y = k / K in [0, 1], J_ell(x y), with
    weights x dx and y dy; then U(delta) = K u(K delta), V(k) = v(k/K) / K.
  * Remark r:svd P:801-811: project onto orthonormal Jacobi(0,1) polynomial bases and take
    a dense SVD  ("jacobi" method).  A second, independent discretization ("nystrom":
    symmetric Nystrom on Gauss-Jacobi(0,1) nodes) must agree with it (pin).
  * Eq. (svdtrunc): Y_eta(delta; ell) = U_eta(delta) exp(-i ell (omega + pi/2)),
    G_eta(k; ell) = Sigma_eta(ell) V_eta(k; ell).
  * global relabel zeta by non-increasing Sigma; keep Sigma > eps (reading R6).
  * ell < 0 from J_{-ell} = (-1)^ell J_ell: same Sigma and U, V * (-1)^ell (reading R7).
"""
from __future__ import annotations

import dataclasses
import math
from typing import Callable, List

import numpy as np
from scipy.special import eval_jacobi, jv, roots_jacobi

from . import bounds as _bounds
from .quadrature import radial_rule


@dataclasses.dataclass
class ModalSVD:
    ell: int
    sigma: np.ndarray                 # all computed singular values, non-increasing
    u: Callable[[np.ndarray, int], np.ndarray]   # u(x, eta): left function on [0, a], x dx-orthonormal
    v: Callable[[np.ndarray, int], np.ndarray]   # v(y, eta): right function on [0, 1], y dy-orthonormal


def _gj_nodes(n, a):
    """Gauss-Jacobi(0,1) on [0,a] for weight x dx: x = a(1+t)/2, x dx = (a^2/4)(1+t) dt."""
    t, om = roots_jacobi(n, 0.0, 1.0)
    return 0.5 * a * (1.0 + t), om * 0.25 * a * a, t


def _fix_sign(vec_on_nodes):
    """Sign convention (reading R7): largest-|entry| of the y-side vector positive."""
    i = int(np.argmax(np.abs(vec_on_nodes)))
    return 1.0 if vec_on_nodes[i] >= 0 else -1.0


def modal_svd_nystrom(ell: int, a: float, n_nodes: int = 128) -> ModalSVD:
    """Symmetrized Nystrom: M_ij = sqrt(wx_i) J_ell(x_i y_j) sqrt(wy_j); Nystrom extension off-node."""
    x, wx, _ = _gj_nodes(n_nodes, a)
    y, wy, _ = _gj_nodes(n_nodes, 1.0)
    M = np.sqrt(wx)[:, None] * jv(ell, x[:, None] * y[None, :]) * np.sqrt(wy)[None, :]
    P, S, QT = np.linalg.svd(M)
    signs = np.array([_fix_sign(QT[e] / np.sqrt(wy)) for e in range(S.size)])
    P = P * signs[None, :]
    QT = QT * signs[:, None]

    def u(xq, eta):  # u(x) = (1/s) int J(x y) v(y) y dy, v(y_j) = QT[eta, j] / sqrt(wy_j)
        xq = np.asarray(xq, dtype=np.float64)
        return (jv(ell, xq[..., None] * y) @ (np.sqrt(wy) * QT[eta])) / S[eta]

    def v(yq, eta):  # v(y) = (1/s) int J(x y) u(x) x dx, u(x_i) = P[i, eta] / sqrt(wx_i)
        yq = np.asarray(yq, dtype=np.float64)
        return (jv(ell, yq[..., None] * x) @ (np.sqrt(wx) * P[:, eta])) / S[eta]

    return ModalSVD(ell, S, u, v)


def modal_svd_jacobi(ell: int, a: float, n_basis: int = 48, n_quad: int = 128) -> ModalSVD:
    """Remark r:svd: tensor-product projection onto orthonormal Jacobi(0,1) bases
    phi_j(x) = sqrt(2(j+1))/a P_j^{(0,1)}(2x/a - 1) on [0,a] (x dx), psi_j(y) likewise on [0,1]."""
    x, wx, tx = _gj_nodes(n_quad, a)
    y, wy, ty = _gj_nodes(n_quad, 1.0)
    j = np.arange(n_basis)
    cx = np.sqrt(2.0 * (j + 1)) / a
    cy = np.sqrt(2.0 * (j + 1))
    Px = cx[:, None] * eval_jacobi(j[:, None], 0.0, 1.0, tx[None, :])   # [nb, nq]
    Py = cy[:, None] * eval_jacobi(j[:, None], 0.0, 1.0, ty[None, :])
    C = (Px * wx) @ jv(ell, x[:, None] * y[None, :]) @ (Py * wy).T     # coefficient matrix
    U, S, VT = np.linalg.svd(C)
    signs = np.array([_fix_sign(VT[e] @ Py) for e in range(S.size)])
    U = U * signs[None, :]
    VT = VT * signs[:, None]

    def u(xq, eta):
        xq = np.asarray(xq, dtype=np.float64)
        t = 2.0 * xq / a - 1.0
        return np.einsum("j,j...->...", U[:, eta] * cx, eval_jacobi(j.reshape((-1,) + (1,) * t.ndim), 0.0, 1.0, t))

    def v(yq, eta):
        yq = np.asarray(yq, dtype=np.float64)
        t = 2.0 * yq - 1.0
        return np.einsum("j,j...->...", VT[eta] * cy, eval_jacobi(j.reshape((-1,) + (1,) * t.ndim), 0.0, 1.0, t))

    return ModalSVD(ell, S, u, v)


@dataclasses.dataclass
class Term:
    ell: int
    eta: int           # 0-based index within the ell block
    sigma: float


@dataclasses.dataclass
class OraclePlan:
    n: int
    K_cycles: float
    k_max: float
    delta_max: float
    W: float
    eps: float
    n_k: int
    n_psi: int
    k: np.ndarray              # radial nodes [n_k]
    w: np.ndarray              # radial weights [n_k]
    shifts: np.ndarray         # [N_t, 2] px
    terms: List[Term]          # zeta order, both signs of ell
    G: np.ndarray              # [H, n_k]  G_zeta(k_m) = Sigma_zeta V_zeta(k_m)
    Y: np.ndarray              # [N_t, H]  Y_zeta(delta_t) = U_zeta(|delta_t|) e^{-i ell (omega_t + pi/2)}
    modal: dict                # ell >= 0 -> ModalSVD
    all_sigma: dict            # ell >= 0 -> all computed singular values

    @property
    def H(self) -> int:
        return len(self.terms)

    @property
    def H_ell(self) -> dict:
        out = {}
        for t in self.terms:
            out[t.ell] = out.get(t.ell, 0) + 1
        return out

    @property
    def H_plus(self) -> int:
        return sum(1 for t in self.terms if t.ell >= 0)


def modal_spectra(W: float, eps: float, method: str = "nystrom", n_nodes: int = 128, ell_max=None):
    """Sigma_eta(ell) for ell = 0..ell_max (default: Theorem 1's cap 2*calH, where H_ell = 0 beyond)."""
    a = 2.0 * math.pi * W
    if ell_max is None:
        ell_max = int(math.ceil(2.0 * _bounds.theorem1_calH(W, eps)))
    out = {}
    for ell in range(0, ell_max + 1):
        if method == "nystrom":
            out[ell] = modal_svd_nystrom(ell, a, n_nodes)
        else:
            out[ell] = modal_svd_jacobi(ell, a, n_basis=min(64, n_nodes // 2), n_quad=n_nodes)
    return out


def order_terms(kept):
    """Global relabel: Sigma desc, then |ell| asc, ell > 0 first, eta asc (reading R8)."""
    return sorted(kept, key=lambda t: (-t.sigma, abs(t.ell), 0 if t.ell > 0 else (1 if t.ell < 0 else 0), t.eta))


def build_plan(n: int, K_cycles: float, delta_max: float, shifts, eps: float, n_k: int, n_psi: int,
               rule: str = "gl", method: str = "nystrom", n_nodes: int = 128) -> OraclePlan:
    """The FTK plan (Sec. 4.5): radial rule, truncated modal SVDs, G_zeta(k_m), Y_zeta(delta_t)."""
    k_max = 2.0 * math.pi * K_cycles / n                 # reading R1: K in cycles per width
    W = delta_max * k_max / (2.0 * math.pi)              # P:284  D = 2 pi W / K
    k, w = radial_rule(n_k, k_max, rule)
    shifts = np.asarray(shifts, dtype=np.float64).reshape(-1, 2)
    modal = modal_spectra(W, eps, method, n_nodes)
    kept = []
    for ell, ms in modal.items():
        for eta, s in enumerate(ms.sigma):
            if s > eps:
                kept.append(Term(ell, eta, float(s)))
                if ell > 0:
                    kept.append(Term(-ell, eta, float(s)))
    terms = order_terms(kept)
    d = np.hypot(shifts[:, 0], shifts[:, 1])
    om = np.arctan2(shifts[:, 1], shifts[:, 0])
    G = np.empty((len(terms), n_k))
    Y = np.empty((shifts.shape[0], len(terms)), dtype=np.complex128)
    for z, t in enumerate(terms):
        ms = modal[abs(t.ell)]
        par = (-1.0) ** abs(t.ell) if t.ell < 0 else 1.0     # J_{-l} = (-1)^l J_l on the V side
        G[z] = t.sigma * par * ms.v(k / k_max, t.eta) / k_max            # Sigma V(k), V(k) = v(k/K)/K
        U = k_max * ms.u(k_max * d, t.eta)                                # U(delta) = K u(K delta)
        Y[:, z] = U * np.exp(-1j * t.ell * (om + 0.5 * math.pi))
    return OraclePlan(n, K_cycles, k_max, delta_max, W, eps, n_k, n_psi, k, w, shifts, terms, G, Y,
                      modal, {l: m.sigma for l, m in modal.items()})


def f_svd(plan: OraclePlan, delta_xy, k, psi):
    """F^SVD(delta, k) = sum_zeta Y_zeta(delta) G_zeta(k) e^{i ell psi}."""
    delta_xy = np.asarray(delta_xy, dtype=np.float64).reshape(-1, 2)
    d = np.hypot(delta_xy[:, 0], delta_xy[:, 1])
    om = np.arctan2(delta_xy[:, 1], delta_xy[:, 0])
    k = np.atleast_1d(np.asarray(k, dtype=np.float64))
    psi = np.atleast_1d(np.asarray(psi, dtype=np.float64))
    out = np.zeros((delta_xy.shape[0], k.size, psi.size), dtype=np.complex128)
    for t in plan.terms:
        ms = plan.modal[abs(t.ell)]
        par = (-1.0) ** abs(t.ell) if t.ell < 0 else 1.0
        Yz = plan.k_max * ms.u(plan.k_max * d, t.eta) * np.exp(-1j * t.ell * (om + 0.5 * math.pi))
        Gz = t.sigma * par * ms.v(k / plan.k_max, t.eta) / plan.k_max
        out += Yz[:, None, None] * Gz[None, :, None] * np.exp(1j * t.ell * psi)[None, None, :]
    return out


def kernel_certificate(plan: OraclePlan, n_psi: int = None):
    """max over (t, m, p) of |F - F^SVD| on the plan's own grid."""
    n_psi = plan.n_psi if n_psi is None else n_psi
    psi = 2.0 * math.pi * np.arange(n_psi) / n_psi
    Fs = f_svd(plan, plan.shifts, plan.k, psi)
    F = np.exp(-1j * plan.k[None, :, None] * (plan.shifts[:, 0, None, None] * np.cos(psi)[None, None, :]
                                               + plan.shifts[:, 1, None, None] * np.sin(psi)[None, None, :]))
    return float(np.max(np.abs(F - Fs)))
