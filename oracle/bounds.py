"""Rank bounds of PAPER.md Sec. 5 (TEST INFRASTRUCTURE ONLY).

Theorem 1: calH = max(pi e^2 W, log(2 pi W / eps)) + 3/2, H <= 2 calH^2,
  and H_ell = 0 for |ell| > 2 calH.
Lemma 2, Eq. (rank): H_ell <= max(0, pi e^2 W - |ell|/2, log(2 pi W/eps) + 3/2 - |ell|/2)
  (reading R17: the +3/2 sits only on the log branch as printed at P:1023).
Remark after Lemma 2: empirical fit H_ell ~ 2.0 (W - |ell|/(2 pi)) + 0.5 log(1/eps).
"""
from __future__ import annotations

import math


def theorem1_calH(W: float, eps: float) -> float:
    return max(math.pi * math.e ** 2 * W, math.log(2.0 * math.pi * W / eps)) + 1.5


def theorem1_total(W: float, eps: float) -> float:
    return 2.0 * theorem1_calH(W, eps) ** 2


def lemma2(ell: int, W: float, eps: float) -> float:
    a = abs(ell) / 2.0
    return max(0.0, math.pi * math.e ** 2 * W - a, math.log(2.0 * math.pi * W / eps) + 1.5 - a)


def empirical_fit(ell: int, W: float, eps: float) -> float:
    return 2.0 * (W - abs(ell) / (2.0 * math.pi)) + 0.5 * math.log(1.0 / eps)
