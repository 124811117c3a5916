"""CPU pin of DESIGN.md section 6 (precision): the tensor-core engine's data path emulated in numpy
(scripts/precision_study.py: every product exact, fp32 sums, the kernels' power-of-two scales) against the
float64 oracle FTK at tiny, 4 pairs.  fp16x3 must stay within the engine's 2.5e-6 bar and near 3xTF32;
bf16x3 (round 1's format) must be clearly worse -- the claim that motivated the change."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "scripts"))
import precision_study as ps  # noqa: E402
import synth  # noqa: E402
from oracle import fb, ftk, kernel_svd as ks  # noqa: E402


def test_fp16x3_emulated_precision_tiny():
    cfg = synth.config("tiny")
    plan = ks.build_plan(cfg.n, cfg.K, synth.delta_max(cfg), synth.shift_list(cfg), cfg.eps, cfg.n_k, cfg.n_psi,
                         n_nodes=96)
    imgs, _ = synth.draw_items(cfg, "images", range(2), plan.k, "planted")
    tpls, _ = synth.draw_items(cfg, "templates", range(2), plan.k)
    A, B = fb.fb_coeffs(imgs), fb.fb_coeffs(tpls)
    na, nb = fb.discrete_norm(imgs, plan.w), fb.discrete_norm(tpls, plan.w)
    X = np.real(ftk.ftk_landscapes(A, B, plan))
    worst = {f: 0.0 for f in ("fp16x3", "tf32x3", "bf16x3")}
    for i in range(2):
        for j in range(2):
            for f in worst:
                e = np.max(np.abs(ps.chain(A[i], B[j], plan, f) - X[i, j])) / (na[i] * nb[j])
                worst[f] = max(worst[f], e)
    assert worst["fp16x3"] <= 2.5e-6, worst
    assert worst["fp16x3"] <= 3.0 * worst["tf32x3"] + 1e-7, worst
    assert worst["bf16x3"] >= 10.0 * worst["fp16x3"], worst


def test_f16_scale_exp_matches_kernel_rule():
    """The emulation's exponent rule is the kernels' (ftk_sm100.cuh f16_scale_exp): x 2^e in (2^13, 2^14]."""
    for x in [1.0, 0.75, 2.0 ** 14, 2.0 ** 14 * 1.0001, 3.1e-20, 7.7e15, 0.0]:
        e = ps.f16_scale_exp(x)
        if x == 0.0:
            assert e == 0
            continue
        y = x * 2.0 ** e
        assert 2.0 ** 13 < y <= 2.0 ** 14, (x, e, y)
