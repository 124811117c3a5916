"""Precision study: the FTK chain (Step 1 split GEMM -> fp32 FFT -> Step 3 split GEMM, the tensor-core engine's
data path in Form B with the real Step-3 operand of reading R13) emulated in numpy under five operand
formats, against the float64 oracle FTK (oracle.ftk.ftk_landscapes) on config-shaped synthetic data:

  fp32     operands and accumulation in float32
  tf32x1   operands rounded to TF32 (10-bit mantissa), one product
  tf32x3   x = hi + lo in TF32, hi*hi + hi*lo + lo*hi
  fp16x3   x scaled by a power of two into (2^13, 2^14] (the operand's bound), x = hi + lo in fp16
           (11-bit significand, subnormals below 2^-14), hi*hi + hi*lo + lo*hi   (the library's engine 0, round 2)
  bf16x3   x = hi + lo in bf16 (8-bit mantissa), hi*hi + hi*lo + lo*hi   (engine 0 in round 1)
  bf16x1   operands rounded to bf16, one product

Products are exact (float64) and summed in float32 per contraction, as the tensor core accumulates in fp32.
Error metric: max |dX| / (||A|| ||B||) over the sampled pairs' full landscapes (the north-star tolerance is
1e-4).  Writes a markdown table (stdout, and --out).  Usage:
    python scripts/precision_study.py [--pairs 8] [--out profiles/r2_precision.md]
Test-infrastructure script: it imports oracle/ (allowed for tests and studies, never for the product).
"""
from __future__ import annotations

import argparse
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from oracle import fb, ftk, kernel_svd as ks  # noqa: E402


def round_mant(x, bits):
    """Round float64 x to a float with `bits` explicit mantissa bits (round to nearest even), fp32 range."""
    x = np.asarray(x, dtype=np.float64)
    m, e = np.frexp(x)
    scale = 2.0 ** (bits + 1)
    return np.ldexp(np.round(m * scale) / scale, e)


def f16_scale_exp(bound):
    """The exponent e with bound 2^e in (2^13, 2^14] (0 for a zero bound), as the kernels compute it."""
    if not bound > 0:
        return 0
    m, e = math.frexp(bound)
    return 14 - (e - 1 if m == 0.5 else e)


def split(x, fmt, bound=None):
    """Operand terms of a format: list of (component) arrays whose products are formed pairwise.  fp16x3 takes
    the operand's bound (scale) and returns the terms unscaled (power-of-two scaling is exact)."""
    if fmt == "fp16x3":
        e = f16_scale_exp(float(np.max(np.abs(x))) if bound is None else bound)
        xs = np.ldexp(np.asarray(x, np.float32).astype(np.float64), e)
        hi = xs.astype(np.float16).astype(np.float64)
        lo = (xs - hi).astype(np.float32).astype(np.float16).astype(np.float64)
        return [np.ldexp(hi, -e), np.ldexp(lo, -e)]
    if fmt == "fp32":
        return [np.asarray(x, np.float32).astype(np.float64)]
    bits = {"tf32x1": 10, "tf32x3": 10, "bf16x3": 7, "bf16x1": 7}[fmt]
    hi = round_mant(np.asarray(x, np.float32).astype(np.float64), bits)
    if fmt.endswith("x1"):
        return [hi]
    lo = round_mant(np.asarray(x, np.float64) - hi, bits)
    return [hi, lo]


def _pairs(n):
    return [(0, 0)] if n == 1 else [(0, 0), (0, 1), (1, 0)]


def dot_rows(A, B, fmt, ba=None, bb=None):
    """out[p] = sum_k A[p, k] B[p, k] with the format's products; float32 result (fp32 accumulation)."""
    As, Bs = split(A, fmt, ba), split(B, fmt, bb)
    acc = sum((As[i] * Bs[j]).sum(-1) for i, j in _pairs(len(As)))
    return acc.astype(np.float32).astype(np.float64)


def matmul(A, B, fmt, ba=None, bb=None):
    """A @ B with the format's products; float32 result."""
    As, Bs = split(A, fmt, ba), split(B, fmt, bb)
    acc = sum(As[i] @ Bs[j] for i, j in _pairs(len(As)))
    return acc.astype(np.float32).astype(np.float64)


def chain(a, b, plan, fmt):
    """Tensor-core engine data path, one pair: a, b FB coefficients [n_k, n_psi]; returns X [N_t, n_psi]."""
    n = a.shape[1]
    zp = [z for z, t in enumerate(plan.terms) if t.ell >= 0]          # ell >= 0 terms (reading R13)
    ells = np.array([plan.terms[z].ell for z in zp])
    g = (2.0 * math.pi * plan.w[None, :] * plan.G[zp]).astype(np.float32).astype(np.float64)  # [Hp, n_k]
    # fp16x3 bounds, as the kernels form them (ftk_tc.cu header): image max, template max x max |g|, and the
    # a-priori bound of Z: |Z_zeta(r)| <= sum_{m,p} |a(m,p)| |g_zeta(m)| |b(m,p+ell)| <= gmax ||a||_F ||b||_F
    amax = float(max(np.abs(a.real).max(), np.abs(a.imag).max()))
    bmax = float(max(np.abs(b.real).max(), np.abs(b.imag).max()))
    gabs = np.abs(g)
    cbound = float(gabs.max()) * bmax
    zbound = float(gabs.max()) * float(np.linalg.norm(a)) * float(np.linalg.norm(b))  # Cauchy-Schwarz over (m, p)
    # Step 1, Form B: Zhat'_z(p) = sum_m a(m, p) g_z(m) conj b(m, p + ell_z)   (real GEMM over [re | im])
    Zh = np.empty((len(zp), n), dtype=np.complex128)
    for zi, l in enumerate(ells):
        c = (g[zi][:, None] * np.conj(np.roll(b, -l, axis=1))).astype(np.complex64).astype(np.complex128)  # [m, p]
        ar, ai, cr, ci = a.real.T, a.imag.T, c.real.T, c.imag.T   # [p, m]
        arow = np.concatenate([ar, ai], 1)                        # image operand rows [p, 2 n_k]
        re = dot_rows(arow, np.concatenate([cr, -ci], 1), fmt, amax, cbound)   # Re-row of the generated operand
        im = dot_rows(arow, np.concatenate([ci, cr], 1), fmt, amax, cbound)    # Im-row
        Zh[zi] = re + 1j * im
    # Step 2 in fp32: Z_z(r) = e^{-2 pi i ell r / n} FFT(Zhat'_z)(r)
    Z = np.fft.fft(Zh.astype(np.complex64), axis=1).astype(np.complex64).astype(np.complex128)
    r = np.arange(n)
    Z = (Z * np.exp(-2j * math.pi * ells[:, None] * r[None, :] / n)).astype(np.complex64).astype(np.complex128)
    # Step 3, real form: X = sum_{ell=0} Re(Y) Re(Z) + sum_{ell>0} (2 Re Y Re Z - 2 Im Y Im Z)
    Yp = plan.Y[:, zp]
    cols_Y, cols_Z = [], []
    for zi, l in enumerate(ells):
        if l == 0:
            cols_Y.append(Yp[:, zi].real)
            cols_Z.append(Z[zi].real)
        else:
            cols_Y += [2.0 * Yp[:, zi].real, -2.0 * Yp[:, zi].imag]
            cols_Z += [Z[zi].real, Z[zi].imag]
    Y3 = np.stack(cols_Y, 1).astype(np.float32).astype(np.float64)      # [N_t, K3]
    Z3 = np.stack(cols_Z, 0)                                            # [K3, n]
    return matmul(Y3, Z3, fmt, None, zbound)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--pairs", type=int, default=8)
    ap.add_argument("--configs", default="tiny,c2,c3,c5")
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    fmts = ["fp32", "tf32x3", "fp16x3", "bf16x3", "tf32x1", "bf16x1"]
    lines = ["| config | pairs | " + " | ".join(fmts) + " |", "|---|---|" + "---|" * len(fmts)]
    for name in args.configs.split(","):
        cfg = synth.config(name)
        plan = ks.build_plan(cfg.n, cfg.K, synth.delta_max(cfg), synth.shift_list(cfg), cfg.eps, cfg.n_k, cfg.n_psi,
                             n_nodes=96)
        ni = max(1, min(cfg.N_im, int(math.ceil(math.sqrt(args.pairs)))))
        nj = max(1, min(cfg.N_tm, (args.pairs + ni - 1) // ni))
        imgs, _ = synth.draw_items(cfg, "images", range(ni), plan.k, "planted" if name == "tiny" else "independent")
        tpls, _ = synth.draw_items(cfg, "templates", range(nj), plan.k)
        A, B = fb.fb_coeffs(imgs), fb.fb_coeffs(tpls)
        na, nb = fb.discrete_norm(imgs, plan.w), fb.discrete_norm(tpls, plan.w)
        X = np.real(ftk.ftk_landscapes(A, B, plan))
        worst = {f: 0.0 for f in fmts}
        for i in range(ni):
            for j in range(nj):
                for f in fmts:
                    e = np.max(np.abs(chain(A[i], B[j], plan, f) - X[i, j])) / (na[i] * nb[j])
                    worst[f] = max(worst[f], e)
        lines.append(f"| {name} | {ni * nj} | " + " | ".join(f"{worst[f]:.1e}" for f in fmts) + " |")
        print(lines[-1], flush=True)
    text = "\n".join(lines)
    print(text)
    if args.out:
        with open(args.out, "w") as fh:
            fh.write(text + "\n")


if __name__ == "__main__":
    main()
