"""Quick A/B of the fused Step 2+3 kernel (k_step23) against the separate k_step2_fft + k_step3_tc path on
the same inputs: per-pair maxima and argmax, per config (debug script; the parity tests are in tests/)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_1905_12317_b200 as pkg  # noqa: E402


def run(cfg, ni, nj, variant):
    # variant: "old" k_step3_tc, "v2" the CTA-pair Step 3 (default), "fused" Steps 2 + 3 (opt-in)
    os.environ["FTK_S23"] = "1" if variant == "fused" else "0"
    os.environ["FTK_S3V2"] = "1" if variant == "v2" else "0"
    p = pkg.FTKPlan(cfg.n, cfg.K, synth.delta_max(cfg), synth.shift_list(cfg), cfg.eps, n_k=cfg.n_k,
                    n_psi=cfg.n_psi, device=0)
    k, w = p.radial()
    imgs, _ = synth.draw_items(cfg, "images", range(ni), k, backend="torch", device="cuda")
    tpls, _ = synth.draw_items(cfg, "templates", range(nj), k, backend="torch", device="cuda")
    p.load_images(imgs)
    p.load_templates(tpls)
    res = p.align(pair_best=True)
    torch.cuda.synchronize()
    t0 = time.time()
    res = p.align(pair_best=True)
    torch.cuda.synchronize()
    dt = time.time() - t0
    pb = pkg.best_to_numpy(res["pair_best"].reshape(-1, 4)).reshape(ni, nj)
    return pb, dt


for name, ni, nj in [("c3", 200, 24), ("c2", 150, 40), ("c5", 260, 40), ("c4", 130, 8), ("tiny", 4, 4)]:
    cfg = synth.config(name)
    a, ta = run(cfg, ni, nj, "old")
    for var in ("v2", "fused"):
        b, tb = run(cfg, ni, nj, var)
        dv = np.abs(a["value"] - b["value"]).max() / np.abs(a["value"]).max()
        same = np.mean((a["shift_idx"] == b["shift_idx"]) & (a["rot_idx"] == b["rot_idx"]))
        print(f"{name} {var}: max |dv|/max|v| = {dv:.2e}, argmax agreement {same:.4f}, time old {ta*1e3:.1f} ms "
              f"{var} {tb*1e3:.1f} ms", flush=True)
