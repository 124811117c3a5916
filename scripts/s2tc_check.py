"""A/B of a kernel option on the same inputs: per-pair maxima and argmax, and explicit-pair landscapes (debug script;
the oracle parity is in tests/).  Default: the tensor-core Step 2 (FTK_S2TC=1) against k_step2_fft (FTK_S2TC=0);
`python scripts/s2tc_check.py FTK_S1CG2 c5` compares FTK_S1CG2=1 against 0 on the listed configs."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_1905_12317_b200 as pkg  # noqa: E402


VAR = sys.argv[1] if len(sys.argv) > 1 else "FTK_S2TC"
ONLY = sys.argv[2].split(",") if len(sys.argv) > 2 else None


def run(cfg, ni, nj, s2tc):
    os.environ[VAR] = "1" if s2tc else "0"
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
    L = p.landscape_pairs([0, ni - 1, min(5, ni - 1)], [0, nj - 1, min(3, nj - 1)]).cpu().numpy()
    return pb, dt, L


for name, ni, nj in [("c5", 4, 3), ("c5", 140, 12), ("c5", 600, 40), ("c3", 300, 20), ("c4", 130, 9), ("c2", 200, 30)]:
    if ONLY and name not in ONLY:
        continue
    cfg = synth.config(name)
    a, ta, La = run(cfg, ni, nj, False)
    b, tb, Lb = run(cfg, ni, nj, True)
    dv = np.abs(a["value"] - b["value"]).max() / np.abs(a["value"]).max()
    same = np.mean((a["shift_idx"] == b["shift_idx"]) & (a["rot_idx"] == b["rot_idx"]))
    dl = np.abs(La - Lb).max() / np.abs(La).max()
    print(f"{name} {ni}x{nj}: pair max |dv|/max|v| = {dv:.2e}, argmax agreement {same:.4f}, landscapes "
          f"max |dL|/max|L| = {dl:.2e}; time fft {ta*1e3:.1f} ms tc {tb*1e3:.1f} ms", flush=True)
