"""Small FTK workload for compute-sanitizer runs (racecheck / synccheck / memcheck): tiny and a ragged c2
subset through ftk_align (tensor-core engine: k_ring_fft, k_prep_image_op, k_step1_tc, k_step2_fft,
k_step3_tc, k_finalize) with per-pair maxima, plus one explicit-pair landscape."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_1905_12317_b200 as pkg  # noqa: E402

for name, ni, nj in [("tiny", 4, 4), ("c2", 6, 20)]:
    cfg = synth.config(name)
    p = pkg.FTKPlan(cfg.n, cfg.K, synth.delta_max(cfg), synth.shift_list(cfg), cfg.eps, n_k=cfg.n_k,
                    n_psi=cfg.n_psi, device=0)
    k, _ = p.radial()
    imgs, _ = synth.draw_items(cfg, "images", range(ni), k)
    tpls, _ = synth.draw_items(cfg, "templates", range(nj), k)
    p.load_images(torch.from_numpy(imgs).cuda())
    p.load_templates(torch.from_numpy(tpls).cuda())
    res = p.align(pair_best=True)
    L = p.landscape_pairs([0, ni - 1], [nj - 1, 0])
    torch.cuda.synchronize()
    b = pkg.best_to_numpy(res["best"])
    print(name, "best values", np.round(b["value"][:3], 4), "landscape max", float(L.max()), flush=True)
print("sanitize case done")
