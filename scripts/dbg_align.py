"""Debug helper: run one ftk_align on a config subset and report success / the failing step.
Usage: FTK_SYNC_DEBUG=1 python scripts/dbg_align.py CONFIG N_IMAGES N_TEMPLATES"""
import os, sys, torch, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth, paper_1905_12317_b200 as pkg
cfg = synth.config(sys.argv[1])
ni, nj = int(sys.argv[2]), int(sys.argv[3])
p = pkg.FTKPlan(cfg.n, cfg.K, synth.delta_max(cfg), synth.shift_list(cfg), cfg.eps, n_k=cfg.n_k, n_psi=cfg.n_psi, device=0)
k, w = p.radial()
imgs, _ = synth.draw_items(cfg, "images", range(ni), k)
tpls, _ = synth.draw_items(cfg, "templates", range(nj), k)
p.load_images(torch.from_numpy(imgs).cuda()); p.load_templates(torch.from_numpy(tpls).cuda())
torch.cuda.synchronize()
print(sys.argv[1:], p.info["H_plus"], p.info["K3p"], end=" ")
try:
    r = p.align(); torch.cuda.synchronize(); print("align ok")
except Exception as e:
    print("align failed", e)
