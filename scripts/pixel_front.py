"""Pixel front end: achieved NUFFT error vs the oracle trapezoid sum, and device throughput.
Usage: python scripts/pixel_front.py   (GPU)"""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth, paper_1905_12317_b200 as pkg
from oracle import pixels

for name in ["tiny", "c2", "c3", "c5"]:
    cfg = synth.config(name)
    p = pkg.FTKPlan(cfg.n, cfg.K, synth.delta_max(cfg), synth.shift_list(cfg), cfg.eps, n_k=cfg.n_k, n_psi=cfg.n_psi, device=0)
    k, _ = p.radial()
    pix, _ = synth.draw_pixel_items(cfg, "images", range(2))
    got = p.polar_from_pixels(torch.from_numpy(pix).cuda()).cpu().numpy()
    rng = np.random.default_rng(0)
    m, q = rng.integers(0, cfg.n_k, 400), rng.integers(0, cfg.n_psi, 400)
    psi = 2 * np.pi * q / cfg.n_psi
    ref = pixels.ft_points(pix[0], k[m] * np.cos(psi), k[m] * np.sin(psi))
    err = np.max(np.abs(got[0, m, q] - ref)) / np.abs(pix[0].astype(np.float64)).sum()
    rel2 = np.linalg.norm(got[0, m, q] - ref) / np.linalg.norm(ref)
    # throughput: N images resident on the device, polar samples + FB coefficients (ftk_load_images_pixels)
    N = {"tiny": 4096, "c2": 4096, "c3": 2048, "c5": 1024}[name]
    x = torch.from_numpy(np.repeat(pix[:1], N, axis=0)).cuda()
    p.load_images_pixels(x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        p.load_images_pixels(x)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(f"{name}: n={cfg.n} max|err|/sum|A| = {err:.2e}, rel L2 = {rel2:.2e}; load_images_pixels {N} images: "
          f"{ms:.2f} ms = {ms * 1e3 / N:.2f} us/image", flush=True)
