"""GPU parity of the pixel front end (Eq. Ahattrap P:302-318 by a type-2 NUFFT,
P:531-541) against the oracle's direct trapezoid sum, and of the whole pixel -> FTK chain against the
oracle FTK on the oracle's polar samples of the same pixels.

Tolerance of the NUFFT stage: |Ahat_gpu - Ahat_oracle| <= 2e-6 sum_ij |A_ij| per sample (kernel width 7 at
upsampling 2 and fp32 FFTs: measured 2-4e-7 of sum |A| at tiny..c5, scripts/pixel_front.py), R23."""
import os

import numpy as np
import pytest

import synth
from oracle import fb, ftk, kernel_svd as ks, pixels

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

NU_TOL = 2e-6
TOL = 1e-4


@pytest.fixture(scope="module")
def pkg():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__ as g
    g.build()
    import paper_1905_12317_b200 as p
    return p


def make(pkg, cfg, **kw):
    return pkg.FTKPlan(cfg.n, cfg.K, synth.delta_max(cfg), synth.shift_list(cfg), cfg.eps, n_k=cfg.n_k,
                       n_psi=cfg.n_psi, device=0, **kw)


@pytest.mark.parametrize("name,ni", [("tiny", 3), ("c2", 4), ("c3", 2)])
def test_polar_from_pixels_vs_oracle(pkg, name, ni):
    cfg = synth.config(name)
    p = make(pkg, cfg)
    k, _ = p.radial()
    pix, _ = synth.draw_pixel_items(cfg, "images", range(ni))
    got = p.polar_from_pixels(torch.from_numpy(pix).cuda()).cpu().numpy()
    ref = pixels.polar_from_pixels(pix, k, cfg.n_psi)
    for a in range(ni):
        l1 = np.abs(pix[a].astype(np.float64)).sum()
        err = np.max(np.abs(got[a] - ref[a])) / l1
        assert err <= NU_TOL, (a, err)
    # host input (chunked H2D) gives the same bits as device input
    assert np.array_equal(p.polar_from_pixels(pix).cpu().numpy(), got)


def test_polar_from_pixels_c5_sampled(pkg):
    cfg = synth.config("c5")
    p = make(pkg, cfg)
    k, _ = p.radial()
    pix, _ = synth.draw_pixel_items(cfg, "templates", [0, 1])
    got = p.polar_from_pixels(torch.from_numpy(pix).cuda()).cpu().numpy()
    rng = np.random.default_rng(3)
    m = rng.integers(0, cfg.n_k, 300)
    q = rng.integers(0, cfg.n_psi, 300)
    psi = 2 * np.pi * q / cfg.n_psi
    for a in range(2):
        ref = pixels.ft_points(pix[a], k[m] * np.cos(psi), k[m] * np.sin(psi))
        err = np.max(np.abs(got[a, m, q] - ref)) / np.abs(pix[a].astype(np.float64)).sum()
        assert err <= NU_TOL, err


def test_ragged_chunks_bitwise(pkg):
    """N = 7 through chunks of 3 (FTK_NU_CHUNK): same bits as one chunk; FB coefficients of a pixel load
    equal the ring FFT of the returned polar samples (ftk_load_images on them)."""
    cfg = synth.config("c2")
    p = make(pkg, cfg)
    pix, _ = synth.draw_pixel_items(cfg, "templates", range(7))
    x = torch.from_numpy(pix).cuda()
    one = p.polar_from_pixels(x).cpu().numpy()
    os.environ["FTK_NU_CHUNK"] = "3"
    try:
        three = p.polar_from_pixels(pix).cpu().numpy()
        p.load_images_pixels(x)
        fb_pix = p.fb_coeffs(0, 0, 7).cpu().numpy()
    finally:
        del os.environ["FTK_NU_CHUNK"]
    assert np.array_equal(one, three)
    p.load_images(torch.from_numpy(one).cuda())
    assert np.array_equal(p.fb_coeffs(0, 0, 7).cpu().numpy(), fb_pix)


@pytest.mark.parametrize("name,ni,nj", [("tiny", 4, 4), ("c2", 5, 12)])
def test_pixels_to_bests_vs_oracle(pkg, name, ni, nj):
    """Pixel images and templates -> ftk_align: landscapes / bests vs the oracle FTK on the oracle's
    trapezoid-sum polar samples of the same pixels (planted images: the truth is recovered)."""
    cfg = synth.config(name)
    p = make(pkg, cfg)
    k, w = p.radial()
    imgs, _ = synth.draw_pixel_items(cfg, "images", range(ni), mode="planted")
    tpls, _ = synth.draw_pixel_items(cfg, "templates", range(nj))
    p.load_images_pixels(torch.from_numpy(imgs).cuda())
    p.load_templates_pixels(tpls)          # host input
    res = p.align(landscape=True)
    torch.cuda.synchronize()
    oplan = ks.build_plan(cfg.n, cfg.K, synth.delta_max(cfg), synth.shift_list(cfg), cfg.eps, cfg.n_k, cfg.n_psi,
                          n_nodes=96)
    A = pixels.polar_from_pixels(imgs, k, cfg.n_psi)
    B = pixels.polar_from_pixels(tpls, k, cfg.n_psi)
    X = np.real(ftk.ftk_landscapes(fb.fb_coeffs(A), fb.fb_coeffs(B), oplan))
    na, nb = fb.discrete_norm(A, w), fb.discrete_norm(B, w)
    L = res["landscape"].cpu().numpy()
    err = np.abs(L - X) / (na[:, None, None, None] * nb[None, :, None, None])
    assert err.max() <= TOL, err.max()
    best = pkg.best_to_numpy(res["best"])
    v, j, t, r, gap = ftk.best_per_image(X)
    for i in range(ni):
        assert abs(best["value"][i] - v[i]) <= TOL * na[i] * nb[j[i]]
        if gap[i] > 2 * TOL * na[i] * nb[j[i]]:
            assert (best["template_idx"][i], best["shift_idx"][i], best["rot_idx"][i]) == (j[i], t[i], r[i])


def test_pixel_template_shards(pkg):
    """world = 2: rank 1 keeps templates [N/2, N) of a pixel load; its FB coefficients equal those of the
    single-rank load bit for bit."""
    cfg = synth.config("c2")
    tpls, _ = synth.draw_pixel_items(cfg, "templates", range(9))
    p1 = make(pkg, cfg)
    p1.load_templates_pixels(tpls)
    pr = make(pkg, cfg, rank=1, world=2)
    pr.load_templates_pixels(torch.from_numpy(tpls).cuda())
    off, nl = pr.info["template_offset"], pr.info["n_templates_local"]
    assert (off, nl) == (4, 5)
    assert np.array_equal(pr.fb_coeffs(1, 0, nl).cpu().numpy(), p1.fb_coeffs(1, off, nl).cpu().numpy())


def test_pixel_errors(pkg):
    import ctypes as C
    cfg = synth.config("tiny")
    p = make(pkg, cfg)
    pix, _ = synth.draw_pixel_items(cfg, "images", range(2))
    L = pkg.lib()
    host_out = np.zeros((2, cfg.n_k, cfg.n_psi), dtype=np.complex64)
    st = L.ftk_polar_from_pixels(p._p, C.c_void_p(pix.ctypes.data), 2, 0, C.c_void_p(host_out.ctypes.data), None)
    assert st == 1                                               # FTK_EINVAL: out must be a device pointer
    assert L.ftk_polar_from_pixels(p._p, None, 2, 0, None, None) == 1
    assert L.ftk_load_images_pixels(p._p, C.c_void_p(pix.ctypes.data), 0, 0, None) == 1
    with pytest.raises(AssertionError):
        p.polar_from_pixels(np.zeros((2, cfg.n, cfg.n + 1), dtype=np.float32))
