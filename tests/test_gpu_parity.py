"""GPU parity: the CUDA path (through the C ABI) against the float64 CPU oracle.

Tolerance (north star): |X_gpu - X_oracle| <= 1e-4 ||A|| ||B|| per inner product, with ||.|| the
discrete bandlimited norm; argmax identical unless the oracle's top-2 gap is within that tolerance.
"""
import math

import numpy as np
import pytest

import synth
from oracle import brute, fb, ftk, kernel_svd as ks

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 1e-4


@pytest.fixture(scope="module")
def pkg():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__ as g
    g.build()
    import paper_1905_12317_b200 as p
    return p


ENGINES = [0, 1]
_OPLANS = {}


def oracle_plan(cfg):
    if cfg.name not in _OPLANS:
        _OPLANS[cfg.name] = ks.build_plan(cfg.n, cfg.K, synth.delta_max(cfg), synth.shift_list(cfg), cfg.eps,
                                          cfg.n_k, cfg.n_psi, n_nodes=96)
    return _OPLANS[cfg.name]


def make(pkg, cfg, engine, **kw):
    return pkg.FTKPlan(cfg.n, cfg.K, synth.delta_max(cfg), synth.shift_list(cfg), cfg.eps, n_k=cfg.n_k,
                       n_psi=cfg.n_psi, device=0, engine=engine, **kw)


def check_best(best, X, na, nb, j_offset=0):
    v, j, t, r, gap = ftk.best_per_image(X)
    for i in range(X.shape[0]):
        tol = TOL * na[i] * nb[j[i]]
        assert abs(best["value"][i] - v[i]) <= tol, (i, best["value"][i], v[i])
        if gap[i] > 2 * tol:
            assert (best["template_idx"][i], best["shift_idx"][i], best["rot_idx"][i]) == (j[i] + j_offset, t[i], r[i])
        # R25: inside the gap rule the GPU's location must still be a near-maximum of the oracle landscape
        xg = np.real(X[i, best["template_idx"][i] - j_offset, best["shift_idx"][i], best["rot_idx"][i]])
        assert xg >= v[i] - 2 * tol, (i, xg, v[i])


@pytest.mark.parametrize("engine", ENGINES)
def test_fb_coeffs_parity(pkg, engine):
    cfg = synth.config("c2")
    p = make(pkg, cfg, engine)
    k, w = p.radial()
    x, _ = synth.draw_items(cfg, "templates", range(5), k)
    p.load_images(torch.from_numpy(x).cuda())
    got = p.fb_coeffs(0, 0, 5).cpu().numpy()
    ref = fb.fb_coeffs(x)
    assert np.max(np.abs(got - ref)) < 2e-6 * np.max(np.abs(ref))


@pytest.mark.parametrize("engine", ENGINES)
def test_tiny_full_landscape(pkg, engine):
    cfg = synth.config("tiny")
    p = make(pkg, cfg, engine)
    k, w = p.radial()
    imgs, _ = synth.draw_items(cfg, "images", range(4), k, "planted")
    tpls, _ = synth.draw_items(cfg, "templates", range(4), k)
    p.load_images(torch.from_numpy(imgs).cuda())
    p.load_templates(torch.from_numpy(tpls).cuda())
    res = p.align(pair_best=True, landscape=True)
    torch.cuda.synchronize()
    X = np.real(ftk.ftk_landscapes(fb.fb_coeffs(imgs), fb.fb_coeffs(tpls), oracle_plan(cfg)))
    na, nb = fb.discrete_norm(imgs, w), fb.discrete_norm(tpls, w)
    L = res["landscape"].cpu().numpy()
    err = np.abs(L - X) / (na[:, None, None, None] * nb[None, :, None, None])
    assert err.max() <= TOL
    best = pkg.best_to_numpy(res["best"])
    check_best(best, X, na, nb)
    # planted truth recovered
    sh = synth.shift_list(cfg)
    for i in range(4):
        j0, t0, r0 = synth.planted_truth(cfg, i, len(sh))
        assert best["template_idx"][i] == j0 and np.allclose(sh[best["shift_idx"][i]], -sh[t0])
        assert best["rot_idx"][i] == (-r0) % cfg.n_psi
    # per-pair maxima agree with the landscape
    pb = pkg.best_to_numpy(res["pair_best"].reshape(-1, 4)).reshape(4, 4)
    for i in range(4):
        for j in range(4):
            assert abs(pb["value"][i, j] - L[i, j].max()) <= 1e-6 * abs(L[i, j]).max()


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("name,ni,nj", [("c2", 6, 40), ("c3", 3, 20)])
def test_config_subsets_vs_oracle(pkg, engine, name, ni, nj):
    """Ragged, several-tile subsets: per-image bests against the oracle's full landscapes."""
    cfg = synth.config(name)
    p = make(pkg, cfg, engine)
    k, w = p.radial()
    imgs, _ = synth.draw_items(cfg, "images", range(ni), k)
    tpls, _ = synth.draw_items(cfg, "templates", range(nj), k)
    p.load_images(torch.from_numpy(imgs).cuda())
    p.load_templates(torch.from_numpy(tpls).cuda())
    best = pkg.best_to_numpy(p.align()["best"])
    X = np.real(ftk.ftk_landscapes(fb.fb_coeffs(imgs), fb.fb_coeffs(tpls), oracle_plan(cfg)))
    check_best(best, X, fb.discrete_norm(imgs, w), fb.discrete_norm(tpls, w))
    # sampled landscapes through ftk_landscape_pairs
    ii, jj = np.array([0, ni - 1, 1]), np.array([nj - 1, 0, 7])
    Lp = p.landscape_pairs(ii, jj).cpu().numpy()
    na, nb = fb.discrete_norm(imgs, w), fb.discrete_norm(tpls, w)
    for n in range(3):
        assert np.max(np.abs(Lp[n] - X[ii[n], jj[n]])) <= TOL * na[ii[n]] * nb[jj[n]]


@pytest.mark.parametrize("engine", ENGINES)
def test_zero_shift_only_and_single_pair(pkg, engine):
    """N_t = 1 (delta = 0) and N_im = N_tm = 1: the rotational correlation (degenerate case)."""
    cfg = synth.config("c2")
    p = pkg.FTKPlan(cfg.n, cfg.K, 2.0, np.zeros((1, 2)), cfg.eps, n_k=cfg.n_k, n_psi=cfg.n_psi, device=0, engine=engine)
    k, w = p.radial()
    x, _ = synth.draw_items(cfg, "images", [3], k)
    y, _ = synth.draw_items(cfg, "templates", [4], k)
    p.load_images(torch.from_numpy(x).cuda())
    p.load_templates(torch.from_numpy(y).cuda())
    L = p.align(landscape=True)["landscape"].cpu().numpy()[0, 0, 0]
    a, b = fb.fb_coeffs(x)[0], fb.fb_coeffs(y)[0]
    q = np.arange(cfg.n_psi)
    ref = np.array([np.real(2 * math.pi * np.sum(w[:, None] * a * np.conj(b) * np.exp(-2j * math.pi * q * r / cfg.n_psi)))
                    for r in range(cfg.n_psi)])
    na, nb = fb.discrete_norm(x, w)[0], fb.discrete_norm(y, w)[0]
    # FTK at delta=0 equals the rotational correlation up to the kernel truncation (<= 4 eps) and fp32
    assert np.max(np.abs(L - ref)) <= 4 * cfg.eps * na * nb


@pytest.mark.parametrize("engine", ENGINES)
def test_host_buffers_and_sharding(pkg, engine):
    """Host-pointer loads and host best output; world=2 shards on one GPU (run one after the other)
    merged with ftk_merge_bests equal the world=1 result exactly; a rank without templates reports -1."""
    cfg = synth.config("c2")
    ni, nj = 5, 9
    p1 = make(pkg, cfg, engine)
    k, w = p1.radial()
    imgs, _ = synth.draw_items(cfg, "images", range(ni), k)
    tpls, _ = synth.draw_items(cfg, "templates", range(nj), k)
    p1.load_images(imgs)                 # host numpy -> H2D inside the call
    p1.load_templates(tpls)
    b1 = p1.align_host()
    recs = []
    for rank in range(2):
        pr = make(pkg, cfg, engine, rank=rank, world=2)
        pr.load_images(torch.from_numpy(imgs).cuda())
        pr.load_templates(torch.from_numpy(tpls).cuda())
        assert pr.info["template_offset"] == (0 if rank == 0 else nj // 2)
        recs.append(pr.align()["best"])
    merged = pkg.merge_bests(torch.cat(recs), 2, ni)
    m = pkg.best_to_numpy(merged)
    assert np.array_equal(m.view(np.int32), b1.view(np.int32))
    # more ranks than templates: rank 3 of 4 with 2 templates owns none
    pe = make(pkg, cfg, engine, rank=0, world=4)
    pe.load_images(torch.from_numpy(imgs).cuda())
    pe.load_templates(torch.from_numpy(tpls[:2]).cuda())
    e = pkg.best_to_numpy(pe.align()["best"])
    assert np.all(e["template_idx"] == -1) and np.all(np.isneginf(e["value"]))


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("name", ["c3", "c4", "c5"])
def test_full_size_sampled(pkg, engine, name):
    """BASELINE.json full sizes in the bench launch configuration: sampled landscapes vs the oracle and
    the exhaustive cross-template argmax property best[i] = max_j pair_best[i, j]."""
    if engine == 1 and name == "c5":
        pytest.skip("SIMT reference engine is too slow for the full c5 sweep")
    cfg = synth.config(name)
    p = make(pkg, cfg, engine)
    k, w = p.radial()
    ni, nj = (cfg.N_im, cfg.N_tm) if name != "c5" else (256, 4096)
    imgs, pim = synth.draw_items(cfg, "images", range(ni), k, backend="torch", device="cuda")
    tpls, ptm = synth.draw_items(cfg, "templates", range(nj), k, backend="torch", device="cuda")
    p.load_images(imgs)
    p.load_templates(tpls)
    res = p.align(pair_best=True)
    torch.cuda.synchronize()
    best = pkg.best_to_numpy(res["best"])
    pb = pkg.best_to_numpy(res["pair_best"].reshape(-1, 4)).reshape(ni, nj)
    # exhaustive: per-image best is the lexicographic max over the per-pair maxima
    jb = np.argmax(pb["value"], axis=1)
    assert np.array_equal(best["value"], pb["value"][np.arange(ni), jb])
    assert np.array_equal(best["template_idx"], jb)
    # sampled pairs vs oracle landscapes
    rng = np.random.default_rng(11)
    ii = rng.integers(0, ni, 3)
    jj = rng.integers(0, nj, 3)
    ii[0], jj[0] = 0, int(jb[0])
    Lp = p.landscape_pairs(ii, jj).cpu().numpy()
    xs = imgs[torch.as_tensor(ii, device="cuda")].cpu().numpy()
    ys = tpls[torch.as_tensor(jj, device="cuda")].cpu().numpy()
    X = np.real(ftk.ftk_landscapes(fb.fb_coeffs(xs), fb.fb_coeffs(ys), oracle_plan(cfg)))
    na, nb = fb.discrete_norm(xs, w), fb.discrete_norm(ys, w)
    for n in range(3):
        assert np.max(np.abs(Lp[n] - X[n, n])) <= TOL * na[n] * nb[n]
        assert abs(pb["value"][ii[n], jj[n]] - X[n, n].max()) <= TOL * na[n] * nb[n]


def test_tc_selftest(pkg):
    """One 128x64x32 bf16 tcgen05.mma with A from TMEM and one with A from SMEM vs a host reference:
    validates the descriptor / TMEM-layout assumptions the tensor-core kernels rely on."""
    import ctypes as C
    ets, ess = C.c_double(-1), C.c_double(-1)
    st = pkg.lib().ftk_tc_selftest(0, C.byref(ets), C.byref(ess))
    assert st == 0
    assert ets.value < 1e-4 and ess.value < 1e-4, (ets.value, ess.value)


@pytest.mark.parametrize("name,mult", [("tiny", 2), ("c2", 4), ("c3", 4)])
def test_n_gamma_more_rotations(pkg, name, mult):
    """n_gamma = mult * n_psi rotations (zero-padded Step 2, reading R21): full landscapes, per-image
    bests and the explicit-pair path against the oracle evaluated at the same angles."""
    cfg = synth.config(name)
    ng = mult * cfg.n_psi
    p = make(pkg, cfg, 0, n_gamma=ng)
    assert p.info["n_gamma"] == ng
    k, w = p.radial()
    imgs, _ = synth.draw_items(cfg, "images", range(3), k)
    tpls, _ = synth.draw_items(cfg, "templates", range(5), k)
    p.load_images(torch.from_numpy(imgs).cuda())
    p.load_templates(torch.from_numpy(tpls).cuda())
    res = p.align(landscape=True)
    torch.cuda.synchronize()
    L = res["landscape"].cpu().numpy()
    X = np.real(ftk.ftk_landscapes(fb.fb_coeffs(imgs), fb.fb_coeffs(tpls), oracle_plan(cfg), n_gamma=ng))
    assert L.shape == X.shape
    na, nb = fb.discrete_norm(imgs, w), fb.discrete_norm(tpls, w)
    err = np.max(np.abs(L - X) / (na[:, None, None, None] * nb[None, :, None, None]))
    assert err <= TOL, err
    check_best(pkg.best_to_numpy(res["best"]), X, na, nb)
    ii, jj = np.array([0, 2]), np.array([4, 1])
    Lp = p.landscape_pairs(ii, jj).cpu().numpy()
    for n in range(2):
        assert np.max(np.abs(Lp[n] - X[ii[n], jj[n]])) <= TOL * na[ii[n]] * nb[jj[n]]


def test_n_gamma_option_errors(pkg):
    cfg = synth.config("tiny")
    for ng, engine in [(96, 0), (32, 0), (2 * cfg.n_psi, 1)]:  # not a power of two; < n_psi; SIMT engine
        with pytest.raises(pkg.FTKError):
            make(pkg, cfg, engine, n_gamma=ng)



# ---------------------------------------------------------------- marginalization epilogue (NEXT-3, R22)
def _marg_check(Lg, X, na, nb, tau):
    """|L_gpu - L_oracle| <= max |dX| / tau + fp32 rounding, max |dX| <= 1e-4 ||A|| ||B|| (north star)."""
    Lo = ftk.log_marginal(X, tau)
    tol = TOL * na[:, None] * nb[None, :] / tau + 1e-5 * np.maximum(1.0, np.abs(Lo))
    err = np.abs(Lg - Lo)
    assert np.all(err <= tol), (err.max(), (err / tol).max())


@pytest.mark.parametrize("name,ni,nj,shift_filter,mult", [
    ("tiny", 4, 4, None, 1),
    ("tiny", 3, 5, "half", 1),     # shifts without a -delta partner + padding columns: the exact path
    ("tiny", 2, 3, None, 2),       # n_gamma = 2 n_psi (reading R21)
    ("c2", 6, 40, None, 1),
    ("c3", 3, 20, None, 1),
])
def test_marginal_vs_oracle(pkg, name, ni, nj, shift_filter, mult):
    cfg = synth.config(name)
    sh = synth.shift_list(cfg)
    if shift_filter == "half":
        sh = sh[sh[:, 1] >= -0.25]
    ng = mult * cfg.n_psi
    p = pkg.FTKPlan(cfg.n, cfg.K, synth.delta_max(cfg), sh, cfg.eps, n_k=cfg.n_k, n_psi=cfg.n_psi, device=0,
                    n_gamma=ng if mult > 1 else 0)
    k, w = p.radial()
    imgs, _ = synth.draw_items(cfg, "images", range(ni), k)
    tpls, _ = synth.draw_items(cfg, "templates", range(nj), k)
    p.load_images(torch.from_numpy(imgs).cuda())
    p.load_templates(torch.from_numpy(tpls).cuda())
    oplan = ks.build_plan(cfg.n, cfg.K, synth.delta_max(cfg), sh, cfg.eps, cfg.n_k, cfg.n_psi, n_nodes=96) \
        if shift_filter else oracle_plan(cfg)
    X = np.real(ftk.ftk_landscapes(fb.fb_coeffs(imgs), fb.fb_coeffs(tpls), oplan, n_gamma=ng))
    na, nb = fb.discrete_norm(imgs, w), fb.discrete_norm(tpls, w)
    scale = float(np.median(na[:, None] * nb[None, :]))
    for f in (0.01, 0.1, 1.0):
        tau = f * scale
        Lg = p.align_marginal(tau).cpu().numpy()
        assert Lg.shape == (ni, nj)
        _marg_check(Lg, X, na, nb, tau)
    # the max / argmax epilogue is unaffected by a preceding marginal call
    check_best(pkg.best_to_numpy(p.align()["best"]), X, na, nb)


@pytest.mark.parametrize("name,ni,nj", [("c5", 256, 512), ("c4", 96, 160)])
def test_marginal_full_size_sampled(pkg, name, ni, nj):
    """c5 sizes (256 images x 512 templates, the bench's Step-3 launch shape) and c4 (3209 shifts: several
    Step-3 rep-groups, whose per-group partials are merged by a finalize kernel): sampled pairs vs the oracle."""
    cfg = synth.config(name)
    p = make(pkg, cfg, 0)
    k, w = p.radial()
    if name == "c4":
        assert p.info["s3_groups"] > 1
    imgs, _ = synth.draw_items(cfg, "images", range(ni), k, backend="torch", device="cuda")
    tpls, _ = synth.draw_items(cfg, "templates", range(nj), k, backend="torch", device="cuda")
    p.load_images(imgs)
    p.load_templates(tpls)
    ii, jj = np.array([0, ni - 1, 17]), np.array([nj - 1, 0, 100])
    xs = imgs[torch.as_tensor(ii, device="cuda")].cpu().numpy()
    ys = tpls[torch.as_tensor(jj, device="cuda")].cpu().numpy()
    na, nb = fb.discrete_norm(xs, w), fb.discrete_norm(ys, w)
    tau = 0.05 * float(np.median(na * nb))
    Lg = p.align_marginal(tau).cpu().numpy()
    assert np.all(np.isfinite(Lg))
    X = np.real(ftk.ftk_landscapes(fb.fb_coeffs(xs), fb.fb_coeffs(ys), oracle_plan(cfg)))
    for n in range(3):
        Lo = ftk.log_marginal(X[n, n], tau)
        assert abs(Lg[ii[n], jj[n]] - Lo) <= TOL * na[n] * nb[n] / tau + 1e-5 * max(1.0, abs(Lo))


def test_marginal_errors(pkg):
    cfg = synth.config("tiny")
    p = make(pkg, cfg, 0)
    k, _ = p.radial()
    x, _ = synth.draw_items(cfg, "images", range(2), k)
    with pytest.raises(pkg.FTKError):          # before the loads
        p.align_marginal(1.0)
    p.load_images(torch.from_numpy(x).cuda())
    p.load_templates(torch.from_numpy(x).cuda())
    for bad in (0.0, -1.0, float("inf"), float("nan")):
        with pytest.raises(pkg.FTKError):
            p.align_marginal(bad)
    ps = make(pkg, cfg, 1)
    ps.load_images(torch.from_numpy(x).cuda())
    ps.load_templates(torch.from_numpy(x).cuda())
    with pytest.raises(pkg.FTKError):          # SIMT engine: max / argmax only
        ps.align_marginal(1.0)


@pytest.mark.parametrize("engine", ENGINES)
def test_small_workspace_many_blocks(pkg, engine):
    """A 16 MB workspace at c3 forces one-template pair blocks over ragged 128-image tiles (140 = 128 + 12):
    per-image bests and per-pair maxima still match the oracle."""
    cfg = synth.config("c3")
    p = make(pkg, cfg, engine, workspace_bytes=16 << 20)
    k, w = p.radial()
    ni, nj = 140, 6
    imgs, _ = synth.draw_items(cfg, "images", range(ni), k)
    tpls, _ = synth.draw_items(cfg, "templates", range(nj), k)
    p.load_images(torch.from_numpy(imgs).cuda())
    p.load_templates(torch.from_numpy(tpls).cuda())
    res = p.align(pair_best=True)
    torch.cuda.synchronize()
    X = np.real(ftk.ftk_landscapes(fb.fb_coeffs(imgs), fb.fb_coeffs(tpls), oracle_plan(cfg)))
    na, nb = fb.discrete_norm(imgs, w), fb.discrete_norm(tpls, w)
    check_best(pkg.best_to_numpy(res["best"]), X, na, nb)
    pb = pkg.best_to_numpy(res["pair_best"].reshape(-1, 4)).reshape(ni, nj)
    assert np.all(np.abs(pb["value"] - X.max(axis=(2, 3))) <= TOL * na[:, None] * nb[None, :])
