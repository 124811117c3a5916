"""GPU parity of the CTF-parameterized factorized kernel (Sec. 6
P:1389-1403; DESIGN reading R24) through the C ABI (ftk_plan_create_ctf) against oracle.ctf.

Tolerance: the north star's |X_gpu - X_oracle| <= 1e-4 ||A|| ||B|| per inner product on the virtual shift
list v = tau * N_t + t (the filters satisfy |c| <= 1, so ||c B|| <= ||B||).  Filter values are computed
from the same input generator (synth.ctf_filters) on each side's own radial nodes.
"""
import numpy as np
import pytest

import synth
from oracle import ctf, fb, ftk
from oracle.quadrature import radial_rule as oracle_radial_rule

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 1e-4
DEF4 = [8000.0, 15000.0, 22000.0, 30000.0]
DEF2 = [10000.0, 20000.0]


@pytest.fixture(scope="module")
def pkg():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__ as g
    g.build()
    import paper_1905_12317_b200 as p
    return p


def _plans(pkg, cfg, defoci, engine, sh=None, **kw):
    sh = synth.shift_list(cfg) if sh is None else sh
    k, _ = pkg.radial_rule(cfg.n, cfg.K, cfg.n_k, 0)
    p = pkg.FTKPlan(cfg.n, cfg.K, synth.delta_max(cfg), sh, cfg.eps, n_k=cfg.n_k, n_psi=cfg.n_psi, device=0,
                    engine=engine, filters=synth.ctf_filters(k, defoci), **kw)
    ko, _ = oracle_radial_rule(cfg.n_k, cfg.k_max)
    op = ctf.build_plan_ctf(cfg.n, cfg.K, synth.delta_max(cfg), sh, cfg.eps, cfg.n_k, cfg.n_psi,
                            synth.ctf_filters(ko, defoci), n_nodes=96)
    return p, op


def _check_best(best, X, na, nb):
    v, j, t, r, gap = ftk.best_per_image(X)
    for i in range(X.shape[0]):
        tol = TOL * na[i] * nb[j[i]]
        assert abs(best["value"][i] - v[i]) <= tol, (i, best["value"][i], v[i])
        if gap[i] > 2 * tol:
            assert (best["template_idx"][i], best["shift_idx"][i], best["rot_idx"][i]) == (j[i], t[i], r[i])
        # R25: a location chosen inside the gap rule is still a near-maximum of the oracle landscape
        xg = np.real(X[i, best["template_idx"][i], best["shift_idx"][i], best["rot_idx"][i]])
        assert xg >= v[i] - 2 * tol, (i, xg, v[i])


@pytest.mark.parametrize("engine", [0, 1])
def test_ctf_tiny_full_landscape(pkg, engine):
    cfg = synth.config("tiny")
    p, op = _plans(pkg, cfg, DEF4, engine)
    assert p.info["H"] == op.H and p.info["N_t"] == 4 * p.info["N_t_base"]
    k, w = p.radial()
    imgs, _ = synth.draw_items(cfg, "images", range(4), k, "planted")
    tpls, _ = synth.draw_items(cfg, "templates", range(4), k)
    p.load_images(torch.from_numpy(imgs).cuda())
    p.load_templates(torch.from_numpy(tpls).cuda())
    res = p.align(pair_best=True, landscape=True)
    torch.cuda.synchronize()
    X = np.real(ftk.ftk_landscapes(fb.fb_coeffs(imgs), fb.fb_coeffs(tpls), op))
    na, nb = fb.discrete_norm(imgs, w), fb.discrete_norm(tpls, w)
    L = res["landscape"].cpu().numpy()
    assert L.shape == X.shape
    err = np.abs(L - X) / (na[:, None, None, None] * nb[None, :, None, None])
    assert err.max() <= TOL
    _check_best(pkg.best_to_numpy(res["best"]), X, na, nb)


@pytest.mark.parametrize("engine", [0, 1])
@pytest.mark.parametrize("name,defoci,ni,nj", [("c2", DEF4, 6, 40), ("c3", DEF2, 3, 20)])
def test_ctf_config_subsets(pkg, engine, name, defoci, ni, nj):
    """Ragged several-tile subsets; c2 x 4 defoci is the widest Step-3 contraction the tensor-core engine
    takes (K3p = 128)."""
    cfg = synth.config(name)
    p, op = _plans(pkg, cfg, defoci, engine)
    k, w = p.radial()
    imgs, _ = synth.draw_items(cfg, "images", range(ni), k)
    tpls, _ = synth.draw_items(cfg, "templates", range(nj), k)
    p.load_images(torch.from_numpy(imgs).cuda())
    p.load_templates(torch.from_numpy(tpls).cuda())
    best = pkg.best_to_numpy(p.align()["best"])
    X = np.real(ftk.ftk_landscapes(fb.fb_coeffs(imgs), fb.fb_coeffs(tpls), op))
    na, nb = fb.discrete_norm(imgs, w), fb.discrete_norm(tpls, w)
    _check_best(best, X, na, nb)
    ii, jj = np.array([0, ni - 1]), np.array([nj - 1, 3])
    Lp = p.landscape_pairs(ii, jj).cpu().numpy()
    for n in range(2):
        assert np.max(np.abs(Lp[n] - X[ii[n], jj[n]])) <= TOL * na[ii[n]] * nb[jj[n]]


def test_ctf_marginal(pkg):
    """Marginalization (reading R22) over shifts, rotations and defocus on a CTF plan."""
    cfg = synth.config("c2")
    p, op = _plans(pkg, cfg, DEF2, 0)
    k, w = p.radial()
    imgs, _ = synth.draw_items(cfg, "images", range(5), k)
    tpls, _ = synth.draw_items(cfg, "templates", range(12), k)
    p.load_images(torch.from_numpy(imgs).cuda())
    p.load_templates(torch.from_numpy(tpls).cuda())
    X = np.real(ftk.ftk_landscapes(fb.fb_coeffs(imgs), fb.fb_coeffs(tpls), op))
    na, nb = fb.discrete_norm(imgs, w), fb.discrete_norm(tpls, w)
    tau = 0.1 * float(np.median(na[:, None] * nb[None, :]))
    Lg = p.align_marginal(tau).cpu().numpy()
    Lo = ftk.log_marginal(X, tau)
    tol = TOL * na[:, None] * nb[None, :] / tau + 1e-5 * np.maximum(1.0, np.abs(Lo))
    assert np.all(np.abs(Lg - Lo) <= tol)


def test_ctf_width_limit(pkg):
    """c5 x 4 defoci needs K3p = 288 > 224: the tensor-core engine refuses (FTK_EINVAL)."""
    cfg = synth.config("c5")
    k, _ = pkg.radial_rule(cfg.n, cfg.K, cfg.n_k, 0)
    f = synth.ctf_filters(k, DEF4)
    with pytest.raises(pkg.FTKError) as e:
        pkg.FTKPlan(cfg.n, cfg.K, synth.delta_max(cfg), synth.shift_list(cfg), cfg.eps, n_k=cfg.n_k,
                    n_psi=cfg.n_psi, device=0, engine=0, filters=f)
    assert e.value.status == 1


@pytest.mark.parametrize("engine", [0, 1])
@pytest.mark.parametrize("name,defoci,ni,nj", [("c3", DEF4, 3, 7), ("c5", DEF2, 2, 3)])
def test_ctf_wide_step3(pkg, engine, name, defoci, ni, nj):
    """Contractions wider than 128 (c3 x 4 defoci: K3p = 224, Step-3 chunks of N = 16; c5 x 2: K3p = 160,
    N = 32) on both engines vs the oracle, with sampled landscapes."""
    cfg = synth.config(name)
    p, op = _plans(pkg, cfg, defoci, engine)
    assert p.info["K3p"] > 128
    k, w = p.radial()
    imgs, _ = synth.draw_items(cfg, "images", range(ni), k)
    tpls, _ = synth.draw_items(cfg, "templates", range(nj), k)
    p.load_images(torch.from_numpy(imgs).cuda())
    p.load_templates(torch.from_numpy(tpls).cuda())
    X = np.real(ftk.ftk_landscapes(fb.fb_coeffs(imgs), fb.fb_coeffs(tpls), op))
    na, nb = fb.discrete_norm(imgs, w), fb.discrete_norm(tpls, w)
    _check_best(pkg.best_to_numpy(p.align()["best"]), X, na, nb)
    ii, jj = np.array([0, ni - 1]), np.array([nj - 1, 0])
    Lp = p.landscape_pairs(ii, jj).cpu().numpy()
    for n in range(2):
        assert np.max(np.abs(Lp[n] - X[ii[n], jj[n]])) <= TOL * na[ii[n]] * nb[jj[n]]


def test_ctf_n_gamma_and_sharding(pkg):
    """CTF plan with n_gamma = 2 n_psi (reading R21) vs the oracle at the same angles, and 2 template shards
    (run one after the other on one GPU) merged with ftk_merge_bests equal to the 1-rank result bitwise."""
    cfg = synth.config("tiny")
    ng = 2 * cfg.n_psi
    p, op = _plans(pkg, cfg, DEF2, 0, n_gamma=ng)
    k, w = p.radial()
    imgs, _ = synth.draw_items(cfg, "images", range(3), k)
    tpls, _ = synth.draw_items(cfg, "templates", range(4), k)
    p.load_images(torch.from_numpy(imgs).cuda())
    p.load_templates(torch.from_numpy(tpls).cuda())
    res = p.align(landscape=True)
    X = np.real(ftk.ftk_landscapes(fb.fb_coeffs(imgs), fb.fb_coeffs(tpls), op, n_gamma=ng))
    na, nb = fb.discrete_norm(imgs, w), fb.discrete_norm(tpls, w)
    L = res["landscape"].cpu().numpy()
    assert L.shape == X.shape
    assert np.max(np.abs(L - X) / (na[:, None, None, None] * nb[None, :, None, None])) <= TOL
    _check_best(pkg.best_to_numpy(res["best"]), X, na, nb)
    b1 = pkg.best_to_numpy(res["best"])
    recs = []
    for rank in range(2):
        pr, _ = _plans(pkg, cfg, DEF2, 0, n_gamma=ng, rank=rank, world=2)
        pr.load_images(torch.from_numpy(imgs).cuda())
        pr.load_templates(torch.from_numpy(tpls).cuda())
        recs.append(pr.align()["best"])
    m = pkg.best_to_numpy(pkg.merge_bests(torch.cat(recs), 2, 3))
    assert np.array_equal(m.view(np.int32), b1.view(np.int32))


def test_ctf_wide_marginal(pkg):
    """Marginalization epilogue (MODE 1) with the narrow Step-3 chunks of a wide CTF plan (c3 x 4 defoci,
    K3p = 224, N = 16)."""
    cfg = synth.config("c3")
    p, op = _plans(pkg, cfg, DEF4, 0)
    assert p.info["K3p"] > 128
    k, w = p.radial()
    imgs, _ = synth.draw_items(cfg, "images", range(3), k)
    tpls, _ = synth.draw_items(cfg, "templates", range(5), k)
    p.load_images(torch.from_numpy(imgs).cuda())
    p.load_templates(torch.from_numpy(tpls).cuda())
    X = np.real(ftk.ftk_landscapes(fb.fb_coeffs(imgs), fb.fb_coeffs(tpls), op))
    na, nb = fb.discrete_norm(imgs, w), fb.discrete_norm(tpls, w)
    for f in (0.02, 0.5):
        tau = f * float(np.median(na[:, None] * nb[None, :]))
        Lg = p.align_marginal(tau).cpu().numpy()
        Lo = ftk.log_marginal(X, tau)
        tol = TOL * na[:, None] * nb[None, :] / tau + 1e-5 * np.maximum(1.0, np.abs(Lo))
        assert np.all(np.abs(Lg - Lo) <= tol)
