"""GPU parity of the PRODUCTION path (tensor-core engine, the kernels and block shapes bench.py times)
against the float64 oracle, at BASELINE.json's full sizes (SURVEY 8(d) "parity sampling"
Eq. fbk3, P:1324 consistency check).

Which kernels each test runs (engine 0):
  * test_landscape_pairs_32       k_step1_tc over each pair's 128-image tile, k_step2_fft (Form B),
                                  k_step3_tc with landscape output (exact epilogue) -- 32 random pairs per
                                  config, element-wise |dX| <= 1e-4 ||A|| ||B|| (north star) and the
                                  engine's own precision claim |dX| <= 2.5e-6 ||A|| ||B|| (DESIGN.md
                                  section 6, fp16x3: emulated worst case 3.9e-7 at tiny).
  * test_pair_best_every_pair     ftk_align as bench.py runs it (k_step1_tc, k_step2_fft, k_step3_tc with the
                                  fast E + |O| epilogue and the resolver): value AND (shift, rot) of every
                                  pair of a >= 2-image-tile subset vs the oracle (argmax: gap rule).
  * test_image_bests_all_templates  per-image bests over ALL templates of the config (4 images at c3/c4,
                                  1 image at c5) vs the oracle.
  * test_bench_block_shape        c5 with 2100 images: one 2048-image Step-1 block (16 image tiles, the
                                  bench's block) plus a ragged one; sampled pair maxima vs the oracle.
  * test_nccl_single_rank         ftk_align with a 1-rank NCCL communicator (the library's all-gather +
                                  device merge): bests equal the oracle's and, bitwise, the plain call.
  * test_poisoned_onchip_state_and_workspace  FTK_POISON: workspace, shared memory and TMEM filled with
                                  0x7B / 0xFF before every block / launch; results bitwise equal (the
                                  initcheck / racecheck stand-in: compute-sanitizer is closed on the pool).
  * test_step2_tensor_core_all_sizes  k_step2_tc<R> (the default Step 2 at n = 512) forced at c2 / c3 / c4
                                  and at c5: sampled landscapes and every pair's max + argmax vs the oracle.
Argmax rule (reading R25): GPU and oracle argmax must agree unless the oracle's top-2 gap is
within 2 x the tolerance (each side may be off by one tolerance).
Set FTK_PARITY_LOG=path to write the max |dX| / (||A|| ||B||) per config as JSON.
"""
import json
import os

import numpy as np
import pytest

import synth
from oracle import fb, ftk, kernel_svd as ks

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 1e-4
PREC = 2.5e-6  # fp16x3 precision bar, 40x inside the north-star tolerance
_OPLANS = {}
_STATS = {}


@pytest.fixture(scope="module")
def pkg():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__ as g
    g.build()
    import paper_1905_12317_b200 as p
    return p


@pytest.fixture(scope="module", autouse=True)
def parity_log():
    yield
    path = os.environ.get("FTK_PARITY_LOG")
    if path and _STATS:
        with open(path, "w") as f:
            json.dump(_STATS, f, indent=1, sort_keys=True)


def note(key, val):
    _STATS[key] = max(float(val), _STATS.get(key, 0.0))


def oracle_plan(cfg):
    if cfg.name not in _OPLANS:
        _OPLANS[cfg.name] = ks.build_plan(cfg.n, cfg.K, synth.delta_max(cfg), synth.shift_list(cfg), cfg.eps,
                                          cfg.n_k, cfg.n_psi, n_nodes=96)
    return _OPLANS[cfg.name]


def make(pkg, cfg, **kw):
    return pkg.FTKPlan(cfg.n, cfg.K, synth.delta_max(cfg), synth.shift_list(cfg), cfg.eps, n_k=cfg.n_k,
                       n_psi=cfg.n_psi, device=0, engine=0, **kw)


def load_gpu(pkg, cfg, ni, nj, **kw):
    p = make(pkg, cfg, **kw)
    k, w = p.radial()
    imgs, _ = synth.draw_items(cfg, "images", range(ni), k, backend="torch", device="cuda")
    tpls, _ = synth.draw_items(cfg, "templates", range(nj), k, backend="torch", device="cuda")
    p.load_images(imgs)
    p.load_templates(tpls)
    return p, w, imgs, tpls


def pair_stats(X):
    """Per pair of X [I, J, N_t, n]: (max, t, r, top-2 gap); argmax ties -> smallest (t, r)."""
    I, J = X.shape[:2]
    flat = X.reshape(I, J, -1)
    idx = np.argmax(flat, axis=2)
    v = np.take_along_axis(flat, idx[..., None], 2)[..., 0]
    part = np.partition(flat, -2, axis=2)
    gap = part[..., -1] - part[..., -2]
    t, r = np.unravel_index(idx, X.shape[2:])
    return v, t, r, gap


@pytest.mark.parametrize("name", ["tiny", "c2", "c3", "c4", "c5"])
def test_landscape_pairs_32(pkg, name):
    cfg = synth.config(name)
    ni, nj = min(cfg.N_im, 300), min(cfg.N_tm, 300)
    p, w, imgs, tpls = load_gpu(pkg, cfg, ni, nj)
    rng = np.random.default_rng(7)
    n = 32
    ii = rng.integers(0, ni, n)
    jj = rng.integers(0, nj, n)
    Lp = p.landscape_pairs(ii, jj).cpu().numpy()
    xs = imgs[torch.as_tensor(ii, device="cuda")].cpu().numpy()
    ys = tpls[torch.as_tensor(jj, device="cuda")].cpu().numpy()
    na, nb = fb.discrete_norm(xs, w), fb.discrete_norm(ys, w)
    a, b = fb.fb_coeffs(xs), fb.fb_coeffs(ys)
    worst = 0.0
    for s in range(n):
        X = np.real(ftk.ftk_landscapes(a[s:s + 1], b[s:s + 1], oracle_plan(cfg)))[0, 0]
        worst = max(worst, np.max(np.abs(Lp[s] - X)) / (na[s] * nb[s]))
    note(f"landscape_pairs_{name}", worst)
    assert worst <= TOL, worst
    assert worst <= PREC, worst


@pytest.mark.parametrize("name,ni,nj", [("c5", 130, 40), ("c4", 130, 8), ("c3", 160, 24)])
def test_pair_best_every_pair(pkg, name, ni, nj):
    """Every pair of a subset spanning 2 image tiles (128 + ragged): the fast E + |O| epilogue and the
    resolver vs the oracle's per-pair maximum and its (shift, rotation).  c4 runs several Step-3 rep-groups."""
    cfg = synth.config(name)
    p, w, imgs, tpls = load_gpu(pkg, cfg, ni, nj)
    if name == "c4":
        assert p.info["s3_groups"] > 1
    res = p.align(pair_best=True)
    torch.cuda.synchronize()
    pb = pkg.best_to_numpy(res["pair_best"].reshape(-1, 4)).reshape(ni, nj)
    xs, ys = imgs.cpu().numpy(), tpls.cpu().numpy()
    na, nb = fb.discrete_norm(xs, w), fb.discrete_norm(ys, w)
    a, b = fb.fb_coeffs(xs), fb.fb_coeffs(ys)
    worst, mism = 0.0, 0
    for i in range(ni):
        X = np.real(ftk.ftk_landscapes(a[i:i + 1], b, oracle_plan(cfg)))
        v, t, r, gap = pair_stats(X)
        tol = TOL * na[i] * nb
        dv = np.abs(pb["value"][i] - v[0])
        worst = max(worst, float(np.max(dv / (na[i] * nb))))
        assert np.all(dv <= tol), (i, dv.max())
        assert np.all(pb["template_idx"][i] == np.arange(nj))
        clear = gap[0] > 2 * tol
        ok = (pb["shift_idx"][i] == t[0]) & (pb["rot_idx"][i] == r[0])
        assert np.all(ok | ~clear), (i, np.where(~ok & clear))
        # R25: every reported location is a near-maximum of the oracle landscape of its pair
        xg = X[0, np.arange(nj), pb["shift_idx"][i], pb["rot_idx"][i]]
        assert np.all(xg >= v[0] - 2 * tol), (i, np.min(xg - v[0] + 2 * tol))
        mism += int(np.sum(~ok))
    note(f"pair_best_value_{name}", worst)
    _STATS[f"pair_best_argmax_near_tie_{name}"] = mism


@pytest.mark.parametrize("name,ni", [("c3", 4), ("c4", 4), ("c5", 1)])
def test_image_bests_all_templates(pkg, name, ni):
    """Per-image bests over ALL N_tm templates of the config (4 images at c3/c4, 1 at c5)."""
    cfg = synth.config(name)
    p, w, imgs, tpls = load_gpu(pkg, cfg, ni, cfg.N_tm)
    best = pkg.best_to_numpy(p.align()["best"])
    xs = imgs.cpu().numpy()
    a, na = fb.fb_coeffs(xs), fb.discrete_norm(xs, w)
    top = np.full((ni, 2), -np.inf)
    arg = np.zeros((ni, 3), dtype=np.int64)
    nb_all = np.empty(cfg.N_tm)
    for j0 in range(0, cfg.N_tm, 64):
        ys = tpls[j0:j0 + 64].cpu().numpy()
        nb_all[j0:j0 + len(ys)] = fb.discrete_norm(ys, w)
        X = np.real(ftk.ftk_landscapes(a, fb.fb_coeffs(ys), oracle_plan(cfg)))
        flat = X.reshape(ni, -1)
        part = np.partition(flat, -2, axis=1)[:, -2:]
        for i in range(ni):
            k = int(np.argmax(flat[i]))
            if flat[i, k] > top[i, 0]:
                top[i, 1] = max(top[i, 0], part[i, 0])
                top[i, 0] = flat[i, k]
                arg[i] = np.unravel_index(k, X.shape[1:])
                arg[i, 0] += j0
            else:
                top[i, 1] = max(top[i, 1], flat[i, k])
    for i in range(ni):
        tol = TOL * na[i] * nb_all[arg[i, 0]]
        assert abs(best["value"][i] - top[i, 0]) <= tol, (i, best["value"][i], top[i, 0])
        note(f"image_best_value_{name}", abs(best["value"][i] - top[i, 0]) / (na[i] * nb_all[arg[i, 0]]))
        if top[i, 0] - top[i, 1] > 2 * tol:
            assert (best["template_idx"][i], best["shift_idx"][i], best["rot_idx"][i]) == tuple(arg[i])


def test_bench_block_shape(pkg):
    """c5 with 2100 images x 3 templates: the first pair block is the bench's 2048-image block (16 Step-1
    image tiles per unit), the second a ragged 52-image block; 64 sampled pair maxima and their
    (shift, rot) vs the oracle, and best[i] = lexicographic max_j pair_best[i, j] for all images."""
    cfg = synth.config("c5")
    ni, nj = 2100, 3
    p, w, imgs, tpls = load_gpu(pkg, cfg, ni, nj)
    res = p.align(pair_best=True)
    torch.cuda.synchronize()
    best = pkg.best_to_numpy(res["best"])
    pb = pkg.best_to_numpy(res["pair_best"].reshape(-1, 4)).reshape(ni, nj)
    jb = np.argmax(pb["value"], axis=1)
    assert np.array_equal(best["value"], pb["value"][np.arange(ni), jb])
    rng = np.random.default_rng(5)
    ii = np.concatenate([[0, 127, 128, 2047, 2048, 2099], rng.integers(0, ni, 58)])
    ys = tpls.cpu().numpy()
    nb, b = fb.discrete_norm(ys, w), fb.fb_coeffs(ys)
    worst = 0.0
    for i in ii:
        x = imgs[int(i):int(i) + 1].cpu().numpy()
        na = fb.discrete_norm(x, w)[0]
        X = np.real(ftk.ftk_landscapes(fb.fb_coeffs(x), b, oracle_plan(cfg)))
        v, t, r, gap = pair_stats(X)
        for j in range(nj):
            tol = TOL * na * nb[j]
            assert abs(pb["value"][i, j] - v[0, j]) <= tol
            worst = max(worst, abs(pb["value"][i, j] - v[0, j]) / (na * nb[j]))
            if gap[0, j] > 2 * tol:
                assert (pb["shift_idx"][i, j], pb["rot_idx"][i, j]) == (t[0, j], r[0, j])
    note("bench_block_c5_pair_value", worst)


def test_nccl_single_rank(pkg):
    """opts.nccl_comm with a 1-rank communicator: ftk_align runs the library's ncclAllGather + device merge;
    the bests equal the oracle's and are bitwise equal to the call without a communicator."""
    cfg = synth.config("c2")
    ni, nj = 6, 40
    comm = pkg.NcclComm(1, 0, 0, pkg.NcclComm.unique_id())
    p = make(pkg, cfg, nccl_comm=comm)
    k, w = p.radial()
    imgs, _ = synth.draw_items(cfg, "images", range(ni), k)
    tpls, _ = synth.draw_items(cfg, "templates", range(nj), k)
    p.load_images(torch.from_numpy(imgs).cuda())
    p.load_templates(torch.from_numpy(tpls).cuda())
    bg = pkg.best_to_numpy(p.align()["best"])
    bh = p.align_host()                         # host output through the same gather
    q = make(pkg, cfg)
    q.load_images(torch.from_numpy(imgs).cuda())
    q.load_templates(torch.from_numpy(tpls).cuda())
    bl = pkg.best_to_numpy(q.align()["best"])
    assert np.array_equal(bg.view(np.int32), bl.view(np.int32))
    assert np.array_equal(bh.view(np.int32), bl.view(np.int32))
    X = np.real(ftk.ftk_landscapes(fb.fb_coeffs(imgs), fb.fb_coeffs(tpls), oracle_plan(cfg)))
    na, nb = fb.discrete_norm(imgs, w), fb.discrete_norm(tpls, w)
    v, j, t, r, gap = ftk.best_per_image(X)
    for i in range(ni):
        tol = TOL * na[i] * nb[j[i]]
        assert abs(bg["value"][i] - v[i]) <= tol
        if gap[i] > 2 * tol:
            assert (bg["template_idx"][i], bg["shift_idx"][i], bg["rot_idx"][i]) == (j[i], t[i], r[i])
    del p
    comm.close()
    # a communicator whose size disagrees with the plan's world is refused at plan creation
    comm2 = pkg.NcclComm(1, 0, 0, pkg.NcclComm.unique_id())
    with pytest.raises(pkg.FTKError):
        make(pkg, cfg, nccl_comm=comm2, rank=0, world=2)
    comm2.close()


def test_landscape_small_workspace(pkg):
    """landscape output with a workspace too small for a full block -- the block shape
    keeps every template in each block (or refuses with FTK_ECAPACITY); never overlapping rows."""
    cfg = synth.config("c3")
    ni, nj = 140, 6
    p = make(pkg, cfg, workspace_bytes=16 << 20)
    k, w = p.radial()
    imgs, _ = synth.draw_items(cfg, "images", range(ni), k)
    tpls, _ = synth.draw_items(cfg, "templates", range(nj), k)
    p.load_images(torch.from_numpy(imgs).cuda())
    p.load_templates(torch.from_numpy(tpls).cuda())
    try:
        L = p.align(landscape=True)["landscape"].cpu().numpy()
    except pkg.FTKError as e:
        assert e.status == 7  # FTK_ECAPACITY
        return
    X = np.real(ftk.ftk_landscapes(fb.fb_coeffs(imgs), fb.fb_coeffs(tpls), oracle_plan(cfg)))
    na, nb = fb.discrete_norm(imgs, w), fb.discrete_norm(tpls, w)
    assert np.max(np.abs(L - X) / (na[:, None, None, None] * nb[None, :, None, None])) <= TOL


def test_landscape_pairs_errors(pkg):
    import ctypes as C
    cfg = synth.config("tiny")
    p = make(pkg, cfg)
    k, _ = p.radial()
    x, _ = synth.draw_items(cfg, "images", range(3), k)
    p.load_images(torch.from_numpy(x).cuda())
    p.load_templates(torch.from_numpy(x).cuda())
    with pytest.raises(pkg.FTKError):
        p.landscape_pairs([0, 5], [0, 1])        # image index out of range
    with pytest.raises(pkg.FTKError):
        p.landscape_pairs([0], [-1])             # template index out of range
    ii = np.array([0, 1], dtype=np.int32)
    out = torch.empty((2, p.info["N_t"], p.info["n_gamma"] - 1), dtype=torch.float32, device="cuda")
    st = pkg.lib().ftk_landscape_pairs(p._p, C.c_void_p(ii.ctypes.data), C.c_void_p(ii.ctypes.data), 2,
                                       C.c_void_p(out.data_ptr()), out.numel(), None)
    assert st == 7                               # FTK_ECAPACITY: host indices accepted, buffer too small


@pytest.mark.parametrize("name,ni,nj,ws_small", [("c3", 260, 24, 16 << 20), ("c5", 140, 12, 64 << 20)])
def test_deterministic_across_runs_and_block_shapes(pkg, name, ni, nj, ws_small):
    """Race / uninitialised-memory canary (compute-sanitizer is not available on the GPU pool): the same
    inputs through the default workspace twice, and through a small workspace (one-template pair blocks
    over ragged image tiles: different grids, block shapes and workspace reuse), must give BITWISE equal
    per-image bests, per-pair maxima and log-marginals.  Every pair's arithmetic is independent of its
    block, so any difference is a race, a stale read or an out-of-bounds write."""
    cfg = synth.config(name)
    runs = []
    for ws in (0, 0, ws_small):
        p = make(pkg, cfg, workspace_bytes=ws)
        k, w = p.radial()
        imgs, _ = synth.draw_items(cfg, "images", range(ni), k, backend="torch", device="cuda")
        tpls, _ = synth.draw_items(cfg, "templates", range(nj), k, backend="torch", device="cuda")
        p.load_images(imgs)
        p.load_templates(tpls)
        res = p.align(pair_best=True)
        torch.cuda.synchronize()
        b = pkg.best_to_numpy(res["best"]).view(np.int32).copy()
        pb = pkg.best_to_numpy(res["pair_best"].reshape(-1, 4)).view(np.int32).copy()
        tau = float(np.median(fb.discrete_norm(imgs[:4].cpu().numpy(), w)) *
                    np.median(fb.discrete_norm(tpls[:4].cpu().numpy(), w))) * 0.1
        lm = p.align_marginal(tau).cpu().numpy().view(np.int32).copy()
        runs.append((b, pb, lm))
        del p
    for other in runs[1:]:
        for x, y in zip(runs[0], other):
            assert np.array_equal(x, y)


@pytest.mark.parametrize("name,ni,nj,ws", [("tiny", 4, 5, 0), ("c3", 260, 6, 0), ("c5", 140, 4, 64 << 20)])
def test_poisoned_onchip_state_and_workspace(pkg, name, ni, nj, ws):
    """initcheck / racecheck stand-in (compute-sanitizer is closed on the GPU pool): with FTK_POISON the
    library fills the pair-block workspace (Zhat', the Step-3 operand) before every block, and every SM's
    shared memory and all 512 TMEM columns before every Step 1 / 2 / 3 launch, with a byte pattern -- 0x7B
    (a large finite fp32 / fp16 value that a max cannot ignore) and 0xFF (NaN).  Per-image bests, per-pair
    maxima, landscapes of explicit pairs and log-marginals must be BITWISE equal to the unpoisoned run: a
    read of shared memory, TMEM or workspace that the same launch did not write first (a missing
    accumulate reset, a stale pipeline stage, a hand-off race) would change them."""
    cfg = synth.config(name)
    rng = np.random.default_rng(7)
    ii = rng.integers(0, ni, 6)
    jj = rng.integers(0, nj, 6)
    runs = []
    for pat in (None, "0x7B", "0xFF"):
        if pat is None:
            os.environ.pop("FTK_POISON", None)
        else:
            os.environ["FTK_POISON"] = pat
        try:
            p, w, imgs, tpls = load_gpu(pkg, cfg, ni, nj, workspace_bytes=ws)
        finally:
            os.environ.pop("FTK_POISON", None)
        res = p.align(pair_best=True)
        L = p.landscape_pairs(ii, jj)
        tau = 0.1 * float(np.median(fb.discrete_norm(imgs[:4].cpu().numpy(), w)) *
                          np.median(fb.discrete_norm(tpls[:4].cpu().numpy(), w)))
        lm = p.align_marginal(tau)
        torch.cuda.synchronize()
        out = [pkg.best_to_numpy(res["best"]).view(np.int32).copy(),
               pkg.best_to_numpy(res["pair_best"].reshape(-1, 4)).view(np.int32).copy(),
               L.cpu().numpy().view(np.int32).copy(), lm.cpu().numpy().view(np.int32).copy()]
        if name == "tiny":
            out.append(p.align(landscape=True)["landscape"].cpu().numpy().view(np.int32).copy())
        assert all(np.all(np.isfinite(x.view(np.float32))) for x in out[2:]), pat
        runs.append(out)
        del p
    for other in runs[1:]:
        for x, y in zip(runs[0], other):
            assert np.array_equal(x, y)


@pytest.mark.parametrize("name,ni,nj", [("c2", 140, 6), ("c3", 140, 5), ("c4", 130, 4), ("c5", 130, 3)])
def test_step2_tensor_core_all_sizes(pkg, name, ni, nj):
    """k_step2_tc (the DFT-64 GEMM form of Step 2) at every n it supports -- n = 128, 256 (forced with
    FTK_S2TC=1; the default there is k_step2_fft) and 512 (its default) -- against the oracle: 12 sampled
    landscapes through ftk_landscape_pairs at the engine's precision bar, and every pair's maximum and
    (shift, rotation) through ftk_align (gap rule R25), with 2-image-tile subsets."""
    cfg = synth.config(name)
    os.environ["FTK_S2TC"] = "1"
    try:
        p, w, imgs, tpls = load_gpu(pkg, cfg, ni, nj)
    finally:
        os.environ.pop("FTK_S2TC", None)
    rng = np.random.default_rng(11)
    ii, jj = rng.integers(0, ni, 12), rng.integers(0, nj, 12)
    L = p.landscape_pairs(ii, jj).cpu().numpy()
    pb = pkg.best_to_numpy(p.align(pair_best=True)["pair_best"].reshape(-1, 4)).reshape(ni, nj)
    a = fb.fb_coeffs(imgs.cpu().numpy().astype(np.complex128))
    b = fb.fb_coeffs(tpls.cpu().numpy().astype(np.complex128))
    na, nb = fb.discrete_norm(imgs.cpu().numpy(), w), fb.discrete_norm(tpls.cpu().numpy(), w)
    plan = oracle_plan(cfg)
    for k in range(12):
        X = np.real(ftk.ftk_landscapes(a[ii[k]:ii[k] + 1], b[jj[k]:jj[k] + 1], plan))[0, 0]
        assert np.max(np.abs(L[k] - X)) / (na[ii[k]] * nb[jj[k]]) <= PREC, (name, k)
    for i in rng.integers(0, ni, 6):
        X = np.real(ftk.ftk_landscapes(a[i:i + 1], b, plan))[0]
        for j in range(nj):
            scale = na[i] * nb[j]
            v = X[j].max()
            assert abs(pb["value"][i, j] - v) <= PREC * scale, (name, i, j)
            t, r = pb["shift_idx"][i, j], pb["rot_idx"][i, j]
            flat = np.sort(X[j].ravel())
            if flat[-1] - flat[-2] > 2 * TOL * scale:
                assert (t, r) == np.unravel_index(np.argmax(X[j]), X[j].shape), (name, i, j)
            else:
                assert X[j][t, r] >= v - TOL * scale, (name, i, j)


@pytest.mark.parametrize("name,ni,nj", [("c3", 260, 7), ("c5", 140, 5)])
def test_step1_cta_pair_bitwise(pkg, name, ni, nj):
    """The opt-in CTA-pair Step 1 (k_step1_cg2, FTK_S1CG2=1: cta_group::2 M = 256, half of every image stage per
    SM) computes the same products in the same order as k_step1_tc: per-pair maxima, per-image bests and explicit-
    pair landscapes must be bitwise equal to the default path (ragged image tiles, odd column-tile counts)."""
    cfg = synth.config(name)
    rng = np.random.default_rng(5)
    ii, jj = rng.integers(0, ni, 6), rng.integers(0, nj, 6)
    outs = []
    for v in ("0", "1"):
        os.environ["FTK_S1CG2"] = v
        try:
            p, w, imgs, tpls = load_gpu(pkg, cfg, ni, nj)
        finally:
            os.environ.pop("FTK_S1CG2", None)
        res = p.align(pair_best=True)
        L = p.landscape_pairs(ii, jj)
        torch.cuda.synchronize()
        outs.append([pkg.best_to_numpy(res["best"]).view(np.int32).copy(),
                     pkg.best_to_numpy(res["pair_best"].reshape(-1, 4)).view(np.int32).copy(),
                     L.cpu().numpy().view(np.int32).copy()])
        del p
    for x, y in zip(*outs):
        assert np.array_equal(x, y)


def test_random_shapes_vs_oracle(pkg):
    """Property test over random small problems on the production engine: random radial order,
    angular grid, shift radius, shift list (1-40 arbitrary off-lattice shifts), tolerance and image / template
    counts (ragged 128-image tiles, single templates).  Per-image bests vs the oracle (value within the
    tolerance, location by the gap rule R25) and sampled landscapes at the engine's precision bar."""
    import dataclasses
    import math
    from hypothesis import HealthCheck, given, settings, strategies as st

    @settings(max_examples=16, deadline=None, suppress_health_check=list(HealthCheck))
    @given(n_k=st.sampled_from([16, 32]), n_psi=st.sampled_from([64, 128, 256, 512]), dmax=st.floats(0.3, 2.0),
           nt=st.integers(1, 40), eps=st.sampled_from([1e-1, 1e-2]), ni=st.integers(1, 150),
           nj=st.integers(1, 5), seed=st.integers(0, 10_000))
    def case(n_k, n_psi, dmax, nt, eps, ni, nj, seed):
        cfg = dataclasses.replace(synth.config("tiny"), n_k=n_k, n_psi=n_psi, eps=eps, seed=seed % 97)
        rng = np.random.default_rng(seed)
        r = dmax * np.sqrt(rng.uniform(0.0, 1.0, nt))
        th = rng.uniform(0.0, 2.0 * math.pi, nt)
        sh = np.stack([r * np.cos(th), r * np.sin(th)], 1)
        p = pkg.FTKPlan(cfg.n, cfg.K, dmax, sh, eps, n_k=n_k, n_psi=n_psi, device=0, engine=0)
        k, w = p.radial()
        imgs, _ = synth.draw_items(cfg, "images", range(ni), k, "planted")
        tpls, _ = synth.draw_items(cfg, "templates", range(nj), k)
        p.load_images(torch.from_numpy(imgs).cuda())
        p.load_templates(torch.from_numpy(tpls).cuda())
        best = pkg.best_to_numpy(p.align()["best"])
        op = ks.build_plan(cfg.n, cfg.K, dmax, sh, eps, n_k, n_psi, n_nodes=64)
        X = np.real(ftk.ftk_landscapes(fb.fb_coeffs(imgs), fb.fb_coeffs(tpls), op))
        na, nb = fb.discrete_norm(imgs, w), fb.discrete_norm(tpls, w)
        v, j, t, rr, gap = ftk.best_per_image(X)
        for i in range(ni):
            scale = na[i] * np.max(nb)
            assert abs(best["value"][i] - v[i]) <= TOL * scale, (i, best["value"][i], v[i])
            if gap[i] > 2 * TOL * scale:
                assert (best["template_idx"][i], best["shift_idx"][i], best["rot_idx"][i]) == (j[i], t[i], rr[i]), i
            else:
                bj, bt, br = best["template_idx"][i], best["shift_idx"][i], best["rot_idx"][i]
                assert X[i, bj, bt, br] >= v[i] - TOL * scale, i
        ii, jj = rng.integers(0, ni, 4), rng.integers(0, nj, 4)
        L = p.landscape_pairs(ii, jj).cpu().numpy()
        for q in range(4):
            assert np.max(np.abs(L[q] - X[ii[q], jj[q]])) <= PREC * na[ii[q]] * nb[jj[q]], q

    case()


def test_fp16x3_extreme_and_mixed_scales(pkg):
    """The fp16x3 arithmetic relies on per-item power-of-two scales.  Images and
    templates spanning 36 decades (1e-18 .. 1e18), an all-zero image and an all-zero template must keep the
    engine's precision bar relative to ||A|| ||B|| in every pair (full landscapes, all pairs), and the zero
    pairs must be exactly zero with the tie rule's (0, 0, 0) best."""
    cfg = synth.config("tiny")
    p = make(pkg, cfg)
    k, w = p.radial()
    imgs, _ = synth.draw_items(cfg, "images", range(6), k, "planted")
    tpls, _ = synth.draw_items(cfg, "templates", range(4), k)
    si = np.array([1e-18, 1e-6, 1.0, 1e6, 1e18, 0.0])
    sj = np.array([1e-15, 1.0, 1e15, 0.0])
    imgs = (imgs * si[:, None, None]).astype(np.complex64)
    tpls = (tpls * sj[:, None, None]).astype(np.complex64)
    p.load_images(torch.from_numpy(imgs).cuda())
    p.load_templates(torch.from_numpy(tpls).cuda())
    ii, jj = np.meshgrid(np.arange(6), np.arange(4), indexing="ij")
    Lp = p.landscape_pairs(ii.ravel(), jj.ravel()).cpu().numpy().reshape(6, 4, p.info["N_t"], p.info["n_gamma"])
    a, b = fb.fb_coeffs(imgs.astype(np.complex128)), fb.fb_coeffs(tpls.astype(np.complex128))
    na, nb = fb.discrete_norm(imgs, w), fb.discrete_norm(tpls, w)
    X = np.real(ftk.ftk_landscapes(a, b, oracle_plan(cfg)))
    for i in range(6):
        for j in range(4):
            if na[i] * nb[j] == 0.0:
                assert np.all(Lp[i, j] == 0.0), (i, j)
                continue
            err = np.max(np.abs(Lp[i, j] - X[i, j])) / (na[i] * nb[j])
            assert err <= PREC, (i, j, err)
    best = pkg.best_to_numpy(p.align()["best"])
    assert best["value"][5] == 0.0
    assert (best["template_idx"][5], best["shift_idx"][5], best["rot_idx"][5]) == (0, 0, 0)


@pytest.mark.parametrize("name,ni,nj", [("c3", 200, 24), ("c5", 260, 12)])
def test_cta_pair_variants_match_default(pkg, name, ni, nj, monkeypatch):
    """The opt-in CTA-pair kernels: the fused Steps 2 + 3 (FTK_S23=1) and the
    Step-3-only CTA-pair kernel (FTK_S3V2=1) against the default k_step2_fft + k_step3_tc on the same inputs:
    the Step-3-only variant bitwise (same operands, same accumulation order), the fused one's per-pair maxima
    within the precision bar of the default ones (its F-point FFT rounds differently)."""
    cfg = synth.config(name)

    def run(s23, s3v2):
        monkeypatch.setenv("FTK_S23", s23)
        monkeypatch.setenv("FTK_S3V2", s3v2)
        p, w, imgs, tpls = load_gpu(pkg, cfg, ni, nj)
        pb = pkg.best_to_numpy(p.align(pair_best=True)["pair_best"].reshape(-1, 4)).reshape(ni, nj)
        na = fb.discrete_norm(imgs.cpu().numpy(), w)
        nb = fb.discrete_norm(tpls.cpu().numpy(), w)
        del p
        return pb, na, nb

    ref, na, nb = run("0", "0")
    v2, _, _ = run("0", "1")
    assert np.array_equal(ref.view(np.int32), v2.view(np.int32))
    fused, _, _ = run("1", "0")
    scale = na[:, None] * nb[None, :]
    assert np.max(np.abs(fused["value"] - ref["value"]) / scale) <= PREC
