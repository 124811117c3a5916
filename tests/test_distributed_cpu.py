"""N > 1 path on CPU: world_size-2 gloo process group, template shards, all-gather of per-image
records and the library's deterministic merge (ftk_merge_bests_host) equal the single-rank answer.
The per-rank records come from the oracle's landscapes restricted to the rank's shard (no GPU)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth
from oracle import fb, ftk, kernel_svd as ks


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _records(X, j_offset):
    """Per-image best over this shard's landscapes X [I, J_local, T, R] -> int32 [I, 4] (ftk_best_t)."""
    v, j, t, r, _ = ftk.best_per_image(X)
    out = np.zeros((X.shape[0], 4), dtype=np.int32)
    out[:, 0] = v.astype(np.float32).view(np.int32)
    out[:, 1] = j + j_offset
    out[:, 2] = t
    out[:, 3] = r
    return out


def _worker(rank, world, port, X, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import __graft_entry__ as g
    g.build()
    import paper_1905_12317_b200 as pkg
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = pkg.shard_range(rank, world, X.shape[1])
    if hi > lo:
        local = torch.from_numpy(_records(X[:, lo:hi], lo))
    else:
        local = torch.tensor([[np.float32(-np.inf).view(np.int32), -1, -1, -1]] * X.shape[0], dtype=torch.int32)
    merged = pkg.gather_and_merge(local)
    q.put((rank, np.asarray(merged)))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,nj", [(2, 5), (2, 1)])
def test_two_rank_gloo_merge_matches_single_rank(world, nj):
    cfg = synth.config("tiny")
    plan = ks.build_plan(cfg.n, cfg.K, synth.delta_max(cfg), synth.shift_list(cfg), cfg.eps, cfg.n_k, cfg.n_psi)
    imgs, _ = synth.draw_items(cfg, "images", range(3), plan.k, "planted")
    tpls, _ = synth.draw_items(cfg, "templates", range(nj), plan.k)
    X = np.real(ftk.ftk_landscapes(fb.fb_coeffs(imgs), fb.fb_coeffs(tpls), plan)).astype(np.float32).astype(np.float64)
    ref = _records(X, 0)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, X, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, merged in res:
        assert np.array_equal(merged, ref), (rank, merged, ref)


def _worker_marg(rank, world, port, X, tau, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import paper_1905_12317_b200 as pkg
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = pkg.shard_range(rank, world, X.shape[1])
    local = torch.from_numpy(ftk.log_marginal(X[:, lo:hi], tau).astype(np.float32).reshape(X.shape[0], hi - lo))
    full = pkg.gather_marginal(local, X.shape[1])
    q.put((rank, np.asarray(full)))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,nj", [(2, 5), (3, 7), (3, 2)])
def test_gloo_gather_marginal_matches_single_rank(world, nj):
    """Template-sharded log-marginals (NEXT-3) gathered over a gloo group equal the single-rank matrix,
    including ranks that own no template (world > N_tm)."""
    cfg = synth.config("tiny")
    plan = ks.build_plan(cfg.n, cfg.K, synth.delta_max(cfg), synth.shift_list(cfg), cfg.eps, cfg.n_k, cfg.n_psi)
    imgs, _ = synth.draw_items(cfg, "images", range(3), plan.k)
    tpls, _ = synth.draw_items(cfg, "templates", range(nj), plan.k)
    X = np.real(ftk.ftk_landscapes(fb.fb_coeffs(imgs), fb.fb_coeffs(tpls), plan))
    tau = 0.1
    ref = ftk.log_marginal(X, tau).astype(np.float32)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_marg, args=(r, world, port, X, tau, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, full in res:
        assert np.array_equal(full, ref), (rank, full, ref)
