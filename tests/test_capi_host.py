"""C-ABI checks that need no GPU: the library loads, exports every symbol include/ftk.h declares,
and the host-side plan (ftk_plan_create with device = -1, untimed plan math) agrees with the oracle."""
import math
import os
import re

import numpy as np
import pytest

import synth
from oracle import kernel_svd as ks, quadrature

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def ftk():
    import __graft_entry__ as g
    g.build()
    import paper_1905_12317_b200 as p
    return p


def test_exports_every_declared_symbol(ftk):
    hdr = open(os.path.join(ROOT, "include", "ftk.h")).read()
    declared = set(re.findall(r"^\s*(?:ftk_status_t|void|const char\*|int)\s+(ftk_\w+)\s*\(", hdr, re.M))
    assert len(declared) >= 18
    L = ftk.lib()
    for name in sorted(declared):
        assert hasattr(L, name), name
    assert set(declared) == set(ftk._ffi.SYMBOLS), set(declared) ^ set(ftk._ffi.SYMBOLS)
    assert L.ftk_version() >= 100


def _host_plan(ftk, name, **kw):
    cfg = synth.config(name)
    return cfg, ftk.FTKPlan(cfg.n, cfg.K, synth.delta_max(cfg), synth.shift_list(cfg), cfg.eps, n_k=cfg.n_k,
                            n_psi=cfg.n_psi, device=-1, **kw)


@pytest.mark.parametrize("name,H,Hp", [("tiny", 27, 15), ("c2", 36, 20), ("c3", 63, 34), ("c5", 94, 50)])
def test_host_plan_matches_oracle(ftk, name, H, Hp):
    cfg, p = _host_plan(ftk, name)
    assert p.info["H"] == H and p.info["H_plus"] == Hp
    k, w = p.radial()
    ko, wo = quadrature.radial_rule(cfg.n_k, cfg.k_max)
    assert np.max(np.abs(k - ko)) < 1e-13 and np.max(np.abs(w - wo)) < 1e-12 * np.max(wo)
    ell, eta, sig = p.terms()
    op = ks.build_plan(cfg.n, cfg.K, synth.delta_max(cfg), synth.shift_list(cfg), cfg.eps, cfg.n_k, cfg.n_psi,
                       n_nodes=96 if name != "tiny" else 64)
    assert list(ell) == [t.ell for t in op.terms] and list(eta) == [t.eta for t in op.terms]
    assert np.max(np.abs(sig - np.array([t.sigma for t in op.terms]))) < 1e-10
    G, Y = p.factors()
    # products Y_zeta(t) G_zeta(k_m) are sign-invariant; compare the assembled per-term rank-1 factors
    for z in range(H):
        P1 = np.outer(Y[:, z], G[z])
        P2 = np.outer(op.Y[:, z], op.G[z])
        assert np.max(np.abs(P1 - P2)) < 1e-8 * max(1.0, np.max(np.abs(P2)))
    assert p.info["certificate"] < 13 * cfg.eps


def test_host_plan_errors(ftk):
    cfg = synth.config("tiny")
    sh = synth.shift_list(cfg)
    with pytest.raises(ftk.FTKError) as e:
        ftk.FTKPlan(cfg.n, cfg.K, 0.5, sh, cfg.eps, n_k=16, n_psi=64, device=-1)    # shifts outside Omega_D
    assert e.value.status == 2
    with pytest.raises(ftk.FTKError) as e:
        ftk.FTKPlan(cfg.n, cfg.K, 1.1, sh, cfg.eps, n_k=16, n_psi=48, device=-1)    # n_psi not a power of two
    assert e.value.status == 1
    cfg2, p = _host_plan(ftk, "tiny")
    with pytest.raises(ftk.FTKError) as e:
        p.align_host()                     # host-only plan: FTK_ESTATE, no device touched
    assert e.value.status == 6


def test_gauss_jacobi_rule_option(ftk):
    cfg, p = _host_plan(ftk, "c2", radial_rule=1)
    k, w = p.radial()
    ko, wo = quadrature.gauss_jacobi_01(cfg.n_k, cfg.k_max)
    assert np.max(np.abs(k - ko)) < 1e-12 and np.max(np.abs(w - wo)) < 1e-12 * np.max(wo)


def test_merge_host_tie_break(ftk):
    # records: value, template, shift, rot (value stored as float32 bits)
    def rec(v, j, t, r):
        return [np.float32(v).view(np.int32), j, t, r]
    g = np.array([rec(1.0, 5, 0, 0), rec(2.0, 9, 1, 1), rec(-np.inf, -1, -1, -1),
                  rec(1.0, 3, 7, 7), rec(2.0, 9, 0, 5), rec(0.5, 1, 1, 1)], dtype=np.int32)
    out = ftk.merge_bests(g, 2, 3)
    vals = out[:, 0].view(np.float32)
    assert vals[0] == 1.0 and out[0, 1] == 3          # equal values -> smaller template
    assert vals[1] == 2.0 and tuple(out[1, 1:]) == (9, 0, 5)   # equal template -> smaller shift
    assert vals[2] == 0.5 and out[2, 1] == 1          # missing record (-1) loses


@pytest.mark.parametrize("name,defoci", [("tiny", [8000.0, 15000.0, 22000.0, 30000.0]), ("c2", [10000.0, 20000.0])])
def test_host_ctf_plan_matches_oracle(ftk, name, defoci):
    """ftk_plan_create_ctf (reading R24) vs oracle.ctf: same terms, Sigma and rank-1 factors on the virtual
    shift list; ftk_radial_rule == the oracle's rule."""
    from oracle import ctf
    cfg = synth.config(name)
    sh = synth.shift_list(cfg)
    k, w = ftk.radial_rule(cfg.n, cfg.K, cfg.n_k, 0)
    ko, wo = quadrature.radial_rule(cfg.n_k, cfg.k_max)
    assert np.max(np.abs(k - ko)) < 1e-13 and np.max(np.abs(w - wo)) < 1e-12 * np.max(wo)
    f = synth.ctf_filters(k, defoci)
    p = ftk.FTKPlan(cfg.n, cfg.K, synth.delta_max(cfg), sh, cfg.eps, n_k=cfg.n_k, n_psi=cfg.n_psi, device=-1,
                    filters=f)
    op = ctf.build_plan_ctf(cfg.n, cfg.K, synth.delta_max(cfg), sh, cfg.eps, cfg.n_k, cfg.n_psi,
                            synth.ctf_filters(ko, defoci), n_nodes=96)
    assert p.info["n_tau"] == len(defoci) and p.info["N_t_base"] == len(sh)
    assert p.info["N_t"] == len(defoci) * len(sh) and p.info["H"] == op.H
    ell, eta, sig = p.terms()
    assert list(ell) == [t.ell for t in op.terms] and list(eta) == [t.eta for t in op.terms]
    assert np.max(np.abs(sig - np.array([t.sigma for t in op.terms]))) < 1e-10
    G, Y = p.factors()
    for z in range(op.H):
        P1 = np.outer(Y[:, z], G[z])
        P2 = np.outer(op.Y[:, z], op.G[z])
        assert np.max(np.abs(P1 - P2)) < 1e-8 * max(1.0, np.max(np.abs(P2)))
    assert abs(p.info["certificate"] - ctf.kernel_certificate_ctf(op, f)) < 1e-9
    t, tau = p.split_ctf_index(np.array([0, len(sh) + 3, p.info["N_t"] - 1]))
    assert list(t) == [0, 3, len(sh) - 1] and list(tau) == [0, 1, len(defoci) - 1]


def test_host_ctf_plan_errors(ftk):
    cfg = synth.config("tiny")
    sh = synth.shift_list(cfg)
    bad = np.ones((2, cfg.n_k))
    bad[1, 3] = np.nan
    with pytest.raises(ftk.FTKError) as e:
        ftk.FTKPlan(cfg.n, cfg.K, synth.delta_max(cfg), sh, cfg.eps, n_k=16, n_psi=64, device=-1, filters=bad)
    assert e.value.status == 1
    L = ftk.lib()
    import ctypes as C
    out = C.c_void_p()
    shp = np.ascontiguousarray(sh)
    st = L.ftk_plan_create_ctf(cfg.n, cfg.K, synth.delta_max(cfg), shp.ctypes.data_as(C.c_void_p), len(sh), 0,
                               None, cfg.eps, None, C.byref(out))
    assert st == 1 and not out.value
    k = np.empty(4)
    assert L.ftk_radial_rule(cfg.n, cfg.K, 4, 7, k.ctypes.data_as(C.c_void_p), k.ctypes.data_as(C.c_void_p)) == 1


def test_nccl_unique_id_and_status(ftk):
    """The NCCL glue loads libnccl.so.2 at run time; a unique id needs no GPU.  FTK_ENCCL has a name."""
    import ctypes as C
    L = ftk.lib()
    assert L.ftk_status_string(9) == b"FTK_ENCCL"
    buf = C.create_string_buffer(128)
    assert L.ftk_nccl_unique_id(buf) == 0
    assert any(buf.raw)
    assert L.ftk_nccl_unique_id(None) == 1          # FTK_EINVAL
    h = C.c_void_p()
    assert L.ftk_nccl_comm_create(buf, 2, 5, -1, C.byref(h)) == 1   # rank >= world


from hypothesis import HealthCheck, given, settings, strategies as st  # noqa: E402


@settings(max_examples=12, deadline=None, suppress_health_check=[HealthCheck.function_scoped_fixture])
@given(dmax=st.floats(0.3, 3.0), eps=st.sampled_from([1e-1, 3e-2, 1e-2, 3e-3]), n_k=st.sampled_from([16, 32]),
       seed=st.integers(0, 10_000))
def test_host_plan_matches_oracle_random(ftk, dmax, eps, n_k, seed):
    """Property test: for random shift radii, tolerances, radial orders and shift lists the C++
    host plan (Nystrom + one-sided Jacobi SVD, truncation Sigma > eps, zeta relabel, G / Y) reproduces the
    float64 oracle's terms, singular values and rank-1 factors Y_zeta G_zeta^T, and its kernel certificate
    stays within the factorization's own error scale."""
    n, K = 32, 16.0
    rng = np.random.default_rng(seed)
    r = dmax * np.sqrt(rng.uniform(0.0, 1.0, 9))
    th = rng.uniform(0.0, 2.0 * math.pi, 9)
    sh = np.concatenate([[[0.0, 0.0]], np.stack([r * np.cos(th), r * np.sin(th)], 1)])
    p = ftk.FTKPlan(n, K, dmax, sh, eps, n_k=n_k, n_psi=64, device=-1)
    op = ks.build_plan(n, K, dmax, sh, eps, n_k, 64, n_nodes=96)
    ell, eta, sig = p.terms()
    ref = np.array([t.sigma for t in op.terms])
    # a singular value within 1e-9 of eps may legitimately fall on either side of the cut (reading R6)
    if np.any(np.abs(ref - eps) < 1e-9) or p.info["H"] != len(op.terms):
        assert abs(p.info["H"] - len(op.terms)) <= 2 and np.min(np.abs(ref - eps)) < 1e-6
        return
    assert list(ell) == [t.ell for t in op.terms] and list(eta) == [t.eta for t in op.terms]
    assert np.max(np.abs(sig - ref)) < 1e-10
    G, Y = p.factors()
    for z in range(len(ref)):
        P1 = np.outer(Y[:, z], G[z])
        P2 = np.outer(op.Y[:, z], op.G[z])
        assert np.max(np.abs(P1 - P2)) < 1e-8 * max(1.0, np.max(np.abs(P2)))
    assert p.info["certificate"] < 13 * eps
