"""Thin Python binding over the C ABI (include/ftk.h).  Argument marshalling only: every step of the
hot path runs in libftk.so's CUDA kernels; torch is used for device memory, streams and
torch.distributed (NCCL) plumbing."""
from __future__ import annotations

import ctypes as C
from typing import Optional

import numpy as np

from . import _ffi

ENGINE_TC = 0     # tcgen05 fp16x3 tensor-core path
ENGINE_SIMT = 1   # CUDA-core fp32 reference kernels
KERNEL_CLASSES = ("load_fft", "step1", "step2", "step3", "finalize")


class FTKError(RuntimeError):
    def __init__(self, status: int, msg: str):
        self.status = status
        super().__init__(f"{_ffi.lib().ftk_status_string(status).decode()}: {msg}")


def _check(st: int, plan_ptr=None):
    if st != 0:
        msg = _ffi.lib().ftk_last_error(plan_ptr).decode() if plan_ptr else ""
        raise FTKError(st, msg)


def _stream_ptr(stream):
    if stream is None:
        try:
            import torch
            if torch.cuda.is_available():
                return C.c_void_p(torch.cuda.current_stream().cuda_stream)
        except ImportError:
            pass
        return C.c_void_p(0)
    if isinstance(stream, int):
        return C.c_void_p(stream)
    return C.c_void_p(stream.cuda_stream)


BEST_DTYPE = np.dtype([("value", "<f4"), ("template_idx", "<i4"), ("shift_idx", "<i4"), ("rot_idx", "<i4")])


def best_to_numpy(t) -> np.ndarray:
    """Device/host int32 [N, 4] record tensor -> structured numpy array (value, template, shift, rot)."""
    a = t.detach().cpu().numpy() if hasattr(t, "detach") else np.asarray(t)
    return np.ascontiguousarray(a).view(BEST_DTYPE).reshape(-1)


def radial_rule(n: int, K: float, n_k: int = 0, rule: int = 0):
    """ftk_radial_rule: the radial nodes/weights (k_m, w_m) a plan with these arguments uses (host)."""
    L = _ffi.lib()
    n_k = n_k if n_k > 0 else int(round(K))
    k, w = np.empty(n_k), np.empty(n_k)
    st = L.ftk_radial_rule(n, float(K), n_k, rule, k.ctypes.data_as(C.c_void_p), w.ctypes.data_as(C.c_void_p))
    if st != 0:
        raise FTKError(st, "ftk_radial_rule failed")
    return k, w


class FTKPlan:
    """One FTK plan (ftk_plan_create) bound to one CUDA device (or host-only with device=-1).

    filters: optional real array [n_tau, n_k] of radial filters (CTFs) on the plan's radial nodes
    (radial_rule()); then the plan is ftk_plan_create_ctf's CTF-parameterized kernel and every result
    indexes the virtual shift v = tau * N_t + t (split_ctf_index)."""

    def __init__(self, n: int, K: float, delta_max: float, shifts, eps: float, *, n_k: int = 0, n_psi: int = 0,
                 radial_rule: int = 0, device: int = 0, rank: int = 0, world: int = 1, engine: int = ENGINE_TC,
                 svd_nodes: int = 0, workspace_bytes: int = 0, n_gamma: int = 0, filters=None, nccl_comm=None):
        self._L = _ffi.lib()
        sh = np.ascontiguousarray(np.asarray(shifts, dtype=np.float64).reshape(-1, 2))
        comm = nccl_comm.handle if isinstance(nccl_comm, NcclComm) else nccl_comm
        opts = _ffi.PlanOpts(n_k, n_psi, radial_rule, device, rank, world, engine, svd_nodes, workspace_bytes,
                             n_gamma, C.c_void_p(comm) if comm else None)
        self._comm_ref = nccl_comm  # the communicator must outlive the plan
        out = C.c_void_p()
        if filters is None:
            st = self._L.ftk_plan_create(n, float(K), float(delta_max), sh.ctypes.data_as(C.c_void_p), sh.shape[0],
                                         float(eps), C.byref(opts), C.byref(out))
        else:
            f = np.ascontiguousarray(np.asarray(filters, dtype=np.float64))
            f = f.reshape(1, -1) if f.ndim == 1 else f
            st = self._L.ftk_plan_create_ctf(n, float(K), float(delta_max), sh.ctypes.data_as(C.c_void_p),
                                             sh.shape[0], f.shape[0], f.ctypes.data_as(C.c_void_p), float(eps),
                                             C.byref(opts), C.byref(out))
        if st != 0:
            raise FTKError(st, "ftk_plan_create failed")
        self._p = out
        self.shifts = sh
        self.device = device
        self._refresh()

    def _refresh(self):
        info = _ffi.PlanInfo()
        _check(self._L.ftk_plan_query(self._p, C.byref(info)), self._p)
        self.info = {f: getattr(info, f) for f, _ in info._fields_}

    def __del__(self):
        p = getattr(self, "_p", None)
        if p:
            self._L.ftk_plan_destroy(p)
            self._p = None

    def split_ctf_index(self, v):
        """Virtual shift index v -> (shift t, filter tau) for CTF plans ((v, 0) for plain plans)."""
        v = np.asarray(v)
        nb = self.info["N_t_base"]
        return v % nb, v // nb

    # ---------------- plan queries (host)
    def radial(self):
        nk = self.info["n_k"]
        k, w = np.empty(nk), np.empty(nk)
        _check(self._L.ftk_plan_radial(self._p, k.ctypes.data_as(C.c_void_p), w.ctypes.data_as(C.c_void_p)), self._p)
        return k, w

    def terms(self):
        H = self.info["H"]
        ell, eta, sig = np.empty(H, np.int32), np.empty(H, np.int32), np.empty(H)
        _check(self._L.ftk_plan_terms(self._p, ell.ctypes.data_as(C.c_void_p), eta.ctypes.data_as(C.c_void_p),
                                      sig.ctypes.data_as(C.c_void_p)), self._p)
        return ell, eta, sig

    def factors(self):
        H, nk, Nt = self.info["H"], self.info["n_k"], self.info["N_t"]
        G, Y = np.empty((H, nk)), np.empty((Nt, H, 2))
        _check(self._L.ftk_plan_factors(self._p, G.ctypes.data_as(C.c_void_p), Y.ctypes.data_as(C.c_void_p)), self._p)
        return G, Y[..., 0] + 1j * Y[..., 1]

    # ---------------- loads
    def _load(self, fn, x, stream):
        import torch
        if isinstance(x, np.ndarray):
            x = torch.from_numpy(np.ascontiguousarray(x.astype(np.complex64, copy=False)))
        assert x.dtype == torch.complex64 and x.dim() == 3, "polar samples must be complex64 [N][n_k][n_psi]"
        assert x.shape[1] == self.info["n_k"] and x.shape[2] == self.info["n_psi"], (tuple(x.shape), self.info)
        x = x.contiguous()
        _check(fn(self._p, C.c_void_p(x.data_ptr()), x.shape[0], 1 if x.is_cuda else 0, _stream_ptr(stream)), self._p)
        self._refresh()

    def load_images(self, polar, stream=None):
        self._load(self._L.ftk_load_images, polar, stream)

    def load_templates(self, polar, stream=None):
        self._load(self._L.ftk_load_templates, polar, stream)

    # ---------------- pixel front end (Eq. Ahattrap by a type-2 NUFFT)
    def _pixels(self, x):
        import torch
        if isinstance(x, np.ndarray):
            x = torch.from_numpy(np.ascontiguousarray(x.astype(np.float32, copy=False)))
        n = self.info["n"]
        assert x.dtype == torch.float32 and x.dim() == 3 and x.shape[1] == n and x.shape[2] == n, \
            f"pixels must be float32 [N][{n}][{n}]"
        return x.contiguous()

    def polar_from_pixels(self, pixels, stream=None):
        """complex64 [N, n_k, n_psi] device tensor of Ahat(k_m, psi_p) from float32 [N, n, n] pixels."""
        import torch
        x = self._pixels(pixels)
        out = torch.empty((x.shape[0], self.info["n_k"], self.info["n_psi"]), dtype=torch.complex64,
                          device=f"cuda:{self.device}")
        _check(self._L.ftk_polar_from_pixels(self._p, C.c_void_p(x.data_ptr()), x.shape[0], 1 if x.is_cuda else 0,
                                             C.c_void_p(out.data_ptr()), _stream_ptr(stream)), self._p)
        return out

    def load_images_pixels(self, pixels, stream=None):
        x = self._pixels(pixels)
        _check(self._L.ftk_load_images_pixels(self._p, C.c_void_p(x.data_ptr()), x.shape[0], 1 if x.is_cuda else 0,
                                              _stream_ptr(stream)), self._p)
        self._refresh()

    def load_templates_pixels(self, pixels, stream=None):
        x = self._pixels(pixels)
        _check(self._L.ftk_load_templates_pixels(self._p, C.c_void_p(x.data_ptr()), x.shape[0],
                                                 1 if x.is_cuda else 0, _stream_ptr(stream)), self._p)
        self._refresh()

    def fb_coeffs(self, which: int, first: int, count: int, stream=None):
        import torch
        out = torch.empty((count, self.info["n_k"], self.info["n_psi"]), dtype=torch.complex64,
                          device=f"cuda:{self.device}")
        _check(self._L.ftk_fb_coeffs(self._p, which, first, count, C.c_void_p(out.data_ptr()), _stream_ptr(stream)),
               self._p)
        return out

    # ---------------- hot path
    def align(self, pair_best: bool = False, landscape: bool = False, stream=None, out=None):
        """Returns dict with 'best' (int32 [N_im,4] device tensor of ftk_best_t), optionally 'pair_best'
        [N_im, N_tm_local, 4] and 'landscape' float [N_im, N_tm_local, N_t, n_gamma]."""
        import torch
        dev = f"cuda:{self.device}"
        NI, NJ = self.info["n_images"], self.info["n_templates_local"]
        best = out if out is not None else torch.empty((NI, 4), dtype=torch.int32, device=dev)
        pb = torch.empty((NI, NJ, 4), dtype=torch.int32, device=dev) if pair_best else None
        land = torch.empty((NI, NJ, self.info["N_t"], self.info["n_gamma"]), dtype=torch.float32, device=dev) \
            if landscape else None
        _check(self._L.ftk_align(self._p, C.c_void_p(best.data_ptr()),
                                 C.c_void_p(pb.data_ptr() if pb is not None else 0),
                                 C.c_void_p(land.data_ptr() if land is not None else 0),
                                 land.numel() if land is not None else 0, _stream_ptr(stream)), self._p)
        res = {"best": best}
        if pb is not None:
            res["pair_best"] = pb
        if land is not None:
            res["landscape"] = land
        return res

    def align_host(self, stream=None) -> np.ndarray:
        """ftk_align with a HOST output buffer (the call copies back and synchronizes)."""
        out = np.empty(self.info["n_images"], dtype=BEST_DTYPE)
        _check(self._L.ftk_align(self._p, C.c_void_p(out.ctypes.data), C.c_void_p(0), C.c_void_p(0), 0,
                                 _stream_ptr(stream)), self._p)
        return out

    def align_marginal(self, tau: float, stream=None, out=None):
        """ftk_align_marginal: float32 [N_im, N_tm_local] device tensor of log sum_{t,r} exp(X / tau)."""
        import torch
        NI, NJ = self.info["n_images"], self.info["n_templates_local"]
        res = out if out is not None else torch.empty((NI, NJ), dtype=torch.float32, device=f"cuda:{self.device}")
        _check(self._L.ftk_align_marginal(self._p, float(tau), C.c_void_p(res.data_ptr()), _stream_ptr(stream)),
               self._p)
        return res

    def landscape_pairs(self, img_idx, tpl_idx, stream=None):
        import torch
        dev = f"cuda:{self.device}"
        ii = torch.as_tensor(np.asarray(img_idx, dtype=np.int32), device=dev)
        jj = torch.as_tensor(np.asarray(tpl_idx, dtype=np.int32), device=dev)
        out = torch.empty((ii.numel(), self.info["N_t"], self.info["n_gamma"]), dtype=torch.float32, device=dev)
        _check(self._L.ftk_landscape_pairs(self._p, C.c_void_p(ii.data_ptr()), C.c_void_p(jj.data_ptr()), ii.numel(),
                                           C.c_void_p(out.data_ptr()), out.numel(), _stream_ptr(stream)), self._p)
        return out

    # ---------------- profiling
    def set_profiling(self, on: bool):
        _check(self._L.ftk_set_profiling(self._p, 1 if on else 0), self._p)

    def kernel_times(self):
        ms = np.zeros(5)
        cnt = np.zeros(5, dtype=np.int64)
        _check(self._L.ftk_kernel_times(self._p, ms.ctypes.data_as(C.c_void_p), cnt.ctypes.data_as(C.c_void_p)), self._p)
        return {k: (float(ms[i]), int(cnt[i])) for i, k in enumerate(KERNEL_CLASSES)}


class NcclComm:
    """An NCCL communicator created through the C ABI (ftk_nccl_unique_id / ftk_nccl_comm_create).  Pass it
    as FTKPlan(nccl_comm=...): ftk_align then all-gathers and merges the per-image bests inside the library
    and returns global bests on every rank.  torch.distributed only carries the 128-byte unique id."""

    def __init__(self, world: int, rank: int, device: int, uid: bytes):
        self._L = _ffi.lib()
        assert len(uid) == 128
        buf = C.create_string_buffer(uid, 128)
        h = C.c_void_p()
        _check(self._L.ftk_nccl_comm_create(buf, world, rank, device, C.byref(h)))
        self.handle = h.value
        self.world, self.rank = world, rank

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        _check(_ffi.lib().ftk_nccl_unique_id(buf))
        return buf.raw

    @classmethod
    def from_group(cls, device: int, group=None):
        """Collective over a torch.distributed group: rank 0 draws the id, the group broadcasts it."""
        import torch
        import torch.distributed as dist
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        uid = cls.unique_id() if rank == 0 else bytes(128)
        t = torch.tensor(list(uid), dtype=torch.uint8)
        if dist.get_backend(group) == "nccl":
            t = t.cuda(device)
        dist.broadcast(t, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
        return cls(world, rank, device, bytes(t.cpu().tolist()))

    def close(self):
        if getattr(self, "handle", None):
            self._L.ftk_nccl_comm_destroy(C.c_void_p(self.handle))
            self.handle = None

    def __del__(self):
        self.close()


def merge_bests(gathered, world: int, n_im: int, out=None, stream=None):
    """Deterministic cross-rank merge (ftk_merge_bests on device tensors, _host on numpy/CPU tensors)."""
    L = _ffi.lib()
    if isinstance(gathered, np.ndarray) or not getattr(gathered, "is_cuda", False):
        g = gathered.numpy() if hasattr(gathered, "numpy") else gathered
        g = np.ascontiguousarray(g, dtype=np.int32).reshape(world * n_im, 4)
        o = np.empty((n_im, 4), dtype=np.int32)
        _check(L.ftk_merge_bests_host(C.c_void_p(g.ctypes.data), world, n_im, C.c_void_p(o.ctypes.data)))
        return o
    import torch
    o = out if out is not None else torch.empty((n_im, 4), dtype=torch.int32, device=gathered.device)
    _check(L.ftk_merge_bests(C.c_void_p(gathered.data_ptr()), world, n_im, C.c_void_p(o.data_ptr()),
                             _stream_ptr(stream)))
    return o


def shard_range(rank: int, world: int, n_total: int):
    """Templates kept by `rank` (mirrors ftk_load_templates): [floor(r N / W), floor((r+1) N / W))."""
    return rank * n_total // world, (rank + 1) * n_total // world


def gather_and_merge(local, group=None, stream=None):
    """All-gather per-rank int32 [N_im, 4] records (NCCL for CUDA tensors, gloo for CPU) and merge them."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    if world == 1:
        return local
    if local.is_cuda:
        gathered = torch.empty((world * local.shape[0], 4), dtype=torch.int32, device=local.device)
        dist.all_gather_into_tensor(gathered, local.contiguous(), group=group)
    else:
        parts = [torch.empty_like(local) for _ in range(world)]
        dist.all_gather(parts, local.contiguous(), group=group)
        gathered = torch.cat(parts)
    out = merge_bests(gathered, world, local.shape[0], stream=stream)
    return out if hasattr(out, "device") else torch.from_numpy(out)


def distributed_align(plan: FTKPlan, group=None, stream=None):
    """Template-sharded alignment.  A plan created with nccl_comm gathers inside ftk_align (the library's
    ncclAllGather + device merge): its result is already global.  Otherwise the per-image records are
    all-gathered through torch.distributed (gloo on CPU) and merged with ftk_merge_bests."""
    local = plan.align(stream=stream)["best"]
    if getattr(plan, "_comm_ref", None) is not None:
        return local
    return gather_and_merge(local, group=group, stream=stream)


def gather_marginal(local, n_tm_total: int, group=None):
    """All-gather per-rank float32 [N_im, N_tm_local] log-marginals (template shards in shard_range order)
    into the full [N_im, N_tm_total] matrix on every rank (NCCL for CUDA tensors, gloo for CPU)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    if world == 1:
        return local
    rank = dist.get_rank(group)
    ni = local.shape[0]
    width = max(hi - lo for lo, hi in (shard_range(r, world, n_tm_total) for r in range(world)))
    pad = torch.full((ni, width), float("-inf"), dtype=torch.float32, device=local.device)
    lo, hi = shard_range(rank, world, n_tm_total)
    pad[:, : hi - lo] = local
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad.contiguous(), group=group)
    out = torch.empty((ni, n_tm_total), dtype=torch.float32, device=local.device)
    for r in range(world):
        lo, hi = shard_range(r, world, n_tm_total)
        out[:, lo:hi] = parts[r][:, : hi - lo]
    return out


def distributed_align_marginal(plan: FTKPlan, tau: float, group=None, stream=None):
    """Template-sharded marginalization (ftk_align_marginal on this rank's shard) gathered to the full
    [N_im, N_tm] matrix of log sum_{t,r} exp(X / tau) on every rank."""
    local = plan.align_marginal(tau, stream=stream)
    return gather_marginal(local, plan.info["n_templates_total"], group=group)
