"""Seeded Gaussian-blob workloads with the shapes of BASELINE.json's five configs.

Stand-in for the paper's GroEL-GroES projections (not in
the container): templates are sums of isotropic Gaussian blobs (the paper's
Fig. 1 uses anisotropic blobs); images are either independent blob
images ("independent", the literal config) or rigidly transformed templates
("planted", the paper's experiment design P:1284).

Units: x, delta in pixels; k in rad/px.  Fourier convention of PAPER.md Eq.
(Ahat) P:196-200:  Ahat(k) = int A(x) exp(-i k.x) dx.  The radial nodes k_m
are an INPUT here (the caller's quadrature); this module never integrates.

Recipe:
  * per item, numpy.random.default_rng([cfg.seed, stream, item]) with
    streams 0 = template blobs, 1 = image blobs / planted choice,
    2 = template noise, 3 = image noise;
  * blob centres uniform in a disc of radius cfg.center_radius px,
    sigma ~ U[1.5, 3] px, amplitude ~ N(0, 1);
  * each clean item is scaled to unit L2 norm in real space, using
    the closed-form Gaussian overlap integral;
  * noise: i.i.d. complex Gaussian per polar sample with Hermitian pairing
    (p <-> p + n_psi/2, conjugated) so real images stay real; variance chosen
    so E||noise||^2 = ||signal||^2 / SNR in the discrete bandlimited norm,
    using sum_m w_m = k_max^2/2 (exact for any rule integrating k dk).
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional, Sequence

import numpy as np

__all__ = [
    "Config", "CONFIGS", "config", "shift_list", "delta_max", "draw_items",
    "blob_params", "polar_samples", "add_noise", "make_polar_set", "planted_truth",
]


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    n: int              # pixels per side
    K: float            # band limit in cycles per image width (BASELINE.json "K"); k_max = 2*pi*K/n rad/px
    n_k: int            # radial quadrature nodes
    n_psi: int          # angles per ring (= rotations n_gamma)
    N_im: int
    N_tm: int
    n_blobs: int
    center_radius: float
    snr: float          # math.inf = noiseless
    spacing: float      # shift lattice pitch, px
    shift_radius: float  # disc radius for the lattice (px); tiny uses a square
    eps: float
    square_lattice: bool = False
    seed: int = 0

    @property
    def k_max(self) -> float:
        return 2.0 * math.pi * self.K / self.n


# BASELINE.json "configs" (same order); seeds are the config index.
CONFIGS = {
    "tiny": Config("tiny", 32, 16.0, 16, 64, 4, 4, 8, 8.0, math.inf, 0.25, 0.75, 1e-3,
                   square_lattice=True, seed=0),
    "c2": Config("c2", 64, 32.0, 32, 128, 256, 256, 16, 16.0, 1.0, 0.25, 2.0, 1e-2, seed=1),
    "c3": Config("c3", 128, 64.0, 64, 256, 1024, 1024, 24, 32.0, 0.1, 0.5, 3.0, 1e-2, seed=2),
    "c4": Config("c4", 128, 64.0, 64, 256, 512, 512, 24, 32.0, 0.1, 0.125, 4.0, 1e-3, seed=3),
    "c5": Config("c5", 256, 128.0, 128, 512, 8192, 4096, 32, 64.0, 0.05, 0.25, 4.0, 1e-2, seed=4),
}


def config(name: str, **overrides) -> Config:
    cfg = CONFIGS[name]
    return dataclasses.replace(cfg, **overrides) if overrides else cfg


def shift_list(cfg: Config) -> np.ndarray:
    """Shift vectors delta_t (px), ordered y-outer / x-inner ascending.  [N_t, 2] float64."""
    s = cfg.spacing
    if cfg.square_lattice:
        r = int(round(cfg.shift_radius / s))
        idx = np.arange(-r, r + 1)
        pts = [(s * i, s * j) for j in idx for i in idx]
    else:
        r = int(math.floor(cfg.shift_radius / s + 1e-9))
        idx = np.arange(-r, r + 1)
        pts = [(s * i, s * j) for j in idx for i in idx
               if math.hypot(s * i, s * j) <= cfg.shift_radius + 1e-9]
    return np.asarray(pts, dtype=np.float64)


def delta_max(cfg: Config) -> float:
    """Radius D of the shift disc Omega_D.  tiny: the 7x7 square's half-diagonal."""
    if cfg.square_lattice:
        return cfg.shift_radius * math.sqrt(2.0)
    return cfg.shift_radius


def _unit_norm_scale(cx, cy, sig, amp) -> float:
    """1/||A||_L2 for A = sum_b amp_b exp(-|x-c_b|^2 / (2 sig_b^2)) (closed-form overlaps)."""
    dx = cx[:, None] - cx[None, :]
    dy = cy[:, None] - cy[None, :]
    s2 = sig[:, None] ** 2 + sig[None, :] ** 2
    ov = 2.0 * math.pi * (sig[:, None] ** 2) * (sig[None, :] ** 2) / s2 * np.exp(-(dx * dx + dy * dy) / (2.0 * s2))
    nrm2 = float(amp @ ov @ amp)
    return 1.0 / math.sqrt(nrm2)


def _draw_blobs(rng, cfg: Config):
    nb = cfg.n_blobs
    u = rng.random(nb)
    th = rng.random(nb) * 2.0 * math.pi
    r = cfg.center_radius * np.sqrt(u)
    cx, cy = r * np.cos(th), r * np.sin(th)
    sig = rng.uniform(1.5, 3.0, nb)
    amp = rng.standard_normal(nb)
    amp = amp * _unit_norm_scale(cx, cy, sig, amp)
    return cx, cy, sig, amp


def planted_truth(cfg: Config, item: int, n_shifts: int):
    """(j0, t0, r0) drawn for planted image `item` (stream 1)."""
    rng = np.random.default_rng([cfg.seed, 1, item, 7])
    return int(rng.integers(cfg.N_tm)), int(rng.integers(n_shifts)), int(rng.integers(cfg.n_psi))


def blob_params(cfg: Config, kind: str, items: Sequence[int], mode: str = "independent"):
    """Blob parameters for the given item indices.

    kind: "templates" or "images"; mode: "independent" or "planted".
    Returns dict of float64 arrays [len(items), n_blobs]: cx, cy, sigma, amp.
    Planted image i = T_{delta_t0} R_{gamma_r0} (template j0): centres -> R_{gamma0} c + delta0
    (the alignment peak is then at (-delta0, -gamma0)).
    """
    items = list(items)
    out = {k: np.empty((len(items), cfg.n_blobs)) for k in ("cx", "cy", "sigma", "amp")}
    shifts = shift_list(cfg) if (kind == "images" and mode == "planted") else None
    for row, it in enumerate(items):
        if kind == "templates":
            cx, cy, sig, amp = _draw_blobs(np.random.default_rng([cfg.seed, 0, it]), cfg)
        elif kind == "images" and mode == "independent":
            cx, cy, sig, amp = _draw_blobs(np.random.default_rng([cfg.seed, 1, it]), cfg)
        elif kind == "images" and mode == "planted":
            j0, t0, r0 = planted_truth(cfg, it, len(shifts))
            cx, cy, sig, amp = _draw_blobs(np.random.default_rng([cfg.seed, 0, j0]), cfg)
            g0 = 2.0 * math.pi * r0 / cfg.n_psi
            c, s = math.cos(g0), math.sin(g0)
            cx, cy = c * cx - s * cy + shifts[t0, 0], s * cx + c * cy + shifts[t0, 1]
        else:
            raise ValueError((kind, mode))
        out["cx"][row], out["cy"][row], out["sigma"][row], out["amp"][row] = cx, cy, sig, amp
    return out


def polar_samples(params, k_nodes, n_psi: int, backend: str = "numpy", device=None, chunk: int = 64):
    """Analytic polar Fourier samples Ahat(k_m, psi_p), psi_p = 2*pi*p/n_psi.

    Ahat(k) = sum_b amp_b 2 pi sig_b^2 exp(-sig_b^2 k^2 / 2) exp(-i k (c_x cos psi + c_y sin psi)).
    Returns complex64 [N_items, n_k, n_psi] (psi fastest); numpy array, or a torch
    tensor on `device` when backend == "torch" (evaluated in float64 there).
    """
    k = np.asarray(k_nodes, dtype=np.float64)
    psi = 2.0 * math.pi * np.arange(n_psi) / n_psi
    n_items = params["cx"].shape[0]
    if backend == "numpy":
        out = np.empty((n_items, k.size, n_psi), dtype=np.complex64)
        cos_p, sin_p = np.cos(psi), np.sin(psi)
        for s in range(0, n_items, chunk):
            e = slice(s, min(s + chunk, n_items))
            cx, cy = params["cx"][e], params["cy"][e]
            sig, amp = params["sigma"][e], params["amp"][e]
            proj = cx[:, :, None] * cos_p[None, None, :] + cy[:, :, None] * sin_p[None, None, :]  # [I,B,P]
            rad = amp[:, :, None] * 2.0 * math.pi * sig[:, :, None] ** 2 * np.exp(-0.5 * sig[:, :, None] ** 2 * k[None, None, :] ** 2)  # [I,B,M]
            ph = np.exp(-1j * k[None, None, :, None] * proj[:, :, None, :])  # [I,B,M,P]
            out[e] = np.einsum("ibm,ibmp->imp", rad, ph).astype(np.complex64)
        return out
    import torch
    dev = torch.device(device if device is not None else "cuda")
    kt = torch.as_tensor(k, device=dev)
    pt = torch.as_tensor(psi, device=dev)
    cos_p, sin_p = torch.cos(pt), torch.sin(pt)
    out = torch.empty((n_items, k.size, n_psi), dtype=torch.complex64, device=dev)
    for s in range(0, n_items, chunk):
        e = slice(s, min(s + chunk, n_items))
        cx = torch.as_tensor(params["cx"][e], device=dev)
        cy = torch.as_tensor(params["cy"][e], device=dev)
        sig = torch.as_tensor(params["sigma"][e], device=dev)
        amp = torch.as_tensor(params["amp"][e], device=dev)
        acc = torch.zeros((cx.shape[0], k.size, n_psi), dtype=torch.complex128, device=dev)
        for b in range(cx.shape[1]):
            proj = cx[:, b, None] * cos_p[None, :] + cy[:, b, None] * sin_p[None, :]          # [I,P]
            rad = amp[:, b, None] * 2.0 * math.pi * sig[:, b, None] ** 2 * torch.exp(-0.5 * sig[:, b, None] ** 2 * kt[None, :] ** 2)  # [I,M]
            ang = -kt[None, :, None] * proj[:, None, :]                                        # [I,M,P]
            acc += rad[:, :, None] * torch.polar(torch.ones_like(ang), ang)
        out[e] = acc.to(torch.complex64)
    return out


def add_noise(samples, cfg: Config, kind: str, items: Sequence[int], snr: Optional[float] = None,
              backend: str = "numpy", torch_seed: Optional[int] = None):
    """Add Hermitian-paired complex white noise in Fourier space, in place.

    Signal items have unit L2 norm, so the discrete bandlimited norm^2 is ~(2 pi)^2;
    noise per sample has E|n|^2 = s^2 with 2 pi s^2 sum_m w_m = (2 pi)^2 / SNR and
    sum_m w_m = k_max^2 / 2.  numpy: one rng per item (streams 2/3); torch: one
    device generator seeded from (cfg.seed, stream) -- a different realization.
    """
    snr = cfg.snr if snr is None else snr
    if not math.isfinite(snr):
        return samples
    stream = 2 if kind == "templates" else 3
    s2 = 4.0 * math.pi / (snr * cfg.k_max ** 2)
    sd = math.sqrt(s2 / 2.0)
    h = cfg.n_psi // 2
    items = list(items)
    if backend == "numpy":
        n_k = samples.shape[1]
        for row, it in enumerate(items):
            rng = np.random.default_rng([cfg.seed, stream, it])
            z = (rng.standard_normal((n_k, h)) + 1j * rng.standard_normal((n_k, h))) * sd
            samples[row, :, :h] += z.astype(np.complex64)
            samples[row, :, h:] += np.conj(z).astype(np.complex64)
        return samples
    import torch
    g = torch.Generator(device=samples.device)
    g.manual_seed(torch_seed if torch_seed is not None else (cfg.seed * 1000003 + stream))
    n_items, n_k = samples.shape[0], samples.shape[1]
    for s in range(0, n_items, 256):
        e = min(s + 256, n_items)
        zr = torch.randn((e - s, n_k, h), generator=g, device=samples.device, dtype=torch.float32) * sd
        zi = torch.randn((e - s, n_k, h), generator=g, device=samples.device, dtype=torch.float32) * sd
        z = torch.complex(zr, zi)
        samples[s:e, :, :h] += z
        samples[s:e, :, h:] += torch.conj(z)
    return samples


def draw_items(cfg: Config, kind: str, items: Sequence[int], k_nodes, mode: str = "independent",
               noise: bool = True, backend: str = "numpy", device=None):
    """Blob parameters -> analytic samples (+ noise).  Returns (samples, params)."""
    p = blob_params(cfg, kind, items, mode)
    x = polar_samples(p, k_nodes, cfg.n_psi, backend=backend, device=device)
    if noise:
        x = add_noise(x, cfg, kind, items, backend=backend)
    return x, p


def make_polar_set(cfg: Config, k_nodes, mode: str = "independent", noise: bool = True,
                   n_images: Optional[int] = None, n_templates: Optional[int] = None,
                   backend: str = "numpy", device=None):
    """Full (or truncated) image and template sets for a config."""
    ni = cfg.N_im if n_images is None else n_images
    nt = cfg.N_tm if n_templates is None else n_templates
    imgs, _ = draw_items(cfg, "images", range(ni), k_nodes, mode, noise, backend, device)
    tpls, _ = draw_items(cfg, "templates", range(nt), k_nodes, "independent", noise, backend, device)
    return imgs, tpls


def pixel_images(params, n: int, noise_sd: float = 0.0, seeds: Optional[Sequence] = None):
    """Blob images sampled at pixel centres: A[i][j] = sum_b amp_b exp(-((x_i - cx_b)^2 + (y_j - cy_b)^2) / 2 sig_b^2)
    with x_i = i - n/2, y_j = j - n/2 px (PAPER.md P:309-312 with the [-1, 1]^2 box in px units, DESIGN R23).
    Optional i.i.d. real Gaussian pixel noise of std `noise_sd` (one rng per item from `seeds`).
    Returns float32 [N_items, n, n] (i slow, j fast)."""
    x = np.arange(n, dtype=np.float64) - n / 2.0
    n_items = params["cx"].shape[0]
    out = np.empty((n_items, n, n), dtype=np.float32)
    for r in range(n_items):
        cx, cy, sig, amp = params["cx"][r], params["cy"][r], params["sigma"][r], params["amp"][r]
        gx = np.exp(-(x[None, :] - cx[:, None]) ** 2 / (2.0 * sig[:, None] ** 2))  # [B, n] over i
        gy = np.exp(-(x[None, :] - cy[:, None]) ** 2 / (2.0 * sig[:, None] ** 2))  # [B, n] over j
        img = np.einsum("b,bi,bj->ij", amp, gx, gy)
        if noise_sd > 0.0:
            img = img + noise_sd * np.random.default_rng(seeds[r]).standard_normal((n, n))
        out[r] = img.astype(np.float32)
    return out


def pixel_images_torch(params, n: int, noise_sd: float = 0.0, seed: int = 0, device=None, chunk: int = 256):
    """pixel_images on the GPU (torch, float64 arithmetic, float32 result); noise from one device
    generator seeded with `seed` (a different realization than the numpy path)."""
    import torch
    dev = torch.device(device if device is not None else "cuda")
    x = torch.arange(n, dtype=torch.float64, device=dev) - n / 2.0
    n_items = params["cx"].shape[0]
    out = torch.empty((n_items, n, n), dtype=torch.float32, device=dev)
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    for s0 in range(0, n_items, chunk):
        e = slice(s0, min(s0 + chunk, n_items))
        cx = torch.as_tensor(params["cx"][e], device=dev)
        cy = torch.as_tensor(params["cy"][e], device=dev)
        sig = torch.as_tensor(params["sigma"][e], device=dev)
        amp = torch.as_tensor(params["amp"][e], device=dev)
        gx = torch.exp(-(x[None, None, :] - cx[:, :, None]) ** 2 / (2.0 * sig[:, :, None] ** 2))  # [I, B, n]
        gy = torch.exp(-(x[None, None, :] - cy[:, :, None]) ** 2 / (2.0 * sig[:, :, None] ** 2))
        img = torch.einsum("ib,ibx,iby->ixy", amp, gx, gy)
        if noise_sd > 0.0:
            img = img + noise_sd * torch.randn(img.shape, generator=g, device=dev, dtype=torch.float64)
        out[e] = img.to(torch.float32)
    return out


def draw_pixel_items(cfg: Config, kind: str, items: Sequence[int], mode: str = "independent", noise: bool = True,
                     backend: str = "numpy", device=None):
    """Pixel images of the config's blob items (same blobs as draw_items) with pixel-domain white noise at
    the config's SNR (||noise||^2 = ||signal||^2 / SNR over the n x n samples; unit-norm signals).
    Returns (pixels float32 [N, n, n], params)."""
    p = blob_params(cfg, kind, items, mode)
    sd = 0.0
    if noise and math.isfinite(cfg.snr):
        sd = math.sqrt(1.0 / (cfg.snr * cfg.n * cfg.n))
    stream = 4 if kind == "templates" else 5
    if backend == "torch":
        return pixel_images_torch(p, cfg.n, sd, seed=cfg.seed * 1000003 + stream, device=device), p
    seeds = [[cfg.seed, stream, it] for it in items]
    return pixel_images(p, cfg.n, sd, seeds), p


def ctf_filters(k_nodes, defocus_A, pixel_A: float = 4.0, kv: float = 300.0, cs_mm: float = 2.7,
                amp_contrast: float = 0.07, bfactor_A2: float = 0.0):
    """Isotropic weak-phase CTFs (the model of Mindell & Grigorieff, which PAPER.md P:1397-1399 cites for
    the defocus parametrization) on radial nodes k [rad/px], one row per defocus [Angstrom]:
        c(s) = -(sqrt(1 - A^2) sin chi(s) + A cos chi(s)) exp(-B s^2 / 4),
        chi(s) = pi lambda dF s^2 - (pi/2) Cs lambda^3 s^4,   s = k / (2 pi pixel_A)  [1/Angstrom],
    lambda the relativistic electron wavelength at kv.  An INPUT generator (the filters are inputs of
    the CTF-parameterized kernel, reading R24); nothing of the method's arithmetic lives here."""
    k = np.asarray(k_nodes, dtype=np.float64)
    V = kv * 1e3
    lam = 12.2643247 / math.sqrt(V * (1.0 + 0.978466e-6 * V))
    cs = cs_mm * 1e7
    s = k / (2.0 * math.pi * pixel_A)
    out = []
    for df in np.atleast_1d(np.asarray(defocus_A, dtype=np.float64)):
        chi = math.pi * lam * df * s ** 2 - 0.5 * math.pi * cs * lam ** 3 * s ** 4
        c = -(math.sqrt(1.0 - amp_contrast ** 2) * np.sin(chi) + amp_contrast * np.cos(chi))
        out.append(c * np.exp(-bfactor_A2 * s ** 2 / 4.0))
    return np.stack(out)
