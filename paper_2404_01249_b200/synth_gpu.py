"""BASELINE config 4 stand-in generated on the device (torch): a microscopy-like
1024^3 fp32 volume — 200k Gaussian puncta (sigma 1-2 voxels, seeded) on a
smooth background with Poisson-like noise — and the moving image made by the
same diffeomorphism recipe as configs 0-3 (velocity N(0,1) smoothed with
sigma 8, tapered at the faces, scaled to 8 voxels max, 6 scaling-and-squaring
steps).  At 1024^3 the numpy recipe of synth.py would need ~100 GB of host
memory, so this one runs on the GPU; it follows the same steps.

Data synthesis only (benchmark / test input); the registration itself runs
through the library.
"""
from __future__ import annotations

import math

import torch
import torch.nn.functional as Fnn


def _gauss_taps(sigma: float, device) -> torch.Tensor:
    r = int(math.ceil(3 * sigma))
    j = torch.arange(-r, r + 1, device=device, dtype=torch.float32)
    t = torch.exp(-0.5 * (j / sigma) ** 2)
    return t / t.sum()


def _smooth_axis(v: torch.Tensor, taps: torch.Tensor, axis: int, circular: bool) -> torch.Tensor:
    """1-D convolution of a (D, H, W) volume along `axis` (0=z, 1=y, 2=x)."""
    r = (taps.numel() - 1) // 2
    x = v.movedim(axis, -1)
    sh = x.shape
    x = x.reshape(-1, 1, sh[-1])
    out = torch.empty_like(x)
    step = 1 << 16  # rows per chunk keeps the padded copy small
    for a in range(0, x.shape[0], step):
        blk = x[a:a + step]
        blk = Fnn.pad(blk, (r, r), mode="circular" if circular else "constant")
        out[a:a + step] = Fnn.conv1d(blk, taps.view(1, 1, -1))
    return out.reshape(sh).movedim(-1, axis)


def smooth(v: torch.Tensor, sigma: float, circular: bool = False) -> torch.Tensor:
    taps = _gauss_taps(sigma, v.device)
    for a in range(3):
        v = _smooth_axis(v, taps, a, circular)
    return v


def _taper(shape, margin: float, device) -> list:
    out = []
    for n in shape:
        i = torch.arange(n, device=device, dtype=torch.float32)
        d = torch.minimum(i, n - 1 - i)
        out.append(0.5 * (1.0 - torch.cos(math.pi * torch.clamp(d / margin, 0.0, 1.0))))
    return out


def _grid(shape, device):
    """identity sampling grid in grid_sample's normalised (x, y, z) order."""
    d, h, w = shape
    zs = torch.linspace(-1, 1, d, device=device)
    ys = torch.linspace(-1, 1, h, device=device)
    xs = torch.linspace(-1, 1, w, device=device)
    return zs, ys, xs


def warp(vol: torch.Tensor, u: torch.Tensor, chunk: int = 64) -> torch.Tensor:
    """vol (D,H,W[,C]) sampled at x + u (u: (D,H,W,3) voxel units, xyz), trilinear,
    clamp-to-edge (align_corners grid == voxel centres), by z-chunks."""
    d, h, w = u.shape[:3]
    multi = vol.dim() == 4
    src = (vol.permute(3, 0, 1, 2) if multi else vol.unsqueeze(0)).unsqueeze(0)
    out = torch.empty_like(vol)
    sx, sy, sz = 2.0 / (w - 1), 2.0 / (h - 1), 2.0 / (d - 1)
    xs = torch.arange(w, device=u.device, dtype=torch.float32)
    ys = torch.arange(h, device=u.device, dtype=torch.float32)
    for z0 in range(0, d, chunk):
        z1 = min(d, z0 + chunk)
        zz = torch.arange(z0, z1, device=u.device, dtype=torch.float32)
        uc = u[z0:z1]
        g = torch.empty((1, z1 - z0, h, w, 3), device=u.device, dtype=torch.float32)
        g[0, ..., 0] = (xs.view(1, 1, w) + uc[..., 0]) * sx - 1
        g[0, ..., 1] = (ys.view(1, h, 1) + uc[..., 1]) * sy - 1
        g[0, ..., 2] = (zz.view(-1, 1, 1) + uc[..., 2]) * sz - 1
        r = Fnn.grid_sample(src, g, mode="bilinear", padding_mode="border", align_corners=True)
        if multi:
            out[z0:z1] = r[0].permute(1, 2, 3, 0)
        else:
            out[z0:z1] = r[0, 0]
        del g, r
    return out


def random_velocity(shape, max_disp: float, gen: torch.Generator, device,
                    sigma: float = 8.0) -> torch.Tensor:
    tz, ty, tx = _taper(shape, min(2.0 * sigma, min(shape) / 4.0), device)
    w = tz.view(-1, 1, 1) * ty.view(1, -1, 1) * tx.view(1, 1, -1)
    v = torch.empty(tuple(shape) + (3,), device=device, dtype=torch.float32)
    for c in range(3):
        n = torch.randn(tuple(shape), generator=gen, device=device, dtype=torch.float32)
        v[..., c] = smooth(n, sigma, circular=True) * w
        del n
    return v * (max_disp / v.abs().max())


def exp_velocity(v: torch.Tensor, steps: int = 6) -> torch.Tensor:
    u = v / float(2 ** steps)
    for _ in range(steps):
        u = u + warp(u, u)
    return u


def puncta_phantom(shape, gen: torch.Generator, device, n_puncta: int = 200_000,
                   sigma_bins=(1.0, 1.25, 1.5, 1.75, 2.0)) -> torch.Tensor:
    """Gaussian puncta (sigma in [1, 2], amplitude U[0.5, 1]) rendered as
    weighted deltas blurred per sigma bin, on a smooth background, with
    Poisson-like noise; normalised to [0, 1]."""
    d, h, w = shape
    img = torch.zeros(shape, device=device, dtype=torch.float32)
    pos = torch.rand((n_puncta, 3), generator=gen, device=device)
    pos = (pos * torch.tensor([d - 1, h - 1, w - 1], device=device)).round().long()
    amp = 0.5 + 0.5 * torch.rand(n_puncta, generator=gen, device=device)
    sig = 1.0 + torch.rand(n_puncta, generator=gen, device=device)
    edges = list(sigma_bins)
    for b in range(len(edges) - 1):
        sel = (sig >= edges[b]) & (sig < edges[b + 1] if b < len(edges) - 2 else sig <= edges[b + 1])
        if not bool(sel.any()):
            continue
        s_mid = 0.5 * (edges[b] + edges[b + 1])
        delta = torch.zeros(shape, device=device, dtype=torch.float32)
        idx = (pos[sel, 0] * h + pos[sel, 1]) * w + pos[sel, 2]
        delta.view(-1).index_add_(0, idx, amp[sel])
        peak = (2 * math.pi * s_mid ** 2) ** 1.5  # unit-peak puncta after the normalised blur
        img += smooth(delta, s_mid) * peak
        del delta
    bg = torch.randn((16, 16, 16), generator=gen, device=device)
    bg = Fnn.interpolate(bg.view(1, 1, 16, 16, 16), size=tuple(shape), mode="trilinear",
                         align_corners=True)[0, 0]
    img += 0.15 + 0.05 * bg
    img.clamp_(min=0.0)
    k = 200.0  # Poisson-like noise: counts at ~200 per unit intensity
    img = torch.poisson(img * k, generator=gen) / k
    lo, hi = img.min(), img.max()
    return (img - lo) / (hi - lo)


def make_config4_pair(device="cuda", seed: int = 0, shape=(1024, 1024, 1024),
                      n_puncta: int = 200_000, max_disp: float = 8.0):
    """(fixed, moving) as (D, H, W) fp32 device tensors."""
    gen = torch.Generator(device=device)
    gen.manual_seed(20240401 * 10 + 4 * 1000 + seed)
    fixed = puncta_phantom(shape, gen, device, n_puncta=n_puncta)
    v = random_velocity(shape, max_disp, gen, device)
    u = exp_velocity(v)
    del v
    moving = warp(fixed, u)
    del u
    return fixed, moving
