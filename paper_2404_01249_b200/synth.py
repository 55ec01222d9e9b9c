"""Seeded synthetic inputs for the BASELINE.json configs.

The paper's datasets (Klein brain MRI, EMPIRE10 lung CT, RnR-ExM) are not
available; these generators stand in for them with the shapes, sizes and value
distributions BASELINE.json names.  They are NOT the reference's own
generators (synth.cpp) — SURVEY.md §8(d) says those must not be substituted.

Every volume is returned as float32 (the reference reads MET_FLOAT volumes,
io.cpp:245-269) in numpy (z, y, x) order, i.e. x-fastest memory.

Moving images follow the shared recipe: velocity v = N(0,1) noise per
component, Gaussian-smoothed with sigma 8 (periodic boundary, so the field is
stationary and its maximum is not an edge artefact), scaled so that max |v| over
all voxels and components equals the stated maximum displacement (BASELINE's
"max N-voxel displacement" is applied to the velocity — documented ambiguity),
then integrated by 6 scaling-and-squaring steps; moving = fixed o exp(v).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
from scipy import ndimage

from ._abi import GridMeta, PyramidSchedule, RegistrationConfig, LOSS_LNCC, LOSS_SSD


def _coords(shape):
    return np.meshgrid(*[np.arange(s, dtype=np.float64) for s in shape], indexing="ij")


def _sample(vol, pts):
    """trilinear, clamp-to-edge sample of a (z,y,x) volume at (z,y,x) points"""
    return ndimage.map_coordinates(vol, pts, order=1, mode="nearest")


def exp_velocity(v: np.ndarray, steps: int = 6) -> np.ndarray:
    """scaling and squaring of v (z,y,x,3 with xyz components) -> displacement"""
    u = v / float(2 ** steps)
    zz, yy, xx = _coords(v.shape[:3])
    for _ in range(steps):
        pts = np.stack([zz + u[..., 2], yy + u[..., 1], xx + u[..., 0]])
        u = u + np.stack([_sample(u[..., c], pts) for c in range(3)], axis=-1)
    return u


def _taper(shape, margin: float):
    """separable raised-cosine window: 0 on the faces, 1 beyond `margin` voxels"""
    w = np.ones(shape)
    for a, n in enumerate(shape):
        i = np.arange(n, dtype=np.float64)
        d = np.minimum(i, n - 1 - i)
        t = 0.5 * (1.0 - np.cos(np.pi * np.clip(d / margin, 0.0, 1.0)))
        sh = [1] * len(shape)
        sh[a] = n
        w = w * t.reshape(sh)
    return w


def random_velocity(shape, max_disp: float, rng: np.random.Generator,
                    sigma: float = 8.0) -> np.ndarray:
    """smoothed N(0,1) noise, tapered to zero over 2 sigma at the volume faces
    (the deformation lives inside the field of view, as in the reference's own
    warp generator, synth.hpp:10-14), max |v| = max_disp"""
    w = _taper(shape, min(2.0 * sigma, min(shape) / 4.0))
    v = np.stack([w * ndimage.gaussian_filter(rng.standard_normal(shape), sigma, mode="wrap")
                  for _ in range(3)], axis=-1)
    return v * (max_disp / np.abs(v).max())


def warp(vol: np.ndarray, u: np.ndarray, order: int = 1) -> np.ndarray:
    zz, yy, xx = _coords(vol.shape)
    pts = np.stack([zz + u[..., 2], yy + u[..., 1], xx + u[..., 0]])
    return ndimage.map_coordinates(vol, pts, order=order, mode="nearest")


@dataclass
class Pair:
    grid: GridMeta
    fixed: np.ndarray           # float32 (z,y,x)
    moving: np.ndarray          # float32
    fixed_labels: np.ndarray    # int32
    moving_labels: np.ndarray   # int32
    truth: np.ndarray           # float64 (z,y,x,3) displacement used for moving
    config: RegistrationConfig
    schedule: PyramidSchedule
    name: str


def _normalise(img):
    lo, hi = img.min(), img.max()
    return (img - lo) / (hi - lo)


def blobs_phantom(shape, rng, n_blobs=12, n_classes=4):
    """config 0: sum of Gaussian blobs + N(0, 0.01), normalised to [0,1]."""
    zz, yy, xx = _coords(shape)
    nz, ny, nx = shape
    cls = np.zeros((n_classes,) + tuple(shape))
    img = np.zeros(shape)
    for k in range(n_blobs):
        c = rng.uniform([0, 0, 0], [nz, ny, nx])
        s = rng.uniform(4.0, 10.0)
        a = rng.uniform(0.3, 1.0)
        b = a * np.exp(-((zz - c[0]) ** 2 + (yy - c[1]) ** 2 + (xx - c[2]) ** 2) / (2 * s * s))
        img += b
        cls[k % n_classes] += b
    img += rng.normal(0.0, 0.01, shape)
    labels = (np.argmax(cls, axis=0) + 1).astype(np.int32)
    labels[cls.max(axis=0) < 0.1] = 0
    return _normalise(img), labels


def head_phantom(shape, rng, n_struct=35):
    """config 1/2: nested ellipsoid shells 0.2/0.5/0.8, bias field, ~35 blob
    structures as labels, N(0, 0.02) noise."""
    zz, yy, xx = _coords(shape)
    nz, ny, nx = shape
    cz, cy, cx = (nz - 1) / 2, (ny - 1) / 2, (nx - 1) / 2
    r = np.sqrt(((zz - cz) / (0.46 * nz)) ** 2 + ((yy - cy) / (0.46 * ny)) ** 2 +
                ((xx - cx) / (0.44 * nx)) ** 2)
    img = np.zeros(shape)
    img[r < 1.0] = 0.2
    img[r < 0.88] = 0.5
    img[r < 0.6] = 0.8
    labels = np.zeros(shape, dtype=np.int32)
    for k in range(n_struct):
        while True:
            c = rng.uniform([0.2 * nz, 0.2 * ny, 0.2 * nx], [0.8 * nz, 0.8 * ny, 0.8 * nx])
            rr = np.sqrt(((c[0] - cz) / (0.46 * nz)) ** 2 + ((c[1] - cy) / (0.46 * ny)) ** 2 +
                         ((c[2] - cx) / (0.44 * nx)) ** 2)
            if rr < 0.8:
                break
        ax = rng.uniform(3.0, 9.0, 3)
        d = ((zz - c[0]) / ax[0]) ** 2 + ((yy - c[1]) / ax[1]) ** 2 + ((xx - c[2]) / ax[2]) ** 2
        m = d < 1.0
        labels[m] = k + 1
        img[m] += rng.uniform(-0.25, 0.25)
    bias = 1.0 + 0.15 * (np.sin(zz / nz * np.pi * rng.uniform(0.5, 1.5)) *
                         np.cos(xx / nx * np.pi * rng.uniform(0.5, 1.5)))
    img = ndimage.gaussian_filter(img, 0.8) * bias
    img += rng.normal(0.0, 0.02, shape)
    return img, labels


def torso_phantom(shape, rng, n_tubes=300):
    """config 3: torso with a low-intensity lung cavity and random-walk vessel
    tubes (radius 1-3 voxels)."""
    zz, yy, xx = _coords(shape)
    nz, ny, nx = shape
    c = np.array([(nz - 1) / 2, (ny - 1) / 2, (nx - 1) / 2])
    body = ((yy - c[1]) / (0.45 * ny)) ** 2 + ((xx - c[2]) / (0.47 * nx)) ** 2 < 1.0
    lung = (((zz - c[0]) / (0.42 * nz)) ** 2 + ((yy - c[1]) / (0.33 * ny)) ** 2 +
            ((xx - c[2]) / (0.38 * nx)) ** 2) < 1.0
    img = np.where(body, 0.7, 0.0)
    img[lung] = 0.1
    vessels = np.zeros(shape)
    for _ in range(n_tubes):
        p = c + rng.uniform(-0.3, 0.3, 3) * np.array(shape)
        d = rng.standard_normal(3)
        d /= np.linalg.norm(d)
        rad = rng.uniform(1.0, 3.0)
        for _ in range(int(rng.integers(10, 40))):
            zi, yi, xi = np.clip(np.round(p).astype(int), 0, np.array(shape) - 1)
            vessels[zi, yi, xi] = max(vessels[zi, yi, xi], rad)
            d += 0.3 * rng.standard_normal(3)
            d /= np.linalg.norm(d)
            p = p + 2.0 * d
    tube = ndimage.grey_dilation(vessels, size=(5, 5, 5)) > 0
    img[tube & lung] = 0.6
    img = ndimage.gaussian_filter(img, 1.0) + rng.normal(0.0, 0.01, shape)
    labels = np.zeros(shape, dtype=np.int32)
    labels[body] = 1
    labels[lung] = 2
    labels[tube & lung] = 3
    return img, labels


CONFIGS = {
    0: dict(shape=(64, 64, 64), max_disp=3.0, scales=(4.0, 2.0, 1.0), iters=(200, 100, 50),
            loss=LOSS_LNCC, radius=2, sigma_grad=1.0, name="cfg0_64cube_blobs_lncc5"),
    1: dict(shape=(224, 192, 160), max_disp=6.0, scales=(4.0, 2.0, 1.0), iters=(200, 100, 50),
            loss=LOSS_LNCC, radius=2, sigma_grad=1.0, name="cfg1_160x192x224_head_lncc5"),
    3: dict(shape=(208, 192, 192), max_disp=10.0, scales=(4.0, 2.0, 1.0), iters=(250, 150, 75),
            loss=LOSS_SSD, radius=2, sigma_grad=1.5, name="cfg3_192x192x208_torso_mse"),
}


def baseline_config(loss=LOSS_LNCC, radius=2, sigma_grad=1.0, conv_window=None,
                    max_iters=0) -> RegistrationConfig:
    """BASELINE optimiser settings: eta 0.5, beta 0.9/0.99, sigma_warp 0.5,
    early stopping off (conv_window > max iterations)."""
    return RegistrationConfig(loss=loss, lncc_radius=radius, eta=0.5, sigma_grad=sigma_grad,
                              sigma_warp=0.5, beta1=0.9, beta2=0.99, eps_adam=1e-8,
                              step_cap=0.5,
                              conv_window=conv_window if conv_window else max_iters + 1,
                              conv_tol=1e-5)


def make_pair(config: int = 0, seed: int = 0, shape=None, iters=None) -> Pair:
    spec = CONFIGS[config]
    shape = tuple(shape or spec["shape"])
    rng = np.random.default_rng(np.random.SeedSequence([20240401, config, seed]))
    if config == 0:
        fixed, labels = blobs_phantom(shape, rng)
    elif config in (1, 2):
        fixed, labels = head_phantom(shape, rng)
    elif config == 3:
        fixed, labels = torso_phantom(shape, rng)
    else:
        raise ValueError(f"no generator for config {config}")
    v = random_velocity(shape, spec["max_disp"], rng)
    u = exp_velocity(v)
    if config == 3:  # affine breathing scale along z about the centre
        s = rng.uniform(0.9, 1.1)
        zc = (shape[0] - 1) / 2
        zz = _coords(shape)[0]
        u[..., 2] += (s - 1.0) * (zz - zc)
    moving = warp(fixed, u)
    mlabels = warp(labels.astype(np.float64), u, order=0).astype(np.int32)
    it = tuple(iters or spec["iters"])
    cfg = baseline_config(spec["loss"], spec["radius"], spec["sigma_grad"], max_iters=max(it))
    grid = GridMeta.make_3d(shape[2], shape[1], shape[0])
    return Pair(grid, fixed.astype(np.float32), moving.astype(np.float32), labels, mlabels,
                u, cfg, PyramidSchedule(spec["scales"], it), spec["name"])
