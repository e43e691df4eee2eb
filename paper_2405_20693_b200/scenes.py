"""Synthetic workloads of BASELINE.json, generated on the host
with NumPy/SciPy. These are data generators for the benchmark and tests, not
compute paths: the same fixture feeds the engine and the CPU reference.

  phantom            Shepp-Logan 3D (simulator.cpp:14-69, Kak & Slaney modified)
  sample_init_cloud  fdk.cpp:203-247 on the phantom (documented deviation: the
                     phantom stands in for the FDK volume; NumPy PCG64 instead
                     of std::mt19937_64, so the draw differs from the C++ one)
  trained_like       per-axis scale *= exp(0.5 N(0,1)) and random rotations, so
                     that anisotropy and the quaternion chain are exercised
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

# simulator.cpp:16-27 (intensity, a, b, c, x0, y0, z0, phi)
SHEPP_LOGAN = [
    (1.0, 0.690, 0.920, 0.810, 0.0, 0.0, 0.0, 0.0),
    (-0.8, 0.6624, 0.874, 0.780, 0.0, -0.0184, 0.0, 0.0),
    (-0.2, 0.110, 0.310, 0.220, 0.22, 0.0, 0.0, -18.0 * math.pi / 180.0),
    (-0.2, 0.160, 0.410, 0.280, -0.22, 0.0, 0.0, 18.0 * math.pi / 180.0),
    (0.1, 0.210, 0.250, 0.410, 0.0, 0.35, -0.15, 0.0),
    (0.1, 0.046, 0.046, 0.050, 0.0, 0.10, 0.25, 0.0),
    (0.1, 0.046, 0.046, 0.050, 0.0, -0.10, 0.25, 0.0),
    (0.1, 0.046, 0.023, 0.050, -0.08, -0.605, 0.0, 0.0),
    (0.1, 0.023, 0.023, 0.020, 0.0, -0.606, 0.0, 0.0),
    (0.1, 0.023, 0.046, 0.020, 0.06, -0.605, 0.0, 0.0),
]


def phantom(n: int, lo=(-1.0, -1.0, -1.0), hi=(1.0, 1.0, 1.0)) -> np.ndarray:
    """phantom_shepp_logan_3d(N^3) -> float32 [Z][Y][X] (x-fastest)."""
    lo = np.asarray(lo, dtype=np.float64)
    hi = np.asarray(hi, dtype=np.float64)
    sp = (hi - lo) / n
    center = 0.5 * (lo + hi)
    half = 0.5 * (hi - lo)
    c = [(lo[k] + (np.arange(n) + 0.5) * sp[k] - center[k]) / half[k] for k in range(3)]
    vol = np.zeros((n, n, n), dtype=np.float32)
    X, Y = np.meshgrid(c[0], c[1], indexing="xy")  # [Y][X]
    for z in range(n):
        zz = c[2][z]
        acc = np.zeros((n, n), dtype=np.float64)
        for inten, a, b, cc, x0, y0, z0, phi in SHEPP_LOGAN:
            dx, dy, dz = X - x0, Y - y0, zz - z0
            co, si = math.cos(phi), math.sin(phi)
            xr = co * dx + si * dy
            yr = -si * dx + co * dy
            q = xr * xr / (a * a) + yr * yr / (b * b) + dz * dz / (cc * cc)
            acc += np.where(q <= 1.0, inten, 0.0)
        vol[z] = acc
    return vol


def sample_trilinear(vol: np.ndarray, lo, spacing, pts: np.ndarray) -> np.ndarray:
    """voxelizer.cpp:16-37 vectorised; vol [Z][Y][X], pts [n,3] (x,y,z)."""
    dims = np.array([vol.shape[2], vol.shape[1], vol.shape[0]])
    g = (pts - np.asarray(lo)) / np.asarray(spacing) - 0.5
    c = np.clip(g, 0.0, dims - 1.0)
    ix = np.minimum(np.floor(c).astype(np.int64), dims - 1)
    f1 = np.minimum(ix + 1, dims - 1)
    w = c - ix
    out = np.zeros(len(pts))
    for dz in (0, 1):
        for dy in (0, 1):
            for dx in (0, 1):
                wt = (w[:, 0] if dx else 1 - w[:, 0]) * (w[:, 1] if dy else 1 - w[:, 1]) * (w[:, 2] if dz else 1 - w[:, 2])
                xi = f1[:, 0] if dx else ix[:, 0]
                yi = f1[:, 1] if dy else ix[:, 1]
                zi = f1[:, 2] if dz else ix[:, 2]
                out += wt * vol[zi, yi, xi]
    return out


def act_density_inv(rho):  # gaussian_cloud.cpp:15-20
    rho = np.asarray(rho, dtype=np.float64)
    return np.where(rho > 30.0, rho, rho + np.log1p(-np.exp(-np.minimum(rho, 30.0))))


def act_scale_inv(s, s_min):  # gaussian_cloud.cpp:30-34
    return np.log(np.asarray(s, dtype=np.float64) - s_min)


@dataclass
class CloudArrays:
    """Raw parameter arrays in the reference's field order (float32, like the .ckpt payload)."""
    s_min: float
    rho_raw: np.ndarray
    pos: np.ndarray
    scale_raw: np.ndarray
    rot: np.ndarray

    @property
    def m(self):
        return int(self.rho_raw.shape[0])

    def as_float64(self):
        return tuple(np.ascontiguousarray(a, dtype=np.float64) for a in (self.rho_raw, self.pos, self.scale_raw,
                                                                          self.rot))


def _raw(s_min, rho, pos, scale, rot) -> CloudArrays:
    q = np.asarray(rot, dtype=np.float64)
    q = q / np.sqrt((q * q).sum(axis=1, keepdims=True))
    f = lambda a: np.ascontiguousarray(np.asarray(a, dtype=np.float32).reshape(-1))
    return CloudArrays(float(s_min), f(act_density_inv(rho)), f(pos), f(act_scale_inv(scale, s_min)), f(q))


def sample_init_cloud(vol: np.ndarray, lo, hi, count: int, tau=0.05, k=0.15, s_min=2e-4, seed=0):
    """fdk.cpp:203-247 on a density volume [Z][Y][X]."""
    from scipy.spatial import cKDTree

    rng = np.random.default_rng(seed)
    n = np.array([vol.shape[2], vol.shape[1], vol.shape[0]])
    lo = np.asarray(lo, dtype=np.float64)
    sp = (np.asarray(hi, dtype=np.float64) - lo) / n
    occ = np.flatnonzero(vol.reshape(-1) > tau)
    if occ.size < count:
        raise ValueError(f"init: only {occ.size} voxels above the density threshold, need {count}")
    pick = rng.choice(occ, size=count, replace=False)
    x = pick % n[0]
    y = (pick // n[0]) % n[1]
    z = pick // (n[0] * n[1])
    pos = lo + (np.stack([x, y, z], axis=1) + 0.5) * sp
    pos += rng.uniform(-0.5, 0.5, size=pos.shape) * sp
    d, _ = cKDTree(pos).query(pos, k=2)
    s = np.maximum(d[:, 1], s_min * (1.0 + 1e-6))
    rho = np.maximum(k * sample_trilinear(vol, lo, sp, pos), 1e-6)
    scale = np.repeat(s[:, None], 3, axis=1)
    rot = np.tile([1.0, 0.0, 0.0, 0.0], (count, 1))
    return rho, pos, scale, rot


def trained_like(rho, pos, scale, rot, s_min, seed=1):
    rng = np.random.default_rng(seed)
    scale = scale * np.exp(0.5 * rng.standard_normal(scale.shape))
    scale = np.maximum(scale, s_min * (1.0 + 1e-6))
    rot = rng.standard_normal((len(rho), 4))
    rot /= np.linalg.norm(rot, axis=1, keepdims=True)
    return rho, pos, scale, rot


def random_cloud(count, pos_radius=0.35, scale_min=0.05, scale_max=0.2, s_min=2e-4, seed=0) -> CloudArrays:
    """tests/helpers.hpp:30-48 analogue (NumPy RNG)."""
    rng = np.random.default_rng(seed)
    rho = rng.uniform(0.2, 1.5, count)
    pos = rng.uniform(-pos_radius, pos_radius, (count, 3))
    scale = rng.uniform(scale_min, scale_max, (count, 3))
    rot = rng.standard_normal((count, 4))
    return _raw(s_min, rho, pos, scale, rot)


# ---------------------------------------------------------------- BASELINE.json configurations
@dataclass
class Workload:
    name: str
    n_vox: int
    m: int
    n_views: int
    res: int
    description: str


CONFIGS = {
    1: Workload("cfg1", 64, 10_000, 25, 128, "Shepp-Logan 64^3, 10k Gaussians, 25 cone-beam views at 128x128"),
    2: Workload("cfg2", 128, 50_000, 50, 256, "128^3 phantom, 50k Gaussians, 50 views at 256x256 (train step)"),
    3: Workload("cfg3", 256, 100_000, 75, 512, "256^3 phantom, 100k Gaussians, 75 cone-beam views at 512x512"),
    4: Workload("cfg4", 256, 200_000, 0, 0, "256^3 grid, 200k Gaussians, voxelizer fwd/bwd"),
    5: Workload("cfg5", 512, 1_000_000, 100, 1024, "512^3, 1M Gaussians, 100 views at 1024x1024"),
}


def make_cloud(cfg: int, seed=0, s_min=2e-4, vol=None) -> CloudArrays:
    w = CONFIGS[cfg]
    if vol is None:
        vol = phantom(w.n_vox)
    rho, pos, scale, rot = sample_init_cloud(vol, (-1, -1, -1), (1, 1, 1), w.m, s_min=s_min, seed=seed)
    rho, pos, scale, rot = trained_like(rho, pos, scale, rot, s_min, seed=seed + 1)
    return _raw(s_min, rho, pos, scale, rot)
