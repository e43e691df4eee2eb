"""Fixture generation on the device — the reference's
simulator.hpp / fdk.hpp API over the C ABI (csrc/fixtures.cu):

  phantom_shepp_logan_3d / phantom_from_ellipsoids   simulator.cpp:14-69
  project_volume                                      simulator.cpp:109-132
  add_noise (host, reference RNG streams)             simulator.cpp:134-158
  simulate_projections                                simulator.cpp:166-189
  fdk_reconstruct                                     fdk.cpp:53-134
  nearest_neighbor_distances                          fdk.cpp:136-201
  sample_init_cloud                                   fdk.cpp:203-247
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional, Sequence, Union

import numpy as np
import torch

from . import _capi
from .engine import Engine, GaussianCloud, GridSpec, ScannerConfig, _check, _ptr, default_engine, grid_for_extent

# simulator.cpp:16-29 (Kak & Slaney 3D, modified intensities):
# intensity, a, b, c, x0, y0, z0, phi_rad
SHEPP_LOGAN_3D = np.array([
    [1.0, 0.690, 0.920, 0.810, 0.0, 0.0, 0.0, 0.0],
    [-0.8, 0.6624, 0.874, 0.780, 0.0, -0.0184, 0.0, 0.0],
    [-0.2, 0.110, 0.310, 0.220, 0.22, 0.0, 0.0, -18.0 * np.pi / 180.0],
    [-0.2, 0.160, 0.410, 0.280, -0.22, 0.0, 0.0, 18.0 * np.pi / 180.0],
    [0.1, 0.210, 0.250, 0.410, 0.0, 0.35, -0.15, 0.0],
    [0.1, 0.046, 0.046, 0.050, 0.0, 0.10, 0.25, 0.0],
    [0.1, 0.046, 0.046, 0.050, 0.0, -0.10, 0.25, 0.0],
    [0.1, 0.046, 0.023, 0.050, -0.08, -0.605, 0.0, 0.0],
    [0.1, 0.023, 0.023, 0.020, 0.0, -0.606, 0.0, 0.0],
    [0.1, 0.023, 0.046, 0.020, 0.06, -0.605, 0.0, 0.0],
], dtype=np.float64)

RAMP, HANN, AUTO = 0, 1, 2  # fdk.hpp RampWindow


@dataclass
class NoiseParams:  # simulator.hpp:43-47
    i0: float = 1e5
    gauss_sigma: float = 10.0
    seed: int = 0


def _eng(engine: Optional[Engine]) -> Engine:
    return engine if engine is not None else default_engine()


def _thetas(theta: Union[float, Sequence[float]]):
    single = isinstance(theta, (int, float))
    th = [float(theta)] if single else [float(t) for t in theta]
    return single, th, (C.c_double * max(1, len(th)))(*th)


def phantom_from_ellipsoids(ellipsoids, dims, lo=(-1.0, -1.0, -1.0), hi=(1.0, 1.0, 1.0),
                            engine: Optional[Engine] = None):
    """Returns (volume [Z][Y][X] float32 device tensor, GridSpec)."""
    eng = _eng(engine)
    e = np.ascontiguousarray(ellipsoids, np.float64).reshape(-1, 8)
    vol = torch.empty((dims[2], dims[1], dims[0]), dtype=torch.float32, device=eng.device)
    _check(eng.lib.sct_phantom(eng._h, e.shape[0], e.ctypes.data_as(_capi.D),
                               (C.c_double * 3)(*[float(x) for x in lo]), (C.c_double * 3)(*[float(x) for x in hi]),
                               (C.c_int32 * 3)(*[int(x) for x in dims]), _ptr(vol)))
    return vol, grid_for_extent(lo, hi, dims)


def phantom_shepp_logan_3d(dims, lo=(-1.0, -1.0, -1.0), hi=(1.0, 1.0, 1.0), engine: Optional[Engine] = None):
    return phantom_from_ellipsoids(SHEPP_LOGAN_3D, dims, lo, hi, engine)


def project_volume(vol: torch.Tensor, grid: GridSpec, config: ScannerConfig, theta_rad, step_mm: float,
                   engine: Optional[Engine] = None) -> torch.Tensor:
    """Clean log-domain projections [n][H][W] (or [H][W] for a scalar angle)."""
    eng = _eng(engine)
    if tuple(vol.shape) != grid.shape_zyx:
        from .engine import DimMismatch
        raise DimMismatch("project_volume: volume dims differ from the grid")
    single, th, arr = _thetas(theta_rad)
    v = vol.to(device=eng.device, dtype=torch.float32).contiguous()
    out = torch.empty((len(th), config.height, config.width), dtype=torch.float32, device=eng.device)
    g, sc = grid._c(), config._c()
    _check(eng.lib.sct_project_volume(eng._h, _ptr(v), C.byref(g), C.byref(sc), arr, len(th), float(step_mm),
                                      _ptr(out)))
    return out[0] if single else out


def add_noise(images, noise: NoiseParams, view0: int = 0) -> torch.Tensor:
    """Poisson + Gaussian detector noise on the host with the reference's per-view
    std::mt19937_64 streams (view v of the batch uses view_rng(seed, view0 + v))."""
    src = images if isinstance(images, torch.Tensor) else torch.as_tensor(np.asarray(images, np.float32))
    single = src.dim() == 2
    h = src.detach().to("cpu", torch.float32).contiguous().clone()
    if single:
        h = h.unsqueeze(0)
    lib = _capi.load()
    _check(lib.sct_add_noise_host(C.c_void_p(h.data_ptr()), h.shape[0], h.shape[2], h.shape[1], float(noise.i0),
                                  float(noise.gauss_sigma), int(noise.seed) & ((1 << 64) - 1), int(view0)))
    return h[0] if single else h


def simulate_projections(phantom: torch.Tensor, grid: GridSpec, config: ScannerConfig, thetas: Sequence[float],
                         step_mm: float, noise: NoiseParams = NoiseParams(), apply_noise: bool = True,
                         engine: Optional[Engine] = None) -> torch.Tensor:
    """simulator.cpp:166-189: device tensor [n][H][W]."""
    eng = _eng(engine)
    clean = project_volume(phantom, grid, config, list(thetas), step_mm, eng)
    if not apply_noise:
        return clean
    return add_noise(clean, noise).to(eng.device)


def fdk_reconstruct(images: torch.Tensor, config: ScannerConfig, thetas: Sequence[float], grid: GridSpec,
                    window: int = AUTO, engine: Optional[Engine] = None) -> torch.Tensor:
    eng = _eng(engine)
    im = images.to(device=eng.device, dtype=torch.float32).contiguous()
    if im.dim() != 3 or tuple(im.shape[1:]) != (config.height, config.width) or im.shape[0] != len(thetas):
        from .engine import DimMismatch
        raise DimMismatch("fdk: projections do not match the scanner / angle list")
    _, th, arr = _thetas(list(thetas))
    vol = torch.empty(grid.shape_zyx, dtype=torch.float32, device=eng.device)
    g, sc = grid._c(), config._c()
    _check(eng.lib.sct_fdk(eng._h, _ptr(im), im.shape[0], C.byref(sc), arr, C.byref(g), int(window), _ptr(vol)))
    return vol


def nearest_neighbor_distances(points: torch.Tensor, engine: Optional[Engine] = None) -> torch.Tensor:
    eng = _eng(engine)
    p = points.to(device=eng.device, dtype=torch.float64).contiguous().reshape(-1, 3)
    out = torch.empty(p.shape[0], dtype=torch.float64, device=eng.device)
    _check(eng.lib.sct_nn_distances(eng._h, p.shape[0], _ptr(p), _ptr(out)))
    return out


def sample_init_cloud(vol: torch.Tensor, grid: GridSpec, count: int, density_threshold: float = 0.05,
                      density_scale: float = 0.15, s_min_mm: float = 2e-4, seed: int = 0,
                      engine: Optional[Engine] = None) -> GaussianCloud:
    """fdk.cpp:203-247 with std::mt19937_64(seed); InitParams defaults (fdk.hpp:23-27)."""
    eng = _eng(engine)
    v = vol.to(device=eng.device, dtype=torch.float32).contiguous()
    e = lambda k: torch.empty(k * count, dtype=torch.float32, device=eng.device)
    cloud = GaussianCloud(s_min_mm, e(1), e(3), e(3), e(4), device=eng.device)
    g, cl = grid._c(), cloud._c()
    _check(eng.lib.sct_sample_init_cloud(eng._h, _ptr(v), C.byref(g), int(count), float(density_threshold),
                                         float(density_scale), float(s_min_mm), int(seed) & ((1 << 64) - 1),
                                         C.byref(cl)))
    return cloud
