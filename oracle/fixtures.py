"""TEST INFRASTRUCTURE — ctypes wrapper of oracle/fixtures_oracle.cpp, the FP64
CPU restatement of the reference's fixture-generation side:
Shepp-Logan phantom, quadrature projector, noise, FDK, nearest-neighbour init.
Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may import it."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import oracle as O

D = C.POINTER(C.c_double)
F = C.POINTER(C.c_float)
I32 = C.POINTER(C.c_int32)
VP = C.c_void_p

# simulator.cpp:16-29 (Kak & Slaney 3D, modified intensities): intensity, a, b, c, x0, y0, z0, phi
SHEPP_LOGAN = np.array([
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

def _lib():
    return O.lib()


def _d(a):
    return a.ctypes.data_as(D)


def _f(a):
    return a.ctypes.data_as(F)


def _i(a):
    return a.ctypes.data_as(I32)


def _grid_args(grid: O.GridSpec):
    return (np.array(grid.dims, np.int32), np.array(grid.origin_mm, np.float64), np.array(grid.spacing_mm, np.float64))


def phantom(dims, lo=(-1.0, -1.0, -1.0), hi=(1.0, 1.0, 1.0), ellipsoids=SHEPP_LOGAN) -> np.ndarray:
    """phantom_from_ellipsoids (simulator.cpp:44-65) as fp32 [Z][Y][X]."""
    e = np.ascontiguousarray(ellipsoids, np.float64)
    out = np.zeros((dims[2], dims[1], dims[0]), np.float32)
    _lib().orc_phantom(e.shape[0], _d(e), _i(np.array(dims, np.int32)), _d(np.array(lo, np.float64)),
                       _d(np.array(hi, np.float64)), _f(out))
    return out


def sample_trilinear(vol: np.ndarray, grid: O.GridSpec, x) -> float:
    v = np.ascontiguousarray(vol, np.float32)
    d, o, s = _grid_args(grid)
    return _lib().orc_sample_trilinear(_f(v), _i(d), _d(o), _d(s), _d(np.array(x, np.float64)))


def project_volume(vol: np.ndarray, grid: O.GridSpec, cfg: O.ScannerConfig, theta: float, step_mm: float):
    """simulator.cpp:109-132: [H][W] float64 line integrals of the trilinear volume."""
    v = np.ascontiguousarray(vol, np.float32)
    d, o, s = _grid_args(grid)
    g, r = cfg._geo()
    out = np.zeros((cfg.detector_res_px[1], cfg.detector_res_px[0]))
    rc = _lib().orc_project_volume(_f(v), _i(d), _d(o), _d(s), _d(g), _i(r), theta, step_mm, _d(out))
    if rc:
        raise O.OracleError("project_volume: step_mm must be > 0")
    return out


def view_seed(master: int, view: int) -> int:
    return _lib().orc_view_seed(master, view)


def add_noise(clean: np.ndarray, i0: float, gauss_sigma: float, seed: int, view: int) -> np.ndarray:
    c = np.ascontiguousarray(clean, np.float32)
    out = np.zeros(c.shape)
    rc = _lib().orc_add_noise(_f(c), c.size, i0, gauss_sigma, seed, view, _d(out))
    if rc:
        raise O.OracleError("add_noise: i0 must be > 0")
    return out


def fdk(images: np.ndarray, cfg: O.ScannerConfig, angles, grid: O.GridSpec, window: int = 2) -> np.ndarray:
    """fdk.cpp:53-134; window 0 ramp, 1 hann, 2 auto. images [n][H][W]."""
    im = np.ascontiguousarray(images, np.float32)
    d, o, s = _grid_args(grid)
    g, r = cfg._geo()
    out = np.zeros(grid.shape_zyx)
    rc = _lib().orc_fdk(_f(im), im.shape[0], _d(g), _i(r), _d(np.array(angles, np.float64)), _i(d), _d(o), _d(s),
                        window, _d(out))
    if rc:
        raise O.OracleError("fdk: need at least 2 views")
    return out


def nn_distances(points: np.ndarray) -> np.ndarray:
    p = np.ascontiguousarray(points, np.float64).reshape(-1, 3)
    out = np.zeros(p.shape[0])
    _lib().orc_nn_distances(p.shape[0], _d(p), _d(out))
    return out


def sample_init_cloud(rng: O.Rng, vol: np.ndarray, grid: O.GridSpec, count: int, threshold=0.05,
                      density_scale=0.15, s_min=2e-4) -> O.Cloud:
    """fdk.cpp:203-247 (raw parameters as add_kernel stores them)."""
    v = np.ascontiguousarray(vol, np.float32)
    d, o, s = _grid_args(grid)
    c = O.Cloud(s_min, np.zeros(count), np.zeros(3 * count), np.zeros(3 * count), np.zeros(4 * count))
    rc = _lib().orc_sample_init_cloud(rng._h, _f(v), _i(d), _d(o), _d(s), count, threshold, density_scale, s_min,
                                      _d(c.rho_raw), _d(c.pos), _d(c.scale_raw), _d(c.rot))
    if rc:
        raise O.DimMismatch("init: too few voxels above the density threshold")
    return c
