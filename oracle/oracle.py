"""ORACLE — test infrastructure only.

ctypes front-end for ``liborc.so`` (``splatct_oracle.cpp``), the FP64 CPU
restatement of the reference hot path. Only ``tests/``, ``__graft_entry__.smoke``
and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` arm may import this
module; the product package never does.

Function names follow the reference's C++ API (rasterizer.hpp:36-64,
voxelizer.hpp:60-72, objectives.hpp:24-31, trainer.cpp:34-36,144-163).
"""
from __future__ import annotations

import contextlib
import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liborc.so")
# the reference itself, compiled from /root/reference by `make -C oracle ref`
# (ref_capi.cpp + ref_shim/); it exports the same orc_* ABI
_REF_LIB_PATH = os.path.join(_HERE, "_ref", "libsplatct_ref.so")
_REF_SRC = "/root/reference/proj/core/src"
_libs: dict = {}
_active = os.environ.get("SCT_ORACLE", "port")

D = C.POINTER(C.c_double)
F = C.POINTER(C.c_float)
I32 = C.POINTER(C.c_int32)
I64 = C.POINTER(C.c_int64)
VP = C.c_void_p


def build(force: bool = False) -> str:
    newest = max(os.path.getmtime(os.path.join(_HERE, s)) for s in ("splatct_oracle.cpp", "fixtures_oracle.cpp"))
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < newest:
        subprocess.run(["make", "-s", "-C", _HERE, "liborc.so"], check=True)
    return _LIB_PATH


def build_ref() -> str | None:
    """Compile the reference's own sources into oracle/_ref (only where
    /root/reference exists; elsewhere the prebuilt .so, if shipped, is used)."""
    if os.path.isdir(_REF_SRC):
        subprocess.run(["make", "-s", "-C", _HERE, "ref"], check=True)
    return _REF_LIB_PATH if os.path.exists(_REF_LIB_PATH) else None


def ref_available() -> bool:
    return os.path.exists(_REF_LIB_PATH)


_SIG = {
    "orc_last_error": (C.c_char_p, []),
    "orc_set_threads": (None, [C.c_int]),
    "orc_max_threads": (C.c_int, []),
    "orc_rng_new": (VP, [C.c_uint64]),
    "orc_rng_free": (None, [VP]),
    "orc_rng_uniform": (C.c_double, [VP, C.c_double, C.c_double]),
    "orc_rng_normal": (C.c_double, [VP]),
    "orc_random_cloud": (None, [VP, C.c_int, C.c_double, C.c_double, C.c_double, C.c_double, D, D, D, D]),
    "orc_kernel_to_raw": (None, [C.c_int, C.c_double, D, D, D, D, D, D]),
    "orc_activate": (None, [C.c_int, C.c_double, D, D, D, D]),
    "orc_random_image": (None, [VP, C.c_int, C.c_double, C.c_double, D]),
    "orc_view_transform": (None, [D, I32, C.c_double, D, D]),
    "orc_detector": (None, [D, I32, D]),
    "orc_local_jacobian": (C.c_int, [D, I32, D, D]),
    "orc_ray_space_point": (None, [D, I32, D, D]),
    "orc_pixel_ray": (None, [D, I32, C.c_double, C.c_int, C.c_int, D, D]),
    "orc_covariance": (None, [C.c_int, C.c_double, D, D, D, D, C.c_int, D]),
    "orc_density_at": (C.c_double, [C.c_int, C.c_double, D, D, D, D, D]),
    "orc_ray_march_density": (C.c_double, [C.c_int, C.c_double, D, D, D, D, D, D, C.c_double]),
    "orc_normalize_rotations": (None, [C.c_int, D]),
    "orc_cov_param_grads": (None, [C.c_int, C.c_double, D, D, D, D, C.c_int, D, D, D]),
    "orc_project_kernel": (C.c_int, [C.c_int, C.c_double, D, D, D, D, C.c_int, D, I32, C.c_double, D, D]),
    "orc_render": (VP, [C.c_int, C.c_double, D, D, D, D, D, I32, C.c_double, D]),
    "orc_render_free": (None, [VP]),
    "orc_render_image": (None, [VP, D]),
    "orc_render_n_visible": (C.c_int, [VP]),
    "orc_render_n_pairs": (C.c_int64, [VP]),
    "orc_render_tile_lists": (None, [VP, I64, I32]),
    "orc_render_visible": (None, [VP, I32, D]),
    "orc_render_backward": (C.c_int, [VP, C.c_int, C.c_double, D, D, D, D, D, I32, C.c_double, D, D,
                                      D, D, D, D, D, I32, D]),
    "orc_raster_chain_from_stats": (None, [C.c_int, C.c_double, D, D, D, D, D, I32, C.c_double, D,
                                           C.c_int, I32, D, D, D, D, D]),
    "orc_grid_for_extent": (None, [D, D, I32, D, D]),
    "orc_voxelize": (None, [C.c_int, C.c_double, D, D, D, D, I32, D, D, C.c_double, D]),
    "orc_voxelize_backward": (C.c_int, [C.c_int, C.c_double, D, D, D, D, I32, D, D, C.c_double, D,
                                        D, D, D, D]),
    "orc_voxel_bins": (C.c_int64, [C.c_int, C.c_double, D, D, D, D, I32, D, D, C.c_double, I64, I32]),
    "orc_random_subvolume_spec": (None, [VP, D, D, D, C.c_int, D]),
    "orc_tv3d": (C.c_int, [I32, D, D, D]),
    "orc_l1": (C.c_int, [C.c_int, D, D, D, D]),
    "orc_dssim": (C.c_int, [C.c_int, C.c_int, D, D, D, D]),
    "orc_adaptive_control": (VP, [VP, C.c_int, C.c_double, C.POINTER(D), D, I32, D, C.c_double,
                                  C.c_double, C.c_double, C.c_double, D]),
    "orc_ac_size": (C.c_int, [VP]),
    "orc_ac_counts": (None, [VP, C.POINTER(C.c_int)]),
    "orc_ac_get": (None, [VP, C.c_int, D]),
    "orc_ac_stats": (None, [VP, D, I32, D]),
    "orc_ac_free": (None, [VP]),
    "orc_normal_draws": (None, [VP, C.c_int, D]),
    "orc_shuffle": (None, [VP, C.c_int, I32]),
    "orc_lr_at": (C.c_double, [C.c_double, C.c_double, C.c_int, C.c_int]),
    "orc_adam_step": (None, [C.c_int64, D, D, D, D, C.c_double, C.c_int, C.c_double, C.c_double,
                             C.c_double]),
    # fixtures (fixtures_oracle.cpp / simulator.cpp, fdk.cpp)
    "orc_phantom": (None, [C.c_int, D, I32, D, D, F]),
    "orc_shepp_logan": (C.c_int, [D, C.c_int]),
    "orc_sample_trilinear": (C.c_double, [F, I32, D, D, D]),
    "orc_project_volume": (C.c_int, [F, I32, D, D, D, I32, C.c_double, C.c_double, D]),
    "orc_view_seed": (C.c_uint64, [C.c_uint64, C.c_int]),
    "orc_add_noise": (C.c_int, [F, C.c_int, C.c_double, C.c_double, C.c_uint64, C.c_int, D]),
    "orc_fdk": (C.c_int, [F, C.c_int, D, I32, D, I32, D, D, C.c_int, D]),
    "orc_nn_distances": (None, [C.c_int, D, D]),
    "orc_sample_init_cloud": (C.c_int, [VP, F, I32, D, D, C.c_int, C.c_double, C.c_double, C.c_double,
                                        D, D, D, D]),
    # reference-only: the training loop and the I/O containers
    "orc_train": (VP, [C.c_int, C.c_double, D, D, D, D, D, I32, C.c_int, D, D, D, I32, C.c_uint64, D,
                       C.c_int, C.POINTER(C.c_int)]),
    "orc_save_cloud": (C.c_int, [C.c_char_p, C.c_int, C.c_double, D, D, D, D]),
    "orc_load_cloud": (C.c_int, [C.c_char_p, C.c_int, C.POINTER(C.c_int), D, D, D, D, D]),
    "orc_write_volume": (C.c_int, [C.c_char_p, I32, D, D, D]),
    "orc_read_volume": (C.c_int, [C.c_char_p, C.c_int64, I32, D, D, D]),
    "orc_write_image": (C.c_int, [C.c_char_p, C.c_int, C.c_int, D]),
    "orc_read_image": (C.c_int, [C.c_char_p, C.c_int64, I32, D]),
}


def _load(kind: str):
    if kind not in _libs:
        if kind == "reference":
            path = _REF_LIB_PATH
            if not os.path.exists(path):
                build_ref()
            if not os.path.exists(path):
                raise OracleError("reference library oracle/_ref/libsplatct_ref.so is not built")
        elif kind == "port":
            path = _LIB_PATH
            if not os.path.exists(path):
                build()
        else:
            raise ValueError(kind)
        L = C.CDLL(path)
        for name, (res, args) in _SIG.items():
            f = getattr(L, name, None)
            if f is None:
                continue
            f.restype = res
            f.argtypes = args
        _libs[kind] = L
    return _libs[kind]


def lib():
    """The active oracle library: "port" (the FP64 restatement, default) or
    "reference" (the reference's own sources, oracle/_ref)."""
    return _load(_active)


def active() -> str:
    return _active


@contextlib.contextmanager
def using(kind: str):
    """Run oracle calls inside the block against `kind` ("port" | "reference")."""
    global _active
    prev = _active
    _load(kind)
    _active = kind
    try:
        yield
    finally:
        _active = prev


def _d(a):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous, (a.dtype, a.flags)
    return a.ctypes.data_as(D)


def _i32(a):
    if a is None:
        return None
    assert a.dtype == np.int32 and a.flags.c_contiguous
    return a.ctypes.data_as(I32)


def _i64(a):
    assert a.dtype == np.int64 and a.flags.c_contiguous
    return a.ctypes.data_as(I64)


class OracleError(RuntimeError):
    pass


class DimMismatch(OracleError):
    pass


def _check(rc):
    if rc == 0:
        return
    msg = lib().orc_last_error().decode()
    if rc == 3:
        raise DimMismatch(msg)
    raise OracleError(msg)


# ----------------------------------------------------------------- types
@dataclass
class ScannerConfig:  # geometry.hpp:12-31 (angles passed per call)
    l_so_mm: float = 8.0
    l_sd_mm: float = 12.0
    detector_size_mm: tuple = (5.6, 5.6)
    detector_res_px: tuple = (128, 128)
    extent_min_mm: tuple = (-1.0, -1.0, -1.0)
    extent_max_mm: tuple = (1.0, 1.0, 1.0)
    near_clip_mm: float = 0.0
    parallel_beam: bool = False  # extension: orthographic projection (no reference code)

    def _geo(self):
        g = np.array([self.l_so_mm, self.l_sd_mm, *self.detector_size_mm, *self.extent_min_mm,
                      *self.extent_max_mm, self.near_clip_mm], dtype=np.float64)
        r = np.array([*self.detector_res_px, int(self.parallel_beam)], dtype=np.int32)
        return g, r


def test_scanner(res: int = 128) -> ScannerConfig:  # tests/helpers.hpp:18-28
    return ScannerConfig(detector_res_px=(res, res))


def full_circle_angles(n: int):  # geometry.cpp:63-67
    return [2.0 * np.pi * i / n for i in range(n)]


@dataclass
class RasterOptions:  # rasterizer.hpp:15-21
    mode: int = 0  # 0 rectified, 1 biased
    lowpass_eps_px: float = 0.3
    dilation_compensation: bool = True
    freeze_jacobian: bool = False
    cull_mahalanobis: float = 3.0348542587702925

    def _arr(self):
        return np.array([self.mode, self.lowpass_eps_px, float(self.dilation_compensation),
                         float(self.freeze_jacobian), self.cull_mahalanobis], dtype=np.float64)


VOXEL_CULL = 3.3681993876652464  # voxelizer.hpp:56


@dataclass
class Cloud:
    """GaussianCloud raw SoA arrays (gaussian_cloud.hpp:62-66), float64."""
    s_min: float
    rho_raw: np.ndarray
    pos: np.ndarray
    scale_raw: np.ndarray
    rot: np.ndarray

    @property
    def m(self):
        return int(self.rho_raw.shape[0])

    def _args(self):
        return (self.m, self.s_min, _d(self.rho_raw), _d(self.pos), _d(self.scale_raw), _d(self.rot))

    def copy(self):
        return Cloud(self.s_min, self.rho_raw.copy(), self.pos.copy(), self.scale_raw.copy(), self.rot.copy())

    @staticmethod
    def from_arrays(s_min, rho_raw, pos, scale_raw, rot):
        f = lambda a: np.ascontiguousarray(np.asarray(a, dtype=np.float64).reshape(-1))
        return Cloud(float(s_min), f(rho_raw), f(pos), f(scale_raw), f(rot))

    @staticmethod
    def empty(s_min=2e-4):
        z = np.zeros(0, dtype=np.float64)
        return Cloud(s_min, z.copy(), z.copy(), z.copy(), z.copy())

    def concat(self, other):
        return Cloud(self.s_min, np.concatenate([self.rho_raw, other.rho_raw]),
                     np.concatenate([self.pos, other.pos]), np.concatenate([self.scale_raw, other.scale_raw]),
                     np.concatenate([self.rot, other.rot]))

    def rho(self):
        m = self.m
        rho = np.zeros(m)
        sc = np.zeros(3 * m)
        lib().orc_activate(m, self.s_min, _d(self.rho_raw), _d(self.scale_raw), _d(rho), _d(sc))
        return rho

    def scale(self):
        m = self.m
        rho = np.zeros(m)
        sc = np.zeros(3 * m)
        lib().orc_activate(m, self.s_min, _d(self.rho_raw), _d(self.scale_raw), _d(rho), _d(sc))
        return sc.reshape(m, 3)


def kernels_to_cloud(s_min, rho, pos, scale, rot) -> Cloud:
    """add_kernel for activated values (gaussian_cloud.cpp:48-55)."""
    rho = np.ascontiguousarray(rho, dtype=np.float64).reshape(-1)
    n = rho.shape[0]
    scale = np.ascontiguousarray(scale, dtype=np.float64).reshape(-1)
    rot = np.ascontiguousarray(rot, dtype=np.float64).reshape(-1)
    rr, sr, qr = np.zeros(n), np.zeros(3 * n), np.zeros(4 * n)
    lib().orc_kernel_to_raw(n, float(s_min), _d(rho), _d(scale), _d(rot), _d(rr), _d(sr), _d(qr))
    return Cloud(float(s_min), rr, np.ascontiguousarray(pos, dtype=np.float64).reshape(-1).copy(), sr, qr)


@dataclass
class Grads:  # CloudGrads (gaussian_cloud.hpp:84-96); accumulate semantics
    rho_raw: np.ndarray
    pos: np.ndarray
    scale_raw: np.ndarray
    rot: np.ndarray

    @staticmethod
    def zeros(m):
        return Grads(np.zeros(m), np.zeros(3 * m), np.zeros(3 * m), np.zeros(4 * m))

    def _args(self):
        return (_d(self.rho_raw), _d(self.pos), _d(self.scale_raw), _d(self.rot))

    def flat(self):
        return np.concatenate([self.rho_raw, self.pos, self.scale_raw, self.rot])


@dataclass
class Stats:  # adaptive-control statistics (gaussian_cloud.hpp:74-77)
    grad2d_norm_accum: np.ndarray
    grad_count: np.ndarray
    grad3d_accum: np.ndarray

    @staticmethod
    def zeros(m):
        return Stats(np.zeros(m), np.zeros(m, dtype=np.int32), np.zeros(3 * m))


class Rng:
    """std::mt19937_64 with libstdc++ distributions (the reference tests' RNG)."""

    def __init__(self, seed: int):
        self._L = lib()
        self._h = self._L.orc_rng_new(seed)

    def __del__(self):
        if getattr(self, "_h", None):
            self._L.orc_rng_free(self._h)
            self._h = None

    def uniform(self, lo=0.0, hi=1.0):
        return lib().orc_rng_uniform(self._h, lo, hi)

    def normal(self):
        return lib().orc_rng_normal(self._h)


def random_cloud(rng: Rng, count: int, pos_radius=0.35, scale_min=0.05, scale_max=0.2, s_min=2e-4) -> Cloud:
    """tests/helpers.hpp:30-48 (same RNG stream as the reference tests)."""
    c = Cloud(s_min, np.zeros(count), np.zeros(3 * count), np.zeros(3 * count), np.zeros(4 * count))
    lib().orc_random_cloud(rng._h, count, pos_radius, scale_min, scale_max, s_min,
                           _d(c.rho_raw), _d(c.pos), _d(c.scale_raw), _d(c.rot))
    return c


def random_image(rng: Rng, w: int, h: int, lo=0.0, hi=1.0) -> np.ndarray:
    out = np.zeros(w * h)
    lib().orc_random_image(rng._h, w * h, lo, hi, _d(out))
    return out.reshape(h, w)


# ----------------------------------------------------------------- geometry
def view_transform(cfg: ScannerConfig, theta: float):
    g, r = cfg._geo()
    rot, t = np.zeros(9), np.zeros(3)
    lib().orc_view_transform(_d(g), _i32(r), theta, _d(rot), _d(t))
    return rot.reshape(3, 3), t


def detector_model(cfg: ScannerConfig):
    g, r = cfg._geo()
    out = np.zeros(4)
    lib().orc_detector(_d(g), _i32(r), _d(out))
    return dict(fx=out[0], fy=out[1], cx=out[2], cy=out[3])


def local_jacobian(cfg: ScannerConfig, p):
    g, r = cfg._geo()
    p = np.ascontiguousarray(p, dtype=np.float64)
    out = np.zeros(9)
    _check(lib().orc_local_jacobian(_d(g), _i32(r), _d(p), _d(out)))
    return out.reshape(3, 3)


def ray_space_point(cfg: ScannerConfig, p):
    g, r = cfg._geo()
    p = np.ascontiguousarray(p, dtype=np.float64)
    out = np.zeros(3)
    lib().orc_ray_space_point(_d(g), _i32(r), _d(p), _d(out))
    return out


def pixel_ray(cfg: ScannerConfig, theta, u, v):
    g, r = cfg._geo()
    o, d = np.zeros(3), np.zeros(3)
    lib().orc_pixel_ray(_d(g), _i32(r), theta, u, v, _d(o), _d(d))
    return o, d


# ----------------------------------------------------------------- cloud math
def covariance_at(cloud: Cloud, i: int):
    out = np.zeros(9)
    lib().orc_covariance(*cloud._args(), i, _d(out))
    return out.reshape(3, 3)


def density_at(cloud: Cloud, x):
    x = np.ascontiguousarray(x, dtype=np.float64)
    return lib().orc_density_at(*cloud._args(), _d(x))


def ray_march_density(cloud: Cloud, origin, direction, step):
    o = np.ascontiguousarray(origin, dtype=np.float64)
    d = np.ascontiguousarray(direction, dtype=np.float64)
    return lib().orc_ray_march_density(*cloud._args(), _d(o), _d(d), step)


def normalize_rotations(cloud: Cloud):
    lib().orc_normalize_rotations(cloud.m, _d(cloud.rot))


def accumulate_covariance_param_grads(cloud: Cloud, i: int, g_sigma, grads: Grads):
    gs = np.ascontiguousarray(g_sigma, dtype=np.float64).reshape(9)
    lib().orc_cov_param_grads(*cloud._args(), i, _d(gs), _d(grads.scale_raw), _d(grads.rot))


# ----------------------------------------------------------------- rasterizer
def project_kernel(cloud: Cloud, i: int, cfg: ScannerConfig, theta: float, opts: RasterOptions = None):
    """rasterizer.hpp:36-38. Returns dict or None when culled."""
    opts = opts or RasterOptions()
    g, r = cfg._geo()
    out = np.zeros(11)
    vis = lib().orc_project_kernel(*cloud._args(), i, _d(g), _i32(r), theta, _d(opts._arr()), _d(out))
    if not vis:
        return None
    return dict(center=out[0:2].copy(), cov=np.array([[out[2], out[3]], [out[3], out[4]]]),
                conic=np.array([[out[5], out[6]], [out[6], out[7]]]), amplitude=out[8], mu=out[9],
                depth=out[10])


class Rendered:
    """RenderedProjection (rasterizer.hpp:41-51), owned by the oracle."""

    def __init__(self, handle, w, h):
        self._h = handle
        self._L = lib()
        self.width, self.height = w, h
        self.tiles_x = (w + 15) // 16
        self.tiles_y = (h + 15) // 16

    def __del__(self):
        if getattr(self, "_h", None):
            self._L.orc_render_free(self._h)
            self._h = None

    @property
    def image(self):
        out = np.zeros(self.width * self.height)
        self._L.orc_render_image(self._h, _d(out))
        return out.reshape(self.height, self.width)

    @property
    def n_visible(self):
        return self._L.orc_render_n_visible(self._h)

    @property
    def n_pairs(self):
        return self._L.orc_render_n_pairs(self._h)

    def tile_lists(self):
        """(offsets[T+1] int64, kernel_idx[pairs] int32), lists in kernel indices."""
        T = self.tiles_x * self.tiles_y
        off = np.zeros(T + 1, dtype=np.int64)
        idx = np.zeros(max(self.n_pairs, 1), dtype=np.int32)
        self._L.orc_render_tile_lists(self._h, _i64(off), _i32(idx))
        return off, idx[: self.n_pairs]

    def visible(self):
        n = self.n_visible
        k = np.zeros(max(n, 1), dtype=np.int32)
        rec = np.zeros(max(n, 1) * 11)
        self._L.orc_render_visible(self._h, _i32(k), _d(rec))
        return k[:n], rec.reshape(-1, 11)[:n]


def render(cloud: Cloud, cfg: ScannerConfig, theta: float, opts: RasterOptions = None) -> Rendered:
    """rasterizer.cpp:112-157"""
    opts = opts or RasterOptions()
    g, r = cfg._geo()
    h = lib().orc_render(*cloud._args(), _d(g), _i32(r), theta, _d(opts._arr()))
    return Rendered(h, cfg.detector_res_px[0], cfg.detector_res_px[1])


def render_backward(cloud: Cloud, cfg: ScannerConfig, theta: float, fwd: Rendered, dL_dimage, grads: Grads,
                    opts: RasterOptions = None, stats: Stats = None):
    """rasterizer.cpp:195-342; accumulates into grads (and stats when given)."""
    opts = opts or RasterOptions()
    g, r = cfg._geo()
    dL = np.ascontiguousarray(dL_dimage, dtype=np.float64)
    if dL.ndim != 2 or dL.shape != (cfg.detector_res_px[1], cfg.detector_res_px[0]):
        raise DimMismatch("render_backward: upstream gradient dims mismatch")
    st = (None, None, None) if stats is None else (_d(stats.grad2d_norm_accum), _i32(stats.grad_count),
                                                     _d(stats.grad3d_accum))
    _check(fwd._L.orc_render_backward(fwd._h, *cloud._args(), _d(g), _i32(r), theta, _d(opts._arr()), _d(dL),
                                     *grads._args(), *st))


def raster_chain_from_stats(cloud: Cloud, cfg: ScannerConfig, theta: float, opts: RasterOptions, kidx, stats6,
                            grads: Grads):
    g, r = cfg._geo()
    kidx = np.ascontiguousarray(kidx, dtype=np.int32)
    stats6 = np.ascontiguousarray(stats6, dtype=np.float64)
    lib().orc_raster_chain_from_stats(*cloud._args(), _d(g), _i32(r), theta, _d(opts._arr()), kidx.shape[0],
                                      _i32(kidx), _d(stats6), *grads._args())


# ----------------------------------------------------------------- voxelizer
@dataclass
class GridSpec:  # voxelizer.hpp:13-24
    dims: tuple
    origin_mm: tuple = (0.0, 0.0, 0.0)
    spacing_mm: tuple = (1.0, 1.0, 1.0)

    def _args(self):
        return (_i32(np.array(self.dims, dtype=np.int32)), _d(np.array(self.origin_mm, dtype=np.float64)),
                _d(np.array(self.spacing_mm, dtype=np.float64)))

    def voxel_center(self, x, y, z):
        return np.array([self.origin_mm[k] + ((x, y, z)[k] + 0.5) * self.spacing_mm[k] for k in range(3)])

    @property
    def shape_zyx(self):
        return (self.dims[2], self.dims[1], self.dims[0])


def grid_for_extent(lo, hi, dims) -> GridSpec:  # voxelizer.cpp:8-14
    lo = np.array(lo, dtype=np.float64)
    hi = np.array(hi, dtype=np.float64)
    o, s = np.zeros(3), np.zeros(3)
    lib().orc_grid_for_extent(_d(lo), _d(hi), _i32(np.array(dims, dtype=np.int32)), _d(o), _d(s))
    return GridSpec(tuple(int(d) for d in dims), tuple(o), tuple(s))


def voxelize(cloud: Cloud, grid: GridSpec, cull: float = VOXEL_CULL) -> np.ndarray:
    """voxelizer.cpp:108-138; returns volume [Z][Y][X] (x-fastest)."""
    vol = np.zeros(grid.shape_zyx)
    a = grid._args()
    lib().orc_voxelize(*cloud._args(), *a, cull, _d(vol))
    return vol


def voxelize_backward(cloud: Cloud, grid: GridSpec, dL_dV, grads: Grads, cull: float = VOXEL_CULL):
    dL = np.ascontiguousarray(dL_dV, dtype=np.float64)
    if dL.shape != grid.shape_zyx:
        raise DimMismatch("voxelize_backward: gradient volume dims mismatch")
    a = grid._args()
    _check(lib().orc_voxelize_backward(*cloud._args(), *a, cull, _d(dL), *grads._args()))


def voxel_bins(cloud: Cloud, grid: GridSpec, cull: float = VOXEL_CULL):
    a = grid._args()
    n = lib().orc_voxel_bins(*cloud._args(), *a, cull, None, None)
    nb = 1
    for d in grid.dims:
        nb *= (d + 7) // 8
    off = np.zeros(nb + 1, dtype=np.int64)
    idx = np.zeros(max(n, 1), dtype=np.int32)
    lib().orc_voxel_bins(*cloud._args(), *a, cull, _i64(off), _i32(idx))
    return off, idx[:n]


def random_subvolume_spec(lo, hi, spacing, d: int, rng: Rng) -> GridSpec:
    lo = np.array(lo, dtype=np.float64)
    hi = np.array(hi, dtype=np.float64)
    sp = np.array(spacing, dtype=np.float64)
    o = np.zeros(3)
    lib().orc_random_subvolume_spec(rng._h, _d(lo), _d(hi), _d(sp), d, _d(o))
    return GridSpec((d, d, d), tuple(o), tuple(sp))


# ----------------------------------------------------------------- objectives
def tv3d_loss(vol: np.ndarray):
    """objectives.cpp:169-202; vol is [Z][Y][X]. Returns (value, grad)."""
    vol = np.ascontiguousarray(vol, dtype=np.float64)
    dims = np.array([vol.shape[2], vol.shape[1], vol.shape[0]], dtype=np.int32)
    grad = np.zeros_like(vol)
    val = C.c_double(0.0)
    _check(lib().orc_tv3d(_i32(dims), _d(vol), C.byref(val), _d(grad)))
    return val.value, grad


def l1_loss(rendered, measured):
    r = np.ascontiguousarray(rendered, dtype=np.float64)
    m = np.ascontiguousarray(measured, dtype=np.float64)
    if r.shape != m.shape:
        raise DimMismatch("l1_loss: image dims differ")
    g = np.zeros_like(r)
    val = C.c_double(0.0)
    _check(lib().orc_l1(r.size, _d(r), _d(m), C.byref(val), _d(g)))
    return val.value, g


def dssim_loss(rendered, measured):
    r = np.ascontiguousarray(rendered, dtype=np.float64)
    m = np.ascontiguousarray(measured, dtype=np.float64)
    if r.shape != m.shape:
        raise DimMismatch("ssim: image dims differ")
    g = np.zeros_like(r)
    val = C.c_double(0.0)
    _check(lib().orc_dssim(r.shape[1], r.shape[0], _d(r), _d(m), C.byref(val), _d(g)))
    return val.value, g


# ----------------------------------------------------------------- adaptive control
ADAM_KEYS = ("m_rho", "v_rho", "m_pos", "v_pos", "m_scale", "v_scale", "m_rot", "v_rot")


def adaptive_control(rng: Rng, cloud: Cloud, adam: dict, stats: Stats, prune_thr=0.005, densify_thr=0.00005,
                     split_frac=0.01, split_factor=1.6, extent_size=(2.0, 2.0, 2.0)):
    """trainer.cpp:167-230. Returns (new Cloud, new adam dict, (pruned, cloned, split))."""
    arrs = [cloud.rho_raw, cloud.pos, cloud.scale_raw, cloud.rot] + [np.ascontiguousarray(adam[k], dtype=np.float64)
                                                                   for k in ADAM_KEYS]
    ptrs = (D * 12)(*[_d(a) for a in arrs])
    ext = np.array(extent_size, dtype=np.float64)
    h = lib().orc_adaptive_control(rng._h, cloud.m, cloud.s_min, ptrs, _d(stats.grad2d_norm_accum),
                                   _i32(stats.grad_count), _d(stats.grad3d_accum), prune_thr, densify_thr,
                                   split_frac, split_factor, _d(ext))
    try:
        n = lib().orc_ac_size(h)
        cnt = (C.c_int * 3)()
        lib().orc_ac_counts(h, cnt)
        strides = (1, 3, 3, 4, 1, 1, 3, 3, 3, 3, 4, 4)
        out = []
        for a in range(12):
            buf = np.zeros(max(1, strides[a] * n))
            lib().orc_ac_get(h, a, _d(buf))
            out.append(buf[: strides[a] * n])
    finally:
        lib().orc_ac_free(h)
    return Cloud(cloud.s_min, *out[:4]), dict(zip(ADAM_KEYS, out[4:])), tuple(cnt)


def shuffle(rng: Rng, values: np.ndarray) -> np.ndarray:
    """std::shuffle on a std::vector<int> (trainer.cpp:270); reference library only."""
    v = np.ascontiguousarray(values, dtype=np.int32).copy()
    _load("reference").orc_shuffle(rng._h, v.size, _i32(v))
    return v


def normal_draws(rng: Rng, n: int) -> np.ndarray:
    out = np.zeros(max(n, 1))
    lib().orc_normal_draws(rng._h, n, _d(out))
    return out[:n]


# ----------------------------------------------------------------- optimizer
def lr_at(lr_init, final_ratio, t, iters):
    return lib().orc_lr_at(lr_init, final_ratio, t, iters)


def adam_step(params, m, v, g, lr, step, beta1=0.9, beta2=0.999, eps=1e-15):
    lib().orc_adam_step(params.size, _d(params), _d(m), _d(v), _d(np.ascontiguousarray(g, dtype=np.float64)),
                        lr, step, beta1, beta2, eps)


def set_threads(n: int):
    lib().orc_set_threads(n)


def max_threads() -> int:
    return lib().orc_max_threads()


# ----------------------------------------------------------------- reference-only entry points
class _RefIO:
    """The reference's container readers/writers (io.cpp:18-213), from oracle/_ref."""

    def __init__(self):
        self.L = _load("reference")

    def _ok(self, rc):
        if rc != 0:
            raise OracleError(self.L.orc_last_error().decode())

    def save_cloud(self, c: "Cloud", path: str):
        self._ok(self.L.orc_save_cloud(path.encode(), *c._args()))

    def load_cloud(self, path: str) -> "Cloud":
        m, s = C.c_int(0), C.c_double(0.0)
        z = np.zeros(1)
        self._ok(self.L.orc_load_cloud(path.encode(), 0, C.byref(m), C.byref(s), _d(z), _d(z), _d(z), _d(z)))
        n = m.value
        c = Cloud(s.value, np.zeros(n), np.zeros(3 * n), np.zeros(3 * n), np.zeros(4 * n))
        self._ok(self.L.orc_load_cloud(path.encode(), n, C.byref(m), C.byref(s), *[_d(a) for a in
                                        (c.rho_raw, c.pos, c.scale_raw, c.rot)]))
        return c

    def write_image(self, img, path: str):
        img = np.ascontiguousarray(img, dtype=np.float64)
        self._ok(self.L.orc_write_image(path.encode(), img.shape[1], img.shape[0], _d(img)))

    def read_image(self, path: str) -> np.ndarray:
        wh = np.zeros(2, np.int32)
        z = np.zeros(1)
        self._ok(self.L.orc_read_image(path.encode(), 0, _i32(wh), _d(z)))
        out = np.zeros(int(wh[0]) * int(wh[1]))
        self._ok(self.L.orc_read_image(path.encode(), out.size, _i32(wh), _d(out)))
        return out.reshape(int(wh[1]), int(wh[0]))

    def write_volume(self, vol, grid: "GridSpec", path: str):
        vol = np.ascontiguousarray(vol, dtype=np.float64)
        self._ok(self.L.orc_write_volume(path.encode(), *grid._args(), _d(vol)))

    def read_volume(self, path: str):
        dims = np.zeros(3, np.int32)
        o, s, z = np.zeros(3), np.zeros(3), np.zeros(1)
        self._ok(self.L.orc_read_volume(path.encode(), 0, _i32(dims), _d(o), _d(s), _d(z)))
        out = np.zeros(int(np.prod(dims)))
        self._ok(self.L.orc_read_volume(path.encode(), out.size, _i32(dims), _d(o), _d(s), _d(out)))
        g = GridSpec(tuple(int(d) for d in dims), tuple(o), tuple(s))
        return out.reshape(g.shape_zyx), g


def reference_io() -> _RefIO:
    return _RefIO()


def ac_stats(h, m):
    out = Stats.zeros(m)
    lib().orc_ac_stats(h, _d(out.grad2d_norm_accum), _i32(out.grad_count), _d(out.grad3d_accum))
    return out


@dataclass
class TrainConfig:  # trainer.hpp:11-45 (fields the hot-path train loop uses)
    iters: int = 30
    lr_position: float = 0.0002
    lr_density: float = 0.01
    lr_scale: float = 0.005
    lr_rotation: float = 0.001
    lr_final_ratio: float = 0.1
    lambda_ssim: float = 0.25
    lambda_tv: float = 0.05
    tv_grid_dim: int = 32
    adaptive_start: int = 500
    adaptive_end: int = 15000
    densify_interval: int = 100
    densify_grad_threshold: float = 0.00005
    prune_density_threshold: float = 0.005
    split_scale_threshold_frac: float = 0.01
    split_factor: float = 1.6
    mode: int = 0
    output_dims: tuple = (64, 64, 64)
    history_interval: int = 10
    seed: int = 0


def train_reference(cloud: Cloud, cfg: ScannerConfig, angles, images, tc: TrainConfig):
    """The reference's own `train` (trainer.cpp:232-345), unmodified, from
    oracle/_ref. images [V][H][W] (un-normalised projections). Returns
    (Cloud, adam dict, Stats, history [n][6] = iter, l1, dssim, tv, total, kernels)."""
    L = _load("reference")
    g, r = cfg._geo()
    imgs = np.ascontiguousarray(images, dtype=np.float64)
    ang = np.ascontiguousarray(angles, dtype=np.float64)
    cd = np.array([tc.lr_position, tc.lr_density, tc.lr_scale, tc.lr_rotation, tc.lr_final_ratio, tc.lambda_ssim,
                   tc.lambda_tv, tc.densify_grad_threshold, tc.prune_density_threshold,
                   tc.split_scale_threshold_frac, tc.split_factor], dtype=np.float64)
    ci = np.array([tc.iters, tc.tv_grid_dim, tc.adaptive_start, tc.adaptive_end, tc.densify_interval, tc.mode,
                   *tc.output_dims, tc.history_interval], dtype=np.int32)
    max_h = tc.iters + 1
    hist = np.zeros(6 * max_h)
    nh = C.c_int(0)
    h = L.orc_train(*cloud._args(), _d(g), _i32(r), len(ang), _d(ang), _d(imgs), _d(cd), _i32(ci), tc.seed,
                    _d(hist), max_h, C.byref(nh))
    if not h:
        raise OracleError(L.orc_last_error().decode())
    try:
        n = L.orc_ac_size(h)
        strides = (1, 3, 3, 4, 1, 1, 3, 3, 3, 3, 4, 4)
        out = []
        for a in range(12):
            buf = np.zeros(max(1, strides[a] * n))
            L.orc_ac_get(h, a, _d(buf))
            out.append(buf[: strides[a] * n])
        st = Stats.zeros(n)
        L.orc_ac_stats(h, _d(st.grad2d_norm_accum), _i32(st.grad_count), _d(st.grad3d_accum))
    finally:
        L.orc_ac_free(h)
    return Cloud(cloud.s_min, *out[:4]), dict(zip(ADAM_KEYS, out[4:])), st, hist[: 6 * nh.value].reshape(-1, 6)
