"""Host-side mirror of the reference's C++ API for the hot path.

Names, argument meaning and error behaviour follow the reference:
  render / render_backward / project_kernel   rasterizer.hpp:36-64
  voxelize / voxelize_backward                voxelizer.hpp:60-67
  tv3d_loss                                   objectives.hpp:31
  l1 + dssim (photometric_loss)               objectives.hpp, trainer.cpp:277-287
  Adam (+ normalize_rotations), lr_at         trainer.cpp:34-36,144-163,310-319
  ScannerConfig / RasterOptions / GridSpec    geometry.hpp:12-31, rasterizer.hpp:15-21, voxelizer.hpp:13-24
  GaussianCloud / CloudGrads                  gaussian_cloud.hpp:31-96
Everything computes through the C ABI of libsplatct_b200.so (include/splatct_gpu.h)
on CUDA device memory held in torch tensors; PyTorch only provides allocation
and streams. Views are batched: ``render`` accepts one angle or a sequence.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Optional, Sequence, Union

import numpy as np
import torch

from . import _capi
from ._capi import sct_adam_state, sct_cloud, sct_grads, sct_grid, sct_raster_opts, sct_scanner, sct_stats


# --------------------------------------------------------------------- errors (common.hpp:27-64)
class SplatctError(RuntimeError):
    pass


class ConfigError(SplatctError):  # exit code 2
    pass


class DataError(SplatctError):  # exit code 3
    pass


class DimMismatch(DataError):
    pass


class DivergenceDetected(SplatctError):  # exit code 4
    pass


class CudaError(SplatctError):  # exit code 5
    pass


def _check(rc: int):
    if rc == 0:
        return
    msg = _capi.load().sct_last_error().decode(errors="replace")
    if rc == 2:
        raise ConfigError(msg)
    if rc == 3:
        raise (DimMismatch if msg.startswith("DimMismatch") else DataError)(msg)
    if rc == 4:
        raise DivergenceDetected(msg)
    if rc == 5:
        raise CudaError(msg)
    raise SplatctError(msg)


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else C.c_void_p(t.data_ptr())


# --------------------------------------------------------------------- geometry / options
@dataclass
class ScannerConfig:
    """geometry.hpp:12-31 (desk-scanner defaults of tests/helpers.hpp:18-28)."""
    l_so_mm: float = 8.0
    l_sd_mm: float = 12.0
    detector_size_mm: tuple = (5.6, 5.6)
    detector_res_px: tuple = (128, 128)
    angles_rad: list = field(default_factory=list)
    extent_min_mm: tuple = (-1.0, -1.0, -1.0)
    extent_max_mm: tuple = (1.0, 1.0, 1.0)
    near_clip_mm: float = 0.0
    parallel_beam: bool = False  # extension (no reference code): orthographic projection

    def near_clip(self):
        return self.near_clip_mm if self.near_clip_mm > 0.0 else 0.01 * self.l_so_mm

    @property
    def width(self):
        return int(self.detector_res_px[0])

    @property
    def height(self):
        return int(self.detector_res_px[1])

    def _c(self) -> sct_scanner:
        s = sct_scanner()
        s.l_so_mm = self.l_so_mm
        s.l_sd_mm = self.l_sd_mm
        s.det_size_mm[:] = [float(x) for x in self.detector_size_mm]
        s.det_res_px[:] = [int(x) for x in self.detector_res_px]
        s.extent_min_mm[:] = [float(x) for x in self.extent_min_mm]
        s.extent_max_mm[:] = [float(x) for x in self.extent_max_mm]
        s.near_clip_mm = self.near_clip_mm
        s.parallel_beam = int(bool(self.parallel_beam))
        return s


def full_circle_angles(n: int):  # geometry.cpp:63-67
    return [2.0 * math.pi * i / n for i in range(n)]


RECTIFIED, BIASED = 0, 1


@dataclass
class RasterOptions:  # rasterizer.hpp:15-21
    mode: int = RECTIFIED
    lowpass_eps_px: float = 0.3
    dilation_compensation: bool = True
    freeze_jacobian: bool = False
    cull_mahalanobis: float = 3.0348542587702925

    def _c(self) -> sct_raster_opts:
        o = sct_raster_opts()
        o.mode = int(self.mode)
        o.lowpass_eps_px = float(self.lowpass_eps_px)
        o.dilation_compensation = int(bool(self.dilation_compensation))
        o.freeze_jacobian = int(bool(self.freeze_jacobian))
        o.cull_mahalanobis = float(self.cull_mahalanobis)
        return o


@dataclass
class VoxelizeOptions:  # voxelizer.hpp:53-57
    cull_mahalanobis: float = 3.3681993876652464


@dataclass
class GridSpec:  # voxelizer.hpp:13-24
    dims: tuple
    origin_mm: tuple = (0.0, 0.0, 0.0)
    spacing_mm: tuple = (1.0, 1.0, 1.0)

    def _c(self) -> sct_grid:
        g = sct_grid()
        g.dims[:] = [int(x) for x in self.dims]
        g.origin_mm[:] = [float(x) for x in self.origin_mm]
        g.spacing_mm[:] = [float(x) for x in self.spacing_mm]
        return g

    @property
    def shape_zyx(self):
        return (int(self.dims[2]), int(self.dims[1]), int(self.dims[0]))

    def voxel_center(self, x, y, z):
        return np.array([self.origin_mm[k] + ((x, y, z)[k] + 0.5) * self.spacing_mm[k] for k in range(3)])

    def voxel_count(self):
        return int(self.dims[0]) * int(self.dims[1]) * int(self.dims[2])


def grid_for_extent(lo, hi, dims) -> GridSpec:  # voxelizer.cpp:8-14
    return GridSpec(tuple(int(d) for d in dims), tuple(float(x) for x in lo),
                    tuple((float(hi[k]) - float(lo[k])) / float(dims[k]) for k in range(3)))


# --------------------------------------------------------------------- cloud / grads
class GaussianCloud:
    """Device SoA parameter store (gaussian_cloud.hpp:31-81), fp32, reference field order:
    rho_raw[M], pos[3M] (xyz per kernel), scale_raw[3M], rot[4M] (w,x,y,z); plus Adam
    moments laid out like the parameters and the adaptive-control statistics."""

    def __init__(self, s_min_mm: float, rho_raw, pos, scale_raw, rot, device="cuda"):
        f = lambda a: torch.as_tensor(np.ascontiguousarray(np.asarray(a, dtype=np.float32).reshape(-1))
                                      if not isinstance(a, torch.Tensor) else a.reshape(-1),
                                      dtype=torch.float32, device=device).contiguous()
        self.s_min = float(s_min_mm)
        self.rho_raw = f(rho_raw)
        self.pos = f(pos)
        self.scale_raw = f(scale_raw)
        self.rot = f(rot)
        m = self.size()
        assert self.pos.numel() == 3 * m and self.scale_raw.numel() == 3 * m and self.rot.numel() == 4 * m
        z = lambda n: torch.zeros(n, dtype=torch.float32, device=self.rho_raw.device)
        self.adam = {k: z(n) for k, n in (("m_rho", m), ("v_rho", m), ("m_pos", 3 * m), ("v_pos", 3 * m),
                                           ("m_scale", 3 * m), ("v_scale", 3 * m), ("m_rot", 4 * m),
                                           ("v_rot", 4 * m))}
        self.grad2d_norm_accum = z(m)
        self.grad_count = torch.zeros(m, dtype=torch.int32, device=self.rho_raw.device)
        self.grad3d_accum = z(3 * m)

    def size(self) -> int:
        return int(self.rho_raw.numel())

    def s_min_mm(self) -> float:
        return self.s_min

    def reset_grad_stats(self):
        self.grad2d_norm_accum.zero_()
        self.grad_count.zero_()
        self.grad3d_accum.zero_()

    def _c(self) -> sct_cloud:
        c = sct_cloud()
        c.m = self.size()
        c.s_min_mm = self.s_min
        c.rho_raw = self.rho_raw.data_ptr()
        c.pos = self.pos.data_ptr()
        c.scale_raw = self.scale_raw.data_ptr()
        c.rot = self.rot.data_ptr()
        return c

    def _stats_c(self) -> sct_stats:
        s = sct_stats()
        s.grad2d_norm_accum = self.grad2d_norm_accum.data_ptr()
        s.grad_count = self.grad_count.data_ptr()
        s.grad3d_accum = self.grad3d_accum.data_ptr()
        return s

    def _adam_c(self) -> sct_adam_state:
        a = sct_adam_state()
        for k, t in self.adam.items():
            setattr(a, k, t.data_ptr())
        return a

    def host_arrays(self):
        return {k: getattr(self, k).detach().cpu().numpy() for k in ("rho_raw", "pos", "scale_raw", "rot")}


class CloudGrads:
    """gaussian_cloud.hpp:84-96 — accumulate (+=) semantics; zero with resize()."""

    def __init__(self, m: int, device="cuda"):
        self.resize(m, device)

    def resize(self, m: int, device="cuda"):
        # one contiguous buffer (11 floats per kernel) so a single collective
        # can reduce all four groups; the group tensors are views into it
        self.buffer = torch.zeros(11 * m, dtype=torch.float32, device=device)
        self.rho_raw, self.pos, self.scale_raw, self.rot = torch.split(self.buffer, [m, 3 * m, 3 * m, 4 * m])

    def zero_(self):
        self.buffer.zero_()

    def flat(self) -> torch.Tensor:
        return self.buffer

    def tensors(self):
        return [self.rho_raw, self.pos, self.scale_raw, self.rot]

    def _c(self) -> sct_grads:
        g = sct_grads()
        g.rho_raw = self.rho_raw.data_ptr()
        g.pos = self.pos.data_ptr()
        g.scale_raw = self.scale_raw.data_ptr()
        g.rot = self.rot.data_ptr()
        return g


# --------------------------------------------------------------------- engine context
class Engine:
    """One sct_ctx bound to a CUDA device and stream (its calls are serialised on it)."""

    def __init__(self, device: Optional[int] = None, stream: Optional[torch.cuda.Stream] = None,
                 deterministic: bool = True):
        if not torch.cuda.is_available():
            raise CudaError("splatct-b200 needs a CUDA device (sm_100a); there is no CPU fallback")
        self.lib = _capi.load()
        self.device_index = torch.cuda.current_device() if device is None else int(device)
        self.device = torch.device("cuda", self.device_index)
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        h = C.c_void_p()
        _check(self.lib.sct_ctx_create(self.device_index, C.c_void_p(self.stream.cuda_stream), C.byref(h)))
        self._h = h
        _check(self.lib.sct_ctx_set_deterministic(self._h, int(deterministic)))

    def __del__(self):
        if getattr(self, "_h", None):
            try:
                self.lib.sct_ctx_destroy(self._h)
            except Exception:
                pass
            self._h = None

    def set_deterministic(self, deterministic: bool = True):
        """Backward reduction: fixed-order per-(tile, kernel) slots (default) or the
        parallel-atomic per-item accumulation (sct_ctx_set_deterministic)."""
        _check(self.lib.sct_ctx_set_deterministic(self._h, int(deterministic)))

    def set_stream(self, stream: torch.cuda.Stream):
        self.stream = stream
        _check(self.lib.sct_ctx_set_stream(self._h, C.c_void_p(stream.cuda_stream)))

    def synchronize(self):
        _check(self.lib.sct_ctx_sync(self._h))

    def kernel_launches(self) -> int:
        return int(self.lib.sct_ctx_kernel_launches(self._h))

    def set_capacity(self, raster_pairs: int = 0, voxel_pairs: int = 0):
        """Sync-free binning: fixed-capacity pair buffers instead of a host readback of
        each binning's pair count (0 = exact mode, the default). Pairs beyond a capacity
        are dropped and recorded; check take_overflow() before trusting results."""
        _check(self.lib.sct_ctx_set_capacity(self._h, int(raster_pairs), int(voxel_pairs)))

    def take_overflow(self) -> bool:
        """Synchronises; True when a capacity-mode binning overflowed since the last call."""
        f = C.c_int32(0)
        _check(self.lib.sct_ctx_take_overflow(self._h, C.byref(f)))
        return bool(f.value)

    def set_timing(self, enable: bool):
        """Bracket every engine launch with CUDA events on the context stream."""
        _check(self.lib.sct_ctx_set_timing(self._h, int(enable)))

    def timing_report(self) -> dict:
        """{kernel: (total_ms, launches)} since the last report (synchronises)."""
        import json
        buf = C.create_string_buffer(1 << 16)
        _check(self.lib.sct_ctx_timing_report(self._h, buf, len(buf)))
        return {k: (float(v[0]), int(v[1])) for k, v in json.loads(buf.value.decode()).items()}

    def voxel_work(self, cloud: "GaussianCloud", grid: "GridSpec", opts: Optional["VoxelizeOptions"] = None):
        """(VGE, pairs) of a full-grid voxelize: the algorithmic work unit of K7/K8."""
        opts = opts or VoxelizeOptions()
        cl, g = cloud._c(), grid._c()
        vge, n = C.c_int64(0), C.c_int64(0)
        _check(self.lib.sct_voxel_work(self._h, C.byref(cl), C.byref(g), float(opts.cull_mahalanobis), C.byref(vge),
                                       C.byref(n)))
        return int(vge.value), int(n.value)

    # ------------------------------------------------------------- rasterizer
    def render(self, cloud: GaussianCloud, config: ScannerConfig, theta_rad: Union[float, Sequence[float]],
               opts: Optional[RasterOptions] = None, out: Optional[torch.Tensor] = None) -> "RenderedProjection":
        opts = opts or RasterOptions()
        single = isinstance(theta_rad, (int, float))
        thetas = [float(theta_rad)] if single else [float(t) for t in theta_rad]
        n = len(thetas)
        if out is None:
            out = torch.empty((n, config.height, config.width), dtype=torch.float32, device=self.device)
        th = (C.c_double * n)(*thetas)
        state = C.c_void_p()
        cl, sc, op = cloud._c(), config._c(), opts._c()
        _check(self.lib.sct_render_fwd(self._h, C.byref(cl), C.byref(sc), th, n, C.byref(op), _ptr(out),
                                       C.byref(state)))
        return RenderedProjection(self, state, out, config, thetas, opts, single)

    def render_backward(self, cloud: GaussianCloud, fwd: "RenderedProjection", dL_dimage: torch.Tensor,
                        grads: CloudGrads, accumulate_stats: bool = False):
        dl = self._check_upstream(fwd, dL_dimage)
        cl, g = cloud._c(), grads._c()
        st = cloud._stats_c() if accumulate_stats else None
        _check(self.lib.sct_render_bwd(self._h, fwd._state, C.byref(cl), _ptr(dl), C.byref(g),
                                       C.byref(st) if st is not None else None))

    def _check_upstream(self, fwd: "RenderedProjection", dL_dimage: torch.Tensor) -> torch.Tensor:
        dl = dL_dimage
        expect = (len(fwd.thetas), fwd.config.height, fwd.config.width)
        if dl.dim() == 2:
            dl = dl.unsqueeze(0)
        if tuple(dl.shape) != expect:
            raise DimMismatch("render_backward: upstream gradient dims mismatch")
        return dl.to(device=self.device, dtype=torch.float32).contiguous()

    def project_kernels(self, cloud: GaussianCloud, config: ScannerConfig, theta_rad: float,
                        opts: Optional[RasterOptions] = None):
        """project_kernel for every kernel (FP64). Returns (visible[m] bool, rec[m,11] float64)."""
        opts = opts or RasterOptions()
        m = cloud.size()
        vis = np.zeros(max(m, 1), dtype=np.int32)
        rec = np.zeros((max(m, 1), 11), dtype=np.float64)
        cl, sc, op = cloud._c(), config._c(), opts._c()
        _check(self.lib.sct_project_kernels(self._h, C.byref(cl), C.byref(sc), float(theta_rad), C.byref(op),
                                            vis.ctypes.data_as(_capi.I32), rec.ctypes.data_as(_capi.D)))
        return vis[:m].astype(bool), rec[:m]

    # ------------------------------------------------------------- voxelizer
    def voxelize(self, cloud: GaussianCloud, grid: GridSpec, opts: Optional[VoxelizeOptions] = None,
                 z_bricks: Optional[tuple] = None, out: Optional[torch.Tensor] = None, keep_state: bool = False):
        """voxelizer.cpp:108-138. keep_state=True returns (volume, VoxelState): the brick lists
        stay alive for voxelize_backward(state=...) instead of being rebuilt (the cloud must
        not change in between)."""
        opts = opts or VoxelizeOptions()
        if out is None:
            out = (torch.empty if z_bricks is None else torch.zeros)(grid.shape_zyx, dtype=torch.float32,
                                                                      device=self.device)
        zb0, zb1 = z_bricks if z_bricks is not None else (0, 2 ** 31 - 1)
        cl, g = cloud._c(), grid._c()
        if keep_state:
            h = C.c_void_p()
            _check(self.lib.sct_voxelize_fwd_state(self._h, C.byref(cl), C.byref(g), float(opts.cull_mahalanobis),
                                                   zb0, zb1, _ptr(out), C.byref(h)))
            return out, VoxelState(self, h, grid)
        _check(self.lib.sct_voxelize_fwd(self._h, C.byref(cl), C.byref(g), float(opts.cull_mahalanobis), zb0, zb1,
                                         _ptr(out)))
        return out

    def voxelize_backward(self, cloud: GaussianCloud, grid: GridSpec, dL_dV: torch.Tensor, grads: CloudGrads,
                          opts: Optional[VoxelizeOptions] = None, z_bricks: Optional[tuple] = None,
                          state: Optional["VoxelState"] = None):
        """voxelizer.cpp:140-224; accumulates into grads. With `state` (from voxelize(keep_state=True))
        the forward's brick lists are reused (grid / cull / slab are the state's)."""
        opts = opts or VoxelizeOptions()
        if tuple(dL_dV.shape) != grid.shape_zyx:
            raise DimMismatch("voxelize_backward: gradient volume dims mismatch")
        dl = dL_dV.to(device=self.device, dtype=torch.float32).contiguous()
        cl, gr = cloud._c(), grads._c()
        if state is not None:
            _check(self.lib.sct_voxelize_bwd_state(self._h, state._h, C.byref(cl), _ptr(dl), C.byref(gr)))
            return
        zb0, zb1 = z_bricks if z_bricks is not None else (0, 2 ** 31 - 1)
        g = grid._c()
        _check(self.lib.sct_voxelize_bwd(self._h, C.byref(cl), C.byref(g), float(opts.cull_mahalanobis), zb0, zb1,
                                         _ptr(dl), C.byref(gr)))

    def voxelize_backward_allreduce(self, cloud: GaussianCloud, grid: GridSpec, dL_dV: torch.Tensor,
                                    grads: CloudGrads, opts: Optional[VoxelizeOptions] = None,
                                    z_bricks: Optional[tuple] = None):
        """voxelize_backward over this rank's z-slab, summed over all ranks before the += into grads."""
        opts = opts or VoxelizeOptions()
        if tuple(dL_dV.shape) != grid.shape_zyx:
            raise DimMismatch("voxelize_backward: gradient volume dims mismatch")
        dl = dL_dV.to(device=self.device, dtype=torch.float32).contiguous()
        zb0, zb1 = z_bricks if z_bricks is not None else (0, 2 ** 31 - 1)
        cl, g, gr = cloud._c(), grid._c(), grads._c()
        _check(self.lib.sct_voxelize_bwd_allreduce(self._h, C.byref(cl), C.byref(g), float(opts.cull_mahalanobis),
                                                   zb0, zb1, _ptr(dl), C.byref(gr)))

    def voxel_bins(self, cloud: GaussianCloud, grid: GridSpec, opts: Optional[VoxelizeOptions] = None):
        opts = opts or VoxelizeOptions()
        cl, g = cloud._c(), grid._c()
        n = C.c_int64(0)
        _check(self.lib.sct_voxel_bins(self._h, C.byref(cl), C.byref(g), float(opts.cull_mahalanobis), C.byref(n),
                                       None, None))
        nb = 1
        for d in grid.dims:
            nb *= (int(d) + 7) // 8
        off = np.zeros(nb + 1, dtype=np.int64)
        idx = np.zeros(max(n.value, 1), dtype=np.int32)
        _check(self.lib.sct_voxel_bins(self._h, C.byref(cl), C.byref(g), float(opts.cull_mahalanobis), C.byref(n),
                                       off.ctypes.data_as(_capi.I64), idx.ctypes.data_as(_capi.I32)))
        return off, idx[: n.value]

    # ------------------------------------------------------------- objectives / optimizer
    def tv3d_loss(self, vol: torch.Tensor, lam: float = 1.0):
        """objectives.cpp:169-202. Returns (value: 0-d float64 device tensor, lam * grad)."""
        if vol.dim() != 3 or min(vol.shape) < 2:
            raise DimMismatch("tv3d_loss: need at least 2 voxels per axis")
        v = vol.contiguous()
        grad = torch.empty_like(v)
        val = torch.empty((), dtype=torch.float64, device=self.device)
        dims = (C.c_int32 * 3)(v.shape[2], v.shape[1], v.shape[0])
        _check(self.lib.sct_tv3d(self._h, _ptr(v), dims, float(lam), _ptr(val), _ptr(grad)))
        return val, grad

    def photometric_loss(self, rendered: torch.Tensor, measured: torch.Tensor, render_scale: float = 1.0,
                         lambda_ssim: float = 0.25, grad_scale: float = 1.0):
        """L1 + lambda * D-SSIM per image (objectives.cpp:113-167) on rendered*render_scale vs measured;
        returns (values [n,2] float64 device: l1, dssim) and dL/dI = (g_l1 + lambda g_dssim) * grad_scale."""
        r = rendered if rendered.dim() == 3 else rendered.unsqueeze(0)
        m = measured if measured.dim() == 3 else measured.unsqueeze(0)
        if r.shape != m.shape:
            raise DimMismatch("photometric loss: image dims differ")
        r, m = r.contiguous(), m.contiguous()
        n, h, w = r.shape
        vals = torch.empty((n, 2), dtype=torch.float64, device=self.device)
        dL = torch.empty_like(r)
        _check(self.lib.sct_photometric_loss(self._h, _ptr(r), _ptr(m), n, w, h, float(render_scale),
                                             float(lambda_ssim), float(grad_scale), _ptr(vals), _ptr(dL)))
        return vals, dL

    def adam_step(self, cloud: GaussianCloud, grads: CloudGrads, t: int, lr: Sequence[float],
                  beta1: float = 0.9, beta2: float = 0.999, eps: float = 1e-15):
        """trainer.cpp:144-163 for pos, rho, scale, rot (lr in that order), then normalize_rotations."""
        cl, st, g = cloud._c(), cloud._adam_c(), grads._c()
        lrs = (C.c_double * 4)(*[float(x) for x in lr])
        _check(self.lib.sct_adam_step(self._h, C.byref(cl), C.byref(st), C.byref(g), int(t), lrs, beta1, beta2, eps))

    def train_step(self, cloud: GaussianCloud, grads: CloudGrads, config: ScannerConfig, theta_rad: float,
                   measured: torch.Tensor, t: int, lr: Sequence[float], values: torch.Tensor,
                   opts: Optional[RasterOptions] = None, render_scale: float = 1.0, grad_scale: float = 1.0,
                   lambda_ssim: float = 0.25, lambda_tv: float = 0.0, tv_grid: Optional[GridSpec] = None,
                   accumulate_stats: bool = True, beta1: float = 0.9, beta2: float = 0.999, eps: float = 1e-15,
                   vox_opts: Optional[VoxelizeOptions] = None, _structs=None):
        """One native training iteration (sct_train_step, trainer.cpp:268-319): render, L1 + D-SSIM,
        zero grads + render_backward (+ adaptive stats), TV on tv_grid when lambda_tv > 0, Adam step t.
        values (device float64 [4]) receives l1, dssim, tv, total. No host synchronisation in
        capacity mode. _structs: cached (scanner, opts, cloud, adam, stats, grads) ctypes structs."""
        if (measured.shape != (config.height, config.width) or measured.dtype != torch.float32
                or not measured.is_contiguous() or measured.device != self.device):
            raise DimMismatch("train_step: measured must be a contiguous float32 [H][W] tensor on the engine's device")
        if values.numel() < 4 or values.dtype != torch.float64:
            raise DimMismatch("train_step: values must be float64 [4]")
        if _structs is None:
            _structs = ((config._c(), (opts or RasterOptions())._c()) +
                        (cloud._c(), cloud._adam_c(), cloud._stats_c(), grads._c()))
        sc, op, cl, ad, st, g = _structs
        a = _capi.sct_train_args()
        a.theta_rad = float(theta_rad)
        a.measured = measured.data_ptr()
        a.render_scale, a.grad_scale = float(render_scale), float(grad_scale)
        a.lambda_ssim, a.lambda_tv = float(lambda_ssim), float(lambda_tv)
        if lambda_tv > 0.0:
            a.tv_grid = tv_grid._c()
        a.cull_mahalanobis = float((vox_opts or VoxelizeOptions()).cull_mahalanobis)
        a.t = int(t)
        a.lr[:] = [float(x) for x in lr]
        a.beta1, a.beta2, a.eps = float(beta1), float(beta2), float(eps)
        a.values_dev = values.data_ptr()
        _check(self.lib.sct_train_step(self._h, C.byref(cl), C.byref(ad), C.byref(st) if accumulate_stats else None,
                                       C.byref(g), C.byref(sc), C.byref(op), C.byref(a)))

    # ------------------------------------------------------------- multi-GPU exchange (comm.cu)
    def comm_init(self, rank: int, world: int, unique_id: Optional[bytes] = None):
        """Context-owned NCCL communicator over `world` ranks. Without ``unique_id`` the id is
        made on rank 0 and broadcast over the default torch.distributed group."""
        if unique_id is None:
            buf = (C.c_uint8 * 128)()
            if rank == 0:
                _check(self.lib.sct_nccl_unique_id(buf))
            if world > 1:
                import torch.distributed as dist
                obj = [bytes(buf)]
                dist.broadcast_object_list(obj, src=0)
                unique_id = obj[0]
            else:
                unique_id = bytes(buf)
        uid = (C.c_uint8 * 128).from_buffer_copy(unique_id)
        _check(self.lib.sct_ctx_comm_init(self._h, int(world), int(rank), uid))

    def comm_info(self):
        n, r = C.c_int32(), C.c_int32()
        _check(self.lib.sct_ctx_comm_info(self._h, C.byref(n), C.byref(r)))
        return int(n.value), int(r.value)

    def allreduce_grads(self, grads: CloudGrads, cloud: Optional[GaussianCloud] = None):
        """In-place sum over ranks of grads (and of cloud's adaptive statistics when given)."""
        g = grads._c()
        st = cloud._stats_c() if cloud is not None else None
        _check(self.lib.sct_allreduce_grads(self._h, int(grads.rho_raw.numel()), C.byref(g),
                                            C.byref(st) if st is not None else None))

    def render_backward_allreduce(self, cloud: GaussianCloud, fwd: "RenderedProjection", dL_dimage: torch.Tensor,
                                  grads: CloudGrads, accumulate_stats: bool = False):
        """render_backward whose contribution is summed over all ranks before the += into grads."""
        dl = self._check_upstream(fwd, dL_dimage)
        cl, g = cloud._c(), grads._c()
        st = cloud._stats_c() if accumulate_stats else None
        _check(self.lib.sct_render_bwd_allreduce(self._h, fwd._state, C.byref(cl), _ptr(dl), C.byref(g),
                                                 C.byref(st) if st is not None else None))

    def adaptive_control(self, cloud: GaussianCloud, extent_size_mm: Sequence[float],
                         prune_density_threshold: float = 0.005, densify_grad_threshold: float = 0.00005,
                         split_scale_threshold_frac: float = 0.01, split_factor: float = 1.6,
                         gauss: Optional[torch.Tensor] = None, generator: Optional[torch.Generator] = None,
                         rng: Optional["HostRng"] = None):
        """trainer.cpp:167-230 on the device: prune, clone, split; returns (new cloud with carried /
        zeroed Adam state and reset statistics, (pruned, cloned, split)). The split positions use
        6 standard-normal draws per split kernel (z, y, x per child): from ``rng`` (the trainer's
        std::mt19937_64 stream, one normal_distribution per call like the reference), or
        ``gauss`` supplied directly, else torch.randn."""
        if not split_factor > 1.0:
            raise ConfigError("train: split_factor must be > 1")
        cl, st = cloud._c(), cloud._stats_c()
        ext = (C.c_double * 3)(*[float(x) for x in extent_size_mm])
        plan, new_m, n_split = C.c_void_p(), C.c_int64(), C.c_int64()
        counts = (C.c_int32 * 3)()
        _check(self.lib.sct_adaptive_plan(self._h, C.byref(cl), C.byref(st), float(prune_density_threshold),
                                          float(densify_grad_threshold), float(split_scale_threshold_frac),
                                          float(split_factor), ext, C.byref(plan), C.byref(new_m),
                                          C.byref(n_split), counts))
        try:
            n, ns = int(new_m.value), int(n_split.value)
            e = lambda k: torch.empty(k * n, dtype=torch.float32, device=self.device)
            out = GaussianCloud(cloud.s_min, e(1), e(3), e(3), e(4), device=self.device)
            if ns > 0:
                if gauss is None:
                    if rng is not None:  # the reference's stream (trainer.cpp:184,213-216)
                        gauss = torch.from_numpy(rng.normal(6 * ns))
                    else:
                        gauss = torch.randn(6 * ns, dtype=torch.float64, device=self.device, generator=generator)
                gauss = gauss.to(device=self.device, dtype=torch.float64).contiguous()
                if gauss.numel() < 6 * ns:
                    raise ConfigError(f"adaptive control: need {6 * ns} normal draws, got {gauss.numel()}")
            ocl, ost, ast = out._c(), out._adam_c(), cloud._adam_c()
            _check(self.lib.sct_adaptive_apply(self._h, plan, C.byref(cl), C.byref(ast),
                                               _ptr(cloud.grad3d_accum), _ptr(gauss) if ns > 0 else None,
                                               C.byref(ocl), C.byref(ost)))
        finally:
            self.lib.sct_adaptive_free(plan)
        return out, tuple(int(x) for x in counts)


class HostRng:
    """The reference trainer's single std::mt19937_64 stream (trainer.cpp:254-258),
    product host code in the engine library (csrc/rng.cu): libstdc++'s engine,
    std::shuffle and distributions, drawn in the reference's order."""

    def __init__(self, seed: int):
        self.lib = _capi.load()
        h = C.c_void_p()
        _check(self.lib.sct_rng_create(int(seed) & ((1 << 64) - 1), C.byref(h)))
        self._h = h

    def shuffle(self, values: np.ndarray) -> np.ndarray:
        """std::shuffle in place (int32 array)."""
        assert values.dtype == np.int32 and values.flags.c_contiguous
        _check(self.lib.sct_rng_shuffle(self._h, values.ctypes.data_as(C.POINTER(C.c_int32)), int(values.size)))
        return values

    def subvolume_origin(self, lo, hi, spacing, d: int):
        a = [(C.c_double * 3)(*[float(x) for x in v]) for v in (lo, hi, spacing)]
        out = (C.c_double * 3)()
        _check(self.lib.sct_rng_subvolume_origin(self._h, a[0], a[1], a[2], int(d), out))
        return tuple(out)

    def normal(self, n: int) -> np.ndarray:
        out = np.zeros(max(1, n), dtype=np.float64)
        _check(self.lib.sct_rng_normal(self._h, int(n), out.ctypes.data_as(C.POINTER(C.c_double))))
        return out[:n]

    def uniform(self, n: int, lo: float = 0.0, hi: float = 1.0) -> np.ndarray:
        out = np.zeros(max(1, n), dtype=np.float64)
        _check(self.lib.sct_rng_uniform(self._h, int(n), float(lo), float(hi),
                                        out.ctypes.data_as(C.POINTER(C.c_double))))
        return out[:n]

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                self.lib.sct_rng_destroy(h)
            except Exception:  # noqa: BLE001 (interpreter shutdown)
                pass
            self._h = None


class VoxelState:
    """Brick lists of one voxelize call, reused by voxelize_backward(state=...)."""

    def __init__(self, engine: Engine, handle, grid: GridSpec):
        self._engine, self._h, self.grid = engine, handle, grid

    def free(self):
        if getattr(self, "_h", None):
            self._engine.lib.sct_vox_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:  # noqa: BLE001 (interpreter shutdown)
            pass


class RenderedProjection:
    """rasterizer.hpp:41-51: images + the forward state (tile lists) for the backward."""

    def __init__(self, engine: Engine, state, images, config, thetas, opts, single):
        self._engine = engine
        self._state = state
        self.images = images
        self.config = config
        self.thetas = thetas
        self.opts = opts
        self._single = single

    @property
    def image(self) -> torch.Tensor:
        return self.images[0] if self._single else self.images

    @property
    def tiles_x(self):
        return (self.config.width + 15) // 16

    @property
    def tiles_y(self):
        return (self.config.height + 15) // 16

    def n_pairs(self) -> int:
        n = C.c_int64(0)
        _check(self._engine.lib.sct_fwd_info(self._state, C.byref(n), None, None, None))
        return int(n.value)

    def work(self):
        """(GPE, pairs): Gaussian-pixel evaluations of this forward (= of its backward)."""
        g, n = C.c_int64(0), C.c_int64(0)
        _check(self._engine.lib.sct_fwd_work(self._state, C.byref(g), C.byref(n)))
        return int(g.value), int(n.value)

    def n_visible(self) -> int:
        n = C.c_int64(0)
        _check(self._engine.lib.sct_fwd_info(self._state, None, None, None, C.byref(n)))
        return int(n.value)

    def tile_lists(self, view: int = 0):
        """(offsets[T+1] int64, kernel_idx int32) — RenderedProjection::tile_visible mapped to
        kernel indices (visible[vi].kernel_index), ascending within each tile."""
        T = self.tiles_x * self.tiles_y
        off = np.zeros(T + 1, dtype=np.int64)
        _check(self._engine.lib.sct_fwd_tile_lists(self._state, view, off.ctypes.data_as(_capi.I64), None))
        idx = np.zeros(max(int(off[-1]), 1), dtype=np.int32)
        _check(self._engine.lib.sct_fwd_tile_lists(self._state, view, off.ctypes.data_as(_capi.I64),
                                                   idx.ctypes.data_as(_capi.I32)))
        return off, idx[: int(off[-1])]

    def free(self):
        if getattr(self, "_state", None):
            self._engine.lib.sct_fwd_free(self._state)
            self._state = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def lr_at(lr_init: float, final_ratio: float, t: int, iters: int) -> float:  # trainer.cpp:34-36
    return float(_capi.load().sct_lr_at(lr_init, final_ratio, t, iters))


# --------------------------------------------------------------------- reference-named free functions
_default: dict = {}


def default_engine() -> Engine:
    dev = torch.cuda.current_device()
    e = _default.get(dev)
    if e is None:
        e = _default[dev] = Engine(dev)
    return e


def render(cloud, config, theta_rad, opts=None):
    return default_engine().render(cloud, config, theta_rad, opts)


def render_backward(cloud, config, theta_rad, fwd, dL_dimage, grads, opts=None, accumulate_stats=False):
    """Reference signature (rasterizer.hpp:61-64). config/theta/opts must match the forward."""
    if opts is not None and opts != fwd.opts:
        raise ConfigError("render_backward: options differ from the forward pass")
    return default_engine().render_backward(cloud, fwd, dL_dimage, grads, accumulate_stats)


def project_kernels(cloud, config, theta_rad, opts=None):
    return default_engine().project_kernels(cloud, config, theta_rad, opts)


def voxelize(cloud, grid, opts=None):
    return default_engine().voxelize(cloud, grid, opts)


def voxelize_backward(cloud, grid, dL_dV, grads, opts=None):
    return default_engine().voxelize_backward(cloud, grid, dL_dV, grads, opts)


def tv3d_loss(vol, lam=1.0):
    return default_engine().tv3d_loss(vol, lam)


class Adam:
    """trainer.cpp:144-163 (beta 0.9/0.999, eps 1e-15, global-step bias correction)."""

    def __init__(self, beta1=0.9, beta2=0.999, eps=1e-15, engine: Optional[Engine] = None):
        self.beta1, self.beta2, self.eps = beta1, beta2, eps
        self.step_count = 0
        self.engine = engine

    def step(self, cloud: GaussianCloud, grads: CloudGrads, lr: Sequence[float]):
        self.step_count += 1
        (self.engine or default_engine()).adam_step(cloud, grads, self.step_count, lr, self.beta1, self.beta2,
                                                    self.eps)
