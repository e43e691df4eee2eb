"""Device-resident training iteration of the reference trainer (BASELINE
configs[1], "full train step"): trainer.cpp:266-330, adaptive control included.

One iteration = render the selected view(s) (rasterizer.cpp:112-157), form
L1 + lambda_ssim * D-SSIM on projections normalised by the dataset maximum and
the matching dL/dI (objectives.cpp:113-167, trainer.cpp:277-287),
render_backward with adaptive statistics (trainer.cpp:288), the TV term on a D^3
sub-grid at the output spacing (voxelize -> tv3d_loss -> lambda_tv-scaled
voxelize_backward, trainer.cpp:290-300), the non-finite check
(trainer.cpp:302-308) and the four Adam groups with the exponential learning
rate followed by quaternion renormalisation (trainer.cpp:310-319) — all on the
GPU through the C ABI; the host only picks the view and the sub-grid origin,
from the reference's own random stream: one std::mt19937_64(cfg.seed)
(trainer.cpp:254-258) with libstdc++'s std::shuffle and distributions
(engine.HostRng, csrc/rng.cu), consumed in the reference's order — view
shuffle at each epoch start, the sub-volume origin every iteration, the split
draws of adaptive control — so a seed selects the same views, sub-grids and
split positions as the reference trainer.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np
import torch

from .engine import (CloudGrads, DataError, DivergenceDetected, Engine, GaussianCloud, GridSpec, HostRng,
                     RasterOptions, ScannerConfig, lr_at)


@dataclass
class TrainConfig:  # trainer.hpp:13-44 (the fields the iteration uses)
    iters: int = 30000
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
    split_scale_threshold_frac: float = 0.01  # of the max extent side
    split_factor: float = 1.6
    output_dims: tuple = (64, 64, 64)
    seed: int = 0
    mode: int = 0
    check_every: int = 1  # iterations between host-side non-finite checks
    # Sync-free binning (Engine.set_capacity): after a calibration iteration in
    # exact mode (the first one, and the first after each adaptive control) the
    # pair buffers get `capacity_margin` x the measured pair counts and no
    # binning reads its count back to the host. Overflow is checked with the
    # non-finite check (every check_every iterations) and raises DataError.
    sync_free: bool = False
    capacity_margin: float = 3.0
    # One native call per iteration (Engine.train_step -> sct_train_step, the same
    # launches in the same order) instead of the call-by-call Python sequence below;
    # calibration iterations of sync-free mode take the Python path (they read counts).
    native: bool = True


def random_subvolume_origin(lo, hi, spacing, d, u):
    """voxelizer.cpp:226-239 with the uniform draws u[3] supplied by the caller."""
    out = []
    for k in range(3):
        span = (hi[k] - lo[k]) - d * spacing[k]
        out.append(lo[k] + u[k] * span if span > 0.0 else 0.5 * (lo[k] + hi[k]) - 0.5 * d * spacing[k])
    return tuple(out)


class Trainer:
    def __init__(self, engine: Engine, cloud: GaussianCloud, scanner: ScannerConfig, angles: Sequence[float],
                 projections: torch.Tensor, cfg: TrainConfig):
        self.eng, self.cloud, self.scanner, self.cfg = engine, cloud, scanner, cfg
        self.angles = list(angles)
        proj = projections.to(engine.device, torch.float32).contiguous()
        norm = float(proj.max().item())  # trainer.cpp:243-246
        if not norm > 0.0:
            norm = 1.0
        self.inv_norm = 1.0 / norm
        self.measured_norm = proj * self.inv_norm  # trainer.cpp:248-252
        self.grads = CloudGrads(cloud.size(), device=engine.device)
        ext = [scanner.extent_max_mm[k] - scanner.extent_min_mm[k] for k in range(3)]
        self.output_spacing = tuple(ext[k] / cfg.output_dims[k] for k in range(3))
        self.opts = RasterOptions(mode=cfg.mode)
        self.t = 0
        self.rng = HostRng(cfg.seed)
        self.order = np.arange(len(self.angles), dtype=np.int32)  # trainer.cpp:255-256
        self.epoch_pos = len(self.angles)  # forces a shuffle on first use
        self._calibrate = cfg.sync_free  # next iteration measures the pair counts (exact mode)

    def next_view(self) -> int:
        """Shuffled epochs (trainer.cpp:269-273): the order is reshuffled in place."""
        if self.epoch_pos >= len(self.angles):
            self.rng.shuffle(self.order)
            self.epoch_pos = 0
        v = int(self.order[self.epoch_pos])
        self.epoch_pos += 1
        return v

    def step(self, view: Optional[int] = None, sub_origin: Optional[tuple] = None) -> dict:
        cfg, eng, cloud = self.cfg, self.eng, self.cloud
        self.t += 1
        t = self.t
        if view is None:
            view = self.next_view()
        calibrate = self._calibrate
        if cfg.native and not calibrate:
            return self._step_native(view, sub_origin)
        if calibrate:
            eng.set_capacity(0, 0)
        fwd = eng.render(cloud, self.scanner, self.angles[view], self.opts)
        raster_pairs = fwd.n_pairs() if calibrate else 0
        vals, dL = eng.photometric_loss(fwd.images, self.measured_norm[view:view + 1], render_scale=self.inv_norm,
                                        lambda_ssim=cfg.lambda_ssim, grad_scale=self.inv_norm)
        self.grads.zero_()  # grads.resize(M), trainer.cpp:283
        eng.render_backward(cloud, fwd, dL, self.grads, accumulate_stats=True)
        fwd.free()
        tv = torch.zeros((), dtype=torch.float64, device=eng.device)
        if cfg.lambda_tv > 0.0:
            if sub_origin is None:  # voxelizer.cpp:226-239 on the trainer's stream
                sub_origin = self.rng.subvolume_origin(self.scanner.extent_min_mm, self.scanner.extent_max_mm,
                                                       self.output_spacing, cfg.tv_grid_dim)
            d = cfg.tv_grid_dim
            sub = GridSpec((d, d, d), sub_origin, self.output_spacing)
            if calibrate:  # the densest sub-grid placement bounds the TV binning
                full = GridSpec(tuple(int(round((self.scanner.extent_max_mm[k] - self.scanner.extent_min_mm[k])
                                                / self.output_spacing[k])) for k in range(3)),
                                tuple(self.scanner.extent_min_mm), self.output_spacing)
                self._voxel_pairs = max(1, eng.voxel_work(cloud, full)[1])
            vol, vstate = eng.voxelize(cloud, sub, keep_state=True)  # bins once for fwd + bwd
            tv, g_tv = eng.tv3d_loss(vol, cfg.lambda_tv)
            eng.voxelize_backward(cloud, sub, g_tv, self.grads, state=vstate)
            vstate.free()
        total = vals[0, 0] + cfg.lambda_ssim * vals[0, 1] + cfg.lambda_tv * tv  # trainer.cpp:302-303
        if cfg.check_every and t % cfg.check_every == 0:
            if not math.isfinite(float(total.item())):
                raise DivergenceDetected(f"non-finite loss at iteration {t}")
            if cfg.sync_free and not calibrate and eng.take_overflow():
                raise DataError(f"sync-free binning exceeded its pair capacity by iteration {t}; "
                                "raise TrainConfig.capacity_margin")
        if calibrate:
            # a sub-grid's pairs are bounded by the full-extent grid's (same brick size; at
            # most 8x from the brick alignment), capped by the margin
            vp = getattr(self, "_voxel_pairs", 0)
            eng.set_capacity(int(cfg.capacity_margin * raster_pairs) + 65536,
                             int(min(8 * vp, cfg.capacity_margin * vp)) + 65536 if cfg.lambda_tv > 0.0 else 0)
            self._calibrate = False
        lrs = [lr_at(cfg.lr_position, cfg.lr_final_ratio, t, cfg.iters),
               lr_at(cfg.lr_density, cfg.lr_final_ratio, t, cfg.iters),
               lr_at(cfg.lr_scale, cfg.lr_final_ratio, t, cfg.iters),
               lr_at(cfg.lr_rotation, cfg.lr_final_ratio, t, cfg.iters)]
        eng.adam_step(cloud, self.grads, t, lrs)  # trainer.cpp:310-319
        adapted = None
        if (cfg.adaptive_start <= t <= cfg.adaptive_end and t > cfg.adaptive_start
                and (t - cfg.adaptive_start) % cfg.densify_interval == 0):  # trainer.cpp:321-323
            adapted = self.adaptive_control()
        return {"iter": t, "view": view, "l1": vals[0, 0], "dssim": vals[0, 1], "tv": tv, "total": total,
                "kernels": self.cloud.size(), "adaptive": adapted}

    def _step_native(self, view: int, sub_origin: Optional[tuple]) -> dict:
        """The iteration of step() as one sct_train_step call (same random draws, same order)."""
        cfg, eng, t = self.cfg, self.eng, self.t
        tv_grid = None
        if cfg.lambda_tv > 0.0:
            if sub_origin is None:
                sub_origin = self.rng.subvolume_origin(self.scanner.extent_min_mm, self.scanner.extent_max_mm,
                                                       self.output_spacing, cfg.tv_grid_dim)
            d = cfg.tv_grid_dim
            tv_grid = GridSpec((d, d, d), sub_origin, self.output_spacing)
        cl = self.cloud
        key = (cl.size(), cl.rho_raw.data_ptr(), cl.pos.data_ptr(), cl.scale_raw.data_ptr(), cl.rot.data_ptr(),
               cl.grad2d_norm_accum.data_ptr(), cl.adam["m_rho"].data_ptr(), self.grads.buffer.data_ptr())
        if getattr(self, "_structs_key", None) != key:  # rebuilt after adaptive control / resize
            self._structs = ((self.scanner._c(), self.opts._c()) +
                             (self.cloud._c(), self.cloud._adam_c(), self.cloud._stats_c(), self.grads._c()))
            self._structs_key = key
        vals = torch.empty(4, dtype=torch.float64, device=eng.device)
        lrs = [lr_at(cfg.lr_position, cfg.lr_final_ratio, t, cfg.iters),
               lr_at(cfg.lr_density, cfg.lr_final_ratio, t, cfg.iters),
               lr_at(cfg.lr_scale, cfg.lr_final_ratio, t, cfg.iters),
               lr_at(cfg.lr_rotation, cfg.lr_final_ratio, t, cfg.iters)]
        eng.train_step(self.cloud, self.grads, self.scanner, self.angles[view], self.measured_norm[view], t, lrs,
                       vals, render_scale=self.inv_norm, grad_scale=self.inv_norm, lambda_ssim=cfg.lambda_ssim,
                       lambda_tv=cfg.lambda_tv, tv_grid=tv_grid, _structs=self._structs)
        total = vals[3]
        if cfg.check_every and t % cfg.check_every == 0:
            if not math.isfinite(float(total.item())):
                raise DivergenceDetected(f"non-finite loss at iteration {t}")
            if cfg.sync_free and eng.take_overflow():
                raise DataError(f"sync-free binning exceeded its pair capacity by iteration {t}; "
                                "raise TrainConfig.capacity_margin")
        adapted = None
        if (cfg.adaptive_start <= t <= cfg.adaptive_end and t > cfg.adaptive_start
                and (t - cfg.adaptive_start) % cfg.densify_interval == 0):  # trainer.cpp:321-323
            adapted = self.adaptive_control()
        return {"iter": t, "view": view, "l1": vals[0], "dssim": vals[1], "tv": vals[2], "total": total,
                "kernels": self.cloud.size(), "adaptive": adapted}

    def adaptive_control(self, gauss: Optional[torch.Tensor] = None):
        """trainer.cpp:167-230 on the device; replaces self.cloud (new size, carried Adam state,
        reset statistics) and resizes the gradient buffer. Returns (pruned, cloned, split)."""
        cfg = self.cfg
        ext = [self.scanner.extent_max_mm[k] - self.scanner.extent_min_mm[k] for k in range(3)]
        self.cloud, counts = self.eng.adaptive_control(
            self.cloud, ext, prune_density_threshold=cfg.prune_density_threshold,
            densify_grad_threshold=cfg.densify_grad_threshold,
            split_scale_threshold_frac=cfg.split_scale_threshold_frac, split_factor=cfg.split_factor, gauss=gauss,
            rng=self.rng if gauss is None else None)
        self.grads.resize(self.cloud.size(), device=self.eng.device)
        self._calibrate = cfg.sync_free  # new kernel count: re-measure the pair counts
        return counts


class NativeTrainer:
    """The reference's train() loop (trainer.cpp:232-345) run entirely in the engine
    library (csrc/trainer.cu, sct_trainer_*): views, TV sub-grid origins and split draws
    from the same std::mt19937_64(cfg.seed) stream as Trainer, adaptive control at the
    same iterations, losses read back only by record(). Equal to Trainer bitwise."""

    def __init__(self, engine: Engine, cloud, scanner: ScannerConfig, angles: Sequence[float],
                 projections, cfg: TrainConfig):
        import ctypes as C
        from . import _capi
        self.eng, self.cfg, self.lib = engine, cfg, _capi.load()
        host = cloud.host_arrays() if isinstance(cloud, GaussianCloud) else cloud
        self._host = {k: np.ascontiguousarray(host[k], dtype=np.float32) for k in ("rho_raw", "pos", "scale_raw",
                                                                                    "rot")}
        s_min = cloud.s_min if isinstance(cloud, GaussianCloud) else float(host["s_min"])
        self.s_min = s_min
        cl = _capi.sct_cloud()
        cl.m, cl.s_min_mm = int(self._host["rho_raw"].size), s_min
        for k, a in self._host.items():
            setattr(cl, k, a.ctypes.data)
        proj = projections.detach().cpu().numpy() if isinstance(projections, torch.Tensor) else projections
        self._proj = np.ascontiguousarray(proj, dtype=np.float32)
        self._angles = (C.c_double * len(angles))(*[float(a) for a in angles])
        c = _capi.sct_train_cfg()
        for k in ("iters", "tv_grid_dim", "adaptive_start", "adaptive_end", "densify_interval", "mode",
                  "check_every"):
            setattr(c, k, int(getattr(cfg, k)))
        for k in ("lr_position", "lr_density", "lr_scale", "lr_rotation", "lr_final_ratio", "lambda_ssim",
                  "lambda_tv", "densify_grad_threshold", "prune_density_threshold", "split_scale_threshold_frac",
                  "split_factor", "capacity_margin"):
            setattr(c, k, float(getattr(cfg, k)))
        c.seed = int(cfg.seed) & ((1 << 64) - 1)
        c.output_dims[:] = [int(x) for x in cfg.output_dims]
        c.sync_free = int(bool(cfg.sync_free))
        h = C.c_void_p()
        sc = scanner._c()
        rc = self.lib.sct_trainer_create(engine._h, C.byref(cl), self._proj.ctypes.data, self._angles, len(angles),
                                         C.byref(sc), C.byref(c), C.byref(h))
        from .engine import _check
        _check(rc)
        self._h = h

    def step(self) -> bool:
        """One iteration; True when adaptive control ran after it."""
        import ctypes as C
        from .engine import _check
        ad = C.c_int32(0)
        _check(self.lib.sct_trainer_step(self._h, C.byref(ad)))
        return bool(ad.value)

    def record(self) -> dict:
        """The last iteration's losses (synchronises), as the reference's HistoryRecord."""
        from . import _capi
        from .engine import _check
        import ctypes as C
        r = _capi.sct_train_record()
        _check(self.lib.sct_trainer_record(self._h, C.byref(r)))
        return {"iter": r.iter, "view": r.view, "l1": r.l1, "dssim": r.dssim, "tv": r.tv, "total": r.total,
                "kernels": int(r.kernels), "adaptive": tuple(r.counts)}

    def state(self) -> dict:
        """Host copies of the cloud, Adam moments and adaptive statistics."""
        import ctypes as C
        from . import _capi
        from .engine import _check
        m = self.record()["kernels"]
        out = {k: np.zeros(n * m, dtype=np.float32) for k, n in (("rho_raw", 1), ("pos", 3), ("scale_raw", 3),
                                                                  ("rot", 4))}
        cl = _capi.sct_cloud()
        cl.m = m
        for k, a in out.items():
            setattr(cl, k, a.ctypes.data)
        adam = {f"{a}_{k}": np.zeros(n * m, dtype=np.float32) for a in ("m", "v")
                for k, n in (("rho", 1), ("pos", 3), ("scale", 3), ("rot", 4))}
        ad = _capi.sct_adam_state()
        for k, a in adam.items():
            setattr(ad, k, a.ctypes.data)
        stats = {"grad2d_norm_accum": np.zeros(m, dtype=np.float32), "grad_count": np.zeros(m, dtype=np.int32),
                 "grad3d_accum": np.zeros(3 * m, dtype=np.float32)}
        st = _capi.sct_stats()
        for k, a in stats.items():
            setattr(st, k, a.ctypes.data)
        _check(self.lib.sct_trainer_download(self._h, C.byref(cl), C.byref(ad), C.byref(st)))
        return {**out, "adam": adam, **stats}

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                self.lib.sct_trainer_destroy(h)
            except Exception:  # noqa: BLE001 (interpreter shutdown)
                pass
            self._h = None
