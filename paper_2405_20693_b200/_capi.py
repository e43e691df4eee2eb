"""ctypes binding of include/splatct_gpu.h (libsplatct_b200.so).

This is the only way the Python layer reaches the engine: there is no
PyTorch/NumPy compute fallback. If the shared library is missing the import
fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# SCT_LIB_VARIANT selects an alternative in-tree build for A/B measurements
# (tools/variants.sh); SCT_CHECKED=1 the checked build (device invariant
# checks, `make checked`); the default is the product library.
LIB_PATH = os.path.join(_HERE, os.environ.get(
    "SCT_LIB_VARIANT", "libsplatct_b200_checked.so" if os.environ.get("SCT_CHECKED") == "1" else "libsplatct_b200.so"))

F = C.POINTER(C.c_float)
D = C.POINTER(C.c_double)
I32 = C.POINTER(C.c_int32)
I64 = C.POINTER(C.c_int64)
VP = C.c_void_p


class sct_scanner(C.Structure):
    _fields_ = [("l_so_mm", C.c_double), ("l_sd_mm", C.c_double), ("det_size_mm", C.c_double * 2),
                ("det_res_px", C.c_int32 * 2), ("extent_min_mm", C.c_double * 3),
                ("extent_max_mm", C.c_double * 3), ("near_clip_mm", C.c_double), ("parallel_beam", C.c_int32)]


class sct_raster_opts(C.Structure):
    _fields_ = [("mode", C.c_int32), ("lowpass_eps_px", C.c_double), ("dilation_compensation", C.c_int32),
                ("freeze_jacobian", C.c_int32), ("cull_mahalanobis", C.c_double)]


class sct_grid(C.Structure):
    _fields_ = [("dims", C.c_int32 * 3), ("origin_mm", C.c_double * 3), ("spacing_mm", C.c_double * 3)]


class sct_cloud(C.Structure):
    _fields_ = [("m", C.c_int64), ("s_min_mm", C.c_double), ("rho_raw", VP), ("pos", VP), ("scale_raw", VP),
                ("rot", VP)]


class sct_grads(C.Structure):
    _fields_ = [("rho_raw", VP), ("pos", VP), ("scale_raw", VP), ("rot", VP)]


class sct_stats(C.Structure):
    _fields_ = [("grad2d_norm_accum", VP), ("grad_count", VP), ("grad3d_accum", VP)]


class sct_adam_state(C.Structure):
    _fields_ = [("m_rho", VP), ("v_rho", VP), ("m_pos", VP), ("v_pos", VP), ("m_scale", VP), ("v_scale", VP),
                ("m_rot", VP), ("v_rot", VP)]


class sct_train_args(C.Structure):
    _fields_ = [("theta_rad", C.c_double), ("measured", VP), ("render_scale", C.c_float), ("grad_scale", C.c_float),
                ("lambda_ssim", C.c_double), ("lambda_tv", C.c_double), ("tv_grid", sct_grid),
                ("cull_mahalanobis", C.c_double), ("t", C.c_int32), ("lr", C.c_double * 4), ("beta1", C.c_double),
                ("beta2", C.c_double), ("eps", C.c_double), ("values_dev", VP)]


class sct_train_cfg(C.Structure):
    _fields_ = [("iters", C.c_int32), ("lr_position", C.c_double), ("lr_density", C.c_double),
                ("lr_scale", C.c_double), ("lr_rotation", C.c_double), ("lr_final_ratio", C.c_double),
                ("lambda_ssim", C.c_double), ("lambda_tv", C.c_double), ("tv_grid_dim", C.c_int32),
                ("adaptive_start", C.c_int32), ("adaptive_end", C.c_int32), ("densify_interval", C.c_int32),
                ("densify_grad_threshold", C.c_double), ("prune_density_threshold", C.c_double),
                ("split_scale_threshold_frac", C.c_double), ("split_factor", C.c_double), ("seed", C.c_uint64),
                ("mode", C.c_int32), ("output_dims", C.c_int32 * 3), ("check_every", C.c_int32),
                ("sync_free", C.c_int32), ("capacity_margin", C.c_double)]


class sct_train_record(C.Structure):
    _fields_ = [("iter", C.c_int32), ("view", C.c_int32), ("l1", C.c_double), ("dssim", C.c_double),
                ("tv", C.c_double), ("total", C.c_double), ("kernels", C.c_int64), ("counts", C.c_int32 * 3)]


P = C.POINTER

SIGNATURES = {
    "sct_ctx_create": (C.c_int, [C.c_int, VP, P(VP)]),
    "sct_ctx_destroy": (C.c_int, [VP]),
    "sct_ctx_set_stream": (C.c_int, [VP, VP]),
    "sct_ctx_sync": (C.c_int, [VP]),
    "sct_ctx_set_deterministic": (C.c_int, [VP, C.c_int]),
    "sct_ctx_set_capacity": (C.c_int, [VP, C.c_int64, C.c_int64]),
    "sct_ctx_take_overflow": (C.c_int, [VP, I32]),
    "sct_last_error": (C.c_char_p, []),
    "sct_version": (C.c_char_p, []),
    "sct_ctx_kernel_launches": (C.c_int64, [VP]),
    "sct_ctx_set_timing": (C.c_int, [VP, C.c_int]),
    "sct_ctx_timing_report": (C.c_int, [VP, C.c_char_p, C.c_int32]),
    "sct_fwd_work": (C.c_int, [VP, I64, I64]),
    "sct_voxel_work": (C.c_int, [VP, P(sct_cloud), P(sct_grid), C.c_double, I64, I64]),
    "sct_render_fwd": (C.c_int, [VP, P(sct_cloud), P(sct_scanner), D, C.c_int32, P(sct_raster_opts), VP, P(VP)]),
    "sct_render_bwd": (C.c_int, [VP, VP, P(sct_cloud), VP, P(sct_grads), P(sct_stats)]),
    "sct_fwd_free": (C.c_int, [VP]),
    "sct_fwd_info": (C.c_int, [VP, I64, I32, I32, I64]),
    "sct_fwd_tile_lists": (C.c_int, [VP, C.c_int32, I64, I32]),
    "sct_project_kernels": (C.c_int, [VP, P(sct_cloud), P(sct_scanner), C.c_double, P(sct_raster_opts), I32, D]),
    "sct_project_kernels_host": (C.c_int, [VP, P(sct_cloud), P(sct_scanner), C.c_double, P(sct_raster_opts), I32,
                                           D]),
    "sct_render_fwd_host": (C.c_int, [VP, P(sct_cloud), P(sct_scanner), D, C.c_int32, P(sct_raster_opts), VP,
                                      P(VP)]),
    "sct_render_bwd_host": (C.c_int, [VP, VP, P(sct_cloud), VP, P(sct_grads), P(sct_stats)]),
    "sct_voxelize_fwd": (C.c_int, [VP, P(sct_cloud), P(sct_grid), C.c_double, C.c_int32, C.c_int32, VP]),
    "sct_voxelize_bwd": (C.c_int, [VP, P(sct_cloud), P(sct_grid), C.c_double, C.c_int32, C.c_int32, VP,
                                   P(sct_grads)]),
    "sct_voxel_bins": (C.c_int, [VP, P(sct_cloud), P(sct_grid), C.c_double, I64, I64, I32]),
    "sct_voxelize_fwd_host": (C.c_int, [VP, P(sct_cloud), P(sct_grid), C.c_double, VP]),
    "sct_voxelize_bwd_host": (C.c_int, [VP, P(sct_cloud), P(sct_grid), C.c_double, VP, P(sct_grads)]),
    "sct_voxelize_fwd_state": (C.c_int, [VP, P(sct_cloud), P(sct_grid), C.c_double, C.c_int32, C.c_int32, VP,
                                         P(VP)]),
    "sct_voxelize_bwd_state": (C.c_int, [VP, VP, P(sct_cloud), VP, P(sct_grads)]),
    "sct_vox_free": (C.c_int, [VP]),
    "sct_tv3d": (C.c_int, [VP, VP, I32, C.c_float, VP, VP]),
    "sct_photometric_loss": (C.c_int, [VP, VP, VP, C.c_int32, C.c_int32, C.c_int32, C.c_float, C.c_float,
                                       C.c_float, VP, VP]),
    "sct_adam_step": (C.c_int, [VP, P(sct_cloud), P(sct_adam_state), P(sct_grads), C.c_int32, D, C.c_double,
                                C.c_double, C.c_double]),
    "sct_lr_at": (C.c_double, [C.c_double, C.c_double, C.c_int32, C.c_int32]),
    "sct_trainer_create": (C.c_int, [VP, P(sct_cloud), VP, D, C.c_int32, P(sct_scanner), P(sct_train_cfg), P(VP)]),
    "sct_trainer_step": (C.c_int, [VP, I32]),
    "sct_trainer_record": (C.c_int, [VP, P(sct_train_record)]),
    "sct_trainer_download": (C.c_int, [VP, P(sct_cloud), P(sct_adam_state), P(sct_stats)]),
    "sct_trainer_destroy": (C.c_int, [VP]),
    "sct_train_step": (C.c_int, [VP, P(sct_cloud), P(sct_adam_state), P(sct_stats), P(sct_grads), P(sct_scanner),
                                 P(sct_raster_opts), P(sct_train_args)]),
    "sct_adaptive_plan": (C.c_int, [VP, P(sct_cloud), P(sct_stats), C.c_double, C.c_double, C.c_double, C.c_double,
                                    D, P(VP), I64, I64, I32]),
    "sct_adaptive_apply": (C.c_int, [VP, VP, P(sct_cloud), P(sct_adam_state), VP, VP, P(sct_cloud),
                                     P(sct_adam_state)]),
    "sct_adaptive_free": (C.c_int, [VP]),
    "sct_phantom": (C.c_int, [VP, C.c_int32, D, D, D, I32, VP]),
    "sct_project_volume": (C.c_int, [VP, VP, P(sct_grid), P(sct_scanner), D, C.c_int32, C.c_double, VP]),
    "sct_add_noise_host": (C.c_int, [VP, C.c_int32, C.c_int32, C.c_int32, C.c_double, C.c_double, C.c_uint64,
                                     C.c_int32]),
    "sct_fdk": (C.c_int, [VP, VP, C.c_int32, P(sct_scanner), D, P(sct_grid), C.c_int32, VP]),
    "sct_nn_distances": (C.c_int, [VP, C.c_int64, VP, VP]),
    "sct_sample_init_cloud": (C.c_int, [VP, VP, P(sct_grid), C.c_int32, C.c_double, C.c_double, C.c_double,
                                        C.c_uint64, P(sct_cloud)]),
    "sct_nccl_unique_id": (C.c_int, [C.POINTER(C.c_uint8)]),
    "sct_ctx_comm_init": (C.c_int, [VP, C.c_int32, C.c_int32, C.POINTER(C.c_uint8)]),
    "sct_ctx_set_comm": (C.c_int, [VP, VP]),
    "sct_ctx_comm_info": (C.c_int, [VP, I32, I32]),
    "sct_allreduce_grads": (C.c_int, [VP, C.c_int64, P(sct_grads), P(sct_stats)]),
    "sct_render_bwd_allreduce": (C.c_int, [VP, VP, P(sct_cloud), VP, P(sct_grads), P(sct_stats)]),
    "sct_voxelize_bwd_allreduce": (C.c_int, [VP, P(sct_cloud), P(sct_grid), C.c_double, C.c_int32, C.c_int32, VP,
                                             P(sct_grads)]),
    "sct_rng_create": (C.c_int, [C.c_uint64, P(VP)]),
    "sct_rng_destroy": (C.c_int, [VP]),
    "sct_rng_shuffle": (C.c_int, [VP, I32, C.c_int32]),
    "sct_rng_subvolume_origin": (C.c_int, [VP, D, D, D, C.c_int32, D]),
    "sct_rng_normal": (C.c_int, [VP, C.c_int64, D]),
    "sct_rng_uniform": (C.c_int, [VP, C.c_int64, C.c_double, C.c_double, D]),
    "sct_host_alloc": (C.c_int, [P(VP), C.c_size_t]),
    "sct_host_free": (C.c_int, [VP]),
    "sct_debug_pointer_type": (C.c_int, [VP]),
}

_lib = None


def load():
    """Load the engine library (raises ImportError if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} not found: the CUDA engine is not built. Run "
                "`python -c 'import __graft_entry__ as g; g.build()'` (nvcc, sm_100a). "
                "There is no CPU fallback.")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def exported_symbols():
    return list(SIGNATURES.keys())
