"""splatct-b200: B200-native (sm_100a) engine for R²-Gaussian's differentiable
hot paths — the rectified X-ray Gaussian rasterizer and the 3D voxelizer,
forward and backward, plus voxel TV, photometric losses and Adam.

The compute lives in libsplatct_b200.so behind the C ABI declared in
include/splatct_gpu.h; this package is the host-side mirror of the reference
C++ API (see engine.py for the file:line map)."""
from .engine import (  # noqa: F401
    BIASED, RECTIFIED, Adam, CloudGrads, ConfigError, CudaError, DataError, DimMismatch, DivergenceDetected, Engine,
    GaussianCloud, GridSpec, RasterOptions, RenderedProjection, ScannerConfig, SplatctError, VoxelizeOptions,
    default_engine, full_circle_angles, grid_for_extent, lr_at, project_kernels, render, render_backward, tv3d_loss,
    voxelize, voxelize_backward)

__version__ = "0.1.0"
