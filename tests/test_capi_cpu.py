"""CPU-side checks of the drop-in boundary: the engine library loads without a
GPU and exports every entry point include/splatct_gpu.h declares."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "splatct_gpu.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sct_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_entry_points():
    fns = declared_functions()
    for f in ("sct_render_fwd", "sct_render_bwd", "sct_voxelize_fwd", "sct_voxelize_bwd", "sct_tv3d",
              "sct_adam_step", "sct_ctx_create"):
        assert f in fns


def test_library_exports_every_declared_symbol():
    from paper_2405_20693_b200 import _capi
    lib = ctypes.CDLL(_capi.LIB_PATH)
    missing = [f for f in declared_functions() if not hasattr(lib, f)]
    assert not missing, missing
    # and the Python binding covers all of them
    assert set(declared_functions()) <= set(_capi.exported_symbols())


def test_library_is_sm100a_only():
    import subprocess
    from paper_2405_20693_b200 import _capi
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _capi.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    for bad in ("sm_80", "sm_90"):
        assert bad not in out


def test_pure_functions_without_gpu():
    from paper_2405_20693_b200 import _capi
    L = _capi.load()
    assert abs(L.sct_lr_at(0.01, 0.1, 15000, 30000) - 0.01 * 0.1 ** 0.5) < 1e-15
    assert L.sct_version().startswith(b"splatct-b200")


def test_host_rng_is_the_reference_stream():
    """engine.HostRng (product host code, csrc/rng.cu) draws the reference trainer's
    std::mt19937_64 stream: epoch shuffles (trainer.cpp:269-273), sub-volume origins
    (voxelizer.cpp:226-239) and one normal_distribution per adaptive-control call
    (trainer.cpp:184) — bit-identical to the reference's own calls (oracle/_ref)."""
    from oracle import oracle as O
    if not O.ref_available():
        pytest.skip("oracle/_ref (the compiled reference) not built")
    from paper_2405_20693_b200.engine import HostRng
    h, r = HostRng(1234), O.Rng(1234)
    order_h = np.arange(75, dtype=np.int32)
    order_r = np.arange(75, dtype=np.int32)
    sp = (2.0 / 64,) * 3
    with O.using("reference"):
        for epoch in range(3):
            h.shuffle(order_h)
            order_r = O.shuffle(r, order_r)
            np.testing.assert_array_equal(order_h, order_r)
            for _ in range(4):
                a = h.subvolume_origin((-1, -1, -1), (1, 1, 1), sp, 32)
                b = O.random_subvolume_spec((-1, -1, -1), (1, 1, 1), sp, 32, r).origin_mm
                assert tuple(a) == tuple(b)
            np.testing.assert_array_equal(h.normal(13), O.normal_draws(r, 13))
