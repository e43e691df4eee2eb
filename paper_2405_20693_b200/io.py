"""Single-file containers of the reference (io.cpp:20-62, 72-213): one JSON
header line, then little-endian float32 payload arrays. Clouds (.ckpt),
volumes (.vol) and images (.img) written here are readable by the reference
and vice versa; the float32 payload is exactly the engine's device layout, so
the device fast path is one read of the whole payload into one pinned staging
buffer and ONE host-to-device copy (the arrays are views of that device
buffer); saving is one device-to-host copy of all arrays into one pinned
buffer and one write.

Extension (the reference does not save optimizer state, io.cpp:201-211): with
``include_adam=True`` the Adam moments are appended after the four parameter
arrays and listed under ``"fields_extra"``; the reference loader reads the
first four arrays and ignores the rest, so such files stay compatible.
"""
from __future__ import annotations

import json
from typing import Optional

import numpy as np
import torch

from .engine import DataError, GaussianCloud, GridSpec


class FileFormatError(DataError):  # common.hpp:37-39
    pass


def _dump_header(h: dict) -> bytes:
    # nlohmann::json::dump(): keys sorted, no whitespace
    return (json.dumps(h, sort_keys=True, separators=(",", ":")) + "\n").encode()


def _write(path: str, header: dict, arrays) -> None:
    try:
        with open(path, "wb") as f:
            f.write(_dump_header(header))
            for a in arrays:
                f.write(np.ascontiguousarray(a, dtype="<f4").tobytes())
    except OSError as e:
        raise DataError(f"cannot write {path}: {e}") from e


def _device_payload(path: str, payload: bytes, count: int, device) -> torch.Tensor:
    """The first `count` floats of the payload on `device`: one pinned staging
    buffer, one (non-blocking) H2D copy."""
    if 4 * count > len(payload):
        raise FileFormatError(f"{path}: truncated payload")
    host = torch.frombuffer(bytearray(payload[:4 * count]), dtype=torch.float32) if count else \
        torch.empty(0, dtype=torch.float32)
    if str(device) == "cpu" or not torch.cuda.is_available():
        return host.clone()
    pinned = torch.empty(count, dtype=torch.float32, pin_memory=True)
    pinned.copy_(host)
    out = torch.empty(count, dtype=torch.float32, device=device)
    out.copy_(pinned, non_blocking=True)
    torch.cuda.current_stream(out.device).synchronize()  # the pinned buffer is released on return
    return out


def _host_arrays(tensors) -> list:
    """Device tensors -> host numpy arrays through ONE device-to-host copy into
    one pinned buffer (one pass over PCIe instead of one per array)."""
    ts = [t.detach().reshape(-1) for t in tensors]
    if not ts or not all(t.is_cuda for t in ts):
        return [t.cpu().numpy() for t in ts]
    flat = torch.cat([t.to(torch.float32) for t in ts])
    pinned = torch.empty(flat.numel(), dtype=torch.float32, pin_memory=True)
    pinned.copy_(flat, non_blocking=True)
    torch.cuda.current_stream(flat.device).synchronize()
    out, off = [], 0
    host = pinned.numpy()
    for t in ts:
        out.append(host[off:off + t.numel()])
        off += t.numel()
    return out


def _read(path: str):
    try:
        f = open(path, "rb")
    except OSError as e:
        raise DataError(f"cannot open {path}") from e
    with f:
        line = f.readline()
        if not line:
            raise FileFormatError(f"{path}: missing header line")
        try:
            h = json.loads(line.decode())
        except (ValueError, UnicodeDecodeError) as e:
            raise FileFormatError(f"{path}: bad header: {e}") from e
        if not isinstance(h, dict):
            raise FileFormatError(f"{path}: bad header")
        if h.get("endianness", "little") != "little":
            raise FileFormatError(f"{path}: only little-endian payloads are supported")
        if h.get("dtype", "float32") != "float32":
            raise FileFormatError(f"{path}: only float32 payloads are supported")
        payload = f.read()
    return h, payload


def _take(path, payload, off, count):
    nbytes = 4 * count
    if off + nbytes > len(payload):
        raise FileFormatError(f"{path}: truncated payload")
    return np.frombuffer(payload, dtype="<f4", count=count, offset=off).astype(np.float32), off + nbytes


# ------------------------------------------------------------------ clouds (io.cpp:171-213)
def save_cloud(cloud: GaussianCloud, path: str, include_adam: bool = False) -> None:
    h = {"kind": "gaussian_cloud", "count": cloud.size(),
         "activations": {"density": "softplus", "scale": "exp_floor"}, "s_min_mm": cloud.s_min,
         "fields": ["rho_raw", "positions_mm", "scales_raw", "rotations_wxyz"], "dtype": "float32",
         "endianness": "little", "version": 1}
    tensors = [cloud.rho_raw, cloud.pos, cloud.scale_raw, cloud.rot]
    if include_adam:
        keys = ["m_rho", "v_rho", "m_pos", "v_pos", "m_scale", "v_scale", "m_rot", "v_rot"]
        h["fields_extra"] = ["adam_" + k for k in keys]
        tensors += [cloud.adam[k] for k in keys]
    _write(path, h, _host_arrays(tensors))


def load_cloud(path: str, device="cuda") -> GaussianCloud:
    h, payload = _read(path)
    if h.get("kind", "") != "gaussian_cloud":
        raise FileFormatError(f"{path}: not a gaussian cloud file")
    m = h.get("count", -1)
    if not isinstance(m, int) or m < 0:
        raise FileFormatError(f"{path}: missing kernel count")
    act = h.get("activations")
    if act is not None and (act.get("density") != "softplus" or act.get("scale") != "exp_floor"):
        raise FileFormatError(f"{path}: unsupported activation names")
    extra = [n for n in (h.get("fields_extra") or []) if n.startswith("adam_")]
    sizes = {"rho": m, "pos": 3 * m, "scale": 3 * m, "rot": 4 * m}
    n_extra = sum(sizes[n[len("adam_"):].split("_", 1)[1]] for n in extra)
    # the parameters (and the optional moments) in one transfer
    dev = _device_payload(path, payload, 11 * m + n_extra, device)
    off = 0
    parts = []
    for n in (m, 3 * m, 3 * m, 4 * m):
        parts.append(dev[off:off + n])
        off += n
    cloud = GaussianCloud(float(h.get("s_min_mm", 1e-4)), *parts, device=device)
    for name in extra:
        k = name[len("adam_"):]
        n = sizes[k.split("_", 1)[1]]
        cloud.adam[k].copy_(dev[off:off + n])
        off += n
    return cloud


# ------------------------------------------------------------------ volumes (io.cpp:72-104)
def write_volume(vol, grid: GridSpec, path: str) -> None:
    v = vol.detach().cpu().numpy() if isinstance(vol, torch.Tensor) else np.asarray(vol)
    h = {"kind": "volume", "dims": [int(d) for d in grid.dims], "spacing_mm": [float(x) for x in grid.spacing_mm],
         "origin_mm": [float(x) for x in grid.origin_mm], "dtype": "float32", "endianness": "little",
         "order": "x-fastest", "version": 1}
    _write(path, h, [v.reshape(-1)])


def read_volume(path: str):
    """Returns (volume [Z][Y][X] float32 numpy, GridSpec)."""
    h, payload = _read(path)
    if h.get("kind", "") != "volume":
        raise FileFormatError(f"{path}: not a volume file")
    try:
        dims = tuple(int(d) for d in h["dims"])
        grid = GridSpec(dims, tuple(float(x) for x in h["origin_mm"]), tuple(float(x) for x in h["spacing_mm"]))
    except (KeyError, TypeError, ValueError) as e:
        raise FileFormatError(f"{path}: bad volume header: {e}") from e
    if len(dims) != 3 or min(dims) <= 0:
        raise FileFormatError(f"{path}: non-positive dims")
    data, _ = _take(path, payload, 0, dims[0] * dims[1] * dims[2])
    return data.reshape(dims[2], dims[1], dims[0]), grid


# ------------------------------------------------------------------ images (io.cpp:106-137)
def write_image(img, path: str, meta: Optional[dict] = None) -> None:
    a = img.detach().cpu().numpy() if isinstance(img, torch.Tensor) else np.asarray(img)
    h = {"kind": "image", "dims": [int(a.shape[1]), int(a.shape[0])], "dtype": "float32", "endianness": "little",
         "order": "row-major", "version": 1}
    if meta:
        h["meta"] = {k: float(v) for k, v in meta.items()}
    _write(path, h, [a.reshape(-1)])


def read_image(path: str):
    """Returns (image [H][W] float32 numpy, meta dict)."""
    h, payload = _read(path)
    if h.get("kind", "") != "image":
        raise FileFormatError(f"{path}: not an image file")
    try:
        w, hh = int(h["dims"][0]), int(h["dims"][1])
    except (KeyError, TypeError, ValueError, IndexError) as e:
        raise FileFormatError(f"{path}: bad image header: {e}") from e
    if w <= 0 or hh <= 0:
        raise FileFormatError(f"{path}: non-positive dims")
    data, _ = _take(path, payload, 0, w * hh)
    return data.reshape(hh, w), dict(h.get("meta", {}))
