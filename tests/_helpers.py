"""Shared test helpers: finite differences (tests/helpers.hpp:79-113) and
tolerance metrics used by the parity tests."""
import numpy as np


def finite_difference_check(cloud, analytic, loss, step=1e-5):
    """Central differences over every raw parameter (helpers.hpp:79-113).

    ``cloud`` is an oracle.Cloud-like object with float64 arrays rho_raw,
    pos, scale_raw, rot (mutated in place and restored); ``analytic`` has the
    same four arrays. Returns (max_err, checked).
    """
    grad_scale = 1e-12
    for g in (analytic.rho_raw, analytic.pos, analytic.scale_raw, analytic.rot):
        if g.size:
            grad_scale = max(grad_scale, float(np.max(np.abs(g))))
    max_err, checked = 0.0, 0
    for name in ("rho_raw", "pos", "scale_raw", "rot"):
        params = getattr(cloud, name)
        grads = getattr(analytic, name)
        for i in range(params.size):
            saved = params[i]
            h = step * max(1.0, abs(saved))
            params[i] = saved + h
            up = loss(cloud)
            params[i] = saved - h
            down = loss(cloud)
            params[i] = saved
            fd = (up - down) / (2.0 * h)
            a = grads[i]
            denom = max(abs(a), abs(fd), 1e-4 * grad_scale)
            max_err = max(max_err, abs(a - fd) / denom)
            checked += 1
    return max_err, checked


def rel_l2(a, b):
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    nb = np.linalg.norm(b)
    if nb == 0.0:
        return float(np.linalg.norm(a))
    return float(np.linalg.norm(a - b) / nb)
