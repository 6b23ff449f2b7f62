"""The reference's kernel plugin seam, served by CUDA.

``permatrace/backend.py:30-33`` re-exports four batch kernels from either its Cython or its numpy
module; this module is the third sibling a maintainer selects with ``PERMATRACE_BACKEND=cuda``
(see INTEGRATION.md).  Same signatures, argument meaning, return dtypes and error behaviour as
``permatrace/_kernels.pyx``; the arithmetic runs in ``csrc/pt_field.cu`` / ``csrc/pt_collision.cu``.
There is deliberately no fallback: if the shared library or the GPU is missing these raise.
"""

from __future__ import annotations

import numpy as np

from . import _cabi

BACKEND = "cuda-sm100a"

__all__ = ["BACKEND", "rbf_values", "sphere_box_hits", "sphere_cylinder_hits", "sphere_sphere_hits"]


def _f64(a, ndim):
    a = np.ascontiguousarray(a, dtype=np.float64)
    if a.ndim != ndim:
        raise ValueError(f"expected a {ndim}-d float64 array")
    return a


def rbf_values(points, support, weights, gamma, bias):
    """sum_j w_j exp(-gamma ||p_i - s_j||^2) + bias for every row p_i (``_kernels.pyx:18-40``)."""
    points, support, weights = _f64(points, 2), _f64(support, 2), _f64(weights, 1)
    if support.shape[1] != points.shape[1] or weights.shape[0] != support.shape[0]:
        raise ValueError("support/weights shape mismatch")
    out = np.empty(points.shape[0], dtype=np.float64)
    if points.shape[0] == 0:
        return out
    ctx = _cabi.context()
    _cabi.check(_cabi.lib.pt_rbf_values(ctx.handle, points.ctypes.data, points.shape[0], points.shape[1],
                                        support.ctypes.data, support.shape[0], weights.ctypes.data,
                                        float(gamma), float(bias), out.ctypes.data))
    return out


def _hits(fn, centers, radii, *params):
    centers, radii = _f64(centers, 2), _f64(radii, 1)
    if centers.shape[1] != 3 or radii.shape[0] != centers.shape[0]:
        raise ValueError("centers must be (m, 3) with one radius per row")
    out = np.zeros(centers.shape[0], dtype=np.uint8)
    if centers.shape[0]:
        ctx = _cabi.context()
        _cabi.check(fn(ctx.handle, centers.ctypes.data, radii.ctypes.data, centers.shape[0],
                       *[float(p) for p in params], out.ctypes.data))
    return out


def sphere_box_hits(centers, radii, lx, ly, lz):
    """1 where a sphere touches an origin-centred axis-aligned box (``_kernels.pyx:43-76``)."""
    return _hits(_cabi.lib.pt_sphere_box_hits, centers, radii, lx, ly, lz)


def sphere_cylinder_hits(centers, radii, height, radius):
    """1 where a sphere touches an origin-centred z-aligned cylinder (``_kernels.pyx:79-104``)."""
    return _hits(_cabi.lib.pt_sphere_cylinder_hits, centers, radii, height, radius)


def sphere_sphere_hits(centers, radii, radius):
    """1 where a sphere touches an origin-centred sphere (``_kernels.pyx:107-122``)."""
    return _hits(_cabi.lib.pt_sphere_sphere_hits, centers, radii, radius)
