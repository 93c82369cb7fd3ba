"""Metrics (proj/include/tessera/metrics.hpp, proj/src/metrics.cpp) plus the
max-abs and L2-relative errors the north star asks for."""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .grid import BasicGrid


@dataclass
class RateReport:
    points_per_step: int
    steps: int
    elapsed_seconds: float
    stencils_per_second: float


def stencils_per_second(extent, steps: int, elapsed_seconds: float) -> RateReport:
    """Eq. 6: prod(extent) * T / time (metrics.cpp:8-20)."""
    if not (elapsed_seconds > 0.0):
        raise ValueError("elapsed time must be positive")
    pts = 1
    for e in extent:
        pts *= int(e)
    return RateReport(pts, int(steps), float(elapsed_seconds),
                      float(pts) * float(steps) / elapsed_seconds)


def _check(a: BasicGrid, ref: BasicGrid) -> None:
    if a.dims != ref.dims:
        raise ValueError("grid dimensionality mismatch")
    if a.extent != ref.extent:
        raise ValueError("grid extent mismatch")


def max_abs(g: BasicGrid) -> float:
    return float(np.max(np.abs(g.interior_view(g.parity).astype(np.float64)), initial=0.0))


def max_rel_deviation(a: BasicGrid, reference: BasicGrid) -> float:
    """max|a-ref| / max(1, max|ref|) over the interior (metrics.cpp:28-39).
    NaN anywhere counts as an infinite deviation."""
    _check(a, reference)
    x = a.interior_view(a.parity).astype(np.float64)
    r = reference.interior_view(reference.parity).astype(np.float64)
    d = np.abs(x - r)
    dev = float(np.inf) if np.isnan(d).any() else float(np.max(d, initial=0.0))
    return dev / max(1.0, float(np.max(np.abs(r), initial=0.0)))


def deviation(a: BasicGrid, reference: BasicGrid) -> dict:
    """max_rel_deviation, max_abs_err and l2_rel_err in one pass."""
    _check(a, reference)
    x = a.interior_view(a.parity).astype(np.float64)
    r = reference.interior_view(reference.parity).astype(np.float64)
    diff = x - r
    d = np.abs(diff)
    maxabs = float(np.inf) if np.isnan(d).any() else float(np.max(d, initial=0.0))
    nr = float(np.sqrt(np.sum(r * r)))
    ne = float(np.sqrt(np.sum(diff * diff)))
    return {
        "max_rel_deviation": maxabs / max(1.0, float(np.max(np.abs(r), initial=0.0))),
        "max_abs_err": maxabs,
        "l2_rel_err": ne / nr if nr > 0 else ne,
        "bitwise_equal": bool(np.array_equal(x.view(np.uint64) if x.dtype == np.float64 else x,
                                             r.view(np.uint64) if r.dtype == np.float64 else r)),
    }
