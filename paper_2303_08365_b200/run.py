"""Time-step run API: the reference's sweep drivers, executed on the B200.

* ``naive_step`` / ``naive_run``  <- proj/include/tessera/naive.hpp:89-100
* ``run_tessellated``             <- proj/src/tiling.cpp:137-184 (the plan's
  tb becomes the number of time steps fused per HBM pass on the GPU)
* ``plan_tiles`` / ``TilePlan``   <- proj/src/tiling.cpp:48-102 (validation and
  plan bookkeeping; the GPU engine chooses its own spatial tiles)
* ``run_gpu``                      the same call with explicit GPU options and
  the device statistics returned.

All of them go through ``tsr_run`` (include/tessera_b200.h): host buffers in,
host buffers out, grid left exactly as the reference leaves it.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

from . import _abi
from .grid import BasicGrid
from .kernel import StencilKernel


@dataclass
class GpuStats:
    device_ms: float
    point_updates: int
    rounds: int
    trailing_steps: int
    kernel_launches: int
    h2d_bytes: int
    d2h_bytes: int
    fused_steps: int
    engine: str
    bytes_exchanged: int = 0
    messages: int = 0
    ghost_recompute_points: int = 0
    ngpus: int = 1
    transport: int = 0


def run_gpu(grid: BasicGrid, kernel: StencilKernel, steps: int, *, fused_steps: int = 0,
            mode: str = "exact", engine: str = "auto", device: int = -1,
            ngpus: int = 1) -> GpuStats:
    """Advances `grid` by `steps` time steps on the GPU (in place, parity
    flipped `steps` times, both buffers as naive_run leaves them).  ngpus > 1
    splits axis 0 into that many slabs on devices 0..ngpus-1 (modulo the
    device count), one host thread driving them (tsr_run with opts.ngpus)."""
    steps = int(steps)
    if steps < 0:
        raise ValueError("negative step count")
    L = _abi.lib()
    st = _abi.TsrStats()
    opts = _abi.make_opts(fused_steps, mode, engine, device, ngpus)
    b0, b1 = grid.c_buffers()
    _abi.check(L.tsr_run(ctypes.byref(kernel.c_struct()), ctypes.byref(grid.c_struct()), b0, b1,
                         grid.parity, steps, ctypes.byref(opts), ctypes.byref(st)))
    if steps & 1:
        grid.flip_parity()
    d = st.as_dict()
    d["engine"] = {0: "none", 1: "generic", 2: "tuned"}.get(d["engine"], "?")
    return GpuStats(**d)


def release_cache() -> None:
    """Frees the device buffers and staging memory tsr_run / tsr_run_multi
    keep between calls (tsr_release_cache)."""
    _abi.check(_abi.lib().tsr_release_cache())


def naive_step(grid: BasicGrid, kernel: StencilKernel) -> None:
    """naive.hpp:89-94 on the GPU."""
    run_gpu(grid, kernel, 1)


def naive_run(grid: BasicGrid, kernel: StencilKernel, steps: int) -> None:
    """naive.hpp:96-100 on the GPU (bitwise equal: exact mode)."""
    run_gpu(grid, kernel, steps)


class TilePlan:
    """Two-phase tessellation plan (tiling.hpp:30-41).  On the GPU only `tb`
    matters (the fused step count); extents and radius are validated like the
    reference so a plan/grid mismatch raises the same errors."""

    def __init__(self, extent, tile, tb, radius, segments):
        self.dims = len(extent)
        self.extent = list(extent)
        self.tile = list(tile)
        self.tb = int(tb)
        self.radius = int(radius)
        self.segments = list(segments)

    @property
    def upright_tiles(self) -> int:
        n = 1
        for s in self.segments:
            n *= s
        return n

    @property
    def inverted_tiles(self) -> int:
        n = 1
        for s in self.segments:
            n *= 2 * s
        return n - self.upright_tiles


def plan_tiles(extent, spatial_tile, tb: int, radius: int) -> TilePlan:
    """tiling.cpp:48-72 validation + segment counts."""
    extent = [int(e) for e in extent]
    spatial_tile = [int(t) for t in spatial_tile]
    if not extent or len(extent) > 3:
        raise ValueError("extent must cover 1 to 3 axes")
    if len(spatial_tile) != len(extent):
        raise ValueError("tile widths must match extent dimensionality")
    if tb < 1:
        raise ValueError("temporal tile height must be >= 1")
    if radius < 1:
        raise ValueError("radius must be >= 1")
    segments = []
    for a, (e, t) in enumerate(zip(extent, spatial_tile)):
        if e < 1:
            raise ValueError("extent must be positive")
        if t < 2 * radius * tb:
            raise ValueError(f"tile width {t} on axis {a} shrinks to empty before {tb} steps: "
                             f"need >= {2 * radius * tb}")
        segments.append(max(1, e // t))
    return TilePlan(extent, spatial_tile, tb, radius, segments)


def run_tessellated(grid: BasicGrid, kernel: StencilKernel, steps: int, plan: TilePlan,
                    threads: int = 1):
    """tiling.cpp:137-184 on the GPU: `plan.tb` steps fused per HBM pass.
    Returns (point_updates, rounds, trailing) as the reference binding does
    (proj/bindings/module.cpp:194-202); `threads` is accepted and ignored
    (the CUDA grid replaces parallel_for)."""
    if grid.dims != kernel.dims:
        raise ValueError("kernel/grid dimensionality mismatch")
    if kernel.radius != plan.radius:
        raise ValueError("plan radius differs from kernel radius")
    if plan.dims != grid.dims:
        raise ValueError("plan dimensionality differs from grid")
    if any(p != e for p, e in zip(plan.extent, grid.extent)):
        raise ValueError("plan extent differs from grid extent")
    if steps < 0:
        raise ValueError("negative step count")
    run_gpu(grid, kernel, steps, fused_steps=plan.tb)
    return grid.interior_points() * steps, steps // plan.tb, steps % plan.tb
