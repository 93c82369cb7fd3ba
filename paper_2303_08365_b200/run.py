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


UPRIGHT, INVERTED = "upright", "inverted"  # PieceKind (tiling.hpp:16)


@dataclass
class Tile:
    """tiling.hpp:18-23: per-axis piece kind, segment / anchor index and
    anchor position; wave = number of inverted axes (0 = phase A)."""
    kind: tuple
    index: tuple
    anchor: tuple
    wave: int


class TilePlan:
    """Two-phase tessellation plan (tiling.hpp:30-41).  On the GPU only `tb`
    matters (the fused step count): the engine streams overlapped tiles
    instead.  The plan itself is built exactly as the reference builds it
    (validation, segment counts, phase A / phase B tile lists ordered by
    wave), so ``upright_tiles`` / ``inverted_tiles`` / ``count_coverage``
    answer as the reference's binding does (module.cpp:180-193)."""

    def __init__(self, extent, tile, tb, radius, segments):
        self.dims = len(extent)
        self.extent = list(extent)
        self.tile = list(tile)
        self.tb = int(tb)
        self.radius = int(radius)
        self.segments = list(segments)
        self.phase_a, self.phase_b = [], []
        # every (kind, index) product over the axes, kinds upright-first
        # (tiling.cpp:80-100); phase B stable-sorted by wave
        combos = [((), ())]
        for a in range(self.dims):
            combos = [(k + (kind,), i + (n,)) for k, i in combos
                      for kind in (UPRIGHT, INVERTED) for n in range(self.segments[a])]
        for kind, index in combos:
            wave = sum(1 for k in kind if k == INVERTED)
            t = Tile(kind, index, tuple(i * w for i, w in zip(index, self.tile)), wave)
            (self.phase_a if wave == 0 else self.phase_b).append(t)
        self.phase_b.sort(key=lambda t: t.wave)

    @property
    def upright_tiles(self) -> int:
        return len(self.phase_a)

    @property
    def inverted_tiles(self) -> int:
        return len(self.phase_b)


def axis_range(plan: TilePlan, axis: int, kind: str, index: int, step: int):
    """tiling.cpp:20-31: cells owned on `axis` by a piece at 0-based step
    `step` of a round, as (lo, hi)."""
    shift = step * plan.radius
    if kind == UPRIGHT:
        lo = index * plan.tile[axis] + shift
        last = index == plan.segments[axis] - 1
        hi = plan.extent[axis] if last else (index + 1) * plan.tile[axis]
        if not last:
            hi -= shift
        return lo, max(lo, hi)
    anchor = index * plan.tile[axis]
    return max(0, anchor - shift), min(plan.extent[axis], anchor + shift)


def tile_range(plan: TilePlan, t: Tile, step: int):
    """tiling.cpp:33-45: the owned box of a tile at a step, (lo, hi) lists."""
    r = [axis_range(plan, a, t.kind[a], t.index[a], step) for a in range(plan.dims)]
    return [x[0] for x in r], [x[1] for x in r]


def count_coverage(plan: TilePlan):
    """tiling.cpp:112-135 / module.cpp:190-193: ownership count of every
    (cell, step) over both phases -> (all_ones, min_count, max_count).  A
    correct plan owns every cell exactly once per step."""
    import numpy as np
    counts = np.zeros([plan.tb] + plan.extent, dtype=np.int32)
    for t in plan.phase_a + plan.phase_b:
        for s in range(plan.tb):
            lo, hi = tile_range(plan, t, s)
            counts[(s,) + tuple(slice(l, h) for l, h in zip(lo, hi))] += 1
    mn, mx = int(counts.min()), int(counts.max())
    return mn == 1 and mx == 1, mn, mx


def plan_tiles(extent, spatial_tile, tb: int, radius: int) -> TilePlan:
    """tiling.cpp:48-102: validation, segment counts and the tile lists."""
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
