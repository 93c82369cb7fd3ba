"""Stencil definition API, mirroring the reference's kernel.hpp / kernel.cpp.

``make_kernel`` validates the exact offset lattice for (dims, shape, radius)
and keeps taps in canonical lexicographic order
(proj/src/kernel.cpp:19-43, 78-116); ``heat_coefficients`` follows
kernel.cpp:118-128; the Table-1 benchmark kernels follow
proj/src/bench.cpp:25-85.  Errors raise ``ValueError`` exactly where the
reference throws ``std::invalid_argument`` (pybind11's mapping).
"""
from __future__ import annotations

import ctypes
import itertools
import math
from dataclasses import dataclass, field
from typing import Iterable, Sequence

from . import _abi

SHAPES = ("star", "box")


def _pad3(off: Sequence[int]) -> tuple[int, int, int]:
    off = tuple(int(v) for v in off)
    if not 1 <= len(off) <= 3:
        raise ValueError("offset needs 1 to 3 components")
    return off + (0,) * (3 - len(off))


def lattice_offsets(dims: int, shape: str, radius: int) -> list[tuple[int, int, int]]:
    """The exact offset lattice, lexicographic (kernel.cpp:19-43)."""
    out = []
    for cur in itertools.product(range(-radius, radius + 1), repeat=dims):
        nonzero = sum(1 for v in cur if v != 0)
        if shape == "box" or nonzero <= 1:
            out.append(_pad3(cur))
    out.sort()
    return out


class StencilKernel:
    """Fixed neighbour pattern with fp64 weights in canonical tap order
    (proj/include/tessera/kernel.hpp:26-51)."""

    def __init__(self, dims: int, shape: str, radius: int,
                 taps: Sequence[tuple[tuple[int, int, int], float]]):
        self._dims = int(dims)
        self._shape = shape
        self._radius = int(radius)
        self._taps = [(tuple(o), float(w)) for o, w in taps]
        s = 0.0
        for _, w in self._taps:
            s += w
        self._weight_sum = s
        self._c = None

    dims = property(lambda self: self._dims)
    shape = property(lambda self: self._shape)
    radius = property(lambda self: self._radius)
    weight_sum = property(lambda self: self._weight_sum)

    def taps(self) -> list[tuple[list[int], float]]:
        """[(offset[:dims], weight)], as the reference binding returns."""
        return [(list(o[: self._dims]), w) for o, w in self._taps]

    def tap_list(self) -> list[tuple[tuple[int, int, int], float]]:
        return list(self._taps)

    def weight_at(self, off: Sequence[int]) -> float:
        off = _pad3(off)
        for o, w in self._taps:
            if o == off:
                return w
        return 0.0

    def line_weights(self, axis: int, transverse: Sequence[int]) -> list[float]:
        """kernel.cpp:64-74."""
        tr = _pad3(transverse)
        w = [0.0] * (2 * self._radius + 1)
        for o, wt in self._taps:
            if all(o[a] == tr[a] for a in range(self._dims) if a != axis):
                w[o[axis] + self._radius] = wt
        return w

    def c_struct(self) -> _abi.TsrKernel:
        """tsr_kernel view of this kernel (arrays kept alive on self)."""
        if self._c is None:
            n = len(self._taps)
            offs = (ctypes.c_int32 * (3 * n))(*[v for o, _ in self._taps for v in o])
            ws = (ctypes.c_double * n)(*[w for _, w in self._taps])
            k = _abi.TsrKernel(self._dims, SHAPES.index(self._shape), self._radius, n,
                               ctypes.cast(offs, ctypes.POINTER(ctypes.c_int32)),
                               ctypes.cast(ws, ctypes.POINTER(ctypes.c_double)))
            self._c = (k, offs, ws)
        return self._c[0]

    def __repr__(self) -> str:
        return (f"<StencilKernel {self._shape} dims={self._dims} radius={self._radius} "
                f"taps={len(self._taps)}>")


def make_kernel(dims: int, shape: str, radius: int,
                weights: Iterable[tuple[Sequence[int], float]]) -> StencilKernel:
    """Builds a kernel after validating the (dims, shape, radius) lattice
    (kernel.cpp:78-116)."""
    if shape not in SHAPES:
        raise ValueError("kernel shape must be 'star' or 'box'")
    if dims < 1 or dims > 3:
        raise ValueError("kernel dims must be 1, 2 or 3")
    if radius < 1:
        raise ValueError("kernel radius must be positive")
    lat = lattice_offsets(dims, shape, radius)
    weights = [(_pad3(o), float(w)) for o, w in weights]
    if len(weights) != len(lat):
        raise ValueError(
            f"kernel offset count mismatch: expected {len(lat)} offsets for {shape} radius "
            f"{radius} in {dims}D, got {len(weights)}")
    for off, w in weights:
        if any(off[a] != 0 for a in range(dims, 3)):
            raise ValueError("offset uses components beyond kernel dims")
        if not math.isfinite(w):
            raise ValueError(f"non-finite kernel weight at offset {off[:dims]}")
    taps = sorted(weights, key=lambda t: t[0])
    for (off, _), want in zip(taps, lat):
        if off != want:
            raise ValueError(
                f"offset set does not match the {shape} lattice (unexpected {off[:dims]})")
    return StencilKernel(dims, shape, radius, taps)


def heat_coefficients(mu: float) -> StencilKernel:
    """2-D 5-point heat kernel: centre 1-4mu, neighbours mu (kernel.cpp:118-128)."""
    if not (mu > 0.0) or mu > 0.25:
        raise ValueError("heat CFL number outside stability range: need 0 < mu <= 0.25")
    return make_kernel(2, "star", 1, [((0, 0), 1.0 - 4.0 * mu), ((-1, 0), mu), ((1, 0), mu),
                                      ((0, -1), mu), ((0, 1), mu)])


def star_kernel(dims: int, radius: int, center: float, ring: Sequence[float]) -> StencilKernel:
    """bench.cpp:25-38."""
    w = [((0, 0, 0), center)]
    for a in range(dims):
        for d in range(1, radius + 1):
            plus = [0, 0, 0]
            minus = [0, 0, 0]
            plus[a], minus[a] = d, -d
            w.append((tuple(plus), ring[d - 1]))
            w.append((tuple(minus), ring[d - 1]))
    return make_kernel(dims, "star", radius, w)


def box_kernel(dims: int, radius: int) -> StencilKernel:
    """bench.cpp:40-58: every tap 1/(2r+1)^dims (computed as 1.0 / pts)."""
    n = 2 * radius + 1
    pts = 1.0
    for _ in range(dims):
        pts *= n
    w = [(off, 1.0 / pts) for off in itertools.product(range(-radius, radius + 1), repeat=dims)]
    return make_kernel(dims, "box", radius, w)


@dataclass
class BenchmarkSpec:
    """bench.hpp:16-25."""
    name: str
    kernel: StencilKernel
    full_extent: list = field(default_factory=list)
    full_steps: int = 0
    tile: list = field(default_factory=list)
    tb: int = 1


_TABLE = None


def benchmark_table() -> list[BenchmarkSpec]:
    """The eight stock benchmarks (bench.cpp:63-85)."""
    global _TABLE
    if _TABLE is None:
        _TABLE = [
            BenchmarkSpec("Heat-1D", star_kernel(1, 1, 0.5, [0.25]), [10_000_000], 100_000,
                          [2_000], 1_000),
            BenchmarkSpec("Star-1D5P", star_kernel(1, 2, 0.5, [0.15, 0.10]), [10_000_000],
                          100_000, [2_000], 500),
            BenchmarkSpec("Heat-2D", heat_coefficients(0.23), [10_000, 10_000], 10_000,
                          [200, 200], 50),
            BenchmarkSpec("Star-2D9P", star_kernel(2, 2, 0.2, [0.12, 0.08]), [10_000, 10_000],
                          10_000, [200, 200], 50),
            BenchmarkSpec("Box-2D9P", box_kernel(2, 1), [10_000, 10_000], 10_000,
                          [2_000, 2_000], 500),
            BenchmarkSpec("Box-2D25P", box_kernel(2, 2), [10_000, 10_000], 10_000, [120, 128],
                          60),
            BenchmarkSpec("Heat-3D", star_kernel(3, 1, 0.25, [0.125]), [1_024, 1_024, 1_024],
                          1_000, [20, 20, 20], 10),
            BenchmarkSpec("Box-3D27P", box_kernel(3, 1), [1_024, 1_024, 1_024], 1_000,
                          [20, 20, 20], 10),
        ]
    return _TABLE


def benchmark_names() -> list[str]:
    return [s.name for s in benchmark_table()]


def find_benchmark(name: str) -> BenchmarkSpec:
    for s in benchmark_table():
        if s.name == name:
            return s
    raise ValueError(f"unknown benchmark: {name}")
