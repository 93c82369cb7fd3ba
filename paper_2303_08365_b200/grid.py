"""Host grid: the reference's double-buffered ``BasicGrid<T>``
(proj/include/tessera/grid.hpp:26-132) over numpy buffers in exactly the
reference's layout (axis 0 outermost, last axis contiguous, halo on every
side), so buffers can be handed to either implementation verbatim.

``pinned=True`` backs both buffers with page-locked memory (via torch) so the
host<->device copies of ``tsr_run`` run at full PCIe rate.
"""
from __future__ import annotations

import ctypes
import struct
from typing import Callable, Sequence

import numpy as np

from . import _abi

MAX_DIMS = 3


class BasicGrid:
    dtype = np.float64
    _tsr_dtype = _abi.TSR_F64

    def __init__(self, extent: Sequence[int], halo: Sequence[int], *, pinned: bool = False):
        extent = [int(e) for e in extent]
        halo = [int(h) for h in halo]
        dims = len(extent)
        if dims < 1 or dims > MAX_DIMS or len(halo) != dims:
            raise ValueError("extent/halo must cover 1 to 3 matching axes")
        total = 1
        for a in range(dims):
            if halo[a] < 0:
                raise ValueError("negative halo width")
            if extent[a] < 2 * halo[a] + 1:
                raise ValueError(
                    f"degenerate extent {extent[a]} on axis {a}: need at least "
                    f"{2 * halo[a] + 1} interior points")
            total *= extent[a] + 2 * halo[a]
        self._dims = dims
        self._extent = extent
        self._halo = halo
        self._padded = [extent[a] + 2 * halo[a] for a in range(dims)]
        self._stride = [0] * dims
        self._stride[dims - 1] = 1
        for a in range(dims - 2, -1, -1):
            self._stride[a] = self._stride[a + 1] * self._padded[a + 1]
        self._parity = 0
        self._pin_keepalive = None
        self._buf = [self._alloc(total, pinned), self._alloc(total, pinned)]

    def _alloc(self, n: int, pinned: bool) -> np.ndarray:
        if pinned:
            import torch  # plumbing only: page-locked host memory
            t = torch.zeros(n, dtype=torch.float64 if self.dtype == np.float64 else torch.float32,
                            pin_memory=True)
            self._pin_keepalive = (self._pin_keepalive or []) + [t]
            return t.numpy()
        return np.zeros(n, dtype=self.dtype)

    # -- geometry ---------------------------------------------------------
    dims = property(lambda self: self._dims)
    parity = property(lambda self: self._parity)
    extent = property(lambda self: list(self._extent))
    halo = property(lambda self: list(self._halo))

    def stride(self, axis: int) -> int:
        return self._stride[axis]

    def flip_parity(self) -> None:
        self._parity ^= 1

    def interior_points(self) -> int:
        n = 1
        for e in self._extent:
            n *= e
        return n

    def buffer_size(self) -> int:
        return self._buf[0].size

    def flat(self, i: int, j: int = 0, k: int = 0) -> int:
        f = (i + self._halo[0]) * self._stride[0]
        if self._dims > 1:
            f += (j + self._halo[1]) * self._stride[1]
        if self._dims > 2:
            f += (k + self._halo[2]) * self._stride[2]
        return f

    # -- buffers ------------------------------------------------------------
    def buffer(self, which: int) -> np.ndarray:
        """Flat buffer `which` (a view; writes go to the grid)."""
        return self._buf[which]

    def padded(self, which: int) -> np.ndarray:
        """Buffer `which` as an ndarray of the padded shape (view)."""
        return self._buf[which].reshape(self._padded)

    def interior_view(self, which: int) -> np.ndarray:
        sl = tuple(slice(h, h + e) for e, h in zip(self._extent, self._halo))
        return self.padded(which)[sl]

    def read_data(self) -> np.ndarray:
        return self._buf[self._parity]

    def write_data(self) -> np.ndarray:
        return self._buf[1 - self._parity]

    def at(self, i: int, j: int = 0, k: int = 0):
        return self._buf[self._parity][self.flat(i, j, k)]

    def set_both(self, i: int, j: int, k: int, value) -> None:
        f = self.flat(i, j, k)
        self._buf[0][f] = value
        self._buf[1][f] = value

    def fill(self, value) -> None:
        self._buf[0][:] = value
        self._buf[1][:] = value

    def initialize(self, fn: Callable[[int, int, int], float]) -> None:
        """Every cell incl. halo, both buffers (grid.hpp:100-104)."""
        rng = [range(-self._halo[a], self._extent[a] + self._halo[a]) if a < self._dims
               else range(0, 1) for a in range(3)]
        for i in rng[0]:
            for j in rng[1]:
                for k in rng[2]:
                    self.set_both(i, j, k, fn(i, j, k))

    def to_numpy(self) -> np.ndarray:
        """Interior copy of the read buffer (module.cpp:36-47)."""
        return np.array(self.interior_view(self._parity), copy=True)

    def copy(self) -> "BasicGrid":
        g = type(self)(self._extent, self._halo)
        g._buf[0][:] = self._buf[0]
        g._buf[1][:] = self._buf[1]
        g._parity = self._parity
        return g

    # -- C-ABI views --------------------------------------------------------
    def c_struct(self) -> _abi.TsrGrid:
        g = _abi.TsrGrid()
        g.dims = self._dims
        g.dtype = self._tsr_dtype
        for a in range(3):
            g.extent[a] = self._extent[a] if a < self._dims else 1
            g.halo[a] = self._halo[a] if a < self._dims else 0
        return g

    def c_buffers(self) -> tuple[int, int]:
        return (self._buf[0].ctypes.data, self._buf[1].ctypes.data)

    def __repr__(self) -> str:
        return f"<{type(self).__name__} {'x'.join(map(str, self._extent))} parity={self._parity}>"


class Grid(BasicGrid):
    """``tessera::Grid`` = ``BasicGrid<double>``."""
    dtype = np.float64
    _tsr_dtype = _abi.TSR_F64


class GridF(BasicGrid):
    """``tessera::GridF`` = ``BasicGrid<float>``."""
    dtype = np.float32
    _tsr_dtype = _abi.TSR_F32


def grid_from_numpy(array, halo: Sequence[int] = (), halo_value: float = 0.0,
                    *, dtype=np.float64, pinned: bool = False) -> BasicGrid:
    """module.cpp:49-67: interior from `array`, halo filled with `halo_value`."""
    arr = np.ascontiguousarray(array, dtype=dtype)
    dims = arr.ndim
    if dims < 1 or dims > MAX_DIMS:
        raise ValueError("array must be 1-D to 3-D")
    halo = list(halo) if len(halo) else [1] * dims
    if len(halo) != dims:
        raise ValueError("halo must match array dimensionality")
    cls = Grid if np.dtype(dtype) == np.float64 else GridF
    g = cls(list(arr.shape), halo, pinned=pinned)
    g.fill(halo_value)
    g.interior_view(0)[...] = arr
    g.interior_view(1)[...] = arr
    return g


def fill_random(grid: BasicGrid, seed: int, lo: float = 0.0, hi: float = 1.0, *,
                skip: int = 0) -> None:
    """random.hpp:20-24 (std::mt19937_64, interior only, both buffers), run by
    the engine library's host code.  `skip` discards that many draws first:
    a slab holding planes [p, ...) of a global grid gets the global stream's
    values with skip = p * (interior cells per plane)."""
    L = _abi.lib()
    b0, b1 = grid.c_buffers()
    _abi.check(L.tsr_fill_random_at(ctypes.byref(grid.c_struct()), b0, b1,
                                    ctypes.c_uint64(seed & (2**64 - 1)), float(lo), float(hi),
                                    ctypes.c_uint64(int(skip))))


# ---- TTRS dump format (proj/src/grid_io.cpp:13-68), fp64 only ---------------
_MAGIC = b"TTRS"


def dump_grid(path: str, g: Grid) -> None:
    if g.dtype != np.float64:
        raise ValueError("grid dump is fp64 only")
    with open(path, "wb") as f:
        f.write(_MAGIC)
        f.write(struct.pack("<II", 1, g.dims))
        f.write(struct.pack(f"<{g.dims}Q", *g.extent))
        f.write(struct.pack(f"<{g.dims}Q", *g.halo))
        f.write(g.read_data().astype("<f8").tobytes())


def load_grid(path: str) -> Grid:
    with open(path, "rb") as f:
        data = f.read()
    if data[:4] != _MAGIC:
        raise RuntimeError(f"bad grid dump magic: {path}")
    ver, dims = struct.unpack_from("<II", data, 4)
    if ver != 1:
        raise RuntimeError("unsupported grid dump version")
    if dims < 1 or dims > 3:
        raise RuntimeError("bad grid dump dimensionality")
    off = 12
    extent = list(struct.unpack_from(f"<{dims}Q", data, off))
    off += 8 * dims
    halo = list(struct.unpack_from(f"<{dims}Q", data, off))
    off += 8 * dims
    g = Grid(extent, halo)
    n = g.buffer_size()
    payload = np.frombuffer(data, dtype="<f8", count=n, offset=off)
    if payload.size != n:
        raise RuntimeError(f"truncated grid dump payload: {path}")
    g.buffer(0)[:] = payload
    g.buffer(1)[:] = payload
    return g
