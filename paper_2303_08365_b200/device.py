"""Device-resident grids: the two buffers of a BasicGrid<T> living in HBM in
the engine's pitched layout (``tsr_layout_of``), advanced without host
round trips.  torch supplies the device memory and streams (plumbing only);
every sweep is a launch of the engine library through ``tsr_advance``.
"""
from __future__ import annotations

import ctypes

from . import _abi
from .grid import BasicGrid
from .kernel import StencilKernel


def layout_of(grid_desc: _abi.TsrGrid) -> _abi.TsrLayout:
    L = _abi.lib()
    lay = _abi.TsrLayout()
    _abi.check(L.tsr_layout_of(ctypes.byref(grid_desc), ctypes.byref(lay)))
    return lay


def _torch_dtype(grid: BasicGrid):
    import torch
    return torch.float64 if grid._tsr_dtype == _abi.TSR_F64 else torch.float32


class DeviceGrid:
    """Device copy of a host grid.  ``advance`` runs fused sweeps on the
    current torch stream; ``download`` writes the state back into a host grid
    exactly as naive_run would have left it."""

    def __init__(self, grid: BasicGrid, device=None, *, upload: bool = True):
        import torch
        self.torch = torch
        self.device = torch.device(device if device is not None else "cuda")
        if self.device.type != "cuda":
            raise ValueError("DeviceGrid needs a CUDA device")
        self.desc = grid.c_struct()
        self.layout = layout_of(self.desc)
        self.dims = grid.dims
        self.extent = grid.extent
        self.halo = grid.halo
        self.esize = 8 if grid._tsr_dtype == _abi.TSR_F64 else 4
        n = self.layout.elements
        self.buf = [torch.empty(n, dtype=_torch_dtype(grid), device=self.device),
                    torch.empty(n, dtype=_torch_dtype(grid), device=self.device)]
        self.cur = 0
        self.steps_done = 0
        self.prev_valid = False
        if upload:
            self.upload(grid)

    def _stream(self, stream=None) -> int:
        s = stream if stream is not None else self.torch.cuda.current_stream(self.device)
        return s.cuda_stream

    def ptr(self, which: int) -> int:
        return self.buf[which].data_ptr()

    def upload(self, grid: BasicGrid, stream=None) -> None:
        """Read buffer of `grid` -> device buffer 0, halo shell -> buffer 1."""
        L = _abi.lib()
        s = self._stream(stream)
        with self.torch.cuda.device(self.device):
            _abi.check(L.tsr_upload(ctypes.byref(self.desc), ctypes.byref(self.layout),
                                    grid.read_data().ctypes.data, self.ptr(0), s))
            _abi.check(L.tsr_copy_halo(ctypes.byref(self.desc), ctypes.byref(self.layout),
                                       self.ptr(0), self.ptr(1), s))
        self.cur = 0
        self.steps_done = 0
        self.prev_valid = False

    def advance(self, kernel: StencilKernel, steps: int, *, fused_steps: int = 0,
                mode: str = "exact", engine: str = "auto", keep_previous: bool = False,
                stream=None) -> _abi.TsrStats:
        L = _abi.lib()
        st = _abi.TsrStats()
        cur = ctypes.c_int32(self.cur)
        opts = _abi.make_opts(fused_steps, mode, engine)
        with self.torch.cuda.device(self.device):
            _abi.check(L.tsr_advance(ctypes.byref(kernel.c_struct()), ctypes.byref(self.desc),
                                     ctypes.byref(self.layout), self.ptr(0), self.ptr(1),
                                     ctypes.byref(cur), int(steps), int(bool(keep_previous)),
                                     ctypes.byref(opts), self._stream(stream),
                                     ctypes.byref(st)))
        self.cur = cur.value
        if steps > 0:
            # One step (or keep_previous) leaves step T-1 in the other buffer.
            self.prev_valid = bool(keep_previous) or steps == 1
        self.steps_done += int(steps)
        return st

    def sweep_range(self, kernel: StencilKernel, lo: int, hi: int, steps: int, *,
                    fused_steps: int = 0, mode: str = "exact", engine: str = "auto",
                    mirror: int = 0, mirror_planes: int = 0, stream=None) -> int:
        """One fused pass of `steps` time steps from the current buffer into
        the other one, storing only the planes [lo, hi) of axis 0
        (tsr_sweep_range).  Does not flip the buffers: a slab round launches
        its interior and seam ranges separately, then calls ``flip``.
        With `mirror` (a device address, e.g. a peer slab's next buffer
        mapped by CUDA IPC) every stored plane p is also written to plane
        p + mirror_planes of that buffer (tsr_sweep_range_mirror).
        Returns the number of kernels launched (0 for an empty range)."""
        if hi <= lo:
            return 0
        L = _abi.lib()
        opts = _abi.make_opts(fused_steps, mode, engine)
        with self.torch.cuda.device(self.device):
            _abi.check(L.tsr_sweep_range_mirror(
                ctypes.byref(kernel.c_struct()), ctypes.byref(self.desc),
                ctypes.byref(self.layout), self.ptr(self.cur), self.ptr(1 - self.cur), int(lo),
                int(hi), int(steps), ctypes.byref(opts), ctypes.c_void_p(mirror or None),
                int(mirror_planes), self._stream(stream)))
        return 1

    def plane_checksums(self, which: int = 0, lo: int = 0, hi: int | None = None, stream=None):
        """64-bit position-mixed checksum of each interior plane [lo, hi) of
        axis 0 of the current (0) or other (1) buffer (tsr_plane_checksums):
        compares a grid with a slab run without moving either."""
        import numpy as np
        hi = self.extent[0] if hi is None else hi
        out = np.zeros(max(0, hi - lo), dtype=np.uint64)
        buf = self.cur if which == 0 else 1 - self.cur
        with self.torch.cuda.device(self.device):
            _abi.check(_abi.lib().tsr_plane_checksums(
                ctypes.byref(self.desc), ctypes.byref(self.layout), self.ptr(buf), int(lo),
                int(hi), out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)),
                self._stream(stream)))
        return out

    def flip(self, steps: int) -> None:
        """Makes the other buffer current after a round of `steps` steps
        written by ``sweep_range`` calls."""
        self.cur ^= 1
        self.steps_done += int(steps)
        self.prev_valid = steps == 1

    def download(self, grid: BasicGrid, stream=None) -> None:
        """Interior of the current buffer -> grid.buffer(final parity); the
        previous step (when kept) -> the other buffer; parity flipped by the
        number of steps advanced since upload."""
        L = _abi.lib()
        s = self._stream(stream)
        if self.steps_done & 1:
            grid.flip_parity()
        bufs = grid.c_buffers()
        with self.torch.cuda.device(self.device):
            _abi.check(L.tsr_download(ctypes.byref(self.desc), ctypes.byref(self.layout),
                                      self.ptr(self.cur), bufs[grid.parity], 1, s))
            if self.steps_done >= 1 and self.prev_valid:
                _abi.check(L.tsr_download(ctypes.byref(self.desc), ctypes.byref(self.layout),
                                          self.ptr(1 - self.cur), bufs[1 - grid.parity], 1, s))
            # the copies were queued on `stream` (or the current stream)
            (stream if stream is not None
             else self.torch.cuda.current_stream(self.device)).synchronize()
        self.steps_done = 0

    # ---- TTRS snapshot / resume (proj/src/grid_io.cpp:34-68) -------------
    def snapshot(self, path: str, stream=None) -> None:
        """Writes the current device state (interior and halo of the
        current buffer) as a TTRS grid dump, the reference's format
        (dump_grid, grid_io.cpp:34-45: fp64 payload; an fp32 grid is
        widened, which is exact).  The device state is untouched, so a long
        run can checkpoint every N steps and keep going."""
        from .grid import Grid, GridF, dump_grid
        cls = Grid if self.esize == 8 else GridF
        host = cls(list(self.extent), list(self.halo))
        L = _abi.lib()
        s = self._stream(stream)
        with self.torch.cuda.device(self.device):
            _abi.check(L.tsr_download(ctypes.byref(self.desc), ctypes.byref(self.layout),
                                      self.ptr(self.cur), host.c_buffers()[0], 0, s))
            (stream if stream is not None
             else self.torch.cuda.current_stream(self.device)).synchronize()
        if self.esize == 4:
            wide = Grid(list(self.extent), list(self.halo))
            wide.buffer(0)[:] = host.buffer(0).astype("f8")
            host = wide
        dump_grid(path, host)

    @classmethod
    def resume(cls, path: str, device=None, dtype: str = "f64") -> "DeviceGrid":
        """A DeviceGrid holding a TTRS dump (load_grid, grid_io.cpp:47-68)
        as its current state; dtype "f32" narrows the payload (exact for a
        dump written from an fp32 grid)."""
        from .grid import GridF, load_grid
        g = load_grid(path)
        if dtype == "f32":
            f = GridF(list(g.extent), list(g.halo))
            for w in (0, 1):
                f.buffer(w)[:] = g.buffer(w).astype("f4")
            g = f
        elif dtype != "f64":
            raise ValueError(f"unknown dtype {dtype!r}")
        return cls(g, device)

