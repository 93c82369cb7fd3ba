"""CPU oracle for the Jacobi stencil sweep — TEST INFRASTRUCTURE ONLY.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's ``cpu_baseline`` /
``--impl reference`` legs may import this package, and only as the checker or
as the timed CPU baseline; the product (paper_2303_08365_b200/) never does.

Two checkers live here:

* ``Oracle`` wraps ``liboracle.so``, the C restatement in oracle.c of the
  reference's apply_box / naive_run / fill_random / max_rel_deviation
  (file:line citations in oracle.c).  Parity is PINNED: tests/test_oracle.py
  checks it bitwise against the reference library and the golden fixtures.
* ``Reference`` wraps ``_ref/libtessera_ref.so``: the UNMODIFIED reference
  sources under /root/reference/proj/src compiled by oracle/Makefile (plus the
  extern "C" shim ref_shim.cpp).  It exists wherever the build ran here (it
  travels to the GPU box inside the repo snapshot).

Both operate in place on grids of the product's host Grid type, whose layout
is the reference's own (proj/include/tessera/grid.hpp:46-49).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libtessera_ref.so")
REF_ROOT = "/root/reference/proj"

_i64p = ctypes.POINTER(ctypes.c_int64)
_i32p = ctypes.POINTER(ctypes.c_int32)
_f64p = ctypes.POINTER(ctypes.c_double)
_vp = ctypes.c_void_p


def build(ref: bool = True) -> None:
    """Builds liboracle.so and (when /root/reference exists) _ref/."""
    subprocess.run(["make", "-s", "-C", HERE, "oracle"], check=True)
    if ref and os.path.isdir(REF_ROOT):
        subprocess.run(["make", "-s", "-j8", "-C", HERE, "ref"], check=True)


class HostGrid:
    """Minimal double-buffered host grid in the reference's own layout
    (proj/include/tessera/grid.hpp:26-132) for callers that must not import
    the product: bench.py's reference arm.  Exposes exactly what the
    checkers below use (extent, halo, dims, dtype, parity, c_buffers,
    flip_parity, read_data)."""

    def __init__(self, extent, halo, dtype=np.float64):
        self.extent = [int(e) for e in extent]
        self.halo = [int(h) for h in halo]
        self.dims = len(self.extent)
        self.dtype = np.dtype(dtype).type
        total = 1
        for e, h in zip(self.extent, self.halo):
            total *= e + 2 * h
        self.parity = 0
        self._buf = [np.zeros(total, self.dtype), np.zeros(total, self.dtype)]

    def c_buffers(self):
        return (self._buf[0].ctypes.data, self._buf[1].ctypes.data)

    def flip_parity(self):
        self.parity ^= 1

    def read_data(self):
        return self._buf[self.parity]

    def interior_points(self) -> int:
        n = 1
        for e in self.extent:
            n *= e
        return n


class RefKernel:
    """Tap list of a Table-1 kernel as the reference library defines it
    (proj/src/bench.cpp:63-85), read through the shim: what the checkers
    need from a StencilKernel (dims, shape, radius, tap_list)."""

    def __init__(self, ref: "Reference", name: str):
        self.dims, self.shape, self.radius, self._taps = ref.benchmark_kernel(name)

    def tap_list(self):
        return list(self._taps)


def _geom(grid):
    ext = (ctypes.c_int64 * 3)(*(grid.extent + [1] * (3 - grid.dims)))
    halo = (ctypes.c_int64 * 3)(*(grid.halo + [0] * (3 - grid.dims)))
    return ext, halo


def _taps(kernel):
    taps = kernel.tap_list()
    offs = (ctypes.c_int32 * (3 * len(taps)))(*[v for o, _ in taps for v in o])
    ws = (ctypes.c_double * len(taps))(*[w for _, w in taps])
    return len(taps), offs, ws


def _sfx(grid) -> str:
    return "f64" if grid.dtype == np.float64 else "f32"


class Oracle:
    """The C restatement (oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build(ref=False)
        self.L = ctypes.CDLL(path)
        for s in ("f64", "f32"):
            getattr(self.L, f"orc_apply_box_{s}").restype = ctypes.c_int64
            getattr(self.L, f"orc_naive_run_{s}").restype = ctypes.c_int
        self.L.orc_mt64_stream.argtypes = [ctypes.c_uint64, ctypes.c_int64, _vp]

    def mt64(self, seed: int, count: int) -> np.ndarray:
        out = np.zeros(count, dtype=np.uint64)
        self.L.orc_mt64_stream(ctypes.c_uint64(seed), count, out.ctypes.data)
        return out

    def fill_random(self, grid, seed: int, lo: float = 0.0, hi: float = 1.0) -> None:
        ext, halo = _geom(grid)
        b0, b1 = grid.c_buffers()
        getattr(self.L, f"orc_fill_random_{_sfx(grid)}")(
            grid.dims, ext, halo, ctypes.c_uint64(seed), ctypes.c_double(lo), ctypes.c_double(hi),
            _vp(b0), _vp(b1))

    def naive_run(self, grid, kernel, steps: int) -> None:
        ext, halo = _geom(grid)
        n, offs, ws = _taps(kernel)
        b0, b1 = grid.c_buffers()
        p = getattr(self.L, f"orc_naive_run_{_sfx(grid)}")(
            grid.dims, ext, halo, n, offs, ws, _vp(b0), _vp(b1), grid.parity,
            ctypes.c_int64(steps))
        if p < 0:
            raise ValueError("oracle naive_run rejected its arguments")
        if p != grid.parity:
            grid.flip_parity()

    def apply_box(self, grid, kernel, lo, hi, read_parity: int) -> int:
        """apply_box on [lo, hi) reading buffer `read_parity`; no flip."""
        ext, halo = _geom(grid)
        n, offs, ws = _taps(kernel)
        lo3 = (ctypes.c_int64 * 3)(*(list(lo) + [0] * (3 - len(lo))))
        hi3 = (ctypes.c_int64 * 3)(*(list(hi) + [1] * (3 - len(hi))))
        bufs = grid.c_buffers()
        return getattr(self.L, f"orc_apply_box_{_sfx(grid)}")(
            grid.dims, ext, halo, n, offs, ws, lo3, hi3, _vp(bufs[read_parity]),
            _vp(bufs[1 - read_parity]))

    def deviation(self, a, ref) -> dict:
        """(max_rel_deviation, max_abs, l2_rel) on the read buffers."""
        ext, halo = _geom(ref)
        out = (ctypes.c_double * 3)()
        getattr(self.L, f"orc_deviation_{_sfx(ref)}")(
            ref.dims, ext, halo, _vp(a.read_data().ctypes.data),
            _vp(ref.read_data().ctypes.data), out)
        return {"max_rel_deviation": out[0], "max_abs_err": out[1], "l2_rel_err": out[2]}


class Reference:
    """The reference library itself (oracle/_ref/libtessera_ref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"reference build missing: {path} (run make -C oracle ref)")
        self.L = ctypes.CDLL(path)
        self.L.ref_last_error.restype = ctypes.c_char_p

    @staticmethod
    def available() -> bool:
        return os.path.exists(REF_SO)

    def _err(self, rc):
        if rc < 0:
            raise ValueError(self.L.ref_last_error().decode())
        return rc

    def threads(self) -> int:
        return self.L.ref_default_threads()

    def benchmark_kernel(self, name: str):
        dims, shape, radius = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        offs = (ctypes.c_int32 * (3 * 125))()
        ws = (ctypes.c_double * 125)()
        n = self._err(self.L.ref_benchmark_kernel(name.encode(), ctypes.byref(dims),
                                                  ctypes.byref(shape), ctypes.byref(radius),
                                                  offs, ws))
        taps = [((offs[3 * t], offs[3 * t + 1], offs[3 * t + 2]), ws[t]) for t in range(n)]
        return dims.value, ("star", "box")[shape.value], radius.value, taps

    def fill_random(self, grid, seed: int, lo: float = 0.0, hi: float = 1.0) -> None:
        ext, halo = _geom(grid)
        b0, b1 = grid.c_buffers()
        self._err(getattr(self.L, f"ref_fill_random_{_sfx(grid)}")(
            grid.dims, ext, halo, ctypes.c_uint64(seed), ctypes.c_double(lo),
            ctypes.c_double(hi), _vp(b0), _vp(b1)))

    def naive_run(self, grid, kernel, steps: int) -> None:
        ext, halo = _geom(grid)
        n, offs, ws = _taps(kernel)
        b0, b1 = grid.c_buffers()
        p = self._err(getattr(self.L, f"ref_naive_run_{_sfx(grid)}")(
            grid.dims, ext, halo, ("star", "box").index(kernel.shape), kernel.radius, n, offs,
            ws, _vp(b0), _vp(b1), grid.parity, ctypes.c_int64(steps)))
        if p != grid.parity:
            grid.flip_parity()

    def run_tessellated(self, grid, kernel, steps: int, tile, tb: int, threads: int = 1):
        """Returns ((point_updates, rounds, trailing), seconds)."""
        ext, halo = _geom(grid)
        n, offs, ws = _taps(kernel)
        b0, b1 = grid.c_buffers()
        t3 = (ctypes.c_int64 * 3)(*(list(tile) + [1] * (3 - len(tile))))
        st = (ctypes.c_int64 * 3)()
        sec = ctypes.c_double()
        p = self._err(self.L.ref_run_tessellated(
            grid.dims, ext, halo, ("star", "box").index(kernel.shape), kernel.radius, n, offs,
            ws, _vp(b0), _vp(b1), grid.parity, ctypes.c_int64(steps), t3, tb, threads, st,
            ctypes.byref(sec)))
        if p != grid.parity:
            grid.flip_parity()
        return (st[0], st[1], st[2]), sec.value

    def time_naive_f32(self, grid, kernel, steps: int) -> float:
        ext, halo = _geom(grid)
        n, offs, ws = _taps(kernel)
        b0, b1 = grid.c_buffers()
        sec = ctypes.c_double()
        p = self._err(self.L.ref_time_naive_f32(
            grid.dims, ext, halo, ("star", "box").index(kernel.shape), kernel.radius, n, offs,
            ws, _vp(b0), _vp(b1), grid.parity, ctypes.c_int64(steps), ctypes.byref(sec)))
        if p != grid.parity:
            grid.flip_parity()
        return sec.value

    def run_heterogeneous(self, grid, kernel, steps: int, tile_width: int, tb: int,
                          threaded: bool = False):
        """Returns (messages, ghost_recompute_points, first_message_bytes, boundary)."""
        ext, halo = _geom(grid)
        n, offs, ws = _taps(kernel)
        b0, b1 = grid.c_buffers()
        log = (ctypes.c_int64 * 3)()
        bnd = ctypes.c_int64()
        p = self._err(self.L.ref_run_heterogeneous(
            grid.dims, ext, halo, ("star", "box").index(kernel.shape), kernel.radius, n, offs,
            ws, _vp(b0), _vp(b1), grid.parity, ctypes.c_int64(steps),
            ctypes.c_int64(tile_width), tb, int(threaded), log, ctypes.byref(bnd)))
        if p != grid.parity:
            grid.flip_parity()
        return log[0], log[1], log[2], bnd.value

    def case_study_heat(self, out_dir: str, extent: int, steps: int, checkpoints, sample_every: int,
                        mu: float = 0.23, sigma: float = 0.0, path: str = "tessellate",
                        threads: int = 1) -> dict:
        """The reference's case_study_heat (case_study.cpp:171-290), run by
        _ref/case_study_ref in its own process: its artifacts in out_dir and
        the result arrays (bit-exact, via hex floats)."""
        exe = os.path.join(HERE, "_ref", "case_study_ref")
        out = subprocess.run([exe, out_dir, str(extent), str(steps), str(sample_every),
                              repr(float(mu)), repr(float(sigma)), path, str(threads),
                              ",".join(str(int(c)) for c in checkpoints)],
                             capture_output=True, text=True)
        if out.returncode != 0:
            raise ValueError(out.stderr.strip())
        res = {"series_steps": [], "center_series": [], "checkpoint_steps": [],
               "checkpoint_errors": [], "final_center": None}
        for line in out.stdout.splitlines():
            tok = line.split()
            if tok[0] == "series":
                res["series_steps"].append(int(tok[1]))
                res["center_series"].append(float.fromhex(tok[2]))
            elif tok[0] == "check":
                v = [float.fromhex(t) for t in tok[2:8]]
                res["checkpoint_steps"].append(int(tok[1]))
                res["checkpoint_errors"].append((v[:3], v[3:]))
            elif tok[0] == "final":
                res["final_center"] = float.fromhex(tok[1])
        return res

    def plan_tiles(self, extent, tile, tb: int, radius: int):
        """The reference's plan_tiles + count_coverage: (upright, inverted,
        (all_ones, min, max), [(kind tuple, index tuple, wave), ...])."""
        d = len(extent)
        ext = (ctypes.c_int64 * 3)(*(list(extent) + [1] * (3 - d)))
        til = (ctypes.c_int64 * 3)(*(list(tile) + [1] * (3 - d)))
        out = (ctypes.c_int64 * 5)()
        cap = 1
        for e, t in zip(extent, tile):
            cap *= 2 * max(1, e // t)
        tl = (ctypes.c_int32 * (7 * cap))()
        self._err(self.L.ref_plan_tiles(d, ext, til, tb, radius, out, tl, ctypes.c_int64(cap)))
        n = out[0] + out[1]
        kinds = ("upright", "inverted")
        tiles = [(tuple(kinds[tl[7 * i + a]] for a in range(d)),
                  tuple(tl[7 * i + 3 + a] for a in range(d)), tl[7 * i + 6]) for i in range(n)]
        return out[0], out[1], (bool(out[2]), out[3], out[4]), tiles
