"""ctypes binding of the C-ABI in include/tessera_b200.h.

The shared library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_2303_08365_b200/csrc``) into ``paper_2303_08365_b200/_native``.
There is no fallback: if the library is missing, every call that needs it
raises ``ImportError`` with the build command.
"""
from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_native", "libtessera_b200.so")

TSR_OK, TSR_EINVAL, TSR_ECUDA, TSR_ENCCL, TSR_ENOMEM, TSR_EUNSUPPORTED = range(6)
TSR_F64, TSR_F32 = 0, 1
TSR_STAR, TSR_BOX = 0, 1
TSR_EXACT, TSR_FAST = 0, 1
ENGINES = {"auto": 0, "generic": 1, "tuned": 2}
MODES = {"exact": TSR_EXACT, "fast": TSR_FAST}

# Every symbol include/tessera_b200.h declares (tests check the .so exports them).
EXPORTED = (
    "tsr_abi_version", "tsr_last_error", "tsr_release_cache", "tsr_check_kernel",
    "tsr_fill_random", "tsr_fill_random_at", "tsr_fill_plate", "tsr_layout_of", "tsr_run", "tsr_upload", "tsr_download",
    "tsr_copy_halo", "tsr_advance", "tsr_query_plan", "tsr_apply_box", "tsr_sweep_range",
    "tsr_sweep_range_mirror", "tsr_ipc_export", "tsr_ipc_open", "tsr_ipc_close",
    "tsr_peer_signal", "tsr_peer_wait", "tsr_peer_round_wait", "tsr_peer_round_signal",
    "tsr_multi_create", "tsr_multi_destroy", "tsr_multi_upload", "tsr_multi_fill_random",
    "tsr_multi_advance", "tsr_multi_download", "tsr_multi_slab_info", "tsr_multi_set_logging",
    "tsr_multi_comm_log", "tsr_multi_plane_checksums", "tsr_plane_checksums", "tsr_run_multi",
)
ABI_VERSION = 3
TSR_XPORT_AUTO, TSR_XPORT_MIRROR, TSR_XPORT_COPY = 0, 1, 2
TRANSPORTS = {"auto": TSR_XPORT_AUTO, "mirror": TSR_XPORT_MIRROR, "copy": TSR_XPORT_COPY}
TSR_PART_POISON = 1


class TsrKernel(ctypes.Structure):
    _fields_ = [
        ("dims", ctypes.c_int32),
        ("shape", ctypes.c_int32),
        ("radius", ctypes.c_int32),
        ("ntaps", ctypes.c_int32),
        ("offsets", ctypes.POINTER(ctypes.c_int32)),
        ("weights", ctypes.POINTER(ctypes.c_double)),
    ]


class TsrGrid(ctypes.Structure):
    _fields_ = [
        ("dims", ctypes.c_int32),
        ("dtype", ctypes.c_int32),
        ("extent", ctypes.c_int64 * 3),
        ("halo", ctypes.c_int64 * 3),
    ]


class TsrLayout(ctypes.Structure):
    _fields_ = [
        ("pitch", ctypes.c_int64 * 3),
        ("origin", ctypes.c_int64),
        ("elements", ctypes.c_int64),
    ]


class TsrOpts(ctypes.Structure):
    _fields_ = [
        ("fused_steps", ctypes.c_int32),
        ("mode", ctypes.c_int32),
        ("engine", ctypes.c_int32),
        ("device", ctypes.c_int32),
        ("ngpus", ctypes.c_int32),
        ("split_axis", ctypes.c_int32),
    ]


class TsrPartition(ctypes.Structure):
    _fields_ = [
        ("ngpus", ctypes.c_int32),
        ("split_axis", ctypes.c_int32),
        ("devices", ctypes.POINTER(ctypes.c_int32)),
        ("boundaries", ctypes.POINTER(ctypes.c_int64)),
        ("transport", ctypes.c_int32),
        ("flags", ctypes.c_int32),
    ]


class TsrSlabInfo(ctypes.Structure):
    _fields_ = [
        ("device", ctypes.c_int32),
        ("cur", ctypes.c_int32),
        ("own_lo", ctypes.c_int64),
        ("own_hi", ctypes.c_int64),
        ("ghost_lo", ctypes.c_int64),
        ("ghost_hi", ctypes.c_int64),
        ("grid", TsrGrid),
        ("layout", TsrLayout),
        ("buf", ctypes.c_void_p * 2),
    ]


class TsrCommRecord(ctypes.Structure):
    _fields_ = [
        ("round", ctypes.c_int64),
        ("from_slab", ctypes.c_int32),
        ("to_slab", ctypes.c_int32),
        ("bytes", ctypes.c_int64),
        ("seam_ms", ctypes.c_double),
        ("seam_t0_ms", ctypes.c_double),
        ("seam_t1_ms", ctypes.c_double),
        ("interior_t0_ms", ctypes.c_double),
        ("interior_t1_ms", ctypes.c_double),
    ]


class TsrIpcHandle(ctypes.Structure):
    _fields_ = [("bytes", ctypes.c_ubyte * 64)]


class TsrStats(ctypes.Structure):
    _fields_ = [
        ("device_ms", ctypes.c_double),
        ("point_updates", ctypes.c_int64),
        ("rounds", ctypes.c_int64),
        ("trailing_steps", ctypes.c_int64),
        ("kernel_launches", ctypes.c_int64),
        ("h2d_bytes", ctypes.c_int64),
        ("d2h_bytes", ctypes.c_int64),
        ("fused_steps", ctypes.c_int32),
        ("engine", ctypes.c_int32),
        ("bytes_exchanged", ctypes.c_int64),
        ("messages", ctypes.c_int64),
        ("ghost_recompute_points", ctypes.c_int64),
        ("ngpus", ctypes.c_int32),
        ("transport", ctypes.c_int32),
    ]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


_lib = None
_lock = threading.Lock()


def lib() -> ctypes.CDLL:
    """Loads the engine library (once); raises if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"B200 sweep engine not built: {LIB_PATH} is missing "
                "(run `python -c 'import __graft_entry__ as g; g.build()'` or "
                "`make -C paper_2303_08365_b200/csrc`)")
        L = ctypes.CDLL(LIB_PATH)
        p, c_void_p = ctypes.POINTER, ctypes.c_void_p
        L.tsr_abi_version.restype = ctypes.c_int
        L.tsr_last_error.restype = ctypes.c_char_p
        L.tsr_release_cache.restype = ctypes.c_int
        L.tsr_check_kernel.argtypes = [p(TsrKernel)]
        L.tsr_fill_random.argtypes = [p(TsrGrid), c_void_p, c_void_p, ctypes.c_uint64,
                                      ctypes.c_double, ctypes.c_double]
        L.tsr_fill_random_at.argtypes = [p(TsrGrid), c_void_p, c_void_p, ctypes.c_uint64,
                                         ctypes.c_double, ctypes.c_double, ctypes.c_uint64]
        L.tsr_fill_plate.argtypes = [p(TsrGrid), c_void_p, c_void_p, ctypes.c_double,
                                     ctypes.c_double, ctypes.c_double]
        L.tsr_layout_of.argtypes = [p(TsrGrid), p(TsrLayout)]
        L.tsr_run.argtypes = [p(TsrKernel), p(TsrGrid), c_void_p, c_void_p, ctypes.c_int32,
                              ctypes.c_int64, p(TsrOpts), p(TsrStats)]
        L.tsr_upload.argtypes = [p(TsrGrid), p(TsrLayout), c_void_p, c_void_p, c_void_p]
        L.tsr_download.argtypes = [p(TsrGrid), p(TsrLayout), c_void_p, c_void_p,
                                   ctypes.c_int32, c_void_p]
        L.tsr_copy_halo.argtypes = [p(TsrGrid), p(TsrLayout), c_void_p, c_void_p, c_void_p]
        L.tsr_advance.argtypes = [p(TsrKernel), p(TsrGrid), p(TsrLayout), c_void_p, c_void_p,
                                  p(ctypes.c_int32), ctypes.c_int64, ctypes.c_int32,
                                  p(TsrOpts), c_void_p, p(TsrStats)]
        L.tsr_query_plan.argtypes = [p(TsrKernel), p(TsrGrid), p(TsrOpts), p(ctypes.c_int32),
                                     p(ctypes.c_int32)]
        L.tsr_apply_box.argtypes = [p(TsrKernel), p(TsrGrid), p(TsrLayout), c_void_p, c_void_p,
                                    p(ctypes.c_int64), p(ctypes.c_int64), p(TsrOpts), c_void_p]
        L.tsr_sweep_range.argtypes = [p(TsrKernel), p(TsrGrid), p(TsrLayout), c_void_p,
                                      c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int32,
                                      p(TsrOpts), c_void_p]
        L.tsr_sweep_range_mirror.argtypes = [p(TsrKernel), p(TsrGrid), p(TsrLayout), c_void_p,
                                             c_void_p, ctypes.c_int64, ctypes.c_int64,
                                             ctypes.c_int32, p(TsrOpts), c_void_p,
                                             ctypes.c_int64, c_void_p]
        L.tsr_ipc_export.argtypes = [c_void_p, p(TsrIpcHandle), p(ctypes.c_int64)]
        L.tsr_ipc_open.argtypes = [p(TsrIpcHandle), p(c_void_p)]
        L.tsr_ipc_close.argtypes = [c_void_p]
        L.tsr_peer_signal.argtypes = [c_void_p, ctypes.c_uint32, c_void_p]
        L.tsr_peer_wait.argtypes = [c_void_p, ctypes.c_uint32, c_void_p]
        L.tsr_peer_round_wait.argtypes = [c_void_p, c_void_p, c_void_p, c_void_p]
        L.tsr_peer_round_signal.argtypes = [c_void_p, c_void_p, c_void_p, c_void_p]
        vp = c_void_p
        L.tsr_multi_create.argtypes = [p(TsrKernel), p(TsrGrid), p(TsrPartition), p(TsrOpts),
                                       p(vp)]
        L.tsr_multi_destroy.argtypes = [vp]
        L.tsr_multi_upload.argtypes = [vp, vp]
        L.tsr_multi_fill_random.argtypes = [vp, ctypes.c_uint64, ctypes.c_double,
                                            ctypes.c_double]
        L.tsr_multi_advance.argtypes = [vp, ctypes.c_int64, ctypes.c_int32, p(TsrStats)]
        L.tsr_multi_download.argtypes = [vp, vp, vp]
        L.tsr_multi_slab_info.argtypes = [vp, ctypes.c_int32, p(TsrSlabInfo)]
        L.tsr_multi_set_logging.argtypes = [vp, ctypes.c_int32]
        L.tsr_multi_comm_log.argtypes = [vp, p(TsrCommRecord), ctypes.c_int64,
                                         p(ctypes.c_int64)]
        L.tsr_multi_plane_checksums.argtypes = [vp, ctypes.c_int32, p(ctypes.c_uint64)]
        L.tsr_plane_checksums.argtypes = [p(TsrGrid), p(TsrLayout), vp, ctypes.c_int64,
                                          ctypes.c_int64, p(ctypes.c_uint64), vp]
        L.tsr_run_multi.argtypes = [p(TsrKernel), p(TsrGrid), vp, vp, ctypes.c_int32,
                                    ctypes.c_int64, p(TsrPartition), ctypes.c_int32, p(TsrOpts),
                                    p(TsrStats)]
        for name in EXPORTED:
            if name not in ("tsr_abi_version", "tsr_last_error"):
                getattr(L, name).restype = ctypes.c_int
        if L.tsr_abi_version() != ABI_VERSION:
            raise ImportError("libtessera_b200.so ABI version mismatch")
        _lib = L
        return L


def check(code: int) -> None:
    """Raises the Python exception matching a tsr_status (pybind11's mapping
    of the reference's std exceptions: invalid_argument -> ValueError)."""
    if code == TSR_OK:
        return
    msg = (lib().tsr_last_error() or b"").decode(errors="replace")
    if code == TSR_EINVAL:
        raise ValueError(msg)
    if code == TSR_ENOMEM:
        raise MemoryError(msg)
    if code == TSR_EUNSUPPORTED:
        raise NotImplementedError(msg)
    raise RuntimeError(msg)


def make_opts(fused_steps: int = 0, mode: str = "exact", engine: str = "auto",
              device: int = -1, ngpus: int = 1) -> TsrOpts:
    if mode not in MODES:
        raise ValueError("mode must be 'exact' or 'fast'")
    if engine not in ENGINES:
        raise ValueError("engine must be 'auto', 'generic' or 'tuned'")
    if fused_steps < 0:
        raise ValueError("fused_steps must be >= 0")
    if ngpus < 1:
        raise ValueError("ngpus must be >= 1")
    return TsrOpts(int(fused_steps), MODES[mode], ENGINES[engine], int(device), int(ngpus), 0)


def make_partition(ngpus: int, devices=None, boundaries=None, transport: str = "auto",
                   poison: bool = False):
    """tsr_partition (arrays kept alive on the returned struct's _keep)."""
    if transport not in TRANSPORTS:
        raise ValueError("transport must be 'auto', 'mirror' or 'copy'")
    part = TsrPartition()
    part.ngpus = int(ngpus)
    part.split_axis = 0
    keep = []
    if devices is not None:
        if len(devices) != ngpus:
            raise ValueError("one device ordinal per slab")
        arr = (ctypes.c_int32 * ngpus)(*devices)
        keep.append(arr)
        part.devices = ctypes.cast(arr, ctypes.POINTER(ctypes.c_int32))
    if boundaries is not None:
        if len(boundaries) != ngpus - 1:
            raise ValueError("ngpus - 1 slab boundaries")
        arr = (ctypes.c_int64 * max(1, ngpus - 1))(*boundaries)
        keep.append(arr)
        part.boundaries = ctypes.cast(arr, ctypes.POINTER(ctypes.c_int64))
    part.transport = TRANSPORTS[transport]
    part.flags = TSR_PART_POISON if poison else 0
    part._keep = keep
    return part


def query_plan(kernel, grid_desc: TsrGrid, fused_steps: int = 0, mode: str = "exact",
               engine: str = "auto") -> tuple[str, int]:
    """(engine, k) the library would use for this kernel and grid."""
    L = lib()
    e, k = ctypes.c_int32(), ctypes.c_int32()
    opts = make_opts(fused_steps, mode, engine)
    check(L.tsr_query_plan(ctypes.byref(kernel.c_struct()), ctypes.byref(grid_desc),
                           ctypes.byref(opts), ctypes.byref(e), ctypes.byref(k)))
    return {1: "generic", 2: "tuned"}[e.value], k.value


def ipc_export(ptr: int) -> tuple[bytes, int]:
    """(64-byte CUDA IPC handle of the allocation holding `ptr`, byte offset
    of `ptr` in it)."""
    h, off = TsrIpcHandle(), ctypes.c_int64()
    check(lib().tsr_ipc_export(ctypes.c_void_p(ptr), ctypes.byref(h), ctypes.byref(off)))
    return bytes(h.bytes), off.value


def ipc_open(handle: bytes) -> int:
    """Maps another process's allocation; returns its base address here."""
    h = TsrIpcHandle()
    ctypes.memmove(h.bytes, handle, 64)
    base = ctypes.c_void_p()
    check(lib().tsr_ipc_open(ctypes.byref(h), ctypes.byref(base)))
    return base.value


def ipc_close(base: int) -> None:
    check(lib().tsr_ipc_close(ctypes.c_void_p(base)))


def grid_desc(extent, halo, dtype: str = "f64") -> TsrGrid:
    g = TsrGrid()
    g.dims = len(extent)
    g.dtype = TSR_F64 if dtype == "f64" else TSR_F32
    for a in range(3):
        g.extent[a] = int(extent[a]) if a < len(extent) else 1
        g.halo[a] = int(halo[a]) if a < len(extent) else 0
    return g
