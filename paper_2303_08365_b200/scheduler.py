"""The reference's heterogeneous scheduler API (proj/include/tessera/scheduler.hpp)
on the memory tier of the B200 engine: slabs of axis 0 on several GPUs, one
host thread driving them through the C-ABI (``tsr_multi_*`` /
``tsr_run_multi`` in include/tessera_b200.h).

Names, arguments and error behaviour follow the reference's binding
(proj/bindings/module.cpp:300-370):

* ``WorkerSpec`` / ``WorkerProfile`` / ``profile_workers``  (scheduler.hpp:20-45)
* ``PartitionPlan`` / ``plan_partition``                   (scheduler.hpp:47-64,
  scheduler.cpp:108-140: boundary = ratio snapped to a tile multiple)
* ``CommCostModel`` / ``comm_cost``                         (scheduler.hpp:66-73,
  scheduler.cpp:142-150: alpha-beta costs)
* ``CommRecord`` / ``CommLog`` / ``dump_comm_log``         (scheduler.hpp:75-92,
  scheduler.cpp:152-159: the per-round CSV)
* ``run_heterogeneous`` / ``run_heterogeneous_instrumented`` (scheduler.hpp:97-124)

The paper's CPU+accelerator split becomes a GPU-only split (north star): the
two workers are two slabs, on two GPUs when the box has them.  ``SlabGrid``
and ``run_multi`` generalise it to P equal (or given) slabs.
"""
from __future__ import annotations

import ctypes
import math
import time
from dataclasses import dataclass, field

from . import _abi
from .grid import BasicGrid
from .kernel import StencilKernel

WORKER_KINDS = ("cpu_like", "accel_like")
STEP_ENGINES = ("naive", "tessellate", "vector", "mm")


@dataclass
class WorkerSpec:
    """scheduler.hpp:20-27.  `engine` is accepted for signature parity (every
    slab runs the B200 engine); `simulated_seconds_per_megastencil` replaces
    timing like the reference's; `device` pins the worker's GPU."""
    kind: str = "cpu_like"
    engine: str = "naive"
    simulated_seconds_per_megastencil: float | None = None
    device: int | None = None

    def __post_init__(self):
        if self.kind not in WORKER_KINDS:
            raise ValueError(f"unknown worker kind '{self.kind}'")
        if self.engine not in STEP_ENGINES:
            raise ValueError(f"unknown step engine '{self.engine}'")


@dataclass
class WorkerProfile:
    """scheduler.hpp:29-38."""
    kind: str = "cpu_like"
    seconds_per_megastencil: float = 0.0
    sample_extent: list = field(default_factory=list)
    iterations: int = 0
    relative_spread: float = 0.0

    def megastencils_per_second(self) -> float:
        return 1.0 / self.seconds_per_megastencil


def profile_workers(a: WorkerSpec, b: WorkerSpec, kernel: StencilKernel, sample_extent,
                    warm_iters: int):
    """scheduler.cpp:61-106: a simulated rate is taken as is; otherwise one
    step of the GPU engine on a fill_random(1) sample grid is timed
    `warm_iters` times after a warm-up on the worker's device."""
    from .grid import Grid, fill_random
    from .run import run_gpu
    if warm_iters < 1:
        raise ValueError("warm_iters must be >= 1")
    sample_extent = [int(e) for e in sample_extent]

    def one(w: WorkerSpec) -> WorkerProfile:
        p = WorkerProfile(kind=w.kind, sample_extent=list(sample_extent),
                          iterations=warm_iters)
        if w.simulated_seconds_per_megastencil is not None:
            p.seconds_per_megastencil = float(w.simulated_seconds_per_megastencil)
            return p
        g = Grid(sample_extent, [kernel.radius] * len(sample_extent))
        fill_random(g, 1)
        dev = -1 if w.device is None else int(w.device)
        run_gpu(g, kernel, 1, device=dev)  # warm-up (kernel load, buffers)
        times = []
        for _ in range(warm_iters):
            t0 = time.perf_counter()
            run_gpu(g, kernel, 1, device=dev)
            times.append(time.perf_counter() - t0)
        mean = sum(times) / len(times)
        p.seconds_per_megastencil = mean / (g.interior_points() / 1e6)
        p.relative_spread = (max(times) - min(times)) / mean if warm_iters > 1 else 0.0
        return p

    return one(a), one(b)


@dataclass
class PartitionPlan:
    """scheduler.hpp:47-64: two-way split of axis 0; the faster worker owns
    rows [0, boundary)."""
    split_axis: int = 0
    boundary: int = 0
    ratio: float = 0.5
    halo_depth: int = 0
    tile_width: int = 0
    tb: int = 1
    radius: int = 1
    bytes_per_exchange: int = 0
    in_flight: int = 2
    first_worker: str = "cpu_like"


def plan_partition(a: WorkerProfile, b: WorkerProfile, extent, tile_width: int, tb: int,
                   radius: int) -> PartitionPlan:
    """scheduler.cpp:108-140, same validation, rounding and tie rule."""
    extent = [int(e) for e in extent]
    if not extent:
        raise ValueError("empty extent")
    if tile_width < 1:
        raise ValueError("tile width must be positive")
    n = extent[0]
    if n < 2 * tile_width:
        raise ValueError("extent along the split axis must cover at least 2 tiles")
    plan = PartitionPlan(tile_width=int(tile_width), tb=int(tb), radius=int(radius),
                         halo_depth=int(radius) * int(tb), in_flight=2)
    ta, tbps = a.megastencils_per_second(), b.megastencils_per_second()
    a_first = ta >= tbps
    plan.first_worker = a.kind if a_first else b.kind
    plan.ratio = max(ta, tbps) / (ta + tbps)
    raw = plan.ratio * float(n)
    k = int(math.floor(raw / float(tile_width) + 0.5))
    k_max = (n - 1) // tile_width
    k = min(max(k, 1), k_max)
    plan.boundary = k * tile_width
    cross = 1
    for e in extent[1:]:
        cross *= e
    plan.bytes_per_exchange = plan.halo_depth * cross * 8 * 2
    return plan


@dataclass
class CommCostModel:
    """scheduler.hpp:66-73: alpha seconds per launch, beta seconds per byte."""
    alpha: float = 1e-5
    beta: float = 1e-9


def comm_cost(model: CommCostModel, k: int, bytes_per_message: int):
    """scheduler.cpp:142-150 -> (per_message_total, batched_total)."""
    if k < 1:
        raise ValueError("message count must be >= 1")
    kd, nb = float(k), float(bytes_per_message)
    return kd * (model.alpha + nb * model.beta), model.alpha + kd * nb * model.beta


@dataclass
class CommRecord:
    """scheduler.hpp:75-81.  On the GPU a record is one seam pass's delivery
    into a neighbour's ghost planes; `wall_seconds` is the device time of the
    sender's seam passes of that round."""
    round: int
    direction: str
    bytes: int
    modeled_cost_alpha_beta: float = 0.0
    wall_seconds: float = 0.0


@dataclass
class CommLog:
    """scheduler.hpp:83-88."""
    records: list = field(default_factory=list)
    ghost_recompute_points: int = 0
    mma_calls: int = 0

    @property
    def messages(self) -> int:
        return len(self.records)

    def rounds_and_bytes(self):
        return [(r.round, r.direction, r.bytes) for r in self.records]


def dump_comm_log(path: str, log: CommLog) -> None:
    """scheduler.cpp:152-159: round,direction,bytes,modeled_cost_alpha_beta,wall_seconds."""
    try:
        f = open(path, "w")
    except OSError as e:
        raise RuntimeError(f"cannot open comm log for writing: {path}") from e
    with f:
        f.write("round,direction,bytes,modeled_cost_alpha_beta,wall_seconds\n")
        for r in log.records:
            f.write(f"{r.round},{r.direction},{r.bytes},{r.modeled_cost_alpha_beta:g},"
                    f"{r.wall_seconds:g}\n")


# ---------------------------------------------------------------------------
# The slab set on the GPUs
# ---------------------------------------------------------------------------

@dataclass
class SlabInfo:
    device: int
    own_lo: int
    own_hi: int
    ghost_lo: int
    ghost_hi: int
    local_extent: list
    buffers: tuple
    cur: int


class SlabGrid:
    """A global grid decomposed into slabs of axis 0, resident in HBM across
    GPUs (``tsr_multi_*``).  One host thread drives every slab: a round is
    the seam passes (storing into the neighbours' ghost planes over peer
    memory) concurrently with the interior pass, ordered across devices by
    CUDA events."""

    def __init__(self, kernel: StencilKernel, extent, halo=None, dtype: str = "f64", *,
                 ngpus: int = 1, devices=None, boundaries=None, transport: str = "auto",
                 fused_steps: int = 0, mode: str = "exact", engine: str = "auto",
                 poison: bool = False):
        L = _abi.lib()
        extent = [int(e) for e in extent]
        halo = [kernel.radius] * len(extent) if halo is None else [int(h) for h in halo]
        self.kernel = kernel
        self.extent, self.halo, self.dtype = extent, halo, dtype
        self.desc = _abi.grid_desc(extent, halo, dtype)
        self._part = _abi.make_partition(ngpus, devices, boundaries, transport, poison)
        self._opts = _abi.make_opts(fused_steps, mode, engine, -1, ngpus)
        self._h = ctypes.c_void_p()
        self._kernel_c = kernel.c_struct()
        _abi.check(L.tsr_multi_create(ctypes.byref(self._kernel_c), ctypes.byref(self.desc),
                                      ctypes.byref(self._part), ctypes.byref(self._opts),
                                      ctypes.byref(self._h)))
        self.ngpus = int(ngpus)
        self.steps_done = 0

    # -- lifetime -------------------------------------------------------------
    def close(self) -> None:
        if self._h:
            _abi.lib().tsr_multi_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 - interpreter shutdown
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- data -----------------------------------------------------------------
    def upload(self, grid: BasicGrid) -> None:
        """The read buffer of a global host grid -> every slab."""
        self._check_grid(grid)
        _abi.check(_abi.lib().tsr_multi_upload(self._h, ctypes.c_void_p(grid.read_data().ctypes.data)))
        self.steps_done = 0

    def fill_random(self, seed: int, lo: float = 0.0, hi: float = 1.0) -> None:
        """fill_random of the global grid (one mt19937_64 stream, halo zero)
        streamed straight into the slabs."""
        _abi.check(_abi.lib().tsr_multi_fill_random(self._h, ctypes.c_uint64(seed), lo, hi))
        self.steps_done = 0

    def advance(self, steps: int, keep_previous: bool = False) -> _abi.TsrStats:
        st = _abi.TsrStats()
        _abi.check(_abi.lib().tsr_multi_advance(self._h, int(steps), int(bool(keep_previous)),
                                                ctypes.byref(st)))
        self.steps_done += int(steps)
        return st

    def download(self, grid: BasicGrid, previous: bool = True) -> None:
        """Owned planes -> grid.buffer(final parity) (and step T-1 -> the
        other buffer when the last round kept it); parity flipped by the
        steps advanced since the upload."""
        self._check_grid(grid)
        if self.steps_done & 1:
            grid.flip_parity()
        b = grid.c_buffers()
        prev = ctypes.c_void_p(b[1 - grid.parity]) if previous else None
        _abi.check(_abi.lib().tsr_multi_download(self._h, ctypes.c_void_p(b[grid.parity]), prev))
        self.steps_done = 0

    def plane_checksums(self, which: int = 0):
        """Per owned global plane 64-bit checksum of the current (0) or
        previous (1) buffers (tsr_multi_plane_checksums)."""
        import numpy as np
        out = np.zeros(self.extent[0], dtype=np.uint64)
        _abi.check(_abi.lib().tsr_multi_plane_checksums(
            self._h, int(which), out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))))
        return out

    def slab(self, i: int) -> SlabInfo:
        info = _abi.TsrSlabInfo()
        _abi.check(_abi.lib().tsr_multi_slab_info(self._h, int(i), ctypes.byref(info)))
        return SlabInfo(info.device, info.own_lo, info.own_hi, info.ghost_lo, info.ghost_hi,
                        [info.grid.extent[a] for a in range(info.grid.dims)],
                        (info.buf[0], info.buf[1]), info.cur)

    def set_logging(self, on: bool = True) -> None:
        _abi.check(_abi.lib().tsr_multi_set_logging(self._h, int(bool(on))))

    def _raw_log(self) -> list:
        """The runtime's delivery records since logging was switched on (or
        since the last read), consumed (tsr_multi_comm_log)."""
        L = _abi.lib()
        n = ctypes.c_int64()
        _abi.check(L.tsr_multi_comm_log(self._h, None, 0, ctypes.byref(n)))
        arr = (_abi.TsrCommRecord * max(1, n.value))()
        _abi.check(L.tsr_multi_comm_log(self._h, arr, n.value, ctypes.byref(n)))
        return list(arr[:n.value])

    def round_timeline(self) -> list:
        """Per slab and round, on the slab's device (ms after its first
        logged round): the seam passes' interval on the seam stream and the
        interior pass's on the second stream — the overlap of exchange and
        compute that the reference gets from its worker threads
        (HaloWorker::run_round, scheduler.cpp:371-406).  Consumes the log."""
        seen, out = set(), []
        for r in self._raw_log():
            key = (int(r.round), int(r.from_slab))
            if key in seen:
                continue
            seen.add(key)
            out.append({"round": key[0], "slab": key[1],
                        "seam": [r.seam_t0_ms, r.seam_t1_ms],
                        "interior": [r.interior_t0_ms, r.interior_t1_ms]})
        out.sort(key=lambda e: (e["round"], e["slab"]))
        return out

    def comm_records(self, model: CommCostModel | None = None) -> list:
        """CommRecords of the rounds run since logging was switched on (or
        since the last call); direction "w{from}_to_w{to}" as the reference
        names its two workers' messages."""
        model = model or CommCostModel()
        out = []
        for r in self._raw_log():
            out.append(CommRecord(int(r.round), f"w{r.from_slab}_to_w{r.to_slab}", int(r.bytes),
                                  model.alpha + float(r.bytes) * model.beta, r.seam_ms / 1e3))
        out.sort(key=lambda r: (r.round, r.direction))
        return out

    def _check_grid(self, grid: BasicGrid) -> None:
        if grid.extent != self.extent or grid.halo != self.halo:
            raise ValueError("grid geometry differs from the slab set's")
        if (grid._tsr_dtype == _abi.TSR_F64) != (self.dtype == "f64"):
            raise ValueError("grid dtype differs from the slab set's")


def run_multi(grid: BasicGrid, kernel: StencilKernel, steps: int, ngpus: int, *, devices=None,
              boundaries=None, transport: str = "auto", fused_steps: int = 0,
              mode: str = "exact", engine: str = "auto", keep_previous: bool = True,
              poison: bool = False) -> _abi.TsrStats:
    """naive_run over `ngpus` slabs in one call (tsr_run_multi): host buffers
    in, host buffers out; with keep_previous the grid ends exactly as
    naive_run leaves it, otherwise only the final read buffer is written
    (run_heterogeneous's post-condition)."""
    steps = int(steps)
    if steps < 0:
        raise ValueError("negative step count")
    part = _abi.make_partition(ngpus, devices, boundaries, transport, poison)
    opts = _abi.make_opts(fused_steps, mode, engine, -1, ngpus)
    st = _abi.TsrStats()
    b0, b1 = grid.c_buffers()
    _abi.check(_abi.lib().tsr_run_multi(
        ctypes.byref(kernel.c_struct()), ctypes.byref(grid.c_struct()), ctypes.c_void_p(b0),
        ctypes.c_void_p(b1), grid.parity, steps, ctypes.byref(part),
        int(bool(keep_previous)), ctypes.byref(opts), ctypes.byref(st)))
    if steps & 1:
        grid.flip_parity()
    return st


def _run_heterogeneous(grid, kernel, steps, plan, first, second, model, poison, mode):
    # run_heterogeneous_impl's checks, in its order (scheduler.cpp:445-461)
    if grid.dims != kernel.dims:
        raise ValueError("kernel/grid dimensionality mismatch")
    if any(h < kernel.radius for h in grid.halo):
        raise ValueError("grid halo too small for kernel radius")
    if steps < 0:
        raise ValueError("negative step count")
    if kernel.radius != plan.radius:
        raise ValueError("partition plan radius differs from kernel radius")
    if plan.halo_depth != plan.radius * plan.tb:
        raise ValueError("partition plan halo depth must be radius*tb")
    n = grid.extent[0]
    b = plan.boundary
    if b <= 0 or b >= n:
        raise ValueError("partition boundary outside the grid")
    if b < plan.halo_depth or n - b < plan.halo_depth:
        raise ValueError("subdomain smaller than the halo depth")
    log = CommLog()
    if steps == 0:
        return log
    import torch
    ndev = max(1, torch.cuda.device_count())
    devices = [w.device if w.device is not None else i % ndev
               for i, w in enumerate((first, second))]
    dtype = "f64" if grid._tsr_dtype == _abi.TSR_F64 else "f32"
    with SlabGrid(kernel, grid.extent, grid.halo, dtype, ngpus=2, devices=devices,
                  boundaries=[b], fused_steps=plan.tb, mode=mode, poison=poison) as sg:
        sg.upload(grid)
        sg.set_logging(True)
        st = sg.advance(steps)
        log.records = sg.comm_records(model)
        # run_heterogeneous scatters the workers' rows into the final read
        # buffer only (scheduler.cpp:555-557)
        if steps & 1:
            grid.flip_parity()
        b0, b1 = grid.c_buffers()
        _abi.check(_abi.lib().tsr_multi_download(sg._h, ctypes.c_void_p((b0, b1)[grid.parity]),
                                                 None))
    log.ghost_recompute_points = int(st.ghost_recompute_points)
    return log


def run_heterogeneous(grid: BasicGrid, kernel: StencilKernel, steps: int, plan: PartitionPlan,
                      first: WorkerSpec, second: WorkerSpec, threaded: bool = True, *,
                      model: CommCostModel | None = None, mode: str = "exact") -> CommLog:
    """scheduler.hpp:109-113 / module.cpp:360-370 on two GPU slabs split at
    plan.boundary; returns the CommLog.  `threaded` is accepted for signature
    parity (one host thread drives both devices; both of the reference's
    drives give the same bits, and so does this one)."""
    return _run_heterogeneous(grid, kernel, int(steps), plan, first, second,
                              model or CommCostModel(), False, mode)


def run_heterogeneous_instrumented(grid: BasicGrid, kernel: StencilKernel, steps: int,
                                   plan: PartitionPlan, first: WorkerSpec, second: WorkerSpec,
                                   threaded: bool = True, *, model: CommCostModel | None = None,
                                   mode: str = "exact") -> CommLog:
    """scheduler.hpp:115-124: NaN in every slab's seam-side halo planes
    (beyond the exchanged ghosts) before stepping, so a read of undelivered
    remote data poisons the result."""
    return _run_heterogeneous(grid, kernel, int(steps), plan, first, second,
                              model or CommCostModel(), True, mode)
