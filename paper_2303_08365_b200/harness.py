"""Benchmark harness of the reference (proj/include/tessera/bench.hpp,
proj/src/bench.cpp:63-312) with the GPU sweep as its executor path.

``run_benchmark(name, path="gpu", scale="desk", threads=1, seed=1, steps=0)``
returns the same dict as the reference binding (proj/bindings/module.cpp:
385-409) plus GPU columns.  As in the reference (bench.cpp:248-260) a row is
first verified at a reduced size, then timed at desk or full scale:

* paths ``gpu`` (engine's fused depth), ``tessellate`` (k = the Table-1 tb,
  clamped like clamp_tb, bench.cpp:104-107) and ``naive`` (k = 1) run on the
  B200; ``hetero`` is the reference's two-worker deep-halo partition
  (bench.cpp:169-189: profile_workers on a <= 64^d sample, plan_partition,
  run_heterogeneous) on two GPU slabs, with its CommLog's message count and
  ghost recompute in the row (``comm_log=`` writes the per-round CSV,
  dump_comm_log); ``vector``/``mm`` are CPU simulators of the reference and
  report ``unsupported``, like its unsupported path/dimension pairings;
* verify compares the tuned engine with the one-thread-per-point generic GPU
  engine (an independent implementation of apply_box; the product never
  calls the CPU oracle) and requires max_rel_deviation <= 1e-12, the
  reference's tolerance;
* ``elapsed_s`` is the wall time of the reference-facing call (host buffers
  in and out, as the reference times execute_path); ``device_s`` is the CUDA
  event time of the same steps run device-resident (DeviceGrid), the sweeps
  alone.
"""
from __future__ import annotations

import time

from .grid import Grid, fill_random
from .kernel import benchmark_table, find_benchmark
from .metrics import deviation, stencils_per_second
from .run import run_gpu

PATHS = ("gpu", "tessellate", "naive", "hetero")
CPU_ONLY = ("vector", "mm")


def clamp_tb(tb: int, min_tile: int, radius: int) -> int:
    """bench.cpp:104-107."""
    return max(1, min(tb, min_tile // (2 * radius)))


def make_setup(spec, scale: str):
    """bench.cpp:192-208 (desk: extents / 20, at least 8)."""
    extent = list(spec.full_extent)
    if scale == "desk":
        extent = [max(e // 20, 8) for e in extent]
    if spec.kernel.dims == 1:
        extent = [(e + 3) // 4 * 4 for e in extent]
    tile = [min(t, e) for t, e in zip(spec.tile, extent)]
    return extent, tile, clamp_tb(spec.tb, min(tile), spec.kernel.radius)


def verify_setup(spec):
    """bench.cpp:210-226."""
    dims, r = spec.kernel.dims, spec.kernel.radius
    extent, tile = {1: ([256], [32]), 2: ([64, 64], [16, 16]), 3: ([24, 24, 24], [8, 8, 8])}[dims]
    return extent, tile, clamp_tb(min(spec.tb, 3), tile[0], r)


def _fused(path: str, tb: int) -> int:
    return {"gpu": 0, "tessellate": tb, "naive": 1, "hetero": tb}[path]


def _hetero(g, k, steps: int, extent, tile, tb: int, mode: str):
    """bench.cpp:169-189 on two GPU slabs: the workers are profiled on a
    sample of at most 64 cells per axis, the plan splits axis 0 on a tile
    multiple, run_heterogeneous advances the grid; returns its CommLog."""
    from .scheduler import (WorkerSpec, plan_partition, profile_workers, run_heterogeneous)
    cpu = WorkerSpec("cpu_like", "tessellate")
    accel = WorkerSpec("accel_like", "mm" if k.dims == 2 else "naive")
    pc, pa = profile_workers(cpu, accel, k, [min(e, 64) for e in extent], 1)
    plan = plan_partition(pc, pa, extent, tile[0], tb, k.radius)
    first, second = (cpu, accel) if plan.first_worker == "cpu_like" else (accel, cpu)
    return run_heterogeneous(g, k, steps, plan, first, second, mode=mode)


def _hbm_peak_gbps() -> float:
    """MEASURED_PEAKS.json's copy bandwidth when present (the roofline
    denominator bench.py uses), else the profiling guide's fallback."""
    import json
    import os
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                        "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"])
    except Exception:
        return 6650.0


def run_benchmark(name: str, path: str = "gpu", scale: str = "desk", threads: int = 1,
                  seed: int = 1, steps: int = 0, mode: str = "exact",
                  verify: bool = True, comm_log: str | None = None) -> dict:
    spec = find_benchmark(name)
    k = spec.kernel
    row = {"name": spec.name, "path": path, "dims": k.dims, "extent": [], "T": 0, "tile": [],
           "Tb": 0, "elapsed_s": 0.0, "stencils_per_s": 0.0, "verify": "skip", "seed": seed,
           "ghost_recompute_points": 0, "mma_calls": 0, "messages": 0,
           "gpus": 1, "k": 0, "device_s": 0.0, "achieved_GBps": 0.0, "roofline_frac": 0.0,
           "max_abs_err": None, "l2_rel_err": None}
    if path in CPU_ONLY:
        row["verify"] = "unsupported"
        return row
    if path not in PATHS:
        raise ValueError(f"unknown executor path: {path}")
    if scale not in ("desk", "full"):
        raise ValueError("scale must be 'desk' or 'full'")

    # verify at the reduced size (T = 6), tuned path vs the generic engine
    if verify:
        vext, _, vtb = verify_setup(spec)
        probe = Grid(vext, [k.radius] * k.dims)
        fill_random(probe, seed)
        check = probe.copy()
        if path == "hetero":
            _hetero(probe, k, 6, vext, verify_setup(spec)[1], vtb, mode)
        else:
            run_gpu(probe, k, 6, fused_steps=_fused(path, vtb), mode=mode)
        run_gpu(check, k, 6, engine="generic")
        d = deviation(probe, check)
        row["verify"] = "pass" if d["max_rel_deviation"] <= 1e-12 else "fail"
        row["max_abs_err"], row["l2_rel_err"] = d["max_abs_err"], d["l2_rel_err"]

    extent, tile, tb = make_setup(spec, scale)
    t_steps = min(spec.full_steps, 1000) if scale == "desk" else spec.full_steps
    if steps > 0:
        t_steps = steps
    row.update(extent=extent, tile=tile, Tb=tb, T=t_steps)
    # warm-up on a small grid: the timed call's kernels (fused and single-step)
    # are loaded by the driver before the clock starts (lazy module loading
    # costs milliseconds per kernel on first launch)
    wext = [min(e, 64) for e in extent]
    warm = Grid(wext, [k.radius] * k.dims)
    run_gpu(warm, k, 2 * max(_fused(path, tb), 1) + 1, fused_steps=_fused(path, tb), mode=mode)
    g = Grid(extent, [k.radius] * k.dims, pinned=True)
    if path != "hetero":
        # and one untimed call of the timed size and length (device cache,
        # chunked round-trip buffers), on the zero grid before it is seeded
        run_gpu(g, k, t_steps, fused_steps=_fused(path, tb), mode=mode)
    fill_random(g, seed)
    if path == "hetero":
        t0 = time.perf_counter()
        log = _hetero(g, k, t_steps, extent, tile, tb, mode)
        elapsed = max(time.perf_counter() - t0, 1e-9)
        rate = stencils_per_second(extent, t_steps, elapsed)
        # the slabs exchange every k = min(tb, engine max) steps: the GPU's
        # deep halo is r*k planes, not r*tb (same bits, more frequent rounds)
        from . import _abi
        _, k_used = _abi.query_plan(k, _abi.grid_desc(extent, [k.radius] * k.dims, "f64"), tb,
                                    mode)
        row.update(elapsed_s=elapsed, stencils_per_s=rate.stencils_per_second, k=k_used, gpus=2,
                   messages=log.messages, ghost_recompute_points=log.ghost_recompute_points,
                   device_s=sum(r.wall_seconds for r in log.records))
        if comm_log:
            from .scheduler import dump_comm_log
            dump_comm_log(comm_log, log)
        return row
    t0 = time.perf_counter()
    st = run_gpu(g, k, t_steps, fused_steps=_fused(path, tb), mode=mode)
    elapsed = max(time.perf_counter() - t0, 1e-9)
    rate = stencils_per_second(extent, t_steps, elapsed)
    # device_s: the same steps device-resident (a short call's run_gpu may
    # take the chunked round trip, whose windows sweep some planes twice)
    dev_s = _device_seconds(g, k, t_steps, st.fused_steps, mode)
    row.update(elapsed_s=elapsed, stencils_per_s=rate.stencils_per_second, k=st.fused_steps,
               device_s=dev_s)
    if dev_s > 0:
        dev_rate = rate.points_per_step * t_steps / dev_s
        row["achieved_GBps"] = dev_rate * 2 * 8 / 1e9
        row["roofline_frac"] = row["achieved_GBps"] / _hbm_peak_gbps()
    return row


def _device_seconds(g, k, steps, fused, mode) -> float:
    """CUDA-event time of `steps` device-resident steps (DeviceGrid,
    tsr_advance) of kernel `k` on grid `g`'s current state, after one
    untimed launch."""
    import torch  # plumbing: device buffers and events
    from .device import DeviceGrid
    dev = torch.device("cuda", torch.cuda.current_device())
    dg = DeviceGrid(g, dev)
    dg.advance(k, max(1, fused), fused_steps=fused, mode=mode)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(dev)
    e0.record()
    dg.advance(k, steps, fused_steps=fused, mode=mode)
    e1.record()
    torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1)
    del dg
    return ms / 1e3


CSV_FIELDS = ("name", "path", "dims", "extent", "T", "tile", "Tb", "elapsed_s",
              "stencils_per_s", "verify", "seed", "ghost_recompute_points", "mma_calls",
              "messages", "gpus", "k", "device_s", "achieved_GBps", "roofline_frac",
              "max_abs_err", "l2_rel_err")


def csv_header() -> str:
    """The reference's 14 columns (bench.cpp:289-292) + the GPU columns."""
    return ",".join(CSV_FIELDS)


def csv_row(row: dict) -> str:
    def fmt(key):
        v = row.get(key)
        if key in ("extent", "tile"):
            return "x".join(str(e) for e in v)
        return "" if v is None else str(v)
    return ",".join(fmt(f) for f in CSV_FIELDS)


def write_csv(path: str, rows) -> None:
    with open(path, "w") as f:
        f.write(csv_header() + "\n")
        for r in rows:
            f.write(csv_row(r) + "\n")


def run_all(path: str = "gpu", scale: str = "desk", seed: int = 1) -> list:
    """Every Table-1 benchmark on one path (the reference CLI's `bench run` loop)."""
    return [run_benchmark(s.name, path=path, scale=scale, seed=seed) for s in benchmark_table()]


def write_csv_file(path: str, rows) -> None:
    """bench.cpp:300-312 name."""
    write_csv(path, rows)
