"""Thermal-diffusion case study (proj/include/tessera/case_study.hpp,
proj/src/case_study.cpp:21-290) on the B200 path.

A square plate with a Gaussian hot spot (peak 100 C) over a 20 C Dirichlet
rim, explicit 5-point heat scheme (mu = 0.23), advanced in FP64 and, as a
precision twin, in FP32; at checkpoints the FP32 field is compared with the
FP64 one (Table-5-style exceedance table).  Both grids stay in HBM for the
whole run; only the centre cell is read back per sample and whole fields
only at checkpoints.  Desk scale is the reference's 480 x 480, 9500 steps;
``apply_full_scale`` is the paper's 9600 x 9600, 3.8e6 steps (PAPER Table 4).

The FP32 twin runs on the GPU in exact mode, which is bitwise the
reference's CPU ``naive_run<float>``, so the error tables are the ones the
reference would print.
"""
from __future__ import annotations

import ctypes
import os
import time
from dataclasses import dataclass, field

import numpy as np

from . import _abi
from .device import DeviceGrid
from .grid import Grid, GridF, dump_grid
from .kernel import heat_coefficients


@dataclass
class ErrorTable:
    """case_study.hpp:16-21."""
    abs_thresholds: tuple = (0.1, 0.5, 1.0)
    rel_thresholds: tuple = (0.01, 0.03, 0.05)
    abs_exceed_pct: list = field(default_factory=lambda: [0.0, 0.0, 0.0])
    rel_exceed_pct: list = field(default_factory=lambda: [0.0, 0.0, 0.0])


def compare_precision(fp64: Grid, other, abs_thresholds=(0.1, 0.5, 1.0),
                      rel_thresholds=(0.01, 0.03, 0.05)) -> ErrorTable:
    """Share of interior points whose |other - fp64| (and relative deviation
    with a 1e-12 floor) exceeds each threshold (case_study.cpp:21-47)."""
    if other.dims != fp64.dims:
        raise ValueError("grid dimensionality mismatch")
    if other.extent != fp64.extent:
        raise ValueError("grid extent mismatch")
    r = fp64.interior_view(fp64.parity).astype(np.float64)
    o = other.interior_view(other.parity).astype(np.float64)
    d = np.abs(o - r)
    rel = d / np.maximum(np.abs(r), 1e-12)
    t = ErrorTable(tuple(abs_thresholds), tuple(rel_thresholds))
    n = r.size
    t.abs_exceed_pct = [100.0 * float(np.count_nonzero(d > a)) / n for a in abs_thresholds]
    t.rel_exceed_pct = [100.0 * float(np.count_nonzero(rel > a)) / n for a in rel_thresholds]
    return t


@dataclass
class CaseStudyConfig:
    """case_study.hpp:31-45 (path is always the GPU here)."""
    plate_side_mm: float = 15.0
    mu: float = 0.23
    extent: int = 480
    steps: int = 9500
    peak_celsius: float = 100.0
    ambient_celsius: float = 20.0
    sigma_cells: float = 0.0  # 0 -> extent / 8
    checkpoints: list = field(default_factory=lambda: [1000, 5000, 9500])
    sample_every: int = 25
    fused_steps: int = 0      # 0 = engine default
    mode: str = "exact"
    snapshot_every: int = 0   # > 0: TTRS snapshots of both fields every N steps (out_dir)


def apply_full_scale(cfg: CaseStudyConfig) -> None:
    """case_study.cpp:118-123: 9600 x 9600, 3.8e6 steps, checkpoints at 1e6,
    2e6 and 3.8e6."""
    cfg.extent = 9600
    cfg.steps = 3_800_000
    cfg.checkpoints = [1_000_000, 2_000_000, 3_800_000]
    cfg.sample_every = 10_000


def parse_case_config(path: str) -> CaseStudyConfig:
    """Line-oriented ``key = value`` config (case_study.cpp:74-116): '#'
    comments, the reference's keys; an unknown key or a line without '='
    raises RuntimeError naming the line.  ``path`` may only name an executor
    this library runs (gpu/naive/tessellate, all on the B200); ``threads`` is
    accepted and ignored (the CUDA grid replaces the worker threads)."""
    cfg = CaseStudyConfig()
    full = False
    try:
        f = open(path)
    except OSError:
        raise RuntimeError(f"cannot open config: {path}") from None
    with f:
        for lineno, line in enumerate(f, 1):
            line = line.split("#", 1)[0].strip()
            if not line:
                continue
            if "=" not in line:
                raise RuntimeError(f"config line {lineno}: expected key = value")
            key, value = (t.strip() for t in line.split("=", 1))
            if key == "extent":
                cfg.extent = int(value)
            elif key == "steps":
                cfg.steps = int(value)
            elif key == "mu":
                cfg.mu = float(value)
            elif key == "peak":
                cfg.peak_celsius = float(value)
            elif key == "ambient":
                cfg.ambient_celsius = float(value)
            elif key == "sigma":
                cfg.sigma_cells = float(value)
            elif key == "plate_side_mm":
                cfg.plate_side_mm = float(value)
            elif key == "path":
                if value not in ("gpu", "naive", "tessellate"):
                    raise ValueError(f"unsupported executor path on the GPU library: {value}")
            elif key == "threads":
                int(value)
            elif key == "sample_every":
                cfg.sample_every = int(value)
            elif key == "full":
                full = value in ("1", "true")
            elif key == "checkpoints":
                cfg.checkpoints = [int(t.strip()) for t in value.split(",")]
            elif key in ("fused_steps", "mode"):  # GPU extensions
                setattr(cfg, key, int(value) if key == "fused_steps" else value)
            else:
                raise RuntimeError(f"config line {lineno}: unknown key '{key}'")
    if full:
        apply_full_scale(cfg)
    heat_coefficients(cfg.mu)  # rejects an unstable CFL number here
    return cfg


def _init(grid, cfg: CaseStudyConfig, sigma: float) -> None:
    """Interior Gaussian over a cold-ambient Dirichlet rim, both buffers
    (case_study.cpp:193-207), evaluated by the engine library's host code
    with std::exp in double and cast to the grid type, as the reference does
    (tsr_fill_plate), so the initial fields are bit-identical to its own."""
    b0, b1 = grid.c_buffers()
    _abi.check(_abi.lib().tsr_fill_plate(ctypes.byref(grid.c_struct()), b0, b1,
                                         float(cfg.ambient_celsius), float(cfg.peak_celsius),
                                         float(sigma)))


def _snapshot_paths(out_dir: str, step: int):
    return (os.path.join(out_dir, f"snapshot_{step}_fp64.ttrs"),
            os.path.join(out_dir, f"snapshot_{step}_fp32.ttrs"))


def case_study_heat(cfg: CaseStudyConfig, out_dir: str | None = None, device=None,
                    resume_step: int | None = None) -> dict:
    """Runs the study; writes center_series.csv, error_table.csv,
    metadata.txt and final.ttrs into `out_dir` when given.

    Long runs (the paper's 3.8e6 steps) checkpoint with
    ``cfg.snapshot_every``: both device fields go to out_dir as TTRS dumps
    (snapshot_<step>_fp64.ttrs / _fp32.ttrs, the reference's grid_io format)
    without leaving HBM; ``resume_step`` restarts from those files and
    produces the rest of the series, tables and artifacts exactly as the
    uninterrupted run does."""
    import torch
    if cfg.extent < 16:
        raise ValueError("plate extent too small")
    if cfg.steps < 0:
        raise ValueError("negative step count")
    for c in cfg.checkpoints:
        if c > cfg.steps:
            raise ValueError("checkpoint beyond the final step")
        if c % cfg.sample_every != 0 and c != cfg.steps:
            raise ValueError("checkpoint must fall on the sampling stride")
    kernel = heat_coefficients(cfg.mu)
    sigma = cfg.sigma_cells if cfg.sigma_cells > 0 else cfg.extent / 8.0
    n = cfg.extent
    fp64 = Grid([n, n], [1, 1])
    fp32 = GridF([n, n], [1, 1])
    _init(fp64, cfg, sigma)
    _init(fp32, cfg, sigma)
    dev = torch.device(device if device is not None else "cuda")
    if resume_step is not None:
        if out_dir is None or cfg.snapshot_every <= 0 or resume_step % cfg.snapshot_every:
            raise ValueError("resume needs out_dir and a step on the snapshot stride")
        if resume_step % cfg.sample_every or resume_step > cfg.steps:
            raise ValueError("resume step must fall on the sampling stride")
        p64, p32 = _snapshot_paths(out_dir, resume_step)
        d64 = DeviceGrid.resume(p64, dev, "f64")
        d32 = DeviceGrid.resume(p32, dev, "f32")
    else:
        d64 = DeviceGrid(fp64, dev)
        d32 = DeviceGrid(fp32, dev)
    center = n // 2

    def center_of(dg: DeviceGrid) -> float:
        e = dg.layout.origin + center * dg.layout.pitch[0] + center
        return float(dg.buf[dg.cur][e].item())

    done = 0 if resume_step is None else int(resume_step)
    res = {"series_steps": [done],
           "center_series": [float(fp64.at(center, center)) if resume_step is None
                             else center_of(d64)],
           "checkpoint_steps": [], "checkpoint_errors": [], "artifacts": []}
    t64 = t32 = 0.0
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    while done < cfg.steps:
        chunk = min(cfg.sample_every, cfg.steps - done)
        ev[0].record()
        d64.advance(kernel, chunk, fused_steps=cfg.fused_steps, mode=cfg.mode)
        ev[1].record()
        d32.advance(kernel, chunk, fused_steps=cfg.fused_steps, mode=cfg.mode)
        ev[2].record()
        done += chunk
        res["series_steps"].append(done)
        res["center_series"].append(center_of(d64))  # synchronises
        t64 += ev[0].elapsed_time(ev[1]) / 1e3
        t32 += ev[1].elapsed_time(ev[2]) / 1e3
        if out_dir and cfg.snapshot_every > 0 and done % cfg.snapshot_every == 0:
            os.makedirs(out_dir, exist_ok=True)
            p64, p32 = _snapshot_paths(out_dir, done)
            d64.snapshot(p64)
            d32.snapshot(p32)
            res["artifacts"] += [p64, p32]
        if done in cfg.checkpoints:
            h64, h32 = Grid([n, n], [1, 1]), GridF([n, n], [1, 1])
            _init(h64, cfg, sigma)
            _init(h32, cfg, sigma)
            d64.download(h64)
            d32.download(h32)
            d64.steps_done = d32.steps_done = 0  # keep stepping from the device state
            res["checkpoint_steps"].append(done)
            res["checkpoint_errors"].append(compare_precision(h64, h32))
            fp64, fp32 = h64, h32
    res["final_center"] = res["center_series"][-1]
    pts = n * n * (cfg.steps - (resume_step or 0))
    res["fp64_device_s"] = t64
    res["fp32_device_s"] = t32
    res["fp64_gstencil_s"] = pts / t64 / 1e9 if t64 > 0 else 0.0
    res["fp32_gstencil_s"] = pts / t32 / 1e9 if t32 > 0 else 0.0
    if out_dir:
        os.makedirs(out_dir, exist_ok=True)
        # the final fp64 field, always (case_study.cpp:241-242)
        if not res["checkpoint_steps"] or res["checkpoint_steps"][-1] != done:
            final = Grid([n, n], [1, 1])
            _init(final, cfg, sigma)
            d64.download(final)
            fp64 = final
        dump_grid(os.path.join(out_dir, "final.ttrs"), fp64)
        res["artifacts"].append(os.path.join(out_dir, "final.ttrs"))
        # the reference's CSV headers and C++ ostream number format (%g)
        with open(os.path.join(out_dir, "center_series.csv"), "w") as f:
            f.write("step,center_c\n")
            for s, c in zip(res["series_steps"], res["center_series"]):
                f.write(f"{s},{c:g}\n")
        with open(os.path.join(out_dir, "error_table.csv"), "w") as f:
            f.write("T,abs_gt_0.1,abs_gt_0.5,abs_gt_1.0,rel_gt_1pct,rel_gt_3pct,rel_gt_5pct\n")
            for s, t in zip(res["checkpoint_steps"], res["checkpoint_errors"]):
                f.write(f"{s}," + ",".join(f"{v:g}" for v in t.abs_exceed_pct + t.rel_exceed_pct)
                        + "\n")
        with open(os.path.join(out_dir, "metadata.txt"), "w") as f:
            f.write(f"plate_side_mm = {cfg.plate_side_mm:g}\nmu = {cfg.mu:g}\n"
                    f"extent = {n}x{n}\nsteps = {cfg.steps}\ninitial = gaussian\n"
                    f"gaussian_peak_c = {cfg.peak_celsius:g}\n"
                    f"gaussian_sigma_cells = {sigma:g}\n"
                    f"ambient_c = {cfg.ambient_celsius:g}\nboundary = dirichlet ambient\n"
                    f"path = gpu ({cfg.mode} mode, fused_steps {cfg.fused_steps or 'auto'})\n"
                    f"fp32_twin = B200 exact mode (bitwise the reference executor's "
                    f"32-bit arithmetic)\n"
                    f"final_center_c = {res['final_center']!r}\n"
                    f"fp64_device_s = {t64:.3f}\nfp32_device_s = {t32:.3f}\n"
                    f"fp64_gstencil_s = {res['fp64_gstencil_s']:.2f}\n"
                    f"fp32_gstencil_s = {res['fp32_gstencil_s']:.2f}\n")
        res["artifacts"] += [os.path.join(out_dir, x) for x in
                             ("center_series.csv", "error_table.csv", "metadata.txt")]
    return res
