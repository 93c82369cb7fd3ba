"""Benchmark of the Jacobi stencil sweep on B200 (driver contract: one JSON line).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c1..c5]
                    [--impl ours|reference] [--fused k] [--mode exact|fast]

Default workload (N=1): BASELINE config C3, the north star's headline target —
Heat-3D 7-point star fp64, 512^3 interior, halo 1, fill_random(seed=1), 1000
time steps.  A "step" is one time step over the whole grid.

N>1 (`--gpus N`, with or without torchrun): the global grid is split along
axis 0 into N slabs, one per GPU, driven by ONE host thread through the C++
slab runtime behind the C-ABI (tsr_multi_*, csrc/multi.cu) — the reference's
own design of one host thread per box.  Weak scaling for the
Heat-3D configs (each GPU owns a 512^3 or 1024^3 slab of a (n*N) x n x n
grid), strong scaling for C4 (1024^3 global).  Every k fused steps each slab
runs its r*k seam planes on one stream, storing every row locally AND into
the neighbour's ghost planes over NVLink peer memory, while its interior runs
on a second stream.  The whole global grid is seeded from ONE fill_random
stream, and after the timed run the per-plane checksums of the slab run are
compared bitwise with a one-GPU run of the same global grid (`parity`).
Under torchrun, ranks > 0 only join the rendezvous (the devices are driven
from rank 0); `--runtime ranks` instead runs one process per GPU with the
torch.distributed slab runner (partition.py).

Arithmetic: Heat-2D/Heat-3D (C1, C3, C5) time FAST mode — one fp64 FMA per
tap in apply_box's order, admitted by the north star within 1e-12 — and every
N=1 line carries `modes`: the EXACT mode (mul + add per tap, bitwise
naive_run) timed on the same input, plus the full-grid max_rel_deviation and
a bitwise flag between the two.  Heat-3D's weights (1/4, 1/8) are powers of
two, so its products are exact and FAST is bitwise EXACT on normal-range data
(the flag shows it).  The box kernels' FAST mode is the separable box sum
(row, column and plane sums times the one weight: C4 8 operations per update
at two fused steps per pass, C2 4.5 instead of Q mode's 9), reported with its
max_rel_deviation from EXACT (<= 1e-5 fp32, <= 1e-12 fp64).

`value` is device-resident throughput (GStencil/s = points * K / time, the
reference's Eq. 6, proj/src/metrics.cpp:8-20), timed with CUDA events on the
streams the sweeps launch on (max over devices).  At N=1 the K timed steps
are captured once into a CUDA graph and replayed between the two events, so
the device is not left waiting on the Python launch path between fused
passes (--no-graph times the launches directly).  `e2e` is the same metric
through the reference-facing call on host buffers in pinned memory (naive_run
-> tsr_run at N=1, tsr_run_multi at N>1): H2D of the read buffer + K steps +
D2H of both buffers.  `--impl reference` times the reference's own CPU path
(oracle/_ref: the unmodified reference sources, run_tessellated with all host
threads) and never loads the product library.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "GStencil/s (fp64) at 1/2/4/8 B200 and % of HBM roofline vs host-CPU ref"
DATA = "synthetic: fill_random(seed=1) U[0,1) interior, zero Dirichlet halo"

CONFIGS = {
    "c1": dict(bench="Heat-2D", extent=[4096, 4096], dtype="f64", steps=100, fused=6,
               mode="fast", workload="C1: 2D heat 5-point star fp64, 4096x4096, 100 timesteps",
               ref_tile=[200, 200], ref_tb=50),
    "c2": dict(bench="Box-2D9P", extent=[16384, 16384], dtype="f64", steps=100, fused=4,
               mode="fast",
               workload="C2: 2D 9-point box fp64, 16384x16384, temporal blocking k=4",
               ref_tile=[2000, 2000], ref_tb=4),
    "c3": dict(bench="Heat-3D", extent=[512, 512, 512], dtype="f64", steps=1000, fused=0,
               mode="fast",
               workload="C3: 3D heat 7-point star fp64, 512^3 per GPU, 1000 timesteps",
               ref_tile=[20, 20, 20], ref_tb=10),
    "c4": dict(bench="Box-3D27P", extent=[1024, 1024, 1024], dtype="f32", steps=100, fused=0,
               mode="fast", strong=True,
               workload="C4: 3D 27-point box fp32, 1024^3 global, slab-partitioned over N GPUs "
                        "(strong scaling), fast mode (separable box sums, within 1e-5)",
               ref_tile=None, ref_tb=None),
    "c5": dict(bench="Heat-3D", extent=[1024, 1024, 1024], dtype="f64", steps=100, fused=0,
               mode="fast", workload="C5: 3D heat 7-point fp64, 1024^3 per GPU (weak scaling)",
               ref_tile=[20, 20, 20], ref_tb=10),
}

HBM_FALLBACK_GBPS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return HBM_FALLBACK_GBPS, "fallback"


# Nominal FP64 / FP32 peaks (148 SMs x 64 FMA lanes x 2 flops x 1.965 GHz; FP32 2x)
# when profiles/fp_peaks.json (tools/microbench/fp64_peak.cu on a B200) is absent.
FP_FALLBACK_TFLOPS = {"f64": 37.2, "f32": 74.4}


def fp_peak(dtype: str):
    """Measured FMA throughput of the pool's B200 (ops/s x 2 flops), best over
    occupancies, from the committed microbenchmark output."""
    try:
        with open(os.path.join(ROOT, "profiles", "fp_peaks.json")) as f:
            d = json.load(f)
        key = "dfma" if dtype == "f64" else "ffma"
        return 2 * max(d["throughput_ops_per_s"][key].values()) / 1e12, "measured"
    except Exception:
        return FP_FALLBACK_TFLOPS[dtype], "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons of the GPUs in use during the
    timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, indices):
        self.indices = [int(i) for i in indices]
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-i", ",".join(map(str, self.indices)), "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except Exception:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        self.proc.wait()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(n)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": sorted(reasons),
                "samples": len(sm), "gpus": self.indices}


# ---------------------------------------------------------------------------
# workload description shared by both arms
# ---------------------------------------------------------------------------

def extents(cfg, n: int):
    """(per-GPU extent, global extent) at n GPUs: weak scaling stacks n
    per-GPU grids along axis 0; C4 (strong) splits its fixed global grid."""
    if cfg.get("strong"):
        glob = list(cfg["extent"])
        per = [glob[0] // n] + glob[1:]
    else:
        per = list(cfg["extent"])
        glob = [per[0] * n] + per[1:]
    return per, glob


def npoints(extent) -> int:
    p = 1
    for e in extent:
        p *= int(e)
    return p


def cfg_scaling(cfg) -> str:
    return "strong" if cfg.get("strong") else "weak"


def bench_config(cfg, n: int, mode: str | None = None) -> dict:
    """The `config` object both arms print (static: no run-time plan keys)."""
    per, glob = extents(cfg, n)
    esize = 8 if cfg["dtype"] == "f64" else 4
    return {"workload": cfg["workload"], "kernel": cfg["bench"], "extent_per_gpu": per,
            "global_extent": glob, "mode": mode or cfg["mode"],
            "parallelism": f"slab{n}" if n > 1 else "single",
            "l2": (f"no flush: the two buffers ({2 * esize * npoints(per) / 1e9:.2f} GB per GPU)"
                   " exceed the 126 MB L2")}


def fused_groups(steps: int, k: int) -> list[int]:
    out = []
    while steps > 0:
        out.append(min(k, steps))
        steps -= out[-1]
    return out


def ncu_traffic(cfg_name: str, kfused: int):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the dominant
    kernel, from the committed ncu launch list of this bench command
    (profiles/ncu_traffic.json, written by tools/launch_summary.py --traffic).
    The entry names the capture it came from; a capture at another fused depth
    is reported as missing (null), never substituted."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f).get(cfg_name)
        if d and d.get("fused_steps") == kfused:
            return d
    except Exception:
        pass
    return None


# ---------------------------------------------------------------------------
# the reference's CPU path (oracle/_ref): cpu_baseline leg and --impl reference
# ---------------------------------------------------------------------------

def _ref_grid(ref, cfg, extent, seed=1):
    """A host grid in the reference's layout filled by the reference's own
    fill_random (random.hpp:20-24) through oracle/_ref: the reference arm and
    the cpu_baseline leg never load the product library."""
    import numpy as np
    import oracle
    g = oracle.HostGrid(extent, [1] * len(extent),
                        np.float64 if cfg["dtype"] == "f64" else np.float32)
    ref.fill_random(g, seed)
    return g


def _ref_sample(cfg, n: int = 1):
    """Per-step sample of the reference's CPU path: one GPU's share of the
    grid for the fp64 configs (run_tessellated with the Table-1 tile and tb,
    all host threads); a 64-plane slab of the full cross-section for C4,
    whose fp32 path in the reference is the single-threaded naive_run<float>
    (it has no threaded fp32 path)."""
    per, _ = extents(cfg, n)
    if cfg["dtype"] == "f64":
        return per, "tessellate"
    return [64] + per[1:], "naive"


def _ref_steps(ref, cfg, g, kernel, steps, threads):
    """Advances g `steps` steps on the reference's path; returns seconds."""
    if steps <= 0:
        return 0.0
    if cfg["dtype"] == "f64":
        _, sec = ref.run_tessellated(g, kernel, steps, cfg["ref_tile"], cfg["ref_tb"], threads)
        return sec
    return ref.time_naive_f32(g, kernel, steps)


def _ref_what(cfg, path, threads):
    if path == "tessellate":
        return (f"reference run_tessellated(tile={cfg['ref_tile']}, tb={cfg['ref_tb']}, "
                f"threads={threads})")
    return "reference naive_run<float> (1 thread: the reference has no threaded fp32 path)"


def cpu_baseline(cfg, n: int = 1, budget_s: float = 12.0):
    """The reference's own CPU path on this host (oracle/_ref) on a bounded
    sample of about `budget_s` seconds (whole tb rounds)."""
    import oracle
    if not oracle.Reference.available():
        return None
    ref = oracle.Reference()
    kernel = oracle.RefKernel(ref, cfg["bench"])
    extent, path = _ref_sample(cfg, n)
    threads = (os.cpu_count() or 1) if path == "tessellate" else 1
    unit = cfg["ref_tb"] if path == "tessellate" else 1
    g = _ref_grid(ref, cfg, extent)
    sec = _ref_steps(ref, cfg, g, kernel, unit, threads)
    steps = unit
    if sec < budget_s / 2:
        more = unit * max(1, min(100, round((budget_s - sec) / max(sec, 1e-3))))
        sec += _ref_steps(ref, cfg, g, kernel, more, threads)
        steps += more
    return {"value": round(g.interior_points() * steps / sec / 1e9, 4), "unit": "GStencil/s",
            "cores": threads, "kind": "reference",
            "sample": (f"{_ref_what(cfg, path, threads)} on a {'x'.join(map(str, extent))} "
                       f"grid{' (one GPU share)' if n > 1 else ''}, T={steps} ({sec:.1f} s)")}


def run_reference_arm(args, cfg):
    """`--impl reference`: the reference's own CPU path (oracle/_ref, the
    unmodified proj/src sources) on this host, rank 0 only.  W untimed steps,
    then exactly K timed steps; a step is one time step over one GPU's share
    of the grid (C1, C2, C3, C5: run_tessellated, all host threads) or over a
    64-plane slab of the cross-section (C4: naive_run<float>, 1 thread)."""
    import oracle
    if int(os.environ.get("RANK", "0")) != 0:
        return
    if not oracle.Reference.available():
        print(json.dumps({"impl": "reference", "unavailable":
                          "oracle/_ref/libtessera_ref.so not built (make -C oracle ref)"}))
        return
    ref = oracle.Reference()
    kernel = oracle.RefKernel(ref, cfg["bench"])
    extent, path = _ref_sample(cfg, args.gpus)
    threads = (os.cpu_count() or 1) if path == "tessellate" else 1
    # run_tessellated runs T mod tb trailing steps as plain single-threaded
    # sweeps (tiling.cpp:177-183): K is rounded up to whole tb rounds so the
    # timed steps are the reference's tessellated path, and `steps` reports
    # the count actually timed.
    unit = cfg["ref_tb"] if path == "tessellate" else 1
    steps = -(-args.steps // unit) * unit
    g = _ref_grid(ref, cfg, extent)
    _ref_steps(ref, cfg, g, kernel, args.warmup, threads)
    sec = _ref_steps(ref, cfg, g, kernel, steps, threads)
    value = round(g.interior_points() * steps / sec / 1e9, 4)
    sample = (f"{_ref_what(cfg, path, threads)} on a {'x'.join(map(str, extent))} grid: "
              f"{args.warmup} untimed + {steps} timed steps ({sec:.2f} s)")
    print(json.dumps({
        "metric": METRIC, "impl": "reference", "value": value, "unit": "GStencil/s",
        "n_gpus": args.gpus, "steps": steps, "steps_requested": args.steps,
        "warmup": args.warmup, "ms_per_step": round(sec * 1e3 / steps, 4),
        "higher_is_better": True,
        "scaling": cfg_scaling(cfg), "vs_baseline": None, "dtype": cfg["dtype"], "data": DATA,
        "config": bench_config(cfg, args.gpus, args.mode),
        "cpu_baseline": {"value": value, "unit": "GStencil/s", "cores": threads,
                         "kind": "reference", "sample": sample},
        "e2e": {"value": value, "unit": "GStencil/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0}}))


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def make_grid(ts, cfg, extent, pinned=False, seed=1):
    cls = ts.Grid if cfg["dtype"] == "f64" else ts.GridF
    g = cls(extent, [1] * len(extent), pinned=pinned)
    ts.fill_random(g, seed)
    return g


def mode_check(ts, torch, cfg, k, host, state, per_gpu, dev, stream, kfused, mode, args,
               total_points, elapsed_ms):
    """The other arithmetic mode on the same input and step count, timed the
    same way, and its full-grid deviation from the timed run (max_rel_deviation,
    metrics.cpp:28-39, and a bitwise flag).  EXACT is apply_box's mul + add
    per tap (bitwise naive_run); FAST contracts them into one FMA, which the
    north star admits within 1e-12 (fp64) / 1e-5 (fp32)."""
    other = "fast" if mode == "exact" else "exact"
    st2 = ts.DeviceGrid(host, dev)
    st2.advance(k, 1, fused_steps=kfused, mode=other)  # the timed run's probe step
    for n in fused_groups(args.warmup, kfused):
        st2.advance(k, n, fused_steps=kfused, mode=other)
    torch.cuda.synchronize(dev)
    groups = fused_groups(args.steps, kfused)
    graph = None
    if not args.no_graph:
        try:
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, capture_error_mode="relaxed"):
                for n in groups:
                    st2.advance(k, n, fused_steps=kfused, mode=other)
        except Exception:
            return None  # (the timed run fell back too)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    if graph is not None:
        graph.replay()
    else:
        for n in groups:
            st2.advance(k, n, fused_steps=kfused, mode=other)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    ms2 = e0.elapsed_time(e1)
    ext3 = [1] * (3 - len(per_gpu)) + list(per_gpu)

    def interior(s):
        lay = s.layout
        return s.buf[s.cur].as_strided(ext3, (lay.pitch[0], lay.pitch[1], 1), lay.origin)

    a, b = interior(state), interior(st2)
    ref = a if mode == "exact" else b
    dev_max = float((a.double() - b.double()).abs().max())
    rel = dev_max / max(1.0, float(ref.double().abs().max()))
    ival = torch.int64 if a.dtype == torch.float64 else torch.int32
    bitwise = bool(torch.equal(a.view(ival), b.view(ival)))
    out = {mode: {"value": round(total_points * args.steps / (elapsed_ms / 1e3) / 1e9, 3)},
           other: {"value": round(total_points * args.steps / (ms2 / 1e3) / 1e9, 3)},
           "fast_vs_exact": {"max_rel_deviation": rel, "bitwise_equal": bitwise,
                             "tolerance": 1e-12 if cfg["dtype"] == "f64" else 1e-5,
                             "grid": "full interior after warmup + steps"}}
    del st2
    return out


def roofline(cfg, cfg_name, k, points_per_gpu, kfused, launch_ms, basis_what):
    esize = 8 if cfg["dtype"] == "f64" else 4
    peak, peak_kind = peaks()
    # Algorithmic bytes of one fused pass on one GPU: 2*sizeof(T) per stencil
    # update (one compulsory read + one write per step), times
    # the k steps the pass advances ("HBM-equivalent" for k > 1).
    alg_bytes = 2 * esize * points_per_gpu * kfused
    achieved = alg_bytes / (launch_ms / 1e3) / 1e9
    traffic = ncu_traffic(cfg_name, kfused)
    # Arithmetic roofline: the reference's apply_box does one multiply and one
    # add per tap (naive.hpp:75-78), i.e. 2 * taps algorithmic flops per update.
    ntaps = len(k.tap_list())
    fpk, fpk_kind = fp_peak(cfg["dtype"])
    arith_tflops = 2 * ntaps * points_per_gpu * kfused / (launch_ms / 1e3) / 1e12
    roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
            "frac": round(achieved / peak, 4),
            "traffic": traffic["bytes_per_launch"] if traffic else None,
            "traffic_source": (f"ncu launch list profiles/{traffic['source']} "
                               f"({traffic['kernel']})") if traffic else
            f"no committed ncu capture of {cfg_name} at k={kfused}",
            "peak_source": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)"
            if peak_kind == "measured" else "fallback (B200_PROFILING.md)",
            "basis": (f"algorithmic {2 * esize} B per stencil update x {kfused} fused steps x "
                      f"{points_per_gpu} points / {basis_what} {launch_ms:.4f} ms")}
    arith = {"bound": "fp64" if cfg["dtype"] == "f64" else "fp32",
             "achieved": round(arith_tflops, 2), "peak": round(fpk, 2), "unit": "TFLOP/s",
             "frac": round(arith_tflops / fpk, 4),
             "basis": (f"algorithmic {2 * ntaps} flops per update ({ntaps} taps x mul+add,"
                       f" apply_box) x {kfused} fused steps / {basis_what}"),
             "peak_source": ("measured FMA rate x 2 (profiles/fp_peaks.json, "
                             "tools/microbench/fp64_peak.cu)") if fpk_kind == "measured"
             else "nominal 148 SM x 64 FMA x 2 x 1.965 GHz (fp32 2x)"}
    return roof, arith


def base_line(args, cfg, n, mode, value, elapsed_ms):
    return {"metric": METRIC, "value": round(value, 3), "unit": "GStencil/s", "n_gpus": n,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(elapsed_ms / args.steps, 5), "higher_is_better": True,
            "scaling": cfg_scaling(cfg), "vs_baseline": None, "dtype": cfg["dtype"],
            "data": DATA, "config": bench_config(cfg, n, mode)}


def pcie_bound(torch, dev, h2d_bytes, d2h_bytes, device_s, wall_s, updates):
    """PCIe floors of one tsr_run call from its host<->device bytes at the
    pinned-copy rates measured here (256 MiB copies, best of 3, CUDA events)
    and the device-resident time of the same steps; frac = floor / wall."""
    n = 256 << 20
    host = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    devb = torch.empty(n, dtype=torch.uint8, device=dev)
    rates = {}
    for name, dst, src in (("h2d", devb, host), ("d2h", host, devb)):
        best = None
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            dst.copy_(src, non_blocking=True)
            e1.record()
            torch.cuda.synchronize(dev)
            ms = e0.elapsed_time(e1)
            best = ms if best is None else min(best, ms)
        rates[name] = n / (best / 1e3) / 1e9
    del host, devb
    up, down = h2d_bytes / (rates["h2d"] * 1e9), d2h_bytes / (rates["d2h"] * 1e9)
    serial = up + down + device_s
    duplex = max(up, down, device_s)
    return {"h2d_gbs": round(rates["h2d"], 2), "d2h_gbs": round(rates["d2h"], 2),
            "floor_serial_s": round(serial, 4), "floor_duplex_s": round(duplex, 4),
            "frac_serial": round(serial / wall_s, 4), "frac_duplex": round(duplex / wall_s, 4),
            "bound_value_duplex": round(updates / duplex / 1e9, 3),
            "basis": "per-call bytes at the pinned-copy rates measured here (one direction at a "
                     "time) and the device time of the same steps (timed region above); serial = "
                     "upload + sweeps + download back to back (the whole-grid round trip), "
                     "duplex = both directions and the sweeps fully overlapped (the ideal of the "
                     "chunked round trip)"}


def guarded(fn, what):
    """Runs one optional leg of the line (e2e, cpu_baseline); a failure there
    is reported in the line instead of losing the measured value."""
    try:
        return fn()
    except Exception as e:  # noqa: BLE001 - reported, not swallowed
        import traceback
        traceback.print_exc(file=sys.stderr)
        return {"value": None, "error": f"{what}: {type(e).__name__}: {e}"[:300]}


def single_e2e(ts, torch, cfg, k, per_gpu, kfused, mode, args, dev, elapsed_ms, points):
    """The metric through run_gpu on pinned host buffers: one untimed call of
    the same length sizes tsr_run's device cache, then the median of three
    timed calls (each continues the last)."""
    hg = make_grid(ts, cfg, per_gpu, pinned=True)
    ts.run_gpu(hg, k, args.steps, fused_steps=kfused, mode=mode)
    walls = []
    for _ in range(3):
        t0 = time.perf_counter()
        st = ts.run_gpu(hg, k, args.steps, fused_steps=kfused, mode=mode)
        walls.append(time.perf_counter() - t0)
    wall = statistics.median(walls)
    del hg
    return {"value": round(points * args.steps / wall / 1e9, 3), "unit": "GStencil/s",
            "h2d_bytes_per_step": round(st.h2d_bytes / args.steps, 1),
            "d2h_bytes_per_step": round(st.d2h_bytes / args.steps, 1),
            "call": "paper_2303_08365_b200.run_gpu(pinned Grid) -> tsr_run",
            "wall_s": round(wall, 4), "walls_s": [round(w, 4) for w in walls],
            "timing": "median of 3 calls after one untimed call of the same length",
            "pcie": pcie_bound(torch, dev, st.h2d_bytes, st.d2h_bytes,
                               elapsed_ms / 1e3, wall, points * args.steps)}


def run_single(args, cfg):
    """N = 1: DeviceGrid (tsr_advance) on cuda:0, CUDA events per fused pass."""
    import torch
    import paper_2303_08365_b200 as ts
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    mode = args.mode or cfg["mode"]
    fused_req = cfg["fused"] if args.fused is None else args.fused
    k = ts.find_benchmark(cfg["bench"]).kernel
    per_gpu, _ = extents(cfg, 1)
    points = npoints(per_gpu)
    stream = torch.cuda.current_stream(dev)

    host = make_grid(ts, cfg, per_gpu)
    state = ts.DeviceGrid(host, dev)
    probe = state.advance(k, 1, fused_steps=fused_req, mode=mode)  # resolves the plan
    kfused, engine = probe.fused_steps, probe.engine
    groups = fused_groups(args.steps, kfused)
    for n in fused_groups(args.warmup, kfused):
        state.advance(k, n, fused_steps=kfused, mode=mode)
    torch.cuda.synchronize(dev)

    # The K timed steps are captured once into a CUDA graph and replayed
    # between two events: the device runs the launches back to back instead
    # of waiting on Python/ctypes per launch (tens of microseconds, the size
    # of a C1 launch).  The per-launch events of the direct path remain the
    # fallback (--no-graph, or a capture the driver refuses).
    graph, launches = None, 0
    if not args.no_graph:
        try:
            graph = torch.cuda.CUDAGraph()
            torch.cuda.synchronize(dev)
            with torch.cuda.graph(graph, capture_error_mode="relaxed"):
                for n in groups:
                    launches += state.advance(k, n, fused_steps=kfused, mode=mode).kernel_launches
        except Exception as e:  # the state advanced on paper only: rebuild it
            print(f"graph capture unavailable ({e}); timing direct launches", file=sys.stderr)
            graph, launches = None, 0
            state = ts.DeviceGrid(host, dev)
            state.advance(k, 1, fused_steps=kfused, mode=mode)
            for n in fused_groups(args.warmup, kfused):
                state.advance(k, n, fused_steps=kfused, mode=mode)
    sampler = ClockSampler([0])
    sampler.start()
    torch.cuda.synchronize(dev)
    if graph is not None:
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record(stream)
        graph.replay()
        ev[1].record(stream)
        torch.cuda.synchronize(dev)
        clocks = sampler.stop()
        elapsed_ms = ev[0].elapsed_time(ev[1])
        launch_ms = elapsed_ms * kfused / args.steps
        basis = "device time per k steps (CUDA-graph replay of the K steps)"
    else:
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(groups) + 1)]
        ev[0].record(stream)
        for i, n in enumerate(groups):
            st = state.advance(k, n, fused_steps=kfused, mode=mode)
            launches += st.kernel_launches
            ev[i + 1].record(stream)
        torch.cuda.synchronize(dev)
        clocks = sampler.stop()
        elapsed_ms = ev[0].elapsed_time(ev[-1])
        full = [ev[i].elapsed_time(ev[i + 1]) for i, n in enumerate(groups) if n == kfused]
        launch_ms = statistics.mean(full) if full else elapsed_ms / max(1, len(groups))
        basis = "mean CUDA-event launch time"
    value = points * args.steps / (elapsed_ms / 1e3) / 1e9
    roof, arith = roofline(cfg, args.config, k, points, kfused, launch_ms, basis)

    modes = None
    if not args.no_mode_check:
        modes = guarded(lambda: mode_check(ts, torch, cfg, k, host, state, per_gpu, dev, stream,
                                           kfused, mode, args, points, elapsed_ms), "modes")
    del state
    e2e = None
    if not args.no_e2e:
        e2e = guarded(lambda: single_e2e(ts, torch, cfg, k, per_gpu, kfused, mode, args, dev,
                                         elapsed_ms, points), "e2e")
    cpu = None if args.no_cpu else guarded(lambda: cpu_baseline(cfg, 1), "cpu_baseline")
    line = base_line(args, cfg, 1, mode, value, elapsed_ms)
    line.update({"plan": {"fused_steps": kfused,
                          "engine": {1: "generic", 2: "tuned"}.get(engine, str(engine)),
                          "launch": "cuda-graph replay" if graph is not None else "direct"},
                 "roofline": roof, "arith": arith, "modes": modes, "cpu_baseline": cpu,
                 "e2e": e2e, "gpu_launches": launches, "clocks": clocks})
    return line


def run_slabs(args, cfg, n):
    """N > 1 from one host thread: SlabGrid (tsr_multi_*) over devices
    0..n-1, seeded from the global fill_random stream, then the in-run
    bitwise check against a one-GPU run of the same global grid."""
    import torch
    import paper_2303_08365_b200 as ts
    ndev = torch.cuda.device_count()
    if ndev < n and not args.share_devices:
        raise SystemExit(f"--gpus {n} but only {ndev} CUDA devices are visible "
                         "(--share-devices maps slabs onto them round-robin)")
    devices = [i % max(1, ndev) for i in range(n)]
    mode = args.mode or cfg["mode"]
    fused_req = cfg["fused"] if args.fused is None else args.fused
    k = ts.find_benchmark(cfg["bench"]).kernel
    per_gpu, glob = extents(cfg, n)
    points_glob = npoints(glob)
    esize = 8 if cfg["dtype"] == "f64" else 4

    sg = ts.SlabGrid(k, glob, dtype=cfg["dtype"], ngpus=n, devices=devices,
                     fused_steps=fused_req, mode=mode)
    sg.fill_random(1)
    st = sg.advance(args.warmup)
    kfused = st.fused_steps
    sampler = ClockSampler(sorted(set(devices)))
    sampler.start()
    st = sg.advance(args.steps)  # synchronises every device on both sides
    clocks = sampler.stop()
    elapsed_ms = st.device_ms
    launches = st.kernel_launches
    comm = {"transport": {1: "peer-mirror", 2: "peer-copy"}.get(st.transport, st.transport),
            "messages": st.messages, "bytes_exchanged": st.bytes_exchanged,
            "ghost_recompute_points": st.ghost_recompute_points, "rounds": st.rounds,
            "trailing_steps": st.trailing_steps, "devices": devices}
    sums = sg.plane_checksums(0)
    sg.close()
    del sg
    value = points_glob * args.steps / (elapsed_ms / 1e3) / 1e9
    roof, arith = roofline(cfg, args.config, k, npoints(per_gpu), kfused,
                           elapsed_ms * kfused / args.steps,
                           "device time per k-step round (seam + interior passes of every "
                           "slab, max over devices)")

    parity = slab_parity(ts, torch, cfg, k, glob, kfused, mode, args, sums, n)
    e2e = None
    host_bytes = 2 * esize * npoints([g + 2 for g in glob])
    if not args.no_e2e and host_bytes <= args.e2e_host_limit_gb * 1e9:
        def multi_e2e():
            hg = make_grid(ts, cfg, glob, pinned=True)
            # one untimed call of the same length (slab allocation, kernel
            # load), then the median of three timed calls
            ts.run_multi(hg, k, args.steps, n, devices=devices, fused_steps=kfused, mode=mode)
            walls = []
            for _ in range(3):
                t0 = time.perf_counter()
                st2 = ts.run_multi(hg, k, args.steps, n, devices=devices, fused_steps=kfused,
                                   mode=mode)
                walls.append(time.perf_counter() - t0)
            wall = statistics.median(walls)
            del hg
            ts.release_cache()
            return {"value": round(points_glob * args.steps / wall / 1e9, 3),
                    "unit": "GStencil/s",
                    "h2d_bytes_per_step": round(st2.h2d_bytes / args.steps, 1),
                    "d2h_bytes_per_step": round(st2.d2h_bytes / args.steps, 1),
                    "call": f"paper_2303_08365_b200.run_multi(pinned Grid, ngpus={n}) -> "
                            "tsr_run_multi", "wall_s": round(wall, 4),
                    "walls_s": [round(w, 4) for w in walls],
                    "timing": "median of 3 calls after one untimed call of the same length"}
        e2e = guarded(multi_e2e, "e2e")
    elif not args.no_e2e:
        e2e = {"value": None, "skipped": f"global host grid {host_bytes / 1e9:.1f} GB exceeds "
                                         f"--e2e-host-limit-gb {args.e2e_host_limit_gb}"}
    cpu = None if args.no_cpu else guarded(lambda: cpu_baseline(cfg, n), "cpu_baseline")
    line = base_line(args, cfg, n, mode, value, elapsed_ms)
    line.update({"plan": {"fused_steps": kfused, "engine": "tuned", "runtime":
                          "one host thread, tsr_multi (csrc/multi.cu)"},
                 "roofline": roof, "arith": arith, "parity": parity, "cpu_baseline": cpu,
                 "e2e": e2e, "gpu_launches": launches, "clocks": clocks, "comm": comm})
    return line


def slab_parity(ts, torch, cfg, k, glob, kfused, mode, args, sums, n):
    """Per-plane checksums of the slab run vs a ONE-GPU run of the same
    global grid (same seed, W + K steps, same plan) on device 0."""
    esize = 8 if cfg["dtype"] == "f64" else 4
    need = 3 * esize * npoints([g + 2 * k.radius * kfused + 2 for g in glob])
    free, _ = torch.cuda.mem_get_info(0)
    if args.no_parity or need > 0.9 * free:
        return {"checked": False, "why": "--no-parity" if args.no_parity else
                f"global grid ({need / 1e9:.1f} GB) exceeds device 0's free HBM"}
    one = ts.SlabGrid(k, glob, dtype=cfg["dtype"], ngpus=1, devices=[0], fused_steps=kfused,
                      mode=mode)
    one.fill_random(1)
    one.advance(args.warmup)
    one.advance(args.steps)
    want = one.plane_checksums(0)
    one.close()
    bad = [int(i) for i in (sums != want).nonzero()[0][:8]]
    return {"checked": True, "bitwise_equal": not bad, "planes": int(len(sums)),
            "first_mismatched_planes": bad,
            "against": "one-GPU run of the same global grid (fill_random(1), W+K steps): "
                       "64-bit checksum of every interior plane"}


def run_ranks(args, cfg):
    """`--runtime ranks` under torchrun: one process per GPU, the
    torch.distributed slab runner (partition.py) with peer-IPC seam stores
    or NCCL send/recv; slabs seeded from the global fill_random stream."""
    import torch
    import torch.distributed as dist
    import paper_2303_08365_b200 as ts
    from paper_2303_08365_b200.partition import SlabRunner, plan_slabs
    world = int(os.environ["WORLD_SIZE"])
    rank = int(os.environ["RANK"])
    ndev = torch.cuda.device_count()
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(1, ndev)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if args.dist_backend == "nccl":
        dist.init_process_group("nccl", device_id=dev)
    else:
        dist.init_process_group("gloo")
    mode = args.mode or cfg["mode"]
    fused_req = cfg["fused"] if args.fused is None else args.fused
    k = ts.find_benchmark(cfg["bench"]).kernel
    per_gpu, glob = extents(cfg, world)
    plan = plan_slabs(glob, k.radius, fused_req or 1, world, rank)
    kw = dict(seed=1, fused_steps=fused_req, mode=mode, overlap=not args.no_overlap)
    try:
        runner = SlabRunner.synthetic(ts, k, plan, cfg["dtype"], dev, transport=args.transport,
                                      graphs=args.transport == "peer", **kw)
    except Exception as e:  # IPC mapping refused on this box: message transport
        if args.transport != "peer":
            raise
        print(f"peer transport unavailable ({e}); using nccl", file=sys.stderr)
        runner = SlabRunner.synthetic(ts, k, plan, cfg["dtype"], dev, transport="nccl", **kw)
    kfused = runner.fused_steps
    groups = fused_groups(args.steps, kfused)
    for g in fused_groups(args.warmup, kfused):
        runner.advance(g)
    torch.cuda.synchronize(dev)
    stream = torch.cuda.current_stream(dev)
    sampler = ClockSampler([local])
    sampler.start()
    dist.barrier()
    torch.cuda.synchronize(dev)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(groups) + 1)]
    launches = 0
    ev[0].record(stream)
    for i, g in enumerate(groups):
        launches += runner.advance(g).kernel_launches
        ev[i + 1].record(stream)
    torch.cuda.synchronize(dev)
    dist.barrier()
    clocks = sampler.stop()
    elapsed_ms = ev[0].elapsed_time(ev[-1])
    full = [ev[i].elapsed_time(ev[i + 1]) for i, g in enumerate(groups) if g == kfused]
    launch_ms = statistics.mean(full) if full else elapsed_ms / max(1, len(groups))
    rdev = dev if args.dist_backend == "nccl" else "cpu"
    t = torch.tensor([elapsed_ms, launch_ms], device=rdev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    elapsed_ms, launch_ms = float(t[0]), float(t[1])
    lt = torch.tensor([launches], device=rdev, dtype=torch.int64)
    dist.all_reduce(lt)
    summary = runner.comm_summary()
    runner.close()
    if rank == 0:
        value = npoints(glob) * args.steps / (elapsed_ms / 1e3) / 1e9
        roof, arith = roofline(cfg, args.config, k, npoints(per_gpu), kfused, launch_ms,
                               "max over ranks of the mean CUDA-event round time")
        line = base_line(args, cfg, world, mode, value, elapsed_ms)
        line.update({"plan": {"fused_steps": kfused, "engine": "tuned",
                              "runtime": f"one process per GPU, SlabRunner ({args.transport})"},
                     "roofline": roof, "arith": arith, "gpu_launches": int(lt[0]),
                     "clocks": clocks, "comm": summary})
        print(json.dumps(line))
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--fused", type=int, default=None)
    ap.add_argument("--mode", default=None, choices=["exact", "fast"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-parity", action="store_true", help="N>1: skip the one-GPU check")
    ap.add_argument("--no-graph", action="store_true",
                    help="N=1: time direct launches instead of a CUDA-graph replay of the K steps")
    ap.add_argument("--no-mode-check", action="store_true",
                    help="skip timing the other arithmetic mode and its deviation check")
    ap.add_argument("--share-devices", action="store_true",
                    help="N>1 on fewer GPUs: slabs mapped onto the visible devices round-robin")
    ap.add_argument("--e2e-host-limit-gb", type=float, default=40.0,
                    help="N>1: skip e2e when the pinned global host grid would exceed this")
    ap.add_argument("--runtime", default="host", choices=["host", "ranks"],
                    help="N>1: one host thread over all GPUs (tsr_multi, default) or one "
                         "process per GPU under torchrun (partition.SlabRunner)")
    ap.add_argument("--no-overlap", action="store_true",
                    help="--runtime ranks: exchange, then the whole slab")
    ap.add_argument("--transport", default="peer", choices=["peer", "nccl"],
                    help="--runtime ranks halo exchange: peer-IPC seam stores or NCCL")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="--runtime ranks: gloo to exercise it with ranks sharing one GPU")
    args = ap.parse_args()
    cfg = dict(CONFIGS[args.config])
    args.steps = cfg["steps"] if args.steps is None else args.steps
    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3")
    if args.steps < 1:
        raise SystemExit("--steps must be >= 1")
    if args.impl == "reference":
        return run_reference_arm(args, cfg)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1 and world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if args.runtime == "ranks":
        if world < 2:
            raise SystemExit("--runtime ranks needs torchrun with WORLD_SIZE = --gpus > 1")
        return run_ranks(args, cfg)
    if rank != 0:
        # torchrun rank > 0: the devices are driven from rank 0's host thread
        return
    line = run_single(args, cfg) if args.gpus == 1 else run_slabs(args, cfg, args.gpus)
    print(json.dumps(line))


if __name__ == "__main__":
    main()
