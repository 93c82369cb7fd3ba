"""Benchmark of the Jacobi stencil sweep on B200 (driver contract: one JSON line).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3]
                    [--impl ours|reference] [--fused k] [--mode exact|fast]

Default workload (N=1): BASELINE config C3, the north star's headline target —
Heat-3D 7-point star fp64, 512^3 interior, halo 1, fill_random(seed=1), 1000
time steps.  A "step" is one time step over the whole grid.  For N>1 every
rank owns a 512^3 slab of a (512*N) x 512 x 512 grid (weak scaling, C5's
slab + deep-halo scheme at C3's per-GPU size); once per k fused steps its seam
pass stores the r*k boundary planes straight into the neighbours' ghost planes
over CUDA-IPC peer memory (--transport peer, default) or they are sent with
NCCL send/recv (--transport nccl).

Arithmetic: Heat-2D/Heat-3D (C1, C3, C5) time FAST mode — one fp64 FMA per
tap in apply_box's order, admitted by the north star within 1e-12 — and every
line carries `modes`: the EXACT mode (mul + add per tap, bitwise naive_run)
timed on the same input, plus the full-grid max_rel_deviation and a bitwise
flag between the two.  Heat-3D's weights (1/4, 1/8) are powers of two, so its
products are exact and FAST is bitwise EXACT on normal-range data (the flag
shows it).  The box kernels (C2, C4) run EXACT: their shared-product Q mode is
as fast as FMA.

`value` is device-resident throughput (GStencil/s = points * K / time, the
reference's Eq. 6, proj/src/metrics.cpp:8-20), timed with CUDA events on the
stream the sweeps launch on, max over ranks.  `e2e` is the same metric through
the reference-facing call (naive_run on host buffers in pinned memory: H2D of
the read buffer + K steps + D2H of both buffers, each one contiguous block).
`--impl reference` times the reference's own CPU path (oracle/_ref: the
unmodified reference sources, run_tessellated with all host threads).
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

CONFIGS = {
    "c1": dict(bench="Heat-2D", extent=[4096, 4096], dtype="f64", steps=100, fused=6,
               mode="fast", workload="C1: 2D heat 5-point star fp64, 4096x4096, 100 timesteps",
               ref_tile=[200, 200], ref_tb=50),
    "c2": dict(bench="Box-2D9P", extent=[16384, 16384], dtype="f64", steps=100, fused=4,
               mode="exact",
               workload="C2: 2D 9-point box fp64, 16384x16384, temporal blocking k=4",
               ref_tile=[2000, 2000], ref_tb=4),
    "c3": dict(bench="Heat-3D", extent=[512, 512, 512], dtype="f64", steps=1000, fused=0,
               mode="fast",
               workload="C3: 3D heat 7-point star fp64, 512^3 per GPU, 1000 timesteps",
               ref_tile=[20, 20, 20], ref_tb=10),
    "c4": dict(bench="Box-3D27P", extent=[1024, 1024, 1024], dtype="f32", steps=100, fused=0,
               mode="exact", strong=True,
               workload="C4: 3D 27-point box fp32, 1024^3 global, slab-partitioned over N GPUs "
                        "(strong scaling), exact mode (shared 1/27 products: bitwise)",
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
    """nvidia-smi clocks / throttle reasons during the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-i", str(self.index), "-lms", "100"], stdout=open(self.path, "w"),
                stderr=subprocess.DEVNULL)
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
                "samples": len(sm)}


def make_grid(ts, cfg, extent, pinned=False, seed=1):
    cls = ts.Grid if cfg["dtype"] == "f64" else ts.GridF
    g = cls(extent, [1] * len(extent), pinned=pinned)
    ts.fill_random(g, seed)
    return g


def fused_groups(steps: int, k: int) -> list[int]:
    out = []
    while steps > 0:
        out.append(min(k, steps))
        steps -= out[-1]
    return out


def ncu_traffic(cfg_name: str, kfused: int):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the dominant
    kernel, from the committed ncu launch list of this bench command
    (profiles/ncu_traffic.json, written by tools/launch_summary.py --traffic),
    or None when the committed capture is for another fused depth."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f).get(cfg_name)
        if d and d.get("fused_steps") == kfused:
            return d
    except Exception:
        pass
    return None


def cpu_baseline(ts, cfg, cfg_name, steps_cap=None):
    """The reference's own CPU path on this host (oracle/_ref), bounded sample."""
    import oracle
    if not oracle.Reference.available():
        return None
    ref = oracle.Reference()
    threads = os.cpu_count() or 1
    k = ts.find_benchmark(cfg["bench"]).kernel
    if cfg["dtype"] == "f64":
        extent = cfg["extent"]
        tb = cfg["ref_tb"]
        g = make_grid(ts, cfg, extent)
        steps = tb * (1 if steps_cap is None else max(1, steps_cap // tb))
        (upd, rounds, trailing), sec = ref.run_tessellated(g, k, steps, cfg["ref_tile"], tb,
                                                           threads)
        if steps_cap is None and sec < 5.0:
            # bounded sample of about 10 s of CPU work (whole tb rounds)
            steps = tb * max(1, min(40, round(10.0 / max(sec, 1e-3))))
            g = make_grid(ts, cfg, extent)
            (upd, rounds, trailing), sec = ref.run_tessellated(g, k, steps, cfg["ref_tile"],
                                                               tb, threads)
        value = upd / sec / 1e9
        return {"value": round(value, 4), "unit": "GStencil/s", "cores": threads,
                "kind": "reference",
                "sample": (f"reference run_tessellated(tile={cfg['ref_tile']}, "
                           f"tb={tb}, threads={threads}) on the full "
                           f"{'x'.join(map(str, extent))} grid, T={steps} ({sec:.1f} s)")}
    # fp32: the reference has no threaded fp32 path; naive_run<float>, 1 thread,
    # on a slab of the full cross-section.
    extent = [64] + cfg["extent"][1:]
    g = make_grid(ts, cfg, extent)
    sec = ref.time_naive_f32(g, k, 1)
    pts = 1
    for e in extent:
        pts *= e
    return {"value": round(pts / sec / 1e9, 4), "unit": "GStencil/s", "cores": 1,
            "kind": "reference",
            "sample": f"reference naive_run<float> 1 thread on a {'x'.join(map(str, extent))} "
                      f"slab, T=1"}


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
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for n in fused_groups(args.steps, kfused):
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


def run_reference_arm(args, cfg, cfg_name):
    import paper_2303_08365_b200 as ts
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    t_steps = min(args.steps, 20)
    cb = cpu_baseline(ts, cfg, cfg_name, steps_cap=t_steps)
    if cb is None:
        print(json.dumps({"impl": "reference", "unavailable":
                          "oracle/_ref/libtessera_ref.so not built (make -C oracle ref)"}))
        return
    line = {"metric": "GStencil/s (fp64) at 1/2/4/8 B200 and % of HBM roofline vs host-CPU ref",
            "impl": "reference", "value": cb["value"], "unit": "GStencil/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": None, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64" if cfg["dtype"] == "f64" else "f32",
            "data": "synthetic: fill_random(seed=1) U[0,1) interior, zero Dirichlet halo",
            "config": {"workload": cfg["workload"], "extent": cfg["extent"]},
            "cpu_baseline": cb,
            "e2e": {"value": cb["value"], "unit": "GStencil/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


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
    ap.add_argument("--no-mode-check", action="store_true",
                    help="skip timing the other arithmetic mode and its deviation check")
    ap.add_argument("--no-overlap", action="store_true",
                    help="N>1: exchange, then the whole slab (no interior/seam split)")
    ap.add_argument("--transport", default="peer", choices=["peer", "nccl"],
                    help="N>1 halo exchange: seam passes storing into the neighbours' ghost "
                         "planes over CUDA-IPC peer memory (default), or NCCL send/recv")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo only to exercise the N>1 path with ranks sharing one GPU")
    args = ap.parse_args()
    cfg = dict(CONFIGS[args.config])
    args.steps = cfg["steps"] if args.steps is None else args.steps
    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3")
    if args.impl == "reference":
        return run_reference_arm(args, cfg, args.config)

    import torch
    import paper_2303_08365_b200 as ts

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    ndev = torch.cuda.device_count()
    if args.dist_backend == "nccl" and world > ndev:
        raise SystemExit(f"--gpus {world} but only {ndev} CUDA devices are visible")
    local = local % ndev
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")

    mode = args.mode or cfg["mode"]
    fused_req = cfg["fused"] if args.fused is None else args.fused
    k = ts.find_benchmark(cfg["bench"]).kernel
    esize = 8 if cfg["dtype"] == "f64" else 4
    strong = cfg.get("strong", False)
    per_gpu = list(cfg["extent"])
    if strong:  # fixed global grid split along axis 0
        per_gpu[0] = cfg["extent"][0] // world
    points_per_gpu = 1
    for e in per_gpu:
        points_per_gpu *= e
    stream = torch.cuda.current_stream(dev)

    if world == 1:
        host = make_grid(ts, cfg, per_gpu)
        state = ts.DeviceGrid(host, dev)
        # resolve the engine's fused step count
        probe = state.advance(k, 1, fused_steps=fused_req, mode=mode)
        kfused = probe.fused_steps
        engine = probe.engine
        advance = lambda n: state.advance(k, n, fused_steps=kfused, mode=mode)  # noqa: E731
        comm = None
    else:
        from paper_2303_08365_b200.partition import SlabRunner, plan_slabs
        kfused_guess = fused_req if fused_req else 1
        glob = list(cfg["extent"]) if strong else [per_gpu[0] * world] + per_gpu[1:]
        plan = plan_slabs(glob, k.radius, kfused_guess, world, rank)
        try:
            runner = SlabRunner.synthetic(ts, k, plan, cfg["dtype"], dev, seed=1 + rank,
                                          fused_steps=fused_req, mode=mode,
                                          overlap=not args.no_overlap, transport=args.transport,
                                          graphs=args.transport == "peer")
        except Exception as e:  # IPC mapping refused on this box: message transport
            if args.transport != "peer":
                raise
            print(f"peer transport unavailable ({e}); using nccl", file=sys.stderr)
            runner = SlabRunner.synthetic(ts, k, plan, cfg["dtype"], dev, seed=1 + rank,
                                          fused_steps=fused_req, mode=mode,
                                          overlap=not args.no_overlap, transport="nccl")
        kfused = runner.fused_steps
        engine = 2
        advance = runner.advance
        comm = runner

    groups = fused_groups(args.steps, kfused)
    for n in fused_groups(args.warmup, kfused):
        advance(n)
    torch.cuda.synchronize(dev)

    sampler = ClockSampler(local)
    sampler.start()
    if dist:
        dist.barrier()
    torch.cuda.synchronize(dev)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(groups) + 1)]
    launches = 0
    ev[0].record(stream)
    for i, n in enumerate(groups):
        st = advance(n)
        launches += st.kernel_launches
        ev[i + 1].record(stream)
    torch.cuda.synchronize(dev)
    if dist:
        dist.barrier()
    clocks = sampler.stop()
    elapsed_ms = ev[0].elapsed_time(ev[-1])
    full = [ev[i].elapsed_time(ev[i + 1]) for i, n in enumerate(groups) if n == kfused]
    launch_ms = statistics.mean(full) if full else elapsed_ms / max(1, len(groups))
    if dist:
        rdev = dev if args.dist_backend == "nccl" else "cpu"
        t = torch.tensor([elapsed_ms, launch_ms], device=rdev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed_ms, launch_ms = float(t[0]), float(t[1])
        lt = torch.tensor([launches], device=rdev, dtype=torch.int64)
        dist.all_reduce(lt)
        launches = int(lt[0])

    total_points = 1
    for e in (cfg["extent"] if strong else [per_gpu[0] * world] + per_gpu[1:]):
        total_points *= e
    value = total_points * args.steps / (elapsed_ms / 1e3) / 1e9
    peak, peak_kind = peaks()
    # Algorithmic bytes of one fused launch on one GPU: 2*sizeof(T) per stencil
    # update (one compulsory read + one write per step), times
    # the k steps the launch advances ("HBM-equivalent" for k > 1).
    alg_bytes = 2 * esize * points_per_gpu * kfused
    achieved = alg_bytes / (launch_ms / 1e3) / 1e9
    traffic = ncu_traffic(args.config, kfused)
    # Arithmetic roofline: the reference's apply_box does one multiply and one
    # add per tap (naive.hpp:75-78), i.e. 2 * taps algorithmic flops per update.
    ntaps = len(k.tap_list())
    fpk, fpk_kind = fp_peak(cfg["dtype"])
    arith_tflops = 2 * ntaps * points_per_gpu * kfused / (launch_ms / 1e3) / 1e12

    modes = None
    if world == 1 and not args.no_mode_check:
        modes = mode_check(ts, torch, cfg, k, host, state, per_gpu, dev, stream, kfused, mode,
                           args, total_points, elapsed_ms)

    e2e = None
    cpu = None
    if rank == 0 and world == 1:
        if not args.no_e2e:
            hg = make_grid(ts, cfg, per_gpu, pinned=True)
            ts.run_gpu(hg, k, min(4, args.steps), fused_steps=kfused, mode=mode)  # warm
            ts.fill_random(hg, 1)
            t0 = time.perf_counter()
            st = ts.run_gpu(hg, k, args.steps, fused_steps=kfused, mode=mode)
            wall = time.perf_counter() - t0
            e2e = {"value": round(total_points * args.steps / wall / 1e9, 3),
                   "unit": "GStencil/s",
                   "h2d_bytes_per_step": round(st.h2d_bytes / args.steps, 1),
                   "d2h_bytes_per_step": round(st.d2h_bytes / args.steps, 1),
                   "call": "paper_2303_08365_b200.run_gpu(pinned Grid) -> tsr_run",
                   "wall_s": round(wall, 4)}
            del hg
        if not args.no_cpu:
            cpu = cpu_baseline(ts, cfg, args.config)

    if comm is not None:
        comm.close()
    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return
    line = {
        "metric": "GStencil/s (fp64) at 1/2/4/8 B200 and % of HBM roofline vs host-CPU ref",
        "value": round(value, 3),
        "unit": "GStencil/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(elapsed_ms / args.steps, 5),
        "higher_is_better": True,
        "scaling": "strong" if strong else "weak",
        "vs_baseline": None,
        "dtype": cfg["dtype"],
        "data": "synthetic: fill_random(seed=1) U[0,1) interior, zero Dirichlet halo",
        "config": {"workload": cfg["workload"], "extent_per_gpu": per_gpu,
                   "global_extent": (list(cfg["extent"]) if strong
                                     else [per_gpu[0] * world] + per_gpu[1:]),
                   "kernel": cfg["bench"], "mode": mode, "fused_steps": kfused,
                   "engine": {1: "generic", 2: "tuned"}.get(engine, str(engine)),
                   "parallelism": f"slab{world}" if world > 1 else "single",
                   "l2": (f"no flush: the two buffers ({2 * esize * points_per_gpu / 1e9:.2f} GB)"
                          " exceed the 126 MB L2")},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                     "unit": "GB/s", "frac": round(achieved / peak, 4),
                     "traffic": traffic["bytes_per_launch"] if traffic else None,
                     "traffic_source": (f"ncu launch list profiles/{traffic['source']} "
                                        f"({traffic['kernel']})") if traffic else None,
                     "peak_source": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)"
                     if peak_kind == "measured" else "fallback (B200_PROFILING.md)",
                     "basis": (f"algorithmic {2 * esize} B per stencil update x {kfused} fused "
                               f"steps per launch / mean CUDA-event launch time "
                               f"{launch_ms:.4f} ms")},
        "arith": {"bound": "fp64" if cfg["dtype"] == "f64" else "fp32",
                  "achieved": round(arith_tflops, 2), "peak": round(fpk, 2), "unit": "TFLOP/s",
                  "frac": round(arith_tflops / fpk, 4),
                  "basis": (f"algorithmic {2 * ntaps} flops per update ({ntaps} taps x mul+add,"
                            f" apply_box) x {kfused} fused steps / mean launch time"),
                  "peak_source": ("measured FMA rate x 2 (profiles/fp_peaks.json, "
                                  "tools/microbench/fp64_peak.cu)") if fpk_kind == "measured"
                  else "nominal 148 SM x 64 FMA x 2 x 1.965 GHz (fp32 2x)"},
        "modes": modes,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clocks,
    }
    if comm is not None:
        line["comm"] = comm.comm_summary()
    print(json.dumps(line))
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
