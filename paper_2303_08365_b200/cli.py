"""Operator CLI: the reference's `bench` tool (proj/tools/bench.cpp:71-129)
rebuilt on argparse (its CLI11 dependency is not vendored) over the GPU path.

    python -m paper_2303_08365_b200 list
    python -m paper_2303_08365_b200 run [--name Heat-2D|a,b|all]
                                        [--path gpu|tessellate|naive|hetero]
                                        [--scale desk|full] [--seed S] [--steps T]
                                        [--no-verify] [--out report.csv] [--mode exact|fast]
                                        [--comm-log rounds.csv]
    python -m paper_2303_08365_b200 case-study [--config FILE] [--path P] [--full] [--out DIR]

Same subcommands, options, output and exit codes as the reference: `run`
prints the CSV header and one row per benchmark and exits 1 if a row failed
verification; `case-study` prints the final centre temperature, the
per-checkpoint exceedance lines and the artifact list; errors print
"error: <what>" and exit 1.  `--threads` is accepted for compatibility and
ignored (the CUDA grid replaces the worker threads).
"""
from __future__ import annotations

import argparse
import sys


def _cmd_list(out) -> int:
    from .kernel import benchmark_table
    out.write(f"{'name':<12} {'pts':<5} {'radius':<7} {'extent':<28} {'T':<12} blocking\n")
    for s in benchmark_table():
        ext = "x".join(str(e) for e in s.full_extent)
        tile = "x".join(str(t) for t in s.tile) + f"x{s.tb}"
        out.write(f"{s.name:<12} {len(s.kernel.taps()):<5} {s.kernel.radius:<7} {ext:<28} "
                  f"{s.full_steps:<12} {tile}\n")
    return 0


def _cmd_run(a, out) -> int:
    from .harness import csv_header, csv_row, run_benchmark, write_csv_file
    from .kernel import benchmark_table, find_benchmark
    if a.name == "all":
        names = [s.name for s in benchmark_table()]
    else:
        names = [find_benchmark(n).name for n in a.name.split(",")]
    rows = []
    out.write(csv_header() + "\n")
    for n in names:
        log = None
        if a.comm_log and a.path == "hetero":  # one CommLog CSV per benchmark
            log = a.comm_log if len(names) == 1 else a.comm_log.replace(".csv", "") + f"_{n}.csv"
        rows.append(run_benchmark(n, path=a.path, scale=a.scale, seed=a.seed, steps=a.steps,
                                  mode=a.mode, verify=not a.no_verify, comm_log=log))
        out.write(csv_row(rows[-1]) + "\n")
        out.flush()
    if a.out:
        write_csv_file(a.out, rows)
        sys.stderr.write(f"report written to {a.out}\n")
    return 0 if all(r["verify"] != "fail" for r in rows) else 1


def _cmd_case_study(a, out) -> int:
    from .case_study import CaseStudyConfig, apply_full_scale, case_study_heat, parse_case_config
    cfg = parse_case_config(a.config) if a.config else CaseStudyConfig()
    if a.path and a.path not in ("gpu", "naive", "tessellate"):
        raise ValueError(f"unsupported executor path on the GPU library: {a.path}")
    if a.full:
        apply_full_scale(cfg)
    res = case_study_heat(cfg, a.out)
    out.write(f"final center temperature: {res['final_center']} C\n")
    for step, t in zip(res["checkpoint_steps"], res["checkpoint_errors"]):
        out.write(f"T={step}  abs>0.1C: {t.abs_exceed_pct[0]}%  abs>0.5C: {t.abs_exceed_pct[1]}%"
                  f"  abs>1.0C: {t.abs_exceed_pct[2]}%  rel>1%: {t.rel_exceed_pct[0]}%\n")
    out.write("artifacts:\n")
    for p in res["artifacts"]:
        out.write(f"  {p}\n")
    return 0


def parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(
        prog="python -m paper_2303_08365_b200",
        description="stencil engine benchmarks and thermal-diffusion case study (B200)")
    sub = ap.add_subparsers(dest="cmd", required=True)
    r = sub.add_parser("run", help="time benchmarks on an executor path")
    r.add_argument("--name", default="Heat-2D", help="benchmark name, comma list, or 'all'")
    r.add_argument("--path", default="gpu", help="gpu|tessellate|naive|hetero (two GPU slabs; "
                   "vector|mm: CPU simulators of the reference, reported unsupported)")
    r.add_argument("--scale", default="desk", choices=["desk", "full"])
    r.add_argument("--threads", type=int, default=1, help="accepted, ignored")
    r.add_argument("--seed", type=int, default=1)
    r.add_argument("--steps", type=int, default=0, help="override the scale's step count")
    r.add_argument("--no-verify", action="store_true", help="skip the reduced-size check")
    r.add_argument("--out", default="", help="CSV report path")
    r.add_argument("--mode", default="exact", choices=["exact", "fast"])
    r.add_argument("--comm-log", default="", help="hetero: per-round CommLog CSV "
                   "(round,direction,bytes,modeled_cost_alpha_beta,wall_seconds)")
    c = sub.add_parser("case-study", help="thermal diffusion on a square plate")
    c.add_argument("--config", default="", help="line-oriented key = value config file")
    c.add_argument("--path", default="", help="executor path override")
    c.add_argument("--threads", type=int, default=0, help="accepted, ignored")
    c.add_argument("--full", action="store_true",
                   help="full-scale configuration (9600x9600, 3.8e6 steps)")
    c.add_argument("--out", default="case_study_out", help="output directory")
    sub.add_parser("list", help="print the benchmark table")
    return ap


def main(argv=None, out=None) -> int:
    out = out or sys.stdout
    a = parser().parse_args(argv)
    try:
        if a.cmd == "list":
            return _cmd_list(out)
        if a.cmd == "run":
            return _cmd_run(a, out)
        return _cmd_case_study(a, out)
    except Exception as e:  # the reference prints what() and exits 1
        sys.stderr.write(f"error: {e}\n")
        return 1
