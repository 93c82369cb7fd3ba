"""Runs the thermal-diffusion case study on the GPU (desk or full scale) and
prints a JSON summary; artifacts go to the given directory.

    python tools/run_case_study.py [--full] [--out DIR] [--fused K]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2303_08365_b200.case_study import CaseStudyConfig, apply_full_scale, case_study_heat


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--full", action="store_true")
    ap.add_argument("--out", default="gpurun_out/case_study")
    ap.add_argument("--fused", type=int, default=6)
    args = ap.parse_args()
    cfg = CaseStudyConfig(fused_steps=args.fused)
    if args.full:
        apply_full_scale(cfg)
    t0 = time.time()
    res = case_study_heat(cfg, args.out)
    wall = time.time() - t0
    summary = {
        "scale": "full" if args.full else "desk", "extent": cfg.extent, "steps": cfg.steps,
        "final_center_celsius": res["final_center"],
        "fp64_device_s": res["fp64_device_s"], "fp64_gstencil_s": res["fp64_gstencil_s"],
        "fp32_device_s": res["fp32_device_s"], "fp32_gstencil_s": res["fp32_gstencil_s"],
        "wall_s": wall,
        "checkpoints": [{"step": s, "abs_exceed_pct": t.abs_exceed_pct,
                         "rel_exceed_pct": t.rel_exceed_pct}
                        for s, t in zip(res["checkpoint_steps"], res["checkpoint_errors"])],
    }
    print(json.dumps(summary))
    with open(os.path.join(args.out, "summary.json"), "w") as f:
        json.dump(summary, f, indent=1)


if __name__ == "__main__":
    main()
