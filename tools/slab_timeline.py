"""Timeline of slab rounds on the GPU (no nsys in this image): a global
Heat-3D grid of P x 512^3 split into P slabs (on P GPUs, or sharing the
visible ones), logged rounds with the seam passes' and the interior pass's
device intervals per slab, and how much of each seam pass ran while the same
slab's interior pass was running.

    python tools/slab_timeline.py [--slabs 2] [--rounds 12] [--out file.json]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2303_08365_b200 as ts  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--slabs", type=int, default=2)
    ap.add_argument("--rounds", type=int, default=12)
    ap.add_argument("--n", type=int, default=512)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    ndev = torch.cuda.device_count()
    devices = [i % ndev for i in range(a.slabs)]
    k = ts.find_benchmark("Heat-3D").kernel
    with ts.SlabGrid(k, [a.n * a.slabs, a.n, a.n], ngpus=a.slabs, devices=devices,
                     fused_steps=3, mode="fast") as sg:
        sg.fill_random(1)
        sg.advance(9)  # warm-up rounds
        sg.set_logging(True)
        st = sg.advance(3 * a.rounds)
        tl = sg.round_timeline()
    rows = []
    for e in tl:
        s0, s1 = e["seam"]
        i0, i1 = e["interior"]
        ov = max(0.0, min(s1, i1) - max(s0, i0))
        e["seam_overlapped_frac"] = ov / (s1 - s0) if s1 > s0 else 0.0
        rows.append(e)
        print(f"round {e['round']:3d} slab {e['slab']}: seam {s0:8.3f}-{s1:8.3f} ms "
              f"interior {i0:8.3f}-{i1:8.3f} ms  seam overlapped {e['seam_overlapped_frac']:.0%}")
    res = {"slabs": a.slabs, "devices": devices, "global_extent": [a.n * a.slabs, a.n, a.n],
           "fused_steps": st.fused_steps, "device_ms": st.device_ms, "rounds": rows,
           "messages": st.messages, "bytes_exchanged": st.bytes_exchanged,
           "mean_seam_overlapped_frac": sum(r["seam_overlapped_frac"] for r in rows) / len(rows)}
    print(json.dumps({k: v for k, v in res.items() if k != "rounds"}))
    if a.out:
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
