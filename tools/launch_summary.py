"""Summarise an ncu --metrics launch list (csv): per kernel, launches, mean
time, mean DRAM read+write per launch, share of total time.  With --traffic
CFG K it also updates profiles/ncu_traffic.json[CFG] with the dominant kernel
(K = its fused steps per launch, which bench.py matches before reporting it)."""
import csv
import json
import os
import sys
from collections import defaultdict


def load(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    idx = {h: i for i, h in enumerate(hdr)}
    per = defaultdict(lambda: defaultdict(dict))
    for r in rows[start + 1:]:
        if len(r) < len(hdr):
            continue
        per[r[idx["ID"]]]["name"] = r[idx["Kernel Name"]]
        per[r[idx["ID"]]]["m"][r[idx["Metric Name"]]] = float(r[idx["Metric Value"]].replace(",", ""))
    return per


def summarise(path):
    per = load(path)
    agg = defaultdict(lambda: {"n": 0, "t": 0.0, "rd": 0.0, "wr": 0.0})
    for lid, d in per.items():
        name = d["name"].split("(")[0].replace("void ", "")
        a = agg[name]
        a["n"] += 1
        a["t"] += d["m"].get("gpu__time_duration.sum", 0.0)
        a["rd"] += d["m"].get("dram__bytes_read.sum", 0.0)
        a["wr"] += d["m"].get("dram__bytes_write.sum", 0.0)
    total = sum(a["t"] for a in agg.values())
    out = []
    for name, a in sorted(agg.items(), key=lambda kv: -kv[1]["t"]):
        out.append({"kernel": name, "launches": a["n"], "mean_ns": a["t"] / a["n"],
                    "share": a["t"] / total, "dram_bytes_per_launch": (a["rd"] + a["wr"]) / a["n"],
                    "dram_read_per_launch": a["rd"] / a["n"], "dram_write_per_launch": a["wr"] / a["n"]})
    return out


if __name__ == "__main__":
    path = sys.argv[1]
    res = summarise(path)
    for r in res:
        print(f"{r['kernel'][:70]:70} n={r['launches']:4d} mean={r['mean_ns']/1e3:9.1f} us "
              f"share={r['share']*100:5.1f}% dram/launch={r['dram_bytes_per_launch']/1e9:.4f} GB")
    if len(sys.argv) > 4 and sys.argv[2] == "--traffic":
        cfg, fused = sys.argv[3], int(sys.argv[4])
        tp = os.path.join(os.path.dirname(__file__), "..", "profiles", "ncu_traffic.json")
        data = json.load(open(tp)) if os.path.exists(tp) else {}
        top = res[0]
        data[cfg] = {"kernel": top["kernel"], "bytes_per_launch": round(top["dram_bytes_per_launch"]),
                     "read": round(top["dram_read_per_launch"]),
                     "write": round(top["dram_write_per_launch"]),
                     "fused_steps": fused,
                     "source": os.path.relpath(os.path.abspath(path),
                                               os.path.abspath(os.path.dirname(tp)))}
        json.dump(data, open(tp, "w"), indent=1)
