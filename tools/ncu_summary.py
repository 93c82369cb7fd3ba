"""Summarise an ncu --set full report: SOL, pipes, stalls, DRAM bytes, opcode mix."""
import csv
import io
import subprocess
import sys
from collections import Counter


def page(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main(rep):
    raw = page(rep, "--page", "raw")
    hdr, vals = raw[0], raw[2]
    m = dict(zip(hdr, vals))
    def g(k):
        try:
            return float(m[k].replace(",", ""))
        except Exception:
            return float("nan")
    print("kernel:", m.get("Kernel Name", "?")[:100])
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__warps_active.avg.pct_of_peak_sustained_active",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
            "launch__registers_per_thread", "launch__grid_size"]
    for k in keys:
        print(f"  {k:70} {m.get(k, '?')}")
    st = []
    for h, v in m.items():
        if "average_warps_issue_stalled" in h and h.endswith("per_issue_active.ratio"):
            try:
                st.append((float(v), h.split("stalled_")[1].split("_per")[0]))
            except ValueError:
                pass
    print("  stalls/issue:", ", ".join(f"{n}={v:.2f}" for v, n in sorted(st, reverse=True)[:8]))
    src = page(rep, "--page", "source", "--print-source", "sass")
    hdr = src[1]
    idx = {h: i for i, h in enumerate(hdr)}
    c, s = Counter(), Counter()
    tot_i = tot_s = 0
    for r in src[2:]:
        toks = r[idx["Source"]].split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") else toks[0]
        op = op.split(".")[0]
        n = int(r[idx["Instructions Executed"]] or 0)
        k = int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
        c[op] += n
        s[op] += k
        tot_i += n
        tot_s += k
    print("  opcode mix (exec% / stall%):",
          ", ".join(f"{op} {n / tot_i * 100:.1f}/{s[op] / max(tot_s, 1) * 100:.1f}"
                    for op, n in c.most_common(12)))


if __name__ == "__main__":
    for rep in sys.argv[1:]:
        main(rep)
