"""Summarise `nvcc -Xptxas -v` logs: kernel, registers, spill bytes, smem."""
import re
import subprocess
import sys

for path in sys.argv[1:]:
    cur = None
    rows = []
    for line in open(path):
        m = re.search(r"Compiling entry function '(\S+)'", line)
        if m:
            cur = {"name": m.group(1), "spill": "0", "regs": "?", "smem": "0"}
            rows.append(cur)
            continue
        if cur is None:
            continue
        m = re.search(r"(\d+) bytes spill stores", line)
        if m:
            cur["spill"] = m.group(1)
        m = re.search(r"Used (\d+) registers", line)
        if m:
            cur["regs"] = m.group(1)
        m = re.search(r"(\d+) bytes smem", line)
        if m:
            cur["smem"] = m.group(1)
    names = subprocess.run(["c++filt"], input="\n".join(r["name"] for r in rows),
                           capture_output=True, text=True).stdout.split("\n")
    for r, n in zip(rows, names):
        n = n.replace("(anonymous namespace)::", "").replace("tsr::", "")
        n = re.sub(r"\(.*", "", n).replace("void ", "")
        print(f"{r['regs']:>4} regs {r['spill']:>6} spill {r['smem']:>6} smem  {n}")
