"""Hot instructions of an ncu source-page SASS csv (gz ok): per instruction
its executed count and stall samples, the top-N by stall, and the stall mix
of the main loop."""
import csv
import gzip
import sys


def rows(path):
    op = gzip.open if path.endswith(".gz") else open
    with op(path, "rt") as f:
        r = list(csv.reader(f))
    hdr = r[1]
    idx = {h: i for i, h in enumerate(hdr)}
    out = []
    for row in r[2:]:
        if len(row) < len(hdr):
            continue
        out.append({"addr": row[idx["Address"]], "src": row[idx["Source"]].strip(),
                    "stall": int(row[idx["Warp Stall Sampling (All Samples)"]] or 0),
                    "exec": int(row[idx["Instructions Executed"]] or 0)})
    return out


def main(path, n=40):
    rs = rows(path)
    tot = sum(r["stall"] for r in rs) or 1
    print(f"{len(rs)} instructions, {tot} stall samples")
    for i, r in enumerate(rs):
        r["i"] = i
    for r in sorted(rs, key=lambda r: -r["stall"])[:n]:
        print(f"{r['i']:5d} {r['stall'] / tot * 100:5.2f}% exec={r['exec']:10d}  {r['src'][:90]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
