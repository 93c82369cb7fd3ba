"""Regenerates the golden fixtures in tests/golden/ from the REFERENCE itself.

* star2d9p_64x64_t12.ttrs — written by the reference's own tool
  (/root/reference/proj/tests/gen_golden.cpp:38-55, compiled unmodified by
  oracle/Makefile into oracle/_ref/gen_golden).  The reference's doctest
  suite checks it bitwise (proj/tests/test_stencil_core.cpp:254-270) but
  does not ship it.
* <case>.npz — naive_run of the reference library (oracle/_ref/
  libtessera_ref.so) on fill_random(seed) grids of every Table-1 kernel
  (proj/src/bench.cpp:63-85), fp64 and fp32: the final read-buffer interior
  ("cur", step T) and the other buffer's interior ("prev", step T-1).

Run here (needs /root/reference):  python tests/golden/make_golden.py
"""
from __future__ import annotations

import json
import os
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import paper_2303_08365_b200 as ts  # noqa: E402  (host Grid type only; no GPU)

# name, benchmark kernel, extent, halo, dtype, seed, steps
CASES = [
    ("heat2d_48x40_t7", "Heat-2D", [48, 40], [1, 1], "f64", 3, 7),
    ("box2d9p_40x36_t8", "Box-2D9P", [40, 36], [1, 1], "f64", 4, 8),
    ("star2d9p_33x30_t6", "Star-2D9P", [33, 30], [2, 2], "f64", 5, 6),
    ("box2d25p_30x28_t4", "Box-2D25P", [30, 28], [2, 2], "f64", 6, 4),
    ("heat3d_20x18x22_t6", "Heat-3D", [20, 18, 22], [1, 1, 1], "f64", 7, 6),
    ("box3d27p_12x14x16_t3", "Box-3D27P", [12, 14, 16], [1, 1, 1], "f64", 9, 3),
    ("box3d27p_f32_16x20x18_t5", "Box-3D27P", [16, 20, 18], [1, 1, 1], "f32", 8, 5),
    ("heat3d_f32_18x16x20_t9", "Heat-3D", [18, 16, 20], [1, 1, 1], "f32", 12, 9),
    ("heat2d_f32_40x44_t10", "Heat-2D", [40, 44], [1, 1], "f32", 13, 10),
    ("heat1d_100_t9", "Heat-1D", [100], [1], "f64", 10, 9),
    ("star1d5p_96_t7", "Star-1D5P", [96], [2], "f64", 11, 7),
]


def main() -> None:
    oracle.build(ref=True)
    os.makedirs("/tmp/tsr_golden", exist_ok=True)
    subprocess.run([os.path.join(oracle.HERE, "_ref", "gen_golden"), "/tmp/tsr_golden"],
                   check=True)
    os.replace("/tmp/tsr_golden/star2d9p_64x64_t12.ttrs",
               os.path.join(HERE, "star2d9p_64x64_t12.ttrs"))
    ref = oracle.Reference()
    index = {}
    for name, bench, extent, halo, dt, seed, steps in CASES:
        cls = ts.Grid if dt == "f64" else ts.GridF
        dims, shape, radius, taps = ref.benchmark_kernel(bench)
        k = ts.make_kernel(dims, shape, radius, [(o[:dims], w) for o, w in taps])
        g = cls(extent, halo)
        ref.fill_random(g, seed)
        ref.naive_run(g, k, steps)
        np.savez_compressed(os.path.join(HERE, name + ".npz"),
                            cur=g.interior_view(g.parity), prev=g.interior_view(1 - g.parity))
        index[name] = {"benchmark": bench, "extent": extent, "halo": halo, "dtype": dt,
                       "seed": seed, "steps": steps, "final_parity": g.parity}
    with open(os.path.join(HERE, "index.json"), "w") as f:
        json.dump(index, f, indent=1)
    print(f"wrote {len(index)} npz fixtures + star2d9p_64x64_t12.ttrs")


if __name__ == "__main__":
    main()
