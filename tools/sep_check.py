"""FAST (separable) Box-3D27P against the oracle for several fused depths
and ragged grids, with a non-zero halo plane (tbbox / box3d SEP paths)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_2303_08365_b200 as ts  # noqa: E402

orc = oracle.Oracle()
k = ts.find_benchmark("Box-3D27P").kernel
worst = 0.0
for kf in (1, 2, 3, 4):
    for ext in ([40, 37, 70], [21, 64, 131], [9, 10, 11], [70, 45, 300]):
        for dt in ("f32", "f64"):
            g = (ts.GridF if dt == "f32" else ts.Grid)(ext, [1, 1, 1])
            orc.fill_random(g, 3)
            g.padded(0)[0] = 2.5
            g.padded(1)[0] = 2.5
            r = g.copy()
            st = ts.run_gpu(g, k, 13, fused_steps=kf, mode="fast")
            orc.naive_run(r, k, 13)
            d = ts.deviation(g, r)
            tol = 1e-5 if dt == "f32" else 1e-12
            flag = "ok" if d["max_rel_deviation"] <= tol else "FAIL"
            worst = max(worst, d["max_rel_deviation"] / tol)
            print(kf, ext, dt, "k =", st.fused_steps, d["max_rel_deviation"], flag, flush=True)
print("worst/tol", worst)
