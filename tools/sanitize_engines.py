"""One small run of every CUDA engine, for compute-sanitizer (memcheck,
racecheck, synccheck): tb3d k=1..3 (TMA ring + mbarriers), box3d k=1..2 and
its separable k-level pipeline, stream2d (cp.async ring; Q and separable
modes), stream1d, the generic engine, the mirrored seam pass of a two-slab
round, each checked against the oracle (bitwise, or within tolerance for the
FAST separable modes) so a sanitizer-visible race that changed results would
also fail here.

    compute-sanitizer --tool racecheck python tools/sanitize_engines.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import paper_2303_08365_b200 as ts  # noqa: E402

CASES = [  # benchmark, extent, steps, fused, dtype
    ("Heat-3D", [20, 24, 70], 3, 1, "f64"),
    ("Heat-3D", [20, 40, 70], 4, 2, "f64"),
    ("Heat-3D", [20, 40, 130], 6, 3, "f64"),
    ("Heat-3D", [18, 40, 70], 3, 3, "f32"),
    ("Box-3D27P", [12, 20, 70], 2, 1, "f32"),
    ("Box-3D27P", [12, 20, 70], 2, 2, "f64"),
    ("Heat-2D", [64, 300], 6, 6, "f64"),
    ("Box-2D9P", [70, 300], 8, 4, "f64"),
    ("Heat-1D", [3000], 8, 8, "f64"),
    ("Box-2D25P", [40, 90], 4, 0, "f64"),
    ("Star-1D5P", [900], 4, 0, "f32"),
]
GENERIC = [("Heat-3D", [12, 14, 20], 2, "f64"), ("Box-3D27P", [8, 10, 12], 2, "f32")]


def main():
    orc = oracle.Oracle()
    for name, ext, steps, fused, dt in CASES:
        k = ts.find_benchmark(name).kernel
        g = (ts.Grid if dt == "f64" else ts.GridF)(ext, [k.radius] * k.dims)
        ts.fill_random(g, 3)
        ref = g.copy()
        st = ts.run_gpu(g, k, steps, fused_steps=fused)
        orc.naive_run(ref, k, steps)
        ok = g.interior_view(g.parity).tobytes() == ref.interior_view(ref.parity).tobytes()
        print(f"{name} {ext} {dt} T={steps} k={st.fused_steps} engine={st.engine}: "
              f"{'bitwise ok' if ok else 'MISMATCH'}", flush=True)
        assert ok
    # FAST-mode separable box kernels (stream2d SEP, box3d k-level pipeline),
    # within the tolerance of the oracle
    for name, ext, steps, fused, dt in [("Box-2D9P", [70, 300], 8, 4, "f64"),
                                        ("Box-3D27P", [14, 20, 70], 5, 2, "f32"),
                                        ("Box-3D27P", [14, 20, 70], 6, 3, "f64"),
                                        ("Box-3D27P", [14, 30, 300], 9, 3, "f32")]:
        k = ts.find_benchmark(name).kernel
        g = (ts.Grid if dt == "f64" else ts.GridF)(ext, [k.radius] * k.dims)
        ts.fill_random(g, 6)
        ref = g.copy()
        st = ts.run_gpu(g, k, steps, fused_steps=fused, mode="fast")
        orc.naive_run(ref, k, steps)
        d = ts.deviation(g, ref)["max_rel_deviation"]
        ok = d <= (1e-12 if dt == "f64" else 1e-5)
        print(f"{name} {ext} {dt} T={steps} k={st.fused_steps} fast: max_rel {d:.2e} "
              f"{'ok' if ok else 'OUT OF TOLERANCE'}", flush=True)
        assert ok
    for name, ext, steps, dt in GENERIC:
        k = ts.find_benchmark(name).kernel
        g = (ts.Grid if dt == "f64" else ts.GridF)(ext, [k.radius] * k.dims)
        ts.fill_random(g, 4)
        ref = g.copy()
        ts.run_gpu(g, k, steps, engine="generic")
        orc.naive_run(ref, k, steps)
        ok = g.interior_view(g.parity).tobytes() == ref.interior_view(ref.parity).tobytes()
        print(f"{name} {ext} {dt} T={steps} engine=generic: {'bitwise ok' if ok else 'MISMATCH'}",
              flush=True)
        assert ok
    # a two-slab round on one device: seam passes storing into the
    # neighbour's ghost planes (mirror), concurrent interior passes
    k = ts.find_benchmark("Heat-3D").kernel
    g = ts.Grid([40, 24, 70], [1, 1, 1])
    ts.fill_random(g, 5)
    ref = g.copy()
    ts.run_multi(g, k, 7, 2, devices=[0, 0], fused_steps=3)
    orc.naive_run(ref, k, 7)
    ok = g.interior_view(g.parity).tobytes() == ref.interior_view(ref.parity).tobytes()
    print(f"two-slab mirror round: {'bitwise ok' if ok else 'MISMATCH'}", flush=True)
    assert ok
    print("SANITIZE_CASES_OK")


if __name__ == "__main__":
    main()
