"""Wall time of tsr_run (run_gpu on a pinned grid) with and without the
chunked round trip, three calls each, for the C1/C3/C4 shapes at short T."""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import paper_2303_08365_b200 as ts  # noqa: E402

T = int(os.environ.get("T", "20"))
for name, extent, dt, mode in (("Heat-2D", [4096, 4096], "f64", "fast"),
                               ("Heat-3D", [512, 512, 512], "f64", "fast"),
                               ("Box-3D27P", [1024, 1024, 1024], "f32", "fast")):
    k = ts.find_benchmark(name).kernel
    cls = ts.Grid if dt == "f64" else ts.GridF
    g = cls(extent, [k.radius] * k.dims, pinned=True)
    ts.fill_random(g, 1)
    for e in ("0", "1", "0", "1"):
        os.environ["TSR_RUN_CHUNKED"] = e
        for i in range(3):
            t0 = time.perf_counter()
            st = ts.run_gpu(g, k, T, mode=mode)
            w = time.perf_counter() - t0
            print(f"{name} chunked={e} call{i}: wall {w*1e3:.1f} ms  device {st.device_ms:.2f} ms "
                  f"launches {st.kernel_launches} k={st.fused_steps} "
                  f"e2e {g.interior_points()*T/w/1e9:.1f} GS/s", flush=True)
    del g
    ts.release_cache() if hasattr(ts, "release_cache") else None
