"""tsr_run wall time against the chunk count (TSR_CHUNKS_MAX) for a few
shapes at short T: median of 5 calls after 2 untimed ones."""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import paper_2303_08365_b200 as ts  # noqa: E402

T = int(os.environ.get("T", "20"))
os.environ["TSR_CHUNK_MIN_MB"] = "0"
for name, extent, dt in (("Heat-2D", [4096, 4096], "f64"), ("Box-2D9P", [16384, 16384], "f64"),
                         ("Heat-3D", [512, 512, 512], "f64")):
    k = ts.find_benchmark(name).kernel
    cls = ts.Grid if dt == "f64" else ts.GridF
    g = cls(extent, [k.radius] * k.dims, pinned=True)
    ts.fill_random(g, 1)
    for mx in ("off", "4", "6", "8", "12", "16", "32"):
        os.environ["TSR_RUN_CHUNKED"] = "0" if mx == "off" else "1"
        os.environ["TSR_CHUNKS_MAX"] = "32" if mx == "off" else mx
        walls = []
        for i in range(7):
            t0 = time.perf_counter()
            ts.run_gpu(g, k, T, mode="fast")
            walls.append(time.perf_counter() - t0)
        w = statistics.median(walls[2:])
        print(f"{name} {extent} T={T} chunks_max={mx}: {w*1e3:.2f} ms "
              f"e2e {g.interior_points()*T/w/1e9:.1f} GS/s", flush=True)
    del g
