"""tsr_run wall time, chunked vs whole-grid round trip, against T for the
full-scale Heat-2D (10000^2) and Heat-3D 512^3 on pinned buffers: where the
redundant window sweeps start to cost more than the overlap saves."""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import paper_2303_08365_b200 as ts  # noqa: E402

for name, extent in (("Heat-2D", [10000, 10000]), ("Heat-3D", [512, 512, 512])):
    k = ts.find_benchmark(name).kernel
    g = ts.Grid(extent, [k.radius] * k.dims, pinned=True)
    ts.fill_random(g, 1)
    for T in (10, 20, 40, 80, 120, 200, 400):
        res = {}
        for ch in ("0", "1"):
            os.environ["TSR_RUN_CHUNKED"] = ch
            walls = []
            for _ in range(4):
                t0 = time.perf_counter()
                st = ts.run_gpu(g, k, T, mode="fast")
                walls.append(time.perf_counter() - t0)
            res[ch] = statistics.median(walls[1:])
        print(f"{name} T={T}: whole {res['0']*1e3:.1f} ms, chunked {res['1']*1e3:.1f} ms "
              f"({res['0']/res['1']:.2f}x)", flush=True)
    del g
