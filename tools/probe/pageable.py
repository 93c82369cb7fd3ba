"""tsr_run on pageable vs pinned host buffers (C3 shape, T=20): median of 3
calls after one untimed call, chunked and whole-grid round trips."""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import paper_2303_08365_b200 as ts  # noqa: E402

T = int(os.environ.get("T", "20"))
k = ts.find_benchmark("Heat-3D").kernel
for pinned in (False, True):
    g = ts.Grid([512, 512, 512], [1, 1, 1], pinned=pinned)
    ts.fill_random(g, 1)
    for ch in ("0", "1"):
        os.environ["TSR_RUN_CHUNKED"] = ch
        walls = []
        for i in range(4):
            t0 = time.perf_counter()
            ts.run_gpu(g, k, T, mode="fast")
            walls.append(time.perf_counter() - t0)
        w = statistics.median(walls[1:])
        print(f"pinned={pinned} chunked={ch}: {w*1e3:.1f} ms e2e "
              f"{g.interior_points()*T/w/1e9:.1f} GS/s  walls {[round(x*1e3,1) for x in walls]}",
              flush=True)
    del g
