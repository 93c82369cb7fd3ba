"""Small tsr_run calls through every round-trip path (whole-grid, chunked
from pinned buffers, chunked staged from pageable buffers, differing
halos), each checked against the oracle: a compute-sanitizer target."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402  (checker only)
import paper_2303_08365_b200 as ts  # noqa: E402

orc = oracle.Oracle()
for name, extent in (("Heat-3D", [96, 20, 36]), ("Heat-2D", [200, 70])):
    k = ts.find_benchmark(name).kernel
    for chunked, pinned, differ in (("0", False, False), ("1", True, False), ("1", False, False),
                                    ("1", False, True)):
        os.environ["TSR_RUN_CHUNKED"] = chunked
        src = ts.Grid(extent, [1] * k.dims)
        ts.fill_random(src, 3)
        g = ts.Grid(extent, [1] * k.dims, pinned=pinned)
        for w in (0, 1):
            g.buffer(w)[:] = src.buffer(w)
        if differ:
            g.padded(1)[0] = 0.5
        ref = g.copy()
        st = ts.run_gpu(g, k, 5, mode="exact")
        orc.naive_run(ref, k, 5)
        ok = all(g.buffer(w).tobytes() == ref.buffer(w).tobytes() for w in (0, 1))
        print(f"{name} chunked={chunked} pinned={pinned} differing_halo={differ}: "
              f"{'bitwise' if ok else 'MISMATCH'} (k={st.fused_steps})", flush=True)
        assert ok
ts.release_cache()
print("roundtrip sanitize target done")
