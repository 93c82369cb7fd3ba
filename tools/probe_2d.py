"""Device-resident GS/s of the 2-D engine over several extents (A/B probe)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2303_08365_b200 as ts

name = sys.argv[1] if len(sys.argv) > 1 else "Box-2D9P"
mode = sys.argv[2] if len(sys.argv) > 2 else "exact"
k = ts.find_benchmark(name).kernel
for ext in ([10000, 10000], [16384, 16384], [10240, 10240], [10000, 10240], [10240, 10000], [4096, 4096]):
    g = ts.Grid(ext, [k.radius] * 2)
    ts.fill_random(g, 1)
    dg = ts.DeviceGrid(g, torch.device("cuda", 0))
    st = dg.advance(k, 8, mode=mode)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    st = dg.advance(k, 40, mode=mode)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(json.dumps({"name": name, "extent": ext, "k": st.fused_steps, "gs": ext[0] * ext[1] * 40 / ms / 1e6}))
    del dg
