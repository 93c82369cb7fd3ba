"""Device-resident GS/s of the 2-D engine against the fused depth k, per
extent and arithmetic mode (default-k choice for 2-D kernels)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2303_08365_b200 as ts  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "Heat-2D"
steps = 120
k = ts.find_benchmark(name).kernel
for ext in ([4096, 4096], [9600, 9600], [16384, 16384]):
    g = ts.Grid(ext, [k.radius] * 2)
    ts.fill_random(g, 1)
    dg = ts.DeviceGrid(g, torch.device("cuda", 0))
    for mode in ("exact", "fast"):
        row = {}
        for kf in (3, 4, 5, 6, 8):
            dg.advance(k, 2 * kf, fused_steps=kf, mode=mode)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            dg.advance(k, steps, fused_steps=kf, mode=mode)
            e1.record()
            torch.cuda.synchronize()
            row[kf] = round(ext[0] * ext[1] * steps / e0.elapsed_time(e1) / 1e6, 1)
        print(json.dumps({"name": name, "extent": ext, "mode": mode, "gs_by_k": row}), flush=True)
    del dg
