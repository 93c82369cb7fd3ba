"""Device-resident GS/s of the 27-point box (fp64 and fp32) against the
fused depth k and arithmetic mode (default-k choice for box3d/tbbox)."""
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import torch  # noqa: E402
import paper_2303_08365_b200 as ts  # noqa: E402

k = ts.find_benchmark("Box-3D27P").kernel
steps = 24
for dt, ext in (("f64", [512, 512, 512]), ("f64", [1024, 1024, 1024]), ("f32", [1024, 1024, 1024])):
    cls = ts.Grid if dt == "f64" else ts.GridF
    g = cls(ext, [1, 1, 1])
    ts.fill_random(g, 1)
    dg = ts.DeviceGrid(g, torch.device("cuda", 0))
    for mode in ("exact", "fast"):
        row = {}
        for kf in (1, 2, 3, 4):
            try:
                st = dg.advance(k, 2 * kf, fused_steps=kf, mode=mode)
            except Exception as e:  # depth beyond the engine's maximum
                row[kf] = str(e)[:40]
                continue
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            st = dg.advance(k, steps, fused_steps=kf, mode=mode)
            e1.record()
            torch.cuda.synchronize()
            row[f"{kf}->{st.fused_steps}"] = round(ext[0] * ext[1] * ext[2] * steps / e0.elapsed_time(e1) / 1e6, 1)
        print(json.dumps({"dtype": dt, "extent": ext, "mode": mode, "gs_by_k": row}), flush=True)
    del dg, g
