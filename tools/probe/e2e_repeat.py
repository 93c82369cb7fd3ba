"""Repeated tsr_run calls (C3 shape, T=20 unless T is set) after a
device-resident warm-up, chunked and whole-grid round trips interleaved:
looks for outlier calls."""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import torch  # noqa: E402
import paper_2303_08365_b200 as ts  # noqa: E402

T = int(os.environ.get("T", "20"))
k = ts.find_benchmark("Heat-3D").kernel
g = ts.Grid([512, 512, 512], [1, 1, 1])
ts.fill_random(g, 1)
st = ts.DeviceGrid(g, torch.device("cuda", 0))
st.advance(k, 60, fused_steps=3, mode="fast")
torch.cuda.synchronize()
hg = ts.Grid([512, 512, 512], [1, 1, 1], pinned=True)
ts.fill_random(hg, 1)
for T_ in (4, T):
    for i in range(8):
        os.environ["TSR_RUN_CHUNKED"] = "1" if i % 2 == 0 else "0"
        t0 = time.perf_counter()
        s = ts.run_gpu(hg, k, T_, fused_steps=3, mode="fast")
        w = time.perf_counter() - t0
        print(f"T={T_} chunked={os.environ['TSR_RUN_CHUNKED']} wall {w*1e3:.1f} ms "
              f"device {s.device_ms:.2f} ms", flush=True)
