"""Where the e2e time of run_gpu goes at C3 (512^3 fp64): transfers vs compute.
Compares the pitched 3-D copies tsr_run does against contiguous copies of the
same byte counts (torch, pinned)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2303_08365_b200 as ts

k = ts.find_benchmark("Heat-3D").kernel
g = ts.Grid([512, 512, 512], [1, 1, 1], pinned=True)
ts.fill_random(g, 1)
for steps in (1, 2, 2, 4, 30, 1000):
    t0 = time.perf_counter()
    st = ts.run_gpu(g, k, steps, fused_steps=3)
    w = time.perf_counter() - t0
    print(f"run_gpu steps={steps}: wall {w*1e3:.1f} ms device {st.device_ms:.1f} ms "
          f"overhead {w*1e3 - st.device_ms:.1f} ms h2d {st.h2d_bytes/1e9:.3f} GB d2h {st.d2h_bytes/1e9:.3f} GB")
n = g.buffer_size() if callable(getattr(g, 'buffer_size', None)) else g.buffer_size
h = torch.empty(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device="cuda")
for _ in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter(); d.copy_(h, non_blocking=True); torch.cuda.synchronize()
    a = time.perf_counter() - t0
    t0 = time.perf_counter(); h.copy_(d, non_blocking=True); torch.cuda.synchronize()
    b = time.perf_counter() - t0
    print(f"contiguous {n*8/1e9:.3f} GB: h2d {a*1e3:.1f} ms ({n*8/a/1e9:.1f} GB/s)  d2h {b*1e3:.1f} ms ({n*8/b/1e9:.1f} GB/s)")
t0 = time.perf_counter(); ok = ts.Grid([512, 512, 512], [1, 1, 1]); print("alloc", time.perf_counter()-t0)
