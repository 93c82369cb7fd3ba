"""Host cost of one slab round (tsr_multi_advance from one host thread):
tiny slabs so the device finishes first, wall time per round per slab."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2303_08365_b200 as ts  # noqa: E402

k = ts.find_benchmark("Heat-3D").kernel
ndev = torch.cuda.device_count()
for P in (1, 2, 4, 8):
    with ts.SlabGrid(k, [24 * P, 32, 64], ngpus=P, devices=[i % ndev for i in range(P)],
                     fused_steps=3, mode="fast") as sg:
        sg.fill_random(1)
        sg.advance(30)
        t0 = time.perf_counter()
        st = sg.advance(300)
        wall = time.perf_counter() - t0
    rounds = st.rounds + (1 if st.trailing_steps else 0)
    print(f"P={P}: {wall / rounds * 1e6:.1f} us host+device per round, "
          f"{wall / rounds / P * 1e6:.1f} us per slab-round; device {st.device_ms / rounds * 1e3:.1f} us "
          f"per round; launches {st.kernel_launches}")
