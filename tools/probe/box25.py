import os, sys, json
sys.path.insert(0, "/root/repo")
import torch, paper_2303_08365_b200 as ts
k = ts.find_benchmark("Box-2D25P").kernel
g = ts.Grid([10000, 10000], [2, 2]); ts.fill_random(g, 1)
for mode in ("exact", "fast"):
    dg = ts.DeviceGrid(g, torch.device("cuda", 0))
    for kf in (1, 2):
        dg.advance(k, 4, fused_steps=kf, mode=mode); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); dg.advance(k, 200, fused_steps=kf, mode=mode); e1.record(); torch.cuda.synchronize()
        print(mode, kf, "device-resident", round(1e8*200/e0.elapsed_time(e1)/1e6, 1), flush=True)
    del dg
    os.environ["TSR_RUN_CHUNKED"] = "0"
    for i in range(2):
        st = ts.run_gpu(g, k, 200, mode=mode)
    print(mode, "tsr_run device_ms", st.device_ms, round(1e8*200/st.device_ms/1e6, 1), "k", st.fused_steps)
