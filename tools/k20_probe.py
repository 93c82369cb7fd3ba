import sys, torch
sys.path.insert(0, '.')
import paper_2303_08365_b200 as ts
import bench
cfg = bench.CONFIGS['c3']
k = ts.find_benchmark('Heat-3D').kernel
host = bench.make_grid(ts, cfg, [512,512,512])
dev = torch.device('cuda', 0)
st = ts.DeviceGrid(host, dev)
st.advance(k, 1, mode='fast')
for n in bench.fused_groups(10, 3): st.advance(k, n, fused_steps=3, mode='fast')
torch.cuda.synchronize()
for K in (20, 20, 60, 300):
    groups = bench.fused_groups(K, 3)
    s = torch.cuda.current_stream()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(groups)+1)]
    torch.cuda.synchronize()
    ev[0].record(s)
    for i, n in enumerate(groups):
        st.advance(k, n, fused_steps=3, mode='fast'); ev[i+1].record(s)
    torch.cuda.synchronize()
    t = [ev[i].elapsed_time(ev[i+1]) for i in range(len(groups))]
    tot = ev[0].elapsed_time(ev[-1])
    print(K, 'total ms', round(tot,3), 'GS/s', round(134217728*K/tot/1e6,1), 'groups', [round(x,3) for x in t[:4]], '...', [round(x,3) for x in t[-3:]])
