import time, ctypes, numpy as np, torch
torch.cuda.init()
cudart = ctypes.CDLL("libcudart.so.12") if False else None
import glob
libs = glob.glob("/usr/local/cuda/lib64/libcudart.so*")
cr = ctypes.CDLL(libs[0])
for gb in (0.25, 1.0, 2.0):
    n = int(gb * (1 << 30))
    a = np.empty(n, dtype=np.uint8); a[::4096] = 1  # touch pages
    t0 = time.perf_counter()
    rc = cr.cudaHostRegister(ctypes.c_void_p(a.ctypes.data), ctypes.c_size_t(n), 0)
    t1 = time.perf_counter()
    rc2 = cr.cudaHostUnregister(ctypes.c_void_p(a.ctypes.data))
    t2 = time.perf_counter()
    print(f"{gb} GB register rc={rc} {1e3*(t1-t0):.1f} ms ({gb/(t1-t0):.1f} GB/s), unregister {1e3*(t2-t1):.1f} ms", flush=True)
    # untouched pages
    b = np.empty(n, dtype=np.uint8)
    t0 = time.perf_counter(); rc = cr.cudaHostRegister(ctypes.c_void_p(b.ctypes.data), ctypes.c_size_t(n), 0); t1 = time.perf_counter()
    cr.cudaHostUnregister(ctypes.c_void_p(b.ctypes.data))
    print(f"   untouched: {1e3*(t1-t0):.1f} ms", flush=True)
print("threads", __import__("os").cpu_count())
