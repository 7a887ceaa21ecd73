"""cudaMalloc timing on this box: fresh 1 GB blocks, after cudaFree, and through the engine's block cache."""
import ctypes, time, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
torch.zeros(1, device="cuda"); torch.cuda.synchronize()
rt = ctypes.CDLL("libcudart.so.12") if os.path.exists("/usr/local/cuda/lib64/libcudart.so.12") else None
if rt is None:
    import glob
    rt = ctypes.CDLL(glob.glob("/usr/local/cuda*/lib64/libcudart.so*")[0])
def malloc(n):
    p = ctypes.c_void_p(); t = time.perf_counter(); rc = rt.cudaMalloc(ctypes.byref(p), ctypes.c_size_t(n)); dt = time.perf_counter() - t
    return p, dt, rc
for rnd in range(3):
    ps = []
    ts = []
    for i in range(6):
        p, dt, rc = malloc(1 << 30); ps.append(p); ts.append(dt * 1e3)
    t = time.perf_counter()
    for p in ps: rt.cudaFree(p)
    rt.cudaDeviceSynchronize()
    print(f"round {rnd}: cudaMalloc 1 GiB x6 ms: {[round(x,1) for x in ts]}, free all {1e3*(time.perf_counter()-t):.1f} ms", flush=True)
