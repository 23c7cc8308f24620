import time, numpy as np, torch, ctypes
cudart = torch.cuda.cudart()
dev = torch.device("cuda", 0)
torch.zeros(1, device=dev)
arrs = [np.random.default_rng(i).random((756, 1008), dtype=np.float32) for i in range(6 * 32)]
tot = sum(a.nbytes for a in arrs)
for rep in range(3):
    t0 = time.perf_counter()
    for a in arrs:
        r = cudart.cudaHostRegister(a.ctypes.data, a.nbytes, 0)
    t1 = time.perf_counter()
    dst = torch.empty(tot // 4, dtype=torch.float32, device=dev)
    off = 0
    torch.cuda.synchronize(); t2 = time.perf_counter()
    for a in arrs:
        dst[off:off + a.size].copy_(torch.from_numpy(a).view(-1), non_blocking=True); off += a.size
    torch.cuda.synchronize(); t3 = time.perf_counter()
    for a in arrs:
        cudart.cudaHostUnregister(a.ctypes.data)
    t4 = time.perf_counter()
    print(f"register {tot/(t1-t0)/1e9:.1f} GB/s ({(t1-t0)*1e3:.1f} ms), copy {tot/(t3-t2)/1e9:.1f} GB/s ({(t3-t2)*1e3:.1f} ms), unregister {(t4-t3)*1e3:.1f} ms, rc {r}")
print("is_pinned after register:", end=" ")
a = arrs[0]; cudart.cudaHostRegister(a.ctypes.data, a.nbytes, 0); print(torch.from_numpy(a).is_pinned()); cudart.cudaHostUnregister(a.ctypes.data)
