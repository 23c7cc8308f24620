import sys, os; sys.path.insert(0, os.getcwd())
import time, numpy as np, torch, concurrent.futures as cf
from paper_2601_04860_b200.staging import Stager
dev = torch.device("cuda", 0)
n = 436 << 20
src = np.random.default_rng(0).random(n // 4, dtype=np.float32)
dst = torch.empty(n // 4, dtype=torch.float32, device=dev)
s = torch.cuda.Stream()
for slot_mb, nslots, th in [(8, 12, 8), (4, 24, 8), (16, 8, 8), (8, 12, 16), (2, 32, 12)]:
    st = Stager(slot_mb << 20, nslots, th)
    for rep in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        st.copy(dst.data_ptr(), src, s); st.flush(); s.synchronize()
        t = time.perf_counter() - t0
    ok = np.array_equal(dst.cpu().numpy(), src)
    print(f"slot {slot_mb} MB x {nslots}, {th} threads: {t*1e3:.1f} ms = {n/t/1e9:.1f} GB/s ok={ok}")
# raw host copy bandwidth with threads
buf = torch.empty(n, dtype=torch.uint8, pin_memory=True).numpy()
for th in (1, 4, 8, 16):
    pool = cf.ThreadPoolExecutor(th)
    t0 = time.perf_counter()
    chunk = n // 64
    futs = [pool.submit(np.copyto, buf[i*chunk:(i+1)*chunk], src.view(np.uint8)[i*chunk:(i+1)*chunk]) for i in range(64)]
    [f.result() for f in futs]
    t = time.perf_counter() - t0
    print(f"host copy {th} threads: {n/t/1e9:.1f} GB/s")
t0=time.perf_counter(); torch.from_numpy(src).to(dev); torch.cuda.synchronize(); t=time.perf_counter()-t0
print(f"pageable torch .to(dev): {n/t/1e9:.1f} GB/s")
pin = torch.from_numpy(src).pin_memory()
t0=time.perf_counter(); pin.to(dev, non_blocking=True); torch.cuda.synchronize(); t=time.perf_counter()-t0
print(f"pinned .to(dev): {n/t/1e9:.1f} GB/s")
