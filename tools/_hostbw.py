"""Does the host zero fill of the result grid slow the H2D / D2H DMAs?"""
import os, sys, time, threading
import numpy as np, torch
dev = torch.device("cuda", 0)
torch.cuda.init()
nb = 436 << 20; nb2 = 99 << 20
hp = torch.empty(nb, dtype=torch.uint8, pin_memory=True)
dd = torch.empty(nb, dtype=torch.uint8, device=dev)
grid = torch.empty(256 ** 3, dtype=torch.float64, pin_memory=True)
s2 = torch.cuda.Stream()
def run(zero, d2h, threads=None):
    if threads: torch.set_num_threads(threads)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if d2h:
        with torch.cuda.stream(s2):
            hp[nb - nb2:].copy_(dd[:nb2], non_blocking=True)
    dd[:nb - nb2].copy_(hp[:nb - nb2], non_blocking=True)
    tz = 0
    if zero:
        z0 = time.perf_counter(); grid.zero_(); tz = time.perf_counter() - z0
    torch.cuda.synchronize()
    torch.set_num_threads(16)
    return 1e3 * (time.perf_counter() - t0), 1e3 * tz
for zero, d2h, th in [(0, 0, None), (1, 0, None), (0, 1, None), (1, 1, None), (1, 1, 4), (1, 1, 2), (1, 0, 4)]:
    r = [run(zero, d2h, th) for _ in range(6)][1:]
    print(f"h2d 337MB zero={zero} d2h={d2h} threads={th}: total {np.median([x[0] for x in r]):.2f} ms, zero fill {np.median([x[1] for x in r]):.2f} ms")
