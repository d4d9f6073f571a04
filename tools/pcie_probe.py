"""PCIe copy rates with pinned memory: one stream vs the same bytes split over K streams (separate
copy engines), both directions.  usage: pcie_probe.py [MiB=1024]"""
import sys
import time

import torch

mib = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
n = mib << 20
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for K in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(K)]
    for name, src, dst in (("h2d", h, d), ("d2h", d, h)):
        best = 1e9
        for rep in range(5):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for k, s in enumerate(streams):
                lo, hi = n * k // K, n * (k + 1) // K
                with torch.cuda.stream(s):
                    dst[lo:hi].copy_(src[lo:hi], non_blocking=True)
            torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t0)
        print(f"{name} {mib} MiB over {K} stream(s): {n / best / 1e9:.2f} GB/s ({best * 1e3:.3f} ms)")
