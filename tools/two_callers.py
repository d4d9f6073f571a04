"""Throughput of the host entry point fpm_polymul with C concurrent callers (host threads, each with
its own pinned operands and product buffer): the calls are reentrant, so one caller's PCIe copies
overlap another caller's kernels.  Prints ms per product for C = 1, 2, 3 and checks every product
against the single-caller result.  usage: two_callers.py [lg=32] [products_per_caller=4]"""
import os
import sys
import threading
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1803_11301_b200 as pkg  # noqa: E402

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 32
per = int(sys.argv[2]) if len(sys.argv) > 2 else 4
bits = 1 << lg
words = bits // 64
out_words = (2 * bits - 1 + 63) // 64
ha = torch.from_numpy(pkg.random_bitpoly(bits, 20261020).view(np.int64)).pin_memory()
hb = torch.from_numpy(pkg.random_bitpoly(bits, 20261021).view(np.int64)).pin_memory()
na, nb = (x.numpy().view(np.uint64) for x in (ha, hb))
outs = [torch.empty(out_words, dtype=torch.int64, pin_memory=True) for _ in range(3)]
nouts = [o.numpy().view(np.uint64) for o in outs]


def caller(k, n):
    for _ in range(n):
        pkg.fp_polymul(na, bits, nb, bits, field=pkg.FIELD_GF128, device=0, out=nouts[k])


for k in range(3):  # warm every buffer (pool growth, graph capture for small products)
    caller(k, 2)
want = nouts[0].copy()
for C in (1, 2, 3):
    if C > 1:  # untimed concurrent round: the pool grows once for every extra concurrent caller
        warm = [threading.Thread(target=caller, args=(k, 1)) for k in range(C)]
        for t in warm:
            t.start()
        for t in warm:
            t.join()
    for k in range(C):
        nouts[k][:] = 0
    th = [threading.Thread(target=caller, args=(k, per)) for k in range(C)]
    t0 = time.perf_counter()
    for t in th:
        t.start()
    for t in th:
        t.join()
    dt = (time.perf_counter() - t0) * 1e3
    ok = all(np.array_equal(nouts[k], want) for k in range(C))
    print(f"lg={lg} callers={C} products={C * per} ms_per_product={dt / (C * per):.3f} all_equal={ok}")
