"""One fpm_polymul_multi product of a 2^lg x 2^lg-bit config with P logical ranks on GPU 0 (host
buffers in, host buffer out), after `reps - 1` warm-ups, with wall-clock timing per call -- the
command profiled by ncu for the sharded conversion's per-rank launch list.
usage: multi_product.py [lg=32] [P=8] [reps=2]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1803_11301_b200 as pkg  # noqa: E402

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 32
P = int(sys.argv[2]) if len(sys.argv) > 2 else 8
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
n = 1 << lg
a = pkg.random_bitpoly(n, 20261020)
b = pkg.random_bitpoly(n, 20261021)
for r in range(reps):
    t0 = time.time()
    c = pkg.fp_polymul_multi(a, n, b, n, [0] * P, field=pkg.FIELD_GF128)
    print(f"rep {r}: {1e3 * (time.time() - t0):.1f} ms (wall, {P} logical ranks on one GPU)")
print("launches", pkg.launch_count())
