"""One device-resident product of a 2^lg x 2^lg-bit config after `reps - 1` warm-ups: the command
profiled by ncu (launch list / full capture).  usage: one_product.py [lg=32] [reps=2] [field=128]"""
import sys

import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import paper_1803_11301_b200 as pkg  # noqa: E402

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 32
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
field = int(sys.argv[3]) if len(sys.argv) > 3 else 128
n = 1 << lg
g = torch.Generator(device="cuda").manual_seed(1)
a = torch.randint(-(1 << 62), 1 << 62, (n // 64,), generator=g, device="cuda", dtype=torch.int64)
b = torch.randint(-(1 << 62), 1 << 62, (n // 64,), generator=g, device="cuda", dtype=torch.int64)
c = torch.empty((2 * n - 1 + 63) // 64, dtype=torch.int64, device="cuda")
for _ in range(reps):
    pkg.fp_polymul_dev(a, n, b, n, c, field=field)
torch.cuda.synchronize()
print("launches", pkg.launch_count())
