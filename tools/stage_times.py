"""Per-stage device times (CUDA events inside the library) of one 2^lg x 2^lg-bit product: median of
`reps` instrumented runs after two warm-ups.  usage: stage_times.py [lg=32] [field=128] [reps=3]
(FPM_LIB=path selects an experiment build of the library)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1803_11301_b200 as pkg  # noqa: E402

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 32
field = int(sys.argv[2]) if len(sys.argv) > 2 else 128
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
n = 1 << lg
g = torch.Generator(device="cuda").manual_seed(1)
a = torch.randint(-(1 << 62), 1 << 62, (n // 64,), generator=g, device="cuda", dtype=torch.int64)
b = torch.randint(-(1 << 62), 1 << 62, (n // 64,), generator=g, device="cuda", dtype=torch.int64)
c = torch.empty((2 * n - 1 + 63) // 64, dtype=torch.int64, device="cuda")
for _ in range(2):
    pkg.fp_polymul_dev(a, n, b, n, c, field=field)
runs = []
for _ in range(reps):
    st = [0.0] * pkg.NUM_STAGES
    pkg.fp_polymul_dev(a, n, b, n, c, field=field, stage_seconds=st)
    torch.cuda.synchronize()
    runs.append(st)
med = [sorted(r[k] for r in runs)[len(runs) // 2] * 1e3 for k in range(pkg.NUM_STAGES)]
tag = os.environ.get("FPM_LIB", "default")
print(f"{tag} lg={lg} field={field} total={sum(med):.3f} ms  " +
      " ".join(f"{k}={v:.3f}" for k, v in zip(pkg.STAGE_NAMES, med)))
