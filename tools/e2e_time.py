"""End-to-end time of the host entry point fpm_polymul (pinned host buffers, both PCIe copies inside)
for one 2^lg x 2^lg-bit product: median of `reps` calls after two warm-ups, with the product's
hash (config 5: compared with the reference's).  usage: e2e_time.py [lg=32] [reps=5] [field=128|64|0]"""
import hashlib
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1803_11301_b200 as pkg  # noqa: E402

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 32
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
field = int(sys.argv[3]) if len(sys.argv) > 3 else 128
bits = 1 << lg
ha = torch.from_numpy(pkg.random_bitpoly(bits, 20261020).view(np.int64)).pin_memory()
hb = torch.from_numpy(pkg.random_bitpoly(bits, 20261021).view(np.int64)).pin_memory()
out = torch.empty((2 * bits - 1 + 63) // 64, dtype=torch.int64, pin_memory=True)
na, nb, no = (x.numpy().view(np.uint64) for x in (ha, hb, out))
ts = []
for k in range(reps + 2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pkg.fp_polymul(na, bits, nb, bits, field=field, device=0, out=no)
    ts.append((time.perf_counter() - t0) * 1e3)
h = hashlib.blake2b(no.tobytes(), digest_size=16).hexdigest()
with open(os.path.join(ROOT, "tests", "golden", "reference_meta.json")) as f:
    ref = json.load(f)["configs"].get(f"{bits}x{bits}", {})
match = (h == ref["blake2b128"]) if ref.get("seed_a") == 20261020 and ref.get("seed_b") == 20261021 else None
print(f"FPM_PRE_A_FRAC={os.environ.get('FPM_PRE_A_FRAC', 'default')} lg={lg} field={field} e2e median {sorted(ts[2:])[reps // 2]:.3f} ms "
      f"(min {min(ts[2:]):.3f})  hash {h}  matches_reference={match}")
