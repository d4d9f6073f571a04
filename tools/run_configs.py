"""Times the device-resident pipeline per BASELINE config with per-stage CUDA-event breakdown and
checks products against the reference (or a stored hash).  Diagnostic tool (uses the oracle)."""
import hashlib
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import oracle  # noqa: E402
import paper_1803_11301_b200 as pkg  # noqa: E402

P = oracle.port()
cfgs = [int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["20", "24", "28"])]
check = len(sys.argv) > 2 and sys.argv[2] == "check"
FIELD = int(__import__("os").environ.get("FPM_FIELD", "128"))  # 128, 64 or 0 (auto)
out = {}
for lg in cfgs:
    n = 1 << lg
    t0 = time.time()
    a = P.random_bitpoly(n, 20261020)
    b = P.random_bitpoly(n, 20261021)
    tgen = time.time() - t0
    da = torch.from_numpy(a.view(np.int64)).cuda()
    db = torch.from_numpy(b.view(np.int64)).cuda()
    wc = (2 * n - 1 + 63) // 64
    dc = torch.zeros(wc, dtype=torch.int64, device="cuda")
    st = [0.0] * 7
    pkg.fp_polymul_dev(da, n, db, n, dc, field=FIELD, stage_seconds=st)  # warm
    torch.cuda.synchronize()
    reps = 3 if lg >= 30 else 5
    st = [0.0] * 7
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    times = []
    for _ in range(reps):
        e0.record()
        pkg.fp_polymul_dev(da, n, db, n, dc, field=FIELD)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    st = [0.0] * 7
    pkg.fp_polymul_dev(da, n, db, n, dc, field=FIELD, stage_seconds=st)
    torch.cuda.synchronize()
    c = dc.cpu().numpy().view(np.uint64)
    h = hashlib.blake2b(c.tobytes(), digest_size=16).hexdigest()
    rec = {"lg": lg, "ms_min": min(times), "ms_med": sorted(times)[len(times) // 2],
           "stages_ms": {k: round(v * 1e3, 3) for k, v in zip(pkg.STAGE_NAMES, st)}, "hash": h}
    if check:
        t0 = time.time()
        R = oracle.ref(f4=(lg >= 32))
        want = R.polymul(a, n, b, n, field=0)
        rec["ref_s"] = time.time() - t0
        rec["match"] = bool(np.array_equal(c, want))
    print(json.dumps(rec), flush=True)
