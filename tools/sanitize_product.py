"""One 2^24 x 2^24-bit GF(2^128) product (l = 18: radix-4 top passes fft_top4_kernel and the tower
tile pass fft_tile_tower_kernel, every basis-conversion kernel) for compute-sanitizer runs:
    compute-sanitizer --tool racecheck|synccheck|memcheck python tools/sanitize_product.py
checked against the golden hash of BASELINE config 3 (tests/golden/reference_meta.json)."""
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1803_11301_b200 as pkg  # noqa: E402

os.environ.setdefault("FPM_GRAPHS", "0")
with open(os.path.join(ROOT, "tests", "golden", "reference_meta.json")) as f:
    c = json.load(f)["configs"]["16777216x16777216"]
a = pkg.random_bitpoly(c["a_bits"], c["seed_a"])
b = pkg.random_bitpoly(c["b_bits"], c["seed_b"])
p = pkg.fp_polymul(a, c["a_bits"], b, c["b_bits"], field=pkg.FIELD_GF128)
ok = hashlib.blake2b(p.tobytes(), digest_size=16).hexdigest() == c["blake2b128"]
print("product matches the reference hash:", ok)
sys.exit(0 if ok else 1)
