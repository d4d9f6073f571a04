"""Generates tests/golden/*.npz from the REAL reference library (oracle/_ref, compiled from
/root/reference/proj by oracle/Makefile).  Run in the build container (where /root/reference exists):

    make -C oracle && python tests/golden/make_golden.py

The fixtures pin the oracle port and the GPU path without needing the reference at test time.
Products at BASELINE scale are stored as blake2b-128 hashes of the product words (configs 1-5);
small cases store full vectors.  Inputs are random_bitpoly(bits, std::mt19937_64(seed))
(proj/src/bitpoly.cpp:19-24), regenerated at test time by oracle.port().random_bitpoly.
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import oracle  # noqa: E402


def h(words: np.ndarray) -> str:
    return hashlib.blake2b(np.ascontiguousarray(words, np.uint64).tobytes(), digest_size=16).hexdigest()


def main(with_big: bool):
    R = oracle.ref()
    out = {}
    c, r, i = R.tables128()
    out["cantor128"], out["rows128"], out["inv_rows128"] = c, r, i
    out["twiddles128_l5"] = R.twiddles128(5)
    # stage vectors (gf128 instantiations)
    a = R.random_bitpoly(1 << 12, 41)
    out["bc_in_4096"] = a
    out["bc_fwd_4096"] = R.basis_cvt(a, 1 << 12)
    out["bc_fwd_bits_4096"] = R.basis_cvt_bits(a, 1 << 12)
    p = R.random_bitpoly(128 << 6, 42)
    out["enc_in_l6"] = p
    out["enc_out_l6"] = R.encode128(p, 6)
    ev = R.random_bitpoly(128 << 7, 43)
    out["bfly_in_l7"] = ev
    out["bfly_fwd_l7"] = R.butterfly128(ev, 7)
    out["bfly_inv_l7"] = R.butterfly128(ev, 7, inverse=True)
    u, v = R.random_bitpoly(128 * 64, 44), R.random_bitpoly(128 * 64, 45)
    out["pw_u"], out["pw_v"], out["pw_out"] = u, v, R.pointwise128(u, v)
    # small products (full vectors), shapes incl. uneven and tiny
    shapes = [(1, 1), (7, 3), (64, 64), (100, 3000), (4095, 4096), (5000, 3000), (1 << 14, (1 << 14) - 17),
              ((1 << 16) + 1, 9)]
    prods = {}
    for k, (la, lb) in enumerate(shapes):
        x, y = R.random_bitpoly(la, 500 + k), R.random_bitpoly(lb, 600 + k)
        prods[f"{la}x{lb}"] = R.polymul(x, la, y, lb, field=0)
    np.savez_compressed(os.path.join(HERE, "reference_small.npz"), **out,
                        **{f"prod_{k}": v for k, v in prods.items()})
    meta = {"shapes": shapes, "seeds": {"a": "500+k", "b": "600+k"}}
    # BASELINE configs: hash of the full product (field auto = the reference default, m=64;
    # products are field independent).  Seeds 20261020 / 20261021.
    cfg = {}
    sizes = [(1, 1 << 20, 1 << 20), (3, 1 << 24, 1 << 24), (3, 1 << 24, (1 << 23) + 12345), (4, 1 << 28, 1 << 28)]
    if with_big:
        sizes.append((5, 1 << 32, 1 << 32))
    for (c_id, la, lb) in sizes:
        t0 = time.time()
        x = R.random_bitpoly(la, 20261020)
        y = R.random_bitpoly(lb, 20261021)
        Rr = oracle.ref(f4=(2 * max(la, lb) >= (1 << 33)))
        prod = Rr.polymul(x, la, y, lb, field=0)
        cfg[f"{la}x{lb}"] = {"config": c_id, "a_bits": la, "b_bits": lb, "seed_a": 20261020, "seed_b": 20261021,
                             "product_bits": la + lb - 1, "blake2b128": h(prod),
                             "library": os.path.basename(Rr.path), "seconds": round(time.time() - t0, 2)}
        print(cfg[f"{la}x{lb}"], flush=True)
    meta["configs"] = cfg
    meta["cfg2_batch"] = cfg2_batch(R)
    path = os.path.join(HERE, "reference_meta.json")
    if not with_big and os.path.exists(path):  # keep the (58 s) config-5 entry of an earlier --big run
        with open(path) as f:
            old = json.load(f).get("configs", {})
        for k, v in old.items():
            cfg.setdefault(k, v)
    with open(path, "w") as f:
        json.dump(meta, f, indent=1)


CFG2_COUNT, CFG2_BITS, CFG2_SEED_A, CFG2_SEED_B = 4096, 1 << 16, 30000, 40000


def cfg2_batch(R):
    """BASELINE config 2: 4096 independent 2^16 x 2^16-bit products; product k multiplies
    random_bitpoly(2^16, 30000 + k) by random_bitpoly(2^16, 40000 + k), each through the reference's
    own fp_polymul (proj/src/polymul.cpp:223-239, auto field).  Stored: the hash of the 4096
    concatenated products (2048 words each, 2^17 - 1 bits) and of product 0 alone."""
    t0 = time.time()
    bits = CFG2_BITS
    prods = []
    for k in range(CFG2_COUNT):
        x = R.random_bitpoly(bits, CFG2_SEED_A + k)
        y = R.random_bitpoly(bits, CFG2_SEED_B + k)
        prods.append(R.polymul(x, bits, y, bits, field=0))
    allw = np.concatenate(prods)
    out = {"count": CFG2_COUNT, "a_bits": bits, "b_bits": bits, "seed_a": f"{CFG2_SEED_A}+k",
           "seed_b": f"{CFG2_SEED_B}+k", "product_words": int(prods[0].size), "blake2b128_all": h(allw),
           "blake2b128_first": h(prods[0]), "library": os.path.basename(R.path),
           "seconds": round(time.time() - t0, 2)}
    print(out, flush=True)
    return out


if __name__ == "__main__":
    main(with_big="--big" in sys.argv)
