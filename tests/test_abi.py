"""CPU tests of the drop-in boundary: the CUDA library loads without a GPU, exports every symbol
include/fpmul_b200.h declares, plans and builds tables host-side, and fails loudly (FPM_ECUDA)
instead of falling back to the CPU when no device is present."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "fpmul_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fpm_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    import paper_1803_11301_b200 as pkg
    L = pkg.lib()
    syms = header_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing


def test_plan_and_tables_host_side():
    import paper_1803_11301_b200 as pkg
    p = pkg.plan_mul(1 << 20, 1 << 20)
    assert (p["n_bits"], p["field_degree"], p["l"], p["n_p"]) == (1 << 21, 64, 15, 1 << 15)
    p = pkg.plan_mul(1 << 32, 1 << 32, pkg.FIELD_GF128)
    assert (p["n_bits"], p["l"]) == (1 << 33, 26)
    with pytest.raises(ValueError):
        pkg.plan_mul(0, 8)
    g = np.load(os.path.join(ROOT, "tests", "golden", "reference_small.npz"))
    c, r, i = pkg.tables128()
    assert np.array_equal(c, g["cantor128"]) and np.array_equal(r, g["rows128"]) and np.array_equal(i, g["inv_rows128"])


def test_argument_errors_match_reference():
    import paper_1803_11301_b200 as pkg
    with pytest.raises(ValueError):
        pkg.encode(np.zeros(3, np.uint64), 3)  # encode.cpp:157-161
    with pytest.raises(ValueError):
        pkg.pointwise_mul(np.zeros(4, np.uint64), np.zeros(2, np.uint64))  # polymul.cpp:244


def test_no_cpu_fallback_without_device():
    import paper_1803_11301_b200 as pkg
    if pkg.device_count() > 0:
        pytest.skip("a GPU is present; this checks the no-device behaviour")
    a = np.ones(4, np.uint64)
    with pytest.raises(pkg.FpmError, match="no CUDA device"):
        pkg.fp_polymul(a, 256, a, 256)


def test_gf64_tables_host_side(port):
    """CantorField<gf64> / EncodeMatrix<gf64> as built by the library (host only) equal the port's,
    and the reference's when it is built here."""
    import oracle
    import paper_1803_11301_b200 as pkg
    c, r, i = pkg.tables64()
    assert np.array_equal(c, port.cantor_basis(64)[0::2])
    pr, pi = port.encode_matrix(64)
    assert np.array_equal(r, pr[0::2]) and np.array_equal(i, pi[0::2])
    if oracle.have_ref():
        rc, rr, ri = oracle.ref().tables64()
        assert np.array_equal(c, rc) and np.array_equal(r, rr) and np.array_equal(i, ri)


@pytest.mark.parametrize("m", [128, 64])
def test_tower_representation_host_side(port, m):
    """The product pipeline's internal tower representation (csrc/tower.cuh; fpm_tower_tables):
    GF(2^m) over its subfield GF(2^8) with basis x^j t^s.  Checked with the oracle port's field
    arithmetic: t is a root of y^8+y^4+y^3+y+1 inside span(v_0..v_7), to_poly[8j+s] = x^j t^s,
    to_r inverts it, tau are the tower coordinates of v_1..v_7, and multiplying by a subfield
    element is the byte-wise GF(2^8) product in tower coordinates (what smul_w computes)."""
    import paper_1803_11301_b200 as pkg
    t, to_poly, to_r, tau = pkg.tower_tables(m)
    mul = lambda a, b: port.pointwise(m, np.asarray(a, np.uint64), np.asarray(b, np.uint64))  # noqa: E731
    one, x = np.array([1, 0], np.uint64), np.array([2, 0], np.uint64)

    def pw(a, e):
        r = one
        for _ in range(e):
            r = mul(r, a)
        return r
    assert not np.any(pw(t, 8) ^ pw(t, 4) ^ pw(t, 3) ^ t ^ one)
    cantor = port.cantor_basis(m).reshape(-1, 2)

    sub = {0}  # span(v_0..v_7) = GF(2^8)
    for c in cantor[:8]:
        sub |= {e ^ (int(c[0]) | int(c[1]) << 64) for e in sub}
    assert len(sub) == 256 and (int(t[0]) | int(t[1]) << 64) in sub
    xj = one
    for j in range(m // 8):
        ts = one
        for s in range(8):
            assert np.array_equal(to_poly[8 * j + s], ts if j == 0 else mul(xj, ts)), (j, s)
            ts = mul(ts, t)
        xj = mul(xj, x)

    def conv(v, rows):  # row-vector times matrix over GF(2)
        acc = np.zeros(2, np.uint64)
        bits = int(v[0]) | int(v[1]) << 64
        for k in range(m):
            if bits >> k & 1:
                acc ^= rows[k]
        return acc
    for k in range(m):
        unit = np.zeros(2, np.uint64)
        unit[k // 64] = np.uint64(1) << np.uint64(k % 64)
        assert np.array_equal(conv(to_poly[k], to_r), unit)
    for b in range(7):
        r = conv(cantor[b + 1], to_r)
        assert int(r[1]) == 0 and int(r[0]) == int(tau[b])

    def gf8(a, b):
        r = 0
        for i in range(8):
            if b >> i & 1:
                r ^= a
            a <<= 1
            if a & 0x100:
                a ^= 0x11B
        return r
    rng = np.random.default_rng(m)
    for _ in range(8):
        u = rng.integers(0, 2**63, 2, dtype=np.uint64)
        if m == 64:
            u[1] = 0
        d = int(rng.integers(1, 128))
        dpoly = np.zeros(2, np.uint64)
        for b in range(7):
            if d >> b & 1:
                dpoly ^= cantor[b + 1]
        ur = conv(u, to_r)
        dr = int(conv(dpoly, to_r)[0])
        want = bytes(gf8(c, dr) for c in ur.tobytes()[: m // 8])
        assert conv(mul(u, dpoly), to_r).tobytes()[: m // 8] == want


def test_shard_fast_path_threshold_host_side():
    """fpm_shard_tower: a coset of 2^l elements runs the single-GPU tower pipeline exactly when the
    product pipeline would (l >= 18: tile depth 10, both operands fused, tower tiles).  Host only."""
    import paper_1803_11301_b200._lib as L
    f = L.lib().fpm_shard_tower
    assert [f(l) for l in (8, 14, 17, 18, 19, 22, 26, 30)] == [0, 0, 0, 1, 1, 1, 1, 1]


def test_random_bitpoly_matches_reference_generator(port):
    """fpm_random_bitpoly = random_bitpoly(n, mt19937_64(seed)) (bitpoly.cpp:19-24), host only: the
    seeded inputs bench.py feeds the GPU are the ones the golden hashes were made from."""
    import paper_1803_11301_b200 as pkg
    for bits, seed in ((1, 3), (64, 20261020), (1000, 20261021), (65536, 30000), (123457, 40007)):
        assert np.array_equal(pkg.random_bitpoly(bits, seed), port.random_bitpoly(bits, seed)), (bits, seed)
    assert pkg.random_bitpoly(0, 1).size == 0


def test_batch_shard_partitions_the_batch():
    from paper_1803_11301_b200.dist import batch_shard
    for count in (1, 7, 4096):
        for P in (1, 2, 3, 8):
            got = [batch_shard(count, P, r) for r in range(P)]
            assert sum(n for _, n in got) == count
            assert all(got[r][0] + got[r][1] == got[r + 1][0] for r in range(P - 1))
            assert max(n for _, n in got) - min(n for _, n in got) <= 1
