"""GPU parity: every stage and the full product through the C-ABI, bit-exact against the oracle
(the reference library compiled from /root/reference when present, else our C restatement)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def rnd_words(rng, bits):
    w = rng.integers(0, 2**63, size=max(1, (bits + 63) // 64), dtype=np.uint64) * np.uint64(2) \
        + rng.integers(0, 2, size=max(1, (bits + 63) // 64), dtype=np.uint64)
    if bits % 64:
        w[-1] &= np.uint64((1 << (bits % 64)) - 1)
    return w[: (bits + 63) // 64] if bits else w[:0]


def test_tables_match(gpu, port):
    c, r, i = gpu.tables128()
    assert np.array_equal(c, port.cantor_basis(128))
    pr, pi = port.encode_matrix(128)
    assert np.array_equal(r, pr) and np.array_equal(i, pi)


def test_gf128_mul(gpu, checker):
    rng = np.random.default_rng(13)
    u = rnd_words(rng, 128 * 4096)
    v = rnd_words(rng, 128 * 4096)
    assert np.array_equal(gpu.gf128_mul(u, v), checker.pointwise(u, v))
    one = np.zeros_like(u)
    one[0::2] = 1
    assert np.array_equal(gpu.gf128_mul(u, one), u)


@pytest.mark.parametrize("lg", list(range(2, 29)))
def test_basis_cvt_roundtrip(gpu, checker, lg):
    n = 1 << lg
    rng = np.random.default_rng(lg)
    w = rnd_words(rng, n)
    fwd = gpu.basis_cvt(w, n)
    assert np.array_equal(fwd, checker.basis_cvt(w, n)), "forward"
    back = gpu.i_basis_cvt(fwd, n)
    assert np.array_equal(back, w), "inverse"
    # declared zero tail (basis_convert.cpp:337-341)
    for content in (n // 2, 3 * n // 8, 1):
        z = rnd_words(rng, content)
        zz = np.zeros(max(1, n // 64), np.uint64)
        zz[: z.size] = z
        assert np.array_equal(gpu.basis_cvt(zz, n, content), checker.basis_cvt(zz, n)), content


@pytest.mark.parametrize("l", [0, 1, 3, 5, 9, 10, 11, 13, 15])
def test_encode_decode(gpu, checker, l):
    rng = np.random.default_rng(100 + l)
    a = rnd_words(rng, 128 << l)
    ev = gpu.encode(a, l)
    assert np.array_equal(ev, checker.encode(a, l))
    assert np.array_equal(gpu.decode(ev, l), a)


@pytest.mark.parametrize("l", [1, 2, 4, 7, 10, 12, 13, 14, 16, 17, 18, 19])
def test_butterfly(gpu, checker, l):
    rng = np.random.default_rng(200 + l)
    ev = rnd_words(rng, 128 << l)
    f = gpu.lch_butterfly(ev, l)
    assert np.array_equal(f, checker.butterfly(ev, l)), "forward"
    assert np.array_equal(gpu.i_lch_butterfly(f, l), ev), "inverse"


@pytest.mark.parametrize("tile", [9, 11, 12])
def test_butterfly_tile_depths(tile):
    """Every shared-memory tile depth (odd ones leave a single radix-2 top layer) gives the same
    transform: run the product in a child process with the FPM_TILE_LOG2 override."""
    import os
    import subprocess
    import sys
    code = (
        "import numpy as np, oracle, paper_1803_11301_b200 as g\n"
        "P = oracle.port()\n"
        "for l in (15, 18):\n"
        "    rng = np.random.default_rng(l)\n"
        "    ev = rng.integers(0, 2**63, size=2 << l, dtype=np.uint64)\n"
        "    f = g.lch_butterfly(ev, l)\n"
        "    assert np.array_equal(f, P.butterfly(128, ev, l, False)), l\n"
        "    assert np.array_equal(g.i_lch_butterfly(f, l), ev), l\n"
        "print('ok')\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True, timeout=600,
                       env=dict(os.environ, FPM_TILE_LOG2=str(tile)))
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


@pytest.mark.parametrize("env", [{}, {"FPM_FUSE_AB": "0"}, {"FPM_TOWER": "0"}, {"FPM_TILE_LOG2": "11", "FPM_TILE_LOG2_64": "12"},
                                 {"FPM_TILE_LOG2": "10", "FPM_TILE_LOG2_64": "10", "FPM_FUSE_AB": "0"},
                                 {"FPM_TILE_LOG2": "12", "FPM_TILE_LOG2_64": "11"}])
@pytest.mark.parametrize("field", [128, 64])
def test_pipeline_schedules(checker, port, env, field):
    """Every tile schedule of the product pipeline -- both operands' tile layers fused into the
    pointwise pass on tower-representation tiles (default), the same on polynomial-representation
    tiles, operand a in its own tile pass, other depths -- gives the reference
    product (child process per environment; l = 18 and 20)."""
    import hashlib
    import os
    import subprocess
    import sys
    shapes = [(1 << 24, (1 << 24) - 3), ((1 << 26) - 5, 1 << 25)]
    code = (
        "import hashlib, oracle, paper_1803_11301_b200 as g\n"
        "P = oracle.port()\n"
        f"for la, lb in {shapes!r}:\n"
        "    a, b = P.random_bitpoly(la, 11 + la), P.random_bitpoly(lb, 13 + lb)\n"
        f"    c = g.fp_polymul(a, la, b, lb, field={field})\n"
        "    print(hashlib.blake2b(c.tobytes(), digest_size=16).hexdigest())\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True, timeout=900,
                       env=dict(os.environ, **env))
    assert r.returncode == 0, r.stderr[-2000:]
    got = r.stdout.split()
    for (la, lb), h in zip(shapes, got):
        a, b = port.random_bitpoly(la, 11 + la), port.random_bitpoly(lb, 13 + lb)
        want = hashlib.blake2b(checker.polymul(a, la, b, lb).tobytes(), digest_size=16).hexdigest()
        assert h == want, (env, la, lb)


SHAPES = [(1, 1), (1, 5), (63, 64), (64, 64), (100, 3000), (4095, 4096), (5000, 3000), (1 << 12, 1 << 12),
          (1 << 14, (1 << 14) - 17), (1 << 16, 1 << 16), ((1 << 16) + 1, 9), ((1 << 17) - 3, (1 << 16) + 5),
          (1 << 18, 1 << 18), (300000, 1 << 19), (1 << 20, 1 << 20), ((1 << 20) + 77, 12345)]


@pytest.mark.parametrize("la,lb", SHAPES)
def test_polymul_shapes(gpu, checker, port, la, lb):
    a = port.random_bitpoly(la, 1000 + la)
    b = port.random_bitpoly(lb, 2000 + lb)
    got = gpu.fp_polymul(a, la, b, lb, field=gpu.FIELD_GF128)
    assert np.array_equal(got, checker.polymul(a, la, b, lb))


@pytest.mark.parametrize("la,lb", SHAPES)
def test_polymul_shapes_gf64(gpu, checker, port, la, lb):
    """The GF(2^64) pipeline (run_pipeline<gf64>, the reference's auto field) gives the same product."""
    a = port.random_bitpoly(la, 3000 + la)
    b = port.random_bitpoly(lb, 4000 + lb)
    want = checker.polymul(a, la, b, lb)
    assert np.array_equal(gpu.fp_polymul(a, la, b, lb, field=gpu.FIELD_GF64), want)
    assert np.array_equal(gpu.fp_polymul(a, la, b, lb, field=gpu.FIELD_AUTO), want)


@pytest.mark.parametrize("lg", [21, 23, 24])
def test_polymul_gf64_large(gpu, checker, port, lg):
    la = 1 << lg
    a = port.random_bitpoly(la, 5000 + lg)
    b = port.random_bitpoly(la - 3, 6000 + lg)
    assert np.array_equal(gpu.fp_polymul(a, la, b, la - 3, field=gpu.FIELD_GF64), checker.polymul(a, la, b, la - 3))


def test_polymul_edge_values(gpu, port):
    # identity, monomial shift, zero, empty (test_polymul.cpp:50-66)
    one = np.array([1], np.uint64)
    b = port.random_bitpoly(50000, 6)
    assert np.array_equal(gpu.fp_polymul(one, 1, b, 50000), b)
    xa = np.zeros(16, np.uint64); xa[1000 // 64] = np.uint64(1 << (1000 % 64))
    xb = np.zeros(65, np.uint64); xb[4096 // 64] = np.uint64(1)
    prod = gpu.fp_polymul(xa, 1001, xb, 4097)
    assert prod.size == (1001 + 4097 - 1 + 63) // 64
    nz = np.flatnonzero(prod)
    assert nz.tolist() == [(1000 + 4096) // 64] and int(prod[nz[0]]) == 1 << ((1000 + 4096) % 64)
    assert gpu.fp_polymul(np.zeros(0, np.uint64), 0, b, 50000).size == 0
    assert not gpu.fp_polymul(b, 50000, np.zeros(1, np.uint64), 17).any()


def test_batch(gpu, port, checker):
    import torch
    la = lb = 1 << 16
    count = 64
    A = np.stack([port.random_bitpoly(la, 7000 + k) for k in range(count)])
    B = np.stack([port.random_bitpoly(lb, 9000 + k) for k in range(count)])
    wa, wb, wc = A.shape[1], B.shape[1], (la + lb - 1 + 63) // 64
    dA = torch.from_numpy(A.view(np.int64)).cuda()
    dB = torch.from_numpy(B.view(np.int64)).cuda()
    dC = torch.zeros((count, wc), dtype=torch.int64, device="cuda")
    gpu.fp_polymul_batch_dev(dA, la, wa, dB, lb, wb, dC, wc, count)
    torch.cuda.synchronize()
    C = dC.cpu().numpy().view(np.uint64)
    for k in (0, 1, count - 1):
        assert np.array_equal(C[k], checker.polymul(A[k], la, B[k], lb)), k


@pytest.mark.parametrize("la,lb,count", [((1 << 16) - 5, 40000, 64), (33000, 1 << 16, 100)])
def test_batch_ragged_operands_tower_path(gpu, checker, la, lb, count):
    """Batches of >= 64 2^17-bit products run the tower-representation batch pipeline (encode in
    the tower representation, one tower tile pass tile per product, decode, the 2^17-bit inverse):
    ragged operand lengths (tail masking, the product trimmed to la + lb - 1 bits) and strides wider
    than the operands, against the oracle."""
    import torch
    A = np.zeros((count, 1100), np.uint64)
    B = np.zeros((count, 1030), np.uint64)
    for k in range(count):
        a = gpu.random_bitpoly(la, 500 + k)
        b = gpu.random_bitpoly(lb, 900 + k)
        A[k, :len(a)] = a
        B[k, :len(b)] = b
        A[k, len(a):] = 0xFFFFFFFFFFFFFFFF  # beyond the operand: must be ignored
    wc = (la + lb - 1 + 63) // 64
    dA = torch.from_numpy(A.view(np.int64)).cuda()
    dB = torch.from_numpy(B.view(np.int64)).cuda()
    dC = torch.zeros((count, wc + 3), dtype=torch.int64, device="cuda")
    gpu.fp_polymul_batch_dev(dA, la, 1100, dB, lb, 1030, dC, wc + 3, count)
    torch.cuda.synchronize()
    C = dC.cpu().numpy().view(np.uint64)
    for k in (0, 1, count // 2, count - 1):
        a = A[k, :(la + 63) // 64].copy()
        if la % 64:
            a[-1] &= (1 << (la % 64)) - 1
        assert np.array_equal(C[k, :wc], checker.polymul(a, la, B[k, :(lb + 63) // 64], lb)), k
        assert not C[k, wc:].any(), k  # nothing written past the product


@pytest.mark.parametrize("count,la,lb", [(300, 1 << 16, (1 << 16) - 9), (40, 20000, 30000)])
def test_batch_host_buffers_pipelined(gpu, checker, count, la, lb):
    """fpm_polymul_batch (host buffers): chunks of >= 64 products with uploads, products and
    downloads overlapped over three device slots (300 products: 5 chunks, every slot reused),
    strided host arrays; equal to the device-buffer batch and the oracle."""
    import torch
    sa, sb = (la + 63) // 64 + 3, (lb + 63) // 64 + 1
    wc = (la + lb - 1 + 63) // 64
    sc = wc + 2
    A = np.zeros(count * sa, np.uint64)
    B = np.zeros(count * sb, np.uint64)
    for k in range(count):
        a = gpu.random_bitpoly(la, 3000 + k)
        b = gpu.random_bitpoly(lb, 4000 + k)
        A[k * sa:k * sa + len(a)] = a
        B[k * sb:k * sb + len(b)] = b
    C = np.zeros(count * sc, np.uint64)
    gpu.fp_polymul_batch(A, la, sa, B, lb, sb, C, sc, count)
    dC = torch.zeros(count * sc, dtype=torch.int64, device="cuda")
    gpu.fp_polymul_batch_dev(torch.from_numpy(A.view(np.int64)).cuda(), la, sa, torch.from_numpy(B.view(np.int64)).cuda(),
                             lb, sb, dC, sc, count)
    torch.cuda.synchronize()
    D = dC.cpu().numpy().view(np.uint64)
    for k in range(count):
        assert np.array_equal(C[k * sc:k * sc + wc], D[k * sc:k * sc + wc]), k
    for k in (0, count - 1):
        want = checker.polymul(A[k * sa:k * sa + (la + 63) // 64], la, B[k * sb:k * sb + (lb + 63) // 64], lb)
        assert np.array_equal(C[k * sc:k * sc + wc], want), k


def _cfg2(gpu):
    import hashlib
    import json
    import os
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_meta.json")) as f:
        meta = json.load(f)["cfg2_batch"]
    bits, count = meta["a_bits"], meta["count"]
    A = np.concatenate([gpu.random_bitpoly(bits, 30000 + k) for k in range(count)])
    B = np.concatenate([gpu.random_bitpoly(bits, 40000 + k) for k in range(count)])
    h = lambda w: hashlib.blake2b(np.ascontiguousarray(w, np.uint64).tobytes(), digest_size=16).hexdigest()
    return meta, bits, count, A, B, h


def test_batch_config2_all_products(gpu):
    """BASELINE config 2 in full: the 4096 products of fpm_polymul_batch_dev (one launch) hash to the
    reference's own 4096 fp_polymul products (tests/golden/make_golden.py, polymul.cpp:223-239)."""
    import torch
    meta, bits, count, A, B, h = _cfg2(gpu)
    wc = meta["product_words"]
    dA = torch.from_numpy(A.view(np.int64)).cuda()
    dB = torch.from_numpy(B.view(np.int64)).cuda()
    dC = torch.full((count * wc,), -1, dtype=torch.int64, device="cuda")
    gpu.fp_polymul_batch_dev(dA, bits, bits // 64, dB, bits, bits // 64, dC, wc, count)
    torch.cuda.synchronize()
    C = dC.cpu().numpy().view(np.uint64)
    assert h(C[:wc]) == meta["blake2b128_first"]
    assert h(C) == meta["blake2b128_all"]


@pytest.mark.parametrize("P", [2, 3, 8])
def test_batch_config2_split_thread_ranks(gpu, P):
    """bench.py's config-2 split (dist.polymul_batch_sharded: contiguous, uneven when P does not
    divide the batch) with P host threads as ranks on one GPU, each writing only its rows of the
    shared product tensor; the assembled batch hashes to the reference's."""
    import threading
    import torch
    from paper_1803_11301_b200.dist import batch_shard, polymul_batch_sharded
    meta, bits, count, A, B, h = _cfg2(gpu)
    wc = meta["product_words"]
    dA = torch.from_numpy(A.view(np.int64)).cuda()
    dB = torch.from_numpy(B.view(np.int64)).cuda()
    dC = torch.full((count * wc,), -1, dtype=torch.int64, device="cuda")
    assert sum(batch_shard(count, P, r)[1] for r in range(P)) == count
    errs = []

    def run(rank):
        try:
            torch.cuda.set_device(0)
            with torch.cuda.stream(torch.cuda.Stream()):
                polymul_batch_sharded(dA, bits, dB, bits, dC, count, P, rank)
                torch.cuda.current_stream().synchronize()
        except Exception as e:  # pragma: no cover - reported below
            errs.append((rank, repr(e)))

    th = [threading.Thread(target=run, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not errs, errs
    torch.cuda.synchronize()
    assert h(dC.cpu().numpy().view(np.uint64)) == meta["blake2b128_all"]


# ---------------------------------------------------------------- GF(2^64) stages (auto field)
def _ref64_or_port(port):
    import oracle
    if oracle.have_ref():
        R = oracle.ref()

        class _R:
            encode = staticmethod(lambda a, l: R.encode64(a, l))
            decode = staticmethod(lambda e, l: R.decode64(e, l))
            butterfly = staticmethod(lambda e, l, base=None, inv=False: R.butterfly64(e, l, base, inv))
            pointwise = staticmethod(lambda u, v: R.pointwise64(u, v))
        return _R()

    class _P:  # the port keeps GF(2^64) elements as {lo, hi = 0}
        encode = staticmethod(lambda a, l: port.encode(64, a, l)[0::2].copy())
        decode = staticmethod(lambda e, l: port.decode(64, np.stack([e, np.zeros_like(e)], 1).ravel(), l))
        butterfly = staticmethod(lambda e, l, base=None, inv=False: port.butterfly(
            64, np.stack([e, np.zeros_like(e)], 1).ravel(), l, inv)[0::2].copy())
        pointwise = staticmethod(lambda u, v: port.pointwise(
            64, np.stack([u, np.zeros_like(u)], 1).ravel(), np.stack([v, np.zeros_like(v)], 1).ravel())[0::2].copy())
    return _P()


@pytest.mark.parametrize("l", [0, 3, 9, 10, 14, 16])
def test_encode_decode64(gpu, port, l):
    chk = _ref64_or_port(port)
    rng = np.random.default_rng(900 + l)
    a = rnd_words(rng, 64 << l)
    ev = gpu.encode64(a, l)
    assert np.array_equal(ev, chk.encode(a, l))
    assert np.array_equal(gpu.decode64(ev, l), a)
    assert np.array_equal(gpu.decode64(ev, l), chk.decode(ev, l))


@pytest.mark.parametrize("l", [1, 4, 7, 8, 9, 12, 13, 16, 19])
def test_butterfly64(gpu, port, l):
    chk = _ref64_or_port(port)
    rng = np.random.default_rng(950 + l)
    ev = rnd_words(rng, 64 << l)
    f = gpu.lch_butterfly64(ev, l)
    assert np.array_equal(f, chk.butterfly(ev, l)), "forward"
    assert np.array_equal(gpu.lch_butterfly64(f, l, inverse=True), ev), "inverse"


def test_butterfly64_any_base(gpu, ref):
    rng = np.random.default_rng(77)
    l = 13
    ev = rnd_words(rng, 64 << l)
    base = (1 << 45) | (0x1234 << 20)  # an arbitrary coset of a sub-FFT
    assert np.array_equal(gpu.lch_butterfly64(ev, l, base=base), ref.butterfly64(ev, l, base=base))
    assert np.array_equal(gpu.lch_butterfly64(ev, l, base=base, inverse=True),
                          ref.butterfly64(ev, l, base=base, inverse=True))


def test_pointwise64(gpu, port):
    chk = _ref64_or_port(port)
    rng = np.random.default_rng(31)
    u = rnd_words(rng, 64 * 5000)
    v = rnd_words(rng, 64 * 5000)
    assert np.array_equal(gpu.pointwise64(u, v), chk.pointwise(u, v))


def test_largest_shapes_fields_agree(gpu):
    """2^33-bit x (2^33 - 337)-bit product (n = 2^34: two top basis-conversion passes, 28/27 FFT
    layers): the GF(2^64) and GF(2^128) transforms give the same product; an all-ones-by-x^k probe
    checks the same path against a closed form."""
    import torch
    n = 1 << 33
    g = torch.Generator(device="cuda").manual_seed(3)
    a = torch.randint(-(1 << 62), 1 << 62, (n // 64,), generator=g, device="cuda", dtype=torch.int64)
    nb = n - 5 * 64 - 17
    b = torch.randint(-(1 << 62), 1 << 62, ((nb + 63) // 64,), generator=g, device="cuda", dtype=torch.int64)
    b[-1] &= (1 << (nb % 64)) - 1
    out = (n + nb - 1 + 63) // 64
    c1 = torch.empty(out, dtype=torch.int64, device="cuda")
    c2 = torch.empty(out, dtype=torch.int64, device="cuda")
    gpu.fp_polymul_dev(a, n, b, nb, c1, field=gpu.FIELD_GF128)
    gpu.fp_polymul_dev(a, n, b, nb, c2, field=gpu.FIELD_GF64)
    torch.cuda.synchronize()
    assert torch.equal(c1, c2)
    # (x^k) * b = b shifted by k bits, through the same 2^34-bit transform
    k = 3 * 64 + 5
    xk = torch.zeros((k + 1 + 63) // 64, dtype=torch.int64, device="cuda")
    xk[k // 64] = 1 << (k % 64)
    c3 = torch.empty((k + 1 + nb - 1 + 63) // 64, dtype=torch.int64, device="cuda")
    gpu.fp_polymul_dev(b, nb, xk, k + 1, c3, field=gpu.FIELD_GF128)
    torch.cuda.synchronize()
    bb = b.cpu().numpy().view(np.uint64)
    got = c3.cpu().numpy().view(np.uint64)
    want = np.zeros(got.size + 1, np.uint64)
    q, r = k // 64, np.uint64(k % 64)
    want[q: q + bb.size] ^= bb << r
    want[q + 1: q + 1 + bb.size] ^= bb >> (np.uint64(64) - r)
    assert np.array_equal(got, want[: got.size]) and not want[got.size:].any()


# ---------------------------------------------------------------- BASELINE configs vs the reference
def _meta():
    import json
    import os
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_meta.json")) as f:
        return json.load(f)["configs"]


@pytest.mark.parametrize("key", ["1048576x1048576", "16777216x16777216", "16777216x8400953",
                                 "268435456x268435456", "4294967296x4294967296"])
def test_baseline_config_products_match_reference_hashes(gpu, port, key):
    """BASELINE configs 1, 3 (equal and unequal), 4 and 5 on the seeded inputs: blake2b-128 of the
    GPU product (both fields) equals the hash of the reference library's product
    (tests/golden/make_golden.py; config 5 with the F4-patched reference build)."""
    import hashlib
    import torch
    c = _meta()[key]
    a = port.random_bitpoly(c["a_bits"], c["seed_a"])
    b = port.random_bitpoly(c["b_bits"], c["seed_b"])
    da = torch.from_numpy(a.view(np.int64)).cuda()
    db = torch.from_numpy(b.view(np.int64)).cuda()
    dc = torch.empty((c["product_bits"] + 63) // 64, dtype=torch.int64, device="cuda")
    for field in (gpu.FIELD_GF128, gpu.FIELD_GF64):
        gpu.fp_polymul_dev(da, c["a_bits"], db, c["b_bits"], dc, field=field)
        torch.cuda.synchronize()
        got = hashlib.blake2b(dc.cpu().numpy().view(np.uint64).tobytes(), digest_size=16).hexdigest()
        assert got == c["blake2b128"], field


def test_config5_host_buffers_match_reference_hash(gpu, port):
    """BASELINE config 5 through the host-buffer entry fpm_polymul (the e2e path: operand b's upload
    overlapping operand a's transforms, the upper 2^32-bit block decoded and converted first -- the
    split decode -- and copied out while the lower block converts): the reference's product hash."""
    import hashlib
    c = _meta()["4294967296x4294967296"]
    a = port.random_bitpoly(c["a_bits"], c["seed_a"])
    b = port.random_bitpoly(c["b_bits"], c["seed_b"])
    got = gpu.fp_polymul(a, c["a_bits"], b, c["b_bits"], field=gpu.FIELD_GF128)
    assert hashlib.blake2b(got.tobytes(), digest_size=16).hexdigest() == c["blake2b128"]


@pytest.mark.parametrize("frac", ["0.5", "1.0", "0.13"])
def test_host_buffers_operand_a_pre_pass(port, frac):
    _pre_pass_case(frac, "FIELD_GF128")


@pytest.mark.parametrize("frac", ["0.5", "1.0"])
def test_host_buffers_operand_a_pre_pass_gf64(port, frac):
    """The same for the GF(2^64) pipeline (fft64_tile_tower_kernel modes 2 / 1)."""
    _pre_pass_case(frac, "FIELD_GF64")


def _pre_pass_case(frac, field):
    """Host-buffer products run part of operand a's tower tile layers ahead of the fused pass
    (fft_tile_tower_kernel modes 2 / 1, FPM_PRE_A_FRAC) while operand b is uploaded; by default only
    2^33-bit products do.  Forced here at l = 22 / 23 (tile depth 12) for several shares, including
    every tile: BASELINE config 4's reference hash and a ragged shape against the device-resident
    product of the default schedule (child process: the knobs are read once)."""
    import hashlib
    import os
    import subprocess
    import sys
    c = _meta()["268435456x268435456"]
    la, lb = (1 << 29) - 12345, (1 << 28) + 777
    code = (
        "import hashlib, numpy as np, torch, paper_1803_11301_b200 as g\n"
        f"a, b = g.random_bitpoly({c['a_bits']}, {c['seed_a']}), g.random_bitpoly({c['b_bits']}, {c['seed_b']})\n"
        f"p = g.fp_polymul(a, {c['a_bits']}, b, {c['b_bits']}, field=g.{field})\n"
        "print(hashlib.blake2b(p.tobytes(), digest_size=16).hexdigest())\n"
        f"a, b = g.random_bitpoly({la}, 71), g.random_bitpoly({lb}, 72)\n"
        f"p = g.fp_polymul(a, {la}, b, {lb}, field=g.{field})\n"
        "da, db = (torch.from_numpy(x.view(np.int64)).cuda() for x in (a, b))\n"
        "dc = torch.empty(p.size, dtype=torch.int64, device='cuda')\n"
        f"g.fp_polymul_dev(da, {la}, db, {lb}, dc, field=g.FIELD_GF128)\n"
        "torch.cuda.synchronize()\n"
        "print(bool(np.array_equal(dc.cpu().numpy().view(np.uint64), p)))\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True, timeout=900,
                       env=dict(os.environ, FPM_PRE_A_FRAC=frac, FPM_PRE_A_MIN_L="22"))
    assert r.returncode == 0, r.stderr[-2000:]
    out = r.stdout.split()
    assert out[0] == c["blake2b128"], frac
    assert out[1] == "True", frac


def _edge_operand(port, kind, bits, seed):
    w = port.random_bitpoly(bits, seed)
    if kind == "sparse":  # density 1/64: AND of six uniform words
        for k in range(1, 6):
            w &= port.random_bitpoly(bits, seed + 1000 * k)
    elif kind == "ones":
        w[:] = np.uint64(0xFFFFFFFFFFFFFFFF)
        if bits % 64:
            w[-1] = np.uint64((1 << (bits % 64)) - 1)
    elif kind == "top":  # exact degree: bit N-1 forced
        w[(bits - 1) // 64] |= np.uint64(1) << np.uint64((bits - 1) % 64)
    return w


@pytest.mark.parametrize("kind", ["sparse", "ones", "top"])
def test_config3_edge_shapes_vs_reference(gpu, ref, port, kind):
    """Config 3's edge shapes at ~2^24 bits, bit-exact against the reference library."""
    la, lb = 1 << 24, (1 << 23) + 12345
    a = _edge_operand(port, kind, la, 71)
    b = _edge_operand(port, kind, lb, 72)
    want = ref.polymul(a, la, b, lb, field=0)
    for field in (gpu.FIELD_GF128, gpu.FIELD_GF64):
        assert np.array_equal(gpu.fp_polymul(a, la, b, lb, field=field), want), (kind, field)


@pytest.mark.parametrize("lg", [28, 32, 33, 34])
def test_basis_cvt_large_roundtrip_and_linearity(gpu, lg):
    """Conversions beyond the oracle's reach (the 2D tile path, the fused 2^33 top pass, the generic
    top passes above it): inverse(forward(x)) = x and forward is GF(2)-linear."""
    import torch
    n = 1 << lg
    g = torch.Generator(device="cuda").manual_seed(lg)
    x = torch.randint(-(1 << 62), 1 << 62, (n // 64,), generator=g, device="cuda", dtype=torch.int64)
    y = torch.randint(-(1 << 62), 1 << 62, (n // 64,), generator=g, device="cuda", dtype=torch.int64)
    fx, fy, fs = x.clone(), y.clone(), x ^ y
    for t in (fx, fy, fs):
        gpu.stage_dev("basis_cvt", t, n, n)
    torch.cuda.synchronize()
    assert torch.equal(fx ^ fy, fs), "linearity"
    gpu.stage_dev("i_basis_cvt", fx, n)
    torch.cuda.synchronize()
    assert torch.equal(fx, x), "round trip"


def test_concurrent_host_calls(gpu, checker):
    """The reference's fp_polymul is safe to call from several threads (its per-field singletons and
    the twiddle-plan cache are mutex-guarded, cantor.cpp:136-140, polymul.cpp:63-74); so is ours:
    four host threads, mixed sizes (tiny shapes use the lazily uploaded row tables) and fields,
    every product checked."""
    import concurrent.futures as cf
    rng = np.random.default_rng(77)
    jobs = []
    for k in range(24):
        la = int(rng.choice([7, 300, 4096, 70000, 1 << 20]))
        lb = int(rng.choice([5, 129, 4096, 1 << 18]))
        a, b = rnd_words(rng, la), rnd_words(rng, lb)
        field = [gpu.FIELD_GF128, gpu.FIELD_GF64, gpu.FIELD_AUTO][k % 3]
        jobs.append((a, la, b, lb, field))
    with cf.ThreadPoolExecutor(4) as ex:
        got = list(ex.map(lambda j: gpu.fp_polymul(j[0], j[1], j[2], j[3], field=j[4]), jobs))
    for (a, la, b, lb, _), g in zip(jobs, got):
        assert np.array_equal(g, checker.polymul(a, la, b, lb)), (la, lb)


def test_concurrent_host_calls_leased_streams(gpu, checker):
    """Host-buffer products above the staged size lease a stream set per call (pipeline, upload and
    download streams; four sets per device) so one caller's PCIe copies overlap another's kernels.
    Six threads (more callers than sets: two wait for a lease) on 2^23..2^26-bit operands in both
    fields; every product against the reference."""
    import concurrent.futures as cf
    rng = np.random.default_rng(78)
    jobs = []
    for k in range(12):
        la = int(rng.choice([1 << 23, (1 << 24) + 77, 1 << 25, (1 << 26) - 5]))
        lb = int(rng.choice([1 << 22, (1 << 24) - 1, 1 << 25]))
        jobs.append((rnd_words(rng, la), la, rnd_words(rng, lb), lb, [gpu.FIELD_GF128, gpu.FIELD_AUTO][k % 2]))
    with cf.ThreadPoolExecutor(6) as ex:
        got = list(ex.map(lambda j: gpu.fp_polymul(j[0], j[1], j[2], j[3], field=j[4]), jobs))
    for (a, la, b, lb, _), g in zip(jobs, got):
        assert np.array_equal(g, checker.polymul(a, la, b, lb)), (la, lb)


@pytest.mark.parametrize("la,lb", [(1, 1), (63, 64), (64, 65), (4095, 4095), (4096, 100), (700, 9000),
                                   (100_000, 77_777), (1 << 20, (1 << 19) + 3)])
def test_karatsuba_mul(gpu, checker, la, lb):
    """karatsuba_mul / naive_mul (polymul.cpp:268-282, polymul.hpp:83-87): the word-level GPU
    product, an algorithm independent of the FFT path, equals the reference product."""
    rng = np.random.default_rng(la * 7 + lb)
    a, b = rnd_words(rng, la), rnd_words(rng, lb)
    want = checker.polymul(a, la, b, lb)
    assert np.array_equal(gpu.karatsuba_mul(a, la, b, lb), want)
    if la < 4096 and lb < 4096:  # the reference's auto-mode bypass (polymul.cpp:226-231)
        assert np.array_equal(gpu.fp_polymul(a, la, b, lb, field=gpu.FIELD_AUTO), want)
    # garbage above the declared length is ignored, as for fp_polymul
    ga, gb = a.copy(), b.copy()
    if la % 64:
        ga[-1] |= np.uint64(~((1 << (la % 64)) - 1) & (2**64 - 1))
    if lb % 64:
        gb[-1] |= np.uint64(~((1 << (lb % 64)) - 1) & (2**64 - 1))
    assert np.array_equal(gpu.karatsuba_mul(ga, la, gb, lb), want)


def test_clmul_words_dev(gpu, checker):
    """naive_mul_words_kernel (detail/kernels.hpp:115-118) on device tensors: full words, out
    overwritten (stale contents must not leak in)."""
    import torch
    rng = np.random.default_rng(5)
    for wa, wb in [(1, 1), (3, 700), (256, 256), (257, 255), (1000, 3000)]:
        a, b = rnd_words(rng, 64 * wa), rnd_words(rng, 64 * wb)
        ta = torch.from_numpy(a.view(np.int64)).cuda()
        tb = torch.from_numpy(b.view(np.int64)).cuda()
        out = torch.full((wa + wb,), -1, dtype=torch.int64, device="cuda")
        gpu.clmul_words_dev(ta, tb, out)
        torch.cuda.synchronize()
        got = out.cpu().numpy().view(np.uint64)
        want = np.zeros(wa + wb, np.uint64)
        w = checker.polymul(a, 64 * wa, b, 64 * wb)
        want[: w.size] = w
        assert np.array_equal(got, want), (wa, wb)


@pytest.mark.parametrize("la,lb", [(1 << 28, (1 << 27) + 12345), ((1 << 28) - 77, 1 << 28), (1 << 32, (1 << 31) + 999)])
def test_concurrent_conversions_device_resident_vs_reference(gpu, ref, la, lb):
    """Device-resident products of >= 2^28 bits convert the two operands on two streams (operand b in
    the upper half of the work array, zero-filled when it does not fill its conversion) and the two
    inverse 2^32-bit blocks of a 2^33-bit product concurrently: unequal and ragged operands,
    bit-exact against the reference library (the F4 build at 2^33 bits)."""
    import oracle
    import torch
    a = gpu.random_bitpoly(la, 91)
    b = gpu.random_bitpoly(lb, 92)
    R = oracle.ref(f4=True) if la + lb > (1 << 32) else ref
    want = R.polymul(a, la, b, lb, field=0)
    da = torch.from_numpy(a.view(np.int64)).cuda()
    db = torch.from_numpy(b.view(np.int64)).cuda()
    dc = torch.empty(len(want), dtype=torch.int64, device="cuda")
    for field in (gpu.FIELD_GF128, gpu.FIELD_GF64):
        gpu.fp_polymul_dev(da, la, db, lb, dc, field=field)
        torch.cuda.synchronize()
        assert np.array_equal(dc.cpu().numpy().view(np.uint64), want), field


def _fuzz_shapes():
    """Seeded random operand lengths, log-uniform over every size class of the pipeline: the
    Karatsuba bypass (< 4096 bits), the one-CTA products (n <= 2^17), graph-replayed small products,
    the unfused / fused tile passes and the first radix-8 top passes (up to ~2^23 bits)."""
    rng = np.random.default_rng(20261021)
    shapes = []
    for _ in range(36):
        la = int(2 ** rng.uniform(0, 23)) + int(rng.integers(0, 3))
        lb = int(2 ** rng.uniform(0, 23)) + int(rng.integers(0, 3))
        shapes.append((la, lb))
    # lengths straddling word and power-of-two boundaries
    shapes += [(65, 127), (4096, 4097), ((1 << 17) - 1, (1 << 17) + 1), ((1 << 21) + 1, (1 << 21) - 1),
               ((1 << 22) - 63, 64), (3, (1 << 22) + 65)]
    return shapes


@pytest.mark.parametrize("la,lb", _fuzz_shapes())
def test_polymul_shape_fuzz(gpu, checker, port, la, lb):
    """fp_polymul (polymul.cpp:223-239) on random ragged shapes: every field choice through the host
    entry point and the device entry point (twice: the second call replays the CUDA graph)."""
    import torch
    a = port.random_bitpoly(la, 7000 + la)
    b = port.random_bitpoly(lb, 8000 + lb)
    want = checker.polymul(a, la, b, lb)
    for field in (gpu.FIELD_GF128, gpu.FIELD_GF64, gpu.FIELD_AUTO):
        assert np.array_equal(gpu.fp_polymul(a, la, b, lb, field=field), want), field
    da = torch.from_numpy(a.view(np.int64)).cuda()
    db = torch.from_numpy(b.view(np.int64)).cuda()
    dc = torch.empty(len(want), dtype=torch.int64, device="cuda")
    for rep in range(2):
        dc.fill_(-1)
        gpu.fp_polymul_dev(da, la, db, lb, dc, field=gpu.FIELD_GF128)
        torch.cuda.synchronize()
        assert np.array_equal(dc.cpu().numpy().view(np.uint64), want), rep


def test_reserve_and_trim_pool(gpu, checker, port):
    """fpm_reserve_pool / fpm_trim_pool: products are unaffected by either (the pool only caches)."""
    la, lb = 300000, 1 << 19
    a, b = port.random_bitpoly(la, 5), port.random_bitpoly(lb, 6)
    want = checker.polymul(a, la, b, lb)
    gpu.reserve_pool(3 << 29)
    assert np.array_equal(gpu.fp_polymul(a, la, b, lb, field=gpu.FIELD_GF128), want)
    gpu.trim_pool()
    assert np.array_equal(gpu.fp_polymul(a, la, b, lb, field=gpu.FIELD_GF128), want)
    with pytest.raises(Exception):
        gpu.reserve_pool(1 << 20, device=63)
    # a failed call leaves no stale CUDA error behind for the next one's launch checks
    assert np.array_equal(gpu.fp_polymul(a, la, b, lb, field=gpu.FIELD_GF128), want)


def test_host_buffers_ragged_2p33_product_matches_device_path(gpu):
    """A ragged 2^33-bit-class product through the host entry point (operand-a pre-pass, split decode,
    overlapped copies) equals the device-resident product of the same operands, which
    test_concurrent_conversions_device_resident_vs_reference pins to the reference."""
    import torch
    la, lb = 1 << 32, (1 << 31) + 999
    a, b = gpu.random_bitpoly(la, 91), gpu.random_bitpoly(lb, 92)
    got = gpu.fp_polymul(a, la, b, lb, field=gpu.FIELD_GF128)
    da, db = (torch.from_numpy(x.view(np.int64)).cuda() for x in (a, b))
    dc = torch.empty(got.size, dtype=torch.int64, device="cuda")
    gpu.fp_polymul_dev(da, la, db, lb, dc, field=gpu.FIELD_GF128)
    torch.cuda.synchronize()
    assert np.array_equal(dc.cpu().numpy().view(np.uint64), got)
    got64 = gpu.fp_polymul(b, lb, a, la, field=gpu.FIELD_AUTO)  # (operands swapped, GF(2^64))
    assert np.array_equal(got64, got)
