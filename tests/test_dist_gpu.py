"""The sharded product driver with the CUDA backend (paper_1803_11301_b200/dist.py GpuBackend) on ONE
GPU: P ranks are host threads sharing the device; exchanges and the column gather go through host
barriers (no kernel ever waits on another).  Checks the device building blocks the multi-GPU path
uses -- encode_cols, decode_cols, bfly_pair, lch_butterfly with a shifted base -- bit-exactly."""
import threading

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


class _Shared:
    def __init__(self, P):
        self.P = P
        self.barrier = threading.Barrier(P)
        self.slots = {}


def _make_backend(shared, rank):
    from paper_1803_11301_b200.dist import GpuBackend

    class ThreadBackend(GpuBackend):
        def world(self):
            return shared.P, rank

        def exchange(self, t, partner):
            torch.cuda.synchronize()
            shared.slots[rank] = t
            shared.barrier.wait()
            theirs = shared.slots[partner].clone()
            torch.cuda.synchronize()
            shared.barrier.wait()
            return theirs

        def gather_columns(self, slice_, plan):
            torch.cuda.synchronize()
            shared.slots[rank] = slice_
            shared.barrier.wait()
            parts = [shared.slots[r].clone() for r in range(shared.P)]
            torch.cuda.synchronize()
            shared.barrier.wait()
            stacked = torch.stack([p.view(128, plan.m // 64) for p in parts], dim=1)
            return stacked.reshape(-1).contiguous()

    return ThreadBackend()


# the last two shapes give cosets of 2^18 elements: the tower fast path (fpm_shard_local_product_dev)
@pytest.mark.parametrize("P,la,lb", [(2, 1 << 18, 1 << 18), (4, 1 << 20, (1 << 20) - 333), (8, 1 << 22, 1 << 21),
                                     (2, 1 << 25, (1 << 25) - 99), (4, 1 << 26, 1 << 25)])
def test_sharded_on_one_gpu(gpu, port, checker, P, la, lb):
    from paper_1803_11301_b200.dist import make_plan, polymul_sharded

    a = port.random_bitpoly(la, 31)
    b = port.random_bitpoly(lb, 32)
    want = checker.polymul(a, la, b, lb)
    shared = _Shared(P)
    out, errs = {}, []

    def run(rank):
        try:
            torch.cuda.set_device(0)
            da = torch.from_numpy(a.view(np.int64).copy()).cuda()
            db = torch.from_numpy(b.view(np.int64).copy()).cuda()
            be = _make_backend(shared, rank)
            res = polymul_sharded(da, la, db, lb, be, make_plan(la, lb, P, rank))
            torch.cuda.synchronize()
            out[rank] = res.cpu().numpy().view(np.uint64)
        except Exception as e:  # pragma: no cover - reported below
            errs.append((rank, repr(e)))
            shared.barrier.abort()

    th = [threading.Thread(target=run, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not errs, errs
    for r in range(P):
        assert np.array_equal(out[r], want), r


def _make_peer_backend(shared, rank, keep):
    """PeerBackend with the IPC hooks replaced by same-process pointers: the exchanged layers read the
    partner thread's buffer directly (as over NVLink), the barriers are host barriers."""
    from paper_1803_11301_b200.dist import PeerBackend

    class ThreadPeerBackend(PeerBackend):
        def world(self):
            return shared.P, rank

        def _alloc(self, nbytes):
            t = torch.empty(nbytes // 8, dtype=torch.int64, device="cuda")
            keep.append(t)
            return t.data_ptr(), t.data_ptr()

        def _publish(self, handles):
            shared.slots[("h", rank)] = handles
            shared.barrier.wait()
            out = [shared.slots[("h", r)] for r in range(shared.P)]
            shared.barrier.wait()
            return out

        def _open(self, handle):
            return handle

        def _close(self, ptr):
            pass

        def _free(self, ptr):
            pass

        def _barrier(self):
            torch.cuda.synchronize()
            shared.barrier.wait()

        def gather_columns(self, slice_, plan):
            torch.cuda.synchronize()
            shared.slots[rank] = slice_
            shared.barrier.wait()
            parts = [shared.slots[r].clone() for r in range(shared.P)]
            torch.cuda.synchronize()
            shared.barrier.wait()
            stacked = torch.stack([p.view(128, plan.m // 64) for p in parts], dim=1)
            return stacked.reshape(-1).contiguous()

    return ThreadPeerBackend()


@pytest.mark.parametrize("P,la,lb", [(2, 1 << 20, 1 << 19), (4, 1 << 25, (1 << 25) - 5), (2, 1 << 26, 1 << 26)])
def test_sharded_peer_exchange_on_one_gpu(gpu, port, checker, P, la, lb):
    """The peer-memory exchange (PeerBackend, fpm_bfly_pair_peer_dev: ping-pong buffers, the
    partner's half read directly by the pair kernel), both for small cosets (stand-alone stage
    kernels) and for >= 2^18-element cosets (tower fast path); two products per backend so the
    buffers are reused."""
    from paper_1803_11301_b200.dist import make_plan, polymul_sharded

    a = port.random_bitpoly(la, 41)
    b = port.random_bitpoly(lb, 42)
    want = checker.polymul(a, la, b, lb)
    shared = _Shared(P)
    out, errs, keep = {}, [], []

    def run(rank):
        try:
            torch.cuda.set_device(0)
            da = torch.from_numpy(a.view(np.int64).copy()).cuda()
            db = torch.from_numpy(b.view(np.int64).copy()).cuda()
            be = _make_peer_backend(shared, rank, keep)
            plan = make_plan(la, lb, P, rank)
            for _ in range(2):
                res = polymul_sharded(da, la, db, lb, be, plan)
            torch.cuda.synchronize()
            out[rank] = res.cpu().numpy().view(np.uint64)
        except Exception as e:  # pragma: no cover - reported below
            errs.append((rank, repr(e)))
            shared.barrier.abort()

    th = [threading.Thread(target=run, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not errs, errs
    for r in range(P):
        assert np.array_equal(out[r], want), r


def test_pair_peer_matches_in_place_pair(gpu):
    """fpm_bfly_pair_peer_dev (out-of-place, partner half from another buffer) equals the in-place
    fpm_bfly_pair_dev for both sides and directions, polynomial and tower representation."""
    import paper_1803_11301_b200._lib as L
    n = 1 << 16
    g = torch.Generator(device="cuda").manual_seed(5)
    mine = torch.randint(-(1 << 62), 1 << 62, (2 * n,), generator=g, device="cuda", dtype=torch.int64)
    theirs = torch.randint(-(1 << 62), 1 << 62, (2 * n,), generator=g, device="cuda", dtype=torch.int64)
    w = np.array([0x0123456789ABCDEF, 0x0FEDCBA987654321], np.uint64)
    s = torch.cuda.current_stream().cuda_stream
    for tower in (0, 1):
        for side in (0, 1):
            for inv in (0, 1):
                ref = mine.clone()
                f = L.lib().fpm_bfly_pair_r_dev if tower else L.lib().fpm_bfly_pair_dev
                L._check(f(ref.data_ptr(), theirs.data_ptr(), n, w.ctypes.data_as(L._u64p), side, inv, s))
                out = torch.empty_like(mine)
                L._check(L.lib().fpm_bfly_pair_peer_dev(mine.data_ptr(), theirs.data_ptr(), out.data_ptr(), n,
                                                        w.ctypes.data_as(L._u64p), side, inv, tower, s))
                torch.cuda.synchronize()
                assert torch.equal(out, ref), (tower, side, inv)


def test_tower_encode_decode_columns_match_polynomial(gpu):
    """fpm_encode_cols_r_dev / fpm_decode_cols_r_dev (tower representation) against the polynomial
    pair: decode_r(encode_r(x)) == decode(encode(x)) == x's column slice, for a column range and
    rows >= 64 zero as in the pipeline."""
    import paper_1803_11301_b200._lib as L
    l, col0, m = 14, 4096, 8192
    n_p = 1 << l
    g = torch.Generator(device="cuda").manual_seed(9)
    poly = torch.randint(-(1 << 62), 1 << 62, (128 * n_p // 64,), generator=g, device="cuda", dtype=torch.int64)
    poly[64 * n_p // 64:] = 0  # rows >= 64 zero
    s = torch.cuda.current_stream().cuda_stream
    outs = []
    for r in (False, True):
        ev = torch.empty(2 * m, dtype=torch.int64, device="cuda")
        enc = L.lib().fpm_encode_cols_r_dev if r else L.lib().fpm_encode_cols_dev
        dec = L.lib().fpm_decode_cols_r_dev if r else L.lib().fpm_decode_cols_dev
        L._check(enc(poly.data_ptr(), l, col0, m, 64, ev.data_ptr(), s))
        sl = torch.empty(128 * m // 64, dtype=torch.int64, device="cuda")
        L._check(dec(ev.data_ptr(), m, sl.data_ptr(), s))
        outs.append((ev.clone(), sl))
    torch.cuda.synchronize()
    assert not torch.equal(outs[0][0], outs[1][0])  # the two representations differ ...
    assert torch.equal(outs[0][1], outs[1][1])      # ... and decode to the same bits
    want = poly.view(128, n_p // 64)[:, col0 // 64:(col0 + m) // 64].reshape(-1)
    assert torch.equal(outs[1][1], want)


@pytest.mark.parametrize("P,la,lb", [(2, 1 << 20, (1 << 20) - 13), (8, 1 << 20, 1 << 20), (2, 1 << 25, (1 << 25) - 99),
                                     (4, 1 << 26, 1 << 25), (8, 1 << 24, 8400953)])
def test_polymul_multi_logical_ranks(gpu, checker, P, la, lb):
    """fpm_polymul_multi -- the single-process multi-GPU entry point (C-ABI) -- with P logical ranks
    on GPU 0: peer-memory exchanges, operand conversions on ranks 0/1, decode into the converting
    rank's array; both coset regimes (stage kernels below 2^18 elements per rank, tower fast path
    above).  Bit-exact against the oracle."""
    a = gpu.random_bitpoly(la, 61)
    b = gpu.random_bitpoly(lb, 62)
    assert np.array_equal(gpu.fp_polymul_multi(a, la, b, lb, [0] * P), checker.polymul(a, la, b, lb))


@pytest.mark.parametrize("key,P", [("268435456x268435456", 4), ("4294967296x4294967296", 2),
                                   ("4294967296x4294967296", 4), ("4294967296x4294967296", 8)])
def test_polymul_multi_baseline_configs(gpu, key, P):
    """BASELINE configs 4 and 5 through fpm_polymul_multi with P logical ranks on GPU 0 against the
    reference's product hash.  Config 5 at P = 2: the two 2^32-bit inverse-conversion blocks on ranks
    0 and 1, the top pass reading rank 1's block; at P = 4 and 8 the sharded conversion -- every
    2^32-bit block on P/2 ranks phase by phase (L1_outer by window, L1_inner + T_r by chunk, T_d by
    column, regathered between phases over peer memory), encode reading and decode writing the column
    owners, the top pass over the window shares."""
    import hashlib
    import json
    import os
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_meta.json")) as f:
        c = json.load(f)["configs"][key]
    a = gpu.random_bitpoly(c["a_bits"], c["seed_a"])
    b = gpu.random_bitpoly(c["b_bits"], c["seed_b"])
    prod = gpu.fp_polymul_multi(a, c["a_bits"], b, c["b_bits"], [0] * P, field=gpu.FIELD_GF128)
    assert hashlib.blake2b(prod.tobytes(), digest_size=16).hexdigest() == c["blake2b128"]


def test_polymul_multi_rejects_bad_rank_counts(gpu):
    a = gpu.random_bitpoly(1 << 20, 1)
    with pytest.raises(ValueError):
        gpu.fp_polymul_multi(a, 1 << 20, a, 1 << 20, [0, 0, 0])
    with pytest.raises(ValueError):  # 2^7 elements per rank
        gpu.fp_polymul_multi(a, 1 << 12, a, 1 << 12, [0] * 64, field=gpu.FIELD_GF128)


@pytest.mark.parametrize("P", [2, 4, 8])
def test_sharded_peer_config5_split_conversions(gpu, P):
    """BASELINE config 5 through dist.polymul_sharded with PeerBackend and thread ranks: at P = 2 the
    split conversions (operand a on rank 0, b on rank 1, encode from peer memory), the decode straight
    into the two 2^32-bit blocks on ranks 0 and 1 and their separate inverse conversions with the
    fused top pass; at P = 4, 8 the sharded conversion (fpm_b32_*: every block on P/2 ranks phase by
    phase); the product hash against the reference's."""
    import hashlib
    import json
    import os
    from paper_1803_11301_b200.dist import make_plan, polymul_sharded
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_meta.json")) as f:
        c = json.load(f)["configs"]["4294967296x4294967296"]
    a = gpu.random_bitpoly(c["a_bits"], c["seed_a"])
    b = gpu.random_bitpoly(c["b_bits"], c["seed_b"])
    shared = _Shared(P)
    out, errs, keep = {}, [], []

    def run(rank):
        try:
            torch.cuda.set_device(0)
            da = torch.from_numpy(a.view(np.int64)).cuda()
            db = torch.from_numpy(b.view(np.int64)).cuda()
            be = _make_peer_backend(shared, rank, keep)
            res = polymul_sharded(da, c["a_bits"], db, c["b_bits"], be, make_plan(c["a_bits"], c["b_bits"], P, rank))
            torch.cuda.synchronize()
            if rank == P - 1:
                out[rank] = hashlib.blake2b(res.cpu().numpy().view(np.uint64).tobytes(), digest_size=16).hexdigest()
            del res, da, db
        except Exception as e:  # pragma: no cover - reported below
            errs.append((rank, repr(e)))
            shared.barrier.abort()

    th = [threading.Thread(target=run, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    keep.clear()
    assert not errs, errs
    assert out[P - 1] == c["blake2b128"]


@pytest.mark.parametrize("Q", [2, 4])
def test_b32_sharded_conversion_c_abi_sequence(gpu, Q):
    """The sharded 2^32-bit conversion driven through its C-ABI exactly as INTEGRATION.md documents
    (fpm_b32_*: L1_outer by window, regather, fix + rows by chunk, regather, T_d by column), Q replicas
    on cuda:0: every column owner's columns equal fpm_basis_cvt_dev's conversion of the whole block;
    then the sharded inverse (T_d^-1 by column, rows^-1 by chunk, L1_outer^-1 by window + fix) brings
    every window owner's words back to the input."""
    import ctypes as C
    from paper_1803_11301_b200 import _lib
    L = gpu.lib()
    chk = _lib._check
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    words = 1 << 26  # 64-bit words of a 2^32-bit block
    x = torch.from_numpy(gpu.random_bitpoly(1 << 32, 777).view(np.int64)).cuda()
    want = x.clone()
    chk(L.fpm_basis_cvt_dev(want.data_ptr(), 1 << 32, 1 << 32, s))
    reps = [x.clone() for _ in range(Q)]
    sides = [torch.empty(256 * 2048 // 2, dtype=torch.int64, device="cuda") for _ in range(Q)]
    group = (C.c_void_p * Q)(*[r.data_ptr() for r in reps])
    WINDOW, CHUNK, COLUMN = 0, 1, 2
    for q in range(Q):
        chk(L.fpm_b32_l1_outer_dev(reps[q].data_ptr(), sides[q].data_ptr(), 0, q, Q, s))
    for q in range(Q):
        chk(L.fpm_b32_regather_dev(reps[q].data_ptr(), group, WINDOW, CHUNK, q, Q, s))
    for q in range(Q):
        c0, c1 = q * 256 // Q, (q + 1) * 256 // Q
        chk(L.fpm_b32_l1_outer_fix_dev(reps[q].data_ptr(), sides[Q - 1].data_ptr(), 0, c0, c1, s))
        chk(L.fpm_b32_rows_dev(reps[q].data_ptr() + c0 * 256 * 2048 * 4, (c1 - c0) * 256, 0, s))
    for q in range(Q):
        chk(L.fpm_b32_regather_dev(reps[q].data_ptr(), group, CHUNK, COLUMN, q, Q, s))
    for q in range(Q):
        chk(L.fpm_b32_cols_dev(reps[q].data_ptr(), 0, q, Q, s))
    torch.cuda.synchronize()
    cols = 2048 // Q  # 32-bit words of a row per owner
    for q in range(Q):
        got = reps[q].view(torch.int32).view(65536, 2048)[:, q * cols:(q + 1) * cols]
        ref = want.view(torch.int32).view(65536, 2048)[:, q * cols:(q + 1) * cols]
        assert torch.equal(got, ref), q
    # inverse, starting from the column owners
    for q in range(Q):
        chk(L.fpm_b32_cols_dev(reps[q].data_ptr(), 1, q, Q, s))
    for q in range(Q):
        chk(L.fpm_b32_regather_dev(reps[q].data_ptr(), group, COLUMN, CHUNK, q, Q, s))
    for q in range(Q):
        c0, c1 = q * 256 // Q, (q + 1) * 256 // Q
        chk(L.fpm_b32_rows_dev(reps[q].data_ptr() + c0 * 256 * 2048 * 4, (c1 - c0) * 256, 1, s))
    for q in range(Q):
        chk(L.fpm_b32_regather_dev(reps[q].data_ptr(), group, CHUNK, WINDOW, q, Q, s))
    for q in range(Q):
        chk(L.fpm_b32_l1_outer_dev(reps[q].data_ptr(), sides[q].data_ptr(), 1, q, Q, s))
    chk(L.fpm_b32_l1_outer_fix_dev(reps[0].data_ptr(), sides[Q - 1].data_ptr(), 1, 0, 256, s))
    for q in range(Q):
        chk(L.fpm_b32_regather_dev(reps[q].data_ptr(), group, WINDOW, CHUNK, q, Q, s))
    torch.cuda.synchronize()
    per = words // Q
    for q in range(Q):
        assert torch.equal(reps[q][q * per:(q + 1) * per], x[q * per:(q + 1) * per]), q


def test_b32_c_abi_rejects_bad_arguments(gpu):
    import ctypes as C
    L = gpu.lib()
    t = torch.zeros(1 << 10, dtype=torch.int64, device="cuda")
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    group = (C.c_void_p * 4)(*([t.data_ptr()] * 4))
    assert L.fpm_b32_regather_dev(t.data_ptr(), group, 0, 1, 0, 3, s) == 1   # Q must be 2 or 4
    assert L.fpm_b32_regather_dev(t.data_ptr(), group, 1, 1, 0, 2, s) == 1   # from == to
    assert L.fpm_b32_l1_outer_dev(t.data_ptr(), None, 0, 0, 2, s) == 1      # no side buffer
    assert L.fpm_b32_rows_dev(t.data_ptr(), 100, 0, s) == 1                  # not whole chunks
    assert L.fpm_b32_cols_dev(t.data_ptr(), 0, 2, 2, s) == 1                 # q >= Q
    assert L.fpm_b32_l1_outer_fix_dev(t.data_ptr(), t.data_ptr(), 0, 3, 300, s) == 1


def test_sharded_peer_config5_per_rank_io_shares(gpu):
    """dist.polymul_sharded(parts=True), 4 thread ranks: every rank passes only its share of its
    operand (operand_part_range) and gets back only its share of the product (product_part_range);
    the assembled shares hash to the reference's config-5 product."""
    import hashlib
    import json
    import os
    from paper_1803_11301_b200.dist import make_plan, operand_part_range, polymul_sharded, product_part_range
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_meta.json")) as f:
        c = json.load(f)["configs"]["4294967296x4294967296"]
    ops = [gpu.random_bitpoly(c["a_bits"], c["seed_a"]), gpu.random_bitpoly(c["b_bits"], c["seed_b"])]
    P = 4
    out_words = (c["a_bits"] + c["b_bits"] - 1 + 63) // 64
    prod = np.zeros(out_words, np.uint64)
    shared = _Shared(P)
    errs, keep = [], []

    def run(rank):
        try:
            torch.cuda.set_device(0)
            plan = make_plan(c["a_bits"], c["b_bits"], P, rank)
            k, w0, n = operand_part_range(plan, rank)
            part = torch.from_numpy(ops[k][w0:w0 + n].view(np.int64).copy()).cuda()
            be = _make_peer_backend(shared, rank, keep)
            res = polymul_sharded(part, c["a_bits"], part, c["b_bits"], be, plan, parts=True)
            torch.cuda.synchronize()
            o0, _ = product_part_range(plan, rank)
            prod[o0:o0 + res.numel()] = res.cpu().numpy().view(np.uint64)
            del res, part
        except Exception as e:  # pragma: no cover - reported below
            errs.append((rank, repr(e)))
            shared.barrier.abort()

    th = [threading.Thread(target=run, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    keep.clear()
    assert not errs, errs
    assert hashlib.blake2b(prod.tobytes(), digest_size=16).hexdigest() == c["blake2b128"]
