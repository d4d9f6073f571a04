"""Multi-process (gloo, CPU) tests of the sharded product's host logic (paper_1803_11301_b200/dist.py):
partition, per-layer partners/sides/twiddles, the sub-FFT base shift, exchanges and the column
gather.  The per-rank compute runs through an oracle backend built on the REAL reference library
(oracle/_ref), so these tests check the decomposition itself; the GPU backend plugs the same driver
into the CUDA C-ABI."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class OracleBackend:
    def __init__(self, R, l):
        self.R, self.l = R, l
        self.tw = R.twiddles128(l)  # plan.mults of plan_butterflies(l, e_{l+64}), layer-major

    def world(self):
        return dist.get_world_size(), dist.get_rank()

    def convert_operand(self, x, bits, n_bits):
        poly = np.zeros(n_bits // 128, np.uint64)
        w = (bits + 63) // 64
        poly[:w] = x[:w]
        if bits % 64:
            poly[w - 1] &= np.uint64((1 << (bits % 64)) - 1)
        count = 64
        while count < bits:
            count <<= 1
        poly[: count // 64] = self.R.basis_cvt(poly[: count // 64], count)
        return poly

    def encode_cols(self, poly, l, col0, ncols):
        full = np.zeros((128 << l) // 64, np.uint64)
        full[: poly.size] = poly
        return self.R.encode128(full, l)[2 * col0: 2 * (col0 + ncols)].copy()

    def exchange(self, arr, partner):
        t = torch.from_numpy(arr.view(np.int64).copy())
        buf = torch.empty_like(t)
        for r in dist.batch_isend_irecv([dist.P2POp(dist.isend, t, partner), dist.P2POp(dist.irecv, buf, partner)]):
            r.wait()
        return buf.numpy().view(np.uint64)

    def twiddle(self, i, b, base):
        assert base == 1 << (self.l + 64)
        k = (1 << (self.l - 1 - i)) - 1 + b  # ButterflyPlan::layer_offset(i) + b (butterfly.hpp:45-48)
        return self.tw[2 * k: 2 * k + 2].copy()

    def pair(self, mine, theirs, w, side, inverse):
        wv = np.tile(w, mine.size // 2)
        mul = lambda x: self.R.pointwise128(wv, x)  # noqa: E731
        if not inverse:
            res = mine ^ mul(theirs) if side == 0 else mine ^ theirs ^ mul(mine)
        else:
            res = mine ^ mul(mine ^ theirs) if side == 0 else mine ^ theirs
        mine[:] = res

    def butterfly(self, ev, l, base, inverse):
        if l:
            ev[:] = self.R.butterfly128_base(ev, l, base & (2**64 - 1), base >> 64, inverse)

    def pointwise(self, u, v):
        return self.R.pointwise128(u, v)

    def decode_cols(self, ev, ncols):
        return self.R.decode128(ev, ncols.bit_length() - 1)

    def gather_columns(self, slice_, plan):
        t = torch.from_numpy(slice_.view(np.int64).copy())
        parts = [torch.empty_like(t) for _ in range(plan.P)]
        dist.all_gather(parts, t)
        stacked = np.stack([p.numpy().view(np.uint64).reshape(128, plan.m // 64) for p in parts], axis=1)
        return stacked.reshape(-1).copy()

    def finish(self, full, n_bits, out_bits):
        out = self.R.basis_cvt(full, n_bits, inverse=True)[: (out_bits + 63) // 64].copy()
        if out_bits % 64:
            out[-1] &= np.uint64((1 << (out_bits % 64)) - 1)
        return out


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, shapes, q):
    import sys
    sys.path.insert(0, ROOT)
    import oracle
    from paper_1803_11301_b200.dist import make_plan, polymul_sharded
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        R = oracle.ref()
        P = oracle.port()
        for la, lb in shapes:
            a, b = P.random_bitpoly(la, 11 + la), P.random_bitpoly(lb, 12 + lb)
            plan = make_plan(la, lb, world, rank)
            got = polymul_sharded(a, la, b, lb, OracleBackend(R, plan.l), plan)
            want = R.polymul(a, la, b, lb, field=128)
            q.put((rank, la, lb, bool(np.array_equal(got, want))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,shapes", [
    (2, [(1 << 17, 1 << 17), ((1 << 17) - 9, 70001)]),
    (4, [(1 << 18, 1 << 18), ((1 << 18) - 100, 3000)]),
])
def test_sharded_product_gloo(ref, world, shapes):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, shapes, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    results = [q.get(timeout=5) for _ in range(world * len(shapes))]
    assert all(p.exitcode == 0 for p in procs)
    assert all(ok for (_, _, _, ok) in results), results


def test_plan_geometry():
    from paper_1803_11301_b200.dist import make_plan
    p = make_plan(1 << 32, 1 << 32, 8, 5)
    assert (p.n_bits, p.l, p.m, p.col0, p.lp) == (1 << 33, 26, 1 << 23, 5 << 23, 23)
    assert p.top_layers(False) == [25, 24, 23] and p.top_layers(True) == [23, 24, 25]
    assert [p.partner(i) for i in (23, 24, 25)] == [4, 7, 1]
    assert [p.side(i) for i in (23, 24, 25)] == [1, 0, 1]
    with pytest.raises(ValueError):
        make_plan(1 << 10, 1 << 10, 8, 0)
    with pytest.raises(ValueError):
        make_plan(1 << 20, 1 << 20, 3, 0)
