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
