"""Sharded single-product multiplication across GPUs (one process per GPU, torch.distributed).

SURVEY.md 8(e): rank g of P owns elements [g*m, (g+1)*m), m = n_p / P, of every EvalVec.

* basis conversion of the operands: with PeerBackend (P >= 2) operand a converts on rank 0 and b on
  rank 1 and every rank encodes its columns straight from the converting rank's memory (CUDA IPC);
  other backends replicate it (every rank holds both inputs);
* encode: element-local -- rank g encodes columns [g*m, (g+1)*m) of the partition matrix;
* forward FFT: layers i >= l' = l - log2 P pair element e with e ^ 2^i, which lives on rank
  g ^ 2^(i - l'): ONE exchange of the rank's whole slice with that partner per layer, then a local
  half-butterfly with the block's (rank-uniform) twiddle C2P((base >> i) ^ 2b), b = g*m >> (i+1);
* layers < l' are a complete sub-FFT on the slice: lch_butterfly(l', base ^ g*m) -- the twiddle
  C2P((base >> i) ^ 2b) with b = (g*m >> (i+1)) + b_local equals C2P(((base ^ g*m) >> i) ^ 2 b_local);
* pointwise: local; inverse FFT mirrors the forward (local layers, then exchanged top layers);
* decode: local columns -> a 128 x m-bit slice; all_gather + column interleave -> the n-bit
  product array; inverse basis conversion (replicated); trim.  PeerBackend instead decodes every
  rank's columns straight into the product array on rank 0 (or, for a 2^33-bit product, the two
  independent 2^32-bit blocks on ranks 0 and 1, converted there, the lower block's top pass reading
  the upper one over peer memory) -- the single-process fpm_polymul_multi's decomposition, over the
  same C-ABI calls.

Cosets of 2^18 or more elements take the single-GPU fast path (backend.tower(l') true): operands
encoded straight into the tower representation, exchanged layers on tower tables, and the local
forward layers of both operands + pointwise product + local inverse layers as ONE call
(local_product: the radix-4 top passes and the fused tower tile pass of k_fft.cu).

Exchange volume per top layer: m * 16 B per rank (config 5, P = 8: 128 MiB).  The compute goes
through a `backend` (GpuBackend here: the CUDA C-ABI; the gloo CPU tests plug in an oracle
backend), so the partition / exchange logic is one piece of code tested on CPU and run on GPUs.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass
class ShardPlan:
    a_bits: int
    b_bits: int
    n_bits: int
    l: int
    P: int
    rank: int

    @property
    def n_p(self) -> int:
        return 1 << self.l

    @property
    def m(self) -> int:
        return self.n_p // self.P

    @property
    def col0(self) -> int:
        return self.rank * self.m

    @property
    def lp(self) -> int:  # local layers
        return self.l - (self.P.bit_length() - 1)

    @property
    def base(self) -> int:  # make_partition_spec<gf128>(l).base = e_{l+64} (encode.cpp:47)
        return 1 << (self.l + 64)

    def top_layers(self, inverse: bool):
        r = range(self.lp, self.l)
        return list(r) if inverse else list(reversed(r))

    def partner(self, i: int) -> int:
        return self.rank ^ (1 << (i - self.lp))

    def side(self, i: int) -> int:
        return (self.rank >> (i - self.lp)) & 1

    def block(self, i: int) -> int:
        return self.col0 >> (i + 1)


def make_plan(a_bits: int, b_bits: int, P: int, rank: int) -> ShardPlan:
    """plan_mul over GF(2^128) (polymul.cpp:187-219) plus the shard geometry."""
    if P & (P - 1):
        raise ValueError("sharded product: the number of ranks must be a power of two")
    mx = max(a_bits, b_bits)
    n = 1
    while n < 2 * mx:
        n <<= 1
    n = max(n, 128)
    l = n.bit_length() - 1 - 7
    plan = ShardPlan(a_bits, b_bits, n, l, P, rank)
    if plan.m < 1024:
        raise ValueError(f"sharded product: {P} ranks need n_p >= {1024 * P} elements (n_p = {plan.n_p})")
    return plan


def batch_shard(count: int, P: int, rank: int) -> tuple[int, int]:
    """Config 2's split of `count` independent products over P ranks (no exchange): rank r takes the
    contiguous range [start, start + n), the first count % P ranks one product more."""
    if P < 1 or not 0 <= rank < P:
        raise ValueError("batch_shard: bad rank / world size")
    q, r = divmod(count, P)
    start = rank * q + min(rank, r)
    return start, q + (1 if rank < r else 0)


def polymul_batch_sharded(a, a_bits: int, b, b_bits: int, c, count: int, P: int, rank: int, lib=None):
    """This rank's share of a batch of `count` products held densely (stride = words per operand /
    product) in the FULL batch tensors a, b, c: only rows [start, start + n) are touched."""
    from . import _lib
    L = lib or _lib
    wa, wb, wc = (a_bits + 63) // 64, (b_bits + 63) // 64, (a_bits + b_bits - 1 + 63) // 64
    start, n = batch_shard(count, P, rank)
    if n:
        L.fp_polymul_batch_dev(a[start * wa:(start + n) * wa], a_bits, wa, b[start * wb:(start + n) * wb], b_bits, wb,
                               c[start * wc:(start + n) * wc], wc, n)
    return start, n


def operand_part_range(plan: ShardPlan, rank: int):
    """The sharded conversion's input share of a rank (P >= 4, 2^32-bit operands): (operand index k,
    first 64-bit word, word count) -- rank g holds words [w0, w0 + n) of operand g // (P/2)."""
    Q = plan.P // 2
    k, q = divmod(rank, Q)
    per = (1 << 26) // Q
    return k, q * per, per


def product_part_range(plan: ShardPlan, rank: int):
    """The sharded conversion's output share of a rank: (first 64-bit word of the product, word
    count before trimming to the product's length) -- the rank's chunks of its 2^32-bit block."""
    Q = plan.P // 2
    k, q = divmod(rank, Q)
    per = (1 << 26) // Q
    return k * (1 << 26) + q * per, per


def polymul_sharded(a, a_bits: int, b, b_bits: int, backend, plan: ShardPlan | None = None, parts: bool = False):
    """Product of two polynomials (backend arrays of packed words) over backend.world ranks;
    every rank returns the full product words.  parts (PeerBackend, sharded conversion): a and b are
    only this rank's input share (operand_part_range; the other operand is ignored) and the rank
    returns only its output share (product_part_range) -- each rank's host I/O is 1/P of the data,
    over its own PCIe link."""
    P, rank = backend.world()
    plan = plan or make_plan(a_bits, b_bits, P, rank)
    r = hasattr(backend, "tower") and backend.tower(plan.lp)           # coset on the fast path
    kw = {"tower": True} if r else {}
    if hasattr(backend, "begin"):
        backend.begin(plan)

    def exchanged(ev, i, inverse):
        w = backend.twiddle(i, plan.block(i), plan.base)
        if hasattr(backend, "exchange_pair"):  # exchange fused into the butterfly (peer memory)
            return backend.exchange_pair(ev, plan.partner(i), w, plan.side(i), inverse, **kw)
        theirs = backend.exchange(ev, plan.partner(i))
        backend.pair(ev, theirs, w, plan.side(i), inverse=inverse, **kw)
        return ev

    # backends with split conversions (PeerBackend, P >= 2): operand a converts on rank 0, b on rank 1,
    # every rank encodes its columns from the converting rank's memory; otherwise replicated
    split = P >= 2 and hasattr(backend, "convert_operands_split")
    polys = backend.convert_operands_split(a, a_bits, b, b_bits, plan, parts) if split else None
    if parts and not split:
        raise ValueError("polymul_sharded: operand parts need a PeerBackend")
    evs = []
    for k, (x, bits) in enumerate(((a, a_bits), (b, b_bits))):
        poly = polys[k] if split else backend.convert_operand(x, bits, plan.n_bits)
        ev = backend.encode_cols(poly, plan.l, plan.col0, plan.m, **kw)  # local columns
        for i in plan.top_layers(inverse=False):                       # exchanged layers
            ev = exchanged(ev, i, False)
        if not r:
            backend.butterfly(ev, plan.lp, plan.base ^ plan.col0, inverse=False)
        evs.append(ev)
    if r:  # local forward layers of both, pointwise, local inverse layers: one call
        c = backend.local_product(evs[0], evs[1], plan.lp, plan.base ^ plan.col0)
    else:
        c = backend.pointwise(evs[0], evs[1])
        backend.butterfly(c, plan.lp, plan.base ^ plan.col0, inverse=True)
    for i in plan.top_layers(inverse=True):
        c = exchanged(c, i, True)
    if split:  # decode into the converting ranks' arrays, inverse conversion split by block
        return backend.finish_split(c, plan, a_bits + b_bits - 1, tower=r, part=parts)
    slice_ = backend.decode_cols(c, plan.m, **kw)                       # 128 rows x m bits
    full = backend.gather_columns(slice_, plan)                         # 128 rows x n_p bits
    return backend.finish(full, plan.n_bits, a_bits + b_bits - 1)       # i_basis_cvt + trim


class GpuBackend:
    """The CUDA C-ABI on torch CUDA tensors (int64 words), NCCL point-to-point exchanges."""

    def __init__(self, group=None):
        import torch
        import torch.distributed as dist

        from . import _lib

        self.torch, self.dist, self.L, self.group = torch, dist, _lib, group

    def world(self):
        d = self.dist
        if not d.is_initialized():
            return 1, 0
        return d.get_world_size(self.group), d.get_rank(self.group)

    def _s(self):
        return self.torch.cuda.current_stream().cuda_stream

    def convert_operand(self, x, bits: int, n_bits: int):
        t = self.torch
        half_words = n_bits // 128
        poly = t.zeros(half_words, dtype=t.int64, device=x.device)
        w = (bits + 63) // 64
        poly[:w] = x[:w]
        if bits % 64:
            poly[w - 1] &= (1 << (bits % 64)) - 1
        count = 1
        while count < bits:
            count <<= 1
        count = max(count, 64)
        self.L.stage_dev("basis_cvt", poly, count, bits, stream=self._s())
        return poly

    def tower(self, l: int) -> bool:
        return bool(self.L.lib().fpm_shard_tower(l))

    def encode_cols(self, poly, l: int, col0: int, ncols: int, tower: bool = False):
        ev = self.torch.empty(2 * ncols, dtype=self.torch.int64, device=poly.device)
        f = self.L.lib().fpm_encode_cols_r_dev if tower else self.L.lib().fpm_encode_cols_dev
        self.L._check(f(poly.data_ptr(), l, col0, ncols, 64, ev.data_ptr(), self._s()))
        return ev

    def exchange(self, t, partner: int):
        d = self.dist
        buf = self.torch.empty_like(t)
        reqs = d.batch_isend_irecv([d.P2POp(d.isend, t, partner, self.group), d.P2POp(d.irecv, buf, partner, self.group)])
        for r in reqs:
            r.wait()
        return buf

    def twiddle(self, i: int, b: int, base: int):
        import ctypes as C

        import numpy as np
        out = np.zeros(2, np.uint64)
        bb = np.array([base & (2**64 - 1), base >> 64], np.uint64)
        self.L._check(self.L.lib().fpm_twiddle128(i, b, bb.ctypes.data_as(self.L._u64p), out.ctypes.data_as(self.L._u64p)))
        return out

    def pair(self, mine, theirs, w, side: int, inverse: bool, tower: bool = False):
        f = self.L.lib().fpm_bfly_pair_r_dev if tower else self.L.lib().fpm_bfly_pair_dev
        self.L._check(f(mine.data_ptr(), theirs.data_ptr(), mine.numel() // 2, w.ctypes.data_as(self.L._u64p), side,
                        int(inverse), self._s()))

    def local_product(self, ea, eb, l: int, base: int):
        import numpy as np
        bb = np.array([base & (2**64 - 1), base >> 64], np.uint64)
        self.L._check(self.L.lib().fpm_shard_local_product_dev(ea.data_ptr(), eb.data_ptr(), l,
                                                               bb.ctypes.data_as(self.L._u64p), self._s()))
        return eb

    def butterfly(self, ev, l: int, base: int, inverse: bool):
        import numpy as np
        if l == 0:
            return
        bb = np.array([base & (2**64 - 1), base >> 64], np.uint64)
        self.L._check(self.L.lib().fpm_lch_butterfly_dev(ev.data_ptr(), l, bb.ctypes.data_as(self.L._u64p),
                                                         int(inverse), self._s()))

    def pointwise(self, u, v):
        self.L.stage_dev("pointwise", u, v, u, u.numel() // 2, stream=self._s())
        return u

    def decode_cols(self, ev, ncols: int, tower: bool = False):
        out = self.torch.empty(128 * ncols // 64, dtype=self.torch.int64, device=ev.device)
        f = self.L.lib().fpm_decode_cols_r_dev if tower else self.L.lib().fpm_decode_cols_dev
        self.L._check(f(ev.data_ptr(), ncols, out.data_ptr(), self._s()))
        return out

    def gather_columns(self, slice_, plan: ShardPlan):
        t = self.torch
        P = plan.P
        parts = [t.empty_like(slice_) for _ in range(P)]
        if P > 1 and self.dist.get_backend(self.group) == "gloo":  # control-plane group (CPU tests,
            host = [t.empty_like(slice_, device="cpu") for _ in range(P)]  # several ranks on one GPU)
            self.dist.all_gather(host, slice_.cpu(), group=self.group)
            parts = [h.to(slice_.device) for h in host]
        elif P > 1:
            self.dist.all_gather(parts, slice_, group=self.group)
        else:
            parts[0] = slice_
        # each part: 128 rows x (m/64) words -> full: 128 rows x (n_p/64) words, columns interleaved by rank
        stacked = t.stack([p.view(128, plan.m // 64) for p in parts], dim=1)  # 128 x P x m/64
        return stacked.reshape(-1).contiguous()

    def finish(self, full, n_bits: int, out_bits: int):
        self.L.stage_dev("i_basis_cvt", full, n_bits, stream=self._s())
        w = (out_bits + 63) // 64
        out = full[:w].clone()
        if out_bits % 64:
            out[w - 1] &= (1 << (out_bits % 64)) - 1
        return out


def C_void(ptr: int):
    import ctypes as C
    return C.c_void_p(ptr)


class DevBuf:
    """A raw device buffer with the two tensor methods the backend's C-ABI calls use."""

    def __init__(self, ptr: int, numel: int, device=None):
        self.ptr, self.n, self.device = ptr, numel, device

    def data_ptr(self) -> int:
        return self.ptr

    def numel(self) -> int:
        return self.n


class _Owners:
    """A converted operand held at its column owners (Q peer replicas, a ctypes pointer array)."""

    def __init__(self, ptrs, Q: int):
        self.ptrs, self.Q = ptrs, Q


class PeerBackend(GpuBackend):
    """GpuBackend with the exchanged layers fused into their butterflies over peer memory (NVLink):
    each rank keeps both operands' evaluation slices in ping-pong pairs of peer-shareable buffers
    (fpm_ipc_alloc; handles exchanged once per plan with all_gather_object, partners' buffers opened
    with fpm_ipc_open), and an exchanged layer is ONE kernel (fpm_bfly_pair_peer_dev) that reads the
    partner's current buffer directly and writes this rank's other one.  A barrier before each
    exchanged layer orders it after every rank's previous step (inputs written, old reads done);
    the local product only touches the buffers partners do not read.  Across products the final
    column all_gather (stream-ordered after every rank's last pair kernel) orders the reuse.
    No NCCL data-path transfer remains except that gather."""

    def __init__(self, group=None):
        super().__init__(group)
        self.key = None
        self.mine, self.peer = [], {}

    def _close(self, ptr):
        self.L._check(self.L.lib().fpm_ipc_close(C_void(ptr)))

    def _free(self, ptr):
        self.L._check(self.L.lib().fpm_ipc_free(C_void(ptr)))

    def close(self):
        """Releases the plan's buffers: partners' handles closed, then (after every rank closed the
        handles to ours) this rank's buffers freed.  Collective: every rank must call it."""
        if self.key is None:
            return
        self._barrier()  # no rank still reads a partner buffer
        for ptrs in self.peer.values():
            for p in ptrs:
                self._close(p)
        for p in getattr(self, "opened", []):
            self._close(p)
        self._barrier()  # every partner closed its mapping of our buffers
        for b in self.mine:
            self._free(b.ptr)
        for p in getattr(self, "owned", []):
            self._free(p)
        self.mine, self.peer, self.key, self.opened, self.owned, self.arrays = [], {}, None, [], [], {}

    # -- split conversions (P >= 2)
    @staticmethod
    def _sharded(plan) -> bool:
        """The sharded 2^32-bit conversion (fpm_b32_*; as fpm_polymul_multi): P >= 4 ranks, P/2 <= 4 per
        block, a 2^33-bit product of two operands that each fill a 2^32-bit conversion."""
        cnt = lambda bits: max(32, 1 << (bits - 1).bit_length())  # noqa: E731
        return (4 <= plan.P <= 8 and plan.n_bits == 1 << 33 and cnt(plan.a_bits) == 1 << 32
                and cnt(plan.b_bits) == 1 << 32)

    @staticmethod
    def _shared_sizes(plan, P, rank):
        if P < 2:
            return {}
        n = plan.n_bits
        if PeerBackend._sharded(plan):  # every rank: a full-size block replica + L1_outer side rows
            return {f"r{rank}": n // 16, f"s{rank}": 256 * 2048 * 4}
        out = {}
        if rank == 0:
            out["x0"] = n // 16
            out["y0"] = n // 16 if n == 1 << 33 else n // 8
        if rank == 1:
            out["x1"] = n // 16
            if n == 1 << 33:
                out["y1"] = n // 16
        return out

    def _ptrs(self, names):
        import ctypes as C
        return (C.c_void_p * len(names))(*[self.arrays[nm] for nm in names])

    def convert_operands_sharded(self, a, a_bits, b, b_bits, plan, parts: bool = False):
        """The sharded conversion: operand k on ranks [kQ, (k+1)Q) (Q = P/2), phase by phase in the
        ranks' replicas -- L1_outer by window, L1_inner + T_r by chunk, T_d by column -- with a barrier
        and a peer-memory regather between phases.  Returns, per operand, its column owners.
        parts: a / b are only this rank's chunk range of its own operand (operand_part_range), pulled
        into the window distribution by a first regather."""
        P, rank = self.world()
        Q = P // 2
        k, q = divmod(rank, Q)
        s = self._s()
        L = self.L.lib()
        chk = self.L._check
        mine, side = self.arrays[f"r{rank}"], self.arrays[f"s{rank}"]
        group = self._ptrs([f"r{k * Q + j}" for j in range(Q)])
        x, bits = ((a, a_bits), (b, b_bits))[k]
        if parts:
            _, w0, per = operand_part_range(plan, rank)
            part_bits = max(0, min(per * 64, bits - w0 * 64))
            chk(L.fpm_load_operand_dev(mine + w0 * 8, per, x.data_ptr(), part_bits, s))
            self._barrier()
            chk(L.fpm_b32_regather_dev(mine, group, 1, 0, q, Q, s))  # CHUNK -> WINDOW
            self._barrier()
        else:
            chk(L.fpm_load_operand_dev(mine, plan.n_bits // 128, x.data_ptr(), bits, s))  # every rank holds the inputs
        chk(L.fpm_b32_l1_outer_dev(mine, side, 0, q, Q, s))
        self._barrier()
        chk(L.fpm_b32_regather_dev(mine, group, 0, 1, q, Q, s))  # WINDOW -> CHUNK
        self._barrier()
        c0, c1 = q * 256 // Q, (q + 1) * 256 // Q
        chk(L.fpm_b32_l1_outer_fix_dev(mine, self.arrays[f"s{k * Q + Q - 1}"], 0, c0, c1, s))
        chk(L.fpm_b32_rows_dev(mine + c0 * 256 * 2048 * 4, (c1 - c0) * 256, 0, s))
        self._barrier()
        chk(L.fpm_b32_regather_dev(mine, group, 1, 2, q, Q, s))  # CHUNK -> COLUMN
        self._barrier()
        chk(L.fpm_b32_cols_dev(mine, 0, q, Q, s))
        self._barrier()  # both converted operands final at their column owners
        return [_Owners(self._ptrs([f"r{kk * Q + j}" for j in range(Q)]), Q) for kk in (0, 1)]

    def convert_operands_split(self, a, a_bits, b, b_bits, plan, parts=False):
        """Rank 0 converts operand a, rank 1 operand b (each into its own shared array); every rank
        then reads both converted operands (peer memory) for its encode.  (P >= 4 with 2^32-bit
        operands: the sharded conversion.)"""
        if self._sharded(plan):
            return self.convert_operands_sharded(a, a_bits, b, b_bits, plan, parts)
        if parts:
            raise ValueError("operand parts need the sharded conversion (P >= 4, 2^32-bit operands)")
        P, rank = self.world()
        s = self._s()
        L = self.L.lib()
        half_words = plan.n_bits // 128
        for k, (x, bits) in enumerate(((a, a_bits), (b, b_bits))):
            if rank == k:
                dst = self.arrays[f"x{k}"]
                self.L._check(L.fpm_load_operand_dev(dst, half_words, x.data_ptr(), bits, s))
                count = 32
                while count < bits:
                    count <<= 1
                self.L._check(L.fpm_basis_cvt_dev(dst, count, bits, s))
        self._barrier()  # both converted operands final before any rank encodes from them
        dev = self.torch.device("cuda", self.torch.cuda.current_device())
        return [DevBuf(self.arrays["x0"], half_words, dev), DevBuf(self.arrays["x1"], half_words, dev)]

    def finish_sharded(self, c, plan, out_bits, tower=False, part=False):
        """The sharded inverse: decode into the column owners of the lower (ranks [0, Q)) and upper
        ([Q, 2Q)) 2^32-bit blocks, T_d^-1 by column, T_r^-1 + L1_inner^-1 by chunk, L1_outer^-1 by
        window (+ fix on rank 0), the top pass, the upper bit fix, a final regather to chunks; then
        every rank copies the whole product from the chunk owners."""
        P, rank = self.world()
        Q = P // 2
        k, q = divmod(rank, Q)
        s = self._s()
        L = self.L.lib()
        chk = self.L._check
        mine, side = self.arrays[f"r{rank}"], self.arrays[f"s{rank}"]
        los = self._ptrs([f"r{j}" for j in range(Q)])
        his = self._ptrs([f"r{Q + j}" for j in range(Q)])
        group = los if k == 0 else his
        chk(L.fpm_decode_cols_owners_dev(c.data_ptr(), plan.m, plan.col0, plan.n_p, los, his, Q, int(tower), s))
        self._barrier()
        chk(L.fpm_b32_cols_dev(mine, 1, q, Q, s))
        self._barrier()
        chk(L.fpm_b32_regather_dev(mine, group, 2, 1, q, Q, s))  # COLUMN -> CHUNK
        self._barrier()
        c0, c1 = q * 256 // Q, (q + 1) * 256 // Q
        chk(L.fpm_b32_rows_dev(mine + c0 * 256 * 2048 * 4, (c1 - c0) * 256, 1, s))
        self._barrier()
        chk(L.fpm_b32_regather_dev(mine, group, 1, 0, q, Q, s))  # CHUNK -> WINDOW
        self._barrier()
        chk(L.fpm_b32_l1_outer_dev(mine, side, 1, q, Q, s))
        self._barrier()
        if q == 0:
            chk(L.fpm_b32_l1_outer_fix_dev(mine, self.arrays[f"s{k * Q + Q - 1}"], 1, 0, 256, s))
        self._barrier()
        if k == 0:
            chk(L.fpm_b32_top_pass_dev(mine, his, q, Q, s))
        self._barrier()  # the lower block read the upper block's (pre-fix) bit 0
        if rank == Q:
            chk(L.fpm_b32_top_bit_fix_dev(mine, self.arrays[f"r{2 * Q - 1}"], s))
        self._barrier()
        chk(L.fpm_b32_regather_dev(mine, group, 0, 1, q, Q, s))  # WINDOW -> CHUNK
        self._barrier()  # the product is final at its chunk owners
        t = self.torch
        w = (out_bits + 63) // 64
        if part:  # only this rank's chunk range of the product
            w0, per = product_part_range(plan, rank)
            n = max(0, min(w, w0 + per) - w0)
            out = t.empty(n, dtype=t.int64, device=c.device)
            if n:
                chk(L.fpm_copy_dev(out.data_ptr(), mine + (w0 - k * (1 << 26)) * 8, n * 8, s))
                if w0 + n == w and out_bits % 64:
                    out[n - 1] &= (1 << (out_bits % 64)) - 1
            self._barrier()  # every rank copied out before the replicas are reused
            return out
        out = t.empty(w, dtype=t.int64, device=c.device)
        per = (1 << 26) // Q  # 64-bit words of a rank's chunks
        for g in range(P):
            kk, qq = divmod(g, Q)
            w0 = kk * (1 << 26) + qq * per
            w1 = min(w, w0 + per)
            if w0 < w1:
                chk(L.fpm_copy_dev(out.data_ptr() + w0 * 8, self.arrays[f"r{g}"] + qq * per * 8, (w1 - w0) * 8, s))
        if out_bits % 64:
            out[w - 1] &= (1 << (out_bits % 64)) - 1
        self._barrier()  # every rank copied out before the replicas are reused
        return out

    def finish_split(self, c, plan, out_bits, tower=False, part=False):
        """Every rank decodes its columns straight into the product array(s); the inverse conversion
        runs on rank 0 (n <= 2^32 bits) or as the two 2^32-bit blocks on ranks 1 and 0 (2^33 bits:
        the lower block's top pass reads rank 1's final block); every rank then copies the product.
        (P >= 4 with 2^32-bit operands: the sharded inverse.)"""
        if self._sharded(plan):
            return self.finish_sharded(c, plan, out_bits, tower, part)
        P, rank = self.world()
        s = self._s()
        L = self.L.lib()
        n, n_p = plan.n_bits, plan.n_p
        blocks = n == 1 << 33
        lo = self.arrays["y0"]
        hi = self.arrays["y1"] if blocks else lo + 64 * (n_p // 8)  # rows 64.. of the n-bit array (bytes)
        self.L._check(L.fpm_decode_cols_split_dev(c.data_ptr(), plan.m, plan.col0, n_p, lo, hi, int(tower), s))
        self._barrier()  # every rank's columns are in place
        if blocks:
            if rank == 1:
                self.L._check(L.fpm_i_basis_cvt_dev(hi, 1 << 32, s))
            self._barrier()
            if rank == 0:
                self.L._check(L.fpm_i_basis_cvt_block32_dev(lo, hi, s))
            self._barrier()  # rank 0 read rank 1's (pre-fix) bit 0
            if rank == 1:
                self.L._check(L.fpm_top_bit_fix_dev(hi, s))
        elif rank == 0:
            self.L._check(L.fpm_i_basis_cvt_dev(lo, n, s))
        self._barrier()  # the product is final
        t = self.torch
        w = (out_bits + 63) // 64
        out = t.empty(w, dtype=t.int64, device=c.device)
        if blocks:
            bw = (1 << 32) // 64
            self.L._check(L.fpm_copy_dev(out.data_ptr(), lo, min(w, bw) * 8, s))
            if w > bw:
                self.L._check(L.fpm_copy_dev(out.data_ptr() + bw * 8, hi, (w - bw) * 8, s))
        else:
            self.L._check(L.fpm_copy_dev(out.data_ptr(), lo, w * 8, s))
        if out_bits % 64:
            out[w - 1] &= (1 << (out_bits % 64)) - 1
        self._barrier()  # every rank copied out before the arrays are reused
        return out

    # -- hooks (the single-GPU thread test overrides these)
    def _alloc(self, nbytes: int):
        import ctypes as C
        import numpy as np
        p = C.c_void_p()
        h = np.zeros(self.L.IPC_HANDLE_BYTES, np.uint8)
        self.L._check(self.L.lib().fpm_ipc_alloc(nbytes, C.byref(p), h.ctypes.data_as(C.POINTER(C.c_uint8))))
        return p.value, bytes(h)

    def _publish(self, handles):
        out = [None] * self.world()[0]
        self.dist.all_gather_object(out, handles, group=self.group)
        return out

    def _open(self, handle):
        import ctypes as C
        import numpy as np
        p = C.c_void_p()
        h = np.frombuffer(handle, np.uint8).copy()
        self.L._check(self.L.lib().fpm_ipc_open(h.ctypes.data_as(C.POINTER(C.c_uint8)), C.byref(p)))
        return p.value

    def _barrier(self):
        self.torch.cuda.current_stream().synchronize()
        self.dist.barrier(group=self.group)

    # -- plan setup: 2 operands x ping/pong of m elements, partners' buffers opened once; with P >= 2
    # also the split conversions' arrays: converted operand a on rank 0, b on rank 1 (n/2 bits each),
    # the product array on rank 0 (n bits) -- or, for a 2^33-bit product, its two 2^32-bit blocks on
    # ranks 0 and 1 -- opened on every rank
    def begin(self, plan):
        P, rank = self.world()
        key = (plan.m, plan.n_bits, P, rank)
        if self.key != key:
            self.close()  # re-key: release the previous plan's buffers and peer mappings
            nbytes = plan.m * 16
            mine = [self._alloc(nbytes) for _ in range(4)]
            shared = self._shared_sizes(plan, P, rank)  # name -> bytes of the arrays this rank owns
            own = {k: self._alloc(v) for k, v in shared.items()}
            allh = self._publish(([h for _, h in mine], {k: h for k, (_, h) in own.items()}))
            dev = self.torch.device("cuda", self.torch.cuda.current_device())
            self.mine = [DevBuf(p, 2 * plan.m, dev) for p, _ in mine]
            self.peer = {}
            for i in range(plan.lp, plan.l):
                g = plan.partner(i)
                if g not in self.peer:
                    self.peer[g] = [self._open(h) for h in allh[g][0]]
            # split-conversion arrays: own pointer or an opened peer mapping (self.opened: to close)
            self.arrays, self.opened, self.owned = {}, [], [p for p, _ in own.values()]
            for g in range(P):
                for name, h in allh[g][1].items():
                    if g == rank:
                        self.arrays[name] = own[name][0]
                    else:
                        self.arrays[name] = self._open(h)
                        self.opened.append(self.arrays[name])
            self.key = key
        self.n_enc = 0
        self.cur = [0, 0]

    def encode_cols(self, poly, l: int, col0: int, ncols: int, tower: bool = False):
        k = self.n_enc  # (poly: a tensor, or a DevBuf over a peer rank's converted operand)
        self.n_enc += 1
        ev = self.mine[2 * k]
        if isinstance(poly, _Owners):  # the sharded conversion's column owners
            self.L._check(self.L.lib().fpm_encode_cols_owners_dev(poly.ptrs, poly.Q, l, col0, ncols, 64, ev.data_ptr(),
                                                                  int(tower), self._s()))
        else:
            f = self.L.lib().fpm_encode_cols_r_dev if tower else self.L.lib().fpm_encode_cols_dev
            self.L._check(f(poly.data_ptr(), l, col0, ncols, 64, ev.data_ptr(), self._s()))
        self.cur[k] = 0
        return ev

    def exchange_pair(self, ev, partner: int, w, side: int, inverse: bool, tower: bool = False):
        k = next(j for j in (0, 1) if self.mine[2 * j + self.cur[j]].ptr == ev.ptr)
        c = self.cur[k]
        out = self.mine[2 * k + 1 - c]
        self._barrier()  # every rank's buffer c is final; nobody still reads buffer 1 - c
        self.L._check(self.L.lib().fpm_bfly_pair_peer_dev(ev.data_ptr(), self.peer[partner][2 * k + c], out.data_ptr(),
                                                          ev.numel() // 2, w.ctypes.data_as(self.L._u64p), side,
                                                          int(inverse), int(tower), self._s()))
        self.cur[k] = 1 - c
        return out

    def pointwise(self, u, v):
        self.L._check(self.L.lib().fpm_pointwise_dev(u.data_ptr(), v.data_ptr(), u.data_ptr(), u.numel() // 2,
                                                     self._s()))
        return u
