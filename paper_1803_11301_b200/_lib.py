"""ctypes binding of libfpmul_b200.so (include/fpmul_b200.h).

Host-buffer calls take numpy uint64 arrays (packed little-endian words, coefficient k = bit k%64
of word k//64, as proj/include/fpmul/bitpoly.hpp).  Device calls take torch CUDA tensors (any
8-byte dtype) and run on the current torch stream.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
IPC_HANDLE_BYTES = 64  # FPM_IPC_HANDLE_BYTES (include/fpmul_b200.h)
LIB_PATH = os.environ.get("FPM_LIB") or os.path.join(HERE, "libfpmul_b200.so")  # FPM_LIB: experiment builds

FIELD_AUTO, FIELD_GF64, FIELD_GF128 = 0, 64, 128
NUM_STAGES = 7
# StageSeconds order (proj/include/fpmul/polymul.hpp:51-59)
STAGE_NAMES = ("basiscvt", "encode", "butterfly", "pointwise", "ibutterfly", "decode", "ibasiscvt")

_u64p = C.POINTER(C.c_uint64)


class FpmError(RuntimeError):
    """A CUDA-side failure (FPM_ECUDA / FPM_ENOMEM)."""


class _Plan(C.Structure):
    _fields_ = [("n_bits", C.c_uint64), ("log2_n", C.c_uint32), ("field_degree", C.c_uint32),
                ("log2_field_degree", C.c_uint32), ("l", C.c_uint32), ("n_p", C.c_uint64)]


_LIB = None


def lib():
    """Loads the in-tree CUDA library; raises if it was not built (no fallback exists)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise FpmError(f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
                           "(there is no CPU fallback for the B200 path)")
        L = C.CDLL(LIB_PATH)
        vp = C.c_void_p
        sz = C.c_size_t
        L.fpm_last_error.restype = C.c_char_p
        L.fpm_version.restype = C.c_char_p
        L.fpm_fft_tile_log2.restype = C.c_uint
        L.fpm_fft_tile_log2.argtypes = [C.c_uint]
        L.fpm_pipeline_fuses_operands.argtypes = [C.c_uint]
        L.fpm_launch_count.restype = C.c_uint64
        L.fpm_launch_count.argtypes = [C.c_int]
        L.fpm_plan_mul.argtypes = [sz, sz, C.c_int, C.POINTER(_Plan)]
        L.fpm_random_bitpoly.argtypes = [sz, C.c_uint64, _u64p]
        L.fpm_polymul.argtypes = [_u64p, sz, _u64p, sz, _u64p, C.c_int, C.c_int, C.POINTER(C.c_double)]
        L.fpm_polymul_dev.argtypes = [vp, sz, vp, sz, vp, C.c_int, vp, C.POINTER(C.c_double)]
        L.fpm_polymul_multi.argtypes = [_u64p, sz, _u64p, sz, _u64p, C.c_int, C.POINTER(C.c_int), C.c_int]
        L.fpm_polymul_n.argtypes = [_u64p, sz, _u64p, sz, _u64p, C.c_int, C.c_int]
        L.fpm_trim_pool.argtypes = [C.c_int]
        L.fpm_reserve_pool.argtypes = [C.c_int, C.c_size_t]
        L.fpm_test_flip_encode_table.argtypes = [C.c_int]
        L.fpm_polymul_batch_dev.argtypes = [vp, sz, sz, vp, sz, sz, vp, sz, sz, vp]
        L.fpm_polymul_batch.argtypes = [_u64p, sz, sz, _u64p, sz, sz, _u64p, sz, sz, C.c_int]
        L.fpm_basis_cvt_dev.argtypes = [vp, sz, sz, vp]
        L.fpm_i_basis_cvt_dev.argtypes = [vp, sz, vp]
        L.fpm_encode_dev.argtypes = [vp, C.c_uint, vp, vp]
        L.fpm_decode_dev.argtypes = [vp, C.c_uint, vp, vp]
        L.fpm_butterfly_dev.argtypes = [vp, C.c_uint, C.c_int, vp]
        L.fpm_pointwise_dev.argtypes = [vp, vp, vp, sz, vp]
        L.fpm_basis_cvt.argtypes = [_u64p, sz, sz, C.c_int]
        L.fpm_i_basis_cvt.argtypes = [_u64p, sz, C.c_int]
        L.fpm_encode.argtypes = [_u64p, C.c_uint, _u64p, C.c_int]
        L.fpm_decode.argtypes = [_u64p, C.c_uint, _u64p, C.c_int]
        L.fpm_butterfly.argtypes = [_u64p, C.c_uint, C.c_int, C.c_int]
        L.fpm_pointwise.argtypes = [_u64p, _u64p, _u64p, sz, C.c_int]
        L.fpm_gf128_mul.argtypes = [_u64p, _u64p, _u64p, sz, C.c_int]
        L.fpm_tables128.argtypes = [_u64p, _u64p, _u64p]
        L.fpm_tables64.argtypes = [_u64p, _u64p, _u64p]
        L.fpm_tower_tables.argtypes = [C.c_int, _u64p, _u64p, _u64p, C.POINTER(C.c_uint8)]
        L.fpm_encode64.argtypes = [_u64p, C.c_uint, _u64p, C.c_int]
        L.fpm_decode64.argtypes = [_u64p, C.c_uint, _u64p, C.c_int]
        L.fpm_lch_butterfly64.argtypes = [_u64p, C.c_uint, C.c_uint64, C.c_int, C.c_int]
        L.fpm_pointwise64.argtypes = [_u64p, _u64p, _u64p, sz, C.c_int]
        L.fpm_lch_butterfly_dev.argtypes = [vp, C.c_uint, _u64p, C.c_int, vp]
        L.fpm_lch_butterfly.argtypes = [_u64p, C.c_uint, _u64p, C.c_int, C.c_int]
        L.fpm_encode_cols_dev.argtypes = [vp, C.c_uint, sz, sz, C.c_int, vp, vp]
        L.fpm_decode_cols_dev.argtypes = [vp, sz, vp, vp]
        L.fpm_bfly_pair_dev.argtypes = [vp, vp, sz, _u64p, C.c_int, C.c_int, vp]
        L.fpm_twiddle128.argtypes = [C.c_uint, C.c_uint64, _u64p, _u64p]
        L.fpm_shard_tower.argtypes = [C.c_uint]
        L.fpm_shard_tower.restype = C.c_int
        L.fpm_encode_cols_r_dev.argtypes = [vp, C.c_uint, sz, sz, C.c_int, vp, vp]
        L.fpm_decode_cols_r_dev.argtypes = [vp, sz, vp, vp]
        L.fpm_bfly_pair_r_dev.argtypes = [vp, vp, sz, _u64p, C.c_int, C.c_int, vp]
        L.fpm_shard_local_product_dev.argtypes = [vp, vp, C.c_uint, _u64p, vp]
        L.fpm_bfly_pair_peer_dev.argtypes = [vp, vp, vp, sz, _u64p, C.c_int, C.c_int, C.c_int, vp]
        L.fpm_load_operand_dev.argtypes = [vp, sz, vp, sz, vp]
        L.fpm_decode_cols_split_dev.argtypes = [vp, sz, sz, sz, vp, vp, C.c_int, vp]
        L.fpm_i_basis_cvt_block32_dev.argtypes = [vp, vp, vp]
        L.fpm_top_bit_fix_dev.argtypes = [vp, vp]
        L.fpm_copy_dev.argtypes = [vp, vp, sz, vp]
        pp = C.POINTER(C.c_void_p)
        L.fpm_b32_regather_dev.argtypes = [vp, pp, C.c_int, C.c_int, C.c_int, C.c_int, vp]
        L.fpm_b32_l1_outer_dev.argtypes = [vp, vp, C.c_int, C.c_int, C.c_int, vp]
        L.fpm_b32_l1_outer_fix_dev.argtypes = [vp, vp, C.c_int, C.c_uint, C.c_uint, vp]
        L.fpm_b32_rows_dev.argtypes = [vp, sz, C.c_int, vp]
        L.fpm_b32_cols_dev.argtypes = [vp, C.c_int, C.c_int, C.c_int, vp]
        L.fpm_b32_top_pass_dev.argtypes = [vp, pp, C.c_int, C.c_int, vp]
        L.fpm_b32_top_bit_fix_dev.argtypes = [vp, vp, vp]
        L.fpm_encode_cols_owners_dev.argtypes = [pp, C.c_int, C.c_uint, sz, sz, C.c_int, vp, C.c_int, vp]
        L.fpm_decode_cols_owners_dev.argtypes = [vp, sz, sz, sz, pp, pp, C.c_int, C.c_int, vp]
        L.fpm_ipc_alloc.argtypes = [sz, C.POINTER(vp), C.POINTER(C.c_uint8)]
        L.fpm_ipc_open.argtypes = [C.POINTER(C.c_uint8), C.POINTER(vp)]
        L.fpm_ipc_close.argtypes = [vp]
        L.fpm_ipc_free.argtypes = [vp]
        L.fpm_karatsuba_mul.argtypes = [_u64p, sz, _u64p, sz, _u64p, C.c_int]
        L.fpm_clmul_words_dev.argtypes = [vp, sz, vp, sz, vp, vp]
        _LIB = L
    return _LIB


def _check(rc: int) -> None:
    if rc == 0:
        return
    msg = lib().fpm_last_error().decode()
    if rc == 1:
        raise ValueError(msg)
    raise FpmError(msg)


def _ptr(a: np.ndarray):
    if a.dtype != np.uint64 or not a.flags["C_CONTIGUOUS"]:
        raise TypeError("expected a C-contiguous uint64 array")
    return a.ctypes.data_as(_u64p)


def _words(bits: int) -> int:
    return (bits + 63) // 64


def _as_u64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.uint64)


def device_count() -> int:
    return int(lib().fpm_device_count())


def trim_pool(device: int = 0) -> None:
    """Returns the library's cached device scratch to the driver (fpm_trim_pool)."""
    _check(lib().fpm_trim_pool(int(device)))


def reserve_pool(nbytes: int, device: int = 0) -> None:
    """Grows the library's scratch pool ahead of time (fpm_reserve_pool): about 5 GiB per concurrent
    2^33-bit host-buffer caller, so that no product pays for fresh device memory inside its call."""
    _check(lib().fpm_reserve_pool(int(device), int(nbytes)))


def launch_count(reset: bool = False) -> int:
    return int(lib().fpm_launch_count(int(reset)))


def fft_tile_log2(l: int) -> int:
    """Product pipeline: butterfly layers below this run in shared-memory tiles, the rest in
    radix-4 passes."""
    return int(lib().fpm_fft_tile_log2(l))


def pipeline_fuses_operands(l: int) -> bool:
    """Whether both operands' tile layers run inside the fused pointwise pass."""
    return bool(lib().fpm_pipeline_fuses_operands(l))


def plan_mul(a_bits: int, b_bits: int, field: int = FIELD_AUTO) -> dict:
    """plan_mul (proj/src/polymul.cpp:187-219)."""
    p = _Plan()
    _check(lib().fpm_plan_mul(a_bits, b_bits, field, C.byref(p)))
    return {k: int(getattr(p, k)) for k, _ in _Plan._fields_}


def random_bitpoly(n_bits: int, seed: int) -> np.ndarray:
    """random_bitpoly(n_bits, std::mt19937_64(seed)) (proj/src/bitpoly.cpp:19-24): packed words."""
    out = np.zeros(max(1, _words(n_bits)), np.uint64)
    _check(lib().fpm_random_bitpoly(n_bits, seed, _ptr(out)))
    return out[: _words(n_bits)]


def tables128():
    """(cantor, rows, inv_rows): CantorField<gf128> basis and EncodeMatrix<gf128> rows, each 256 words."""
    out = [np.zeros(256, np.uint64) for _ in range(3)]
    _check(lib().fpm_tables128(*[_ptr(o) for o in out]))
    return tuple(out)


# ----------------------------------------------------------------------------- host buffers
def fp_polymul(a, a_bits: int, b, b_bits: int, field: int = FIELD_AUTO, device: int = 0,
               stage_seconds: list | None = None, out: np.ndarray | None = None) -> np.ndarray:
    """fp_polymul (proj/src/polymul.cpp:223-239): returns ceil((a_bits+b_bits-1)/64) words
    (written into `out` when given, e.g. a pinned buffer)."""
    a, b = _as_u64(a), _as_u64(b)
    if a.size < _words(a_bits) or b.size < _words(b_bits):
        raise ValueError("fp_polymul: word arrays shorter than the declared bit lengths")
    if a_bits == 0 or b_bits == 0:
        return np.zeros(0, np.uint64)
    if out is not None:
        if out.dtype != np.uint64 or out.size < _words(a_bits + b_bits - 1):
            raise ValueError("fp_polymul: output buffer too small")
        c = out
    else:
        c = np.zeros(_words(a_bits + b_bits - 1), np.uint64)
    st = (C.c_double * NUM_STAGES)()
    _check(lib().fpm_polymul(_ptr(a), a_bits, _ptr(b), b_bits, _ptr(c), field, device,
                             st if stage_seconds is not None else None))
    if stage_seconds is not None:
        stage_seconds[:] = list(st)
    return c


def fp_polymul_multi(a, a_bits: int, b, b_bits: int, devices, field: int = FIELD_AUTO,
                     out: np.ndarray | None = None) -> np.ndarray:
    """fp_polymul sharded over several GPUs from this process (fpm_polymul_multi): `devices` lists
    the logical ranks (a power of two; a device may repeat, e.g. [0, 0, 0, 0])."""
    a, b = _as_u64(a), _as_u64(b)
    if a.size < _words(a_bits) or b.size < _words(b_bits):
        raise ValueError("fp_polymul_multi: word arrays shorter than the declared bit lengths")
    if a_bits == 0 or b_bits == 0:
        return np.zeros(0, np.uint64)
    c = out if out is not None else np.zeros(_words(a_bits + b_bits - 1), np.uint64)
    if c.dtype != np.uint64 or c.size < _words(a_bits + b_bits - 1):
        raise ValueError("fp_polymul_multi: output buffer too small")
    devs = (C.c_int * len(devices))(*devices)
    _check(lib().fpm_polymul_multi(_ptr(a), a_bits, _ptr(b), b_bits, _ptr(c), field, devs, len(devices)))
    return c


def karatsuba_mul(a, a_bits: int, b, b_bits: int, device: int = 0) -> np.ndarray:
    """karatsuba_mul (proj/src/polymul.cpp:268-282): the exact product by word-level carry-less
    multiplication on the GPU, no FFT -- the independent cross-check of fp_polymul."""
    a, b = _as_u64(a), _as_u64(b)
    if a.size < _words(a_bits) or b.size < _words(b_bits):
        raise ValueError("karatsuba_mul: word arrays shorter than the declared bit lengths")
    if a_bits == 0 or b_bits == 0:
        return np.zeros(0, np.uint64)
    c = np.zeros(_words(a_bits + b_bits - 1), np.uint64)
    _check(lib().fpm_karatsuba_mul(_ptr(a), a_bits, _ptr(b), b_bits, _ptr(c), device))
    return c


naive_mul = karatsuba_mul  # polymul.hpp:83: the same exact product


def basis_cvt(w, n_bits: int, content_bits: int | None = None, device: int = 0) -> np.ndarray:
    """basis_cvt (proj/src/basis_convert.cpp:337-341); returns the converted copy."""
    w = _as_u64(w).copy()
    if w.size < _words(n_bits):
        raise ValueError("basis_cvt: word array shorter than n_bits")
    cb = (1 << 64) - 1 if content_bits is None else content_bits
    _check(lib().fpm_basis_cvt(_ptr(w), n_bits, cb, device))
    return w


def i_basis_cvt(w, n_bits: int, device: int = 0) -> np.ndarray:
    w = _as_u64(w).copy()
    if w.size < _words(n_bits):
        raise ValueError("i_basis_cvt: word array shorter than n_bits")
    _check(lib().fpm_i_basis_cvt(_ptr(w), n_bits, device))
    return w


def tables64():
    """(cantor, rows, inv_rows) of CantorField<gf64> / EncodeMatrix<gf64>, 64 words each."""
    out = [np.zeros(64, np.uint64) for _ in range(3)]
    _check(lib().fpm_tables64(*[_ptr(o) for o in out]))
    return tuple(out)


def tower_tables(field_degree: int):
    """(t, to_poly, to_r, tau) of the pipeline's internal tower representation (fpm_tower_tables):
    t as 2 words, to_poly / to_r as (m, 2) word arrays, tau as 8 bytes.  Host only."""
    t = np.zeros(2, np.uint64)
    tp = np.zeros(2 * field_degree, np.uint64)
    tr = np.zeros(2 * field_degree, np.uint64)
    tau = np.zeros(8, np.uint8)
    _check(lib().fpm_tower_tables(field_degree, _ptr(t), _ptr(tp), _ptr(tr), tau.ctypes.data_as(C.POINTER(C.c_uint8))))
    return t, tp.reshape(-1, 2), tr.reshape(-1, 2), tau


def encode64(poly, l: int, device: int = 0) -> np.ndarray:
    """encode<gf64> with make_partition_spec<gf64>(l): 64 rows of 2^l bits -> 2^l uint64 elements."""
    poly = _as_u64(poly)
    if l >= 32:
        raise ValueError("PartitionSpec: l must satisfy l < m/2")
    if poly.size != max(1, (64 << l) // 64):
        raise ValueError("encode: input length must be m * n_p bits")
    ev = np.zeros(1 << l, np.uint64)
    _check(lib().fpm_encode64(_ptr(poly), l, _ptr(ev), device))
    return ev


def decode64(ev, l: int, device: int = 0) -> np.ndarray:
    ev = _as_u64(ev)
    if l >= 32:
        raise ValueError("PartitionSpec: l must satisfy l < m/2")
    if ev.size != (1 << l):
        raise ValueError("decode: length must equal n_p")
    poly = np.zeros(max(1, (64 << l) // 64), np.uint64)
    _check(lib().fpm_decode64(_ptr(ev), l, _ptr(poly), device))
    return poly


def lch_butterfly64(ev, l: int, base: int | None = None, inverse: bool = False, device: int = 0) -> np.ndarray:
    """lch_butterfly<gf64> / i_lch_butterfly<gf64> with plan_butterflies(l, base); base defaults to
    the partition base e_{l+32}."""
    ev = _as_u64(ev).copy()
    if ev.size != (1 << l):
        raise ValueError("lch_butterfly: vector length does not match plan")
    b = (1 << (l + 32)) if base is None else base
    _check(lib().fpm_lch_butterfly64(_ptr(ev), l, b, int(inverse), device))
    return ev


def pointwise64(u, v, device: int = 0) -> np.ndarray:
    u, v = _as_u64(u), _as_u64(v)
    if u.size != v.size:
        raise ValueError("pointwise_mul: length mismatch")
    out = np.zeros_like(u)
    _check(lib().fpm_pointwise64(_ptr(u), _ptr(v), _ptr(out), u.size, device))
    return out


def encode(poly, l: int, device: int = 0) -> np.ndarray:
    """encode<gf128> with make_partition_spec<gf128>(l) (proj/src/encode.cpp:165-193)."""
    poly = _as_u64(poly)
    if l >= 64:
        raise ValueError("PartitionSpec: l must satisfy l < m/2")
    if poly.size * 64 != (128 << l):
        raise ValueError("encode: input length must be m * n_p bits")
    ev = np.zeros(2 << l, np.uint64)
    _check(lib().fpm_encode(_ptr(poly), l, _ptr(ev), device))
    return ev


def decode(ev, l: int, device: int = 0) -> np.ndarray:
    ev = _as_u64(ev)
    if l >= 64:
        raise ValueError("PartitionSpec: l must satisfy l < m/2")
    if ev.size != (2 << l):
        raise ValueError("decode: length must equal n_p")
    poly = np.zeros(max(1, (128 << l) // 64), np.uint64)
    _check(lib().fpm_decode(_ptr(ev), l, _ptr(poly), device))
    return poly


def butterfly(ev, l: int, inverse: bool = False, device: int = 0) -> np.ndarray:
    ev = _as_u64(ev).copy()
    if ev.size != (2 << l):
        raise ValueError("lch_butterfly: vector length does not match plan")
    _check(lib().fpm_butterfly(_ptr(ev), l, int(inverse), device))
    return ev


def lch_butterfly(ev, l: int, device: int = 0) -> np.ndarray:
    """lch_butterfly<gf128> with plan_butterflies(l, make_partition_spec(l).base)."""
    return butterfly(ev, l, False, device)


def i_lch_butterfly(ev, l: int, device: int = 0) -> np.ndarray:
    return butterfly(ev, l, True, device)


def pointwise_mul(u, v, device: int = 0) -> np.ndarray:
    """pointwise_mul<gf128> (proj/src/polymul.cpp:241-257)."""
    u, v = _as_u64(u), _as_u64(v)
    if u.size != v.size:
        raise ValueError("pointwise_mul: length mismatch")
    out = np.zeros_like(u)
    _check(lib().fpm_pointwise(_ptr(u), _ptr(v), _ptr(out), u.size // 2, device))
    return out


def gf128_mul(a, b, device: int = 0) -> np.ndarray:
    return pointwise_mul(a, b, device)


# ----------------------------------------------------------------------------- device buffers
def _dptr(t) -> int:
    if t is None:
        return 0
    if not t.is_cuda or not t.is_contiguous() or t.element_size() != 8:
        raise TypeError("expected a contiguous CUDA tensor of 8-byte elements")
    return t.data_ptr()


def _stream(stream):
    if stream is not None:
        return stream
    import torch
    return torch.cuda.current_stream().cuda_stream


def clmul_words_dev(a, b, out, stream=None) -> None:
    """naive_mul_words_kernel (detail/kernels.hpp:115-118) on device tensors: out[0 .. a.numel() +
    b.numel()) = a * b carry-less (overwritten)."""
    if out.numel() < a.numel() + b.numel():
        raise ValueError("clmul_words_dev: output shorter than a + b words")
    _check(lib().fpm_clmul_words_dev(_dptr(a), a.numel(), _dptr(b), b.numel(), _dptr(out), _stream(stream)))


def fp_polymul_dev(a, a_bits: int, b, b_bits: int, c, field: int = FIELD_AUTO, stream=None,
                   stage_seconds: list | None = None) -> None:
    """fp_polymul on device-resident tensors; c must hold ceil((a_bits+b_bits-1)/64) words."""
    if a_bits and b_bits:
        if a.numel() < _words(a_bits) or b.numel() < _words(b_bits):
            raise ValueError("fp_polymul_dev: operand tensors shorter than the declared bit lengths")
        if c.numel() < _words(a_bits + b_bits - 1):
            raise ValueError("fp_polymul_dev: product tensor shorter than ceil((a_bits+b_bits-1)/64) words")
    st = (C.c_double * NUM_STAGES)()
    _check(lib().fpm_polymul_dev(_dptr(a), a_bits, _dptr(b), b_bits, _dptr(c), field, _stream(stream),
                                 st if stage_seconds is not None else None))
    if stage_seconds is not None:
        stage_seconds[:] = [x + y for x, y in zip(stage_seconds, st)] if len(stage_seconds) == NUM_STAGES else list(st)


def fp_polymul_batch_dev(a, a_bits: int, a_stride: int, b, b_bits: int, b_stride: int, c, c_stride: int,
                         count: int, stream=None) -> None:
    """count independent products: a[k*a_stride ..] (a_bits) x b[k*b_stride ..] (b_bits) -> c[k*c_stride ..]."""
    if count and a_bits and b_bits:
        wa, wb, wc = _words(a_bits), _words(b_bits), _words(a_bits + b_bits - 1)
        if a_stride < wa or b_stride < wb or c_stride < wc:
            raise ValueError("fp_polymul_batch_dev: a stride is shorter than its operand / product")
        for t, stride, w, name in ((a, a_stride, wa, "a"), (b, b_stride, wb, "b"), (c, c_stride, wc, "c")):
            if t.numel() < (count - 1) * stride + w:
                raise ValueError(f"fp_polymul_batch_dev: tensor {name} shorter than (count-1)*stride + words")
    _check(lib().fpm_polymul_batch_dev(_dptr(a), a_bits, a_stride, _dptr(b), b_bits, b_stride, _dptr(c),
                                       c_stride, count, _stream(stream)))


def fp_polymul_batch(a, a_bits: int, a_stride: int, b, b_bits: int, b_stride: int, c, c_stride: int, count: int,
                     device: int = 0) -> None:
    """fp_polymul_batch_dev on HOST numpy uint64 arrays (fpm_polymul_batch: chunked, uploads, products
    and downloads overlapped); c is filled in place."""
    a, b = _as_u64(a), _as_u64(b)
    if c.dtype != np.uint64 or not c.flags.c_contiguous:
        raise ValueError("fp_polymul_batch: c must be a contiguous uint64 array")
    if count and a_bits and b_bits:
        wa, wb, wc = _words(a_bits), _words(b_bits), _words(a_bits + b_bits - 1)
        if a_stride < wa or b_stride < wb or c_stride < wc:
            raise ValueError("fp_polymul_batch: a stride is shorter than its operand / product")
        for t, stride, w, name in ((a, a_stride, wa, "a"), (b, b_stride, wb, "b"), (c, c_stride, wc, "c")):
            if t.size < (count - 1) * stride + w:
                raise ValueError(f"fp_polymul_batch: array {name} shorter than (count-1)*stride + words")
    _check(lib().fpm_polymul_batch(_ptr(a), a_bits, a_stride, _ptr(b), b_bits, b_stride, _ptr(c), c_stride, count,
                                   device))


def stage_dev(name: str, *args, stream=None) -> None:
    """Device-buffer stage entry points: basis_cvt(w, n_bits, content_bits), i_basis_cvt(w, n_bits),
    encode(poly, l, ev), decode(ev, l, poly), butterfly(ev, l, inverse), pointwise(u, v, out, n)."""
    L, s = lib(), _stream(stream)
    if name == "basis_cvt":
        w, n_bits, cb = args
        _check(L.fpm_basis_cvt_dev(_dptr(w), n_bits, cb, s))
    elif name == "i_basis_cvt":
        w, n_bits = args
        _check(L.fpm_i_basis_cvt_dev(_dptr(w), n_bits, s))
    elif name == "encode":
        poly, l, ev = args
        _check(L.fpm_encode_dev(_dptr(poly), l, _dptr(ev), s))
    elif name == "decode":
        ev, l, poly = args
        _check(L.fpm_decode_dev(_dptr(ev), l, _dptr(poly), s))
    elif name == "butterfly":
        ev, l, inv = args
        _check(L.fpm_butterfly_dev(_dptr(ev), l, int(inv), s))
    elif name == "pointwise":
        u, v, out, n = args
        _check(L.fpm_pointwise_dev(_dptr(u), _dptr(v), _dptr(out), n, s))
    else:
        raise ValueError(f"unknown stage {name!r}")
