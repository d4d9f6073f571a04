"""oracle -- TEST INFRASTRUCTURE ONLY: the checker and CPU baseline, never the product.

Two CPU implementations of the reference's fp_polymul path, both loaded with ctypes:

* ``port``: our plain-C restatement (``oracle/port/fpo.c``), every function citing the
  reference file:line it follows.  Built by ``make -C oracle port`` into ``oracle/_build``.
* ``ref``:  the UNMODIFIED reference library compiled from ``/root/reference/proj/src`` by
  ``oracle/Makefile`` into ``oracle/_ref/libfpmul_ref.so`` (plus ``libfpmul_ref_f4.so``, the
  same sources with the one-line ``digit_size`` overflow fix, needed for
  products of >= 2^33 bits).  Exposed through our C-ABI shim ``oracle/ref_shim.cpp``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and the
``--impl reference`` arm) may import this package.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "_build", "libfpmul_port.so")
REF_SO = os.path.join(HERE, "_ref", "libfpmul_ref.so")
REF_F4_SO = os.path.join(HERE, "_ref", "libfpmul_ref_f4.so")

_u64p = C.POINTER(C.c_uint64)


def build(quiet: bool = True) -> None:
    """Builds the port (always) and the reference libraries (when /root/reference exists)."""
    out = subprocess.run(["make", "-C", HERE, "-j8"], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout[-2000:] + out.stderr[-4000:])
    if not quiet:
        print(out.stdout)


def _ptr(a: np.ndarray):
    assert a.dtype == np.uint64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(_u64p)


def words_for(bits: int) -> int:
    return (bits + 63) // 64


# ----------------------------------------------------------------------------- port
class _Port:
    def __init__(self, path: str = PORT_SO):
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        L.fpo_random_bitpoly.argtypes = [C.c_size_t, C.c_uint64, _u64p]
        L.fpo_basis_cvt.argtypes = [_u64p, C.c_size_t]
        L.fpo_i_basis_cvt.argtypes = [_u64p, C.c_size_t]
        L.fpo_encode.argtypes = [C.c_uint, _u64p, C.c_uint, _u64p]
        L.fpo_decode.argtypes = [C.c_uint, _u64p, C.c_uint, _u64p]
        L.fpo_butterfly.argtypes = [C.c_uint, _u64p, C.c_uint, C.c_int]
        L.fpo_pointwise.argtypes = [C.c_uint, _u64p, _u64p, _u64p, C.c_size_t]
        L.fpo_plan_mul.argtypes = [C.c_size_t, C.c_size_t, C.c_int, _u64p]
        L.fpo_fft_polymul.argtypes = [C.c_uint, _u64p, C.c_size_t, _u64p, C.c_size_t, _u64p]
        L.fpo_naive_mul.argtypes = [_u64p, C.c_size_t, _u64p, C.c_size_t, _u64p]
        L.fpo_cantor_basis.argtypes = [C.c_uint, _u64p]
        L.fpo_encode_matrix.argtypes = [C.c_uint, _u64p, _u64p]
        L.fpo_last_error.restype = C.c_char_p
        self.L = L

    def _chk(self, rc):
        if rc:
            raise (ValueError if rc == 1 else RuntimeError)(self.L.fpo_last_error().decode())

    def random_bitpoly(self, n_bits: int, seed: int) -> np.ndarray:
        out = np.zeros(max(1, words_for(n_bits)), np.uint64)
        if n_bits:
            self.L.fpo_random_bitpoly(n_bits, seed, _ptr(out))
        return out[: words_for(n_bits)]

    def basis_cvt(self, w: np.ndarray, n_bits: int, inverse: bool = False) -> np.ndarray:
        w = np.ascontiguousarray(w, np.uint64).copy()
        fn = self.L.fpo_i_basis_cvt if inverse else self.L.fpo_basis_cvt
        self._chk(fn(_ptr(w), n_bits))
        return w

    def encode(self, m: int, a: np.ndarray, l: int) -> np.ndarray:
        ev = np.zeros(2 << l, np.uint64)
        self._chk(self.L.fpo_encode(m, _ptr(np.ascontiguousarray(a, np.uint64)), l, _ptr(ev)))
        return ev

    def decode(self, m: int, ev: np.ndarray, l: int) -> np.ndarray:
        a = np.zeros(max(1, (m << l) // 64), np.uint64)
        self._chk(self.L.fpo_decode(m, _ptr(np.ascontiguousarray(ev, np.uint64)), l, _ptr(a)))
        return a

    def butterfly(self, m: int, ev: np.ndarray, l: int, inverse: bool = False) -> np.ndarray:
        ev = np.ascontiguousarray(ev, np.uint64).copy()
        self._chk(self.L.fpo_butterfly(m, _ptr(ev), l, int(inverse)))
        return ev

    def pointwise(self, m: int, u: np.ndarray, v: np.ndarray) -> np.ndarray:
        out = np.zeros_like(u)
        self.L.fpo_pointwise(m, _ptr(u), _ptr(v), _ptr(out), u.size // 2)
        return out

    def plan_mul(self, a_bits: int, b_bits: int, field: int = 0):
        out = np.zeros(6, np.uint64)
        self._chk(self.L.fpo_plan_mul(a_bits, b_bits, field, _ptr(out)))
        return tuple(int(x) for x in out)

    def fft_polymul(self, m: int, a, a_bits, b, b_bits) -> np.ndarray:
        ob = a_bits + b_bits - 1 if a_bits and b_bits else 0
        c = np.zeros(max(1, words_for(ob)), np.uint64)
        a = np.ascontiguousarray(a, np.uint64)
        b = np.ascontiguousarray(b, np.uint64)
        self._chk(self.L.fpo_fft_polymul(m, _ptr(a), a_bits, _ptr(b), b_bits, _ptr(c)))
        return c[: words_for(ob)]

    def naive_mul(self, a, a_bits, b, b_bits) -> np.ndarray:
        ob = a_bits + b_bits - 1 if a_bits and b_bits else 0
        c = np.zeros(max(1, words_for(ob)), np.uint64)
        self.L.fpo_naive_mul(_ptr(np.ascontiguousarray(a, np.uint64)), a_bits,
                             _ptr(np.ascontiguousarray(b, np.uint64)), b_bits, _ptr(c))
        return c[: words_for(ob)]

    def cantor_basis(self, m: int) -> np.ndarray:
        out = np.zeros(2 * m, np.uint64)
        self._chk(self.L.fpo_cantor_basis(m, _ptr(out)))
        return out

    def encode_matrix(self, m: int):
        rows = np.zeros(2 * m, np.uint64)
        inv = np.zeros(2 * m, np.uint64)
        self._chk(self.L.fpo_encode_matrix(m, _ptr(rows), _ptr(inv)))
        return rows, inv


# ----------------------------------------------------------------------------- reference
class _Ref:
    """The real reference library (unmodified sources) behind oracle/ref_shim.cpp."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle` where /root/reference exists")
        L = C.CDLL(path)
        L.ref_polymul.argtypes = [_u64p, C.c_size_t, _u64p, C.c_size_t, _u64p, C.c_int, C.c_int,
                                  C.POINTER(C.c_double)]
        L.ref_karatsuba.argtypes = [_u64p, C.c_size_t, _u64p, C.c_size_t, _u64p]
        L.ref_plan_mul.argtypes = [C.c_size_t, C.c_size_t, C.c_int, _u64p]
        L.ref_random_bitpoly.argtypes = [C.c_size_t, C.c_uint64, _u64p]
        L.ref_basis_cvt.argtypes = [_u64p, C.c_size_t, C.c_size_t, C.c_int]
        L.ref_i_basis_cvt.argtypes = [_u64p, C.c_size_t, C.c_int]
        L.ref_basis_cvt_bits.argtypes = [_u64p, C.c_size_t, C.c_int]
        L.ref_encode128.argtypes = [_u64p, C.c_uint, _u64p, C.c_int]
        L.ref_decode128.argtypes = [_u64p, C.c_uint, _u64p, C.c_int]
        L.ref_butterfly128.argtypes = [_u64p, C.c_uint, C.c_int, C.c_int]
        L.ref_pointwise128.argtypes = [_u64p, _u64p, _u64p, C.c_size_t]
        L.ref_butterfly128_base.argtypes = [_u64p, C.c_uint, C.c_uint64, C.c_uint64, C.c_int]
        L.ref_gf128_mul.argtypes = [_u64p, _u64p, _u64p]
        L.ref_tables128.argtypes = [_u64p, _u64p, _u64p]
        L.ref_twiddles128.argtypes = [C.c_uint, _u64p]
        L.ref_encode64.argtypes = [_u64p, C.c_uint, _u64p]
        L.ref_decode64.argtypes = [_u64p, C.c_uint, _u64p]
        L.ref_butterfly64.argtypes = [_u64p, C.c_uint, C.c_uint64, C.c_int]
        L.ref_pointwise64.argtypes = [_u64p, _u64p, _u64p, C.c_size_t]
        L.ref_tables64.argtypes = [_u64p, _u64p, _u64p]
        L.ref_last_error.restype = C.c_char_p
        L.ref_set_threads.argtypes = [C.c_int]
        self.L = L
        self.path = path

    def _chk(self, rc):
        if rc:
            raise (ValueError if rc == 1 else RuntimeError)(self.L.ref_last_error().decode())

    def max_threads(self) -> int:
        return int(self.L.ref_max_threads())

    def set_threads(self, n: int) -> None:
        self.L.ref_set_threads(n)

    def polymul(self, a, a_bits, b, b_bits, field=0, parallel=True, stages=False):
        ob = a_bits + b_bits - 1 if a_bits and b_bits else 0
        c = np.zeros(max(1, words_for(ob)), np.uint64)
        st = (C.c_double * 7)()
        self._chk(self.L.ref_polymul(_ptr(np.ascontiguousarray(a, np.uint64)), a_bits,
                                     _ptr(np.ascontiguousarray(b, np.uint64)), b_bits, _ptr(c),
                                     field, int(parallel), st if stages else None))
        c = c[: words_for(ob)]
        return (c, list(st)) if stages else c

    def karatsuba(self, a, a_bits, b, b_bits):
        ob = a_bits + b_bits - 1 if a_bits and b_bits else 0
        c = np.zeros(max(1, words_for(ob)), np.uint64)
        self._chk(self.L.ref_karatsuba(_ptr(np.ascontiguousarray(a, np.uint64)), a_bits,
                                       _ptr(np.ascontiguousarray(b, np.uint64)), b_bits, _ptr(c)))
        return c[: words_for(ob)]

    def plan_mul(self, a_bits, b_bits, field=0):
        out = np.zeros(6, np.uint64)
        self._chk(self.L.ref_plan_mul(a_bits, b_bits, field, _ptr(out)))
        return tuple(int(x) for x in out)

    def random_bitpoly(self, n_bits, seed):
        out = np.zeros(max(1, words_for(n_bits)), np.uint64)
        if n_bits:
            self.L.ref_random_bitpoly(n_bits, seed, _ptr(out))
        return out[: words_for(n_bits)]

    def basis_cvt(self, w, n_bits, content_bits=None, inverse=False, parallel=True):
        w = np.ascontiguousarray(w, np.uint64).copy()
        if inverse:
            self._chk(self.L.ref_i_basis_cvt(_ptr(w), n_bits, int(parallel)))
        else:
            cb = n_bits if content_bits is None else content_bits
            self._chk(self.L.ref_basis_cvt(_ptr(w), n_bits, cb, int(parallel)))
        return w

    def basis_cvt_bits(self, w, n_bits, inverse=False):
        w = np.ascontiguousarray(w, np.uint64).copy()
        self._chk(self.L.ref_basis_cvt_bits(_ptr(w), n_bits, int(inverse)))
        return w

    def encode128(self, a, l, parallel=True):
        ev = np.zeros(2 << l, np.uint64)
        self._chk(self.L.ref_encode128(_ptr(np.ascontiguousarray(a, np.uint64)), l, _ptr(ev), int(parallel)))
        return ev

    def decode128(self, ev, l, parallel=True):
        a = np.zeros(max(1, (128 << l) // 64), np.uint64)
        self._chk(self.L.ref_decode128(_ptr(np.ascontiguousarray(ev, np.uint64)), l, _ptr(a), int(parallel)))
        return a

    def butterfly128(self, ev, l, inverse=False, parallel=True):
        ev = np.ascontiguousarray(ev, np.uint64).copy()
        self._chk(self.L.ref_butterfly128(_ptr(ev), l, int(inverse), int(parallel)))
        return ev

    def butterfly128_base(self, ev, l, base_lo, base_hi, inverse=False):
        ev = np.ascontiguousarray(ev, np.uint64).copy()
        self._chk(self.L.ref_butterfly128_base(_ptr(ev), l, base_lo, base_hi, int(inverse)))
        return ev

    def pointwise128(self, u, v):
        out = np.zeros_like(u)
        self._chk(self.L.ref_pointwise128(_ptr(u), _ptr(v), _ptr(out), u.size // 2))
        return out

    def gf128_mul(self, a, b):
        out = np.zeros(2, np.uint64)
        self.L.ref_gf128_mul(_ptr(np.ascontiguousarray(a, np.uint64)),
                             _ptr(np.ascontiguousarray(b, np.uint64)), _ptr(out))
        return out

    def tables128(self):
        c = np.zeros(256, np.uint64)
        r = np.zeros(256, np.uint64)
        i = np.zeros(256, np.uint64)
        self.L.ref_tables128(_ptr(c), _ptr(r), _ptr(i))
        return c, r, i

    # gf64 stages (the reference's auto field)
    def encode64(self, a, l):
        ev = np.zeros(1 << l, np.uint64)
        self._chk(self.L.ref_encode64(_ptr(np.ascontiguousarray(a, np.uint64)), l, _ptr(ev)))
        return ev

    def decode64(self, ev, l):
        a = np.zeros(max(1, (64 << l) // 64), np.uint64)
        self._chk(self.L.ref_decode64(_ptr(np.ascontiguousarray(ev, np.uint64)), l, _ptr(a)))
        return a

    def butterfly64(self, ev, l, base=None, inverse=False):
        ev = np.ascontiguousarray(ev, np.uint64).copy()
        b = (1 << (l + 32)) if base is None else base
        self._chk(self.L.ref_butterfly64(_ptr(ev), l, b, int(inverse)))
        return ev

    def pointwise64(self, u, v):
        out = np.zeros_like(u)
        self._chk(self.L.ref_pointwise64(_ptr(u), _ptr(v), _ptr(out), u.size))
        return out

    def tables64(self):
        c, r, i = (np.zeros(64, np.uint64) for _ in range(3))
        self.L.ref_tables64(_ptr(c), _ptr(r), _ptr(i))
        return c, r, i

    def twiddles128(self, l):
        out = np.zeros(2 * ((1 << l) - 1) if l else 2, np.uint64)
        self._chk(self.L.ref_twiddles128(l, _ptr(out)))
        return out


_port = None
_ref = {}


def port() -> _Port:
    global _port
    if _port is None:
        _port = _Port()
    return _port


def ref(f4: bool = False) -> _Ref:
    key = REF_F4_SO if f4 else REF_SO
    if key not in _ref:
        _ref[key] = _Ref(key)
    return _ref[key]


def have_ref() -> bool:
    return os.path.exists(REF_SO)
