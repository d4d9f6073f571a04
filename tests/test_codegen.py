"""CPU test of the generated register-level basis conversions (csrc/conv_regs_gen.cuh): the header is
compiled with g++ (CUDA intrinsics stubbed) and every aligned 2^r-bit span of random 256-bit rows is
compared with the oracle's pass-by-pass conversion (proj/src/basis_convert.cpp semantics)."""
import ctypes as C
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_1803_11301_b200", "csrc")

HARNESS = r"""
#include <cstdint>
#include <cstring>
#define __device__
#define __constant__
#define __forceinline__ inline
static inline uint32_t __funnelshift_r(uint32_t lo, uint32_t hi, unsigned s) { s &= 31; return s ? (lo >> s) | (hi << (32 - s)) : lo; }
#include "conv_regs_gen.cuh"
extern "C" void run(int r, int inv, uint32_t* w) {
  uint32_t a[8]; memcpy(a, w, 32);
  if (inv) fpm::conv_regs<true>(r, a); else fpm::conv_regs<false>(r, a);
  memcpy(w, a, 32);
}
extern "C" int rowsched(int g, int k, int which) {
  return which == 0 ? fpm::kRowSchedN[g] : which == 1 ? fpm::kRowSchedS[g][k] : fpm::kRowSchedD[g][k];
}
"""


def _lib(tmp_path):
    src = tmp_path / "h.cpp"
    src.write_text(HARNESS)
    so = tmp_path / "libh.so"
    subprocess.run(["g++", "-O1", "-shared", "-fPIC", "-I", CSRC, str(src), "-o", str(so)], check=True)
    return C.CDLL(str(so))


def test_generated_header_is_current(tmp_path):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "gen_conv_regs.py")], capture_output=True,
                         text=True, check=True).stdout
    assert out == open(os.path.join(CSRC, "conv_regs_gen.cuh")).read(), "regenerate conv_regs_gen.cuh"


def test_register_conversions_match_oracle(tmp_path, port):
    L = _lib(tmp_path)
    rng = np.random.default_rng(0)
    for r in range(1, 9):
        n = 1 << r
        for _ in range(20):
            row = rng.integers(0, 2**32, 8, dtype=np.uint64).astype(np.uint32)
            w = row.copy()
            L.run(r, 0, w.ctypes.data_as(C.c_void_p))
            bits = np.unpackbits(row.view(np.uint8), bitorder="little")
            want = bits.copy()
            for s in range(0, 256, n):
                seg = np.concatenate([bits[s:s + n], np.zeros((-n) % 64, np.uint8)])
                words = np.packbits(seg, bitorder="little").view(np.uint64)
                want[s:s + n] = np.unpackbits(port.basis_cvt(words, n).view(np.uint8), bitorder="little")[:n]
            assert np.array_equal(np.unpackbits(w.view(np.uint8), bitorder="little"), want), r
            L.run(r, 1, w.ctypes.data_as(C.c_void_p))
            assert np.array_equal(w, row), r


def test_row_schedules(tmp_path):
    sys.path.insert(0, os.path.join(ROOT, "tools", "models"))
    from bc_model import build
    L = _lib(tmp_path)
    for g in range(9):
        sc = []
        build(sc, 1 << g, 1)
        assert L.rowsched(g, 0, 0) == len(sc)
        for k, (S, D) in enumerate(sc):
            assert (L.rowsched(g, k, 1), L.rowsched(g, k, 2)) == (S, D)
