"""paper_1803_11301_b200 -- B200-native Frobenius-partition additive-FFT multiplication of GF(2)[x]
polynomials (arXiv 1803.11301), over GF(2^128).

The product is the CUDA library ``libfpmul_b200.so`` (C-ABI in ``include/fpmul_b200.h``; C++
mirror of the reference ``fpmul::`` API in ``cpp/include/fpmul``).  This module is a thin ctypes
host layer over that C-ABI, mirroring the reference names (``fp_polymul``, ``plan_mul``,
``basis_cvt``, ``encode``, ``lch_butterfly`` ... from /root/reference/proj/include/fpmul) with
the same argument meaning and error behaviour (ValueError for the reference's
``std::invalid_argument``, RuntimeError otherwise).  There is no CPU fallback: every call goes to
the GPU and fails loudly when the library or a device is missing.
"""
from __future__ import annotations

from ._lib import (  # noqa: F401
    FIELD_AUTO,
    FIELD_GF64,
    FIELD_GF128,
    NUM_STAGES,
    STAGE_NAMES,
    LIB_PATH,
    FpmError,
    basis_cvt,
    butterfly,
    decode,
    device_count,
    encode,
    fp_polymul,
    fp_polymul_multi,
    karatsuba_mul,
    naive_mul,
    clmul_words_dev,
    fp_polymul_batch,
    fp_polymul_batch_dev,
    fp_polymul_dev,
    gf128_mul,
    i_basis_cvt,
    i_lch_butterfly,
    launch_count,
    lch_butterfly,
    lib,
    decode64,
    encode64,
    fft_tile_log2,
    pipeline_fuses_operands,
    lch_butterfly64,
    pointwise64,
    tables64,
    plan_mul,
    pointwise_mul,
    random_bitpoly,
    reserve_pool,
    trim_pool,
    stage_dev,
    tables128,
    tower_tables,
)

__all__ = [n for n in dir() if not n.startswith("_")]
