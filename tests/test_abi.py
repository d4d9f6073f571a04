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
