import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests through the C-ABI")
    config.addinivalue_line("markers", "slow: long-running (large configs)")


@pytest.fixture(scope="session")
def port():
    import oracle
    return oracle.port()


@pytest.fixture(scope="session")
def ref():
    import oracle
    if not oracle.have_ref():
        pytest.skip("reference library not built (oracle/_ref); run make -C oracle where /root/reference exists")
    return oracle.ref()


@pytest.fixture(scope="session")
def checker():
    """The strongest available oracle: the reference library when built, else the C port."""
    import oracle
    if oracle.have_ref():
        R = oracle.ref()
        class _C:
            name = "reference"
            def polymul(self, a, la, b, lb):
                return R.polymul(a, la, b, lb, field=128)
            basis_cvt = staticmethod(lambda w, n, content=None: R.basis_cvt(w, n, content))
            i_basis_cvt = staticmethod(lambda w, n: R.basis_cvt(w, n, inverse=True))
            encode = staticmethod(lambda a, l: R.encode128(a, l))
            decode = staticmethod(lambda e, l: R.decode128(e, l))
            butterfly = staticmethod(lambda e, l, inv=False: R.butterfly128(e, l, inv))
            pointwise = staticmethod(lambda u, v: R.pointwise128(u, v))
        return _C()
    P = oracle.port()
    class _P:
        name = "port"
        def polymul(self, a, la, b, lb):
            return P.fft_polymul(128, a, la, b, lb)
        basis_cvt = staticmethod(lambda w, n, content=None: P.basis_cvt(w, n))
        i_basis_cvt = staticmethod(lambda w, n: P.basis_cvt(w, n, inverse=True))
        encode = staticmethod(lambda a, l: P.encode(128, a, l))
        decode = staticmethod(lambda e, l: P.decode(128, e, l))
        butterfly = staticmethod(lambda e, l, inv=False: P.butterfly(128, e, l, inv))
        pointwise = staticmethod(lambda u, v: P.pointwise(128, u, v))
    return _P()


@pytest.fixture(scope="session")
def gpu():
    import paper_1803_11301_b200 as pkg
    if pkg.device_count() == 0:
        pytest.fail("no CUDA device visible: the gpu tests must run on a B200 (no CPU fallback exists)")
    return pkg
