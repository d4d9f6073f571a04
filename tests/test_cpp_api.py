"""The reference's C++ API through the B200 backend: tests/cpp/test_api.cpp compiled against the
mirror headers (paper_1803_11301_b200/cpp/include/fpmul) and linked to libfpmul_b200.so."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_1803_11301_b200")


@pytest.fixture(scope="module")
def test_api(tmp_path_factory):
    out = tmp_path_factory.mktemp("cpp") / "test_api"
    subprocess.run(["g++", "-std=c++20", "-O1", "-Wall", "-I", os.path.join(PKG, "cpp", "include"),
                    os.path.join(ROOT, "tests", "cpp", "test_api.cpp"), "-L", PKG, "-lfpmul_b200",
                    f"-Wl,-rpath,{PKG}", "-o", str(out)], check=True)
    return str(out)


def test_cpp_api_host_parts(test_api):
    r = subprocess.run([test_api, "cpu"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASS" in r.stdout


@pytest.mark.gpu
def test_cpp_api_on_gpu(test_api):
    r = subprocess.run([test_api], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]
    assert "PASS" in r.stdout


@pytest.mark.gpu
def test_cpp_api_multi_gpu_logical_ranks(test_api):
    """MulOptions::devices = {0, ..., 0}: fp_polymul sharded over P = 2/4/8 logical ranks through
    the C++ API (fpm_polymul_multi), against karatsuba_mul and the single-GPU pipeline."""
    r = subprocess.run([test_api, "multi"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]
    assert "PASS" in r.stdout
