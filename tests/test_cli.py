"""The reference's `fpmul` command line (proj/tools/fpmul_main.cpp) on the B200 backend:
paper_1803_11301_b200/fpmul_b200 {mul, selftest, bench}; exit codes 0 ok / 1 verification failure /
2 usage or I/O error; file format of proj/src/io.cpp (LE bytes, trimmed output)."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_1803_11301_b200", "fpmul_b200")


def run(*args, timeout=600):
    if not os.path.exists(CLI):
        pytest.skip("CLI not built (make -C paper_1803_11301_b200/csrc)")
    return subprocess.run([CLI, *args], capture_output=True, text=True, timeout=timeout)


def test_usage_errors():
    assert run().returncode == 2
    assert run("frobnicate").returncode == 2
    assert run("bench", "--min-log", "3").returncode == 2
    assert run("bench", "--min-log", "5", "--max-log", "3").returncode == 2
    assert run("mul", "a").returncode == 2
    assert run("mul", "/nonexistent/a", "/nonexistent/b", "/tmp/out", "--field", "256").returncode == 2
    r = run("mul", "/nonexistent/a", "/nonexistent/b", "/tmp/out")
    assert r.returncode == 2 and "cannot open" in r.stderr


def _write_poly(path, words, bits):
    nbytes = (bits + 7) // 8
    data = words.view(np.uint8)[:nbytes].copy()
    if bits % 8:
        data[-1] &= (1 << (bits % 8)) - 1
    data.tofile(path)


@pytest.mark.gpu
@pytest.mark.parametrize("field", ["auto", "64", "128"])
def test_mul_files(tmp_path, port, checker, field):
    la, lb = 300001, 123457
    a = port.random_bitpoly(la, 11)
    b = port.random_bitpoly(lb, 12)
    a[-1] |= np.uint64(1) << np.uint64((la - 1) % 64)  # exact degrees
    b[-1] |= np.uint64(1) << np.uint64((lb - 1) % 64)
    _write_poly(tmp_path / "a.bin", a, la)
    _write_poly(tmp_path / "b.bin", b, lb)
    r = run("mul", str(tmp_path / "a.bin"), str(tmp_path / "b.bin"), str(tmp_path / "c.bin"), "--field", field)
    assert r.returncode == 0, r.stderr
    assert f"product bit length: {la + lb - 1}" in r.stdout
    want = checker.polymul(a, la, b, lb)
    got = np.fromfile(tmp_path / "c.bin", np.uint8)
    assert got.size == (la + lb - 1 + 7) // 8
    assert np.array_equal(got, want.view(np.uint8)[: got.size])


@pytest.mark.gpu
def test_selftest_and_fault_injection():
    r = run("selftest", "--seed", "7")
    assert r.returncode == 0, r.stdout + r.stderr
    assert "selftest passed" in r.stdout
    r = run("selftest", "--inject-encode-fault")
    assert r.returncode == 1
    assert "encode.gf128.encode/decode round-trip" in r.stderr


@pytest.mark.gpu
def test_bench_csv(tmp_path):
    csv = tmp_path / "b.csv"
    r = run("bench", "--min-log", "12", "--max-log", "14", "--reps", "3", "--csv", str(csv), "--field", "128")
    assert r.returncode == 0, r.stderr
    lines = csv.read_text().strip().splitlines()
    assert lines[0] == ("log2_size_words,n_bits,m,reps,mean_s,basiscvt_s,encode_s,butterfly_s,pointwise_s,"
                        "ibutterfly_s,decode_s,ibasiscvt_s")
    assert [int(x.split(",")[0]) for x in lines[1:]] == [12, 13, 14]
    assert all(int(x.split(",")[2]) == 128 for x in lines[1:])
