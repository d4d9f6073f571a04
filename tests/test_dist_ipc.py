"""The cross-process data plane of the sharded product: P separate processes on cuda:0, each
running the unmodified PeerBackend (paper_1803_11301_b200/dist.py) with a gloo process group for
control and REAL CUDA-IPC buffers for data (fpm_ipc_alloc/open/close/free; the exchanged layers read
the partner process's buffer inside fpm_bfly_pair_peer_dev).  Bit-exact against the oracle.  (Two
processes on one GPU cannot run NCCL, so NCCL itself is exercised only on multi-GPU boxes.)"""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("P,la,lb", [(2, 1 << 25, (1 << 25) - 777), (4, 1 << 26, 1 << 26), (2, 1 << 20, 1 << 19)])
def test_peer_backend_two_processes(gpu, checker, tmp_path, P, la, lb):
    a = gpu.random_bitpoly(la, 41)
    b = gpu.random_bitpoly(lb, 42)
    want = checker.polymul(a, la, b, lb)
    port = _free_port()
    outs = [str(tmp_path / f"r{r}.npy") for r in range(P)]
    procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "_ipc_rank.py"), str(r), str(P), str(port), str(la),
                               str(lb), "2", outs[r]], stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
             for r in range(P)]
    logs = []
    try:
        for p in procs:
            logs.append(p.communicate(timeout=600)[0])
    finally:
        for p in procs:
            if p.poll() is None:
                p.kill()
    for r, p in enumerate(procs):
        assert p.returncode == 0, f"rank {r} failed:\n{logs[r][-3000:]}"
    for r in range(P):
        assert np.array_equal(np.load(outs[r]), want), r


@pytest.mark.parametrize("P", [4])
def test_peer_backend_processes_config5_sharded_conversion(gpu, tmp_path, P):
    """BASELINE config 5 over P separate processes (gloo control, CUDA-IPC data): the sharded
    conversion -- every 2^32-bit block on P/2 processes phase by phase, regathered through the other
    processes' IPC replicas (fpm_b32_*), encode / decode at the column owners -- bit-exact against the
    reference's product hash on every rank."""
    import json
    with open(os.path.join(HERE, "golden", "reference_meta.json")) as f:
        c = json.load(f)["configs"]["4294967296x4294967296"]
    port = _free_port()
    outs = [str(tmp_path / f"r{r}.hash") for r in range(P)]
    procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "_ipc_rank.py"), str(r), str(P), str(port),
                               str(c["a_bits"]), str(c["b_bits"]), "1", outs[r], str(c["seed_a"]), str(c["seed_b"])],
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
             for r in range(P)]
    logs = []
    try:
        for p in procs:
            logs.append(p.communicate(timeout=900)[0])
    finally:
        for p in procs:
            if p.poll() is None:
                p.kill()
    for r, p in enumerate(procs):
        assert p.returncode == 0, f"rank {r} failed:\n{logs[r][-3000:]}"
    for r in range(P):
        with open(outs[r]) as f:
            assert f.read() == c["blake2b128"], r
