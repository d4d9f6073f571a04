"""One rank of tests/test_dist_ipc.py: a separate PROCESS on cuda:0 running the unmodified
PeerBackend (paper_1803_11301_b200/dist.py) -- gloo process group for control, real CUDA-IPC buffers
(fpm_ipc_alloc / fpm_ipc_open / fpm_ipc_close / fpm_ipc_free) for the exchanged butterfly layers."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    rank, P, port, la, lb, products, out = (int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]),
                                            int(sys.argv[5]), int(sys.argv[6]), sys.argv[7])
    seed_a, seed_b = (int(sys.argv[8]), int(sys.argv[9])) if len(sys.argv) > 9 else (41, 42)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=P)
    import paper_1803_11301_b200 as pkg
    from paper_1803_11301_b200.dist import PeerBackend, make_plan, polymul_sharded

    a = pkg.random_bitpoly(la, seed_a)
    b = pkg.random_bitpoly(lb, seed_b)
    da = torch.from_numpy(a.view(np.int64).copy()).cuda()
    db = torch.from_numpy(b.view(np.int64).copy()).cuda()
    be = PeerBackend()
    plan = make_plan(la, lb, P, rank)
    for _ in range(products):  # the ping-pong IPC buffers are reused across products
        res = polymul_sharded(da, la, db, lb, be, plan)
    torch.cuda.synchronize()
    if out.endswith(".hash"):  # large products: the blake2b-128 of the product words
        import hashlib
        with open(out, "w") as f:
            f.write(hashlib.blake2b(res.cpu().numpy().view(np.uint64).tobytes(), digest_size=16).hexdigest())
    else:
        np.save(out, res.cpu().numpy().view(np.uint64))
    be.close()  # collective release of the peer mappings and buffers
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
