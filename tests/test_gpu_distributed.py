"""torchrun-style multi-process path on the GPU: two ranks (gloo for the
plumbing, both on the box's one GPU — their kernels never wait on each other)
run pipeline.run on their strided shards through the CUDA path, and rank 0's
gathered potentials and the per-rank Neumann data are bitwise those of one
process (the gloo CPU tests in test_distributed.py cover the host logic)."""
from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]
pytestmark = pytest.mark.gpu


def _problem():
    sys.path.insert(0, str(ROOT))
    from paper_1210_1491_b200 import workloads

    w = workloads.config5(1500)
    t = workloads.make_targets(w, 2000, seed=5)
    return w, t


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist

    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    sys.path.insert(0, str(ROOT))
    from paper_1210_1491_b200 import pipeline

    w, t = _problem()
    u, near, res, panels = pipeline.run(w, t, device=0, n_paths=256)
    q.put((rank, res.dudn, u, near))
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_bitwise_equal_to_one(gpu):
    from paper_1210_1491_b200 import pipeline

    w, t = _problem()
    u1, near1, res1, _ = pipeline.run(w, t, device=0, n_paths=256)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 31500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p_ in procs:
        p_.start()
    got = {}
    for _ in range(2):
        r, dudn, u, near = q.get(timeout=600)
        got[r] = (dudn, u, near)
    for p_ in procs:
        p_.join(timeout=120)
        assert p_.exitcode == 0
    dudn = np.empty(w.n_bp)
    dudn[0::2], dudn[1::2] = got[0][0], got[1][0]
    assert dudn.tobytes() == res1.dudn.tobytes()
    assert got[0][1].tobytes() == u1.tobytes() and (got[0][2] == near1).all()
