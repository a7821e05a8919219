"""World-size-2 gloo tests of the sharded DtN host logic (CPU): strided
shards keep global stream ids, so per-point results and the gathered boundary
data are bitwise identical to the single-process run (the multi-GPU analogue
of the reference's worker-count determinism test, tests/test_wos.cpp:118-133).
The per-rank compute here is the CPU oracle (test infrastructure)."""
from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]


def _compute(ids, w, n_paths):
    sys.path.insert(0, str(ROOT / "tests"))
    import oracle_lib as O
    from paper_1210_1491_b200 import nodes
    from paper_1210_1491_b200.wos import WosConfig

    orc = O.oracle()
    cfg = WosConfig(eps_shell=w.eps, n_paths=n_paths, seed=w.seed)
    out = []
    for b in ids:
        pos = nodes.patch_node_positions(w.points[b:b + 1], w.axes[b:b + 1], w.radii[b], None,
                                         w.dirs[int(w.cls[b])])[0]
        st, est, steps = O.or_estimate(orc, w.scene.to_c(), cfg.to_c(), pos,
                                       base=int(b) * w.n_nodes, workers=1)
        assert st == 0
        out.append([est["mean"].sum(), est["variance"].sum(), float(steps.sum())])
    return np.array(out).reshape(-1, 3)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sys.path.insert(0, str(ROOT))
    from paper_1210_1491_b200 import distributed as D
    from paper_1210_1491_b200 import workloads

    w = workloads.config1(24)
    ids = D.shard_ids(w.n_bp, rank, world)
    local = torch.from_numpy(_compute(ids, w, 64))
    full = D.allgather_strided(local, w.n_bp)
    if rank == 0:
        q.put(full.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_shards_cover_and_partition():
    from paper_1210_1491_b200 import distributed as D

    for n, world in [(10, 1), (10, 3), (7, 8), (100000, 8)]:
        ids = np.concatenate([D.shard_ids(n, r, world) for r in range(world)])
        assert np.array_equal(np.sort(ids), np.arange(n))
        assert sum(D.shard_counts(n, world)) == n


def test_gloo_world2_bitwise_equal_to_single_process():
    sys.path.insert(0, str(ROOT))
    from paper_1210_1491_b200 import workloads

    w = workloads.config1(24)
    single = _compute(np.arange(w.n_bp), w, 64)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p_ in procs:
        p_.start()
    full = q.get(timeout=300)
    for p_ in procs:
        p_.join(timeout=60)
        assert p_.exitcode == 0
    assert full.tobytes() == single.tobytes()


def _raise_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sys.path.insert(0, str(ROOT))
    from paper_1210_1491_b200 import distributed as D

    # rank 1's shard had a SolverError (soft status 10), rank 0's none: both
    # must raise before the next collective, and the all-gather after an OK
    # round must still complete on both
    D.raise_together(0)
    D.allgather_strided(torch.zeros((1, 1)), world)
    try:
        D.raise_together(10 if rank == 1 else 0)
        q.put((rank, "no raise"))
    except Exception as e:  # noqa: BLE001
        q.put((rank, type(e).__name__))
    dist.barrier()
    dist.destroy_process_group()


def test_soft_errors_raise_on_every_rank():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 30500 + os.getpid() % 1000
    procs = [ctx.Process(target=_raise_worker, args=(r, 2, port, q)) for r in range(2)]
    for p_ in procs:
        p_.start()
    got = dict(q.get(timeout=300) for _ in range(2))
    for p_ in procs:
        p_.join(timeout=60)
        assert p_.exitcode == 0
    assert got == {0: "SolverError", 1: "SolverError"}
