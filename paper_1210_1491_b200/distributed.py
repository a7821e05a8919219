"""Multi-GPU plumbing of the DtN path (one process per GPU, torch.distributed).

Boundary points are independent, so the
walks, the collocation and the solves shard with no communication: rank r
owns the global points r, r + N, r + 2N, ... (strided, so cavity and face
points, whose walks cost differently, spread evenly) and keeps their GLOBAL
ids in its Philox streams — every point's result is bitwise the same for any
N. The only exchange is one all-gather of the per-point boundary records
(the panels of the integral representation, 9 doubles each) before the
potential evaluation, whose targets shard the same way. NCCL on GPUs, gloo in
the CPU tests.
"""
from __future__ import annotations

import numpy as np


def shard_ids(n: int, rank: int, world: int) -> np.ndarray:
    """Global indices owned by `rank` (strided)."""
    return np.arange(rank, n, world, dtype=np.int64)


def shard_counts(n: int, world: int) -> list[int]:
    return [len(range(r, n, world)) for r in range(world)]


def allgather_strided(local, n_total: int, group=None):
    """Inverse of shard_ids: gather every rank's rows (local: torch tensor
    (n_local, ...) of the rows it owns, in shard order) into the full
    (n_total, ...) array in global order, on every rank. One all_gather of
    equal-size padded blocks (NCCL all_gather_into_tensor on GPUs)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world == 1:
        return local.clone()
    counts = shard_counts(n_total, world)
    width = max(counts)
    pad = torch.zeros((width,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    out = torch.empty((world * width,) + tuple(local.shape[1:]), dtype=local.dtype,
                      device=local.device)
    if (hasattr(dist, "all_gather_into_tensor") and local.device.type == "cuda"
            and dist.get_backend(group) == "nccl"):
        dist.all_gather_into_tensor(out, pad, group=group)
    elif local.device.type == "cuda":  # gloo (tests): through host memory
        parts = [torch.empty_like(pad, device="cpu") for _ in range(world)]
        dist.all_gather(parts, pad.cpu(), group=group)
        out.copy_(torch.cat(parts))
    else:
        dist.all_gather(list(out.chunk(world)), pad, group=group)
    full = torch.empty((n_total,) + tuple(local.shape[1:]), dtype=local.dtype,
                       device=local.device)
    for r in range(world):
        full[r::world] = out[r * width: r * width + counts[r]]
    return full


def raise_together(status: int, device=None, group=None) -> None:
    """Every rank raises if any rank's soft status (bw_status from a sharded
    call with soft=True) is non-zero: one all-reduce (MAX) of the code before
    the caller's next collective, so no rank is left waiting in it."""
    import torch
    import torch.distributed as dist

    from .errors import STATUS_TO_EXC, Error

    worst = int(status)
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        t = torch.tensor([worst], dtype=torch.int64,
                         device=torch.device("cuda", device) if device is not None
                         and dist.get_backend(group) == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
        worst = int(t.item())
    if worst:
        raise STATUS_TO_EXC.get(worst, Error)(
            f"status {worst} on {'this or another rank' if worst != status else 'this rank'} "
            "(per-point detail in the DtN status array)")


def boundary_panels(points, axes, areas, u, dudn_axis) -> np.ndarray:
    """Integral-representation panels (field_eval.hpp:12-22): normals point INTO
    the region where u is evaluated (the solution domain = the patch axis),
    dudn along that normal."""
    P = np.empty((len(points), 9))
    P[:, 0:3] = points
    P[:, 3:6] = axes
    P[:, 6] = areas
    P[:, 7] = u
    P[:, 8] = dudn_axis
    return P
