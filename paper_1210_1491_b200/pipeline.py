"""The full BASELINE config-5 pipeline on one or many GPUs (one process each):

  K1 WOS over all Gamma nodes -> K4 collocation -> K2 batched LU -> K5 point
  values (each rank: its strided shard of boundary points, no communication)
  -> all-gather of the boundary panels (NCCL; 72 B per point)
  -> K3 potential sum at this rank's shard of the targets -> gather to rank 0.

Boundary panels for the integral representation (field_eval.hpp:12-22): one
per boundary point, area = (area of its surface piece) / (points on it),
normal INTO the solution domain, u = Dirichlet data, dudn along that normal.
"""
from __future__ import annotations

import numpy as np

from . import dtn
from .distributed import allgather_strided, raise_together, shard_ids
from .geometry import SceneKind


def panel_areas(w) -> np.ndarray:
    """Surface area represented by each boundary point."""
    area = np.empty(w.n_bp)
    if w.scene.kind == SceneKind.Sphere:
        area[:] = 4.0 * np.pi * w.scene.sphere_radius ** 2 / w.n_bp
    elif w.scene.kind == SceneKind.Box:
        lo, hi = np.array(w.scene.box_lo), np.array(w.scene.box_hi)
        for f in range(6):
            ax = f // 2
            on = np.isclose(w.points[:, ax], hi[ax] if f & 1 else lo[ax]) & \
                np.isclose(np.abs(w.axes[:, ax]), 1.0)
            others = [k for k in range(3) if k != ax]
            area[on] = np.prod(hi[others] - lo[others]) / max(on.sum(), 1)
    else:
        cav = w.extra["cavities"]
        lo, hi = np.array(w.scene.box_lo), np.array(w.scene.box_hi)
        face = w.cls == 0
        for f in range(6):
            ax = f // 2
            on = face & np.isclose(w.points[:, ax], hi[ax] if f & 1 else lo[ax]) & \
                np.isclose(np.abs(w.axes[:, ax]), 1.0)
            others = [k for k in range(3) if k != ax]
            area[on] = np.prod(hi[others] - lo[others]) / max(on.sum(), 1)
        for i, c in enumerate(cav):
            on = w.cls == 1 + i
            if on.any():
                area[on] = 4.0 * np.pi * c[3] ** 2 / on.sum()
    return area


def run(w, targets: np.ndarray, device: int = 0, n_paths: int | None = None,
        dtn_cfg=None, timer=None, rng: int = 0):
    """Run the pipeline on this rank. Returns (u at all targets on rank 0 or
    None, near flags, per-rank DtN result). `timer(name)` is called at phase
    boundaries if given (CUDA-event timing by the caller)."""
    import torch
    import torch.distributed as dist

    from . import _native as N
    from .field_eval import evaluate_device

    rank = dist.get_rank() if dist.is_initialized() else 0
    world = dist.get_world_size() if dist.is_initialized() else 1
    dev = torch.device("cuda", device)
    ctx = N.context(device)
    stream = torch.cuda.current_stream(dev)
    ctx.set_stream(stream.cuda_stream)
    dcfg = dtn_cfg or dtn.DtnConfig()
    cfg = w.wos_config(n_paths, rng)

    ids = shard_ids(w.n_bp, rank, world)
    n_loc = len(ids)
    patches = dtn.patches_for(w)[ids]
    d_patches = torch.from_numpy(patches.view(np.uint8).copy()).to(dev)
    d_ids = torch.from_numpy(ids).to(dev)
    d_dirs = torch.from_numpy(w.dirs).to(dev)
    d_wts = torch.from_numpy(np.ascontiguousarray(w.weights)).to(dev)
    d_dudn = torch.empty(n_loc, dtype=torch.float64, device=dev)
    d_err = torch.empty(n_loc, dtype=torch.float64, device=dev)
    d_status = torch.empty(n_loc, dtype=torch.int32, device=dev)
    d_steps = torch.empty(n_loc * w.n_nodes, dtype=torch.int64, device=dev)
    if timer:
        timer("start")
    rc = dtn.dtn_solve_device(w.scene, cfg, dcfg, d_patches.data_ptr(), d_ids.data_ptr(), n_loc,
                              d_dirs.data_ptr(), d_wts.data_ptr(), w.dirs.shape[0], w.n_nodes,
                              d_dudn.data_ptr(), d_err.data_ptr(), d_status.data_ptr(), None,
                              d_steps.data_ptr(), device=device, soft=True)
    raise_together(rc, device)  # before the all-gather: all ranks raise, or none
    if timer:
        timer("dtn")
    # local panels: point, normal into the domain, area, u, dudn along that normal
    area = panel_areas(w)[ids]
    u_bp = w.scene.phi(w.points[ids])
    loc = torch.empty((n_loc, 9), dtype=torch.float64, device=dev)
    loc[:, 0:3] = torch.from_numpy(w.points[ids]).to(dev)
    loc[:, 3:6] = torch.from_numpy(w.axes[ids]).to(dev)
    loc[:, 6] = torch.from_numpy(area).to(dev)
    loc[:, 7] = torch.from_numpy(np.asarray(u_bp, np.float64)).to(dev)
    loc[:, 8] = -d_dudn  # outward -> along the into-domain normal
    panels = allgather_strided(loc, w.n_bp)
    if timer:
        timer("allgather")
    t_ids = shard_ids(len(targets), rank, world)
    d_t = torch.from_numpy(np.ascontiguousarray(targets[t_ids])).to(dev)
    d_u = torch.empty(len(t_ids), dtype=torch.float64, device=dev)
    d_near = torch.empty(len(t_ids), dtype=torch.uint8, device=dev)
    evaluate_device(panels.data_ptr(), w.n_bp, d_t.data_ptr(), len(t_ids), d_u.data_ptr(),
                    d_near.data_ptr(), device=device)
    if timer:
        timer("potential")
    u_all = allgather_strided(d_u[:, None], len(targets))[:, 0]
    near_all = allgather_strided(d_near[:, None].to(torch.float64), len(targets))[:, 0] > 0
    if timer:
        timer("gather")
    res = dtn.DtnResult(d_dudn.cpu().numpy(), d_err.cpu().numpy(), d_status.cpu().numpy())
    res.steps = int(d_steps.sum().item())
    if rank == 0:
        return u_all.cpu().numpy(), near_all.cpu().numpy(), res, panels.cpu().numpy()
    return None, None, res, None
