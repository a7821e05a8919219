"""Argument validation at the C boundary (advisor findings): walk counts the
device cannot count, patch classes outside the Gamma-rule table, and the
device-pointer DtN entry with node counts beyond its kernels — all rejected
with BW_ERR_INVALID (ValueError) before any kernel reads out of bounds."""
from __future__ import annotations

import numpy as np
import pytest
import torch

import paper_1210_1491_b200 as bw
from paper_1210_1491_b200 import dtn, workloads

pytestmark = pytest.mark.gpu


def test_n_paths_beyond_int32_rejected(gpu):
    s = bw.Scene.sphere(1.0, bw.DomainSide.Interior, 1.0)
    with pytest.raises(ValueError):
        bw.estimate_u_batch(s, [[0, 0, 0.1]], bw.WosConfig(n_paths=2**31))
    with pytest.raises(ValueError):
        bw.estimate_u_batch(s, [[0, 0, 0.1]], bw.WosConfig(n_paths=10, rng=7))


def test_statistical_mode_shell_floor(gpu):
    """BW_RNG_PHILOX4X32 resolves distances to ~3e-12 of the boundary's size:
    a shell below 1e-9 of it is refused (the parity mode takes any shell)."""
    s = bw.Scene.sphere(2.0, bw.DomainSide.Interior, 1.0)
    with pytest.raises(ValueError):
        bw.estimate_u_batch(s, [[0, 0, 0.1]], bw.WosConfig(n_paths=8, eps_shell=1e-9, rng=1))
    bw.estimate_u_batch(s, [[0, 0, 0.1]], bw.WosConfig(n_paths=8, eps_shell=4e-9, rng=1))
    bw.estimate_u_batch(s, [[0, 0, 0.1]], bw.WosConfig(n_paths=8, eps_shell=1e-11, rng=0))


def test_bad_class_rejected_host_and_device(gpu):
    w = workloads.config4(2000).subset(np.arange(4))
    P = dtn.patches_for(w)
    P["cls"][2] = 5  # one class only
    cfg = w.wos_config(n_paths=32)
    with pytest.raises(ValueError):
        dtn.dtn_solve(w.scene, cfg, P, w.dirs, w.weights)
    dev = torch.device("cuda", 0)
    d_p = torch.from_numpy(P.view(np.uint8).copy()).to(dev)
    d_dirs = torch.from_numpy(w.dirs).to(dev)
    d_w = torch.from_numpy(np.ascontiguousarray(w.weights)).to(dev)
    out = [torch.empty(4, dtype=t, device=dev) for t in (torch.float64, torch.float64, torch.int32)]
    with pytest.raises(ValueError):
        dtn.dtn_solve_device(w.scene, cfg, dtn.DtnConfig(), d_p.data_ptr(), None, 4,
                             d_dirs.data_ptr(), d_w.data_ptr(), 1, w.n_nodes,
                             *(o.data_ptr() for o in out), device=0)
    # the same arrays with a valid class run
    P["cls"][2] = 0
    d_p = torch.from_numpy(P.view(np.uint8).copy()).to(dev)
    dtn.dtn_solve_device(w.scene, cfg, dtn.DtnConfig(), d_p.data_ptr(), None, 4,
                         d_dirs.data_ptr(), d_w.data_ptr(), 1, w.n_nodes,
                         *(o.data_ptr() for o in out), device=0)
    torch.cuda.synchronize()
    assert torch.isfinite(out[0]).all()
