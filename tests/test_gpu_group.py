"""Several devices inside the library (bw_group_*): sharded DtN and the config-5
pipeline with an NCCL all-gather. On the one-GPU box: n = 1 runs NCCL as a
single-rank communicator; n = 2, 3 with the device id repeated run the same
sharding with device-to-device copies in place of NCCL. Every result must be
bitwise the single-device one (wos.hpp:43-44 across devices)."""
from __future__ import annotations

import numpy as np
import pytest

import oracle_lib as O
from paper_1210_1491_b200 import DeviceGroup, dtn, pipeline, workloads

pytestmark = pytest.mark.gpu


def _mixed_cfg3(n=90):
    full = workloads.config3()
    idx = np.unique(np.linspace(0, full.n_bp - 1, n).astype(np.int64))
    return full.subset(idx)


@pytest.mark.parametrize("devices", [[0], [0, 0], [0, 0, 0]])
def test_group_dtn_bitwise_equals_single_device(gpu, devices):
    w = _mixed_cfg3()
    cfg = w.wos_config(n_paths=256)
    ref = dtn.dtn_solve(w.scene, cfg, dtn.patches_for(w), w.dirs, w.weights)
    g = DeviceGroup(devices)
    assert g.size == len(devices) and g.uses_nccl == (len(devices) == 1)
    res, steps, ms = g.dtn_solve(w.scene, cfg, dtn.patches_for(w), w.dirs, w.weights)
    assert res.dudn.tobytes() == ref.dudn.tobytes()
    assert res.err.tobytes() == ref.err.tobytes()
    assert (res.status == ref.status).all()
    assert steps > 0 and ms > 0
    # global ids: a permuted batch with its bp_ids gives each point's same bits
    perm = np.random.default_rng(3).permutation(w.n_bp)
    res2, steps2, _ = g.dtn_solve(w.scene, cfg, dtn.patches_for(w)[perm], w.dirs, w.weights,
                                  bp_ids=perm)
    assert res2.dudn.tobytes() == ref.dudn[perm].tobytes() and steps2 == steps
    g.close()


def test_group_pipeline_bitwise_across_devices_and_matches_oracle(gpu, orc):
    w = workloads.config5(2000)
    t = workloads.make_targets(w, 3000, seed=5)
    area = pipeline.panel_areas(w)
    u_bp = np.asarray(w.scene.phi(w.points), np.float64)
    cfg = w.wos_config(n_paths=512)
    out = []
    for devices in ([0], [0, 0, 0]):
        g = DeviceGroup(devices)
        out.append(g.pipeline(w.scene, cfg, dtn.patches_for(w), w.dirs, w.weights, area, u_bp, t))
        g.close()
    a, b = out
    assert a.u.tobytes() == b.u.tobytes() and (a.near == b.near).all()
    assert a.dtn.dudn.tobytes() == b.dtn.dudn.tobytes() and a.walk_steps == b.walk_steps
    assert set(a.phase_ms) == {"dtn", "exchange", "potential"}
    # the same Neumann data as the single-device DtN, and the potential of the
    # panels it implies equals the long-double oracle sum to 1e-10
    ref = dtn.dtn_solve(w.scene, cfg, dtn.patches_for(w), w.dirs, w.weights)
    assert a.dtn.dudn.tobytes() == ref.dudn.tobytes()
    panels = np.concatenate([w.points, w.axes, area[:, None], u_bp[:, None],
                             -a.dtn.dudn[:, None]], axis=1)
    u_ref, near_ref = O.or_potential(orc, panels, t, long_double=True)
    assert (a.near == near_ref).all()
    ok = ~a.near
    assert (np.abs(a.u[ok] - u_ref[ok]) / (np.abs(u_ref[ok]) + 1e-3)).max() < 1e-10
    assert np.isnan(a.u[a.near]).all()


def test_group_soft_errors_do_not_hang(gpu):
    """A ReliabilityError on one shard (max_steps = 1: every walk fails) is
    reported by the group with all outputs written; nothing hangs."""
    w = workloads.config4(20000).subset(np.arange(8))
    cfg = w.wos_config(n_paths=64)
    cfg.max_steps = 1
    g = DeviceGroup([0, 0])
    with pytest.raises(Exception) as ei:
        g.dtn_solve(w.scene, cfg, dtn.patches_for(w), w.dirs, w.weights)
    assert type(ei.value).__name__ == "ReliabilityError"
    assert len(ei.value.result.dudn) == w.n_bp
    g.close()


def test_k3_on_cfg5_panel_set_matches_long_double_oracle(gpu, orc):
    """K3 on config 5's own 2e5-panel set (exact du/dn) at 2,000 targets drawn
    like the benchmark's, near-field flags included: <= 1e-10 relative to the
    compensated long-double oracle sum."""
    from paper_1210_1491_b200 import field_eval

    w = workloads.config5()
    area = pipeline.panel_areas(w)
    dudn_in = (w.exact_grad(w.points) * w.axes).sum(axis=1)
    panels = np.concatenate([w.points, w.axes, area[:, None],
                             np.asarray(w.scene.phi(w.points))[:, None], dudn_in[:, None]], axis=1)
    t = workloads.make_targets(w, 1000000, seed=5)
    t = t[np.linspace(0, len(t) - 1, 2000).astype(np.int64)]
    # a few targets right at the boundary to exercise the near-field flag
    t = np.concatenate([t, w.points[:5] + 1e-4 * w.axes[:5]])
    u, near = field_eval.evaluate_batch(panels, t)
    u_ref, near_ref = O.or_potential(orc, panels, t, long_double=True)
    assert (near == near_ref).all() and near[-5:].all()
    ok = ~near
    assert (np.abs(u[ok] - u_ref[ok]) / np.abs(u_ref[ok])).max() < 1e-10
