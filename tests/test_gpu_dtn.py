"""GPU parity of the DtN path (K1 -> K4 -> K2 -> K5) against the CPU oracle
(oracle/biewos_patch.c, itself bit-identical to the reference's assemble, see
tests/test_patch_oracle.py) given identical Gamma node values, and accuracy
against the analytic Neumann data."""
from __future__ import annotations

import numpy as np
import pytest

import oracle_lib as O
from paper_1210_1491_b200 import dtn, nodes, workloads

pytestmark = pytest.mark.gpu


def _oracle_dudn(orc, w, res, idx):
    sc = w.scene.to_c()
    P = dtn.patches_for(w)
    out = []
    for b in idx:
        cls = int(w.cls[b])
        gy = O.or_patch_nodes(orc, w.points[b:b + 1], w.axes[b:b + 1], w.radii[b], None,
                              w.dirs[cls])[0]
        e = res.node_est[b]
        ok = e["n"] > 0
        gw = np.where(ok, w.weights[cls] * w.radii[b] ** 2, 0.0)
        gu = np.where(ok, e["mean"], 0.0)
        guv = np.where(ok, e["variance"] / np.maximum(e["n"], 1), 0.0)
        d, err, st = O.or_patch_point(orc, sc, P[b], gy, gw, gu, guv)
        out.append((-d, err, st))
    return np.array(out)


@pytest.mark.parametrize("cfg", [1, 4, 3])
def test_dtn_matches_oracle_given_node_values(gpu, orc, cfg):
    if cfg == 1:
        w = workloads.config1().subset(np.array([0, 137, 500, 999]))
    elif cfg == 4:
        w = workloads.config4(20000).subset(np.array([3, 7000, 15000]))
    else:
        full = workloads.config3()
        face = np.where(full.cls == 0)[0]
        cav = np.where(full.cls > 0)[0]
        w = full.subset(np.concatenate([face[[100, 4000]], cav[[0, 500, 1500]]]))
    res = dtn.dtn_solve_workload(w, n_paths=256, return_nodes=True)
    ref = _oracle_dudn(orc, w, res, range(w.n_bp))
    assert (ref[:, 2] == 0).all() and (res.status == 0).all()
    scale = np.abs(ref[:, 0]) + 1e-3 * np.abs(ref[:, 0]).max()
    assert (np.abs(res.dudn - ref[:, 0]) / scale).max() < 1e-10
    assert np.allclose(res.err, ref[:, 1], rtol=1e-8)


def test_dtn_unit_ball_accuracy(gpu):
    """cfg1 data (u = x^2 - y^2 + z on the unit ball): Neumann data within the
    propagated WOS error plus the m = 54 discretisation bias (<0.5%)."""
    w = workloads.config1().subset(np.arange(0, 1000, 50))
    res = dtn.dtn_solve_workload(w, n_paths=10000)
    exact = w.exact_dudn_outward()
    gscale = np.abs(w.exact_grad(w.points)).max(axis=1)
    dev = np.abs(res.dudn - exact)
    assert (dev < 5 * res.err + 5e-3 * gscale).all(), np.max(dev / (res.err + 1e-3))
    assert (res.status == 0).all()


def test_dtn_cube_edges(gpu):
    """cfg2: hemispheres shrink near edges/corners so no patch is clipped
    (workloads.edge_clear_radii); a full-size corner patch is flagged."""
    w = workloads.config2()
    idx = np.array([0, 32 * 16 + 16])  # a corner cell and a face-centre cell of face x=0
    sub = w.subset(idx)
    assert sub.radii[0] < 0.016 and sub.radii[1] == 0.05
    res = dtn.dtn_solve_workload(sub, n_paths=256)
    assert (res.status == 0).all()
    sub.radii[:] = 0.05  # the unshrunk corner hemisphere pokes out of the cube
    res = dtn.dtn_solve_workload(sub, n_paths=256)
    assert res.status[0] & 1 and not res.status[1] & 1


def test_dtn_cube_accuracy(gpu):
    w = workloads.config2()
    idx = np.arange(0, w.n_bp, 97)
    sub = w.subset(idx)
    res = dtn.dtn_solve_workload(sub, n_paths=4096)
    exact = sub.exact_dudn_outward()
    gscale = np.abs(sub.exact_grad(sub.points)).max(axis=1) + 1.0
    assert (res.status == 0).all()
    assert (np.abs(res.dudn - exact) < 6 * res.err + 1e-2 * gscale).mean() > 0.98


def _mixed_cfg3(n_face=6, n_cav=6, n_edge=3):
    """cfg3 points: face interiors (one canonical class), cavities (several
    classes) and edge-shrunk face patches (singleton classes)."""
    full = workloads.config3()
    face = np.where((full.cls == 0) & (full.radii == full.a))[0]
    edge = np.where((full.cls == 0) & (full.radii < full.a))[0]
    cav = np.where(full.cls > 0)[0]
    rng = np.random.default_rng(7)
    idx = np.concatenate([rng.choice(face, n_face, replace=False),
                          rng.choice(cav, n_cav, replace=False),
                          rng.choice(edge, n_edge, replace=False)])
    return full.subset(idx)


def _nodes(w, n_paths=256):
    return dtn.dtn_solve_workload(w, n_paths=n_paths, return_nodes=True)


@pytest.mark.parametrize("which", ["cfg4", "cfg3", "cfg2"])
def test_class_tables_match_per_patch(gpu, orc, which):
    """K7 (congruence-class tables) and K4 -> K2 -> K5 on identical node
    estimates agree with the CPU oracle (scaled as in the oracle test above)
    and with each other; same propagated error and status. Gate 2e-10: on
    the cfg3 mix both device paths sit ~1e-10 from the oracle on cavity points
    whose Neumann value is small against the data scale (the oracle's own
    sequential double sums; K7 sums compensated, K4 in panel order)."""
    if which == "cfg4":
        w = workloads.config4(20000).subset(np.array([0, 3, 7000, 15000, 19999]))
    elif which == "cfg3":
        w = _mixed_cfg3()
    else:
        w = workloads.config2().subset(np.array([0, 17, 32 * 16 + 16, 3000, 6143]))
    res = _nodes(w)
    P = dtn.patches_for(w)
    a = dtn.dtn_neumann(w.scene, P, w.dirs, w.weights, res.node_est, method=dtn.DTN_CLASSES)
    b = dtn.dtn_neumann(w.scene, P, w.dirs, w.weights, res.node_est, method=dtn.DTN_PER_PATCH)
    assert np.array_equal(a.dudn, res.dudn) and np.array_equal(a.err, res.err)
    ref = _oracle_dudn(orc, w, res, range(w.n_bp))
    # du/dn = sum_g c_g u_g with c_g ~ 1/a_b: on an edge-shrunk patch the
    # terms grow like a / a_b against a result of the data's scale, and so does
    # the rounding of any summation order (K7 compensated, K4 and the oracle in
    # panel order)
    scale = (np.abs(ref[:, 0]) + 1e-3 * np.abs(ref[:, 0]).max()) * np.maximum(1.0, w.a / w.radii)
    assert (np.abs(a.dudn - ref[:, 0]) / scale).max() < 2e-10
    assert (np.abs(b.dudn - ref[:, 0]) / scale).max() < 2e-10
    assert (np.abs(a.dudn - b.dudn) / scale).max() < 2e-10
    # the north star's 1e-10 relative gate, norm-wise over the batch
    nref = np.abs(ref[:, 0]).max()
    assert np.abs(a.dudn - ref[:, 0]).max() / nref < 1e-10
    assert np.abs(b.dudn - ref[:, 0]).max() / nref < 1e-10
    assert np.allclose(a.err, b.err, rtol=1e-9)
    assert np.allclose(a.err, ref[:, 1], rtol=1e-8)
    assert np.array_equal(a.status, b.status)


def _both(w, P, est):
    a = dtn.dtn_neumann(w.scene, P, w.dirs, w.weights, est, method=dtn.DTN_CLASSES)
    b = dtn.dtn_neumann(w.scene, P, w.dirs, w.weights, est, method=dtn.DTN_PER_PATCH)
    assert np.array_equal(a.status, b.status)
    scale = np.abs(b.dudn) + 1e-3 * np.abs(b.dudn).max()
    assert (np.abs(a.dudn - b.dudn) / scale).max() < 2e-10
    assert np.allclose(a.err, b.err, rtol=1e-9)
    return a


def test_class_tables_invalid_nodes(gpu):
    """Patches whose Gamma nodes leave the domain (status bit 0): the nodes drop
    out of b exactly as in K4 (their Kg columns are removed)."""
    w = workloads.config2().subset(np.array([0, 5, 32 * 16 + 16]))
    w.radii[:] = 0.05  # corner hemispheres poke out of the cube
    res = _nodes(w)
    a = _both(w, dtn.patches_for(w), res.node_est)
    assert a.status[0] & 1 and not a.status[2] & 1


def test_class_tables_self_classes(gpu):
    """A sphere patch whose axis is not radial is no rigid image of the
    canonical patch: it becomes its own class (exemplar = itself)."""
    w = workloads.config4(20000).subset(np.array([3, 7000, 15000]))
    res = _nodes(w)
    P = dtn.patches_for(w)
    P["axis"][1] = P["axis"][1] + np.array([2e-3, -1e-3, 1e-3])
    P["axis"][1] /= np.linalg.norm(P["axis"][1])
    _both(w, P, res.node_est)


def test_class_tables_batch_independent(gpu):
    """A point's result does not depend on which other points share the call
    (class tables are built from the class key alone): bitwise, so sharded
    runs agree with one-GPU runs."""
    w = _mixed_cfg3()
    res = _nodes(w)
    P = dtn.patches_for(w)
    full = dtn.dtn_neumann(w.scene, P, w.dirs, w.weights, res.node_est)
    for sel in (np.array([0, 7, 14]), np.arange(1, w.n_bp, 2), np.array([5])):
        part = dtn.dtn_neumann(w.scene, P[sel], w.dirs, w.weights, res.node_est[sel])
        assert np.array_equal(part.dudn, full.dudn[sel])
        assert np.array_equal(part.err, full.err[sel])


def _hits(gpu):
    import ctypes as C

    h = C.c_uint64(0)
    gpu.check(gpu.lib.bw_dtn_class_cache_hits(gpu.handle, C.byref(h)))
    return h.value


def test_class_tables_reused_across_calls(gpu):
    """The library keeps the congruence classes (and, single chunk, their
    tables) of the last patch set: a repeated Neumann stage on the same
    patches hits the cache and returns bitwise the same data — also with new
    node estimates and other Dirichlet data, which the tables do not depend
    on; a changed patch, another mesh or another rule miss it and rebuild."""
    w = _mixed_cfg3()
    res = _nodes(w)
    P = dtn.patches_for(w)
    first = dtn.dtn_neumann(w.scene, P, w.dirs, w.weights, res.node_est)
    h0 = _hits(gpu)
    again = dtn.dtn_neumann(w.scene, P, w.dirs, w.weights, res.node_est)
    assert _hits(gpu) == h0 + 1
    assert np.array_equal(first.dudn, again.dudn) and np.array_equal(first.err, again.err)
    assert np.array_equal(first.status, again.status)
    # new estimates on the same geometry: a hit, and equal to a cold build
    est2 = res.node_est.copy()
    est2["mean"] *= 1.25
    warm = dtn.dtn_neumann(w.scene, P, w.dirs, w.weights, est2)
    assert _hits(gpu) == h0 + 2
    P2 = P.copy()
    P2["a"][3] *= 0.5  # one patch changes: a miss
    other = dtn.dtn_neumann(w.scene, P2, w.dirs, w.weights, est2)
    assert _hits(gpu) == h0 + 2
    assert not np.array_equal(other.dudn, warm.dudn)
    cold = dtn.dtn_neumann(w.scene, P, w.dirs, w.weights, est2)  # rebuilt from scratch
    assert _hits(gpu) == h0 + 2
    assert np.array_equal(cold.dudn, warm.dudn) and np.array_equal(cold.err, warm.err)
    # the per-patch path never touches the cache
    dtn.dtn_neumann(w.scene, P, w.dirs, w.weights, est2, method=dtn.DTN_PER_PATCH)
    assert _hits(gpu) == h0 + 2
