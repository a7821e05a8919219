"""Local Dirichlet-to-Neumann map on the B200: the whole-boundary driver.

For every boundary point: K1 estimates u at the Gamma nodes of its hemisphere
(WOS); the local BIE of its patch (the reference's `assemble`,
patch_solver.cpp:197-309, second kind by default) is solved (PartialPivLU,
patch_solver.cpp:314-324) and the Neumann value read off the fan panels around
the point. By default this goes through congruence-class tables (K7: A, its LU
and the kernel values once per class of rigidly congruent patches, a
compensated dot product with the data per point); `dtn_neumann(...,
method=DTN_PER_PATCH)` runs the per-patch structure instead (K4 assembly, K2
batched LU, K5 point value). The reference has no whole-boundary driver (it
solves one patch per call, patch_solver.cpp:331-335); this is the additive
batch API.

Conventions: a patch's axis points INTO the solution domain;
`dudn` is returned along the domain-OUTWARD normal (-axis).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N

PATCH_DTYPE = np.dtype([("o", "<f8", 3), ("axis", "<f8", 3), ("sc", "<f8", 3), ("a", "<f8"),
                        ("R", "<f8"), ("surf", "<i4"), ("cls", "<i4")])


class BwDtnConfig(C.Structure):
    _fields_ = [("bands", C.c_int32), ("azimuth", C.c_int32), ("gauss_polar", C.c_int32),
                ("near_depth", C.c_int32), ("solve_tol", C.c_double), ("kind", C.c_int32),
                ("reserved", C.c_int32)]


BIE_SECOND, BIE_FIRST = 0, 1  # patch_solver.hpp:61 BieKind (second kind is the default)


@dataclass
class DtnConfig:
    bands: int = 5        # m = azimuth (2 bands - 1) = 54 panels
    azimuth: int = 6
    gauss_polar: int = 20  # patch_solver.hpp:34
    near_depth: int = 2    # patch_solver.hpp:35
    solve_tol: float = 1e-10  # patch_solver.cpp:319
    kind: int = BIE_SECOND    # BIE_FIRST: A = int G, b with dG/dn_y (patch_solver.cpp:285-305)

    @property
    def m(self) -> int:
        return self.azimuth * (2 * self.bands - 1)

    def to_c(self) -> BwDtnConfig:
        return BwDtnConfig(self.bands, self.azimuth, self.gauss_polar, self.near_depth,
                           self.solve_tol, int(self.kind), 0)


def patches_for(w) -> np.ndarray:
    """bw_patch records of a workloads.Workload: the local surface of each
    boundary point is the unit sphere (cfg1/4), the face plane (cfg2, box faces)
    or its cavity sphere (cfg3/5)."""
    from .geometry import SceneKind

    p = np.zeros(w.n_bp, PATCH_DTYPE)
    p["o"] = w.points
    p["axis"] = w.axes
    p["a"] = w.radii
    p["cls"] = w.cls
    if w.scene.kind == SceneKind.Sphere:
        p["surf"] = 0
        p["R"] = w.scene.sphere_radius
    elif w.scene.kind == SceneKind.Box:
        p["surf"] = 1
    else:
        cav = w.extra["cavities"]
        on_cav = w.cls > 0
        p["surf"] = np.where(on_cav, 0, 1)
        ci = np.maximum(w.cls - 1, 0)
        p["sc"] = np.where(on_cav[:, None], cav[ci, :3], 0.0)
        p["R"] = np.where(on_cav, cav[ci, 3], 0.0)
    return p


@dataclass
class DtnResult:
    dudn: np.ndarray     # along the domain-outward normal
    err: np.ndarray      # propagated WOS error (est_error average)
    status: np.ndarray   # bit0 clipped patch, bit1 solver failure
    node_est: np.ndarray | None = None
    steps: np.ndarray | None = None


def dtn_solve(scene, wos_cfg, patches: np.ndarray, local_dirs, weights, dtn_cfg=None,
              bp_ids=None, point_id_base: int = 0, return_nodes: bool = False,
              device=None) -> DtnResult:
    """Neumann data at every boundary point (bw_dtn_solve)."""
    ctx = N.context(device)
    dtn_cfg = dtn_cfg or DtnConfig()
    P = np.ascontiguousarray(patches, dtype=PATCH_DTYPE)
    L = np.ascontiguousarray(np.asarray(local_dirs, np.float64))
    if L.ndim == 2:
        L = L[None]
    Wt = np.ascontiguousarray(np.asarray(weights, np.float64).reshape(L.shape[0], L.shape[1]))
    n_bp, n_cls, n_nodes = len(P), L.shape[0], L.shape[1]
    ids = None if bp_ids is None else N.as_c(bp_ids, np.int64)
    dudn = np.empty(n_bp)
    err = np.empty(n_bp)
    status = np.empty(n_bp, np.int32)
    est = np.zeros((n_bp, n_nodes), N.ESTIMATE_DTYPE) if return_nodes else None
    steps = np.zeros((n_bp, n_nodes), np.int64) if return_nodes else None
    sc, wc, dc = scene.to_c(), wos_cfg.to_c(), dtn_cfg.to_c()
    rc = ctx.lib.bw_dtn_solve(ctx.handle, C.byref(sc), C.byref(wc), C.byref(dc), P.ctypes.data,
                              N.ptr(ids), n_bp, N.ptr(L), N.ptr(Wt), n_cls, n_nodes,
                              int(point_id_base), N.ptr(dudn), N.ptr(err), N.ptr(status),
                              None if est is None else est.ctypes.data, N.ptr(steps))
    res = DtnResult(dudn, err, status, est, steps)
    try:
        ctx.check(rc)
    except Exception as e:
        e.result = res
        raise
    return res


DTN_CLASSES, DTN_PER_PATCH = 0, 1  # bw_dtn_neumann methods (include/biewos_b200.h)


def dtn_neumann(scene, patches: np.ndarray, local_dirs, weights, node_est: np.ndarray,
                dtn_cfg=None, method: int = DTN_CLASSES, device=None) -> DtnResult:
    """The Neumann stage alone from given Gamma node estimates (bw_dtn_neumann):
    DTN_CLASSES = congruence-class tables (K7), DTN_PER_PATCH = K4 -> K2 -> K5."""
    ctx = N.context(device)
    dtn_cfg = dtn_cfg or DtnConfig()
    P = np.ascontiguousarray(patches, dtype=PATCH_DTYPE)
    L = np.ascontiguousarray(np.asarray(local_dirs, np.float64))
    if L.ndim == 2:
        L = L[None]
    Wt = np.ascontiguousarray(np.asarray(weights, np.float64).reshape(L.shape[0], L.shape[1]))
    n_bp, n_cls, n_nodes = len(P), L.shape[0], L.shape[1]
    E = np.ascontiguousarray(node_est, dtype=N.ESTIMATE_DTYPE).reshape(n_bp, n_nodes)
    dudn = np.empty(n_bp)
    err = np.empty(n_bp)
    status = np.empty(n_bp, np.int32)
    sc, dc = scene.to_c(), dtn_cfg.to_c()
    rc = ctx.lib.bw_dtn_neumann(ctx.handle, C.byref(sc), C.byref(dc), P.ctypes.data, n_bp,
                                N.ptr(L), N.ptr(Wt), n_cls, n_nodes, E.ctypes.data, int(method),
                                N.ptr(dudn), N.ptr(err), N.ptr(status))
    res = DtnResult(dudn, err, status)
    try:
        ctx.check(rc)
    except Exception as e:
        e.result = res
        raise
    return res


@dataclass
class NeumannField:  # patch_solver.hpp:78-82, one row per patch
    dudn: np.ndarray       # (n_bp, m) along the panel normals (into the domain)
    r: np.ndarray          # (n_bp, m) |centroid - o|
    est_error: np.ndarray  # (n_bp, m) |A^-1 b_se|
    status: np.ndarray     # (n_bp,) bit0 nodes outside the domain, bit1 solver failure


def solve_patch(scene, patches: np.ndarray, local_dirs, weights, node_est: np.ndarray,
                dtn_cfg=None, device=None) -> NeumannField:
    """solve_patch (patch_solver.cpp:311-335) for many patches (bw_solve_patch):
    the per-panel Neumann field of each patch from its Gamma node estimates."""
    ctx = N.context(device)
    dtn_cfg = dtn_cfg or DtnConfig()
    P = np.ascontiguousarray(patches, dtype=PATCH_DTYPE)
    L = np.ascontiguousarray(np.asarray(local_dirs, np.float64))
    if L.ndim == 2:
        L = L[None]
    Wt = np.ascontiguousarray(np.asarray(weights, np.float64).reshape(L.shape[0], L.shape[1]))
    n_bp, n_cls, n_nodes = len(P), L.shape[0], L.shape[1]
    E = np.ascontiguousarray(node_est, dtype=N.ESTIMATE_DTYPE).reshape(n_bp, n_nodes)
    m = dtn_cfg.m
    dudn, r, err = np.empty((n_bp, m)), np.empty((n_bp, m)), np.empty((n_bp, m))
    status = np.empty(n_bp, np.int32)
    sc, dc = scene.to_c(), dtn_cfg.to_c()
    rc = ctx.lib.bw_solve_patch(ctx.handle, C.byref(sc), C.byref(dc), P.ctypes.data, n_bp,
                                N.ptr(L), N.ptr(Wt), n_cls, n_nodes, E.ctypes.data, N.ptr(dudn),
                                N.ptr(r), N.ptr(err), N.ptr(status))
    res = NeumannField(dudn, r, err, status)
    try:
        ctx.check(rc)
    except Exception as e:
        e.result = res
        raise
    return res


def dtn_solve_workload(w, dtn_cfg=None, n_paths=None, bp_ids=None, return_nodes=False,
                       device=None, rng: int = 0) -> DtnResult:
    cfg = w.wos_config(n_paths, rng)
    return dtn_solve(w.scene, cfg, patches_for(w), w.dirs, w.weights, dtn_cfg, bp_ids=bp_ids,
                     return_nodes=return_nodes, device=device)


SOFT_STATUS = (5, 10)  # BW_ERR_RELIABILITY, BW_ERR_SOLVER: outputs written, details in status


def dtn_solve_device(scene, wos_cfg, dtn_cfg, d_patches, d_bp_ids, n_bp, d_dirs, d_weights,
                     n_cls, n_nodes, d_dudn, d_err, d_status, d_node_est=None, d_steps=None,
                     point_id_base=0, stream=None, device=None, soft: bool = False) -> int:
    """Device-pointer variant (bw_dtn_solve_d): inputs already in HBM.
    soft=True returns BW_ERR_RELIABILITY / BW_ERR_SOLVER instead of raising
    (every output is written, the per-point detail is in d_status): a sharded
    caller must agree across ranks on raising before its next collective, or the
    ranks without the failing point would block in it (distributed.raise_together)."""
    ctx = N.context(device)
    if stream is not None:
        ctx.set_stream(stream)
    sc, wc, dc = scene.to_c(), wos_cfg.to_c(), dtn_cfg.to_c()
    rc = ctx.lib.bw_dtn_solve_d(ctx.handle, C.byref(sc), C.byref(wc), C.byref(dc), d_patches,
                                d_bp_ids, n_bp, d_dirs, d_weights, n_cls, n_nodes,
                                int(point_id_base), d_dudn, d_err, d_status, d_node_est, d_steps)
    if soft and rc in SOFT_STATUS:
        return int(rc)
    ctx.check(rc)
    return 0
