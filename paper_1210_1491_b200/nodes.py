"""Boundary points, hemisphere frames and Gamma node rules (host setup).

  gauss_legendre(n)              quadrature.cpp:7-35 (same Newton iteration)
  gamma_rule(nt, np_, theta_max) theta Gauss-Legendre x phi uniform node rule of the
                                 BASELINE configs
  fibonacci_sphere(n)            SURVEY.md 8(d) cfg1/4 lattice
  cube_face_points(k)            cfg2: k x k cell-centred grid per face
  frame(axis)                    greens.cpp:98-105 orthonormal completion
  wos_patch_nodes(...)           K1 over all Gamma nodes of many boundary points
"""
from __future__ import annotations

import ctypes as C
import math

import numpy as np

from . import _native as N

PI = 3.14159265358979323846


def gauss_legendre(n: int):
    if n < 1 or n > 64:
        from .errors import GeometryError

        raise GeometryError("gauss_legendre: order must be in [1,64]")
    x = np.zeros(n)
    w = np.zeros(n)
    m = (n + 1) // 2
    for i in range(1, m + 1):
        z = math.cos(PI * (i - 0.25) / (n + 0.5))
        while True:
            p1, p2 = 1.0, 0.0
            for j in range(1, n + 1):
                p3 = p2
                p2 = p1
                p1 = ((2.0 * j - 1.0) * z * p2 - (j - 1.0) * p3) / j
            pp = n * (z * p1 - p2) / (z * z - 1.0)
            z1 = z
            z = z1 - p1 / pp
            if abs(z - z1) <= 1e-15:
                break
        x[i - 1] = -z
        x[n - i] = z
        w[i - 1] = 2.0 / ((1.0 - z * z) * pp * pp)
        w[n - i] = w[i - 1]
    if n % 2 == 1:
        x[n // 2] = 0.0
    return x, w


def gamma_rule(n_theta: int, n_phi: int, theta_max: float):
    """Local unit directions (n_theta*n_phi, 3), row-major [theta][phi], and
    weights for the unit sphere (GL weight x theta_max/2 x 2pi/n_phi x sin theta)."""
    x, w = gauss_legendre(n_theta)
    th = theta_max * 0.5 * (x + 1.0)
    ph = 2.0 * PI * np.arange(n_phi) / n_phi
    st, ct = np.sin(th), np.cos(th)
    dirs = np.empty((n_theta, n_phi, 3))
    dirs[..., 0] = st[:, None] * np.cos(ph)[None, :]
    dirs[..., 1] = st[:, None] * np.sin(ph)[None, :]
    dirs[..., 2] = ct[:, None]
    wts = (w * 0.5 * theta_max * st)[:, None] * np.full(n_phi, 2.0 * PI / n_phi)[None, :]
    return dirs.reshape(-1, 3), wts.reshape(-1)


def fibonacci_sphere(n: int, radius: float = 1.0) -> np.ndarray:
    i = np.arange(n, dtype=np.float64)
    z = 1.0 - (2.0 * i + 1.0) / n
    r = np.sqrt(1.0 - z * z)
    ph = i * (PI * (3.0 - math.sqrt(5.0)))
    return radius * np.stack([r * np.cos(ph), r * np.sin(ph), z], axis=1)


def cube_face_points(k: int, lo=(0.0, 0.0, 0.0), hi=(1.0, 1.0, 1.0)):
    """k x k cell-centred points per face, faces in feature order
    x=lo, x=hi, y=lo, y=hi, z=lo, z=hi. Returns (points, inward normals, face id)."""
    lo, hi = np.asarray(lo, float), np.asarray(hi, float)
    c = (np.arange(k) + 0.5) / k
    u, v = np.meshgrid(c, c, indexing="ij")
    u, v = u.ravel(), v.ravel()
    pts, nrm, fid = [], [], []
    for f in range(6):
        ax = f // 2
        others = [a for a in range(3) if a != ax]
        p = np.empty((k * k, 3))
        p[:, ax] = hi[ax] if f & 1 else lo[ax]
        p[:, others[0]] = lo[others[0]] + u * (hi[others[0]] - lo[others[0]])
        p[:, others[1]] = lo[others[1]] + v * (hi[others[1]] - lo[others[1]])
        n = np.zeros((k * k, 3))
        n[:, ax] = -1.0 if f & 1 else 1.0
        pts.append(p)
        nrm.append(n)
        fid.append(np.full(k * k, f, np.int32))
    return np.concatenate(pts), np.concatenate(nrm), np.concatenate(fid)


def frame(axis):
    """(e1, e2) completing a unit axis (greens.cpp:98-105), vectorised."""
    axis = np.asarray(axis, dtype=np.float64).reshape(-1, 3)
    ref = np.where(np.abs(axis[:, :1]) < 0.9, [[1.0, 0.0, 0.0]], [[0.0, 1.0, 0.0]])
    e1 = np.cross(axis, ref)
    e1 /= np.linalg.norm(e1, axis=1, keepdims=True)
    e2 = np.cross(axis, e1)
    return e1, e2


def patch_node_positions(centers, axes, radii, cls, local_dirs):
    """Host evaluation of the node formula used by K1 (for drivers and tests)."""
    centers = np.asarray(centers, float).reshape(-1, 3)
    axes = np.asarray(axes, float).reshape(-1, 3)
    e1, e2 = frame(axes)
    L = np.asarray(local_dirs, float)
    if L.ndim == 2:
        L = L[None]
    cls = np.zeros(len(centers), np.int64) if cls is None else np.asarray(cls)
    l = L[cls]  # (n_bp, n_nodes, 3)
    w = l[..., :1] * e1[:, None, :] + l[..., 1:2] * e2[:, None, :] + l[..., 2:3] * axes[:, None, :]
    return centers[:, None, :] + np.asarray(radii, float).reshape(-1, 1, 1) * w


def wos_patch_nodes(scene, cfg, centers, axes, radii, local_dirs, cls=None,
                    point_id_base: int = 0, bp_ids=None, device=None):
    """K1 over the Gamma nodes of n_bp boundary points (bw_wos_patch_nodes).
    Returns (estimates (n_bp, n_nodes) ESTIMATE_DTYPE, steps (n_bp, n_nodes))."""
    ctx = N.context(device)
    centers = N.as_c(centers, np.float64, 3)
    axes = N.as_c(axes, np.float64, 3)
    n_bp = len(centers)
    radii = N.as_c(np.broadcast_to(np.asarray(radii, np.float64), (n_bp,)), np.float64)
    L = np.ascontiguousarray(np.asarray(local_dirs, np.float64))
    if L.ndim == 2:
        L = L[None]
    n_cls, n_nodes = L.shape[0], L.shape[1]
    cls_a = None if cls is None else N.as_c(cls, np.int32)
    ids = None if bp_ids is None else N.as_c(bp_ids, np.int64)
    out = np.zeros((n_bp, n_nodes), N.ESTIMATE_DTYPE)
    steps = np.zeros((n_bp, n_nodes), np.int64)
    sc, cf = scene.to_c(), cfg.to_c()
    rc = ctx.lib.bw_wos_patch_nodes(ctx.handle, C.byref(sc), C.byref(cf), N.ptr(centers),
                                    N.ptr(axes), N.ptr(radii), N.ptr(cls_a), N.ptr(ids), n_bp,
                                    N.ptr(L),
                                    n_cls, n_nodes, int(point_id_base), out.ctypes.data,
                                    N.ptr(steps))
    try:
        ctx.check(rc)
    except Exception as e:
        e.estimates, e.steps = out, steps
        raise
    return out, steps


def wos_patch_nodes_device(scene, cfg, d_centers, d_axes, d_radii, d_cls, d_bp_ids, n_bp, d_dirs,
                           n_cls, n_nodes, point_id_base, d_out, d_steps, stream=None,
                           device=None):
    """Device-pointer variant (bw_wos_patch_nodes_d): all arrays already in HBM."""
    ctx = N.context(device)
    if stream is not None:
        ctx.set_stream(stream)
    sc, cf = scene.to_c(), cfg.to_c()
    ctx.check(ctx.lib.bw_wos_patch_nodes_d(ctx.handle, C.byref(sc), C.byref(cf), d_centers,
                                           d_axes, d_radii, d_cls, d_bp_ids, n_bp, d_dirs, n_cls,
                                           n_nodes,
                                           int(point_id_base), d_out, d_steps))
