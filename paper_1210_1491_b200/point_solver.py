"""Flat-boundary point formula (the reference's point_solver, next-row f2):
du/dn(x) = Sigma1' + Sigma2' along -axis, for one or many boundary points.

  cap_rule(n)                 quadrature.cpp:37-53 (unit-radius table)
  ring_rule_unit(n, dfrac)    quadrature.cpp:55-71 (in units of a)
  sigma1_prime / sigma2_prime point_solver.cpp:119-174
  solve_point(scene, frame, n_g1, n_g2, delta, cfg[, sampler])  point_solver.cpp:195-208
  solve_points(...)           the batch: K1 over all cap nodes, K6 per point
The node estimates come from K1 (bw_wos_patch_nodes) with point ids = cap
node index, exactly as sigma1_prime's estimate_u_batch(scene, pts, cfg)
(point_solver.cpp:160-166), so the walks are the reference's walks.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .dtn import PATCH_DTYPE
from .errors import ApplicabilityError, GeometryError
from .geometry import SceneKind
from .nodes import gauss_legendre, patch_node_positions, wos_patch_nodes

PI = 3.14159265358979323846


def cap_rule(n: int):
    """Local unit directions (n*n, 3) and unit-radius weights of the cap rule:
    theta_i = (pi/4)(x_i + 1), phi_j = pi (x_j + 1), w_i w_j (pi^2/4) sin theta_i."""
    if n < 2:
        raise GeometryError("cap_rule: need n >= 2")
    x, w = gauss_legendre(n)
    dirs, wts = [], []
    for i in range(n):
        th = PI / 4.0 * (x[i] + 1.0)
        elem = (PI * PI / 4.0) * math.sin(th)
        for j in range(n):
            ph = PI * (x[j] + 1.0)
            dirs.append([math.sin(th) * math.cos(ph), math.sin(th) * math.sin(ph), math.cos(th)])
            wts.append(w[i] * w[j] * elem)
    return np.array(dirs), np.array(wts)


def ring_rule_unit(n: int, delta_frac: float) -> np.ndarray:
    """(n*n, 4) table {rho/a, cos psi, sin psi, weight/a^2} of
    ring_rule(a, delta = delta_frac a, n) (quadrature.cpp:55-71); the
    trigonometry is done here with the host libm, like the reference."""
    if not (delta_frac > 0) or delta_frac >= 1.0:
        raise GeometryError("ring_rule: need 0 < delta < a")
    x, w = gauss_legendre(n)
    out = []
    for i in range(n):
        rho = delta_frac + (1.0 - delta_frac) * 0.5 * (x[i] + 1.0)
        wr = w[i] * 0.5 * (1.0 - delta_frac)
        for j in range(n):
            psi = PI * (x[j] + 1.0)
            out.append([rho, math.cos(psi), math.sin(psi), wr * w[j] * PI * rho])
    return np.array(out)


@dataclass
class HemisphereFrame:  # greens.hpp:16-30 (centre, radius, axis into the solution side)
    center: tuple
    radius: float
    axis: tuple = (0.0, 0.0, 1.0)


@dataclass
class PointNeumannResult:  # point_solver.hpp:13-22
    sigma1: float
    sigma2: float
    total: float
    std_error: float
    a: float
    delta: float
    n_g1: int
    n_g2: int


def _patches(centers, axes, radii) -> np.ndarray:
    c = np.asarray(centers, float).reshape(-1, 3)
    p = np.zeros(len(c), PATCH_DTYPE)
    p["o"] = c
    p["axis"] = np.asarray(axes, float).reshape(-1, 3)
    p["a"] = np.broadcast_to(np.asarray(radii, float), (len(c),))
    p["surf"] = 1
    return p


def point_formula(scene, patches, cap_dirs, cap_weights, est, ring, device=None):
    """K6 over many points: returns (total, sigma1, sigma2, std_error) arrays."""
    ctx = N.context(device)
    P = np.ascontiguousarray(patches, dtype=PATCH_DTYPE)
    n = len(P)
    D = N.as_c(cap_dirs, np.float64, 3)
    Wt = N.as_c(cap_weights, np.float64)
    E = np.ascontiguousarray(est, dtype=N.ESTIMATE_DTYPE).reshape(n, len(D))
    R = N.as_c(ring, np.float64, 4)
    out = [np.empty(n) for _ in range(4)]
    sc = scene.to_c()
    ctx.check(ctx.lib.bw_point_formula(ctx.handle, C.byref(sc), P.ctypes.data, n, N.ptr(D),
                                       N.ptr(Wt), len(D), E.ctypes.data, N.ptr(R), len(R),
                                       *[N.ptr(o) for o in out]))
    return tuple(out)


def solve_points(scene, centers, axes, radii, n_g1, n_g2, delta_frac, cfg, device=None):
    """Point formula at many flat-boundary points (one K1 launch + one K6)."""
    if scene.kind == SceneKind.Sphere:
        raise ApplicabilityError("point solver requires a flat boundary scene")
    dirs, wts = cap_rule(n_g1)
    est, _ = wos_patch_nodes(scene, cfg, centers, axes, radii, dirs, device=device)
    return point_formula(scene, _patches(centers, axes, radii), dirs, wts, est,
                         ring_rule_unit(n_g2, delta_frac), device)


def solve_point(scene, frame: HemisphereFrame, n_g1: int, n_g2: int, delta: float, cfg,
                sampler=None, device=None) -> PointNeumannResult:
    """point_solver.cpp:195-208 (with an optional PotentialSampler, :202-208)."""
    if scene.kind == SceneKind.Sphere:
        raise ApplicabilityError("point solver requires a flat boundary scene")
    a = float(frame.radius)
    dirs, wts = cap_rule(n_g1)
    c = np.asarray(frame.center, float)[None]
    ax = np.asarray(frame.axis, float)[None]
    if sampler is None:
        est, _ = wos_patch_nodes(scene, cfg, c, ax, a, dirs, device=device)
    else:
        pos = patch_node_positions(c, ax, a, None, dirs)[0]
        est = np.zeros((1, len(pos)), N.ESTIMATE_DTYPE)
        for i, y in enumerate(pos):
            e = sampler(y, i)
            est[0, i] = (e.mean, e.variance, e.n, e.n_infinity, e.n_failed)
    total, s1, s2, se = point_formula(scene, _patches(c, ax, a), dirs, wts, est,
                                      ring_rule_unit(n_g2, delta / a), device)
    return PointNeumannResult(float(s1[0]), float(s2[0]), float(total[0]), float(se[0]), a,
                              delta, n_g1, n_g2)
