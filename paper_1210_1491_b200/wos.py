"""Walk-on-spheres entry points: the reference's wos.hpp API on the B200 kernel.

Same names, argument meaning and error behaviour as proj/include/biewos/wos.hpp:
  walk(scene, start, cfg, point_id, path_id)            wos.hpp:32-34
  exit_value(scene, rec)                                wos.hpp:37
  estimate_u(scene, p, cfg, point_id=0)                 wos.hpp:40-41
  estimate_u_batch(scene, points, cfg, point_id_base=0) wos.hpp:45-46
  wos_sampler(scene, cfg)                               wos.hpp:49-50
All run the sm_100a kernels in libbiewos_b200.so through the C-ABI.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .errors import ReliabilityError
from .geometry import Scene, kExitFailed, kExitInfinity

ESTIMATE_DTYPE = N.ESTIMATE_DTYPE
RNG_PHILOX4X64, RNG_PHILOX4X32 = 0, 1  # bw_rng_kind


@dataclass
class WosConfig:  # wos.hpp:13-20
    eps_shell: float = 1e-5
    trunc_radius: float = 1e5
    n_paths: int = 1000
    max_steps: int = 10000
    seed: int = 0
    workers: int = 1  # affects speed only, never results (meaningless on device)
    # additive (include/biewos_b200.h bw_wos_config): RNG_PHILOX4X64 is the
    # reference's RngStream bit for bit; RNG_PHILOX4X32 a statistically
    # equivalent Philox4x32-10 stream. eps_rel: patch nodes walk with
    # eps_b = min(eps_shell, eps_rel * a_b) (0 = off).
    rng: int = 0
    eps_rel: float = 0.0

    def to_c(self) -> N.BwWosConfig:
        c = N.BwWosConfig()
        c.eps_shell = self.eps_shell
        c.trunc_radius = self.trunc_radius
        c.n_paths = int(self.n_paths)
        c.max_steps = int(self.max_steps)
        c.seed = int(self.seed) & 0xFFFFFFFFFFFFFFFF
        c.rng = int(self.rng)
        c.eps_rel = float(self.eps_rel)
        return c


@dataclass
class Estimate:  # wos.hpp:22-29
    mean: float = 0.0
    variance: float = 0.0
    n: int = 0
    n_infinity: int = 0
    n_failed: int = 0

    def std_error(self) -> float:  # wos.cpp:55-57
        return float(np.sqrt(self.variance / self.n)) if self.n > 0 else 0.0

    @staticmethod
    def from_record(r) -> "Estimate":
        return Estimate(float(r["mean"]), float(r["variance"]), int(r["n"]),
                        int(r["n_infinity"]), int(r["n_failed"]))


@dataclass
class ExitRecord:  # geometry.hpp:28-32
    point: np.ndarray
    feature: int
    steps: int


def std_error(est: np.ndarray) -> np.ndarray:
    """Vectorised Estimate::std_error over an ESTIMATE_DTYPE array."""
    n = est["n"].astype(np.float64)
    with np.errstate(invalid="ignore", divide="ignore"):
        return np.where(n > 0, np.sqrt(est["variance"] / np.maximum(n, 1)), 0.0)


def walk_batch(scene: Scene, starts, cfg: WosConfig, point_ids, path_ids, device=None):
    """One trajectory per row (wos.cpp:61-85). Returns (exit_points, features, steps)."""
    ctx = N.context(device)
    starts = N.as_c(starts, np.float64, 3)
    n = len(starts)
    pids = N.as_c(np.broadcast_to(np.asarray(point_ids, dtype=np.uint64), (n,)), np.uint64)
    paths = N.as_c(np.broadcast_to(np.asarray(path_ids, dtype=np.uint64), (n,)), np.uint64)
    ex = np.empty((n, 3), np.float64)
    feat = np.empty(n, np.int32)
    steps = np.empty(n, np.int32)
    sc, cf = scene.to_c(), cfg.to_c()
    ctx.check(ctx.lib.bw_walk(ctx.handle, C.byref(sc), C.byref(cf), N.ptr(starts), n,
                              N.ptr(pids), N.ptr(paths), N.ptr(ex), N.ptr(feat), N.ptr(steps)))
    return ex, feat, steps


@dataclass
class DistanceQuery:  # geometry.hpp:66-70
    distance: float
    feature: int


def nearest_feature_batch(scene: Scene, points, device=None, walk_distance: bool = False):
    """nearest_feature (geometry.cpp:131-155) for many points on the device
    (bw_nearest_feature): (distance, feature[, K1 walk-loop distance])."""
    ctx = N.context(device)
    pts = N.as_c(points, np.float64, 3)
    n = len(pts)
    d, f = np.empty(n), np.empty(n, np.int32)
    dw = np.empty(n) if walk_distance else None
    sc = scene.to_c()
    ctx.check(ctx.lib.bw_nearest_feature(ctx.handle, C.byref(sc), N.ptr(pts), n, N.ptr(d),
                                         N.ptr(f), N.ptr(dw)))
    return (d, f, dw) if walk_distance else (d, f)


def nearest_feature(scene: Scene, p, device=None) -> DistanceQuery:
    d, f = nearest_feature_batch(scene, np.asarray(p, np.float64)[None], device)
    return DistanceQuery(float(d[0]), int(f[0]))


def distance_to_boundary(scene: Scene, p, device=None) -> DistanceQuery:
    """geometry.cpp:157-171: DomainError on or outside the solution domain."""
    ctx = N.context(device)
    pts = N.as_c(np.asarray(p, np.float64)[None], np.float64, 3)
    d, f = np.empty(1), np.empty(1, np.int32)
    sc = scene.to_c()
    ctx.check(ctx.lib.bw_distance_to_boundary(ctx.handle, C.byref(sc), N.ptr(pts), 1, N.ptr(d),
                                              N.ptr(f)))
    return DistanceQuery(float(d[0]), int(f[0]))


def classify_exit_batch(scene: Scene, points, eps: float, trunc_radius: float, device=None):
    """classify_exit (geometry.cpp:222-239) for many points (bw_classify_exit):
    (projected points, features); ClassificationError if any point is neither
    near the boundary nor truncated."""
    ctx = N.context(device)
    pts = N.as_c(points, np.float64, 3)
    n = len(pts)
    q, f = np.empty((n, 3)), np.empty(n, np.int32)
    sc = scene.to_c()
    ctx.check(ctx.lib.bw_classify_exit(ctx.handle, C.byref(sc), N.ptr(pts), n, float(eps),
                                       float(trunc_radius), N.ptr(q), N.ptr(f)))
    return q, f


def classify_exit(scene: Scene, p, eps: float, trunc_radius: float, device=None) -> ExitRecord:
    q, f = classify_exit_batch(scene, np.asarray(p, np.float64)[None], eps, trunc_radius, device)
    return ExitRecord(q[0], int(f[0]), 0)


def walk(scene: Scene, start, cfg: WosConfig, point_id: int, path_id: int) -> ExitRecord:
    ex, f, s = walk_batch(scene, np.asarray(start, dtype=np.float64)[None], cfg, point_id, path_id)
    return ExitRecord(ex[0], int(f[0]), int(s[0]))


def exit_value(scene: Scene, rec: ExitRecord) -> float:  # wos.cpp:87-93
    if rec.feature == kExitInfinity:
        return 0.0
    if rec.feature == kExitFailed:
        raise ReliabilityError("no boundary value for a failed path")
    if scene.piecewise_const:
        return float(scene.feature_potential[rec.feature])
    return float(scene.dirichlet(rec.point))


def estimate_u_batch_full(scene: Scene, points, cfg: WosConfig, point_id_base: int = 0,
                          device=None):
    """estimate_u_batch plus the per-point WOS step counts.

    Returns (estimates [ESTIMATE_DTYPE], steps [int64]). Raises ReliabilityError
    when any point has more than 0.1% failed walks (wos.cpp:43-44), like the
    reference; the exception carries `.estimates` and `.steps`.
    """
    ctx = N.context(device)
    pts = N.as_c(points, np.float64, 3)
    n = len(pts)
    out = np.zeros(n, ESTIMATE_DTYPE)
    steps = np.zeros(n, np.int64)
    if n == 0:
        return out, steps
    sc, cf = scene.to_c(), cfg.to_c()
    rc = ctx.lib.bw_wos_estimate(ctx.handle, C.byref(sc), C.byref(cf), N.ptr(pts), n,
                                 int(point_id_base), out.ctypes.data, N.ptr(steps))
    try:
        ctx.check(rc)
    except Exception as e:
        e.estimates, e.steps = out, steps
        raise
    return out, steps


def estimate_u_batch(scene: Scene, points, cfg: WosConfig, point_id_base: int = 0,
                     device=None) -> np.ndarray:
    """wos.cpp:95-132 on the B200: per-point estimates, point ids base + index.

    Bit-identical for any launch geometry / device count (wos.hpp:43-44)."""
    return estimate_u_batch_full(scene, points, cfg, point_id_base, device)[0]


def estimate_u(scene: Scene, p, cfg: WosConfig, point_id: int = 0, device=None) -> Estimate:
    est = estimate_u_batch(scene, np.asarray(p, dtype=np.float64)[None], cfg, point_id, device)
    return Estimate.from_record(est[0])


def wos_sampler(scene: Scene, cfg: WosConfig):
    """PotentialSampler (wos.hpp:48-50): (y, point_id) -> Estimate."""
    return lambda y, point_id: estimate_u(scene, y, cfg, point_id)


def estimate_u_batch_device(scene: Scene, d_points: int, n: int, cfg: WosConfig,
                            point_id_base: int, d_out: int, d_steps: int | None,
                            stream: int | None = None, device=None) -> None:
    """Device-pointer variant (bw_wos_estimate_d): inputs already in HBM."""
    ctx = N.context(device)
    if stream is not None:
        ctx.set_stream(stream)
    sc, cf = scene.to_c(), cfg.to_c()
    ctx.check(ctx.lib.bw_wos_estimate_d(ctx.handle, C.byref(sc), C.byref(cf), d_points, n,
                                        int(point_id_base), d_out, d_steps))
