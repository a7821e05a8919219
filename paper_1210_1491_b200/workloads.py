"""The five BASELINE.json configurations as seeded synthetic workloads.

BASELINE.json names synthetic problems (no dataset): these builders fix every
generator the reference lacks once, for the oracle, the
tests and bench.py alike:
  cfg1/cfg4  interior unit ball, u = x^2 - y^2 + z, Fibonacci boundary points
  cfg2       interior unit cube, u = exp(sqrt2 pi x) sin(pi y) sin(pi z),
             32 x 32 cell-centred points per face
  cfg3/cfg5  [-1,1]^3 minus 64 cavities (rejection-sampled from a Philox
             stream, seed 3), u = 1/|x - c0|, points split by area
A boundary point b carries a hemisphere frame: centre, unit axis pointing into
the solution domain (the reference's "object-outward" normal, patch_solver.hpp:
16,27), radius a and a node class (theta_max of its Gamma). Gamma nodes are
theta-Gauss-Legendre x phi-uniform.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .geometry import DomainSide, ExpSinSin, PointSource, Quadratic, Scene
from .nodes import cube_face_points, fibonacci_sphere, gamma_rule

M64 = (1 << 64) - 1
_M0, _M1 = 0xD2E7470EE14C6C93, 0xCA5A826395121157
_W0, _W1 = 0x9E3779B97F4A7C15, 0xBB67AE8584CAA73B


def _mulhilo(a: np.ndarray, b: int):
    """Vectorised 64x64 -> 128 multiply of uint64 arrays by a constant."""
    a = a.astype(np.uint64)
    m32 = np.uint64(0xFFFFFFFF)
    al, ah = a & m32, a >> np.uint64(32)
    bl, bh = np.uint64(b & 0xFFFFFFFF), np.uint64(b >> 32)
    ll, lh, hl, hh = al * bl, al * bh, ah * bl, ah * bh
    mid = (ll >> np.uint64(32)) + (lh & m32) + (hl & m32)
    lo = (ll & m32) | ((mid & m32) << np.uint64(32))
    hi = hh + (lh >> np.uint64(32)) + (hl >> np.uint64(32)) + (mid >> np.uint64(32))
    return hi, lo


def philox_blocks(c0, c1, c2, c3, k0: int, k1: int) -> np.ndarray:
    """Philox4x64-10 (rng.hpp:25-38), vectorised over counters. Host setup only."""
    c = [np.asarray(x, dtype=np.uint64).copy() for x in (c0, c1, c2, c3)]
    for r in range(10):
        if r > 0:
            k0 = (k0 + _W0) & M64
            k1 = (k1 + _W1) & M64
        hi0, lo0 = _mulhilo(c[0], _M0)
        hi1, lo1 = _mulhilo(c[2], _M1)
        c = [hi1 ^ c[1] ^ np.uint64(k0), lo1, hi0 ^ c[3] ^ np.uint64(k1), lo0]
    return np.stack(c, axis=-1)


def stream_doubles(seed: int, point_id: int, path_id: int, domain: int, n: int) -> np.ndarray:
    """First n doubles of RngStream(seed, point_id, path_id, domain) (rng.hpp:44-60)."""
    nb = (n + 3) // 4
    blk = np.arange(nb, dtype=np.uint64)
    out = philox_blocks(blk, np.full(nb, path_id, np.uint64), np.full(nb, point_id, np.uint64),
                        np.full(nb, domain, np.uint64), seed & M64,
                        0x1BD11BDAA9FC1A22 ^ domain).reshape(-1)[:n]
    return (out >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


DOMAIN_CAVITIES = 2  # RNG domain tags of the generators (0 = WOS, 1 = last-passage)
DOMAIN_TARGETS = 3
DOMAIN_FACES = 4


def make_cavities(n: int = 64, seed: int = 3, clearance: float = 0.04,
                  box: float = 0.8, rmin: float = 0.05, rmax: float = 0.1) -> np.ndarray:
    """Rejection-sampled non-overlapping cavities: attempt t draws 4 doubles
    (cx, cy, cz, r) from RngStream(seed, 0, t, DOMAIN_CAVITIES); accept when
    |c - c_j| > r + r_j + clearance for every accepted j (clearance = 2a keeps
    each Gamma clear of other cavities)."""
    acc = []
    t = 0
    while len(acc) < n:
        u = stream_doubles(seed, 0, t, DOMAIN_CAVITIES, 4)
        c = -box + 2 * box * u[:3]
        r = rmin + (rmax - rmin) * u[3]
        if all(np.linalg.norm(c - a[:3]) > r + a[3] + clearance for a in acc):
            acc.append(np.array([*c, r]))
        t += 1
        if t > 100000:
            raise RuntimeError("cavity rejection sampling did not converge")
    return np.array(acc)


def largest_remainder(weights, total: int) -> np.ndarray:
    w = np.asarray(weights, float)
    q = w / w.sum() * total
    base = np.floor(q).astype(np.int64)
    rem = total - base.sum()
    order = np.argsort(-(q - base), kind="stable")
    base[order[:rem]] += 1
    return base


def r2_points(n: int, offset: int = 0) -> np.ndarray:
    """R2 low-discrepancy points in [0,1)^2 (plastic-number additive recurrence)."""
    g = 1.32471795724474602596
    i = np.arange(offset, offset + n, dtype=np.float64) + 1
    return np.stack([np.mod(0.5 + i / g, 1.0), np.mod(0.5 + i / (g * g), 1.0)], axis=1)


@dataclass
class Workload:
    name: str
    scene: Scene
    points: np.ndarray        # (n_bp, 3) boundary points
    axes: np.ndarray          # (n_bp, 3) unit normals into the solution domain
    a: float                  # hemisphere radius
    cls: np.ndarray           # (n_bp,) node class
    theta_max: np.ndarray     # (n_cls,) Gamma rim angle per class
    n_theta: int
    n_phi: int
    n_paths: int
    eps: float
    seed: int
    exact_u: object = None
    exact_grad: object = None
    radii: np.ndarray = field(default=None)    # (n_bp,) per-point hemisphere radius
    # per-point shell eps_b = min(eps, eps_rel a_b) (bw_wos_config.eps_rel): only
    # hemispheres shrunk below eps / eps_rel (edge and corner points of the box
    # faces, config 3/5) walk with a thinner shell, so the eps bias of du/dn,
    # O(eps_b / a_b), stays <= 1e-3 relative to the data's variation
    eps_rel: float = 1e-3
    dirs: np.ndarray = field(default=None)     # (n_cls, n_nodes, 3)
    weights: np.ndarray = field(default=None)  # (n_cls, n_nodes) unit-sphere weights
    extra: dict = field(default_factory=dict)

    def __post_init__(self):
        if self.radii is None:
            self.radii = np.full(len(self.points), float(self.a))
        d, w = [], []
        for tm in self.theta_max:
            di, wi = gamma_rule(self.n_theta, self.n_phi, float(tm))
            d.append(di)
            w.append(wi)
        self.dirs = np.ascontiguousarray(np.stack(d))
        self.weights = np.stack(w)

    @property
    def n_bp(self) -> int:
        return len(self.points)

    @property
    def n_nodes(self) -> int:
        return self.n_theta * self.n_phi

    def subset(self, idx) -> "Workload":
        w = Workload(self.name, self.scene, self.points[idx], self.axes[idx], self.a,
                     self.cls[idx], self.theta_max, self.n_theta, self.n_phi, self.n_paths,
                     self.eps, self.seed, self.exact_u, self.exact_grad,
                     radii=self.radii[idx], eps_rel=self.eps_rel)
        w.extra = dict(self.extra)
        return w

    def eps_of(self, b) -> np.ndarray:
        """The shell thickness boundary point(s) b walk with."""
        r = np.asarray(self.radii)[b]
        return np.minimum(self.eps, self.eps_rel * r) if self.eps_rel > 0 else np.full_like(r, self.eps)

    def wos_config(self, n_paths=None, rng: int = 0, eps=None):
        from .wos import WosConfig

        return WosConfig(eps_shell=self.eps if eps is None else float(eps),
                         n_paths=n_paths or self.n_paths, seed=self.seed, rng=rng,
                         eps_rel=self.eps_rel if eps is None else 0.0)

    def exact_dudn_outward(self) -> np.ndarray:
        """Analytic du/dn along the domain-OUTWARD normal (= -axis)."""
        return -(self.exact_grad(self.points) * self.axes).sum(axis=1)


def _ball(name, n_bp, a, n_theta, n_phi, n_paths, eps, seed):
    q = Quadratic(g=(0.0, 0.0, 1.0), q=(1.0, -1.0, 0.0, 0.0, 0.0, 0.0))
    scene = Scene.sphere(1.0, DomainSide.Interior, q)
    pts = fibonacci_sphere(n_bp, 1.0)
    axes = -pts / np.linalg.norm(pts, axis=1, keepdims=True)
    return Workload(name, scene, pts, axes, a, np.zeros(n_bp, np.int32),
                    np.array([math.acos(a / 2.0)]), n_theta, n_phi, n_paths, eps, seed,
                    exact_u=q, exact_grad=q.grad)


def config1(n_bp: int = 1000) -> Workload:
    return _ball("cfg1_unit_ball", n_bp, 0.2, 16, 32, 10000, 1e-4, 1)


def config4(n_bp: int = 100000) -> Workload:
    return _ball("cfg4_unit_ball_scaling", n_bp, 0.05, 8, 16, 4096, 1e-5, 4)


def edge_clear_radii(points, axes, lo, hi, a: float, margin: float = 0.9) -> np.ndarray:
    """Hemisphere radius per face point: a, shrunk near edges and corners so
    the hemisphere (and so every Gamma node and the patch disk) stays inside
    the box: a_b = min(a, margin * distance d to the nearest other face plane).
    margin 0.9 keeps every Gamma node >= 0.1 d from the other faces (0.999 put
    rim nodes within ~2 eps of them). The points then walk with a shell
    eps_b = min(eps, eps_rel a_b) (Workload.eps_rel). The reference has no
    edge/corner construction; this is the documented deviation."""
    lo, hi = np.asarray(lo, float), np.asarray(hi, float)
    r = np.full(len(points), float(a))
    for k in range(3):
        other = np.abs(axes[:, k]) < 0.5  # the face is not normal to axis k
        d = np.minimum(points[:, k] - lo[k], hi[k] - points[:, k])
        r = np.where(other, np.minimum(r, margin * d), r)
    return r


def config2(k: int = 32) -> Workload:
    phi = ExpSinSin(1.0, (math.sqrt(2.0) * math.pi, math.pi, math.pi))
    scene = Scene.box((0, 0, 0), (1, 1, 1), phi)
    pts, nrm, _ = cube_face_points(k)
    return Workload("cfg2_unit_cube", scene, pts, nrm, 0.05, np.zeros(len(pts), np.int32),
                    np.array([math.pi / 2]), 8, 16, 4096, 1e-5, 2, exact_u=phi,
                    exact_grad=phi.grad,
                    radii=edge_clear_radii(pts, nrm, (0, 0, 0), (1, 1, 1), 0.05))


def _cavity_box(name, n_bp, a, seed):
    cav = make_cavities(64, 3, clearance=2 * 0.02)
    src = PointSource(q=1.0, s=tuple(cav[0, :3]))
    scene = Scene.box_with_cavities((-1, -1, -1), (1, 1, 1), cav, src)
    areas = np.concatenate([np.full(6, 4.0), 4 * np.pi * cav[:, 3] ** 2])
    counts = largest_remainder(areas, n_bp)
    pts, axes, cls = [], [], []
    off = 0
    for f in range(6):
        n = int(counts[f])
        uv = r2_points(n, off) * 2.0 - 1.0
        off += n
        ax = f // 2
        others = [k for k in range(3) if k != ax]
        p = np.empty((n, 3))
        p[:, ax] = 1.0 if f & 1 else -1.0
        p[:, others[0]], p[:, others[1]] = uv[:, 0], uv[:, 1]
        nrm = np.zeros((n, 3))
        nrm[:, ax] = -1.0 if f & 1 else 1.0
        pts.append(p)
        axes.append(nrm)
        cls.append(np.zeros(n, np.int32))
    for i, c in enumerate(cav):
        n = int(counts[6 + i])
        u = fibonacci_sphere(n, 1.0) if n > 0 else np.zeros((0, 3))
        pts.append(c[:3] + c[3] * u)
        axes.append(u)
        cls.append(np.full(n, 1 + i, np.int32))
    theta_max = np.concatenate([[math.pi / 2], np.arccos(-a / (2 * cav[:, 3]))])
    P, AX, CL = np.concatenate(pts), np.concatenate(axes), np.concatenate(cls)
    radii = np.where(CL == 0, edge_clear_radii(P, AX, (-1, -1, -1), (1, 1, 1), a), a)
    w = Workload(name, scene, P, AX, a, CL, theta_max, 8, 16, 4096, 1e-5, seed, exact_u=src,
                 exact_grad=src.grad, radii=radii)
    w.extra["cavities"] = cav
    return w


def config3(n_bp: int = 20000) -> Workload:
    return _cavity_box("cfg3_box_64_cavities", n_bp, 0.02, 3)


def config5(n_bp: int = 200000, n_targets: int = 1000000) -> Workload:
    w = _cavity_box("cfg5_full_pipeline", n_bp, 0.02, 5)
    w.extra["n_targets"] = n_targets
    return w


def make_targets(w: Workload, n: int, seed: int = 5) -> np.ndarray:
    """Uniform targets in the box rejecting cavity interiors: candidate t uses
    RngStream(seed, 0, t, DOMAIN_TARGETS) (3 doubles)."""
    cav = w.extra["cavities"]
    out = np.empty((0, 3))
    start = 0
    while len(out) < n:
        m = int((n - len(out)) * 1.1) + 16
        t = np.arange(start, start + m, dtype=np.uint64)
        blk = philox_blocks(np.zeros(m, np.uint64), t, np.zeros(m, np.uint64),
                            np.full(m, DOMAIN_TARGETS, np.uint64), seed,
                            0x1BD11BDAA9FC1A22 ^ DOMAIN_TARGETS)
        u = (blk[:, :3] >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
        x = -1.0 + 2.0 * u
        ok = np.ones(m, bool)
        for c in cav:
            ok &= np.linalg.norm(x - c[:3], axis=1) > c[3]
        out = np.concatenate([out, x[ok]])
        start += m
    return out[:n]


CONFIGS = {1: config1, 2: config2, 3: config3, 4: config4, 5: config5}
