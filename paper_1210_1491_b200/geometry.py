"""Scene + Dirichlet data: host mirror of biewos::Scene (geometry.hpp:38-64).

Factories keep the reference's names (Scene.half_space, Scene.sphere,
geometry.cpp:34-92) and add the BASELINE geometries the reference lacks
(Scene.box, Scene.box_with_cavities). Dirichlet data must be one of the closed
forms below: the reference's std::function phi (geometry.hpp:34) cannot run
on a device, and an arbitrary Python callable is refused with
ApplicabilityError (there is no CPU fallback).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from enum import IntEnum

import numpy as np

from ._native import BwScene
from .errors import ApplicabilityError, GeometryError


class SceneKind(IntEnum):  # geometry.hpp:11 (+ BOX, BOX_CAVITIES)
    HalfSpace = 0
    PlateSet = 1
    ThinDisk = 2
    Sphere = 3
    Box = 4
    BoxCavities = 5


class DomainSide(IntEnum):  # geometry.hpp:12
    Exterior = 0
    Interior = 1


kExitInfinity = -1  # geometry.hpp:25
kExitFailed = -2    # geometry.hpp:26


# ---- closed-form Dirichlet data (bw_phi_kind) ----
@dataclass(frozen=True)
class Quadratic:
    """u = c + g.x + Qxx x^2 + Qyy y^2 + Qzz z^2 + Qxy xy + Qxz xz + Qyz yz."""
    c: float = 0.0
    g: tuple = (0.0, 0.0, 0.0)
    q: tuple = (0.0, 0.0, 0.0, 0.0, 0.0, 0.0)  # xx, yy, zz, xy, xz, yz
    kind = 1

    def params(self):
        return [self.c, *self.g, *self.q]

    def __call__(self, y):
        y = np.asarray(y, dtype=float)
        x0, x1, x2 = y[..., 0], y[..., 1], y[..., 2]
        q = self.q
        return (self.c + self.g[0] * x0 + self.g[1] * x1 + self.g[2] * x2 + q[0] * x0 * x0
                + q[1] * x1 * x1 + q[2] * x2 * x2 + q[3] * x0 * x1 + q[4] * x0 * x2
                + q[5] * x1 * x2)

    def grad(self, y):
        y = np.asarray(y, dtype=float)
        x0, x1, x2 = y[..., 0], y[..., 1], y[..., 2]
        q = self.q
        return np.stack([self.g[0] + 2 * q[0] * x0 + q[3] * x1 + q[4] * x2,
                         self.g[1] + 2 * q[1] * x1 + q[3] * x0 + q[5] * x2,
                         self.g[2] + 2 * q[2] * x2 + q[4] * x0 + q[5] * x1], axis=-1)


@dataclass(frozen=True)
class ExpSinSin:
    """u = A exp(kx (x - x0)) sin(ky (y - y0)) sin(kz (z - z0))."""
    A: float = 1.0
    k: tuple = (0.0, 0.0, 0.0)
    origin: tuple = (0.0, 0.0, 0.0)
    kind = 2

    def params(self):
        return [self.A, *self.k, *self.origin]

    def __call__(self, y):
        y = np.asarray(y, dtype=float) - np.asarray(self.origin)
        return (self.A * np.exp(self.k[0] * y[..., 0]) * np.sin(self.k[1] * y[..., 1])
                * np.sin(self.k[2] * y[..., 2]))

    def grad(self, y):
        y = np.asarray(y, dtype=float) - np.asarray(self.origin)
        kx, ky, kz = self.k
        e = self.A * np.exp(kx * y[..., 0])
        sy, cy = np.sin(ky * y[..., 1]), np.cos(ky * y[..., 1])
        sz, cz = np.sin(kz * y[..., 2]), np.cos(kz * y[..., 2])
        return np.stack([kx * e * sy * sz, ky * e * cy * sz, kz * e * sy * cz], axis=-1)


@dataclass(frozen=True)
class SinSin:
    """u = A sin(kx (x - x0)) sin(ky (y - y0)) (runner.cpp:318-324, four_plates_sine)."""
    A: float = 1.0
    k: tuple = (1.0, 1.0)
    origin: tuple = (0.0, 0.0)
    kind = 4

    def params(self):
        return [self.A, *self.k, *self.origin]

    def __call__(self, y):
        y = np.asarray(y, dtype=float)
        return (self.A * np.sin(self.k[0] * (y[..., 0] - self.origin[0]))
                * np.sin(self.k[1] * (y[..., 1] - self.origin[1])))


@dataclass(frozen=True)
class PointSource:
    """u = c + q / |x - s|."""
    q: float = 1.0
    s: tuple = (0.0, 0.0, 0.0)
    c: float = 0.0
    kind = 3

    def params(self):
        return [self.q, *self.s, self.c]

    def __call__(self, y):
        r = np.asarray(y, dtype=float) - np.asarray(self.s)
        return self.c + self.q / np.linalg.norm(r, axis=-1)

    def grad(self, y):
        r = np.asarray(y, dtype=float) - np.asarray(self.s)
        d = np.linalg.norm(r, axis=-1)
        return -self.q * r / (d ** 3)[..., None]


@dataclass
class Scene:
    kind: SceneKind = SceneKind.HalfSpace
    side: DomainSide = DomainSide.Exterior
    plane_z: float = 0.0
    sphere_radius: float = 0.0
    box_lo: tuple = (0.0, 0.0, 0.0)
    box_hi: tuple = (0.0, 0.0, 0.0)
    cavities: np.ndarray | None = None  # n x 4 (cx, cy, cz, r)
    plates: np.ndarray | None = None    # n x 4 (x0, x1, y0, y1) on z = 0 (geometry.hpp:14-18)
    disk_radius: float = 0.0
    piecewise_const: bool = False
    feature_potential: list = field(default_factory=list)
    dirichlet: object = None

    # ---- factories (geometry.cpp:34-92) ----
    @staticmethod
    def half_space(plane_z: float, phi) -> "Scene":
        return Scene(kind=SceneKind.HalfSpace, plane_z=plane_z, dirichlet=phi)

    @staticmethod
    def plate_set(plates, phi=None) -> "Scene":
        """plates: n x 5 (x0, x1, y0, y1, potential) -> piecewise constant data
        (geometry.cpp:42-50), or n x 4 plus a closed-form phi (:52-59)."""
        P = np.asarray(plates, dtype=np.float64)
        s = Scene(kind=SceneKind.PlateSet, plates=np.ascontiguousarray(P[:, :4]))
        if phi is None:
            s.piecewise_const, s.feature_potential = True, [float(v) for v in P[:, 4]]
        else:
            s.dirichlet = phi
        return s

    @staticmethod
    def four_plates(potentials) -> "Scene":  # geometry.cpp:61-64, quadrants I..IV
        v = list(potentials)
        return Scene.plate_set([[0, 1, 0, 1, v[0]], [-1, 0, 0, 1, v[1]], [-1, 0, -1, 0, v[2]],
                                [0, 1, -1, 0, v[3]]])

    @staticmethod
    def thin_disk(radius: float, potential: float) -> "Scene":  # geometry.cpp:66-73
        return Scene(kind=SceneKind.ThinDisk, disk_radius=float(radius), piecewise_const=True,
                     feature_potential=[float(potential)])

    @staticmethod
    def sphere(radius: float, side: DomainSide, phi) -> "Scene":
        if isinstance(phi, (int, float)):
            return Scene(kind=SceneKind.Sphere, sphere_radius=radius, side=side,
                         piecewise_const=True, feature_potential=[float(phi)])
        return Scene(kind=SceneKind.Sphere, sphere_radius=radius, side=side, dirichlet=phi)

    @staticmethod
    def box(lo, hi, phi) -> "Scene":
        s = Scene(kind=SceneKind.Box, side=DomainSide.Interior, box_lo=tuple(map(float, lo)),
                  box_hi=tuple(map(float, hi)))
        if isinstance(phi, (list, tuple)) and len(phi) == 6:
            s.piecewise_const, s.feature_potential = True, [float(v) for v in phi]
        else:
            s.dirichlet = phi
        return s

    @staticmethod
    def box_with_cavities(lo, hi, cavities, phi) -> "Scene":
        cav = np.ascontiguousarray(np.asarray(cavities, dtype=np.float64).reshape(-1, 4))
        if len(cav) > 1024:
            raise GeometryError("at most 1024 cavities")
        return Scene(kind=SceneKind.BoxCavities, side=DomainSide.Interior,
                     box_lo=tuple(map(float, lo)), box_hi=tuple(map(float, hi)), cavities=cav,
                     dirichlet=phi)

    def feature_count(self) -> int:
        if self.kind == SceneKind.Box:
            return 6
        if self.kind == SceneKind.BoxCavities:
            return 6 + len(self.cavities)
        if self.kind == SceneKind.PlateSet:
            return len(self.plates)
        return 1

    def phi(self, y, feature=None):
        """Dirichlet data at on-boundary points y (host evaluation for drivers/tests)."""
        if self.piecewise_const:
            return np.asarray(self.feature_potential)[feature]
        return self.dirichlet(y)

    def to_c(self) -> BwScene:
        """bw_scene image. The returned struct keeps its arrays alive."""
        s = BwScene()
        s.kind = int(self.kind)
        s.side = int(self.side)
        s.plane_z = self.plane_z
        s.sphere_radius = self.sphere_radius
        for k in range(3):
            s.box_lo[k] = self.box_lo[k]
            s.box_hi[k] = self.box_hi[k]
        keep = []
        if self.kind == SceneKind.BoxCavities:
            cav = np.ascontiguousarray(self.cavities, dtype=np.float64)
            keep.append(cav)
            s.n_cavities = len(cav)
            s.cavities = cav.ctypes.data_as(C.POINTER(C.c_double))
        if self.kind == SceneKind.PlateSet:
            pl = np.ascontiguousarray(self.plates, dtype=np.float64)
            keep.append(pl)
            s.n_plates = len(pl)
            s.plates = pl.ctypes.data_as(C.POINTER(C.c_double))
        s.disk_radius = self.disk_radius
        if self.piecewise_const:
            fp = np.ascontiguousarray(self.feature_potential, dtype=np.float64)
            if len(fp) != self.feature_count():
                raise GeometryError("feature_potential needs one value per feature")
            keep.append(fp)
            s.phi_kind = 0
            s.feature_potential = fp.ctypes.data_as(C.POINTER(C.c_double))
        else:
            phi = self.dirichlet
            if not hasattr(phi, "kind") or not hasattr(phi, "params"):
                raise ApplicabilityError(
                    "Dirichlet data must be a closed form (Quadratic, ExpSinSin, PointSource) "
                    "to run on the device; there is no CPU fallback")
            s.phi_kind = int(phi.kind)
            for i, v in enumerate(phi.params()):
                s.phi[i] = float(v)
        s._keep = keep  # lifetime of the pointed-to arrays
        return s
