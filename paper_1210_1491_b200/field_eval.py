"""Integral-representation potential (field_eval.hpp:12-27) on the B200.

  BoundaryPanel / BoundaryData  field_eval.hpp:12-22
  evaluate(data, x)             field_eval.hpp:27, field_eval.cpp:7-19
  evaluate_batch(panels, X)     additive batch API (many targets, one launch)
Panels are an (n, 9) float64 array {px,py,pz, nx,ny,nz, area, u, dudn}.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _native as N


@dataclass
class BoundaryPanel:
    point: tuple
    normal: tuple
    area: float
    u: float
    dudn: float


@dataclass
class BoundaryData:
    panels: list = field(default_factory=list)

    def as_array(self) -> np.ndarray:
        return panels_array(self.panels)


def panels_array(panels) -> np.ndarray:
    if isinstance(panels, BoundaryData):
        panels = panels.panels
    if isinstance(panels, np.ndarray):
        return N.as_c(panels, np.float64, 9)
    return np.array([[*p.point, *p.normal, p.area, p.u, p.dudn] for p in panels],
                    dtype=np.float64).reshape(-1, 9)


def evaluate_batch(panels, targets, flag_near: bool = True, device=None):
    """u at every target. With flag_near, near-field targets come back NaN with
    near[i] = True; otherwise any near-field target raises NearFieldError
    (field_eval.cpp:12-13). Returns (u, near)."""
    ctx = N.context(device)
    P = panels_array(panels)
    T = N.as_c(targets, np.float64, 3)
    u = np.empty(len(T), np.float64)
    near = np.zeros(len(T), np.uint8) if flag_near else None
    ctx.check(ctx.lib.bw_potential(ctx.handle, N.ptr(P), len(P), N.ptr(T), len(T), N.ptr(u),
                                   N.ptr(near)))
    return u, (near.astype(bool) if near is not None else np.zeros(len(T), bool))


def evaluate(data, x, device=None) -> float:
    """field_eval.cpp:7-19: raises NearFieldError within one panel diameter."""
    u, _ = evaluate_batch(data, np.asarray(x, dtype=np.float64)[None], flag_near=False,
                          device=device)
    return float(u[0])


def evaluate_device(d_panels: int, n_panels: int, d_targets: int, n_t: int, d_u: int,
                    d_near: int | None, stream: int | None = None, device=None) -> int:
    """Device-pointer variant; returns the near-field count."""
    import ctypes as C

    ctx = N.context(device)
    if stream is not None:
        ctx.set_stream(stream)
    cnt = C.c_int64(0)
    ctx.check(ctx.lib.bw_potential_d(ctx.handle, d_panels, n_panels, d_targets, n_t, d_u,
                                     d_near, C.byref(cnt)))
    return cnt.value
