"""Last-passage estimator on the B200 (the reference's last_passage.hpp/.cpp,
next-row f3): estimate_lp(scene, frame, n_paths, cfg, allow_general_data)."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _native as N


class BwLpResult(C.Structure):
    _fields_ = [("sigma_lp", C.c_double), ("std_error", C.c_double), ("n_paths", C.c_int64),
                ("n_infinity", C.c_int64), ("n_failed", C.c_int64)]


@dataclass
class LastPassageResult:  # last_passage.hpp:10-17
    sigma_lp: float = 0.0
    std_error: float = 0.0
    n_paths: int = 0
    n_infinity: int = 0
    n_failed: int = 0
    feature_counts: list = field(default_factory=list)


def estimate_lp(scene, frame, n_paths: int, cfg, allow_general_data: bool = False,
                device=None) -> LastPassageResult:
    """last_passage.cpp:53-112 on the device (paths of stream domain 1)."""
    ctx = N.context(device)
    c = np.ascontiguousarray(frame.center, np.float64)
    ax = np.ascontiguousarray(frame.axis, np.float64)
    counts = np.zeros(scene.feature_count(), np.int64)
    out = BwLpResult()
    sc, cf = scene.to_c(), cfg.to_c()
    ctx.check(ctx.lib.bw_estimate_lp(ctx.handle, C.byref(sc), C.byref(cf), N.ptr(c),
                                     float(frame.radius), N.ptr(ax), int(n_paths),
                                     int(bool(allow_general_data)), C.byref(out),
                                     N.ptr(counts)))
    return LastPassageResult(out.sigma_lp, out.std_error, out.n_paths, out.n_infinity,
                             out.n_failed, counts.tolist())
