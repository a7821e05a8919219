"""ctypes bindings of the TEST ORACLE (oracle/_build/liboracle.so, the C
restatement) and of the reference itself (oracle/_ref/libbiewos_ref.so, the
reference's own sources compiled by oracle/Makefile). Test infrastructure only.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
ORACLE_SO = ROOT / "oracle" / "_build" / "liboracle.so"
REF_SO = ROOT / "oracle" / "_ref" / "libbiewos_ref.so"

ESTIMATE_DTYPE = np.dtype([("mean", "<f8"), ("variance", "<f8"), ("n", "<i8"),
                           ("n_infinity", "<i8"), ("n_failed", "<i8")])
_P = C.c_void_p


def _build_oracle():
    if not ORACLE_SO.exists():
        subprocess.run(["make", "-C", str(ROOT / "oracle")], check=True, capture_output=True)


def oracle() -> C.CDLL:
    _build_oracle()
    lib = C.CDLL(str(ORACLE_SO))
    lib.or_philox_block.argtypes = [_P, _P, _P]
    lib.or_rng_doubles.argtypes = [C.c_uint64] * 4 + [C.c_int64, _P]
    lib.or_rng_u64s.argtypes = [C.c_uint64] * 4 + [C.c_int64, _P]
    lib.or_philox4x32_blocks.argtypes = [_P, _P, C.c_int64, _P]
    lib.or_rng32_u64s.argtypes = [C.c_uint64] * 3 + [C.c_int64, _P]
    lib.or_rng32_doubles.argtypes = [C.c_uint64] * 3 + [C.c_int64, _P]
    lib.or_nearest_feature.argtypes = [_P, _P, _P]
    lib.or_nearest_feature.restype = C.c_double
    lib.or_in_domain.argtypes = [_P, _P]
    lib.or_walk.argtypes = [_P, _P, _P, C.c_int64, _P, _P, _P, _P, _P]
    lib.or_estimate_u_batch.argtypes = [_P, _P, _P, C.c_int64, C.c_uint64, C.c_int, _P, _P]
    lib.or_patch_nodes.argtypes = [_P, _P, _P, _P, C.c_int64, _P, C.c_int32, _P]
    lib.or_gauss_legendre.argtypes = [C.c_int, _P, _P]
    lib.or_gamma_rule.argtypes = [C.c_int, C.c_int, C.c_double, _P, _P]
    lib.or_fibonacci_sphere.argtypes = [C.c_int64, C.c_double, _P]
    lib.or_potential.argtypes = [_P, C.c_int64, _P, C.c_int64, _P, _P]
    lib.or_potential_ld.argtypes = [_P, C.c_int64, _P, C.c_int64, _P, _P]
    lib.or_lu_solve_batched.argtypes = [C.c_int, C.c_int64, _P, _P, C.c_int, _P, _P, _P]
    lib.or_eval_phi.argtypes = [_P, _P, C.c_int]
    lib.or_eval_phi.restype = C.c_double
    return lib


def ref_available() -> bool:
    if not REF_SO.exists() and Path("/root/reference/proj/src").exists():
        subprocess.run(["make", "-C", str(ROOT / "oracle"), "ref"], capture_output=True)
    return REF_SO.exists()


def ref() -> C.CDLL:
    lib = C.CDLL(str(REF_SO))
    lib.ref_philox_block.argtypes = [_P, _P, _P]
    lib.ref_rng_doubles.argtypes = [C.c_uint64] * 4 + [C.c_int64, _P]
    lib.ref_walk.argtypes = [_P, _P, _P, C.c_int64, _P, _P, _P, _P, _P]
    lib.ref_estimate_u_batch.argtypes = [_P, _P, _P, C.c_int64, C.c_uint64, C.c_int, _P]
    lib.ref_evaluate.argtypes = [_P, C.c_int64, _P, C.c_int64, _P, _P]
    lib.ref_gauss_legendre.argtypes = [C.c_int, _P, _P]
    return lib


def p(a):
    return None if a is None else a.ctypes.data


# ---- convenience wrappers shared by tests/bench ----

def or_eval_phi(lib, scene_c, y, feature=0) -> float:
    return lib.or_eval_phi(C.byref(scene_c), p(np.ascontiguousarray(y, np.float64)), feature)


def or_walk(lib, scene_c, cfg_c, starts, pids, paths):
    starts = np.ascontiguousarray(starts, np.float64).reshape(-1, 3)
    n = len(starts)
    pids = np.ascontiguousarray(np.broadcast_to(np.asarray(pids, np.uint64), (n,)))
    paths = np.ascontiguousarray(np.broadcast_to(np.asarray(paths, np.uint64), (n,)))
    ex = np.empty((n, 3))
    f = np.empty(n, np.int32)
    s = np.empty(n, np.int32)
    st = lib.or_walk(C.byref(scene_c), C.byref(cfg_c), p(starts), n, p(pids), p(paths), p(ex),
                     p(f), p(s))
    return st, ex, f, s


def ref_walk(lib, scene_c, cfg_c, starts, pids, paths):
    starts = np.ascontiguousarray(starts, np.float64).reshape(-1, 3)
    n = len(starts)
    pids = np.ascontiguousarray(np.broadcast_to(np.asarray(pids, np.uint64), (n,)))
    paths = np.ascontiguousarray(np.broadcast_to(np.asarray(paths, np.uint64), (n,)))
    ex = np.empty((n, 3))
    f = np.empty(n, np.int32)
    s = np.empty(n, np.int32)
    st = lib.ref_walk(C.byref(scene_c), C.byref(cfg_c), p(starts), n, p(pids), p(paths), p(ex),
                      p(f), p(s))
    return st, ex, f, s


def or_estimate(lib, scene_c, cfg_c, pts, base=0, workers=None):
    pts = np.ascontiguousarray(pts, np.float64).reshape(-1, 3)
    out = np.zeros(len(pts), ESTIMATE_DTYPE)
    steps = np.zeros(len(pts), np.int64)
    workers = workers or (os.cpu_count() or 1)
    st = lib.or_estimate_u_batch(C.byref(scene_c), C.byref(cfg_c), p(pts), len(pts), base,
                                 workers, out.ctypes.data, p(steps))
    return st, out, steps


def ref_estimate(lib, scene_c, cfg_c, pts, base=0, workers=None):
    pts = np.ascontiguousarray(pts, np.float64).reshape(-1, 3)
    out = np.zeros(len(pts), ESTIMATE_DTYPE)
    workers = workers or (os.cpu_count() or 1)
    st = lib.ref_estimate_u_batch(C.byref(scene_c), C.byref(cfg_c), p(pts), len(pts), base,
                                  workers, out.ctypes.data)
    return st, out


def or_potential(lib, panels, targets, long_double=False):
    panels = np.ascontiguousarray(panels, np.float64).reshape(-1, 9)
    targets = np.ascontiguousarray(targets, np.float64).reshape(-1, 3)
    u = np.empty(len(targets))
    near = np.zeros(len(targets), np.uint8)
    fn = lib.or_potential_ld if long_double else lib.or_potential
    fn(p(panels), len(panels), p(targets), len(targets), p(u), p(near))
    return u, near.astype(bool)


def or_patch_nodes(lib, centers, axes, radii, cls, dirs):
    centers = np.ascontiguousarray(centers, np.float64).reshape(-1, 3)
    axes = np.ascontiguousarray(axes, np.float64).reshape(-1, 3)
    radii = np.ascontiguousarray(np.broadcast_to(np.asarray(radii, np.float64), (len(centers),)))
    dirs = np.ascontiguousarray(dirs, np.float64)
    n_nodes = dirs.shape[-2]
    cls_a = None if cls is None else np.ascontiguousarray(cls, np.int32)
    out = np.empty((len(centers), n_nodes, 3))
    lib.or_patch_nodes(p(centers), p(axes), p(radii), p(cls_a), len(centers), p(dirs), n_nodes,
                       p(out))
    return out


def or_patch_point(lib, scene_c, patch, gy, gw, gu, guv, bands=5, azimuth=6, gauss_polar=20,
                   near_depth=2):
    """CPU oracle of one patch solve: returns (dudn along the INTO-domain axis,
    its est_error average, status)."""
    f = lib.or_solve_patch_point
    f.argtypes = [_P, _P, _P, C.c_int, _P, C.c_double, C.c_double, C.c_int, C.c_int, C.c_int,
                  C.c_int, _P, _P, _P, _P, C.c_int, _P, _P, _P, _P]
    o = np.ascontiguousarray(patch["o"], np.float64)
    ax = np.ascontiguousarray(patch["axis"], np.float64)
    sc = np.ascontiguousarray(patch["sc"], np.float64)
    gy = np.ascontiguousarray(gy, np.float64)
    gw, gu, guv = (np.ascontiguousarray(v, np.float64) for v in (gw, gu, guv))
    d, e = C.c_double(), C.c_double()
    st = f(C.byref(scene_c), p(o), p(ax), int(patch["surf"]), p(sc), float(patch["R"]),
           float(patch["a"]), bands, azimuth, gauss_polar, near_depth, p(gy), p(gw), p(gu),
           p(guv), len(gu), C.byref(d), C.byref(e), None, None)
    return d.value, e.value, st
