"""ctypes binding of the C-ABI (include/biewos_b200.h) and the error mapping.

The library is the product: there is no Python or CPU fallback. If the shared
object is missing or no B200 is visible, every call raises.
"""
from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

import numpy as np

from .errors import STATUS_TO_EXC, Error

LIB_PATH = Path(os.environ.get("BW_LIB_PATH") or
                Path(__file__).resolve().parent / "_lib" / "libbiewos_b200.so")

# ---- structs (must match include/biewos_b200.h) ----


class BwScene(C.Structure):
    _fields_ = [
        ("kind", C.c_int32),
        ("side", C.c_int32),
        ("plane_z", C.c_double),
        ("sphere_radius", C.c_double),
        ("box_lo", C.c_double * 3),
        ("box_hi", C.c_double * 3),
        ("n_cavities", C.c_int32),
        ("phi_kind", C.c_int32),
        ("cavities", C.POINTER(C.c_double)),
        ("feature_potential", C.POINTER(C.c_double)),
        ("phi", C.c_double * 16),
        ("n_plates", C.c_int32),
        ("reserved", C.c_int32),
        ("plates", C.POINTER(C.c_double)),
        ("disk_radius", C.c_double),
    ]


class BwWosConfig(C.Structure):
    _fields_ = [
        ("eps_shell", C.c_double),
        ("trunc_radius", C.c_double),
        ("n_paths", C.c_int64),
        ("max_steps", C.c_int32),
        ("rng", C.c_int32),
        ("seed", C.c_uint64),
        ("eps_rel", C.c_double),
    ]


# numpy view of bw_estimate / biewos::Estimate (wos.hpp:22-29)
ESTIMATE_DTYPE = np.dtype([("mean", "<f8"), ("variance", "<f8"), ("n", "<i8"),
                           ("n_infinity", "<i8"), ("n_failed", "<i8")])

EXPORTS = [
    "bw_abi_version", "bw_init", "bw_finalize", "bw_last_error", "bw_launch_count", "bw_set_stream",
    "bw_synchronize", "bw_device_info", "bw_philox_blocks", "bw_walk", "bw_wos_estimate",
    "bw_nearest_feature", "bw_distance_to_boundary", "bw_classify_exit",
    "bw_wos_estimate_d", "bw_wos_patch_nodes", "bw_wos_patch_nodes_d", "bw_potential",
    "bw_potential_d", "bw_lu_solve_batched", "bw_lu_solve_batched_d", "bw_measure_fp64_peak",
    "bw_dtn_assemble_d", "bw_dtn_point_values_d", "bw_dtn_solve", "bw_dtn_solve_d",
    "bw_dtn_neumann", "bw_dtn_neumann_d", "bw_solve_patch",
    "bw_point_formula", "bw_point_formula_d", "bw_estimate_lp", "bw_diag_sqrt",
    "bw_diag_wos_stream", "bw_philox4x32_blocks", "bw_diag_wos_stream32", "bw_diag_stat_math", "bw_dtn_class_cache_hits",
    "bw_group_init", "bw_group_finalize", "bw_group_size", "bw_group_context",
    "bw_group_last_error", "bw_group_launch_count", "bw_group_dtn_solve", "bw_group_pipeline",
]

_P = C.c_void_p
_lib = None
_lock = threading.Lock()


def load_library() -> C.CDLL:
    """Load libbiewos_b200.so (build it first with paper_1210_1491_b200.build)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_1210_1491_b200.build` "
                              "(no CPU fallback exists)")
        lib = C.CDLL(str(LIB_PATH))
        st = C.c_int
        lib.bw_abi_version.restype = C.c_int32
        lib.bw_init.argtypes = [C.c_int, C.POINTER(_P)]
        lib.bw_init.restype = st
        lib.bw_finalize.argtypes = [_P]
        lib.bw_finalize.restype = st
        lib.bw_launch_count.argtypes = [_P, C.POINTER(C.c_uint64)]
        lib.bw_launch_count.restype = st
        lib.bw_last_error.argtypes = [_P]
        lib.bw_last_error.restype = C.c_char_p
        lib.bw_set_stream.argtypes = [_P, _P]
        lib.bw_set_stream.restype = st
        lib.bw_synchronize.argtypes = [_P]
        lib.bw_synchronize.restype = st
        lib.bw_device_info.argtypes = [_P, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
        lib.bw_device_info.restype = st
        lib.bw_philox_blocks.argtypes = [_P, _P, _P, C.c_int64, _P]
        lib.bw_philox_blocks.restype = st
        lib.bw_philox4x32_blocks.argtypes = [_P, _P, _P, C.c_int64, _P]
        lib.bw_philox4x32_blocks.restype = st
        lib.bw_diag_wos_stream32.argtypes = [_P, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int32, _P]
        lib.bw_diag_wos_stream32.restype = st
        sc, cf = C.POINTER(BwScene), C.POINTER(BwWosConfig)
        lib.bw_walk.argtypes = [_P, sc, cf, _P, C.c_int64, _P, _P, _P, _P, _P]
        lib.bw_walk.restype = st
        lib.bw_nearest_feature.argtypes = [_P, sc, _P, C.c_int64, _P, _P, _P]
        lib.bw_nearest_feature.restype = st
        lib.bw_distance_to_boundary.argtypes = [_P, sc, _P, C.c_int64, _P, _P]
        lib.bw_distance_to_boundary.restype = st
        lib.bw_classify_exit.argtypes = [_P, sc, _P, C.c_int64, C.c_double, C.c_double, _P, _P]
        lib.bw_classify_exit.restype = st
        lib.bw_walk.restype = st
        for fn in (lib.bw_wos_estimate, lib.bw_wos_estimate_d):
            fn.argtypes = [_P, sc, cf, _P, C.c_int64, C.c_uint64, _P, _P]
            fn.restype = st
        for fn in (lib.bw_wos_patch_nodes, lib.bw_wos_patch_nodes_d):
            fn.argtypes = [_P, sc, cf, _P, _P, _P, _P, _P, C.c_int64, _P, C.c_int32,
                           C.c_int32, C.c_uint64, _P, _P]
            fn.restype = st
        lib.bw_potential.argtypes = [_P, _P, C.c_int64, _P, C.c_int64, _P, _P]
        lib.bw_potential.restype = st
        lib.bw_potential_d.argtypes = [_P, _P, C.c_int64, _P, C.c_int64, _P, _P,
                                       C.POINTER(C.c_int64)]
        lib.bw_potential_d.restype = st
        for fn in (lib.bw_lu_solve_batched, lib.bw_lu_solve_batched_d):
            fn.argtypes = [_P, C.c_int32, C.c_int64, _P, _P, C.c_int32, C.c_double, _P, _P, _P]
            fn.restype = st
        lib.bw_dtn_assemble_d.argtypes = [_P, sc, _P, C.c_int64, _P, _P, C.c_int32, C.c_int32,
                                          _P, _P, _P, _P, _P, _P]
        lib.bw_dtn_assemble_d.restype = st
        lib.bw_dtn_point_values_d.argtypes = [_P, C.c_int64, _P, _P, _P, _P, _P, _P, _P, _P]
        lib.bw_dtn_point_values_d.restype = st
        for fn in (lib.bw_dtn_solve, lib.bw_dtn_solve_d):
            fn.argtypes = [_P, sc, cf, _P, _P, _P, C.c_int64, _P, _P, C.c_int32, C.c_int32,
                           C.c_uint64, _P, _P, _P, _P, _P]
            fn.restype = st
        lib.bw_solve_patch.argtypes = [_P, sc, _P, _P, C.c_int64, _P, _P, C.c_int32, C.c_int32, _P,
                                       _P, _P, _P, _P]
        lib.bw_solve_patch.restype = st
        for fn in (lib.bw_dtn_neumann, lib.bw_dtn_neumann_d):
            fn.argtypes = [_P, sc, _P, _P, C.c_int64, _P, _P, C.c_int32, C.c_int32, _P,
                           C.c_int32, _P, _P, _P]
            fn.restype = st
        for fn in (lib.bw_point_formula, lib.bw_point_formula_d):
            fn.argtypes = [_P, sc, _P, C.c_int64, _P, _P, C.c_int32, _P, _P, C.c_int32, _P, _P,
                           _P, _P]
            fn.restype = st
        lib.bw_estimate_lp.argtypes = [_P, sc, cf, _P, C.c_double, _P, C.c_int64, C.c_int32, _P,
                                       _P]
        lib.bw_estimate_lp.restype = st
        lib.bw_measure_fp64_peak.argtypes = [_P, C.POINTER(C.c_double), C.POINTER(C.c_double)]
        lib.bw_measure_fp64_peak.restype = st
        if hasattr(lib, "bw_diag_sqrt"):  # diagnostic; absent from older A/B builds
            lib.bw_diag_sqrt.argtypes = [_P, _P, C.c_int64, _P, _P]
            lib.bw_diag_sqrt.restype = st
        if hasattr(lib, "bw_dtn_class_cache_hits"):
            lib.bw_dtn_class_cache_hits.argtypes = [_P, _P]
            lib.bw_dtn_class_cache_hits.restype = st
        if hasattr(lib, "bw_diag_stat_math"):
            lib.bw_diag_stat_math.argtypes = [_P, _P, _P, C.c_int64, _P, _P, _P]
            lib.bw_diag_stat_math.restype = st
        if hasattr(lib, "bw_diag_wos_stream"):
            lib.bw_diag_wos_stream.argtypes = [_P, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int32, _P]
            lib.bw_diag_wos_stream.restype = st
        lib.bw_group_init.argtypes = [C.c_int32, _P, C.POINTER(_P)]
        lib.bw_group_init.restype = st
        lib.bw_group_finalize.argtypes = [_P]
        lib.bw_group_finalize.restype = st
        lib.bw_group_size.argtypes = [_P, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
        lib.bw_group_size.restype = st
        lib.bw_group_context.argtypes = [_P, C.c_int32]
        lib.bw_group_context.restype = _P
        lib.bw_group_last_error.argtypes = [_P]
        lib.bw_group_last_error.restype = C.c_char_p
        lib.bw_group_launch_count.argtypes = [_P, C.POINTER(C.c_uint64)]
        lib.bw_group_launch_count.restype = st
        lib.bw_group_dtn_solve.argtypes = [_P, sc, cf, _P, _P, _P, C.c_int64, _P, _P, C.c_int32,
                                           C.c_int32, C.c_uint64, _P, _P, _P,
                                           C.POINTER(C.c_int64), C.POINTER(C.c_double)]
        lib.bw_group_dtn_solve.restype = st
        lib.bw_group_pipeline.argtypes = [_P, sc, cf, _P, _P, C.c_int64, _P, _P, C.c_int32,
                                          C.c_int32, C.c_uint64, _P, _P, _P, C.c_int64, _P, _P,
                                          _P, _P, _P, C.POINTER(C.c_int64), _P]
        lib.bw_group_pipeline.restype = st
        _lib = lib
        return lib


class Context:
    """One bw_ctx per (process, device): owns device scratch and the stream."""

    def __init__(self, device: int = 0):
        self.lib = load_library()
        self.device = device
        h = _P()
        rc = self.lib.bw_init(device, C.byref(h))
        if rc != 0:
            raise STATUS_TO_EXC.get(rc, Error)(
                f"bw_init(device={device}) failed with status {rc}: no usable sm_100 device "
                "(there is no CPU fallback)")
        self.handle = h

    def check(self, rc: int) -> None:
        if rc != 0:
            msg = self.lib.bw_last_error(self.handle).decode() or f"status {rc}"
            raise STATUS_TO_EXC.get(rc, Error)(msg)

    def set_stream(self, stream_handle: int | None) -> None:
        self.check(self.lib.bw_set_stream(self.handle, stream_handle or None))

    def device_info(self) -> tuple[int, int]:
        sm, clk = C.c_int32(), C.c_int32()
        self.check(self.lib.bw_device_info(self.handle, C.byref(sm), C.byref(clk)))
        return sm.value, clk.value

    def launch_count(self) -> int:
        """Kernels this context has launched so far (bw_launch_count)."""
        n = C.c_uint64()
        self.check(self.lib.bw_launch_count(self.handle, C.byref(n)))
        return int(n.value)

    def fp64_peak(self) -> tuple[float, float]:
        """Measured DFMA throughput (TFLOP/s) and the kernel time (ms)."""
        tf, ms = C.c_double(), C.c_double()
        self.check(self.lib.bw_measure_fp64_peak(self.handle, C.byref(tf), C.byref(ms)))
        return tf.value, ms.value

    def close(self) -> None:
        if getattr(self, "handle", None):
            self.lib.bw_finalize(self.handle)
            self.handle = None


_contexts: dict[int, Context] = {}


def context(device: int | None = None) -> Context:
    """The process-wide context of `device` (default: torch's current device)."""
    if device is None:
        device = _current_device()
    with _lock:
        ctx = _contexts.get(device)
    if ctx is None:
        ctx = Context(device)
        with _lock:
            _contexts[device] = ctx
    return ctx


def _current_device() -> int:
    try:
        import torch

        if torch.cuda.is_available():
            return torch.cuda.current_device()
    except Exception:  # torch is plumbing only; its absence is not an error here
        pass
    return 0


def ptr(a: np.ndarray | None) -> int | None:
    return None if a is None else a.ctypes.data


def as_c(a, dtype, shape_last: int | None = None) -> np.ndarray:
    """Contiguous numpy copy/view with the given dtype (and trailing dim)."""
    arr = np.ascontiguousarray(np.asarray(a, dtype=dtype))
    if shape_last is not None:
        arr = arr.reshape(-1, shape_last)
    return arr
