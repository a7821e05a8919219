"""Several GPUs of one process behind the C-ABI (bw_group_*): the DtN path and
the config-5 pipeline sharded over devices inside the library, with one NCCL
all-gather of the panel records before the potential sum.

The reference runs estimate_u_batch on `workers` threads with results
independent of the worker count (wos.hpp:19,43-44; parallel.hpp:14-40); a
DeviceGroup gives the same guarantee across GPUs: boundary point b runs on
device b mod n with its global stream ids, and the results are bitwise those
of the single-device calls for any n. (torchrun + torch.distributed is the
other multi-GPU form, one process per GPU: distributed.py, pipeline.py.)
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .dtn import PATCH_DTYPE, DtnConfig, DtnResult
from .errors import STATUS_TO_EXC, Error


@dataclass
class PipelineResult:
    u: np.ndarray          # potential at the targets (NaN where near-field)
    near: np.ndarray       # near-field flags
    dtn: DtnResult         # Neumann data of every boundary point
    walk_steps: int
    phase_ms: dict         # max over devices: dtn, exchange, potential


class DeviceGroup:
    """bw_group over `devices` (distinct ids: NCCL; a repeated id stands one GPU
    in for several ranks with device-to-device copies — tests only)."""

    def __init__(self, devices):
        self.devices = [int(d) for d in devices]
        if len(set(self.devices)) == len(self.devices) > 0:
            # the library dlopens NCCL and reuses one already in the process:
            # make it torch's (newer) one when torch is around
            try:
                import torch  # noqa: F401
            except Exception:
                pass
        self.lib = N.load_library()
        ids = np.asarray(self.devices, np.int32)
        h = C.c_void_p()
        rc = self.lib.bw_group_init(len(ids), ids.ctypes.data, C.byref(h))
        if rc != 0:
            raise STATUS_TO_EXC.get(rc, Error)(f"bw_group_init({self.devices}) failed: status {rc}")
        self.handle = h
        n, nccl = C.c_int32(), C.c_int32()
        self.check(self.lib.bw_group_size(self.handle, C.byref(n), C.byref(nccl)))
        self.size, self.uses_nccl = n.value, bool(nccl.value)

    def check(self, rc: int) -> None:
        if rc != 0:
            msg = self.lib.bw_group_last_error(self.handle).decode() or f"status {rc}"
            raise STATUS_TO_EXC.get(rc, Error)(msg)

    def launch_count(self) -> int:
        n = C.c_uint64()
        self.check(self.lib.bw_group_launch_count(self.handle, C.byref(n)))
        return int(n.value)

    def close(self) -> None:
        if getattr(self, "handle", None):
            self.lib.bw_group_finalize(self.handle)
            self.handle = None

    def __del__(self):
        self.close()

    def dtn_solve(self, scene, wos_cfg, patches, local_dirs, weights, dtn_cfg=None, bp_ids=None,
                  point_id_base: int = 0):
        """bw_group_dtn_solve: (DtnResult, walk_steps, device_ms)."""
        dtn_cfg = dtn_cfg or DtnConfig()
        P = np.ascontiguousarray(patches, dtype=PATCH_DTYPE)
        L = np.ascontiguousarray(np.asarray(local_dirs, np.float64))
        if L.ndim == 2:
            L = L[None]
        Wt = np.ascontiguousarray(np.asarray(weights, np.float64).reshape(L.shape[0], L.shape[1]))
        n_bp = len(P)
        ids = None if bp_ids is None else N.as_c(bp_ids, np.int64)
        dudn, err, status = np.empty(n_bp), np.empty(n_bp), np.empty(n_bp, np.int32)
        steps, ms = C.c_int64(), C.c_double()
        sc, wc, dc = scene.to_c(), wos_cfg.to_c(), dtn_cfg.to_c()
        rc = self.lib.bw_group_dtn_solve(self.handle, C.byref(sc), C.byref(wc), C.byref(dc),
                                         P.ctypes.data, N.ptr(ids), n_bp, N.ptr(L), N.ptr(Wt),
                                         L.shape[0], L.shape[1], int(point_id_base), N.ptr(dudn),
                                         N.ptr(err), N.ptr(status), C.byref(steps), C.byref(ms))
        res = DtnResult(dudn, err, status)
        try:
            self.check(rc)
        except Exception as e:
            e.result = res
            raise
        return res, int(steps.value), float(ms.value)

    def pipeline(self, scene, wos_cfg, patches, local_dirs, weights, area, u_bp, targets,
                 dtn_cfg=None, point_id_base: int = 0) -> PipelineResult:
        """bw_group_pipeline: DtN -> NCCL all-gather of the panels -> potential."""
        dtn_cfg = dtn_cfg or DtnConfig()
        P = np.ascontiguousarray(patches, dtype=PATCH_DTYPE)
        L = np.ascontiguousarray(np.asarray(local_dirs, np.float64))
        if L.ndim == 2:
            L = L[None]
        Wt = np.ascontiguousarray(np.asarray(weights, np.float64).reshape(L.shape[0], L.shape[1]))
        n_bp = len(P)
        A = N.as_c(area, np.float64)
        U = N.as_c(u_bp, np.float64)
        T = N.as_c(targets, np.float64, 3)
        n_t = len(T)
        u, near = np.empty(n_t), np.zeros(n_t, np.uint8)
        dudn, err, status = np.empty(n_bp), np.empty(n_bp), np.empty(n_bp, np.int32)
        steps, ph = C.c_int64(), np.zeros(3)
        sc, wc, dc = scene.to_c(), wos_cfg.to_c(), dtn_cfg.to_c()
        rc = self.lib.bw_group_pipeline(self.handle, C.byref(sc), C.byref(wc), C.byref(dc),
                                        P.ctypes.data, n_bp, N.ptr(L), N.ptr(Wt), L.shape[0],
                                        L.shape[1], int(point_id_base), N.ptr(A), N.ptr(U),
                                        N.ptr(T), n_t, N.ptr(u), N.ptr(near), N.ptr(dudn),
                                        N.ptr(err), N.ptr(status), C.byref(steps), N.ptr(ph))
        res = PipelineResult(u, near.astype(bool), DtnResult(dudn, err, status),
                             int(steps.value), dict(zip(("dtn", "exchange", "potential"), ph)))
        try:
            self.check(rc)
        except Exception as e:
            e.result = res
            raise
        return res
