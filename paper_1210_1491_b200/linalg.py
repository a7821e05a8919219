"""Batched dense LU solve (K2) — the per-patch Eigen::PartialPivLU + solve +
residual gate of patch_solver.cpp:314-324, for many patches in one launch."""
from __future__ import annotations

import numpy as np

from . import _native as N
from .errors import SolverError


def lu_solve_batched(A, B, tol: float = 1e-10, raise_on_fail: bool = True, device=None):
    """A: (n, m, m), B: (n, nrhs, m) or (n, m). Returns (X, resid, info).

    resid[s] = ||A x0 - b0|| / max(||b0||, 1e-300); info 0 ok, 1 singular,
    2 residual > tol / non-finite. With raise_on_fail a failing system raises
    SolverError (patch_solver.cpp:319-323)."""
    ctx = N.context(device)
    A = np.ascontiguousarray(np.asarray(A, dtype=np.float64))
    B = np.asarray(B, dtype=np.float64)
    squeeze = B.ndim == 2
    if squeeze:
        B = B[:, None, :]
    B = np.ascontiguousarray(B)
    n, m, _ = A.shape
    nrhs = B.shape[1]
    X = np.empty_like(B)
    resid = np.empty(n, np.float64)
    info = np.empty(n, np.int32)
    rc = ctx.lib.bw_lu_solve_batched(ctx.handle, m, n, N.ptr(A), N.ptr(B), nrhs, tol, N.ptr(X),
                                     N.ptr(resid), N.ptr(info))
    if rc == 10 and not raise_on_fail:
        rc = 0
    try:
        ctx.check(rc)
    except SolverError as e:
        e.X, e.resid, e.info = X, resid, info
        raise
    return (X[:, 0, :] if squeeze else X), resid, info
