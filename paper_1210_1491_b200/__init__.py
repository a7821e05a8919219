"""paper_1210_1491_b200 — B200-native BIE-WOS / local-DtN hot path.

The walk-on-spheres estimator, batched per-patch LU and the potential sum of
arXiv 1210.1491's local Dirichlet-to-Neumann method, as hand-written sm_100a
fp64 kernels behind a C-ABI (include/biewos_b200.h). This package is the host
mirror of the reference's C++ API (proj/include/biewos/*.hpp): same names,
argument meaning and exception classes. There is no CPU fallback.
"""
from .errors import (ApplicabilityError, ClassificationError, DomainError, Error,
                     ExtrapolationError, GeometryError, NearFieldError, ReliabilityError,
                     SingularityError, SolverError)
from .group import DeviceGroup, PipelineResult
from .field_eval import BoundaryData, BoundaryPanel, evaluate, evaluate_batch
from .geometry import (DomainSide, ExpSinSin, PointSource, Quadratic, Scene, SceneKind, SinSin,
                       kExitFailed, kExitInfinity)
from .last_passage import LastPassageResult, estimate_lp
from .linalg import lu_solve_batched
from .point_solver import HemisphereFrame, PointNeumannResult, solve_point, solve_points
from .wos import (ESTIMATE_DTYPE, DistanceQuery, Estimate, ExitRecord, WosConfig,
                  classify_exit, classify_exit_batch, distance_to_boundary, estimate_u,
                  estimate_u_batch, estimate_u_batch_full, exit_value, nearest_feature,
                  nearest_feature_batch, walk, walk_batch, wos_sampler)

__all__ = [
    "ApplicabilityError", "ClassificationError", "DomainError", "Error", "ExtrapolationError",
    "GeometryError", "NearFieldError", "ReliabilityError", "SingularityError", "SolverError",
    "BoundaryData", "BoundaryPanel", "evaluate", "evaluate_batch", "DomainSide", "ExpSinSin",
    "PointSource", "Quadratic", "Scene", "SceneKind", "SinSin", "kExitFailed", "kExitInfinity",
    "lu_solve_batched", "ESTIMATE_DTYPE", "Estimate", "ExitRecord", "WosConfig", "estimate_u",
    "estimate_u_batch", "estimate_u_batch_full", "exit_value", "walk", "walk_batch",
    "DistanceQuery", "classify_exit", "classify_exit_batch", "distance_to_boundary",
    "nearest_feature", "nearest_feature_batch",
    "wos_sampler", "DeviceGroup", "PipelineResult",
]
