"""Exception classes of the reference (proj/include/biewos/types.hpp:22-45),
keyed by the bw_status codes of include/biewos_b200.h."""


class Error(RuntimeError):
    """biewos::Error (types.hpp:22)."""


class DomainError(Error):
    """point on or outside the solution domain (types.hpp:25)"""


class ClassificationError(Error):
    """exit point could not be matched to a boundary feature (types.hpp:27)"""


class SingularityError(Error):
    """coincident kernel arguments (types.hpp:29)"""


class GeometryError(Error):
    """argument off the surface it must lie on (types.hpp:31)"""


class ReliabilityError(Error):
    """too many failed paths / unusable statistics (types.hpp:33)"""


class ApplicabilityError(Error):
    """estimator used outside its validity class (types.hpp:35)"""


class ExtrapolationError(Error):
    """interpolation target outside grid coverage (types.hpp:37)"""


class NearFieldError(Error):
    """evaluation point too close to a panel (types.hpp:39)"""


class ConfigError(Error):
    """config file problems (types.hpp:41)"""


class SolverError(Error):
    """linear solve failed or residual out of contract (types.hpp:43)"""


class CudaError(Error):
    """device/runtime failure; the product has no CPU fallback"""


STATUS_TO_EXC = {
    1: DomainError, 2: ClassificationError, 3: SingularityError, 4: GeometryError,
    5: ReliabilityError, 6: ApplicabilityError, 7: ExtrapolationError, 8: NearFieldError,
    9: ConfigError, 10: SolverError, 64: CudaError, 65: ValueError,
}
