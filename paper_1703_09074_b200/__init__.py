"""B200-native randomized CP decomposition (arXiv 1703.09074) hot path.

The GPU library (csrc/, built to librcpg.so) implements the reference's
rcp::decompose(randomized = true, method = als) path; `rcp` mirrors the
reference's C++ API on top of its C ABI (include/rcpg.h).
"""
from .rcp import (  # noqa: F401
    ALS, BCD, COMPRESS, EIGENVECTORS, FACTORS, GAUSSIAN, INIT, LU, NOISE, QR, RANDOM, UNIFORM,
    CompressConfig, CompressionResult, Context, CudaError, DecomposeConfig, DeviceTensor, FitTrace, Kruskal,
    ModeBasis, SolverError, als_solve, compress, decompose, default_context, derive_seed, plu_basis, recover,
    relative_error,
    sketch_matrix, stream_id, stream_pass, thin_qr, comm_unique_id, comm_init_loopback, slab_range,
    BoundReport, projection_residual, theorem_bound, validate_bound, TRIAL,
)
from ._lib import LIB_PATH, build  # noqa: F401

__all__ = [
    "CompressConfig", "DecomposeConfig", "Kruskal", "FitTrace", "SolverError", "ModeBasis", "CompressionResult",
    "compress", "decompose", "als_solve", "recover", "relative_error", "sketch_matrix", "stream_pass", "comm_unique_id", "comm_init_loopback", "slab_range", "plu_basis", "thin_qr", "DeviceTensor", "Context",
    "BoundReport", "projection_residual", "theorem_bound", "validate_bound",
]
