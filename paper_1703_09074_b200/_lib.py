"""ctypes binding of the in-tree CUDA library librcpg.so (include/rcpg.h).

There is no CPU fallback: if the extension is missing or no CUDA device is
present, every compute call raises.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

_HERE = os.path.dirname(os.path.abspath(__file__))
# RCPG_LIB: load another build of the same library (A/B timing of two builds)
LIB_PATH = os.environ.get("RCPG_LIB") or os.path.join(_HERE, "librcpg.so")

RCPG_OK, RCPG_INVALID_ARGUMENT, RCPG_SOLVER_ERROR, RCPG_CUDA_ERROR, RCPG_OOM, RCPG_NCCL_ERROR = range(6)
RCPG_F32, RCPG_F64 = 0, 1


class CompressConfigC(C.Structure):
    """rcpg_compress_config (include/rcpg.h) = rcp::CompressConfig (compress.hpp:23-33)."""
    _fields_ = [
        ("target_rank", C.c_int64),
        ("oversampling", C.c_int64),
        ("power_iterations", C.c_int32),
        ("distribution", C.c_int32),
        ("stabilizer", C.c_int32),
        ("modes_present", C.c_int32),
        ("n_modes", C.c_int64),
        ("modes", C.POINTER(C.c_int64)),
        ("seed", C.c_uint64),
    ]


class DecomposeConfigC(C.Structure):
    """rcpg_decompose_config = rcp::DecomposeConfig (solve.hpp:22-31)."""
    _fields_ = [
        ("rank", C.c_int64),
        ("method", C.c_int32),
        ("randomized", C.c_int32),
        ("compress", CompressConfigC),
        ("tol", C.c_double),
        ("max_iter", C.c_int32),
        ("init", C.c_int32),
        ("seed", C.c_uint64),
    ]


class ResultC(C.Structure):
    _fields_ = [
        ("weights", C.c_void_p),
        ("factors", C.c_void_p),
        ("trace_iteration", C.POINTER(C.c_int32)),
        ("trace_fit", C.POINTER(C.c_double)),
        ("trace_seconds", C.POINTER(C.c_double)),
        ("trace_capacity", C.c_int32),
        ("iterations", C.c_int32),
        ("converged", C.c_int32),
        ("final_relative_error", C.c_double),
    ]


def build(force: bool = False) -> None:
    """Compile librcpg.so for sm_100a in-tree (nvcc, see csrc/Makefile)."""
    args = ["make", "-s", "-j8", "-C", os.path.join(_HERE, "csrc")]
    if force:
        subprocess.run(args[:-2] + ["-C", os.path.join(_HERE, "csrc"), "clean"], check=True)
    subprocess.run(args, check=True)


_lib = None

# every symbol include/rcpg.h declares, with its ctypes signature
_V, _I32, _I64, _U64, _D = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_double
SIGNATURES = {
    "rcpg_create": (_I32, [C.c_int, C.POINTER(C.c_void_p)]),
    "rcpg_destroy": (None, [_V]),
    "rcpg_last_error": (C.c_char_p, [_V]),
    "rcpg_last_error_iteration": (_I32, [_V]),
    "rcpg_version": (C.c_char_p, []),
    "rcpg_tensor_upload": (_I32, [_V, C.c_int, _I32, _V, _V, C.POINTER(C.c_void_p)]),
    "rcpg_tensor_wrap_device": (_I32, [_V, C.c_int, _I32, _V, _V, C.POINTER(C.c_void_p)]),
    "rcpg_tensor_download": (_I32, [_V, _V, _V]),
    "rcpg_tensor_device_ptr": (_V, [_V]),
    "rcpg_tensor_free": (None, [_V]),
    "rcpg_compress": (_I32, [_V, _V, C.POINTER(CompressConfigC), C.POINTER(C.c_void_p)]),
    "rcpg_compressed_order": (_I32, [_V]),
    "rcpg_compressed_shape": (None, [_V, _V]),
    "rcpg_compressed_download": (_I32, [_V, _V, _V]),
    "rcpg_compressed_basis_info": (None, [_V, _I32, _V, _V, _V, _V]),
    "rcpg_compressed_basis_download": (_I32, [_V, _V, _I32, _V]),
    "rcpg_compressed_free": (None, [_V]),
    "rcpg_decompose": (_I32, [_V, _V, C.POINTER(DecomposeConfigC), C.POINTER(ResultC)]),
    "rcpg_decompose_host": (_I32, [_V, C.c_int, _I32, _V, _V, C.POINTER(DecomposeConfigC), C.POINTER(ResultC)]),
    "rcpg_relative_error": (_I32, [_V, _V, _I64, _V, _V, C.POINTER(C.c_double)]),
    "rcpg_recover": (_I32, [_V, C.c_int, _I32, _I64, _V, _V, _V, _V, _V, _V, _V, _V, _V]),
    "rcpg_als_solve": (_I32, [_V, _V, C.POINTER(DecomposeConfigC), C.POINTER(ResultC)]),
    "rcpg_sketch_matrix": (_I32, [_V, C.c_int, _U64, _I64, _I64, _I64, _I32, _V]),
    "rcpg_comm_unique_id": (_I32, [_V]),
    "rcpg_comm_init_nccl": (_I32, [_V, C.c_int32, C.c_int32, _V]),
    "rcpg_comm_init_loopback": (_I32, [_V, C.c_int32]),
    "rcpg_comm_rank": (_I32, [_V, _V, _V]),
    "rcpg_slab_range": (None, [_I64, C.c_int32, C.c_int32, _V, _V]),
    "rcpg_tensor_slab": (_I32, [_V, _V, _I64, _I64, _V]),
    "rcpg_tensor_upload_slab": (_I32, [_V, C.c_int, C.c_int32, _V, _I64, _I64, _V, _V]),
    "rcpg_tensor_slab_mode": (_I32, [_V, _V, C.c_int32, _I64, _I64, _V]),
    "rcpg_tensor_upload_slab_mode": (_I32, [_V, C.c_int, C.c_int32, _V, C.c_int32, _I64, _I64, _V, _V]),
    "rcpg_stream_pass": (_I32, [_V, C.c_int, C.c_int32, _I64, _I64, _I64, _I64, _V, _V, _V]),
    "rcpg_plu_basis": (_I32, [_V, C.c_int, _I64, _I64, _V, _V]),
    "rcpg_thin_qr": (_I32, [_V, C.c_int, _I64, _I64, _V, _V, _V]),
    "rcpg_pass_timings": (_I32, [_V, C.c_char_p, _I32, _V, _V, _I32]),
    "rcpg_pass_offsets": (_I32, [_V, _V, _I32]),
    "rcpg_kernel_launches": (_I64, [_V]),
    "rcpg_synth": (_I32, [_V, C.c_int, _I32, _V, _I64, _V, _V, _D, _U64, C.POINTER(C.c_void_p)]),
    "rcpg_synchronize": (_I32, [_V]),
    "rcpg_set_option": (_I32, [_V, C.c_char_p, _I64]),
    "rcpg_projection_residual": (_I32, [_V, _V, _V, C.POINTER(C.c_double)]),
    "rcpg_theorem_bound": (_I32, [_V, _V, _I64, _I64, _V, C.POINTER(C.c_double)]),
    "rcpg_projection_residual_bases": (_I32, [_V, _V, _V, _V, _V, C.POINTER(C.c_double)]),
    "rcpg_get_option": (_I32, [_V, C.c_char_p, C.POINTER(C.c_int64)]),
    "rcpg_bench_factor": (_I32, [_V, C.c_int, _I32, _I64, _I64, _I32, C.POINTER(C.c_double)]),
    "rcpg_event_record": (_I32, [_V, _I32]),
    "rcpg_event_elapsed": (_I32, [_V, _I32, _I32, C.POINTER(C.c_double)]),
    "rcpg_host_register": (_I32, [_V, _V, C.c_size_t]),
    "rcpg_host_unregister": (_I32, [_V, _V]),
}


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build the CUDA extension first "
                "(python -c 'import __graft_entry__ as g; g.build()'); there is no CPU fallback")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib
