"""ctypes binding of libsphbi_cuda.so (the C-ABI declared in include/sphbi_cuda.h).

There is no CPU fallback: if the shared library is missing or no sm_100 GPU is
visible, every call raises. The library is built in-tree by
``paper_2507_21686_b200.build.build_native()`` (or ``__graft_entry__.build()``).
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

LIB_DIR = Path(__file__).resolve().parent / "_lib"
# SPHBI_LIB: a variant build of the same library (tools/build_variant.sh; code-shape sweeps)
LIB_PATH = Path(os.environ["SPHBI_LIB"]) if os.environ.get("SPHBI_LIB") else LIB_DIR / "libsphbi_cuda.so"

MAX_COEFFICIENTS = 17
NUM_COUNTERS = 19

# sphbi_status codes (include/sphbi_cuda.h)
OK = 0
ERR_DOMAIN = 1
ERR_INVALID_ARGUMENT = 2
ERR_UNSUPPORTED_FORM = 3
ERR_SINGULAR_INPUT = 4
ERR_LOGIC = 5
ERR_CUDA = 6
ERR_NO_DEVICE = 7
ERR_OUT_OF_MEMORY = 8
ERR_INTERNAL = 9

MEM_HOST = 0
MEM_DEVICE = 1

DECOMP_EDGES = 0
DECOMP_REFERENCE = 1
DECOMP_HYBRID = 2

c_double_p = ctypes.POINTER(ctypes.c_double)
c_int64_p = ctypes.POINTER(ctypes.c_int64)
c_uint32_p = ctypes.POINTER(ctypes.c_uint32)
c_int32_p = ctypes.POINTER(ctypes.c_int32)


class KernelDesc(ctypes.Structure):
    _fields_ = [
        ("n_coefficients", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
        ("coefficients", ctypes.c_double * MAX_COEFFICIENTS),
        ("normalization", ctypes.c_double),
    ]


class Stats(ctypes.Structure):
    _fields_ = [
        ("n_pairs", ctypes.c_int64),
        ("n_candidates", ctypes.c_int64),
        ("status_bits", ctypes.c_uint32),
        ("reserved", ctypes.c_uint32),
        ("ms_pairs", ctypes.c_double),
        ("ms_eval", ctypes.c_double),
        ("ms_reduce", ctypes.c_double),
    ]


EXPORTED_SYMBOLS = (
    "sphbi_ctx_create",
    "sphbi_ctx_destroy",
    "sphbi_ctx_set_stream",
    "sphbi_ctx_synchronize",
    "sphbi_ctx_enable_counters",
    "sphbi_ctx_set_decomposition",
    "sphbi_ctx_set_precision",
    "sphbi_ctx_last_precision",
    "sphbi_read_counters",
    "sphbi_last_error",
    "sphbi_ctx_launch_count",
    "sphbi_kernel_validate",
    "sphbi_integrate_pairs",
    "sphbi_integrate_regions",
    "sphbi_evaluate",
    "sphbi_pair_counts",
    "sphbi_integrate_pairs_p3",
    "sphbi_evaluate_p3",
    "sphbi_measure_fp64_peak",
    "sphbi_evaluate_piecewise",
    "sphbi_bases_create",
    "sphbi_bases_info",
    "sphbi_bases_read",
    "sphbi_bases_apply",
    "sphbi_bases_destroy",
    "sphbi_bases_apply_pairs",
    "sphbi_boundary_normals",
)

_lib = None


def load() -> ctypes.CDLL:
    """Load libsphbi_cuda.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise RuntimeError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(str(LIB_PATH))
    P = ctypes.c_void_p
    lib.sphbi_ctx_create.argtypes = [ctypes.c_int, ctypes.POINTER(P)]
    lib.sphbi_ctx_destroy.argtypes = [P]
    lib.sphbi_ctx_set_stream.argtypes = [P, P]
    lib.sphbi_ctx_synchronize.argtypes = [P]
    lib.sphbi_ctx_enable_counters.argtypes = [P, ctypes.c_int]
    lib.sphbi_ctx_set_decomposition.argtypes = [P, ctypes.c_int32]
    lib.sphbi_ctx_set_precision.argtypes = [P, ctypes.c_int32]
    lib.sphbi_ctx_last_precision.argtypes = [P]
    lib.sphbi_ctx_last_precision.restype = ctypes.c_int32
    lib.sphbi_read_counters.argtypes = [P, ctypes.POINTER(ctypes.c_uint64), ctypes.c_int]
    lib.sphbi_last_error.restype = ctypes.c_char_p
    lib.sphbi_ctx_launch_count.argtypes = [P]
    lib.sphbi_ctx_launch_count.restype = ctypes.c_int64
    lib.sphbi_kernel_validate.argtypes = [ctypes.POINTER(KernelDesc)]
    lib.sphbi_integrate_pairs.argtypes = [P, ctypes.POINTER(KernelDesc), ctypes.c_double, ctypes.c_int64,
                                          P, P, P, ctypes.c_int32, P, P, ctypes.c_int]
    lib.sphbi_integrate_regions.argtypes = [P, ctypes.POINTER(KernelDesc), ctypes.c_int64, P, P, P, P, P]
    lib.sphbi_evaluate.argtypes = [P, ctypes.POINTER(KernelDesc), ctypes.c_double, ctypes.c_int64, P,
                                   ctypes.c_int64, P, P, ctypes.c_int64, P, P, P, P, P,
                                   ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(Stats), ctypes.c_int]
    lib.sphbi_pair_counts.argtypes = [P, ctypes.c_double, ctypes.c_int64, P, ctypes.c_int64, P, P,
                                      ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(Stats), ctypes.c_int]
    lib.sphbi_integrate_pairs_p3.argtypes = [P, ctypes.POINTER(KernelDesc), ctypes.c_double, ctypes.c_int64,
                                             P, P, P, P, P, ctypes.c_int]
    lib.sphbi_evaluate_p3.argtypes = lib.sphbi_evaluate.argtypes
    lib.sphbi_measure_fp64_peak.argtypes = [P, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]
    lib.sphbi_evaluate_piecewise.argtypes = [P, ctypes.c_int32, ctypes.POINTER(KernelDesc), P, ctypes.c_double,
                                             ctypes.c_int64, P, ctypes.c_int64, P, P, ctypes.c_int64, P, P, P, P, P,
                                             ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(Stats), ctypes.c_int]
    lib.sphbi_bases_create.argtypes = [P, ctypes.POINTER(KernelDesc), ctypes.c_double, ctypes.c_int64, P,
                                       ctypes.c_int64, P, ctypes.c_int64, P, P, ctypes.POINTER(Stats), ctypes.c_int,
                                       ctypes.POINTER(P)]
    I64 = ctypes.POINTER(ctypes.c_int64)
    lib.sphbi_bases_info.argtypes = [P, I64, I64, I64]
    lib.sphbi_bases_read.argtypes = [P, P, P, ctypes.c_int]
    lib.sphbi_bases_apply.argtypes = [P, ctypes.c_int32, P, P, P, P, P, P, ctypes.POINTER(ctypes.c_double),
                                      ctypes.c_int]
    lib.sphbi_bases_destroy.argtypes = [P]
    lib.sphbi_bases_apply_pairs.argtypes = [P, P, P, P, ctypes.c_int]
    lib.sphbi_boundary_normals.argtypes = [P, P, ctypes.c_int]
    _lib = lib
    return lib


def last_error() -> str:
    return load().sphbi_last_error().decode(errors="replace")
