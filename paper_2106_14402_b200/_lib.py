"""ctypes binding of libslapcu.so (the C-ABI declared in include/slapcu.h).

The product path always goes through this library; if it is missing the
import fails loudly -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SLAPCU_LIB") or os.path.join(HERE, "libslapcu.so")  # SLAPCU_LIB: A/B builds

# slapcu_status
OK = 0
STATUS_NAMES = {
    1: "DimError",
    2: "ShapeError",
    3: "InternalError",
    4: "NameError",
    5: "BudgetError",
    6: "IndexError",
    7: "InvalidArgument",
    8: "CudaError",
    9: "OutOfMemory",
    10: "DeadlockError",
}

# slapcu_semiring
PLUS_TIMES_F64, PLUS_TIMES_F32, PLUS_TIMES_I64, MIN_PLUS_I32, MIN_PLUS_F64, OR_AND_U8 = range(6)
# slapcu_alg
ALG_HEAP, ALG_HASH, ALG_HYBRID = 0, 1, 2
# slapcu_option
(OPT_TILE_ROWS_LOG2, OPT_SYM_TILE_ROWS_LOG2, OPT_LIGHT_NNZ_MAX, OPT_LIGHT_FLOPS_MAX, OPT_DETERMINISTIC, OPT_PROFILE,
 OPT_DENSE_FLOPS_MIN, OPT_DENSE_TILE_ROWS_LOG2, OPT_ASYNC_FINISH, OPT_DIRECT_TILE_ROWS_LOG2,
 OPT_DIRECT_SPLIT_FLOPS, OPT_DIRECT_MARK_MODE, OPT_DIRECT_FORM_THREADS, OPT_DIRECT_EMIT_THREADS,
 OPT_DIRECT_DENSE_RUN_MIN, OPT_DIRECT_PERSISTENT, OPT_DIRECT_QUADS,
 OPT_DIRECT_VALUE_TILE_ROWS_LOG2, OPT_DIRECT_VALUE_THREADS, OPT_SUMMA_CONCAT,
 OPT_DIRECT_VALUE_HASH, OPT_DIRECT_VALUE_RANK, OPT_DIRECT_VALUE_INTERLEAVE, OPT_DIRECT_TILE_MAJOR,
 OPT_DIRECT_FORM_WALK, OPT_DIRECT_SHORT_RUN, OPT_DIRECT_VALUE_TMAJOR, OPT_DIRECT_WORDS,
 OPT_DIRECT_ESC, OPT_DIRECT_VALUE_DENSE_ROWS, OPT_DIRECT_VALUE_DENSE_ONLY, OPT_DIRECT_VALUE_L2,
 OPT_DIRECT_VALUE_FORM, OPT_DIRECT_VALUE_TINY_RUN, OPT_DIRECT_VALUE_ROWS) = range(35)
NUM_KERNEL_CLASSES = 10
KERNEL_CLASSES = ["other", "flops", "bin", "sym_light", "sym_heavy", "scan", "num_light", "num_heavy", "merge", "gen"]


class CscView(C.Structure):
    """slapcu_csc (device pointers)."""

    _fields_ = [
        ("nrows", C.c_int64),
        ("ncols", C.c_int64),
        ("nnz", C.c_int64),
        ("colptr", C.c_void_p),
        ("rowids", C.c_void_p),
        ("vals", C.c_void_p),
    ]


class CscOut(C.Structure):
    """slapcu_csc_out / slapcu_host_csc."""

    _fields_ = [
        ("nrows", C.c_int64),
        ("ncols", C.c_int64),
        ("nnz", C.c_int64),
        ("colptr", C.c_void_p),
        ("rowids", C.c_void_p),
        ("vals", C.c_void_p),
    ]


class DistStats(C.Structure):
    """slapcu_dist_stats (summa.hpp:15-20 DistKernelStats + timings)."""

    _fields_ = [
        ("stages", C.c_int),
        ("flops", C.c_int64),
        ("nnz_out", C.c_int64),
        ("layer_warning", C.c_int),
        ("ms_total", C.c_float),
        ("ms_local", C.c_float),
        ("ms_merge", C.c_float),
        ("ms_exposed_bcast", C.c_float),
    ]


class Tiling(C.Structure):
    """slapcu_tiling (host pointers; see grid.tiling_2d / tiling_3d)."""

    _fields_ = [
        ("nr", C.c_int),
        ("nc", C.c_int),
        ("row_cuts", C.c_void_p),
        ("col_cuts", C.c_void_p),
        ("owner", C.c_void_p),
    ]


# typedef int (*slapcu_batch_consumer)(void*, int, int64_t, int64_t, const slapcu_host_csc*)
BatchConsumer = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.c_int64, C.c_int64, C.POINTER(CscOut))

# (name, restype, argtypes) for every entry point of include/slapcu.h
_P = C.c_void_p
_I = C.c_int
_L = C.c_int64
_PV = C.POINTER(CscView)
_PO = C.POINTER(CscOut)
SIGNATURES = [
    ("slapcu_abi_version", _I, []),
    ("slapcu_status_name", C.c_char_p, [_I]),
    ("slapcu_ctx_create", _I, [C.POINTER(_P), _I, _P]),
    ("slapcu_ctx_destroy", _I, [_P]),
    ("slapcu_ctx_set_stream", _I, [_P, _P]),
    ("slapcu_ctx_invalidate", _I, [_P]),
    ("slapcu_ctx_synchronize", _I, [_P]),
    ("slapcu_ctx_last_error", C.c_char_p, [_P]),
    ("slapcu_ctx_set_option", _I, [_P, _I, _L]),
    ("slapcu_ctx_kernel_launches", _L, [_P]),
    ("slapcu_ctx_last_phase_ms", _I, [_P, C.POINTER(C.c_float), C.POINTER(C.c_float)]),
    ("slapcu_ctx_kernel_stats", _I, [_P, _I, C.POINTER(_L), C.POINTER(C.c_double)]),
    ("slapcu_ctx_reset_stats", _I, [_P]),
    ("slapcu_kernel_class_name", C.c_char_p, [_I]),
    ("slapcu_semiring_value_size", _I, [_I]),
    ("slapcu_semiring_from_name", _I, [C.c_char_p, C.c_char_p, C.POINTER(_I)]),
    ("slapcu_alg_from_name", _I, [C.c_char_p, C.POINTER(_I)]),
    ("slapcu_estimate_flops", _I, [_P, _PV, _PV, _P, C.POINTER(_L)]),
    ("slapcu_spgemm_symbolic", _I, [_P, _PV, _PV, _I, _P, C.POINTER(_L)]),
    ("slapcu_spgemm_numeric", _I, [_P, _PV, _PV, _I, _I, _P, _P, _P]),
    ("slapcu_spgemm_begin", _I, [_P, _PV, _PV, _I, _I, _L, _P, C.POINTER(_L)]),
    ("slapcu_spgemm_finish", _I, [_P, _PV, _PV, _I, _P, _P]),
    ("slapcu_spgemm_direct", _I, [_P, _PV, _PV, _I, _I, _L, _P, _P, _P, C.POINTER(_L)]),
    ("slapcu_spgemm", _I, [_P, _PV, _PV, _I, _I, _PO]),
    ("slapcu_spgemm_host", _I, [_P, _PO, _PO, _I, _I, _PO]),
    ("slapcu_batched_spgemm_host", _I, [_P, _PO, _PO, _I, _I, _I, _P, _L, BatchConsumer, _P, C.POINTER(_L)]),
    ("slapcu_csc_free", _I, [_P, _PO]),
    ("slapcu_device_count", _I, [C.POINTER(_I)]),
    ("slapcu_estimate_flops_host", _I, [_P, _PO, _PO, _P, C.POINTER(_L)]),
    ("slapcu_symbolic_nnz_host", _I, [_P, _PO, _PO, _I, _P]),
    ("slapcu_csc_upload", _I, [_P, _PO, _I, _PO]),
    ("slapcu_dcsc_upload", _I, [_P, _L, _L, _L, _P, _P, _P, _P, _I, _PO]),
    ("slapcu_csc_download", _I, [_P, _PV, _I, _PO]),
    ("slapcu_mcl_step", _I, [_P, _PV, _I, C.c_double, C.c_double, _PO]),
    ("slapcu_host_free", None, [_PO]),
    ("slapcu_dcsc_colptr", _I, [_P, _L, _L, _P, _P, _P]),
    ("slapcu_merge_symbolic", _I, [_P, _I, _PV, _P, C.POINTER(_L)]),
    ("slapcu_merge_numeric", _I, [_P, _I, _PV, _I, _P, _P, _P]),
    ("slapcu_gen_rmat", _I, [_P, _I, _I, C.c_uint64, C.c_double, C.c_double, C.c_double, C.c_double, _PO]),
    ("slapcu_gen_er", _I, [_P, _L, _L, C.c_uint64, _I, _PO]),
    ("slapcu_gen_one_per_row", _I, [_P, _L, _L, C.c_uint64, _PO]),
    ("slapcu_fill_values", _I, [_P, _I, _I, _PV, _P]),
    ("slapcu_permute_symmetric", _I, [_P, _PV, C.c_uint64, _I, _PO]),
    ("slapcu_slice_cols", _I, [_P, _PV, _I, _L, _L, _PO]),
    ("slapcu_column_checksums", _I, [_P, _PV, _I, _I, _P]),
    ("slapcu_comm_unique_id", _I, [_P]),
    ("slapcu_comm_create", _I, [C.POINTER(_P), _P, _I, _I, _P]),
    ("slapcu_comm_destroy", _I, [_P]),
    ("slapcu_comm_counters", _I, [_P, _I, C.POINTER(_L), C.POINTER(_L)]),
    ("slapcu_summa2d", _I, [_P, _PV, _PV, _I, _I, _PO, C.POINTER(DistStats)]),
    ("slapcu_ca3d", _I, [_P, _I, _PV, _PV, _I, _I, _PO, C.POINTER(DistStats)]),
    ("slapcu_dist_symbolic_col_nnz", _I, [_P, _PV, _PV, _P, _L]),
    ("slapcu_mcl_step_dist", _I, [_P, _I, _I, _I, _PV, _I, C.c_double, C.c_double, _PO]),
    ("slapcu_redistribute", _I, [_P, _PV, _L, _L, _L, _L, _I, C.POINTER(Tiling), _I, _PO, C.POINTER(_L),
                                 C.POINTER(_L)]),
    ("slapcu_cb2b_header", _I, [C.c_char_p, C.POINTER(_L), C.POINTER(_L), C.POINTER(_L)]),
    ("slapcu_write_cb2b", _I, [_P, C.c_char_p, _PV, _L, _L, _L, _L]),
    ("slapcu_read_cb2b", _I, [_P, C.c_char_p, _I, _I, _PO, C.POINTER(_L), C.POINTER(_L), C.POINTER(_L),
                              C.POINTER(_L)]),
    ("slapcu_distribute_triples", _I, [_P, _L, _P, _P, _P, _L, _L, _I, C.POINTER(Tiling), _I, _PO, C.POINTER(_L),
                                       C.POINTER(_L)]),
]

_lib = None


def load(path: str = LIB_PATH) -> C.CDLL:
    """Loads libslapcu.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build it with `python -m paper_2106_14402_b200._build` "
            "(there is no CPU fallback for the SpGEMM path)"
        )
    lib = C.CDLL(path)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


_cudart = None


def cudart() -> C.CDLL:
    """The CUDA runtime libslapcu.so links against (for raw async copies)."""
    global _cudart
    if _cudart is None:
        load()
        _cudart = C.CDLL("libcudart.so.12")
        _cudart.cudaMemcpyAsync.restype = C.c_int
        _cudart.cudaMemcpyAsync.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int, C.c_void_p]
    return _cudart


def symbol_names():
    return [s[0] for s in SIGNATURES]
