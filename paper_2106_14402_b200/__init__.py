"""B200-native semiring SpGEMM for 2D/3D Sparse SUMMA (CombBLAS 2.0 hot path).

The product is libslapcu.so (CUDA for sm_100a behind the C-ABI in
include/slapcu.h).  This package is the host-side mirror of the reference's
C++ interface (slap::local_spgemm, summa2d_spgemm, ca3d_spgemm,
batched_spgemm, ...) over that C-ABI; torch supplies device memory, streams
and torch.distributed plumbing only.
"""
from . import errors
from ._lib import load as load_library
from .spgemm import (
    Context,
    CscMatrix,
    DeviceCsc,
    MinPlusF64,
    MinPlusI32,
    OrAnd,
    PlusTimesF32,
    PlusTimesF64,
    PlusTimesI64,
    SEMIRINGS,
    Semiring,
    SpGemmAlg,
    column_checksums,
    dcsc_to_csc,
    default_context,
    estimate_flops,
    fill_values,
    gen_er,
    gen_one_per_row,
    gen_rmat,
    local_spgemm,
    mcl_step,
    merge,
    permute_symmetric,
    semiring_from_name,
    slice_cols,
    spgemm_alg_from_name,
    symbolic_nnz,
)

__all__ = [n for n in dir() if not n.startswith("_")]
