/*
 * slapcu.h -- C-ABI of the B200-native semiring SpGEMM library (libslapcu.so).
 *
 * This is the drop-in boundary for the hot path of the reference ("slap",
 * /root/reference/proj, a CombBLAS 2.0 embodiment): the local semiring
 * SpGEMM that 2D/3D Sparse SUMMA calls once per stage, the stage-partial merge,
 * and the distributed drivers around them.  Plain C types only: device
 * pointers, sizes, an opaque context and int status codes.  No exceptions
 * cross this boundary; status codes map 1:1 onto the reference's slap::Error
 * kinds (error.hpp:27-36) via slapcu_status_name().
 *
 * Layout (all matrices): CSC, int64 colptr[ncols+1], int32 rowids[nnz] with
 * rows strictly ascending inside every column, values of the semiring's
 * element type.  The reference stores colptr in its int32 local index type
 * (local_matrix.hpp:26-82, dist_matrix.hpp:18), which overflows at nnz >= 2^31
 * (spgemm.hpp:289-292); 64-bit offsets remove that limit here.
 *
 * Reference interface each entry point replaces is cited on its declaration
 * (paths relative to /root/reference/proj/core/include/slap/).
 */
#ifndef SLAPCU_H
#define SLAPCU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SLAPCU_ABI_VERSION 1

/* error.hpp:10-36: Error kinds.  SLAPCU_ERR_INTERNAL is the reference's
 * Error("InternalError") raised when numeric != symbolic (spgemm.hpp:323-324). */
typedef enum {
    SLAPCU_OK = 0,
    SLAPCU_ERR_DIM = 1,      /* DimError   (spgemm.hpp:57-64, summa.hpp:116-122)   */
    SLAPCU_ERR_SHAPE = 2,    /* ShapeError (summa.hpp:112-115, spgemm3d.hpp:27-30) */
    SLAPCU_ERR_INTERNAL = 3, /* Error("InternalError")                             */
    SLAPCU_ERR_NAME = 4,     /* NameError  (spgemm.hpp:19-24, semiring.cpp)        */
    SLAPCU_ERR_BUDGET = 5,   /* BudgetError (batched.hpp:122-148)                  */
    SLAPCU_ERR_INDEX = 6,    /* IndexError                                         */
    SLAPCU_ERR_INVALID = 7,  /* bad argument (null pointer, unsupported id)        */
    SLAPCU_ERR_CUDA = 8,     /* CUDA runtime failure                               */
    SLAPCU_ERR_NOMEM = 9,    /* device allocation failure                          */
    SLAPCU_ERR_COMM = 10,    /* NCCL failure / collective mismatch (DeadlockError) */
    SLAPCU_ERR_STOCHASTIC = 11, /* StochasticityError (algorithms.cpp:271-275, mcl_step input) */
    SLAPCU_ERR_IO = 12,         /* IoError     (binary_io.cpp, mm_io.cpp:15-20)             */
    SLAPCU_ERR_FORMAT = 13      /* FormatError (binary_io.cpp: magic / version / truncation) */
} slapcu_status;

/* semiring.hpp:36-93.  Ids are stable (shared with oracle/oracle.h). */
typedef enum {
    SLAPCU_PLUS_TIMES_F64 = 0, /* PlusTimes<double>  */
    SLAPCU_PLUS_TIMES_F32 = 1, /* PlusTimes<float>   */
    SLAPCU_PLUS_TIMES_I64 = 2, /* PlusTimes<int64_t> */
    SLAPCU_MIN_PLUS_I32 = 3,   /* MinPlus<int32_t>   (zero = INT32_MAX) */
    SLAPCU_MIN_PLUS_F64 = 4,   /* MinPlus<double>    (zero = +inf)      */
    SLAPCU_OR_AND_U8 = 5       /* OrAnd, uint8 0/1                      */
} slapcu_semiring;

/* spgemm.hpp:17 SpGemmAlg.  On the GPU these are accumulator policies:
 * hybrid = binned by work (smem hash for light columns, row-tiled dense
 * bitmap accumulator for heavy ones); hash = same bins; heap = force the
 * sorted dense-tile path for every column.  Output is identical for all. */
typedef enum { SLAPCU_ALG_HEAP = 0, SLAPCU_ALG_HASH = 1, SLAPCU_ALG_HYBRID = 2 } slapcu_alg;

/* One CSC operand in DEVICE memory. */
typedef struct {
    int64_t nrows, ncols, nnz;
    const int64_t* colptr; /* [ncols+1] */
    const int32_t* rowids; /* [nnz]     */
    const void* vals;      /* [nnz] of the semiring element type */
} slapcu_csc;

/* A CSC result whose device buffers were allocated by the library
 * (free with slapcu_csc_free). */
typedef struct {
    int64_t nrows, ncols, nnz;
    int64_t* colptr;
    int32_t* rowids;
    void* vals;
} slapcu_csc_out;

/* The same layout in HOST memory (used by the reference-facing one-shot call). */
typedef slapcu_csc_out slapcu_host_csc;

typedef struct slapcu_ctx_s* slapcu_ctx;

/* ---------------------------------------------------------------- context */

/* A context = one device + one CUDA stream + a stream-ordered workspace and
 * the per-product plan cached between the symbolic and numeric phases.
 * `stream` is a cudaStream_t (NULL = the legacy default stream).  Calls on a
 * context are stream-ordered and not reentrant; use one context per host thread. */
slapcu_status slapcu_ctx_create(slapcu_ctx* out, int device, void* stream);
/* Waits for the context's work, frees its workspace and trims the device's
 * stream-ordered memory pool (which keeps freed workspace cached while
 * contexts are alive) back to what live allocations hold. */
slapcu_status slapcu_ctx_destroy(slapcu_ctx ctx);
slapcu_status slapcu_ctx_set_stream(slapcu_ctx ctx, void* stream);
/* Drops every per-operand cache of the context (A tile pointers, dense-run
 * bitmaps, the symbolic->numeric plan).  Never needed for correctness: the
 * caches are keyed on a content fingerprint of A's pattern, recomputed on every
 * call; the benchmark calls it once per step so per-A setup is timed. */
slapcu_status slapcu_ctx_invalidate(slapcu_ctx ctx);
/* Waits for the context's stream and reports any deferred error. */
slapcu_status slapcu_ctx_synchronize(slapcu_ctx ctx);
const char* slapcu_ctx_last_error(slapcu_ctx ctx);
const char* slapcu_status_name(slapcu_status s); /* "DimError", "ShapeError", ... */
int slapcu_abi_version(void);

/* Tuning / test knobs (defaults are the production policy). */
typedef enum {
    SLAPCU_OPT_TILE_ROWS_LOG2 = 0,    /* row-tile height of the dense accumulators (default 18) */
    SLAPCU_OPT_SYM_TILE_ROWS_LOG2 = 1,/* row-tile height of the symbolic bitmap    (default 19) */
    SLAPCU_OPT_LIGHT_NNZ_MAX = 2,     /* numeric: columns above this use the dense tile path */
    SLAPCU_OPT_LIGHT_FLOPS_MAX = 3,   /* symbolic: columns above this use the bitmap path   */
    SLAPCU_OPT_DETERMINISTIC = 4,     /* 1: floating-point semirings fold every output entry in the
                                         reference's order (ascending k, spgemm.hpp:156-159, :251-255) on
                                         the ESC path -- bit-identical to slap::local_spgemm and run-to-run
                                         reproducible; 0 (default): semiring atomics, within tolerance */
    SLAPCU_OPT_PROFILE = 5,           /* 1: CUDA events around every launch, per-class device time */
    SLAPCU_OPT_DENSE_FLOPS_MIN = 6,   /* fused path: byte-flag tiles for columns with flops >= v
                                         (-1 auto = nrows/4, 0 = off) */
    SLAPCU_OPT_DENSE_TILE_ROWS_LOG2 = 7, /* byte-flag tile height (default 17 = 128 KB) */
    SLAPCU_OPT_ASYNC_FINISH = 8,      /* 1: slapcu_spgemm_finish returns without waiting; its
                                         InternalError surfaces at the next call on the context
                                         or at slapcu_ctx_synchronize */
    SLAPCU_OPT_DIRECT_TILE_ROWS_LOG2 = 9,  /* direct path: rows per (column, row tile) item (default 17) */
    SLAPCU_OPT_DIRECT_SPLIT_FLOPS = 10,    /* direct path: items with more multiplies than this are formed
                                              by several CTAs over equal-flops parts of B(:,j) (>= 1024) */
    SLAPCU_OPT_DIRECT_MARK_MODE = 11,      /* retired (round 2): only 0 (test-then-set, summary by ballots) */
    SLAPCU_OPT_DIRECT_FORM_THREADS = 12,   /* direct path: threads per form CTA (128, 256, 512) */
    SLAPCU_OPT_DIRECT_EMIT_THREADS = 13,   /* retired (round 2): only 128 (one 4-warp CTA per item) */
    SLAPCU_OPT_DIRECT_DENSE_RUN_MIN = 14,  /* direct path: A(:,k) runs inside one row tile with at least
                                              this many entries are OR-ed as cached tile bitmaps
                                              (row form only; default 4096, 0 = never) */
    SLAPCU_OPT_DIRECT_PERSISTENT = 15,     /* direct path form kernel: 1 persistent CTAs taking units by
                                              ticket, 0 one CTA per unit */
    SLAPCU_OPT_DIRECT_QUADS = 16,          /* retired (round 2): only 0 */
    SLAPCU_OPT_DIRECT_VALUE_TILE_ROWS_LOG2 = 17, /* direct path value pass, sub-tile mode (VALUE_RANK = 0):
                                                    rows per shared value array (10..15, default 13) */
    SLAPCU_OPT_DIRECT_VALUE_THREADS = 18,  /* direct path value pass: threads per CTA (256, 512) */
    SLAPCU_OPT_SUMMA_CONCAT = 19,          /* SUMMA / 3D layers: 1 (default) = all stage blocks are
                                              broadcast, then ONE concatenated-k product forms C(i,j)
                                              (no stage partials, no merge); 0 = per-stage products
                                              double-buffered against the broadcasts + stage merge */
    SLAPCU_OPT_DIRECT_VALUE_HASH = 20,     /* direct path value pass: 1 (= 13) / 13 / 14 = items with
                                              <= 2^(v-1) outputs take one walk into a shared hash table of
                                              2^v slots keyed by their rows; 0 = every item takes the rank
                                              chunks (or the row sub-tiles when VALUE_RANK = 0).  Default
                                              (auto): 0 for 4-byte values with rank chunks, else 13 */
    SLAPCU_OPT_DIRECT_VALUE_RANK = 21,     /* direct path value pass: larger items are folded in rank
                                              chunks of at most this many outputs (4096..16384; default
                                              10240 for 4-byte, 4096 for 8-byte accumulators);
                                              0 = row sub-tiles of 2^VTL rows */
    SLAPCU_OPT_DIRECT_VALUE_INTERLEAVE = 22, /* direct path value pass: A's rows and values gathered as
                                              one interleaved pair per product -- 1 (default) for 4-byte
                                              values (8-byte pairs), 2 also for 8-byte values (16-byte
                                              pairs); 0 = from the two arrays */
    SLAPCU_OPT_DIRECT_TILE_MAJOR = 23,     /* direct path form: 1 = work units ordered by row tile, heaviest
                                              first inside a tile (the tile's A slice stays in L2);
                                              0 = heaviest first over all tiles */
    SLAPCU_OPT_DIRECT_FORM_WALK = 24,      /* retired (round 2): only 0 (256-element units) */
    SLAPCU_OPT_DIRECT_SHORT_RUN = 25,      /* direct path form: runs (A column x row tile) shorter than this
                                              are walked by their own thread (0 = default 8) */
    SLAPCU_OPT_DIRECT_VALUE_TMAJOR = 26,   /* direct path value pass: 1 = 4096-row tile pointers stored
                                              tile-major and rank chunks run in row-block order */
    SLAPCU_OPT_DIRECT_WORDS = 27,          /* direct path form: 1 = walk A as (32-row word, row mask) pairs
                                              (built per A): one shared update per distinct word of a run */
    SLAPCU_OPT_DIRECT_ESC = 28,            /* direct path: 1 = every semiring on the ESC (expand, stable sort
                                              by row, left fold) path; 0 = bitmap / hash paths; -1 (default)
                                              = value semirings whose sampled compression flops / nnz(C) is
                                              below 2 (spgemm.hpp:54's hybrid threshold) take ESC */
    SLAPCU_OPT_DIRECT_VALUE_DENSE_ROWS = 29, /* direct path value pass: chunks spanning at most this many rows
                                              (multiple of 4096, <= 32768) fold by row offset into a dense
                                              shared array, without rank lookups (0 = the rank chunk size) */
    SLAPCU_OPT_DIRECT_VALUE_DENSE_ONLY = 30, /* retired (round 2, measured 2.6x slower on MinPlus C3): only 0 */
    SLAPCU_OPT_DIRECT_VALUE_L2 = 31,       /* retired (round 2: global-atomic folds, one walk per form unit,
                                              measured 501 -> 609 ms on MinPlus C3): only 0 */
    SLAPCU_OPT_DIRECT_VALUE_FORM = 32,     /* direct path, semirings with values: log2 rows of the value
                                              form's item tile (one product walk folds values into a dense
                                              shared array of the tile and stashes them in row order; emit
                                              copies them into C).  0 (default) = off (pattern form + the
                                              value pass: measured faster at C3, whose 2^14-row items are
                                              too many and too small), -1 = auto (2^14 rows for accumulators
                                              of <= 4 bytes, 2^13 for 8 bytes), 12..15 = that height */
    SLAPCU_OPT_DIRECT_VALUE_TINY_RUN = 33, /* direct path value walks: runs (A column x tile) of at most this
                                              many products are folded by their own thread with 4 loads in
                                              flight; longer runs below 32 are packed 32 products per warp
                                              step, 32 and up cut into warp units.  -1 = default */
    SLAPCU_OPT_DIRECT_VALUE_ROWS = 34      /* direct path, 4-byte values (every item in rank chunks): 1 =
                                              the value pass writes C's rows beside the values from the
                                              form pass's stash and the emit pass is skipped (measured
                                              slower, MinPlus C3 409 -> 458 ms: its per-thread row stores
                                              are not staged like emit's); 0 (default) = emit writes them */
} slapcu_option;
slapcu_status slapcu_ctx_set_option(slapcu_ctx ctx, slapcu_option opt, int64_t value);

/* Per-kernel-class device time collected with SLAPCU_OPT_PROFILE (events on
 * the context stream).  Classes: 0 other, 1 flops, 2 bin, 3 sym_light,
 * 4 sym_heavy, 5 scan, 6 num_light, 7 num_heavy, 8 merge, 9 gen. */
#define SLAPCU_NUM_KERNEL_CLASSES 10
slapcu_status slapcu_ctx_kernel_stats(slapcu_ctx ctx, int cls, int64_t* launches, double* ms);
slapcu_status slapcu_ctx_reset_stats(slapcu_ctx ctx);
const char* slapcu_kernel_class_name(int cls);

/* Number of kernels this context launched since creation (for bench reports). */
int64_t slapcu_ctx_kernel_launches(slapcu_ctx ctx);

/* Elapsed device time of the last numeric phase's dominant kernels, ms
 * (CUDA events on the context stream). */
slapcu_status slapcu_ctx_last_phase_ms(slapcu_ctx ctx, float* symbolic_ms, float* numeric_ms);

int slapcu_semiring_value_size(slapcu_semiring sr);
/* semiring.cpp builtin_semiring + dtype: ("plus_times","f64") etc. */
slapcu_status slapcu_semiring_from_name(const char* name, const char* dtype, slapcu_semiring* out);
/* spgemm.hpp:19-24 spgemm_alg_from_name */
slapcu_status slapcu_alg_from_name(const char* name, slapcu_alg* out);

/* --------------------------------------------------- local SpGEMM phases */

/* Phase 1, spgemm.hpp:68-88 estimate_flops: per-column multiply counts of
 * C = A*B into flops_per_col (device, int64[B.ncols], may be NULL) and the
 * total into *total (host). */
slapcu_status slapcu_estimate_flops(slapcu_ctx ctx, const slapcu_csc* A, const slapcu_csc* B,
                                    int64_t* flops_per_col, int64_t* total);

/* Phase 2, spgemm.hpp:118-138 symbolic_nnz + the colptr prefix sum
 * (spgemm.hpp:289-293): writes C's colptr (device, int64[B.ncols+1]) and
 * *c_nnz (host).  Values of A/B are not read. */
slapcu_status slapcu_spgemm_symbolic(slapcu_ctx ctx, const slapcu_csc* A, const slapcu_csc* B, slapcu_alg alg,
                                     int64_t* c_colptr, int64_t* c_nnz);

/* Phase 3, spgemm.hpp:297-330 numeric pass: fills C's rowids/vals (device,
 * caller-allocated, sized by phase 2) for the colptr phase 2 produced on the
 * same context.  Rows come out ascending per column, no explicit zeros are
 * pruned.  SLAPCU_ERR_INTERNAL if any column's numeric count
 * disagrees with the symbolic count (spgemm.hpp:323-324). */
slapcu_status slapcu_spgemm_numeric(slapcu_ctx ctx, const slapcu_csc* A, const slapcu_csc* B, slapcu_semiring sr,
                                    slapcu_alg alg, const int64_t* c_colptr, int32_t* c_rowids, void* c_vals);

/* Single-product-pass form of the same contract (the production path):
 * begin() forms every output column once, sorted, into a staging area owned
 * by the context and writes C's colptr + *c_nnz; the caller allocates rowids
 * / vals; finish() lays the staged columns out (and, for value semirings,
 * accumulates heavy columns' values at their popcount rank).  Staging needs
 * sum_j min(flops_j, A.nrows) entries; if that exceeds staging_budget_bytes
 * (> 0) begin() fails with SLAPCU_ERR_BUDGET and the caller batches columns
 * (batched.hpp:153-170).  A and B must be the same objects in both calls. */
slapcu_status slapcu_spgemm_begin(slapcu_ctx ctx, const slapcu_csc* A, const slapcu_csc* B, slapcu_semiring sr,
                                  slapcu_alg alg, int64_t staging_budget_bytes, int64_t* c_colptr, int64_t* c_nnz);
slapcu_status slapcu_spgemm_finish(slapcu_ctx ctx, const slapcu_csc* A, const slapcu_csc* B, slapcu_semiring sr,
                                   int32_t* c_rowids, void* c_vals);

/* Single pass straight into caller buffers (the production path for the
 * Boolean C3 headline): C's colptr, rowids and values are written in place
 * after one walk over the products -- heavy columns are cut into (column, row
 * tile) items, each formed in a shared-memory bitmap and kept as a compact
 * stash (bitmap or non-zero word list, ~1 byte per output entry), then placed
 * by a scan of the item counts and expanded straight into C; there is no
 * row-id staging copy and no second product pass.  `capacity` = entries the caller's
 * c_rowids / c_vals hold; sum_j min(flops_j, A.nrows) (from
 * slapcu_estimate_flops) always suffices.  If C needs more, nothing beyond
 * capacity is written, *c_nnz gets the exact requirement and the call
 * returns SLAPCU_ERR_BUDGET.  OrAnd operands without stored zeros take the
 * in-place path; other semirings are formed by the begin/finish pair into
 * the same buffers (same contract).  Same output as local_spgemm. */
slapcu_status slapcu_spgemm_direct(slapcu_ctx ctx, const slapcu_csc* A, const slapcu_csc* B, slapcu_semiring sr,
                                   slapcu_alg alg, int64_t capacity, int64_t* c_colptr, int32_t* c_rowids,
                                   void* c_vals, int64_t* c_nnz);

/* spgemm.hpp:275-330 local_spgemm, all three phases, C allocated on the
 * device by the library: the direct single pass into a bound-sized scratch,
 * then exactly sized buffers; falls back to begin/finish, then to the
 * symbolic/numeric pair, when that scratch / the staging area does not fit. */
slapcu_status slapcu_spgemm(slapcu_ctx ctx, const slapcu_csc* A, const slapcu_csc* B, slapcu_semiring sr,
                            slapcu_alg alg, slapcu_csc_out* C);

/* local_spgemm with HOST operands and a HOST result (malloc'd; free with
 * slapcu_host_free): H2D copies, the three phases, D2H copies.  This is the
 * call the reference-side C++ template shim binds. */
slapcu_status slapcu_spgemm_host(slapcu_ctx ctx, const slapcu_host_csc* A, const slapcu_host_csc* B,
                                 slapcu_semiring sr, slapcu_alg alg, slapcu_host_csc* C);

/* batched.hpp:153-170 batched_spgemm (with batched.hpp:122-148 planning) for
 * HOST operands: A and B are copied to the device once, then for every column
 * range r of B, in order, C_r = A * B(:, range_r) is formed on the device and
 * read back into pinned host memory, and consumer(user, r, col_begin, col_end,
 * C_r) is called on the calling thread (batch r+1's product overlaps batch r's
 * read-back).  C_r is a host CSC with colptr rebased to 0; its buffers belong
 * to the library and are valid only during the call.  `col_ranges` holds
 * nranges [begin, end) pairs partitioning B's columns (ShapeError otherwise,
 * batched.hpp:157-163), or NULL: the library plans the fewest ranges whose
 * output bound sum_j min(flops_j, nrows) * (4 + value bytes) fits
 * `budget_bytes` (BudgetError if one column alone exceeds it).  A non-zero
 * consumer return aborts with SLAPCU_ERR_INVALID.  *total_nnz = nnz(C). */
typedef int (*slapcu_batch_consumer)(void* user, int batch, int64_t col_begin, int64_t col_end,
                                     const slapcu_host_csc* C_r);
slapcu_status slapcu_batched_spgemm_host(slapcu_ctx ctx, const slapcu_host_csc* A, const slapcu_host_csc* B,
                                         slapcu_semiring sr, slapcu_alg alg, int nranges, const int64_t* col_ranges,
                                         int64_t budget_bytes, slapcu_batch_consumer consumer, void* user,
                                         int64_t* total_nnz);

slapcu_status slapcu_csc_free(slapcu_ctx ctx, slapcu_csc_out* C);

/* spgemm.hpp:68-88 estimate_flops and spgemm.hpp:118-138 symbolic_nnz for
 * HOST operands (pattern only; values are not read): per-column results into
 * host arrays of B.ncols.  DimError on an inner-dimension mismatch. */
slapcu_status slapcu_estimate_flops_host(slapcu_ctx ctx, const slapcu_host_csc* A, const slapcu_host_csc* B,
                                         int64_t* flops_per_col, int64_t* total);
slapcu_status slapcu_symbolic_nnz_host(slapcu_ctx ctx, const slapcu_host_csc* A, const slapcu_host_csc* B,
                                       slapcu_alg alg, int64_t* counts);

/* Number of CUDA devices visible to this process (0 when none). */
slapcu_status slapcu_device_count(int* n);
/* Host CSC -> library-allocated device CSC (free with slapcu_csc_free). */
slapcu_status slapcu_csc_upload(slapcu_ctx ctx, const slapcu_host_csc* h, slapcu_semiring sr, slapcu_csc_out* d);
/* Host DCSC (local_matrix.hpp:88-150: jc[nzc] nonempty column ids, cp[nzc+1]
 * offsets, int32 like the reference's LocalIdx) -> device CSC: the arrays are
 * copied as they are and the dense int64 colptr is built on the device
 * (slapcu_dcsc_colptr), so a SUMMA block goes to the GPU without a host
 * conversion.  Free with slapcu_csc_free. */
slapcu_status slapcu_dcsc_upload(slapcu_ctx ctx, int64_t nrows, int64_t ncols, int64_t nzc, const int32_t* jc,
                                 const int32_t* cp, const int32_t* rowids, const void* vals, slapcu_semiring sr,
                                 slapcu_csc_out* d);
/* Device CSC (any colptr base) -> malloc'd host CSC with colptr rebased to 0
 * (free with slapcu_host_free). */
slapcu_status slapcu_csc_download(slapcu_ctx ctx, const slapcu_csc* d, slapcu_semiring sr, slapcu_host_csc* h);
void slapcu_host_free(slapcu_host_csc* C);

/* algorithms.cpp:267-293 mcl_step on one device: expansion
 * C = A*A (the direct single pass), inflation v -> v^inflation, pruning of
 * entries with v < prune_threshold, column renormalisation (a column whose
 * kept sum is 0 is left as is).  sr: PlusTimes f64 (the reference's type) or
 * f32 (config C4).  Input columns must sum to 1 within 1e-9 (f64) / 1e-5
 * (f32), else SLAPCU_ERR_STOCHASTIC; non-square A or inflation <= 0 give
 * SLAPCU_ERR_SHAPE.  C is allocated by the library (slapcu_csc_free). */
slapcu_status slapcu_mcl_step(slapcu_ctx ctx, const slapcu_csc* A, slapcu_semiring sr, double inflation,
                              double prune_threshold, slapcu_csc_out* C);

/* ------------------------------------------------------- format adapters */

/* local_matrix.hpp:88-150 DcscMatrix -> dense device colptr: scatters the
 * nzc (jc, cp) pairs (int32, device) into colptr (int64[ncols+1]).  The
 * reference looks columns up by binary search on every access
 * (local_matrix.hpp:115-121); the device kernels index colptr directly. */
slapcu_status slapcu_dcsc_colptr(slapcu_ctx ctx, int64_t ncols, int64_t nzc, const int32_t* jc, const int32_t* cp,
                                 int64_t* colptr);

/* ------------------------------------------------------ merge (SUMMA/3D) */

/* local_matrix.hpp:166-188 sort_and_combine as the SUMMA stage merge
 * (summa.hpp:145-156) and the 3D fiber merge (spgemm3d.hpp:257-262): C =
 * parts[0] (+) parts[1] (+) ... with every coincident entry left-folded with
 * sr.add in part order -- the order the reference's stable sort yields.
 * All parts share one shape.  Two phases like the SpGEMM. */
slapcu_status slapcu_merge_symbolic(slapcu_ctx ctx, int nparts, const slapcu_csc* parts, int64_t* c_colptr,
                                    int64_t* c_nnz);
slapcu_status slapcu_merge_numeric(slapcu_ctx ctx, int nparts, const slapcu_csc* parts, slapcu_semiring sr,
                                   const int64_t* c_colptr, int32_t* c_rowids, void* c_vals);

/* -------------------------------------------- synthetic inputs on device */

/* algorithms.cpp:71-113 gen_rmat, bit-identical (Rng rng.hpp:12-45, one
 * stream per edge draw, symmetrized, self loops dropped, duplicates
 * collapsed).  Allocates the pattern (vals = NULL). */
slapcu_status slapcu_gen_rmat(slapcu_ctx ctx, int scale, int edge_factor, uint64_t seed, double a, double b,
                              double c, double d, slapcu_csc_out* out);
/* oracles.hpp:205-217 random_triples as an n x n Erdos-Renyi matrix: `draws`
 * (row, col, value) draws from one Rng(seed) stream, duplicates keep the first
 * draw; values U[0,1) stored as double if with_values. */
slapcu_status slapcu_gen_er(slapcu_ctx ctx, int64_t n, int64_t draws, uint64_t seed, int with_values,
                            slapcu_csc_out* out);
/* Tall-skinny B for config C5: n x ncols, exactly one nonzero per row at
 * column Rng(seed) draw 2i mod ncols, value U[0,1) from draw 2i+1. */
slapcu_status slapcu_gen_one_per_row(slapcu_ctx ctx, int64_t n, int64_t ncols, uint64_t seed, slapcu_csc_out* out);
/* Value recipes, written into `vals` (device, nnz of sr's type):
 * kind 0 ones, 1 U[0,1), 2 U[0,10), 3 int 1+h%255, 4 1/deg(col), 5 int 1+h%9,
 * where h = splitmix64((i<<32) ^ j). */
slapcu_status slapcu_fill_values(slapcu_ctx ctx, slapcu_semiring sr, int kind, const slapcu_csc* m, void* vals);
/* Symmetric relabelling P*A*P^T with a seed-deterministic permutation (the
 * balanced alternative to dist_matrix.hpp:191-212 random_permute for A*A). */
slapcu_status slapcu_permute_symmetric(slapcu_ctx ctx, const slapcu_csc* A, uint64_t seed, slapcu_semiring sr,
                                       slapcu_csc_out* out);

/* Column slice B(:, [c0, c1)) as a new device CSC (batched.hpp:43-66 slice_cols). */
slapcu_status slapcu_slice_cols(slapcu_ctx ctx, const slapcu_csc* B, slapcu_semiring sr, int64_t c0, int64_t c1,
                                slapcu_csc_out* out);

/* Per-column 64-bit checksums of (row, value bits) (device uint64[ncols]);
 * with_values=0 hashes the pattern only.  Matches oracle/orc_column_checksums. */
slapcu_status slapcu_column_checksums(slapcu_ctx ctx, const slapcu_csc* m, slapcu_semiring sr, int with_values,
                                      uint64_t* sums);

/* ---------------------------------------------------- distributed drivers */

/* One process (or host thread) per GPU.  Communicators are NCCL over
 * NVLink/NVSwitch.  slapcu_comm_unique_id fills a 128-byte ncclUniqueId that
 * rank 0 shares with the others out of band (torch.distributed store, MPI,
 * a file...). */
typedef struct slapcu_comm_s* slapcu_comm;
slapcu_status slapcu_comm_unique_id(void* id128);
slapcu_status slapcu_comm_create(slapcu_comm* out, slapcu_ctx ctx, int rank, int nranks, const void* id128);
slapcu_status slapcu_comm_destroy(slapcu_comm comm);

/* comm.hpp:31-53 CommCounters analogue: per-kind call counts / bytes sent by
 * this rank (kind: 0 broadcast, 1 alltoallv, 2 reduce, 3 allgatherv). */
slapcu_status slapcu_comm_counters(slapcu_comm comm, int kind, int64_t* calls, int64_t* bytes);

/* Per-call record, summa.hpp:15-20 DistKernelStats + timing. */
typedef struct {
    int stages;
    int64_t flops;   /* this rank's multiplies */
    int64_t nnz_out; /* this rank's output nonzeros */
    int layer_warning;
    float ms_total, ms_local, ms_merge, ms_exposed_bcast; /* device-event timings */
} slapcu_dist_stats;

/* summa.hpp:106-163 summa2d_spgemm on a q x q grid (rank = i*q + j,
 * grid.hpp:15-24).  A_local / B_local are this rank's blocks (rows
 * A.row_offsets[i].., cols A.col_offsets[j].., layout.hpp:60-66 block_offsets);
 * C_local is allocated.  Stage s broadcasts A(i,s) on the row communicator and
 * B(s,j) on the column communicator (ncclBroadcast), double-buffered against
 * the stage multiply; the q partials are merged once with
 * slapcu_merge (stage order).  Collective over all ranks of `comm`. */
slapcu_status slapcu_summa2d(slapcu_comm comm, const slapcu_csc* A_local, const slapcu_csc* B_local,
                             slapcu_semiring sr, slapcu_alg alg, slapcu_csc_out* C_local,
                             slapcu_dist_stats* stats);

/* batched.hpp:70-117 dist_symbolic_col_nnz on the q x q grid of `comm`:
 * exact per-output-column counts of A*B (pattern SUMMA, column-communicator
 * allreduce, row-communicator all-gather).  Every rank receives all `ncols`
 * counts of B's columns in `counts` (HOST int64[ncols]).  Collective. */
slapcu_status slapcu_dist_symbolic_col_nnz(slapcu_comm comm, const slapcu_csc* A_local, const slapcu_csc* B_local,
                                           int64_t* counts, int64_t ncols);

/* algorithms.cpp:267-293 mcl_step on a pr x pc grid (rank = i*pc + j, A_local
 * = block (i, j) with block_offsets geometry): column sums reduced over the
 * grid column and checked (1e-9 f64 / 1e-5 f32; SLAPCU_ERR_STOCHASTIC on every
 * rank), expansion A*A by slapcu_summa2d (layers <= 1; square grid) or, for
 * layers = c > 1, redistribute to the regular 3D layout (split columns /
 * rows), slapcu_ca3d, redistribute back (all on the device, over NCCL), then
 * inflation, pruning (kept iff !(v < prune_threshold)) and renormalisation by
 * the kept column sums reduced over the grid column.  sr: PlusTimes f64 or
 * f32.  C_local: this rank's block of the result (allocated).  Collective. */
slapcu_status slapcu_mcl_step_dist(slapcu_comm comm, int pr, int pc, int layers, const slapcu_csc* A_local,
                                   slapcu_semiring sr, double inflation, double prune_threshold,
                                   slapcu_csc_out* C_local);

/* spgemm3d.hpp:21-106 ca3d_spgemm on a c x q x q grid (regular variant,
 * grid.cpp:57 rank = l*q*q + i*q + j): A split by columns, B by rows; per
 * layer SUMMA, then C_int's columns are split into c pieces (block_offsets)
 * and exchanged over the fiber (grouped ncclSend/ncclRecv after a count
 * exchange), then merged.  C_local is this rank's piece. */
slapcu_status slapcu_ca3d(slapcu_comm comm, int layers, const slapcu_csc* A_local, const slapcu_csc* B_local,
                          slapcu_semiring sr, slapcu_alg alg, slapcu_csc_out* C_local, slapcu_dist_stats* stats);


/* ------------------------------------------------- redistribution (8f rank 2)
 *
 * A target layout is a tiling of the global nrows x ncols matrix: nr+1 row
 * cuts, nc+1 column cuts (non-decreasing, from 0 to nrows / ncols) and the
 * owning rank of tile (i, j) at owner[i*nc + j]; nr*nc == nranks and every
 * rank owns exactly one tile.  All pointers are HOST pointers and every rank
 * passes the same tiling (checked: SLAPCU_ERR_SHAPE otherwise).  The 2D
 * (grid.hpp:15-24, block_offsets) and regular 3D (dist_matrix3d.hpp:54-80)
 * layouts are built by paper_2106_14402_b200/grid.py tiling_2d / tiling_3d. */
typedef struct {
    int nr, nc;
    const int64_t* row_cuts;
    const int64_t* col_cuts;
    const int32_t* owner;
} slapcu_tiling;

/* redistribute_3d (dist_matrix3d.hpp:117-170, regular variant) /
 * redistribute_2d (dist_matrix3d.hpp:250-261), generalised: this rank's block
 * `local` (block-local indices, global offsets row_start / col_start) is
 * routed entry by entry to the owners of the target tiles (grouped
 * ncclSend/ncclRecv after one count all-gather) and the received entries are
 * assembled into this rank's tile as canonical CSC (allocated; free with
 * slapcu_csc_free); out_row_start / out_col_start receive the tile's global
 * offsets.  combine: 0 keeps the first of duplicate coordinates in arrival
 * order (source rank, then source order), 1 folds them with the semiring add
 * (local_matrix.hpp:167-188).  An entry outside nrows x ncols fails on every
 * rank with SLAPCU_ERR_INDEX.  Collective over all ranks of `comm`. */
slapcu_status slapcu_redistribute(slapcu_comm comm, const slapcu_csc* local, int64_t row_start, int64_t col_start,
                                  int64_t nrows, int64_t ncols, slapcu_semiring sr, const slapcu_tiling* target,
                                  int combine, slapcu_csc_out* out, int64_t* out_row_start, int64_t* out_col_start);

/* distribute_triples (dist_matrix.hpp:89-119): `count` global (row, col, val)
 * triples in DEVICE arrays (int64 rows / cols) from this rank, routed to the
 * target tiles and assembled as above (duplicates: combine 0 keep-first,
 * 1 semiring add, like the reference's `add` argument). */
slapcu_status slapcu_distribute_triples(slapcu_comm comm, int64_t count, const int64_t* rows, const int64_t* cols,
                                        const void* vals, int64_t nrows, int64_t ncols, slapcu_semiring sr,
                                        const slapcu_tiling* target, int combine, slapcu_csc_out* out,
                                        int64_t* out_row_start, int64_t* out_col_start);


/* ------------------------------------------------ CB2B binary I/O (8f rank 4)
 *
 * binary_io.hpp:10-28 format: "CB2B", uint32 version 1, int64 nrows / ncols /
 * nnz, then nnz records (int64 row, int64 col, f64 value), little-endian.
 * Values are f64 (semiring PLUS_TIMES_F64 or MIN_PLUS_F64 blocks). */

/* Header only (no communicator): SLAPCU_ERR_IO if unreadable,
 * SLAPCU_ERR_FORMAT on bad magic / version / size mismatch. */
slapcu_status slapcu_cb2b_header(const char* path, int64_t* nrows, int64_t* ncols, int64_t* nnz);

/* write_binary (binary_io.cpp): rank 0 writes the header, every rank writes
 * its block's records (column-major block order, global indices) at its
 * exclusive-scan offset -- records are built on the device and streamed
 * through pinned buffers.  Collective; the file is complete on return.
 * The format stores fp64 values (the reference's write_binary is
 * double-only): local->vals must hold 8-byte doubles (PLUS_TIMES_F64 /
 * MIN_PLUS_F64 blocks); other value widths are not converted. */
slapcu_status slapcu_write_cb2b(slapcu_comm comm, const char* path, const slapcu_csc* local, int64_t row_start,
                                int64_t col_start, int64_t nrows, int64_t ncols);

/* read_binary (binary_io.cpp): rank r reads records [nnz*r/p, nnz*(r+1)/p),
 * streams them to the device, and the entries are routed to the pr x pc 2D
 * layout (rank = i*pc + j) by the redistribution above (keep-first).  Returns
 * this rank's block (allocated), its global offsets and the global dims. */
slapcu_status slapcu_read_cb2b(slapcu_comm comm, const char* path, int pr, int pc, slapcu_csc_out* out,
                               int64_t* out_row_start, int64_t* out_col_start, int64_t* nrows, int64_t* ncols);

#ifdef __cplusplus
}
#endif
#endif /* SLAPCU_H */
