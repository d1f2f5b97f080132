/*
 * oracle.h -- CPU restatement of the reference's semiring SpGEMM hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_2106_14402_b200/)
 * links, imports or executes this code.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may call it, and only as
 * the checker or the timed CPU baseline, never as the thing measured or shipped.
 *
 * Parity of this restatement is PINNED two ways (see tests/test_oracle.py):
 *   1. the reference's own golden vectors (test_localkernels.cpp:69-142,
 *      acceptance.cpp:58-97 style randomized checks), and
 *   2. bit-for-bit comparison with the unmodified reference compiled from
 *      /root/reference/proj sources into oracle/_ref/libslapref.so
 *      (oracle/Makefile, oracle/ref_shim.cpp), plus committed fixtures in
 *      tests/golden/ generated from it.
 *
 * Every function cites the reference file:line it restates
 * (paths relative to /root/reference/proj/core/include/slap/ unless noted).
 */
#ifndef SLAP_ORACLE_H
#define SLAP_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Semiring ids: same numbering as include/slapcu.h (checked by a test). */
enum {
    ORC_PLUS_TIMES_F64 = 0, /* PlusTimes<double>       semiring.hpp:36-44 */
    ORC_PLUS_TIMES_F32 = 1, /* PlusTimes<float>        semiring.hpp:36-44 */
    ORC_PLUS_TIMES_I64 = 2, /* PlusTimes<int64_t>      semiring.hpp:36-44 */
    ORC_MIN_PLUS_I32 = 3,   /* MinPlus<int32_t>        semiring.hpp:58-74 */
    ORC_MIN_PLUS_F64 = 4,   /* MinPlus<double>         semiring.hpp:58-74 */
    ORC_OR_AND_U8 = 5       /* OrAnd (uint8 0/1)       semiring.hpp:48-56 */
};

/* CSC with 64-bit column pointers and 32-bit row ids (the device layout). */
typedef struct {
    int64_t nrows, ncols, nnz;
    int64_t* colptr; /* ncols+1 */
    int32_t* rowids; /* nnz, strictly ascending per column */
    void* vals;      /* nnz values of the semiring's type (may be NULL for pattern) */
} orc_csc;

int orc_value_size(int sr);

/* rng.hpp:12-45 (splitmix64 finalizer and counter-based stream). */
uint64_t orc_mix(uint64_t z);
uint64_t orc_rng_init(uint64_t seed, uint64_t stream);
uint64_t orc_rng_next(uint64_t* state);

/* algorithms.cpp:71-113 gen_rmat (+ distribute_triples keep-first dedup,
 * dist_matrix.hpp:89-119).  Pattern only (values are 1.0 in the reference).
 * Allocates colptr/rowids (free with orc_free). */
int orc_gen_rmat(int scale, int edge_factor, uint64_t seed, double a, double b, double c, double d,
                 orc_csc* out);

/* oracles.hpp:205-217 random_triples restated for a square n x n ER matrix:
 * `draws` (row, col, value) draws from one Rng(seed) stream, dedup keep-first,
 * values U[0,1) as double.  Allocates. */
int orc_gen_er(int64_t n, int64_t draws, uint64_t seed, orc_csc* out);

/* Value recipes: fill `vals` for the pattern of m.
 * kind 0: 1 (of the semiring type)      kind 1: U[0,1) coordinate hash
 * kind 2: 10*U[0,1)                      kind 3: int32 1 + h mod 255
 * kind 4: 1/deg(col) as the type         kind 5: small int 1..9 from hash */
int orc_fill_values(int sr, int kind, const orc_csc* m, void* vals);

/* spgemm.hpp:68-88 estimate_flops; returns total, fills per-column if non-NULL. */
int64_t orc_estimate_flops(const orc_csc* a, const orc_csc* b, int64_t* per_col);

/* spgemm.hpp:118-138 symbolic_nnz (pattern-union count per output column). */
int64_t orc_symbolic_nnz(const orc_csc* a, const orc_csc* b, int64_t* counts, int threads);

/* spgemm.hpp:275-330 local_spgemm: Gustavson by output column, each output
 * entry folded with sr.add in ascending inner index k (the order both the
 * heap, spgemm.hpp:156-159, and hash, spgemm.hpp:251-255, accumulators use),
 * rows sorted ascending.  Allocates c->colptr/rowids/vals.  Restricted to the
 * output column range [col_begin, col_end) of B when col_end > col_begin
 * (column slicing preserves every column bit-for-bit). */
int orc_spgemm(int sr, const orc_csc* a, const orc_csc* b, int64_t col_begin, int64_t col_end,
               orc_csc* c, int threads);

/* local_matrix.hpp:166-188 sort_and_combine as used by the SUMMA / 3D merge
 * (summa.hpp:145-156, spgemm3d.hpp:257-262): the parts are appended in order,
 * stable-sorted by (col,row) and duplicates left-folded with sr.add.  All parts
 * share one shape.  Allocates. */
int orc_merge(int sr, int nparts, const orc_csc* parts, orc_csc* out);

/* Per-column 64-bit checksums of (row, value bits) used for size-independent
 * parity at full scale. */
void orc_column_checksums(int sr, const orc_csc* m, uint64_t* sums);

void orc_free(void* p);

#ifdef __cplusplus
}
#endif
#endif
