/*
 * oracle.c -- CPU restatement of the reference SpGEMM hot path (TEST
 * INFRASTRUCTURE ONLY; see oracle.h for the rules and the pinning).
 *
 * Reference paths are relative to /root/reference/proj/core/include/slap/
 * unless prefixed.
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define GOLDEN 0x9e3779b97f4a7c15ULL

/* ------------------------------------------------------------ rng.hpp:12-45 */

uint64_t orc_mix(uint64_t z) { /* rng.hpp:34-41 */
    z ^= z >> 30;
    z *= 0xbf58476d1ce4e5b9ULL;
    z ^= z >> 27;
    z *= 0x94d049bb133111ebULL;
    z ^= z >> 31;
    return z;
}

uint64_t orc_rng_init(uint64_t seed, uint64_t stream) { /* rng.hpp:16-17 */
    return orc_mix(seed * GOLDEN + stream + 1);
}

uint64_t orc_rng_next(uint64_t* state) { /* rng.hpp:19-22 */
    *state += GOLDEN;
    return orc_mix(*state);
}

static double rng_next_double(uint64_t* s) { /* rng.hpp:26-28 */
    return (double)(orc_rng_next(s) >> 11) * 0x1.0p-53;
}

int orc_value_size(int sr) {
    switch (sr) {
    case ORC_PLUS_TIMES_F64: return 8;
    case ORC_PLUS_TIMES_F32: return 4;
    case ORC_PLUS_TIMES_I64: return 8;
    case ORC_MIN_PLUS_I32: return 4;
    case ORC_MIN_PLUS_F64: return 8;
    case ORC_OR_AND_U8: return 1;
    }
    return 0;
}

void orc_free(void* p) { free(p); }

/* ------------------------------------------------ COO -> canonical CSC build */

typedef struct {
    uint64_t key; /* col << 32 | row */
    int64_t e;    /* draw index (keep-first tie break) */
    double v;
} ent_t;

static int cmp_ent(const void* x, const void* y) {
    const ent_t* a = (const ent_t*)x;
    const ent_t* b = (const ent_t*)y;
    if (a->key != b->key) return (a->key > b->key) - (a->key < b->key);
    return (a->e > b->e) - (a->e < b->e);
}

static int cmp_u32(const void* x, const void* y) {
    uint32_t a = *(const uint32_t*)x, b = *(const uint32_t*)y;
    return (a > b) - (a < b);
}

/* Pattern-only canonical CSC from (col<<32|row) keys: sort rows inside each
 * column, drop repeats (distribute_triples keep-first, dist_matrix.hpp:89-119;
 * build_dcsc, local_matrix.hpp:207-221). */
static int keys_to_csc(const uint64_t* keys, int64_t m, int64_t n, orc_csc* out) {
    int64_t* colptr = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
    uint32_t* rows = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(m ? m : 1));
    int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n ? n : 1));
    int64_t* newptr = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
    int32_t* outrows = (int32_t*)malloc(sizeof(int32_t) * (size_t)(m ? m : 1));
    if (!colptr || !rows || !fill || !newptr || !outrows) return -1;
    for (int64_t e = 0; e < m; ++e) colptr[(keys[e] >> 32) + 1]++;
    for (int64_t j = 0; j < n; ++j) colptr[j + 1] += colptr[j];
    memcpy(fill, colptr, sizeof(int64_t) * (size_t)n);
    for (int64_t e = 0; e < m; ++e) {
        int64_t j = (int64_t)(keys[e] >> 32);
        rows[fill[j]++] = (uint32_t)(keys[e] & 0xffffffffULL);
    }
    free(fill);
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t j = 0; j < n; ++j) {
        int64_t b = colptr[j], e = colptr[j + 1];
        if (e - b > 1) qsort(rows + b, (size_t)(e - b), sizeof(uint32_t), cmp_u32);
        int64_t u = 0;
        for (int64_t i = b; i < e; ++i)
            if (i == b || rows[i] != rows[i - 1]) rows[b + u++] = rows[i];
        newptr[j + 1] = u;
    }
    for (int64_t j = 0; j < n; ++j) newptr[j + 1] += newptr[j];
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t j = 0; j < n; ++j) {
        int64_t cnt = newptr[j + 1] - newptr[j];
        for (int64_t i = 0; i < cnt; ++i) outrows[newptr[j] + i] = (int32_t)rows[colptr[j] + i];
    }
    free(rows);
    free(colptr);
    out->ncols = n;
    out->nnz = newptr[n];
    out->colptr = newptr;
    out->rowids = outrows;
    out->vals = NULL;
    return 0;
}

/* --------------------------------------------- algorithms.cpp:71-113 gen_rmat */

int orc_gen_rmat(int scale, int edge_factor, uint64_t seed, double a, double b, double c, double d,
                 orc_csc* out) {
    if (scale < 1 || scale > 30) return -1;
    (void)d;
    const int64_t n = (int64_t)1 << scale;
    const int64_t edges = (int64_t)edge_factor * n;
    const double ab = a + b, abc = ab + c; /* algorithms.cpp:89-90 */
    uint64_t* keys = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(2 * edges));
    if (!keys) return -1;
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < edges; ++e) {
        /* algorithms.cpp:92-93: Rng(seed, e + 0x524d4154) per edge */
        uint64_t st = orc_rng_init(seed, (uint64_t)e + 0x524d4154ULL);
        int64_t i = 0, j = 0;
        for (int level = 0; level < scale; ++level) { /* algorithms.cpp:95-107 */
            const double u = rng_next_double(&st);
            int qi = 0, qj = 0;
            if (u < a) {
            } else if (u < ab) {
                qj = 1;
            } else if (u < abc) {
                qi = 1;
            } else {
                qi = 1;
                qj = 1;
            }
            i = (i << 1) | qi;
            j = (j << 1) | qj;
        }
        if (i == j) { /* algorithms.cpp:108: no self loops */
            keys[2 * e] = ~0ULL;
            keys[2 * e + 1] = ~0ULL;
        } else { /* algorithms.cpp:109-110: symmetrize */
            keys[2 * e] = ((uint64_t)j << 32) | (uint64_t)i;
            keys[2 * e + 1] = ((uint64_t)i << 32) | (uint64_t)j;
        }
    }
    int64_t m = 0;
    for (int64_t e = 0; e < 2 * edges; ++e)
        if (keys[e] != ~0ULL) keys[m++] = keys[e];
    out->nrows = n;
    int rc = keys_to_csc(keys, m, n, out);
    free(keys);
    return rc;
}

/* ----------------------------------- oracles.hpp:205-217 random_triples (ER) */

int orc_gen_er(int64_t n, int64_t draws, uint64_t seed, orc_csc* out) {
    ent_t* es = (ent_t*)malloc(sizeof(ent_t) * (size_t)(draws ? draws : 1));
    if (!es || n <= 0) return -1;
    const uint64_t st0 = orc_rng_init(seed, 0);
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < draws; ++e) {
        /* oracles.hpp:212-214: row, col, value drawn in that order from one
         * stream; after k calls the splitmix state is st0 + k*GOLDEN */
        uint64_t s = st0 + (uint64_t)(3 * e) * GOLDEN;
        uint64_t r = orc_rng_next(&s) % (uint64_t)n;
        uint64_t cc = orc_rng_next(&s) % (uint64_t)n;
        double v = (double)(orc_rng_next(&s) >> 11) * 0x1.0p-53;
        es[e].key = (cc << 32) | r;
        es[e].e = e;
        es[e].v = v;
    }
    qsort(es, (size_t)draws, sizeof(ent_t), cmp_ent);
    int64_t* colptr = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
    int32_t* rows = (int32_t*)malloc(sizeof(int32_t) * (size_t)(draws ? draws : 1));
    double* vals = (double*)malloc(sizeof(double) * (size_t)(draws ? draws : 1));
    int64_t m = 0;
    for (int64_t e = 0; e < draws; ++e) {
        if (e > 0 && es[e].key == es[e - 1].key) continue; /* keep first draw */
        rows[m] = (int32_t)(es[e].key & 0xffffffffULL);
        vals[m] = es[e].v;
        colptr[(es[e].key >> 32) + 1]++;
        ++m;
    }
    for (int64_t j = 0; j < n; ++j) colptr[j + 1] += colptr[j];
    free(es);
    out->nrows = n;
    out->ncols = n;
    out->nnz = m;
    out->colptr = colptr;
    out->rowids = rows;
    out->vals = vals;
    return 0;
}

/* ---------------------------------------------------------- value recipes */

static inline uint64_t coord_hash(int64_t i, int64_t j) {
    return orc_mix(((uint64_t)i << 32) ^ (uint64_t)j);
}

int orc_fill_values(int sr, int kind, const orc_csc* m, void* vals) {
#pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t j = 0; j < m->ncols; ++j) {
        const int64_t b = m->colptr[j], e = m->colptr[j + 1];
        const int64_t deg = e - b;
        for (int64_t p = b; p < e; ++p) {
            const int64_t i = m->rowids[p];
            const uint64_t h = coord_hash(i, j);
            const double u = (double)(h >> 11) * 0x1.0p-53;
            double dv;
            int64_t iv;
            switch (kind) {
            case 0: dv = 1.0; iv = 1; break;
            case 1: dv = u; iv = 1 + (int64_t)(h % 255); break;
            case 2: dv = 10.0 * u; iv = 1 + (int64_t)(h % 255); break;
            case 3: iv = 1 + (int64_t)(h % 255); dv = (double)iv; break;
            case 4: dv = 1.0 / (double)deg; iv = 1; break;
            case 5: iv = 1 + (int64_t)(h % 9); dv = (double)iv; break;
            default: dv = 1.0; iv = 1; break;
            }
            switch (sr) {
            case ORC_PLUS_TIMES_F64:
            case ORC_MIN_PLUS_F64: ((double*)vals)[p] = dv; break;
            case ORC_PLUS_TIMES_F32:
                ((float*)vals)[p] = (kind == 4) ? 1.0f / (float)deg : (float)dv;
                break;
            case ORC_PLUS_TIMES_I64: ((int64_t*)vals)[p] = iv; break;
            case ORC_MIN_PLUS_I32: ((int32_t*)vals)[p] = (int32_t)iv; break;
            case ORC_OR_AND_U8: ((uint8_t*)vals)[p] = 1; break;
            }
        }
    }
    return 0;
}

/* ------------------------------------------- spgemm.hpp:68-88 estimate_flops */

int64_t orc_estimate_flops(const orc_csc* a, const orc_csc* b, int64_t* per_col) {
    int64_t total = 0;
#pragma omp parallel for schedule(dynamic, 1024) reduction(+ : total)
    for (int64_t j = 0; j < b->ncols; ++j) {
        int64_t f = 0;
        for (int64_t p = b->colptr[j]; p < b->colptr[j + 1]; ++p) {
            const int64_t k = b->rowids[p];
            f += a->colptr[k + 1] - a->colptr[k];
        }
        if (per_col) per_col[j] = f;
        total += f;
    }
    return total;
}

/* -------------------------------------------- spgemm.hpp:118-138 symbolic_nnz */

int64_t orc_symbolic_nnz(const orc_csc* a, const orc_csc* b, int64_t* counts, int threads) {
    int64_t total = 0;
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#else
    (void)threads;
#endif
#pragma omp parallel reduction(+ : total)
    {
        /* PatternSpa (spgemm.hpp:94-112): flags + touched list */
        char* seen = (char*)calloc((size_t)a->nrows + 1, 1);
        int32_t* touched = (int32_t*)malloc(sizeof(int32_t) * (size_t)(a->nrows + 1));
#pragma omp for schedule(dynamic, 64)
        for (int64_t j = 0; j < b->ncols; ++j) {
            int64_t cnt = 0;
            for (int64_t p = b->colptr[j]; p < b->colptr[j + 1]; ++p) {
                const int64_t k = b->rowids[p];
                for (int64_t q = a->colptr[k]; q < a->colptr[k + 1]; ++q) {
                    const int32_t r = a->rowids[q];
                    if (!seen[r]) {
                        seen[r] = 1;
                        touched[cnt++] = r;
                    }
                }
            }
            for (int64_t t = 0; t < cnt; ++t) seen[touched[t]] = 0;
            counts[j] = cnt;
            total += cnt;
        }
        free(seen);
        free(touched);
    }
    return total;
}

/* ------------------------------------------ spgemm.hpp:275-330 local_spgemm */

/* Semiring algebra, semiring.hpp:36-74. */
#define DEFINE_SR(NAME, T, MUL, ADD)                                        \
    static inline T NAME##_mul(T a, T b) { return MUL; }                    \
    static inline T NAME##_add(T a, T b) { return ADD; }

DEFINE_SR(ptf64, double, a * b, a + b)
DEFINE_SR(ptf32, float, a * b, a + b)
DEFINE_SR(pti64, int64_t, (int64_t)((uint64_t)a * (uint64_t)b), (int64_t)((uint64_t)a + (uint64_t)b))
DEFINE_SR(mpi32, int32_t, (int32_t)((uint32_t)a + (uint32_t)b), (a < b ? a : b))
DEFINE_SR(mpf64, double, a + b, (a < b ? a : b))
DEFINE_SR(oru8, uint8_t, (uint8_t)((a && b) ? 1 : 0), (uint8_t)((a || b) ? 1 : 0))

/* One output column, Gustavson with a dense SPA: entries are created by the
 * first product and folded with add in ascending k (B(:,j) is row-sorted),
 * which is the accumulation order of spgemm_heap_column (spgemm.hpp:156-199)
 * and spgemm_hash_column (spgemm.hpp:251-255); rows are then emitted ascending
 * (spgemm.hpp:259-264).  Returns the column's nnz. */
#define DEFINE_COLUMN(NAME, T)                                                                   \
    static int64_t NAME##_column(const orc_csc* a, const orc_csc* b, int64_t j, char* seen,      \
                                 int32_t* touched, T* acc, int32_t* out_rows, T* out_vals) {     \
        const T* av = (const T*)a->vals;                                                         \
        const T* bv = (const T*)b->vals;                                                         \
        int64_t cnt = 0;                                                                         \
        for (int64_t p = b->colptr[j]; p < b->colptr[j + 1]; ++p) {                              \
            const int64_t k = b->rowids[p];                                                      \
            const T bval = bv[p];                                                                \
            for (int64_t q = a->colptr[k]; q < a->colptr[k + 1]; ++q) {                          \
                const int32_t r = a->rowids[q];                                                  \
                const T prod = NAME##_mul(av[q], bval);                                          \
                if (!seen[r]) {                                                                  \
                    seen[r] = 1;                                                                 \
                    acc[r] = prod;                                                               \
                    touched[cnt++] = r;                                                          \
                } else {                                                                         \
                    acc[r] = NAME##_add(acc[r], prod);                                           \
                }                                                                                \
            }                                                                                    \
        }                                                                                        \
        if (cnt > 1) qsort(touched, (size_t)cnt, sizeof(int32_t), cmp_i32);                      \
        for (int64_t t = 0; t < cnt; ++t) {                                                      \
            const int32_t r = touched[t];                                                        \
            if (out_rows) {                                                                      \
                out_rows[t] = r;                                                                 \
                out_vals[t] = acc[r];                                                            \
            }                                                                                    \
            seen[r] = 0;                                                                         \
        }                                                                                        \
        return cnt;                                                                              \
    }

static int cmp_i32(const void* x, const void* y) {
    int32_t a = *(const int32_t*)x, b = *(const int32_t*)y;
    return (a > b) - (a < b);
}

DEFINE_COLUMN(ptf64, double)
DEFINE_COLUMN(ptf32, float)
DEFINE_COLUMN(pti64, int64_t)
DEFINE_COLUMN(mpi32, int32_t)
DEFINE_COLUMN(mpf64, double)
DEFINE_COLUMN(oru8, uint8_t)

static int64_t run_column(int sr, const orc_csc* a, const orc_csc* b, int64_t j, char* seen, int32_t* touched,
                          void* acc, int32_t* out_rows, void* out_vals) {
    switch (sr) {
    case ORC_PLUS_TIMES_F64: return ptf64_column(a, b, j, seen, touched, (double*)acc, out_rows, (double*)out_vals);
    case ORC_PLUS_TIMES_F32: return ptf32_column(a, b, j, seen, touched, (float*)acc, out_rows, (float*)out_vals);
    case ORC_PLUS_TIMES_I64: return pti64_column(a, b, j, seen, touched, (int64_t*)acc, out_rows, (int64_t*)out_vals);
    case ORC_MIN_PLUS_I32: return mpi32_column(a, b, j, seen, touched, (int32_t*)acc, out_rows, (int32_t*)out_vals);
    case ORC_MIN_PLUS_F64: return mpf64_column(a, b, j, seen, touched, (double*)acc, out_rows, (double*)out_vals);
    case ORC_OR_AND_U8: return oru8_column(a, b, j, seen, touched, (uint8_t*)acc, out_rows, (uint8_t*)out_vals);
    }
    return -1;
}

int orc_spgemm(int sr, const orc_csc* a, const orc_csc* b, int64_t col_begin, int64_t col_end, orc_csc* c,
               int threads) {
    if (a->ncols != b->nrows) return -2; /* DimError, spgemm.hpp:57-64 */
    const int vs = orc_value_size(sr);
    if (vs == 0) return -3;
    if (col_end <= col_begin) {
        col_begin = 0;
        col_end = b->ncols;
    }
    const int64_t nc = col_end - col_begin;
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#else
    (void)threads;
#endif
    /* phase 2: symbolic counts (spgemm.hpp:287) -> colptr (spgemm.hpp:289-293,
     * 64-bit here: the reference's int32 colptr overflows at 2^31) */
    int64_t* colptr = (int64_t*)calloc((size_t)nc + 1, sizeof(int64_t));
    if (!colptr) return -1;
    int fail = 0;
#pragma omp parallel
    {
        char* seen = (char*)calloc((size_t)a->nrows + 1, 1);
        int32_t* touched = (int32_t*)malloc(sizeof(int32_t) * (size_t)(a->nrows + 1));
        void* acc = malloc((size_t)vs * (size_t)(a->nrows + 1));
        if (!seen || !touched || !acc) fail = 1;
#pragma omp for schedule(dynamic, 16)
        for (int64_t j = 0; j < nc; ++j) {
            if (fail) continue;
            colptr[j + 1] = run_column(sr, a, b, col_begin + j, seen, touched, acc, NULL, NULL);
        }
        free(seen);
        free(touched);
        free(acc);
    }
    if (fail) return -1;
    for (int64_t j = 0; j < nc; ++j) colptr[j + 1] += colptr[j];
    const int64_t total = colptr[nc];
    int32_t* rows = (int32_t*)malloc(sizeof(int32_t) * (size_t)(total ? total : 1));
    void* vals = malloc((size_t)vs * (size_t)(total ? total : 1));
    if (!rows || !vals) return -1;
    /* phase 3: numeric */
#pragma omp parallel
    {
        char* seen = (char*)calloc((size_t)a->nrows + 1, 1);
        int32_t* touched = (int32_t*)malloc(sizeof(int32_t) * (size_t)(a->nrows + 1));
        void* acc = malloc((size_t)vs * (size_t)(a->nrows + 1));
#pragma omp for schedule(dynamic, 16)
        for (int64_t j = 0; j < nc; ++j) {
            int64_t got = run_column(sr, a, b, col_begin + j, seen, touched, acc, rows + colptr[j],
                                     (char*)vals + (size_t)vs * (size_t)colptr[j]);
            if (got != colptr[j + 1] - colptr[j]) fail = 2; /* spgemm.hpp:323-324 */
        }
        free(seen);
        free(touched);
        free(acc);
    }
    c->nrows = a->nrows;
    c->ncols = nc;
    c->nnz = total;
    c->colptr = colptr;
    c->rowids = rows;
    c->vals = vals;
    return fail ? -4 : 0;
}

/* ---------------------------- local_matrix.hpp:166-188 sort_and_combine merge */

#define DEFINE_FOLD(NAME, T)                                                   \
    static void NAME##_fold(void* acc, const void* v) {                        \
        *(T*)acc = NAME##_add(*(T*)acc, *(const T*)v);                          \
    }
DEFINE_FOLD(ptf64, double)
DEFINE_FOLD(ptf32, float)
DEFINE_FOLD(pti64, int64_t)
DEFINE_FOLD(mpi32, int32_t)
DEFINE_FOLD(mpf64, double)
DEFINE_FOLD(oru8, uint8_t)

int orc_merge(int sr, int nparts, const orc_csc* parts, orc_csc* out) {
    if (nparts < 1) return -1;
    const int vs = orc_value_size(sr);
    void (*fold)(void*, const void*) = NULL;
    switch (sr) {
    case ORC_PLUS_TIMES_F64: fold = ptf64_fold; break;
    case ORC_PLUS_TIMES_F32: fold = ptf32_fold; break;
    case ORC_PLUS_TIMES_I64: fold = pti64_fold; break;
    case ORC_MIN_PLUS_I32: fold = mpi32_fold; break;
    case ORC_MIN_PLUS_F64: fold = mpf64_fold; break;
    case ORC_OR_AND_U8: fold = oru8_fold; break;
    default: return -3;
    }
    const int64_t n = parts[0].ncols, m = parts[0].nrows;
    for (int s = 1; s < nparts; ++s)
        if (parts[s].ncols != n || parts[s].nrows != m) return -2;
    int64_t cap = 0;
    for (int s = 0; s < nparts; ++s) cap += parts[s].nnz;
    int64_t* colptr = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
    int32_t* rows = (int32_t*)malloc(sizeof(int32_t) * (size_t)(cap ? cap : 1));
    char* vals = (char*)malloc((size_t)vs * (size_t)(cap ? cap : 1));
    if (!colptr || !rows || !vals) return -1;
    /* Per column: a stable (row, part) order is exactly what the stable sort
     * over parts appended in stage order yields (summa.hpp:145-147 append,
     * local_matrix.hpp:172-175 stable_sort); equal rows fold left in part
     * order (local_matrix.hpp:179-186). */
    int64_t o = 0;
    int64_t* pos = (int64_t*)malloc(sizeof(int64_t) * (size_t)nparts);
    for (int64_t j = 0; j < n; ++j) {
        for (int s = 0; s < nparts; ++s) pos[s] = parts[s].colptr[j];
        for (;;) {
            int best = -1;
            int32_t br = 0;
            for (int s = 0; s < nparts; ++s) {
                if (pos[s] < parts[s].colptr[j + 1]) {
                    int32_t r = parts[s].rowids[pos[s]];
                    if (best < 0 || r < br) {
                        best = s;
                        br = r;
                    }
                }
            }
            if (best < 0) break;
            rows[o] = br;
            memcpy(vals + (size_t)vs * (size_t)o, (const char*)parts[best].vals + (size_t)vs * (size_t)pos[best],
                   (size_t)vs);
            pos[best]++;
            for (int s = best + 1; s < nparts; ++s) {
                if (pos[s] < parts[s].colptr[j + 1] && parts[s].rowids[pos[s]] == br) {
                    fold(vals + (size_t)vs * (size_t)o, (const char*)parts[s].vals + (size_t)vs * (size_t)pos[s]);
                    pos[s]++;
                }
            }
            ++o;
        }
        colptr[j + 1] = o;
    }
    free(pos);
    out->nrows = m;
    out->ncols = n;
    out->nnz = o;
    out->colptr = colptr;
    out->rowids = rows;
    out->vals = vals;
    return 0;
}

/* ------------------------------------------------------------- checksums */

void orc_column_checksums(int sr, const orc_csc* m, uint64_t* sums) {
    const int vs = m->vals ? orc_value_size(sr) : 0;
#pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t j = 0; j < m->ncols; ++j) {
        uint64_t s = 0;
        for (int64_t p = m->colptr[j]; p < m->colptr[j + 1]; ++p) {
            uint64_t bits = 0;
            if (vs) memcpy(&bits, (const char*)m->vals + (size_t)vs * (size_t)p, (size_t)vs);
            s += orc_mix(((uint64_t)(uint32_t)m->rowids[p] * GOLDEN) ^ bits);
        }
        sums[j] = s;
    }
}
