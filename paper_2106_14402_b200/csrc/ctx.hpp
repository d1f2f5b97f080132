// ctx.hpp -- host-side context, workspace and launch bookkeeping shared by
// the CUDA translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <functional>
#include <string>
#include <tuple>
#include <utility>
#include <vector>

#include "common.cuh"
#include "slapcu.h"

struct slapcu_ctx_s;

namespace slapcu {

// Device CSC view (colptr int64, rowids int32, typed values).
// colptr values may be offset (a column window of a larger matrix): entries
// of column j live at rw[cp[j] .. cp[j+1]).  `base` = cp[0] and `span` =
// cp[ncols] - cp[0] are filled on the host by resolve() before launches.
struct DevCsc {
    int64_t nrows = 0, ncols = 0, nnz = 0;
    const int64_t* cp = nullptr;
    const int32_t* rw = nullptr;
    const void* v = nullptr;
    int64_t base = 0, span = 0;
};

inline DevCsc view(const slapcu_csc& m) { return DevCsc{m.nrows, m.ncols, m.nnz, m.colptr, m.rowids, m.vals}; }

// Stream-ordered device buffer from the default memory pool.
class DevBuf {
public:
    DevBuf() = default;
    DevBuf(size_t bytes, cudaStream_t s) : s_(s) { alloc(bytes); }
    ~DevBuf() { release(); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p_(o.p_), n_(o.n_), s_(o.s_) { o.p_ = nullptr; o.n_ = 0; }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) {
            release();
            p_ = o.p_;
            n_ = o.n_;
            s_ = o.s_;
            o.p_ = nullptr;
            o.n_ = 0;
        }
        return *this;
    }
    void reset(size_t bytes, cudaStream_t s) {
        if (bytes <= n_ && p_) { s_ = s; return; }
        release();
        s_ = s;
        alloc(bytes);
    }
    template <class T>
    T* as() const { return static_cast<T*>(p_); }
    void* get() const { return p_; }
    size_t size() const { return n_; }
    void release() {
        if (p_) cudaFreeAsync(p_, s_);
        p_ = nullptr;
        n_ = 0;
    }
    void* detach() { void* p = p_; p_ = nullptr; n_ = 0; return p; }

private:
    void alloc(size_t bytes) {
        if (bytes == 0) bytes = 16;
        SLAPCU_CUDA(cudaMallocAsync(&p_, bytes, s_));
        n_ = bytes;
    }
    void* p_ = nullptr;
    size_t n_ = 0;
    cudaStream_t s_ = nullptr;
};

// State carried from the symbolic phase to the numeric phase of one product.
struct Plan {
    const void* a_key = nullptr;  // identity of the operands the plan is for
    const void* b_key = nullptr;
    int64_t a_ncols = -1, b_ncols = -1, b_nnz = -1, b_base = -1;
    DevBuf flops;   // int64[B.ncols]
    DevBuf counts;  // int64[B.ncols + 1]
    DevBuf cursor;  // int32[B.nnz] per-B-entry row-tile cursors
    bool valid = false;
};

struct Bins {
    std::vector<int> count;   // per bin
    std::vector<int> offset;  // per bin
    DevBuf list;              // int32[n_nonzero]
};

// State of a fused product carried from spgemm_begin to spgemm_finish.
struct FusedState {
    bool valid = false;
    const void* a_key = nullptr;
    const void* b_key = nullptr;
    int sr = -1;
    int64_t ncols = -1, nnz = 0;
    const int64_t* colptr = nullptr;
    bool ones = false;
    DevBuf srows, svals, cnt, soff, scur, seg_off, seg_cnt, items;
    Bins bins;
    int nlight_bins = 0, tile_log2 = 0, T = 0;
};

struct Options {
    int tile_rows_log2 = 18;      // numeric dense-tile height
    int sym_tile_rows_log2 = 19;  // symbolic bitmap height
    int64_t light_nnz_max = 4096;     // numeric hash path if nnz <= this
    int64_t light_flops_max = 16384;  // symbolic hash path if flops <= this
    // fused byte-flag path if flops >= this (-1 auto = nrows/4, 0 off).  Off by
    // default: measured slower than the bitmap path at R-MAT s20 (8 row tiles
    // of byte flags re-walk B per tile and the separate launch serialises).
    int64_t dense_flops_min = 0;
    int dense_tile_rows_log2 = 17;    // byte-flag tile height (128 KB of flags)
    bool async_finish = false;        // finish() returns without waiting (errors surface later)
    int direct_tile_rows_log2 = 0;    // direct path: row-tile height of an item (0 = auto: 17, 18 above 2^20 rows)
    int64_t direct_light_flops_max = 1024;  // direct path: hash path for columns up to this many flops
    int64_t direct_dense_run_min = 4096;    // direct path: A runs (column x tile) this long are OR-ed
                                            // as precomputed tile bitmaps (0 = never)
    int direct_value_tile_log2 = 13;        // direct path value pass: rows per shared value array
    int direct_values_fallback = 0;
    int summa_concat = 1;                   // SUMMA: one concatenated-k product per call (no stage merge)
    int direct_value_threads = 512;
    int direct_value_hash = -1;  // -1 auto: off for 4-byte values (rank chunks take every item), 13 for 8-byte
    int direct_value_interleave = 1;       // value pass: values gathered with their rows (0 off, 1 4-byte, 2 all)
    int direct_value_rank = -1;  // value pass: large items by rank chunks of this many outputs (0 = sub-tiles,
                                 // -1 = by accumulator width: 10240 for 4-byte, 4096 for 8-byte)
    int direct_tile_major = 1;              // form: work units ordered by row tile, then heaviest first
    int deterministic = 0;                  // 1: every product by ESC (the reference's fold order, bit-exact fp)
    int direct_esc = -1;                    // 1: ESC for every semiring, 0: bitmap / hash paths, -1 auto (value
                                            // semirings with sampled compression < 2 take ESC)
    int direct_words = 1;                   // form: walk A's (32-row word, mask) pairs instead of its rows
    int direct_value_dense_rows = 0;        // value pass: chunks spanning <= this many rows fold by row offset (0 = cap)
    int direct_value_tmajor = 1;            // value pass: tile-major 4096-row pointer table + chunks in row order
    int direct_value_rows = 0;              // 1: value pass writes C's rows too (emit skipped; measured slower)
    int direct_value_tiny_run = -1;         // value walks: runs this short folded by their own thread (-1 default)
    int direct_value_form = 0;              // value semirings: one walk folding values in a 2^v-row tile
                                            // (-1 auto: 14 for <= 4-byte accumulators, 13 for 8; 0 = value pass)
    int direct_short_run = 0;               // form: runs shorter than this walked per thread (0 = default 8)
    int direct_persistent = 1;              // form kernel: persistent CTAs (1) or one CTA per unit (0)
    int direct_form_threads = 256;          // CTA size of the form kernel (128, 256, 512)
    int direct_emit_threads = 128;          // CTA size of the emit kernel (128, 256)
    int64_t direct_split_flops = 1 << 20;  // direct path: items above this many multiplies are
                                          // formed by several CTAs (equal-flops B-entry parts)
};

// Workspace of the direct (in-place) path, kept across calls.
struct DirectCache {
    FusedState light;  // light columns: staged hash output (fused.cu kernels)
    DevBuf atp;        // A tile pointers int32[A.ncols][T+1]
    uint64_t atp_key = 0;  // pattern fingerprint of the A they were built for (pattern_fingerprint)
    int64_t atp_ncols = -1, atp_nnz = -1;
    int atp_tl = -1;
    bool atp_valid = false;
    DevBuf dslot, dbm;  // dense A runs: slot per (k, tile), tile bitmaps
    DevBuf aw, awcp, watp;  // word form of A: (word, mask) pairs, their colptr, word tile pointers
    uint64_t aw_key = 0;
    int aw_tl = -1;
    int64_t aw_ncols = -1;
    bool aw_valid = false;
    DevBuf atpv;        // A tile pointers at the value-pass sub-tile height
    uint64_t atpv_key = 0;
    int64_t atpv_ncols = -1, atpv_nnz = -1;
    int atpv_tl = -1;
    bool atpv_valid = false;
    bool atpv_tmajor = false;
    int ndense = 0, dense_min = -1;
    DevBuf lp, hcnt, hl, items, ifl, sres, soff, units, order, stash, partial, cnt, form, hoff, rbc;
    DevBuf dist_rw, dist_v;  // SUMMA concatenated product: bound-sized output scratch
    DevBuf eblocks;          // emit work list: (item, block) pairs
    int64_t last_nnz = -1;  // exact nnz(C) of the last call (also on BudgetError)
    int64_t nunits = 0;     // form work units of the last call (the L2 value pass reuses them)
};

// Kernel classes for the per-class device-time breakdown (profiling mode).
enum KClass {
    KC_OTHER = 0,
    KC_FLOPS,
    KC_BIN,
    KC_SYM_LIGHT,
    KC_SYM_HEAVY,
    KC_SCAN,
    KC_NUM_LIGHT,
    KC_NUM_HEAVY,
    KC_MERGE,
    KC_GEN,
    KC_COUNT
};

struct Prof {
    bool on = false;
    std::vector<std::tuple<int, cudaEvent_t, cudaEvent_t>> pending;
    std::vector<cudaEvent_t> pool;
    double ms[KC_COUNT] = {};
    int64_t n[KC_COUNT] = {};
};

struct Ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    int64_t launches = 0;
    Options opt;
    Plan plan;
    FusedState fused;
    DirectCache direct;
    std::string last_error;
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
    float sym_ms = 0.f, num_ms = 0.f;
    int smem_optin = 0;
    int num_sms = 0;
    Prof prof;
    int cur_cls = KC_OTHER;
    int* err_host = nullptr;   // pinned, deferred error flag of an async finish()
    bool err_pending = false;
    DevBuf err_flag;      // int
    DevBuf scratch_small; // misc small counters
    // host batched path: pinned read-back buffers, grown on demand and kept
    struct {
        void* pinned[2] = {nullptr, nullptr};
        size_t bytes[2] = {0, 0};
    } host;
    // merge state carried from merge_symbolic to merge_numeric
    struct {
        DevBuf ranks, tot, counts;
        const void* key0 = nullptr;
        int q = 0;
        int64_t ncols = -1;
    } merge;
};

Ctx& ctx_of(slapcu_ctx c);

// Device memory a new workspace can take: what the driver reports free plus
// what the stream-ordered pool holds cached but unused (the pool keeps freed
// workspace, release threshold = max) -- sizing by the free memory alone made
// the ESC group size depend on what earlier products left cached.
inline size_t device_available(const Ctx& c) {
    size_t fr = 0, tot = 0;
    if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) return 0;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, c.device) == cudaSuccess) {
        uint64_t reserved = 0, used = 0;
        if (cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved) == cudaSuccess &&
            cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used) == cudaSuccess && reserved > used)
            fr += size_t(reserved - used);
    }
    return fr;
}

// Reads cp[0] and cp[ncols] (synchronizes the context stream).
void resolve(Ctx& c, DevCsc& m);
uint64_t pattern_fingerprint(Ctx& c, const DevCsc& m);  // resolved m

// spgemm.cu
void spgemm_flops(Ctx& c, const DevCsc& A, const DevCsc& B, int64_t* flops_dev, int64_t* total);
int64_t spgemm_symbolic(Ctx& c, const DevCsc& A, const DevCsc& B, int alg, int64_t* c_colptr);
void spgemm_numeric(Ctx& c, const DevCsc& A, const DevCsc& B, int sr, int alg, const int64_t* c_colptr,
                    int32_t* c_rowids, void* c_vals);
// fused.cu: single-product-pass begin/finish
int64_t fused_begin(Ctx& c, const DevCsc& A, const DevCsc& B, int sr, int alg, int64_t* c_colptr,
                    int64_t staging_budget_bytes);
void fused_finish(Ctx& c, const DevCsc& A, const DevCsc& B, int sr, int32_t* c_rowids, void* c_vals);
void ctx_settle(Ctx& c);
// fused.cu helpers shared with the direct path
void fused_light_launch(Ctx& c, int sr, bool ones, int bin, const DevCsc& A, const DevCsc& B, const int* list, int n,
                        const int64_t* flops, FusedState& f);
void fused_copy_light(Ctx& c, int sr, bool ones, const int* list, int n, const FusedState& f, const int64_t* c_colptr,
                      int32_t* c_rowids, void* c_vals);
// direct.cu: single product pass straight into C; direct_exact returns exactly
// sized library-owned buffers (false when the bound-sized scratch exceeds budget)
bool direct_exact(Ctx& c, const DevCsc& A, const DevCsc& B, int sr, int alg, int64_t budget, int64_t** colptr,
                  int32_t** rowids, void** vals, int64_t* nnz, bool copy_out = true);
// host.cu: batched product of host operands, per-batch host consumer
int64_t batched_host(Ctx& c, const slapcu_host_csc& A, const slapcu_host_csc& B, int sr, int alg, int nranges,
                     const int64_t* ranges, int64_t budget, slapcu_batch_consumer consumer, void* user);
void free_host_cache(Ctx& c);
// esc.cu: expand / stable segmented sort / left fold (reference fold order)
int64_t esc_spgemm(Ctx& c, const DevCsc& A, const DevCsc& B, int sr, int64_t capacity, int64_t* c_colptr, int32_t* crw,
                   void* cv);
int64_t direct_spgemm(Ctx& c, const DevCsc& A, const DevCsc& B, int sr, int alg, int64_t capacity, int64_t* c_colptr,
                      int32_t* c_rowids, void* c_vals);
void any_zero_u8(Ctx& c, const uint8_t* v, int64_t n, int* flag);
void dcsc_colptr(Ctx& c, int64_t ncols, int64_t nzc, const int32_t* jc, const int32_t* cp, int64_t* colptr);
void exclusive_scan_i64(Ctx& c, const int64_t* in, int64_t* out, int64_t n);

// mcl.cu: algorithms.cpp:267-293 mcl_step around the direct product
void mcl_step(Ctx& c, const DevCsc& A, int sr, double inflation, double prune, slapcu_csc_out* out);
void mcl_block_colsums(Ctx& c, const DevCsc& A, int sr, double* sums);
bool mcl_sums_bad(Ctx& c, const double* sums, int64_t n, double tol);
void mcl_block_epilogue(Ctx& c, const DevCsc& E, int sr, double inflation, double prune,
                        const std::function<void(double*, int64_t)>& reduce, slapcu_csc_out* out);

// merge.cu
int64_t merge_symbolic(Ctx& c, int nparts, const DevCsc* parts, int64_t* c_colptr);
void merge_numeric(Ctx& c, int nparts, const DevCsc* parts, int sr, const int64_t* c_colptr, int32_t* c_rowids,
                   void* c_vals);

// gen.cu
void gen_rmat(Ctx& c, int scale, int ef, uint64_t seed, double a, double b, double cc, double d, slapcu_csc_out* out);
void gen_er(Ctx& c, int64_t n, int64_t draws, uint64_t seed, bool with_values, slapcu_csc_out* out);
void gen_one_per_row(Ctx& c, int64_t n, int64_t ncols, uint64_t seed, slapcu_csc_out* out);
void fill_values(Ctx& c, int sr, int kind, const DevCsc& m, void* vals);
void permute_symmetric(Ctx& c, const DevCsc& A, uint64_t seed, int sr, slapcu_csc_out* out);
void slice_cols(Ctx& c, const DevCsc& B, int sr, int64_t c0, int64_t c1, slapcu_csc_out* out);
void column_checksums(Ctx& c, const DevCsc& m, int sr, bool with_values, uint64_t* sums);

// ---- profiling: CUDA events around every launch on the context stream

inline cudaEvent_t prof_event(Ctx& c) {
    if (!c.prof.pool.empty()) {
        cudaEvent_t e = c.prof.pool.back();
        c.prof.pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    SLAPCU_CUDA(cudaEventCreate(&e));
    return e;
}

// Resolves recorded event pairs into the per-class totals (synchronizes).
inline void prof_flush(Ctx& c) {
    for (auto& [cls, a, b] : c.prof.pending) {
        cudaEventSynchronize(b);
        float t = 0.f;
        cudaEventElapsedTime(&t, a, b);
        c.prof.ms[cls] += t;
        c.prof.n[cls] += 1;
        c.prof.pool.push_back(a);
        c.prof.pool.push_back(b);
    }
    c.prof.pending.clear();
}

// Enqueues f() (one or more launches) bracketed by events when profiling.
template <class F>
inline void timed(Ctx& c, int cls, F&& f) {
    if (!c.prof.on) {
        f();
        return;
    }
    cudaEvent_t a = prof_event(c), b = prof_event(c);
    SLAPCU_CUDA(cudaEventRecord(a, c.stream));
    f();
    SLAPCU_CUDA(cudaEventRecord(b, c.stream));
    c.prof.pending.emplace_back(cls, a, b);
}

struct KScope {
    Ctx& c;
    int prev;
    KScope(Ctx& c_, int k) : c(c_), prev(c_.cur_cls) { c.cur_cls = k; }
    ~KScope() { c.cur_cls = prev; }
};

template <class K, class... Args>
inline void launch(Ctx& c, K kernel, dim3 grid, dim3 block, size_t smem, Args... args) {
    if (grid.x == 0 || grid.y == 0 || grid.z == 0) return;
    timed(c, c.cur_cls, [&] {
        kernel<<<grid, block, smem, c.stream>>>(args...);
        SLAPCU_LAUNCH_CHECK();
    });
    ++c.launches;
}

}  // namespace slapcu
