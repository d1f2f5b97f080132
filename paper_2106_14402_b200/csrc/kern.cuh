// kern.cuh -- device building blocks shared by the SpGEMM translation units
// (binning spec, product walking, shared-memory hashing, group sync) and the
// host helpers that launch them.
#pragma once

#include <algorithm>
#include <vector>

#include "ctx.hpp"

namespace slapcu {

struct BinSpec {
    int nlight;            // light bins 0..nlight-1, heavy bin = nlight
    int64_t thr[12];       // light bin b holds key <= thr[b]
    int64_t light_max;     // key > light_max -> heavy
    int all_heavy;         // alg == heap
    int key_is_nnz;        // 0: key = flops[j]; 1: key = Ccp[j+1]-Ccp[j]
};

__device__ __forceinline__ int bin_of_key(const BinSpec& s, int64_t key) {
    if (key <= 0) return -1;
    if (s.all_heavy || key > s.light_max) return s.nlight;
    for (int b = 0; b < s.nlight; ++b)
        if (key <= s.thr[b]) return b;
    return s.nlight;
}

// ============================================================ product walking

// Sub-group width for walking A(:,k): the power of two closest above the
// column's mean A-column length, so short A columns do not idle a warp.
__device__ __forceinline__ int pick_sg(int64_t flops, int64_t nb, int G) {
    const int64_t avg = nb > 0 ? (flops + nb - 1) / nb : 1;
    int sg = 1;
    while (sg < avg && sg < 32 && sg < G) sg <<= 1;
    return sg;
}

template <int LOG2S>
__device__ __forceinline__ unsigned hslot(int r) {
    return ((unsigned)r * 0x9E3779B1u) >> (32 - LOG2S);
}

// Insert row id into an open-addressing table of 2^LOG2S int keys (-1 empty),
// linear probing.  Returns the slot; *is_new tells whether it was inserted.
template <int LOG2S>
__device__ __forceinline__ int hash_insert(int* keys, int r, bool* is_new) {
    constexpr unsigned MASK = (1u << LOG2S) - 1u;
    unsigned h = hslot<LOG2S>(r);
    for (;;) {
        int k = keys[h];
        if (k == r) {
            *is_new = false;
            return (int)h;
        }
        if (k == -1) {
            int old = atomicCAS(&keys[h], -1, r);
            if (old == -1) {
                *is_new = true;
                return (int)h;
            }
            if (old == r) {
                *is_new = false;
                return (int)h;
            }
        }
        h = (h + 1) & MASK;
    }
}

template <int G, int CPB>
__device__ __forceinline__ void group_sync(int g) {
    if constexpr (G == 32)
        __syncwarp();
    else if constexpr (CPB == 1)
        __syncthreads();
    else
        named_sync(1 + g, G);
}

template <int G, int CPB>
__device__ __forceinline__ long long group_sum(long long v, int g, int lane, long long* red) {
    v = warp_reduce_sum64(v);
    if constexpr (G == 32) {
        return v;
    } else {
        constexpr int W = G / 32;
        if ((lane & 31) == 0) red[g * W + (lane >> 5)] = v;
        group_sync<G, CPB>(g);
        long long s = 0;
#pragma unroll
        for (int w = 0; w < W; ++w) s += red[g * W + w];
        group_sync<G, CPB>(g);
        return s;
    }
}


// Walks the entries of A(:,k), k in B(:,j), whose rows fall in [.., t1) of
// the current row tile, starting from the per-B-entry cursor (A columns are
// row-sorted, so each tile continues where the previous one stopped).
// f(p, i, r) is called per product.  If write_cursor, the lane that owns the
// first out-of-tile position records it for the next tile.  Cursors are
// double-buffered by tile parity (read cur_in, write cur_out) so no lane can
// overwrite a start position another lane of its sub-group has yet to read.
template <class F>
__device__ __forceinline__ void walk_tile(const DevCsc& A, const DevCsc& B, int64_t bs, int64_t be, int sg, int tid,
                                          int nt, int t, int ntiles, int t1, const int32_t* __restrict__ cur_in,
                                          int32_t* __restrict__ cur_out, bool write_cursor, F&& f) {
    const int sub = tid / sg, nsub = nt / sg, sl = tid % sg;
    for (int64_t i = bs + sub; i < be; i += nsub) {
        const int k = B.rw[i];
        const int64_t as = A.cp[k], ae = A.cp[k + 1];
        if (ntiles == 1) {
            for (int64_t p = as + sl; p < ae; p += sg) f(p, i, A.rw[p]);
            continue;
        }
        const int64_t start = (t == 0) ? as : as + cur_in[i - B.base];
        int64_t p = start + sl;
        for (; p < ae; p += sg) {
            const int r = A.rw[p];
            if (r >= t1) break;
            f(p, i, r);
        }
        if (write_cursor) {
            if (p > ae) p = ae;
            const bool mine = (p == start) || (A.rw[p - 1] < t1);
            if (mine) cur_out[i - B.base] = (int32_t)(p - as);
        }
    }
}

__device__ __forceinline__ long long block_sum_ll(long long v, long long* red) {
    v = warp_reduce_sum64(v);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    long long s = 0;
    if (threadIdx.x == 0)
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += red[i];
    return s;  // valid on thread 0
}


// walk_tile with memory-level parallelism: every lane issues U independent
// row-id loads before applying f to them, so a warp keeps U sectors of A in
// flight instead of one (the product loop is L2-latency bound otherwise).
// Same contract (tile range, cursors) as walk_tile.
template <int U, class F>
__device__ __forceinline__ void walk_tile_ilp(const DevCsc& A, const DevCsc& B, int64_t bs, int64_t be, int sg,
                                              int tid, int nt, int t, int ntiles, int t1,
                                              const int32_t* __restrict__ cur_in, int32_t* __restrict__ cur_out,
                                              bool write_cursor, F&& f) {
    const int sub = tid / sg, nsub = nt / sg, sl = tid % sg;
    for (int64_t i = bs + sub; i < be; i += nsub) {
        const int k = B.rw[i];
        const int64_t as = A.cp[k], ae = A.cp[k + 1];
        const int64_t start = (ntiles == 1 || t == 0) ? as : as + cur_in[i - B.base];
        int64_t p = start + sl;
        int64_t stop = -1;
        while (stop < 0) {
            int r[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int64_t q = p + int64_t(u) * sg;
                r[u] = q < ae ? __ldg(&A.rw[q]) : INT_MAX;
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (stop < 0) {
                    if (r[u] < t1)
                        f(p + int64_t(u) * sg, i, r[u]);
                    else
                        stop = p + int64_t(u) * sg;
                }
            }
            p += int64_t(U) * sg;
        }
        if (write_cursor && ntiles > 1) {
            if (stop > ae) stop = ae;
            const bool mine = (stop == start) || (A.rw[stop - 1] < t1);
            if (mine) cur_out[i - B.base] = (int32_t)(stop - as);
        }
    }
}

// Batch functor adapting a per-product callable f(p, i, row).
template <class F>
struct PerProduct {
    F f;
    template <int U>
    __device__ __forceinline__ void batch(int64_t p, int width, int64_t i, const int* r, int ok) {
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (ok & (1 << u)) f(p + int64_t(u) * width, i, r[u]);
    }
};
template <class F>
__device__ __forceinline__ PerProduct<F> per_product(F f) {
    return PerProduct<F>{f};
}

// Products of ONE B entry i (A column k, entries [start, ae)) restricted to
// rows < t1, walked by `width` threads of which this is thread `sl`, U loads
// in flight per thread.  Returns nothing; writes the tile cursor through
// cur_out_i (may be null) from the thread that owns the first out-of-tile
// position.
template <int U, class F>
__device__ __forceinline__ void walk_entry(const int32_t* __restrict__ Arw, int64_t i, int64_t as, int64_t start,
                                           int64_t ae, int sl, int width, int t1, int32_t* cur_out_i, F&& f) {
    int64_t p = start + sl;
    int64_t stop = -1;
    while (stop < 0) {
        int r[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t q = p + int64_t(u) * width;
            r[u] = q < ae ? __ldg(&Arw[q]) : INT_MAX;
        }
        // hand the whole batch to f so it can issue its own dependent loads
        // (values) for all U products before consuming any of them
        int ok = 0;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (stop < 0) {
                if (r[u] < t1)
                    ok |= 1 << u;
                else
                    stop = p + int64_t(u) * width;
            }
        }
        f.template batch<U>(p, width, i, r, ok);
        p += int64_t(U) * width;
    }
    if (cur_out_i) {
        if (stop > ae) stop = ae;
        const bool mine = (stop == start) || (Arw[stop - 1] < t1);
        if (mine) *cur_out_i = (int32_t)(stop - as);
    }
}

// Shared state of walk_balanced (static shared memory of the caller).
struct WalkShared {
    int next;      // dynamic hand-out of short entries
    int nlong;     // long entries collected this round
    int list[1024];  // their B positions (relative to bs); >= blockDim.x
};

// Load-balanced walk of all products of column j inside one row tile.  A
// column's share of the work is its remaining length; R-MAT columns mix hub
// A columns (10^4 entries) with short ones, and a static entry->sub-group map
// leaves most warps waiting at the next barrier for the one holding the hub
// (ncu: `barrier` was the top stall).  Here entries with >= `big` remaining
// products are walked by the whole CTA cooperatively (collected NT at a time
// into shared memory), and the others are handed out to sub-groups of sg
// lanes through a shared atomic counter.  Must be called by all threads of
// the CTA (contains barriers); NT <= 1024.
template <int U, class S, class F>
__device__ __forceinline__ void walk_balanced_from(const DevCsc& A, const DevCsc& B, int64_t bs, int64_t be, int sg,
                                                   int t1, int32_t* __restrict__ cur_out, int64_t big,
                                                   WalkShared& ws, S&& start_of, F&& f);

template <int U, class F>
__device__ __forceinline__ void walk_balanced(const DevCsc& A, const DevCsc& B, int64_t bs, int64_t be, int sg,
                                              int t, int ntiles, int t1, const int32_t* __restrict__ cur_in,
                                              int32_t* __restrict__ cur_out, int64_t big, WalkShared& ws, F&& f) {
    const bool tiled = ntiles > 1;
    auto start_of = [&](int64_t i, int64_t as, int64_t) -> int64_t {
        return (!tiled || t == 0) ? as : as + cur_in[i - B.base];
    };
    walk_balanced_from<U>(A, B, bs, be, sg, t1, tiled ? cur_out : nullptr, big, ws, start_of, f);
}

// Same walk with a caller-supplied start position per B entry
// (start_of(i, as, ae) -> first position to visit); cursors are written only
// when cur_out is non-null.
template <int U, class S, class F>
__device__ __forceinline__ void walk_balanced_from(const DevCsc& A, const DevCsc& B, int64_t bs, int64_t be, int sg,
                                                   int t1, int32_t* __restrict__ cur_out, int64_t big,
                                                   WalkShared& ws, S&& start_of, F&& f) {
    const int tid = threadIdx.x, nt = blockDim.x;
    const bool tiled = cur_out != nullptr;
    const int64_t nb = be - bs;
    // phase A: long entries, whole CTA per entry
    for (int64_t base = 0; base < nb; base += nt) {
        if (tid == 0) ws.nlong = 0;
        __syncthreads();
        const int64_t i = bs + base + tid;
        if (base + tid < nb) {
            const int k = B.rw[i];
            const int64_t as = A.cp[k], ae = A.cp[k + 1];
            if (ae - start_of(i, as, ae) >= big) ws.list[atomicAdd(&ws.nlong, 1)] = (int)(base + tid);
        }
        __syncthreads();
        const int nl = ws.nlong;
        for (int li = 0; li < nl; ++li) {
            const int64_t ii = bs + ws.list[li];
            const int k = B.rw[ii];
            const int64_t as = A.cp[k], ae = A.cp[k + 1];
            walk_entry<U>(A.rw, ii, as, start_of(ii, as, ae), ae, tid, nt, t1, tiled ? cur_out + (ii - B.base) : nullptr,
                          f);
        }
        __syncthreads();
    }
    // phase B: short entries, dynamic hand-out to sub-groups
    if (tid == 0) ws.next = 0;
    __syncthreads();
    const int lane = tid & 31, sl = lane % sg, subs = 32 / sg;
    for (;;) {
        int got = 0;
        if (lane == 0) got = atomicAdd(&ws.next, subs);
        got = __shfl_sync(0xffffffffu, got, 0);
        if (got >= nb) break;
        const int64_t e = got + lane / sg;
        if (e < nb) {
            const int64_t i = bs + e;
            const int k = B.rw[i];
            const int64_t as = A.cp[k], ae = A.cp[k + 1];
            const int64_t st = start_of(i, as, ae);
            if (ae - st < big)
                walk_entry<U>(A.rw, i, as, st, ae, sl, sg, t1, tiled ? cur_out + (i - B.base) : nullptr, f);
        }
    }
    __syncthreads();
}

// Position of the n-th (0-based) set bit of w (n < popc(w)): branch-free
// halving on popcounts (the __fns intrinsic is a software loop on sm_100).
__device__ __forceinline__ int nth_set_bit(unsigned w, int n) {
    int pos = 0;
#pragma unroll
    for (int half = 16; half > 0; half >>= 1) {
        const unsigned lo = w & ((1u << half) - 1u);
        const int c = __popc(lo);
        const bool up = n >= c;
        n -= up ? c : 0;
        pos += up ? half : 0;
        w = up ? (w >> half) : lo;
    }
    return pos;
}

// Writes the set bits of a warp's 32 bitmap words (word w0+lane) as row ids
// rb_lane + bit to out[base ...] in order, 32 consecutive entries per store:
// output element o is found by a shuffle search for the lane whose exclusive
// prefix covers o, then the bit by popcount halving.
__device__ __forceinline__ void emit_rows_coalesced(unsigned bits, int row_base, int32_t* __restrict__ out,
                                                    int lane) {
    int tot;
    const int ex = warp_excl_scan(__popc(bits), lane, &tot);
    for (int o0 = 0; o0 < tot; o0 += 32) {
        const int o = o0 + lane;
        // largest lane l with ex_l <= o (ex is non-decreasing across lanes)
        int lo = 0;
#pragma unroll
        for (int step = 16; step > 0; step >>= 1) {
            const int cand = lo + step;
            const int exc = __shfl_sync(0xffffffffu, ex, cand & 31);
            if (cand < 32 && exc <= o) lo = cand;
        }
        const unsigned w = __shfl_sync(0xffffffffu, bits, lo);
        const int rb = __shfl_sync(0xffffffffu, row_base, lo);
        const int exl = __shfl_sync(0xffffffffu, ex, lo);
        if (o < tot) out[o] = rb + nth_set_bit(w, o - exl);
    }
}

// 32-bit shared-window addresses and raw shared loads / atomics: the generic
// pointer form makes the compiler rebuild the shared base (S2R + LEA) for
// every product.
__device__ __forceinline__ unsigned smem_addr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned lds_u32(unsigned a) {
    unsigned v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ unsigned atoms_or(unsigned a, unsigned v) {
    unsigned o;
    asm volatile("atom.shared.or.b32 %0, [%1], %2;" : "=r"(o) : "r"(a), "r"(v) : "memory");
    return o;
}

// Per-word exclusive popcount prefix of a W-word bitmap (the rank of every
// set bit among the tile's set bits) into pre[], chunk bases in chunk[];
// returns the tile's popcount (all threads).  Uses warp scans inside 32-word
// chunks, then one warp scans the chunk totals.
__device__ __forceinline__ int bitmap_ranks(const unsigned* __restrict__ bm, int* __restrict__ pre,
                                            int* __restrict__ chunk, int W, int* total_sh) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    const int nch = (W + 31) >> 5;
    for (int c = warp; c < nch; c += nw) {
        const int w = c * 32 + lane;
        const int x = w < W ? __popc(bm[w]) : 0;
        int tot;
        const int ex = warp_excl_scan(x, lane, &tot);
        if (w < W) pre[w] = ex;
        if (lane == 0) chunk[c] = tot;
    }
    __syncthreads();
    if (warp == 0) {
        int run = 0;
        for (int b0 = 0; b0 < nch; b0 += 32) {
            const int c = b0 + lane;
            const int x = c < nch ? chunk[c] : 0;
            int tot;
            const int ex = warp_excl_scan(x, lane, &tot);
            if (c < nch) chunk[c] = run + ex;
            run += tot;
        }
        if (lane == 0) *total_sh = run;
    }
    __syncthreads();
    for (int w = tid; w < W; w += blockDim.x) pre[w] += chunk[w >> 5];
    __syncthreads();
    return *total_sh;
}

// bitmap_ranks with half the rank storage: pre16[w] is the exclusive prefix
// inside w's 32-word chunk (<= 992, fits 16 bits) and chunk[c] the chunk
// base, so rank(row) = chunk[w>>5] + pre16[w] + popc(low bits of bm[w]).
__device__ __forceinline__ int bitmap_ranks16(const unsigned* __restrict__ bm, uint16_t* __restrict__ pre16,
                                              int* __restrict__ chunk, int W, int* total_sh) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    const int nch = (W + 31) >> 5;
    for (int c = warp; c < nch; c += nw) {
        const int w = c * 32 + lane;
        const int x = w < W ? __popc(bm[w]) : 0;
        int tot;
        const int ex = warp_excl_scan(x, lane, &tot);
        if (w < W) pre16[w] = (uint16_t)ex;
        if (lane == 0) chunk[c] = tot;
    }
    __syncthreads();
    if (warp == 0) {
        int run = 0;
        for (int b0 = 0; b0 < nch; b0 += 32) {
            const int c = b0 + lane;
            const int x = c < nch ? chunk[c] : 0;
            int tot;
            const int ex = warp_excl_scan(x, lane, &tot);
            if (c < nch) chunk[c] = run + ex;
            run += tot;
        }
        if (lane == 0) *total_sh = run;
    }
    __syncthreads();
    return *total_sh;
}

// Zero n words of shared memory with 16-byte stores (n a multiple of 4 or the
// tail handled word-wise).
__device__ __forceinline__ void smem_zero(unsigned* p, int n) {
    const int n4 = n >> 2;
    uint4* q = reinterpret_cast<uint4*>(p);
    for (int i = threadIdx.x; i < n4; i += blockDim.x) q[i] = make_uint4(0u, 0u, 0u, 0u);
    for (int i = (n4 << 2) + threadIdx.x; i < n; i += blockDim.x) p[i] = 0u;
}

// ---------------------------------------------------------------- host side

// Opt in to more than the default 48 KB of dynamic shared memory.  The
// kernels also hold a few bytes of static shared memory, which counts
// against the same 48 KB default, hence the margin.
template <class K>
void ensure_smem(K kernel, size_t smem) {
    // static + dynamic may pass the 48 KB default even when the dynamic part
    // alone does not, so opt in whenever a kernel carries static state too
    if (smem > 16 * 1024) SLAPCU_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
}

int grid_for(Ctx& c, int64_t work, int block, int per_sm = 8);
void make_bins(Ctx& c, int64_t n, const int64_t* flops, const int64_t* ccp, const BinSpec& spec, int64_t* zero_counts,
               Bins& bins);
void check_operands(const DevCsc& A, const DevCsc& B);
void prepare_plan(Ctx& c, const DevCsc& A, const DevCsc& B);
bool plan_matches(const Ctx& c, const DevCsc& A, const DevCsc& B);

}  // namespace slapcu
