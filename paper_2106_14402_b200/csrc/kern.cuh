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


// ---------------------------------------------------------------- host side

struct Bins {
    std::vector<int> count;   // per bin
    std::vector<int> offset;  // per bin
    DevBuf list;              // int32[n_nonzero]
};

// Opt in to more than the default 48 KB of dynamic shared memory.  The
// kernels also hold a few bytes of static shared memory, which counts
// against the same 48 KB default, hence the margin.
template <class K>
void ensure_smem(K kernel, size_t smem) {
    if (smem > 40 * 1024) SLAPCU_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
}

int grid_for(Ctx& c, int64_t work, int block, int per_sm = 8);
void make_bins(Ctx& c, int64_t n, const int64_t* flops, const int64_t* ccp, const BinSpec& spec, int64_t* zero_counts,
               Bins& bins);
void check_operands(const DevCsc& A, const DevCsc& B);
void prepare_plan(Ctx& c, const DevCsc& A, const DevCsc& B);
bool plan_matches(const Ctx& c, const DevCsc& A, const DevCsc& B);

}  // namespace slapcu
