// spgemm.cu -- local semiring SpGEMM C = A*B (CSC x CSC -> CSC) for sm_100a.
//
// Restates the three phases of slap::local_spgemm (reference
// proj/core/include/slap/spgemm.hpp:275-330) as GPU passes:
//
//   phase 1  k_flops            flops_j = sum_{k in B(:,j)} nnz(A(:,k))  (spgemm.hpp:68-88)
//   binning  k_bin_*            columns -> work classes (the GPU form of the
//                               flops-balanced thread split, spgemm.hpp:297-299)
//   phase 2  k_sym_light        exact nnz per column, shared-memory hash of row ids
//            k_sym_heavy        ... row-tiled shared-memory bitmap for heavy columns
//                               (spgemm.hpp:118-138 PatternSpa)
//   scan     cub ExclusiveSum   colptr in int64 (spgemm.hpp:289-293, no 2^31 limit)
//   phase 3  k_num_light        shared-memory hash accumulator (spgemm.hpp:211-266)
//                               + in-smem bitonic sort of the column (:259-260)
//            k_num_heavy        row-tiled dense accumulator: bitmap -> popcount
//                               rank -> values in rank order, sorted by
//                               construction (replaces the heap merge, :146-206)
//
// Everything is HBM/L2/smem-bound integer and byte work: no tensor cores.
// Output columns are canonical (rows ascending), numeric count must equal the
// symbolic count per column or the call fails with InternalError
// (spgemm.hpp:323-324).
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "kern.cuh"

namespace slapcu {

// ===================================================================== phase 1

// Entry-parallel over B's entries (spgemm.hpp:68-88): each thread takes a
// contiguous run of kFlopsRun entries, finds the column of its first entry by
// binary search on colptr and advances from there, adding nnz(A(:,k)) per
// entry and flushing each column's partial sum with one 64-bit atomic into
// flops[] (zeroed by the caller).  A warp per column left the R-MAT hub
// columns (up to 64K entries) serialised on one warp: a 1.2 ms tail per batch.
constexpr int kFlopsRun = 8;
__global__ void __launch_bounds__(256) k_flops(const int64_t* __restrict__ Acp, const int64_t* __restrict__ Bcp,
                                               const int32_t* __restrict__ Brw, int64_t ncols,
                                               unsigned long long* __restrict__ flops,
                                               unsigned long long* __restrict__ total) {
    const int64_t eb = Bcp[0], ee = Bcp[ncols];
    const int64_t nthreads = int64_t(gridDim.x) * blockDim.x;
    unsigned long long mine = 0;
    for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;; t += nthreads) {
        const int64_t e0 = eb + t * kFlopsRun;
        if (e0 >= ee) break;
        const int64_t e1 = e0 + kFlopsRun < ee ? e0 + kFlopsRun : ee;
        int64_t lo = 0, hi = ncols;  // Bcp[lo] <= e0 < Bcp[hi]
        while (hi - lo > 1) {
            const int64_t mid = (lo + hi) >> 1;
            if (Bcp[mid] <= e0) lo = mid; else hi = mid;
        }
        int64_t c = lo, cend = Bcp[c + 1];
        unsigned long long f = 0;
        int k[kFlopsRun];
#pragma unroll
        for (int q = 0; q < kFlopsRun; ++q) k[q] = e0 + q < e1 ? Brw[e0 + q] : 0;
        unsigned long long d[kFlopsRun];
#pragma unroll
        for (int q = 0; q < kFlopsRun; ++q) d[q] = e0 + q < e1 ? (unsigned long long)(Acp[k[q] + 1] - Acp[k[q]]) : 0ull;
#pragma unroll
        for (int q = 0; q < kFlopsRun; ++q) {
            const int64_t e = e0 + q;
            if (e >= e1) break;
            while (e >= cend) {  // next non-empty column
                if (f && flops) atomicAdd(&flops[c], f);
                mine += f;
                f = 0;
                ++c;
                cend = Bcp[c + 1];
            }
            f += d[q];
        }
        if (f && flops) atomicAdd(&flops[c], f);
        mine += f;
    }
    const unsigned long long w = (unsigned long long)warp_reduce_sum64((long long)mine);
    if ((threadIdx.x & 31) == 0 && total && w) atomicAdd(total, w);
}

// ===================================================================== binning

__global__ void __launch_bounds__(256) k_bin_count(int64_t n, const int64_t* __restrict__ flops,
                                                   const int64_t* __restrict__ ccp, BinSpec spec,
                                                   int8_t* __restrict__ bin_of, int* __restrict__ counts,
                                                   int64_t* __restrict__ zero_counts) {
    __shared__ int h[16];
    if (threadIdx.x < 16) h[threadIdx.x] = 0;
    __syncthreads();
    for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < n; j += int64_t(gridDim.x) * blockDim.x) {
        const int64_t key = spec.key_is_nnz ? (ccp[j + 1] - ccp[j]) : flops[j];
        const int b = bin_of_key(spec, key);
        bin_of[j] = (int8_t)b;
        if (b >= 0)
            atomicAdd(&h[b], 1);
        else if (zero_counts)
            zero_counts[j] = 0;
    }
    __syncthreads();
    if (threadIdx.x <= spec.nlight && h[threadIdx.x]) atomicAdd(&counts[threadIdx.x], h[threadIdx.x]);
}

__global__ void __launch_bounds__(256) k_bin_fill(int64_t n, const int8_t* __restrict__ bin_of,
                                                  int* __restrict__ cursor, int* __restrict__ list) {
    for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < n; j += int64_t(gridDim.x) * blockDim.x) {
        const int b = bin_of[j];
        if (b < 0) continue;
        // aggregate lanes that share a bin
        const unsigned peers = __match_any_sync(__activemask(), b);
        const int lane = threadIdx.x & 31;
        const int leader = __ffs(peers) - 1;
        int base = 0;
        if (lane == leader) base = atomicAdd(&cursor[b], __popc(peers));
        base = __shfl_sync(peers, base, leader);
        list[base + __popc(peers & ((1u << lane) - 1u))] = (int)j;
    }
}

__global__ void k_gather_keys(int n, const int* __restrict__ list, const int64_t* __restrict__ flops,
                              int64_t* __restrict__ keys) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) keys[i] = flops[list[i]];
}

// ============================================================ phase 2: light

// One group of G threads per column, CPB columns per block; a 2^LOG2S-slot
// key table in shared memory per column (slots >= 2*flops_j so the load
// factor stays <= 1/2 for the worst case of all-distinct rows).
template <int LOG2S, int G, int CPB>
__global__ void __launch_bounds__(G* CPB) k_sym_light(DevCsc A, DevCsc B, const int* __restrict__ cols, int n,
                                                      const int64_t* __restrict__ flops, int64_t* __restrict__ counts) {
    constexpr int S = 1 << LOG2S;
    extern __shared__ int sm_keys[];
    __shared__ long long red[(G * CPB) / 32];
    const int g = threadIdx.x / G, lane = threadIdx.x % G;
    int* keys = sm_keys + g * S;
    const int ci = blockIdx.x * CPB + g;
    const bool active = ci < n;
    const int j = active ? cols[ci] : 0;
    for (int s = lane; s < S; s += G) keys[s] = -1;
    group_sync<G, CPB>(g);
    long long cnt = 0;
    if (active) {
        const int64_t bs = B.cp[j], be = B.cp[j + 1];
        const int sg = pick_sg(flops[j], be - bs, G);
        const int sub = lane / sg, nsub = G / sg, sl = lane % sg;
        for (int64_t i = bs + sub; i < be; i += nsub) {
            const int k = B.rw[i];
            const int64_t as = A.cp[k], ae = A.cp[k + 1];
            for (int64_t p = as + sl; p < ae; p += sg) {
                bool nw;
                hash_insert<LOG2S>(keys, A.rw[p], &nw);
                cnt += nw;
            }
        }
    }
    cnt = group_sum<G, CPB>(cnt, g, lane, red);
    if (active && lane == 0) counts[j] = cnt;
}

// ============================================================ phase 2: heavy
// One CTA per heavy column; row tiles of 2^tile_log2 rows, each a shared-memory
// bitmap; count = popcount (PatternSpa::count, spgemm.hpp:107).
template <int NT>
__global__ void __launch_bounds__(NT) k_sym_heavy(DevCsc A, DevCsc B, const int* __restrict__ cols, int n,
                                                  const int64_t* __restrict__ flops, int64_t* __restrict__ counts,
                                                  int tile_log2, int32_t* __restrict__ cursor) {
    extern __shared__ unsigned bm[];
    __shared__ long long red[NT / 32];
    const int j = cols[blockIdx.x];
    const int64_t bs = B.cp[j], be = B.cp[j + 1];
    const int sg = pick_sg(flops[j], be - bs, 32);
    const int64_t R = int64_t(1) << tile_log2;
    const int ntiles = (int)((A.nrows + R - 1) >> tile_log2);
    long long total = 0;
    for (int t = 0; t < ntiles; ++t) {
        const int64_t t0 = int64_t(t) << tile_log2;
        const int64_t rows = min(R, A.nrows - t0);
        const int W = (int)((rows + 31) >> 5);
        for (int w = threadIdx.x; w < W; w += NT) bm[w] = 0u;
        __syncthreads();
        walk_tile(A, B, bs, be, sg, threadIdx.x, NT, t, ntiles, (int)(t0 + rows), cursor + (t & 1) * B.span,
                  cursor + ((t + 1) & 1) * B.span, true,
                  [&](int64_t, int64_t, int r) {
                      const int rr = r - (int)t0;
                      atomicOr(&bm[rr >> 5], 1u << (rr & 31));
                  });
        __syncthreads();
        long long c = 0;
        for (int w = threadIdx.x; w < W; w += NT) c += __popc(bm[w]);
        total += block_sum_ll(c, red);
        __syncthreads();
    }
    if (threadIdx.x == 0) counts[j] = total;
}

// ============================================================ phase 3: light

template <int SRID, bool ONES, int LOG2S, int G, int CPB>
__global__ void __launch_bounds__(G* CPB)
    k_num_light(DevCsc A, DevCsc B, const int* __restrict__ cols, int n, const int64_t* __restrict__ flops,
                const int64_t* __restrict__ Ccp, int32_t* __restrict__ Crw, typename Sr<SRID>::T* __restrict__ Cv,
                int* __restrict__ err) {
    using S_ = Sr<SRID>;
    using T = typename S_::T;
    using Acc = typename S_::Acc;
    constexpr int S = 1 << LOG2S;
    constexpr int PER = S / G;
    static_assert(PER >= 1 && PER <= 16, "per-thread slots");
    extern __shared__ __align__(16) unsigned char sm_raw[];
    Acc* vals_all = reinterpret_cast<Acc*>(sm_raw);                       // [CPB*S]
    int* keys_all = reinterpret_cast<int*>(sm_raw + sizeof(Acc) * CPB * S);  // [CPB*S]
    __shared__ int ctr[CPB];
    const int g = threadIdx.x / G, lane = threadIdx.x % G;
    int* keys = keys_all + g * S;
    Acc* vals = vals_all + g * S;
    const int ci = blockIdx.x * CPB + g;
    const bool active = ci < n;
    const int j = active ? cols[ci] : 0;
    const T* Av = static_cast<const T*>(A.v);
    const T* Bv = static_cast<const T*>(B.v);
    for (int s = lane; s < S; s += G) {
        keys[s] = -1;
        if constexpr (!ONES) vals[s] = S_::identity();
    }
    if (lane == 0) ctr[g] = 0;
    group_sync<G, CPB>(g);
    if (active) {
        const int64_t bs = B.cp[j], be = B.cp[j + 1];
        const int sg = pick_sg(flops[j], be - bs, G);
        const int sub = lane / sg, nsub = G / sg, sl = lane % sg;
        for (int64_t i = bs + sub; i < be; i += nsub) {
            const int k = B.rw[i];
            const int64_t as = A.cp[k], ae = A.cp[k + 1];
            T bval{};
            if constexpr (!ONES) bval = Bv[i];
            for (int64_t p = as + sl; p < ae; p += sg) {
                bool nw;
                const int slot = hash_insert<LOG2S>(keys, A.rw[p], &nw);
                if constexpr (!ONES) S_::atomic_acc(&vals[slot], S_::mul(Av[p], bval));
            }
        }
    }
    group_sync<G, CPB>(g);
    // compaction: pull own slots into registers, then write densely
    int kk[PER];
    Acc vv[PER];
#pragma unroll
    for (int q = 0; q < PER; ++q) {
        kk[q] = keys[lane + q * G];
        if constexpr (!ONES) vv[q] = vals[lane + q * G];
    }
    group_sync<G, CPB>(g);
#pragma unroll
    for (int q = 0; q < PER; ++q) {
        if (kk[q] != -1) {
            const int pos = warp_agg_inc(&ctr[g]);
            keys[pos] = kk[q];
            if constexpr (!ONES) vals[pos] = vv[q];
        }
    }
    group_sync<G, CPB>(g);
    const int m = ctr[g];
    int P = 1;
    while (P < m) P <<= 1;
    for (int s = m + lane; s < P; s += G) keys[s] = INT_MAX;
    group_sync<G, CPB>(g);
    // bitonic sort of keys[0..P) carrying vals
    for (int kk2 = 2; kk2 <= P; kk2 <<= 1) {
        for (int jj = kk2 >> 1; jj > 0; jj >>= 1) {
            for (int i = lane; i < P; i += G) {
                const int ixj = i ^ jj;
                if (ixj > i) {
                    const int a = keys[i], b = keys[ixj];
                    const bool up = (i & kk2) == 0;
                    if ((a > b) == up) {
                        keys[i] = b;
                        keys[ixj] = a;
                        if constexpr (!ONES) {
                            Acc t = vals[i];
                            vals[i] = vals[ixj];
                            vals[ixj] = t;
                        }
                    }
                }
            }
            group_sync<G, CPB>(g);
        }
    }
    if (active) {
        const int64_t o = Ccp[j];
        const int64_t expected = Ccp[j + 1] - o;
        if (m != expected) {
            if (lane == 0) atomicExch(err, 1);
        } else {
            for (int i = lane; i < m; i += G) {
                Crw[o + i] = keys[i];
                if constexpr (ONES)
                    Cv[o + i] = (T)1;
                else
                    Cv[o + i] = S_::out(vals[i]);
            }
        }
    }
}

// ============================================================ phase 3: heavy

// One CTA per heavy column.  Per row tile: (1) bitmap of present rows, (2)
// per-word popcount prefix = the rank of every present row among the tile's
// nonzeros (an order-preserving, collision-free slot map), (3) rows emitted in
// order straight from the bitmap, (4) values accumulated at their rank in
// shared memory (global memory when the tile holds more than `cap` entries),
// (5) values stored in order.  No sort is needed.
template <int SRID, bool ONES, int NT>
__global__ void __launch_bounds__(NT)
    k_num_heavy(DevCsc A, DevCsc B, const int* __restrict__ cols, int n, const int64_t* __restrict__ flops,
                const int64_t* __restrict__ Ccp, int32_t* __restrict__ Crw, typename Sr<SRID>::T* __restrict__ Cv,
                int tile_log2, int cap, int32_t* __restrict__ cursor, int* __restrict__ err) {
    using S_ = Sr<SRID>;
    using T = typename S_::T;
    using Acc = typename S_::Acc;
    extern __shared__ __align__(16) unsigned char sm_raw[];
    const int64_t R = int64_t(1) << tile_log2;
    const int WMAX = (int)(R >> 5);
    Acc* vals = reinterpret_cast<Acc*>(sm_raw);                                   // [cap]
    unsigned* bm = reinterpret_cast<unsigned*>(sm_raw + sizeof(Acc) * cap);       // [WMAX]
    int* pre = reinterpret_cast<int*>(bm + WMAX);                                 // [WMAX]
    int* chunk = pre + WMAX;                                                      // [WMAX/32]
    __shared__ int tile_nnz_sh;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int NW = NT / 32;
    const T* Av = static_cast<const T*>(A.v);
    const T* Bv = static_cast<const T*>(B.v);

    const int j = cols[blockIdx.x];
    const int64_t bs = B.cp[j], be = B.cp[j + 1];
    const int sg = pick_sg(flops[j], be - bs, 32);
    const int ntiles = (int)((A.nrows + R - 1) >> tile_log2);
    const int64_t out0 = Ccp[j];
    const int64_t expected = Ccp[j + 1] - out0;
    int64_t written = 0;

    for (int t = 0; t < ntiles; ++t) {
        const int64_t t0 = int64_t(t) << tile_log2;
        const int64_t rows = min(R, A.nrows - t0);
        const int W = (int)((rows + 31) >> 5);
        const int t1 = (int)(t0 + rows);
        for (int w = tid; w < W; w += NT) bm[w] = 0u;
        __syncthreads();
        // (1) pattern
        int32_t* cin = cursor + (t & 1) * B.span;
        int32_t* cout = cursor + ((t + 1) & 1) * B.span;
        walk_tile(A, B, bs, be, sg, tid, NT, t, ntiles, t1, cin, cout, ONES, [&](int64_t, int64_t, int r) {
            const int rr = r - (int)t0;
            atomicOr(&bm[rr >> 5], 1u << (rr & 31));
        });
        __syncthreads();
        // (2) ranks: warp-level scan inside 32-word chunks, then across chunks
        const int nch = (W + 31) >> 5;
        for (int c = warp; c < nch; c += NW) {
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
            if (lane == 0) tile_nnz_sh = run;
        }
        __syncthreads();
        const int tile_nnz = tile_nnz_sh;
        for (int w = tid; w < W; w += NT) pre[w] += chunk[w >> 5];
        __syncthreads();
        if (written + tile_nnz > expected) {
            if (tid == 0) atomicExch(err, 1);
            return;
        }
        const int64_t ob = out0 + written;
        // (3) rows in order
        for (int w = tid; w < W; w += NT) {
            unsigned bits = bm[w];
            int64_t pos = ob + pre[w];
            const int rb = (int)t0 + (w << 5);
            while (bits) {
                const int b = __ffs(bits) - 1;
                bits &= bits - 1u;
                Crw[pos++] = rb + b;
            }
        }
        if constexpr (ONES) {
            for (int i = tid; i < tile_nnz; i += NT) Cv[ob + i] = (T)1;
        } else {
            const bool in_smem = tile_nnz <= cap;
            if (in_smem) {
                for (int i = tid; i < tile_nnz; i += NT) vals[i] = S_::identity();
            } else {
                for (int i = tid; i < tile_nnz; i += NT) Cv[ob + i] = S_::out(S_::identity());
            }
            __syncthreads();
            // (4) values at their rank
            walk_tile(A, B, bs, be, sg, tid, NT, t, ntiles, t1, cin, cout, true, [&](int64_t p, int64_t i, int r) {
                const int rr = r - (int)t0;
                const int w = rr >> 5;
                const int idx = pre[w] + __popc(bm[w] & ((1u << (rr & 31)) - 1u));
                const Acc v = S_::mul(Av[p], Bv[i]);
                if (in_smem)
                    S_::atomic_acc(&vals[idx], v);
                else
                    S_::atomic_acc_global(&Cv[ob + idx], v);
            });
            __syncthreads();
            // (5) values in order
            if (in_smem)
                for (int i = tid; i < tile_nnz; i += NT) Cv[ob + i] = S_::out(vals[i]);
        }
        written += tile_nnz;
        __syncthreads();
    }
    if (tid == 0 && written != expected) atomicExch(err, 1);
}

// ====================================================== misc small kernels

__global__ void k_any_zero_u8(int64_t n, const uint8_t* __restrict__ v, int* __restrict__ flag) {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        if (v[i] == 0) {
            *flag = 1;
            return;
        }
}

// ============================================================ host helpers

constexpr int kNumLightSym = 10;
constexpr int kNumLightNum = 8;

int grid_for(Ctx& c, int64_t work, int block, int per_sm) {
    int64_t g = ceil_div(work, block);
    int64_t cap = int64_t(c.num_sms) * per_sm;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    return (int)g;
}

// Two-pass binning of the columns by key; heavy bin sorted by flops desc (LPT).
void make_bins(Ctx& c, int64_t n, const int64_t* flops, const int64_t* ccp, const BinSpec& spec, int64_t* zero_counts,
               Bins& bins) {
    const int nb = spec.nlight + 1;
    KScope ks(c, KC_BIN);
    DevBuf bin_of(std::max<int64_t>(n, 1), c.stream);
    DevBuf cnt(sizeof(int) * 16, c.stream);
    SLAPCU_CUDA(cudaMemsetAsync(cnt.get(), 0, sizeof(int) * 16, c.stream));
    launch(c, k_bin_count, dim3(grid_for(c, n, 256)), dim3(256), 0, n, flops, ccp, spec, bin_of.as<int8_t>(),
           cnt.as<int>(), zero_counts);
    std::vector<int> h(16, 0);
    SLAPCU_CUDA(cudaMemcpyAsync(h.data(), cnt.get(), sizeof(int) * 16, cudaMemcpyDeviceToHost, c.stream));
    SLAPCU_CUDA(cudaStreamSynchronize(c.stream));
    bins.count.assign(h.begin(), h.begin() + nb);
    bins.offset.assign(nb, 0);
    int tot = 0;
    for (int b = 0; b < nb; ++b) {
        bins.offset[b] = tot;
        tot += bins.count[b];
    }
    bins.list.reset(sizeof(int) * std::max(tot, 1), c.stream);
    if (tot == 0) return;
    SLAPCU_CUDA(cudaMemcpyAsync(cnt.get(), bins.offset.data(), sizeof(int) * nb, cudaMemcpyHostToDevice, c.stream));
    launch(c, k_bin_fill, dim3(grid_for(c, n, 256)), dim3(256), 0, n, (const int8_t*)bin_of.as<int8_t>(),
           cnt.as<int>(), bins.list.as<int>());
    // LPT order for the heavy bin: heaviest columns first
    const int hc = bins.count[spec.nlight];
    if (hc > 1) {
        int* hl = bins.list.as<int>() + bins.offset[spec.nlight];
        DevBuf keys_in(sizeof(int64_t) * hc, c.stream), keys_out(sizeof(int64_t) * hc, c.stream),
            vals_out(sizeof(int) * hc, c.stream);
        launch(c, k_gather_keys, dim3(grid_for(c, hc, 256)), dim3(256), 0, hc, (const int*)hl, flops,
               keys_in.as<int64_t>());
        size_t tb = 0;
        SLAPCU_CUDA(cub::DeviceRadixSort::SortPairsDescending(nullptr, tb, keys_in.as<int64_t>(),
                                                              keys_out.as<int64_t>(), hl, vals_out.as<int>(), hc, 0,
                                                              64, c.stream));
        DevBuf tmp(tb, c.stream);
        timed(c, KC_BIN, [&] {
            SLAPCU_CUDA(cub::DeviceRadixSort::SortPairsDescending(tmp.get(), tb, keys_in.as<int64_t>(),
                                                                  keys_out.as<int64_t>(), hl, vals_out.as<int>(), hc,
                                                                  0, 64, c.stream));
        });
        ++c.launches;
        SLAPCU_CUDA(cudaMemcpyAsync(hl, vals_out.get(), sizeof(int) * hc, cudaMemcpyDeviceToDevice, c.stream));
    }
}

BinSpec sym_spec(const Ctx& c, int alg) {
    BinSpec s{};
    s.nlight = kNumLightSym;
    for (int b = 0; b < kNumLightSym; ++b) s.thr[b] = int64_t(32) << b;  // 32 .. 16384
    s.light_max = std::min<int64_t>(c.opt.light_flops_max, s.thr[kNumLightSym - 1]);
    s.all_heavy = alg == SLAPCU_ALG_HEAP;
    s.key_is_nnz = 0;
    return s;
}

BinSpec num_spec(const Ctx& c, int alg) {
    BinSpec s{};
    s.nlight = kNumLightNum;
    for (int b = 0; b < kNumLightNum; ++b) s.thr[b] = int64_t(32) << b;  // 32 .. 4096
    s.light_max = std::min<int64_t>(c.opt.light_nnz_max, s.thr[kNumLightNum - 1]);
    s.all_heavy = alg == SLAPCU_ALG_HEAP;
    s.key_is_nnz = 1;
    return s;
}

void check_operands(const DevCsc& A, const DevCsc& B) {
    if (A.ncols != B.nrows)
        throw Fail{SLAPCU_ERR_DIM, "spgemm inner dims: A is " + std::to_string(A.nrows) + "x" +
                                       std::to_string(A.ncols) + ", B is " + std::to_string(B.nrows) + "x" +
                                       std::to_string(B.ncols)};
    if (A.nrows > INT32_MAX - 64 || B.nrows > INT32_MAX - 64)
        throw Fail{SLAPCU_ERR_SHAPE, "row dimension exceeds the 32-bit row id width"};
    if (B.ncols > INT32_MAX) throw Fail{SLAPCU_ERR_SHAPE, "column dimension exceeds 2^31"};
    if ((A.nnz && (!A.cp || !A.rw)) || (B.nnz && (!B.cp || !B.rw)) || !A.cp || !B.cp)
        throw Fail{SLAPCU_ERR_INVALID, "null operand pointer"};
}

void prepare_plan(Ctx& c, const DevCsc& A, const DevCsc& B) {
    Plan& p = c.plan;
    p.flops.reset(sizeof(int64_t) * std::max<int64_t>(B.ncols, 1), c.stream);
    p.counts.reset(sizeof(int64_t) * (B.ncols + 1), c.stream);
    p.cursor.reset(sizeof(int32_t) * 2 * std::max<int64_t>(B.span, 1), c.stream);
    KScope ks(c, KC_FLOPS);
    SLAPCU_CUDA(cudaMemsetAsync(p.flops.get(), 0, sizeof(int64_t) * std::max<int64_t>(B.ncols, 1), c.stream));
    const int64_t runs = (std::max<int64_t>(B.span, B.nnz) + kFlopsRun - 1) / kFlopsRun;
    if (B.ncols > 0)
        launch(c, k_flops, dim3(grid_for(c, std::max<int64_t>(runs, 1), 256, 16)), dim3(256), 0, A.cp, B.cp, B.rw,
               B.ncols, reinterpret_cast<unsigned long long*>(p.flops.as<int64_t>()), (unsigned long long*)nullptr);
    p.a_key = A.cp;
    p.b_key = B.cp;
    p.a_ncols = A.ncols;
    p.b_ncols = B.ncols;
    p.b_nnz = B.span;
    p.b_base = B.base;
    p.valid = true;
}

bool plan_matches(const Ctx& c, const DevCsc& A, const DevCsc& B) {
    const Plan& p = c.plan;
    return p.valid && p.a_key == A.cp && p.b_key == B.cp && p.a_ncols == A.ncols && p.b_ncols == B.ncols &&
           p.b_nnz == B.span && p.b_base == B.base;
}

namespace {

// ---- light launch tables

template <int LOG2S, int G, int CPB>
void launch_sym_light(Ctx& c, const DevCsc& A, const DevCsc& B, const int* list, int n, const int64_t* flops,
                      int64_t* counts) {
    const size_t smem = sizeof(int) * (size_t(CPB) << LOG2S);
    auto k = k_sym_light<LOG2S, G, CPB>;
    ensure_smem(k, smem);
    launch(c, k, dim3((unsigned)ceil_div(n, CPB)), dim3(G * CPB), smem, A, B, list, n, flops, counts);
}

template <int SRID, bool ONES, int LOG2S, int G, int CPB>
void launch_num_light(Ctx& c, const DevCsc& A, const DevCsc& B, const int* list, int n, const int64_t* flops,
                      const int64_t* ccp, int32_t* crw, void* cv, int* err) {
    using Acc = typename Sr<SRID>::Acc;
    const size_t smem = (sizeof(Acc) + sizeof(int)) * (size_t(CPB) << LOG2S);
    auto k = k_num_light<SRID, ONES, LOG2S, G, CPB>;
    ensure_smem(k, smem);
    launch(c, k, dim3((unsigned)ceil_div(n, CPB)), dim3(G * CPB), smem, A, B, list, n, flops, ccp, crw,
           static_cast<typename Sr<SRID>::T*>(cv), err);
}

template <int SRID, bool ONES>
void launch_num_bin(Ctx& c, int b, const DevCsc& A, const DevCsc& B, const int* list, int n, const int64_t* flops,
                    const int64_t* ccp, int32_t* crw, void* cv, int* err) {
    switch (b) {
    case 0: launch_num_light<SRID, ONES, 6, 32, 8>(c, A, B, list, n, flops, ccp, crw, cv, err); break;
    case 1: launch_num_light<SRID, ONES, 7, 32, 8>(c, A, B, list, n, flops, ccp, crw, cv, err); break;
    case 2: launch_num_light<SRID, ONES, 8, 32, 8>(c, A, B, list, n, flops, ccp, crw, cv, err); break;
    case 3: launch_num_light<SRID, ONES, 9, 64, 4>(c, A, B, list, n, flops, ccp, crw, cv, err); break;
    case 4: launch_num_light<SRID, ONES, 10, 128, 2>(c, A, B, list, n, flops, ccp, crw, cv, err); break;
    case 5: launch_num_light<SRID, ONES, 11, 256, 1>(c, A, B, list, n, flops, ccp, crw, cv, err); break;
    case 6: launch_num_light<SRID, ONES, 12, 512, 1>(c, A, B, list, n, flops, ccp, crw, cv, err); break;
    case 7: launch_num_light<SRID, ONES, 13, 1024, 1>(c, A, B, list, n, flops, ccp, crw, cv, err); break;
    }
}

constexpr int kHeavyThreads = 512;

size_t heavy_fixed_smem(int tile_log2) {
    const size_t W = size_t(1) << (tile_log2 - 5);
    const size_t NCH = (W + 31) / 32;
    return W * 4 * 2 + NCH * 4 + 64;
}

template <int SRID, bool ONES>
void launch_num_heavy(Ctx& c, const DevCsc& A, const DevCsc& B, const int* list, int n, const int64_t* flops,
                      const int64_t* ccp, int32_t* crw, void* cv, int* err) {
    using Acc = typename Sr<SRID>::Acc;
    int tl = c.opt.tile_rows_log2;
    // never tile finer than needed: one tile when the rows fit
    while (tl > 10 && (int64_t(1) << (tl - 1)) >= A.nrows) --tl;
    const size_t fixed = heavy_fixed_smem(tl);
    // two CTAs per SM when the bitmap leaves room; otherwise one
    size_t budget = std::min<size_t>(size_t(c.smem_optin), size_t(110) * 1024);
    if (budget < fixed + 1024 * sizeof(Acc)) budget = size_t(c.smem_optin);
    int cap = ONES ? 0 : (int)((budget - fixed) / sizeof(Acc));
    if (cap < 0) cap = 0;
    const size_t smem = fixed + size_t(cap) * sizeof(Acc);
    if (smem > size_t(c.smem_optin)) throw Fail{SLAPCU_ERR_INVALID, "tile too large for shared memory"};
    auto k = k_num_heavy<SRID, ONES, kHeavyThreads>;
    ensure_smem(k, smem);
    launch(c, k, dim3(n), dim3(kHeavyThreads), smem, A, B, list, n, flops, ccp, crw,
           static_cast<typename Sr<SRID>::T*>(cv), tl, cap, c.plan.cursor.as<int32_t>(), err);
}

}  // namespace

// ================================================================ host API

void spgemm_flops(Ctx& c, const DevCsc& A, const DevCsc& B, int64_t* flops_dev, int64_t* total) {
    check_operands(A, B);
    DevBuf tot(sizeof(unsigned long long), c.stream);
    SLAPCU_CUDA(cudaMemsetAsync(tot.get(), 0, sizeof(unsigned long long), c.stream));
    KScope ks(c, KC_FLOPS);
    if (flops_dev) SLAPCU_CUDA(cudaMemsetAsync(flops_dev, 0, sizeof(int64_t) * std::max<int64_t>(B.ncols, 1), c.stream));
    // grid-stride over the entries: the grid is sized from an upper bound
    // (a column window carries its parent's nnz)
    const int64_t runs = (std::max<int64_t>(B.span, B.nnz) + kFlopsRun - 1) / kFlopsRun;
    if (B.ncols > 0)
        launch(c, k_flops, dim3(grid_for(c, std::max<int64_t>(runs, 1), 256, 16)), dim3(256), 0, A.cp, B.cp, B.rw,
               B.ncols, reinterpret_cast<unsigned long long*>(flops_dev), tot.as<unsigned long long>());
    unsigned long long h = 0;
    SLAPCU_CUDA(cudaMemcpyAsync(&h, tot.get(), sizeof(h), cudaMemcpyDeviceToHost, c.stream));
    SLAPCU_CUDA(cudaStreamSynchronize(c.stream));
    if (total) *total = (int64_t)h;
}

void exclusive_scan_i64(Ctx& c, const int64_t* in, int64_t* out, int64_t n) {
    size_t tb = 0;
    SLAPCU_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, n, c.stream));
    DevBuf tmp(tb, c.stream);
    timed(c, KC_SCAN, [&] { SLAPCU_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(), tb, in, out, n, c.stream)); });
    ++c.launches;
}

int64_t spgemm_symbolic(Ctx& c, const DevCsc& A_, const DevCsc& B_, int alg, int64_t* c_colptr) {
    check_operands(A_, B_);
    DevCsc A = A_, B = B_;
    resolve(c, A);
    resolve(c, B);
    if (!c_colptr) throw Fail{SLAPCU_ERR_INVALID, "null colptr"};
    SLAPCU_CUDA(cudaEventRecord(c.ev[0], c.stream));
    prepare_plan(c, A, B);
    int64_t* flops = c.plan.flops.as<int64_t>();
    int64_t* counts = c.plan.counts.as<int64_t>();
    SLAPCU_CUDA(cudaMemsetAsync(counts + B.ncols, 0, sizeof(int64_t), c.stream));
    Bins bins;
    const BinSpec spec = sym_spec(c, alg);
    make_bins(c, B.ncols, flops, nullptr, spec, counts, bins);
    const int* L = bins.list.as<int>();
    for (int b = 0; b <= spec.nlight; ++b) {
        const int n = bins.count[b];
        if (!n) continue;
        const int* l = L + bins.offset[b];
        KScope ks(c, b < spec.nlight ? KC_SYM_LIGHT : KC_SYM_HEAVY);
        switch (b) {
        case 0: launch_sym_light<6, 32, 8>(c, A, B, l, n, flops, counts); break;
        case 1: launch_sym_light<7, 32, 8>(c, A, B, l, n, flops, counts); break;
        case 2: launch_sym_light<8, 32, 8>(c, A, B, l, n, flops, counts); break;
        case 3: launch_sym_light<9, 64, 4>(c, A, B, l, n, flops, counts); break;
        case 4: launch_sym_light<10, 128, 2>(c, A, B, l, n, flops, counts); break;
        case 5: launch_sym_light<11, 256, 1>(c, A, B, l, n, flops, counts); break;
        case 6: launch_sym_light<12, 256, 1>(c, A, B, l, n, flops, counts); break;
        case 7: launch_sym_light<13, 512, 1>(c, A, B, l, n, flops, counts); break;
        case 8: launch_sym_light<14, 512, 1>(c, A, B, l, n, flops, counts); break;
        case 9: launch_sym_light<15, 1024, 1>(c, A, B, l, n, flops, counts); break;
        default: {
            int tl = c.opt.sym_tile_rows_log2;
            while (tl > 10 && (int64_t(1) << (tl - 1)) >= A.nrows) --tl;
            const size_t smem = (size_t(1) << (tl - 5)) * 4;
            if (smem > size_t(c.smem_optin)) throw Fail{SLAPCU_ERR_INVALID, "symbolic tile too large"};
            auto k = k_sym_heavy<kHeavyThreads>;
            ensure_smem(k, smem);
            launch(c, k, dim3(n), dim3(kHeavyThreads), smem, A, B, l, n, (const int64_t*)flops, counts, tl,
                   c.plan.cursor.as<int32_t>());
        }
        }
    }
    exclusive_scan_i64(c, counts, c_colptr, B.ncols + 1);
    int64_t total = 0;
    SLAPCU_CUDA(cudaMemcpyAsync(&total, c_colptr + B.ncols, sizeof(int64_t), cudaMemcpyDeviceToHost, c.stream));
    SLAPCU_CUDA(cudaEventRecord(c.ev[1], c.stream));
    SLAPCU_CUDA(cudaStreamSynchronize(c.stream));
    cudaEventElapsedTime(&c.sym_ms, c.ev[0], c.ev[1]);
    prof_flush(c);
    return total;
}

void spgemm_numeric(Ctx& c, const DevCsc& A_, const DevCsc& B_, int sr, int alg, const int64_t* ccp, int32_t* crw,
                    void* cv) {
    check_operands(A_, B_);
    DevCsc A = A_, B = B_;
    resolve(c, A);
    resolve(c, B);
    if (!ccp) throw Fail{SLAPCU_ERR_INVALID, "null colptr"};
    if (value_size(sr) == 0) throw Fail{SLAPCU_ERR_INVALID, "unknown semiring"};
    if ((A.nnz && !A.v) || (B.nnz && !B.v)) throw Fail{SLAPCU_ERR_INVALID, "operand values are null"};
    SLAPCU_CUDA(cudaEventRecord(c.ev[2], c.stream));
    if (!plan_matches(c, A, B)) prepare_plan(c, A, B);
    const int64_t* flops = c.plan.flops.as<int64_t>();
    c.err_flag.reset(sizeof(int) * 2, c.stream);
    int* err = c.err_flag.as<int>();
    SLAPCU_CUDA(cudaMemsetAsync(err, 0, sizeof(int) * 2, c.stream));
    // OrAnd fast path: if no stored value is 0 every product is 1
    bool ones = false;
    if (sr == SLAPCU_OR_AND_U8) {
        launch(c, k_any_zero_u8, dim3(grid_for(c, A.span, 256)), dim3(256), 0, A.span, (const uint8_t*)A.v + A.base,
               err + 1);
        launch(c, k_any_zero_u8, dim3(grid_for(c, B.span, 256)), dim3(256), 0, B.span, (const uint8_t*)B.v + B.base,
               err + 1);
        int hz = 0;
        SLAPCU_CUDA(cudaMemcpyAsync(&hz, err + 1, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
        SLAPCU_CUDA(cudaStreamSynchronize(c.stream));
        ones = hz == 0;
    }
    Bins bins;
    const BinSpec spec = num_spec(c, alg);
    make_bins(c, B.ncols, flops, ccp, spec, nullptr, bins);
    const int* L = bins.list.as<int>();
    dispatch_sr(sr, [&](auto id) {
        constexpr int ID = decltype(id)::value;
        for (int b = 0; b <= spec.nlight; ++b) {
            const int n = bins.count[b];
            if (!n) continue;
            const int* l = L + bins.offset[b];
            KScope ks(c, b < spec.nlight ? KC_NUM_LIGHT : KC_NUM_HEAVY);
            if (b < spec.nlight) {
                if constexpr (ID == SLAPCU_OR_AND_U8) {
                    if (ones)
                        launch_num_bin<ID, true>(c, b, A, B, l, n, flops, ccp, crw, cv, err);
                    else
                        launch_num_bin<ID, false>(c, b, A, B, l, n, flops, ccp, crw, cv, err);
                } else {
                    launch_num_bin<ID, false>(c, b, A, B, l, n, flops, ccp, crw, cv, err);
                }
            } else {
                if constexpr (ID == SLAPCU_OR_AND_U8) {
                    if (ones)
                        launch_num_heavy<ID, true>(c, A, B, l, n, flops, ccp, crw, cv, err);
                    else
                        launch_num_heavy<ID, false>(c, A, B, l, n, flops, ccp, crw, cv, err);
                } else {
                    launch_num_heavy<ID, false>(c, A, B, l, n, flops, ccp, crw, cv, err);
                }
            }
        }
    });
    int herr = 0;
    SLAPCU_CUDA(cudaMemcpyAsync(&herr, err, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
    SLAPCU_CUDA(cudaEventRecord(c.ev[3], c.stream));
    SLAPCU_CUDA(cudaStreamSynchronize(c.stream));
    cudaEventElapsedTime(&c.num_ms, c.ev[2], c.ev[3]);
    prof_flush(c);
    if (herr) throw Fail{SLAPCU_ERR_INTERNAL, "numeric column nnz disagrees with symbolic count"};
}

// DCSC (jc, cp) -> dense colptr: empty columns take the start of the next
// stored column.  Built as: colptr[j] = cp[#stored columns < j].
__global__ void k_dcsc_dense(int64_t ncols, int64_t nzc, const int32_t* __restrict__ jc,
                             const int32_t* __restrict__ cp, int64_t* __restrict__ colptr) {
    for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j <= ncols;
         j += int64_t(gridDim.x) * blockDim.x) {
        // lower_bound of j in jc
        int64_t lo = 0, hi = nzc;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (jc[mid] < j)
                lo = mid + 1;
            else
                hi = mid;
        }
        colptr[j] = cp[lo];
    }
}

void any_zero_u8(Ctx& c, const uint8_t* v, int64_t n, int* flag) {
    launch(c, k_any_zero_u8, dim3(grid_for(c, n, 256)), dim3(256), 0, n, v, flag);
}

void resolve(Ctx& c, DevCsc& m) {
    int64_t ends[2] = {0, 0};
    if (m.ncols > 0) {
        SLAPCU_CUDA(cudaMemcpyAsync(&ends[0], m.cp, sizeof(int64_t), cudaMemcpyDeviceToHost, c.stream));
        SLAPCU_CUDA(cudaMemcpyAsync(&ends[1], m.cp + m.ncols, sizeof(int64_t), cudaMemcpyDeviceToHost, c.stream));
        SLAPCU_CUDA(cudaStreamSynchronize(c.stream));
    } else if (m.cp) {
        SLAPCU_CUDA(cudaMemcpyAsync(&ends[0], m.cp, sizeof(int64_t), cudaMemcpyDeviceToHost, c.stream));
        SLAPCU_CUDA(cudaStreamSynchronize(c.stream));
        ends[1] = ends[0];
    }
    m.base = ends[0];
    m.span = ends[1] - ends[0];
    if (m.span < 0) throw Fail{SLAPCU_ERR_INVALID, "colptr is not monotone"};
}

// Content fingerprint of an operand's PATTERN (column lengths and row ids),
// order-dependent through the position mix: keys the per-A caches of the
// direct path, so an A rewritten in place (same pointer, same nnz) or a new A
// at a reused address is never served stale tile pointers.  One read of
// colptr + rowids (~25 us for R-MAT s20's 157 MB), reduced by atomics.
__global__ void k_fingerprint(int64_t ncols, const int64_t* __restrict__ cp, const int32_t* __restrict__ rw,
                              int64_t base, int64_t span, unsigned long long* __restrict__ out) {
    auto mix = [](unsigned long long z) {
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        return z ^ (z >> 31);
    };
    unsigned long long h = 0;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    const int64_t t0 = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    for (int64_t j = t0; j < ncols; j += stride)
        h += mix((unsigned long long)(cp[j + 1] - cp[j]) * 0x9e3779b97f4a7c15ull + (unsigned long long)j);
    for (int64_t i = t0; i < span; i += stride)
        h += mix(((unsigned long long)i << 32) ^ (unsigned)rw[base + i] ^ 0x5bd1e995ull);
    for (int o = 16; o > 0; o >>= 1) h += __shfl_xor_sync(0xffffffffu, h, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(out, h);
}

uint64_t pattern_fingerprint(Ctx& c, const DevCsc& m) {
    DevBuf acc(sizeof(unsigned long long), c.stream);
    SLAPCU_CUDA(cudaMemsetAsync(acc.get(), 0, sizeof(unsigned long long), c.stream));
    const int64_t work = std::max<int64_t>(std::max<int64_t>(m.ncols, m.span), 1);
    launch(c, k_fingerprint, dim3(grid_for(c, work, 256, 4)), dim3(256), 0, m.ncols, m.cp, m.rw, m.base, m.span,
           acc.as<unsigned long long>());
    unsigned long long h = 0;
    SLAPCU_CUDA(cudaMemcpyAsync(&h, acc.get(), sizeof(h), cudaMemcpyDeviceToHost, c.stream));
    SLAPCU_CUDA(cudaStreamSynchronize(c.stream));
    return (uint64_t)h ^ ((uint64_t)m.nrows << 17) ^ (uint64_t)m.ncols;
}

void dcsc_colptr(Ctx& c, int64_t ncols, int64_t nzc, const int32_t* jc, const int32_t* cp, int64_t* colptr) {
    launch(c, k_dcsc_dense, dim3(grid_for(c, ncols + 1, 256)), dim3(256), 0, ncols, nzc, jc, cp, colptr);
}

}  // namespace slapcu
