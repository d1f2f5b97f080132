// fused.cu -- single-product-pass SpGEMM ("begin" / "finish").
//
// The two-phase symbolic -> numeric contract of slap::local_spgemm
// (spgemm.hpp:286-330) walks every product twice on the GPU (count, then form).
// This path forms every output column ONCE, already sorted, into a staging
// area carved out by a global atomic cursor, and only then lays the columns
// out canonically:
//
//   begin   k_flops + bins by flops
//           K1 light  (flops <= L):  shared-memory hash of (row, value),
//                                    compaction, bitonic sort -> staging
//           K1 heavy  (flops >  L):  row-tiled shared-memory bitmap of the
//                                    pattern (atomicOr), per-chunk popcount
//                                    scan -> sorted rows -> staging segments
//           scan of the per-column counts -> C colptr (int64)
//   finish  K2: staged rows/values copied into C (values 1 for Boolean
//           all-ones operands)
//           K3 (heavy columns, semirings with values): bitmap rebuilt from
//           C's sorted rows, popcount ranks, one pass over the products
//           accumulating at rank in shared memory.
//
// Product passes: 1 for Boolean (the C3 headline), 2 for value semirings on
// heavy columns, 1 for light columns.  Staging holds at most
// sum_j min(flops_j, nrows) entries; when that exceeds the budget begin()
// fails with BudgetError and callers batch columns (batched.hpp:153-170).
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "kern.cuh"

namespace slapcu {

// ------------------------------------------------------------------ K1 light

template <int SRID, bool ONES, int LOG2S, int G, int CPB>
__global__ void __launch_bounds__(G* CPB)
    k_fused_light(DevCsc A, DevCsc B, const int* __restrict__ cols, int n, const int64_t* __restrict__ flops,
                  int64_t* __restrict__ cnt, int64_t* __restrict__ soff, int32_t* __restrict__ srows,
                  typename Sr<SRID>::T* __restrict__ svals, unsigned long long* __restrict__ scur) {
    using S_ = Sr<SRID>;
    using T = typename S_::T;
    using Acc = typename S_::Acc;
    constexpr int S = 1 << LOG2S;
    constexpr int PER = S / G;
    static_assert(PER >= 1 && PER <= 16, "per-thread slots");
    extern __shared__ __align__(16) unsigned char sm_raw[];
    Acc* vals_all = reinterpret_cast<Acc*>(sm_raw);
    int* keys_all = reinterpret_cast<int*>(sm_raw + (ONES ? 0 : sizeof(Acc) * CPB * S));
    __shared__ int ctr[CPB];
    __shared__ unsigned long long off_sh[CPB];
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
                const int slot = hash_insert<LOG2S>(keys, __ldg(&A.rw[p]), &nw);
                if constexpr (!ONES) S_::atomic_acc(&vals[slot], S_::mul(Av[p], bval));
            }
        }
    }
    group_sync<G, CPB>(g);
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
    if constexpr (G == 32 && PER <= 4) {
        // one warp per column (<= 128 entries): rank by counting -- every key
        // is compared with the column's keys read as shared-memory broadcasts,
        // and goes straight to its sorted place in the staging area (C2, ER
        // d = 8, bin of <= 64 products: 0.94 -> 0.82 ms; at <= 256 entries the
        // bitonic network is cheaper: 2.1 -> 2.5 ms)
        if (active && lane == 0) {
            const unsigned long long off = atomicAdd(scur, (unsigned long long)m);
            off_sh[g] = off;
            cnt[j] = m;
            soff[j] = (int64_t)off;
        }
        __syncwarp();
        if (active) {
            const int64_t off = (int64_t)off_sh[g];
            const int nq = (m + 31) >> 5;
            int mk[PER], rk[PER];
#pragma unroll
            for (int q = 0; q < PER; ++q) {
                const int i = lane + q * 32;
                mk[q] = i < m ? keys[i] : INT_MAX;
                rk[q] = 0;
            }
            for (int x = 0; x < m; ++x) {
                const int kx = keys[x];
#pragma unroll
                for (int q = 0; q < PER; ++q)
                    if (q < nq) rk[q] += kx < mk[q];
            }
#pragma unroll
            for (int q = 0; q < PER; ++q) {
                const int i = lane + q * 32;
                if (i < m) {
                    srows[off + rk[q]] = mk[q];
                    if constexpr (!ONES) svals[off + rk[q]] = S_::out(vals[i]);
                }
            }
        }
        return;
    }
    int P = 1;
    while (P < m) P <<= 1;
    for (int s = m + lane; s < P; s += G) keys[s] = INT_MAX;
    group_sync<G, CPB>(g);
    for (int k2 = 2; k2 <= P; k2 <<= 1) {
        for (int jj = k2 >> 1; jj > 0; jj >>= 1) {
            for (int i = lane; i < P; i += G) {
                const int ixj = i ^ jj;
                if (ixj > i) {
                    const int a = keys[i], b = keys[ixj];
                    if ((a > b) == ((i & k2) == 0)) {
                        keys[i] = b;
                        keys[ixj] = a;
                        if constexpr (!ONES) {
                            const Acc t = vals[i];
                            vals[i] = vals[ixj];
                            vals[ixj] = t;
                        }
                    }
                }
            }
            group_sync<G, CPB>(g);
        }
    }
    if (active && lane == 0) {
        const unsigned long long off = atomicAdd(scur, (unsigned long long)m);
        off_sh[g] = off;
        cnt[j] = m;
        soff[j] = (int64_t)off;
    }
    group_sync<G, CPB>(g);
    if (active) {
        const int64_t off = (int64_t)off_sh[g];
        for (int i = lane; i < m; i += G) {
            srows[off + i] = keys[i];
            if constexpr (!ONES) svals[off + i] = S_::out(vals[i]);
        }
    }
}

// ------------------------------------------------------------------ K1 heavy

// One CTA per heavy column.  Per row tile: bitmap via shared atomics (the only
// per-product work), 32-word chunk popcounts, chunk scan, one global atomic
// to reserve the tile's staging segment, rows emitted in order.
template <int NT>
__global__ void __launch_bounds__(NT)
    k_fused_heavy(DevCsc A, DevCsc B, const int* __restrict__ cols, int n, const int64_t* __restrict__ flops,
                  int tile_log2, int32_t* __restrict__ cursor, int64_t* __restrict__ cnt, int32_t* __restrict__ srows,
                  unsigned long long* __restrict__ scur, int64_t* __restrict__ seg_off, int* __restrict__ seg_cnt,
                  int T) {
    extern __shared__ __align__(16) unsigned bm[];
    const int64_t R = int64_t(1) << tile_log2;
    const int WMAX = (int)(R >> 5);
    int* chunk = reinterpret_cast<int*>(bm + WMAX);  // [WMAX/32]
    __shared__ unsigned long long off_sh;
    __shared__ int tot_sh;
    __shared__ WalkShared ws;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int NW = NT / 32;
    const int j = cols[blockIdx.x];
    const int64_t bs = B.cp[j], be = B.cp[j + 1];
    const int sg = pick_sg(flops[j], be - bs, 32);
    const int ntiles = (int)((A.nrows + R - 1) >> tile_log2);
    long long total = 0;
    for (int t = 0; t < ntiles; ++t) {
        const int64_t t0 = int64_t(t) << tile_log2;
        const int64_t rows = min(R, A.nrows - t0);
        const int W = (int)((rows + 31) >> 5);
        const int nch = (W + 31) >> 5;
        smem_zero(bm, W);
        __syncthreads();
        const int t0i = (int)t0;
        unsigned* bmp = bm;
        walk_balanced<4>(A, B, bs, be, sg, t, ntiles, (int)(t0 + rows), cursor + (t & 1) * B.span,
                         cursor + ((t + 1) & 1) * B.span, int64_t(4) * NT, ws,
                         per_product([bmp, t0i](int64_t, int64_t, int r) {
                             const int rr = r - t0i;
                             atomicOr(&bmp[rr >> 5], 1u << (rr & 31));
                         }));
        for (int c = warp; c < nch; c += NW) {
            const int w = c * 32 + lane;
            int x = w < W ? __popc(bm[w]) : 0;
            x = warp_reduce_sum(x);
            if (lane == 0) chunk[c] = x;
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
            if (lane == 0) {
                tot_sh = run;
                const unsigned long long off = atomicAdd(scur, (unsigned long long)run);
                off_sh = off;
                seg_off[int64_t(blockIdx.x) * T + t] = (int64_t)off;
                seg_cnt[int64_t(blockIdx.x) * T + t] = run;
            }
        }
        __syncthreads();
        const int64_t off = (int64_t)off_sh;
        for (int c = warp; c < nch; c += NW) {
            const int w = c * 32 + lane;
            emit_rows_coalesced(w < W ? bm[w] : 0u, (int)t0 + (w << 5), srows + off + chunk[c], lane);
        }
        total += tot_sh;
        __syncthreads();
    }
    if (tid == 0) cnt[j] = total;
}

// ------------------------------------------------------- K1 heavy, byte flags

// For the heaviest columns (flops >> rows per tile) the per-product shared
// atomic of k_fused_heavy is the bottleneck (ncu: ~10 L1 wavefronts per warp
// ATOMS).  Here a product is a plain byte store flags[row] = 1 (benign races:
// every writer stores the same value), and the pattern is recovered by
// scanning the tile's flag bytes twice (chunk counts, then coalesced emit +
// clear).  Tiles of 2^tile_log2 rows of byte flags (128 KB at 2^17), one CTA
// of NT threads per column.  Output = staging segments exactly like
// k_fused_heavy (seg index = column slot * T + tile).
__device__ __forceinline__ unsigned byte_mask16(uint4 v) {
    // flags are exactly 0 or 1: gather byte k's low bit into bit k
    auto m4 = [](unsigned x) { return (x & 1u) | ((x >> 7) & 2u) | ((x >> 14) & 4u) | ((x >> 21) & 8u); };
    return m4(v.x) | (m4(v.y) << 4) | (m4(v.z) << 8) | (m4(v.w) << 12);
}

template <int NT>
__global__ void __launch_bounds__(NT)
    k_fused_dense(DevCsc A, DevCsc B, const int* __restrict__ cols, int n, const int64_t* __restrict__ flops,
                  int tile_log2, int32_t* __restrict__ cursor, int64_t* __restrict__ cnt, int32_t* __restrict__ srows,
                  unsigned long long* __restrict__ scur, int64_t* __restrict__ seg_off, int* __restrict__ seg_cnt,
                  int T) {
    extern __shared__ __align__(16) unsigned char flags[];
    const int64_t R = int64_t(1) << tile_log2;
    int* chunk = reinterpret_cast<int*>(flags + R);  // [R/512] chunk bases
    __shared__ unsigned long long off_sh;
    __shared__ int tot_sh;
    __shared__ WalkShared ws;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int NW = NT / 32;
    const int j = cols[blockIdx.x];
    const int64_t bs = B.cp[j], be = B.cp[j + 1];
    const int sg = pick_sg(flops[j], be - bs, 32);
    const int ntiles = (int)((A.nrows + R - 1) >> tile_log2);
    smem_zero(reinterpret_cast<unsigned*>(flags), (int)(R >> 2));
    __syncthreads();
    long long total = 0;
    for (int t = 0; t < ntiles; ++t) {
        const int64_t t0 = int64_t(t) << tile_log2;
        const int64_t rows = min(R, A.nrows - t0);
        const int nch = (int)((rows + 511) >> 9);  // 512-byte chunks (32 lanes x 16 B)
        const int t0i = (int)t0;
        unsigned char* fl = flags;
        walk_balanced<4>(A, B, bs, be, sg, t, ntiles, (int)(t0 + rows), cursor + (t & 1) * B.span,
                         cursor + ((t + 1) & 1) * B.span, int64_t(4) * NT, ws,
                         per_product([fl, t0i](int64_t, int64_t, int r) { fl[r - t0i] = 1; }));
        const uint4* f4 = reinterpret_cast<const uint4*>(flags);
        for (int c = warp; c < nch; c += NW) {
            int x = __popc(byte_mask16(f4[c * 32 + lane]));
            x = warp_reduce_sum(x);
            if (lane == 0) chunk[c] = x;
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
            if (lane == 0) {
                tot_sh = run;
                const unsigned long long off = atomicAdd(scur, (unsigned long long)run);
                off_sh = off;
                seg_off[int64_t(blockIdx.x) * T + t] = (int64_t)off;
                seg_cnt[int64_t(blockIdx.x) * T + t] = run;
            }
        }
        __syncthreads();
        const int64_t off = (int64_t)off_sh;
        uint4* fw = reinterpret_cast<uint4*>(flags);
        for (int c = warp; c < nch; c += NW) {
            const uint4 v = fw[c * 32 + lane];
            const unsigned m = byte_mask16(v);
            emit_rows_coalesced(m, t0i + c * 512 + lane * 16, srows + off + chunk[c], lane);
            if (m) fw[c * 32 + lane] = make_uint4(0u, 0u, 0u, 0u);  // clear for the next tile
        }
        total += tot_sh;
        __syncthreads();
    }
    if (tid == 0) cnt[j] = total;
}

// ----------------------------------------------------------------------- K2

template <class T, bool ONES>
__global__ void __launch_bounds__(256)
    k_copy_light(const int* __restrict__ cols, int n, const int64_t* __restrict__ soff, const int64_t* __restrict__ Ccp,
                 const int32_t* __restrict__ srows, const T* __restrict__ svals, int32_t* __restrict__ Crw,
                 T* __restrict__ Cv) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
    for (int64_t ci = warp; ci < n; ci += nwarps) {
        const int j = cols[ci];
        const int64_t src = soff[j], dst = Ccp[j], m = Ccp[j + 1] - dst;
        for (int64_t i = lane; i < m; i += 32) {
            Crw[dst + i] = srows[src + i];
            if constexpr (ONES)
                Cv[dst + i] = (T)1;
            else
                Cv[dst + i] = svals[src + i];
        }
    }
}

template <class T, bool ONES>
__global__ void __launch_bounds__(256)
    k_copy_heavy(const int* __restrict__ cols, int T_, const int64_t* __restrict__ seg_off,
                 const int* __restrict__ seg_cnt, const int32_t* __restrict__ srows, const int64_t* __restrict__ Ccp,
                 int32_t* __restrict__ Crw, T* __restrict__ Cv) {
    const int j = cols[blockIdx.x];
    int64_t dst = Ccp[j];
    for (int t = 0; t < T_; ++t) {
        const int64_t src = seg_off[int64_t(blockIdx.x) * T_ + t];
        const int m = seg_cnt[int64_t(blockIdx.x) * T_ + t];
        for (int i = threadIdx.x; i < m; i += blockDim.x) {
            Crw[dst + i] = srows[src + i];
            if constexpr (ONES) Cv[dst + i] = (T)1;
        }
        dst += m;
    }
}

// ----------------------------------------------------------------------- K3

// Value accumulation for a batch of U products of one B entry: all U value
// loads are issued before any rank lookup / atomic, so the A-value gathers
// overlap like the row-id gathers do.
template <int SRID>
struct ValueBatch {
    using S_ = Sr<SRID>;
    using T = typename S_::T;
    using Acc = typename S_::Acc;
    const T* __restrict__ Av;
    const T* __restrict__ Bv;
    const unsigned* bm;
    const uint16_t* pre16;
    const int* chunk;
    Acc* vals;
    int r_lo;
    template <int U>
    __device__ __forceinline__ void batch(int64_t p, int width, int64_t i, const int* r, int ok) {
        if (!ok) return;  // bit 0 set whenever any bit is (the batch stops at the first miss)
        const T bv = Bv[i];
        T av[U];
        // unpredicated loads (a lane past the batch end re-reads position p)
        // so the compiler issues all U before the first use
#pragma unroll
        for (int u = 0; u < U; ++u) av[u] = Av[(ok & (1 << u)) ? p + int64_t(u) * width : p];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (ok & (1 << u)) {
                const int rr = r[u] - r_lo;
                const int w = rr >> 5;
                const int idx = chunk[w >> 5] + pre16[w] + __popc(bm[w] & ((1u << (rr & 31)) - 1u));
                S_::atomic_acc(&vals[idx], S_::mul(av[u], bv));
            }
        }
    }
};

// Values of heavy columns for semirings with values: per row tile the bitmap
// is rebuilt from C's (sorted) rows, popcount prefixes give every row its
// rank, one pass over the products accumulates at rank in shared memory (or
// straight into C when the tile holds more than `cap` entries).
template <int SRID, int NT>
__global__ void __launch_bounds__(NT)
    k_values_heavy(DevCsc A, DevCsc B, const int* __restrict__ cols, int n, const int64_t* __restrict__ flops,
                   const int64_t* __restrict__ Ccp, const int32_t* __restrict__ Crw,
                   typename Sr<SRID>::T* __restrict__ Cv, int tile_log2, int cap, int32_t* __restrict__ cursor,
                   int* __restrict__ err) {
    using S_ = Sr<SRID>;
    using T = typename S_::T;
    using Acc = typename S_::Acc;
    extern __shared__ __align__(16) unsigned char sm_raw[];
    const int64_t R = int64_t(1) << tile_log2;
    const int WMAX = (int)(R >> 5);
    Acc* vals = reinterpret_cast<Acc*>(sm_raw);
    unsigned* bm = reinterpret_cast<unsigned*>(sm_raw + sizeof(Acc) * cap);
    int* chunk = reinterpret_cast<int*>(bm + WMAX);                    // [WMAX/32]
    uint16_t* pre16 = reinterpret_cast<uint16_t*>(chunk + WMAX / 32);  // [WMAX]
    __shared__ int tot_sh;
    __shared__ int64_t hi_sh;
    __shared__ WalkShared ws;
    const int tid = threadIdx.x;
    const T* Av = static_cast<const T*>(A.v);
    const T* Bv = static_cast<const T*>(B.v);
    const int j = cols[blockIdx.x];
    const int64_t bs = B.cp[j], be = B.cp[j + 1];
    const int sg = pick_sg(flops[j], be - bs, 32);
    const int64_t ce = Ccp[j + 1];
    int64_t lo = Ccp[j];
    // Chunks are row ranges [r_lo, r_hi) holding at most `cap` output entries
    // (so values always accumulate in shared memory) and at most R rows (the
    // bitmap).  C's rows are known and sorted, so the boundaries come from C
    // itself; the product cursors advance monotonically as for fixed tiles.
    int r_lo = 0;
    for (int t = 0; lo < ce; ++t) {  // no output entries left -> no products left
        if (tid == 0) {
            const int64_t e_cap = lo + cap;
            const int64_t r_cand = e_cap < ce ? (int64_t)Crw[e_cap] : A.nrows;
            const int r_hi = (int)min(min(r_cand, int64_t(r_lo) + R), A.nrows);
            int64_t a = lo, b = min(ce, e_cap);
            while (a < b) {
                const int64_t mid = (a + b) >> 1;
                if (Crw[mid] < r_hi)
                    a = mid + 1;
                else
                    b = mid;
            }
            hi_sh = a;
            tot_sh = r_hi;
        }
        __syncthreads();
        const int64_t hi = hi_sh;
        const int r_hi = tot_sh;
        const int W = (r_hi - r_lo + 31) >> 5;
        smem_zero(bm, W);
        __syncthreads();
        for (int64_t e = lo + tid; e < hi; e += NT) {
            const int rr = Crw[e] - r_lo;
            atomicOr(&bm[rr >> 5], 1u << (rr & 31));
        }
        __syncthreads();
        const int tile_nnz = bitmap_ranks16(bm, pre16, chunk, W, &tot_sh);
        if (tile_nnz != hi - lo) {
            if (tid == 0) atomicExch(err, 1);
            return;
        }
        for (int i = tid; i < tile_nnz; i += NT) vals[i] = S_::identity();
        __syncthreads();
        // ntiles = 2 selects the cursor-driven walk (chunk count is data dependent)
        walk_balanced<8>(A, B, bs, be, sg, t, 2, r_hi, cursor + (t & 1) * B.span, cursor + ((t + 1) & 1) * B.span,
                         int64_t(8) * NT, ws, ValueBatch<SRID>{Av, Bv, bm, pre16, chunk, vals, r_lo});
        for (int i = tid; i < tile_nnz; i += NT) Cv[lo + i] = S_::out(vals[i]);
        lo = hi;
        r_lo = r_hi;
        __syncthreads();
    }
    if (tid == 0 && lo != ce) atomicExch(err, 1);
}

// ---------------------------------------------------- K3 as independent items

// One work item of the value pass: rows [r_lo, r_hi) of column `col`, whose
// output entries are C[lo, hi) (at most cap of them, at most R rows).
struct VItem {
    int col, r_lo, r_hi, pad;
    int64_t lo, hi;
};

// Cuts every heavy column's output into items (one thread per column; C's
// rows are sorted, so the boundaries are binary searches in C itself).
// fill == false: counts items per column into nit[h]; fill == true: writes
// them at items[off[h] ...].
// Columns with at most `split_flops` multiplies become ONE whole-column item
// (pad = 1: the CTA walks all its chunks with tile cursors, no searches);
// heavier ones are cut into independent single-chunk items (pad = 0).
__global__ void k_values_plan(const int* __restrict__ cols, int n, const int64_t* __restrict__ Ccp,
                              const int32_t* __restrict__ Crw, int64_t nrows, int64_t R, int cap, bool fill,
                              int64_t* __restrict__ nit, const int64_t* __restrict__ off, VItem* __restrict__ items,
                              const int64_t* __restrict__ flops, int64_t split_flops) {
    for (int h = blockIdx.x * blockDim.x + threadIdx.x; h < n; h += gridDim.x * blockDim.x) {
        const int j = cols[h];
        const int64_t ce = Ccp[j + 1];
        if (flops[j] <= split_flops) {
            if (fill) items[off[h]] = VItem{j, 0, (int)nrows, 1, Ccp[j], ce};
            else nit[h] = 1;
            continue;
        }
        int64_t lo = Ccp[j];
        int r_lo = 0;
        int64_t k = 0;
        while (lo < ce) {
            const int64_t e_cap = lo + cap;
            const int64_t r_cand = e_cap < ce ? (int64_t)Crw[e_cap] : nrows;
            const int r_hi = (int)min(min(r_cand, int64_t(r_lo) + R), nrows);
            int64_t a = lo, b = min(ce, e_cap);
            while (a < b) {
                const int64_t mid = (a + b) >> 1;
                if (Crw[mid] < r_hi)
                    a = mid + 1;
                else
                    b = mid;
            }
            if (a > lo) {  // skip row ranges without output (no products either)
                if (fill) items[off[h] + k] = VItem{j, r_lo, r_hi, 0, lo, a};
                ++k;
            }
            lo = a;
            r_lo = r_hi;
        }
        if (!fill) nit[h] = k;
    }
}

// One CTA per item: bitmap of the item's output rows (from C), 16-bit
// popcount ranks, values accumulated at rank in shared memory over all
// products with rows in [r_lo, r_hi) (start positions by binary search, so
// items of one column are independent and spread over SMs -- the heaviest
// column no longer serialises on one SM).
template <int SRID, int NT>
__global__ void __launch_bounds__(NT)
    k_values_items(DevCsc A, DevCsc B, const VItem* __restrict__ items, const int64_t* __restrict__ flops,
                   const int32_t* __restrict__ Crw, typename Sr<SRID>::T* __restrict__ Cv, int tile_log2, int cap,
                   int32_t* __restrict__ cursor, int* __restrict__ err) {
    using S_ = Sr<SRID>;
    using T = typename S_::T;
    using Acc = typename S_::Acc;
    extern __shared__ __align__(16) unsigned char sm_raw[];
    const int64_t R = int64_t(1) << tile_log2;
    const int WMAX = (int)(R >> 5);
    Acc* vals = reinterpret_cast<Acc*>(sm_raw);
    unsigned* bm = reinterpret_cast<unsigned*>(sm_raw + ((sizeof(Acc) * size_t(cap) + 15) & ~size_t(15)));
    int* chunk = reinterpret_cast<int*>(bm + WMAX);
    uint16_t* pre16 = reinterpret_cast<uint16_t*>(chunk + WMAX / 32);
    __shared__ int tot_sh, rhi_sh;
    __shared__ int64_t hi_sh;
    __shared__ WalkShared ws;
    const int tid = threadIdx.x;
    const T* Av = static_cast<const T*>(A.v);
    const T* Bv = static_cast<const T*>(B.v);
    const VItem it = items[blockIdx.x];
    const int j = it.col;
    const int64_t bs = B.cp[j], be = B.cp[j + 1];
    const int sg = pick_sg(flops[j], be - bs, 32);
    const int32_t* Arw = A.rw;
    const bool whole = it.pad == 1;  // all chunks of the column here, tile cursors between chunks
    int64_t lo = it.lo;
    int r_lo = it.r_lo;
    for (int t = 0; lo < it.hi; ++t) {
        int64_t hi;
        int r_hi;
        if (whole) {
            if (tid == 0) {
                const int64_t e_cap = lo + cap;
                const int64_t r_cand = e_cap < it.hi ? (int64_t)Crw[e_cap] : A.nrows;
                const int rh = (int)min(min(r_cand, int64_t(r_lo) + R), A.nrows);
                int64_t a = lo, b = min(it.hi, e_cap);
                while (a < b) {
                    const int64_t mid = (a + b) >> 1;
                    if (Crw[mid] < rh)
                        a = mid + 1;
                    else
                        b = mid;
                }
                hi_sh = a;
                rhi_sh = rh;
            }
            __syncthreads();
            hi = hi_sh;
            r_hi = rhi_sh;
        } else {
            hi = it.hi;
            r_hi = it.r_hi;
        }
        const int W = (r_hi - r_lo + 31) >> 5;
        smem_zero(bm, W);
        __syncthreads();
        for (int64_t e = lo + tid; e < hi; e += NT) {
            const int rr = Crw[e] - r_lo;
            atomicOr(&bm[rr >> 5], 1u << (rr & 31));
        }
        __syncthreads();
        const int tile_nnz = bitmap_ranks16(bm, pre16, chunk, W, &tot_sh);
        if (tile_nnz != hi - lo) {
            if (tid == 0) atomicExch(err, 1);
            return;
        }
        for (int i = tid; i < tile_nnz; i += NT) vals[i] = S_::identity();
        __syncthreads();
        ValueBatch<SRID> vb{Av, Bv, bm, pre16, chunk, vals, r_lo};
        if (whole) {
            // cursor-driven like k_fused_heavy's tiles (ntiles = 2: chunk count is data dependent)
            walk_balanced<8>(A, B, bs, be, sg, t, 2, r_hi, cursor + (t & 1) * B.span,
                             cursor + ((t + 1) & 1) * B.span, int64_t(8) * NT, ws, vb);
        } else {
            const int rl = r_lo;
            auto start_of = [Arw, rl](int64_t, int64_t as, int64_t ae) -> int64_t {
                if (rl == 0) return as;
                int64_t a = as, b = ae;  // first position with row >= rl
                while (a < b) {
                    const int64_t mid = (a + b) >> 1;
                    if (__ldg(&Arw[mid]) < rl)
                        a = mid + 1;
                    else
                        b = mid;
                }
                return a;
            };
            walk_balanced_from<8>(A, B, bs, be, sg, r_hi, nullptr, int64_t(8) * NT, ws, start_of, vb);
        }
        for (int i = tid; i < tile_nnz; i += NT) Cv[lo + i] = S_::out(vals[i]);
        lo = hi;
        r_lo = r_hi;
        __syncthreads();
    }
}

__global__ void k_count_ge(int n, const int* __restrict__ list, const int64_t* __restrict__ flops, int64_t thr,
                           int* __restrict__ out) {
    int c = 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) c += flops[list[i]] >= thr;
    c = warp_reduce_sum(c);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

// Staging bound: sum_j min(flops_j, nrows) (entries any column can produce).
__global__ void k_stage_bound(int64_t n, const int64_t* __restrict__ flops, int64_t nrows,
                              unsigned long long* __restrict__ out) {
    unsigned long long s = 0;
    for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < n; j += int64_t(gridDim.x) * blockDim.x)
        s += (unsigned long long)min(flops[j], nrows);
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(out, s);
}

// ==================================================================== host

namespace {

constexpr int kFusedHeavyThreads = 512;
constexpr int kValuesThreads = 1024;

template <int SRID, bool ONES, int LOG2S, int G, int CPB>
void launch_fused_light(Ctx& c, const DevCsc& A, const DevCsc& B, const int* list, int n, const int64_t* flops,
                        FusedState& f) {
    using Acc = typename Sr<SRID>::Acc;
    const size_t smem = ((ONES ? 0 : sizeof(Acc)) + sizeof(int)) * (size_t(CPB) << LOG2S);
    auto k = k_fused_light<SRID, ONES, LOG2S, G, CPB>;
    ensure_smem(k, smem);
    launch(c, k, dim3((unsigned)ceil_div(n, CPB)), dim3(G * CPB), smem, A, B, list, n, flops, f.cnt.as<int64_t>(),
           f.soff.as<int64_t>(), f.srows.as<int32_t>(), static_cast<typename Sr<SRID>::T*>(f.svals.get()),
           f.scur.as<unsigned long long>());
}

template <int SRID, bool ONES>
void launch_fused_light_bin(Ctx& c, int b, const DevCsc& A, const DevCsc& B, const int* l, int n,
                            const int64_t* flops, FusedState& f) {
    switch (b) {
    case 0: launch_fused_light<SRID, ONES, 6, 32, 8>(c, A, B, l, n, flops, f); break;
    case 1: launch_fused_light<SRID, ONES, 7, 32, 8>(c, A, B, l, n, flops, f); break;
    case 2: launch_fused_light<SRID, ONES, 8, 32, 8>(c, A, B, l, n, flops, f); break;
    case 3: launch_fused_light<SRID, ONES, 9, 64, 4>(c, A, B, l, n, flops, f); break;
    case 4: launch_fused_light<SRID, ONES, 10, 128, 2>(c, A, B, l, n, flops, f); break;
    case 5: launch_fused_light<SRID, ONES, 11, 256, 1>(c, A, B, l, n, flops, f); break;
    case 6: launch_fused_light<SRID, ONES, 12, 512, 1>(c, A, B, l, n, flops, f); break;
    case 7: launch_fused_light<SRID, ONES, 13, 1024, 1>(c, A, B, l, n, flops, f); break;
    }
}

int heavy_tile_log2(int want, int64_t nrows) {
    int tl = want;
    while (tl > 10 && (int64_t(1) << (tl - 1)) >= nrows) --tl;
    return tl;
}

}  // namespace

void fused_light_launch(Ctx& c, int sr, bool ones, int bin, const DevCsc& A, const DevCsc& B, const int* list, int n,
                        const int64_t* flops, FusedState& f) {
    dispatch_sr(sr, [&](auto id) {
        constexpr int ID = decltype(id)::value;
        if constexpr (ID == SLAPCU_OR_AND_U8) {
            if (ones) {
                launch_fused_light_bin<ID, true>(c, bin, A, B, list, n, flops, f);
                return;
            }
        }
        launch_fused_light_bin<ID, false>(c, bin, A, B, list, n, flops, f);
    });
}

// Staged light columns into C (values 1 for all-one OrAnd operands).
void fused_copy_light(Ctx& c, int sr, bool ones, const int* list, int n, const FusedState& f, const int64_t* c_colptr,
                      int32_t* crw, void* cv) {
    const int g = grid_for(c, int64_t(n) * 32, 256, 16);
    dispatch_sr(sr, [&](auto id) {
        constexpr int ID = decltype(id)::value;
        using T = typename Sr<ID>::T;
        if (ones)
            launch(c, k_copy_light<T, true>, dim3(g), dim3(256), 0, list, n, (const int64_t*)f.soff.as<int64_t>(),
                   c_colptr, (const int32_t*)f.srows.as<int32_t>(), (const T*)nullptr, crw, static_cast<T*>(cv));
        else
            launch(c, k_copy_light<T, false>, dim3(g), dim3(256), 0, list, n, (const int64_t*)f.soff.as<int64_t>(),
                   c_colptr, (const int32_t*)f.srows.as<int32_t>(), (const T*)f.svals.get(), crw,
                   static_cast<T*>(cv));
    });
}

int64_t fused_begin(Ctx& c, const DevCsc& A_, const DevCsc& B_, int sr, int alg, int64_t* c_colptr,
                    int64_t staging_budget_bytes) {
    check_operands(A_, B_);
    if (!c_colptr) throw Fail{SLAPCU_ERR_INVALID, "null colptr"};
    const int vs = value_size(sr);
    if (vs == 0) throw Fail{SLAPCU_ERR_INVALID, "unknown semiring"};
    DevCsc A = A_, B = B_;
    resolve(c, A);
    resolve(c, B);
    if ((A.span && !A.v) || (B.span && !B.v)) throw Fail{SLAPCU_ERR_INVALID, "operand values are null"};
    ctx_settle(c);  // the previous finish() on this context may still be running
    SLAPCU_CUDA(cudaEventRecord(c.ev[0], c.stream));
    FusedState& f = c.fused;
    f.valid = false;
    prepare_plan(c, A, B);
    const int64_t* flops = c.plan.flops.as<int64_t>();
    // Boolean fast path: no stored zero -> every product is 1
    f.ones = false;
    if (sr == SLAPCU_OR_AND_U8) {
        c.err_flag.reset(sizeof(int) * 2, c.stream);
        int* fl = c.err_flag.as<int>();
        SLAPCU_CUDA(cudaMemsetAsync(fl, 0, sizeof(int) * 2, c.stream));
        any_zero_u8(c, (const uint8_t*)A.v + A.base, A.span, fl + 1);
        any_zero_u8(c, (const uint8_t*)B.v + B.base, B.span, fl + 1);
        int hz = 0;
        SLAPCU_CUDA(cudaMemcpyAsync(&hz, fl + 1, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
        SLAPCU_CUDA(cudaStreamSynchronize(c.stream));
        f.ones = hz == 0;
    }
    // staging bound
    DevBuf bnd(sizeof(unsigned long long), c.stream);
    SLAPCU_CUDA(cudaMemsetAsync(bnd.get(), 0, sizeof(unsigned long long), c.stream));
    {
        KScope ks(c, KC_FLOPS);
        launch(c, k_stage_bound, dim3(grid_for(c, B.ncols, 256)), dim3(256), 0, B.ncols, flops, A.nrows,
               bnd.as<unsigned long long>());
    }
    unsigned long long bound = 0;
    SLAPCU_CUDA(cudaMemcpyAsync(&bound, bnd.get(), sizeof(bound), cudaMemcpyDeviceToHost, c.stream));
    SLAPCU_CUDA(cudaStreamSynchronize(c.stream));
    const int64_t stage_bytes = (int64_t)bound * (4 + (f.ones ? 0 : vs));
    if (staging_budget_bytes > 0 && stage_bytes > staging_budget_bytes)
        throw Fail{SLAPCU_ERR_BUDGET, "staging needs " + std::to_string(stage_bytes) + " bytes, budget " +
                                          std::to_string(staging_budget_bytes) + "; batch the columns"};
    f.srows.reset(sizeof(int32_t) * std::max<unsigned long long>(bound, 1), c.stream);
    if (!f.ones) f.svals.reset(size_t(vs) * std::max<unsigned long long>(bound, 1), c.stream);
    f.cnt.reset(sizeof(int64_t) * (B.ncols + 1), c.stream);
    f.soff.reset(sizeof(int64_t) * std::max<int64_t>(B.ncols, 1), c.stream);
    f.scur.reset(sizeof(unsigned long long), c.stream);
    SLAPCU_CUDA(cudaMemsetAsync(f.scur.get(), 0, sizeof(unsigned long long), c.stream));
    SLAPCU_CUDA(cudaMemsetAsync(f.cnt.as<int64_t>() + B.ncols, 0, sizeof(int64_t), c.stream));
    // bins by flops: light = shared hash, heavy = row-tiled bitmap
    BinSpec spec{};
    spec.nlight = 8;
    for (int b = 0; b < 8; ++b) spec.thr[b] = int64_t(32) << b;
    int64_t lmax = std::max<int64_t>(256, std::min<int64_t>(A.nrows / 128, 4096));
    if (c.opt.light_flops_max != Options{}.light_flops_max) lmax = std::min<int64_t>(c.opt.light_flops_max, 4096);
    spec.light_max = lmax;
    spec.all_heavy = alg == SLAPCU_ALG_HEAP;
    spec.key_is_nnz = 0;
    make_bins(c, B.ncols, flops, nullptr, spec, f.cnt.as<int64_t>(), f.bins);
    const int* L = f.bins.list.as<int>();
    const int nheavy = f.bins.count[spec.nlight];
    f.nlight_bins = spec.nlight;
    f.tile_log2 = heavy_tile_log2(c.opt.sym_tile_rows_log2, A.nrows);
    const int tb = (int)((A.nrows + (int64_t(1) << f.tile_log2) - 1) >> f.tile_log2);
    // byte-flag path for the heaviest columns (the heavy list is sorted by
    // flops, descending, so they are its first `ndense` entries)
    const int dense_log2 = heavy_tile_log2(std::min(c.opt.dense_tile_rows_log2, 17), A.nrows);
    const int td = (int)((A.nrows + (int64_t(1) << dense_log2) - 1) >> dense_log2);
    int ndense = 0;
    const int64_t dthr = c.opt.dense_flops_min < 0 ? std::max<int64_t>(A.nrows / 4, 1) : c.opt.dense_flops_min;
    if (nheavy && c.opt.dense_flops_min != 0) {
        DevBuf nd(sizeof(int), c.stream);
        SLAPCU_CUDA(cudaMemsetAsync(nd.get(), 0, sizeof(int), c.stream));
        KScope ks(c, KC_BIN);
        launch(c, k_count_ge, dim3(grid_for(c, nheavy, 256)), dim3(256), 0, nheavy, L + f.bins.offset[spec.nlight],
               flops, dthr, nd.as<int>());
        SLAPCU_CUDA(cudaMemcpyAsync(&ndense, nd.get(), sizeof(int), cudaMemcpyDeviceToHost, c.stream));
        SLAPCU_CUDA(cudaStreamSynchronize(c.stream));
    }
    f.T = std::max(tb, ndense ? td : 1);
    if (nheavy) {
        f.seg_off.reset(sizeof(int64_t) * int64_t(nheavy) * std::max(f.T, 1), c.stream);
        f.seg_cnt.reset(sizeof(int) * int64_t(nheavy) * std::max(f.T, 1), c.stream);
        SLAPCU_CUDA(cudaMemsetAsync(f.seg_cnt.get(), 0, sizeof(int) * int64_t(nheavy) * std::max(f.T, 1), c.stream));
    }
    dispatch_sr(sr, [&](auto id) {
        constexpr int ID = decltype(id)::value;
        for (int b = 0; b < spec.nlight; ++b) {
            const int n = f.bins.count[b];
            if (!n) continue;
            KScope ks(c, KC_SYM_LIGHT);
            if constexpr (ID == SLAPCU_OR_AND_U8) {
                if (f.ones)
                    launch_fused_light_bin<ID, true>(c, b, A, B, L + f.bins.offset[b], n, flops, f);
                else
                    launch_fused_light_bin<ID, false>(c, b, A, B, L + f.bins.offset[b], n, flops, f);
            } else {
                launch_fused_light_bin<ID, false>(c, b, A, B, L + f.bins.offset[b], n, flops, f);
            }
        }
    });
    const int* HL = L + f.bins.offset[spec.nlight];
    if (ndense) {
        KScope ks(c, KC_SYM_HEAVY);
        const size_t R = size_t(1) << dense_log2;
        const size_t smem = R + (R / 512) * 4 + 16;
        auto k = k_fused_dense<1024>;
        ensure_smem(k, smem);
        launch(c, k, dim3(ndense), dim3(1024), smem, A, B, HL, ndense, flops, dense_log2,
               c.plan.cursor.as<int32_t>(), f.cnt.as<int64_t>(), f.srows.as<int32_t>(),
               f.scur.as<unsigned long long>(), f.seg_off.as<int64_t>(), f.seg_cnt.as<int>(), f.T);
    }
    if (nheavy > ndense) {
        KScope ks(c, KC_SYM_HEAVY);
        const size_t W = size_t(1) << (f.tile_log2 - 5);
        const size_t smem = W * 4 + ((W + 31) / 32) * 4 + 16;
        const int nb = nheavy - ndense;
        // segment slots continue after the dense columns'
        int64_t* so = f.seg_off.as<int64_t>() + int64_t(ndense) * f.T;
        int* sc = f.seg_cnt.as<int>() + int64_t(ndense) * f.T;
        // a bitmap above ~96 KB leaves room for one CTA per SM: give it 1024 threads
        auto go = [&](auto k, int nt) {
            ensure_smem(k, smem);
            launch(c, k, dim3(nb), dim3(nt), smem, A, B, HL + ndense, nb, flops, f.tile_log2,
                   c.plan.cursor.as<int32_t>(), f.cnt.as<int64_t>(), f.srows.as<int32_t>(),
                   f.scur.as<unsigned long long>(), so, sc, f.T);
        };
        if (smem > 96 * 1024)
            go(k_fused_heavy<1024>, 1024);
        else
            go(k_fused_heavy<kFusedHeavyThreads>, kFusedHeavyThreads);
    }
    {
        KScope ks(c, KC_SCAN);
        exclusive_scan_i64(c, f.cnt.as<int64_t>(), c_colptr, B.ncols + 1);
    }
    int64_t total = 0;
    SLAPCU_CUDA(cudaMemcpyAsync(&total, c_colptr + B.ncols, sizeof(int64_t), cudaMemcpyDeviceToHost, c.stream));
    SLAPCU_CUDA(cudaEventRecord(c.ev[1], c.stream));
    SLAPCU_CUDA(cudaStreamSynchronize(c.stream));
    cudaEventElapsedTime(&c.sym_ms, c.ev[0], c.ev[1]);
    prof_flush(c);
    f.a_key = A.cp;
    f.b_key = B.cp;
    f.sr = sr;
    f.ncols = B.ncols;
    f.nnz = total;
    f.colptr = c_colptr;
    f.valid = true;
    return total;
}

void fused_finish(Ctx& c, const DevCsc& A_, const DevCsc& B_, int sr, int32_t* crw, void* cv) {
    FusedState& f = c.fused;
    if (!f.valid || f.a_key != A_.cp || f.b_key != B_.cp || f.sr != sr || f.ncols != B_.ncols)
        throw Fail{SLAPCU_ERR_INVALID, "spgemm_finish without a matching spgemm_begin on this context"};
    DevCsc A = A_, B = B_;
    resolve(c, A);
    resolve(c, B);
    SLAPCU_CUDA(cudaEventRecord(c.ev[2], c.stream));
    const int* L = f.bins.list.as<int>();
    const int nheavy = f.bins.count[f.nlight_bins];
    int nlight = 0;
    for (int b = 0; b < f.nlight_bins; ++b) nlight += f.bins.count[b];
    c.err_flag.reset(sizeof(int) * 2, c.stream);
    int* err = c.err_flag.as<int>();
    SLAPCU_CUDA(cudaMemsetAsync(err, 0, sizeof(int) * 2, c.stream));
    const int64_t* flops = c.plan.flops.as<int64_t>();
    dispatch_sr(sr, [&](auto id) {
        constexpr int ID = decltype(id)::value;
        using T = typename Sr<ID>::T;
        using Acc = typename Sr<ID>::Acc;
        T* Cv = static_cast<T*>(cv);
        KScope ks(c, KC_NUM_LIGHT);
        if (nlight) {
            const int g = grid_for(c, int64_t(nlight) * 32, 256, 16);
            if (f.ones)
                launch(c, k_copy_light<T, true>, dim3(g), dim3(256), 0, L, nlight, (const int64_t*)f.soff.as<int64_t>(),
                       (const int64_t*)f.colptr, (const int32_t*)f.srows.as<int32_t>(), (const T*)nullptr, crw, Cv);
            else
                launch(c, k_copy_light<T, false>, dim3(g), dim3(256), 0, L, nlight,
                       (const int64_t*)f.soff.as<int64_t>(), (const int64_t*)f.colptr,
                       (const int32_t*)f.srows.as<int32_t>(), (const T*)f.svals.get(), crw, Cv);
        }
        if (nheavy) {
            const int* hl = L + f.bins.offset[f.nlight_bins];
            if (f.ones)
                launch(c, k_copy_heavy<T, true>, dim3(nheavy), dim3(256), 0, hl, f.T,
                       (const int64_t*)f.seg_off.as<int64_t>(), (const int*)f.seg_cnt.as<int>(),
                       (const int32_t*)f.srows.as<int32_t>(), (const int64_t*)f.colptr, crw, Cv);
            else
                launch(c, k_copy_heavy<T, false>, dim3(nheavy), dim3(256), 0, hl, f.T,
                       (const int64_t*)f.seg_off.as<int64_t>(), (const int*)f.seg_cnt.as<int>(),
                       (const int32_t*)f.srows.as<int32_t>(), (const int64_t*)f.colptr, crw, Cv);
            if (!f.ones) {
                KScope ks2(c, KC_NUM_HEAVY);
                // One CTA of 1024 threads per SM: bitmap + 16-bit ranks for up to
                // 2^19 rows (98 KB) and the rest of the SM's shared memory for
                // the item's values.  Items (<= cap entries, <= 2^19 rows) are
                // planned from C's rows and processed independently.
                const int tl = heavy_tile_log2(std::min(c.opt.tile_rows_log2 + 1, 19), A.nrows);
                const size_t W = size_t(1) << (tl - 5);
                const size_t fixed = W * 4 + ((W + 31) / 32) * 4 + W * 2 + 64;
                const size_t budget = size_t(c.smem_optin) - 8 * 1024;  // static state + reserve
                const int cap = (int)((budget - fixed) / sizeof(Acc)) & ~3;
                const size_t smem = fixed + size_t(cap) * sizeof(Acc) + 16;
                DevBuf nit(sizeof(int64_t) * (nheavy + 1), c.stream), ioff(sizeof(int64_t) * (nheavy + 1), c.stream);
                SLAPCU_CUDA(cudaMemsetAsync(nit.as<int64_t>() + nheavy, 0, sizeof(int64_t), c.stream));
                const int pg = grid_for(c, nheavy, 128);
                // columns above this many multiplies are split over several CTAs
                const int64_t split = int64_t(4) << 20;
                launch(c, k_values_plan, dim3(pg), dim3(128), 0, hl, nheavy, (const int64_t*)f.colptr,
                       (const int32_t*)crw, A.nrows, int64_t(1) << tl, cap, false, nit.as<int64_t>(),
                       (const int64_t*)nullptr, (VItem*)nullptr, flops, split);
                exclusive_scan_i64(c, nit.as<int64_t>(), ioff.as<int64_t>(), nheavy + 1);
                int64_t nitems = 0;
                SLAPCU_CUDA(cudaMemcpyAsync(&nitems, ioff.as<int64_t>() + nheavy, sizeof(int64_t),
                                            cudaMemcpyDeviceToHost, c.stream));
                SLAPCU_CUDA(cudaStreamSynchronize(c.stream));
                if (nitems > INT32_MAX) throw Fail{SLAPCU_ERR_INVALID, "too many value-pass items"};
                f.items.reset(sizeof(VItem) * std::max<int64_t>(nitems, 1), c.stream);
                launch(c, k_values_plan, dim3(pg), dim3(128), 0, hl, nheavy, (const int64_t*)f.colptr,
                       (const int32_t*)crw, A.nrows, int64_t(1) << tl, cap, true, nit.as<int64_t>(),
                       (const int64_t*)ioff.as<int64_t>(), f.items.as<VItem>(), flops, split);
                auto k = k_values_items<ID, kValuesThreads>;
                ensure_smem(k, smem);
                launch(c, k, dim3((unsigned)nitems), dim3(kValuesThreads), smem, A, B,
                       (const VItem*)f.items.as<VItem>(), flops, (const int32_t*)crw, Cv, tl, cap,
                       c.plan.cursor.as<int32_t>(), err);
            }
        }
    });
    if (!c.err_host) SLAPCU_CUDA(cudaMallocHost((void**)&c.err_host, sizeof(int)));
    SLAPCU_CUDA(cudaMemcpyAsync(c.err_host, err, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
    SLAPCU_CUDA(cudaEventRecord(c.ev[3], c.stream));
    c.err_pending = true;
    if (!c.opt.async_finish) ctx_settle(c);
}

// Completes an asynchronous finish(): waits for the context stream and raises
// the deferred InternalError, if any.
void ctx_settle(Ctx& c) {
    if (!c.err_pending) return;
    c.err_pending = false;
    SLAPCU_CUDA(cudaStreamSynchronize(c.stream));
    cudaEventElapsedTime(&c.num_ms, c.ev[2], c.ev[3]);
    prof_flush(c);
    if (*c.err_host) throw Fail{SLAPCU_ERR_INTERNAL, "numeric column nnz disagrees with symbolic count"};
}

}  // namespace slapcu
