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
        walk_balanced<4>(A, B, bs, be, sg, t, ntiles, (int)(t0 + rows), cursor + (t & 1) * B.span,
                         cursor + ((t + 1) & 1) * B.span, int64_t(4) * NT, ws, [&](int64_t, int64_t, int r) {
                             const int rr = r - (int)t0;
                             atomicOr(&bm[rr >> 5], 1u << (rr & 31));
                         });
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
    int* pre = reinterpret_cast<int*>(bm + WMAX);
    int* chunk = pre + WMAX;
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
        const int tile_nnz = bitmap_ranks(bm, pre, chunk, W, &tot_sh);
        if (tile_nnz != hi - lo) {
            if (tid == 0) atomicExch(err, 1);
            return;
        }
        for (int i = tid; i < tile_nnz; i += NT) vals[i] = S_::identity();
        __syncthreads();
        // ntiles = 2 selects the cursor-driven walk (chunk count is data dependent)
        walk_balanced<4>(A, B, bs, be, sg, t, 2, r_hi, cursor + (t & 1) * B.span, cursor + ((t + 1) & 1) * B.span,
                         int64_t(4) * NT, ws, [&](int64_t p, int64_t i, int r) {
                             const int rr = r - r_lo;
                             const int w = rr >> 5;
                             const int idx = pre[w] + __popc(bm[w] & ((1u << (rr & 31)) - 1u));
                             S_::atomic_acc(&vals[idx], S_::mul(Av[p], Bv[i]));
                         });
        for (int i = tid; i < tile_nnz; i += NT) Cv[lo + i] = S_::out(vals[i]);
        lo = hi;
        r_lo = r_hi;
        __syncthreads();
    }
    if (tid == 0 && lo != ce) atomicExch(err, 1);
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
constexpr int kValuesThreads = 512;

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
    f.T = (int)((A.nrows + (int64_t(1) << f.tile_log2) - 1) >> f.tile_log2);
    if (nheavy) {
        f.seg_off.reset(sizeof(int64_t) * int64_t(nheavy) * std::max(f.T, 1), c.stream);
        f.seg_cnt.reset(sizeof(int) * int64_t(nheavy) * std::max(f.T, 1), c.stream);
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
    if (nheavy) {
        KScope ks(c, KC_SYM_HEAVY);
        const size_t W = size_t(1) << (f.tile_log2 - 5);
        const size_t smem = W * 4 + ((W + 31) / 32) * 4 + 16;
        auto k = k_fused_heavy<kFusedHeavyThreads>;
        ensure_smem(k, smem);
        launch(c, k, dim3(nheavy), dim3(kFusedHeavyThreads), smem, A, B, L + f.bins.offset[spec.nlight], nheavy,
               flops, f.tile_log2, c.plan.cursor.as<int32_t>(), f.cnt.as<int64_t>(), f.srows.as<int32_t>(),
               f.scur.as<unsigned long long>(), f.seg_off.as<int64_t>(), f.seg_cnt.as<int>(), f.T);
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
                // bitmap + ranks for up to 2^17 rows, the rest of ~113 KB (two
                // CTAs per SM) holds the chunk's values
                const int tl = heavy_tile_log2(std::min(c.opt.tile_rows_log2, 17), A.nrows);
                const size_t W = size_t(1) << (tl - 5);
                const size_t fixed = W * 8 + ((W + 31) / 32) * 4 + 64;
                // 112 KB: two CTAs per SM once the per-CTA reserved 1 KB and the
                // static shared state are added (228 KB per SM)
                size_t budget = std::min<size_t>(size_t(c.smem_optin), size_t(108) * 1024);
                if (budget < fixed + 1024 * sizeof(Acc)) budget = size_t(c.smem_optin);
                // multiple of 4 entries keeps the bitmap behind the values 16-byte aligned
                const int cap = (int)((budget - fixed) / sizeof(Acc)) & ~3;
                const size_t smem = fixed + size_t(cap) * sizeof(Acc);
                auto k = k_values_heavy<ID, kValuesThreads>;
                ensure_smem(k, smem);
                launch(c, k, dim3(nheavy), dim3(kValuesThreads), smem, A, B, hl, nheavy, flops,
                       (const int64_t*)f.colptr, (const int32_t*)crw, Cv, tl, cap, c.plan.cursor.as<int32_t>(), err);
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

}  // namespace slapcu
