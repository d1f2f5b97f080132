// direct.cu -- one-pass SpGEMM that writes C in place (no staging of heavy
// columns).
//
// The reference forms C in two passes, symbolic counts then numeric fill
// (spgemm.hpp:286-330), so every product is walked twice.  fused.cu walks
// once but stages every output column and copies it into place, which costs
// 8 extra bytes of HBM traffic per output entry -- at R-MAT s20 that is more
// than C itself.  Here heavy columns are cut into (column, row tile) items,
// laid out in C order, and each item is formed in a shared-memory bitmap,
// counted, given its output offset by a decoupled look-back over the items
// before it, and emitted straight into C:
//
//   A tile pointers   Atp[k][t] = first position of A(:,k) with row >= t*R
//                     (per A, cached): an item walks exactly its rows of every
//                     A(:,k), k in B(:,j), with no cursors and no searches.
//   light columns     (flops <= L) shared-memory hash + sort (fused.cu), staged;
//                     they hold ~1% of C and are copied at the end.
//   dense items       (flops > H) formed first by k_tile_dense, kept as a
//                     global bitmap (R/8 bytes) with their count pre-published,
//                     so no item in the ordered pass waits behind a long one.
//   k_tile_direct     persistent CTAs take items by ticket in C order: walk,
//                     count (touched-word summary, so sparse items never scan
//                     the whole bitmap), look back, emit rows + values.
//   colptr            = exclusive scan of light + heavy per-column counts.
//
// Pattern semirings only (OrAnd); value semirings use fused.cu.
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "kern.cuh"

namespace slapcu {

namespace {

constexpr int kShortRun = 32;   // runs shorter than this are walked by one thread
constexpr int kUnit = 512;      // products per warp work unit on long runs
constexpr unsigned long long kFlagAgg = 1ull << 62, kFlagIncl = 2ull << 62, kValMask = (1ull << 62) - 1;

__device__ __forceinline__ void st_release(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// Look-back reads only use the state word itself, so relaxed suffices (an
// acquire load invalidates L1 on every spin).
__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Exclusive block-wide scan of one int per thread; *total gets the sum.
template <int NT>
__device__ __forceinline__ int block_excl_scan(int v, int* wsum, int* total) {
    constexpr int NW = NT / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int wt;
    const int ex = warp_excl_scan(v, lane, &wt);
    if (lane == 0) wsum[warp] = wt;
    __syncthreads();
    if (warp == 0) {
        const int x = lane < NW ? wsum[lane] : 0;
        int t;
        const int e = warp_excl_scan(x, lane, &t);
        if (lane < NW) wsum[lane] = e;
        if (lane == 0) wsum[NW] = t;
    }
    __syncthreads();
    const int r = ex + wsum[warp];
    *total = wsum[NW];
    return r;
}

template <int NT>
struct WalkSm {
    int wsum[NT / 32 + 1];
    int ustart[NT];
    int len[NT];
    int64_t start[NT];
};

// Marks row rr of the current tile (bitmap at shared address bmA): test
// before set (a plain shared load is a broadcast for lanes hitting one word,
// and most products of a dense column find their bit already set); the first
// touch of a word also sets its summary bit (summary at sumA).
template <bool SUMM>
__device__ __forceinline__ void mark(unsigned bmA, unsigned sumA, int rr) {
    const int w = rr >> 5;
    const unsigned a = bmA + (unsigned(w) << 2);
    const unsigned b = 1u << (rr & 31);
    if (!(lds_u32(a) & b)) {
        const unsigned old = atoms_or(a, b);
        if (SUMM && old == 0) atoms_or(sumA + (unsigned(w >> 5) << 2), 1u << (w & 31));
    }
}

// All products of item (column j of B, row tile t) into the tile bitmap.
// B entries are taken NT at a time; a thread walks its own run when it is
// short, long runs are cut into units of kUnit products that the warps walk
// lane-strided with U loads in flight (coalesced, balanced across warps).
template <int NT, int U, bool SUMM>
__device__ __forceinline__ void tile_walk(const DevCsc& A, const DevCsc& B, const int32_t* __restrict__ Atp, int T,
                                          int j, int t, int t0, unsigned* bm, unsigned* summ, WalkSm<NT>& sh) {
    constexpr int NW = NT / 32;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t bs = B.cp[j], be = B.cp[j + 1];
    const int32_t* __restrict__ Arw = A.rw;
    const unsigned bmA = smem_addr(bm), sumA = SUMM ? smem_addr(summ) : 0u;
    for (int64_t base = bs; base < be; base += NT) {
        const int64_t i = base + tid;
        int units = 0, len = 0;
        int64_t s = 0;
        if (i < be) {
            const int k = B.rw[i];
            const int32_t* tp = Atp + int64_t(k) * (T + 1) + t;
            const int lo = tp[0], hi = tp[1];
            s = A.cp[k] + lo;
            len = hi - lo;
            if (len < kShortRun) {
                const int32_t* q = Arw + s;
                for (int x = 0; x < len; ++x) mark<SUMM>(bmA, sumA, __ldg(q + x) - t0);
                len = 0;
            } else {
                units = (len + kUnit - 1) / kUnit;
            }
        }
        int tot;
        const int ex = block_excl_scan<NT>(units, sh.wsum, &tot);
        sh.ustart[tid] = ex;
        sh.len[tid] = len;
        sh.start[tid] = s;
        __syncthreads();
        for (int u = warp; u < tot; u += NW) {
            // entry owning unit u: the last e with ustart[e] <= u
            int lo = 0, hi = NT - 1;
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (sh.ustart[mid] <= u)
                    lo = mid;
                else
                    hi = mid - 1;
            }
            const int c0 = (u - sh.ustart[lo]) * kUnit;
            const int32_t* run = Arw + sh.start[lo] + c0;
            const int m = min(kUnit, sh.len[lo] - c0);
            for (int x = lane; x < m; x += 32 * U) {
                int r[U];
#pragma unroll
                for (int v = 0; v < U; ++v) r[v] = x + 32 * v < m ? __ldg(run + x + 32 * v) : -1;
#pragma unroll
                for (int v = 0; v < U; ++v)
                    if (r[v] >= 0) mark<SUMM>(bmA, sumA, r[v] - t0);
            }
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------ dense items

// One CTA per dense item: bitmap of the tile -> global (W words), count
// pre-published into the look-back state as an aggregate.
template <int NT>
__global__ void __launch_bounds__(NT)
    k_tile_dense(DevCsc A, DevCsc B, const int32_t* __restrict__ Atp, int T, int TL, const int2* __restrict__ items,
                 const int* __restrict__ dlist, unsigned* __restrict__ gbm, unsigned long long* __restrict__ state) {
    extern __shared__ __align__(16) unsigned bm[];
    __shared__ WalkSm<NT> sh;
    __shared__ int red[NT / 32];
    const int W = 1 << (TL - 5);
    const int item = dlist[blockIdx.x];
    const int2 it = items[item];
    smem_zero(bm, W);
    __syncthreads();
    tile_walk<NT, 4, false>(A, B, Atp, T, it.x, it.y, it.y << TL, bm, nullptr, sh);
    uint4* dst = reinterpret_cast<uint4*>(gbm + int64_t(blockIdx.x) * W);
    const uint4* src = reinterpret_cast<const uint4*>(bm);
    int cnt = 0;
    for (int q = threadIdx.x; q < W / 4; q += NT) {
        const uint4 x = src[q];
        dst[q] = x;
        cnt += __popc(x.x) + __popc(x.y) + __popc(x.z) + __popc(x.w);
    }
    cnt = warp_reduce_sum(cnt);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = cnt;
    __syncthreads();
    if (threadIdx.x == 0) {
        long long s = 0;
        for (int w = 0; w < NT / 32; ++w) s += red[w];
        state[item] = kFlagAgg | (unsigned long long)s;
    }
}

// ------------------------------------------------------------ ordered pass

struct DirectArgs {
    DevCsc A, B;
    const int32_t* Atp;
    int T, TL;
    const int2* items;
    const int* dslot;  // per item: slot in gbm, or -1
    int nitems;
    const unsigned* gbm;
    unsigned long long* state;
    int* ticket;
    const int64_t* lp;  // light prefix per column
    unsigned long long* hcnt;  // heavy entries per column
    int32_t* crw;
    uint8_t* cv;
    int64_t capacity;
    int* overflow;
};

template <int NT>
__global__ void __launch_bounds__(NT) k_tile_direct(DirectArgs g) {
    constexpr int NW = NT / 32;
    extern __shared__ __align__(16) unsigned char sm_raw[];
    const int W = 1 << (g.TL - 5), WS = W >> 5;
    unsigned* bm = reinterpret_cast<unsigned*>(sm_raw);
    unsigned* summ = bm + W;                                       // [WS]
    int* chunk = reinterpret_cast<int*>(summ + WS);                // [W/32 + 1] chunk bases
    uint16_t* tl = reinterpret_cast<uint16_t*>(chunk + W / 32 + 1);  // [W] touched words
    __shared__ WalkSm<NT> sh;
    __shared__ int item_sh, ntouch_sh;
    __shared__ unsigned long long excl_sh;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    smem_zero(bm, W + WS);
    __syncthreads();
    for (;;) {
        if (tid == 0) item_sh = atomicAdd(g.ticket, 1);
        __syncthreads();
        const int item = item_sh;
        if (item >= g.nitems) break;
        const int2 it = g.items[item];
        const int j = it.x, t = it.y, t0 = t << g.TL;
        const int ds = g.dslot[item];
        if (ds < 0) {
            tile_walk<NT, 4, true>(g.A, g.B, g.Atp, g.T, j, t, t0, bm, summ, sh);
        } else {
            const uint4* src = reinterpret_cast<const uint4*>(g.gbm + int64_t(ds) * W);
            uint4* d4 = reinterpret_cast<uint4*>(bm);
            for (int q = tid; q < W / 4; q += NT) d4[q] = src[q];
            for (int q = tid; q < WS; q += NT) summ[q] = ~0u;
            __syncthreads();
        }
        // touched words in order: summary popcounts -> scan -> list
        {
            unsigned s = 0;
            int c = 0;
            for (int q = tid; q < WS; q += NT) {  // WS <= NT for TL <= 5 + 5 + log2(NT)
                s = summ[q];
                c = __popc(s);
            }
            int tot;
            int base = block_excl_scan<NT>(c, sh.wsum, &tot);
            if (tid < WS) {
                while (s) {
                    const int b = __ffs(s) - 1;
                    s &= s - 1;
                    tl[base++] = (uint16_t)(tid * 32 + b);
                }
            }
            if (tid == 0) ntouch_sh = tot;
            __syncthreads();
        }
        const int U = ntouch_sh;
        const int nch = (U + 31) >> 5;
        for (int cc = warp; cc < nch; cc += NW) {
            const int u = cc * 32 + lane;
            int x = u < U ? __popc(bm[tl[u]]) : 0;
            x = warp_reduce_sum(x);
            if (lane == 0) chunk[cc] = x;
        }
        __syncthreads();
        if (warp == 0) {
            int run = 0;
            for (int b0 = 0; b0 < nch; b0 += 32) {
                const int cix = b0 + lane;
                const int x = cix < nch ? chunk[cix] : 0;
                int tt;
                const int e = warp_excl_scan(x, lane, &tt);
                if (cix < nch) chunk[cix] = run + e;
                run += tt;
            }
            const unsigned long long cnt = (unsigned long long)run;
            // decoupled look-back over the items before this one (C order)
            unsigned long long excl = 0;
            if (item == 0) {
                if (lane == 0) st_release(&g.state[0], kFlagIncl | cnt);
            } else {
                if (ds < 0 && lane == 0) st_release(&g.state[item], kFlagAgg | cnt);
                long long q0 = item - 1;
                for (;;) {
                    const long long q = q0 - lane;
                    const unsigned long long s = q >= 0 ? ld_relaxed(&g.state[q]) : kFlagIncl;
                    const unsigned fl = (unsigned)(s >> 62);
                    const unsigned incl = __ballot_sync(0xffffffffu, fl == 2);
                    const unsigned ready = __ballot_sync(0xffffffffu, fl != 0);
                    const int L = incl ? __ffs(incl) - 1 : 31;
                    const unsigned need = L == 31 ? 0xffffffffu : ((2u << L) - 1u);
                    if ((ready & need) != need) {
                        __nanosleep(32);
                        continue;
                    }
                    unsigned long long v = lane <= L ? (s & kValMask) : 0ull;
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                    excl += v;
                    if (incl) break;
                    q0 -= 32;
                }
                if (lane == 0) st_release(&g.state[item], kFlagIncl | (excl + cnt));
            }
            if (lane == 0) {
                excl_sh = excl;
                chunk[nch] = run;
                atomicAdd(&g.hcnt[j], cnt);
            }
        }
        __syncthreads();
        const int cnt = chunk[nch];
        const int64_t off = g.lp[j] + (int64_t)excl_sh;
        if (off + cnt <= g.capacity) {
            for (int cc = warp; cc < nch; cc += NW) {
                const int u = cc * 32 + lane;
                const int w = u < U ? tl[u] : 0;
                emit_rows_coalesced(u < U ? bm[w] : 0u, t0 + (w << 5), g.crw + off + chunk[cc], lane);
            }
            if (g.cv)
                for (int q = tid; q < cnt; q += NT) g.cv[off + q] = 1;
        } else if (tid == 0) {
            atomicExch(g.overflow, 1);
        }
        __syncthreads();
        for (int u = tid; u < U; u += NT) bm[tl[u]] = 0u;
        for (int q = tid; q < WS; q += NT) summ[q] = 0u;
        __syncthreads();
    }
}

// ------------------------------------------------------------ item setup

// Atp[k][t] (int32, relative to A.cp[k]) = first entry of A(:,k) with row >=
// t << TL, for t = 0..T.
__global__ void k_tile_ptr(DevCsc A, int TL, int T, int32_t* __restrict__ Atp) {
    const int64_t n = A.ncols * int64_t(T + 1);
    for (int64_t x = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; x < n; x += int64_t(gridDim.x) * blockDim.x) {
        const int64_t k = x / (T + 1);
        const int t = (int)(x - k * (T + 1));
        const int64_t as = A.cp[k], ae = A.cp[k + 1];
        int64_t lo = as, hi = ae;
        if (t == 0) {
            hi = as;
        } else if (t == T) {
            lo = ae;
        } else {
            const int64_t bound = int64_t(t) << TL;
            while (lo < hi) {
                const int64_t mid = (lo + hi) >> 1;
                if (A.rw[mid] < bound)
                    lo = mid + 1;
                else
                    hi = mid;
            }
        }
        Atp[x] = (int32_t)(lo - as);
    }
}

// Per heavy column (in column order) and tile: multiplies, and the number of
// tiles with work.  One warp per column.
__global__ void k_item_flops(DevCsc A, DevCsc B, const int32_t* __restrict__ Atp, int T, const int* __restrict__ hl,
                             int nh, int64_t* __restrict__ iflops, int64_t* __restrict__ nit) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
    for (int64_t h = w0; h < nh; h += nw) {
        const int j = hl[h];
        const int64_t bs = B.cp[j], be = B.cp[j + 1];
        int64_t items = 0;
        for (int t = 0; t < T; ++t) {
            long long f = 0;
            for (int64_t i = bs + lane; i < be; i += 32) {
                const int32_t* tp = Atp + int64_t(B.rw[i]) * (T + 1) + t;
                f += tp[1] - tp[0];
            }
            f = warp_reduce_sum64(f);
            if (lane == 0) iflops[h * T + t] = f;
            items += f > 0;
        }
        if (lane == 0) nit[h] = items;
    }
}

__global__ void k_item_fill(const int* __restrict__ hl, int nh, int T, const int64_t* __restrict__ iflops,
                            const int64_t* __restrict__ ioff, int64_t dense_min, int2* __restrict__ items,
                            int* __restrict__ dflag) {
    for (int64_t h = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; h < nh; h += int64_t(gridDim.x) * blockDim.x) {
        int64_t o = ioff[h];
        const int j = hl[h];
        for (int t = 0; t < T; ++t) {
            const int64_t f = iflops[h * T + t];
            if (f > 0) {
                items[o] = make_int2(j, t);
                dflag[o] = f >= dense_min ? 1 : 0;
                ++o;
            }
        }
    }
}

// dslot[i] = exclusive prefix of dflag at dense items, -1 elsewhere; dlist
// inverts it.
__global__ void k_dense_slots(int n, const int* __restrict__ dflag, const int* __restrict__ dpre,
                              int* __restrict__ dslot, int* __restrict__ dlist) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        if (dflag[i]) {
            dslot[i] = dpre[i];
            dlist[dpre[i]] = i;
        } else {
            dslot[i] = -1;
        }
    }
}

__global__ void k_add_counts(int64_t n, const int64_t* __restrict__ a, const unsigned long long* __restrict__ b,
                             int64_t* __restrict__ out) {
    for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < n; j += int64_t(gridDim.x) * blockDim.x)
        out[j] = a[j] + (int64_t)b[j];
}

__global__ void k_mark_heavy(int64_t n, const int64_t* __restrict__ flops, int64_t lmax, bool all_heavy,
                             int* __restrict__ flag) {
    for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < n; j += int64_t(gridDim.x) * blockDim.x)
        flag[j] = flops[j] > 0 && (all_heavy || flops[j] > lmax);
}

__global__ void k_scatter_heavy(int64_t n, const int* __restrict__ flag, const int* __restrict__ pre,
                                int* __restrict__ hl) {
    for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < n; j += int64_t(gridDim.x) * blockDim.x)
        if (flag[j]) hl[pre[j]] = (int)j;
}

void excl_scan_i32(Ctx& c, const int* in, int* out, int64_t n) {
    size_t tb = 0;
    SLAPCU_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, n, c.stream));
    DevBuf tmp(tb, c.stream);
    timed(c, KC_SCAN, [&] { SLAPCU_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(), tb, in, out, n, c.stream)); });
    ++c.launches;
}

template <class T>
T d2h(Ctx& c, const T* p) {
    T v{};
    SLAPCU_CUDA(cudaMemcpyAsync(&v, p, sizeof(T), cudaMemcpyDeviceToHost, c.stream));
    SLAPCU_CUDA(cudaStreamSynchronize(c.stream));
    return v;
}

constexpr int kDirectThreads = 256;
constexpr int kDenseThreads = 512;

}  // namespace

int direct_tile_log2(const Ctx& c, int64_t nrows) {
    int tl = std::min(c.opt.direct_tile_rows_log2, 18);  // summary words <= threads per CTA
    while (tl > 10 && (int64_t(1) << (tl - 1)) >= nrows) --tl;
    return tl;
}

// Tile pointers of A for row tiles of 2^TL rows (cached on the context).
static const int32_t* tile_pointers(Ctx& c, const DevCsc& A, int TL, int T) {
    DirectCache& d = c.direct;
    if (d.atp_valid && d.atp_key == A.cp && d.atp_ncols == A.ncols && d.atp_tl == TL && d.atp_nnz == A.nnz)
        return d.atp.as<int32_t>();
    d.atp.reset(sizeof(int32_t) * size_t(A.ncols) * (T + 1), c.stream);
    KScope ks(c, KC_BIN);
    launch(c, k_tile_ptr, dim3(grid_for(c, A.ncols * (T + 1), 256)), dim3(256), 0, A, TL, T, d.atp.as<int32_t>());
    d.atp_key = A.cp;
    d.atp_ncols = A.ncols;
    d.atp_nnz = A.nnz;
    d.atp_tl = TL;
    d.atp_valid = true;
    return d.atp.as<int32_t>();
}

// Fallback for semirings with values (and OrAnd operands holding stored
// zeros, whose pattern is structural but whose values are not all 1): the
// fused begin/finish pair into the caller's buffers.
static int64_t direct_fallback(Ctx& c, const DevCsc& A, const DevCsc& B, int sr, int alg, int64_t capacity,
                               int64_t* c_colptr, int32_t* crw, void* cv) {
    const int64_t nnz = fused_begin(c, A, B, sr, alg, c_colptr, 0);
    c.direct.last_nnz = nnz;
    if (nnz > capacity)
        throw Fail{SLAPCU_ERR_BUDGET, "output needs " + std::to_string(nnz) + " entries, capacity " +
                                          std::to_string(capacity)};
    fused_finish(c, A, B, sr, crw, cv);
    ctx_settle(c);
    return nnz;
}

int64_t direct_spgemm(Ctx& c, const DevCsc& A_, const DevCsc& B_, int sr, int alg, int64_t capacity,
                      int64_t* c_colptr, int32_t* crw, void* cv) {
    check_operands(A_, B_);
    if (!c_colptr) throw Fail{SLAPCU_ERR_INVALID, "null colptr"};
    if (value_size(sr) == 0) throw Fail{SLAPCU_ERR_INVALID, "unknown semiring"};
    if (capacity > 0 && (!crw || !cv)) throw Fail{SLAPCU_ERR_INVALID, "null output buffers"};
    DevCsc A = A_, B = B_;
    resolve(c, A);
    resolve(c, B);
    if ((A.span && !A.v) || (B.span && !B.v)) throw Fail{SLAPCU_ERR_INVALID, "operand values are null"};
    ctx_settle(c);
    if (sr != SLAPCU_OR_AND_U8) return direct_fallback(c, A_, B_, sr, alg, capacity, c_colptr, crw, cv);
    // OrAnd: if no stored value is 0 every product is 1 (pattern only)
    c.err_flag.reset(sizeof(int) * 2, c.stream);
    int* fl = c.err_flag.as<int>();
    SLAPCU_CUDA(cudaMemsetAsync(fl, 0, sizeof(int) * 2, c.stream));
    any_zero_u8(c, (const uint8_t*)A.v + A.base, A.span, fl + 1);
    any_zero_u8(c, (const uint8_t*)B.v + B.base, B.span, fl + 1);
    if (d2h(c, fl + 1) != 0) return direct_fallback(c, A_, B_, sr, alg, capacity, c_colptr, crw, cv);
    const bool ones = true;
    SLAPCU_CUDA(cudaEventRecord(c.ev[0], c.stream));
    DirectCache& d = c.direct;
    FusedState& f = d.light;
    f.ones = true;
    prepare_plan(c, A, B);
    const int64_t* flops = c.plan.flops.as<int64_t>();
    const int64_t n = B.ncols;

    // ---- light columns: shared hash, staged (fused.cu kernels)
    BinSpec spec{};
    spec.nlight = 8;
    for (int b = 0; b < 8; ++b) spec.thr[b] = int64_t(32) << b;
    int64_t lmax = std::max<int64_t>(256, std::min<int64_t>(A.nrows / 128, 4096));
    if (c.opt.light_flops_max != Options{}.light_flops_max) lmax = std::min<int64_t>(c.opt.light_flops_max, 4096);
    spec.light_max = lmax;
    spec.all_heavy = alg == SLAPCU_ALG_HEAP;
    f.cnt.reset(sizeof(int64_t) * (n + 1), c.stream);
    SLAPCU_CUDA(cudaMemsetAsync(f.cnt.get(), 0, sizeof(int64_t) * (n + 1), c.stream));
    make_bins(c, n, flops, nullptr, spec, f.cnt.as<int64_t>(), f.bins);
    int nlight = 0;
    int64_t light_bound = 0;
    for (int b = 0; b < spec.nlight; ++b) {
        nlight += f.bins.count[b];
        light_bound += int64_t(f.bins.count[b]) * std::min<int64_t>(spec.thr[b], A.nrows);
    }
    f.srows.reset(sizeof(int32_t) * std::max<int64_t>(light_bound, 1), c.stream);
    f.soff.reset(sizeof(int64_t) * std::max<int64_t>(n, 1), c.stream);
    f.scur.reset(sizeof(unsigned long long), c.stream);
    SLAPCU_CUDA(cudaMemsetAsync(f.scur.get(), 0, sizeof(unsigned long long), c.stream));
    const int* L = f.bins.list.as<int>();
    for (int b = 0; b < spec.nlight; ++b) {
        const int nb = f.bins.count[b];
        if (!nb) continue;
        KScope ks(c, KC_SYM_LIGHT);
        fused_light_launch(c, sr, ones, b, A, B, L + f.bins.offset[b], nb, flops, f);
    }
    // light prefix per column (heavy columns count 0 here)
    d.lp.reset(sizeof(int64_t) * (n + 1), c.stream);
    {
        KScope ks(c, KC_SCAN);
        exclusive_scan_i64(c, f.cnt.as<int64_t>(), d.lp.as<int64_t>(), n + 1);
    }

    // ---- heavy columns in column order, cut into row-tile items
    const int nh = f.bins.count[spec.nlight];
    const int TL = direct_tile_log2(c, A.nrows);
    const int T = (int)((A.nrows + (int64_t(1) << TL) - 1) >> TL);
    const int W = 1 << (TL - 5);
    d.hcnt.reset(sizeof(unsigned long long) * std::max<int64_t>(n, 1), c.stream);
    SLAPCU_CUDA(cudaMemsetAsync(d.hcnt.get(), 0, sizeof(unsigned long long) * std::max<int64_t>(n, 1), c.stream));
    DevBuf misc(sizeof(int) * 4, c.stream);
    SLAPCU_CUDA(cudaMemsetAsync(misc.get(), 0, sizeof(int) * 4, c.stream));
    int* ticket = misc.as<int>();
    int* overflow = misc.as<int>() + 1;
    if (nh > 0) {
        const int32_t* Atp = tile_pointers(c, A, TL, T);
        KScope ks(c, KC_BIN);
        DevBuf hflag(sizeof(int) * (n + 1), c.stream), hpre(sizeof(int) * (n + 1), c.stream);
        launch(c, k_mark_heavy, dim3(grid_for(c, n, 256)), dim3(256), 0, n, flops, lmax, spec.all_heavy != 0,
               hflag.as<int>());
        excl_scan_i32(c, hflag.as<int>(), hpre.as<int>(), n);
        d.hl.reset(sizeof(int) * nh, c.stream);
        launch(c, k_scatter_heavy, dim3(grid_for(c, n, 256)), dim3(256), 0, n, (const int*)hflag.as<int>(),
               (const int*)hpre.as<int>(), d.hl.as<int>());
        DevBuf iflops(sizeof(int64_t) * int64_t(nh) * T, c.stream);
        DevBuf nit(sizeof(int64_t) * (nh + 1), c.stream), ioff(sizeof(int64_t) * (nh + 1), c.stream);
        SLAPCU_CUDA(cudaMemsetAsync(nit.as<int64_t>() + nh, 0, sizeof(int64_t), c.stream));
        launch(c, k_item_flops, dim3(grid_for(c, int64_t(nh) * 32, 256)), dim3(256), 0, A, B, Atp, T,
               (const int*)d.hl.as<int>(), nh, iflops.as<int64_t>(), nit.as<int64_t>());
        exclusive_scan_i64(c, nit.as<int64_t>(), ioff.as<int64_t>(), nh + 1);
        const int64_t nitems64 = d2h(c, ioff.as<int64_t>() + nh);
        if (nitems64 > INT32_MAX) throw Fail{SLAPCU_ERR_INVALID, "too many tile items"};
        const int nitems = (int)nitems64;
        d.items.reset(sizeof(int2) * std::max(nitems, 1), c.stream);
        DevBuf dflag(sizeof(int) * (nitems + 1), c.stream), dpre(sizeof(int) * (nitems + 1), c.stream);
        SLAPCU_CUDA(cudaMemsetAsync(dflag.as<int>() + nitems, 0, sizeof(int), c.stream));
        const int64_t dense_min = c.opt.direct_dense_flops_min > 0 ? c.opt.direct_dense_flops_min : INT64_MAX;
        launch(c, k_item_fill, dim3(grid_for(c, nh, 256)), dim3(256), 0, (const int*)d.hl.as<int>(), nh, T,
               (const int64_t*)iflops.as<int64_t>(), (const int64_t*)ioff.as<int64_t>(), dense_min,
               d.items.as<int2>(), dflag.as<int>());
        excl_scan_i32(c, dflag.as<int>(), dpre.as<int>(), nitems + 1);
        const int ndense = d2h(c, dpre.as<int>() + nitems);
        d.dslot.reset(sizeof(int) * std::max(nitems, 1), c.stream);
        d.dlist.reset(sizeof(int) * std::max(ndense, 1), c.stream);
        launch(c, k_dense_slots, dim3(grid_for(c, nitems, 256)), dim3(256), 0, nitems, (const int*)dflag.as<int>(),
               (const int*)dpre.as<int>(), d.dslot.as<int>(), d.dlist.as<int>());
        d.state.reset(sizeof(unsigned long long) * std::max(nitems, 1), c.stream);
        SLAPCU_CUDA(cudaMemsetAsync(d.state.get(), 0, sizeof(unsigned long long) * std::max(nitems, 1), c.stream));
        d.gbm.reset(sizeof(unsigned) * size_t(W) * std::max(ndense, 1), c.stream);
        KScope ks2(c, KC_SYM_HEAVY);
        if (ndense > 0) {
            const size_t smem = sizeof(unsigned) * W;
            auto go = [&](auto k) {
                ensure_smem(k, smem);
                launch(c, k, dim3(ndense), dim3(kDenseThreads), smem, A, B, Atp, T, TL, (const int2*)d.items.as<int2>(),
                       (const int*)d.dlist.as<int>(), d.gbm.as<unsigned>(), d.state.as<unsigned long long>());
            };
            go(k_tile_dense<kDenseThreads>);
        }
        DirectArgs g{A, B, Atp, T, TL, (const int2*)d.items.as<int2>(), (const int*)d.dslot.as<int>(), nitems,
                     (const unsigned*)d.gbm.as<unsigned>(), d.state.as<unsigned long long>(), ticket,
                     (const int64_t*)d.lp.as<int64_t>(), d.hcnt.as<unsigned long long>(), crw,
                     static_cast<uint8_t*>(cv), capacity, overflow};
        const size_t smem = sizeof(unsigned) * (W + W / 32) + sizeof(int) * (W / 32 + 1) + sizeof(uint16_t) * W + 16;
        auto go = [&](auto k) {
            ensure_smem(k, smem);
            int per_sm = 0;
            SLAPCU_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kDirectThreads, smem));
            const int grid = std::max(1, std::min(nitems, per_sm * c.num_sms));
            launch(c, k, dim3(grid), dim3(kDirectThreads), smem, g);
        };
        go(k_tile_direct<kDirectThreads>);
    }
    // ---- colptr = scan(light + heavy counts); light columns copied into place
    {
        KScope ks(c, KC_SCAN);
        DevBuf tot(sizeof(int64_t) * (n + 1), c.stream);
        SLAPCU_CUDA(cudaMemsetAsync(tot.as<int64_t>() + n, 0, sizeof(int64_t), c.stream));
        launch(c, k_add_counts, dim3(grid_for(c, n, 256)), dim3(256), 0, n, (const int64_t*)f.cnt.as<int64_t>(),
               (const unsigned long long*)d.hcnt.as<unsigned long long>(), tot.as<int64_t>());
        exclusive_scan_i64(c, tot.as<int64_t>(), c_colptr, n + 1);
    }
    const int64_t total = d2h(c, c_colptr + n);
    const int ovf = d2h(c, overflow);
    d.last_nnz = total;
    if (ovf || total > capacity)
        throw Fail{SLAPCU_ERR_BUDGET, "output needs " + std::to_string(total) + " entries, capacity " +
                                          std::to_string(capacity)};
    if (nlight) {
        KScope ks(c, KC_NUM_LIGHT);
        fused_copy_light(c, ones, L, nlight, f, c_colptr, crw, cv);
    }
    SLAPCU_CUDA(cudaEventRecord(c.ev[1], c.stream));
    SLAPCU_CUDA(cudaStreamSynchronize(c.stream));
    cudaEventElapsedTime(&c.sym_ms, c.ev[0], c.ev[1]);
    prof_flush(c);
    return total;
}

}  // namespace slapcu
