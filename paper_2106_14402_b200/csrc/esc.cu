// esc.cu -- expand / sort / compress (ESC) product: the sort-merge path for
// low-compression columns and the deterministic (reference-order) fold.
//
// Per output column j every product A(i,k) * B(k,j) is written out in the
// reference's enumeration order (B(:,j) entries ascending in k, then A(:,k)
// ascending in i), the column's products are sorted by row with a STABLE
// segmented radix sort, and each run of equal rows is folded left to right
// with the semiring add.  That is exactly the reference's per-entry fold
// order (heap: ties by stream = ascending k, spgemm.hpp:156-159; hash:
// upserts in B-column order, spgemm.hpp:251-255), so floating-point
// PlusTimes comes out BIT-identical to slap::local_spgemm, not just within
// tolerance -- the atomics of the bitmap / hash paths fold in arrival order.
// The cost is ~(8 + 2 sizeof(value)) bytes per product moved a few times
// (expand, 3 radix passes over 20-22-bit row keys, fold), which is the cheaper
// side when the compression factor flops / nnz(C) is near 1 (configs C2, C5)
// and the price of determinism elsewhere.
#include <cub/cub.cuh>

#include <algorithm>
#include <string>
#include <vector>

#include "kern.cuh"

namespace slapcu {

namespace {

// Products of each B entry of columns [j0, j1): nnz(A(:,k)).
__global__ void k_entry_len(DevCsc A, DevCsc B, int64_t e0, int64_t ne, int64_t* __restrict__ len) {
    for (int64_t x = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; x < ne; x += int64_t(gridDim.x) * blockDim.x) {
        const int k = B.rw[e0 + x];
        len[x] = A.cp[k + 1] - A.cp[k];
    }
}

// Column (relative to the group) of each B entry of the group.
__global__ void k_entry_col(int64_t ncols, const int64_t* __restrict__ Bcp, int64_t e0, int* __restrict__ col) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
    for (int64_t j = w0; j < ncols; j += nw)
        for (int64_t x = Bcp[j] + lane; x < Bcp[j + 1]; x += 32) col[x - e0] = (int)j;
}

// Expand: a warp takes 32 B entries; their products are contiguous in the
// output (eoff is the prefix of the entries' A column lengths), so the warp
// walks that range with consecutive lanes on consecutive products -- reads of
// A and writes of keys / values coalesced -- finding each product's entry by a
// 5-step search over the lanes' prefix (shuffles).  The key is
// (column << row_bits) | row, so ONE stable radix sort over the group orders
// products by (column, row) and keeps the enumeration order (ascending k)
// inside every run.
template <int SRID, class K>
__global__ void k_expand(DevCsc A, DevCsc B, int64_t e0, int64_t ne, const int64_t* __restrict__ eoff,
                         const int* __restrict__ ecol, int row_bits, K* __restrict__ keys,
                         typename Sr<SRID>::Acc* __restrict__ vals) {
    using S_ = Sr<SRID>;
    using T = typename S_::T;
    const T* Av = static_cast<const T*>(A.v);
    const T* Bv = static_cast<const T*>(B.v);
    const int lane = threadIdx.x & 31;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t base = int64_t(blockIdx.x) * blockDim.x + (threadIdx.x & ~31); base < ne; base += stride) {
        const int64_t x = base + lane;
        int64_t s = 0;
        int len = 0;
        T b{};
        K hi = 0;
        if (x < ne) {
            const int k = B.rw[e0 + x];
            b = Bv[e0 + x];
            hi = K(ecol[x]) << row_bits;
            s = A.cp[k];
            len = (int)(A.cp[k + 1] - s);
        }
        const int64_t o0 = __shfl_sync(0xffffffffu, x < ne ? eoff[x] : 0, 0);  // the warp's first product
        int tot;
        const int ex = warp_excl_scan(len, lane, &tot);
        // kExpandU warp steps at a time: every lane has kExpandU independent
        // (row, value) gathers in flight (one step at a time left the kernel
        // latency-bound: long_scoreboard 86%, C5 expand 3.5 ms)
        constexpr int kExpandU = 4;
        for (int q0 = 0; q0 < tot; q0 += 32 * kExpandU) {
            int64_t pp[kExpandU];
            T bv[kExpandU];
            K hv[kExpandU];
#pragma unroll
            for (int u = 0; u < kExpandU; ++u) {
                const int q = q0 + 32 * u + lane;
                // owner: the last lane whose prefix is <= q (lanes with len 0 are skipped by <=)
                int src = 0;
#pragma unroll
                for (int step = 16; step > 0; step >>= 1) {
                    const int cand = src + step;
                    const int exc = __shfl_sync(0xffffffffu, ex, cand & 31);
                    if (cand < 32 && exc <= q) src = cand;
                }
                const int exs = __shfl_sync(0xffffffffu, ex, src);
                pp[u] = (int64_t)__shfl_sync(0xffffffffu, (long long)s, src) + (q - exs);
                hv[u] = __shfl_sync(0xffffffffu, hi, src);
                bv[u] = __shfl_sync(0xffffffffu, b, src);
            }
            int r[kExpandU];
            T a[kExpandU];
#pragma unroll
            for (int u = 0; u < kExpandU; ++u) {
                if (q0 + 32 * u + lane < tot) {
                    r[u] = __ldg(&A.rw[pp[u]]);
                    a[u] = Av[pp[u]];
                }
            }
#pragma unroll
            for (int u = 0; u < kExpandU; ++u) {
                const int q = q0 + 32 * u + lane;
                if (q < tot) {
                    keys[o0 + q] = hv[u] | K(r[u]);
                    vals[o0 + q] = S_::mul(a[u], bv[u]);
                }
            }
        }
    }
}

// Columns with at most kSmallSort products: one CTA sorts the column's
// products in shared memory by (row, enumeration index) -- a bitonic network
// on 64-bit keys, stable by construction -- and writes them permuted into the
// sorted arrays.  (One global radix sort over millions of short columns is
// 5 passes over every product; this is one.)
constexpr int kSmallSort = 2048;

template <class K, class V>
__global__ void __launch_bounds__(256) k_sort_small(const int* __restrict__ cols, const int* __restrict__ beg,
                                                    const int* __restrict__ end, K row_mask, const K* __restrict__ k0,
                                                    const V* __restrict__ v0, K* __restrict__ k1, V* __restrict__ v1) {
    __shared__ unsigned long long sk[kSmallSort];
    const int j = cols[blockIdx.x];
    const int b = beg[j], n = end[j] - b;
    int N = 1;
    while (N < n) N <<= 1;
    for (int q = threadIdx.x; q < N; q += blockDim.x)
        sk[q] = q < n ? ((unsigned long long)(k0[b + q] & row_mask) << 11) | (unsigned long long)q : ~0ull;
    __syncthreads();
    for (int size = 2; size <= N; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int q = threadIdx.x; q < (N >> 1); q += blockDim.x) {
                const int lo = 2 * q - (q & (stride - 1)), hi = lo + stride;
                const bool up = (lo & size) == 0;
                const unsigned long long x = sk[lo], y = sk[hi];
                if ((x > y) == up) {
                    sk[lo] = y;
                    sk[hi] = x;
                }
            }
            __syncthreads();
        }
    }
    for (int q = threadIdx.x; q < n; q += blockDim.x) {
        const int src = (int)(sk[q] & 2047ull);
        k1[b + q] = k0[b + src];
        v1[b + q] = v0[b + src];
    }
}

// Columns with at most kWarpSort products: one WARP each (8 per CTA), the
// same bitonic network in the warp's slice of shared memory, __syncwarp only.
constexpr int kWarpSort = 256;

// <= 32 * R products: the network in registers, element e = r * 32 + lane --
// partners across lanes by shuffles, across registers in-thread (no shared
// round trip per stage; C2's columns of 64-128 products).
template <int R, class K, class V>
__device__ __forceinline__ void warp_reg_sort(int n, int N, int lane, int b, K row_mask, const K* __restrict__ k0,
                                              const V* __restrict__ v0, K* __restrict__ k1, V* __restrict__ v1) {
    unsigned long long x[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int e = r * 32 + lane;
        x[r] = e < n ? ((unsigned long long)(k0[b + e] & row_mask) << 11) | (unsigned long long)e : ~0ull;
    }
    for (int size = 2; size <= N; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            if (stride >= 32) {  // partner register r ^ (stride / 32), same lane (constant indices:
                                 // a runtime register index would put x in local memory)
                auto cx = [&](unsigned long long& a, unsigned long long& c, int r) {
                    const bool asc = ((r * 32 + lane) & size) == 0;
                    const unsigned long long lo = a < c ? a : c, hi = a < c ? c : a;
                    a = asc ? lo : hi;
                    c = asc ? hi : lo;
                };
                if (stride == 32) {
                    cx(x[0], x[1], 0);
                    if constexpr (R == 4) cx(x[2], x[3], 2);
                } else if constexpr (R == 4) {  // stride 64
                    cx(x[0], x[2], 0);
                    cx(x[1], x[3], 1);
                }
                continue;
            }
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int e = r * 32 + lane;
                const unsigned long long y = __shfl_xor_sync(0xffffffffu, x[r], stride);
                const bool keep_min = ((e & stride) == 0) == ((e & size) == 0);
                x[r] = keep_min ? (x[r] < y ? x[r] : y) : (x[r] < y ? y : x[r]);
            }
        }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int q = r * 32 + lane;
        if (q < n) {
            const int src = (int)(x[r] & 2047ull);
            k1[b + q] = k0[b + src];
            v1[b + q] = v0[b + src];
        }
    }
}

template <class K, class V>
__global__ void __launch_bounds__(256) k_sort_warp(int ncols, const int* __restrict__ cols, const int* __restrict__ beg,
                                                   const int* __restrict__ end, K row_mask, const K* __restrict__ k0,
                                                   const V* __restrict__ v0, K* __restrict__ k1, V* __restrict__ v1) {
    __shared__ unsigned long long skw[8][kWarpSort];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int ci = blockIdx.x * 8 + w;
    if (ci >= ncols) return;
    unsigned long long* sk = skw[w];
    const int j = cols[ci];
    const int b = beg[j], n = end[j] - b;
    int N = 1;
    while (N < n) N <<= 1;
    if (N <= 64) {
        warp_reg_sort<2>(n, N, lane, b, row_mask, k0, v0, k1, v1);
        return;
    }
    // (65-128 products in 4 registers per lane measured slower than the shared
    // network: C2 sort 1.66 -> 1.79 ms)
    for (int q = lane; q < N; q += 32)
        sk[q] = q < n ? ((unsigned long long)(k0[b + q] & row_mask) << 11) | (unsigned long long)q : ~0ull;
    __syncwarp();
    for (int size = 2; size <= N; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int q = lane; q < (N >> 1); q += 32) {
                const int lo = 2 * q - (q & (stride - 1)), hi = lo + stride;
                const bool up = (lo & size) == 0;
                const unsigned long long x = sk[lo], y = sk[hi];
                if ((x > y) == up) {
                    sk[lo] = y;
                    sk[hi] = x;
                }
            }
            __syncwarp();
        }
    }
    for (int q = lane; q < n; q += 32) {
        const int src = (int)(sk[q] & 2047ull);
        k1[b + q] = k0[b + src];
        v1[b + q] = v0[b + src];
    }
}

// Columns of a group by product count: 2..kWarpSort -> tiny (one warp each),
// ..kSmallSort -> small (one CTA each), more -> a long column (flag[0]).
// (On the device: a host pass over millions of light columns cost more than
// the sorts, C2 ESC 9.8 ms.)
__global__ void k_esc_classify(int64_t ng, const int64_t* __restrict__ flops, int* __restrict__ tiny,
                               int* __restrict__ small, int* __restrict__ counts) {
    for (int64_t jj = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; jj < ng; jj += int64_t(gridDim.x) * blockDim.x) {
        const int64_t pj = flops[jj];
        if (pj > 1 && pj <= kWarpSort)
            tiny[atomicAdd(&counts[0], 1)] = (int)jj;
        else if (pj > kWarpSort && pj <= kSmallSort)
            small[atomicAdd(&counts[1], 1)] = (int)jj;
        else if (pj > kSmallSort)
            counts[2] = 1;
    }
}

// Segment (column) begin/end offsets of the group's products.
__global__ void k_seg_bounds(int64_t ncols, const int64_t* __restrict__ Bcp, int64_t e0, const int64_t* __restrict__ eoff,
                             int* __restrict__ beg, int* __restrict__ end) {
    for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < ncols; j += int64_t(gridDim.x) * blockDim.x) {
        beg[j] = (int)eoff[Bcp[j] - e0];
        end[j] = (int)eoff[Bcp[j + 1] - e0];
    }
}

// Run heads: a (column, row) key differing from its predecessor.
template <class K>
__global__ void k_run_heads(int64_t P, const K* __restrict__ keys, int* __restrict__ head) {
    for (int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; p <= P; p += int64_t(gridDim.x) * blockDim.x)
        head[p] = p < P && (p == 0 || keys[p] != keys[p - 1]);
}

// Fold each run left to right (the reference's order) and write (row, value).
template <int SRID, class K>
__global__ void k_fold(int64_t P, const K* __restrict__ keys, const typename Sr<SRID>::Acc* __restrict__ vals,
                       const int* __restrict__ head, const int* __restrict__ ex, int64_t obase, K row_mask,
                       int32_t* __restrict__ crw, typename Sr<SRID>::T* __restrict__ cv) {
    using S_ = Sr<SRID>;
    for (int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; p < P; p += int64_t(gridDim.x) * blockDim.x) {
        if (!head[p]) continue;
        typename S_::Acc acc = vals[p];
        for (int64_t q = p + 1; q < P && !head[q]; ++q) acc = S_::add(acc, vals[q]);
        const int64_t o = obase + ex[p];
        crw[o] = (int32_t)(keys[p] & row_mask);
        cv[o] = S_::out(acc);
    }
}

__global__ void k_esc_colptr(int64_t ncols, const int* __restrict__ beg, const int* __restrict__ ex, int64_t obase,
                             int64_t* __restrict__ cp) {
    for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < ncols; j += int64_t(gridDim.x) * blockDim.x)
        cp[j] = obase + ex[beg[j]];
}

template <class T>
T d2h1(Ctx& c, const T* p) {
    T v{};
    SLAPCU_CUDA(cudaMemcpyAsync(&v, p, sizeof(T), cudaMemcpyDeviceToHost, c.stream));
    SLAPCU_CUDA(cudaStreamSynchronize(c.stream));
    return v;
}

}  // namespace

// C = A * B by ESC into caller buffers (capacity entries); returns nnz(C).
// Columns are processed in groups of at most `group_max` products (int32
// sort offsets; bounded scratch).  BudgetError (exact nnz in c.direct.last_nnz)
// when C needs more than `capacity` entries -- nothing past capacity is written.
int64_t esc_spgemm(Ctx& c, const DevCsc& A_, const DevCsc& B_, int sr, int64_t capacity, int64_t* c_colptr,
                   int32_t* crw, void* cv) {
    check_operands(A_, B_);
    DevCsc A = A_, B = B_;
    resolve(c, A);
    resolve(c, B);
    const int64_t n = B.ncols;
    // per-column products, on the host for grouping
    DevBuf fl(sizeof(int64_t) * std::max<int64_t>(n, 1), c.stream);
    int64_t total = 0;
    spgemm_flops(c, A, B, fl.as<int64_t>(), &total);
    const size_t fr = device_available(c);
    const int64_t per_prod = 2 * 8 + 2 * 4 + 2 * 8;  // keys x2 (<= 8 bytes), head, ex, values x2 (<= 8 bytes)
    const int64_t group_max = std::max<int64_t>(1, std::min<int64_t>(int64_t(1) << 30, int64_t(fr / 3) / per_prod));
    // per-column counts and B's column pointers on the host only when the
    // product needs several groups (one group: the bounds are B's span)
    const bool one_group = total <= group_max;
    std::vector<int64_t> hf, hbcp;
    if (!one_group) {
        hf.resize(size_t(std::max<int64_t>(n, 1)));
        hbcp.resize(size_t(n) + 1);
        if (n) SLAPCU_CUDA(cudaMemcpyAsync(hf.data(), fl.get(), sizeof(int64_t) * n, cudaMemcpyDeviceToHost, c.stream));
        SLAPCU_CUDA(cudaMemcpyAsync(hbcp.data(), B.cp, sizeof(int64_t) * (n + 1), cudaMemcpyDeviceToHost, c.stream));
        SLAPCU_CUDA(cudaStreamSynchronize(c.stream));
    }
    int64_t obase = 0;
    int64_t j0 = 0;
    bool over = false;  // past capacity: keep counting for the exact requirement, write nothing
    dispatch_sr(sr, [&](auto idc) {
        constexpr int ID = decltype(idc)::value;
        using Acc = typename Sr<ID>::Acc;
        using T = typename Sr<ID>::T;
        while (j0 < n) {
            // the group: columns [j0, j1) with at most group_max products (a single larger column is an error)
            int64_t j1 = j0, P = 0;
            if (one_group) {
                j1 = n;
                P = total;
            } else {
                while (j1 < n && (j1 == j0 || P + hf[j1] <= group_max)) P += hf[j1++];
            }
            if (P > INT32_MAX)
                throw Fail{SLAPCU_ERR_BUDGET, "ESC: column " + std::to_string(j0) + " has " + std::to_string(P) +
                                                  " products (int32 sort offsets)"};
            const int64_t ng = j1 - j0;
            const int64_t e0 = one_group ? B.base : hbcp[j0], ne = one_group ? B.span : hbcp[j1] - e0;
            int row_bits = 1, col_bits = 1;
            while ((int64_t(1) << row_bits) < A.nrows) ++row_bits;
            while ((int64_t(1) << col_bits) < ng) ++col_bits;
            const bool narrow = row_bits + col_bits <= 32;
            int64_t gnnz = 0;
            auto run = [&](auto kz) {
                using K = decltype(kz);
                DevBuf len(sizeof(int64_t) * (ne + 1), c.stream), eoff(sizeof(int64_t) * (ne + 1), c.stream),
                    ecol(sizeof(int) * std::max<int64_t>(ne, 1), c.stream);
                SLAPCU_CUDA(cudaMemsetAsync(len.as<int64_t>() + ne, 0, sizeof(int64_t), c.stream));
                DevBuf k0(sizeof(K) * std::max<int64_t>(P, 1), c.stream), k1(sizeof(K) * std::max<int64_t>(P, 1), c.stream);
                DevBuf v0(sizeof(Acc) * std::max<int64_t>(P, 1), c.stream),
                    v1(sizeof(Acc) * std::max<int64_t>(P, 1), c.stream);
                DevBuf beg(sizeof(int) * std::max<int64_t>(ng, 1), c.stream), end(sizeof(int) * std::max<int64_t>(ng, 1), c.stream);
                DevBuf head(sizeof(int) * (P + 1), c.stream), ex(sizeof(int) * (P + 1), c.stream);
                {
                    KScope ks(c, KC_SYM_HEAVY);
                    if (ne) {
                        launch(c, k_entry_len, dim3(grid_for(c, ne, 256)), dim3(256), 0, A, B, e0, ne, len.as<int64_t>());
                        launch(c, k_entry_col, dim3(grid_for(c, ng * 32, 256)), dim3(256), 0, ng, (const int64_t*)(B.cp + j0),
                               e0, ecol.as<int>());
                    }
                    exclusive_scan_i64(c, len.as<int64_t>(), eoff.as<int64_t>(), ne + 1);
                    if (ne)
                        launch(c, k_expand<ID, K>, dim3(grid_for(c, ne, 256)), dim3(256), 0, A, B, e0, ne,
                               (const int64_t*)eoff.as<int64_t>(), (const int*)ecol.as<int>(), row_bits, k0.as<K>(),
                               v0.as<Acc>());
                    launch(c, k_seg_bounds, dim3(grid_for(c, ng, 256)), dim3(256), 0, ng, (const int64_t*)(B.cp + j0), e0,
                           (const int64_t*)eoff.as<int64_t>(), beg.as<int>(), end.as<int>());
                    if (P) {
                        // groups of short columns: one warp (<= 256 products) or CTA (<= 2048)
                        // per column, shared-memory sorts; a group holding any longer column:
                        // ONE stable LSD radix sort over the (column, row) keys of the group
                        // (cub's segmented sort runs a long segment on one CTA)
                        DevBuf lists(sizeof(int) * 2 * size_t(std::max<int64_t>(ng, 1)), c.stream),
                            lcnt(sizeof(int) * 3, c.stream);
                        SLAPCU_CUDA(cudaMemsetAsync(lcnt.get(), 0, sizeof(int) * 3, c.stream));
                        int* dtiny = lists.as<int>();
                        int* dsmall = dtiny + ng;
                        launch(c, k_esc_classify, dim3(grid_for(c, ng, 256)), dim3(256), 0, ng,
                               (const int64_t*)(fl.as<int64_t>() + j0), dtiny, dsmall, lcnt.as<int>());
                        int hc[3];
                        SLAPCU_CUDA(cudaMemcpyAsync(hc, lcnt.get(), sizeof(hc), cudaMemcpyDeviceToHost, c.stream));
                        SLAPCU_CUDA(cudaStreamSynchronize(c.stream));
                        int ntiny = hc[0], nsmall = hc[1];
                        const bool any_long = hc[2] != 0;
                        if (any_long) {
                            size_t tb = 0;
                            const int bits = row_bits + col_bits;
                            SLAPCU_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, k0.as<K>(), k1.as<K>(), v0.as<Acc>(),
                                                                        v1.as<Acc>(), (int)P, 0, bits, c.stream));
                            DevBuf tmp(tb, c.stream);
                            timed(c, KC_SYM_HEAVY, [&] {
                                SLAPCU_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), tb, k0.as<K>(), k1.as<K>(),
                                                                            v0.as<Acc>(), v1.as<Acc>(), (int)P, 0, bits,
                                                                            c.stream));
                            });
                            ++c.launches;
                            ntiny = nsmall = 0;
                        } else if (int64_t(ntiny) + nsmall < ng) {  // 0 / 1-product columns: as they are
                            SLAPCU_CUDA(cudaMemcpyAsync(k1.get(), k0.get(), sizeof(K) * P, cudaMemcpyDeviceToDevice, c.stream));
                            SLAPCU_CUDA(cudaMemcpyAsync(v1.get(), v0.get(), sizeof(Acc) * P, cudaMemcpyDeviceToDevice, c.stream));
                        }
                        if (ntiny) {
                            launch(c, k_sort_warp<K, Acc>, dim3((unsigned)((ntiny + 7) / 8)), dim3(256), 0,
                                   ntiny, (const int*)dtiny, (const int*)beg.as<int>(),
                                   (const int*)end.as<int>(), K((int64_t(1) << row_bits) - 1), (const K*)k0.as<K>(),
                                   (const Acc*)v0.as<Acc>(), k1.as<K>(), v1.as<Acc>());
                        }
                        if (nsmall) {
                            launch(c, k_sort_small<K, Acc>, dim3((unsigned)nsmall), dim3(256), 0, (const int*)dsmall,
                                   (const int*)beg.as<int>(), (const int*)end.as<int>(),
                                   K((int64_t(1) << row_bits) - 1), (const K*)k0.as<K>(), (const Acc*)v0.as<Acc>(),
                                   k1.as<K>(), v1.as<Acc>());
                        }
                    }
                    launch(c, k_run_heads<K>, dim3(grid_for(c, P + 1, 256)), dim3(256), 0, P, (const K*)k1.as<K>(),
                           head.as<int>());
                }
                {
                    KScope ks(c, KC_SCAN);
                    size_t tb = 0;
                    SLAPCU_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, head.as<int>(), ex.as<int>(), P + 1, c.stream));
                    DevBuf tmp(tb, c.stream);
                    timed(c, KC_SCAN, [&] {
                        SLAPCU_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(), tb, head.as<int>(), ex.as<int>(), P + 1,
                                                                  c.stream));
                    });
                    ++c.launches;
                }
                gnnz = d2h1(c, ex.as<int>() + P);
                launch(c, k_esc_colptr, dim3(grid_for(c, ng, 256)), dim3(256), 0, ng, (const int*)beg.as<int>(),
                       (const int*)ex.as<int>(), obase, c_colptr + j0);
                if (obase + gnnz > capacity) over = true;
                if (P && !over) {
                    KScope ks(c, KC_NUM_HEAVY);
                    launch(c, k_fold<ID, K>, dim3(grid_for(c, P, 256)), dim3(256), 0, P, (const K*)k1.as<K>(),
                           (const Acc*)v1.as<Acc>(), (const int*)head.as<int>(), (const int*)ex.as<int>(), obase,
                           K((int64_t(1) << row_bits) - 1), crw, static_cast<T*>(cv));
                }
            };
            if (narrow)
                run(uint32_t(0));
            else
                run(uint64_t(0));
            obase += gnnz;
            j0 = j1;
        }
    });
    SLAPCU_CUDA(cudaMemcpyAsync(c_colptr + n, &obase, sizeof(int64_t), cudaMemcpyHostToDevice, c.stream));
    SLAPCU_CUDA(cudaStreamSynchronize(c.stream));
    c.direct.last_nnz = obase;
    if (over)
        throw Fail{SLAPCU_ERR_BUDGET, "output needs " + std::to_string(obase) + " entries, capacity " +
                                          std::to_string(capacity)};
    return obase;
}

}  // namespace slapcu
