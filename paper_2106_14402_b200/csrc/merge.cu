// merge.cu -- multiway merge of q sorted partial results, C = P0 (+) P1 (+) ...
//
// The reference accumulates every SUMMA stage's partial C into one Triples
// list in stage order (summa.hpp:145-147), then build_dcsc stable-sorts it by
// (col,row) and left-folds coincident entries with sr.add
// (local_matrix.hpp:166-188).  The 3D driver does the same after its fiber
// exchange (spgemm3d.hpp:257-262).  Because every partial is already a
// canonical CSC, the GPU never sorts: per column, an entry of part s is the
// FIRST occurrence of its row iff no earlier part holds that row (binary
// search), its output slot is the number of distinct rows below it
// (per-part ranks of first occurrences), and its value is the left fold over
// parts s, s+1, ... in stage order -- the exact fold order of the stable sort,
// so the merge is bit-identical to the reference's for every semiring.
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "ctx.hpp"

namespace slapcu {

constexpr int kMaxParts = 16;

struct PartSet {
    int q;
    const int64_t* cp[kMaxParts];
    const int32_t* rw[kMaxParts];
    const void* v[kMaxParts];
    int32_t* firstrank[kMaxParts];  // per input entry: rank among the part's first occurrences in its column
};

__device__ __forceinline__ int64_t lower_bound_i32(const int32_t* __restrict__ a, int64_t lo, int64_t hi, int key) {
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (a[mid] < key)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}

// Pass 1 (symbolic): one warp per column.  Entries of part s are visited in
// row order 32 at a time; a ballot over "first occurrence" gives each entry its
// rank.  tot[s*ncols + j] = number of first occurrences of part s in column j.
__global__ void __launch_bounds__(256) k_merge_count(PartSet P, int64_t ncols, int32_t* __restrict__ tot,
                                                     int64_t* __restrict__ counts) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
    for (int64_t j = warp; j < ncols; j += nwarps) {
        int64_t total = 0;
        for (int s = 0; s < P.q; ++s) {
            const int64_t cs = P.cp[s][j], ce = P.cp[s][j + 1];
            int run = 0;
            for (int64_t b = cs; b < ce; b += 32) {
                const int64_t e = b + lane;
                bool first = false;
                if (e < ce) {
                    const int r = P.rw[s][e];
                    first = true;
                    for (int s2 = 0; s2 < s && first; ++s2) {
                        const int64_t lo = P.cp[s2][j], hi = P.cp[s2][j + 1];
                        const int64_t x = lower_bound_i32(P.rw[s2], lo, hi, r);
                        if (x < hi && P.rw[s2][x] == r) first = false;
                    }
                }
                const unsigned m = __ballot_sync(0xffffffffu, first);
                if (e < ce) P.firstrank[s][e] = run + __popc(m & ((1u << lane) - 1u));
                run += __popc(m);
            }
            if (lane == 0) tot[int64_t(s) * ncols + j] = run;
            total += run;
        }
        if (lane == 0) counts[j] = total;
    }
}

// Pass 2 (numeric): every first occurrence finds its slot and folds the
// values of the same row from the later parts in part order.
template <int SRID>
__global__ void __launch_bounds__(256) k_merge_write(PartSet P, int64_t ncols, const int32_t* __restrict__ tot,
                                                     const int64_t* __restrict__ Ccp, int32_t* __restrict__ Crw,
                                                     typename Sr<SRID>::T* __restrict__ Cv) {
    using S_ = Sr<SRID>;
    using T = typename S_::T;
    const int lane = threadIdx.x & 31;
    const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
    for (int64_t j = warp; j < ncols; j += nwarps) {
        const int64_t ob = Ccp[j];
        for (int s = 0; s < P.q; ++s) {
            const int64_t cs = P.cp[s][j], ce = P.cp[s][j + 1];
            const T* vs = static_cast<const T*>(P.v[s]);
            for (int64_t e = cs + lane; e < ce; e += 32) {
                const int r = P.rw[s][e];
                const int fr = P.firstrank[s][e];
                bool first = true;
                int64_t pos = fr;
                for (int s2 = 0; s2 < P.q; ++s2) {
                    if (s2 == s) continue;
                    const int64_t lo = P.cp[s2][j], hi = P.cp[s2][j + 1];
                    const int64_t x = lower_bound_i32(P.rw[s2], lo, hi, r);
                    if (s2 < s && x < hi && P.rw[s2][x] == r) {
                        first = false;
                        break;
                    }
                    pos += (x < hi) ? P.firstrank[s2][x] : tot[int64_t(s2) * ncols + j];
                }
                if (!first) continue;
                // left fold in part order (local_matrix.hpp:179-186)
                typename S_::Acc acc = (typename S_::Acc)0;
                if constexpr (SRID == SLAPCU_OR_AND_U8)
                    acc = vs[e] ? 1u : 0u;
                else
                    acc = (typename S_::Acc)vs[e];
                for (int s2 = s + 1; s2 < P.q; ++s2) {
                    const int64_t lo = P.cp[s2][j], hi = P.cp[s2][j + 1];
                    const int64_t x = lower_bound_i32(P.rw[s2], lo, hi, r);
                    if (x < hi && P.rw[s2][x] == r) {
                        const T* v2 = static_cast<const T*>(P.v[s2]);
                        typename S_::Acc o;
                        if constexpr (SRID == SLAPCU_OR_AND_U8)
                            o = v2[x] ? 1u : 0u;
                        else
                            o = (typename S_::Acc)v2[x];
                        acc = S_::add(acc, o);
                    }
                }
                Crw[ob + pos] = r;
                Cv[ob + pos] = S_::out(acc);
            }
        }
    }
}

namespace {

using MergeScratch = decltype(Ctx::merge);

MergeScratch& scratch_for(Ctx& c) { return c.merge; }

// Parts may be column windows (colptr not starting at 0): their entry range
// [base, base+span) is read from the device and the per-entry rank scratch is
// addressed with the same absolute indices.
PartSet make_parts(Ctx& c, int q, const DevCsc* parts_in, MergeScratch& ms, bool alloc) {
    if (q < 1 || q > kMaxParts) throw Fail{SLAPCU_ERR_INVALID, "merge supports 1..16 parts"};
    for (int s = 1; s < q; ++s)
        if (parts_in[s].nrows != parts_in[0].nrows || parts_in[s].ncols != parts_in[0].ncols)
            throw Fail{SLAPCU_ERR_DIM, "merge parts have different shapes"};
    DevCsc parts[kMaxParts];
    for (int s = 0; s < q; ++s) {
        parts[s] = parts_in[s];
        resolve(c, parts[s]);
    }
    PartSet P{};
    P.q = q;
    int64_t tot_nnz = 0;
    for (int s = 0; s < q; ++s) tot_nnz += parts[s].span;
    if (alloc) ms.ranks.reset(sizeof(int32_t) * std::max<int64_t>(tot_nnz, 1), c.stream);
    int64_t off = 0;
    for (int s = 0; s < q; ++s) {
        P.cp[s] = parts[s].cp;
        P.rw[s] = parts[s].rw;
        P.v[s] = parts[s].v;
        P.firstrank[s] = ms.ranks.as<int32_t>() + off - parts[s].base;
        off += parts[s].span;
    }
    return P;
}

}  // namespace

int64_t merge_symbolic(Ctx& c, int q, const DevCsc* parts, int64_t* c_colptr) {
    KScope ks(c, KC_MERGE);
    MergeScratch& ms = scratch_for(c);
    PartSet P = make_parts(c, q, parts, ms, true);
    const int64_t n = parts[0].ncols;
    ms.tot.reset(sizeof(int32_t) * std::max<int64_t>(n * q, 1), c.stream);
    ms.counts.reset(sizeof(int64_t) * (n + 1), c.stream);
    SLAPCU_CUDA(cudaMemsetAsync(ms.counts.as<int64_t>() + n, 0, sizeof(int64_t), c.stream));
    int64_t blocks = std::min<int64_t>(ceil_div(n * 32, 256), int64_t(c.num_sms) * 16);
    launch(c, k_merge_count, dim3((unsigned)std::max<int64_t>(blocks, 1)), dim3(256), 0, P, n, ms.tot.as<int32_t>(),
           ms.counts.as<int64_t>());
    exclusive_scan_i64(c, ms.counts.as<int64_t>(), c_colptr, n + 1);
    int64_t total = 0;
    SLAPCU_CUDA(cudaMemcpyAsync(&total, c_colptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost, c.stream));
    SLAPCU_CUDA(cudaStreamSynchronize(c.stream));
    ms.key0 = parts[0].cp;
    ms.q = q;
    ms.ncols = n;
    return total;
}

void merge_numeric(Ctx& c, int q, const DevCsc* parts, int sr, const int64_t* c_colptr, int32_t* c_rowids,
                   void* c_vals) {
    MergeScratch& ms = scratch_for(c);
    if (ms.key0 != parts[0].cp || ms.q != q || ms.ncols != parts[0].ncols) {
        // symbolic state missing: recompute it (colptr is recomputed into scratch)
        DevBuf tmp(sizeof(int64_t) * (parts[0].ncols + 1), c.stream);
        merge_symbolic(c, q, parts, tmp.as<int64_t>());
    }
    PartSet P = make_parts(c, q, parts, ms, false);
    KScope ks(c, KC_MERGE);
    const int64_t n = parts[0].ncols;
    int64_t blocks = std::min<int64_t>(ceil_div(n * 32, 256), int64_t(c.num_sms) * 16);
    dispatch_sr(sr, [&](auto id) {
        constexpr int ID = decltype(id)::value;
        launch(c, k_merge_write<ID>, dim3((unsigned)std::max<int64_t>(blocks, 1)), dim3(256), 0, P, n,
               (const int32_t*)ms.tot.as<int32_t>(), c_colptr, c_rowids, static_cast<typename Sr<ID>::T*>(c_vals));
    });
    SLAPCU_CUDA(cudaStreamSynchronize(c.stream));
    prof_flush(c);
}

}  // namespace slapcu
