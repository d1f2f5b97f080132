// redist.cu -- device-side redistribution of a distributed sparse matrix
// (SURVEY.md 8f rank 2), over NCCL instead of the reference's simulated
// alltoallv:
//
//   distribute_triples   dist_matrix.hpp:89-119   COO -> 2D blocks, duplicates
//                                                 combined with `add`
//   redistribute_3d      dist_matrix3d.hpp:117-170 (regular variant)
//                                                 2D blocks -> c x q x q blocks
//   redistribute_2d      dist_matrix3d.hpp:250-261 3D blocks -> 2D blocks
//
// All three are one operation: every entry of this rank's input goes to the
// owner of the target tile holding its global (row, col).  A target layout is
// a tiling -- row cuts, column cuts and the owning rank of each tile -- that
// the host builds from the reference's geometry (grid.py tiling_2d /
// tiling_3d); each rank owns exactly one tile.
//
// Steps, all on this rank's stream:
//   route     one thread per entry: global coordinates (the column of a CSC
//             entry by binary search on colptr), tile by binary search on the
//             cuts held in shared memory, target-local (row, col), and a
//             shared-memory histogram of destinations;
//   partition stable radix sort of the destinations (keeps each rank's
//             entries in input order, as the reference's per-peer push order);
//   exchange  one all-gather of [counts, error flags, layout digest], then
//             grouped ncclSend/ncclRecv of rows, cols, values (NCCL has no
//             alltoallv); received parts land in source-rank order like
//             comm.alltoallv's concatenation (dist_matrix3d.hpp:170-174);
//   assemble  stable radix sort by (col, row) and one pass over the runs of
//             equal keys: keep-first or the semiring add folded left in
//             arrival order (local_matrix.hpp:167-188 sort_and_combine), then
//             colptr by binary search over the sorted columns.
// Out-of-range entries (IndexError, dist_matrix.hpp:101-106) and ranks that
// disagree on the layout are detected in the all-gather, so every rank fails
// the same way before any data moves.
#include <cub/cub.cuh>

#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cerrno>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "comm.hpp"
#include "kern.cuh"

namespace slapcu {
namespace {

constexpr int kMaxCuts = 1024;  // tiles per dimension (p <= 1024)
constexpr int kMaxRanks = 1024;

struct Tiling {
    int nr = 0, nc = 0;
    std::vector<int64_t> rc, cc;  // nr+1 / nc+1 cuts
    std::vector<int32_t> owner;   // nr*nc
};

__device__ __forceinline__ int tile_of(const int64_t* cuts, int n, int64_t x) {
    // last tile t with cuts[t] <= x (empty tiles share a cut and are skipped)
    int lo = 0, hi = n;  // cuts[lo] <= x < cuts[hi]
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (cuts[mid] <= x) lo = mid; else hi = mid;
    }
    return lo;
}

// Source: CSC block (block-local rows/cols + offsets) or global triples.
struct Src {
    int64_t n = 0;
    // CSC
    const int64_t* cp = nullptr;
    const int32_t* rw = nullptr;
    int64_t ncols = 0, base = 0, rs = 0, cs = 0;
    // triples
    const int64_t* grow = nullptr;
    const int64_t* gcol = nullptr;
};

template <bool CSC>
__global__ void k_route(Src s, int64_t m, int64_t n, int nr, int nc, int p, const int64_t* __restrict__ cuts,
                        const int32_t* __restrict__ owner, int32_t* __restrict__ dest, int32_t* __restrict__ lr,
                        int32_t* __restrict__ lc, unsigned long long* __restrict__ counts, int* __restrict__ bad) {
    extern __shared__ int64_t sm[];
    int64_t* rc = sm;
    int64_t* cc = sm + nr + 1;
    unsigned* hist = reinterpret_cast<unsigned*>(cc + nc + 1);
    for (int t = threadIdx.x; t <= nr; t += blockDim.x) rc[t] = cuts[t];
    for (int t = threadIdx.x; t <= nc; t += blockDim.x) cc[t] = cuts[nr + 1 + t];
    for (int t = threadIdx.x; t < p; t += blockDim.x) hist[t] = 0;
    __syncthreads();
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < s.n; e += int64_t(gridDim.x) * blockDim.x) {
        int64_t r, c;
        if constexpr (CSC) {
            const int64_t g = s.base + e;
            int64_t lo = 0, hi = s.ncols;  // cp[lo] <= g < cp[hi]
            while (hi - lo > 1) {
                const int64_t mid = (lo + hi) >> 1;
                if (s.cp[mid] <= g) lo = mid; else hi = mid;
            }
            r = s.rs + s.rw[g];
            c = s.cs + lo;
        } else {
            r = s.grow[e];
            c = s.gcol[e];
        }
        if (r < 0 || r >= m || c < 0 || c >= n) {
            atomicExch(bad, 1);
            dest[e] = 0;
            lr[e] = lc[e] = 0;
            continue;
        }
        const int ti = tile_of(rc, nr, r), tj = tile_of(cc, nc, c);
        const int d = owner[ti * nc + tj];
        dest[e] = d;
        lr[e] = int32_t(r - rc[ti]);
        lc[e] = int32_t(c - cc[tj]);
        atomicAdd(&hist[d], 1u);
    }
    __syncthreads();
    for (int t = threadIdx.x; t < p; t += blockDim.x)
        if (hist[t]) atomicAdd(&counts[t], (unsigned long long)hist[t]);
}

template <class W>
__global__ void k_pack(int64_t n, const int64_t* __restrict__ order, const int32_t* __restrict__ lr,
                       const int32_t* __restrict__ lc, const W* __restrict__ v, int64_t vbase, int32_t* __restrict__ srow,
                       int32_t* __restrict__ scol, W* __restrict__ sval) {
    for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < n; k += int64_t(gridDim.x) * blockDim.x) {
        const int64_t e = order[k];
        srow[k] = lr[e];
        scol[k] = lc[e];
        sval[k] = v[vbase + e];
    }
}

__global__ void k_iota(int64_t n, int64_t* __restrict__ out) {
    for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < n; k += int64_t(gridDim.x) * blockDim.x)
        out[k] = k;
}

__global__ void k_keys(int64_t n, const int32_t* __restrict__ r, const int32_t* __restrict__ c, int rbits,
                       uint64_t* __restrict__ key) {
    for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < n; k += int64_t(gridDim.x) * blockDim.x)
        key[k] = (uint64_t(uint32_t(c[k])) << rbits) | uint32_t(r[k]);
}

__global__ void k_heads(int64_t n, const uint64_t* __restrict__ key, int64_t* __restrict__ head) {
    for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < n; k += int64_t(gridDim.x) * blockDim.x)
        head[k] = (k == 0 || key[k] != key[k - 1]) ? 1 : 0;
}

// One thread per run of equal keys: keep-first, or the semiring add folded
// left in arrival order with the value rounded to T after every step (the
// reference's `vals.back() = add(vals.back(), v)` on VT).
template <int ID, bool ADD>
__global__ void k_combine(int64_t n, const uint64_t* __restrict__ key, const int64_t* __restrict__ order,
                          const int64_t* __restrict__ pos, const typename Sr<ID>::T* __restrict__ v, int rbits,
                          int32_t* __restrict__ orow, int32_t* __restrict__ ocol, typename Sr<ID>::T* __restrict__ ov) {
    using S = Sr<ID>;
    using T = typename S::T;
    using Acc = typename S::Acc;
    const uint64_t rmask = (uint64_t(1) << rbits) - 1;
    for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < n; k += int64_t(gridDim.x) * blockDim.x) {
        const uint64_t kk = key[k];
        if (k > 0 && key[k - 1] == kk) continue;
        T acc = v[order[k]];
        if constexpr (ADD) {
            for (int64_t j = k + 1; j < n && key[j] == kk; ++j) acc = S::out(S::add(Acc(acc), Acc(v[order[j]])));
        }
        const int64_t o = pos[k];
        orow[o] = int32_t(kk & rmask);
        ocol[o] = int32_t(kk >> rbits);
        ov[o] = acc;
    }
}

__global__ void k_colptr_from_cols(int64_t ncols, int64_t u, const int32_t* __restrict__ col, int64_t* __restrict__ cp) {
    for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j <= ncols; j += int64_t(gridDim.x) * blockDim.x) {
        int64_t lo = 0, hi = u;  // first index with col >= j
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (col[mid] < j) lo = mid + 1; else hi = mid;
        }
        cp[j] = lo;
    }
}

int bits_for(int64_t v) {  // bits to hold values in [0, v)
    int b = 0;
    while (b < 62 && (int64_t(1) << b) < v) ++b;
    return b;
}

uint64_t digest(const Tiling& t, int64_t m, int64_t n, int sr, int combine) {
    uint64_t h = mix64(uint64_t(m) * kGolden ^ uint64_t(n));
    auto add = [&](uint64_t x) { h = mix64(h ^ (x + kGolden)); };
    add(uint64_t(t.nr));
    add(uint64_t(t.nc));
    for (int64_t x : t.rc) add(uint64_t(x));
    for (int64_t x : t.cc) add(uint64_t(x));
    for (int32_t x : t.owner) add(uint64_t(uint32_t(x)));
    add(uint64_t(sr));
    add(uint64_t(combine));
    return h;
}

Tiling read_tiling(const slapcu_tiling* t, int p, int64_t m, int64_t n) {
    if (!t || !t->row_cuts || !t->col_cuts || !t->owner) throw Fail{SLAPCU_ERR_INVALID, "null target tiling"};
    if (t->nr < 1 || t->nc < 1 || t->nr > kMaxCuts || t->nc > kMaxCuts)
        throw Fail{SLAPCU_ERR_SHAPE, "target tiling needs 1..1024 tiles per dimension"};
    Tiling g;
    g.nr = t->nr;
    g.nc = t->nc;
    g.rc.assign(t->row_cuts, t->row_cuts + g.nr + 1);
    g.cc.assign(t->col_cuts, t->col_cuts + g.nc + 1);
    g.owner.assign(t->owner, t->owner + size_t(g.nr) * g.nc);
    if (g.rc.front() != 0 || g.rc.back() != m || g.cc.front() != 0 || g.cc.back() != n)
        throw Fail{SLAPCU_ERR_SHAPE, "target cuts must span [0, nrows) x [0, ncols)"};
    for (int i = 0; i < g.nr; ++i)
        if (g.rc[i + 1] < g.rc[i]) throw Fail{SLAPCU_ERR_SHAPE, "row cuts must be non-decreasing"};
    for (int j = 0; j < g.nc; ++j)
        if (g.cc[j + 1] < g.cc[j]) throw Fail{SLAPCU_ERR_SHAPE, "column cuts must be non-decreasing"};
    if (int64_t(g.nr) * g.nc != p) throw Fail{SLAPCU_ERR_SHAPE, "target tiling must have one tile per rank"};
    std::vector<int> seen(p, 0);
    for (int32_t o : g.owner) {
        if (o < 0 || o >= p || seen[o]) throw Fail{SLAPCU_ERR_SHAPE, "tile owners must be a permutation of the ranks"};
        seen[o] = 1;
    }
    return g;
}

template <class W>
void pack(Ctx& c, int64_t n, const int64_t* order, const int32_t* lr, const int32_t* lc, const void* v, int64_t vbase,
          int32_t* sr_, int32_t* sc, void* sv) {
    launch(c, k_pack<W>, dim3(grid_for(c, n, 256)), dim3(256), 0, n, order, lr, lc, static_cast<const W*>(v), vbase,
           sr_, sc, static_cast<W*>(sv));
}

void redistribute(slapcu_comm_s* cm, Ctx& c, const Src& src, const void* vals, int64_t vbase, bool csc, int64_t m,
                  int64_t n, int sr, const slapcu_tiling* target, int combine, slapcu_csc_out* out, int64_t* ors,
                  int64_t* ocs) {
    const int vs = value_size(sr);
    if (vs == 0) throw Fail{SLAPCU_ERR_INVALID, "unknown semiring"};
    if (combine != 0 && combine != 1) throw Fail{SLAPCU_ERR_INVALID, "combine: 0 keep-first, 1 semiring add"};
    if (m < 0 || n < 0) throw Fail{SLAPCU_ERR_SHAPE, "negative global dimensions"};
    const int p = cm->nranks, me = cm->rank;
    if (p > kMaxRanks) throw Fail{SLAPCU_ERR_SHAPE, "redistribution supports up to 1024 ranks"};
    const Tiling g = read_tiling(target, p, m, n);
    int mt = 0;
    while (g.owner[mt] != me) ++mt;
    const int ti = mt / g.nc, tj = mt % g.nc;
    const int64_t tr = g.rc[ti + 1] - g.rc[ti], tc = g.cc[tj + 1] - g.cc[tj];
    if (tr > INT32_MAX || tc > INT32_MAX) throw Fail{SLAPCU_ERR_SHAPE, "target tile exceeds int32 local indices"};
    const int64_t ne = src.n;
    if (ne > 0 && !vals) throw Fail{SLAPCU_ERR_INVALID, "null values"};

    // phase trace (SLAPCU_REDIST_TRACE=1): host wall time per phase, stream-synchronised
    static const bool trace = std::getenv("SLAPCU_REDIST_TRACE") != nullptr;
    auto t_last = std::chrono::steady_clock::now();
    auto mark = [&](const char* what) {
        if (!trace) return;
        cudaStreamSynchronize(c.stream);
        const auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[redist r%d] %-10s %8.3f ms\n", me, what,
                     std::chrono::duration<double, std::milli>(now - t_last).count());
        t_last = now;
    };
    mark("setup");
    // ---- route
    DevBuf cuts(sizeof(int64_t) * (g.nr + g.nc + 2), c.stream), own(sizeof(int32_t) * g.owner.size(), c.stream);
    std::vector<int64_t> hc(g.rc);
    hc.insert(hc.end(), g.cc.begin(), g.cc.end());
    SLAPCU_CUDA(cudaMemcpyAsync(cuts.get(), hc.data(), sizeof(int64_t) * hc.size(), cudaMemcpyHostToDevice, c.stream));
    SLAPCU_CUDA(cudaMemcpyAsync(own.get(), g.owner.data(), sizeof(int32_t) * g.owner.size(), cudaMemcpyHostToDevice,
                                c.stream));
    const int64_t ne1 = std::max<int64_t>(ne, 1);
    DevBuf dest(sizeof(int32_t) * ne1, c.stream), lr(sizeof(int32_t) * ne1, c.stream), lc(sizeof(int32_t) * ne1, c.stream);
    // [0,p) counts, p: bad flag, p+1: layout digest -- all-gathered as one row
    const int W = p + 2;
    DevBuf meta(sizeof(int64_t) * W * (p + 1), c.stream);
    int64_t* mine = meta.as<int64_t>() + int64_t(W) * p;
    SLAPCU_CUDA(cudaMemsetAsync(mine, 0, sizeof(int64_t) * W, c.stream));
    if (ne > 0) {
        const size_t smem = sizeof(int64_t) * (g.nr + g.nc + 2) + sizeof(unsigned) * p;
        auto k = csc ? k_route<true> : k_route<false>;
        ensure_smem(k, smem);
        launch(c, k, dim3(grid_for(c, ne, 256)), dim3(256), smem, src, m, n, g.nr, g.nc, p,
               (const int64_t*)cuts.as<int64_t>(), (const int32_t*)own.as<int32_t>(), dest.as<int32_t>(),
               lr.as<int32_t>(), lc.as<int32_t>(), reinterpret_cast<unsigned long long*>(mine),
               reinterpret_cast<int*>(mine + p));
    }
    const uint64_t dg = digest(g, m, n, sr, combine);
    SLAPCU_CUDA(cudaMemcpyAsync(mine + p + 1, &dg, sizeof(uint64_t), cudaMemcpyHostToDevice, c.stream));
    mark("route");
    // ---- partition by destination (stable)
    DevBuf order(sizeof(int64_t) * ne1, c.stream);
    const int dbits = std::max(1, bits_for(p));
    if (ne > 0) {
        DevBuf ord0(sizeof(int64_t) * ne1, c.stream), dsort(sizeof(int32_t) * ne1, c.stream);
        launch(c, k_iota, dim3(grid_for(c, ne, 256)), dim3(256), 0, ne, ord0.as<int64_t>());
        size_t tb = 0;
        SLAPCU_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, dest.as<int32_t>(), dsort.as<int32_t>(),
                                                    ord0.as<int64_t>(), order.as<int64_t>(), ne, 0, dbits, c.stream));
        DevBuf tmp(tb, c.stream);
        SLAPCU_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), tb, dest.as<int32_t>(), dsort.as<int32_t>(),
                                                    ord0.as<int64_t>(), order.as<int64_t>(), ne, 0, dbits, c.stream));
    }
    DevBuf srow(sizeof(int32_t) * ne1, c.stream), scol(sizeof(int32_t) * ne1, c.stream), sval(size_t(vs) * ne1, c.stream);
    if (ne > 0) {
        switch (vs) {
        case 1: pack<uint8_t>(c, ne, order.as<int64_t>(), lr.as<int32_t>(), lc.as<int32_t>(), vals, vbase,
                              srow.as<int32_t>(), scol.as<int32_t>(), sval.get()); break;
        case 4: pack<uint32_t>(c, ne, order.as<int64_t>(), lr.as<int32_t>(), lc.as<int32_t>(), vals, vbase,
                               srow.as<int32_t>(), scol.as<int32_t>(), sval.get()); break;
        default: pack<uint64_t>(c, ne, order.as<int64_t>(), lr.as<int32_t>(), lc.as<int32_t>(), vals, vbase,
                                srow.as<int32_t>(), scol.as<int32_t>(), sval.get()); break;
        }
    }
    mark("partition");
    // ---- exchange: counts / flags / digest, then the entries
    SLAPCU_NCCL(ncclAllGather(mine, meta.get(), W, ncclInt64, cm->world, c.stream));
    std::vector<int64_t> all(size_t(W) * p);
    SLAPCU_CUDA(cudaMemcpyAsync(all.data(), meta.get(), sizeof(int64_t) * W * p, cudaMemcpyDeviceToHost, c.stream));
    SLAPCU_CUDA(cudaStreamSynchronize(c.stream));
    cm->calls[kAllgatherv] += 1;
    cm->bytes[kAllgatherv] += sizeof(int64_t) * W;
    for (int r = 0; r < p; ++r)
        if (uint64_t(all[size_t(W) * r + p + 1]) != dg)
            throw Fail{SLAPCU_ERR_SHAPE, "ranks disagree on the target layout of the redistribution"};
    for (int r = 0; r < p; ++r)
        if (all[size_t(W) * r + p])
            throw Fail{SLAPCU_ERR_INDEX, "entry outside " + std::to_string(m) + "x" + std::to_string(n) +
                                             " on rank " + std::to_string(r)};
    std::vector<int64_t> soff(p + 1, 0), roff(p + 1, 0);
    for (int r = 0; r < p; ++r) {
        soff[r + 1] = soff[r] + all[size_t(W) * me + r];
        roff[r + 1] = roff[r] + all[size_t(W) * r + me];
    }
    const int64_t R = roff[p];
    const int64_t R1 = std::max<int64_t>(R, 1);
    DevBuf rrow(sizeof(int32_t) * R1, c.stream), rcol(sizeof(int32_t) * R1, c.stream), rval(size_t(vs) * R1, c.stream);
    // own part: a device copy, no NCCL
    const int64_t own_n = soff[me + 1] - soff[me];
    if (own_n) {
        SLAPCU_CUDA(cudaMemcpyAsync(rrow.as<int32_t>() + roff[me], srow.as<int32_t>() + soff[me], sizeof(int32_t) * own_n,
                                    cudaMemcpyDeviceToDevice, c.stream));
        SLAPCU_CUDA(cudaMemcpyAsync(rcol.as<int32_t>() + roff[me], scol.as<int32_t>() + soff[me], sizeof(int32_t) * own_n,
                                    cudaMemcpyDeviceToDevice, c.stream));
        SLAPCU_CUDA(cudaMemcpyAsync(rval.as<char>() + size_t(vs) * roff[me], sval.as<char>() + size_t(vs) * soff[me],
                                    size_t(vs) * own_n, cudaMemcpyDeviceToDevice, c.stream));
    }
    int64_t sent = 0;
    SLAPCU_NCCL(ncclGroupStart());
    for (int r = 0; r < p; ++r) {
        if (r == me) continue;
        const int64_t sn = soff[r + 1] - soff[r], rn = roff[r + 1] - roff[r];
        if (sn) {
            SLAPCU_NCCL(ncclSend(srow.as<int32_t>() + soff[r], size_t(sn), ncclInt32, r, cm->world, c.stream));
            SLAPCU_NCCL(ncclSend(scol.as<int32_t>() + soff[r], size_t(sn), ncclInt32, r, cm->world, c.stream));
            SLAPCU_NCCL(ncclSend(sval.as<char>() + size_t(vs) * soff[r], size_t(sn) * vs, ncclUint8, r, cm->world,
                                 c.stream));
            sent += (8 + vs) * sn;
        }
        if (rn) {
            SLAPCU_NCCL(ncclRecv(rrow.as<int32_t>() + roff[r], size_t(rn), ncclInt32, r, cm->world, c.stream));
            SLAPCU_NCCL(ncclRecv(rcol.as<int32_t>() + roff[r], size_t(rn), ncclInt32, r, cm->world, c.stream));
            SLAPCU_NCCL(ncclRecv(rval.as<char>() + size_t(vs) * roff[r], size_t(rn) * vs, ncclUint8, r, cm->world,
                                 c.stream));
        }
    }
    SLAPCU_NCCL(ncclGroupEnd());
    cm->calls[kAlltoallv] += 1;
    cm->bytes[kAlltoallv] += sent;
    // send-side scratch is dead once the group completes on the stream
    dest.release();
    lr.release();
    lc.release();
    order.release();

    mark("exchange");
    // ---- assemble the local tile
    out->nrows = tr;
    out->ncols = tc;
    *ors = g.rc[ti];
    *ocs = g.cc[tj];
    const int rbits = bits_for(tr), cbits = bits_for(tc);
    SLAPCU_CUDA(cudaMallocAsync((void**)&out->colptr, sizeof(int64_t) * (tc + 1), c.stream));
    if (R == 0) {
        out->nnz = 0;
        SLAPCU_CUDA(cudaMemsetAsync(out->colptr, 0, sizeof(int64_t) * (tc + 1), c.stream));
        SLAPCU_CUDA(cudaMallocAsync((void**)&out->rowids, sizeof(int32_t), c.stream));
        SLAPCU_CUDA(cudaMallocAsync(&out->vals, size_t(vs), c.stream));
        SLAPCU_CUDA(cudaStreamSynchronize(c.stream));
        return;
    }
    DevBuf key(sizeof(uint64_t) * R, c.stream), keys(sizeof(uint64_t) * R, c.stream);
    DevBuf ord0(sizeof(int64_t) * R, c.stream), ord(sizeof(int64_t) * R, c.stream);
    launch(c, k_keys, dim3(grid_for(c, R, 256)), dim3(256), 0, R, (const int32_t*)rrow.as<int32_t>(),
           (const int32_t*)rcol.as<int32_t>(), rbits, key.as<uint64_t>());
    launch(c, k_iota, dim3(grid_for(c, R, 256)), dim3(256), 0, R, ord0.as<int64_t>());
    {
        const int end_bit = std::max(1, rbits + cbits);
        size_t tb = 0;
        SLAPCU_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, key.as<uint64_t>(), keys.as<uint64_t>(),
                                                    ord0.as<int64_t>(), ord.as<int64_t>(), R, 0, end_bit, c.stream));
        DevBuf tmp(tb, c.stream);
        SLAPCU_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), tb, key.as<uint64_t>(), keys.as<uint64_t>(),
                                                    ord0.as<int64_t>(), ord.as<int64_t>(), R, 0, end_bit, c.stream));
    }
    DevBuf head(sizeof(int64_t) * (R + 1), c.stream), pos(sizeof(int64_t) * (R + 1), c.stream);
    launch(c, k_heads, dim3(grid_for(c, R, 256)), dim3(256), 0, R, (const uint64_t*)keys.as<uint64_t>(),
           head.as<int64_t>());
    SLAPCU_CUDA(cudaMemsetAsync(head.as<int64_t>() + R, 0, sizeof(int64_t), c.stream));
    exclusive_scan_i64(c, head.as<int64_t>(), pos.as<int64_t>(), R + 1);
    int64_t U = 0;
    SLAPCU_CUDA(cudaMemcpyAsync(&U, pos.as<int64_t>() + R, sizeof(int64_t), cudaMemcpyDeviceToHost, c.stream));
    SLAPCU_CUDA(cudaStreamSynchronize(c.stream));
    out->nnz = U;
    DevBuf ucol(sizeof(int32_t) * U, c.stream);
    SLAPCU_CUDA(cudaMallocAsync((void**)&out->rowids, sizeof(int32_t) * U, c.stream));
    SLAPCU_CUDA(cudaMallocAsync(&out->vals, size_t(vs) * U, c.stream));
    dispatch_sr(sr, [&](auto id) {
        constexpr int ID = decltype(id)::value;
        using T = typename Sr<ID>::T;
        auto k = combine ? k_combine<ID, true> : k_combine<ID, false>;
        launch(c, k, dim3(grid_for(c, R, 256)), dim3(256), 0, R, (const uint64_t*)keys.as<uint64_t>(),
               (const int64_t*)ord.as<int64_t>(), (const int64_t*)pos.as<int64_t>(), (const T*)rval.get(), rbits,
               out->rowids, ucol.as<int32_t>(), static_cast<T*>(out->vals));
    });
    launch(c, k_colptr_from_cols, dim3(grid_for(c, tc + 1, 256)), dim3(256), 0, tc, U,
           (const int32_t*)ucol.as<int32_t>(), out->colptr);
    SLAPCU_CUDA(cudaStreamSynchronize(c.stream));
    mark("assemble");
}

// ------------------------------------------------------------ CB2B binary I/O
// binary_io.hpp:10-28 / binary_io.cpp.  Records are (int64 row, int64 col,
// f64 value); they are built / taken apart on the device and streamed
// through two pinned staging buffers so the file I/O of chunk k overlaps the
// copy of chunk k-1.

constexpr int64_t kHeaderBytes = 32;
constexpr int64_t kRecBytes = 24;
constexpr int64_t kChunkRecs = int64_t(1) << 21;  // 48 MB per staging buffer
const char kMagic[4] = {'C', 'B', '2', 'B'};
constexpr uint32_t kVersion = 1;

struct Fd {
    int fd = -1;
    ~Fd() {
        if (fd >= 0) ::close(fd);
    }
};

struct Pinned {
    void* p = nullptr;
    explicit Pinned(size_t bytes) { SLAPCU_CUDA(cudaHostAlloc(&p, bytes, cudaHostAllocDefault)); }
    ~Pinned() {
        if (p) cudaFreeHost(p);
    }
};

struct Header {
    int64_t m = 0, n = 0, nnz = 0;
};

Header read_header(const char* path) {
    if (!path) throw Fail{SLAPCU_ERR_INVALID, "null path"};
    Fd f;
    f.fd = ::open(path, O_RDONLY);
    if (f.fd < 0) throw Fail{SLAPCU_ERR_IO, std::string("cannot open '") + path + "': " + std::strerror(errno)};
    struct stat st {};
    if (::fstat(f.fd, &st) != 0) throw Fail{SLAPCU_ERR_IO, std::string("cannot stat '") + path + "'"};
    const int64_t size = st.st_size;
    if (size < kHeaderBytes) throw Fail{SLAPCU_ERR_FORMAT, "file too short for a binary matrix header"};
    unsigned char hb[kHeaderBytes];
    if (::pread(f.fd, hb, kHeaderBytes, 0) != kHeaderBytes) throw Fail{SLAPCU_ERR_IO, "header read failed"};
    if (std::memcmp(hb, kMagic, 4) != 0) throw Fail{SLAPCU_ERR_FORMAT, std::string("bad magic in '") + path + "'"};
    uint32_t ver = 0;
    std::memcpy(&ver, hb + 4, 4);
    if (ver != kVersion) throw Fail{SLAPCU_ERR_FORMAT, "unsupported binary version " + std::to_string(ver)};
    Header h;
    std::memcpy(&h.m, hb + 8, 8);
    std::memcpy(&h.n, hb + 16, 8);
    std::memcpy(&h.nnz, hb + 24, 8);
    if (h.m < 0 || h.n < 0 || h.nnz < 0) throw Fail{SLAPCU_ERR_FORMAT, "negative header field"};
    if (h.nnz > (INT64_MAX - kHeaderBytes) / kRecBytes || size != kHeaderBytes + h.nnz * kRecBytes)
        throw Fail{SLAPCU_ERR_FORMAT, "file size " + std::to_string(size) + " does not match " +
                                          std::to_string(h.nnz) + " declared records"};
    return h;
}

void pread_all(int fd, void* dst, int64_t bytes, int64_t off) {
    char* d = static_cast<char*>(dst);
    while (bytes > 0) {
        const ssize_t r = ::pread(fd, d, size_t(std::min<int64_t>(bytes, int64_t(1) << 30)), off);
        if (r <= 0) throw Fail{SLAPCU_ERR_FORMAT, "truncated record section"};
        d += r;
        off += r;
        bytes -= r;
    }
}

void pwrite_all(int fd, const void* src, int64_t bytes, int64_t off) {
    const char* s_ = static_cast<const char*>(src);
    while (bytes > 0) {
        const ssize_t r = ::pwrite(fd, s_, size_t(std::min<int64_t>(bytes, int64_t(1) << 30)), off);
        if (r <= 0) throw Fail{SLAPCU_ERR_IO, std::string("write failed: ") + std::strerror(errno)};
        s_ += r;
        off += r;
        bytes -= r;
    }
}

__global__ void k_split_records(int64_t n, const int64_t* __restrict__ rec, int64_t* __restrict__ rows,
                                int64_t* __restrict__ cols, int64_t* __restrict__ vals) {
    for (int64_t w = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; w < 3 * n; w += int64_t(gridDim.x) * blockDim.x) {
        const int64_t x = rec[w];
        const int64_t e = w / 3;
        switch (w - 3 * e) {
        case 0: rows[e] = x; break;
        case 1: cols[e] = x; break;
        default: vals[e] = x; break;
        }
    }
}

__global__ void k_make_records(int64_t n, const int64_t* __restrict__ cp, const int32_t* __restrict__ rw,
                               const int64_t* __restrict__ v, int64_t ncols, int64_t base, int64_t rs, int64_t cs,
                               int64_t* __restrict__ rec) {
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n; e += int64_t(gridDim.x) * blockDim.x) {
        const int64_t g = base + e;
        int64_t lo = 0, hi = ncols;  // cp[lo] <= g < cp[hi]
        while (hi - lo > 1) {
            const int64_t mid = (lo + hi) >> 1;
            if (cp[mid] <= g) lo = mid; else hi = mid;
        }
        rec[3 * e] = rs + rw[g];
        rec[3 * e + 1] = cs + lo;
        rec[3 * e + 2] = v[g];
    }
}

// All-gather of a few int64 per rank over the world communicator (also the
// collective's synchronisation point).
std::vector<int64_t> allgather_small(slapcu_comm_s* cm, Ctx& c, const std::vector<int64_t>& mine) {
    const int p = cm->nranks, w = int(mine.size());
    DevBuf d(sizeof(int64_t) * w * (p + 1), c.stream);
    SLAPCU_CUDA(cudaMemcpyAsync(d.as<int64_t>() + int64_t(w) * p, mine.data(), sizeof(int64_t) * w,
                                cudaMemcpyHostToDevice, c.stream));
    SLAPCU_NCCL(ncclAllGather(d.as<int64_t>() + int64_t(w) * p, d.get(), w, ncclInt64, cm->world, c.stream));
    std::vector<int64_t> all(size_t(w) * p);
    SLAPCU_CUDA(cudaMemcpyAsync(all.data(), d.get(), sizeof(int64_t) * w * p, cudaMemcpyDeviceToHost, c.stream));
    SLAPCU_CUDA(cudaStreamSynchronize(c.stream));
    return all;
}

struct OutGuard {  // frees a half-built output on failure
    Ctx& c;
    slapcu_csc_out* o;
    bool ok = false;
    ~OutGuard() {
        if (ok || !o) return;
        if (o->colptr) cudaFreeAsync(o->colptr, c.stream);
        if (o->rowids) cudaFreeAsync(o->rowids, c.stream);
        if (o->vals) cudaFreeAsync(o->vals, c.stream);
        *o = slapcu_csc_out{};
    }
};

}  // namespace
}  // namespace slapcu

using namespace slapcu;

extern "C" {

slapcu_status slapcu_redistribute(slapcu_comm cm, const slapcu_csc* local, int64_t row_start, int64_t col_start,
                                  int64_t nrows, int64_t ncols, slapcu_semiring sr, const slapcu_tiling* target,
                                  int combine, slapcu_csc_out* out, int64_t* out_row_start, int64_t* out_col_start) {
    if (!cm || !local || !out || !out_row_start || !out_col_start) return SLAPCU_ERR_INVALID;
    Ctx& c = ctx_of(cm->ctx);
    *out = slapcu_csc_out{};
    OutGuard guard{c, out};
    try {
        SLAPCU_CUDA(cudaSetDevice(c.device));
        DevCsc A = view(*local);
        resolve(c, A);
        Src s;
        s.n = A.span;
        s.cp = A.cp;
        s.rw = A.rw;
        s.ncols = A.ncols;
        s.base = A.base;
        s.rs = row_start;
        s.cs = col_start;
        redistribute(cm, c, s, A.v, A.base, true, nrows, ncols, sr, target, combine, out, out_row_start, out_col_start);
        guard.ok = true;
        return SLAPCU_OK;
    } catch (const Fail& e) {
        c.last_error = e.msg;
        return e.st;
    }
}

slapcu_status slapcu_distribute_triples(slapcu_comm cm, int64_t count, const int64_t* rows, const int64_t* cols,
                                        const void* vals, int64_t nrows, int64_t ncols, slapcu_semiring sr,
                                        const slapcu_tiling* target, int combine, slapcu_csc_out* out,
                                        int64_t* out_row_start, int64_t* out_col_start) {
    if (!cm || !out || !out_row_start || !out_col_start || count < 0) return SLAPCU_ERR_INVALID;
    if (count > 0 && (!rows || !cols)) return SLAPCU_ERR_INVALID;
    Ctx& c = ctx_of(cm->ctx);
    *out = slapcu_csc_out{};
    OutGuard guard{c, out};
    try {
        SLAPCU_CUDA(cudaSetDevice(c.device));
        Src s;
        s.n = count;
        s.grow = rows;
        s.gcol = cols;
        redistribute(cm, c, s, vals, 0, false, nrows, ncols, sr, target, combine, out, out_row_start, out_col_start);
        guard.ok = true;
        return SLAPCU_OK;
    } catch (const Fail& e) {
        c.last_error = e.msg;
        return e.st;
    }
}

}  // extern "C"

extern "C" {

slapcu_status slapcu_cb2b_header(const char* path, int64_t* nrows, int64_t* ncols, int64_t* nnz) {
    try {
        const Header h = read_header(path);
        if (nrows) *nrows = h.m;
        if (ncols) *ncols = h.n;
        if (nnz) *nnz = h.nnz;
        return SLAPCU_OK;
    } catch (const Fail& e) {
        return e.st;
    }
}

slapcu_status slapcu_write_cb2b(slapcu_comm cm, const char* path, const slapcu_csc* local, int64_t row_start,
                                int64_t col_start, int64_t nrows, int64_t ncols) {
    if (!cm || !local || !path) return SLAPCU_ERR_INVALID;
    Ctx& c = ctx_of(cm->ctx);
    try {
        SLAPCU_CUDA(cudaSetDevice(c.device));
        DevCsc A = view(*local);
        resolve(c, A);
        const int p = cm->nranks, me = cm->rank;
        const int64_t ne = A.span;
        if (ne > 0 && !A.v) throw Fail{SLAPCU_ERR_INVALID, "null values"};
        // records of my block on the device
        DevBuf rec(size_t(kRecBytes) * std::max<int64_t>(ne, 1), c.stream);
        if (ne > 0)
            launch(c, k_make_records, dim3(grid_for(c, ne, 256)), dim3(256), 0, ne, A.cp, A.rw,
                   static_cast<const int64_t*>(A.v), A.ncols, A.base, row_start, col_start, rec.as<int64_t>());
        // counts (dist_nnz + exscan, binary_io.cpp) ...
        auto cnt = allgather_small(cm, c, {ne});
        int64_t total = 0, before = 0;
        for (int r = 0; r < p; ++r) {
            if (r < me) before += cnt[r];
            total += cnt[r];
        }
        // ... rank 0 creates the file with the header; everyone learns whether it could
        int64_t ok = 1;
        std::string err;
        if (me == 0) {
            Fd f;
            f.fd = ::open(path, O_WRONLY | O_CREAT | O_TRUNC, 0644);
            if (f.fd < 0) {
                ok = 0;
                err = std::string("cannot create '") + path + "': " + std::strerror(errno);
            } else {
                unsigned char hb[kHeaderBytes];
                std::memcpy(hb, kMagic, 4);
                std::memcpy(hb + 4, &kVersion, 4);
                const int64_t dims[3] = {nrows, ncols, total};
                std::memcpy(hb + 8, dims, sizeof dims);
                try {
                    pwrite_all(f.fd, hb, kHeaderBytes, 0);
                    if (::ftruncate(f.fd, kHeaderBytes + total * kRecBytes) != 0) throw Fail{SLAPCU_ERR_IO, "ftruncate"};
                } catch (const Fail& e) {
                    ok = 0;
                    err = e.msg;
                }
            }
        }
        auto hdr = allgather_small(cm, c, {ok});
        if (!hdr[0]) throw Fail{SLAPCU_ERR_IO, me == 0 ? err : "rank 0 could not create '" + std::string(path) + "'"};
        // my records at 32 + before*24, streamed through two pinned buffers
        ok = 1;
        try {
            Fd f;
            f.fd = ::open(path, O_WRONLY);
            if (f.fd < 0) throw Fail{SLAPCU_ERR_IO, std::string("cannot open '") + path + "' for writing"};
            if (ne > 0) {
                Pinned buf0(size_t(kChunkRecs) * kRecBytes), buf1(size_t(kChunkRecs) * kRecBytes);
                void* bufs[2] = {buf0.p, buf1.p};
                cudaEvent_t ev[2];
                SLAPCU_CUDA(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
                SLAPCU_CUDA(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
                struct Ev {
                    cudaEvent_t* e;
                    ~Ev() {
                        cudaEventDestroy(e[0]);
                        cudaEventDestroy(e[1]);
                    }
                } evg{ev};
                const int64_t nchunks = (ne + kChunkRecs - 1) / kChunkRecs;
                auto issue = [&](int64_t k) {
                    const int64_t o = k * kChunkRecs, m = std::min(kChunkRecs, ne - o);
                    SLAPCU_CUDA(cudaMemcpyAsync(bufs[k & 1], rec.as<char>() + o * kRecBytes, size_t(m) * kRecBytes,
                                                cudaMemcpyDeviceToHost, c.stream));
                    SLAPCU_CUDA(cudaEventRecord(ev[k & 1], c.stream));
                };
                issue(0);
                for (int64_t k = 0; k < nchunks; ++k) {
                    SLAPCU_CUDA(cudaEventSynchronize(ev[k & 1]));
                    if (k + 1 < nchunks) issue(k + 1);  // next copy overlaps this write
                    const int64_t o = k * kChunkRecs, m = std::min(kChunkRecs, ne - o);
                    pwrite_all(f.fd, bufs[k & 1], m * kRecBytes, kHeaderBytes + (before + o) * kRecBytes);
                }
            }
        } catch (const Fail& e) {
            ok = 0;
            err = e.msg;
        }
        auto done = allgather_small(cm, c, {ok});
        for (int r = 0; r < p; ++r)
            if (!done[r]) throw Fail{SLAPCU_ERR_IO, ok ? "rank " + std::to_string(r) + " failed to write its records" : err};
        cm->calls[kAllgatherv] += 3;
        return SLAPCU_OK;
    } catch (const Fail& e) {
        c.last_error = e.msg;
        return e.st;
    }
}

slapcu_status slapcu_read_cb2b(slapcu_comm cm, const char* path, int pr, int pc, slapcu_csc_out* out,
                               int64_t* out_row_start, int64_t* out_col_start, int64_t* nrows, int64_t* ncols) {
    if (!cm || !path || !out || !out_row_start || !out_col_start) return SLAPCU_ERR_INVALID;
    Ctx& c = ctx_of(cm->ctx);
    *out = slapcu_csc_out{};
    OutGuard guard{c, out};
    try {
        SLAPCU_CUDA(cudaSetDevice(c.device));
        const int p = cm->nranks, me = cm->rank;
        if (pr < 1 || pc < 1 || int64_t(pr) * pc != p)
            throw Fail{SLAPCU_ERR_SHAPE, std::to_string(pr) + "x" + std::to_string(pc) + " grid on " +
                                             std::to_string(p) + " ranks"};
        const Header h = read_header(path);
        const int64_t lo = h.nnz * me / p, hi = h.nnz * (me + 1) / p, ne = hi - lo;
        DevBuf rec(size_t(kRecBytes) * std::max<int64_t>(ne, 1), c.stream);
        if (ne > 0) {
            Fd f;
            f.fd = ::open(path, O_RDONLY);
            if (f.fd < 0) throw Fail{SLAPCU_ERR_IO, std::string("cannot open '") + path + "'"};
            Pinned buf0(size_t(kChunkRecs) * kRecBytes), buf1(size_t(kChunkRecs) * kRecBytes);
            void* bufs[2] = {buf0.p, buf1.p};
            cudaEvent_t ev[2];
            SLAPCU_CUDA(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
            SLAPCU_CUDA(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
            struct Ev {
                cudaEvent_t* e;
                ~Ev() {
                    cudaEventDestroy(e[0]);
                    cudaEventDestroy(e[1]);
                }
            } evg{ev};
            const int64_t nchunks = (ne + kChunkRecs - 1) / kChunkRecs;
            for (int64_t k = 0; k < nchunks; ++k) {
                if (k >= 2) SLAPCU_CUDA(cudaEventSynchronize(ev[k & 1]));  // buffer free again
                const int64_t o = k * kChunkRecs, m = std::min(kChunkRecs, ne - o);
                pread_all(f.fd, bufs[k & 1], m * kRecBytes, kHeaderBytes + (lo + o) * kRecBytes);
                SLAPCU_CUDA(cudaMemcpyAsync(rec.as<char>() + o * kRecBytes, bufs[k & 1], size_t(m) * kRecBytes,
                                            cudaMemcpyHostToDevice, c.stream));
                SLAPCU_CUDA(cudaEventRecord(ev[k & 1], c.stream));
            }
            SLAPCU_CUDA(cudaStreamSynchronize(c.stream));
        }
        const int64_t ne1 = std::max<int64_t>(ne, 1);
        DevBuf rows(sizeof(int64_t) * ne1, c.stream), cols(sizeof(int64_t) * ne1, c.stream),
            vals(sizeof(int64_t) * ne1, c.stream);
        if (ne > 0)
            launch(c, k_split_records, dim3(grid_for(c, 3 * ne, 256)), dim3(256), 0, ne,
                   (const int64_t*)rec.as<int64_t>(), rows.as<int64_t>(), cols.as<int64_t>(), vals.as<int64_t>());
        rec.release();
        // read_binary routes with distribute_triples onto block_offsets rows / cols
        std::vector<int64_t> rc(pr + 1), cc(pc + 1);
        for (int i = 0; i < pr; ++i) rc[i] = int64_t(i) * (h.m / pr);
        rc[pr] = h.m;
        for (int j = 0; j < pc; ++j) cc[j] = int64_t(j) * (h.n / pc);
        cc[pc] = h.n;
        std::vector<int32_t> owner(size_t(pr) * pc);
        for (int k = 0; k < pr * pc; ++k) owner[k] = k;
        slapcu_tiling t{pr, pc, rc.data(), cc.data(), owner.data()};
        Src s;
        s.n = ne;
        s.grow = rows.as<int64_t>();
        s.gcol = cols.as<int64_t>();
        redistribute(cm, c, s, vals.get(), 0, false, h.m, h.n, SLAPCU_PLUS_TIMES_F64, &t, 0, out, out_row_start,
                     out_col_start);
        if (nrows) *nrows = h.m;
        if (ncols) *ncols = h.n;
        guard.ok = true;
        return SLAPCU_OK;
    } catch (const Fail& e) {
        c.last_error = e.msg;
        return e.st;
    }
}

}  // extern "C"
