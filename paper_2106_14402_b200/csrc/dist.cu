// dist.cu -- 2D Sparse SUMMA and 3D communication-avoiding SpGEMM over NCCL.
//
// Replaces the reference's simulated transport (comm.hpp:178-348, ranks are
// threads rendezvousing on a mutex) with one process (or host thread) per GPU
// and NCCL communicators over NVLink 5 / NVSwitch:
//
//   summa2d_spgemm (summa.hpp:106-163)
//     stage s: A(i,s) broadcast on the row communicator, B(s,j) on the column
//     communicator (summa.hpp:133-140 broadcast_block) -- here ncclBroadcast of
//     the CSC arrays straight out of the owner's device buffers, issued on a
//     dedicated comm stream one stage AHEAD of the local multiply into the other
//     half of a double buffer, so stage s+1's transfer overlaps stage s's
//     SpGEMM; the partials are merged once at the end in stage order
//     (summa.hpp:156) by the device multiway merge.
//   ca3d_spgemm (spgemm3d.hpp:21-106)
//     per-layer SUMMA, C_int split into c column pieces (block_offsets), one
//     fiber exchange (counts all-gathered, then grouped ncclSend/ncclRecv --
//     NCCL has no alltoallv), merge in fiber order.
//
// Block metadata (dims, nnz) of every rank is all-gathered once per call, so
// every rank knows every broadcast's size up front (NCCL needs matching
// counts) and shape errors are detected consistently on all ranks before any
// data collective is posted.
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "kern.cuh"

#include "comm.hpp"

namespace slapcu {
namespace {

bool is_square(int64_t v, int64_t* root) {
    if (v < 0) return false;
    int64_t r = (int64_t)std::llround(std::sqrt((double)v));
    for (int64_t c = std::max<int64_t>(r - 1, 0); c <= r + 1; ++c)
        if (c * c == v) {
            *root = c;
            return true;
        }
    return false;
}

ncclComm_t split(slapcu_comm_s* cm, const std::string& name, int color, int key) {
    auto it = cm->splits.find(name);
    if (it != cm->splits.end()) return it->second;
    ncclComm_t out = nullptr;
    SLAPCU_NCCL(ncclCommSplit(cm->world, color, key, &out, nullptr));
    cm->splits[name] = out;
    return out;
}

// Block metadata of every rank (kMeta int64 each): A then B as
// [nrows, ncols, colptr base, entry count] -- operands may be column windows
// whose colptr does not start at 0 (batched.hpp slices).
constexpr int kMeta = 8;
enum { MA_R = 0, MA_C, MA_BASE, MA_NZ, MB_R, MB_C, MB_BASE, MB_NZ };

std::vector<int64_t> allgather_meta(slapcu_comm_s* cm, Ctx& c, const DevCsc& A, const DevCsc& B) {
    const int p = cm->nranks;
    int64_t mine[kMeta] = {A.nrows, A.ncols, A.base, A.span, B.nrows, B.ncols, B.base, B.span};
    DevBuf d(sizeof(int64_t) * kMeta * (p + 1), c.stream);
    SLAPCU_CUDA(cudaMemcpyAsync(d.as<int64_t>() + kMeta * p, mine, sizeof(mine), cudaMemcpyHostToDevice, c.stream));
    SLAPCU_NCCL(ncclAllGather(d.as<int64_t>() + kMeta * p, d.as<int64_t>(), kMeta, ncclInt64, cm->world, c.stream));
    std::vector<int64_t> h(kMeta * p);
    SLAPCU_CUDA(cudaMemcpyAsync(h.data(), d.get(), sizeof(int64_t) * kMeta * p, cudaMemcpyDeviceToHost, c.stream));
    SLAPCU_CUDA(cudaStreamSynchronize(c.stream));
    cm->calls[kAllgatherv] += 1;
    cm->bytes[kAllgatherv] += sizeof(mine);
    return h;
}

// One owned device CSC.
struct Block {
    DevBuf cp, rw, v;
    int64_t nrows = 0, ncols = 0, nnz = 0;
    DevCsc view() const { return DevCsc{nrows, ncols, nnz, cp.as<int64_t>(), rw.as<int32_t>(), v.get()}; }
};

// Receive slot for a broadcast block, sized for the largest block it holds.
struct Slot {
    DevBuf cp, rw, v;
    void reserve(Ctx& c, int64_t ncols, int64_t nnz, int vs) {
        cp.reset(sizeof(int64_t) * (ncols + 1), c.stream);
        rw.reset(sizeof(int32_t) * std::max<int64_t>(nnz, 1), c.stream);
        v.reset(size_t(vs) * std::max<int64_t>(nnz, 1), c.stream);
    }
};

// ncclBroadcast of one CSC block (three arrays) from group rank `root`.  The
// root broadcasts in place from its own block (only its entry range
// [base, base+nnz)); the others receive into slot.  colptr travels unchanged,
// so a receiver addresses the entries through pointers shifted by -base
// (never dereferenced outside [base, base+nnz)).
DevCsc bcast_block(slapcu_comm_s* cm, ncclComm_t comm, int my_group_rank, int root, const DevCsc& mine,
                   int64_t nrows, int64_t ncols, int64_t base, int64_t nnz, int vs, Slot& slot, cudaStream_t s) {
    const bool am_root = my_group_rank == root;
    int64_t* cp = am_root ? const_cast<int64_t*>(mine.cp) : slot.cp.as<int64_t>();
    int32_t* rw = am_root ? const_cast<int32_t*>(mine.rw) + base : slot.rw.as<int32_t>();
    char* v = am_root ? static_cast<char*>(const_cast<void*>(mine.v)) + size_t(vs) * base
                      : static_cast<char*>(slot.v.get());
    SLAPCU_NCCL(ncclBroadcast(cp, cp, size_t(ncols + 1), ncclInt64, root, comm, s));
    if (nnz) {
        SLAPCU_NCCL(ncclBroadcast(rw, rw, size_t(nnz), ncclInt32, root, comm, s));
        SLAPCU_NCCL(ncclBroadcast(v, v, size_t(nnz) * vs, ncclUint8, root, comm, s));
    }
    if (am_root) {
        cm->calls[kBcast] += 1;  // one logical block broadcast, like comm.hpp:202-218
        cm->bytes[kBcast] += sizeof(int64_t) * (ncols + 1) + (sizeof(int32_t) + vs) * nnz;
    } else {
        cm->calls[kBcast] += 1;
    }
    return DevCsc{nrows, ncols, nnz, cp, rw - base, v - size_t(vs) * base, base, nnz};
}

// Local multiply into an owned block (symbolic -> allocate -> numeric).
void local_multiply(Ctx& c, const DevCsc& A, const DevCsc& B, int sr, int alg, Block& out, float* ms) {
    const int vs = value_size(sr);
    out.nrows = A.nrows;
    out.ncols = B.ncols;
    out.cp.reset(sizeof(int64_t) * (B.ncols + 1), c.stream);
    // single product pass when its staging area fits in half the free memory,
    // else the two-pass symbolic -> numeric contract
    const size_t fr = device_available(c);
    bool fused = true;
    try {
        out.nnz = fused_begin(c, A, B, sr, alg, out.cp.as<int64_t>(), int64_t(fr / 2));
    } catch (const Fail& e) {
        if (e.st != SLAPCU_ERR_BUDGET) throw;
        fused = false;
        out.nnz = spgemm_symbolic(c, A, B, alg, out.cp.as<int64_t>());
    }
    out.rw.reset(sizeof(int32_t) * std::max<int64_t>(out.nnz, 1), c.stream);
    out.v.reset(size_t(vs) * std::max<int64_t>(out.nnz, 1), c.stream);
    if (fused)
        fused_finish(c, A, B, sr, out.rw.as<int32_t>(), out.v.get());
    else
        spgemm_numeric(c, A, B, sr, alg, out.cp.as<int64_t>(), out.rw.as<int32_t>(), out.v.get());
    *ms += c.sym_ms + c.num_ms;
}

void merge_blocks(Ctx& c, const std::vector<DevCsc>& parts, int sr, slapcu_csc_out* C) {
    const int vs = value_size(sr);
    const int64_t n = parts[0].ncols;
    C->nrows = parts[0].nrows;
    C->ncols = n;
    SLAPCU_CUDA(cudaMallocAsync((void**)&C->colptr, sizeof(int64_t) * (n + 1), c.stream));
    C->nnz = merge_symbolic(c, (int)parts.size(), parts.data(), C->colptr);
    SLAPCU_CUDA(cudaMallocAsync((void**)&C->rowids, sizeof(int32_t) * std::max<int64_t>(C->nnz, 1), c.stream));
    SLAPCU_CUDA(cudaMallocAsync(&C->vals, size_t(vs) * std::max<int64_t>(C->nnz, 1), c.stream));
    merge_numeric(c, (int)parts.size(), parts.data(), sr, C->colptr, C->rowids, C->vals);
}

void move_out(Ctx& c, Block& b, slapcu_csc_out* C) {
    C->nrows = b.nrows;
    C->ncols = b.ncols;
    C->nnz = b.nnz;
    C->colptr = static_cast<int64_t*>(b.cp.detach());
    C->rowids = static_cast<int32_t*>(b.rw.detach());
    C->vals = b.v.detach();
    (void)c;
}

struct Timer {
    cudaEvent_t a = nullptr, b = nullptr;
    Timer() {
        cudaEventCreate(&a);
        cudaEventCreate(&b);
    }
    ~Timer() {
        cudaEventDestroy(a);
        cudaEventDestroy(b);
    }
    float ms() {
        float t = 0.f;
        cudaEventElapsedTime(&t, a, b);
        return t;
    }
};

// ---- concatenated-k local multiply (no partial merge)
//
// C(i,j) = sum_s A(i,s) B(s,j) is formed as ONE product [A(i,0) .. A(i,q-1)] x
// [B(0,j); ..; B(q-1,j)] once every stage's blocks have arrived: the stage
// partials of summa.hpp:145-156 -- each nearly as large as C(i,j) itself for
// A*A -- and their merge disappear.  Exact semirings are bit-identical to the
// stage-order fold; PlusTimes fp64 stays within the north_star tolerance.

__global__ void k_cat_colptr(const int64_t* __restrict__ in, int64_t K, int64_t pre, int64_t* __restrict__ out,
                             int last) {
    const int64_t n = K + (last ? 1 : 0);
    for (int64_t x = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; x < n; x += int64_t(gridDim.x) * blockDim.x)
        out[x] = in[x] - in[0] + pre;
}

struct VStack {
    const int64_t* cp[8];
    const int32_t* rw[8];
    const char* v[8];
    int64_t koff[8];
    int q;
};

__global__ void k_vstack_count(VStack vs, int64_t n, int64_t* __restrict__ cnt) {
    for (int64_t x = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; x < n; x += int64_t(gridDim.x) * blockDim.x) {
        int64_t t = 0;
        for (int s = 0; s < vs.q; ++s) t += vs.cp[s][x + 1] - vs.cp[s][x];
        cnt[x] = t;
    }
}

__global__ void k_vstack_fill(VStack vs, int vsize, int64_t n, const int64_t* __restrict__ ocp,
                              int32_t* __restrict__ orw, char* __restrict__ ov) {
    const int lane = threadIdx.x & 31;
    for (int64_t x = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; x < n;
         x += (int64_t(gridDim.x) * blockDim.x) >> 5) {
        int64_t o = ocp[x];
        for (int s = 0; s < vs.q; ++s) {
            const int64_t a = vs.cp[s][x], b = vs.cp[s][x + 1];
            const int32_t add = (int32_t)vs.koff[s];
            for (int64_t e = a + lane; e < b; e += 32) {
                orw[o + (e - a)] = vs.rw[s][e] + add;
                for (int k = 0; k < vsize; ++k) ov[(o + (e - a)) * vsize + k] = vs.v[s][e * vsize + k];
            }
            o += b - a;
        }
    }
}

// [A_0 .. A_{q-1}] (column concatenation) and [B_0; ..; B_{q-1}] (row
// concatenation) of the received stage blocks, then one direct product.
void concat_multiply(Ctx& c, const std::vector<DevCsc>& As, const std::vector<DevCsc>& Bs, int sr, int alg,
                     Block& out, float* ms) {
    const int q = (int)As.size();
    const int vs = value_size(sr);
    if (q > 8) throw Fail{SLAPCU_ERR_INTERNAL, "concat_multiply: at most 8 parts (VStack)"};
    int64_t K = 0, annz = 0, bnnz = 0;
    for (int s = 0; s < q; ++s) {
        K += As[s].ncols;
        annz += As[s].span;
        bnnz += Bs[s].span;
    }
    const int64_t M = As[0].nrows, N = Bs[0].ncols;
    Block Ac, Bc;
    Ac.nrows = M; Ac.ncols = K; Ac.nnz = annz;
    Ac.cp.reset(sizeof(int64_t) * (K + 1), c.stream);
    Ac.rw.reset(sizeof(int32_t) * std::max<int64_t>(annz, 1), c.stream);
    Ac.v.reset(size_t(vs) * std::max<int64_t>(annz, 1), c.stream);
    int64_t koff = 0, pre = 0;
    for (int s = 0; s < q; ++s) {
        const DevCsc& a = As[s];
        launch(c, k_cat_colptr, dim3(grid_for(c, a.ncols + 1, 256)), dim3(256), 0, a.cp, a.ncols, pre,
               Ac.cp.as<int64_t>() + koff, s == q - 1 ? 1 : 0);
        if (a.span) {
            SLAPCU_CUDA(cudaMemcpyAsync(Ac.rw.as<int32_t>() + pre, a.rw + a.base, sizeof(int32_t) * a.span,
                                        cudaMemcpyDeviceToDevice, c.stream));
            SLAPCU_CUDA(cudaMemcpyAsync(static_cast<char*>(Ac.v.get()) + size_t(vs) * pre,
                                        static_cast<const char*>(a.v) + size_t(vs) * a.base, size_t(vs) * a.span,
                                        cudaMemcpyDeviceToDevice, c.stream));
        }
        koff += a.ncols;
        pre += a.span;
    }
    VStack st{};
    st.q = q;
    int64_t ko = 0;
    for (int s = 0; s < q; ++s) {
        st.cp[s] = Bs[s].cp;
        st.rw[s] = Bs[s].rw;
        st.v[s] = static_cast<const char*>(Bs[s].v);
        st.koff[s] = ko;
        ko += Bs[s].nrows;
    }
    Bc.nrows = ko; Bc.ncols = N; Bc.nnz = bnnz;
    Bc.cp.reset(sizeof(int64_t) * (N + 1), c.stream);
    Bc.rw.reset(sizeof(int32_t) * std::max<int64_t>(bnnz, 1), c.stream);
    Bc.v.reset(size_t(vs) * std::max<int64_t>(bnnz, 1), c.stream);
    {
        DevBuf cnt(sizeof(int64_t) * (N + 1), c.stream);
        SLAPCU_CUDA(cudaMemsetAsync(cnt.as<int64_t>() + N, 0, sizeof(int64_t), c.stream));
        launch(c, k_vstack_count, dim3(grid_for(c, N, 256)), dim3(256), 0, st, N, cnt.as<int64_t>());
        exclusive_scan_i64(c, cnt.as<int64_t>(), Bc.cp.as<int64_t>(), N + 1);
        launch(c, k_vstack_fill, dim3(grid_for(c, N * 32, 256)), dim3(256), 0, st, vs, N,
               (const int64_t*)Bc.cp.as<int64_t>(), Bc.rw.as<int32_t>(), static_cast<char*>(Bc.v.get()));
    }
    const DevCsc A = Ac.view(), B = Bc.view();
    // output sized by the bound sum_j min(flops_j, M)
    DevBuf fl(sizeof(int64_t) * std::max<int64_t>(N, 1), c.stream);
    int64_t tot = 0;
    spgemm_flops(c, A, B, fl.as<int64_t>(), &tot);
    std::vector<int64_t> hf(N);
    if (N) SLAPCU_CUDA(cudaMemcpyAsync(hf.data(), fl.get(), sizeof(int64_t) * N, cudaMemcpyDeviceToHost, c.stream));
    SLAPCU_CUDA(cudaStreamSynchronize(c.stream));
    int64_t cap = 0;
    for (int64_t x = 0; x < N; ++x) cap += std::min(hf[x], M);
    out.nrows = M;
    out.ncols = N;
    out.cp.reset(sizeof(int64_t) * (N + 1), c.stream);
    // the product lands in a bound-sized scratch kept on the context (no
    // per-call allocation of ~3x the output), then moves into exact buffers
    DirectCache& d = c.direct;
    d.dist_rw.reset(sizeof(int32_t) * std::max<int64_t>(cap, 1), c.stream);
    d.dist_v.reset(size_t(vs) * std::max<int64_t>(cap, 1), c.stream);
    cudaEvent_t e0, e1;
    SLAPCU_CUDA(cudaEventCreate(&e0));
    SLAPCU_CUDA(cudaEventCreate(&e1));
    SLAPCU_CUDA(cudaEventRecord(e0, c.stream));
    out.nnz = direct_spgemm(c, A, B, sr, alg, cap, out.cp.as<int64_t>(), d.dist_rw.as<int32_t>(), d.dist_v.get());
    out.rw.reset(sizeof(int32_t) * std::max<int64_t>(out.nnz, 1), c.stream);
    out.v.reset(size_t(vs) * std::max<int64_t>(out.nnz, 1), c.stream);
    if (out.nnz) {
        SLAPCU_CUDA(cudaMemcpyAsync(out.rw.get(), d.dist_rw.get(), sizeof(int32_t) * out.nnz, cudaMemcpyDeviceToDevice,
                                    c.stream));
        SLAPCU_CUDA(cudaMemcpyAsync(out.v.get(), d.dist_v.get(), size_t(vs) * out.nnz, cudaMemcpyDeviceToDevice,
                                    c.stream));
    }
    SLAPCU_CUDA(cudaEventRecord(e1, c.stream));
    SLAPCU_CUDA(cudaEventSynchronize(e1));
    float t = 0.f;
    cudaEventElapsedTime(&t, e0, e1);
    *ms += t;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
}

// Multiplicative identity of each semiring (one ⊗ id = id ⊗ one = value).
template <int ID>
typename Sr<ID>::T mul_one() {
    if constexpr (ID == SLAPCU_MIN_PLUS_I32 || ID == SLAPCU_MIN_PLUS_F64)
        return typename Sr<ID>::T(0);
    else
        return typename Sr<ID>::T(1);
}

__global__ void k_identity(int64_t n, int64_t* __restrict__ cp, int32_t* __restrict__ rw, char* __restrict__ v,
                           const char* __restrict__ one, int vsize) {
    for (int64_t x = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; x <= n; x += int64_t(gridDim.x) * blockDim.x) {
        cp[x] = x;
        if (x < n) {
            rw[x] = (int32_t)x;
            for (int k = 0; k < vsize; ++k) v[x * vsize + k] = one[k];
        }
    }
}

// C = P0 (+) P1 (+) ... as the product [P0 .. Pq-1] x [I; ..; I] on the direct
// path (bitmap union per row tile instead of per-entry binary searches).
// Exact semirings are bit-identical to the stage-order fold; PlusTimes fp64
// folds in atomic order (north_star tolerance 1e-12).
void fast_merge(Ctx& c, std::vector<DevCsc> parts, int sr, int alg, slapcu_csc_out* C, float* ms) {
    const int vs = value_size(sr);
    for (auto& p : parts) resolve(c, p);
    if (parts.size() > 8) {  // the concatenated product stacks at most 8 parts: multiway merge instead
        merge_blocks(c, parts, sr, C);
        return;
    }
    const int64_t N = parts[0].ncols;
    Block id;
    id.nrows = N;
    id.ncols = N;
    id.nnz = N;
    id.cp.reset(sizeof(int64_t) * (N + 1), c.stream);
    id.rw.reset(sizeof(int32_t) * std::max<int64_t>(N, 1), c.stream);
    id.v.reset(size_t(vs) * std::max<int64_t>(N, 1), c.stream);
    char one[8] = {0};
    dispatch_sr(sr, [&](auto idc) {
        constexpr int ID = decltype(idc)::value;
        const auto o = mul_one<ID>();
        std::memcpy(one, &o, sizeof(o));
    });
    DevBuf done(8, c.stream);
    SLAPCU_CUDA(cudaMemcpyAsync(done.get(), one, 8, cudaMemcpyHostToDevice, c.stream));
    launch(c, k_identity, dim3(grid_for(c, N + 1, 256)), dim3(256), 0, N, id.cp.as<int64_t>(), id.rw.as<int32_t>(),
           static_cast<char*>(id.v.get()), (const char*)done.get(), vs);
    DevCsc iv = id.view();
    resolve(c, iv);
    std::vector<DevCsc> ids(parts.size(), iv);
    Block out;
    concat_multiply(c, parts, ids, sr, alg, out, ms);
    move_out(c, out, C);
}

// The q-stage SUMMA over a q x q (layer) grid.  `gr_row`/`gr_col` are this
// rank's group ranks in the row / column communicators (= its column / row
// coordinate); meta_of(i,j) returns the metadata index of grid rank (i,j).
template <class MetaOf>
void summa_stages(slapcu_comm_s* cm, Ctx& c, ncclComm_t row, ncclComm_t col, int q, int myi, int myj,
                  const DevCsc& A, const DevCsc& B, int sr, int alg, const std::vector<int64_t>& meta, MetaOf meta_of,
                  std::vector<Block>& partials, slapcu_dist_stats* st) {
    const int vs = value_size(sr);
    // size the double buffer for the largest block this rank will receive
    int64_t a_nc = 0, a_nz = 0, b_nc = 0, b_nz = 0;
    for (int s = 0; s < q; ++s) {
        const int64_t* ma = &meta[kMeta * meta_of(myi, s)];
        const int64_t* mb = &meta[kMeta * meta_of(s, myj)];
        a_nc = std::max(a_nc, ma[MA_C]);
        a_nz = std::max(a_nz, ma[MA_NZ]);
        b_nc = std::max(b_nc, mb[MB_C]);
        b_nz = std::max(b_nz, mb[MB_NZ]);
    }
    if (q == 1 && c.opt.summa_concat) {  // one stage: the local product alone, on the direct path
        float local_ms = 0.f;
        if (A.ncols != B.nrows) throw Fail{SLAPCU_ERR_DIM, "SUMMA inner dims disagree"};
        int64_t f = 0;
        spgemm_flops(c, A, B, nullptr, &f);
        if (st) st->flops += f;
        partials.resize(1);
        concat_multiply(c, {A}, {B}, sr, alg, partials[0], &local_ms);
        if (st) {
            st->ms_local += local_ms;
            st->stages = 1;
        }
        return;
    }
    const bool concat = c.opt.summa_concat && q > 1 && q <= 8;
    std::vector<Slot> sa(concat ? q : 2), sb(concat ? q : 2);
    const int nslots = concat ? q : (q > 1 ? 2 : 1);
    for (int k = 0; k < nslots; ++k) {
        sa[k].reserve(c, a_nc, a_nz, vs);
        sb[k].reserve(c, b_nc, b_nz, vs);
    }
    std::vector<cudaEvent_t> bc_done(q), slot_free(2);
    for (auto& e : bc_done) SLAPCU_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (auto& e : slot_free) SLAPCU_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    std::vector<DevCsc> sa_view(q), sb_view(q);
    // the comm stream must not start before the inputs are ready on the compute stream
    cudaEvent_t ready;
    SLAPCU_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
    SLAPCU_CUDA(cudaEventRecord(ready, c.stream));
    SLAPCU_CUDA(cudaStreamWaitEvent(cm->comm_stream, ready, 0));
    auto issue = [&](int s) {
        const int slot = concat ? s : s % 2;
        if (!concat && s >= 2) SLAPCU_CUDA(cudaStreamWaitEvent(cm->comm_stream, slot_free[slot], 0));
        const int64_t* ma = &meta[kMeta * meta_of(myi, s)];
        const int64_t* mb = &meta[kMeta * meta_of(s, myj)];
        SLAPCU_NCCL(ncclGroupStart());
        sa_view[s] = bcast_block(cm, row, myj, s, A, ma[MA_R], ma[MA_C], ma[MA_BASE], ma[MA_NZ], vs, sa[slot],
                                 cm->comm_stream);
        sb_view[s] = bcast_block(cm, col, myi, s, B, mb[MB_R], mb[MB_C], mb[MB_BASE], mb[MB_NZ], vs, sb[slot],
                                 cm->comm_stream);
        SLAPCU_NCCL(ncclGroupEnd());
        SLAPCU_CUDA(cudaEventRecord(bc_done[s], cm->comm_stream));
    };
    float local_ms = 0.f, exposed = 0.f;
    Timer w;
    if (concat) {
        // every stage's broadcasts are issued at once; the multiply waits for all
        partials.resize(1);
        for (int s = 0; s < q; ++s) issue(s);
        SLAPCU_CUDA(cudaEventRecord(w.a, c.stream));
        for (int s = 0; s < q; ++s) SLAPCU_CUDA(cudaStreamWaitEvent(c.stream, bc_done[s], 0));
        SLAPCU_CUDA(cudaEventRecord(w.b, c.stream));
        SLAPCU_CUDA(cudaEventSynchronize(w.b));
        exposed = w.ms();
        for (int s = 0; s < q; ++s) {
            if (sa_view[s].ncols != sb_view[s].nrows)
                throw Fail{SLAPCU_ERR_DIM, "SUMMA stage blocks misaligned on the inner dimension"};
            int64_t f = 0;
            spgemm_flops(c, sa_view[s], sb_view[s], nullptr, &f);
            if (st) st->flops += f;
        }
        concat_multiply(c, sa_view, sb_view, sr, alg, partials[0], &local_ms);
        SLAPCU_CUDA(cudaStreamSynchronize(cm->comm_stream));
        for (auto& e : bc_done) cudaEventDestroy(e);
        for (auto& e : slot_free) cudaEventDestroy(e);
        cudaEventDestroy(ready);
        if (st) {
            st->ms_local += local_ms;
            st->ms_exposed_bcast += exposed;
            st->stages = q;
        }
        return;
    }
    partials.resize(q);
    if (q > 1) issue(0);
    for (int s = 0; s < q; ++s) {
        if (q > 1 && s + 1 < q) issue(s + 1);  // prefetch the next stage while this one multiplies
        DevCsc a = A, b = B;
        if (q > 1) {
            SLAPCU_CUDA(cudaEventRecord(w.a, c.stream));
            SLAPCU_CUDA(cudaStreamWaitEvent(c.stream, bc_done[s], 0));
            SLAPCU_CUDA(cudaEventRecord(w.b, c.stream));
            SLAPCU_CUDA(cudaEventSynchronize(w.b));
            exposed += w.ms();
            a = sa_view[s];
            b = sb_view[s];
        }
        if (a.ncols != b.nrows) throw Fail{SLAPCU_ERR_DIM, "SUMMA stage blocks misaligned on the inner dimension"};
        int64_t f = 0;
        spgemm_flops(c, a, b, nullptr, &f);
        if (st) st->flops += f;
        local_multiply(c, a, b, sr, alg, partials[s], &local_ms);
        SLAPCU_CUDA(cudaEventRecord(slot_free[s % 2], c.stream));
    }
    SLAPCU_CUDA(cudaStreamSynchronize(c.stream));
    SLAPCU_CUDA(cudaStreamSynchronize(cm->comm_stream));
    for (auto& e : bc_done) cudaEventDestroy(e);
    for (auto& e : slot_free) cudaEventDestroy(e);
    cudaEventDestroy(ready);
    if (st) {
        st->ms_local += local_ms;
        st->ms_exposed_bcast += exposed;
        st->stages = q;
    }
}

}  // namespace
}  // namespace slapcu

using namespace slapcu;

extern "C" {

slapcu_status slapcu_comm_unique_id(void* id128) {
    if (!id128) return SLAPCU_ERR_INVALID;
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) return SLAPCU_ERR_COMM;
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    std::memcpy(id128, &id, sizeof(id));
    return SLAPCU_OK;
}

slapcu_status slapcu_comm_create(slapcu_comm* out, slapcu_ctx ctx, int rank, int nranks, const void* id128) {
    if (!out || !ctx || !id128 || nranks < 1 || rank < 0 || rank >= nranks) return SLAPCU_ERR_INVALID;
    *out = nullptr;
    auto* cm = new slapcu_comm_s;
    cm->ctx = ctx;
    cm->rank = rank;
    cm->nranks = nranks;
    Ctx& c = ctx_of(ctx);
    try {
        SLAPCU_CUDA(cudaSetDevice(c.device));
        SLAPCU_CUDA(cudaStreamCreateWithFlags(&cm->comm_stream, cudaStreamNonBlocking));
        ncclUniqueId id;
        std::memcpy(&id, id128, sizeof(id));
        SLAPCU_NCCL(ncclCommInitRank(&cm->world, nranks, id, rank));
    } catch (const Fail& e) {
        c.last_error = e.msg;
        if (cm->comm_stream) cudaStreamDestroy(cm->comm_stream);
        delete cm;
        return e.st;
    }
    *out = cm;
    return SLAPCU_OK;
}

slapcu_status slapcu_comm_destroy(slapcu_comm cm) {
    if (!cm) return SLAPCU_ERR_INVALID;
    cudaSetDevice(ctx_of(cm->ctx).device);
    for (auto& kv : cm->splits) ncclCommDestroy(kv.second);
    if (cm->world) ncclCommDestroy(cm->world);
    if (cm->comm_stream) cudaStreamDestroy(cm->comm_stream);
    delete cm;
    return SLAPCU_OK;
}

slapcu_status slapcu_comm_counters(slapcu_comm cm, int kind, int64_t* calls, int64_t* bytes) {
    if (!cm || kind < 0 || kind > 3) return SLAPCU_ERR_INVALID;
    if (calls) *calls = cm->calls[kind];
    if (bytes) *bytes = cm->bytes[kind];
    return SLAPCU_OK;
}

slapcu_status slapcu_summa2d(slapcu_comm cm, const slapcu_csc* A_local, const slapcu_csc* B_local,
                             slapcu_semiring sr, slapcu_alg alg, slapcu_csc_out* C_local, slapcu_dist_stats* stats) {
    if (!cm || !A_local || !B_local || !C_local) return SLAPCU_ERR_INVALID;
    Ctx& c = ctx_of(cm->ctx);
    try {
        SLAPCU_CUDA(cudaSetDevice(c.device));
        if (value_size(sr) == 0) throw Fail{SLAPCU_ERR_INVALID, "unknown semiring"};
        int64_t q = 0;
        if (!is_square(cm->nranks, &q))
            throw Fail{SLAPCU_ERR_SHAPE, "2D SUMMA needs a square process grid, got p=" + std::to_string(cm->nranks)};
        if (stats) *stats = slapcu_dist_stats{};
        Timer total;
        SLAPCU_CUDA(cudaEventRecord(total.a, c.stream));
        DevCsc A = view(*A_local), B = view(*B_local);
        resolve(c, A);
        resolve(c, B);
        const int i = cm->rank / (int)q, j = cm->rank % (int)q;
        std::vector<int64_t> meta;
        ncclComm_t row = nullptr, col = nullptr;
        if (q > 1) {
            meta = allgather_meta(cm, c, A, B);
            // summa.hpp:116-122: every stage pair must agree on the inner extent
            for (int ii = 0; ii < q; ++ii)
                for (int jj = 0; jj < q; ++jj)
                    for (int s = 0; s < q; ++s)
                        if (meta[kMeta * (ii * q + s) + MA_C] != meta[kMeta * (s * q + jj) + MB_R])
                            throw Fail{SLAPCU_ERR_DIM, "SUMMA inner block offsets of A and B disagree"};
            row = split(cm, "row2d", i, j);
            col = split(cm, "col2d", j, i);
        } else {
            meta = {A.nrows, A.ncols, A.base, A.span, B.nrows, B.ncols, B.base, B.span};
            if (A.ncols != B.nrows) throw Fail{SLAPCU_ERR_DIM, "SUMMA inner dims disagree"};
        }
        std::vector<Block> partials;
        summa_stages(cm, c, row, col, (int)q, i, j, A, B, sr, alg, meta,
                     [&](int ii, int jj) { return q > 1 ? ii * (int)q + jj : 0; }, partials, stats);
        Timer mt;
        SLAPCU_CUDA(cudaEventRecord(mt.a, c.stream));
        if (partials.size() == 1) {
            move_out(c, partials[0], C_local);
        } else {
            std::vector<DevCsc> pv;
            for (auto& p : partials) pv.push_back(p.view());
            merge_blocks(c, pv, sr, C_local);
        }
        SLAPCU_CUDA(cudaEventRecord(mt.b, c.stream));
        SLAPCU_CUDA(cudaEventRecord(total.b, c.stream));
        SLAPCU_CUDA(cudaStreamSynchronize(c.stream));
        if (stats) {
            stats->ms_merge = mt.ms();
            stats->ms_total = total.ms();
            stats->nnz_out = C_local->nnz;
        }
        return SLAPCU_OK;
    } catch (const Fail& e) {
        c.last_error = e.msg;
        return e.st;
    }
}

__global__ void k_col_counts(int64_t n, const int64_t* __restrict__ cp, int64_t* __restrict__ out) {
    for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < n; j += int64_t(gridDim.x) * blockDim.x)
        out[j] = cp[j + 1] - cp[j];
}

// batched.hpp:70-117 dist_symbolic_col_nnz: the pattern product over the
// q x q grid (OrAnd SUMMA on all-one copies of the operands' patterns), its
// per-column counts summed over the grid column (allreduce on the column
// communicator) and concatenated over the grid row (all-gather on the row
// communicator): every rank returns all of B's column counts.
slapcu_status slapcu_dist_symbolic_col_nnz(slapcu_comm cm, const slapcu_csc* A_local, const slapcu_csc* B_local,
                                           int64_t* counts, int64_t ncols) {
    if (!cm || !A_local || !B_local || !counts) return SLAPCU_ERR_INVALID;
    Ctx& c = ctx_of(cm->ctx);
    try {
        SLAPCU_CUDA(cudaSetDevice(c.device));
        int64_t q = 0;
        if (!is_square(cm->nranks, &q))
            throw Fail{SLAPCU_ERR_SHAPE, "2D SUMMA needs a square process grid, got p=" + std::to_string(cm->nranks)};
        DevCsc A = view(*A_local), B = view(*B_local);
        resolve(c, A);
        resolve(c, B);
        // pattern operands: values all 1 (u8), addressed like the originals
        const int64_t mx = std::max<int64_t>(std::max<int64_t>(A.span, B.span), 1);
        DevBuf ones(size_t(mx), c.stream);
        SLAPCU_CUDA(cudaMemsetAsync(ones.get(), 1, size_t(mx), c.stream));
        slapcu_csc ap = *A_local, bp = *B_local;
        ap.vals = static_cast<const char*>(ones.get()) - A.base;
        bp.vals = static_cast<const char*>(ones.get()) - B.base;
        slapcu_csc_out cpat{};
        const slapcu_status st =
            slapcu_summa2d(cm, &ap, &bp, SLAPCU_OR_AND_U8, SLAPCU_ALG_HASH, &cpat, nullptr);
        if (st != SLAPCU_OK) return st;
        struct FreeOut {
            Ctx& c;
            slapcu_csc_out& o;
            ~FreeOut() {
                if (o.colptr) cudaFreeAsync(o.colptr, c.stream);
                if (o.rowids) cudaFreeAsync(o.rowids, c.stream);
                if (o.vals) cudaFreeAsync(o.vals, c.stream);
            }
        } free_pat{c, cpat};
        const int i = cm->rank / (int)q, j = cm->rank % (int)q;
        const int64_t nl = B.ncols;
        // every grid column's block width (row all-gather of the local widths)
        std::vector<int64_t> widths(size_t(q), nl);
        ncclComm_t row = nullptr, col = nullptr;
        if (q > 1) {
            row = split(cm, "row2d", i, j);
            col = split(cm, "col2d", j, i);
            DevBuf w(sizeof(int64_t) * (q + 1), c.stream);
            SLAPCU_CUDA(cudaMemcpyAsync(w.as<int64_t>() + q, &nl, sizeof(int64_t), cudaMemcpyHostToDevice, c.stream));
            SLAPCU_NCCL(ncclAllGather(w.as<int64_t>() + q, w.as<int64_t>(), 1, ncclInt64, row, c.stream));
            SLAPCU_CUDA(cudaMemcpyAsync(widths.data(), w.get(), sizeof(int64_t) * q, cudaMemcpyDeviceToHost, c.stream));
            SLAPCU_CUDA(cudaStreamSynchronize(c.stream));
        }
        int64_t total = 0, wmax = 1;
        for (auto x : widths) {
            total += x;
            wmax = std::max(wmax, x);
        }
        if (total != ncols)
            throw Fail{SLAPCU_ERR_DIM, "column blocks sum to " + std::to_string(total) + ", B has " +
                                           std::to_string(ncols) + " columns"};
        DevBuf loc(sizeof(int64_t) * wmax * (q + 1), c.stream);
        int64_t* mine = loc.as<int64_t>() + wmax * q;
        SLAPCU_CUDA(cudaMemsetAsync(mine, 0, sizeof(int64_t) * wmax, c.stream));
        if (nl) launch(c, k_col_counts, dim3(grid_for(c, nl, 256)), dim3(256), 0, nl, (const int64_t*)cpat.colptr, mine);
        if (q > 1) {
            // batched.hpp:109-110 col_comm.allreduce_vec, :111-112 row_comm.allgatherv (padded to the widest block)
            SLAPCU_NCCL(ncclAllReduce(mine, mine, size_t(wmax), ncclInt64, ncclSum, col, c.stream));
            SLAPCU_NCCL(ncclAllGather(mine, loc.as<int64_t>(), size_t(wmax), ncclInt64, row, c.stream));
            cm->calls[kReduce] += 1;
            cm->bytes[kReduce] += sizeof(int64_t) * nl;
            cm->calls[kAllgatherv] += 1;
            cm->bytes[kAllgatherv] += sizeof(int64_t) * nl;
        } else {
            SLAPCU_CUDA(cudaMemcpyAsync(loc.get(), mine, sizeof(int64_t) * wmax, cudaMemcpyDeviceToDevice, c.stream));
        }
        int64_t o = 0;
        for (int b = 0; b < (int)q; ++b) {
            if (widths[b])
                SLAPCU_CUDA(cudaMemcpyAsync(counts + o, loc.as<int64_t>() + int64_t(b) * wmax, sizeof(int64_t) * widths[b],
                                            cudaMemcpyDeviceToHost, c.stream));
            o += widths[b];
        }
        SLAPCU_CUDA(cudaStreamSynchronize(c.stream));
        return SLAPCU_OK;
    } catch (const Fail& e) {
        c.last_error = e.msg;
        return e.st;
    }
}

// layout.hpp:60-66 block_offsets: parts-1 equal blocks, remainder to the last.
static std::vector<int64_t> block_offsets(int64_t ext, int parts) {
    std::vector<int64_t> o(size_t(parts) + 1);
    const int64_t q = ext / parts;
    for (int i = 0; i < parts; ++i) o[i] = int64_t(i) * q;
    o[parts] = ext;
    return o;
}

// algorithms.cpp:267-293 mcl_step on a pr x pc grid (rank = i*pc + j):
// column sums of the input reduced over the grid column and checked (1e-9
// f64 / 1e-5 f32, StochasticityError on every rank), the expansion A*A by the
// 2D SUMMA (layers <= 1, square grid) or -- layers = c > 1 -- by
// redistribute_3d x2 -> ca3d -> redistribute_2d on the device
// (dist_matrix3d.hpp:117-261 regular variant), then inflation / pruning /
// renormalisation with the kept column sums reduced over the grid column.
slapcu_status slapcu_mcl_step_dist(slapcu_comm cm, int pr, int pc, int layers, const slapcu_csc* A_local,
                                   slapcu_semiring sr, double inflation, double prune_threshold,
                                   slapcu_csc_out* C_local) {
    if (!cm || !A_local || !C_local) return SLAPCU_ERR_INVALID;
    Ctx& c = ctx_of(cm->ctx);
    try {
        SLAPCU_CUDA(cudaSetDevice(c.device));
        if (sr != SLAPCU_PLUS_TIMES_F64 && sr != SLAPCU_PLUS_TIMES_F32)
            throw Fail{SLAPCU_ERR_INVALID, "mcl step: PlusTimes f64 or f32"};
        if (pr < 1 || pc < 1 || pr * pc != cm->nranks)
            throw Fail{SLAPCU_ERR_SHAPE, "grid " + std::to_string(pr) + "x" + std::to_string(pc) + " does not match " +
                                             std::to_string(cm->nranks) + " ranks"};
        if (!(inflation > 0.0)) throw Fail{SLAPCU_ERR_SHAPE, "inflation exponent must be positive"};
        DevCsc A = view(*A_local);
        resolve(c, A);
        const int i = cm->rank / pc, j = cm->rank % pc;
        // global dims from every rank's block dims (grid column 0 rows, grid row 0 cols)
        const std::vector<int64_t> meta = allgather_meta(cm, c, A, A);
        int64_t m = 0, n = 0;
        for (int ii = 0; ii < pr; ++ii) m += meta[kMeta * (ii * pc) + MA_R];
        for (int jj = 0; jj < pc; ++jj) n += meta[kMeta * jj + MA_C];
        if (m != n) throw Fail{SLAPCU_ERR_SHAPE, "mcl step needs a square matrix"};
        const double tol = sr == SLAPCU_PLUS_TIMES_F64 ? 1e-9 : 1e-5;
        ncclComm_t col = split(cm, "col2d_" + std::to_string(pr) + "x" + std::to_string(pc), j, i);
        auto col_reduce = [&](double* v, int64_t len) {
            if (len) SLAPCU_NCCL(ncclAllReduce(v, v, size_t(len), ncclDouble, ncclSum, col, c.stream));
            cm->calls[kReduce] += 1;
            cm->bytes[kReduce] += sizeof(double) * len;
        };
        {  // algorithms.cpp:270-275 stochasticity check
            DevBuf sums(sizeof(double) * std::max<int64_t>(A.ncols, 1), c.stream);
            mcl_block_colsums(c, A, sr, sums.as<double>());
            col_reduce(sums.as<double>(), A.ncols);
            int bad = mcl_sums_bad(c, sums.as<double>(), A.ncols, tol) ? 1 : 0;
            DevBuf f(sizeof(int), c.stream);
            SLAPCU_CUDA(cudaMemcpyAsync(f.get(), &bad, sizeof(int), cudaMemcpyHostToDevice, c.stream));
            SLAPCU_NCCL(ncclAllReduce(f.get(), f.get(), 1, ncclInt32, ncclMax, cm->world, c.stream));
            SLAPCU_CUDA(cudaMemcpyAsync(&bad, f.get(), sizeof(int), cudaMemcpyDeviceToHost, c.stream));
            SLAPCU_CUDA(cudaStreamSynchronize(c.stream));
            if (bad) throw Fail{SLAPCU_ERR_STOCHASTIC, "input column sums deviate from 1"};
        }
        slapcu_csc_out E{};
        struct FreeOut {
            Ctx& c;
            slapcu_csc_out& o;
            ~FreeOut() {
                if (o.colptr) cudaFreeAsync(o.colptr, c.stream);
                if (o.rowids) cudaFreeAsync(o.rowids, c.stream);
                if (o.vals) cudaFreeAsync(o.vals, c.stream);
            }
        } free_e{c, E};
        if (layers <= 1) {
            if (pr != pc) throw Fail{SLAPCU_ERR_SHAPE, "2D SUMMA needs a square process grid"};
            const slapcu_status st = slapcu_summa2d(cm, A_local, A_local, sr, SLAPCU_ALG_HYBRID, &E, nullptr);
            if (st != SLAPCU_OK) return st;
        } else {
            const int p = cm->nranks;
            if (p % layers) throw Fail{SLAPCU_ERR_SHAPE, "cannot split ranks into layers"};
            int64_t q = 0;
            if (!is_square(p / layers, &q)) throw Fail{SLAPCU_ERR_SHAPE, "p/c is not a perfect square"};
            const auto ro = block_offsets(m, pr), co = block_offsets(n, pc);
            // regular 3D tilings (dist_matrix3d.hpp:54-80): the split dimension in c slabs of q pieces
            auto tiling3 = [&](bool split_cols, std::vector<int64_t>& rc, std::vector<int64_t>& cc,
                               std::vector<int32_t>& own) {
                const auto slabs = block_offsets(n, layers);
                std::vector<int64_t> cuts;
                for (int l = 0; l < layers; ++l) {
                    const auto sub = block_offsets(slabs[l + 1] - slabs[l], (int)q);
                    for (int x = 0; x < q; ++x) cuts.push_back(slabs[l] + sub[x]);
                }
                cuts.push_back(n);
                const auto other = block_offsets(m, (int)q);
                own.clear();
                if (split_cols) {
                    rc = other;
                    cc = cuts;
                    for (int ii = 0; ii < q; ++ii)
                        for (int lj = 0; lj < layers * q; ++lj)
                            own.push_back((lj / (int)q) * (int)(q * q) + ii * (int)q + lj % (int)q);
                } else {
                    rc = cuts;
                    cc = other;
                    for (int li = 0; li < layers * q; ++li)
                        for (int jj = 0; jj < q; ++jj)
                            own.push_back((li / (int)q) * (int)(q * q) + (li % (int)q) * (int)q + jj);
                }
            };
            std::vector<int64_t> rc1, cc1, rc2, cc2;
            std::vector<int32_t> o1, o2;
            tiling3(true, rc1, cc1, o1);
            tiling3(false, rc2, cc2, o2);
            slapcu_tiling t1{(int)rc1.size() - 1, (int)cc1.size() - 1, rc1.data(), cc1.data(), o1.data()};
            slapcu_tiling t2{(int)rc2.size() - 1, (int)cc2.size() - 1, rc2.data(), cc2.data(), o2.data()};
            slapcu_csc_out A3{}, B3{}, C3{};
            FreeOut fa{c, A3}, fb{c, B3}, fc{c, C3};
            int64_t rs = 0, cs = 0;
            slapcu_status st = slapcu_redistribute(cm, A_local, ro[i], co[j], m, n, sr, &t1, 0, &A3, &rs, &cs);
            if (st != SLAPCU_OK) return st;
            st = slapcu_redistribute(cm, A_local, ro[i], co[j], m, n, sr, &t2, 0, &B3, &rs, &cs);
            if (st != SLAPCU_OK) return st;
            const slapcu_csc a3{A3.nrows, A3.ncols, A3.nnz, A3.colptr, A3.rowids, A3.vals};
            const slapcu_csc b3{B3.nrows, B3.ncols, B3.nnz, B3.colptr, B3.rowids, B3.vals};
            st = slapcu_ca3d(cm, layers, &a3, &b3, sr, SLAPCU_ALG_HYBRID, &C3, nullptr);
            if (st != SLAPCU_OK) return st;
            // C3 is split by columns like A3: this rank's piece of its layer's column block
            const int qq = (int)(q * q), l = cm->rank / qq, i3 = (cm->rank % qq) / (int)q, j3 = cm->rank % (int)q;
            // spgemm3d.hpp:86-90: C3 rows = A3's row block, columns = B3's column
            // block (split rows: n cut into q blocks) cut into c pieces, piece l
            const auto qb = block_offsets(n, (int)q);
            const auto pieces = block_offsets(qb[j3 + 1] - qb[j3], layers);
            const int64_t c3_col = qb[j3] + pieces[l];
            const int64_t c3_row = block_offsets(m, (int)q)[i3];
            std::vector<int32_t> own2d;
            for (int ii = 0; ii < pr; ++ii)
                for (int jj = 0; jj < pc; ++jj) own2d.push_back(ii * pc + jj);
            slapcu_tiling t2d{pr, pc, ro.data(), co.data(), own2d.data()};
            const slapcu_csc c3v{C3.nrows, C3.ncols, C3.nnz, C3.colptr, C3.rowids, C3.vals};
            st = slapcu_redistribute(cm, &c3v, c3_row, c3_col, m, n, sr, &t2d, 0, &E, &rs, &cs);
            if (st != SLAPCU_OK) return st;
        }
        const DevCsc ev{E.nrows, E.ncols, E.nnz, E.colptr, E.rowids, E.vals};
        mcl_block_epilogue(c, ev, sr, inflation, prune_threshold, col_reduce, C_local);
        SLAPCU_CUDA(cudaStreamSynchronize(c.stream));
        return SLAPCU_OK;
    } catch (const Fail& e) {
        c.last_error = e.msg;
        return e.st;
    }
}

slapcu_status slapcu_ca3d(slapcu_comm cm, int layers, const slapcu_csc* A_local, const slapcu_csc* B_local,
                          slapcu_semiring sr, slapcu_alg alg, slapcu_csc_out* C_local, slapcu_dist_stats* stats) {
    if (!cm || !A_local || !B_local || !C_local) return SLAPCU_ERR_INVALID;
    Ctx& c = ctx_of(cm->ctx);
    try {
        SLAPCU_CUDA(cudaSetDevice(c.device));
        const int vs = value_size(sr);
        if (vs == 0) throw Fail{SLAPCU_ERR_INVALID, "unknown semiring"};
        const int p = cm->nranks;
        if (layers < 1 || p % layers != 0)
            throw Fail{SLAPCU_ERR_SHAPE, "cannot split " + std::to_string(p) + " ranks into " + std::to_string(layers) +
                                             " layers"};
        int64_t q = 0;
        if (!is_square(p / layers, &q))
            throw Fail{SLAPCU_ERR_SHAPE, "p/c = " + std::to_string(p / layers) + " is not a perfect square"};
        if (stats) *stats = slapcu_dist_stats{};
        const bool warn = (double)layers > std::cbrt((double)p) + 1e-9;  // spgemm3d.hpp:38-41
        if (stats) stats->layer_warning = warn;
        Timer total;
        SLAPCU_CUDA(cudaEventRecord(total.a, c.stream));
        DevCsc A = view(*A_local), B = view(*B_local);
        resolve(c, A);
        resolve(c, B);
        const int qq = (int)(q * q);
        const int l = cm->rank / qq, i = (cm->rank % qq) / (int)q, j = cm->rank % (int)q;  // grid.cpp:57
        std::vector<int64_t> meta = allgather_meta(cm, c, A, B);
        for (int ii = 0; ii < q; ++ii)
            for (int jj = 0; jj < q; ++jj)
                for (int s = 0; s < q; ++s)
                    if (meta[kMeta * (l * qq + ii * (int)q + s) + MA_C] != meta[kMeta * (l * qq + s * (int)q + jj) + MB_R])
                        throw Fail{SLAPCU_ERR_DIM, "3D SpGEMM stage blocks misaligned on the inner dimension"};
        ncclComm_t row = nullptr, col = nullptr;
        if (q > 1) {
            row = split(cm, "row3d_" + std::to_string(layers), l * (int)q + i, j);
            col = split(cm, "col3d_" + std::to_string(layers), l * (int)q + j, i);
        }
        ncclComm_t fiber = split(cm, "fiber3d_" + std::to_string(layers), i * (int)q + j, l);
        // per-layer SUMMA
        std::vector<Block> partials;
        summa_stages(cm, c, row, col, (int)q, i, j, A, B, sr, alg, meta,
                     [&](int ii, int jj) { return l * qq + ii * (int)q + jj; }, partials, stats);
        Timer mt;
        SLAPCU_CUDA(cudaEventRecord(mt.a, c.stream));
        // C_int: the layer's merged product (a view; owned by partials[0] or cint_out)
        slapcu_csc_out cint_out{};
        DevCsc ci;
        if (partials.size() == 1) {
            ci = partials[0].view();
        } else {
            std::vector<DevCsc> pv;
            for (auto& pp : partials) pv.push_back(pp.view());
            float fm = 0.f;
            if (c.opt.summa_concat)
                fast_merge(c, pv, sr, alg, &cint_out, &fm);
            else
                merge_blocks(c, pv, sr, &cint_out);
            partials.clear();
            ci = DevCsc{cint_out.nrows, cint_out.ncols, cint_out.nnz, cint_out.colptr, cint_out.rowids, cint_out.vals};
        }
        struct FreeOut {
            Ctx& c;
            slapcu_csc_out& o;
            ~FreeOut() {
                if (o.colptr) cudaFreeAsync(o.colptr, c.stream);
                if (o.rowids) cudaFreeAsync(o.rowids, c.stream);
                if (o.vals) cudaFreeAsync(o.vals, c.stream);
            }
        } free_cint{c, cint_out};
        // spgemm3d.hpp:65-79: split C_int's columns into c pieces and exchange
        const int c_ = layers;
        std::vector<int64_t> poff(c_ + 1);
        const int64_t qc = ci.ncols / c_;
        for (int k = 0; k < c_; ++k) poff[k] = int64_t(k) * qc;  // layout.hpp:60-66
        poff[c_] = ci.ncols;
        std::vector<int64_t> hcp(ci.ncols + 1);
        SLAPCU_CUDA(cudaMemcpyAsync(hcp.data(), ci.cp, sizeof(int64_t) * (ci.ncols + 1),
                                    cudaMemcpyDeviceToHost, c.stream));
        SLAPCU_CUDA(cudaStreamSynchronize(c.stream));
        // counts: my nnz per piece, all-gathered over the fiber
        std::vector<int64_t> mine(c_);
        for (int k = 0; k < c_; ++k) mine[k] = hcp[poff[k + 1]] - hcp[poff[k]];
        DevBuf dcnt(sizeof(int64_t) * c_ * (c_ + 1), c.stream);
        SLAPCU_CUDA(cudaMemcpyAsync(dcnt.as<int64_t>() + c_ * c_, mine.data(), sizeof(int64_t) * c_,
                                    cudaMemcpyHostToDevice, c.stream));
        SLAPCU_NCCL(ncclAllGather(dcnt.as<int64_t>() + c_ * c_, dcnt.as<int64_t>(), c_, ncclInt64, fiber, c.stream));
        std::vector<int64_t> allc(c_ * c_);
        SLAPCU_CUDA(cudaMemcpyAsync(allc.data(), dcnt.get(), sizeof(int64_t) * c_ * c_, cudaMemcpyDeviceToHost, c.stream));
        SLAPCU_CUDA(cudaStreamSynchronize(c.stream));
        // rebased colptr of each outgoing piece
        const int64_t my_cols = poff[l + 1] - poff[l];
        std::vector<Block> pieces(c_);
        std::vector<DevBuf> send_cp(c_);
        for (int k = 0; k < c_; ++k) {
            const int64_t nc = poff[k + 1] - poff[k];
            std::vector<int64_t> pc(nc + 1);
            for (int64_t x = 0; x <= nc; ++x) pc[x] = hcp[poff[k] + x] - hcp[poff[k]];
            send_cp[k].reset(sizeof(int64_t) * (nc + 1), c.stream);
            SLAPCU_CUDA(cudaMemcpyAsync(send_cp[k].get(), pc.data(), sizeof(int64_t) * (nc + 1),
                                        cudaMemcpyHostToDevice, c.stream));
            SLAPCU_CUDA(cudaStreamSynchronize(c.stream));
        }
        for (int src = 0; src < c_; ++src) {
            const int64_t nz = allc[src * c_ + l];  // what src sends me
            pieces[src].nrows = ci.nrows;
            pieces[src].ncols = my_cols;
            pieces[src].nnz = nz;
            if (src == l) continue;
            pieces[src].cp.reset(sizeof(int64_t) * (my_cols + 1), c.stream);
            pieces[src].rw.reset(sizeof(int32_t) * std::max<int64_t>(nz, 1), c.stream);
            pieces[src].v.reset(size_t(vs) * std::max<int64_t>(nz, 1), c.stream);
        }
        SLAPCU_NCCL(ncclGroupStart());
        int64_t sent = 0;
        for (int k = 0; k < c_; ++k) {
            if (k == l) continue;
            const int64_t nc = poff[k + 1] - poff[k];
            const int64_t nz = mine[k];
            const int64_t e0 = hcp[poff[k]];
            SLAPCU_NCCL(ncclSend(send_cp[k].get(), size_t(nc + 1), ncclInt64, k, fiber, c.stream));
            if (nz) {
                SLAPCU_NCCL(ncclSend(const_cast<int32_t*>(ci.rw) + e0, size_t(nz), ncclInt32, k, fiber, c.stream));
                SLAPCU_NCCL(ncclSend(static_cast<char*>(const_cast<void*>(ci.v)) + size_t(vs) * e0, size_t(nz) * vs, ncclUint8, k,
                                     fiber, c.stream));
            }
            sent += sizeof(int64_t) * (nc + 1) + (sizeof(int32_t) + vs) * nz;
            const int64_t rz = allc[k * c_ + l];
            SLAPCU_NCCL(ncclRecv(pieces[k].cp.get(), size_t(my_cols + 1), ncclInt64, k, fiber, c.stream));
            if (rz) {
                SLAPCU_NCCL(ncclRecv(pieces[k].rw.get(), size_t(rz), ncclInt32, k, fiber, c.stream));
                SLAPCU_NCCL(ncclRecv(pieces[k].v.get(), size_t(rz) * vs, ncclUint8, k, fiber, c.stream));
            }
        }
        SLAPCU_NCCL(ncclGroupEnd());
        cm->calls[kAlltoallv] += 1;  // one fiber alltoallv (spgemm3d.hpp:78-79)
        cm->bytes[kAlltoallv] += sent;
        // own piece: a view into C_int
        std::vector<DevCsc> pv(c_);
        for (int k = 0; k < c_; ++k) {
            if (k == l)
                pv[k] = DevCsc{ci.nrows, my_cols, mine[l], send_cp[l].as<int64_t>(),
                               const_cast<int32_t*>(ci.rw) + hcp[poff[l]],
                               static_cast<const char*>(ci.v) + size_t(vs) * hcp[poff[l]]};
            else
                pv[k] = pieces[k].view();
        }
        float fm = 0.f;
        if (c.opt.summa_concat)
            fast_merge(c, pv, sr, alg, C_local, &fm);
        else
            merge_blocks(c, pv, sr, C_local);
        SLAPCU_CUDA(cudaEventRecord(mt.b, c.stream));
        SLAPCU_CUDA(cudaEventRecord(total.b, c.stream));
        SLAPCU_CUDA(cudaStreamSynchronize(c.stream));
        if (stats) {
            stats->ms_merge = mt.ms();
            stats->ms_total = total.ms();
            stats->nnz_out = C_local->nnz;
        }
        return SLAPCU_OK;
    } catch (const Fail& e) {
        c.last_error = e.msg;
        return e.st;
    }
}

}  // extern "C"
