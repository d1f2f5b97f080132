// slapcu_slap.hpp -- the reference-side binding: GPU drop-ins for slap's local
// SpGEMM built on the C-ABI of slapcu.h.
//
// A maintainer of the reference adds this header next to slap's own and links
// libslapcu.so; call sites switch from slap::local_spgemm to
// slapcu_slap::local_spgemm with the same arguments (spgemm.hpp:275-280):
//
//     auto c = slapcu_slap::local_spgemm(a, b, slap::PlusTimesF64{}, slap::SpGemmAlg::hybrid, threads);
//
// Contract mirrored from the reference:
//   * AMat / BMat are slap::CscMatrix or slap::DcscMatrix with int32 local
//     indices (SparseColMatrix, local_matrix.hpp:152-159);
//   * DimError on an inner-dimension mismatch (spgemm.hpp:57-64), ShapeError
//     when nnz(C) does not fit the int32 CscMatrix the reference returns
//     (spgemm.hpp:289-292), Error("InternalError") when the numeric count
//     disagrees with the symbolic one (spgemm.hpp:323-324);
//   * output canonical: rows strictly ascending per column, no zero pruning.
// `threads` is accepted for signature parity; all arithmetic runs on the GPU.
//
// Also here (same names and contracts as the reference):
//   estimate_flops / symbolic_nnz            spgemm.hpp:68-88, :118-138
//   summa2d_spgemm(DistSparseMat2D...)       summa.hpp:106-163
//   ca3d_spgemm(DistSparseMat3D...)          spgemm3d.hpp:21-106
//   dist_symbolic_col_nnz / plan_batches_by_budget / batched_spgemm
//                                            batched.hpp:70-170
// The distributed drop-ins are collective like the reference's: every rank
// thread of slap::run_world calls them.  Rank r of the grid drives GPU r
// (one GPU per rank; ShapeError when the grid has more ranks than devices).
// The NCCL communicator is built once per rank thread and grid shape from an
// ncclUniqueId that grid rank 0 broadcasts over the grid's own slap::Comm
// (one generic broadcast in CommCounters); blocks travel as DCSC straight to
// the device (slapcu_dcsc_upload) and every data collective of the product
// then runs on NCCL.
#pragma once

#include <cstdint>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

#include <algorithm>
#include <array>
#include <cmath>
#include <iostream>
#include <map>
#include <utility>

#include "slap/batched.hpp"
#include "slap/comm.hpp"
#include "slap/dist_matrix.hpp"
#include "slap/dist_matrix3d.hpp"
#include "slap/error.hpp"
#include "slap/grid.hpp"
#include "slap/layout.hpp"
#include "slap/local_matrix.hpp"
#include "slap/semiring.hpp"
#include "slap/spgemm.hpp"
#include "slap/spgemm3d.hpp"
#include "slap/summa.hpp"
#include "slapcu.h"

namespace slapcu_slap {

template <class SR>
struct semiring_id;  // only the semirings libslapcu implements compile
template <>
struct semiring_id<slap::PlusTimes<double>> {
    static constexpr slapcu_semiring value = SLAPCU_PLUS_TIMES_F64;
};
template <>
struct semiring_id<slap::PlusTimes<float>> {
    static constexpr slapcu_semiring value = SLAPCU_PLUS_TIMES_F32;
};
template <>
struct semiring_id<slap::PlusTimes<std::int64_t>> {
    static constexpr slapcu_semiring value = SLAPCU_PLUS_TIMES_I64;
};
template <>
struct semiring_id<slap::MinPlus<std::int32_t>> {
    static constexpr slapcu_semiring value = SLAPCU_MIN_PLUS_I32;
};
template <>
struct semiring_id<slap::MinPlus<double>> {
    static constexpr slapcu_semiring value = SLAPCU_MIN_PLUS_F64;
};
template <>
struct semiring_id<slap::OrAnd> {
    static constexpr slapcu_semiring value = SLAPCU_OR_AND_U8;
};

inline slapcu_alg alg_of(slap::SpGemmAlg a) {
    switch (a) {
    case slap::SpGemmAlg::heap: return SLAPCU_ALG_HEAP;
    case slap::SpGemmAlg::hash: return SLAPCU_ALG_HASH;
    default: return SLAPCU_ALG_HYBRID;
    }
}

// status -> the reference's exception kinds (error.hpp:27-36)
inline void raise(slapcu_status st, slapcu_ctx ctx) {
    if (st == SLAPCU_OK) return;
    const std::string msg = ctx ? slapcu_ctx_last_error(ctx) : "";
    switch (st) {
    case SLAPCU_ERR_DIM: throw slap::DimError(msg);
    case SLAPCU_ERR_SHAPE: throw slap::ShapeError(msg);
    case SLAPCU_ERR_NAME: throw slap::NameError(msg);
    case SLAPCU_ERR_BUDGET: throw slap::BudgetError(msg);
    case SLAPCU_ERR_INDEX: throw slap::IndexError(msg);
    default: throw slap::Error(slapcu_status_name(st), msg);
    }
}

// One context per host thread (contexts are stream-ordered, not reentrant).
inline slapcu_ctx thread_context(int device = 0) {
    thread_local slapcu_ctx ctx = nullptr;
    if (!ctx) raise(slapcu_ctx_create(&ctx, device, nullptr), nullptr);
    return ctx;
}

// Host CSC (int64 colptr) view of any slap column matrix.
template <class M, class VT>
struct HostCsc {
    std::vector<std::int64_t> colptr;
    std::vector<std::int32_t> rowids;
    std::vector<VT> vals;
    slapcu_host_csc view{};

    explicit HostCsc(const M& m) {
        colptr.assign(static_cast<std::size_t>(m.ncols()) + 1, 0);
        rowids.reserve(m.nnz());
        vals.reserve(m.nnz());
        m.for_each_col([&](typename M::col_view c) {  // ascending nonempty columns
            colptr[static_cast<std::size_t>(c.col) + 1] = static_cast<std::int64_t>(c.nnz());
            for (std::size_t k = 0; k < c.nnz(); ++k) {
                rowids.push_back(static_cast<std::int32_t>(c.rows[k]));
                vals.push_back(c.vals[k]);
            }
        });
        for (std::size_t j = 0; j + 1 < colptr.size(); ++j) colptr[j + 1] += colptr[j];
        view = slapcu_host_csc{static_cast<std::int64_t>(m.nrows()), static_cast<std::int64_t>(m.ncols()),
                               static_cast<std::int64_t>(rowids.size()), colptr.data(), rowids.data(),
                               vals.data()};
    }
};

/// GPU drop-in for slap::local_spgemm (spgemm.hpp:275-330).
template <slap::SparseColMatrix AMat, slap::SparseColMatrix BMat, slap::SemiringConcept SR>
    requires std::same_as<typename AMat::value_type, typename SR::left_type> &&
             std::same_as<typename BMat::value_type, typename SR::right_type>
slap::CscMatrix<typename AMat::index_type, typename SR::result_type>
local_spgemm(const AMat& a, const BMat& b, const SR&, slap::SpGemmAlg alg = slap::SpGemmAlg::hybrid,
             int threads = 1) {
    (void)threads;
    using IT = typename AMat::index_type;
    using R = typename SR::result_type;
    if (static_cast<std::int64_t>(a.ncols()) != static_cast<std::int64_t>(b.nrows()))
        throw slap::DimError("spgemm inner dims: A is " + std::to_string(static_cast<long long>(a.nrows())) + "x" +
                             std::to_string(static_cast<long long>(a.ncols())) + ", B is " +
                             std::to_string(static_cast<long long>(b.nrows())) + "x" +
                             std::to_string(static_cast<long long>(b.ncols())));
    HostCsc<AMat, typename AMat::value_type> ha(a);
    HostCsc<BMat, typename BMat::value_type> hb(b);
    slapcu_ctx ctx = thread_context();
    slapcu_host_csc hc{};
    raise(slapcu_spgemm_host(ctx, &ha.view, &hb.view, semiring_id<SR>::value, alg_of(alg), &hc), ctx);
    struct Free {
        slapcu_host_csc* p;
        ~Free() { slapcu_host_free(p); }
    } guard{&hc};
    if (hc.nnz > std::numeric_limits<IT>::max())
        throw slap::ShapeError("nnz(C) = " + std::to_string(static_cast<long long>(hc.nnz)) +
                               " exceeds the int32 local index of CscMatrix; use the device API");
    std::vector<IT> colptr(static_cast<std::size_t>(hc.ncols) + 1);
    for (std::size_t j = 0; j < colptr.size(); ++j) colptr[j] = static_cast<IT>(hc.colptr[j]);
    std::vector<IT> rowids(hc.rowids, hc.rowids + hc.nnz);
    const R* v = static_cast<const R*>(hc.vals);
    std::vector<R> vals(v, v + hc.nnz);
    return slap::CscMatrix<IT, R>(static_cast<IT>(hc.nrows), static_cast<IT>(hc.ncols), std::move(colptr),
                                  std::move(rowids), std::move(vals));
}

/// GPU drop-in for slap::estimate_flops (spgemm.hpp:68-88).
template <slap::SparseColMatrix AMat, slap::SparseColMatrix BMat>
slap::SpGemmEstimate estimate_flops(const AMat& a, const BMat& b) {
    if (static_cast<std::int64_t>(a.ncols()) != static_cast<std::int64_t>(b.nrows()))
        throw slap::DimError("spgemm inner dims: A has " + std::to_string(static_cast<long long>(a.ncols())) +
                             " columns, B has " + std::to_string(static_cast<long long>(b.nrows())) + " rows");
    HostCsc<AMat, typename AMat::value_type> ha(a);
    HostCsc<BMat, typename BMat::value_type> hb(b);
    slapcu_ctx ctx = thread_context();
    slap::SpGemmEstimate est;
    est.flops_per_column.assign(static_cast<std::size_t>(b.ncols()), 0);
    raise(slapcu_estimate_flops_host(ctx, &ha.view, &hb.view, est.flops_per_column.data(), &est.total_flops), ctx);
    return est;
}

/// GPU drop-in for slap::symbolic_nnz (spgemm.hpp:118-138).
template <slap::SparseColMatrix AMat, slap::SparseColMatrix BMat>
std::vector<std::int64_t> symbolic_nnz(const AMat& a, const BMat& b, int threads = 1) {
    (void)threads;
    if (static_cast<std::int64_t>(a.ncols()) != static_cast<std::int64_t>(b.nrows()))
        throw slap::DimError("spgemm inner dims: A has " + std::to_string(static_cast<long long>(a.ncols())) +
                             " columns, B has " + std::to_string(static_cast<long long>(b.nrows())) + " rows");
    HostCsc<AMat, typename AMat::value_type> ha(a);
    HostCsc<BMat, typename BMat::value_type> hb(b);
    slapcu_ctx ctx = thread_context();
    std::vector<std::int64_t> counts(static_cast<std::size_t>(b.ncols()), 0);
    raise(slapcu_symbolic_nnz_host(ctx, &ha.view, &hb.view, SLAPCU_ALG_HYBRID, counts.data()), ctx);
    return counts;
}

// ------------------------------------------------------------ distributed

namespace detail {

// Per rank thread: its device context and the NCCL communicators it built,
// keyed by (transport of the world, grid shape tag).
struct RankGpu {
    slapcu_ctx ctx = nullptr;
    int device = -1;
    std::map<std::pair<const void*, std::string>, slapcu_comm> comms;
    ~RankGpu() {
        for (auto& kv : comms) slapcu_comm_destroy(kv.second);
        if (ctx) slapcu_ctx_destroy(ctx);
    }
};

inline RankGpu& rank_gpu() {
    thread_local RankGpu r;
    return r;
}

// The grid communicator `grid_comm` (group rank = grid rank) as an NCCL
// communicator whose rank `nccl_rank` follows the driver's numbering
// (2D: i*q + j, 3D regular: l*q*q + i*q + j).  Collective on first use.
inline std::pair<slapcu_ctx, slapcu_comm> gpu_comm(const slap::Comm& grid_comm, int nccl_rank, const std::string& tag) {
    slap::Comm cm = grid_comm;
    int ndev = 0;
    slapcu_device_count(&ndev);
    if (ndev < 1) throw slap::Error("CudaError", "no CUDA device for the GPU drop-in");
    if (cm.size() > ndev)
        throw slap::ShapeError("GPU SUMMA runs one rank per GPU: grid has " + std::to_string(cm.size()) +
                               " ranks, " + std::to_string(ndev) + " devices");
    RankGpu& r = rank_gpu();
    if (!r.ctx || r.device != cm.rank()) {
        for (auto& kv : r.comms) slapcu_comm_destroy(kv.second);
        r.comms.clear();
        if (r.ctx) slapcu_ctx_destroy(r.ctx);
        r.ctx = nullptr;
        raise(slapcu_ctx_create(&r.ctx, cm.rank(), nullptr), nullptr);
        r.device = cm.rank();
    }
    const auto key = std::make_pair(static_cast<const void*>(&cm.transport()), tag + "/" + std::to_string(cm.size()));
    auto it = r.comms.find(key);
    if (it != r.comms.end()) return {r.ctx, it->second};
    std::vector<unsigned char> id(128, 0);
    if (cm.rank() == 0) raise(slapcu_comm_unique_id(id.data()), nullptr);
    id = cm.broadcast(0, id);
    slapcu_comm comm = nullptr;
    raise(slapcu_comm_create(&comm, r.ctx, nccl_rank, cm.size(), id.data()), r.ctx);
    r.comms[key] = comm;
    return {r.ctx, comm};
}

// A DCSC block on the device (freed by the destructor).
struct DevBlock {
    slapcu_ctx ctx;
    slapcu_csc_out d{};
    template <class VT>
    DevBlock(slapcu_ctx c, const slap::DcscMatrix<slap::LocalIdx, VT>& m, slapcu_semiring sr) : ctx(c) {
        raise(slapcu_dcsc_upload(ctx, m.nrows(), m.ncols(), static_cast<std::int64_t>(m.nzc()), m.jc().data(),
                                 m.cp().data(), m.rowids().data(), m.vals().data(), sr, &d),
              ctx);
    }
    ~DevBlock() { slapcu_csc_free(ctx, &d); }
    slapcu_csc view() const { return slapcu_csc{d.nrows, d.ncols, d.nnz, d.colptr, d.rowids, d.vals}; }
    slapcu_csc window(std::int64_t c0, std::int64_t c1) const {  // columns [c0, c1) (no copy)
        return slapcu_csc{d.nrows, c1 - c0, d.nnz, d.colptr + c0, d.rowids, d.vals};
    }
};

// Device result -> DcscMatrix (block-local indices) and free.
template <class R>
slap::DcscMatrix<slap::LocalIdx, R> take_dcsc(slapcu_ctx ctx, slapcu_csc_out& c, slapcu_semiring sr) {
    struct Free {
        slapcu_ctx ctx;
        slapcu_csc_out& c;
        ~Free() { slapcu_csc_free(ctx, &c); }
    } guard{ctx, c};
    const slapcu_csc v{c.nrows, c.ncols, c.nnz, c.colptr, c.rowids, c.vals};
    slapcu_host_csc h{};
    raise(slapcu_csc_download(ctx, &v, sr, &h), ctx);
    struct FreeH {
        slapcu_host_csc* p;
        ~FreeH() { slapcu_host_free(p); }
    } hguard{&h};
    if (h.nnz > std::numeric_limits<slap::LocalIdx>::max())
        throw slap::ShapeError("block nnz exceeds the local index width");
    std::vector<slap::LocalIdx> jc, cp{0}, rows(h.rowids, h.rowids + h.nnz);
    const R* hv = static_cast<const R*>(h.vals);
    std::vector<R> vals(hv, hv + h.nnz);
    for (std::int64_t j = 0; j < h.ncols; ++j)
        if (h.colptr[j + 1] > h.colptr[j]) {
            jc.push_back(static_cast<slap::LocalIdx>(j));
            cp.push_back(static_cast<slap::LocalIdx>(h.colptr[j + 1]));
        }
    return slap::DcscMatrix<slap::LocalIdx, R>(slap::detail::narrow_dim(h.nrows, "row"),
                                               slap::detail::narrow_dim(h.ncols, "col"), std::move(jc),
                                               std::move(cp), std::move(rows), std::move(vals));
}

template <class VT1, class VT2>
void summa_checks(const slap::DistSparseMat2D<VT1>& a, const slap::DistSparseMat2D<VT2>& b) {  // summa.hpp:112-122
    if (!a.grid.square())
        throw slap::ShapeError("2D SUMMA needs a square process grid, got " + std::to_string(a.grid.pr) + "x" +
                               std::to_string(a.grid.pc));
    if (a.grid.pr != b.grid.pr || a.grid.pc != b.grid.pc) throw slap::ShapeError("SUMMA operands live on different grids");
    if (a.ncols != b.nrows)
        throw slap::DimError("SUMMA inner dims: A is " + std::to_string(static_cast<long long>(a.nrows)) + "x" +
                             std::to_string(static_cast<long long>(a.ncols)) + ", B is " +
                             std::to_string(static_cast<long long>(b.nrows)) + "x" +
                             std::to_string(static_cast<long long>(b.ncols)));
    if (a.col_offsets != b.row_offsets) throw slap::DimError("SUMMA inner block offsets of A and B disagree");
}

}  // namespace detail

/// GPU drop-in for slap::summa2d_spgemm (summa.hpp:106-163): the q stage
/// broadcasts run as ncclBroadcast over NVLink, the local multiply on the GPU.
template <class VT1, class VT2, slap::SemiringConcept SR>
    requires std::same_as<VT1, typename SR::left_type> && std::same_as<VT2, typename SR::right_type>
slap::DistSparseMat2D<typename SR::result_type>
summa2d_spgemm(const slap::DistSparseMat2D<VT1>& a, const slap::DistSparseMat2D<VT2>& b, const SR&,
               slap::SpGemmAlg alg = slap::SpGemmAlg::hybrid, int threads = 1, slap::DistKernelStats* stats = nullptr) {
    (void)threads;
    using R = typename SR::result_type;
    detail::summa_checks(a, b);
    const slapcu_semiring sr = semiring_id<SR>::value;
    auto [ctx, comm] = detail::gpu_comm(a.grid.comm, a.grid.myrow * a.grid.pc + a.grid.mycol, "2d");
    detail::DevBlock da(ctx, a.local, sr), db(ctx, b.local, sr);
    const slapcu_csc av = da.view(), bv = db.view();
    slapcu_csc_out cd{};
    slapcu_dist_stats st{};
    raise(slapcu_summa2d(comm, &av, &bv, sr, alg_of(alg), &cd, &st), ctx);
    slap::DistSparseMat2D<R> c;
    c.grid = a.grid;
    c.nrows = a.nrows;
    c.ncols = b.ncols;
    c.row_offsets = a.row_offsets;
    c.col_offsets = b.col_offsets;
    c.local = detail::take_dcsc<R>(ctx, cd, sr);
    if (stats) {
        stats->stages = a.grid.pr;
        stats->flops = st.flops;
        stats->nnz_out = static_cast<std::int64_t>(c.local.nnz());
    }
    return c;
}

/// GPU drop-in for slap::ca3d_spgemm (spgemm3d.hpp:21-106): per-layer SUMMA
/// on NCCL, the fiber exchange as grouped ncclSend/ncclRecv, the merge on
/// the GPU.  Either conversion variant: NCCL ranks follow the 3D coordinates.
template <class VT1, class VT2, slap::SemiringConcept SR>
    requires std::same_as<VT1, typename SR::left_type> && std::same_as<VT2, typename SR::right_type>
slap::DistSparseMat3D<typename SR::result_type>
ca3d_spgemm(const slap::DistSparseMat3D<VT1>& a3, const slap::DistSparseMat3D<VT2>& b3, const SR&,
            slap::SpGemmAlg alg = slap::SpGemmAlg::hybrid, int threads = 1, slap::DistKernelStats* stats = nullptr) {
    (void)threads;
    using R = typename SR::result_type;
    if (a3.split != slap::SplitDim::cols) throw slap::ShapeError("3D SpGEMM expects A split along columns");
    if (b3.split != slap::SplitDim::rows) throw slap::ShapeError("3D SpGEMM expects B split along rows");
    if (a3.grid.nlayers != b3.grid.nlayers || a3.grid.q != b3.grid.q || a3.grid.variant != b3.grid.variant)
        throw slap::ShapeError("3D SpGEMM operands live on different grids");
    if (a3.ncols != b3.nrows)
        throw slap::DimError("3D SpGEMM inner dims: A has " + std::to_string(static_cast<long long>(a3.ncols)) +
                             " columns, B has " + std::to_string(static_cast<long long>(b3.nrows)) + " rows");
    const int c = a3.grid.nlayers, q = a3.grid.q, p = a3.grid.size();
    const bool warn = static_cast<double>(c) > std::cbrt(static_cast<double>(p)) + 1e-9;
    if (warn && a3.grid.comm.rank() == 0)
        std::cerr << "ca3d_spgemm: layer count " << c << " exceeds cbrt(p) = cbrt(" << p
                  << "); inter-layer exchange may dominate\n";
    const slapcu_semiring sr = semiring_id<SR>::value;
    const int l = a3.grid.mylayer, i = a3.grid.myrow(), j = a3.grid.mycol();
    auto [ctx, comm] = detail::gpu_comm(a3.grid.comm, l * q * q + i * q + j, "3d");
    detail::DevBlock da(ctx, a3.local, sr), db(ctx, b3.local, sr);
    const slapcu_csc av = da.view(), bv = db.view();
    slapcu_csc_out cd{};
    slapcu_dist_stats st{};
    raise(slapcu_ca3d(comm, c, &av, &bv, sr, alg_of(alg), &cd, &st), ctx);
    auto piece_off = slap::block_offsets(b3.col_len, c);
    slap::DistSparseMat3D<R> c3;
    c3.grid = a3.grid;
    c3.split = slap::SplitDim::cols;
    c3.nrows = a3.nrows;
    c3.ncols = b3.ncols;
    c3.row_start = a3.row_start;
    c3.row_len = a3.row_len;
    c3.col_start = b3.col_start + piece_off[static_cast<std::size_t>(l)];
    c3.col_len = piece_off[static_cast<std::size_t>(l) + 1] - piece_off[static_cast<std::size_t>(l)];
    c3.local = detail::take_dcsc<R>(ctx, cd, sr);
    if (stats) {
        stats->stages = q;
        stats->flops = st.flops;
        stats->nnz_out = static_cast<std::int64_t>(c3.local.nnz());
        stats->layer_warning = warn;
    }
    return c3;
}

/// GPU drop-in for slap::dist_symbolic_col_nnz (batched.hpp:70-117).
template <class VT1, class VT2>
std::vector<std::int64_t> dist_symbolic_col_nnz(const slap::DistSparseMat2D<VT1>& a, const slap::DistSparseMat2D<VT2>& b,
                                                int threads = 1) {
    (void)threads;
    detail::summa_checks(a, b);
    auto [ctx, comm] = detail::gpu_comm(a.grid.comm, a.grid.myrow * a.grid.pc + a.grid.mycol, "2d");
    // the pattern is all that is read; values go up as the operand's own type
    const slapcu_semiring s1 = semiring_id<slap::OrAnd>::value;
    auto pat = [](const auto& m) {  // the block's pattern with 1-byte values
        std::vector<std::uint8_t> ones(m.nnz(), 1);
        return slap::DcscMatrix<slap::LocalIdx, std::uint8_t>(m.nrows(), m.ncols(), m.jc(), m.cp(), m.rowids(),
                                                               std::move(ones));
    };
    detail::DevBlock da(ctx, pat(a.local), s1), db(ctx, pat(b.local), s1);
    const slapcu_csc av = da.view(), bv = db.view();
    std::vector<std::int64_t> counts(static_cast<std::size_t>(b.ncols), 0);
    raise(slapcu_dist_symbolic_col_nnz(comm, &av, &bv, counts.data(), b.ncols), ctx);
    return counts;
}

/// GPU drop-in for slap::plan_batches_by_budget (batched.hpp:122-148).
template <class VT1, class VT2>
slap::BatchPlan plan_batches_by_budget(const slap::DistSparseMat2D<VT1>& a, const slap::DistSparseMat2D<VT2>& b,
                                       std::int64_t budget_bytes, int threads = 1) {
    if (budget_bytes <= 0) throw slap::BudgetError("memory budget must be positive");
    auto counts = slapcu_slap::dist_symbolic_col_nnz(a, b, threads);
    const std::int64_t per_entry = slap::kBatchEntryBytes;
    slap::BatchPlan plan;
    slap::GlobalIdx start = 0;
    std::int64_t cur = 0;
    for (slap::GlobalIdx j = 0; j < static_cast<slap::GlobalIdx>(counts.size()); ++j) {
        const std::int64_t cost = counts[static_cast<std::size_t>(j)] * per_entry;
        if (cost > budget_bytes)
            throw slap::BudgetError("output column " + std::to_string(static_cast<long long>(j)) + " alone needs " +
                                    std::to_string(static_cast<long long>(cost)) + " bytes, budget is " +
                                    std::to_string(static_cast<long long>(budget_bytes)));
        if (cur + cost > budget_bytes) {
            plan.col_ranges.emplace_back(start, j);
            plan.est_entries.push_back(cur / per_entry);
            start = j;
            cur = 0;
        }
        cur += cost;
    }
    plan.col_ranges.emplace_back(start, static_cast<slap::GlobalIdx>(counts.size()));
    plan.est_entries.push_back(cur / per_entry);
    return plan;
}

/// GPU drop-in for slap::batched_spgemm (batched.hpp:153-170): A and B's
/// blocks go to the device once; batch r's B slice is a column window of the
/// device block (no slice_cols copy), multiplied by the GPU SUMMA, and the
/// consumer gets (r, s, e, C_r) with C_r laid out like slice_cols(b, s, e)
/// would lay it out.
template <class VT1, class VT2, slap::SemiringConcept SR, class Consumer>
    requires std::same_as<VT1, typename SR::left_type> && std::same_as<VT2, typename SR::right_type>
void batched_spgemm(const slap::DistSparseMat2D<VT1>& a, const slap::DistSparseMat2D<VT2>& b, const slap::BatchPlan& plan,
                    const SR&, slap::SpGemmAlg alg, int threads, Consumer&& consumer) {
    (void)threads;
    using R = typename SR::result_type;
    if (plan.batches() < 1) throw slap::ShapeError("batch plan is empty");
    slap::GlobalIdx expect = 0;
    for (const auto& [s, e] : plan.col_ranges) {
        if (s != expect || e < s) throw slap::ShapeError("batch ranges must partition B's columns in order");
        expect = e;
    }
    if (expect != b.ncols) throw slap::ShapeError("batch ranges must cover all columns of B");
    detail::summa_checks(a, b);
    const slapcu_semiring sr = semiring_id<SR>::value;
    auto [ctx, comm] = detail::gpu_comm(a.grid.comm, a.grid.myrow * a.grid.pc + a.grid.mycol, "2d");
    detail::DevBlock da(ctx, a.local, sr), db(ctx, b.local, sr);
    const slapcu_csc av = da.view();
    const slap::GlobalIdx cs = b.col_start(), ce = b.col_end();
    for (int r = 0; r < plan.batches(); ++r) {
        const auto [s, e] = plan.col_ranges[static_cast<std::size_t>(r)];
        // this rank's block of the slice: global columns [max(cs, s), min(ce, e)),
        // empty (a zero-width window at the block's edge) when the range misses it
        const slap::GlobalIdx w0 = std::clamp<slap::GlobalIdx>(s - cs, 0, ce - cs);
        const slap::GlobalIdx w1 = std::clamp<slap::GlobalIdx>(e - cs, w0, ce - cs);
        const slapcu_csc bv = db.window(w0, w1);
        slapcu_csc_out cd{};
        slapcu_dist_stats st{};
        raise(slapcu_summa2d(comm, &av, &bv, sr, alg_of(alg), &cd, &st), ctx);
        slap::DistSparseMat2D<R> cr;
        cr.grid = a.grid;
        cr.nrows = a.nrows;
        cr.ncols = e - s;
        cr.row_offsets = a.row_offsets;
        cr.col_offsets.resize(b.col_offsets.size());
        for (std::size_t i = 0; i < b.col_offsets.size(); ++i)
            cr.col_offsets[i] = std::min(std::max(b.col_offsets[i], s), e) - s;
        cr.local = detail::take_dcsc<R>(ctx, cd, sr);
        consumer(r, s, e, cr);
    }
}

}  // namespace slapcu_slap
