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
#pragma once

#include <cstdint>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

#include "slap/error.hpp"
#include "slap/local_matrix.hpp"
#include "slap/semiring.hpp"
#include "slap/spgemm.hpp"
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

}  // namespace slapcu_slap
