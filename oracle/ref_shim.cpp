// ref_shim.cpp -- C entry points over the UNMODIFIED reference library
// (/root/reference/proj/core), compiled in place by oracle/Makefile into
// oracle/_ref/libslapref.so.  TEST INFRASTRUCTURE ONLY: used to pin the C
// restatement (oracle.c), to generate tests/golden fixtures, and as the timed
// CPU baseline ("kind": "reference") in bench.py.  No reference source is
// copied into this repository; this file only calls the reference's public
// templates.
//
// Layout at this boundary: CSC with int64 colptr / int32 rowids, like the
// device library.  The reference's own local index type is int32
// (dist_matrix.hpp:18, spgemm.hpp:281), so inputs are narrowed on entry and the
// call fails with -5 when nnz(C) >= 2^31 would overflow its colptr.

#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <limits>
#include <type_traits>
#include <vector>

#include "slap/algorithms.hpp"
#include "slap/batched.hpp"
#include "slap/binary_io.hpp"
#include "slap/spgemm.hpp"
#include "slap/spgemm3d.hpp"
#include "slap/summa.hpp"

using namespace slap;
using I = std::int32_t;

extern "C" {
typedef struct {
    int64_t nrows, ncols, nnz;
    int64_t* colptr;
    int32_t* rowids;
    void* vals;
} ref_csc;
}

namespace {

template <class VT>
CscMatrix<I, VT> to_ref_csc(const ref_csc& m) {
    std::vector<I> cp(static_cast<std::size_t>(m.ncols) + 1);
    for (int64_t j = 0; j <= m.ncols; ++j) cp[static_cast<std::size_t>(j)] = static_cast<I>(m.colptr[j]);
    std::vector<I> rows(m.rowids, m.rowids + m.nnz);
    std::vector<VT> vals(static_cast<std::size_t>(m.nnz));
    if (m.nnz) std::memcpy(vals.data(), m.vals, sizeof(VT) * static_cast<std::size_t>(m.nnz));
    return CscMatrix<I, VT>(static_cast<I>(m.nrows), static_cast<I>(m.ncols), std::move(cp), std::move(rows),
                            std::move(vals));
}

template <class VT>
Triples<GlobalIdx, VT> to_triples64(const ref_csc& m) {
    Triples<GlobalIdx, VT> t;
    t.nrows = m.nrows;
    t.ncols = m.ncols;
    const VT* v = static_cast<const VT*>(m.vals);
    for (int64_t j = 0; j < m.ncols; ++j)
        for (int64_t p = m.colptr[j]; p < m.colptr[j + 1]; ++p) t.push_back(m.rowids[p], j, v[p]);
    return t;
}

template <class VT>
void from_triples64(const Triples<GlobalIdx, VT>& t, ref_csc* out) {
    out->nrows = t.nrows;
    out->ncols = t.ncols;
    out->nnz = static_cast<int64_t>(t.size());
    out->colptr = static_cast<int64_t*>(std::calloc(static_cast<std::size_t>(t.ncols) + 1, sizeof(int64_t)));
    out->rowids = static_cast<int32_t*>(std::malloc(sizeof(int32_t) * (t.size() ? t.size() : 1)));
    out->vals = std::malloc(sizeof(VT) * (t.size() ? t.size() : 1));
    VT* ov = static_cast<VT*>(out->vals);
    for (std::size_t e = 0; e < t.size(); ++e) {  // gather_matrix output is (col,row)-sorted
        out->colptr[t.cols[e] + 1]++;
        out->rowids[e] = static_cast<int32_t>(t.rows[e]);
        ov[e] = t.vals[e];
    }
    for (int64_t j = 0; j < t.ncols; ++j) out->colptr[j + 1] += out->colptr[j];
}

template <class IT, class VT>
void from_csc(const CscMatrix<IT, VT>& c, ref_csc* out) {
    out->nrows = c.nrows();
    out->ncols = c.ncols();
    out->nnz = static_cast<int64_t>(c.nnz());
    out->colptr = static_cast<int64_t*>(std::malloc(sizeof(int64_t) * (static_cast<std::size_t>(c.ncols()) + 1)));
    for (std::size_t j = 0; j <= static_cast<std::size_t>(c.ncols()); ++j) out->colptr[j] = c.colptr()[j];
    out->rowids = static_cast<int32_t*>(std::malloc(sizeof(int32_t) * (c.nnz() ? c.nnz() : 1)));
    out->vals = std::malloc(sizeof(VT) * (c.nnz() ? c.nnz() : 1));
    if (c.nnz()) {
        std::memcpy(out->rowids, c.rowids().data(), sizeof(int32_t) * c.nnz());
        std::memcpy(out->vals, c.vals().data(), sizeof(VT) * c.nnz());
    }
}

CscMatrix<I, std::uint8_t> pattern_csc(const ref_csc& m) {
    std::vector<I> cp(static_cast<std::size_t>(m.ncols) + 1);
    for (int64_t j = 0; j <= m.ncols; ++j) cp[static_cast<std::size_t>(j)] = static_cast<I>(m.colptr[j]);
    return CscMatrix<I, std::uint8_t>(static_cast<I>(m.nrows), static_cast<I>(m.ncols), std::move(cp),
                                      std::vector<I>(m.rowids, m.rowids + m.nnz),
                                      std::vector<std::uint8_t>(static_cast<std::size_t>(m.nnz), 1));
}

// Same pattern with a value array of ones (owned by a static buffer per call).
ref_csc ones_view(const ref_csc& m) {
    static thread_local std::vector<std::uint8_t> ones;
    ones.assign(static_cast<std::size_t>(m.nnz) + 1, 1);
    ref_csc v = m;
    v.vals = ones.data();
    return v;
}

// Semiring ids follow include/slapcu.h.
template <class F>
int with_semiring(int sr, F&& f) {
    switch (sr) {
    case 0: return f(PlusTimes<double>{});
    case 1: return f(PlusTimes<float>{});
    case 2: return f(PlusTimes<std::int64_t>{});
    case 3: return f(MinPlus<std::int32_t>{});
    case 4: return f(MinPlus<double>{});
    case 5: return f(OrAnd{});
    }
    return -3;
}

SpGemmAlg alg_of(int a) { return a == 0 ? SpGemmAlg::heap : a == 1 ? SpGemmAlg::hash : SpGemmAlg::hybrid; }

int error_code(const std::exception& e) {
    if (const auto* err = dynamic_cast<const Error*>(&e)) {
        if (err->kind() == "DimError") return -2;
        if (err->kind() == "ShapeError") return -6;
        if (err->kind() == "BudgetError") return -7;
        if (err->kind() == "InternalError") return -4;
        if (err->kind() == "StochasticityError") return -8;
    }
    return -1;
}


// Block-local CSC of a DCSC / CSC local block (for_each_col order).
template <class M>
void from_local(const M& m, int64_t nrows, int64_t ncols, ref_csc* out) {
    using VT = std::remove_cv_t<std::remove_reference_t<decltype(m.vals()[0])>>;
    out->nrows = nrows;
    out->ncols = ncols;
    out->nnz = static_cast<int64_t>(m.nnz());
    out->colptr = static_cast<int64_t*>(std::calloc(static_cast<std::size_t>(ncols) + 1, sizeof(int64_t)));
    out->rowids = static_cast<int32_t*>(std::malloc(sizeof(int32_t) * (m.nnz() ? m.nnz() : 1)));
    out->vals = std::malloc(sizeof(VT) * (m.nnz() ? m.nnz() : 1));
    VT* ov = static_cast<VT*>(out->vals);
    int64_t e = 0;
    m.for_each_col([&](auto cv) {
        out->colptr[cv.col + 1] = static_cast<int64_t>(cv.nnz());
        for (std::size_t k = 0; k < cv.nnz(); ++k, ++e) {
            out->rowids[e] = cv.rows[k];
            ov[e] = cv.vals[k];
        }
    });
    for (int64_t j = 0; j < ncols; ++j) out->colptr[j + 1] += out->colptr[j];
}

}  // namespace

extern "C" {

void ref_free(void* p) { std::free(p); }

/// spgemm.hpp:275-330 local_spgemm(a, b, sr, alg, threads) on CSC x CSC
/// (b_dcsc != 0 builds B as DcscMatrix like the SUMMA blocks).
int ref_local_spgemm(int sr, int alg, int threads, const ref_csc* a, const ref_csc* b, int b_dcsc, ref_csc* c) {
    try {
        return with_semiring(sr, [&](auto s) -> int {
            using VT = typename decltype(s)::left_type;
            auto am = to_ref_csc<VT>(*a);
            auto bm = to_ref_csc<VT>(*b);
            auto sym = symbolic_nnz(am, bm, threads);
            std::int64_t total = 0;
            for (auto v : sym) total += v;
            if (total > std::numeric_limits<I>::max()) return -5;  // int32 colptr overflow (spgemm.hpp:289-292)
            if (b_dcsc) {
                auto bd = csc_to_dcsc(bm);
                from_csc(local_spgemm(am, bd, s, alg_of(alg), threads), c);
            } else {
                from_csc(local_spgemm(am, bm, s, alg_of(alg), threads), c);
            }
            return 0;
        });
    } catch (const std::exception& e) {
        return error_code(e);
    }
}

/// Timed reference run for the CPU baseline: converts A and the column range
/// [c0, c1) of B into the reference's CscMatrix OUTSIDE the timed region, then
/// times exactly one slap::local_spgemm call (spgemm.hpp:275-330) with
/// `threads` worker threads.  Returns 0 and writes seconds, output nnz and the
/// multiply count (estimate_flops) of the slice; -5 if nnz(C) would overflow
/// the reference's int32 colptr.  When `c` is non-null the slice's product
/// C(:, c0:c1) is returned too (converted after the timed region), so the
/// benchmark checks the GPU output of the same columns against it.
int ref_time_local_spgemm(int sr, int alg, int threads, const ref_csc* a, const ref_csc* b, int64_t c0, int64_t c1,
                          double* seconds, int64_t* nnz_out, int64_t* flops_out, ref_csc* c) {
    try {
        return with_semiring(sr, [&](auto s) -> int {
            using VT = typename decltype(s)::left_type;
            auto am = to_ref_csc<VT>(*a);
            ref_csc bs{b->nrows, c1 - c0, b->colptr[c1] - b->colptr[c0], nullptr,
                       b->rowids + b->colptr[c0], static_cast<const VT*>(b->vals) ? const_cast<VT*>(static_cast<const VT*>(b->vals)) + b->colptr[c0] : nullptr};
            std::vector<int64_t> cp(static_cast<std::size_t>(c1 - c0) + 1);
            for (int64_t j = c0; j <= c1; ++j) cp[static_cast<std::size_t>(j - c0)] = b->colptr[j] - b->colptr[c0];
            bs.colptr = cp.data();
            auto bm = to_ref_csc<VT>(bs);
            auto est = estimate_flops(am, bm);
            auto sym = symbolic_nnz(am, bm, threads);
            std::int64_t total = 0;
            for (auto v : sym) total += v;
            if (total > std::numeric_limits<I>::max()) return -5;
            const auto t0 = std::chrono::steady_clock::now();
            auto cm = local_spgemm(am, bm, s, alg_of(alg), threads);
            const auto t1 = std::chrono::steady_clock::now();
            *seconds = std::chrono::duration<double>(t1 - t0).count();
            *nnz_out = static_cast<int64_t>(cm.nnz());
            *flops_out = est.total_flops;
            if (c) from_csc(cm, c);
            return 0;
        });
    } catch (const std::exception& e) {
        return error_code(e);
    }
}

/// spgemm.hpp:68-88
int64_t ref_estimate_flops(const ref_csc* a, const ref_csc* b, int64_t* per_col) {
    try {
        auto A = pattern_csc(*a);
        auto B = pattern_csc(*b);
        auto est = estimate_flops(A, B);
        if (per_col)
            for (std::size_t j = 0; j < est.flops_per_column.size(); ++j) per_col[j] = est.flops_per_column[j];
        return est.total_flops;
    } catch (const std::exception& e) {
        return error_code(e);
    }
}

/// spgemm.hpp:118-138
int ref_symbolic_nnz(const ref_csc* a, const ref_csc* b, int threads, int64_t* counts) {
    try {
        auto A = pattern_csc(*a);
        auto B = pattern_csc(*b);
        auto s = symbolic_nnz(A, B, threads);
        for (std::size_t j = 0; j < s.size(); ++j) counts[j] = s[j];
        return 0;
    } catch (const std::exception& e) {
        return error_code(e);
    }
}

/// algorithms.cpp:71-113 gen_rmat on a 1x1 grid (pattern; values are 1.0).
int ref_gen_rmat(int scale, int edge_factor, uint64_t seed, ref_csc* out) {
    try {
        int rc = 0;
        run_world(1, [&](Comm& w) {
            auto g = make_grid2d(w, 1, 1);
            RmatParams p;
            p.scale = scale;
            p.edge_factor = edge_factor;
            p.seed = seed;
            auto m = gen_rmat(p, g);
            auto csc = dcsc_to_csc(m.local);
            from_csc(csc, out);
            std::free(out->vals);
            out->vals = nullptr;
        });
        return rc;
    } catch (const std::exception& e) {
        return error_code(e);
    }
}

/// algorithms.cpp:267-293 mcl_step (expansion A*A in PlusTimes<double>,
/// inflation pow, prune below the threshold, column renormalisation) on a
/// sqrt(p) x sqrt(p) grid of rank threads (layers > 1: the 3D expansion).
int ref_mcl_step(int p, int layers, const ref_csc* a, double inflation, double prune, ref_csc* c) {
    try {
        auto ta = to_triples64<double>(*a);
        run_world(p, [&](Comm& w) {
            auto g = make_square_grid2d(w);
            auto first = [](const double& x, const double&) { return x; };
            Triples<GlobalIdx, double> ma;
            ma.nrows = ta.nrows;
            ma.ncols = ta.ncols;
            if (w.rank() == 0) ma = ta;
            auto da = distribute_triples(ma, g, ta.nrows, ta.ncols, first);
            MclOptions opt;
            opt.inflation = inflation;
            opt.prune_threshold = prune;
            opt.layers = layers;
            auto dc = mcl_step(da, opt);
            auto got = gather_matrix(dc);
            if (w.rank() == 0) from_triples64(got, c);
        });
        return 0;
    } catch (const std::exception& e) {
        return error_code(e);
    }
}

/// summa.hpp:106-163 summa2d_spgemm on a sqrt(p) x sqrt(p) grid of rank threads
/// (comm.cpp:135-175 run_world).  Inputs/outputs are global CSC.
int ref_summa2d(int sr, int alg, int p, int threads, const ref_csc* a, const ref_csc* b, ref_csc* c,
                int64_t* stage_count, int64_t* bcast_calls) {
    try {
        return with_semiring(sr, [&](auto s) -> int {
            using VT = typename decltype(s)::left_type;
            auto ta = to_triples64<VT>(*a);
            auto tb = to_triples64<VT>(*b);
            auto counters = run_world(p, [&](Comm& w) {
                auto g = make_square_grid2d(w);
                auto first = [](const VT& x, const VT&) { return x; };
                Triples<GlobalIdx, VT> ma, mb;
                ma.nrows = ta.nrows;
                ma.ncols = ta.ncols;
                mb.nrows = tb.nrows;
                mb.ncols = tb.ncols;
                if (w.rank() == 0) {
                    ma = ta;
                    mb = tb;
                }
                auto da = distribute_triples(ma, g, ta.nrows, ta.ncols, first);
                auto db = distribute_triples(mb, g, tb.nrows, tb.ncols, first);
                DistKernelStats st;
                auto dc = summa2d_spgemm(da, db, s, alg_of(alg), threads, &st);
                auto got = gather_matrix(dc);
                if (w.rank() == 0) {
                    from_triples64(got, c);
                    if (stage_count) *stage_count = st.stages;
                }
            });
            if (bcast_calls) *bcast_calls = counters[0].kind(Coll::broadcast).calls;
            return 0;
        });
    } catch (const std::exception& e) {
        return error_code(e);
    }
}

/// spgemm3d.hpp:21-106 ca3d_spgemm with layers c on p ranks (regular variant);
/// inputs are distributed on a 2D grid (pr x pc) and redistributed
/// (dist_matrix3d.hpp:117-219) exactly as acceptance.cpp:140-160 does.
int ref_ca3d(int sr, int alg, int p, int pr, int pc, int layers, int threads, const ref_csc* a, const ref_csc* b,
             ref_csc* c) {
    try {
        return with_semiring(sr, [&](auto s) -> int {
            using VT = typename decltype(s)::left_type;
            auto ta = to_triples64<VT>(*a);
            auto tb = to_triples64<VT>(*b);
            run_world(p, [&](Comm& w) {
                auto g = make_grid2d(w, pr, pc);
                auto first = [](const VT& x, const VT&) { return x; };
                Triples<GlobalIdx, VT> ma, mb;
                ma.nrows = ta.nrows;
                ma.ncols = ta.ncols;
                mb.nrows = tb.nrows;
                mb.ncols = tb.ncols;
                if (w.rank() == 0) {
                    ma = ta;
                    mb = tb;
                }
                auto da = distribute_triples(ma, g, ta.nrows, ta.ncols, first);
                auto db = distribute_triples(mb, g, tb.nrows, tb.ncols, first);
                auto g3 = make_grid3d(w, layers);
                auto c3 = ca3d_spgemm(redistribute_3d(da, g3, SplitDim::cols), redistribute_3d(db, g3, SplitDim::rows),
                                      s, alg_of(alg), threads);
                auto got = gather_matrix(c3);
                if (w.rank() == 0) from_triples64(got, c);
            });
            return 0;
        });
    } catch (const std::exception& e) {
        return error_code(e);
    }
}

/// batched.hpp:122-148 plan_batches_by_budget on a sqrt(p) x sqrt(p) grid;
/// writes up to max_ranges [start,end) pairs and the per-range entry
/// estimates, returns the number of ranges (or < 0 on error).
int ref_plan_batches(int p, int threads, const ref_csc* a, const ref_csc* b, int64_t budget, int64_t* ranges,
                     int64_t* est_entries, int max_ranges) {
    try {
        auto ta = to_triples64<std::uint8_t>(ones_view(*a));
        auto tb = to_triples64<std::uint8_t>(ones_view(*b));
        int nr = 0;
        run_world(p, [&](Comm& w) {
            auto g = make_square_grid2d(w);
            auto first = [](const std::uint8_t& x, const std::uint8_t&) { return x; };
            Triples<GlobalIdx, std::uint8_t> ma, mb;
            ma.nrows = ta.nrows;
            ma.ncols = ta.ncols;
            mb.nrows = tb.nrows;
            mb.ncols = tb.ncols;
            if (w.rank() == 0) {
                ma = ta;
                mb = tb;
            }
            auto da = distribute_triples(ma, g, ta.nrows, ta.ncols, first);
            auto db = distribute_triples(mb, g, tb.nrows, tb.ncols, first);
            auto plan = plan_batches_by_budget(da, db, budget, threads);
            if (w.rank() == 0) {
                nr = plan.batches();
                for (int r = 0; r < nr && r < max_ranges; ++r) {
                    ranges[2 * r] = plan.col_ranges[static_cast<std::size_t>(r)].first;
                    ranges[2 * r + 1] = plan.col_ranges[static_cast<std::size_t>(r)].second;
                    est_entries[r] = plan.est_entries[static_cast<std::size_t>(r)];
                }
            }
        });
        return nr;
    } catch (const std::exception& e) {
        return error_code(e);
    }
}

/// local_matrix.hpp:166-188 build_csc over parts appended in order (the SUMMA
/// merge, summa.hpp:145-156).
int ref_merge(int sr, int nparts, const ref_csc* parts, ref_csc* out) {
    try {
        return with_semiring(sr, [&](auto s) -> int {
            using VT = typename decltype(s)::left_type;
            Triples<I, VT> t;
            t.nrows = static_cast<I>(parts[0].nrows);
            t.ncols = static_cast<I>(parts[0].ncols);
            for (int q = 0; q < nparts; ++q) {
                const VT* v = static_cast<const VT*>(parts[q].vals);
                for (int64_t j = 0; j < parts[q].ncols; ++j)
                    for (int64_t e = parts[q].colptr[j]; e < parts[q].colptr[j + 1]; ++e)
                        t.push_back(parts[q].rowids[e], static_cast<I>(j), v[e]);
            }
            auto csc = build_csc(t, [&](const VT& x, const VT& y) { return s.add(x, y); });
            from_csc(csc, out);
            return 0;
        });
    } catch (const std::exception& e) {
        return error_code(e);
    }
}

/// distribute_triples (dist_matrix.hpp:89-119) of triples held by source
/// ranks src[k] onto a pr x pc grid, duplicates combined keep-first
/// (combine 0) or with the semiring add (1); mode 1 continues with
/// redistribute_3d(layers, split) (dist_matrix3d.hpp:117-170, regular), mode
/// 2 with redistribute_2d back to the pr x pc grid (:250-261).  Rank r's
/// resulting local block goes to blocks[r] (block-local CSC) with its global
/// offsets.
int ref_redistribute(int sr, int p, int pr, int pc, int mode, int layers, int split_rows, int combine,
                     int64_t nrows, int64_t ncols, int64_t n, const int32_t* src, const int64_t* rows,
                     const int64_t* cols, const void* vals, ref_csc* blocks, int64_t* row_start, int64_t* col_start) {
    try {
        return with_semiring(sr, [&](auto s) -> int {
            using VT = typename decltype(s)::left_type;
            const VT* v = static_cast<const VT*>(vals);
            run_world(p, [&](Comm& w) {
                Triples<GlobalIdx, VT> mine;
                mine.nrows = nrows;
                mine.ncols = ncols;
                for (int64_t k = 0; k < n; ++k)
                    if (src[k] == w.rank()) mine.push_back(rows[k], cols[k], v[k]);
                auto g = make_grid2d(w, pr, pc);
                auto first = [](const VT& x, const VT&) { return x; };
                auto add = [&](const VT& x, const VT& y) { return static_cast<VT>(s.add(x, y)); };
                auto d2 = combine ? distribute_triples(mine, g, nrows, ncols, add)
                                  : distribute_triples(mine, g, nrows, ncols, first);
                const int r = w.rank();
                if (mode == 0) {
                    from_local(d2.local, d2.row_end() - d2.row_start(), d2.col_end() - d2.col_start(), &blocks[r]);
                    row_start[r] = d2.row_start();
                    col_start[r] = d2.col_start();
                    return;
                }
                auto g3 = make_grid3d(w, layers);
                auto d3 = redistribute_3d(d2, g3, split_rows ? SplitDim::rows : SplitDim::cols);
                if (mode == 1) {
                    from_local(d3.local, d3.row_len, d3.col_len, &blocks[r]);
                    row_start[r] = d3.row_start;
                    col_start[r] = d3.col_start;
                    return;
                }
                auto b2 = redistribute_2d(d3, g);
                from_local(b2.local, b2.row_end() - b2.row_start(), b2.col_end() - b2.col_start(), &blocks[r]);
                row_start[r] = b2.row_start();
                col_start[r] = b2.col_start();
            });
            return 0;
        });
    } catch (const std::exception& e) {
        return error_code(e);
    }
}

/// write_binary (binary_io.cpp) of the global f64 matrix `a` distributed by
/// distribute_triples onto pr x pc rank threads.
int ref_write_binary(int p, int pr, int pc, const ref_csc* a, const char* path) {
    try {
        auto t = to_triples64<double>(*a);
        run_world(p, [&](Comm& w) {
            auto g = make_grid2d(w, pr, pc);
            Triples<GlobalIdx, double> mine;
            mine.nrows = t.nrows;
            mine.ncols = t.ncols;
            if (w.rank() == 0) mine = t;
            auto first = [](const double& x, const double&) { return x; };
            write_binary(distribute_triples(mine, g, t.nrows, t.ncols, first), path);
        });
        return 0;
    } catch (const std::exception& e) {
        if (const auto* err = dynamic_cast<const Error*>(&e)) {
            if (err->kind() == "IoError") return -9;
            if (err->kind() == "FormatError") return -10;
        }
        return error_code(e);
    }
}

/// read_binary (binary_io.cpp) onto pr x pc rank threads; rank r's block to
/// blocks[r] with its global offsets.
int ref_read_binary(const char* path, int p, int pr, int pc, ref_csc* blocks, int64_t* row_start, int64_t* col_start) {
    try {
        run_world(p, [&](Comm& w) {
            auto g = make_grid2d(w, pr, pc);
            auto d = read_binary(path, g);
            const int r = w.rank();
            from_local(d.local, d.row_end() - d.row_start(), d.col_end() - d.col_start(), &blocks[r]);
            row_start[r] = d.row_start();
            col_start[r] = d.col_start();
        });
        return 0;
    } catch (const std::exception& e) {
        if (const auto* err = dynamic_cast<const Error*>(&e)) {
            if (err->kind() == "IoError") return -9;
            if (err->kind() == "FormatError") return -10;
        }
        return error_code(e);
    }
}

}  // extern "C"
