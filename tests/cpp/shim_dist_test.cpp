// Drop-in check of the distributed and phase drop-ins of include/slapcu_slap.hpp:
// the same collective call sites with the reference's templates (CPU, the
// simulated transport) and with slapcu_slap:: (GPU + NCCL) inside one
// slap::run_world, compared on rank 0 after gather_matrix -- bit-exact for
// PlusTimes<int64> / OrAnd / MinPlus<int32>, rel 1e-12 for PlusTimes<double>
// (acceptance.cpp:49-54; the SUMMA fold order differs, summa.hpp:156).
//   estimate_flops / symbolic_nnz      spgemm.hpp:68-88, :118-138
//   summa2d_spgemm                     summa.hpp:106-163 (p = 1, 4)
//   ca3d_spgemm                        spgemm3d.hpp:21-106 (c x 1 x 1 for p = 1, 2, 4)
//   dist_symbolic_col_nnz, plan_batches_by_budget, batched_spgemm  batched.hpp:70-170
// p is limited to the visible GPUs (one rank per GPU).  Prints SHIM_DIST_OK.
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "slap/rng.hpp"
#include "slap/triples.hpp"
#include "slapcu_slap.hpp"

using namespace slap;

template <class VT, class Val>
Triples<GlobalIdx, VT> random_global(Rng& rng, GlobalIdx m, GlobalIdx n, double density, Val val) {
    Triples<GlobalIdx, VT> t;
    t.nrows = m;
    t.ncols = n;
    const auto target = static_cast<std::int64_t>(density * static_cast<double>(m) * static_cast<double>(n));
    for (std::int64_t e = 0; e < target; ++e) {
        const auto r = static_cast<GlobalIdx>(rng.next_below(static_cast<std::uint64_t>(m)));
        const auto c = static_cast<GlobalIdx>(rng.next_below(static_cast<std::uint64_t>(n)));
        t.push_back(r, c, val(rng));
    }
    return t;
}

template <class VT>
DistSparseMat2D<VT> dist_from(const Triples<GlobalIdx, VT>& global, const Grid2D& grid) {
    Triples<GlobalIdx, VT> mine;
    mine.nrows = global.nrows;
    mine.ncols = global.ncols;
    if (grid.comm.rank() == 0) mine = global;
    return distribute_triples(mine, grid, global.nrows, global.ncols, [](const VT& a, const VT&) { return a; });
}

template <class VT>
bool same(const Triples<GlobalIdx, VT>& a, const Triples<GlobalIdx, VT>& b, bool exact) {
    if (a.nrows != b.nrows || a.ncols != b.ncols || a.rows != b.rows || a.cols != b.cols) return false;
    for (std::size_t k = 0; k < a.size(); ++k) {
        const double x = static_cast<double>(a.vals[k]), y = static_cast<double>(b.vals[k]);
        if (exact ? x != y : std::abs(x - y) > 1e-12 * std::max({1.0, std::abs(x), std::abs(y)})) return false;
    }
    return true;
}

std::mutex g_mu;
std::atomic<int> g_fail{0};
const bool g_trace = std::getenv("SLAPCU_SHIM_TRACE") != nullptr;
#define TRACE(what)                                                                 \
    do {                                                                            \
        if (g_trace) {                                                              \
            std::lock_guard<std::mutex> lk_(g_mu);                                  \
            std::fprintf(stderr, "[rank %d] %s\n", w.rank(), what);                  \
        }                                                                           \
    } while (0)
void fail(const char* what, int p) {
    std::lock_guard<std::mutex> lk(g_mu);
    std::printf("SHIM_DIST_FAIL %s p=%d\n", what, p);
    ++g_fail;
}

template <class SR, class Val>
void check_2d(int p, const SR& sr, Val val, bool exact, std::uint64_t seed) {
    using VT = typename SR::left_type;
    Rng rng(seed);
    const GlobalIdx m = 97 + static_cast<GlobalIdx>(rng.next_below(60)), k = 83, n = 101;
    auto ga = random_global<VT>(rng, m, k, 0.08, val);
    auto gb = random_global<VT>(rng, k, n, 0.08, val);
    const int q = static_cast<int>(std::lround(std::sqrt(p)));
    WorldOptions opt;
    opt.timeout = std::chrono::milliseconds(180000);  // first CUDA / NCCL init on a fresh box
    run_world(p, [&](Comm& w) {
        auto grid = make_grid2d(w, q, q);
        auto a = dist_from(ga, grid);
        auto b = dist_from(gb, grid);
        DistKernelStats s1, s2;
        TRACE("2d: reference summa");
        auto want = slap::summa2d_spgemm(a, b, sr, SpGemmAlg::hybrid, 1, &s1);
        TRACE("2d: gpu summa");
        auto got = slapcu_slap::summa2d_spgemm(a, b, sr, SpGemmAlg::hybrid, 1, &s2);
        TRACE("2d: gather");
        auto tw = gather_matrix(want), tg = gather_matrix(got);
        if (w.rank() == 0 && !same(tw, tg, exact)) fail("summa2d", p);
        if (s1.stages != s2.stages || s1.nnz_out != s2.nnz_out) fail("summa2d stats", p);
        // batched.hpp: counts, plan, batches
        TRACE("2d: counts");
        auto cw = slap::dist_symbolic_col_nnz(a, b);
        auto cg = slapcu_slap::dist_symbolic_col_nnz(a, b);
        TRACE("2d: plans");
        if (cw != cg) fail("dist_symbolic_col_nnz", p);
        std::int64_t cmax = 1;
        for (auto x : cw) cmax = std::max(cmax, x);
        const std::int64_t budget = 16 * 3 * cmax;  // a few batches
        auto pw = slap::plan_batches_by_budget(a, b, budget);
        auto pg = slapcu_slap::plan_batches_by_budget(a, b, budget);
        if (pw.col_ranges != pg.col_ranges || pw.est_entries != pg.est_entries) fail("plan_batches_by_budget", p);
        std::vector<Triples<GlobalIdx, typename SR::result_type>> bw, bg;
        TRACE("2d: batched");
        slap::batched_spgemm(a, b, pw, sr, SpGemmAlg::hash, 1,
                             [&](int, GlobalIdx, GlobalIdx, const auto& cr) { bw.push_back(gather_matrix(cr)); });
        slapcu_slap::batched_spgemm(a, b, pw, sr, SpGemmAlg::hash, 1,
                                    [&](int, GlobalIdx, GlobalIdx, const auto& cr) { bg.push_back(gather_matrix(cr)); });
        if (bw.size() != bg.size()) fail("batched_spgemm count", p);
        for (std::size_t r = 0; r < std::min(bw.size(), bg.size()); ++r)
            if (w.rank() == 0 && !same(bw[r], bg[r], exact)) fail("batched_spgemm batch", p);
        TRACE("2d: errors");
        // error contract: inner-dimension mismatch -> DimError on every rank before any collective
        auto bad = dist_from(random_global<VT>(rng, k + 1, n, 0.05, val), grid);
        try {
            slapcu_slap::summa2d_spgemm(a, bad, sr);
            fail("summa2d DimError", p);
        } catch (const DimError&) {
        }
    }, opt);
}

template <class SR, class Val>
void check_3d(int p, int feeder_pr, int feeder_pc, const SR& sr, Val val, bool exact, std::uint64_t seed) {
    using VT = typename SR::left_type;
    Rng rng(seed);
    const GlobalIdx m = 90, k = 77, n = 95;
    auto ga = random_global<VT>(rng, m, k, 0.1, val);
    auto gb = random_global<VT>(rng, k, n, 0.1, val);
    WorldOptions opt;
    opt.timeout = std::chrono::milliseconds(180000);
    run_world(p, [&](Comm& w) {
        auto g2 = make_grid2d(w, feeder_pr, feeder_pc);
        auto a2 = dist_from(ga, g2);
        auto b2 = dist_from(gb, g2);
        auto g3 = make_grid3d(w, p);  // c = p layers of 1 x 1
        auto a3 = redistribute_3d(a2, g3, SplitDim::cols);
        auto b3 = redistribute_3d(b2, g3, SplitDim::rows);
        DistKernelStats s1, s2;
        TRACE("3d: reference");
        auto want = slap::ca3d_spgemm(a3, b3, sr, SpGemmAlg::hybrid, 1, &s1);
        TRACE("3d: gpu");
        auto got = slapcu_slap::ca3d_spgemm(a3, b3, sr, SpGemmAlg::hybrid, 1, &s2);
        TRACE("3d: done");
        if (want.col_start != got.col_start || want.col_len != got.col_len) fail("ca3d piece", p);
        auto tw = gather_matrix(want), tg = gather_matrix(got);
        if (w.rank() == 0 && !same(tw, tg, exact)) fail("ca3d", p);
        if (s1.layer_warning != s2.layer_warning || s1.stages != s2.stages) fail("ca3d stats", p);
    }, opt);
}

int main() {
    int ndev = 0;
    slapcu_device_count(&ndev);
    if (ndev < 1) {
        std::printf("SHIM_DIST_SKIP no device\n");
        return 0;
    }
    // local phase drop-ins
    {
        Rng rng(7);
        for (int t = 0; t < 20; ++t) {
            auto ta = random_global<double>(rng, 120, 90, 0.05, [](Rng& r) { return r.next_double(); });
            auto tb = random_global<double>(rng, 90, 70, 0.05, [](Rng& r) { return r.next_double(); });
            Triples<LocalIdx, double> a32, b32;
            a32.nrows = 120, a32.ncols = 90, b32.nrows = 90, b32.ncols = 70;
            for (std::size_t e = 0; e < ta.size(); ++e) a32.push_back((LocalIdx)ta.rows[e], (LocalIdx)ta.cols[e], ta.vals[e]);
            for (std::size_t e = 0; e < tb.size(); ++e) b32.push_back((LocalIdx)tb.rows[e], (LocalIdx)tb.cols[e], tb.vals[e]);
            auto first = [](const double& x, const double&) { return x; };
            auto a = build_csc(a32, first);
            auto b = build_dcsc(b32, first);
            auto e1 = slap::estimate_flops(a, b), e2 = slapcu_slap::estimate_flops(a, b);
            if (e1.total_flops != e2.total_flops || e1.flops_per_column != e2.flops_per_column) fail("estimate_flops", 1);
            if (slap::symbolic_nnz(a, b, 2) != slapcu_slap::symbolic_nnz(a, b, 2)) fail("symbolic_nnz", 1);
        }
    }
    auto i64 = [](Rng& r) { return static_cast<std::int64_t>(r.next_below(9) + 1); };
    auto f64 = [](Rng& r) { return r.next_double() * 10.0; };
    auto i32 = [](Rng& r) { return static_cast<std::int32_t>(r.next_below(255) + 1); };
    auto ones = [](Rng&) { return std::uint8_t{1}; };
    for (int p : {1, 4}) {
        if (p > ndev) continue;
        check_2d(p, PlusTimesI64{}, i64, true, 11 + p);
        check_2d(p, PlusTimesF64{}, f64, false, 21 + p);
        check_2d(p, MinPlus<std::int32_t>{}, i32, true, 31 + p);
        check_2d(p, OrAnd{}, ones, true, 41 + p);
    }
    const int feeders[5][2] = {{0, 0}, {1, 1}, {1, 2}, {0, 0}, {2, 2}};
    for (int p : {1, 2, 4}) {
        if (p > ndev) continue;
        check_3d(p, feeders[p][0], feeders[p][1], PlusTimesI64{}, i64, true, 51 + p);
        check_3d(p, feeders[p][0], feeders[p][1], PlusTimesF64{}, f64, false, 61 + p);
    }
    if (g_fail) return 1;
    std::printf("SHIM_DIST_OK devices=%d\n", ndev);
    return 0;
}
