// Drop-in check of include/slapcu_slap.hpp: the same call sites with
// slap::local_spgemm (reference, CPU) and slapcu_slap::local_spgemm (GPU via
// the C-ABI) must agree -- bit-exact for integer / Boolean / MinPlus, rel 1e-12
// for fp64 -- on the reference's own worked example (test_localkernels.cpp:126-131)
// and on random CSC x DCSC pairs (acceptance.cpp:58-97 style).  Built in the
// container against the reference headers (tests/test_abi.py); the binary runs
// on the GPU box (tests/test_gpu_shim.py).  Prints SHIM_OK.
#include <cmath>
#include <cstdio>

#include "slap/rng.hpp"
#include "slap/triples.hpp"
#include "slapcu_slap.hpp"

using namespace slap;
using I = std::int32_t;

template <class VT, class Val>
Triples<I, VT> random_triples(Rng& rng, I m, I n, double density, Val val) {
    Triples<I, VT> t;
    t.nrows = m;
    t.ncols = n;
    const auto target = static_cast<std::int64_t>(density * m * n);
    for (std::int64_t e = 0; e < target; ++e) {
        const auto r = static_cast<I>(rng.next_below(static_cast<std::uint64_t>(m)));
        const auto c = static_cast<I>(rng.next_below(static_cast<std::uint64_t>(n)));
        t.push_back(r, c, val(rng));
    }
    return t;
}

template <class SR, class Val>
bool check(const SR& sr, Val val, bool exact, int trials, std::uint64_t seed) {
    using VT = typename SR::left_type;
    Rng rng(seed);
    auto first = [](const VT& x, const VT&) { return x; };
    for (int t = 0; t < trials; ++t) {
        const auto m = static_cast<I>(rng.next_below(120) + 2);
        const auto n = static_cast<I>(rng.next_below(120) + 2);
        const auto k = static_cast<I>(rng.next_below(120) + 2);
        const double d = 0.01 + 0.29 * rng.next_double();
        auto a = build_csc(random_triples<VT>(rng, m, n, d, val), first);
        auto b = build_dcsc(random_triples<VT>(rng, n, k, d, val), first);
        for (auto alg : {SpGemmAlg::heap, SpGemmAlg::hash, SpGemmAlg::hybrid}) {
            auto want = slap::local_spgemm(a, b, sr, alg, 2);
            auto got = slapcu_slap::local_spgemm(a, b, sr, alg, 2);
            if (got.colptr() != want.colptr() || got.rowids() != want.rowids()) return false;
            for (std::size_t e = 0; e < want.nnz(); ++e) {
                const double x = static_cast<double>(got.vals()[e]), y = static_cast<double>(want.vals()[e]);
                if (exact ? x != y : std::abs(x - y) > 1e-12 * std::max({1.0, std::abs(x), std::abs(y)})) return false;
            }
        }
    }
    return true;
}

int main() {
    // worked example
    Triples<I, std::int64_t> ta, tb;
    ta.nrows = ta.ncols = tb.nrows = tb.ncols = 2;
    ta.push_back(0, 0, 1);
    ta.push_back(1, 0, 2);
    ta.push_back(1, 1, 3);
    tb.push_back(0, 1, 4);
    tb.push_back(1, 0, 5);
    auto add = [](const std::int64_t& x, const std::int64_t& y) { return x + y; };
    auto c = to_triples(slapcu_slap::local_spgemm(build_csc(ta, add), build_csc(tb, add), PlusTimesI64{}));
    if (c.rows != std::vector<I>{1, 0, 1} || c.cols != std::vector<I>{0, 1, 1} ||
        c.vals != std::vector<std::int64_t>{15, 4, 8}) {
        std::printf("SHIM_FAIL worked example\n");
        return 1;
    }
    bool ok = true;
    ok = ok && check(PlusTimesI64{}, [](Rng& r) { return static_cast<std::int64_t>(r.next_below(9) + 1); }, true, 20, 1);
    ok = ok && check(OrAnd{}, [](Rng&) { return std::uint8_t{1}; }, true, 20, 2);
    ok = ok && check(MinPlus<std::int32_t>{}, [](Rng& r) { return static_cast<std::int32_t>(r.next_below(255) + 1); },
                     true, 20, 3);
    ok = ok && check(PlusTimesF64{}, [](Rng& r) { return r.next_double() * 10.0; }, false, 20, 4);
    // DimError passes through as the reference's exception kind
    try {
        Triples<I, double> bad;
        bad.nrows = 3;
        bad.ncols = 2;
        auto m = build_csc(bad, [](const double& x, const double&) { return x; });
        (void)slapcu_slap::local_spgemm(m, m, PlusTimesF64{});
        ok = false;
    } catch (const slap::DimError&) {
    }
    std::printf(ok ? "SHIM_OK\n" : "SHIM_FAIL\n");
    return ok ? 0 : 1;
}
