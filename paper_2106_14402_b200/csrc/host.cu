// host.cu -- batched_spgemm with HOST operands and a per-batch HOST consumer.
//
// The reference runs A * B(:, range_r) per column batch and hands each batch
// product to a consumer (batched.hpp:153-170); plan_batches_by_budget sizes
// the ranges so one batch's output fits a memory budget (batched.hpp:122-148).
// Here the operands come from host memory and every batch product is
// delivered in (pinned) host memory: H2D of A and B once, then per batch
// one direct product into a device buffer and the D2H of its result on a copy
// stream, so batch r+1's product overlaps batch r's read-back (the PCIe
// transfer is the long pole of a host-resident C3: 118.6 GB of output).
// The consumer runs on the calling thread; its buffers are valid during the
// call only (they are reused two batches later).
#include <algorithm>
#include <string>
#include <vector>

#include "kern.cuh"

namespace slapcu {

namespace {

void* grow_pinned(Ctx& c, int slot, size_t bytes) {
    auto& h = c.host;
    if (h.bytes[slot] >= bytes) return h.pinned[slot];
    if (h.pinned[slot]) SLAPCU_CUDA(cudaFreeHost(h.pinned[slot]));
    h.pinned[slot] = nullptr;
    h.bytes[slot] = 0;
    // 25% headroom: batch outputs vary, re-pinning is slow (~0.1 s/GB)
    const size_t want = bytes + bytes / 4 + 4096;
    if (cudaHostAlloc(&h.pinned[slot], want, cudaHostAllocDefault) != cudaSuccess) {
        cudaGetLastError();
        h.pinned[slot] = nullptr;
        throw Fail{SLAPCU_ERR_NOMEM, "pinned host allocation of " + std::to_string(want) + " bytes failed"};
    }
    h.bytes[slot] = want;
    return h.pinned[slot];
}

struct Event {
    cudaEvent_t e = nullptr;
    Event() { SLAPCU_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming)); }
    ~Event() {
        if (e) cudaEventDestroy(e);
    }
};

struct Stream {
    cudaStream_t s = nullptr;
    Stream() { SLAPCU_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking)); }
    ~Stream() {
        if (s) {
            cudaStreamSynchronize(s);
            cudaStreamDestroy(s);
        }
    }
};

}  // namespace

void free_host_cache(Ctx& c) {
    for (int i = 0; i < 2; ++i) {
        if (c.host.pinned[i]) cudaFreeHost(c.host.pinned[i]);
        c.host.pinned[i] = nullptr;
        c.host.bytes[i] = 0;
    }
}

// Column ranges for batched.hpp:122-148 semantics with the product's flops
// bound in place of the symbolic count (no symbolic pre-pass): the fewest
// contiguous ranges whose bound * entry_bytes fits the budget.
std::vector<std::pair<int64_t, int64_t>> plan_by_bound(const std::vector<int64_t>& bound, int64_t entry_bytes,
                                                       int64_t budget) {
    if (budget <= 0) throw Fail{SLAPCU_ERR_BUDGET, "memory budget must be positive"};
    std::vector<std::pair<int64_t, int64_t>> r;
    int64_t start = 0, cur = 0;
    const int64_t n = (int64_t)bound.size();
    for (int64_t j = 0; j < n; ++j) {
        const int64_t cost = bound[j] * entry_bytes;
        if (cost > budget)
            throw Fail{SLAPCU_ERR_BUDGET, "output column " + std::to_string(j) + " alone needs " + std::to_string(cost) +
                                              " bytes, budget is " + std::to_string(budget)};
        if (cur + cost > budget) {
            r.emplace_back(start, j);
            start = j;
            cur = 0;
        }
        cur += cost;
    }
    r.emplace_back(start, n);
    return r;
}

int64_t batched_host(Ctx& c, const slapcu_host_csc& Ah, const slapcu_host_csc& Bh, int sr, int alg, int nranges,
                     const int64_t* ranges, int64_t budget, slapcu_batch_consumer consumer, void* user) {
    const int vs = value_size(sr);
    if (vs <= 0) throw Fail{SLAPCU_ERR_INVALID, "unknown semiring"};
    if (Ah.ncols != Bh.nrows)
        throw Fail{SLAPCU_ERR_DIM, "spgemm inner dims: A is " + std::to_string(Ah.nrows) + "x" +
                                       std::to_string(Ah.ncols) + ", B is " + std::to_string(Bh.nrows) + "x" +
                                       std::to_string(Bh.ncols)};
    if (!consumer) throw Fail{SLAPCU_ERR_INVALID, "null consumer"};
    // ---- operands to the device (one copy; pinned sources overlap nothing else here)
    DevBuf acp(sizeof(int64_t) * (Ah.ncols + 1), c.stream), arw(sizeof(int32_t) * std::max<int64_t>(Ah.nnz, 1), c.stream),
        av(size_t(vs) * std::max<int64_t>(Ah.nnz, 1), c.stream);
    DevBuf bcp(sizeof(int64_t) * (Bh.ncols + 1), c.stream), brw(sizeof(int32_t) * std::max<int64_t>(Bh.nnz, 1), c.stream),
        bv(size_t(vs) * std::max<int64_t>(Bh.nnz, 1), c.stream);
    auto h2d = [&](void* d, const void* h, size_t n) {
        if (n) SLAPCU_CUDA(cudaMemcpyAsync(d, h, n, cudaMemcpyHostToDevice, c.stream));
    };
    h2d(acp.get(), Ah.colptr, sizeof(int64_t) * (Ah.ncols + 1));
    h2d(arw.get(), Ah.rowids, sizeof(int32_t) * Ah.nnz);
    if (Ah.vals) h2d(av.get(), Ah.vals, size_t(vs) * Ah.nnz);
    h2d(bcp.get(), Bh.colptr, sizeof(int64_t) * (Bh.ncols + 1));
    h2d(brw.get(), Bh.rowids, sizeof(int32_t) * Bh.nnz);
    if (Bh.vals) h2d(bv.get(), Bh.vals, size_t(vs) * Bh.nnz);
    DevCsc A{Ah.nrows, Ah.ncols, Ah.nnz, acp.as<int64_t>(), arw.as<int32_t>(), av.get()};
    DevCsc B{Bh.nrows, Bh.ncols, Bh.nnz, bcp.as<int64_t>(), brw.as<int32_t>(), bv.get()};
    DevCsc Ar = A, Br = B;
    resolve(c, Ar);
    resolve(c, Br);
    // ---- per-column bound min(flops_j, nrows): plan (if none given) and capacity
    const int64_t n = B.ncols;
    std::vector<int64_t> bound(size_t(std::max<int64_t>(n, 1)), 0);
    if (n) {
        DevBuf fl(sizeof(int64_t) * n, c.stream);
        int64_t tot = 0;
        spgemm_flops(c, Ar, Br, fl.as<int64_t>(), &tot);
        SLAPCU_CUDA(cudaMemcpyAsync(bound.data(), fl.get(), sizeof(int64_t) * n, cudaMemcpyDeviceToHost, c.stream));
        SLAPCU_CUDA(cudaStreamSynchronize(c.stream));
        for (auto& x : bound) x = std::min(x, A.nrows);
    }
    std::vector<std::pair<int64_t, int64_t>> plan;
    if (ranges) {
        if (nranges < 1) throw Fail{SLAPCU_ERR_SHAPE, "batch plan is empty"};
        int64_t expect = 0;
        for (int r = 0; r < nranges; ++r) {
            const int64_t s = ranges[2 * r], e = ranges[2 * r + 1];
            if (s != expect || e < s) throw Fail{SLAPCU_ERR_SHAPE, "batch ranges must partition B's columns in order"};
            expect = e;
            plan.emplace_back(s, e);
        }
        if (expect != n) throw Fail{SLAPCU_ERR_SHAPE, "batch ranges must cover all columns of B"};
    } else {
        plan = plan_by_bound(std::vector<int64_t>(bound.begin(), bound.begin() + n), 4 + vs, budget);
    }
    int64_t cap = 1, maxcols = 1;
    for (auto& [s, e] : plan) {
        int64_t b = 0;
        for (int64_t j = s; j < e; ++j) b += bound[j];
        cap = std::max(cap, b);
        maxcols = std::max(maxcols, e - s);
    }
    // ---- two device output sets, a copy stream, events
    DevBuf ocp[2], orw[2], ov[2];
    for (int i = 0; i < std::min<int>(2, (int)plan.size()); ++i) {
        ocp[i] = DevBuf(sizeof(int64_t) * (maxcols + 1), c.stream);
        orw[i] = DevBuf(sizeof(int32_t) * cap, c.stream);
        ov[i] = DevBuf(size_t(vs) * cap, c.stream);
    }
    Stream cs;
    Event produced[2], copied[2];
    struct Pending {
        int r = -1;
        int64_t nnz = 0;
        void* h = nullptr;
    } pend[2];
    int64_t total = 0;
    auto deliver = [&](Pending& p) {
        if (p.r < 0) return;
        SLAPCU_CUDA(cudaEventSynchronize(copied[p.r & 1].e));
        const auto [s, e] = plan[size_t(p.r)];
        const int64_t nc = e - s;
        int64_t* hcp = static_cast<int64_t*>(p.h);
        int32_t* hrw = reinterpret_cast<int32_t*>(hcp + nc + 1);
        void* hv = reinterpret_cast<char*>(hrw) + ((sizeof(int32_t) * p.nnz + 15) & ~size_t(15));
        slapcu_host_csc out{A.nrows, nc, p.nnz, hcp, hrw, hv};
        const int rc = consumer(user, p.r, s, e, &out);
        p.r = -1;
        if (rc != 0) throw Fail{SLAPCU_ERR_INVALID, "batch consumer returned " + std::to_string(rc)};
    };
    for (int r = 0; r < (int)plan.size(); ++r) {
        const int k = r & 1;
        const auto [s, e] = plan[size_t(r)];
        // device set k is free once batch r-2's read-back finished
        SLAPCU_CUDA(cudaStreamWaitEvent(c.stream, copied[k].e, 0));
        DevCsc w = B;
        w.ncols = e - s;
        w.cp = B.cp + s;
        const int64_t nnz = direct_spgemm(c, A, w, sr, alg, cap, ocp[k].as<int64_t>(), orw[k].as<int32_t>(), ov[k].get());
        total += nnz;
        // batch r-1's read-back has been running during this product: hand it over
        // (also frees pinned set k^1 for batch r+1)
        deliver(pend[k ^ 1]);
        // batch r-2's pinned set (k) was delivered in the previous iteration
        const size_t hb = sizeof(int64_t) * (w.ncols + 1) + ((sizeof(int32_t) * nnz + 15) & ~size_t(15)) + size_t(vs) * nnz;
        void* h = grow_pinned(c, k, hb);
        SLAPCU_CUDA(cudaEventRecord(produced[k].e, c.stream));
        SLAPCU_CUDA(cudaStreamWaitEvent(cs.s, produced[k].e, 0));
        int64_t* hcp = static_cast<int64_t*>(h);
        int32_t* hrw = reinterpret_cast<int32_t*>(hcp + w.ncols + 1);
        char* hv = reinterpret_cast<char*>(hrw) + ((sizeof(int32_t) * nnz + 15) & ~size_t(15));
        SLAPCU_CUDA(cudaMemcpyAsync(hcp, ocp[k].get(), sizeof(int64_t) * (w.ncols + 1), cudaMemcpyDeviceToHost, cs.s));
        if (nnz) {
            SLAPCU_CUDA(cudaMemcpyAsync(hrw, orw[k].get(), sizeof(int32_t) * nnz, cudaMemcpyDeviceToHost, cs.s));
            SLAPCU_CUDA(cudaMemcpyAsync(hv, ov[k].get(), size_t(vs) * nnz, cudaMemcpyDeviceToHost, cs.s));
        }
        SLAPCU_CUDA(cudaEventRecord(copied[k].e, cs.s));
        pend[k] = Pending{r, nnz, h};
    }
    const int last = (int)plan.size() - 1;
    deliver(pend[(last - 1) & 1]);  // (no-op when already delivered)
    deliver(pend[last & 1]);
    SLAPCU_CUDA(cudaStreamSynchronize(c.stream));
    return total;
}

}  // namespace slapcu
