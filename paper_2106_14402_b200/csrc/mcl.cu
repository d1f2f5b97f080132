// mcl.cu -- the Markov-clustering step around the SpGEMM.
//
// algorithms.cpp:267-293 mcl_step: input columns must sum to 1 (1e-9,
// StochasticityError), expansion C = A*A in PlusTimes, inflation v -> v^e,
// pruning of entries below the threshold (kept iff !(v < thr)), and column
// renormalisation (v / column sum; a zero-sum column is left as is,
// algorithms.cpp:55-67).  The expansion is the direct single-pass product;
// inflation, pruning and the column sums are one counting pass over C, the
// renormalised survivors one writing pass (warp per column, sums in double).
#include <cub/cub.cuh>

#include <cmath>
#include <functional>

#include "kern.cuh"

namespace slapcu {
namespace {

template <class T>
__global__ void k_col_sum_check(int64_t ncols, const int64_t* __restrict__ cp, const T* __restrict__ v, double tol,
                                int* __restrict__ bad) {
    const int lane = threadIdx.x & 31;
    for (int64_t j = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; j < ncols;
         j += (int64_t(gridDim.x) * blockDim.x) >> 5) {
        double s = 0;
        for (int64_t e = cp[j] + lane; e < cp[j + 1]; e += 32) s += (double)v[e];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0 && fabs(s - 1.0) > tol) atomicExch(bad, 1);
    }
}

// v^e rounded to T.  MCL's usual inflation 2 is a double product (exact for
// f32 inputs, correctly rounded for f64 like a correctly rounded pow); a
// general double pow costs ~50x more and made the epilogue compute-bound.
enum { kPow = 0, kSquare = 1, kIdentity = 2 };
template <class T, int MODE>
__device__ __forceinline__ T inflate(T v, double e) {
    if constexpr (MODE == kSquare) return (T)((double)v * (double)v);
    else if constexpr (MODE == kIdentity) return v;
    else return (T)pow((double)v, e);
}

// kept entries per column and the column sum of the kept (inflated) values.
// Warp per column; each lane keeps kU independent loads in flight (the pass
// is a 12 GB stream at C4 and one load per lane per trip left it latency-bound).
constexpr int kU = 4;

template <class T, int MODE>
__global__ void k_mcl_count(int64_t ncols, const int64_t* __restrict__ cp, const T* __restrict__ v, double e,
                            double thr, int64_t* __restrict__ kept, double* __restrict__ sums) {
    const int lane = threadIdx.x & 31;
    for (int64_t j = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; j < ncols;
         j += (int64_t(gridDim.x) * blockDim.x) >> 5) {
        const int64_t b1 = cp[j + 1];
        double s = 0;
        int k = 0;
        for (int64_t q = cp[j] + lane; q < b1; q += 32 * kU) {
            T x[kU];
#pragma unroll
            for (int u = 0; u < kU; ++u) x[u] = q + 32 * u < b1 ? v[q + 32 * u] : T(0);
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                if (q + 32 * u < b1) {
                    const T y = inflate<T, MODE>(x[u], e);
                    if (!((double)y < thr)) {
                        s += (double)y;
                        ++k;
                    }
                }
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            s += __shfl_xor_sync(0xffffffffu, s, o);
            k += __shfl_xor_sync(0xffffffffu, k, o);
        }
        if (lane == 0) {
            kept[j] = k;
            sums[j] = s;
        }
    }
}

// survivors in order (warp ballot compaction), divided by the column sum;
// row ids are read only for survivors
template <class T, int MODE>
__global__ void k_mcl_write(int64_t ncols, const int64_t* __restrict__ cp, const int32_t* __restrict__ rw,
                            const T* __restrict__ v, double e, double thr, const double* __restrict__ sums,
                            const int64_t* __restrict__ ocp, int32_t* __restrict__ orw, T* __restrict__ ov) {
    const int lane = threadIdx.x & 31;
    for (int64_t j = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; j < ncols;
         j += (int64_t(gridDim.x) * blockDim.x) >> 5) {
        const int64_t b1 = cp[j + 1];
        if (ocp[j + 1] == ocp[j]) continue;  // nothing survives in this column
        const double s = sums[j];
        int64_t o = ocp[j];
        for (int64_t b = cp[j]; b < b1; b += 32 * kU) {
            T x[kU];
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const int64_t q = b + 32 * u + lane;
                x[u] = q < b1 ? v[q] : T(0);
            }
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const int64_t q = b + 32 * u + lane;
                bool keep = false;
                T y = T(0);
                if (q < b1) {
                    y = inflate<T, MODE>(x[u], e);
                    keep = !((double)y < thr);
                }
                const unsigned m = __ballot_sync(0xffffffffu, keep);
                if (keep) {
                    const int64_t at = o + __popc(m & ((1u << lane) - 1u));
                    orw[at] = rw[q];
                    ov[at] = s != 0.0 ? (T)((double)y / s) : y;
                }
                o += __popc(m);
            }
        }
    }
}

template <class T>
__global__ void k_col_sums(int64_t ncols, const int64_t* __restrict__ cp, const T* __restrict__ v,
                           double* __restrict__ sums) {
    const int lane = threadIdx.x & 31;
    for (int64_t j = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; j < ncols;
         j += (int64_t(gridDim.x) * blockDim.x) >> 5) {
        double s = 0;
        for (int64_t e = cp[j] + lane; e < cp[j + 1]; e += 32) s += (double)v[e];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) sums[j] = s;
    }
}

__global__ void k_sums_check(int64_t n, const double* __restrict__ s, double tol, int* __restrict__ bad) {
    for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < n; j += int64_t(gridDim.x) * blockDim.x)
        if (fabs(s[j] - 1.0) > tol) atomicExch(bad, 1);
}

}  // namespace

// Block pieces of mcl_step for the distributed driver (dist.cu): column sums
// of a block (double), the sum check, and the epilogue of an expanded block
// whose column sums are reduced by `reduce` (the grid-column allreduce)
// between the counting and the writing pass.
void mcl_block_colsums(Ctx& c, const DevCsc& A, int sr, double* sums) {
    dispatch_sr(sr, [&](auto id) {
        constexpr int ID = decltype(id)::value;
        if constexpr (ID == SLAPCU_PLUS_TIMES_F64 || ID == SLAPCU_PLUS_TIMES_F32) {
            using T = typename Sr<ID>::T;
            if (A.ncols)
                launch(c, k_col_sums<T>, dim3(grid_for(c, A.ncols * 32, 256)), dim3(256), 0, A.ncols, A.cp,
                       static_cast<const T*>(A.v), sums);
        } else {
            throw Fail{SLAPCU_ERR_INVALID, "mcl step: PlusTimes f64 or f32"};
        }
    });
}

bool mcl_sums_bad(Ctx& c, const double* sums, int64_t n, double tol) {
    DevBuf bad(sizeof(int), c.stream);
    SLAPCU_CUDA(cudaMemsetAsync(bad.get(), 0, sizeof(int), c.stream));
    if (n) launch(c, k_sums_check, dim3(grid_for(c, n, 256)), dim3(256), 0, n, sums, tol, bad.as<int>());
    int h = 0;
    SLAPCU_CUDA(cudaMemcpyAsync(&h, bad.get(), sizeof(int), cudaMemcpyDeviceToHost, c.stream));
    SLAPCU_CUDA(cudaStreamSynchronize(c.stream));
    return h != 0;
}

void mcl_block_epilogue(Ctx& c, const DevCsc& E_, int sr, double inflation, double prune,
                        const std::function<void(double*, int64_t)>& reduce, slapcu_csc_out* out) {
    DevCsc E = E_;
    resolve(c, E);
    const int64_t n = E.ncols;
    dispatch_sr(sr, [&](auto id) {
        constexpr int ID = decltype(id)::value;
        if constexpr (ID == SLAPCU_PLUS_TIMES_F64 || ID == SLAPCU_PLUS_TIMES_F32) {
            using T = typename Sr<ID>::T;
            DevBuf kept(sizeof(int64_t) * (n + 1), c.stream), sums(sizeof(double) * std::max<int64_t>(n, 1), c.stream);
            SLAPCU_CUDA(cudaMemsetAsync(kept.as<int64_t>() + n, 0, sizeof(int64_t), c.stream));
            const int mode = inflation == 2.0 ? kSquare : inflation == 1.0 ? kIdentity : kPow;
            auto kc = mode == kSquare ? k_mcl_count<T, kSquare> : mode == kIdentity ? k_mcl_count<T, kIdentity>
                                                                                    : k_mcl_count<T, kPow>;
            auto kw = mode == kSquare ? k_mcl_write<T, kSquare> : mode == kIdentity ? k_mcl_write<T, kIdentity>
                                                                                    : k_mcl_write<T, kPow>;
            if (n)
                launch(c, kc, dim3(grid_for(c, n * 32, 256)), dim3(256), 0, n, E.cp, static_cast<const T*>(E.v),
                       inflation, prune, kept.as<int64_t>(), sums.as<double>());
            reduce(sums.as<double>(), n);  // kept entries are local; their sums span the grid column
            out->nrows = E.nrows;
            out->ncols = n;
            SLAPCU_CUDA(cudaMallocAsync((void**)&out->colptr, sizeof(int64_t) * (n + 1), c.stream));
            exclusive_scan_i64(c, kept.as<int64_t>(), out->colptr, n + 1);
            SLAPCU_CUDA(cudaMemcpyAsync(&out->nnz, out->colptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost, c.stream));
            SLAPCU_CUDA(cudaStreamSynchronize(c.stream));
            SLAPCU_CUDA(cudaMallocAsync((void**)&out->rowids, sizeof(int32_t) * std::max<int64_t>(out->nnz, 1), c.stream));
            SLAPCU_CUDA(cudaMallocAsync(&out->vals, sizeof(T) * std::max<int64_t>(out->nnz, 1), c.stream));
            if (n)
                launch(c, kw, dim3(grid_for(c, n * 32, 256)), dim3(256), 0, n, E.cp, E.rw, static_cast<const T*>(E.v),
                       inflation, prune, (const double*)sums.as<double>(), (const int64_t*)out->colptr, out->rowids,
                       static_cast<T*>(out->vals));
        } else {
            throw Fail{SLAPCU_ERR_INVALID, "mcl step: PlusTimes f64 or f32"};
        }
    });
}

void mcl_step(Ctx& c, const DevCsc& A_, int sr, double inflation, double prune, slapcu_csc_out* out) {
    if (sr != SLAPCU_PLUS_TIMES_F64 && sr != SLAPCU_PLUS_TIMES_F32)
        throw Fail{SLAPCU_ERR_INVALID, "mcl step: PlusTimes f64 or f32"};
    if (A_.nrows != A_.ncols) throw Fail{SLAPCU_ERR_SHAPE, "mcl step needs a square matrix"};
    if (!(inflation > 0.0)) throw Fail{SLAPCU_ERR_SHAPE, "inflation exponent must be positive"};
    DevCsc A = A_;
    resolve(c, A);
    const int64_t n = A.ncols;
    // f32 inputs carry ~1e-7 of rounding per column sum; f64 uses the reference's 1e-9
    const double tol = sr == SLAPCU_PLUS_TIMES_F64 ? 1e-9 : 1e-5;
    dispatch_sr(sr, [&](auto id) {
        constexpr int ID = decltype(id)::value;
        if constexpr (ID == SLAPCU_PLUS_TIMES_F64 || ID == SLAPCU_PLUS_TIMES_F32) {
            using T = typename Sr<ID>::T;
            DevBuf bad(sizeof(int), c.stream);
            SLAPCU_CUDA(cudaMemsetAsync(bad.get(), 0, sizeof(int), c.stream));
            launch(c, k_col_sum_check<T>, dim3(grid_for(c, n * 32, 256)), dim3(256), 0, n, A.cp,
                   static_cast<const T*>(A.v), tol, bad.as<int>());
            int hbad = 0;
            SLAPCU_CUDA(cudaMemcpyAsync(&hbad, bad.get(), sizeof(int), cudaMemcpyDeviceToHost, c.stream));
            SLAPCU_CUDA(cudaStreamSynchronize(c.stream));
            if (hbad) throw Fail{SLAPCU_ERR_STOCHASTIC, "input column sums deviate from 1"};
            // expansion
            int64_t* ecp = nullptr;
            int32_t* erw = nullptr;
            void* ev = nullptr;
            int64_t enz = 0;
            // the expansion stays in the context's product scratch; the
            // epilogue reads it there (no exactly-sized copy of C)
            if (!direct_exact(c, A, A, sr, SLAPCU_ALG_HYBRID, 0, &ecp, &erw, &ev, &enz, false))
                throw Fail{SLAPCU_ERR_NOMEM, "mcl expansion does not fit"};
            struct Free {
                Ctx& c;
                void* p;
                ~Free() {
                    if (p) cudaFreeAsync(p, c.stream);
                }
            } fe{c, ecp};
            DevBuf kept(sizeof(int64_t) * (n + 1), c.stream), sums(sizeof(double) * std::max<int64_t>(n, 1), c.stream);
            SLAPCU_CUDA(cudaMemsetAsync(kept.as<int64_t>() + n, 0, sizeof(int64_t), c.stream));
            const int mode = inflation == 2.0 ? kSquare : inflation == 1.0 ? kIdentity : kPow;
            auto kc = mode == kSquare ? k_mcl_count<T, kSquare> : mode == kIdentity ? k_mcl_count<T, kIdentity>
                                                                                    : k_mcl_count<T, kPow>;
            auto kw = mode == kSquare ? k_mcl_write<T, kSquare> : mode == kIdentity ? k_mcl_write<T, kIdentity>
                                                                                    : k_mcl_write<T, kPow>;
            launch(c, kc, dim3(grid_for(c, n * 32, 256)), dim3(256), 0, n, (const int64_t*)ecp,
                   (const T*)ev, inflation, prune, kept.as<int64_t>(), sums.as<double>());
            out->nrows = n;
            out->ncols = n;
            SLAPCU_CUDA(cudaMallocAsync((void**)&out->colptr, sizeof(int64_t) * (n + 1), c.stream));
            exclusive_scan_i64(c, kept.as<int64_t>(), out->colptr, n + 1);
            SLAPCU_CUDA(cudaMemcpyAsync(&out->nnz, out->colptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost, c.stream));
            SLAPCU_CUDA(cudaStreamSynchronize(c.stream));
            SLAPCU_CUDA(cudaMallocAsync((void**)&out->rowids, sizeof(int32_t) * std::max<int64_t>(out->nnz, 1), c.stream));
            SLAPCU_CUDA(cudaMallocAsync(&out->vals, sizeof(T) * std::max<int64_t>(out->nnz, 1), c.stream));
            launch(c, kw, dim3(grid_for(c, n * 32, 256)), dim3(256), 0, n, (const int64_t*)ecp,
                   (const int32_t*)erw, (const T*)ev, inflation, prune, (const double*)sums.as<double>(),
                   (const int64_t*)out->colptr, out->rowids, static_cast<T*>(out->vals));
        }
    });
}

}  // namespace slapcu
