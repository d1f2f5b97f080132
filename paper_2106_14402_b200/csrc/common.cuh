// common.cuh -- shared device helpers and the semiring functors for sm_100a.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <climits>
#include <cmath>
#include <string>

#include "slapcu.h"

namespace slapcu {

// ------------------------------------------------------------- error plumbing

struct Fail {
    slapcu_status st;
    std::string msg;
};

#define SLAPCU_CUDA(call)                                                                                  \
    do {                                                                                                   \
        cudaError_t e_ = (call);                                                                           \
        if (e_ != cudaSuccess)                                                                             \
            throw ::slapcu::Fail{e_ == cudaErrorMemoryAllocation ? SLAPCU_ERR_NOMEM : SLAPCU_ERR_CUDA,      \
                                 std::string(#call) + ": " + cudaGetErrorString(e_)};                       \
    } while (0)

#define SLAPCU_LAUNCH_CHECK() SLAPCU_CUDA(cudaGetLastError())

// ------------------------------------------------------------------ semirings
// semiring.hpp:36-74.  `Acc` is the accumulator type held in shared memory
// (OrAnd accumulates in a 32-bit word so it can use native smem atomics).
// `mul` and `add` restate the reference functors exactly; `atomic_acc` is
// the commutative-associative fold applied concurrently (order differs from
// the reference's ascending-k fold only for floating point, where the
// north_star tolerance applies).

template <int ID>
struct Sr;

template <>
struct Sr<SLAPCU_PLUS_TIMES_F64> {
    using T = double;
    using Acc = double;
    static __device__ __forceinline__ Acc mul(T a, T b) { return a * b; }
    static __device__ __forceinline__ Acc add(Acc a, Acc b) { return a + b; }
    static __device__ __forceinline__ Acc identity() { return 0.0; }
    static __device__ __forceinline__ void atomic_acc(Acc* p, Acc v) { atomicAdd(p, v); }
    static __device__ __forceinline__ void atomic_acc_global(T* p, Acc v) { atomicAdd(p, v); }
    static __device__ __forceinline__ T out(Acc a) { return a; }
};

template <>
struct Sr<SLAPCU_PLUS_TIMES_F32> {
    using T = float;
    using Acc = float;
    static __device__ __forceinline__ Acc mul(T a, T b) { return a * b; }
    static __device__ __forceinline__ Acc add(Acc a, Acc b) { return a + b; }
    static __device__ __forceinline__ Acc identity() { return 0.0f; }
    static __device__ __forceinline__ void atomic_acc(Acc* p, Acc v) { atomicAdd(p, v); }
    static __device__ __forceinline__ void atomic_acc_global(T* p, Acc v) { atomicAdd(p, v); }
    static __device__ __forceinline__ T out(Acc a) { return a; }
};

template <>
struct Sr<SLAPCU_PLUS_TIMES_I64> {
    using T = int64_t;
    using Acc = unsigned long long;  // two's-complement wraparound add
    static __device__ __forceinline__ Acc mul(T a, T b) { return (Acc)a * (Acc)b; }
    static __device__ __forceinline__ Acc add(Acc a, Acc b) { return a + b; }
    static __device__ __forceinline__ Acc identity() { return 0ull; }
    static __device__ __forceinline__ void atomic_acc(Acc* p, Acc v) { atomicAdd(p, v); }
    static __device__ __forceinline__ void atomic_acc_global(T* p, Acc v) {
        atomicAdd(reinterpret_cast<unsigned long long*>(p), v);
    }
    static __device__ __forceinline__ T out(Acc a) { return (T)a; }
};

template <>
struct Sr<SLAPCU_MIN_PLUS_I32> {
    using T = int32_t;
    using Acc = int;
    static __device__ __forceinline__ Acc mul(T a, T b) { return (int)((unsigned)a + (unsigned)b); }
    static __device__ __forceinline__ Acc add(Acc a, Acc b) { return a < b ? a : b; }
    static __device__ __forceinline__ Acc identity() { return INT_MAX; }
    static __device__ __forceinline__ void atomic_acc(Acc* p, Acc v) { atomicMin(p, v); }
    static __device__ __forceinline__ void atomic_acc_global(T* p, Acc v) { atomicMin(p, v); }
    static __device__ __forceinline__ T out(Acc a) { return a; }
};

__device__ __forceinline__ void atomic_min_f64(double* p, double v) {
    // add(a,b) = a < b ? a : b (semiring.hpp:69): replace unless the stored
    // value is strictly smaller.
    unsigned long long* q = reinterpret_cast<unsigned long long*>(p);
    unsigned long long old = *q;
    while (!(__longlong_as_double((long long)old) < v)) {
        unsigned long long prev = atomicCAS(q, old, (unsigned long long)__double_as_longlong(v));
        if (prev == old) break;
        old = prev;
    }
}

template <>
struct Sr<SLAPCU_MIN_PLUS_F64> {
    using T = double;
    using Acc = double;
    static __device__ __forceinline__ Acc mul(T a, T b) { return a + b; }
    static __device__ __forceinline__ Acc add(Acc a, Acc b) { return a < b ? a : b; }
    static __device__ __forceinline__ Acc identity() { return __longlong_as_double(0x7ff0000000000000ll); }
    static __device__ __forceinline__ void atomic_acc(Acc* p, Acc v) { atomic_min_f64(p, v); }
    static __device__ __forceinline__ void atomic_acc_global(T* p, Acc v) { atomic_min_f64(p, v); }
    static __device__ __forceinline__ T out(Acc a) { return a; }
};

template <>
struct Sr<SLAPCU_OR_AND_U8> {
    using T = uint8_t;
    using Acc = unsigned;
    static __device__ __forceinline__ Acc mul(T a, T b) { return (a && b) ? 1u : 0u; }
    static __device__ __forceinline__ Acc add(Acc a, Acc b) { return (a || b) ? 1u : 0u; }
    static __device__ __forceinline__ Acc identity() { return 0u; }
    static __device__ __forceinline__ void atomic_acc(Acc* p, Acc v) {
        if (v) atomicOr(p, 1u);
    }
    static __device__ __forceinline__ void atomic_acc_global(T* p, Acc v) {
        if (v) {
            uintptr_t a = reinterpret_cast<uintptr_t>(p);
            unsigned* w = reinterpret_cast<unsigned*>(a & ~uintptr_t(3));
            atomicOr(w, 1u << (8 * (a & 3)));
        }
    }
    static __device__ __forceinline__ T out(Acc a) { return (T)(a ? 1 : 0); }
};

inline int value_size(int sr) {
    switch (sr) {
    case SLAPCU_PLUS_TIMES_F64: return 8;
    case SLAPCU_PLUS_TIMES_F32: return 4;
    case SLAPCU_PLUS_TIMES_I64: return 8;
    case SLAPCU_MIN_PLUS_I32: return 4;
    case SLAPCU_MIN_PLUS_F64: return 8;
    case SLAPCU_OR_AND_U8: return 1;
    }
    return 0;
}

// Calls f(std::integral_constant<int, ID>) for a runtime semiring id.
template <class F>
void dispatch_sr(int sr, F&& f) {
    switch (sr) {
    case SLAPCU_PLUS_TIMES_F64: f(std::integral_constant<int, SLAPCU_PLUS_TIMES_F64>{}); return;
    case SLAPCU_PLUS_TIMES_F32: f(std::integral_constant<int, SLAPCU_PLUS_TIMES_F32>{}); return;
    case SLAPCU_PLUS_TIMES_I64: f(std::integral_constant<int, SLAPCU_PLUS_TIMES_I64>{}); return;
    case SLAPCU_MIN_PLUS_I32: f(std::integral_constant<int, SLAPCU_MIN_PLUS_I32>{}); return;
    case SLAPCU_MIN_PLUS_F64: f(std::integral_constant<int, SLAPCU_MIN_PLUS_F64>{}); return;
    case SLAPCU_OR_AND_U8: f(std::integral_constant<int, SLAPCU_OR_AND_U8>{}); return;
    }
    throw Fail{SLAPCU_ERR_INVALID, "unknown semiring id " + std::to_string(sr)};
}

// ------------------------------------------------------------------ helpers

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {  // rng.hpp:34-41
    z ^= z >> 30;
    z *= 0xbf58476d1ce4e5b9ull;
    z ^= z >> 27;
    z *= 0x94d049bb133111ebull;
    z ^= z >> 31;
    return z;
}

constexpr uint64_t kGolden = 0x9e3779b97f4a7c15ull;

__device__ __forceinline__ int warp_reduce_sum(int v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ long long warp_reduce_sum64(long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// exclusive prefix sum within a full warp
__device__ __forceinline__ int warp_excl_scan(int v, int lane, int* total) {
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    *total = __shfl_sync(0xffffffffu, x, 31);
    return x - v;
}

// Warp-aggregated increment of a shared or global counter.
__device__ __forceinline__ int warp_agg_inc(int* ctr) {
    unsigned m = __activemask();
    int lane = threadIdx.x & 31;
    int leader = __ffs(m) - 1;
    int base = 0;
    if (lane == leader) base = atomicAdd(ctr, __popc(m));
    base = __shfl_sync(m, base, leader);
    return base + __popc(m & ((1u << lane) - 1u));
}

// Named barrier over `nthreads` threads (a multiple of 32); id 1..15.
__device__ __forceinline__ void named_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace slapcu
