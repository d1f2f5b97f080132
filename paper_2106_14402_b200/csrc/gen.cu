// gen.cu -- synthetic inputs built on the device, bit-identical to the
// reference generators, plus small format utilities (value recipes, symmetric
// permutation, column slices, per-column checksums).
//
//   gen_rmat        algorithms.cpp:71-113 (Rng, rng.hpp:12-45; one counter-based
//                   stream per edge draw, symmetrize, drop self loops, dedup)
//   gen_er          oracles.hpp:205-217 random_triples (row, col, value drawn in
//                   that order from ONE Rng stream -- splitmix is counter-based,
//                   so draw m is mix(state0 + (m+1)*golden) and every draw is
//                   computed independently), keep-first dedup
//   gen_one_per_row tall-skinny B of config C5
#include <cub/cub.cuh>

#include <algorithm>

#include "ctx.hpp"

namespace slapcu {

__device__ __forceinline__ uint64_t rng_init(uint64_t seed, uint64_t stream) {  // rng.hpp:16-17
    return mix64(seed * kGolden + stream + 1);
}
__device__ __forceinline__ uint64_t rng_draw(uint64_t state0, uint64_t m) {  // m-th next_u64 (0-based)
    return mix64(state0 + (m + 1) * kGolden);
}
__device__ __forceinline__ double u53(uint64_t x) { return (double)(x >> 11) * 0x1.0p-53; }  // rng.hpp:26-28

// key = col << scale | row ; invalid (self loop) = all ones in 2*scale bits,
// which is the (n-1, n-1) self loop and therefore never a valid edge.
__global__ void k_rmat_edges(int scale, int64_t edges, uint64_t seed, double a, double ab, double abc,
                             uint64_t* __restrict__ keys) {
    const uint64_t invalid = (scale >= 32) ? ~0ull : ((1ull << (2 * scale)) - 1ull);
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < edges;
         e += int64_t(gridDim.x) * blockDim.x) {
        uint64_t st = rng_init(seed, (uint64_t)e + 0x524d4154ull);
        uint64_t i = 0, j = 0;
        for (int level = 0; level < scale; ++level) {
            st += kGolden;
            const double u = u53(mix64(st));
            int qi = 0, qj = 0;
            if (u < a) {
            } else if (u < ab) {
                qj = 1;
            } else if (u < abc) {
                qi = 1;
            } else {
                qi = 1;
                qj = 1;
            }
            i = (i << 1) | qi;
            j = (j << 1) | qj;
        }
        if (i == j) {
            keys[2 * e] = invalid;
            keys[2 * e + 1] = invalid;
        } else {
            keys[2 * e] = (j << scale) | i;
            keys[2 * e + 1] = (i << scale) | j;
        }
    }
}

// colptr[j] = lower_bound(keys, j * stride); rowids = key % stride.
__global__ void k_keys_to_csc(int64_t m, int64_t ncols, int64_t stride, const uint64_t* __restrict__ keys,
                              int64_t* __restrict__ colptr, int32_t* __restrict__ rowids) {
    const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t nt = int64_t(gridDim.x) * blockDim.x;
    for (int64_t e = tid; e < m; e += nt) rowids[e] = (int32_t)(keys[e] % (uint64_t)stride);
    for (int64_t j = tid; j <= ncols; j += nt) {
        const uint64_t key = (uint64_t)j * (uint64_t)stride;
        int64_t lo = 0, hi = m;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (keys[mid] < key)
                lo = mid + 1;
            else
                hi = mid;
        }
        colptr[j] = lo;
    }
}

__global__ void k_er_draws(int64_t draws, int64_t n, uint64_t st0, uint64_t* __restrict__ keys,
                           int64_t* __restrict__ idx) {
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < draws;
         e += int64_t(gridDim.x) * blockDim.x) {
        const uint64_t r = rng_draw(st0, 3 * (uint64_t)e) % (uint64_t)n;
        const uint64_t c = rng_draw(st0, 3 * (uint64_t)e + 1) % (uint64_t)n;
        keys[e] = c * (uint64_t)n + r;
        idx[e] = e;
    }
}

__global__ void k_er_values(int64_t m, uint64_t st0, const int64_t* __restrict__ idx, double* __restrict__ vals) {
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < m; e += int64_t(gridDim.x) * blockDim.x)
        vals[e] = u53(rng_draw(st0, 3 * (uint64_t)idx[e] + 2));
}

__global__ void k_opr_draws(int64_t n, int64_t ncols, uint64_t st0, uint64_t* __restrict__ keys) {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const uint64_t c = rng_draw(st0, 2 * (uint64_t)i) % (uint64_t)ncols;
        keys[i] = c * (uint64_t)n + (uint64_t)i;
    }
}

__global__ void k_opr_values(int64_t m, uint64_t st0, const int32_t* __restrict__ rows, double* __restrict__ vals) {
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < m; e += int64_t(gridDim.x) * blockDim.x)
        vals[e] = u53(rng_draw(st0, 2 * (uint64_t)rows[e] + 1));
}

// Value recipes, one warp per column.
template <class T>
__global__ void k_fill_values(int64_t ncols, const int64_t* __restrict__ cp, const int32_t* __restrict__ rw, int kind,
                              int is_float32, T* __restrict__ vals) {
    const int lane = threadIdx.x & 31;
    for (int64_t j = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; j < ncols;
         j += (int64_t(gridDim.x) * blockDim.x) >> 5) {
        const int64_t b = cp[j], e = cp[j + 1];
        const int64_t deg = e - b;
        for (int64_t p = b + lane; p < e; p += 32) {
            const uint64_t h = mix64(((uint64_t)(uint32_t)rw[p] << 32) ^ (uint64_t)j);
            const double u = u53(h);
            double dv;
            int64_t iv;
            switch (kind) {
            case 0: dv = 1.0; iv = 1; break;
            case 1: dv = u; iv = 1 + (int64_t)(h % 255); break;
            case 2: dv = 10.0 * u; iv = 1 + (int64_t)(h % 255); break;
            case 3: iv = 1 + (int64_t)(h % 255); dv = (double)iv; break;
            case 4: dv = 1.0 / (double)deg; iv = 1; break;
            case 5: iv = 1 + (int64_t)(h % 9); dv = (double)iv; break;
            default: dv = 1.0; iv = 1;
            }
            if constexpr (sizeof(T) == 1) {
                vals[p] = (T)1;
            } else if constexpr (std::is_floating_point<T>::value) {
                if (is_float32 && kind == 4)
                    vals[p] = (T)(1.0f / (float)deg);
                else
                    vals[p] = (T)dv;
            } else {
                vals[p] = (T)iv;
            }
        }
    }
}

__global__ void k_column_checksums(int64_t ncols, const int64_t* __restrict__ cp, const int32_t* __restrict__ rw,
                                   const unsigned char* __restrict__ vals, int vs, uint64_t* __restrict__ sums) {
    const int lane = threadIdx.x & 31;
    for (int64_t j = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; j < ncols;
         j += (int64_t(gridDim.x) * blockDim.x) >> 5) {
        unsigned long long s = 0;
        for (int64_t p = cp[j] + lane; p < cp[j + 1]; p += 32) {
            uint64_t bits = 0;
            for (int b = 0; b < vs; ++b) bits |= (uint64_t)vals[p * vs + b] << (8 * b);
            s += mix64(((uint64_t)(uint32_t)rw[p] * kGolden) ^ bits);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) sums[j] = s;
    }
}

// Symmetric relabelling: new id of i is its rank under a random sort key.
__global__ void k_perm_keys(int64_t n, uint64_t seed, uint64_t* __restrict__ key, int64_t* __restrict__ ids) {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        key[i] = mix64(seed * kGolden ^ mix64((uint64_t)i + 0x7065726dull));
        ids[i] = i;
    }
}
__global__ void k_invert(int64_t n, const int64_t* __restrict__ sorted_ids, int64_t* __restrict__ newid) {
    for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < n; r += int64_t(gridDim.x) * blockDim.x)
        newid[sorted_ids[r]] = r;
}
__global__ void k_perm_entries(int64_t ncols, const int64_t* __restrict__ cp, const int32_t* __restrict__ rw,
                               const int64_t* __restrict__ newid, int64_t stride, uint64_t* __restrict__ keys,
                               int64_t* __restrict__ src) {
    const int lane = threadIdx.x & 31;
    for (int64_t j = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; j < ncols;
         j += (int64_t(gridDim.x) * blockDim.x) >> 5) {
        const uint64_t nj = (uint64_t)newid[j];
        for (int64_t p = cp[j] + lane; p < cp[j + 1]; p += 32) {
            keys[p] = nj * (uint64_t)stride + (uint64_t)newid[rw[p]];
            src[p] = p;
        }
    }
}
__global__ void k_gather_bytes(int64_t m, int vs, const int64_t* __restrict__ src, const unsigned char* __restrict__ in,
                               unsigned char* __restrict__ out) {
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < m; e += int64_t(gridDim.x) * blockDim.x)
        for (int b = 0; b < vs; ++b) out[e * vs + b] = in[src[e] * vs + b];
}
__global__ void k_shift_colptr(int64_t n, const int64_t* __restrict__ in, int64_t base, int64_t* __restrict__ out) {
    for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j <= n; j += int64_t(gridDim.x) * blockDim.x)
        out[j] = in[j] - base;
}

namespace {

int blocks_for(Ctx& c, int64_t work, int block = 256) {
    int64_t g = ceil_div(std::max<int64_t>(work, 1), block);
    return (int)std::min<int64_t>(g, int64_t(c.num_sms) * 16);
}

void sort_keys(Ctx& c, uint64_t* keys, uint64_t* keys_alt, int64_t m, int end_bit) {
    cub::DoubleBuffer<uint64_t> db(keys, keys_alt);
    size_t tb = 0;
    SLAPCU_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, db, m, 0, end_bit, c.stream));
    DevBuf tmp(tb, c.stream);
    SLAPCU_CUDA(cub::DeviceRadixSort::SortKeys(tmp.get(), tb, db, m, 0, end_bit, c.stream));
    ++c.launches;
    if (db.Current() != keys)
        SLAPCU_CUDA(cudaMemcpyAsync(keys, db.Current(), sizeof(uint64_t) * m, cudaMemcpyDeviceToDevice, c.stream));
}

template <class V>
void sort_pairs(Ctx& c, uint64_t* keys, uint64_t* keys_alt, V* vals, V* vals_alt, int64_t m, int end_bit) {
    cub::DoubleBuffer<uint64_t> dk(keys, keys_alt);
    cub::DoubleBuffer<V> dv(vals, vals_alt);
    size_t tb = 0;
    SLAPCU_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, dk, dv, m, 0, end_bit, c.stream));
    DevBuf tmp(tb, c.stream);
    SLAPCU_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), tb, dk, dv, m, 0, end_bit, c.stream));
    ++c.launches;
    if (dk.Current() != keys)
        SLAPCU_CUDA(cudaMemcpyAsync(keys, dk.Current(), sizeof(uint64_t) * m, cudaMemcpyDeviceToDevice, c.stream));
    if (dv.Current() != vals)
        SLAPCU_CUDA(cudaMemcpyAsync(vals, dv.Current(), sizeof(V) * m, cudaMemcpyDeviceToDevice, c.stream));
}

int bits_for(uint64_t maxkey) {
    int b = 1;
    while (b < 64 && (maxkey >> b)) ++b;
    return b;
}

// keep the first of each run of equal keys (stable: lowest draw index first)
int64_t unique_by_key(Ctx& c, const uint64_t* keys, const int64_t* vals, uint64_t* okeys, int64_t* ovals, int64_t m) {
    DevBuf nsel(sizeof(int64_t), c.stream);
    size_t tb = 0;
    SLAPCU_CUDA(cub::DeviceSelect::UniqueByKey(nullptr, tb, keys, vals, okeys, ovals, nsel.as<int64_t>(), m, c.stream));
    DevBuf tmp(tb, c.stream);
    SLAPCU_CUDA(
        cub::DeviceSelect::UniqueByKey(tmp.get(), tb, keys, vals, okeys, ovals, nsel.as<int64_t>(), m, c.stream));
    ++c.launches;
    int64_t h = 0;
    SLAPCU_CUDA(cudaMemcpyAsync(&h, nsel.get(), sizeof(int64_t), cudaMemcpyDeviceToHost, c.stream));
    SLAPCU_CUDA(cudaStreamSynchronize(c.stream));
    return h;
}

void alloc_out(Ctx& c, slapcu_csc_out* out, int64_t nrows, int64_t ncols, int64_t nnz, int vs) {
    out->nrows = nrows;
    out->ncols = ncols;
    out->nnz = nnz;
    SLAPCU_CUDA(cudaMallocAsync((void**)&out->colptr, sizeof(int64_t) * (ncols + 1), c.stream));
    SLAPCU_CUDA(cudaMallocAsync((void**)&out->rowids, sizeof(int32_t) * std::max<int64_t>(nnz, 1), c.stream));
    out->vals = nullptr;
    if (vs) SLAPCU_CUDA(cudaMallocAsync(&out->vals, size_t(vs) * std::max<int64_t>(nnz, 1), c.stream));
}

}  // namespace

void gen_rmat(Ctx& c, int scale, int ef, uint64_t seed, double a, double b, double cc, double d, slapcu_csc_out* out) {
    KScope ks(c, KC_GEN);
    (void)d;
    if (scale < 1 || scale > 30) throw Fail{SLAPCU_ERR_SHAPE, "rmat scale must be in 1..30"};
    if (std::abs(a + b + cc + d - 1.0) > 1e-12) throw Fail{SLAPCU_ERR_SHAPE, "rmat quadrant probabilities must sum to 1"};
    const int64_t n = int64_t(1) << scale;
    const int64_t edges = int64_t(ef) * n;
    const int64_t m2 = 2 * edges;
    DevBuf k1(sizeof(uint64_t) * std::max<int64_t>(m2, 1), c.stream), k2(sizeof(uint64_t) * std::max<int64_t>(m2, 1), c.stream);
    launch(c, k_rmat_edges, dim3(blocks_for(c, edges)), dim3(256), 0, scale, edges, seed, a, a + b, a + b + cc,
           k1.as<uint64_t>());
    sort_keys(c, k1.as<uint64_t>(), k2.as<uint64_t>(), m2, 2 * scale);
    // unique keys (values unused: reuse unique_by_key with dummy indices)
    DevBuf nsel(sizeof(int64_t), c.stream);
    size_t tb = 0;
    SLAPCU_CUDA(cub::DeviceSelect::Unique(nullptr, tb, k1.as<uint64_t>(), k2.as<uint64_t>(), nsel.as<int64_t>(), m2,
                                          c.stream));
    DevBuf tmp(tb, c.stream);
    SLAPCU_CUDA(cub::DeviceSelect::Unique(tmp.get(), tb, k1.as<uint64_t>(), k2.as<uint64_t>(), nsel.as<int64_t>(), m2,
                                          c.stream));
    ++c.launches;
    int64_t mu = 0;
    SLAPCU_CUDA(cudaMemcpyAsync(&mu, nsel.get(), sizeof(int64_t), cudaMemcpyDeviceToHost, c.stream));
    SLAPCU_CUDA(cudaStreamSynchronize(c.stream));
    // drop the trailing invalid marker
    const uint64_t invalid = (1ull << (2 * scale)) - 1ull;
    uint64_t last = 0;
    if (mu > 0) {
        SLAPCU_CUDA(cudaMemcpyAsync(&last, k2.as<uint64_t>() + mu - 1, sizeof(uint64_t), cudaMemcpyDeviceToHost, c.stream));
        SLAPCU_CUDA(cudaStreamSynchronize(c.stream));
        if (last == invalid) --mu;
    }
    alloc_out(c, out, n, n, mu, 0);
    launch(c, k_keys_to_csc, dim3(blocks_for(c, std::max(mu, n + 1))), dim3(256), 0, mu, n, n,
           (const uint64_t*)k2.as<uint64_t>(), out->colptr, out->rowids);
    SLAPCU_CUDA(cudaStreamSynchronize(c.stream));
}

void gen_er(Ctx& c, int64_t n, int64_t draws, uint64_t seed, bool with_values, slapcu_csc_out* out) {
    KScope ks(c, KC_GEN);
    if (n <= 0 || n > INT32_MAX) throw Fail{SLAPCU_ERR_SHAPE, "ER dimension out of range"};
    const uint64_t st0 = mix64(seed * kGolden + 0 + 1);
    DevBuf k1(sizeof(uint64_t) * std::max<int64_t>(draws, 1), c.stream), k2(sizeof(uint64_t) * std::max<int64_t>(draws, 1), c.stream);
    DevBuf v1(sizeof(int64_t) * std::max<int64_t>(draws, 1), c.stream), v2(sizeof(int64_t) * std::max<int64_t>(draws, 1), c.stream);
    launch(c, k_er_draws, dim3(blocks_for(c, draws)), dim3(256), 0, draws, n, st0, k1.as<uint64_t>(), v1.as<int64_t>());
    const int eb = bits_for((uint64_t)n * (uint64_t)n);
    sort_pairs<int64_t>(c, k1.as<uint64_t>(), k2.as<uint64_t>(), v1.as<int64_t>(), v2.as<int64_t>(), draws, eb);
    const int64_t mu = unique_by_key(c, k1.as<uint64_t>(), v1.as<int64_t>(), k2.as<uint64_t>(), v2.as<int64_t>(), draws);
    alloc_out(c, out, n, n, mu, with_values ? 8 : 0);
    launch(c, k_keys_to_csc, dim3(blocks_for(c, std::max(mu, n + 1))), dim3(256), 0, mu, n, n,
           (const uint64_t*)k2.as<uint64_t>(), out->colptr, out->rowids);
    if (with_values)
        launch(c, k_er_values, dim3(blocks_for(c, mu)), dim3(256), 0, mu, st0, (const int64_t*)v2.as<int64_t>(),
               static_cast<double*>(out->vals));
    SLAPCU_CUDA(cudaStreamSynchronize(c.stream));
}

void gen_one_per_row(Ctx& c, int64_t n, int64_t ncols, uint64_t seed, slapcu_csc_out* out) {
    KScope ks(c, KC_GEN);
    if (n <= 0 || n > INT32_MAX || ncols <= 0) throw Fail{SLAPCU_ERR_SHAPE, "one-per-row dims out of range"};
    const uint64_t st0 = mix64(seed * kGolden + 0 + 1);
    DevBuf k1(sizeof(uint64_t) * n, c.stream), k2(sizeof(uint64_t) * n, c.stream);
    launch(c, k_opr_draws, dim3(blocks_for(c, n)), dim3(256), 0, n, ncols, st0, k1.as<uint64_t>());
    sort_keys(c, k1.as<uint64_t>(), k2.as<uint64_t>(), n, bits_for((uint64_t)ncols * (uint64_t)n));
    alloc_out(c, out, n, ncols, n, 8);
    launch(c, k_keys_to_csc, dim3(blocks_for(c, n + 1)), dim3(256), 0, n, ncols, n, (const uint64_t*)k1.as<uint64_t>(),
           out->colptr, out->rowids);
    launch(c, k_opr_values, dim3(blocks_for(c, n)), dim3(256), 0, n, st0, (const int32_t*)out->rowids,
           static_cast<double*>(out->vals));
    SLAPCU_CUDA(cudaStreamSynchronize(c.stream));
}

void fill_values(Ctx& c, int sr, int kind, const DevCsc& m, void* vals) {
    KScope ks(c, KC_GEN);
    const int g = blocks_for(c, m.ncols * 32);
    switch (value_size(sr)) {
    case 1: launch(c, k_fill_values<uint8_t>, dim3(g), dim3(256), 0, m.ncols, m.cp, m.rw, kind, 0, (uint8_t*)vals); break;
    case 4:
        if (sr == SLAPCU_PLUS_TIMES_F32)
            launch(c, k_fill_values<float>, dim3(g), dim3(256), 0, m.ncols, m.cp, m.rw, kind, 1, (float*)vals);
        else
            launch(c, k_fill_values<int32_t>, dim3(g), dim3(256), 0, m.ncols, m.cp, m.rw, kind, 0, (int32_t*)vals);
        break;
    case 8:
        if (sr == SLAPCU_PLUS_TIMES_I64)
            launch(c, k_fill_values<int64_t>, dim3(g), dim3(256), 0, m.ncols, m.cp, m.rw, kind, 0, (int64_t*)vals);
        else
            launch(c, k_fill_values<double>, dim3(g), dim3(256), 0, m.ncols, m.cp, m.rw, kind, 0, (double*)vals);
        break;
    default: throw Fail{SLAPCU_ERR_INVALID, "unknown semiring"};
    }
}

void column_checksums(Ctx& c, const DevCsc& m, int sr, bool with_values, uint64_t* sums) {
    KScope ks(c, KC_GEN);
    const int vs = (with_values && m.v) ? value_size(sr) : 0;
    launch(c, k_column_checksums, dim3(blocks_for(c, m.ncols * 32)), dim3(256), 0, m.ncols, m.cp, m.rw,
           (const unsigned char*)m.v, vs, sums);
}

void permute_symmetric(Ctx& c, const DevCsc& A, uint64_t seed, int sr, slapcu_csc_out* out) {
    KScope ks(c, KC_GEN);
    if (A.nrows != A.ncols) throw Fail{SLAPCU_ERR_SHAPE, "symmetric permutation needs a square matrix"};
    const int64_t n = A.nrows, m = A.nnz;
    const int vs = A.v ? value_size(sr) : 0;
    DevBuf pk(sizeof(uint64_t) * n, c.stream), pk2(sizeof(uint64_t) * n, c.stream);
    DevBuf ids(sizeof(int64_t) * n, c.stream), ids2(sizeof(int64_t) * n, c.stream), newid(sizeof(int64_t) * n, c.stream);
    launch(c, k_perm_keys, dim3(blocks_for(c, n)), dim3(256), 0, n, seed, pk.as<uint64_t>(), ids.as<int64_t>());
    sort_pairs<int64_t>(c, pk.as<uint64_t>(), pk2.as<uint64_t>(), ids.as<int64_t>(), ids2.as<int64_t>(), n, 64);
    launch(c, k_invert, dim3(blocks_for(c, n)), dim3(256), 0, n, (const int64_t*)ids.as<int64_t>(), newid.as<int64_t>());
    DevBuf k1(sizeof(uint64_t) * std::max<int64_t>(m, 1), c.stream), k2(sizeof(uint64_t) * std::max<int64_t>(m, 1), c.stream);
    DevBuf s1(sizeof(int64_t) * std::max<int64_t>(m, 1), c.stream), s2(sizeof(int64_t) * std::max<int64_t>(m, 1), c.stream);
    launch(c, k_perm_entries, dim3(blocks_for(c, A.ncols * 32)), dim3(256), 0, A.ncols, A.cp, A.rw,
           (const int64_t*)newid.as<int64_t>(), n, k1.as<uint64_t>(), s1.as<int64_t>());
    sort_pairs<int64_t>(c, k1.as<uint64_t>(), k2.as<uint64_t>(), s1.as<int64_t>(), s2.as<int64_t>(), m,
                        bits_for((uint64_t)n * (uint64_t)n));
    alloc_out(c, out, n, n, m, vs);
    launch(c, k_keys_to_csc, dim3(blocks_for(c, std::max(m, n + 1))), dim3(256), 0, m, n, n,
           (const uint64_t*)k1.as<uint64_t>(), out->colptr, out->rowids);
    if (vs)
        launch(c, k_gather_bytes, dim3(blocks_for(c, m)), dim3(256), 0, m, vs, (const int64_t*)s1.as<int64_t>(),
               (const unsigned char*)A.v, (unsigned char*)out->vals);
    SLAPCU_CUDA(cudaStreamSynchronize(c.stream));
}

void slice_cols(Ctx& c, const DevCsc& B, int sr, int64_t c0, int64_t c1, slapcu_csc_out* out) {
    KScope ks(c, KC_GEN);
    if (c0 < 0 || c1 < c0 || c1 > B.ncols) throw Fail{SLAPCU_ERR_INDEX, "column slice out of range"};
    int64_t lo = 0, hi = 0;
    SLAPCU_CUDA(cudaMemcpyAsync(&lo, B.cp + c0, sizeof(int64_t), cudaMemcpyDeviceToHost, c.stream));
    SLAPCU_CUDA(cudaMemcpyAsync(&hi, B.cp + c1, sizeof(int64_t), cudaMemcpyDeviceToHost, c.stream));
    SLAPCU_CUDA(cudaStreamSynchronize(c.stream));
    const int vs = B.v ? value_size(sr) : 0;
    alloc_out(c, out, B.nrows, c1 - c0, hi - lo, vs);
    launch(c, k_shift_colptr, dim3(blocks_for(c, c1 - c0 + 1)), dim3(256), 0, c1 - c0, B.cp + c0, lo, out->colptr);
    if (hi > lo) {
        SLAPCU_CUDA(cudaMemcpyAsync(out->rowids, B.rw + lo, sizeof(int32_t) * (hi - lo), cudaMemcpyDeviceToDevice, c.stream));
        if (vs)
            SLAPCU_CUDA(cudaMemcpyAsync(out->vals, (const char*)B.v + size_t(vs) * lo, size_t(vs) * (hi - lo),
                                        cudaMemcpyDeviceToDevice, c.stream));
    }
    SLAPCU_CUDA(cudaStreamSynchronize(c.stream));
}

}  // namespace slapcu
