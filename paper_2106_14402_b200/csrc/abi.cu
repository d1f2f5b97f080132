// abi.cu -- the extern "C" boundary (include/slapcu.h).  Exceptions never
// cross it: every entry point maps slapcu::Fail onto a status code and keeps
// the message in the context (slapcu_ctx_last_error).
#include <cstdlib>
#include <cstring>
#include <new>

#include "ctx.hpp"

struct slapcu_ctx_s {
    slapcu::Ctx c;
};

namespace slapcu {

Ctx& ctx_of(slapcu_ctx c) { return c->c; }

namespace {

template <class F>
slapcu_status guarded(slapcu_ctx ctx, F&& f) {
    if (!ctx) return SLAPCU_ERR_INVALID;
    try {
        SLAPCU_CUDA(cudaSetDevice(ctx->c.device));
        ctx_settle(ctx->c);  // surface a deferred error of an asynchronous finish()
        f(ctx->c);
        ctx->c.last_error.clear();
        return SLAPCU_OK;
    } catch (const Fail& e) {
        ctx->c.last_error = e.msg;
        return e.st;
    } catch (const std::bad_alloc&) {
        ctx->c.last_error = "host allocation failed";
        return SLAPCU_ERR_NOMEM;
    } catch (const std::exception& e) {
        ctx->c.last_error = e.what();
        return SLAPCU_ERR_INTERNAL;
    }
}

void require(bool ok, slapcu_status st, const char* msg) {
    if (!ok) throw Fail{st, msg};
}

void alloc_csc_out(Ctx& c, slapcu_csc_out* C, int64_t nrows, int64_t ncols, int64_t nnz, int vs) {
    C->nrows = nrows;
    C->ncols = ncols;
    C->nnz = nnz;
    C->colptr = nullptr;
    C->rowids = nullptr;
    C->vals = nullptr;
    SLAPCU_CUDA(cudaMallocAsync((void**)&C->colptr, sizeof(int64_t) * (ncols + 1), c.stream));
    SLAPCU_CUDA(cudaMallocAsync((void**)&C->rowids, sizeof(int32_t) * std::max<int64_t>(nnz, 1), c.stream));
    SLAPCU_CUDA(cudaMallocAsync(&C->vals, size_t(vs) * std::max<int64_t>(nnz, 1), c.stream));
}

}  // namespace
}  // namespace slapcu

using namespace slapcu;

extern "C" {

int slapcu_abi_version(void) { return SLAPCU_ABI_VERSION; }

const char* slapcu_status_name(slapcu_status s) {
    switch (s) {
    case SLAPCU_OK: return "Ok";
    case SLAPCU_ERR_DIM: return "DimError";
    case SLAPCU_ERR_SHAPE: return "ShapeError";
    case SLAPCU_ERR_INTERNAL: return "InternalError";
    case SLAPCU_ERR_NAME: return "NameError";
    case SLAPCU_ERR_BUDGET: return "BudgetError";
    case SLAPCU_ERR_INDEX: return "IndexError";
    case SLAPCU_ERR_INVALID: return "InvalidArgument";
    case SLAPCU_ERR_CUDA: return "CudaError";
    case SLAPCU_ERR_NOMEM: return "OutOfMemory";
    case SLAPCU_ERR_COMM: return "DeadlockError";
    case SLAPCU_ERR_IO: return "IoError";
    case SLAPCU_ERR_FORMAT: return "FormatError";
    case SLAPCU_ERR_STOCHASTIC: return "StochasticityError";
    }
    return "Unknown";
}

slapcu_status slapcu_ctx_create(slapcu_ctx* out, int device, void* stream) {
    if (!out) return SLAPCU_ERR_INVALID;
    *out = nullptr;
    slapcu_ctx ctx = new (std::nothrow) slapcu_ctx_s;
    if (!ctx) return SLAPCU_ERR_NOMEM;
    ctx->c.device = device;
    ctx->c.stream = static_cast<cudaStream_t>(stream);
    slapcu_status st = guarded(ctx, [&](Ctx& c) {
        SLAPCU_CUDA(cudaDeviceGetAttribute(&c.smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
        SLAPCU_CUDA(cudaDeviceGetAttribute(&c.num_sms, cudaDevAttrMultiProcessorCount, device));
        for (auto& e : c.ev) SLAPCU_CUDA(cudaEventCreate(&e));
        // keep freed workspace cached in the stream-ordered pool
        cudaMemPool_t pool;
        SLAPCU_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
        uint64_t thr = UINT64_MAX;
        SLAPCU_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    });
    if (st != SLAPCU_OK) {
        delete ctx;
        return st;
    }
    *out = ctx;
    return SLAPCU_OK;
}

slapcu_status slapcu_ctx_destroy(slapcu_ctx ctx) {
    if (!ctx) return SLAPCU_ERR_INVALID;
    cudaSetDevice(ctx->c.device);
    cudaStreamSynchronize(ctx->c.stream);
    for (auto& e : ctx->c.ev)
        if (e) cudaEventDestroy(e);
    if (ctx->c.err_host) cudaFreeHost(ctx->c.err_host);
    free_host_cache(ctx->c);
    const int dev = ctx->c.device;
    delete ctx;  // (its workspace goes back to the device's stream-ordered pool ...)
    // ... and the pool, which keeps freed memory cached while contexts work
    // (release threshold = max), returns what no allocation holds to the device
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        cudaDeviceSynchronize();
        cudaMemPoolTrimTo(pool, 0);
    }
    return SLAPCU_OK;
}

slapcu_status slapcu_ctx_synchronize(slapcu_ctx ctx) {
    return guarded(ctx, [&](Ctx& c) { SLAPCU_CUDA(cudaStreamSynchronize(c.stream)); });
}

slapcu_status slapcu_ctx_invalidate(slapcu_ctx ctx) {
    return guarded(ctx, [&](Ctx& c) {
        c.direct.atp_valid = false;
        c.direct.atpv_valid = false;
        c.direct.aw_valid = false;
        c.plan.valid = false;
    });
}

slapcu_status slapcu_ctx_set_stream(slapcu_ctx ctx, void* stream) {
    return guarded(ctx, [&](Ctx& c) { c.stream = static_cast<cudaStream_t>(stream); });
}

const char* slapcu_ctx_last_error(slapcu_ctx ctx) { return ctx ? ctx->c.last_error.c_str() : "null context"; }

slapcu_status slapcu_ctx_set_option(slapcu_ctx ctx, slapcu_option opt, int64_t v) {
    return guarded(ctx, [&](Ctx& c) {
        switch (opt) {
        case SLAPCU_OPT_TILE_ROWS_LOG2:
            require(v >= 10 && v <= 20, SLAPCU_ERR_INVALID, "tile rows log2 must be in 10..20");
            c.opt.tile_rows_log2 = (int)v;
            break;
        case SLAPCU_OPT_SYM_TILE_ROWS_LOG2:
            require(v >= 10 && v <= 20, SLAPCU_ERR_INVALID, "symbolic tile rows log2 must be in 10..20");
            c.opt.sym_tile_rows_log2 = (int)v;
            break;
        case SLAPCU_OPT_LIGHT_NNZ_MAX: c.opt.light_nnz_max = v; break;
        case SLAPCU_OPT_DIRECT_TILE_ROWS_LOG2:
            require(v == 0 || (v >= 10 && v <= 18), SLAPCU_ERR_INVALID, "direct tile rows log2: 0 (auto) or 10..18");
            c.opt.direct_tile_rows_log2 = (int)v;
            break;
        // retired experiments (measured slower, removed in round 2): only the default is accepted
        case SLAPCU_OPT_DIRECT_MARK_MODE:
            require(v == 0, SLAPCU_ERR_INVALID, "mark mode: removed (0 = test-then-set, summary by ballots)");
            break;
        case SLAPCU_OPT_DIRECT_PERSISTENT: c.opt.direct_persistent = v != 0; break;
        case SLAPCU_OPT_DIRECT_TILE_MAJOR: c.opt.direct_tile_major = v != 0; break;
        case SLAPCU_OPT_DIRECT_FORM_WALK:
            require(v == 0, SLAPCU_ERR_INVALID, "form walk: removed (0 = 256-element units)");
            break;
        case SLAPCU_OPT_DIRECT_WORDS: c.opt.direct_words = v != 0; break;
        case SLAPCU_OPT_DIRECT_VALUE_DENSE_ROWS:
            require(v == 0 || (v >= 4096 && v <= 32768 && v % 4096 == 0), SLAPCU_ERR_INVALID,
                    "value dense rows: 0 (= rank chunk) or a multiple of 4096 up to 32768");
            c.opt.direct_value_dense_rows = (int)v;
            break;
        // retired (measured slower, round 2): only the default is accepted
        case SLAPCU_OPT_DIRECT_VALUE_L2: require(v == 0, SLAPCU_ERR_INVALID, "value L2 folds: removed"); break;
        case SLAPCU_OPT_DIRECT_VALUE_DENSE_ONLY:
            require(v == 0, SLAPCU_ERR_INVALID, "dense-only value chunks: removed");
            break;
        case SLAPCU_OPT_DIRECT_VALUE_TMAJOR: c.opt.direct_value_tmajor = v != 0; break;
        case SLAPCU_OPT_DIRECT_VALUE_ROWS: c.opt.direct_value_rows = v != 0; break;
        case SLAPCU_OPT_DIRECT_VALUE_TINY_RUN:
            require(v >= -1 && v <= 64, SLAPCU_ERR_INVALID, "value tiny run: -1 (default) or 0..64");
            c.opt.direct_value_tiny_run = (int)v;
            break;
        case SLAPCU_OPT_DIRECT_VALUE_FORM:
            require(v == -1 || v == 0 || (v >= 12 && v <= 15), SLAPCU_ERR_INVALID,
                    "value form tile rows log2: -1 (auto), 0 (off) or 12..15");
            c.opt.direct_value_form = (int)v;
            break;
        case SLAPCU_OPT_DIRECT_SHORT_RUN:
            require(v >= 0 && v <= 256, SLAPCU_ERR_INVALID, "short run threshold: 0 (default) .. 256");
            c.opt.direct_short_run = (int)v;
            break;
        case SLAPCU_OPT_DIRECT_QUADS: require(v == 0, SLAPCU_ERR_INVALID, "quads: removed"); break;
        case SLAPCU_OPT_DIRECT_VALUE_TILE_ROWS_LOG2:
            require(v >= 10 && v <= 15, SLAPCU_ERR_INVALID, "value tile rows log2 must be in 10..15");
            c.opt.direct_value_tile_log2 = (int)v;
            break;
        case SLAPCU_OPT_SUMMA_CONCAT: c.opt.summa_concat = v != 0; break;
        case SLAPCU_OPT_DIRECT_VALUE_RANK:
            require(v == 0 || (v >= 4096 && v <= 16384), SLAPCU_ERR_INVALID, "value rank chunk: 0 or 4096..16384");
            c.opt.direct_value_rank = (int)v;
            break;
        case SLAPCU_OPT_DIRECT_VALUE_INTERLEAVE:
            require(v >= 0 && v <= 2, SLAPCU_ERR_INVALID, "value interleave: 0, 1 or 2");
            c.opt.direct_value_interleave = (int)v;
            break;
        case SLAPCU_OPT_DIRECT_VALUE_HASH:
            require(v == 0 || v == 1 || v == 13 || v == 14, SLAPCU_ERR_INVALID, "value hash: 0, 1, 13 or 14");
            c.opt.direct_value_hash = (int)v;
            break;
        case SLAPCU_OPT_DIRECT_VALUE_THREADS:
            require(v == 256 || v == 512, SLAPCU_ERR_INVALID, "value threads: 256 or 512");
            c.opt.direct_value_threads = (int)v;
            break;
        case SLAPCU_OPT_DIRECT_FORM_THREADS:
            require(v == 128 || v == 256 || v == 512, SLAPCU_ERR_INVALID, "form threads: 128, 256 or 512");
            c.opt.direct_form_threads = (int)v;
            break;
        case SLAPCU_OPT_DIRECT_EMIT_THREADS:
            require(v == 0 || v == 128, SLAPCU_ERR_INVALID, "emit: one 128-thread CTA per item (warp-per-block removed)");
            break;
        case SLAPCU_OPT_DIRECT_DENSE_RUN_MIN:
            require(v >= 0, SLAPCU_ERR_INVALID, "dense run threshold must be >= 0");
            c.opt.direct_dense_run_min = v;
            break;
        case SLAPCU_OPT_DIRECT_SPLIT_FLOPS:
            require(v >= 1024, SLAPCU_ERR_INVALID, "split threshold must be >= 1024");
            c.opt.direct_split_flops = v;
            break;
        case SLAPCU_OPT_LIGHT_FLOPS_MAX:
            c.opt.light_flops_max = v;
            c.opt.direct_light_flops_max = v;
            break;
        case SLAPCU_OPT_DETERMINISTIC: c.opt.deterministic = v != 0; break;
        case SLAPCU_OPT_DIRECT_ESC:
            require(v >= -1 && v <= 1, SLAPCU_ERR_INVALID, "ESC: -1 (auto), 0 (off) or 1 (always)");
            c.opt.direct_esc = (int)v;
            break;
        case SLAPCU_OPT_DENSE_FLOPS_MIN: c.opt.dense_flops_min = v; break;
        case SLAPCU_OPT_ASYNC_FINISH: c.opt.async_finish = v != 0; break;
        case SLAPCU_OPT_DENSE_TILE_ROWS_LOG2:
            require(v >= 10 && v <= 17, SLAPCU_ERR_INVALID, "dense tile rows log2 must be in 10..17");
            c.opt.dense_tile_rows_log2 = (int)v;
            break;
        case SLAPCU_OPT_PROFILE:
            prof_flush(c);
            c.prof.on = v != 0;
            break;
        default: throw Fail{SLAPCU_ERR_INVALID, "unknown option"};
        }
    });
}

slapcu_status slapcu_ctx_kernel_stats(slapcu_ctx ctx, int cls, int64_t* launches, double* ms) {
    return guarded(ctx, [&](Ctx& c) {
        require(cls >= 0 && cls < KC_COUNT, SLAPCU_ERR_INVALID, "kernel class out of range");
        prof_flush(c);
        if (launches) *launches = c.prof.n[cls];
        if (ms) *ms = c.prof.ms[cls];
    });
}

slapcu_status slapcu_ctx_reset_stats(slapcu_ctx ctx) {
    return guarded(ctx, [&](Ctx& c) {
        prof_flush(c);
        for (int k = 0; k < KC_COUNT; ++k) {
            c.prof.ms[k] = 0.0;
            c.prof.n[k] = 0;
        }
    });
}

const char* slapcu_kernel_class_name(int cls) {
    static const char* names[KC_COUNT] = {"other", "flops", "bin", "sym_light", "sym_heavy",
                                          "scan", "num_light", "num_heavy", "merge", "gen"};
    return (cls >= 0 && cls < KC_COUNT) ? names[cls] : "unknown";
}

int64_t slapcu_ctx_kernel_launches(slapcu_ctx ctx) { return ctx ? ctx->c.launches : -1; }

slapcu_status slapcu_ctx_last_phase_ms(slapcu_ctx ctx, float* sym, float* num) {
    return guarded(ctx, [&](Ctx& c) {
        if (sym) *sym = c.sym_ms;
        if (num) *num = c.num_ms;
    });
}

int slapcu_semiring_value_size(slapcu_semiring sr) { return value_size(sr); }

slapcu_status slapcu_semiring_from_name(const char* name, const char* dtype, slapcu_semiring* out) {
    if (!name || !out) return SLAPCU_ERR_INVALID;
    const std::string n(name), d(dtype ? dtype : "");
    if (n == "plus_times" && (d == "f64" || d.empty())) *out = SLAPCU_PLUS_TIMES_F64;
    else if (n == "plus_times" && d == "f32") *out = SLAPCU_PLUS_TIMES_F32;
    else if (n == "plus_times" && d == "i64") *out = SLAPCU_PLUS_TIMES_I64;
    else if (n == "min_plus" && d == "i32") *out = SLAPCU_MIN_PLUS_I32;
    else if (n == "min_plus" && (d == "f64" || d.empty())) *out = SLAPCU_MIN_PLUS_F64;
    else if ((n == "or_and" || n == "boolean") && (d == "u8" || d == "bool" || d.empty())) *out = SLAPCU_OR_AND_U8;
    else return SLAPCU_ERR_NAME;
    return SLAPCU_OK;
}

slapcu_status slapcu_alg_from_name(const char* name, slapcu_alg* out) {
    if (!name || !out) return SLAPCU_ERR_INVALID;
    const std::string n(name);
    if (n == "heap") *out = SLAPCU_ALG_HEAP;
    else if (n == "hash") *out = SLAPCU_ALG_HASH;
    else if (n == "hybrid") *out = SLAPCU_ALG_HYBRID;
    else return SLAPCU_ERR_NAME;
    return SLAPCU_OK;
}

slapcu_status slapcu_estimate_flops(slapcu_ctx ctx, const slapcu_csc* A, const slapcu_csc* B, int64_t* flops_per_col,
                                    int64_t* total) {
    return guarded(ctx, [&](Ctx& c) {
        require(A && B, SLAPCU_ERR_INVALID, "null operand");
        spgemm_flops(c, view(*A), view(*B), flops_per_col, total);
    });
}

slapcu_status slapcu_spgemm_symbolic(slapcu_ctx ctx, const slapcu_csc* A, const slapcu_csc* B, slapcu_alg alg,
                                     int64_t* c_colptr, int64_t* c_nnz) {
    return guarded(ctx, [&](Ctx& c) {
        require(A && B && c_colptr, SLAPCU_ERR_INVALID, "null argument");
        const int64_t nnz = spgemm_symbolic(c, view(*A), view(*B), alg, c_colptr);
        if (c_nnz) *c_nnz = nnz;
    });
}

slapcu_status slapcu_spgemm_numeric(slapcu_ctx ctx, const slapcu_csc* A, const slapcu_csc* B, slapcu_semiring sr,
                                    slapcu_alg alg, const int64_t* c_colptr, int32_t* c_rowids, void* c_vals) {
    return guarded(ctx, [&](Ctx& c) {
        require(A && B && c_colptr, SLAPCU_ERR_INVALID, "null argument");
        spgemm_numeric(c, view(*A), view(*B), sr, alg, c_colptr, c_rowids, c_vals);
    });
}

slapcu_status slapcu_spgemm_begin(slapcu_ctx ctx, const slapcu_csc* A, const slapcu_csc* B, slapcu_semiring sr,
                                  slapcu_alg alg, int64_t staging_budget_bytes, int64_t* c_colptr, int64_t* c_nnz) {
    return guarded(ctx, [&](Ctx& c) {
        require(A && B && c_colptr, SLAPCU_ERR_INVALID, "null argument");
        const int64_t nnz = fused_begin(c, view(*A), view(*B), sr, alg, c_colptr, staging_budget_bytes);
        if (c_nnz) *c_nnz = nnz;
    });
}

slapcu_status slapcu_spgemm_finish(slapcu_ctx ctx, const slapcu_csc* A, const slapcu_csc* B, slapcu_semiring sr,
                                   int32_t* c_rowids, void* c_vals) {
    return guarded(ctx, [&](Ctx& c) {
        require(A && B, SLAPCU_ERR_INVALID, "null argument");
        fused_finish(c, view(*A), view(*B), sr, c_rowids, c_vals);
    });
}

slapcu_status slapcu_spgemm_direct(slapcu_ctx ctx, const slapcu_csc* A, const slapcu_csc* B, slapcu_semiring sr,
                                   slapcu_alg alg, int64_t capacity, int64_t* c_colptr, int32_t* c_rowids,
                                   void* c_vals, int64_t* c_nnz) {
    if (ctx) ctx->c.direct.last_nnz = -1;
    const slapcu_status st = guarded(ctx, [&](Ctx& c) {
        require(A && B && c_colptr, SLAPCU_ERR_INVALID, "null argument");
        require(capacity >= 0, SLAPCU_ERR_INVALID, "negative capacity");
        c.direct.last_nnz = direct_spgemm(c, view(*A), view(*B), sr, alg, capacity, c_colptr, c_rowids, c_vals);
    });
    if (ctx && c_nnz) *c_nnz = ctx->c.direct.last_nnz;
    return st;
}

// Largest staging area the one-shot call will take: half the free device memory.
static int64_t default_staging_budget(Ctx& c) { return int64_t(device_available(c) / 2); }

slapcu_status slapcu_spgemm(slapcu_ctx ctx, const slapcu_csc* A, const slapcu_csc* B, slapcu_semiring sr,
                            slapcu_alg alg, slapcu_csc_out* C) {
    return guarded(ctx, [&](Ctx& c) {
        require(A && B && C, SLAPCU_ERR_INVALID, "null argument");
        const int vs = value_size(sr);
        require(vs > 0, SLAPCU_ERR_INVALID, "unknown semiring");
        const DevCsc a = view(*A), b = view(*B);
        // production path: one product pass into an exactly sized C
        int64_t nnz = 0;
        int64_t* dcp = nullptr;
        int32_t* drw = nullptr;
        void* dv = nullptr;
        if (direct_exact(c, a, b, sr, alg, default_staging_budget(c), &dcp, &drw, &dv, &nnz)) {
            C->nrows = a.nrows;
            C->ncols = b.ncols;
            C->nnz = nnz;
            C->colptr = dcp;
            C->rowids = drw;
            C->vals = dv;
            return;
        }
        int64_t* cp = nullptr;
        SLAPCU_CUDA(cudaMallocAsync((void**)&cp, sizeof(int64_t) * (b.ncols + 1), c.stream));
        bool fused = true;
        try {
            try {
                nnz = fused_begin(c, a, b, sr, alg, cp, default_staging_budget(c));
            } catch (const Fail& e) {
                if (e.st != SLAPCU_ERR_BUDGET) throw;
                fused = false;  // staging does not fit: two-pass path needs none
                nnz = spgemm_symbolic(c, a, b, alg, cp);
            }
        } catch (...) {
            cudaFreeAsync(cp, c.stream);
            throw;
        }
        C->nrows = a.nrows;
        C->ncols = b.ncols;
        C->nnz = nnz;
        C->colptr = cp;
        C->rowids = nullptr;
        C->vals = nullptr;
        SLAPCU_CUDA(cudaMallocAsync((void**)&C->rowids, sizeof(int32_t) * std::max<int64_t>(nnz, 1), c.stream));
        SLAPCU_CUDA(cudaMallocAsync(&C->vals, size_t(vs) * std::max<int64_t>(nnz, 1), c.stream));
        if (fused)
            fused_finish(c, a, b, sr, C->rowids, C->vals);
        else
            spgemm_numeric(c, a, b, sr, alg, cp, C->rowids, C->vals);
    });
}

slapcu_status slapcu_device_count(int* n) {
    if (!n) return SLAPCU_ERR_INVALID;
    *n = 0;
    if (cudaGetDeviceCount(n) != cudaSuccess) {
        cudaGetLastError();
        *n = 0;
    }
    return SLAPCU_OK;
}

slapcu_status slapcu_csc_upload(slapcu_ctx ctx, const slapcu_host_csc* h, slapcu_semiring sr, slapcu_csc_out* d) {
    return guarded(ctx, [&](Ctx& c) {
        require(h && d, SLAPCU_ERR_INVALID, "null argument");
        const int vs = value_size(sr);
        require(vs > 0, SLAPCU_ERR_INVALID, "unknown semiring");
        alloc_csc_out(c, d, h->nrows, h->ncols, h->nnz, vs);
        SLAPCU_CUDA(cudaMemcpyAsync(d->colptr, h->colptr, sizeof(int64_t) * (h->ncols + 1), cudaMemcpyHostToDevice,
                                    c.stream));
        if (h->nnz) {
            SLAPCU_CUDA(cudaMemcpyAsync(d->rowids, h->rowids, sizeof(int32_t) * h->nnz, cudaMemcpyHostToDevice, c.stream));
            if (h->vals)
                SLAPCU_CUDA(cudaMemcpyAsync(d->vals, h->vals, size_t(vs) * h->nnz, cudaMemcpyHostToDevice, c.stream));
        }
        SLAPCU_CUDA(cudaStreamSynchronize(c.stream));
    });
}

slapcu_status slapcu_dcsc_upload(slapcu_ctx ctx, int64_t nrows, int64_t ncols, int64_t nzc, const int32_t* jc,
                                 const int32_t* cp, const int32_t* rowids, const void* vals, slapcu_semiring sr,
                                 slapcu_csc_out* d) {
    return guarded(ctx, [&](Ctx& c) {
        require(d && (nzc == 0 || (jc && cp)), SLAPCU_ERR_INVALID, "null argument");
        const int vs = value_size(sr);
        require(vs > 0, SLAPCU_ERR_INVALID, "unknown semiring");
        const int64_t nnz = nzc ? cp[nzc] : 0;
        alloc_csc_out(c, d, nrows, ncols, nnz, vs);
        DevBuf djc(sizeof(int32_t) * std::max<int64_t>(nzc, 1), c.stream),
            dcp(sizeof(int32_t) * (nzc + 1), c.stream);
        if (nzc) {
            SLAPCU_CUDA(cudaMemcpyAsync(djc.get(), jc, sizeof(int32_t) * nzc, cudaMemcpyHostToDevice, c.stream));
            SLAPCU_CUDA(cudaMemcpyAsync(dcp.get(), cp, sizeof(int32_t) * (nzc + 1), cudaMemcpyHostToDevice, c.stream));
        } else {
            SLAPCU_CUDA(cudaMemsetAsync(dcp.get(), 0, sizeof(int32_t), c.stream));
        }
        // local_matrix.hpp:88-150 (jc, cp) -> dense colptr on the device
        dcsc_colptr(c, ncols, nzc, djc.as<int32_t>(), dcp.as<int32_t>(), d->colptr);
        if (nnz) {
            SLAPCU_CUDA(cudaMemcpyAsync(d->rowids, rowids, sizeof(int32_t) * nnz, cudaMemcpyHostToDevice, c.stream));
            if (vals) SLAPCU_CUDA(cudaMemcpyAsync(d->vals, vals, size_t(vs) * nnz, cudaMemcpyHostToDevice, c.stream));
        }
        SLAPCU_CUDA(cudaStreamSynchronize(c.stream));
    });
}

slapcu_status slapcu_csc_download(slapcu_ctx ctx, const slapcu_csc* d, slapcu_semiring sr, slapcu_host_csc* h) {
    return guarded(ctx, [&](Ctx& c) {
        require(h && d, SLAPCU_ERR_INVALID, "null argument");
        const int vs = value_size(sr);
        require(vs > 0, SLAPCU_ERR_INVALID, "unknown semiring");
        DevCsc m = view(*d);
        resolve(c, m);
        *h = slapcu_host_csc{m.nrows, m.ncols, m.span, nullptr, nullptr, nullptr};
        h->colptr = static_cast<int64_t*>(std::malloc(sizeof(int64_t) * (m.ncols + 1)));
        h->rowids = static_cast<int32_t*>(std::malloc(sizeof(int32_t) * std::max<int64_t>(m.span, 1)));
        h->vals = std::malloc(size_t(vs) * std::max<int64_t>(m.span, 1));
        if (!h->colptr || !h->rowids || !h->vals) {
            slapcu_host_free(h);
            throw Fail{SLAPCU_ERR_NOMEM, "host allocation failed"};
        }
        SLAPCU_CUDA(cudaMemcpyAsync(h->colptr, m.cp, sizeof(int64_t) * (m.ncols + 1), cudaMemcpyDeviceToHost, c.stream));
        if (m.span) {
            SLAPCU_CUDA(cudaMemcpyAsync(h->rowids, m.rw + m.base, sizeof(int32_t) * m.span, cudaMemcpyDeviceToHost,
                                        c.stream));
            if (m.v)
                SLAPCU_CUDA(cudaMemcpyAsync(h->vals, static_cast<const char*>(m.v) + size_t(vs) * m.base,
                                            size_t(vs) * m.span, cudaMemcpyDeviceToHost, c.stream));
        }
        SLAPCU_CUDA(cudaStreamSynchronize(c.stream));
        for (int64_t j = 0; j <= m.ncols; ++j) h->colptr[j] -= m.base;
    });
}

// Pattern of a host CSC on the device (colptr + rowids; values are not read
// by estimate_flops / symbolic_nnz).
struct PatternUpload {
    DevBuf cp, rw;
    DevCsc m;
    PatternUpload(Ctx& c, const slapcu_host_csc& h)
        : cp(sizeof(int64_t) * (h.ncols + 1), c.stream), rw(sizeof(int32_t) * std::max<int64_t>(h.nnz, 1), c.stream) {
        SLAPCU_CUDA(cudaMemcpyAsync(cp.get(), h.colptr, sizeof(int64_t) * (h.ncols + 1), cudaMemcpyHostToDevice, c.stream));
        if (h.nnz)
            SLAPCU_CUDA(cudaMemcpyAsync(rw.get(), h.rowids, sizeof(int32_t) * h.nnz, cudaMemcpyHostToDevice, c.stream));
        m = DevCsc{h.nrows, h.ncols, h.nnz, cp.as<int64_t>(), rw.as<int32_t>(), nullptr};
    }
};

static void host_dims(const slapcu_host_csc* A, const slapcu_host_csc* B) {
    require(A && B, SLAPCU_ERR_INVALID, "null operand");
    if (A->ncols != B->nrows)
        throw Fail{SLAPCU_ERR_DIM, "spgemm inner dims: A is " + std::to_string(A->nrows) + "x" +
                                       std::to_string(A->ncols) + ", B is " + std::to_string(B->nrows) + "x" +
                                       std::to_string(B->ncols)};
}

slapcu_status slapcu_estimate_flops_host(slapcu_ctx ctx, const slapcu_host_csc* A, const slapcu_host_csc* B,
                                         int64_t* flops_per_col, int64_t* total) {
    return guarded(ctx, [&](Ctx& c) {
        host_dims(A, B);
        PatternUpload a(c, *A), b(c, *B);
        DevBuf fl(sizeof(int64_t) * std::max<int64_t>(B->ncols, 1), c.stream);
        int64_t tot = 0;
        spgemm_flops(c, a.m, b.m, fl.as<int64_t>(), &tot);
        if (flops_per_col && B->ncols)
            SLAPCU_CUDA(cudaMemcpyAsync(flops_per_col, fl.get(), sizeof(int64_t) * B->ncols, cudaMemcpyDeviceToHost,
                                        c.stream));
        SLAPCU_CUDA(cudaStreamSynchronize(c.stream));
        if (total) *total = tot;
    });
}

slapcu_status slapcu_symbolic_nnz_host(slapcu_ctx ctx, const slapcu_host_csc* A, const slapcu_host_csc* B,
                                       slapcu_alg alg, int64_t* counts) {
    return guarded(ctx, [&](Ctx& c) {
        host_dims(A, B);
        require(counts || B->ncols == 0, SLAPCU_ERR_INVALID, "null counts");
        PatternUpload a(c, *A), b(c, *B);
        DevBuf cp(sizeof(int64_t) * (B->ncols + 1), c.stream);
        spgemm_symbolic(c, a.m, b.m, alg, cp.as<int64_t>());
        std::vector<int64_t> h(size_t(B->ncols) + 1);
        SLAPCU_CUDA(cudaMemcpyAsync(h.data(), cp.get(), sizeof(int64_t) * (B->ncols + 1), cudaMemcpyDeviceToHost,
                                    c.stream));
        SLAPCU_CUDA(cudaStreamSynchronize(c.stream));
        for (int64_t j = 0; j < B->ncols; ++j) counts[j] = h[j + 1] - h[j];
    });
}

slapcu_status slapcu_batched_spgemm_host(slapcu_ctx ctx, const slapcu_host_csc* A, const slapcu_host_csc* B,
                                         slapcu_semiring sr, slapcu_alg alg, int nranges, const int64_t* col_ranges,
                                         int64_t budget_bytes, slapcu_batch_consumer consumer, void* user,
                                         int64_t* total_nnz) {
    int64_t tot = -1;
    const slapcu_status st = guarded(ctx, [&](Ctx& c) {
        require(A && B, SLAPCU_ERR_INVALID, "null argument");
        tot = batched_host(c, *A, *B, sr, alg, nranges, col_ranges, budget_bytes, consumer, user);
    });
    if (total_nnz) *total_nnz = tot;
    return st;
}

slapcu_status slapcu_spgemm_host(slapcu_ctx ctx, const slapcu_host_csc* A, const slapcu_host_csc* B,
                                 slapcu_semiring sr, slapcu_alg alg, slapcu_host_csc* C) {
    return guarded(ctx, [&](Ctx& c) {
        require(A && B && C, SLAPCU_ERR_INVALID, "null argument");
        const int vs = value_size(sr);
        require(vs > 0, SLAPCU_ERR_INVALID, "unknown semiring");
        if (A->ncols != B->nrows)
            throw Fail{SLAPCU_ERR_DIM, "spgemm inner dims: A is " + std::to_string(A->nrows) + "x" +
                                           std::to_string(A->ncols) + ", B is " + std::to_string(B->nrows) + "x" +
                                           std::to_string(B->ncols)};
        slapcu_csc_out dA{}, dB{};
        alloc_csc_out(c, &dA, A->nrows, A->ncols, A->nnz, vs);
        alloc_csc_out(c, &dB, B->nrows, B->ncols, B->nnz, vs);
        auto h2d = [&](void* d, const void* h, size_t n) {
            if (n) SLAPCU_CUDA(cudaMemcpyAsync(d, h, n, cudaMemcpyHostToDevice, c.stream));
        };
        h2d(dA.colptr, A->colptr, sizeof(int64_t) * (A->ncols + 1));
        h2d(dA.rowids, A->rowids, sizeof(int32_t) * A->nnz);
        h2d(dA.vals, A->vals, size_t(vs) * A->nnz);
        h2d(dB.colptr, B->colptr, sizeof(int64_t) * (B->ncols + 1));
        h2d(dB.rowids, B->rowids, sizeof(int32_t) * B->nnz);
        h2d(dB.vals, B->vals, size_t(vs) * B->nnz);
        slapcu_csc a{dA.nrows, dA.ncols, dA.nnz, dA.colptr, dA.rowids, dA.vals};
        slapcu_csc b{dB.nrows, dB.ncols, dB.nnz, dB.colptr, dB.rowids, dB.vals};
        slapcu_csc_out dC{};
        auto cleanup = [&]() {
            for (void* p : {(void*)dA.colptr, (void*)dA.rowids, dA.vals, (void*)dB.colptr, (void*)dB.rowids, dB.vals,
                            (void*)dC.colptr, (void*)dC.rowids, dC.vals})
                if (p) cudaFreeAsync(p, c.stream);
        };
        try {
            const DevCsc av = view(a), bv = view(b);
            int64_t nnz = 0;
            // entries are read back straight out of the product scratch (no device copy)
            int32_t* srw = nullptr;
            void* sv = nullptr;
            if (direct_exact(c, av, bv, sr, alg, default_staging_budget(c), &dC.colptr, &srw, &sv, &nnz, false)) {
                dC.rowids = nullptr;
                dC.vals = nullptr;
            } else {
                SLAPCU_CUDA(cudaMallocAsync((void**)&dC.colptr, sizeof(int64_t) * (bv.ncols + 1), c.stream));
                nnz = spgemm_symbolic(c, av, bv, alg, dC.colptr);
                SLAPCU_CUDA(cudaMallocAsync((void**)&dC.rowids, sizeof(int32_t) * std::max<int64_t>(nnz, 1), c.stream));
                SLAPCU_CUDA(cudaMallocAsync(&dC.vals, size_t(vs) * std::max<int64_t>(nnz, 1), c.stream));
                spgemm_numeric(c, av, bv, sr, alg, dC.colptr, dC.rowids, dC.vals);
            }
            C->nrows = av.nrows;
            C->ncols = bv.ncols;
            C->nnz = nnz;
            C->colptr = static_cast<int64_t*>(std::malloc(sizeof(int64_t) * (bv.ncols + 1)));
            C->rowids = static_cast<int32_t*>(std::malloc(sizeof(int32_t) * std::max<int64_t>(nnz, 1)));
            C->vals = std::malloc(size_t(vs) * std::max<int64_t>(nnz, 1));
            if (!C->colptr || !C->rowids || !C->vals) throw std::bad_alloc();
            SLAPCU_CUDA(cudaMemcpyAsync(C->colptr, dC.colptr, sizeof(int64_t) * (bv.ncols + 1), cudaMemcpyDeviceToHost,
                                        c.stream));
            if (nnz) {
                SLAPCU_CUDA(cudaMemcpyAsync(C->rowids, srw ? srw : dC.rowids, sizeof(int32_t) * nnz,
                                            cudaMemcpyDeviceToHost, c.stream));
                SLAPCU_CUDA(cudaMemcpyAsync(C->vals, srw ? sv : dC.vals, size_t(vs) * nnz, cudaMemcpyDeviceToHost,
                                            c.stream));
            }
            SLAPCU_CUDA(cudaStreamSynchronize(c.stream));
        } catch (...) {
            cleanup();
            throw;
        }
        cleanup();
    });
}

slapcu_status slapcu_mcl_step(slapcu_ctx ctx, const slapcu_csc* A, slapcu_semiring sr, double inflation,
                              double prune_threshold, slapcu_csc_out* C) {
    return guarded(ctx, [&](Ctx& c) {
        require(A && C, SLAPCU_ERR_INVALID, "null argument");
        *C = slapcu_csc_out{};
        mcl_step(c, view(*A), sr, inflation, prune_threshold, C);
    });
}

slapcu_status slapcu_csc_free(slapcu_ctx ctx, slapcu_csc_out* C) {
    return guarded(ctx, [&](Ctx& c) {
        if (!C) return;
        for (void* p : {(void*)C->colptr, (void*)C->rowids, C->vals})
            if (p) SLAPCU_CUDA(cudaFreeAsync(p, c.stream));
        C->colptr = nullptr;
        C->rowids = nullptr;
        C->vals = nullptr;
    });
}

void slapcu_host_free(slapcu_host_csc* C) {
    if (!C) return;
    std::free(C->colptr);
    std::free(C->rowids);
    std::free(C->vals);
    C->colptr = nullptr;
    C->rowids = nullptr;
    C->vals = nullptr;
}

slapcu_status slapcu_dcsc_colptr(slapcu_ctx ctx, int64_t ncols, int64_t nzc, const int32_t* jc, const int32_t* cp,
                                 int64_t* colptr) {
    return guarded(ctx, [&](Ctx& c) {
        require(cp && colptr && (nzc == 0 || jc), SLAPCU_ERR_INVALID, "null argument");
        dcsc_colptr(c, ncols, nzc, jc, cp, colptr);
    });
}

slapcu_status slapcu_merge_symbolic(slapcu_ctx ctx, int nparts, const slapcu_csc* parts, int64_t* c_colptr,
                                    int64_t* c_nnz) {
    return guarded(ctx, [&](Ctx& c) {
        require(parts && c_colptr && nparts >= 1, SLAPCU_ERR_INVALID, "bad merge arguments");
        std::vector<DevCsc> v(nparts);
        for (int s = 0; s < nparts; ++s) v[s] = view(parts[s]);
        const int64_t n = merge_symbolic(c, nparts, v.data(), c_colptr);
        if (c_nnz) *c_nnz = n;
    });
}

slapcu_status slapcu_merge_numeric(slapcu_ctx ctx, int nparts, const slapcu_csc* parts, slapcu_semiring sr,
                                   const int64_t* c_colptr, int32_t* c_rowids, void* c_vals) {
    return guarded(ctx, [&](Ctx& c) {
        require(parts && c_colptr && nparts >= 1, SLAPCU_ERR_INVALID, "bad merge arguments");
        std::vector<DevCsc> v(nparts);
        for (int s = 0; s < nparts; ++s) v[s] = view(parts[s]);
        merge_numeric(c, nparts, v.data(), sr, c_colptr, c_rowids, c_vals);
    });
}

slapcu_status slapcu_gen_rmat(slapcu_ctx ctx, int scale, int edge_factor, uint64_t seed, double a, double b, double cc,
                              double d, slapcu_csc_out* out) {
    return guarded(ctx, [&](Ctx& c) {
        require(out, SLAPCU_ERR_INVALID, "null output");
        gen_rmat(c, scale, edge_factor, seed, a, b, cc, d, out);
    });
}

slapcu_status slapcu_gen_er(slapcu_ctx ctx, int64_t n, int64_t draws, uint64_t seed, int with_values,
                            slapcu_csc_out* out) {
    return guarded(ctx, [&](Ctx& c) {
        require(out, SLAPCU_ERR_INVALID, "null output");
        gen_er(c, n, draws, seed, with_values != 0, out);
    });
}

slapcu_status slapcu_gen_one_per_row(slapcu_ctx ctx, int64_t n, int64_t ncols, uint64_t seed, slapcu_csc_out* out) {
    return guarded(ctx, [&](Ctx& c) {
        require(out, SLAPCU_ERR_INVALID, "null output");
        gen_one_per_row(c, n, ncols, seed, out);
    });
}

slapcu_status slapcu_fill_values(slapcu_ctx ctx, slapcu_semiring sr, int kind, const slapcu_csc* m, void* vals) {
    return guarded(ctx, [&](Ctx& c) {
        require(m && vals, SLAPCU_ERR_INVALID, "null argument");
        fill_values(c, sr, kind, view(*m), vals);
    });
}

slapcu_status slapcu_permute_symmetric(slapcu_ctx ctx, const slapcu_csc* A, uint64_t seed, slapcu_semiring sr,
                                       slapcu_csc_out* out) {
    return guarded(ctx, [&](Ctx& c) {
        require(A && out, SLAPCU_ERR_INVALID, "null argument");
        permute_symmetric(c, view(*A), seed, sr, out);
    });
}

slapcu_status slapcu_slice_cols(slapcu_ctx ctx, const slapcu_csc* B, slapcu_semiring sr, int64_t c0, int64_t c1,
                                slapcu_csc_out* out) {
    return guarded(ctx, [&](Ctx& c) {
        require(B && out, SLAPCU_ERR_INVALID, "null argument");
        slice_cols(c, view(*B), sr, c0, c1, out);
    });
}

slapcu_status slapcu_column_checksums(slapcu_ctx ctx, const slapcu_csc* m, slapcu_semiring sr, int with_values,
                                      uint64_t* sums) {
    return guarded(ctx, [&](Ctx& c) {
        require(m && sums, SLAPCU_ERR_INVALID, "null argument");
        column_checksums(c, view(*m), sr, with_values != 0, sums);
    });
}

}  // extern "C"
