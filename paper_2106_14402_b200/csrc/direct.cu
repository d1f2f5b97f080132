// direct.cu -- single product pass that writes C in place.
//
// The reference forms C in two passes, symbolic counts then numeric fill
// (spgemm.hpp:286-330), so every product is walked twice.  fused.cu walks
// once but stages every output row id and copies it into place: 8 extra bytes
// of HBM traffic per output entry, more than C itself (5 bytes for OrAnd).
// Here heavy columns are cut into (column, row tile) ITEMS and the product
// walk is decoupled from placement through a compact per-item stash:
//
//   A tile pointers  Atp[k][t] = first position of A(:,k) with row >= t*R
//                    (per A, cached): an item walks exactly its rows of every
//                    A(:,k), k in B(:,j) -- no cursors, no searches.
//   form   (k_tile_form)  one CTA per work unit, heaviest first: shared-memory
//                    bitmap of the tile (test-before-set atomics), then the
//                    item's count and its stash in the smaller of two forms:
//                    the whole bitmap (R/8 bytes) or the list of non-zero
//                    words (6 bytes each).  Items with more than `split`
//                    multiplies are cut by B entries into equal-flops parts
//                    whose partial bitmaps are OR-ed by k_tile_combine.
//   place  item offsets = exclusive scan of item counts (C order) + the light
//                    prefix of the column; colptr = scan of per-column counts.
//   emit   (k_tile_emit)  one CTA per item: expands the stash into sorted row
//                    ids written straight into C (coalesced), values 1.
//   light columns (flops <= L) use the shared hash of fused.cu, staged; they
//                    hold ~1% of C and are copied into place at the end.
//
// Stash traffic at R-MAT scale 16/20 is ~0.8 bytes per output entry (C's
// words are dense: ~7 entries per touched 32-row word), against 8 for
// staging row ids.  Pattern semirings only (OrAnd with all-one operands);
// other semirings go through fused.cu with the same contract.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "kern.cuh"

namespace slapcu {

namespace {

#ifndef SLAPCU_SHORT_RUN
#define SLAPCU_SHORT_RUN 8  // measured best of 4..64 on C3 (form 103.6 -> 100.7 ms)
#endif
constexpr int kShortRun = SLAPCU_SHORT_RUN;  // runs shorter than this are walked by one thread
#ifndef SLAPCU_UNIT
#define SLAPCU_UNIT 256
#endif
constexpr int kUnit = SLAPCU_UNIT;  // products per warp work unit on long runs
#ifndef SLAPCU_FORM_U
#define SLAPCU_FORM_U 4  // loads in flight per lane on long runs
#endif

__host__ __device__ __forceinline__ int64_t lmin(int64_t a, int64_t b) { return a < b ? a : b; }

constexpr int kEmitWPL = 4;                    // stash words per lane in a warp block
constexpr int kEmitBlock = 32 * kEmitWPL;      // words per warp block
constexpr int kEmitStage = 1024;               // entries per staging round
constexpr int kRbcWords = 128;                 // value pass: row blocks of 128 words (4096 rows)
constexpr int kMaxBlocks = 128;                // W / kEmitBlock for row tiles up to 2^19 (emit holds 4 x 32)

// Every item's stash starts with a header of per-block output counts (one
// int per kEmitBlock words of the stash body), so the emitter needs no
// counting pass; padded to 16 bytes.
__host__ __device__ __forceinline__ int stash_header_words(int W) {
    const int nb = (W + kEmitBlock - 1) / kEmitBlock;
    return (nb + 3) & ~3;
}

// Exclusive block-wide scan of one int per thread; *total gets the sum.
template <int NT>
__device__ __forceinline__ int block_excl_scan(int v, int* wsum, int* total) {
    constexpr int NW = NT / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int wt;
    const int ex = warp_excl_scan(v, lane, &wt);
    if (lane == 0) wsum[warp] = wt;
    __syncthreads();
    if (warp == 0) {
        const int x = lane < NW ? wsum[lane] : 0;
        int t;
        const int e = warp_excl_scan(x, lane, &t);
        if (lane < NW) wsum[lane] = e;
        if (lane == 0) wsum[NW] = t;
    }
    __syncthreads();
    const int r = ex + wsum[warp];
    *total = wsum[NW];
    __syncthreads();
    return r;
}

template <int NT>
struct WalkSm {
    int wsum[NT / 32 + 1];
    int ustart[NT + 1];
    int len[NT];
    int64_t start[NT];
    int ndense, nlong;
    int dense[NT];  // dense-run bitmap slots met in this batch of B entries
};

// Dense A runs: A(:,k) restricted to row tile t with at least `dmin` entries
// is kept (per A, cached) as a bitmap of the tile, so an item OR-s whole words
// (one coalesced load + one conflict-free shared update per 32 rows) instead
// of marking each product.  slot[k*T + t] = bitmap index or -1.
struct DenseRuns {
    const int* slot;
    const unsigned* bm;
    int dmin;  // 0: none
};

// Sets bits `b` of the bitmap word at shared address `a`, test before set: a
// plain shared load is a broadcast for lanes hitting one word, and most
// updates of a dense column find their bits already set (without the test:
// +20%, round 1).  The touched-word summary is rebuilt by ballots after the
// walk.  (No "memory" clobber: the bitmap is only read back after a
// __syncthreads, and a clobber would stop the compiler from issuing the next
// updates' global loads ahead of these shared updates.)
__device__ __forceinline__ void set_bits(unsigned a, unsigned b) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t.reg .b32 x;\n\t"
        "ld.shared.u32 x, [%0];\n\t"
        "and.b32 x, x, %1;\n\t"
        "setp.ne.u32 p, x, %1;\n\t"
        "@p red.shared.or.b32 [%0], %1;\n\t}" ::"r"(a),
        "r"(b));
}

// Marks absolute row rr (bmA: the bitmap base shifted by the tile origin).
__device__ __forceinline__ void mark(unsigned bmA, int rr) { set_bits(bmA + (unsigned(rr >> 5) << 2), 1u << (rr & 31)); }

// Marks a (32-row word, row mask) pair of the word form of A.
__device__ __forceinline__ void mark_word(unsigned bmA, int2 e) {
    set_bits(bmA + (unsigned(e.x) << 2), (unsigned)e.y);
}

// One element of a run: a row id (row form of A) or a (word, mask) pair
// (word form).
__device__ __forceinline__ void mark_el(unsigned bmA, int32_t r) { mark(bmA, r); }
__device__ __forceinline__ void mark_el(unsigned bmA, int2 e) { mark_word(bmA, e); }

// All updates of B entries [b0, b1) (column j) whose rows lie in tile t, into
// the tile bitmap.  A's elements are rows (ET = int32_t) or, in the word form
// (ET = int2), (32-row word, row mask) pairs: rows sharing a word cost one
// update -- at R-MAT s20 A*A the 70.1e9 multiplies are 36.9e9 word updates
// (runs of 512-4096 rows compress 1.9x).  Entries are taken NT at a time; a
// thread walks its own run when it is short, long runs are cut into units of
// kUnit elements that the warps walk lane-strided with U loads in flight
// (coalesced, balanced across warps; a warp's units are increasing, so the
// entry owning a unit is found by advancing, not searching).  Row-form runs of
// at least dr.dmin rows OR a cached tile bitmap instead.
// Tried and slower (same box): packing the long runs' elements evenly over the
// warps (101 -> 107 ms), a warp-independent walk without block barriers (101 ->
// 155 ms), lane-contiguous quads merged per word (+22%, round 1).
template <int NT, int U, class ET>
__device__ __forceinline__ void tile_walk(const ET* __restrict__ Ael, const int64_t* __restrict__ Acp, const DevCsc& B,
                                          const int32_t* __restrict__ Atp, int T, int64_t b0, int64_t b1, int t,
                                          int t0, unsigned* bm, WalkSm<NT>& sh, const DenseRuns& dr, int W,
                                          int short_run) {
    constexpr int NW = NT / 32;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned bm0 = smem_addr(bm);
    const unsigned bmA = bm0 - (unsigned(t0 >> 5) << 2);  // absolute rows / words index the tile directly
    // (sh.ndense and sh.nlong are zeroed by the caller before a barrier)
    for (int64_t base = b0; base < b1; base += NT) {
        const int64_t i = base + tid;
        if (i < b1) {
            const int k = B.rw[i];
            const int32_t* tp = Atp + int64_t(k) * (T + 1) + t;
            const int lo = tp[0], hi = tp[1];
            const int64_t s = Acp[k] + lo;
            const int len = hi - lo;
            if (dr.dmin && len >= dr.dmin) {
                sh.dense[atomicAdd(&sh.ndense, 1)] = dr.slot[int64_t(k) * T + t];
            } else if (len < short_run) {
                // (packing the short runs per warp, 32 elements per step with a shuffle
                // owner search, measured slower on the same box: form 83.8 -> 88.7 ms)
                // loads in groups of 4 so a short run is not a chain of L2 round trips
                const ET* q = Ael + s;
                int x = 0;
                for (; x + 4 <= len; x += 4) {
                    const ET e0 = __ldg(q + x), e1 = __ldg(q + x + 1), e2 = __ldg(q + x + 2), e3 = __ldg(q + x + 3);
                    mark_el(bmA, e0);
                    mark_el(bmA, e1);
                    mark_el(bmA, e2);
                    mark_el(bmA, e3);
                }
                for (; x < len; ++x) mark_el(bmA, __ldg(q + x));
            } else {
                // long run: into the compact list (order is irrelevant)
                const unsigned peers = __activemask();
                const int leader = __ffs(peers) - 1;
                int pos = 0;
                if (lane == leader) pos = atomicAdd(&sh.nlong, __popc(peers));
                pos = __shfl_sync(peers, pos, leader) + __popc(peers & ((1u << lane) - 1u));
                sh.len[pos] = len;
                sh.start[pos] = s;
            }
        }
        __syncthreads();
        const int nl = sh.nlong;
        const int units = tid < nl ? (sh.len[tid] + kUnit - 1) / kUnit : 0;
        int tot;
        const int ex = block_excl_scan<NT>(units, sh.wsum, &tot);
        sh.ustart[tid] = ex;
        if (tid == 0) sh.ustart[nl] = tot;
        __syncthreads();
        // warp w takes the contiguous unit range [u0, u1): one search for the
        // owning long run, then it only advances (every long run has units)
        const int u0 = (int)((int64_t(tot) * warp) / NW), u1 = (int)((int64_t(tot) * (warp + 1)) / NW);
        int e = 0;
        if (u0 < u1) {
            int lo = 0, hi = nl - 1;
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (sh.ustart[mid] <= u0)
                    lo = mid;
                else
                    hi = mid - 1;
            }
            e = lo;
        }
        for (int u = u0; u < u1; ++u) {
            if (sh.ustart[e + 1] <= u) ++e;
            const int c0 = (u - sh.ustart[e]) * kUnit;
            const ET* run = Ael + sh.start[e] + c0;
            const int m = min(kUnit, sh.len[e] - c0);
            int x = lane;
            for (; x + 32 * (U - 1) < m; x += 32 * U) {
                ET r[U];
#pragma unroll
                for (int v = 0; v < U; ++v) r[v] = __ldg(run + x + 32 * v);
#pragma unroll
                for (int v = 0; v < U; ++v) mark_el(bmA, r[v]);
            }
            // (tail one load per trip: issuing the tail's loads together, predicated,
            // measured slower on the same box, form 83.3 -> 86.2 ms)
            for (; x < m; x += 32) mark_el(bmA, __ldg(run + x));
        }
        // dense runs of this batch: OR whole words of their tile bitmaps
        const int nd = sh.ndense;
        for (int di = 0; di < nd; ++di) {
            const uint4* src = reinterpret_cast<const uint4*>(dr.bm + int64_t(sh.dense[di]) * W);
            for (int q = tid; q < (W >> 2); q += NT) {
                const uint4 v = __ldg(src + q);
                const unsigned a = bm0 + (unsigned(q) << 4);
                if (v.x) set_bits(a, v.x);
                if (v.y) set_bits(a + 4, v.y);
                if (v.z) set_bits(a + 8, v.z);
                if (v.w) set_bits(a + 12, v.w);
            }
        }
        __syncthreads();
        if (tid == 0) {
            sh.ndense = 0;
            sh.nlong = 0;
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------- form

struct FormArgs {
    DevCsc A, B;
    const int32_t* Atp;
    DenseRuns dr;
    int T, TL;
    const int2* items;      // (column, tile) in C order
    const int4* units;      // (item, b0, b1 relative to B.cp[j], partial slot or -1)
    const int* order;       // units, heaviest first
    unsigned* stash;        // per item: bitmap or word list
    const int64_t* soff;    // stash offset per item (words)
    const int64_t* sres;    // stash words reserved per item
    unsigned* partial;      // partial bitmaps of split items (W words per slot)
    int64_t* cnt;           // output entries per item
    int* form;              // -1 bitmap, else number of listed words
    unsigned long long* hcnt;  // output entries per column (heavy part)
    int* ticket;
    int nunits;
    int* rbc;  // per item entries per 4096-row block (value semirings), or null
    int short_run;  // runs shorter than this are walked by their own thread
    const int2* Aw;        // word form of A (words mode), or null
    const int64_t* Awcp;   // its column pointers
};

// Count, choose the stash form and write it, then clear the bitmap (whole
// CTA).  bm holds the item's tile bitmap and summ its touched-word summary
// (W/32 words); tl is shared scratch for W word indices.
template <int NT>
__device__ __forceinline__ void stash_bitmap(unsigned* bm, unsigned* summ, uint16_t* tl, int W, int* wsum, int* red,
                                             int* bcs, int64_t item, int j, unsigned* stash, int64_t sres,
                                             int64_t* cnt, int* form, unsigned long long* hcnt, int* rbc) {
    constexpr int NW = NT / 32;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int WS = W >> 5;
    if (rbc) {  // entries per 4096-row block (value pass sub-tile ranges)
        const int nrb = (W + kRbcWords - 1) / kRbcWords;
        for (int b = warp; b < nrb; b += NW) {
            int x = 0;
#pragma unroll
            for (int q = 0; q < kRbcWords / 32; ++q) {
                const int w = b * kRbcWords + q * 32 + lane;
                x += w < W ? __popc(bm[w]) : 0;
            }
            x = warp_reduce_sum(x);
            if (lane == 0) rbc[item * nrb + b] = x;
        }
    }
    // touched words in order: summary popcounts -> scan -> list (WS <= NT)
    unsigned sw = 0;
    if (tid < WS) {
        sw = summ[tid];
        summ[tid] = 0u;
    }
    int U;
    int base = block_excl_scan<NT>(__popc(sw), wsum, &U);
    while (sw) {
        tl[base++] = (uint16_t)(tid * 32 + __ffs(sw) - 1);
        sw &= sw - 1u;
    }
    __syncthreads();
    const int HB = stash_header_words(W);
    const int64_t lw = int64_t(U) + (U + 1) / 2;  // words + 16-bit word indices
    const bool list = lw < W && lw <= sres - HB;
    unsigned* body = stash + HB;
    int myc = 0;
    if (list) {
        // a warp covers 32 consecutive list positions: one warp sum per group
        uint16_t* idx = reinterpret_cast<uint16_t*>(body + U);
        for (int q0 = 0; q0 < U; q0 += NT) {
            const int q = q0 + tid;
            int c = 0;
            if (q < U) {
                const int w = tl[q];
                const unsigned x = bm[w];
                bm[w] = 0u;
                body[q] = x;
                idx[q] = (uint16_t)w;
                c = __popc(x);
            }
            myc += c;
            c = warp_reduce_sum(c);
            if (lane == 0 && c) atomicAdd(&bcs[(q0 + warp * 32) / kEmitBlock], c);
        }
    } else {
        // a warp covers 32 consecutive uint4 = one block of 128 words
        uint4* d4 = reinterpret_cast<uint4*>(body);
        uint4* s4 = reinterpret_cast<uint4*>(bm);
        for (int q0 = 0; q0 < W / 4; q0 += NT) {
            const int q = q0 + tid;
            int c = 0;
            if (q < W / 4) {
                const uint4 x = s4[q];
                d4[q] = x;
                s4[q] = make_uint4(0u, 0u, 0u, 0u);
                c = __popc(x.x) + __popc(x.y) + __popc(x.z) + __popc(x.w);
            }
            myc += c;
            c = warp_reduce_sum(c);
            if (lane == 0 && c) atomicAdd(&bcs[((q0 + warp * 32) * 4) / kEmitBlock], c);
        }
    }
    myc = warp_reduce_sum(myc);
    if (lane == 0) red[warp] = myc;
    __syncthreads();
    const int nb = ((list ? U : W) + kEmitBlock - 1) / kEmitBlock;
    for (int b = tid; b < nb; b += NT) {
        stash[b] = (unsigned)bcs[b];
        bcs[b] = 0;
    }
    if (tid == 0) {
        long long c = 0;
        for (int w = 0; w < NW; ++w) c += red[w];
        cnt[item] = c;
        form[item] = list ? U : -1;
        atomicAdd(&hcnt[j], (unsigned long long)c);
    }
}

// Persistent: each CTA takes work units (heaviest first) by ticket.
#ifdef SLAPCU_FORM_MINB
#define SLAPCU_FORM_BOUNDS __launch_bounds__(NT, SLAPCU_FORM_MINB)
#else
#define SLAPCU_FORM_BOUNDS __launch_bounds__(NT)
#endif
__host__ __device__ __forceinline__ size_t form_tail_offset(int W) {
    return (sizeof(unsigned) * size_t(W + W / 32) + 15) & ~size_t(15);
}

template <int NT, bool WORDS>
__global__ void SLAPCU_FORM_BOUNDS k_tile_form(FormArgs g) {
    extern __shared__ __align__(16) unsigned char sm_raw[];
    const int W = 1 << (g.TL - 5);
    unsigned* bm = reinterpret_cast<unsigned*>(sm_raw);
    unsigned* summ = bm + W;  // [W/32]
    // the stash's word list (after the walk) and the walk's batch state share
    // one region: 4 KB less shared memory per CTA, one more CTA per SM
    unsigned char* shared_tail = sm_raw + form_tail_offset(W);
    uint16_t* tl = reinterpret_cast<uint16_t*>(shared_tail);  // [W]
    WalkSm<NT>& sh = *reinterpret_cast<WalkSm<NT>*>(shared_tail);
    __shared__ int wsum2[NT / 32 + 1];
    __shared__ int red[NT / 32];
    __shared__ int ticket_sh;
    __shared__ int bcs[kMaxBlocks];
    smem_zero(bm, W + W / 32);
    for (int b = threadIdx.x; b < kMaxBlocks; b += NT) bcs[b] = 0;
    for (;;) {
        if (threadIdx.x == 0) {
            ticket_sh = atomicAdd(g.ticket, 1);
            sh.ndense = 0;
            sh.nlong = 0;
        }
        __syncthreads();
        const int ui = ticket_sh;
        if (ui >= g.nunits) break;
        const int4 u = g.units[g.order[ui]];
        const int2 it = g.items[u.x];
        const int64_t bs = g.B.cp[it.x];
        if constexpr (WORDS)
            tile_walk<NT, SLAPCU_FORM_U, int2>(g.Aw, g.Awcp, g.B, g.Atp, g.T, bs + u.y, bs + u.z, it.y, it.y << g.TL, bm, sh,
                                   DenseRuns{nullptr, nullptr, 0}, W, g.short_run);
        else
            tile_walk<NT, SLAPCU_FORM_U, int32_t>(g.A.rw, g.A.cp, g.B, g.Atp, g.T, bs + u.y, bs + u.z, it.y, it.y << g.TL, bm, sh,
                                      g.dr, W, g.short_run);
        if (u.w < 0) {  // summary by ballots over the bitmap
            const int lane = threadIdx.x & 31;
            for (int cc = threadIdx.x >> 5; cc < W / 32; cc += NT / 32) {
                const unsigned nz = __ballot_sync(0xffffffffu, bm[cc * 32 + lane] != 0u);
                if (lane == 0) summ[cc] = nz;
            }
            __syncthreads();
        }
        if (u.w >= 0) {  // one part of a split item: partial bitmap out, then clear
            uint4* d4 = reinterpret_cast<uint4*>(g.partial + int64_t(u.w) * W);
            uint4* s4 = reinterpret_cast<uint4*>(bm);
            for (int q = threadIdx.x; q < W / 4; q += NT) {
                d4[q] = s4[q];
                s4[q] = make_uint4(0u, 0u, 0u, 0u);
            }
            for (int q = threadIdx.x; q < W / 32; q += NT) summ[q] = 0u;
        } else {
            stash_bitmap<NT>(bm, summ, tl, W, wsum2, red, bcs, u.x, it.x, g.stash + g.soff[u.x], g.sres[u.x], g.cnt,
                             g.form, g.hcnt, g.rbc);
        }
        __syncthreads();
    }
}

// OR of the partial bitmaps of each split item -> its stash (bitmap or list).
template <int NT>
__global__ void __launch_bounds__(NT)
    k_tile_combine(int TL, const int2* __restrict__ items, const int* __restrict__ sitems,
                   const int* __restrict__ spart, const int* __restrict__ snp, const unsigned* __restrict__ partial,
                   unsigned* __restrict__ stash, const int64_t* __restrict__ soff, const int64_t* __restrict__ sres,
                   int64_t* __restrict__ cnt, int* __restrict__ form, unsigned long long* __restrict__ hcnt,
                   int* __restrict__ rbc) {
    constexpr int NW = NT / 32;
    extern __shared__ __align__(16) unsigned char sm_raw[];
    const int W = 1 << (TL - 5);
    unsigned* bm = reinterpret_cast<unsigned*>(sm_raw);
    unsigned* summ = bm + W;
    uint16_t* tl = reinterpret_cast<uint16_t*>(summ + W / 32);
    __shared__ int red[NW];
    __shared__ int wsum[NW + 1];
    __shared__ int bcs[kMaxBlocks];
    for (int b = threadIdx.x; b < kMaxBlocks; b += NT) bcs[b] = 0;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int item = sitems[blockIdx.x];
    const int np = snp[blockIdx.x];
    const unsigned* p0 = partial + int64_t(spart[blockIdx.x]) * W;
    for (int cc = warp; cc < W / 32; cc += NW) {
        const int w = cc * 32 + lane;
        unsigned x = 0;
        for (int p = 0; p < np; ++p) x |= p0[int64_t(p) * W + w];
        bm[w] = x;
        const unsigned nz = __ballot_sync(0xffffffffu, x != 0u);
        if (lane == 0) summ[cc] = nz;
    }
    __syncthreads();
    stash_bitmap<NT>(bm, summ, tl, W, wsum, red, bcs, item, items[item].x, stash + soff[item], sres[item], cnt, form,
                     hcnt, rbc);
}

// ------------------------------------------------------------------- emit

struct EmitArgs {
    const int2* items;
    const int64_t* cnt;
    const int* form;
    const unsigned* stash;
    const int64_t* soff;
    const int64_t* hoff;  // exclusive scan of cnt over items
    const int64_t* lp;    // light prefix per column
    int TL;
    int32_t* crw;
    uint8_t* cv;      // values written by emit (null: the value pass writes them)
    int vsize;        // bytes per value
    uint4 vpattern;   // 16 bytes of the value to write (1s for OrAnd)
    int nitems;
    const uint8_t* vst;    // value form: every item's values in row order (else null: vpattern)
    const int64_t* voff;   // their first entry per item
};

// Per-warp shared state of the emission.
struct EmitWarp {
    uint2 wr[kEmitBlock];         // the block's non-zero words (x) and their row bases (y), in order
    int stage[kEmitStage + 8];    // one round of outputs, co-aligned with the destination
};

// Rows of one warp block written to out[0, E) in order.  Lane l's non-zero
// words are ws->wr[pos, pos + nz) holding cnt set bits.  Outputs go in
// rounds of kEmitStage: lane l produces a contiguous run of `per` outputs
// (per odd, so the lanes' stage writes hit distinct banks) -- one search for
// its first word and bit, then it walks bits serially -- into a stage
// co-aligned with `out`, then the round is stored with 16-byte stores.
__device__ __forceinline__ void emit_block(EmitWarp* ws, int pos, int ex, int E, int32_t* __restrict__ out,
                                           int lane) {
    const int shift = (int)((reinterpret_cast<uintptr_t>(out) >> 2) & 3);
    for (int R0 = 0; R0 < E; R0 += kEmitStage) {
        const int RE = min(kEmitStage, E - R0);
        const int per = ((RE + 31) >> 5) | 1;
        const int my0 = R0 + min(lane * per, RE), my1 = R0 + min(lane * per + per, RE);
        // owner lane of output my0: the largest l with ex_l <= my0
        int src = 0;
#pragma unroll
        for (int step = 16; step > 0; step >>= 1) {
            const int cand = src + step;
            const int exc = __shfl_sync(0xffffffffu, ex, cand & 31);
            if (cand < 32 && exc <= my0) src = cand;
        }
        const int exs = __shfl_sync(0xffffffffu, ex, src);
        const int poss = __shfl_sync(0xffffffffu, pos, src);
        if (my0 < my1) {
            int k = my0 - exs;
            int wi = poss;
            uint2 cur = ws->wr[wi];
            for (;;) {  // word of the owner lane holding output my0 (all words non-zero)
                const int c = __popc(cur.x);
                if (k < c) break;
                k -= c;
                cur = ws->wr[++wi];
            }
            unsigned w = cur.x;
            if (k) w &= ~((1u << nth_set_bit(w, k)) - 1u);  // drop the k lowest set bits
            int rb = (int)cur.y;
            // pointer-stepped walk with a count-down (fewer address / compare
            // instructions per output than indexing by o)
            int* sp = ws->stage + shift - R0 + my0;
            const uint2* wp = &ws->wr[wi];
            int left = my1 - my0;
            // (loading the next word one step ahead measured slower: emit 39.8 -> 40.5 ms)
            do {
                if (w == 0u) {
                    const uint2 nw = *++wp;
                    w = nw.x;
                    rb = (int)nw.y;
                }
                *sp++ = rb + (__ffs(w) - 1);
                w &= w - 1u;
            } while (--left);
        }
        __syncwarp();
        // stage[shift + i] -> out[R0 + i]; both 16-byte aligned where (shift + i) % 4 == 0
        int32_t* dst = out + R0;
        const int h = min(RE, (4 - shift) & 3);
        if (lane < h) dst[lane] = ws->stage[shift + lane];
        const int nb = (RE - h) >> 2;
        const uint4* s4 = reinterpret_cast<const uint4*>(ws->stage + shift + h);
        uint4* d4 = reinterpret_cast<uint4*>(dst + h);
        for (int q = lane; q < nb; q += 32) d4[q] = s4[q];
        const int tl = h + (nb << 2);
        if (tl + lane < RE) dst[tl + lane] = ws->stage[shift + tl + lane];
        __syncwarp();
    }
}

// (__launch_bounds__(NT) alone: 56 registers; an explicit minimum of 1 block
// lets the compiler take 80 and emit loses 20% to occupancy; 12 spills)
#ifdef SLAPCU_EMIT_MINB
#define SLAPCU_EMIT_BOUNDS __launch_bounds__(NT, SLAPCU_EMIT_MINB)
#else
#define SLAPCU_EMIT_BOUNDS __launch_bounds__(NT)
#endif
template <int NT>
__global__ void SLAPCU_EMIT_BOUNDS k_tile_emit(EmitArgs g) {
    // one warp per item (NW items per CTA; default 1): most items stash 1-4
    // blocks of 128 words, so the warps of a multi-warp item CTA idled (4
    // warps per item 42.7 ms, 2: 40.9, 1: 39.1 at C3)
    constexpr int NW = NT / 32;
    __shared__ EmitWarp wsm[NW];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int item = blockIdx.x * NW + warp;
    if (item >= g.nitems) return;
    const int2 it = g.items[item];
    const int64_t c = g.cnt[item];
    const int64_t off = g.lp[it.x] + g.hoff[item];
    const int U = g.form[item];
    const int W = 1 << (g.TL - 5);
    const int nwords = U >= 0 ? U : W;
    const unsigned* hdr = g.stash + g.soff[item];
    const unsigned* words = hdr + stash_header_words(W);
    const uint16_t* idx = U >= 0 ? reinterpret_cast<const uint16_t*>(words + U) : nullptr;
    const int nblk = (nwords + kEmitBlock - 1) / kEmitBlock;
    const int t0 = it.y << g.TL;
    EmitWarp* ws = &wsm[warp];
    // block counts -> exclusive block bases, held as 4 registers per lane
    // (block b at lane b % 32, register b / 32; up to 128 blocks)
    int hv[4], hb[4];
    int run = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int bi = k * 32 + lane;
        hv[k] = bi < nblk ? (int)hdr[bi] : 0;
        int tot;
        hb[k] = run + warp_excl_scan(hv[k], lane, &tot);
        run += tot;
    }
    auto sel = [](const int (&r)[4], int k) { return k == 0 ? r[0] : k == 1 ? r[1] : k == 2 ? r[2] : r[3]; };
    // words of block b (4 per lane), prefetched one block ahead
    auto load = [&](int b, unsigned (&xs)[kEmitWPL], int (&wi)[kEmitWPL]) {
#pragma unroll
        for (int q = 0; q < kEmitWPL; ++q) {
            const int w = b * kEmitBlock + lane * kEmitWPL + q;
            const bool ok = b < nblk && w < nwords;
            xs[q] = ok ? words[w] : 0u;
            wi[q] = ok ? (idx ? (int)idx[w] : w) : 0;
        }
    };
    unsigned xs[kEmitWPL];
    int wi[kEmitWPL];
    load(0, xs, wi);
    for (int b = 0; b < nblk; ++b) {
        unsigned xn[kEmitWPL];
        int wn[kEmitWPL];
        load(b + 1, xn, wn);
        const int E = __shfl_sync(0xffffffffu, sel(hv, b >> 5), b & 31);
        const int bbase = __shfl_sync(0xffffffffu, sel(hb, b >> 5), b & 31);
        if (E) {
            int cnt = 0, nz = 0;
#pragma unroll
            for (int q = 0; q < kEmitWPL; ++q) {
                cnt += __popc(xs[q]);
                nz += xs[q] != 0u;
            }
            // one scan for both: set bits (<= 128 per lane) high, non-zero words low
            int tot;
            const int packed = warp_excl_scan((cnt << 16) | nz, lane, &tot);
            const int pos = packed & 0xffff, ex = packed >> 16;
            int p = pos;
#pragma unroll
            for (int q = 0; q < kEmitWPL; ++q) {
                if (xs[q]) {
                    ws->wr[p] = make_uint2(xs[q], (unsigned)(t0 + (wi[q] << 5)));
                    ++p;
                }
            }
            __syncwarp();
            emit_block(ws, pos, ex, E, g.crw + off + bbase, lane);
        }
#pragma unroll
        for (int q = 0; q < kEmitWPL; ++q) {
            xs[q] = xn[q];
            wi[q] = wn[q];
        }
    }
    if (g.cv && g.vst) {
        // values from the value form's stash (same order as the rows)
        if (c > 0) {
            const int64_t vo = g.voff[item];
            if (g.vsize == 4) {
                const unsigned* s = reinterpret_cast<const unsigned*>(g.vst) + vo;
                unsigned* d = reinterpret_cast<unsigned*>(g.cv) + off;
                for (int64_t q = lane; q < c; q += 32) d[q] = __ldg(s + q);
            } else if (g.vsize == 8) {
                const unsigned long long* s = reinterpret_cast<const unsigned long long*>(g.vst) + vo;
                unsigned long long* d = reinterpret_cast<unsigned long long*>(g.cv) + off;
                for (int64_t q = lane; q < c; q += 32) d[q] = __ldg(s + q);
            } else {
                for (int64_t q = lane; q < c * g.vsize; q += 32) g.cv[off * g.vsize + q] = g.vst[vo * g.vsize + q];
            }
        }
    } else if (g.cv) {
        // values: c copies of the pattern value (head elements, 16-byte body, tail elements)
        uint8_t* v = g.cv + off * g.vsize;
        const int64_t bytes = c * g.vsize;
        const int64_t head = lmin(bytes, (16 - (reinterpret_cast<uintptr_t>(v) & 15)) & 15);
        const uint4 pat = g.vpattern;
        auto pbyte = [pat](int b) {  // byte b of the 16-byte pattern (no address taken: no stack copy)
            const unsigned wd = b < 8 ? (b < 4 ? pat.x : pat.y) : (b < 12 ? pat.z : pat.w);
            return (uint8_t)(wd >> ((b & 3) * 8));
        };
        for (int64_t q = lane; q < head; q += 32) v[q] = pbyte((int)(q % g.vsize));
        const int64_t body = (bytes - head) >> 4;
        uint4* v4 = reinterpret_cast<uint4*>(v + head);
        for (int64_t q = lane; q < body; q += 32) v4[q] = pat;  // (head is a multiple of vsize)
        for (int64_t q = head + (body << 4) + lane; q < bytes; q += 32) v[q] = pbyte((int)(q % g.vsize));
    }
}

// ------------------------------------------------------------ value pass

// Values of the items for semirings with values (and OrAnd operands with
// stored zeros), after the emit pass has written C's rows.  One CTA per item;
// the item's tile is walked in sub-tiles of 2^VTL rows with a dense shared
// value array indexed by row (no ranks needed): every product of the
// sub-tile is folded in with the semiring's atomic, then the item's output
// entries that fall in the sub-tile (a contiguous range of C, found by
// binary search in its sorted rows) take their values and the touched slots
// are reset to the identity.  A second walk over the products -- the pattern
// walk (k_tile_form) only touches row ids.
struct ValueArgs {
    DevCsc A, B;
    const int32_t* Atpv;  // A tile pointers at 2^VTL rows
    int Tv, VTL, TL;
    const int32_t* Atp;   // A tile pointers at 2^TL rows (the items' tiles)
    int T;
    const int2* items;
    const int* list;      // the items this launch handles
    const int64_t* cnt;
    const int64_t* hoff;
    const int64_t* lp;
    const int* rbc;       // entries per 4096-row block of every item
    const int32_t* crw;
    void* cv;
    const void* arv;      // A's (row, value bits) interleaved (int2 for 4-byte, int4 for 8-byte values), or null
    int64_t tv_stride;    // > 0: Atpv is tile-major (entry (k, t) at t * tv_stride + k), else column-major
    int tiny;             // runs of at most this many products are folded by their own thread
    const unsigned* stash;  // the form pass's per-item stash (bitmap or word list), its offsets and forms
    const int64_t* soff;
    const int* form;
    int32_t* rows_out;      // rank chunks also write C's rows (the emit pass is skipped), or null
};

// One product's A row and value: from the interleaved copy when there is one
// (one 8-byte gather, one sector), else from the two arrays.
// (IL is resolved once per walk: a runtime test here was if-converted into
// both loads, predicated, on every product -- 7% of the value pass's issue)
template <bool IL, class T_>
__device__ __forceinline__ void load_prod(const int32_t* __restrict__ Arw, const T_* Av, const void* __restrict__ Arv,
                                          int64_t p, int& r, T_& a) {
    if constexpr (IL && sizeof(T_) == 4) {
        const int2 e = __ldg(static_cast<const int2*>(Arv) + p);
        r = e.x;
        memcpy(&a, &e.y, 4);
    } else if constexpr (IL && sizeof(T_) == 8) {  // (row, pad, value): one 16-byte load
        const int4 e = __ldg(static_cast<const int4*>(Arv) + p);
        r = e.x;
        const unsigned long long bits = (unsigned long long)(unsigned)e.z | ((unsigned long long)(unsigned)e.w << 32);
        memcpy(&a, &bits, 8);
    } else {
        r = __ldg(&Arw[p]);
        a = Av[p];
    }
}

__global__ void k_interleave_rv8(int64_t n, const int32_t* __restrict__ rw, const long long* __restrict__ v,
                                 int4* __restrict__ out) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const unsigned long long x = (unsigned long long)__ldg(v + i);
        out[i] = make_int4(__ldg(rw + i), 0, (int)(unsigned)x, (int)(unsigned)(x >> 32));
    }
}

__global__ void k_interleave_rv(int64_t n, const int32_t* __restrict__ rw, const int32_t* __restrict__ v,
                                int2* __restrict__ out) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        out[i] = make_int2(__ldg(rw + i), __ldg(v + i));
}

template <int SRID, int NT>
struct ValueWalkSm {
    using T = typename Sr<SRID>::T;
    int wsum[NT / 32 + 1];
    int ustart[NT + 1];
    int ulen[NT];
    int64_t ustartp[NT];
    T ubval[NT];
    int nlong;
};

// Warp shuffle of a semiring value (1-byte values travel as int).
template <class T_>
__device__ __forceinline__ T_ shfl_val(T_ v, int src) {
    if constexpr (sizeof(T_) < 4)
        return (T_)__shfl_sync(0xffffffffu, (int)v, src);
    else if constexpr (sizeof(T_) == 8 && !std::is_floating_point<T_>::value)
        return (T_)__shfl_sync(0xffffffffu, (long long)v, src);
    else
        return __shfl_sync(0xffffffffu, v, src);
}

// Every product of B(:,j) whose A row lies in tile `t` of the pointer table
// `tp0` (T+1 entries per A column) is handed to fold(row, product) -- for the
// value passes the semiring's atomic into *slot(row) (into<S_>(slot)).  Runs
// of >= 32 products are cut into 256-product warp units; shorter runs are
// packed 32 products per warp step (the owning B entry found by a search over
// the batch's product prefix), so no thread walks a run alone through a chain
// of dependent loads.
#ifndef SLAPCU_VTINY
#define SLAPCU_VTINY 0  // with the per-warp shuffle packing, runs of 1-2 pack too (MinPlus C3 413.8 -> 410.0 ms)
#endif
constexpr int kValueTinyRun = SLAPCU_VTINY;  // value walk: runs this short are folded by their own thread
#ifndef SLAPCU_VALUE_U
#define SLAPCU_VALUE_U 8  // MinPlus C3: 2 / 4 / 8 -> 469 / 454 / 443 ms (latency-bound gathers)
#endif
#ifndef SLAPCU_VALUE_UNIT
#define SLAPCU_VALUE_UNIT 128  // MinPlus C3 (same box): 128 / 256 / 512 -> 407.6 / 409.6 / 428.3 ms
#endif
constexpr int kValueU = SLAPCU_VALUE_U;        // value walk: products per lane per trip on long runs
constexpr int kValueUnit = SLAPCU_VALUE_UNIT;  // value walk: products per warp work unit on long runs
#ifdef SLAPCU_VCOUNT
// entry visits, nonempty runs, products, batches, products in rank / dense chunks,
// products in runs of <= 2 / 3..31 / >= 32 (debug variant)
__device__ unsigned long long g_vcount[12];
#endif
// (A test-then-min before the atomic -- skip products that do not lower the
// slot -- measured no faster on MinPlus C3: 445 -> 462 ms.)
template <class S_, class Slot>
struct AtomicInto {
    Slot slot;
    __device__ __forceinline__ void operator()(int r, typename S_::Acc v) const {
        typename S_::Acc* p = slot(r);
        S_::atomic_acc(p, v);
    }
};
template <class S_, class Slot>
__device__ __forceinline__ AtomicInto<S_, Slot> into(Slot s) {
    return AtomicInto<S_, Slot>{s};
}

template <int SRID, int NT, bool IL, class Fold>
__device__ __forceinline__ void value_walk_il(const DevCsc& A, const DevCsc& B, const int32_t* __restrict__ Atab, int T,
                                              int t, int j, ValueWalkSm<SRID, NT>& sh, Fold fold, int t_hi,
                                              const void* __restrict__ Arv, int64_t tstride, int vtag, int64_t eb0,
                                              int64_t eb1, int tiny) {
    using S_ = Sr<SRID>;
    using T_ = typename S_::T;
    constexpr int NW = NT / 32;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const T_* Av = static_cast<const T_*>(A.v);
    const T_* Bv = static_cast<const T_*>(B.v);
    const int32_t* __restrict__ Arw = A.rw;
    const int64_t bs = eb0 >= 0 ? eb0 : B.cp[j], be = eb0 >= 0 ? eb1 : B.cp[j + 1];
    for (int64_t base = bs; base < be; base += NT) {
        const int64_t i = base + tid;
        int slen = 0, units = 0;
        int64_t sst = 0;
        T_ sbv{};
        if (i < be) {
            const int k = B.rw[i];
            const int th = t_hi < 0 ? t + 1 : t_hi;  // tiles [t, th) of the table
            int rlo, rhi;
            if (tstride > 0) {  // tile-major table: a chunk's two rows are small and stay in L2
                rlo = __ldg(Atab + int64_t(t) * tstride + k);
                rhi = __ldg(Atab + int64_t(th) * tstride + k);
            } else {
                const int32_t* tp = Atab + int64_t(k) * (T + 1);
                rlo = tp[t];
                rhi = tp[th];
            }
            const int len = rhi - rlo;
#ifdef SLAPCU_VCOUNT
            atomicAdd(&g_vcount[0], 1ull);
            if (len > 0) atomicAdd(&g_vcount[1], 1ull);
            atomicAdd(&g_vcount[2], (unsigned long long)(len > 0 ? len : 0));
            if (tid == 0) atomicAdd(&g_vcount[3], 1ull);
            if (len > 0) {
                atomicAdd(&g_vcount[4 + vtag], (unsigned long long)len);
                atomicAdd(&g_vcount[len <= 2 ? 8 : len < 32 ? 9 : 10], (unsigned long long)len);
            }
#endif
            if (len > 0) {
                const int64_t st = A.cp[k] + rlo;
                const T_ bv = Bv[i];
                if (len <= tiny) {
                    // short run: folded by this thread, loads in groups of 4 in
                    // flight (no packing search -- 9 shared loads per product)
                    int x = 0;
                    for (; x + 4 <= len; x += 4) {
                        int r[4];
                        T_ a[4];
#pragma unroll
                        for (int v = 0; v < 4; ++v) load_prod<IL>(Arw, Av, Arv, st + x + v, r[v], a[v]);
#pragma unroll
                        for (int v = 0; v < 4; ++v) fold(r[v], S_::mul(a[v], bv));
                    }
                    for (; x < len; ++x) {
                        int r0;
                        T_ a0;
                        load_prod<IL>(Arw, Av, Arv, st + x, r0, a0);
                        fold(r0, S_::mul(a0, bv));
                    }
                } else if (len < 32) {
                    slen = len;
                    sst = st;
                    sbv = bv;
                } else {  // long run: this thread's slot of the batch
                    units = (len + kValueUnit - 1) / kValueUnit;
                    sh.ulen[tid] = len;
                    sh.ustartp[tid] = st;
                    sh.ubval[tid] = bv;
                }
            }
        }
        // packed short runs of this warp's entries, before the barrier: 32
        // products per warp step, the owner lane of product q found by a
        // 5-step search over the lanes' prefix (shuffles; lanes without a
        // packed run are skipped by <=)
        {
            int stot;
            const int ex = warp_excl_scan(slen, lane, &stot);
            for (int q0 = 0; q0 < stot; q0 += 32) {
                const int q = q0 + lane;
                int src = 0;
#pragma unroll
                for (int step = 16; step > 0; step >>= 1) {
                    const int cand = src + step;
                    const int exc = __shfl_sync(0xffffffffu, ex, cand & 31);
                    if (cand < 32 && exc <= q) src = cand;
                }
                const int exs = __shfl_sync(0xffffffffu, ex, src);
                const int64_t ss = (int64_t)__shfl_sync(0xffffffffu, (long long)sst, src);
                const T_ bb = shfl_val(sbv, src);
                if (q < stot) {
                    int r;
                    T_ av;
                    load_prod<IL>(Arw, Av, Arv, ss + (q - exs), r, av);
                    fold(r, S_::mul(av, bb));
                }
            }
        }
        // long runs: thread slots, unit prefix = warp scan + warp bases (two
        // barriers per batch of entries; the slot list needs no atomics or resets)
        int wtot;
        const int uex = warp_excl_scan(units, lane, &wtot);
        if (lane == 31) sh.wsum[warp] = wtot;
        __syncthreads();
        int wb = 0, tot = 0;
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            const int x = sh.wsum[w];
            wb += w < warp ? x : 0;
            tot += x;
        }
        sh.ustart[tid] = wb + uex;
        if (tid == 0) sh.ustart[NT] = tot;
        __syncthreads();
        const int u0 = (int)((int64_t(tot) * warp) / NW), u1 = (int)((int64_t(tot) * (warp + 1)) / NW);
        int e = 0;
        if (u0 < u1) {  // the slot owning unit u0: the last slot whose prefix is <= u0
            int a = 0, b = NT - 1;
            while (a < b) {
                const int mid = (a + b + 1) >> 1;
                if (sh.ustart[mid] <= u0)
                    a = mid;
                else
                    b = mid - 1;
            }
            e = a;
        }
        for (int u = u0; u < u1; ++u) {
            while (sh.ustart[e + 1] <= u) ++e;  // (slots without a long run hold no units)
            const int c0 = (u - sh.ustart[e]) * kValueUnit;
            const int64_t p0 = sh.ustartp[e] + c0;
            const int m = min(kValueUnit, sh.ulen[e] - c0);
            const T_ bv = sh.ubval[e];
            // kValueU products per lane per trip: independent gathers in flight
            for (int x = lane; x < m; x += 32 * kValueU) {
                int r[kValueU];
                T_ a[kValueU];
#pragma unroll
                for (int v = 0; v < kValueU; ++v) {
                    r[v] = -1;
                    if (x + 32 * v < m) load_prod<IL>(Arw, Av, Arv, p0 + x + 32 * v, r[v], a[v]);
                }
#pragma unroll
                for (int v = 0; v < kValueU; ++v)
                    if (r[v] >= 0) fold(r[v], S_::mul(a[v], bv));
            }
        }
        __syncthreads();  // (the next batch rewrites the slots; skipping this and the unit-prefix
                          // barrier for batches without long runs measured slower: 414 -> 424 ms,
                          // the double-buffered counts pushed the 40-register walk into spills)
    }
}

template <int SRID, int NT, class Fold>
__device__ __forceinline__ void value_walk(const DevCsc& A, const DevCsc& B, const int32_t* __restrict__ Atab, int T,
                                           int t, int j, ValueWalkSm<SRID, NT>& sh, Fold fold, int t_hi = -1,
                                           const void* __restrict__ Arv = nullptr, int64_t tstride = 0,
                                           int vtag = 0, int64_t eb0 = -1, int64_t eb1 = -1,
                                           int tiny = kValueTinyRun) {
    if (Arv)
        value_walk_il<SRID, NT, true>(A, B, Atab, T, t, j, sh, fold, t_hi, Arv, tstride, vtag, eb0, eb1, tiny);
    else
        value_walk_il<SRID, NT, false>(A, B, Atab, T, t, j, sh, fold, t_hi, Arv, tstride, vtag, eb0, eb1, tiny);
}

// Values of the large items: one CTA per (item, sub-tile of 2^VTL rows) with
// a dense shared value array indexed by row.  The sub-tile's output entries
// are a contiguous range of C (from the item's row-block counts); products
// only land on those rows, so only they are initialised.
template <int SRID, int NT>
__global__ void __launch_bounds__(NT) k_tile_values(ValueArgs g) {
    using S_ = Sr<SRID>;
    using T = typename S_::T;
    using Acc = typename S_::Acc;
    extern __shared__ __align__(16) unsigned char sm_raw[];
    Acc* val = reinterpret_cast<Acc*>(sm_raw);
    __shared__ ValueWalkSm<SRID, NT> sh;
    __shared__ int64_t range_sh[2];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nsub = 1 << (g.TL - g.VTL);
    const int item = g.list[blockIdx.x / nsub], s = blockIdx.x % nsub;
    const int2 it = g.items[item];
    const int j = it.x;
    const int ts = (it.y << (g.TL - g.VTL)) + s;
    const int s0 = ts << g.VTL;
    if (warp == 0) {  // this sub-tile's output entries C[lo, hi) from the row-block counts
        const int W = 1 << (g.TL - 5);
        const int nrb = (W + kRbcWords - 1) / kRbcWords;
        const int per = max(1, (1 << (g.VTL - 5)) / kRbcWords);  // row blocks per sub-tile
        const int* rb = g.rbc + int64_t(item) * nrb;
        int before = 0, inside = 0;
        for (int b = lane; b < nrb; b += 32) {
            const int x = rb[b];
            before += b < s * per ? x : 0;
            inside += (b >= s * per && b < (s + 1) * per) ? x : 0;
        }
        before = warp_reduce_sum(before);
        inside = warp_reduce_sum(inside);
        if (lane == 0) {
            const int64_t off = g.lp[j] + g.hoff[item];
            range_sh[0] = off + before;
            range_sh[1] = off + before + inside;
            sh.nlong = 0;
        }
    }
    __syncthreads();
    const int64_t lo = range_sh[0], hi = range_sh[1];
    if (lo == hi) return;
    for (int64_t q = lo + tid; q < hi; q += NT) val[g.crw[q] - s0] = S_::identity();
    __syncthreads();
    value_walk<SRID, NT>(g.A, g.B, g.Atpv, g.Tv, ts, j, sh, into<S_>([val, s0](int r) { return &val[r - s0]; }), -1,
                         g.arv, 0, 0, -1, -1, g.tiny);
    T* Cv = static_cast<T*>(g.cv);
    for (int64_t q = lo + tid; q < hi; q += NT) Cv[q] = S_::out(val[g.crw[q] - s0]);
}

// Values of the small items (at most HS/2 output entries): one CTA per item,
// one walk over its products, values in a shared open-addressing table keyed
// by the item's output rows (built first from C's rows, so a product only
// probes -- it never inserts).
template <int SRID, int NT, int LOG2HS>
__global__ void __launch_bounds__(NT) k_item_values_hash(ValueArgs g) {
    using S_ = Sr<SRID>;
    using T = typename S_::T;
    using Acc = typename S_::Acc;
    constexpr int HS = 1 << LOG2HS;
    extern __shared__ __align__(16) unsigned char sm_raw[];
    Acc* val = reinterpret_cast<Acc*>(sm_raw);
    int* key = reinterpret_cast<int*>(sm_raw + sizeof(Acc) * HS);
    __shared__ ValueWalkSm<SRID, NT> sh;
    const int tid = threadIdx.x;
    const int item = g.list[blockIdx.x];
    const int2 it = g.items[item];
    const int j = it.x;
    const int64_t off = g.lp[j] + g.hoff[item];
    const int64_t c = g.cnt[item];
    for (int q = tid; q < HS; q += NT) key[q] = -1;
    if (tid == 0) sh.nlong = 0;
    __syncthreads();
    auto home = [](int r) { return (int)(((unsigned)r * 0x9E3779B1u) >> (32 - LOG2HS)); };
    for (int64_t q = tid; q < c; q += NT) {
        const int r = g.crw[off + q];
        int h = home(r);
        while (atomicCAS(&key[h], -1, r) != -1) h = (h + 1) & (HS - 1);
        val[h] = S_::identity();
    }
    __syncthreads();
    auto slot = [key, val, home](int r) {
        int h = home(r);
        while (key[h] != r) h = (h + 1) & (HS - 1);
        return &val[h];
    };
    value_walk<SRID, NT>(g.A, g.B, g.Atp, g.T, it.y, j, sh, into<S_>(slot), -1, g.arv, 0, 0, -1, -1, g.tiny);
    T* Cv = static_cast<T*>(g.cv);
    for (int64_t q = tid; q < c; q += NT) Cv[off + q] = S_::out(*slot(g.crw[off + q]));
}

// Values of the large items by rank chunks: an item's 4096-row blocks are
// grouped greedily into chunks of at most `cap` output entries; one CTA per
// chunk rebuilds the chunk's row bitmap from C's rows, turns it into ranks
// (16-bit prefixes inside 32-word groups + group bases) and folds every
// product of the chunk's rows into a rank-indexed shared value array -- one
// walk over B(:,j) per chunk instead of one per fixed row sub-tile.
struct RankChunk {
    int item, b0, b1, pad;
};

template <int SRID, int NT>
// (3 CTAs per SM: the shared footprint allows 3 at 8192 4-byte slots; without the
// bound the compiler takes 51 registers and 512-thread CTAs drop to 2 per SM)
__global__ void __launch_bounds__(NT, 3) k_item_values_rank(ValueArgs g, const RankChunk* __restrict__ chunks, int cap,
                                                         int dense_rows) {
    using S_ = Sr<SRID>;
    using T = typename S_::T;
    using Acc = typename S_::Acc;
    constexpr int kBlkRows = kRbcWords * 32;  // 4096
    extern __shared__ __align__(16) unsigned char sm_raw[];
    const int W = 1 << (g.TL - 5);
    Acc* val = reinterpret_cast<Acc*>(sm_raw);
    unsigned* bm = reinterpret_cast<unsigned*>(sm_raw + ((sizeof(Acc) * size_t(max(cap, dense_rows)) + 15) & ~size_t(15)));
    uint16_t* pre16 = reinterpret_cast<uint16_t*>(bm + W);  // [W]
    __shared__ ValueWalkSm<SRID, NT> sh;
    __shared__ int64_t range_sh[2];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const RankChunk ch = chunks[blockIdx.x];
    const int2 it = g.items[ch.item];
    const int j = it.x;
    const int r0 = (it.y << g.TL) + ch.b0 * kBlkRows;
    const int nwords = (ch.b1 - ch.b0) * kRbcWords;
    if (warp == 0) {
        const int nrb = (W + kRbcWords - 1) / kRbcWords;
        const int* rb = g.rbc + int64_t(ch.item) * nrb;
        int before = 0, inside = 0;
        for (int b = lane; b < nrb; b += 32) {
            const int x = rb[b];
            before += b < ch.b0 ? x : 0;
            inside += (b >= ch.b0 && b < ch.b1) ? x : 0;
        }
        before = warp_reduce_sum(before);
        inside = warp_reduce_sum(inside);
        if (lane == 0) {
            const int64_t off = g.lp[j] + g.hoff[ch.item];
            range_sh[0] = off + before;
            range_sh[1] = off + before + inside;
            sh.nlong = 0;
        }
    }
    // dense chunks (their rows fit the value array): values indexed by row
    // offset -- no bitmap, no ranks, one shared atomic per product
    const bool dense = nwords * 32 <= dense_rows;
    // (nwords is a multiple of 128 and bm 16-byte aligned)
    for (int q = tid; q < (nwords >> 2); q += NT) reinterpret_cast<uint4*>(bm)[q] = make_uint4(0u, 0u, 0u, 0u);
    if (dense)
        for (int q = tid; q < nwords * 32; q += NT) val[q] = S_::identity();
    __syncthreads();
    const int64_t lo = range_sh[0], hi = range_sh[1];
    const int n = (int)(hi - lo);
    // (the last chunk of an item ends at the item's last row block, which can lie
    // past the matrix's last 4096-row block when nrows is not a multiple of 2^TL)
    const int ts0 = min((it.y << (g.TL - g.VTL)) + ch.b0, g.Tv), ts1 = min((it.y << (g.TL - g.VTL)) + ch.b1, g.Tv);
    T* Cv = static_cast<T*>(g.cv);
    // The chunk's pattern comes straight from the item's stash (bitmap or
    // word list, ~0.8 bytes per output), not from C's rows (4 bytes per
    // output and a shared atomic each; this pass no longer depends on the
    // emit pass -- run beside it on a second stream it measured no faster,
    // the value pass fills the SMs alone): thread tid takes a
    // contiguous range of stash entries (words of the chunk's span, or the
    // whole list, whose 16-bit word indices are sorted) and one block scan of
    // their popcounts gives every word's first output pre16[w].  A product's
    // rank slot is pre16[w] + popc(bits below it in the word): two shared
    // loads.  (Words without outputs keep a stale prefix; no product lands in
    // them.)
    {
        const unsigned* body = g.stash + g.soff[ch.item] + stash_header_words(W);
        const int U = g.form[ch.item];
        const int wb = ch.b0 * kRbcWords;
        const uint16_t* idx = U >= 0 ? reinterpret_cast<const uint16_t*>(body + U) : nullptr;
        const int ne = U >= 0 ? U : nwords;
        const int per = (ne + NT - 1) / NT;
        const int e0 = min(ne, tid * per), e1 = min(ne, e0 + per);
        auto word_of = [&](int e, unsigned& x) {  // chunk-relative word of entry e (or -1), its bits
            if (!idx) {
                x = __ldg(body + wb + e);
                return e;
            }
            const int w = int(__ldg(idx + e)) - wb;
            x = (w >= 0 && w < nwords) ? __ldg(body + e) : 0u;
            return (w >= 0 && w < nwords) ? w : -1;
        };
        int c = 0;
        for (int e = e0; e < e1; ++e) {
            unsigned x;
            if (word_of(e, x) >= 0) c += __popc(x);
        }
        int tot;
        int pfx = block_excl_scan<NT>(c, sh.wsum, &tot);
        for (int e = e0; e < e1; ++e) {
            unsigned x;
            const int w = word_of(e, x);
            if (w >= 0 && x) {
                bm[w] = x;
                pre16[w] = (uint16_t)pfx;
                pfx += __popc(x);
            }
        }
        if (!dense)
            for (int q = tid; q < n; q += NT) val[q] = S_::identity();
    }
    __syncthreads();
    if (dense) {  // values indexed by row offset; outputs in row order from the chunk's bitmap
        value_walk<SRID, NT>(g.A, g.B, g.Atpv, g.Tv, ts0, j, sh, into<S_>([val, r0](int r) { return &val[r - r0]; }), ts1,
                             g.arv, g.tv_stride, 1, -1, -1, g.tiny);
        const int per = (nwords + NT - 1) / NT;
        const int w0 = min(nwords, tid * per), w1 = min(nwords, w0 + per);
        int32_t* rows = g.rows_out;
        for (int w = w0; w < w1; ++w) {
            unsigned x = bm[w];
            int o = pre16[w];
            while (x) {
                const int b = __ffs(x) - 1;
                if (rows) rows[lo + o] = r0 + (w << 5) + b;
                Cv[lo + o++] = S_::out(val[(w << 5) + b]);
                x &= x - 1u;
            }
        }
        return;
    }
    auto slot = [bm, pre16, val, r0](int r) {
        const int rr = r - r0;
        const int w = rr >> 5;
        return &val[pre16[w] + __popc(bm[w] & ((1u << (rr & 31)) - 1u))];
    };
    value_walk<SRID, NT>(g.A, g.B, g.Atpv, g.Tv, ts0, j, sh, into<S_>(slot), ts1, g.arv, g.tv_stride, 0, -1, -1,
                         g.tiny);
    for (int q = tid; q < n; q += NT) Cv[lo + q] = S_::out(val[q]);
    if (g.rows_out) {  // C's rows of the chunk, in order, from its bitmap (thread-contiguous words)
        const int per = (nwords + NT - 1) / NT;
        const int w0 = min(nwords, tid * per), w1 = min(nwords, w0 + per);
        for (int w = w0; w < w1; ++w) {
            unsigned x = bm[w];
            int o = pre16[w];
            while (x) {
                g.rows_out[lo + o++] = r0 + (w << 5) + __ffs(x) - 1;
                x &= x - 1u;
            }
        }
    }
}

// Rank chunks of the large items (thread per item, greedy over row blocks).
// Chunks never start or end on an empty 4096-row block.  A chunk may grow
// past `cap` outputs while its span stays within `dense_blocks` blocks (it is
// then folded by row offset, no ranks); beyond that span it holds at most
// `cap` outputs (rank slots).
__global__ void k_rank_chunks(int n, const int* __restrict__ list, const int* __restrict__ rbc, int nrb, int cap,
                              int dense_blocks, const int64_t* __restrict__ coff, int64_t* __restrict__ ccount,
                              RankChunk* __restrict__ out) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int item = list[i];
        const int* rb = rbc + int64_t(item) * nrb;
        int64_t k = 0, acc = 0;
        int b0 = -1, blast = -1;
        for (int b = 0; b < nrb; ++b) {
            const int x = rb[b];
            if (x == 0) continue;
            if (b0 >= 0 && b + 1 - b0 > dense_blocks && acc + x > cap) {
                if (out) out[coff[i] + k] = RankChunk{item, b0, blast + 1, 0};
                ++k;
                b0 = -1;
            }
            if (b0 < 0) {
                b0 = b;
                acc = 0;
            }
            acc += x;
            blast = b;
        }
        if (b0 >= 0) {
            if (out) out[coff[i] + k] = RankChunk{item, b0, blast + 1, 0};
            ++k;
        }
        if (!out) ccount[i] = k;
    }
}

__global__ void k_value_split(int nitems, const int64_t* __restrict__ cnt, int64_t hcap, int* __restrict__ small,
                              int* __restrict__ large, int* __restrict__ counts) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nitems; i += gridDim.x * blockDim.x) {
        if (cnt[i] <= hcap)
            small[atomicAdd(&counts[0], 1)] = i;
        else
            large[atomicAdd(&counts[1], 1)] = i;
    }
}

// ------------------------------------------------------------ value form
//
// Semirings with values in ONE product walk: items are (column j, tile of 2^TL
// rows) with TL small enough that the tile's accumulators fit in shared
// memory (2^14 x 4 bytes, 2^13 x 8 bytes).  Every product of the item is
// folded into val[row - t0] with the semiring's atomic and marks the row in a
// bitmap; the item then writes its values in row order to a value stash (a
// bump cursor hands out the space) and its pattern stash exactly like
// k_tile_form, and emit copies the values beside the rows.  This replaces the
// pattern walk + value re-walk pair (k_tile_form + k_item_values_rank), whose
// rank chunks re-walked B(:,j) once per chunk.  The reference folds a column's
// products into one accumulator the same way (spgemm.hpp:251-255).
//
// For MinPlus (add = min, zero = +inf, semiring.hpp:58-69) the fold tests
// first: a product only takes the atomic when it lowers the slot, and only the
// product meeting an untouched slot (still the identity) marks its row --
// slots only decrease, so the thread that moves a slot off the identity is one
// that saw it there.  Other semirings mark every product (test-then-set).
template <int SRID>
struct MinSentinel : std::false_type {};
template <>
struct MinSentinel<SLAPCU_MIN_PLUS_I32> : std::true_type {};
template <>
struct MinSentinel<SLAPCU_MIN_PLUS_F64> : std::true_type {};

struct VFormArgs {
    DevCsc A, B;
    const int32_t* tab;  // A tile pointers at 2^TL rows: tile-major (tstride = A.ncols) or per column (tstride 0)
    int64_t tstride;
    int T, TL;
    const int2* items;
    const int4* units;
    const int* order;
    unsigned* stash;
    const int64_t* soff;
    const int64_t* sres;
    unsigned char* partial;  // split items: per part slot W bitmap words, then 2^TL accumulators
    int64_t pslot_bytes;
    int64_t* cnt;
    int* form;
    unsigned long long* hcnt;
    int* ticket;
    int nunits;
    const void* arv;           // A's (row, value) interleaved (4-byte values) or null
    void* vst;                 // value stash: each item's values in row order
    int64_t* voff;             // per item: its first entry in vst
    unsigned long long* vcur;  // bump cursor into vst
    int64_t vcap;              // entries of vst
    int* overflow;
    int tiny;                  // runs of at most this many products are folded by their own thread
};

template <int SRID>
__device__ __forceinline__ void vfold(typename Sr<SRID>::Acc* val, unsigned bm0, int rr, typename Sr<SRID>::Acc v) {
    using S_ = Sr<SRID>;
    using Acc = typename S_::Acc;
    if constexpr (MinSentinel<SRID>::value) {
        const Acc cur = *reinterpret_cast<volatile Acc*>(&val[rr]);
        if (cur == S_::identity()) mark(bm0, rr);
        if (v < cur) S_::atomic_acc(&val[rr], v);
    } else {
        mark(bm0, rr);
        S_::atomic_acc(&val[rr], v);
    }
}

// The item's values in row order -> the value stash (and val back to the
// identity), then its pattern stash (stash_bitmap: count, bitmap or word
// list, clears bm).  Thread tid owns a contiguous range of bitmap words, so
// one block scan of its output count places its values.
template <int SRID, int NT>
__device__ __forceinline__ void vform_finish(typename Sr<SRID>::Acc* val, unsigned* bm, unsigned* summ, uint16_t* tl,
                                             int* wsum, int* red, int* bcs, int item, int j, const VFormArgs& g) {
    using S_ = Sr<SRID>;
    using T = typename S_::T;
    constexpr int NW = NT / 32;
    __shared__ long long vbase_sh;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int W = 1 << (g.TL - 5);
    const int P = (W + NT - 1) / NT;
    const int w0 = min(W, tid * P), w1 = min(W, w0 + P);
    int c = 0;
    for (int w = w0; w < w1; ++w) c += __popc(bm[w]);
    int tot;
    int o = block_excl_scan<NT>(c, wsum, &tot);
    if (tid == 0) {
        long long b = -1;
        if (tot > 0) {
            b = (long long)atomicAdd(g.vcur, (unsigned long long)tot);
            if (b + tot > g.vcap) {
                atomicExch(g.overflow, 1);
                b = -1;
            }
        }
        vbase_sh = b;
        g.voff[item] = b;
    }
    __syncthreads();
    const long long vb = vbase_sh;
    T* vst = static_cast<T*>(g.vst) + (vb >= 0 ? vb : 0);
    for (int w = w0; w < w1; ++w) {
        unsigned x = bm[w];
        while (x) {
            const int r = (w << 5) + __ffs(x) - 1;
            x &= x - 1u;
            if (vb >= 0) vst[o] = S_::out(val[r]);
            ++o;
            val[r] = S_::identity();
        }
    }
    for (int cc = warp; cc < W / 32; cc += NW) {
        const unsigned nz = __ballot_sync(0xffffffffu, bm[cc * 32 + lane] != 0u);
        if (lane == 0) summ[cc] = nz;
    }
    __syncthreads();
    stash_bitmap<NT>(bm, summ, tl, W, wsum, red, bcs, item, j, g.stash + g.soff[item], g.sres[item], g.cnt, g.form,
                     g.hcnt, nullptr);
}

__host__ __device__ __forceinline__ size_t vform_smem(int TL, size_t acc) {
    const size_t R = size_t(1) << TL, W = R >> 5;
    return ((acc * R + sizeof(unsigned) * (W + W / 32) + sizeof(uint16_t) * W) + 15) & ~size_t(15);
}

// Persistent like k_tile_form: CTAs take work units (row tile, then heaviest
// first) by ticket; a unit walks its B-entry range of the item's column.
template <int SRID, int NT>
__global__ void __launch_bounds__(NT) k_value_form(VFormArgs g) {
    using S_ = Sr<SRID>;
    using Acc = typename S_::Acc;
    extern __shared__ __align__(16) unsigned char sm_raw[];
    const int R = 1 << g.TL, W = R >> 5;
    Acc* val = reinterpret_cast<Acc*>(sm_raw);
    unsigned* bm = reinterpret_cast<unsigned*>(sm_raw + sizeof(Acc) * size_t(R));
    unsigned* summ = bm + W;
    uint16_t* tl = reinterpret_cast<uint16_t*>(summ + W / 32);
    __shared__ ValueWalkSm<SRID, NT> sh;
    __shared__ int wsum2[NT / 32 + 1];
    __shared__ int red[NT / 32];
    __shared__ int bcs[kMaxBlocks];
    __shared__ int ticket_sh;
    for (int q = threadIdx.x; q < R; q += NT) val[q] = S_::identity();
    smem_zero(bm, W + W / 32);
    for (int b = threadIdx.x; b < kMaxBlocks; b += NT) bcs[b] = 0;
    const unsigned bm0 = smem_addr(bm);
    for (;;) {
        if (threadIdx.x == 0) {
            ticket_sh = atomicAdd(g.ticket, 1);
            sh.nlong = 0;
        }
        __syncthreads();
        const int ui = ticket_sh;
        if (ui >= g.nunits) break;
        const int4 u = g.units[g.order[ui]];
        const int2 it = g.items[u.x];
        const int64_t bs = g.B.cp[it.x];
        const int t0 = it.y << g.TL;
        value_walk<SRID, NT>(
            g.A, g.B, g.tab, g.T, it.y, it.x, sh, [val, bm0, t0](int r, Acc v) { vfold<SRID>(val, bm0, r - t0, v); },
            -1, g.arv, g.tstride, 0, bs + u.y, bs + u.z, g.tiny);
        if (u.w >= 0) {  // one part of a split item: partial bitmap and accumulators out, then reset
            unsigned char* slot = g.partial + int64_t(u.w) * g.pslot_bytes;
            unsigned* pb = reinterpret_cast<unsigned*>(slot);
            Acc* pv = reinterpret_cast<Acc*>(slot + sizeof(unsigned) * W);
            for (int q = threadIdx.x; q < W; q += NT) {
                pb[q] = bm[q];
                bm[q] = 0u;
            }
            for (int q = threadIdx.x; q < R; q += NT) {
                pv[q] = val[q];
                val[q] = S_::identity();
            }
        } else {
            vform_finish<SRID, NT>(val, bm, summ, tl, wsum2, red, bcs, u.x, it.x, g);
        }
        __syncthreads();
    }
}

// Split items: the parts' partial bitmaps OR-ed and accumulators folded (part
// order), then the same finish.  One CTA per split item.
template <int SRID, int NT>
__global__ void __launch_bounds__(NT)
    k_value_combine(VFormArgs g, const int* __restrict__ sitems, const int* __restrict__ spart,
                    const int* __restrict__ snp) {
    using S_ = Sr<SRID>;
    using Acc = typename S_::Acc;
    extern __shared__ __align__(16) unsigned char sm_raw[];
    const int R = 1 << g.TL, W = R >> 5;
    Acc* val = reinterpret_cast<Acc*>(sm_raw);
    unsigned* bm = reinterpret_cast<unsigned*>(sm_raw + sizeof(Acc) * size_t(R));
    unsigned* summ = bm + W;
    uint16_t* tl = reinterpret_cast<uint16_t*>(summ + W / 32);
    __shared__ int wsum[NT / 32 + 1];
    __shared__ int red[NT / 32];
    __shared__ int bcs[kMaxBlocks];
    for (int b = threadIdx.x; b < kMaxBlocks; b += NT) bcs[b] = 0;
    const int item = sitems[blockIdx.x];
    const int np = snp[blockIdx.x];
    const unsigned char* p0 = g.partial + int64_t(spart[blockIdx.x]) * g.pslot_bytes;
    for (int w = threadIdx.x; w < W; w += NT) {
        unsigned x = 0;
        for (int p = 0; p < np; ++p) {
            const unsigned char* sl = p0 + int64_t(p) * g.pslot_bytes;
            const unsigned xp = reinterpret_cast<const unsigned*>(sl)[w];
            const Acc* pv = reinterpret_cast<const Acc*>(sl + sizeof(unsigned) * W);
            for (unsigned y = xp; y; y &= y - 1u) {
                const int b = __ffs(y) - 1, r = (w << 5) + b;
                val[r] = ((x >> b) & 1u) ? S_::add(val[r], pv[r]) : pv[r];
            }
            x |= xp;
        }
        bm[w] = x;
    }
    __syncthreads();
    vform_finish<SRID, NT>(val, bm, summ, tl, wsum, red, bcs, item, g.items[item].x, g);
}

// Upper bound of the heavy output entries: sum over items of min(multiplies, 2^TL).
__global__ void k_sum_min(int64_t n, const int64_t* __restrict__ f, int64_t cap, unsigned long long* __restrict__ out) {
    long long s = 0;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        s += lmin(f[i], cap);
    s = warp_reduce_sum64(s);
    if ((threadIdx.x & 31) == 0 && s) atomicAdd(out, (unsigned long long)s);
}

// ------------------------------------------------------------ item setup

// Atp[k][t] (int32, relative to A.cp[k]) = first entry of A(:,k) with row >=
// t << TL, for t = 0..T.
__global__ void k_tile_ptr(DevCsc A, int TL, int T, int32_t* __restrict__ Atp) {
    const int64_t n = A.ncols * int64_t(T + 1);
    for (int64_t x = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; x < n; x += int64_t(gridDim.x) * blockDim.x) {
        const int64_t k = x / (T + 1);
        const int t = (int)(x - k * (T + 1));
        const int64_t as = A.cp[k], ae = A.cp[k + 1];
        int64_t lo = as, hi = ae;
        if (t == 0) {
            hi = as;
        } else if (t == T) {
            lo = ae;
        } else {
            const int64_t bound = int64_t(t) << TL;
            while (lo < hi) {
                const int64_t mid = (lo + hi) >> 1;
                if (A.rw[mid] < bound)
                    lo = mid + 1;
                else
                    hi = mid;
            }
        }
        Atp[x] = (int32_t)(lo - as);
    }
}

// Word form of A: entry p starts a new (column, 32-row word) pair -- its word
// differs from its predecessor's (thread per entry, coalesced), or it starts
// a column (k_word_colstart, after).
__global__ void k_word_flag(DevCsc A, int* __restrict__ flag) {
    for (int64_t x = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; x < A.span; x += int64_t(gridDim.x) * blockDim.x)
        flag[x] = x == 0 || (A.rw[A.base + x] >> 5) != (A.rw[A.base + x - 1] >> 5);
}

__global__ void k_word_colstart(DevCsc A, int* __restrict__ flag) {
    for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < A.ncols; k += int64_t(gridDim.x) * blockDim.x)
        if (A.cp[k + 1] > A.cp[k]) flag[A.cp[k] - A.base] = 1;
}

// ex = exclusive scan of flag (span + 1 entries): word entry of p is
// ex[p] + flag[p] - 1; its mask is the OR of its rows' bits.
__global__ void k_word_fill(DevCsc A, const int* __restrict__ ex, const int* __restrict__ flag, int2* __restrict__ Aw) {
    for (int64_t x = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; x < A.span; x += int64_t(gridDim.x) * blockDim.x) {
        const int r = A.rw[A.base + x];
        const int idx = ex[x] + flag[x] - 1;
        if (flag[x]) Aw[idx].x = r >> 5;
        atomicOr(reinterpret_cast<unsigned*>(&Aw[idx].y), 1u << (r & 31));
    }
}

__global__ void k_word_cp(int64_t ncols, const int64_t* __restrict__ cp, int64_t base, const int* __restrict__ ex,
                          int64_t* __restrict__ Awcp) {
    for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k <= ncols; k += int64_t(gridDim.x) * blockDim.x)
        Awcp[k] = ex[cp[k] - base];
}

// Word tile pointers: first word entry of column k with word >= t << (TL-5).
__global__ void k_word_tile_ptr(int64_t ncols, const int64_t* __restrict__ Awcp, const int2* __restrict__ Aw, int TL,
                                int T, int32_t* __restrict__ Atp) {
    const int64_t n = ncols * int64_t(T + 1);
    for (int64_t x = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; x < n; x += int64_t(gridDim.x) * blockDim.x) {
        const int64_t k = x / (T + 1);
        const int t = (int)(x - k * (T + 1));
        const int64_t as = Awcp[k], ae = Awcp[k + 1];
        int64_t lo = as, hi = ae;
        if (t == 0) {
            hi = as;
        } else if (t == T) {
            lo = ae;
        } else {
            const int bound = t << (TL - 5);
            while (lo < hi) {
                const int64_t mid = (lo + hi) >> 1;
                if (Aw[mid].x < bound)
                    lo = mid + 1;
                else
                    hi = mid;
            }
        }
        Atp[x] = (int32_t)(lo - as);
    }
}

// Tile-major layout of the same table: AtpT[t][k], t = 0..T (one row of
// A.ncols entries per tile boundary).
__global__ void k_tile_ptr_t(DevCsc A, int TL, int T, int32_t* __restrict__ AtpT) {
    // (a thread-per-column merge of rows and tile bounds measured slower: 3.7 -> 10 ms at
    // C3, the hub columns' threads walk tens of thousands of rows alone)
    const int64_t n = A.ncols * int64_t(T + 1);
    for (int64_t x = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; x < n; x += int64_t(gridDim.x) * blockDim.x) {
        const int t = (int)(x / A.ncols);
        const int64_t k = x - int64_t(t) * A.ncols;
        const int64_t as = A.cp[k], ae = A.cp[k + 1];
        int64_t lo = as, hi = ae;
        if (t == 0) {
            hi = as;
        } else if (t == T) {
            lo = ae;
        } else {
            const int64_t bound = int64_t(t) << TL;
            while (lo < hi) {
                const int64_t mid = (lo + hi) >> 1;
                if (A.rw[mid] < bound)
                    lo = mid + 1;
                else
                    hi = mid;
            }
        }
        AtpT[x] = (int32_t)(lo - as);
    }
}

// Rank chunks in row-block order (key = absolute first 4096-row block), so
// the CTAs running together share A's rows and the table's rows in L2.
__global__ void k_chunk_keys(int64_t n, const RankChunk* __restrict__ ch, const int2* __restrict__ items, int TL,
                             int* __restrict__ key, int* __restrict__ idx) {
    for (int64_t x = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; x < n; x += int64_t(gridDim.x) * blockDim.x) {
        key[x] = (items[ch[x].item].y << (TL - 12)) + ch[x].b0;
        idx[x] = (int)x;
    }
}

__global__ void k_chunk_gather(int64_t n, const RankChunk* __restrict__ in, const int* __restrict__ order,
                               RankChunk* __restrict__ out) {
    for (int64_t x = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; x < n; x += int64_t(gridDim.x) * blockDim.x)
        out[x] = in[order[x]];
}

__global__ void k_dense_flag(int64_t nkt, int T, const int32_t* __restrict__ Atp, int dmin, int* __restrict__ flag) {
    for (int64_t x = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; x < nkt; x += int64_t(gridDim.x) * blockDim.x) {
        const int64_t k = x / T;
        const int t = (int)(x - k * T);
        const int32_t* tp = Atp + k * (T + 1) + t;
        flag[x] = (tp[1] - tp[0]) >= dmin;
    }
}

__global__ void k_dense_slot(int64_t nkt, const int* __restrict__ flag, const int* __restrict__ pre,
                             int* __restrict__ slot, int2* __restrict__ runs, int T) {
    for (int64_t x = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; x < nkt; x += int64_t(gridDim.x) * blockDim.x) {
        if (flag[x]) {
            slot[x] = pre[x];
            runs[pre[x]] = make_int2((int)(x / T), (int)(x % T));
        } else {
            slot[x] = -1;
        }
    }
}

// One CTA per dense run: its rows of the tile as a bitmap.
template <int NT>
__global__ void __launch_bounds__(NT)
    k_dense_build(DevCsc A, const int32_t* __restrict__ Atp, int T, int TL, const int2* __restrict__ runs,
                  unsigned* __restrict__ out) {
    extern __shared__ __align__(16) unsigned bmd[];
    const int W = 1 << (TL - 5);
    const int2 r = runs[blockIdx.x];
    smem_zero(bmd, W);
    __syncthreads();
    const int32_t* tp = Atp + int64_t(r.x) * (T + 1) + r.y;
    const int64_t s = A.cp[r.x] + tp[0], e = A.cp[r.x] + tp[1];
    const int t0 = r.y << TL;
    for (int64_t p = s + threadIdx.x; p < e; p += NT) {
        const int rr = A.rw[p] - t0;
        atomicOr(&bmd[rr >> 5], 1u << (rr & 31));
    }
    __syncthreads();
    uint4* d4 = reinterpret_cast<uint4*>(out + int64_t(blockIdx.x) * W);
    const uint4* s4 = reinterpret_cast<const uint4*>(bmd);
    for (int q = threadIdx.x; q < W / 4; q += NT) d4[q] = s4[q];
}

// Per heavy column (column order) and tile: multiplies, and the number of
// tiles with work.  One warp per column, 8 tiles per pass over B(:,j).
__global__ void k_item_flops(DevCsc B, const int32_t* __restrict__ Atp, int T, const int* __restrict__ hl, int nh,
                             const int64_t* __restrict__ flops, int64_t* __restrict__ iflops,
                             int64_t* __restrict__ nit) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
    for (int64_t h = w0; h < nh; h += nw) {
        const int j = hl[h];
        const int64_t bs = B.cp[j], be = B.cp[j + 1];
        const bool small = flops[j] < (int64_t(1) << 31);  // 32-bit sums: one redux per tile
        int64_t items = 0;
        for (int tb = 0; tb < T; tb += 8) {
            long long f[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            const int nt = min(8, T - tb);
            for (int64_t i = bs + lane; i < be; i += 32) {
                const int32_t* tp = Atp + int64_t(B.rw[i]) * (T + 1) + tb;
                int prev = tp[0];
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    if (q < nt) {
                        const int nx = tp[q + 1];
                        f[q] += nx - prev;
                        prev = nx;
                    }
                }
            }
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                if (q < nt) {
                    const long long sum =
                        small ? (long long)__reduce_add_sync(0xffffffffu, (unsigned)f[q]) : warp_reduce_sum64(f[q]);
                    if (lane == 0) iflops[h * T + tb + q] = sum;
                    items += sum > 0;
                }
            }
        }
        if (lane == 0) nit[h] = items;
    }
}

// Chunked variant: heavy column h's B entries are cut into chunks of
// kItemChunk; a warp per chunk adds its per-tile flops into iflops (zeroed)
// with one atomic per non-zero tile, so hub columns (tens of thousands of
// entries) are spread over many warps instead of serialising one.
constexpr int kItemChunk = 1024;

__global__ void k_item_chunks(DevCsc B, const int* __restrict__ hl, int nh, int64_t* __restrict__ nch) {
    for (int64_t h = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; h < nh; h += int64_t(gridDim.x) * blockDim.x) {
        const int j = hl[h];
        nch[h] = (B.cp[j + 1] - B.cp[j] + kItemChunk - 1) / kItemChunk;
    }
}

__global__ void k_item_chunk_fill(int nh, const int64_t* __restrict__ choff, int* __restrict__ chh) {
    for (int64_t h = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; h < nh; h += int64_t(gridDim.x) * blockDim.x)
        for (int64_t q = choff[h]; q < choff[h + 1]; ++q) chh[q] = (int)h;
}

__global__ void k_item_flops_chunked(DevCsc B, const int32_t* __restrict__ Atp, int T, const int* __restrict__ hl,
                                     const int64_t* __restrict__ choff, const int* __restrict__ chh, int64_t nchunks,
                                     unsigned long long* __restrict__ iflops) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
    for (int64_t q = w0; q < nchunks; q += nw) {
        const int h = chh[q];
        const int j = hl[h];
        const int64_t bs = B.cp[j] + (q - choff[h]) * kItemChunk;
        const int64_t be = min(B.cp[j + 1], bs + kItemChunk);
        for (int tb = 0; tb < T; tb += 8) {
            unsigned long long g[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            const int nt = min(8, T - tb);
            for (int64_t i = bs + lane; i < be; i += 32) {
                const int32_t* tp = Atp + int64_t(B.rw[i]) * (T + 1) + tb;
                int prev = tp[0];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    if (u < nt) {
                        const int nx = tp[u + 1];
                        g[u] += (unsigned long long)(nx - prev);
                        prev = nx;
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                if (u < nt) {
                    const unsigned long long sum = (unsigned long long)warp_reduce_sum64((long long)g[u]);
                    if (lane == 0 && sum) atomicAdd(&iflops[int64_t(h) * T + tb + u], sum);
                }
            }
        }
    }
}

__global__ void k_item_count(int nh, int T, const int64_t* __restrict__ iflops, int64_t* __restrict__ nit) {
    for (int64_t h = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; h < nh; h += int64_t(gridDim.x) * blockDim.x) {
        int64_t k = 0;
        for (int t = 0; t < T; ++t) k += iflops[h * T + t] > 0;
        nit[h] = k;
    }
}

// Items in C order; per item its work-unit count (split when above `split`
// multiplies), stash reservation and partial-slot count.
__global__ void k_item_fill(const int* __restrict__ hl, int nh, int T, int W, const int64_t* __restrict__ iflops,
                            const int64_t* __restrict__ ioff, int64_t split, int max_parts, int2* __restrict__ items,
                            int64_t* __restrict__ ifl, int64_t* __restrict__ np, int64_t* __restrict__ sres,
                            int64_t* __restrict__ pslots) {
    for (int64_t h = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; h < nh; h += int64_t(gridDim.x) * blockDim.x) {
        int64_t o = ioff[h];
        const int j = hl[h];
        for (int t = 0; t < T; ++t) {
            const int64_t f = iflops[h * T + t];
            if (f <= 0) continue;
            items[o] = make_int2(j, t);
            ifl[o] = f;
            const int64_t p = f > split ? lmin(max_parts, (f + split - 1) / split) : 1;
            np[o] = p;
            pslots[o] = p > 1 ? p : 0;
            // 4-word multiples keep every stash 16-byte aligned (bitmap copies are uint4)
            sres[o] = stash_header_words(W) +
                      (p > 1 ? W : (lmin(W, (3 * lmin(f, W) + 1) / 2 + 1) + 3) & ~int64_t(3));
            ++o;
        }
    }
}

// Work units of unsplit items: the whole column range, in item order.
// Sort key of a work unit: its multiplies (heaviest first, LPT), and with
// tile_major the row tile above them, so that the units of one row tile run
// together and its A slice stays L2-resident (T - 1 - t: ascending tiles
// under the descending sort).
__device__ __forceinline__ int64_t unit_key(int64_t f, int t, int T, int tile_major) {
    const int64_t ff = f < (int64_t(1) << 40) ? f : (int64_t(1) << 40) - 1;
    return tile_major ? (int64_t(T - 1 - t) << 40) | ff : ff;
}

__global__ void k_unit_fill_whole(const DevCsc B, int nitems, const int2* __restrict__ items,
                                  const int64_t* __restrict__ ifl, const int64_t* __restrict__ np,
                                  const int64_t* __restrict__ uoff, int4* __restrict__ units,
                                  int64_t* __restrict__ ukey, int T, int tile_major) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nitems; i += gridDim.x * blockDim.x) {
        if (np[i] != 1) continue;
        const int j = items[i].x;
        units[uoff[i]] = make_int4(i, 0, (int)(B.cp[j + 1] - B.cp[j]), -1);
        ukey[uoff[i]] = unit_key(ifl[i], items[i].y, T, tile_major);
    }
}

// Work units of split items: equal-flops B-entry ranges (one CTA per split
// item scans its column's run lengths in this tile).
template <int NT>
__global__ void __launch_bounds__(NT)
    k_unit_fill_split(DevCsc B, const int32_t* __restrict__ Atp, int T, const int* __restrict__ sitems,
                      const int2* __restrict__ items, const int64_t* __restrict__ ifl, const int64_t* __restrict__ np,
                      const int64_t* __restrict__ uoff, const int64_t* __restrict__ poff, int4* __restrict__ units,
                      int64_t* __restrict__ ukey, int tile_major) {
    __shared__ int wsum[NT / 32 + 1];
    __shared__ long long run_sh;
    __shared__ int bnd[65];
    const int item = sitems[blockIdx.x];
    const int2 it = items[item];
    const int64_t p = np[item];
    const int64_t bs = B.cp[it.x], be = B.cp[it.x + 1];
    const int64_t u0 = uoff[item];
    const int64_t f = ifl[item];
    // part q ends after the entry whose inclusive flops prefix first reaches ceil(q*f/p)
    if (threadIdx.x == 0) run_sh = 0;
    if (threadIdx.x <= p) bnd[threadIdx.x] = threadIdx.x == p ? (int)(be - bs) : 0;
    __syncthreads();
    for (int64_t base = bs; base < be; base += NT) {
        const int64_t i = base + threadIdx.x;
        int len = 0;
        if (i < be) {
            const int32_t* tp = Atp + int64_t(B.rw[i]) * (T + 1) + it.y;
            len = tp[1] - tp[0];
        }
        int tot;
        const long long ex = (long long)block_excl_scan<NT>(len, wsum, &tot) + run_sh;
        const long long in = ex + len;
        if (len > 0) {
            // parts whose target ceil(q*f/p) lies in (ex, in]: start at the
            // first q with target > ex instead of testing every part
            for (int64_t q = (ex * p + f) / f > 1 ? (ex * p + f) / f : 1; q < p; ++q) {
                const long long tg = (q * f + p - 1) / p;
                if (tg > in) break;
                if (tg > ex) bnd[q] = (int)(i - bs + 1);
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) run_sh += tot;
        __syncthreads();
    }
    if (threadIdx.x < p) {
        const int lo = bnd[threadIdx.x], hi = max(lo, bnd[threadIdx.x + 1]);
        units[u0 + threadIdx.x] = make_int4(item, lo, hi, (int)(poff[item] + threadIdx.x));
        ukey[u0 + threadIdx.x] = unit_key(f / p, it.y, T, tile_major);
    }
}

__global__ void k_split_list(int nitems, const int64_t* __restrict__ np, const int64_t* __restrict__ poff,
                             int* __restrict__ sitems, int* __restrict__ spart, int* __restrict__ snp,
                             int* __restrict__ nsplit) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nitems; i += gridDim.x * blockDim.x) {
        if (np[i] > 1) {
            const int s = atomicAdd(nsplit, 1);
            sitems[s] = i;
            spart[s] = (int)poff[i];
            snp[s] = (int)np[i];
        }
    }
}

__global__ void k_iota(int n, int* __restrict__ v) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) v[i] = i;
}

__global__ void k_add_counts(int64_t n, const int64_t* __restrict__ a, const unsigned long long* __restrict__ b,
                             int64_t* __restrict__ out) {
    for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < n; j += int64_t(gridDim.x) * blockDim.x)
        out[j] = a[j] + (int64_t)b[j];
}

__global__ void k_mark_heavy(int64_t n, const int64_t* __restrict__ flops, int64_t lmax, bool all_heavy,
                             int* __restrict__ flag) {
    for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < n; j += int64_t(gridDim.x) * blockDim.x)
        flag[j] = flops[j] > 0 && (all_heavy || flops[j] > lmax);
}

__global__ void k_scatter_heavy(int64_t n, const int* __restrict__ flag, const int* __restrict__ pre,
                                int* __restrict__ hl) {
    for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < n; j += int64_t(gridDim.x) * blockDim.x)
        if (flag[j]) hl[pre[j]] = (int)j;
}

void excl_scan_i32(Ctx& c, const int* in, int* out, int64_t n) {
    size_t tb = 0;
    SLAPCU_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, n, c.stream));
    DevBuf tmp(tb, c.stream);
    timed(c, KC_SCAN, [&] { SLAPCU_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(), tb, in, out, n, c.stream)); });
    ++c.launches;
}

template <class T>
T d2h(Ctx& c, const T* p) {
    T v{};
    SLAPCU_CUDA(cudaMemcpyAsync(&v, p, sizeof(T), cudaMemcpyDeviceToHost, c.stream));
    SLAPCU_CUDA(cudaStreamSynchronize(c.stream));
    return v;
}

constexpr int kFormThreads = 256;  // split-item combine
constexpr int kMaxParts = 64;

}  // namespace

// 16 bytes of the value emit writes: 1s for the OrAnd pattern path, the
// semiring's identity (semiring.hpp zero()) for the global-atomic value pass.
static uint4 value_pattern(int sr, bool ones) {
    unsigned char b[16] = {};
    if (ones) {
        for (auto& x : b) x = 1;
    } else if (sr == SLAPCU_MIN_PLUS_I32) {
        const int32_t v = INT32_MAX;
        for (int q = 0; q < 4; ++q) std::memcpy(b + 4 * q, &v, 4);
    } else if (sr == SLAPCU_MIN_PLUS_F64) {
        const double v = INFINITY;
        for (int q = 0; q < 2; ++q) std::memcpy(b + 8 * q, &v, 8);
    }  // PlusTimes: +0
    uint4 r;
    std::memcpy(&r, b, 16);
    return r;
}

// Value walks: runs of at most this many products are folded by their own thread.
static int value_tiny_run(const Ctx& c) {
    return c.opt.direct_value_tiny_run >= 0 ? c.opt.direct_value_tiny_run : kValueTinyRun;
}

// Value form (semirings with values): log2 rows of an item tile whose
// accumulators fit in shared memory, or 0 when the pattern form + value pass
// run instead (option 0, or OrAnd operands without stored zeros).
static int value_form_log2(const Ctx& c, int sr, bool ones, int64_t nrows) {
    if (ones || c.opt.direct_value_form == 0) return 0;
    const size_t acc = sr == SLAPCU_OR_AND_U8 ? 4 : size_t(value_size(sr));
    int tl = c.opt.direct_value_form > 0 ? c.opt.direct_value_form : (acc <= 4 ? 14 : 13);
    while (tl > 10 && vform_smem(tl, acc) + 24 * 1024 > size_t(c.smem_optin)) --tl;
    while (tl > 10 && (int64_t(1) << (tl - 1)) >= nrows) --tl;
    return tl;
}

int direct_tile_log2(const Ctx& c, int64_t nrows) {
    // auto: 2^17-row tiles up to 2^20 rows, 2^18 above (fewer items walking
    // the same B columns when rows are many and columns sparse)
    int tl = c.opt.direct_tile_rows_log2 > 0 ? c.opt.direct_tile_rows_log2 : (nrows > (int64_t(1) << 20) ? 18 : 17);
    while (tl > 10 && (int64_t(1) << (tl - 1)) >= nrows) --tl;
    return tl;
}

// Tile pointers of A for row tiles of 2^TL rows (cached on the context).
// The cache is keyed on the CONTENT of A's pattern (fp = pattern_fingerprint),
// never on its address: SUMMA receive slots and pooled buffers reuse
// addresses for different operands.
static const int32_t* tile_pointers(Ctx& c, const DevCsc& A, uint64_t fp, int TL, int T, bool dense = true) {
    DirectCache& d = c.direct;
    const int dmin = dense ? (int)std::min<int64_t>(c.opt.direct_dense_run_min, INT32_MAX) : 0;
    if (d.atp_valid && d.atp_key == fp && d.atp_ncols == A.ncols && d.atp_tl == TL && d.atp_nnz == A.nnz &&
        d.dense_min == dmin)
        return d.atp.as<int32_t>();
    d.atp.reset(sizeof(int32_t) * size_t(A.ncols) * (T + 1), c.stream);
    KScope ks(c, KC_BIN);
    launch(c, k_tile_ptr, dim3(grid_for(c, A.ncols * (T + 1), 256)), dim3(256), 0, A, TL, T, d.atp.as<int32_t>());
    d.ndense = 0;
    d.dense_min = dmin;
    if (dmin > 0) {
        const int64_t nkt = A.ncols * int64_t(T);
        DevBuf flag(sizeof(int) * (nkt + 1), c.stream), pre(sizeof(int) * (nkt + 1), c.stream);
        SLAPCU_CUDA(cudaMemsetAsync(flag.as<int>() + nkt, 0, sizeof(int), c.stream));
        launch(c, k_dense_flag, dim3(grid_for(c, nkt, 256)), dim3(256), 0, nkt, T, (const int32_t*)d.atp.as<int32_t>(),
               dmin, flag.as<int>());
        excl_scan_i32(c, flag.as<int>(), pre.as<int>(), nkt + 1);
        d.ndense = d2h(c, pre.as<int>() + nkt);
        d.dslot.reset(sizeof(int) * std::max<int64_t>(nkt, 1), c.stream);
        DevBuf runs(sizeof(int2) * std::max(d.ndense, 1), c.stream);
        launch(c, k_dense_slot, dim3(grid_for(c, nkt, 256)), dim3(256), 0, nkt, (const int*)flag.as<int>(),
               (const int*)pre.as<int>(), d.dslot.as<int>(), runs.as<int2>(), T);
        const int W = 1 << (TL - 5);
        d.dbm.reset(sizeof(unsigned) * size_t(W) * std::max(d.ndense, 1), c.stream);
        if (d.ndense > 0) {
            auto k = k_dense_build<256>;
            ensure_smem(k, sizeof(unsigned) * W);
            launch(c, k, dim3(d.ndense), dim3(256), sizeof(unsigned) * W, A, (const int32_t*)d.atp.as<int32_t>(), T,
                   TL, (const int2*)runs.as<int2>(), d.dbm.as<unsigned>());
        }
    }
    d.atp_key = fp;
    d.atp_ncols = A.ncols;
    d.atp_nnz = A.nnz;
    d.atp_tl = TL;
    d.atp_valid = true;
    return d.atp.as<int32_t>();
}

// Word form of A and its tile pointers (cached like Atp, same fingerprint key).
static const int32_t* word_pointers(Ctx& c, const DevCsc& A, uint64_t fp, int TL, int T) {
    DirectCache& d = c.direct;
    if (d.aw_valid && d.aw_key == fp && d.aw_tl == TL && d.aw_ncols == A.ncols) return d.watp.as<int32_t>();
    KScope ks(c, KC_BIN);
    const int64_t span = A.span;
    DevBuf flag(sizeof(int) * (span + 1), c.stream), ex(sizeof(int) * (span + 1), c.stream);
    SLAPCU_CUDA(cudaMemsetAsync(flag.as<int>() + span, 0, sizeof(int), c.stream));
    if (span) launch(c, k_word_flag, dim3(grid_for(c, span, 256)), dim3(256), 0, A, flag.as<int>());
    if (A.ncols) launch(c, k_word_colstart, dim3(grid_for(c, A.ncols, 256)), dim3(256), 0, A, flag.as<int>());
    excl_scan_i32(c, flag.as<int>(), ex.as<int>(), span + 1);
    const int nw = d2h(c, ex.as<int>() + span);
    d.aw.reset(sizeof(int2) * std::max(nw, 1), c.stream);
    SLAPCU_CUDA(cudaMemsetAsync(d.aw.get(), 0, sizeof(int2) * std::max(nw, 1), c.stream));
    if (span)
        launch(c, k_word_fill, dim3(grid_for(c, span, 256)), dim3(256), 0, A, (const int*)ex.as<int>(),
               (const int*)flag.as<int>(), d.aw.as<int2>());
    d.awcp.reset(sizeof(int64_t) * (A.ncols + 1), c.stream);
    launch(c, k_word_cp, dim3(grid_for(c, A.ncols + 1, 256)), dim3(256), 0, A.ncols, A.cp, A.base,
           (const int*)ex.as<int>(), d.awcp.as<int64_t>());
    d.watp.reset(sizeof(int32_t) * size_t(A.ncols) * (T + 1), c.stream);
    launch(c, k_word_tile_ptr, dim3(grid_for(c, A.ncols * (T + 1), 256)), dim3(256), 0, A.ncols,
           (const int64_t*)d.awcp.as<int64_t>(), (const int2*)d.aw.as<int2>(), TL, T, d.watp.as<int32_t>());
    d.aw_key = fp;
    d.aw_tl = TL;
    d.aw_ncols = A.ncols;
    d.aw_valid = true;
    return d.watp.as<int32_t>();
}

// Tile pointers at the value-pass sub-tile height (cached like Atp).
static const int32_t* value_tile_pointers(Ctx& c, const DevCsc& A, uint64_t fp, int VTL, int Tv, bool tmajor = false) {
    DirectCache& d = c.direct;
    if (d.atpv_valid && d.atpv_key == fp && d.atpv_ncols == A.ncols && d.atpv_tl == VTL && d.atpv_nnz == A.nnz &&
        d.atpv_tmajor == tmajor)
        return d.atpv.as<int32_t>();
    d.atpv.reset(sizeof(int32_t) * size_t(A.ncols) * (Tv + 1), c.stream);
    KScope ks(c, KC_BIN);
    if (tmajor)
        launch(c, k_tile_ptr_t, dim3(grid_for(c, A.ncols * (Tv + 1), 256)), dim3(256), 0, A, VTL, Tv,
               d.atpv.as<int32_t>());
    else
        launch(c, k_tile_ptr, dim3(grid_for(c, A.ncols * (Tv + 1), 256)), dim3(256), 0, A, VTL, Tv,
               d.atpv.as<int32_t>());
    d.atpv_tmajor = tmajor;
    d.atpv_key = fp;
    d.atpv_ncols = A.ncols;
    d.atpv_nnz = A.nnz;
    d.atpv_tl = VTL;
    d.atpv_valid = true;
    return d.atpv.as<int32_t>();
}

// Fallback for semirings with values (and OrAnd operands holding stored
// zeros, whose pattern is structural but whose values are not all 1): the
// fused begin/finish pair into the caller's buffers.
static int64_t direct_fallback(Ctx& c, const DevCsc& A, const DevCsc& B, int sr, int alg, int64_t capacity,
                               int64_t* c_colptr, int32_t* crw, void* cv) {
    const int64_t nnz = fused_begin(c, A, B, sr, alg, c_colptr, 0);
    c.direct.last_nnz = nnz;
    if (nnz > capacity)
        throw Fail{SLAPCU_ERR_BUDGET, "output needs " + std::to_string(nnz) + " entries, capacity " +
                                          std::to_string(capacity)};
    fused_finish(c, A, B, sr, crw, cv);
    ctx_settle(c);
    return nnz;
}

// The reference picks the accumulator per column by compression: hash iff
// flops_j / nnz(C(:,j)) >= 2 (spgemm.hpp:54, :312-317), else the k-way merge.
// Here the choice is per product for value semirings: the compression of 8
// evenly spaced windows of <= 256 columns (exact symbolic counts) decides
// between the bitmap path and the sort-merge (ESC) path, whose cost is per
// product rather than per output entry and wins when cf is near 1 (C2, C5).
// Compression of up to 16 sampled columns, exactly: one CTA per sampled
// column marks its rows in a global bitmap (atomicOr; a newly set bit is a
// new output entry), at most kSampleProducts products per column.
constexpr int kSampleCols = 16;
constexpr int64_t kSampleProducts = 1 << 20;
constexpr int64_t kEscAutoMaxProducts = int64_t(1) << 28;

constexpr int kSampleParts = 16;  // CTAs per sampled column (its B entries interleaved)

__global__ void __launch_bounds__(256) k_sample_cf(DevCsc A, DevCsc B, const int* __restrict__ cols, int words,
                                                   unsigned* __restrict__ bm, unsigned long long* __restrict__ out) {
    const int sc = blockIdx.x / kSampleParts, part = blockIdx.x % kSampleParts;
    const int64_t j = cols[sc];
    unsigned* m = bm + int64_t(sc) * words;
    unsigned long long f = 0, s = 0;
    int64_t done = 0;
    for (int64_t i = B.cp[j] + part; i < B.cp[j + 1] && done < kSampleProducts / kSampleParts; i += kSampleParts) {
        const int k = B.rw[i];
        const int64_t a0 = A.cp[k], a1 = A.cp[k + 1];
        for (int64_t p = a0 + threadIdx.x; p < a1; p += blockDim.x) {
            const int r = A.rw[p];
            const unsigned bit = 1u << (r & 31);
            ++f;
            if (!(atomicOr(&m[r >> 5], bit) & bit)) ++s;
        }
        done += a1 - a0;
    }
    for (int o = 16; o > 0; o >>= 1) {
        f += __shfl_xor_sync(0xffffffffu, f, o);
        s += __shfl_xor_sync(0xffffffffu, s, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&out[0], f);
        atomicAdd(&out[1], s);
    }
}

// The reference picks the accumulator per column by compression: hash iff
// flops_j / nnz(C(:,j)) >= 2 (spgemm.hpp:54, :312-317), else the k-way merge.
// Here, for value semirings, per product: products of at most 2^28
// multiplies whose sampled compression is below 2 go to the sort-merge (ESC)
// path, which costs per product rather than per output entry (C5: 12.8 ->
// ~5 ms; C2, light columns of ~64 products at compression 1.0: 5.4 -> 4.7 ms
// once ESC kept its per-column work on the device).  Heavy products sample
// columns at flops quantiles, light ones evenly spaced columns.
static bool esc_preferred(Ctx& c, const DevCsc& A, const DevCsc& B) {
    const int64_t n = B.ncols;
    if (n == 0) return false;
    DevBuf fl(sizeof(int64_t) * n, c.stream);
    int64_t total = 0;
    spgemm_flops(c, A, B, fl.as<int64_t>(), &total);
    // ESC moves ~40 bytes per product: only products it finishes in a few
    // milliseconds are candidates (a misjudged large product would cost seconds)
    if (total > kEscAutoMaxProducts) return false;
    const int64_t words64 = (A.nrows + 31) / 32;
    if (words64 > (int64_t(1) << 22)) return false;  // (sample bitmaps of > 16 MB each: not worth it)
    std::vector<int> cols;
    if (total <= 4096 * n) {
        // light columns on average (C2: 64 products each): evenly spaced sample
        // columns -- no per-column counts on the host (1M columns: a ms of copy)
        for (int q = 0; q < kSampleCols; ++q) {
            const int j = (int)((n * (2 * q + 1)) / (2 * kSampleCols));
            if (cols.empty() || cols.back() != j) cols.push_back(j);
        }
    } else {
        // sampled columns at evenly spaced quantiles of the cumulative flops, so
        // the columns holding most of the work are the ones measured
        std::vector<int64_t> hf(static_cast<size_t>(n));
        SLAPCU_CUDA(cudaMemcpyAsync(hf.data(), fl.get(), sizeof(int64_t) * n, cudaMemcpyDeviceToHost, c.stream));
        SLAPCU_CUDA(cudaStreamSynchronize(c.stream));
        int64_t acc = 0;
        int next = 0;
        for (int64_t j = 0; j < n && next < kSampleCols; ++j) {
            acc += hf[size_t(j)];
            while (next < kSampleCols && acc * kSampleCols > total * next) {
                if (cols.empty() || cols.back() != (int)j) cols.push_back((int)j);
                ++next;
            }
        }
    }
    const int ns = (int)cols.size();
    const int words = (int)words64;
    DevBuf dcols(sizeof(int) * std::max(ns, 1), c.stream);
    SLAPCU_CUDA(cudaMemcpyAsync(dcols.get(), cols.data(), sizeof(int) * ns, cudaMemcpyHostToDevice, c.stream));
    DevBuf bm(sizeof(unsigned) * size_t(words) * ns, c.stream), cnt(sizeof(unsigned long long) * 2, c.stream);
    SLAPCU_CUDA(cudaMemsetAsync(bm.get(), 0, sizeof(unsigned) * size_t(words) * ns, c.stream));
    SLAPCU_CUDA(cudaMemsetAsync(cnt.get(), 0, sizeof(unsigned long long) * 2, c.stream));
    launch(c, k_sample_cf, dim3(ns * kSampleParts), dim3(256), 0, A, B, (const int*)dcols.as<int>(), words,
           bm.as<unsigned>(), cnt.as<unsigned long long>());
    unsigned long long h[2] = {0, 0};
    SLAPCU_CUDA(cudaMemcpyAsync(h, cnt.get(), sizeof(h), cudaMemcpyDeviceToHost, c.stream));
    SLAPCU_CUDA(cudaStreamSynchronize(c.stream));
    return h[1] > 0 && h[0] < 2 * h[1];
}

int64_t direct_spgemm(Ctx& c, const DevCsc& A_, const DevCsc& B_, int sr, int alg, int64_t capacity,
                      int64_t* c_colptr, int32_t* crw, void* cv) {
    check_operands(A_, B_);
    if (!c_colptr) throw Fail{SLAPCU_ERR_INVALID, "null colptr"};
    if (value_size(sr) == 0) throw Fail{SLAPCU_ERR_INVALID, "unknown semiring"};
    if (capacity > 0 && (!crw || !cv)) throw Fail{SLAPCU_ERR_INVALID, "null output buffers"};
    DevCsc A = A_, B = B_;
    resolve(c, A);
    resolve(c, B);
    if ((A.span && !A.v) || (B.span && !B.v)) throw Fail{SLAPCU_ERR_INVALID, "operand values are null"};
    ctx_settle(c);
    // sort-merge (ESC) path: the reference's fold order for every output entry
    // (bit-exact floating point), or forced for any semiring
    const bool fp = sr == SLAPCU_PLUS_TIMES_F64 || sr == SLAPCU_PLUS_TIMES_F32 || sr == SLAPCU_MIN_PLUS_F64;
    if ((c.opt.deterministic && fp) || c.opt.direct_esc == 1 ||
        (c.opt.direct_esc < 0 && sr != SLAPCU_OR_AND_U8 && esc_preferred(c, A, B))) {
        SLAPCU_CUDA(cudaEventRecord(c.ev[0], c.stream));
        const int64_t nz = esc_spgemm(c, A_, B_, sr, capacity, c_colptr, crw, cv);
        SLAPCU_CUDA(cudaEventRecord(c.ev[1], c.stream));
        SLAPCU_CUDA(cudaStreamSynchronize(c.stream));
        cudaEventElapsedTime(&c.sym_ms, c.ev[0], c.ev[1]);
        prof_flush(c);
        return nz;
    }
    if (c.opt.direct_values_fallback && sr != SLAPCU_OR_AND_U8)
        return direct_fallback(c, A_, B_, sr, alg, capacity, c_colptr, crw, cv);
    // OrAnd: if no stored value is 0 every product is 1 (pattern only, values
    // written as 1); otherwise -- and for every other semiring -- the pattern
    // is structural and a value pass follows the emit pass
    bool ones = false;
    if (sr == SLAPCU_OR_AND_U8) {
        c.err_flag.reset(sizeof(int) * 2, c.stream);
        int* fl = c.err_flag.as<int>();
        SLAPCU_CUDA(cudaMemsetAsync(fl, 0, sizeof(int) * 2, c.stream));
        any_zero_u8(c, (const uint8_t*)A.v + A.base, A.span, fl + 1);
        any_zero_u8(c, (const uint8_t*)B.v + B.base, B.span, fl + 1);
        ones = d2h(c, fl + 1) == 0;
    }
    SLAPCU_CUDA(cudaEventRecord(c.ev[0], c.stream));
    DirectCache& d = c.direct;
    FusedState& f = d.light;
    const uint64_t afp = pattern_fingerprint(c, A);
    f.ones = ones;
    prepare_plan(c, A, B);
    const int64_t* flops = c.plan.flops.as<int64_t>();
    const int64_t n = B.ncols;

    // ---- light columns: shared hash, staged (fused.cu kernels)
    BinSpec spec{};
    spec.nlight = 8;
    for (int b = 0; b < 8; ++b) spec.thr[b] = int64_t(32) << b;
    // columns above 1024 multiplies go to the tile items: the hash kernels'
    // block-wide sorts of 2-8K keys cost more than a few small tile items
    int64_t lmax = std::min<int64_t>(c.opt.direct_light_flops_max, 4096);
    spec.light_max = lmax;
    spec.all_heavy = alg == SLAPCU_ALG_HEAP;
    f.cnt.reset(sizeof(int64_t) * (n + 1), c.stream);
    SLAPCU_CUDA(cudaMemsetAsync(f.cnt.get(), 0, sizeof(int64_t) * (n + 1), c.stream));
    make_bins(c, n, flops, nullptr, spec, f.cnt.as<int64_t>(), f.bins);
    int nlight = 0;
    int64_t light_bound = 0;
    for (int b = 0; b < spec.nlight; ++b) {
        nlight += f.bins.count[b];
        light_bound += int64_t(f.bins.count[b]) * std::min<int64_t>(spec.thr[b], A.nrows);
    }
    f.srows.reset(sizeof(int32_t) * std::max<int64_t>(light_bound, 1), c.stream);
    if (!ones) f.svals.reset(size_t(value_size(sr)) * std::max<int64_t>(light_bound, 1), c.stream);
    f.soff.reset(sizeof(int64_t) * std::max<int64_t>(n, 1), c.stream);
    f.scur.reset(sizeof(unsigned long long), c.stream);
    SLAPCU_CUDA(cudaMemsetAsync(f.scur.get(), 0, sizeof(unsigned long long), c.stream));
    const int* L = f.bins.list.as<int>();
    for (int b = 0; b < spec.nlight; ++b) {
        const int nb = f.bins.count[b];
        if (!nb) continue;
        KScope ks(c, KC_SYM_LIGHT);
        fused_light_launch(c, sr, ones, b, A, B, L + f.bins.offset[b], nb, flops, f);
    }
    // light prefix per column (heavy columns count 0 here)
    d.lp.reset(sizeof(int64_t) * (n + 1), c.stream);
    {
        KScope ks(c, KC_SCAN);
        exclusive_scan_i64(c, f.cnt.as<int64_t>(), d.lp.as<int64_t>(), n + 1);
    }

    // ---- heavy columns in column order, cut into row-tile items
    const int nh = f.bins.count[spec.nlight];
    // value form: one walk folds the values in small shared tiles (no value pass)
    const int vtl = value_form_log2(c, sr, ones, A.nrows);
    const bool vform = vtl > 0;
    const int TL = vform ? vtl : direct_tile_log2(c, A.nrows);
    const int T = (int)((A.nrows + (int64_t(1) << TL) - 1) >> TL);
    const int W = 1 << (TL - 5);
    d.hcnt.reset(sizeof(unsigned long long) * std::max<int64_t>(n, 1), c.stream);
    SLAPCU_CUDA(cudaMemsetAsync(d.hcnt.get(), 0, sizeof(unsigned long long) * std::max<int64_t>(n, 1), c.stream));
    int nitems = 0;
    // words mode: the form walks A's (word, mask) pairs (one shared update
    // per distinct word of a run) instead of its rows
    const bool words = !vform && c.opt.direct_words != 0 && A.span < INT32_MAX;
    DevBuf vst, voff, vcur, arv_form;  // value form: value stash, per-item offsets, bump cursor + overflow flag
    if (nh > 0) {
        const int32_t* Atp = words ? word_pointers(c, A, afp, TL, T) : tile_pointers(c, A, afp, TL, T, !vform);
        KScope ks(c, KC_BIN);
        DevBuf hflag(sizeof(int) * (n + 1), c.stream), hpre(sizeof(int) * (n + 1), c.stream);
        launch(c, k_mark_heavy, dim3(grid_for(c, n, 256)), dim3(256), 0, n, flops, lmax, spec.all_heavy != 0,
               hflag.as<int>());
        excl_scan_i32(c, hflag.as<int>(), hpre.as<int>(), n);
        d.hl.reset(sizeof(int) * nh, c.stream);
        launch(c, k_scatter_heavy, dim3(grid_for(c, n, 256)), dim3(256), 0, n, (const int*)hflag.as<int>(),
               (const int*)hpre.as<int>(), d.hl.as<int>());
        DevBuf iflops(sizeof(int64_t) * int64_t(nh) * T, c.stream);
        DevBuf nit(sizeof(int64_t) * (nh + 1), c.stream), ioff(sizeof(int64_t) * (nh + 1), c.stream);
        SLAPCU_CUDA(cudaMemsetAsync(nit.as<int64_t>() + nh, 0, sizeof(int64_t), c.stream));
        {
            DevBuf nch(sizeof(int64_t) * (nh + 1), c.stream), choff(sizeof(int64_t) * (nh + 1), c.stream);
            SLAPCU_CUDA(cudaMemsetAsync(nch.as<int64_t>() + nh, 0, sizeof(int64_t), c.stream));
            launch(c, k_item_chunks, dim3(grid_for(c, nh, 256)), dim3(256), 0, B, (const int*)d.hl.as<int>(), nh,
                   nch.as<int64_t>());
            exclusive_scan_i64(c, nch.as<int64_t>(), choff.as<int64_t>(), nh + 1);
            const int64_t nchunks = d2h(c, choff.as<int64_t>() + nh);
            DevBuf chh(sizeof(int) * std::max<int64_t>(nchunks, 1), c.stream);
            launch(c, k_item_chunk_fill, dim3(grid_for(c, nh, 256)), dim3(256), 0, nh,
                   (const int64_t*)choff.as<int64_t>(), chh.as<int>());
            SLAPCU_CUDA(cudaMemsetAsync(iflops.get(), 0, sizeof(int64_t) * int64_t(nh) * T, c.stream));
            launch(c, k_item_flops_chunked, dim3(grid_for(c, nchunks * 32, 256)), dim3(256), 0, B, Atp, T,
                   (const int*)d.hl.as<int>(), (const int64_t*)choff.as<int64_t>(), (const int*)chh.as<int>(),
                   nchunks, reinterpret_cast<unsigned long long*>(iflops.as<int64_t>()));
            launch(c, k_item_count, dim3(grid_for(c, nh, 256)), dim3(256), 0, nh, T,
                   (const int64_t*)iflops.as<int64_t>(), nit.as<int64_t>());
        }
        exclusive_scan_i64(c, nit.as<int64_t>(), ioff.as<int64_t>(), nh + 1);
        const int64_t nitems64 = d2h(c, ioff.as<int64_t>() + nh);
        if (nitems64 > INT32_MAX) throw Fail{SLAPCU_ERR_INVALID, "too many tile items"};
        nitems = (int)nitems64;
        const size_t ni1 = size_t(nitems) + 1;
        d.items.reset(sizeof(int2) * ni1, c.stream);
        d.ifl.reset(sizeof(int64_t) * ni1, c.stream);
        DevBuf np(sizeof(int64_t) * ni1, c.stream), uoff(sizeof(int64_t) * ni1, c.stream);
        DevBuf psl(sizeof(int64_t) * ni1, c.stream), poff(sizeof(int64_t) * ni1, c.stream);
        d.sres.reset(sizeof(int64_t) * ni1, c.stream);
        d.soff.reset(sizeof(int64_t) * ni1, c.stream);
        SLAPCU_CUDA(cudaMemsetAsync(np.as<int64_t>() + nitems, 0, sizeof(int64_t), c.stream));
        SLAPCU_CUDA(cudaMemsetAsync(psl.as<int64_t>() + nitems, 0, sizeof(int64_t), c.stream));
        SLAPCU_CUDA(cudaMemsetAsync(d.sres.as<int64_t>() + nitems, 0, sizeof(int64_t), c.stream));
        const int64_t split = std::max<int64_t>(c.opt.direct_split_flops, 1024);
        launch(c, k_item_fill, dim3(grid_for(c, nh, 256)), dim3(256), 0, (const int*)d.hl.as<int>(), nh, T, W,
               (const int64_t*)iflops.as<int64_t>(), (const int64_t*)ioff.as<int64_t>(), split, kMaxParts,
               d.items.as<int2>(), d.ifl.as<int64_t>(), np.as<int64_t>(), d.sres.as<int64_t>(), psl.as<int64_t>());
        exclusive_scan_i64(c, np.as<int64_t>(), uoff.as<int64_t>(), nitems + 1);
        exclusive_scan_i64(c, psl.as<int64_t>(), poff.as<int64_t>(), nitems + 1);
        exclusive_scan_i64(c, d.sres.as<int64_t>(), d.soff.as<int64_t>(), nitems + 1);
        int64_t tail[3];
        SLAPCU_CUDA(cudaMemcpyAsync(&tail[0], uoff.as<int64_t>() + nitems, 8, cudaMemcpyDeviceToHost, c.stream));
        SLAPCU_CUDA(cudaMemcpyAsync(&tail[1], poff.as<int64_t>() + nitems, 8, cudaMemcpyDeviceToHost, c.stream));
        SLAPCU_CUDA(cudaMemcpyAsync(&tail[2], d.soff.as<int64_t>() + nitems, 8, cudaMemcpyDeviceToHost, c.stream));
        SLAPCU_CUDA(cudaStreamSynchronize(c.stream));
        const int64_t nunits = tail[0], nslots = tail[1], swords = tail[2];
        d.nunits = nunits;
        if (nunits > INT32_MAX || nslots > INT32_MAX) throw Fail{SLAPCU_ERR_INVALID, "too many work units"};
        d.units.reset(sizeof(int4) * std::max<int64_t>(nunits, 1), c.stream);
        DevBuf ukey(sizeof(int64_t) * std::max<int64_t>(nunits, 1), c.stream);
        // split items (parts of one item are formed by several CTAs, then OR-ed)
        DevBuf sl(sizeof(int) * 3 * (size_t(nitems) + 1), c.stream), ns(sizeof(int), c.stream);
        SLAPCU_CUDA(cudaMemsetAsync(ns.get(), 0, sizeof(int), c.stream));
        int* si = sl.as<int>();
        int nsplit = 0;
        if (nslots > 0) {
            launch(c, k_split_list, dim3(grid_for(c, nitems, 256)), dim3(256), 0, nitems,
                   (const int64_t*)np.as<int64_t>(), (const int64_t*)poff.as<int64_t>(), si, si + nitems,
                   si + 2 * nitems, ns.as<int>());
            nsplit = d2h(c, ns.as<int>());
        }
        launch(c, k_unit_fill_whole, dim3(grid_for(c, nitems, 256)), dim3(256), 0, B, nitems,
               (const int2*)d.items.as<int2>(), (const int64_t*)d.ifl.as<int64_t>(), (const int64_t*)np.as<int64_t>(),
               (const int64_t*)uoff.as<int64_t>(), d.units.as<int4>(), ukey.as<int64_t>(), T, c.opt.direct_tile_major);
        if (nsplit > 0)
            launch(c, k_unit_fill_split<256>, dim3(nsplit), dim3(256), 0, B, Atp, T, (const int*)si,
                   (const int2*)d.items.as<int2>(), (const int64_t*)d.ifl.as<int64_t>(),
                   (const int64_t*)np.as<int64_t>(), (const int64_t*)uoff.as<int64_t>(),
                   (const int64_t*)poff.as<int64_t>(), d.units.as<int4>(), ukey.as<int64_t>(), c.opt.direct_tile_major);
        // heaviest units first (LPT)
        d.order.reset(sizeof(int) * std::max<int64_t>(nunits, 1), c.stream);
        {
            DevBuf idx(sizeof(int) * std::max<int64_t>(nunits, 1), c.stream),
                kout(sizeof(int64_t) * std::max<int64_t>(nunits, 1), c.stream);
            launch(c, k_iota, dim3(grid_for(c, nunits, 256)), dim3(256), 0, (int)nunits, idx.as<int>());
            size_t tb = 0;
            SLAPCU_CUDA(cub::DeviceRadixSort::SortPairsDescending(nullptr, tb, ukey.as<int64_t>(), kout.as<int64_t>(),
                                                                  idx.as<int>(), d.order.as<int>(), (int)nunits, 0,
                                                                  62, c.stream));
            DevBuf tmp(tb, c.stream);
            timed(c, KC_BIN, [&] {
                SLAPCU_CUDA(cub::DeviceRadixSort::SortPairsDescending(tmp.get(), tb, ukey.as<int64_t>(),
                                                                      kout.as<int64_t>(), idx.as<int>(),
                                                                      d.order.as<int>(), (int)nunits, 0, 62,
                                                                      c.stream));
            });
            ++c.launches;
        }
        d.stash.reset(sizeof(unsigned) * std::max<int64_t>(swords, 4), c.stream);
        const size_t vacc = sr == SLAPCU_OR_AND_U8 ? 4 : size_t(value_size(sr));
        const int64_t pslot_bytes =
            vform ? int64_t((sizeof(unsigned) * size_t(W) + vacc * (size_t(1) << TL) + 15) & ~size_t(15))
                  : int64_t(sizeof(unsigned) * size_t(W));
        d.partial.reset(size_t(pslot_bytes) * std::max<int64_t>(nslots, 1), c.stream);
        d.cnt.reset(sizeof(int64_t) * ni1, c.stream);
        d.form.reset(sizeof(int) * ni1, c.stream);
        d.hoff.reset(sizeof(int64_t) * ni1, c.stream);
        SLAPCU_CUDA(cudaMemsetAsync(d.cnt.as<int64_t>() + nitems, 0, sizeof(int64_t), c.stream));
        KScope ks2(c, KC_SYM_HEAVY);
        const int nrb = (W + kRbcWords - 1) / kRbcWords;
        int* rbc = nullptr;
        if (!ones && !vform) {
            d.rbc.reset(sizeof(int) * size_t(nitems) * nrb, c.stream);
            rbc = d.rbc.as<int>();
        }
        const DenseRuns dr{(!words && d.ndense > 0) ? (const int*)d.dslot.as<int>() : nullptr,
                           (const unsigned*)d.dbm.as<unsigned>(), (!words && d.ndense > 0) ? d.dense_min : 0};
        FormArgs g{A, B, Atp, dr, T, TL, (const int2*)d.items.as<int2>(), (const int4*)d.units.as<int4>(),
                   (const int*)d.order.as<int>(), d.stash.as<unsigned>(), (const int64_t*)d.soff.as<int64_t>(),
                   (const int64_t*)d.sres.as<int64_t>(), d.partial.as<unsigned>(), d.cnt.as<int64_t>(),
                   d.form.as<int>(), d.hcnt.as<unsigned long long>(), nullptr, 0, rbc,
                   c.opt.direct_short_run > 0 ? c.opt.direct_short_run : kShortRun,
                   words ? (const int2*)d.aw.as<int2>() : nullptr, words ? (const int64_t*)d.awcp.as<int64_t>() : nullptr};
        DevBuf tick(sizeof(int), c.stream);
        SLAPCU_CUDA(cudaMemsetAsync(tick.get(), 0, sizeof(int), c.stream));
        g.ticket = tick.as<int>();
        g.nunits = (int)nunits;
        auto form = [&](auto kf, int nt) {
            const size_t walk = nt == 512 ? sizeof(WalkSm<512>) : nt == 128 ? sizeof(WalkSm<128>) : sizeof(WalkSm<256>);
            const size_t smem = form_tail_offset(W) + std::max(sizeof(uint16_t) * W, walk);
            ensure_smem(kf, smem);
            int per_sm = 0;
            SLAPCU_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kf, nt, smem));
            const int64_t grid = c.opt.direct_persistent ? std::max<int64_t>(1, std::min<int64_t>(nunits, int64_t(per_sm) * c.num_sms))
                                                         : nunits;
            launch(c, kf, dim3((unsigned)grid), dim3(nt), smem, g);
        };
        const int ft = c.opt.direct_form_threads;
        if (vform) {
            // value stash: at most min(multiplies, 2^TL) entries per item, and no more than C holds
            DevBuf smin(sizeof(unsigned long long), c.stream);
            SLAPCU_CUDA(cudaMemsetAsync(smin.get(), 0, sizeof(unsigned long long), c.stream));
            if (nitems > 0)
                launch(c, k_sum_min, dim3(grid_for(c, nitems, 256)), dim3(256), 0, int64_t(nitems),
                       (const int64_t*)d.ifl.as<int64_t>(), int64_t(1) << TL, smin.as<unsigned long long>());
            const int64_t vcap = std::min<int64_t>(std::max<int64_t>(capacity, 0),
                                                   (int64_t)d2h(c, smin.as<unsigned long long>()));
            vst = DevBuf(size_t(value_size(sr)) * std::max<int64_t>(vcap, 1), c.stream);
            voff = DevBuf(sizeof(int64_t) * ni1, c.stream);
            vcur = DevBuf(sizeof(unsigned long long) * 2, c.stream);
            SLAPCU_CUDA(cudaMemsetAsync(vcur.get(), 0, sizeof(unsigned long long) * 2, c.stream));
            const void* arvp = nullptr;
            if (value_size(sr) == 4 && A.span > 0 && c.opt.direct_value_interleave) {
                arv_form = DevBuf(sizeof(int2) * size_t(A.span), c.stream);
                launch(c, k_interleave_rv, dim3(grid_for(c, A.span, 256)), dim3(256), 0, A.span, A.rw + A.base,
                       static_cast<const int32_t*>(A.v) + A.base, arv_form.as<int2>());
                arvp = arv_form.as<int2>() - A.base;
            } else if (value_size(sr) == 8 && A.span > 0 && c.opt.direct_value_interleave == 2) {
                arv_form = DevBuf(sizeof(int4) * size_t(A.span), c.stream);
                launch(c, k_interleave_rv8, dim3(grid_for(c, A.span, 256)), dim3(256), 0, A.span, A.rw + A.base,
                       static_cast<const long long*>(A.v) + A.base, arv_form.as<int4>());
                arvp = arv_form.as<int4>() - A.base;
            }
            // the walk reads the tile-major table (a row tile's two rows stay in L2 while its units run)
            const bool tmaj = c.opt.direct_value_tmajor != 0;
            VFormArgs vg{A, B, tmaj ? value_tile_pointers(c, A, afp, TL, T, true) : Atp, tmaj ? A.ncols : 0, T, TL,
                         (const int2*)d.items.as<int2>(), (const int4*)d.units.as<int4>(), (const int*)d.order.as<int>(),
                         d.stash.as<unsigned>(), (const int64_t*)d.soff.as<int64_t>(),
                         (const int64_t*)d.sres.as<int64_t>(), d.partial.as<unsigned char>(), pslot_bytes,
                         d.cnt.as<int64_t>(), d.form.as<int>(), d.hcnt.as<unsigned long long>(), tick.as<int>(),
                         (int)nunits, arvp, vst.get(), voff.as<int64_t>(), vcur.as<unsigned long long>(), vcap,
                         reinterpret_cast<int*>(vcur.as<unsigned long long>() + 1), value_tiny_run(c)};
            const size_t smem = vform_smem(TL, vacc);
            dispatch_sr(sr, [&](auto id) {
                constexpr int ID = decltype(id)::value;
                auto go = [&](auto kf, int nt) {
                    ensure_smem(kf, smem);
                    int per_sm = 0;
                    SLAPCU_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kf, nt, smem));
                    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(nunits, int64_t(std::max(per_sm, 1)) * c.num_sms));
                    launch(c, kf, dim3((unsigned)grid), dim3(nt), smem, vg);
                };
                if (c.opt.direct_value_threads == 512)
                    go(k_value_form<ID, 512>, 512);
                else
                    go(k_value_form<ID, 256>, 256);
                if (nsplit > 0) {
                    auto kc = k_value_combine<ID, 256>;
                    ensure_smem(kc, smem);
                    launch(c, kc, dim3(nsplit), dim3(256), smem, vg, (const int*)si, (const int*)(si + nitems),
                           (const int*)(si + 2 * nitems));
                }
            });
        } else if (words)
            ft == 512 ? form(k_tile_form<512, true>, 512) : ft == 128 ? form(k_tile_form<128, true>, 128)
                                                          : form(k_tile_form<256, true>, 256);
        else
            ft == 512 ? form(k_tile_form<512, false>, 512) : ft == 128 ? form(k_tile_form<128, false>, 128)
                                                           : form(k_tile_form<256, false>, 256);
        if (nsplit > 0 && !vform) {
            auto kc = k_tile_combine<kFormThreads>;
            const size_t smem = sizeof(unsigned) * (W + W / 32) + sizeof(uint16_t) * W;
            ensure_smem(kc, smem);
            launch(c, kc, dim3(nsplit), dim3(kFormThreads), smem, TL, (const int2*)d.items.as<int2>(),
                   (const int*)si, (const int*)(si + nitems), (const int*)(si + 2 * nitems),
                   (const unsigned*)d.partial.as<unsigned>(), d.stash.as<unsigned>(),
                   (const int64_t*)d.soff.as<int64_t>(), (const int64_t*)d.sres.as<int64_t>(), d.cnt.as<int64_t>(),
                   d.form.as<int>(), d.hcnt.as<unsigned long long>(), rbc);
        }
        exclusive_scan_i64(c, d.cnt.as<int64_t>(), d.hoff.as<int64_t>(), nitems + 1);
    }
    // ---- colptr = scan(light + heavy counts)
    {
        KScope ks(c, KC_SCAN);
        DevBuf tot(sizeof(int64_t) * (n + 1), c.stream);
        SLAPCU_CUDA(cudaMemsetAsync(tot.as<int64_t>() + n, 0, sizeof(int64_t), c.stream));
        launch(c, k_add_counts, dim3(grid_for(c, n, 256)), dim3(256), 0, n, (const int64_t*)f.cnt.as<int64_t>(),
               (const unsigned long long*)d.hcnt.as<unsigned long long>(), tot.as<int64_t>());
        exclusive_scan_i64(c, tot.as<int64_t>(), c_colptr, n + 1);
    }
    const int64_t total = d2h(c, c_colptr + n);
    d.last_nnz = total;
    if (vform && nitems > 0 && total <= capacity &&
        d2h(c, reinterpret_cast<const int*>(vcur.as<unsigned long long>() + 1)) != 0)
        throw Fail{SLAPCU_ERR_CUDA, "value form: value stash overflow"};
    if (total > capacity)
        throw Fail{SLAPCU_ERR_BUDGET, "output needs " + std::to_string(total) + " entries, capacity " +
                                          std::to_string(capacity)};
    // value pass parameters: rank chunks (every item, 4-byte values) or the
    // small-item hash table + rank chunks (8-byte values)
    const bool rank_path = c.opt.direct_value_rank != 0 && TL >= 12;
    const int hopt = c.opt.direct_value_hash >= 0 ? c.opt.direct_value_hash
                                                  : ((value_size(sr) == 4 && rank_path) ? 0 : 1);
    // option: 4-byte values, every item through rank chunks (they read the form's
    // stash, not C's rows): the chunks write C's rows too and the emit pass is
    // skipped -- measured slower (409 -> 458 ms at MinPlus C3: the chunks' row
    // stores are per thread, emit stages them for 16-byte stores)
    const bool rows_by_values = nitems > 0 && !ones && !vform && rank_path && hopt == 0 &&
                                c.opt.direct_value_rows != 0;
    if (nitems > 0 && !rows_by_values) {
        KScope ks(c, KC_NUM_HEAVY);
        EmitArgs e{(const int2*)d.items.as<int2>(), (const int64_t*)d.cnt.as<int64_t>(), (const int*)d.form.as<int>(),
                   (const unsigned*)d.stash.as<unsigned>(), (const int64_t*)d.soff.as<int64_t>(),
                   (const int64_t*)d.hoff.as<int64_t>(), (const int64_t*)d.lp.as<int64_t>(), TL, crw,
                   (ones || vform) ? static_cast<uint8_t*>(cv) : nullptr,  // 1s / the value form's values, else the value pass
                   value_size(sr), value_pattern(sr, ones), nitems,
                   vform ? (const uint8_t*)vst.get() : nullptr, vform ? (const int64_t*)voff.as<int64_t>() : nullptr};
        const size_t smem = 0;
        auto emit = [&](auto ke, int nt) {
            ensure_smem(ke, smem);
            launch(c, ke, dim3((unsigned)((nitems + nt / 32 - 1) / (nt / 32))), dim3(nt), smem, e);
        };
#ifndef SLAPCU_EMIT_NT
#define SLAPCU_EMIT_NT 32  // one warp, one item per CTA (C3: 39.1 ms; 2 / 4 / 8 items per CTA 44.4 / 41.2 / 50.7:
                            // a CTA lives as long as its largest item)
#endif
        emit(k_tile_emit<SLAPCU_EMIT_NT>, SLAPCU_EMIT_NT);  // (per-warp state is static shared memory)
    }
    if (nitems > 0 && !ones && !vform) {
        KScope ks(c, KC_NUM_HEAVY);
        // sub-tiles are whole 4096-row blocks of the item (or the item itself)
        const int VTL = std::min(TL, std::max(12, c.opt.direct_value_tile_log2));
        const int Tv = (int)((A.nrows + (int64_t(1) << VTL) - 1) >> VTL);
        // (one cached table at a time: only the sub-tile path needs 2^VTL rows)
        const int32_t* Atpv = rank_path ? nullptr : value_tile_pointers(c, A, afp, VTL, Tv);
        const int32_t* Atp = tile_pointers(c, A, afp, TL, T);
        // small items (<= kHashCap outputs) take the one-walk hash kernel
        // auto (hopt above): 4-byte values take every item through the rank chunks (C3 MinPlus
        // 561 -> 531 ms, C4 product 66.1 -> 63.9 ms); 8-byte values keep the hash kernel for small items
        const int hlog2 = hopt >= 14 ? 14 : 13;  // table slots (load <= 1/2)
        const int64_t hcap = hopt ? (int64_t(1) << hlog2) / 2 : -1;
        DevBuf lists(sizeof(int) * (2 * size_t(nitems) + 2), c.stream), lc(sizeof(int) * 2, c.stream);
        SLAPCU_CUDA(cudaMemsetAsync(lc.get(), 0, sizeof(int) * 2, c.stream));
        int* small = lists.as<int>();
        int* large = small + nitems;
        launch(c, k_value_split, dim3(grid_for(c, nitems, 256)), dim3(256), 0, nitems,
               (const int64_t*)d.cnt.as<int64_t>(), hcap, small, large, lc.as<int>());
        int nsl[2];
        SLAPCU_CUDA(cudaMemcpyAsync(nsl, lc.get(), sizeof(nsl), cudaMemcpyDeviceToHost, c.stream));
        SLAPCU_CUDA(cudaStreamSynchronize(c.stream));
        ValueArgs va{A, B, Atpv, Tv, VTL, TL, Atp, T, (const int2*)d.items.as<int2>(), nullptr,
                     (const int64_t*)d.cnt.as<int64_t>(), (const int64_t*)d.hoff.as<int64_t>(),
                     (const int64_t*)d.lp.as<int64_t>(), (const int*)d.rbc.as<int>(), crw, cv, nullptr, 0,
                     value_tiny_run(c), (const unsigned*)d.stash.as<unsigned>(), (const int64_t*)d.soff.as<int64_t>(),
                     (const int*)d.form.as<int>(), rows_by_values ? crw : nullptr};
        // 4-byte values: A's rows and values interleaved, so a product's gather
        // is one 8-byte load (one sector) instead of one from each array
        DevBuf arv;
        if (value_size(sr) == 4 && A.span > 0 && c.opt.direct_value_interleave) {
            arv = DevBuf(sizeof(int2) * size_t(A.span), c.stream);
            launch(c, k_interleave_rv, dim3(grid_for(c, A.span, 256)), dim3(256), 0, A.span, A.rw + A.base,
                   static_cast<const int32_t*>(A.v) + A.base, arv.as<int2>());
            va.arv = arv.as<int2>() - A.base;
        } else if (value_size(sr) == 8 && A.span > 0 && c.opt.direct_value_interleave == 2) {
            // opt-in: at C2 / C5 (fp64, cf ~1-1.4) the 16-byte copy did not pay (C5 12.0 -> 12.2 ms)
            arv = DevBuf(sizeof(int4) * size_t(A.span), c.stream);
            launch(c, k_interleave_rv8, dim3(grid_for(c, A.span, 256)), dim3(256), 0, A.span, A.rw + A.base,
                   static_cast<const long long*>(A.v) + A.base, arv.as<int4>());
            va.arv = arv.as<int4>() - A.base;
        }
        dispatch_sr(sr, [&](auto id) {
            constexpr int ID = decltype(id)::value;
            using Acc = typename Sr<ID>::Acc;
            if (nsl[0] > 0) {
                va.list = small;
                const size_t smem = (sizeof(Acc) + sizeof(int)) << hlog2;
                auto go = [&](auto k, int nt) {
                    ensure_smem(k, smem);
                    launch(c, k, dim3(nsl[0]), dim3(nt), smem, va);
                };
                const bool wide = c.opt.direct_value_threads == 512;
                if (hlog2 == 14)
                    wide ? go(k_item_values_hash<ID, 512, 14>, 512) : go(k_item_values_hash<ID, 256, 14>, 256);
                else
                    wide ? go(k_item_values_hash<ID, 512, 13>, 512) : go(k_item_values_hash<ID, 256, 13>, 256);
            }
            if (nsl[1] > 0 && rank_path) {
                // large items by rank chunks over 4096-row blocks (tile pointers at 2^12 rows)
                // 8192 4-byte slots keep 3 CTAs of 512 threads per SM (C3 MinPlus: values
                // 498 -> 441 ms vs 4096; 6144 467, 10240 508, 12288 492 ms)
                const int cap = c.opt.direct_value_rank > 0 ? c.opt.direct_value_rank : (sizeof(Acc) <= 4 ? 10240 : 4096);
                // chunks spanning at most dense_rows rows fold by row offset (no ranks)
                constexpr int kBlkRows4096 = 4096;
                int dense_rows = std::max(
                    cap, (c.opt.direct_value_dense_rows > 0 ? c.opt.direct_value_dense_rows : cap) / kBlkRows4096 * kBlkRows4096);
                while (dense_rows > cap && sizeof(Acc) * size_t(dense_rows) + sizeof(unsigned) * W + sizeof(uint16_t) * W +
                                                   sizeof(int) * (W / 32) + 16 > size_t(c.smem_optin) - 8192)
                    dense_rows -= kBlkRows4096;  // (a larger dense span than shared memory holds)
                const int chunk_cap = cap;
                const int T12 = (int)((A.nrows + 4095) >> 12);
                ValueArgs vr = va;
                const bool tmajor = c.opt.direct_value_tmajor != 0;
                vr.Atpv = value_tile_pointers(c, A, afp, 12, T12, tmajor);
                vr.Tv = T12;
                vr.VTL = 12;
                vr.tv_stride = tmajor ? A.ncols : 0;
                const int nrb = (W + kRbcWords - 1) / kRbcWords;
                DevBuf ccount(sizeof(int64_t) * (size_t(nsl[1]) + 1), c.stream),
                    coff(sizeof(int64_t) * (size_t(nsl[1]) + 1), c.stream);
                SLAPCU_CUDA(cudaMemsetAsync(ccount.as<int64_t>() + nsl[1], 0, sizeof(int64_t), c.stream));
                launch(c, k_rank_chunks, dim3(grid_for(c, nsl[1], 256)), dim3(256), 0, nsl[1], (const int*)large,
                       (const int*)d.rbc.as<int>(), nrb, chunk_cap, dense_rows / kBlkRows4096, (const int64_t*)nullptr,
                       ccount.as<int64_t>(), (RankChunk*)nullptr);
                exclusive_scan_i64(c, ccount.as<int64_t>(), coff.as<int64_t>(), nsl[1] + 1);
                const int64_t nch = d2h(c, coff.as<int64_t>() + nsl[1]);
                DevBuf chunks(sizeof(RankChunk) * std::max<int64_t>(nch, 1), c.stream);
                launch(c, k_rank_chunks, dim3(grid_for(c, nsl[1], 256)), dim3(256), 0, nsl[1], (const int*)large,
                       (const int*)d.rbc.as<int>(), nrb, chunk_cap, dense_rows / kBlkRows4096,
                       (const int64_t*)coff.as<int64_t>(), ccount.as<int64_t>(), chunks.as<RankChunk>());
                if (c.opt.direct_value_tmajor && nch > 1) {  // row-block order (L2 locality of A and the table)
                    DevBuf key(sizeof(int) * nch, c.stream), kout(sizeof(int) * nch, c.stream),
                        idx(sizeof(int) * nch, c.stream), ord(sizeof(int) * nch, c.stream),
                        sorted(sizeof(RankChunk) * nch, c.stream);
                    launch(c, k_chunk_keys, dim3(grid_for(c, nch, 256)), dim3(256), 0, nch,
                           (const RankChunk*)chunks.as<RankChunk>(), (const int2*)d.items.as<int2>(), TL, key.as<int>(),
                           idx.as<int>());
                    size_t tb = 0;
                    SLAPCU_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, key.as<int>(), kout.as<int>(), idx.as<int>(),
                                                                ord.as<int>(), (int)nch, 0, 31, c.stream));
                    DevBuf tmp(tb, c.stream);
                    timed(c, KC_BIN, [&] {
                        SLAPCU_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), tb, key.as<int>(), kout.as<int>(),
                                                                    idx.as<int>(), ord.as<int>(), (int)nch, 0, 31,
                                                                    c.stream));
                    });
                    ++c.launches;
                    launch(c, k_chunk_gather, dim3(grid_for(c, nch, 256)), dim3(256), 0, nch,
                           (const RankChunk*)chunks.as<RankChunk>(), (const int*)ord.as<int>(), sorted.as<RankChunk>());
                    chunks = std::move(sorted);
                }
                const size_t smem = ((sizeof(Acc) * size_t(std::max(cap, dense_rows)) + 15) & ~size_t(15)) +
                                    sizeof(unsigned) * W + sizeof(uint16_t) * W + sizeof(int) * (W / 32) + 16;
                auto gor = [&](auto k, int nt) {
                    ensure_smem(k, smem);
                    launch(c, k, dim3((unsigned)nch), dim3(nt), smem, vr, (const RankChunk*)chunks.as<RankChunk>(),
                           cap, dense_rows);
                };
                if (c.opt.direct_value_threads == 512)
                    gor(k_item_values_rank<ID, 512>, 512);
                else
                    gor(k_item_values_rank<ID, 256>, 256);
            } else if (nsl[1] > 0) {
                va.list = large;
                const size_t smem = sizeof(Acc) * (size_t(1) << VTL);
                if (smem > size_t(c.smem_optin) - 16 * 1024)
                    throw Fail{SLAPCU_ERR_INVALID, "value tile too large for shared memory"};
                auto go = [&](auto k, int nt) {
                    ensure_smem(k, smem);
                    launch(c, k, dim3((unsigned)(int64_t(nsl[1]) << (TL - VTL))), dim3(nt), smem, va);
                };
                if (c.opt.direct_value_threads == 512)
                    go(k_tile_values<ID, 512>, 512);
                else
                    go(k_tile_values<ID, 256>, 256);
            }
        });
    }
    if (nlight) {
        KScope ks(c, KC_NUM_LIGHT);
        fused_copy_light(c, sr, ones, L, nlight, f, c_colptr, crw, cv);
    }
    SLAPCU_CUDA(cudaEventRecord(c.ev[1], c.stream));
    SLAPCU_CUDA(cudaStreamSynchronize(c.stream));
    cudaEventElapsedTime(&c.sym_ms, c.ev[0], c.ev[1]);
    prof_flush(c);
    return total;
}

// The direct product into library-owned, exactly sized buffers (the
// one-shot / host / distributed entry points): C lands in a bound-sized
// scratch kept on the context, then moves into cudaMallocAsync'd buffers of
// nnz entries.  Returns false (nothing allocated) when the scratch would not
// fit in `budget` bytes -- callers then take the staged or two-pass path.
bool direct_exact(Ctx& c, const DevCsc& A_, const DevCsc& B_, int sr, int alg, int64_t budget, int64_t** cp,
                  int32_t** rw, void** v, int64_t* nnz, bool copy_out) {
    check_operands(A_, B_);
    const int vs = value_size(sr);
    DevCsc A = A_, B = B_;
    resolve(c, A);
    resolve(c, B);
    const int64_t N = B.ncols;
    DevBuf fl(sizeof(int64_t) * std::max<int64_t>(N, 1), c.stream);
    int64_t tot = 0;
    spgemm_flops(c, A, B, fl.as<int64_t>(), &tot);
    // the output bound sum_j min(flops_j, nrows), reduced on the device (one 8-byte read back)
    DevBuf bsum(sizeof(unsigned long long), c.stream);
    SLAPCU_CUDA(cudaMemsetAsync(bsum.get(), 0, sizeof(unsigned long long), c.stream));
    if (N)
        launch(c, k_sum_min, dim3(grid_for(c, N, 256)), dim3(256), 0, N, (const int64_t*)fl.as<int64_t>(), A.nrows,
               bsum.as<unsigned long long>());
    const int64_t cap = (int64_t)d2h(c, bsum.as<unsigned long long>());
    if (budget > 0 && cap * (4 + vs) > budget) return false;
    DirectCache& d = c.direct;
    d.dist_rw.reset(sizeof(int32_t) * std::max<int64_t>(cap, 1), c.stream);
    d.dist_v.reset(size_t(vs) * std::max<int64_t>(cap, 1), c.stream);
    SLAPCU_CUDA(cudaMallocAsync((void**)cp, sizeof(int64_t) * (N + 1), c.stream));
    try {
        *nnz = direct_spgemm(c, A_, B_, sr, alg, cap, *cp, d.dist_rw.as<int32_t>(), d.dist_v.get());
    } catch (...) {
        cudaFreeAsync(*cp, c.stream);
        *cp = nullptr;
        throw;
    }
    if (!copy_out) {  // entries stay in the context's scratch (valid until the next direct call)
        *rw = d.dist_rw.as<int32_t>();
        *v = d.dist_v.get();
        return true;
    }
    SLAPCU_CUDA(cudaMallocAsync((void**)rw, sizeof(int32_t) * std::max<int64_t>(*nnz, 1), c.stream));
    SLAPCU_CUDA(cudaMallocAsync(v, size_t(vs) * std::max<int64_t>(*nnz, 1), c.stream));
    if (*nnz) {
        SLAPCU_CUDA(cudaMemcpyAsync(*rw, d.dist_rw.get(), sizeof(int32_t) * *nnz, cudaMemcpyDeviceToDevice, c.stream));
        SLAPCU_CUDA(cudaMemcpyAsync(*v, d.dist_v.get(), size_t(vs) * *nnz, cudaMemcpyDeviceToDevice, c.stream));
    }
    return true;
}

}  // namespace slapcu

#ifdef SLAPCU_VCOUNT
// debug variant only: value-walk counters (entry visits, nonempty runs, products, batches)
extern "C" int slapcu_debug_vcount(unsigned long long* out, int reset) {
    cudaMemcpyFromSymbol(out, slapcu::g_vcount, sizeof(unsigned long long) * 12);
    if (reset) {
        unsigned long long z[12] = {};
        cudaMemcpyToSymbol(slapcu::g_vcount, z, sizeof(z));
    }
    return 0;
}
#endif
