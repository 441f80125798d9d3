// ops.cu — homomorphic statistics (K-STAT), regional reductions (K-REG) and
// integer finite-difference stencils (K-STEN).
//
// Exactness: integer sums are accumulated in int128 per thread and reduced
// deterministically (per-CTA partials + one finalize CTA); the host finishes
// with the reference's own Python-int expressions (analytics/stats.py:58-62,
// 69-77, 92, 118, 130-138), so scalars are bit-identical.  Stencil outputs
// reproduce the reference's fp64 rounding sequence exactly (int stencil, one
// multiply by eps or 2*eps — analytics/fields.py:67-80 — or, in the float
// domain, fields.py:83-93 operation by operation), then round to the output
// type.
#include <cstdio>
#include <cstdlib>
#include "tile.cuh"
#include "async.cuh"
#include "moments.cuh"
#include "wtiles.cuh"
#include "stencil.cuh"

namespace hszg {

constexpr int RED_THREADS = 256;

__device__ __forceinline__ uint64_t sq64(int v) { return (uint64_t)((int64_t)v * (int64_t)v); }

// ---- per-chunk accumulators for the fused stream reductions -----------------

// mode 1/2: sum over the row-major box of w * p with w = (N0-i0)(N1-i1)(N2-i2)
// (stats.py:88 for HSZP, the separable Lorenzo weights of stats.py:95-112)
struct WeightedChunk {
    int64_t N0, N1, N2;
    int64_t w0, i1, i2;
    i128 csum;
    __device__ __forceinline__ void begin(const SegGeo& sg, const ChunkLoc& L, const int32_t*) {
        N0 = sg.n[0]; N1 = sg.n[1]; N2 = sg.n[2];
        const int64_t plane = N1 * N2;
        const int64_t i0 = L.start / plane;
        const int64_t rem = L.start - i0 * plane;
        i1 = rem / N2;
        i2 = rem - i1 * N2;
        w0 = N0 - i0;
        csum = 0;
    }
    __device__ __forceinline__ void take(Acc&, int, int32_t v) {
        const int64_t w12 = (N1 - i1) * (N2 - i2);
        csum += (i128)w12 * (i128)v;
        if (++i2 == N2) {
            i2 = 0;
            ++i1;   // chunks never cross planes (segments are planes / rows / 1-D blocks)
        }
    }
    __device__ __forceinline__ void end(Acc& a, int count) {
        a.s1 += csum * (i128)w0;
        a.count += count;
    }
};

// mode 3: q = p + M_b in stream order (HSZX*): sum, sum of squares, min, max
struct MetaChunk {
    int32_t m;
    __device__ __forceinline__ void begin(const SegGeo&, const ChunkLoc& L, const int32_t* meta) { m = __ldg(meta + L.seg); }
    __device__ __forceinline__ void take(Acc& a, int, int32_t v) {
        const int32_t q = v + m;
        a.s1 += q;
        a.s2 += (i128)((int64_t)q * (int64_t)q);
        a.vmin = min(a.vmin, q);
        a.vmax = max(a.vmax, q);
    }
    __device__ __forceinline__ void end(Acc& a, int count) { a.count += count; }
};

template <class CA>
__global__ void __launch_bounds__(TILE_CHUNKS) k_reduce_tiles(SegGeo sg, const uint8_t* payload, uint64_t len,
                                                             const uint64_t* offsets, const int32_t* meta,
                                                             HszgSums* partials) {
    TileCtx t = tile_stage(sg, payload, len, offsets, blockIdx.x);
    Acc a;
    a.init();
    const int64_t c = t.c0 + threadIdx.x;
    if (c < t.c1) {
        const ChunkLoc L = locate_chunk(sg, c);
        CA ca;
        ca.begin(sg, L, meta);
        decode_chunk_words(t.words, (uint32_t)(offsets[c] - t.base), L.count,
                           [&](int j, int32_t v) { ca.take(a, j, v); });
        ca.end(a, L.count);
    }
    block_reduce(a);
    if (threadIdx.x == 0) store_sums(partials + blockIdx.x, a);
}

// Grid-strided 256-chunk tiles with double-buffered staging: the byte range of the CTA's next tile is
// copied with 16-B cp.async into the other buffer while the current one decodes (two barriers per
// tile).  Each thread's index entries (chunk start / end bytes) and one auxiliary word per chunk
// (aux(c), e.g. its block mean) are loaded two tiles ahead, so no global-load latency sits between a
// tile's barriers.  body(c, words, rel, valid, aux) handles chunk c (words: the staged bytes, rel: its
// byte offset there); every thread of the CTA calls it each tile (valid = false past the last chunk),
// so warps stay converged for warp-uniform decode decisions.
struct NoAux {
    __device__ __forceinline__ int32_t operator()(int64_t) const { return 0; }
};

template <typename Body, typename Aux = NoAux>
__device__ __forceinline__ void staged_tiles(const uint8_t* __restrict__ payload, uint64_t len,
                                             const uint64_t* __restrict__ offsets, int64_t n_chunks, uint8_t* smem,
                                             uint32_t buf_bytes, Body body, Aux aux = Aux()) {
    // byte ranges of the CTA's i-th tile in slot i % 3: a thread one iteration ahead writes a slot no
    // thread still reads (barrier A of the next iteration separates the third)
    __shared__ uint64_t s_lo[3], s_hi[3];
    const int64_t tiles = (n_chunks + TILE_CHUNKS - 1) / TILE_CHUNKS;
    const int64_t G = gridDim.x;
    struct Ent {
        uint64_t off, end;
        int32_t aux;
    };
    auto fetch = [&](int64_t t, Ent& e) {          // this thread's chunk of tile t: start / end bytes, aux
        const int64_t c = t * TILE_CHUNKS + threadIdx.x;
        if (t < tiles && c < n_chunks) {
            e.off = __ldg(offsets + c);
            e.end = c + 1 < n_chunks ? __ldg(offsets + c + 1) : payload_end(offsets, n_chunks, len);
            e.aux = aux(c);
        }
    };
    auto publish = [&](int64_t t, int r, const Ent& e) {   // the tile's byte range, from its first / last chunk
        const int64_t c0 = t * TILE_CHUNKS;
        const int nch = (int)(n_chunks - c0 < TILE_CHUNKS ? n_chunks - c0 : TILE_CHUNKS);
        if (threadIdx.x == 0) s_lo[r] = e.off;
        if ((int)threadIdx.x == nch - 1) s_hi[r] = e.end;
    };
    auto issue = [&](int b, int r) {
        uint4* sb = reinterpret_cast<uint4*>(smem + (size_t)b * buf_bytes);
        const uint64_t base = s_lo[r] & ~(uint64_t)15;
        const uint32_t nvec = (uint32_t)((s_hi[r] - base + 15) >> 4);
        const uint4* g = reinterpret_cast<const uint4*>(payload + base);
        for (uint32_t i = threadIdx.x; i < nvec; i += blockDim.x) cp_async16(sb + i, g + i);
        if (threadIdx.x == 0) sb[nvec] = make_uint4(0, 0, 0, 0);   // the bit cursor's look-ahead word
        cp_async_commit();
    };
    int64_t t = blockIdx.x;
    if (t >= tiles) return;
    Ent A = {0, 0, 0}, B = {0, 0, 0};
    fetch(t, A);
    publish(t, 0, A);
    fetch(t + G, B);
    __syncthreads();
    issue(0, 0);
    for (int i = 0; t < tiles; t += G, i++) {
        const int b = i & 1, r = i % 3, rn = (i + 1) % 3;
        const int64_t tn = t + G;
        const Ent cur = A;
        if (tn < tiles) publish(tn, rn, B);         // B was loaded an iteration ago
        A = B;
        fetch(tn + G, B);                           // two tiles ahead: consumed next iteration
        __syncthreads();                            // (A) next range visible; buffer b^1 no longer read
        if (tn < tiles) issue(b ^ 1, rn);
        else cp_async_commit();                     // keep one group per iteration
        cp_async_wait<1>();                         // this thread's copies of tile t landed
        __syncthreads();                            // (B) everyone's
        const int64_t c = t * TILE_CHUNKS + threadIdx.x;
        const uint64_t base = s_lo[r] & ~(uint64_t)15;
        const bool valid = c < n_chunks;
        body(c, reinterpret_cast<const uint32_t*>(smem + (size_t)b * buf_bytes), valid ? (uint32_t)(cur.off - base) : 0u,
             valid, cur.aux);
    }
    cp_async_wait<0>();
}

// Exact per-thread accumulation of q = p + m moments from chunk moments of p (32 full values):
//   sum q = sum p + 32 m,  sum q^2 = sum p^2 + 2 m sum p + 32 m^2.
// Narrow chunks (|sum p| < 2^24, sum p^2 < 2^40, |m| < 2^25) accumulate the three terms in 64-bit
// registers, folded into int128 every 2048 chunks (bounds: 2^51, 2^60, 2^61); the rest take the
// 128-bit algebra directly.
struct QMomAcc {
    int64_t s1 = 0;
    i128 s2 = 0;
    uint64_t sq = 0;
    int64_t msp = 0;
    uint64_t mm = 0;
    int n = 0;
    __device__ __forceinline__ void fold() {
        s2 += (i128)sq + 2 * (i128)msp + 32 * (i128)mm;
        sq = 0;
        msp = 0;
        mm = 0;
        n = 0;
    }
    __device__ __forceinline__ void add(const ChunkMoments& r, int64_t m) {
        s1 += r.sp + 32 * m;
        if (r.sq >> 40 == 0 && r.sp > -(1ll << 24) && r.sp < (1ll << 24) && m > -(1ll << 25) && m < (1ll << 25)) {
            sq += (uint64_t)r.sq;
            msp += m * r.sp;
            mm += (uint64_t)(m * m);
            if (++n == 2048) fold();
        } else {
            s2 += (i128)r.sq + (i128)(2 * m) * (i128)r.sp + (i128)(32 * m) * (i128)m;
        }
    }
    __device__ __forceinline__ i128 total() {
        fold();
        return s2;
    }
};

// MetaChunk fast path: every chunk full and every segment full-size (chunk c belongs to segment
// c / cps): per chunk the lean moments of p (moments.cuh), then the q algebra above; the block mean
// comes with the index entries (warp_tiles, wtiles.cuh).  One partial per CTA.
template <bool MINMAX>
__global__ void __launch_bounds__(256, HSZG_WT_MINB_S) k_reduce_meta_fast(const uint8_t* __restrict__ payload, uint64_t len,
                                                                  const uint64_t* __restrict__ offsets, int64_t n_chunks,
                                                                  MetaAux aux, int64_t n, HszgSums* partials,
                                                                  uint32_t buf_bytes) {
    extern __shared__ __align__(16) uint8_t smem[];
    Acc a;
    a.init();
    QMomAcc q;
    warp_tiles(payload, len, offsets, n_chunks, smem + (threadIdx.x >> 5) * WT_NS * buf_bytes, buf_bytes,
               wt_bars(smem, buf_bytes), [&](int64_t, const uint32_t* words, uint32_t rel, bool valid, int32_t m) {
        const ChunkMoments r = chunk_moments<false, MINMAX>(words, rel, valid);
        if (!valid) return;
        q.add(r, m);
        if (MINMAX) {
            a.vmin = min(a.vmin, r.mn + m);
            a.vmax = max(a.vmax, r.mx + m);
        }
    }, aux);
    a.s1 = q.s1;
    a.s2 = q.total();
    block_reduce(a);
    if (threadIdx.x == 0) {
        a.count = blockIdx.x ? 0 : n;
        store_sums(partials + blockIdx.x, a);
    }
}

// WeightedChunk fast path (stats.py:80-112: sum of (N0-i0)(N1-i1)(N2-i2) p over the box): every chunk
// full and inside one row (n2 % 32 == 0), so a chunk starting at (i0, i1, x0) contributes
// (N0-i0)(N1-i1)[(N2-x0) S - T] with S = sum p_j, T = sum j p_j — the lean moments with TSUM;
// warp-private tiles as k_reduce_meta_fast.
__global__ void __launch_bounds__(256, HSZG_WT_MINB_S) k_reduce_weighted_fast(const uint8_t* __restrict__ payload,
                                                                      uint64_t len,
                                                                      const uint64_t* __restrict__ offsets,
                                                                      int64_t n_chunks, int64_t N0, int64_t N1,
                                                                      int64_t N2, int64_t n, HszgSums* partials,
                                                                      uint32_t buf_bytes) {
    extern __shared__ __align__(16) uint8_t smem[];
    Acc a;
    a.init();
    const int64_t cpr = N2 / kChunkCap;
    i128 s1 = 0;
    warp_tiles(payload, len, offsets, n_chunks, smem + (threadIdx.x >> 5) * WT_NS * buf_bytes, buf_bytes,
               wt_bars(smem, buf_bytes), [&](int64_t c, const uint32_t* words, uint32_t rel, bool valid, int32_t) {
        const ChunkMoments r = chunk_moments<true, false>(words, rel, valid);
        if (!valid) return;
        const int64_t row = c / cpr, x0 = (c - row * cpr) * kChunkCap;
        const int64_t i0 = row / N1, i1 = row - i0 * N1;
        const i128 inner = (i128)(N2 - x0) * r.sp - r.tp;
        s1 += (i128)((N0 - i0) * (N1 - i1)) * inner;
    });
    a.s1 = s1;
    block_reduce(a);
    if (threadIdx.x == 0) {
        a.count = blockIdx.x ? 0 : n;
        store_sums(partials + blockIdx.x, a);
    }
}

// ---- HSZP variance by tile algebra (stats.py:168-173 sums of q = cumsum(p), compressors.py:212) ----
// q_i = C_t + L_i inside a 32-chunk warp tile t, C_t = q just before the tile (the exclusive prefix of
// the tile totals, exact in int32 wrap-around because every q fits int32) and L_i the tile-local prefix.
//   sum q = sum_t (n_t C_t + sum L),   sum q^2 = sum_t (sum L^2 + 2 C_t sum L + n_t C_t^2)
// k_hszp_tile_sums decodes each tile once (warp-private TMA tiles, running-prefix chunk moments, a warp
// scan of the chunk totals) and writes (T_t, sum L, sum L^2); k_hszp_tile_combine scans T_t and folds
// the algebra in int128.  No look-back chain, q never stored.
struct HszpTileRec {
    int64_t T;         // tile total of p
    int64_t s1;        // sum of the tile-local prefixes L
    uint64_t s2lo;     // sum L^2 (u128)
    uint64_t s2hi;
    int64_t mn, mx;    // min / max of L (q = C_t + L: the extrema of q follow in the combine)
};

__global__ void __launch_bounds__(256, HSZG_WT_MINB_S) k_hszp_tile_sums(const uint8_t* __restrict__ payload, uint64_t len,
                                                        const uint64_t* __restrict__ offsets, int64_t n_chunks,
                                                        HszpTileRec* rec, uint32_t buf_bytes) {
    extern __shared__ __align__(16) uint8_t smem[];
    const int lane = threadIdx.x & 31;
    warp_tiles(payload, len, offsets, n_chunks, smem + (threadIdx.x >> 5) * WT_NS * buf_bytes, buf_bytes,
               wt_bars(smem, buf_bytes), [&](int64_t c, const uint32_t* words, uint32_t rel, bool valid, int32_t) {
        const PrefixMoments r = prefix_moments(words, rel, valid);
        int64_t inc = r.T;                                   // warp inclusive scan of the chunk totals
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int64_t o = __shfl_up_sync(0xffffffffu, inc, d);
            if (lane >= d) inc += o;
        }
        const int64_t E = inc - r.T;                          // chunk offset inside the tile
        int64_t s1 = 32 * E + r.S1;
        i128 s2 = (i128)r.S2 + (i128)(2 * E) * (i128)r.S1 + (i128)(32 * E) * (i128)E;
        int64_t mn = E + r.mn, mx = E + r.mx;
        if (!valid) {
            s1 = 0;
            s2 = 0;
            mn = INT64_MAX;
            mx = INT64_MIN;
        }
        uint64_t lo = (uint64_t)(u128)s2, hi = (uint64_t)((u128)s2 >> 64);
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
            s1 += (int64_t)__shfl_down_sync(0xffffffffu, (unsigned long long)s1, d);
            const uint64_t olo = __shfl_down_sync(0xffffffffu, lo, d), ohi = __shfl_down_sync(0xffffffffu, hi, d);
            const u128 t = (((u128)hi << 64) | lo) + (((u128)ohi << 64) | olo);
            lo = (uint64_t)t;
            hi = (uint64_t)(t >> 64);
            mn = min(mn, (int64_t)__shfl_down_sync(0xffffffffu, (unsigned long long)mn, d));
            mx = max(mx, (int64_t)__shfl_down_sync(0xffffffffu, (unsigned long long)mx, d));
        }
        const int64_t total = __shfl_sync(0xffffffffu, inc, 31);
        if (lane == 0) rec[c >> 5] = HszpTileRec{total, s1, lo, hi, mn, mx};
    });
}

// Tile combine over NB CTAs: CTA b owns tiles [b*per, (b+1)*per), each thread a contiguous run of them.
constexpr int HC_THREADS = 256;

__device__ __forceinline__ void hc_range(int64_t tiles, int64_t& t0, int64_t& t1) {
    const int64_t per = (tiles + gridDim.x - 1) / gridDim.x;
    const int64_t b0 = blockIdx.x * per, b1 = b0 + per < tiles ? b0 + per : tiles;
    const int64_t tp = (per + HC_THREADS - 1) / HC_THREADS;
    t0 = b0 + threadIdx.x * tp;
    t1 = t0 + tp < b1 ? t0 + tp : b1;
    if (t0 > b1) t0 = b1;
}

// phase 1: each CTA's wrap-around sum of its tile totals
__global__ void __launch_bounds__(HC_THREADS) k_hszp_block_totals(const HszpTileRec* __restrict__ rec, int64_t tiles,
                                                                  uint32_t* __restrict__ bt) {
    int64_t t0, t1;
    hc_range(tiles, t0, t1);
    uint32_t sum = 0;
    for (int64_t t = t0; t < t1; t++) sum += (uint32_t)rec[t].T;
    for (int d = 16; d > 0; d >>= 1) sum += __shfl_down_sync(0xffffffffu, sum, d);
    __shared__ uint32_t ws[HC_THREADS / 32];
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = sum;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t v = 0;
        for (int i = 0; i < HC_THREADS / 32; i++) v += ws[i];
        bt[blockIdx.x] = v;
    }
}

// phase 2: carries (exclusive prefix of the CTA totals, then of the threads' runs) and the int128 algebra
__global__ void __launch_bounds__(HC_THREADS) k_hszp_tile_combine(const HszpTileRec* __restrict__ rec, int64_t tiles,
                                                                  int64_t n, const uint32_t* __restrict__ bt,
                                                                  HszgSums* partials) {
    __shared__ uint32_t s_run[HC_THREADS];
    __shared__ uint32_t s_base;
    uint32_t base = 0;
    for (int i = threadIdx.x; i < (int)blockIdx.x; i += HC_THREADS) base += bt[i];
    for (int d = 16; d > 0; d >>= 1) base += __shfl_down_sync(0xffffffffu, base, d);
    if (threadIdx.x == 0) s_base = 0;
    __syncthreads();
    if ((threadIdx.x & 31) == 0) atomicAdd(&s_base, base);
    int64_t t0, t1;
    hc_range(tiles, t0, t1);
    uint32_t sum = 0;
    for (int64_t t = t0; t < t1; t++) sum += (uint32_t)rec[t].T;
    s_run[threadIdx.x] = sum;
    __syncthreads();
    for (int d = 1; d < HC_THREADS; d <<= 1) {              // inclusive scan (uint32 wrap)
        const uint32_t v = threadIdx.x >= (unsigned)d ? s_run[threadIdx.x - d] : 0u;
        __syncthreads();
        s_run[threadIdx.x] += v;
        __syncthreads();
    }
    uint32_t carry = s_base + s_run[threadIdx.x] - sum;    // q just before this thread's first tile
    Acc a;
    a.init();
    for (int64_t t = t0; t < t1; t++) {
        const HszpTileRec r = rec[t];
        const int64_t C = (int32_t)carry;
        const int64_t nt = (t + 1) * 1024 <= n ? 1024 : n - t * 1024;
        const i128 L2 = (i128)(((u128)r.s2hi << 64) | r.s2lo);
        a.s1 += (i128)nt * C + r.s1;
        a.s2 += L2 + (i128)(2 * C) * (i128)r.s1 + (i128)(nt * C) * (i128)C;
        a.vmin = min(a.vmin, (int32_t)(C + r.mn));            // every q fits int32
        a.vmax = max(a.vmax, (int32_t)(C + r.mx));
        carry += (uint32_t)r.T;
    }
    block_reduce(a);
    if (threadIdx.x == 0) {
        a.count = blockIdx.x ? 0 : n;
        store_sums(partials + blockIdx.x, a);
    }
}

// HSZP (full chunks, canonical) sums of q without the scan: 0 = done, 1 = not applicable
constexpr int HC_BLOCKS = 148 * 4;

size_t hszp_tile_sums_ws(const HszgGeom* g, const HszgStream* s) {
    if (g->kind != HSZG_HSZP || !s->canonical || g->n_chunks * kChunkCap != g->n) return 0;
    const int64_t tiles = (g->n_chunks + 31) / 32;
    return (((size_t)tiles * sizeof(HszpTileRec) + 255) & ~(size_t)255) + HC_BLOCKS * 4 +
           (size_t)(HC_BLOCKS + 1) * sizeof(HszgSums) + 512;
}

}  // namespace hszg
int hszg_finalize_sums(HszgSums* partials, int64_t nparts, HszgSums* out, cudaStream_t st);
namespace hszg {

int hszp_tile_sums(const HszgGeom* g, const HszgStream* s, HszgSums* out_dev, void* ws, size_t ws_bytes,
                   cudaStream_t st) {
    const size_t need = hszp_tile_sums_ws(g, s);
    if (need == 0 || ws_bytes < need) return 1;
    const int64_t tiles = (g->n_chunks + 31) / 32;
    char* w = reinterpret_cast<char*>(ws);
    HszpTileRec* rec = reinterpret_cast<HszpTileRec*>(w);
    const size_t ro = ((size_t)tiles * sizeof(HszpTileRec) + 255) & ~(size_t)255;
    uint32_t* bt = reinterpret_cast<uint32_t*>(w + ro);
    HszgSums* partials = reinterpret_cast<HszgSums*>(w + ro + ((HC_BLOCKS * 4 + 255) & ~255));
    size_t sm;
    uint32_t sb;
    const unsigned grid = wtile_grid(k_hszp_tile_sums, s->max_bitwidth, g->n_chunks, &sm, &sb);
    k_hszp_tile_sums<<<grid, 256, sm, st>>>(s->payload, s->payload_len, s->offsets, g->n_chunks, rec, sb);
    const int nb = (int)(tiles < HC_BLOCKS ? tiles : HC_BLOCKS);
    k_hszp_block_totals<<<nb, HC_THREADS, 0, st>>>(rec, tiles, bt);
    k_hszp_tile_combine<<<nb, HC_THREADS, 0, st>>>(rec, tiles, g->n, bt, partials);
    if (cudaGetLastError() != cudaSuccess) return -1;
    return ::hszg_finalize_sums(partials, nb, out_dev, st) == HSZG_OK ? 0 : -1;
}

// ---- K-REG fused from the bytes (HSZX*: regions of q = p + M_b, no reconstruction) -------------
// Regions tile the box like grid.partition with extents R (a multiple of the block extents B on every
// axis, so each block lies in exactly one region).  Per chunk: the lean moments of p plus the block
// mean (exact q moments), keyed by region; a warp-segmented inclusive scan over the 32 lanes (consecutive
// chunks share a block, hence a region) leaves each run's total on its last lane, which adds it into
// the region's accumulator (int64 S1, S2 as four 32-bit limbs in u64 words, int32 min / max atomics).
// k_region_accum_finish turns the accumulators into the region_buffer layout (s1, s2 lo / hi, size,
// qmin, qmax) for k_region_finalize.
struct RegAccum {
    unsigned long long s1;      // two's complement int64
    unsigned long long l[4];    // S2 limbs (32-bit parts, limb 3 signed)
    int qmin, qmax;
    unsigned long long pad[2];
};
static_assert(sizeof(RegAccum) == 64, "RegAccum layout");

__global__ void k_region_accum_init(RegAccum* acc, int64_t nr) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nr; r += (int64_t)gridDim.x * blockDim.x) {
        RegAccum a;
        a.s1 = 0;
        a.l[0] = a.l[1] = a.l[2] = a.l[3] = 0;
        a.qmin = INT32_MAX;
        a.qmax = INT32_MIN;
        a.pad[0] = a.pad[1] = 0;
        acc[r] = a;
    }
}

struct RegionMap {
    int64_t rg[3];      // region grid
    int64_t bpr[3];     // blocks per region extent (R / B)
};

__global__ void __launch_bounds__(256, HSZG_WT_MINB_S) k_region_fused(SegGeo sg, RegionMap rm, const uint8_t* __restrict__ payload,
                                                              uint64_t len, const uint64_t* __restrict__ offsets,
                                                              const int32_t* __restrict__ meta, bool full_segs,
                                                              int64_t cps, RegAccum* acc, uint32_t buf_bytes) {
    extern __shared__ __align__(16) uint8_t smem[];
    const int lane = threadIdx.x & 31;
    warp_tiles(payload, len, offsets, sg.n_chunks, smem + (threadIdx.x >> 5) * WT_NS * buf_bytes, buf_bytes,
               wt_bars(smem, buf_bytes), [&](int64_t c, const uint32_t* words, uint32_t rel, bool valid, int32_t) {
        const ChunkMoments r = chunk_moments<false, true>(words, rel, valid);
        int64_t key = -1 - lane;                  // lanes without a chunk: unique keys, zero moments
        int64_t s1 = 0;
        i128 s2 = 0;
        int mn = INT32_MAX, mx = INT32_MIN;
        if (valid) {
            int64_t seg;
            if (full_segs) seg = c / cps;
            else seg = locate_chunk(sg, c).seg;
            const int64_t b2 = seg % sg.G[2];
            const int64_t t = seg / sg.G[2];
            const int64_t b1 = t % sg.G[1];
            const int64_t b0 = t / sg.G[1];
            key = ((b0 / rm.bpr[0]) * rm.rg[1] + b1 / rm.bpr[1]) * rm.rg[2] + b2 / rm.bpr[2];
            const int64_t m = __ldg(meta + seg);
            s1 = r.sp + 32 * m;
            s2 = (i128)r.sq + (i128)(2 * m) * (i128)r.sp + (i128)(32 * m) * (i128)m;
            mn = r.mn + (int32_t)m;
            mx = r.mx + (int32_t)m;
        }
        // inclusive segmented scan over runs of equal keys (a key may recur after another run: runs,
        // not keys, are the segments — each run's last lane adds its run into the region)
        const int64_t prev = __shfl_up_sync(0xffffffffu, key, 1);
        const unsigned heads = __ballot_sync(0xffffffffu, lane == 0 || prev != key);
        const int run = __popc(heads & (0xffffffffu >> (31 - lane)));
        uint64_t lo = (uint64_t)(u128)s2, hi = (uint64_t)((u128)s2 >> 64);
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int ok = __shfl_up_sync(0xffffffffu, run, d);
            const int64_t o1 = __shfl_up_sync(0xffffffffu, s1, d);
            const uint64_t olo = __shfl_up_sync(0xffffffffu, lo, d);
            const uint64_t ohi = __shfl_up_sync(0xffffffffu, hi, d);
            const int omn = __shfl_up_sync(0xffffffffu, mn, d);
            const int omx = __shfl_up_sync(0xffffffffu, mx, d);
            if (lane >= d && ok == run) {
                s1 += o1;
                const u128 tt = (((u128)hi << 64) | lo) + (((u128)ohi << 64) | olo);
                lo = (uint64_t)tt;
                hi = (uint64_t)(tt >> 64);
                mn = min(mn, omn);
                mx = max(mx, omx);
            }
        }
        const int64_t next = __shfl_down_sync(0xffffffffu, key, 1);
        if (valid && (lane == 31 || next != key)) {
            RegAccum* a = acc + key;
            atomicAdd(&a->s1, (unsigned long long)s1);
            acc_add_i128(a->l, (i128)(((u128)hi << 64) | lo));
            atomicMin(&a->qmin, mn);
            atomicMax(&a->qmax, mx);
        }
    });
}

// accumulators -> region_buffer words (s1, s2 lo / hi, size, qmin, qmax); sizes in closed form
// Regions that are exactly the stream's blocks (region extent = block extent on every axis, every block full,
// CPS = chunks per block dividing 32): a block's chunks sit in CPS consecutive lanes of one warp tile, so the
// region is reduced by log2(CPS) xor-shuffle steps and its group leader writes the region_buffer entry itself
// (one writer per region: no accumulator, no atomics, no init / finish kernels; key = chunk / CPS).
template <int CPS>
__global__ void __launch_bounds__(256, HSZG_WT_MINB_S) k_region_blocks(const uint8_t* __restrict__ payload, uint64_t len,
                                                               const uint64_t* __restrict__ offsets, int64_t n_chunks,
                                                               const int32_t* __restrict__ meta, int64_t bsize,
                                                               int64_t* s1o, uint64_t* s2lo, int64_t* s2hi,
                                                               int32_t* qmin, int32_t* qmax, int64_t* size,
                                                               uint32_t buf_bytes) {
    extern __shared__ __align__(16) uint8_t smem[];
    const int lane = threadIdx.x & 31;
    warp_tiles(payload, len, offsets, n_chunks, smem + (threadIdx.x >> 5) * WT_NS * buf_bytes, buf_bytes,
               wt_bars(smem, buf_bytes), [&](int64_t c, const uint32_t* words, uint32_t rel, bool valid, int32_t) {
        const ChunkMoments r = chunk_moments<false, true>(words, rel, valid);
        const int64_t seg = c / CPS;
        const int64_t m = valid ? (int64_t)__ldg(meta + seg) : 0;
        int64_t s1 = valid ? r.sp + 32 * m : 0;
        const u128 s2 = valid ? (u128)((i128)r.sq + (i128)(2 * m) * (i128)r.sp + (i128)(32 * m) * (i128)m) : (u128)0;
        uint64_t lo = (uint64_t)s2, hi = (uint64_t)(s2 >> 64);
        int mn = valid ? r.mn + (int32_t)m : INT32_MAX, mx = valid ? r.mx + (int32_t)m : INT32_MIN;
#pragma unroll
        for (int d = 1; d < CPS; d <<= 1) {
            s1 += __shfl_xor_sync(0xffffffffu, s1, d);
            const uint64_t olo = __shfl_xor_sync(0xffffffffu, lo, d), ohi = __shfl_xor_sync(0xffffffffu, hi, d);
            const u128 t = (((u128)hi << 64) | lo) + (((u128)ohi << 64) | olo);
            lo = (uint64_t)t;
            hi = (uint64_t)(t >> 64);
            mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, d));
            mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, d));
        }
        if (valid && (lane & (CPS - 1)) == 0) {
            s1o[seg] = s1;
            s2lo[seg] = lo;
            s2hi[seg] = (int64_t)hi;
            qmin[seg] = mn;
            qmax[seg] = mx;
            size[seg] = bsize;
        }
    });
}

__global__ void k_region_accum_finish(const RegAccum* acc, int64_t n0, int64_t n1, int64_t n2, int64_t R0, int64_t R1,
                                      int64_t R2, int64_t g1, int64_t g2, int64_t nr, int64_t* s1, uint64_t* s2lo,
                                      int64_t* s2hi, int32_t* qmin, int32_t* qmax, int64_t* size) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nr; r += (int64_t)gridDim.x * blockDim.x) {
        const RegAccum a = acc[r];
        s1[r] = (int64_t)a.s1;
        const u128 v = (u128)a.l[0] + ((u128)a.l[1] << 32) + ((u128)a.l[2] << 64) + ((u128)(int64_t)a.l[3] << 96);
        s2lo[r] = (uint64_t)v;
        s2hi[r] = (int64_t)(uint64_t)(v >> 64);
        qmin[r] = a.qmin;
        qmax[r] = a.qmax;
        const int64_t r2 = r % g2, t = r / g2, r1 = t % g1, r0 = t / g1;
        const int64_t e0 = (r0 + 1) * R0 <= n0 ? R0 : n0 - r0 * R0;
        const int64_t e1 = (r1 + 1) * R1 <= n1 ? R1 : n1 - r1 * R1;
        const int64_t e2 = (r2 + 1) * R2 <= n2 ? R2 : n2 - r2 * R2;
        size[r] = e0 * e1 * e2;
    }
}

// same reduction over an already-decoded stream-order array (non-canonical containers)
template <class CA>
__global__ void k_reduce_chunks_array(SegGeo sg, const int32_t* p, const int32_t* meta, HszgSums* partials) {
    Acc a;
    a.init();
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < sg.n_chunks;
         c += (int64_t)gridDim.x * blockDim.x) {
        const ChunkLoc L = locate_chunk(sg, c);
        CA ca;
        ca.begin(sg, L, meta);
        for (int j = 0; j < L.count; j++) ca.take(a, j, p[L.start + j]);
        ca.end(a, L.count);
    }
    block_reduce(a);
    if (threadIdx.x == 0) store_sums(partials + blockIdx.x, a);
}

// mode 4: sum(M_b * S_b) over the metadata (stats.py:69-77)
__global__ void k_reduce_meta(SegGeo sg, const int32_t* meta, HszgSums* partials) {
    Acc a;
    a.init();
    const int64_t nb = sg.G[0] * sg.G[1] * sg.G[2];
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b2 = b % sg.G[2];
        const int64_t r = b / sg.G[2];
        const int64_t b1 = r % sg.G[1];
        const int64_t b0 = r / sg.G[1];
        const int64_t size = seg_ext(sg, 0, b0) * seg_ext(sg, 1, b1) * seg_ext(sg, 2, b2);
        a.s1 += (i128)size * (i128)meta[b];
        a.count += size;
    }
    block_reduce(a);
    if (threadIdx.x == 0) store_sums(partials + blockIdx.x, a);
}

// mode 0 over int32 arrays: sum, sum of squares, min, max
__global__ void k_reduce_i32(const int32_t* src, int64_t n, HszgSums* partials) {
    Acc a;
    a.init();
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t s1 = 0;
    u128 s2 = 0;
    const bool aligned = (reinterpret_cast<uintptr_t>(src) & 15) == 0;
    int64_t head = 0;
    if (aligned) {
        const int4* v4 = reinterpret_cast<const int4*>(src);
        const int64_t n4 = n >> 2;
        int mn = INT32_MAX, mx = INT32_MIN;
        auto take = [&](const int4 v) {
            s1 += (int64_t)v.x + v.y + v.z + v.w;
            s2 += (u128)(sq64(v.x) + sq64(v.y));        // squares <= 2^62: pair sums fit 64 bits
            s2 += (u128)(sq64(v.z) + sq64(v.w));
            mn = min(mn, min(min(v.x, v.y), min(v.z, v.w)));
            mx = max(mx, max(max(v.x, v.y), max(v.z, v.w)));
        };
        int64_t i = tid;
        for (; i + 3 * stride < n4; i += 4 * stride) {   // four 16-B loads in flight per thread
            const int4 v0 = __ldg(v4 + i), v1 = __ldg(v4 + i + stride);
            const int4 v2 = __ldg(v4 + i + 2 * stride), v3 = __ldg(v4 + i + 3 * stride);
            take(v0);
            take(v1);
            take(v2);
            take(v3);
        }
        for (; i < n4; i += stride) take(__ldg(v4 + i));
        a.vmin = mn;
        a.vmax = mx;
        head = n4 << 2;
    }
    a.s2 += (i128)s2;
    for (int64_t i = head + tid; i < n; i += stride) {
        const int32_t v = src[i];
        s1 += v;
        a.s2 += (i128)((int64_t)v * v);
        a.vmin = min(a.vmin, v);
        a.vmax = max(a.vmax, v);
    }
    a.s1 += s1;   // per-thread int64 partial: <= n/(4*threads) terms of |v| <= 2^31, far from overflow
    block_reduce(a);
    if (threadIdx.x == 0) {
        a.count = blockIdx.x ? 0 : n;
        store_sums(partials + blockIdx.x, a);
    }
}

// stage-4 float sums: f1 = sum(fl(q*s)), f2 = sum((fl(q*s) - mean)^2)
__global__ void k_reduce_f64(const int32_t* q, int64_t n, double s, const double* mean, HszgSums* partials) {
    Acc a;
    a.init();
    const double mu = mean ? *mean : 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double d = __dmul_rn((double)q[i], s);
        a.f1 = __dadd_rn(a.f1, d);
        if (mean) {
            const double e = __dsub_rn(d, mu);
            a.f2 = __dadd_rn(a.f2, __dmul_rn(e, e));
        }
    }
    block_reduce(a);
    if (threadIdx.x == 0) {
        a.count = blockIdx.x ? 0 : n;
        store_sums(partials + blockIdx.x, a);
    }
}

__global__ void k_reduce_dot(const int32_t* x, const int32_t* y, int64_t n, HszgSums* partials) {
    Acc a;
    a.init();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        a.s1 += (i128)((int64_t)x[i] * (int64_t)y[i]);
    block_reduce(a);
    if (threadIdx.x == 0) {
        a.count = blockIdx.x ? 0 : n;
        store_sums(partials + blockIdx.x, a);
    }
}

__global__ void k_finalize(const HszgSums* partials, int64_t nparts, HszgSums* out) {
    Acc a;
    a.init();
    // fixed per-thread striding + fixed tree: deterministic float sums too
    for (int64_t i = threadIdx.x; i < nparts; i += blockDim.x) a.merge(load_sums(partials + i));
    block_reduce(a);
    if (threadIdx.x == 0) store_sums(out, a);
}

// ---- regional reductions (N2-N4) --------------------------------------------------

__global__ void k_region_reduce(const int32_t* q, int64_t n0, int64_t n1, int64_t n2, int64_t R0, int64_t R1,
                                int64_t R2, int64_t g1, int64_t g2, int64_t* s1, uint64_t* s2lo, int64_t* s2hi,
                                int32_t* qmin, int32_t* qmax, int64_t* size) {
    const int64_t r = blockIdx.x;
    const int64_t r2 = r % g2;
    const int64_t rr = r / g2;
    const int64_t r1 = rr % g1;
    const int64_t r0 = rr / g1;
    const int64_t z0 = r0 * R0, y0 = r1 * R1, x0 = r2 * R2;
    const int e0 = (int)((z0 + R0 <= n0 ? R0 : n0 - z0));
    const int e1 = (int)((y0 + R1 <= n1 ? R1 : n1 - y0));
    const int e2 = (int)((x0 + R2 <= n2 ? R2 : n2 - x0));
    const int tot = e0 * e1 * e2;
    Acc a;
    a.init();
    for (int i = threadIdx.x; i < tot; i += blockDim.x) {
        const int zy = i / e2;
        const int x = i - zy * e2;
        const int z = zy / e1;
        const int y = zy - z * e1;
        const int32_t v = __ldg(q + ((z0 + z) * n1 + (y0 + y)) * n2 + x0 + x);
        a.s1 += v;
        a.s2 += (i128)((int64_t)v * v);
        a.vmin = min(a.vmin, v);
        a.vmax = max(a.vmax, v);
    }
    block_reduce(a);
    if (threadIdx.x == 0) {
        s1[r] = (int64_t)a.s1;
        s2lo[r] = (uint64_t)a.s2;
        s2hi[r] = (int64_t)(a.s2 >> 64);
        qmin[r] = a.vmin;
        qmax[r] = a.vmax;
        size[r] = tot;
    }
}

// Row-streaming variant for regions R2 = 4..128 wide (a power of two) over 16-B rows: one CTA per
// (region plane, region row) sweeps its R0 x R1 grid rows across the full width with 16-B loads,
// each thread owning four x-points of one region; the R2/4 threads of a region then combine by
// shuffles.  Coalesced and with ~R0*R1 loads in flight per thread (k_region_reduce: one CTA per
// region, scattered 4-byte loads).
constexpr int RR_THREADS = 128;   // 512 x-points per pass (R2 divides 512)

__global__ void __launch_bounds__(RR_THREADS) k_region_rows(const int32_t* __restrict__ q, int64_t n0, int64_t n1,
                                                            int64_t n2, int R0, int R1, int R2, int64_t g1, int64_t g2,
                                                            int64_t* s1o, uint64_t* s2lo, int64_t* s2hi, int32_t* qmin,
                                                            int32_t* qmax, int64_t* size) {
    const int64_t r1 = blockIdx.x, r0 = blockIdx.y;
    const int64_t z0 = r0 * R0, y0 = r1 * R1;
    const int e0 = (int)(z0 + R0 <= n0 ? R0 : n0 - z0);
    const int e1 = (int)(y0 + R1 <= n1 ? R1 : n1 - y0);
    const int rows = e0 * e1;
    const int seg = R2 >> 2;                     // threads per region (power of two <= 32)
    const int lane = threadIdx.x & 31;
    for (int64_t xb = 0; xb < n2; xb += 4 * RR_THREADS) {
        const int64_t x = xb + 4 * (int64_t)threadIdx.x;
        const bool act = x < n2;
        int64_t s1 = 0;
        u128 s2 = 0;
        int mn = INT32_MAX, mx = INT32_MIN;
        if (act) {
#pragma unroll 4
            for (int k = 0; k < rows; k++) {
                const int z = k / e1, y = k - z * e1;
                const int4 v = __ldg(reinterpret_cast<const int4*>(q + ((z0 + z) * n1 + y0 + y) * n2 + x));
                s1 += (int64_t)v.x + v.y + v.z + v.w;
                s2 += (u128)(sq64(v.x) + sq64(v.y));  // each square <= 2^62: pair sums fit 64 bits
                s2 += (u128)(sq64(v.z) + sq64(v.w));
                mn = min(mn, min(min(v.x, v.y), min(v.z, v.w)));
                mx = max(mx, max(max(v.x, v.y), max(v.z, v.w)));
            }
        }
        uint64_t lo = (uint64_t)s2, hi = (uint64_t)(s2 >> 64);
        for (int d = 1; d < seg; d <<= 1) {
            s1 += (int64_t)__shfl_xor_sync(0xffffffffu, (unsigned long long)s1, d);
            const uint64_t olo = __shfl_xor_sync(0xffffffffu, (unsigned long long)lo, d);
            const uint64_t ohi = __shfl_xor_sync(0xffffffffu, (unsigned long long)hi, d);
            const u128 t = (((u128)hi << 64) | lo) + (((u128)ohi << 64) | olo);
            lo = (uint64_t)t;
            hi = (uint64_t)(t >> 64);
            mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, d));
            mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, d));
        }
        if (act && (lane & (seg - 1)) == 0) {
            const int64_t r2 = x / R2;
            const int64_t r = (r0 * g1 + r1) * g2 + r2;
            const int64_t e2 = (r2 + 1) * R2 <= n2 ? R2 : n2 - r2 * R2;
            s1o[r] = s1;
            s2lo[r] = lo;
            s2hi[r] = (int64_t)hi;
            qmin[r] = mn;
            qmax[r] = mx;
            size[r] = (int64_t)rows * e2;
        }
    }
}

__global__ void k_region_finalize(const int64_t* s1, const uint64_t* s2lo, const int64_t* s2hi, const int32_t* qmin,
                                  const int32_t* qmax, const int64_t* size, int64_t nr, double two_eps, double tau,
                                  double* mean, double* var, double* fmin, double* fmax, unsigned long long* count) {
    unsigned long long cnt = 0;
    const double s2e = __dmul_rn(two_eps, two_eps);
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nr; r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t n = size[r];
        mean[r] = __dmul_rn(__ddiv_rn((double)s1[r], (double)n), two_eps);
        if (n < 2) {
            var[r] = __longlong_as_double(0x7ff8000000000000ll);
        } else {
            const i128 S2 = (i128)(((u128)(uint64_t)s2hi[r] << 64) | s2lo[r]);
            const i128 num = (i128)n * S2 - (i128)s1[r] * (i128)s1[r];
            const double numd = (num >= 0 && num < ((i128)1 << 63)) ? (double)(int64_t)num
                              : __dadd_rn(__dmul_rn((double)(int64_t)(num >> 64), 18446744073709551616.0),
                                          __ull2double_rn((uint64_t)num));
            var[r] = __dmul_rn(__ddiv_rn(numd, (double)(n * (n - 1))), s2e);
        }
        const double lo = __dmul_rn((double)qmin[r], two_eps), hi = __dmul_rn((double)qmax[r], two_eps);
        fmin[r] = lo;
        fmax[r] = hi;
        if (lo < tau && tau <= hi) cnt++;
    }
    for (int d = 16; d > 0; d >>= 1) cnt += __shfl_down_sync(0xffffffffu, cnt, d);
    if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(count, cnt);
}

// float64 input sums: f1 = sum(x), f2 = sum((x-mean)^2)
__global__ void k_reduce_flt(const double* x, int64_t n, const double* mean, HszgSums* partials) {
    Acc a;
    a.init();
    const double mu = mean ? *mean : 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double d = __ldg(x + i);
        a.f1 = __dadd_rn(a.f1, d);
        if (mean) {
            const double e = __dsub_rn(d, mu);
            a.f2 = __dadd_rn(a.f2, __dmul_rn(e, e));
        }
    }
    block_reduce(a);
    if (threadIdx.x == 0) {
        a.count = blockIdx.x ? 0 : n;
        store_sums(partials + blockIdx.x, a);
    }
}

// ---- stencils -----------------------------------------------------------------------

struct StencilArgs {
    int op;
    int nd;             // original dimensionality
    int ncomp;
    int float_domain;   // 0: int32 q (stage 2/3), 1: int32 q read as fl(q*2eps) (stage 4), 2: float64 input grids
    int out_type;
    int64_t n[3];       // box dims (leading 1s for 1-D / 2-D)
    const void* q[3];
    double eps[3];
    double two_eps[3];
    void* out[4];
    int64_t zlo;        // first box plane (axis 0) to compute; outputs are indexed from it
    int64_t gz0;        // global axis-0 coordinate of box plane 0 (window / rank offset)
    int64_t gN0;        // global axis-0 extent (boundary layers are global)
};

__device__ __forceinline__ int64_t gext(const StencilArgs& A, int a) { return a == 0 ? A.gN0 : A.n[a]; }

__device__ __forceinline__ void put(const StencilArgs& A, int k, int64_t i, double v) {
    if (A.out_type == HSZG_F32) reinterpret_cast<float*>(A.out[k])[i] = __double2float_rn(v);
    else reinterpret_cast<double*>(A.out[k])[i] = v;
}

__device__ __forceinline__ int32_t qv(const StencilArgs& A, int c, int64_t i) {
    return __ldg(reinterpret_cast<const int32_t*>(A.q[c]) + i);
}
// float-domain value of component c at i: the stage-4 float fl(q*2eps) or a float64 input
__device__ __forceinline__ double fv(const StencilArgs& A, int c, int64_t i) {
    if (A.float_domain == 2) return __ldg(reinterpret_cast<const double*>(A.q[c]) + i);
    return __dmul_rn((double)qv(A, c, i), A.two_eps[c]);
}

// derivative of component c along original axis k at box position (i0,i1,i2), linear i
__device__ __forceinline__ double deriv(const StencilArgs& A, int c, int k, const int64_t* idx, int64_t i,
                                        int64_t* dint) {
    const int a = 3 - A.nd + k;
    const int64_t s = a == 2 ? 1 : (a == 1 ? A.n[2] : A.n[1] * A.n[2]);
    if (idx[a] == 0 || idx[a] == gext(A, a) - 1) {
        if (dint) *dint = 0;
        return 0.0;
    }
    if (A.float_domain) return __ddiv_rn(__dsub_rn(fv(A, c, i + s), fv(A, c, i - s)), 2.0);   // fields.py:85
    const int64_t d = (int64_t)qv(A, c, i + s) - (int64_t)qv(A, c, i - s);                    // fields.py:43
    if (dint) *dint = d;
    return __dmul_rn((double)d, A.eps[c]);                   // fields.py:70
}

__device__ __forceinline__ double laplacian_at(const StencilArgs& A, const int64_t* idx, int64_t i) {
    for (int k = 0; k < A.nd; k++) {
        const int a = 3 - A.nd + k;
        if (!(idx[a] > 0 && idx[a] < gext(A, a) - 1)) return 0.0;
    }
    if (A.float_domain) {
        // fields.py:47-60 on float64 values: acc = (-2*nd)*v; acc = acc + lo + hi per axis
        double acc = __dmul_rn((double)(-2 * A.nd), fv(A, 0, i));
        for (int k = 0; k < A.nd; k++) {
            const int a = 3 - A.nd + k;
            const int64_t st = a == 2 ? 1 : (a == 1 ? A.n[2] : A.n[1] * A.n[2]);
            acc = __dadd_rn(acc, fv(A, 0, i - st));
            acc = __dadd_rn(acc, fv(A, 0, i + st));
        }
        return acc;
    }
    int64_t acc = -2 * (int64_t)A.nd * qv(A, 0, i);
    for (int k = 0; k < A.nd; k++) {
        const int a = 3 - A.nd + k;
        const int64_t st = a == 2 ? 1 : (a == 1 ? A.n[2] : A.n[1] * A.n[2]);
        acc += (int64_t)qv(A, 0, i - st) + (int64_t)qv(A, 0, i + st);
    }
    return __dmul_rn((double)acc, A.two_eps[0]);   // fields.py:79
}

__global__ void k_stencil(StencilArgs A) {
    const int64_t i2 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i2 >= A.n[2]) return;
    const int64_t i1 = blockIdx.y;
    const int64_t i0 = A.zlo + blockIdx.z;
    const int64_t idx[3] = {A.gz0 + i0, i1, i2};          // global coordinates (boundary tests)
    const int64_t i = (i0 * A.n[1] + i1) * A.n[2] + i2;   // input index
    const int64_t oi = ((i0 - A.zlo) * A.n[1] + i1) * A.n[2] + i2;   // output index
    switch (A.op) {
        case HSZG_OP_DERIV:
            for (int k = 0; k < A.nd; k++) put(A, k, oi, deriv(A, 0, k, idx, i, nullptr));
            break;
        case HSZG_OP_LAPLACIAN:
            put(A, 0, oi, laplacian_at(A, idx, i));
            break;
        case HSZG_OP_GRAD_LAP:
            for (int k = 0; k < A.nd; k++) put(A, k, oi, deriv(A, 0, k, idx, i, nullptr));
            put(A, A.nd, oi, laplacian_at(A, idx, i));
            break;
        case HSZG_OP_GRADMAG: {
            if (A.float_domain) {
                double s = 0.0;
                for (int k = 0; k < A.nd; k++) {
                    const double d = deriv(A, 0, k, idx, i, nullptr);
                    s = __dadd_rn(s, __dmul_rn(d, d));
                }
                put(A, 0, oi, __dsqrt_rn(s));
            } else {
                u128 s = 0;
                for (int k = 0; k < A.nd; k++) {
                    int64_t d;
                    deriv(A, 0, k, idx, i, &d);
                    const uint64_t ad = (uint64_t)(d < 0 ? -d : d);
                    s += (u128)ad * ad;
                }
                double sd;
                if ((uint64_t)(s >> 64) == 0) sd = __ull2double_rn((uint64_t)s);
                else sd = __dadd_rn(__dmul_rn(__ull2double_rn((uint64_t)(s >> 64)), 18446744073709551616.0),
                                    __ull2double_rn((uint64_t)s));
                put(A, 0, oi, __dmul_rn(__dsqrt_rn(sd), A.eps[0]));
            }
            break;
        }
        case HSZG_OP_DIVERGENCE: {
            double acc = deriv(A, 0, 0, idx, i, nullptr);        // fields.py:219-221
            for (int k = 1; k < A.ncomp; k++) acc = __dadd_rn(acc, deriv(A, k, k, idx, i, nullptr));
            put(A, 0, oi, acc);
            break;
        }
        case HSZG_OP_CURL: {
            if (A.ncomp == 2) {                                     // fields.py:228-231
                put(A, 0, oi, __dsub_rn(deriv(A, 0, 1, idx, i, nullptr), deriv(A, 1, 0, idx, i, nullptr)));
            } else {                                                // fields.py:232-236
                put(A, 0, oi, __dsub_rn(deriv(A, 2, 1, idx, i, nullptr), deriv(A, 1, 2, idx, i, nullptr)));
                put(A, 1, oi, __dsub_rn(deriv(A, 0, 2, idx, i, nullptr), deriv(A, 2, 0, idx, i, nullptr)));
                put(A, 2, oi, __dsub_rn(deriv(A, 1, 0, idx, i, nullptr), deriv(A, 0, 1, idx, i, nullptr)));
            }
            break;
        }
        default:
            break;
    }
}

}  // namespace hszg

using namespace hszg;

int hszg_set_cuda_error(HszgErr* err, cudaError_t e, const char* where);
int hszg_launch_decode(const HszgGeom* g, const HszgStream* s, int32_t* out, cudaStream_t st, HszgErr* err);

static inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

static const int kMaxParts = 148 * 16;

size_t hszg_reduce_ws_bytes(int64_t tiles) {
    const int64_t parts = tiles > kMaxParts ? tiles : kMaxParts;
    return (size_t)(parts + 1) * sizeof(HszgSums) + 256;
}

static int finalize(HszgSums* partials, int64_t nparts, HszgSums* out, cudaStream_t st) {
    k_finalize<<<1, 1024, 0, st>>>(partials, nparts, out);
    return cudaGetLastError() == cudaSuccess ? HSZG_OK : HSZG_CUDA;
}

int hszg_finalize_sums(HszgSums* partials, int64_t nparts, HszgSums* out, cudaStream_t st) {
    return finalize(partials, nparts, out, st);
}

extern "C" int hszg_reduce_stream(const HszgGeom* g, const HszgStream* s, int mode, HszgSums* out_dev, void* ws,
                                  size_t ws_bytes, void* stream, HszgErr* err) {
    err->status = HSZG_OK;
    cudaStream_t st = as_stream(stream);
    const SegGeo sg = make_seggeo(*g);
    HszgSums* partials = reinterpret_cast<HszgSums*>(ws);
    const bool no_extrema = (mode & HSZG_REDUCE_NO_EXTREMA) != 0;   // vmin / vmax not wanted (statistics)
    mode &= ~HSZG_REDUCE_NO_EXTREMA;
    if (mode == 4) {
        if (!s->metadata) {
            err->status = HSZG_INVALID_ARG;
            snprintf(err->message, sizeof(err->message), "stream has no block-mean metadata");
            return HSZG_INVALID_ARG;
        }
        const int64_t nb = sg.G[0] * sg.G[1] * sg.G[2];
        const int grid = grid_for(nb, RED_THREADS, kMaxParts);
        k_reduce_meta<<<grid, RED_THREADS, 0, st>>>(sg, s->metadata, partials);
        return finalize(partials, grid, out_dev, st);
    }
    if (mode < 1 || mode > 3) {
        err->status = HSZG_INVALID_ARG;
        snprintf(err->message, sizeof(err->message), "unknown reduction mode %d", mode);
        return HSZG_INVALID_ARG;
    }
    const int64_t tiles = (g->n_chunks + TILE_CHUNKS - 1) / TILE_CHUNKS;
    if (g->n_chunks == 0) {
        HszgSums z = {};
        cudaMemcpyAsync(out_dev, &z, sizeof(z), cudaMemcpyHostToDevice, st);
        return HSZG_OK;
    }
    if (s->canonical) {
        if (ws_bytes < hszg_reduce_ws_bytes(tiles)) {
            err->status = HSZG_INVALID_ARG;
            snprintf(err->message, sizeof(err->message), "workspace too small for reduction");
            return HSZG_INVALID_ARG;
        }
        const size_t smem = tile_smem_bytes(s->max_bitwidth);
        bool full_segs = g->n_chunks * kChunkCap == g->n && (sg.B[0] * sg.B[1] * sg.B[2]) % kChunkCap == 0;
        for (int a = 0; a < 3; a++) full_segs = full_segs && sg.E[a] == sg.B[a];
        if (mode != 3 && g->n_chunks * kChunkCap == g->n && sg.n[2] % kChunkCap == 0) {
            size_t sm;
            uint32_t bb;
            const unsigned grid = wtile_grid(k_reduce_weighted_fast, s->max_bitwidth, g->n_chunks, &sm, &bb);
            k_reduce_weighted_fast<<<grid, 256, sm, st>>>(s->payload, s->payload_len, s->offsets, g->n_chunks,
                                                         sg.n[0], sg.n[1], sg.n[2], g->n, partials, bb);
            { const cudaError_t e_ = cudaGetLastError(); if (e_ != cudaSuccess) return hszg_set_cuda_error(err, e_, "reduce tiles"); }
            return finalize(partials, grid, out_dev, st);
        }
        if (mode == 3 && full_segs) {
            const int64_t cps = (sg.B[0] * sg.B[1] * sg.B[2]) / kChunkCap;
            MetaAux aux{s->metadata, cps, -1};
            for (int k = 0; k < 40; k++)
                if (cps == (int64_t)1 << k) aux.shift = k;
            size_t sm;
            uint32_t bb;
            unsigned grid;
            if (no_extrema) {
                grid = wtile_grid(k_reduce_meta_fast<false>, s->max_bitwidth, g->n_chunks, &sm, &bb);
                k_reduce_meta_fast<false><<<grid, 256, sm, st>>>(s->payload, s->payload_len, s->offsets,
                                                                g->n_chunks, aux, g->n, partials, bb);
            } else {
                grid = wtile_grid(k_reduce_meta_fast<true>, s->max_bitwidth, g->n_chunks, &sm, &bb);
                k_reduce_meta_fast<true><<<grid, 256, sm, st>>>(s->payload, s->payload_len, s->offsets,
                                                               g->n_chunks, aux, g->n, partials, bb);
            }
            { const cudaError_t e_ = cudaGetLastError(); if (e_ != cudaSuccess) return hszg_set_cuda_error(err, e_, "reduce tiles"); }
            return finalize(partials, grid, out_dev, st);
        }
        if (mode == 3)
            allow_smem(k_reduce_tiles<MetaChunk>, smem),
            k_reduce_tiles<MetaChunk><<<(unsigned)tiles, TILE_CHUNKS, smem, st>>>(sg, s->payload, s->payload_len,
                                                                                s->offsets, s->metadata, partials);
        else
            allow_smem(k_reduce_tiles<WeightedChunk>, smem),
            k_reduce_tiles<WeightedChunk><<<(unsigned)tiles, TILE_CHUNKS, smem, st>>>(
                sg, s->payload, s->payload_len, s->offsets, s->metadata, partials);
        { const cudaError_t e_ = cudaGetLastError(); if (e_ != cudaSuccess) return hszg_set_cuda_error(err, e_, "reduce tiles"); }
        return finalize(partials, tiles, out_dev, st);
    }
    // non-canonical: decode into the workspace tail, then reduce per chunk
    const size_t head = hszg_reduce_ws_bytes(kMaxParts);
    if (ws_bytes < head + (size_t)g->n * 4) {
        err->status = HSZG_INVALID_ARG;
        snprintf(err->message, sizeof(err->message), "workspace too small for reduction");
        return HSZG_INVALID_ARG;
    }
    int32_t* p = reinterpret_cast<int32_t*>(reinterpret_cast<char*>(ws) + head);
    int r = hszg_launch_decode(g, s, p, st, err);
    if (r) return r;
    const int grid = grid_for(g->n_chunks, RED_THREADS, kMaxParts);
    if (mode == 3) k_reduce_chunks_array<MetaChunk><<<grid, RED_THREADS, 0, st>>>(sg, p, s->metadata, partials);
    else k_reduce_chunks_array<WeightedChunk><<<grid, RED_THREADS, 0, st>>>(sg, p, s->metadata, partials);
    return finalize(partials, grid, out_dev, st);
}

extern "C" int hszg_reduce_array(const HszgGeom* g, const int32_t* p, const int32_t* metadata, int mode,
                                 HszgSums* out_dev, void* ws, size_t ws_bytes, void* stream) {
    cudaStream_t st = as_stream(stream);
    const SegGeo sg = make_seggeo(*g);
    if (ws_bytes < hszg_reduce_ws_bytes(0)) return HSZG_INVALID_ARG;
    HszgSums* partials = reinterpret_cast<HszgSums*>(ws);
    const int grid = grid_for(g->n_chunks, RED_THREADS, kMaxParts);
    if (mode == 3) k_reduce_chunks_array<MetaChunk><<<grid, RED_THREADS, 0, st>>>(sg, p, metadata, partials);
    else if (mode == 1 || mode == 2)
        k_reduce_chunks_array<WeightedChunk><<<grid, RED_THREADS, 0, st>>>(sg, p, metadata, partials);
    else return HSZG_INVALID_ARG;
    return finalize(partials, grid, out_dev, st);
}

extern "C" int hszg_reduce_i32(const int32_t* src, int64_t n, HszgSums* out_dev, void* ws, size_t ws_bytes,
                               void* stream) {
    cudaStream_t st = as_stream(stream);
    if (ws_bytes < hszg_reduce_ws_bytes(0)) return HSZG_INVALID_ARG;
    HszgSums* partials = reinterpret_cast<HszgSums*>(ws);
    const int grid = grid_for(n / 4 + 1, RED_THREADS * 8, kMaxParts);
    k_reduce_i32<<<grid, RED_THREADS, 0, st>>>(src, n, partials);
    return finalize(partials, grid, out_dev, st);
}

extern "C" int hszg_reduce_f64(const int32_t* q, int64_t n, double scale, const double* mean_dev, HszgSums* out_dev,
                               void* ws, size_t ws_bytes, void* stream) {
    cudaStream_t st = as_stream(stream);
    if (ws_bytes < hszg_reduce_ws_bytes(0)) return HSZG_INVALID_ARG;
    HszgSums* partials = reinterpret_cast<HszgSums*>(ws);
    const int grid = grid_for(n, RED_THREADS * 8, kMaxParts);
    k_reduce_f64<<<grid, RED_THREADS, 0, st>>>(q, n, scale, mean_dev, partials);
    return finalize(partials, grid, out_dev, st);
}

extern "C" int hszg_reduce_dot(const int32_t* a, const int32_t* b, int64_t n, HszgSums* out_dev, void* ws,
                               size_t ws_bytes, void* stream) {
    cudaStream_t st = as_stream(stream);
    if (ws_bytes < hszg_reduce_ws_bytes(0)) return HSZG_INVALID_ARG;
    HszgSums* partials = reinterpret_cast<HszgSums*>(ws);
    const int grid = grid_for(n, RED_THREADS * 8, kMaxParts);
    k_reduce_dot<<<grid, RED_THREADS, 0, st>>>(a, b, n, partials);
    return finalize(partials, grid, out_dev, st);
}

static void box3(int32_t ndims, const int64_t* dims, int64_t* n) {
    n[0] = n[1] = n[2] = 1;
    for (int k = 0; k < ndims; k++) n[3 - ndims + k] = dims[k];
}

extern "C" int hszg_region_reduce(const int32_t* q, int32_t ndims, const int64_t* dims, const int64_t* region,
                                  int64_t* s1, uint64_t* s2_lo, int64_t* s2_hi, int32_t* qmin, int32_t* qmax,
                                  int64_t* size, void* stream) {
    if (ndims < 1 || ndims > 3) return HSZG_INVALID_ARG;
    int64_t n[3], R[3] = {1, 1, 1};
    box3(ndims, dims, n);
    for (int k = 0; k < ndims; k++) {
        const int64_t r = region[k] < dims[k] ? region[k] : dims[k];
        if (r < 1) return HSZG_INVALID_ARG;
        R[3 - ndims + k] = r;
    }
    const int64_t g0 = (n[0] + R[0] - 1) / R[0], g1 = (n[1] + R[1] - 1) / R[1], g2 = (n[2] + R[2] - 1) / R[2];
    const int64_t nr = g0 * g1 * g2;
    if (nr == 0) return HSZG_OK;
    const int64_t seg = R[2] / 4;
    static const char* rm = getenv("HSZG_REGION");           // 'b': one-CTA-per-region kernel (A/B runs)
    if (R[2] % 4 == 0 && seg <= 32 && (seg & (seg - 1)) == 0 && n[2] % 4 == 0 &&
        (reinterpret_cast<uintptr_t>(q) & 15) == 0 && g0 <= 65535 && g1 < INT32_MAX && R[0] * R[1] < INT32_MAX &&
        !(rm && rm[0] == 'b')) {
        k_region_rows<<<dim3((unsigned)g1, (unsigned)g0), RR_THREADS, 0, as_stream(stream)>>>(
            q, n[0], n[1], n[2], (int)R[0], (int)R[1], (int)R[2], g1, g2, s1, s2_lo, s2_hi, qmin, qmax, size);
        return cudaGetLastError() == cudaSuccess ? HSZG_OK : HSZG_CUDA;
    }
    const int64_t rs = R[0] * R[1] * R[2];
    const int threads = rs >= 1024 ? 256 : (rs >= 256 ? 128 : 64);
    k_region_reduce<<<(unsigned)nr, threads, 0, as_stream(stream)>>>(q, n[0], n[1], n[2], R[0], R[1], R[2], g1, g2,
                                                                     s1, s2_lo, s2_hi, qmin, qmax, size);
    return cudaGetLastError() == cudaSuccess ? HSZG_OK : HSZG_CUDA;
}

// Region reduction straight from an HSZX* stream (stage 2 / 3 integers q = p + M_b): see k_region_fused.
// region[] in the ORIGINAL dims (clipped to them); every extent must be a multiple of the block extent
// (or reach the grid end) and every chunk must be full.  Returns HSZG_UNSUPPORTED_STAGE when not
// applicable (the caller reconstructs q and runs hszg_region_reduce).  ws: >= nr * 64 bytes.
extern "C" int hszg_region_stream(const HszgGeom* g, const HszgStream* s, const int64_t* region, int64_t* s1,
                                  uint64_t* s2_lo, int64_t* s2_hi, int32_t* qmin, int32_t* qmax, int64_t* size,
                                  void* ws, size_t ws_bytes, void* stream, HszgErr* err) {
    err->status = HSZG_OK;
    cudaStream_t st = as_stream(stream);
    if ((g->kind != 2 && g->kind != 3) || !s->canonical || !s->metadata || g->n_chunks * kChunkCap != g->n)
        return HSZG_UNSUPPORTED_STAGE;
    const SegGeo sg = make_seggeo(*g);
    // regions in box coordinates (the box is the original dims, leading 1s for 2-D / 1-D)
    const int nd = g->ndims;
    int64_t R[3] = {1, 1, 1};
    for (int k = 0; k < nd; k++) {
        const int64_t r = region[k] < g->dims[k] ? region[k] : g->dims[k];
        if (r < 1) return HSZG_INVALID_ARG;
        R[3 - nd + k] = r;
    }
    if (g->kind == 2 && !(sg.n[0] == 1 && sg.n[1] == 1 && R[0] == 1 && R[1] == 1)) {
        // HSZX: 1-D blocks of the flat stream; regions must be 1-D too
        return HSZG_UNSUPPORTED_STAGE;
    }
    RegionMap rm;
    for (int a = 0; a < 3; a++) {
        rm.rg[a] = (sg.n[a] + R[a] - 1) / R[a];
        if (R[a] % sg.B[a] != 0 && R[a] < sg.n[a]) return HSZG_UNSUPPORTED_STAGE;
        rm.bpr[a] = R[a] >= sg.n[a] ? sg.G[a] : R[a] / sg.B[a];
    }
    const int64_t nr = rm.rg[0] * rm.rg[1] * rm.rg[2];
    if (ws_bytes < (size_t)nr * sizeof(RegAccum)) return HSZG_INVALID_ARG;
    RegAccum* acc = reinterpret_cast<RegAccum*>(ws);
    bool full_segs = (sg.B[0] * sg.B[1] * sg.B[2]) % kChunkCap == 0;
    for (int a = 0; a < 3; a++) full_segs = full_segs && sg.E[a] == sg.B[a];
    const int64_t cps = (sg.B[0] * sg.B[1] * sg.B[2]) / kChunkCap;
    if (full_segs && rm.bpr[0] == 1 && rm.bpr[1] == 1 && rm.bpr[2] == 1 && cps >= 1 && cps <= 32 &&
        (cps & (cps - 1)) == 0 && nr == g->n_chunks / cps) {
        // region = block: the one-writer kernel (no accumulator)
        size_t sm;
        uint32_t bb;
        const int64_t bs = sg.B[0] * sg.B[1] * sg.B[2];
#define HSZG_RB(C)                                                                                              \
        do {                                                                                                    \
            const unsigned grid = wtile_grid(k_region_blocks<C>, s->max_bitwidth, g->n_chunks, &sm, &bb);      \
            k_region_blocks<C><<<grid, 256, sm, st>>>(s->payload, s->payload_len, s->offsets, g->n_chunks,      \
                                                      s->metadata, bs, s1, s2_lo, s2_hi, qmin, qmax, size, bb); \
        } while (0)
        switch (cps) {
            case 1: HSZG_RB(1); break;
            case 2: HSZG_RB(2); break;
            case 4: HSZG_RB(4); break;
            case 8: HSZG_RB(8); break;
            case 16: HSZG_RB(16); break;
            default: HSZG_RB(32); break;
        }
#undef HSZG_RB
        { const cudaError_t e_ = cudaGetLastError(); if (e_ != cudaSuccess) return hszg_set_cuda_error(err, e_, "region blocks"); }
        return HSZG_OK;
    }
    k_region_accum_init<<<grid_for(nr, 256, 148 * 8), 256, 0, st>>>(acc, nr);
    size_t sm;
    uint32_t bb;
    const unsigned grid = wtile_grid(k_region_fused, s->max_bitwidth, g->n_chunks, &sm, &bb);
    k_region_fused<<<grid, 256, sm, st>>>(sg, rm, s->payload, s->payload_len, s->offsets, s->metadata, full_segs, cps,
                                          acc, bb);
    { const cudaError_t e_ = cudaGetLastError(); if (e_ != cudaSuccess) return hszg_set_cuda_error(err, e_, "region fused"); }
    k_region_accum_finish<<<grid_for(nr, 256, 148 * 8), 256, 0, st>>>(acc, sg.n[0], sg.n[1], sg.n[2], R[0], R[1], R[2],
                                                                     rm.rg[1], rm.rg[2], nr, s1, s2_lo, s2_hi, qmin,
                                                                     qmax, size);
    return cudaGetLastError() == cudaSuccess ? HSZG_OK : HSZG_CUDA;
}

static int stencil_impl(int op, int32_t ndims, const int64_t* dims, int32_t ncomp, const void* const* q,
                        const double* eps, int float_domain, int32_t out_type, void* const* out, int64_t zlo,
                        int64_t zhi, int64_t gz0, int64_t gN0, cudaStream_t st);

extern "C" int hszg_stencil(int op, int32_t ndims, const int64_t* dims, int32_t ncomp, const void* const* q,
                            const double* eps, int float_domain, int32_t out_type, void* const* out, void* stream) {
    const int64_t n0 = ndims == 3 ? dims[0] : 1;
    return stencil_impl(op, ndims, dims, ncomp, q, eps, float_domain, out_type, out, 0, n0, 0, n0,
                        as_stream(stream));
}

extern "C" int hszg_stencil_window(int op, const int64_t* dims, int32_t ncomp, const void* const* q, const double* eps,
                                   int float_domain, int32_t out_type, void* const* out, int64_t zlo, int64_t zhi,
                                   int64_t gz0, int64_t gN0, void* stream) {
    return stencil_impl(op, 3, dims, ncomp, q, eps, float_domain, out_type, out, zlo, zhi, gz0, gN0,
                        as_stream(stream));
}

// ---- the hot stencil: 3-D gradient (3 comps) + Laplacian of int32 q into fp32 grids -------------
// Four x-consecutive points per thread: one 16-B load per neighbour row (x+-1 from the adjacent
// lanes by shuffle), fp64 scaling exactly as fields.py:70/79 (one rounding) then one cast to fp32,
// and 16-B streaming stores (evict-first: the q window stays in L2 for its z/y neighbours).
namespace hszg {

__device__ __forceinline__ float4 scale4(int64_t a, int64_t b, int64_t c, int64_t d, double s) {
    return make_float4(__double2float_rn(__dmul_rn((double)a, s)), __double2float_rn(__dmul_rn((double)b, s)),
                       __double2float_rn(__dmul_rn((double)c, s)), __double2float_rn(__dmul_rn((double)d, s)));
}

constexpr int GL_THREADS = 128;   // 512 x-points per CTA row

__global__ void __launch_bounds__(GL_THREADS) k_grad_lap_f32(const int32_t* __restrict__ q, int64_t n1, int64_t n2,
                                                             int64_t zlo, int64_t gz0, int64_t gN0, double eps,
                                                             double two_eps, float* __restrict__ o0,
                                                             float* __restrict__ o1, float* __restrict__ o2,
                                                             float* __restrict__ o3) {
    const int lane = threadIdx.x & 31;
    const int64_t x = ((int64_t)blockIdx.x * GL_THREADS + threadIdx.x) * 4;
    const int64_t y = blockIdx.y;
    const int64_t z = zlo + blockIdx.z;               // box plane
    const int64_t gz = gz0 + z;                       // global plane
    const int64_t plane = n1 * n2;
    const bool active = x < n2;
    const int64_t xi = active ? x : 0;
    const int32_t* row = q + z * plane + y * n2;
    int4 c = make_int4(0, 0, 0, 0);
    if (active) c = __ldg(reinterpret_cast<const int4*>(row + xi));
    // x neighbours: previous lane's .w, next lane's .x; warp edges load their own
    int left = __shfl_up_sync(0xffffffffu, c.w, 1);
    int right = __shfl_down_sync(0xffffffffu, c.x, 1);
    if (active && lane == 0 && xi > 0) left = __ldg(row + xi - 1);
    if (active && lane == 31 && xi + 4 < n2) right = __ldg(row + xi + 4);
    if (!active) return;
    const bool zin = gz > 0 && gz < gN0 - 1;
    const bool yin = y > 0 && y < n1 - 1;
    int4 zm = make_int4(0, 0, 0, 0), zp = zm, ym = zm, yp = zm;
    if (zin) {
        zm = __ldg(reinterpret_cast<const int4*>(row - plane + xi));
        zp = __ldg(reinterpret_cast<const int4*>(row + plane + xi));
    }
    if (yin) {
        ym = __ldg(reinterpret_cast<const int4*>(row - n2 + xi));
        yp = __ldg(reinterpret_cast<const int4*>(row + n2 + xi));
    }
    const int64_t o = (z - zlo) * plane + y * n2 + xi;
    // d/dz (axis 0), d/dy (axis 1): zero on their boundary layers (fields.py:34-44)
    float4 dz = make_float4(0.f, 0.f, 0.f, 0.f), dy = dz, dx, lp = dz;
    if (zin) dz = scale4((int64_t)zp.x - zm.x, (int64_t)zp.y - zm.y, (int64_t)zp.z - zm.z, (int64_t)zp.w - zm.w, eps);
    if (yin) dy = scale4((int64_t)yp.x - ym.x, (int64_t)yp.y - ym.y, (int64_t)yp.z - ym.z, (int64_t)yp.w - ym.w, eps);
    // d/dx (axis 2): zero at x = 0 and x = n2-1
    int64_t d0 = (int64_t)c.y - left, d1 = (int64_t)c.z - c.x, d2 = (int64_t)c.w - c.y, d3 = (int64_t)right - c.z;
    if (xi == 0) d0 = 0;
    if (xi + 3 >= n2 - 1) d3 = 0;
    dx = scale4(d0, d1, d2, d3, eps);
    if (zin && yin) {   // Laplacian: zero on every boundary layer (fields.py:47-60)
        int64_t l0 = (int64_t)zm.x + zp.x + ym.x + yp.x + left + c.y - 6ll * c.x;
        int64_t l1 = (int64_t)zm.y + zp.y + ym.y + yp.y + c.x + c.z - 6ll * c.y;
        int64_t l2 = (int64_t)zm.z + zp.z + ym.z + yp.z + c.y + c.w - 6ll * c.z;
        int64_t l3 = (int64_t)zm.w + zp.w + ym.w + yp.w + c.z + right - 6ll * c.w;
        if (xi == 0) l0 = 0;
        if (xi + 3 >= n2 - 1) l3 = 0;
        lp = scale4(l0, l1, l2, l3, two_eps);
    }
    __stcs(reinterpret_cast<float4*>(o0 + o), dz);
    __stcs(reinterpret_cast<float4*>(o1 + o), dy);
    __stcs(reinterpret_cast<float4*>(o2 + o), dx);
    __stcs(reinterpret_cast<float4*>(o3 + o), lp);
}

// ---- vectorised K-STEN: every op of k_stencil on 2-D / 3-D int32 grids, four x-points per thread ----
// Same per-point arithmetic as deriv / laplacian_at / k_stencil (so bit-identical results), but
// 16-B neighbour-row loads (x+-1 by shuffle), no per-point index math and 16/32-B streaming stores.
constexpr int SV_THREADS = 128;
constexpr int SV_ZC = 8;          // planes per CTA of the 3-D z-sliding stencil

struct Nb4 {            // one component around four x-points: centre, z+-1, y+-1 rows and the x edges
    int4 c, zm, zp, ym, yp;
    int l, r;
};

__device__ __forceinline__ Nb4 nb4_load(const int32_t* q, int64_t plane, int64_t n2, int64_t off, bool active,
                                        bool zin, bool yin, int lane, int64_t xi) {
    Nb4 b;
    const int4 z4 = make_int4(0, 0, 0, 0);
    b.c = b.zm = b.zp = b.ym = b.yp = z4;
    if (active) b.c = __ldg(reinterpret_cast<const int4*>(q + off));
    b.l = __shfl_up_sync(0xffffffffu, b.c.w, 1);     // every lane takes part in the shuffles
    b.r = __shfl_down_sync(0xffffffffu, b.c.x, 1);
    if (!active) return b;
    if (lane == 0 && xi > 0) b.l = __ldg(q + off - 1);
    if (lane == 31 && xi + 4 < n2) b.r = __ldg(q + off + 4);
    if (zin) {
        b.zm = __ldg(reinterpret_cast<const int4*>(q + off - plane));
        b.zp = __ldg(reinterpret_cast<const int4*>(q + off + plane));
    }
    if (yin) {
        b.ym = __ldg(reinterpret_cast<const int4*>(q + off - n2));
        b.yp = __ldg(reinterpret_cast<const int4*>(q + off + n2));
    }
    return b;
}

__device__ __forceinline__ int el(const int4& v, int j) { return j == 0 ? v.x : (j == 1 ? v.y : (j == 2 ? v.z : v.w)); }
// x-neighbours of point j: (x-1, x+1)
__device__ __forceinline__ int xm1(const Nb4& b, int j) { return j == 0 ? b.l : el(b.c, j - 1); }
__device__ __forceinline__ int xp1(const Nb4& b, int j) { return j == 3 ? b.r : el(b.c, j + 1); }

struct Pt4 {            // per-thread geometry shared by every component
    bool zin, yin, x0, xl;   // interior along z / y; point 0 at x = 0; point 3 at x = n2-1
};

// derivative of one component along BOX axis a at point j (deriv(): fields.py:43/70, stage 4: :85)
__device__ __forceinline__ double dv4(const Nb4& b, const Pt4& p, int a, int j, double eps, double two_eps, bool fd) {
    int m, h;
    if (a == 0) {
        if (!p.zin) return 0.0;
        m = el(b.zm, j), h = el(b.zp, j);
    } else if (a == 1) {
        if (!p.yin) return 0.0;
        m = el(b.ym, j), h = el(b.yp, j);
    } else {
        if ((j == 0 && p.x0) || (j == 3 && p.xl)) return 0.0;
        m = xm1(b, j), h = xp1(b, j);
    }
    if (fd) return __ddiv_rn(__dsub_rn(__dmul_rn((double)h, two_eps), __dmul_rn((double)m, two_eps)), 2.0);
    return __dmul_rn((double)((int64_t)h - (int64_t)m), eps);
}
// integer derivative (GRADMAG)
__device__ __forceinline__ int64_t di4(const Nb4& b, const Pt4& p, int a, int j) {
    if (a == 0) return p.zin ? (int64_t)el(b.zp, j) - el(b.zm, j) : 0;
    if (a == 1) return p.yin ? (int64_t)el(b.yp, j) - el(b.ym, j) : 0;
    if ((j == 0 && p.x0) || (j == 3 && p.xl)) return 0;
    return (int64_t)xp1(b, j) - xm1(b, j);
}
template <int ND>
__device__ __forceinline__ double lap4(const Nb4& b, const Pt4& p, int j, double two_eps, bool fd) {
    if ((ND == 3 && !p.zin) || !p.yin || (j == 0 && p.x0) || (j == 3 && p.xl)) return 0.0;
    if (fd) {   // fields.py:47-60 in float64, axis order z (3-D), y, x
        double acc = __dmul_rn((double)(-2 * ND), __dmul_rn((double)el(b.c, j), two_eps));
        if (ND == 3) {
            acc = __dadd_rn(acc, __dmul_rn((double)el(b.zm, j), two_eps));
            acc = __dadd_rn(acc, __dmul_rn((double)el(b.zp, j), two_eps));
        }
        acc = __dadd_rn(acc, __dmul_rn((double)el(b.ym, j), two_eps));
        acc = __dadd_rn(acc, __dmul_rn((double)el(b.yp, j), two_eps));
        acc = __dadd_rn(acc, __dmul_rn((double)xm1(b, j), two_eps));
        acc = __dadd_rn(acc, __dmul_rn((double)xp1(b, j), two_eps));
        return acc;
    }
    int64_t acc = -2 * (int64_t)ND * el(b.c, j) + (int64_t)el(b.ym, j) + el(b.yp, j) + xm1(b, j) + xp1(b, j);
    if (ND == 3) acc += (int64_t)el(b.zm, j) + el(b.zp, j);
    return __dmul_rn((double)acc, two_eps);
}

__device__ __forceinline__ void st4(float* o, int64_t i, const double* v) {
    __stcs(reinterpret_cast<float4*>(o + i), make_float4(__double2float_rn(v[0]), __double2float_rn(v[1]),
                                                         __double2float_rn(v[2]), __double2float_rn(v[3])));
}
__device__ __forceinline__ void st4(double* o, int64_t i, const double* v) {
    __stcs(reinterpret_cast<double2*>(o + i), make_double2(v[0], v[1]));
    __stcs(reinterpret_cast<double2*>(o + i + 2), make_double2(v[2], v[3]));
}

// FD: float-domain input (stage 4: q read as fl(q * 2eps)) — a template parameter so the integer
// (stage 2/3) kernels carry no float-domain code (they were issue-bound on it: 81% issue slots)
template <int OP, int ND, typename OutT, bool FD>
__global__ void __launch_bounds__(SV_THREADS) k_stencil_v4(StencilArgs A, int zc, int64_t zend) {
    const int lane = threadIdx.x & 31;
    const int64_t xi0 = ((int64_t)blockIdx.x * SV_THREADS + threadIdx.x) * 4;
    const bool active = xi0 < A.n[2];
    const int64_t xi = active ? xi0 : 0;
    const int64_t y = blockIdx.y;
    const int64_t n1 = A.n[1], n2 = A.n[2], plane = n1 * n2, nbox = A.n[0];
    const int64_t zs = A.zlo + (int64_t)blockIdx.z * zc;
    const int64_t ze = zs + zc < zend ? zs + zc : zend;
    Pt4 p;
    p.yin = y > 0 && y < n1 - 1;
    p.x0 = xi == 0;
    p.xl = xi + 3 >= n2 - 1;
    constexpr bool fd = FD;
    constexpr int a0 = 3 - ND;                        // box axis of original axis 0
    constexpr int NC = (OP == HSZG_OP_DIVERGENCE || OP == HSZG_OP_CURL) ? ND : 1;
    const int4 z4 = make_int4(0, 0, 0, 0);
    // the thread slides along z through zc planes: rows z-1, z, z+1 stay in registers; the loads of
    // the next plane (its y+-1 rows and x edges, and row z+2) are issued before plane z is computed
    int4 cm[NC], cc[NC], cp[NC], ymn[NC], ypn[NC];
    int eln[NC], ern[NC];
    auto load_nb = [&](int c, int64_t zz, int4& ym, int4& yp, int& el, int& er) {
        const int32_t* row = reinterpret_cast<const int32_t*>(A.q[c]) + zz * plane + y * n2 + xi;
        ym = active && p.yin ? __ldg(reinterpret_cast<const int4*>(row - n2)) : z4;
        yp = active && p.yin ? __ldg(reinterpret_cast<const int4*>(row + n2)) : z4;
        el = lane == 0 && active && xi > 0 ? __ldg(row - 1) : 0;
        er = lane == 31 && active && xi + 4 < n2 ? __ldg(row + 4) : 0;
    };
#pragma unroll
    for (int c = 0; c < NC; c++) {
        const int32_t* col = reinterpret_cast<const int32_t*>(A.q[c]) + y * n2 + xi;
        cc[c] = active ? __ldg(reinterpret_cast<const int4*>(col + zs * plane)) : z4;
        cm[c] = active && zs > 0 ? __ldg(reinterpret_cast<const int4*>(col + (zs - 1) * plane)) : z4;
        cp[c] = active && zs + 1 < nbox ? __ldg(reinterpret_cast<const int4*>(col + (zs + 1) * plane)) : z4;
        load_nb(c, zs, ymn[c], ypn[c], eln[c], ern[c]);
    }
    for (int64_t z = zs; z < ze; z++) {
    p.zin = ND == 3 && A.gz0 + z > 0 && A.gz0 + z < A.gN0 - 1;
    Nb4 b[NC];
    int4 nx[NC];
#pragma unroll
    for (int c = 0; c < NC; c++) {
        b[c].c = cc[c];
        b[c].zm = cm[c];
        b[c].zp = cp[c];
        b[c].ym = ymn[c];
        b[c].yp = ypn[c];
        b[c].l = __shfl_up_sync(0xffffffffu, cc[c].w, 1);
        b[c].r = __shfl_down_sync(0xffffffffu, cc[c].x, 1);
        if (lane == 0) b[c].l = eln[c];
        if (lane == 31) b[c].r = ern[c];
        const int32_t* row = reinterpret_cast<const int32_t*>(A.q[c]) + z * plane + y * n2 + xi;
        nx[c] = active && z + 1 < ze && z + 2 < nbox ? __ldg(reinterpret_cast<const int4*>(row + 2 * plane)) : z4;
        if (z + 1 < ze) load_nb(c, z + 1, ymn[c], ypn[c], eln[c], ern[c]);
    }
    const int64_t oi = (z - A.zlo) * plane + y * n2 + xi;
    if (active) {
    double v[4];
    auto D = [&](int c, int k, int j) { return dv4(b[c], p, a0 + k, j, A.eps[c], A.two_eps[c], fd); };
    OutT* const* out = reinterpret_cast<OutT* const*>(A.out);
    if (OP == HSZG_OP_DERIV || OP == HSZG_OP_GRAD_LAP) {
#pragma unroll
        for (int k = 0; k < ND; k++) {
#pragma unroll
            for (int j = 0; j < 4; j++) v[j] = D(0, k, j);
            st4(out[k], oi, v);
        }
    }
    if (OP == HSZG_OP_LAPLACIAN || OP == HSZG_OP_GRAD_LAP) {
#pragma unroll
        for (int j = 0; j < 4; j++) v[j] = lap4<ND>(b[0], p, j, A.two_eps[0], fd);
        st4(out[OP == HSZG_OP_GRAD_LAP ? ND : 0], oi, v);
    }
    if (OP == HSZG_OP_GRADMAG) {
#pragma unroll
        for (int j = 0; j < 4; j++) {
            if (fd) {
                double s = 0.0;
#pragma unroll
                for (int k = 0; k < ND; k++) {
                    const double d = D(0, k, j);
                    s = __dadd_rn(s, __dmul_rn(d, d));
                }
                v[j] = __dsqrt_rn(s);
            } else {
                u128 s = 0;
#pragma unroll
                for (int k = 0; k < ND; k++) {
                    const int64_t d = di4(b[0], p, a0 + k, j);
                    const uint64_t ad = (uint64_t)(d < 0 ? -d : d);
                    s += (u128)ad * ad;
                }
                const double sd = (uint64_t)(s >> 64) == 0
                                      ? __ull2double_rn((uint64_t)s)
                                      : __dadd_rn(__dmul_rn(__ull2double_rn((uint64_t)(s >> 64)), 18446744073709551616.0),
                                                  __ull2double_rn((uint64_t)s));
                v[j] = __dmul_rn(__dsqrt_rn(sd), A.eps[0]);
            }
        }
        st4(out[0], oi, v);
    }
    if (OP == HSZG_OP_DIVERGENCE) {
#pragma unroll
        for (int j = 0; j < 4; j++) {
            double acc = D(0, 0, j);
#pragma unroll
            for (int k = 1; k < NC; k++) acc = __dadd_rn(acc, D(k, k, j));
            v[j] = acc;
        }
        st4(out[0], oi, v);
    }
    if (OP == HSZG_OP_CURL) {
        if (ND == 2) {
#pragma unroll
            for (int j = 0; j < 4; j++) v[j] = __dsub_rn(D(0, 1, j), D(1 % NC, 0, j));
            st4(out[0], oi, v);
        } else {
#pragma unroll
            for (int j = 0; j < 4; j++) v[j] = __dsub_rn(D(2 % NC, 1, j), D(1 % NC, 2 % ND, j));
            st4(out[0], oi, v);
#pragma unroll
            for (int j = 0; j < 4; j++) v[j] = __dsub_rn(D(0, 2 % ND, j), D(2 % NC, 0, j));
            st4(out[1], oi, v);
#pragma unroll
            for (int j = 0; j < 4; j++) v[j] = __dsub_rn(D(1 % NC, 0, j), D(0, 1, j));
            st4(out[2], oi, v);
        }
    }
    }   // active
#pragma unroll
    for (int c = 0; c < NC; c++) {
        cm[c] = cc[c];
        cc[c] = cp[c];
        cp[c] = nx[c];
    }
    }   // z
}

template <int ND, typename OutT, bool FD>
static void launch_sv4_fd(const StencilArgs& A, dim3 grid, int zc, int64_t zend, cudaStream_t st) {
    switch (A.op) {
        case HSZG_OP_DERIV: k_stencil_v4<HSZG_OP_DERIV, ND, OutT, FD><<<grid, SV_THREADS, 0, st>>>(A, zc, zend); break;
        case HSZG_OP_LAPLACIAN:
            k_stencil_v4<HSZG_OP_LAPLACIAN, ND, OutT, FD><<<grid, SV_THREADS, 0, st>>>(A, zc, zend);
            break;
        case HSZG_OP_GRAD_LAP:
            k_stencil_v4<HSZG_OP_GRAD_LAP, ND, OutT, FD><<<grid, SV_THREADS, 0, st>>>(A, zc, zend);
            break;
        case HSZG_OP_GRADMAG:
            k_stencil_v4<HSZG_OP_GRADMAG, ND, OutT, FD><<<grid, SV_THREADS, 0, st>>>(A, zc, zend);
            break;
        case HSZG_OP_DIVERGENCE:
            k_stencil_v4<HSZG_OP_DIVERGENCE, ND, OutT, FD><<<grid, SV_THREADS, 0, st>>>(A, zc, zend);
            break;
        case HSZG_OP_CURL: k_stencil_v4<HSZG_OP_CURL, ND, OutT, FD><<<grid, SV_THREADS, 0, st>>>(A, zc, zend); break;
        default: break;
    }
}

template <int ND, typename OutT>
static void launch_sv4(const StencilArgs& A, dim3 grid, int zc, int64_t zend, cudaStream_t st) {
    if (A.float_domain == 1) launch_sv4_fd<ND, OutT, true>(A, grid, zc, zend, st);
    else launch_sv4_fd<ND, OutT, false>(A, grid, zc, zend, st);
}

}  // namespace hszg

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

static int stencil_impl(int op, int32_t ndims, const int64_t* dims, int32_t ncomp, const void* const* q,
                        const double* eps, int float_domain, int32_t out_type, void* const* out, int64_t zlo,
                        int64_t zhi, int64_t gz0, int64_t gN0, cudaStream_t st) {
    if (op == HSZG_OP_GRAD_LAP && ndims == 3 && ncomp == 1 && float_domain == 0 && out_type == HSZG_F32 &&
        dims[2] % 4 == 0 && dims[2] >= 4 && aligned16(q[0]) && aligned16(out[0]) && aligned16(out[1]) &&
        aligned16(out[2]) && aligned16(out[3]) && dims[1] <= 65535 && zhi - zlo <= 65535) {
        if (zhi - zlo < 1) return HSZG_OK;
        dim3 grid((unsigned)((dims[2] / 4 + GL_THREADS - 1) / GL_THREADS), (unsigned)dims[1], (unsigned)(zhi - zlo));
        k_grad_lap_f32<<<grid, GL_THREADS, 0, st>>>(reinterpret_cast<const int32_t*>(q[0]), dims[1], dims[2], zlo,
                                                     gz0, gN0, eps[0], 2.0 * eps[0],
                                                     reinterpret_cast<float*>(out[0]), reinterpret_cast<float*>(out[1]),
                                                     reinterpret_cast<float*>(out[2]), reinterpret_cast<float*>(out[3]));
        return cudaGetLastError() == cudaSuccess ? HSZG_OK : HSZG_CUDA;
    }
    if (ndims < 1 || ndims > 3 || ncomp < 1 || ncomp > 3) return HSZG_INVALID_ARG;
    if (out_type != HSZG_F32 && out_type != HSZG_F64) return HSZG_INVALID_ARG;
    StencilArgs A = {};
    A.op = op;
    A.nd = ndims;
    A.ncomp = ncomp;
    A.float_domain = float_domain;
    A.out_type = out_type;
    box3(ndims, dims, A.n);
    for (int c = 0; c < ncomp; c++) {
        A.q[c] = q[c];
        A.eps[c] = eps[c];
        A.two_eps[c] = 2.0 * eps[c];
    }
    int nout = 1;
    if (op == HSZG_OP_DERIV) nout = ndims;
    if (op == HSZG_OP_GRAD_LAP) nout = ndims + 1;
    if (op == HSZG_OP_CURL) nout = ncomp == 2 ? 1 : 3;
    for (int k = 0; k < nout; k++) A.out[k] = out[k];
    A.zlo = zlo;
    A.gz0 = gz0;
    A.gN0 = gN0;
    if (zhi - zlo < 1) return HSZG_OK;
    if (A.n[1] > 65535 || zhi - zlo > 65535) return HSZG_INVALID_ARG;
    if (A.n[0] * A.n[1] * A.n[2] == 0) return HSZG_OK;
    bool vec = ndims >= 2 && float_domain <= 1 && A.n[2] % 4 == 0 &&
               ((op == HSZG_OP_DIVERGENCE || op == HSZG_OP_CURL) ? ncomp == ndims : true);
    for (int c = 0; c < ncomp; c++) vec = vec && aligned16(q[c]);
    for (int k = 0; k < nout; k++) vec = vec && aligned16(out[k]);
    static const char* sv = getenv("HSZG_STENCIL");          // 's': scalar k_stencil only (A/B runs)
    if (vec && !(sv && sv[0] == 's')) {
        const int zc = ndims == 3 ? SV_ZC : 1;                 // planes per CTA (z sliding)
        const dim3 g4((unsigned)((A.n[2] / 4 + SV_THREADS - 1) / SV_THREADS), (unsigned)A.n[1],
                      (unsigned)((zhi - zlo + zc - 1) / zc));
        if (ndims == 3) {
            if (out_type == HSZG_F32) launch_sv4<3, float>(A, g4, zc, zhi, st);
            else launch_sv4<3, double>(A, g4, zc, zhi, st);
        } else {
            if (out_type == HSZG_F32) launch_sv4<2, float>(A, g4, zc, zhi, st);
            else launch_sv4<2, double>(A, g4, zc, zhi, st);
        }
        return cudaGetLastError() == cudaSuccess ? HSZG_OK : HSZG_CUDA;
    }
    dim3 grid((unsigned)((A.n[2] + 255) / 256), (unsigned)A.n[1], (unsigned)(zhi - zlo));
    k_stencil<<<grid, 256, 0, st>>>(A);
    return cudaGetLastError() == cudaSuccess ? HSZG_OK : HSZG_CUDA;
}

extern "C" int hszg_region_finalize(const int64_t* s1, const uint64_t* s2_lo, const int64_t* s2_hi, const int32_t* qmin,
                                    const int32_t* qmax, const int64_t* size, int64_t n_regions, double two_eps,
                                    double tau, double* mean, double* var, double* fmin, double* fmax,
                                    unsigned long long* count_dev, void* stream) {
    cudaStream_t st = as_stream(stream);
    cudaMemsetAsync(count_dev, 0, 8, st);
    if (n_regions <= 0) return HSZG_OK;
    k_region_finalize<<<grid_for(n_regions, 256, 148 * 8), 256, 0, st>>>(s1, s2_lo, s2_hi, qmin, qmax, size, n_regions,
                                                                         two_eps, tau, mean, var, fmin, fmax, count_dev);
    return cudaGetLastError() == cudaSuccess ? HSZG_OK : HSZG_CUDA;
}

extern "C" int hszg_reduce_flt(const double* x, int64_t n, const double* mean_dev, HszgSums* out_dev, void* ws,
                               size_t ws_bytes, void* stream) {
    cudaStream_t st = as_stream(stream);
    if (ws_bytes < hszg_reduce_ws_bytes(0)) return HSZG_INVALID_ARG;
    HszgSums* partials = reinterpret_cast<HszgSums*>(ws);
    const int grid = grid_for(n, RED_THREADS * 8, kMaxParts);
    k_reduce_flt<<<grid, RED_THREADS, 0, st>>>(x, n, mean_dev, partials);
    return finalize(partials, grid, out_dev, st);
}

extern "C" int hszg_sums_combine(const HszgSums* parts, int64_t n, HszgSums* out, void* stream) {
    return finalize(const_cast<HszgSums*>(parts), n, out, as_stream(stream));
}
