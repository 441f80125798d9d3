// recon.cu — stage 3 (prediction reversion, K-REC-*) and stage 4 (K-DEQ epilogue).
//
// Reference: recorrelate (compressors.py:201-226) and the stage-4 dequantize
// q.astype(float64) * (2.0*eps) (stages.py:88).
//   HSZX    : q = p + M_b, stream order == row-major          -> k_stream_full<1> (full chunks) /
//                                                                 k_tile_stream<add_meta>
//   HSZX_ND : q = p + M_b scattered block-contiguous -> row-major -> k_stream_full<2> / k_tile_blocks_fast /
//                                                                 k_tile_blocks (smem transpose)
//   HSZP    : q = inclusive cumsum of p over the flat stream  -> k_tile_scan(_fast) (decoupled look-back)
//   HSZP_ND : q = cumsum along every axis (Lorenzo inverse)     -> 3-D, n2 % 32 == 0: hszg_band_scan +
//             z prefix (k_col_scan / k_col_scan_bands); otherwise decode + row scan + column scans
//   hszg_quantized_sums: the HSZP / 3-D HSZP_ND scans reduce q instead of storing it
// All arithmetic is int32 with wrap-around: every prefix equals a q value,
// which fits int32, so modular sums are exact (the reference casts its int64
// result back to int32, compressors.py:226).
#include <cstdio>
#include <cstdlib>
#include <type_traits>
#include "tile.cuh"
#include "lookback.cuh"
#include "wtiles.cuh"
#include "moments.cuh"

extern "C" int hszg_band_scan(const HszgGeom* g, const HszgStream* s, int64_t band_rows, void* L, int32_t* A,
                              int32_t* strip_edges, int l_int16, int32_t* l_overflow, int ctas_per_sm, void* stream,
                              HszgErr* err);

namespace hszg {

// HSZG_STREAM_FULL=0 keeps the shared-tile kernels (A/B runs)
static bool sf_off() {
    static const char* e = getenv("HSZG_STREAM_FULL");
    return e && e[0] == '0';
}

template <typename OutT>
struct Conv;
template <>
struct Conv<int32_t> {
    __device__ __forceinline__ static int32_t go(int32_t q, double) { return q; }
};
template <>
struct Conv<float> {
    __device__ __forceinline__ static float go(int32_t q, double s) { return __double2float_rn(__dmul_rn((double)q, s)); }
};
template <>
struct Conv<double> {
    __device__ __forceinline__ static double go(int32_t q, double s) { return __dmul_rn((double)q, s); }
};

// ---- stream-order tiles (HSZX; also stage 2 with add_meta=false) ------------

template <bool AddMeta, typename OutT>
__global__ void __launch_bounds__(TILE_CHUNKS) k_tile_stream(SegGeo sg, const uint8_t* payload, uint64_t len,
                                                            const uint64_t* offsets, const int32_t* meta,
                                                            double two_eps, OutT* out) {
    TileCtx t = tile_stage(sg, payload, len, offsets, blockIdx.x);
    const int64_t c = t.c0 + threadIdx.x;
    if (c < t.c1) {
        const ChunkLoc L = locate_chunk(sg, c);
        const int local = (int)(L.start - t.e0);
        const int32_t m = AddMeta ? __ldg(meta + L.seg) : 0;
        int32_t* vals = t.vals;
        decode_chunk_words(t.words, (uint32_t)(offsets[c] - t.base), L.count,
                           [&](int j, int32_t v) { vals[pad_idx(local + j)] = v + m; });
    }
    __syncthreads();
    const int n = (int)(t.e1 - t.e0);
    for (int i = threadIdx.x; i < n; i += blockDim.x) out[t.e0 + i] = Conv<OutT>::go(t.vals[pad_idx(i)], two_eps);
}

// ---- HSZX_ND: groups of k blocks along the last axis, transposed to row-major -----

struct BlockTiles {
    int64_t k;        // segments per tile
    int64_t tpr;      // tiles per segment row = ceil(G2 / k)
};

template <typename OutT>
__global__ void __launch_bounds__(TILE_CHUNKS) k_tile_blocks(SegGeo sg, BlockTiles bt, const uint8_t* payload,
                                                            uint64_t len, const uint64_t* offsets,
                                                            const int32_t* meta, double two_eps, OutT* out) {
    extern __shared__ __align__(16) uint8_t tile_smem[];
    __shared__ uint64_t s_lo, s_hi;
    __shared__ int64_t s_c0, s_c1, s_e0;
    const int64_t tile = blockIdx.x;
    const int64_t row = tile / bt.tpr;             // segment row (b0, b1)
    const int64_t tb = tile - row * bt.tpr;
    const int64_t b0 = row / sg.G[1];
    const int64_t b1 = row - b0 * sg.G[1];
    const int64_t b2a = tb * bt.k;
    const int64_t b2b = (b2a + bt.k < sg.G[2]) ? b2a + bt.k : sg.G[2];
    const int c0cls = b0 == sg.G[0] - 1, c1cls = b1 == sg.G[1] - 1;
    const int64_t s0 = seg_ext(sg, 0, b0), s1 = seg_ext(sg, 1, b1);
    if (threadIdx.x == 0) {
        s_c0 = seg_chunk_start(sg, b0, b1, b2a);
        const int64_t last = b2b - 1;
        s_c1 = seg_chunk_start(sg, b0, b1, last) + sg.cpb[(c0cls << 2) | (c1cls << 1) | (last == sg.G[2] - 1)];
        s_lo = offsets[s_c0];
        s_hi = s_c1 < sg.n_chunks ? offsets[s_c1] : payload_end(offsets, sg.n_chunks, len);
        s_e0 = seg_elem_start(sg, b0, b1, b2a);
    }
    __syncthreads();
    const uint64_t base = s_lo & ~(uint64_t)15;
    const uint64_t nvec = (s_hi - base + 15) >> 4;
    int32_t* vals = reinterpret_cast<int32_t*>(tile_smem);
    uint4* sb = reinterpret_cast<uint4*>(tile_smem + (size_t)TILE_VALS * 4);
    const uint4* g = reinterpret_cast<const uint4*>(payload + base);
    for (uint64_t i = threadIdx.x; i < nvec; i += blockDim.x) sb[i] = __ldg(g + i);
    if (threadIdx.x == 0) sb[nvec] = make_uint4(0, 0, 0, 0);
    const uint32_t* words = reinterpret_cast<const uint32_t*>(sb);
    __syncthreads();
    // Tile geometry in 32-bit: the tile's segments are one segment-row slice, all full along x
    // except possibly the last one, so chunk -> (segment, chunk-in-segment) needs no 64-bit division.
    const int B2 = (int)sg.B[2];
    const int nlast = (int)(b2b - 1 - b2a);                 // index of the last segment in the tile
    const int last_ext = (int)seg_ext(sg, 2, b2b - 1);
    const int S1 = (int)s1;
    const int plane01 = (int)(s0 * s1);                     // rows of a segment (z, y pairs)
    const int segsz = plane01 * B2;                         // values in a full segment
    const int cpb = (segsz + kChunkCap - 1) / kChunkCap;    // chunks in a full segment
    const int lastsz = plane01 * last_ext;
    const int nch = (int)(s_c1 - s_c0);
    const int64_t mbase = (b0 * sg.G[1] + b1) * sg.G[2] + b2a;
    for (int ci = threadIdx.x; ci < nch; ci += blockDim.x) {
        int seg = ci / cpb;
        if (seg > nlast) seg = nlast;
        const int j = ci - seg * cpb;
        const int size = seg == nlast ? lastsz : segsz;
        const int left = size - j * kChunkCap;
        const int count = left < kChunkCap ? left : kChunkCap;
        const int local = seg * segsz + j * kChunkCap;
        const int32_t m = __ldg(meta + mbase + seg);
        decode_chunk_words(words, (uint32_t)(offsets[s_c0 + ci] - base), count,
                           [&](int jj, int32_t v) { vals[pad_idx(local + jj)] = v + m; });
    }
    __syncthreads();
    // row-major write-out of the (s0, s1, W) box
    const int64_t x0 = b2a * sg.B[2];
    const int64_t xe = (b2b == sg.G[2]) ? sg.n[2] : b2b * sg.B[2];
    const int W = (int)(xe - x0);
    const int64_t z0 = b0 * sg.B[0], y0 = b1 * sg.B[1];
    const int64_t n1 = sg.n[1], n2 = sg.n[2];
    if ((int)blockDim.x % W == 0) {
        // every thread keeps one x column: the per-x parts are loop invariant
        const int xl = threadIdx.x % W;
        const int step = blockDim.x / W;
        const int t = xl / B2;
        const int xi = xl - t * B2;
        const int s2t = (t == nlast) ? last_ext : B2;
        int zy = threadIdx.x / W;
        int zl = zy / S1, yl = zy - zl * S1;
        for (; zy < plane01; zy += step) {
            const int local = t * segsz + zy * s2t + xi;
            out[((z0 + zl) * n1 + (y0 + yl)) * n2 + x0 + xl] = Conv<OutT>::go(vals[pad_idx(local)], two_eps);
            yl += step;
            while (yl >= S1) {
                yl -= S1;
                zl++;
            }
        }
    } else {
        const int total = plane01 * W;
        for (int i = threadIdx.x; i < total; i += blockDim.x) {
            const int zy = i / W;
            const int xl = i - zy * W;
            const int t = xl / B2;
            const int xi = xl - t * B2;
            const int s2t = (t == nlast) ? last_ext : B2;
            const int local = t * segsz + zy * s2t + xi;
            const int zl = zy / S1, yl = zy - zl * S1;
            out[((z0 + zl) * n1 + (y0 + yl)) * n2 + x0 + xl] = Conv<OutT>::go(vals[pad_idx(local)], two_eps);
        }
    }
}

// Fast variant for full blocks (every n[i] % B[i] == 0, B2 % 4 == 0, 32 | B0*B1*B2 and
// 256 % (2048 / (B0*B1)) == 0, e.g. 8x8x8): the tile is k = 8192 / |block| whole blocks along x
// (a (B0, B1, k*B2) box), decoded with decode32 into the 36-word chunk layout, then written
// row-major with one 16-byte load + 16-byte store per 4 values; every thread keeps one int4
// column of the box (gpr = k*B2/4 columns, 256/gpr rows per pass).
template <typename OutT>
__device__ __forceinline__ void store4(OutT* p, int4 v, double s);
template <>
__device__ __forceinline__ void store4<int32_t>(int32_t* p, int4 v, double) {
    *reinterpret_cast<int4*>(p) = v;
}
template <>
__device__ __forceinline__ void store4<float>(float* p, int4 v, double s) {
    *reinterpret_cast<float4*>(p) = make_float4(Conv<float>::go(v.x, s), Conv<float>::go(v.y, s),
                                                Conv<float>::go(v.z, s), Conv<float>::go(v.w, s));
}
template <>
__device__ __forceinline__ void store4<double>(double* p, int4 v, double s) {
    reinterpret_cast<double2*>(p)[0] = make_double2(Conv<double>::go(v.x, s), Conv<double>::go(v.y, s));
    reinterpret_cast<double2*>(p)[1] = make_double2(Conv<double>::go(v.z, s), Conv<double>::go(v.w, s));
}

template <typename OutT>
__global__ void __launch_bounds__(TILE_CHUNKS) k_tile_blocks_fast(SegGeo sg, BlockTiles bt,
                                                                 const uint8_t* __restrict__ payload, uint64_t len,
                                                                 const uint64_t* __restrict__ offsets,
                                                                 const int32_t* __restrict__ meta, double two_eps,
                                                                 OutT* __restrict__ out) {
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ uint64_t s_lo, s_hi;
    int32_t* tile = reinterpret_cast<int32_t*>(smem);
    uint4* sb = reinterpret_cast<uint4*>(smem + kFastTileBytes);
    const int B0 = (int)sg.B[0], B1 = (int)sg.B[1], B2 = (int)sg.B[2];
    const int segsz = B0 * B1 * B2;
    const int cps = segsz >> 5;                               // chunks per block
    const int64_t tile_id = blockIdx.x;
    const int64_t row = tile_id / bt.tpr;                     // block row (b0, b1)
    const int64_t b2a = (tile_id - row * bt.tpr) * bt.k;
    const int nseg = (int)(sg.G[2] - b2a < bt.k ? sg.G[2] - b2a : bt.k);
    const int nch = nseg * cps;
    const int64_t c0 = (row * sg.G[2] + b2a) * cps;           // all blocks full: chunk = block * cps + j
    if (threadIdx.x == 0) {
        s_lo = offsets[c0];
        s_hi = c0 + nch < sg.n_chunks ? offsets[c0 + nch] : payload_end(offsets, sg.n_chunks, len);
    }
    __syncthreads();
    const uint64_t base = stage_range(payload, s_lo, s_hi, sb);
    uint32_t rel = 0;
    int32_t m = 0;
    if ((int)threadIdx.x < nch) {
        rel = (uint32_t)(__ldg(offsets + c0 + threadIdx.x) - base);
        m = __ldg(meta + row * sg.G[2] + b2a + threadIdx.x / cps);
    }
    __syncthreads();
    if ((int)threadIdx.x < nch)
        decode32<false>(reinterpret_cast<const uint32_t*>(sb), rel, tile + threadIdx.x * kChunkStride, m);
    __syncthreads();
    const int gpr = (int)bt.k * B2 / 4;                       // int4 columns of a full tile row
    const int gi = threadIdx.x % gpr;
    const int step = TILE_CHUNKS / gpr;
    if (4 * gi >= nseg * B2) return;
    const int t = (4 * gi) / B2, xl = 4 * gi - t * B2;
    const int64_t b0 = row / sg.G[1], b1 = row - b0 * sg.G[1];
    const int64_t n1 = sg.n[1], n2 = sg.n[2];
    OutT* o = out + (b0 * B0 * n1 + b1 * B1) * n2 + b2a * B2 + 4 * gi;
    const int plane01 = B0 * B1;
    int zy = threadIdx.x / gpr;
    int zl = zy / B1, yl = zy - zl * B1;
    for (; zy < plane01; zy += step) {
        const int local = zy * B2 + xl;                       // within block t
        const int ch = t * cps + (local >> 5);
        const int4 v = *reinterpret_cast<const int4*>(tile + ch * kChunkStride + (local & 31));
        store4<OutT>(o + ((int64_t)zl * n1 + yl) * n2, v, two_eps);
        yl += step;
        while (yl >= B1) {
            yl -= B1;
            zl++;
        }
    }
}

static bool blocks_fast_ok(const SegGeo& sg) {
    const int64_t B0 = sg.B[0], B1 = sg.B[1], B2 = sg.B[2];
    const int64_t segsz = B0 * B1 * B2;
    if (sg.n[0] % B0 || sg.n[1] % B1 || sg.n[2] % B2 || B2 % 4 || segsz % 32 || segsz > TILE_ELEMS) return false;
    if ((int64_t)TILE_ELEMS % segsz) return false;
    const int64_t gpr = (TILE_ELEMS / segsz) * B2 / 4;
    return gpr >= 1 && TILE_CHUNKS % gpr == 0;
}

// ---- HSZP: flat inclusive scan with decoupled look-back -------------------------

template <typename OutT>
__global__ void __launch_bounds__(TILE_CHUNKS) k_tile_scan(SegGeo sg, const uint8_t* payload, uint64_t len,
                                                          const uint64_t* offsets, LBState st, double two_eps,
                                                          OutT* out) {
    __shared__ unsigned int s_tile;
    __shared__ unsigned long long s_prefix;
    if (threadIdx.x == 0) s_tile = atomicAdd(st.ticket, 1u);
    __syncthreads();
    const int64_t tile = s_tile;
    TileCtx t = tile_stage(sg, payload, len, offsets, tile);
    const int64_t c = t.c0 + threadIdx.x;
    uint32_t run = 0;
    int local = 0, count = 0;
    int32_t* vals = t.vals;
    if (c < t.c1) {
        const ChunkLoc L = locate_chunk(sg, c);
        local = (int)(L.start - t.e0);
        count = L.count;
        decode_chunk_words(t.words, (uint32_t)(offsets[c] - t.base), L.count, [&](int j, int32_t v) {
            run += (uint32_t)v;
            vals[pad_idx(local + j)] = (int32_t)run;
        });
    }
    unsigned long long tot;
    const unsigned long long excl = block_exclusive_u64((unsigned long long)run, &tot);
    if (threadIdx.x < 32) {
        const unsigned long long e = lookback_exclusive_warp32(st, tile, (uint32_t)tot);
        if (threadIdx.x == 0) s_prefix = e;
    }
    __syncthreads();
    const uint32_t add = (uint32_t)(s_prefix + excl);
    for (int j = 0; j < count; j++) vals[pad_idx(local + j)] = (int32_t)((uint32_t)vals[pad_idx(local + j)] + add);
    __syncthreads();
    const int n = (int)(t.e1 - t.e0);
    for (int i = threadIdx.x; i < n; i += blockDim.x) out[t.e0 + i] = Conv<OutT>::go(t.vals[pad_idx(i)], two_eps);
}

// Fast variant when every chunk is full (n_chunks * 32 == N: chunk c holds stream values 32c..32c+31):
// TMA-free 16-B staging, decode32 (inclusive chunk prefix) into the 36-word layout, block scan of the
// chunk sums + the same warp look-back, then 16-B stores of value + (tile prefix + chunk prefix).
template <typename OutT>
__global__ void __launch_bounds__(TILE_CHUNKS) k_tile_scan_fast(const uint8_t* __restrict__ payload, uint64_t len,
                                                               const uint64_t* __restrict__ offsets, int64_t n_chunks,
                                                               LBState st, double two_eps, OutT* __restrict__ out,
                                                               HszgSums* partials) {
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ unsigned int s_tile;
    __shared__ unsigned long long s_prefix;
    __shared__ uint64_t s_lo, s_hi;
    __shared__ uint32_t s_add[TILE_CHUNKS];
    int32_t* tile = reinterpret_cast<int32_t*>(smem);
    uint4* sb = reinterpret_cast<uint4*>(smem + kFastTileBytes);
    if (threadIdx.x == 0) s_tile = atomicAdd(st.ticket, 1u);
    __syncthreads();
    const int64_t t = s_tile;
    const int64_t c0 = t * TILE_CHUNKS;
    const int nch = (int)(n_chunks - c0 < TILE_CHUNKS ? n_chunks - c0 : TILE_CHUNKS);
    if (threadIdx.x == 0) {
        s_lo = offsets[c0];
        s_hi = c0 + nch < n_chunks ? offsets[c0 + nch] : payload_end(offsets, n_chunks, len);
    }
    __syncthreads();
    const uint64_t base = stage_range(payload, s_lo, s_hi, sb);
    const uint32_t rel = (int)threadIdx.x < nch ? (uint32_t)(__ldg(offsets + c0 + threadIdx.x) - base) : 0u;
    __syncthreads();
    uint32_t run = 0;
    if ((int)threadIdx.x < nch)
        run = decode32<true>(reinterpret_cast<const uint32_t*>(sb), rel, tile + threadIdx.x * kChunkStride, 0);
    unsigned long long tot;
    const unsigned long long excl = block_exclusive_u64((unsigned long long)run, &tot);
    if (threadIdx.x < 32) {
        const unsigned long long e = lookback_exclusive_warp32(st, t, (uint32_t)tot);
        if (threadIdx.x == 0) s_prefix = e;
    }
    __syncthreads();
    s_add[threadIdx.x] = (uint32_t)(s_prefix + excl);
    __syncthreads();
    if (partials) {                                    // hszg_quantized_sums: reduce q instead of storing it
        int64_t s1 = 0;
        u128 s2 = 0;
        int mn = INT32_MAX, mx = INT32_MIN;
        for (int g = threadIdx.x; g < nch * 8; g += TILE_CHUNKS) {
            const int ch = g >> 3;
            const int4 v = *reinterpret_cast<const int4*>(tile + ch * kChunkStride + ((g & 7) << 2));
            const uint32_t a = s_add[ch];
            const int4 q = make_int4((int)((uint32_t)v.x + a), (int)((uint32_t)v.y + a), (int)((uint32_t)v.z + a),
                                     (int)((uint32_t)v.w + a));
            s1 += (int64_t)q.x + q.y + q.z + q.w;
            s2 += (u128)((uint64_t)((int64_t)q.x * q.x) + (uint64_t)((int64_t)q.y * q.y));
            s2 += (u128)((uint64_t)((int64_t)q.z * q.z) + (uint64_t)((int64_t)q.w * q.w));
            mn = min(mn, min(min(q.x, q.y), min(q.z, q.w)));
            mx = max(mx, max(max(q.x, q.y), max(q.z, q.w)));
        }
        Acc acc;
        acc.init();
        acc.s1 = s1;
        acc.s2 = (i128)s2;
        acc.vmin = mn;
        acc.vmax = mx;
        block_reduce(acc);
        if (threadIdx.x == 0) {
            acc.count = (int64_t)nch * kChunkCap;
            store_sums(partials + t, acc);
        }
        return;
    }
    OutT* o = out + c0 * kChunkCap;
    for (int g = threadIdx.x; g < nch * 8; g += TILE_CHUNKS) {
        const int ch = g >> 3;
        const int4 v = *reinterpret_cast<const int4*>(tile + ch * kChunkStride + ((g & 7) << 2));
        const uint32_t a = s_add[ch];
        store4<OutT>(o + 4 * g, make_int4((int)((uint32_t)v.x + a), (int)((uint32_t)v.y + a), (int)((uint32_t)v.z + a),
                                          (int)((uint32_t)v.w + a)), two_eps);
    }
}

// 4 values of a P2 row: int32 (16 B) or int16 (8 B, the narrow band-local prefixes)
__device__ __forceinline__ int4 ld_p2x4(const int32_t* p) { return __ldg(reinterpret_cast<const int4*>(p)); }
__device__ __forceinline__ int4 ld_p2x4(const int16_t* p) {
    const uint2 h = __ldg(reinterpret_cast<const uint2*>(p));
    return make_int4((int32_t)(int16_t)(h.x & 0xffffu), (int32_t)h.x >> 16, (int32_t)(int16_t)(h.y & 0xffffu),
                     (int32_t)h.y >> 16);
}

// V values of a P2 row (V = 4 or 2)
template <int V> struct P2Vec;
template <> struct P2Vec<4> {
    template <typename T> static __device__ __forceinline__ void ld(const T* p, int32_t* v) {
        const int4 t = ld_p2x4(p);
        v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
    }
};
template <> struct P2Vec<2> {
    static __device__ __forceinline__ void ld(const int32_t* p, int32_t* v) {
        const int2 t = __ldg(reinterpret_cast<const int2*>(p));
        v[0] = t.x; v[1] = t.y;
    }
    static __device__ __forceinline__ void ld(const int16_t* p, int32_t* v) {
        const uint32_t h = __ldg(reinterpret_cast<const uint32_t*>(p));
        v[0] = (int32_t)(int16_t)(h & 0xffffu); v[1] = (int32_t)h >> 16;
    }
};

// z prefix (one band per plane: L is the plane's 2-D prefix) reduced instead of stored: V columns per
// thread (one 16-B / 8-B / 4-B load per plane; Lc % 4 == 0 and a 16-B aligned src), U planes in flight.
// Planes with few column groups (512^2: 65536 int4 groups = 14 warps per SM) take V = 2 in 128-thread
// CTAs: the per-column chains (prefix, 64-bit sum, 128-bit sum of squares) are latency-bound, so twice
// the threads with half the work each run faster (512^3: 107 -> 87 us; one column per thread: 108 us).
template <typename SrcT, int V, int U>
__global__ void __launch_bounds__(256) k_col_scan_sums_v4(const SrcT* __restrict__ src, int64_t M, int64_t Lc,
                                                          HszgSums* partials) {
    const int64_t l = V * (blockIdx.x * (int64_t)blockDim.x + threadIdx.x);
    int64_t s1 = 0;
    u128 s2 = 0;
    int mn = INT32_MAX, mx = INT32_MIN;
    if (l < Lc) {
        uint32_t acc[V];
#pragma unroll
        for (int j = 0; j < V; j++) acc[j] = 0;
        const SrcT* c = src + l;
        auto take = [&](const int32_t* w) {
            uint64_t sq = 0;                    // V squares < 2^64 (|q| <= 2^31)
#pragma unroll
            for (int j = 0; j < V; j++) {
                acc[j] += (uint32_t)w[j];
                const int q = (int)acc[j];
                s1 += q;
                sq += (uint64_t)((int64_t)q * q);
                mn = min(mn, q);
                mx = max(mx, q);
            }
            s2 += (u128)sq;
        };
        int64_t m = 0;
        for (; m + U <= M; m += U) {
            int32_t v[U][V];
#pragma unroll
            for (int k = 0; k < U; k++) P2Vec<V>::ld(c + (m + k) * Lc, v[k]);
#pragma unroll
            for (int k = 0; k < U; k++) take(v[k]);
        }
        for (; m < M; m++) {
            int32_t v[V];
            P2Vec<V>::ld(c + m * Lc, v);
            take(v);
        }
    }
    Acc a;
    a.init();
    a.s1 = s1;
    a.s2 = (i128)s2;
    a.vmin = mn;
    a.vmax = mx;
    block_reduce(a);
    const int64_t cols = Lc - V * blockIdx.x * (int64_t)blockDim.x;
    const int64_t active = cols < V * (int64_t)blockDim.x ? cols : V * (int64_t)blockDim.x;
    if (threadIdx.x == 0) {
        a.count = active * M;
        store_sums(partials + blockIdx.x, a);
    }
}

// launch: four columns per thread in 256-thread CTAs, or two in 128-thread CTAs for small planes
template <typename SrcT>
static int64_t launch_col_scan_sums(const SrcT* src, int64_t M, int64_t Lc, HszgSums* partials, cudaStream_t st) {
    static const int force = getenv("HSZG_CSS_V") ? atoi(getenv("HSZG_CSS_V")) : 0;     // A/B runs: 2 or 4
    const bool narrow = force ? force == 2 : Lc / 4 < (int64_t)148 * 1024;
    if (narrow) {
        const int64_t nb = (Lc / 2 + 127) / 128;
        k_col_scan_sums_v4<SrcT, 2, 8><<<(unsigned)nb, 128, 0, st>>>(src, M, Lc, partials);
        return nb;
    }
    const int64_t nb = (Lc / 4 + 255) / 256;
    k_col_scan_sums_v4<SrcT, 4, 4><<<(unsigned)nb, 256, 0, st>>>(src, M, Lc, partials);
    return nb;
}

// ---- full-chunk streams without a shared value tile (register-resident chunks) ----------------
// Every chunk full (chunk c = stream values 32c .. 32c+31) and every segment full-size: a CTA stages
// the byte range of 256 chunks (16-B loads, ~15 KB of shared memory, so many CTAs per SM overlap their
// phases), each thread decodes its chunk with decode32s and stores it straight from registers
// (8 x 16-B stores per thread; every 128-B line is completed by one thread, merged in L2).
//   Mode 0: p (stage 2)   Mode 1: p + M_b (HSZX stage 3/4)
//   Mode 2: p + M_b scattered from block-contiguous to row-major (HSZX_ND stage 3/4; rows of B2 | 32
//           values, so a chunk is whole block rows and every 16-B store completes its sectors)
// (A register variant of the HSZP look-back scan measured slower than k_tile_scan_fast: 0.41 vs
// 0.34 ms at 512^3 — the look-back chain wants short-lived CTAs.)
constexpr int SF_THREADS = TILE_CHUNKS;

template <int Mode, typename OutT>
__global__ void __launch_bounds__(SF_THREADS) k_stream_full(const uint8_t* __restrict__ payload, uint64_t len,
                                                           const uint64_t* __restrict__ offsets, int64_t n_chunks,
                                                           const int32_t* __restrict__ meta, int64_t cps,
                                                           double two_eps, OutT* __restrict__ out, SegGeo sg) {
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ uint64_t s_lo, s_hi;
    uint4* sb = reinterpret_cast<uint4*>(smem);
    const int64_t c0 = (int64_t)blockIdx.x * SF_THREADS;
    const int nch = (int)(n_chunks - c0 < SF_THREADS ? n_chunks - c0 : SF_THREADS);
    const bool mine = (int)threadIdx.x < nch;
    const int64_t c = c0 + threadIdx.x;
    uint64_t off = 0;
    int32_t m = 0;
    if (mine) {
        off = __ldg(offsets + c);
        if (threadIdx.x == 0) s_lo = off;
        if ((int)threadIdx.x == nch - 1) s_hi = c + 1 < n_chunks ? __ldg(offsets + c + 1) : payload_end(offsets, n_chunks, len);
        if (Mode != 0) m = __ldg(meta + c / cps);
    }
    __syncthreads();
    const uint64_t base = stage_range(payload, s_lo, s_hi, sb);
    __syncthreads();
    if (!mine) return;
    if (Mode != 2) {
        OutT* o = out + c * kChunkCap;
        decode32s<false>(reinterpret_cast<const uint32_t*>(sb), (uint32_t)(off - base), m,
                         [&](int q, int4 v) { store4<OutT>(o + 4 * q, v, two_eps); });
        return;
    }
    // chunk j of block b: block-row-major values 32j .. 32j+31
    const uint32_t b = (uint32_t)(c / cps), j = (uint32_t)(c - (int64_t)b * cps);
    const uint32_t G1 = (uint32_t)sg.G[1], G2 = (uint32_t)sg.G[2], B1 = (uint32_t)sg.B[1], B2 = (uint32_t)sg.B[2];
    const uint32_t r = b / G2, b2 = b - r * G2, b0 = r / G1, b1 = r - b0 * G1;
    const int64_t n1 = sg.n[1], n2 = sg.n[2];
    OutT* ob = out + ((int64_t)b0 * sg.B[0] * n1 + (int64_t)b1 * B1) * n2 + (int64_t)b2 * B2;
    decode32s<false>(reinterpret_cast<const uint32_t*>(sb), (uint32_t)(off - base), m, [&](int q, int4 v) {
        const uint32_t l = 32 * j + 4 * q;
        const uint32_t row = l / B2, xl = l - row * B2;
        const uint32_t zl = row / B1, yl = row - zl * B1;
        store4<OutT>(ob + ((int64_t)zl * n1 + yl) * n2 + xl, v, two_eps);
    });
}

// full chunks and full-size segments (chunk c of segment c / cps)
static bool stream_full_ok(const HszgGeom* g, const SegGeo& sg, const void* out) {
    bool ok = g->n_chunks * kChunkCap == g->n && (sg.B[0] * sg.B[1] * sg.B[2]) % kChunkCap == 0 &&
              (reinterpret_cast<uintptr_t>(out) & 15) == 0;
    for (int a = 0; a < 3; a++) ok = ok && sg.E[a] == sg.B[a];
    return ok;
}

// Stream-order outputs (stage 2 p; HSZX stage 3/4 q = p + M_b, whose stream order is row-major) from
// warp-private 32-chunk tiles (wtiles.cuh): each lane decodes its chunk into the warp's shared tile
// (36-word chunk stride, 16-B stores), then the warp writes the tile's 1024 contiguous values with
// coalesced 16-B stores (512 B per warp instruction instead of 32 scattered 16-B pieces).
constexpr size_t WS_TILE_BYTES = (size_t)32 * kChunkStride * 4;

template <int Mode, typename OutT>
__global__ void __launch_bounds__(256, HSZG_WT_MINB_R) k_wt_stream(const uint8_t* __restrict__ payload, uint64_t len,
                                                   const uint64_t* __restrict__ offsets, int64_t n_chunks, MetaAux aux,
                                                   double two_eps, OutT* __restrict__ out, uint32_t sb_bytes) {
    extern __shared__ __align__(16) uint8_t smem[];
    const int lane = threadIdx.x & 31;
    int32_t* tile = reinterpret_cast<int32_t*>(wt_scratch(smem, sb_bytes, WS_TILE_BYTES));
    auto body = [&](int64_t c, const uint32_t* words, uint32_t rel, bool valid, int32_t m) {
        if (valid) decode32<false>(words, rel, tile + lane * kChunkStride, Mode ? m : 0);
        __syncwarp();
        const int64_t c0 = c - lane;
        const int nv = n_chunks - c0 < 32 ? (int)(n_chunks - c0) : 32;
        OutT* o = out + c0 * kChunkCap;
#pragma unroll
        for (int i = 0; i < 8; i++) {
            const int idx = 128 * i + 4 * lane;
            if ((idx >> 5) < nv)
                store4<OutT>(o + idx, *reinterpret_cast<const int4*>(tile + (idx >> 5) * kChunkStride + (idx & 31)),
                             two_eps);
        }
        __syncwarp();
    };
    if (Mode) warp_tiles(payload, len, offsets, n_chunks, smem + (threadIdx.x >> 5) * WT_NS * sb_bytes, sb_bytes,
                         wt_bars(smem, sb_bytes), body, aux);
    else warp_tiles(payload, len, offsets, n_chunks, smem + (threadIdx.x >> 5) * WT_NS * sb_bytes, sb_bytes,
                    wt_bars(smem, sb_bytes), body);
}

// HSZX_ND stage 3 / 4 with power-of-two block extents (B2 >= 4) and full blocks: the warp's tile
// (32 chunks, 1024 block-contiguous values: whole blocks or a part of one) is written to the row-major
// grid a float4 at a time — lane pairs write whole 32-B rows of 8^3 blocks, every sector full.  Block
// origins are computed once per tile (one lane per block) and shuffled to the writers.
struct BlkGeo {
    int lb0, lb1, lb2, lbs;           // log2 of the block extents, of the block size
    int64_t G1, G2, n1, n2;
    int pre;                          // lbs <= 10 and block-local offsets fit int32: per-lane offsets precomputed
};

template <typename OutT>
__global__ void __launch_bounds__(256, HSZG_WT_MINB_R) k_wt_blocks(const uint8_t* __restrict__ payload, uint64_t len,
                                                   const uint64_t* __restrict__ offsets, int64_t n_chunks, MetaAux aux,
                                                   BlkGeo bg, double two_eps, OutT* __restrict__ out, uint32_t sb_bytes) {
    extern __shared__ __align__(16) uint8_t smem[];
    const int lane = threadIdx.x & 31;
    int32_t* tile = reinterpret_cast<int32_t*>(wt_scratch(smem, sb_bytes, WS_TILE_BYTES));
    const int nblk = bg.lbs >= 10 ? 1 : 1 << (10 - bg.lbs);          // blocks per full tile (<= 32)
    // Blocks of <= 1024 values tile a 1024-value warp tile exactly, so store i of this lane always lands
    // in the same block of the tile at the same block-local offset: both are computed once here
    // (bg.pre: the host checked that the local offsets fit int32) instead of per store.
    int32_t loff[8];
    int lblk[8];
#pragma unroll
    for (int i = 0; i < 8; i++) {
        const int idx = 128 * i + 4 * lane;
        lblk[i] = bg.pre ? idx >> bg.lbs : 0;
        const int l = bg.pre ? idx & ((1 << bg.lbs) - 1) : 0;
        const int xl = l & ((1 << bg.lb2) - 1), yl = (l >> bg.lb2) & ((1 << bg.lb1) - 1), zl = l >> (bg.lb1 + bg.lb2);
        loff[i] = bg.pre ? (int32_t)(((int64_t)zl * bg.n1 + yl) * bg.n2 + xl) : 0;
    }
    warp_tiles(payload, len, offsets, n_chunks, smem + (threadIdx.x >> 5) * WT_NS * sb_bytes, sb_bytes,
               wt_bars(smem, sb_bytes), [&](int64_t c, const uint32_t* words, uint32_t rel, bool valid, int32_t m) {
        if (valid) decode32<false>(words, rel, tile + lane * kChunkStride, m);
        const int64_t c0 = c - lane;
        const int nv = n_chunks - c0 < 32 ? (int)(n_chunks - c0) : 32;
        const int64_t v0 = c0 * kChunkCap;
        const int64_t bfirst = v0 >> bg.lbs;
        int64_t org = 0;
        if (lane < nblk) {
            const int64_t b = bfirst + lane;
            const int64_t b2 = b % bg.G2, r = b / bg.G2;
            const int64_t b1 = r % bg.G1, b0 = r / bg.G1;
            org = (((b0 << bg.lb0) * bg.n1) + (b1 << bg.lb1)) * bg.n2 + (b2 << bg.lb2);
        }
        __syncwarp();
        if (bg.pre) {
#pragma unroll
            for (int i = 0; i < 8; i++) {
                const int64_t ob = __shfl_sync(0xffffffffu, org, lblk[i]);
                const int idx = 128 * i + 4 * lane;
                if ((idx >> 5) < nv)
                    store4<OutT>(out + ob + loff[i],
                                 *reinterpret_cast<const int4*>(tile + (idx >> 5) * kChunkStride + (idx & 31)), two_eps);
            }
            __syncwarp();
            return;
        }
        const int64_t bmask = ((int64_t)1 << bg.lbs) - 1;
#pragma unroll
        for (int i = 0; i < 8; i++) {
            const int idx = 128 * i + 4 * lane;
            const int64_t v = v0 + idx;
            const int bl = (int)((v >> bg.lbs) - bfirst);
            const int64_t ob = __shfl_sync(0xffffffffu, org, bl & 31);
            if ((idx >> 5) < nv) {
                const int64_t l = v & bmask;
                const int64_t xl = l & ((1 << bg.lb2) - 1);
                const int64_t yl = (l >> bg.lb2) & ((1 << bg.lb1) - 1);
                const int64_t zl = l >> (bg.lb1 + bg.lb2);
                store4<OutT>(out + ob + (zl * bg.n1 + yl) * bg.n2 + xl,
                             *reinterpret_cast<const int4*>(tile + (idx >> 5) * kChunkStride + (idx & 31)), two_eps);
            }
        }
        __syncwarp();
    }, aux);
}

static int ilog2_exact(int64_t v) {
    for (int k = 0; k < 62; k++)
        if (v == (int64_t)1 << k) return k;
    return -1;
}

// ---- HSZP stage 3 / 4 in three passes over warp tiles (compressors.py:212, the flat inclusive cumsum) ----
// (1) k_hszp_tile_totals: the wrap-around total of p over each 32-chunk tile (lean chunk sums);
// (2) k_hszp_carries: C_t = exclusive prefix of the tile totals (uint32 wrap-around is exact: every q
//     fits int32), two multi-CTA passes; (3) k_wt_prefix_stream: decode with the in-chunk prefix into the
// warp's shared tile, add C_t + the chunk's offset in the tile (warp scan), coalesced 16-B stores.  No
// look-back chain: every tile is independent once the carries are known.
__global__ void __launch_bounds__(256, HSZG_WT_MINB_R) k_hszp_tile_totals(const uint8_t* __restrict__ payload, uint64_t len,
                                                          const uint64_t* __restrict__ offsets, int64_t n_chunks,
                                                          uint32_t* __restrict__ tot, uint32_t sb) {
    extern __shared__ __align__(16) uint8_t smem[];
    const int lane = threadIdx.x & 31;
    warp_tiles(payload, len, offsets, n_chunks, smem + (threadIdx.x >> 5) * WT_NS * sb, sb, wt_bars(smem, sb),
               [&](int64_t c, const uint32_t* words, uint32_t rel, bool valid, int32_t) {
        uint32_t t = (uint32_t)chunk_moments<false, false>(words, rel, valid).sp;
        for (int d = 16; d > 0; d >>= 1) t += __shfl_down_sync(0xffffffffu, t, d);
        if (lane == 0) tot[c >> 5] = t;
    });
}

constexpr int HCS_THREADS = 256;
constexpr int HCS_BLOCKS = 148 * 4;

__device__ __forceinline__ void hcs_range(int64_t tiles, int64_t& t0, int64_t& t1) {
    const int64_t per = (tiles + gridDim.x - 1) / gridDim.x;
    const int64_t b0 = blockIdx.x * per, b1 = b0 + per < tiles ? b0 + per : tiles;
    const int64_t tp = (per + HCS_THREADS - 1) / HCS_THREADS;
    t0 = b0 + threadIdx.x * tp;
    t1 = t0 + tp < b1 ? t0 + tp : b1;
    if (t0 > b1) t0 = b1;
}

__global__ void __launch_bounds__(HCS_THREADS) k_hszp_carry_blocks(const uint32_t* __restrict__ tot, int64_t tiles,
                                                                   uint32_t* __restrict__ bt) {
    int64_t t0, t1;
    hcs_range(tiles, t0, t1);
    uint32_t sum = 0;
    for (int64_t t = t0; t < t1; t++) sum += tot[t];
    for (int d = 16; d > 0; d >>= 1) sum += __shfl_down_sync(0xffffffffu, sum, d);
    __shared__ uint32_t ws[HCS_THREADS / 32];
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = sum;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t v = 0;
        for (int i = 0; i < HCS_THREADS / 32; i++) v += ws[i];
        bt[blockIdx.x] = v;
    }
}

// in place: tot[t] -> C_t (exclusive prefix)
__global__ void __launch_bounds__(HCS_THREADS) k_hszp_carries(uint32_t* __restrict__ tot, int64_t tiles,
                                                              const uint32_t* __restrict__ bt) {
    __shared__ uint32_t s_run[HCS_THREADS];
    __shared__ uint32_t s_base;
    uint32_t base = 0;
    for (int i = threadIdx.x; i < (int)blockIdx.x; i += HCS_THREADS) base += bt[i];
    for (int d = 16; d > 0; d >>= 1) base += __shfl_down_sync(0xffffffffu, base, d);
    if (threadIdx.x == 0) s_base = 0;
    __syncthreads();
    if ((threadIdx.x & 31) == 0) atomicAdd(&s_base, base);
    int64_t t0, t1;
    hcs_range(tiles, t0, t1);
    uint32_t sum = 0;
    for (int64_t t = t0; t < t1; t++) sum += tot[t];
    s_run[threadIdx.x] = sum;
    __syncthreads();
    for (int d = 1; d < HCS_THREADS; d <<= 1) {
        const uint32_t v = threadIdx.x >= (unsigned)d ? s_run[threadIdx.x - d] : 0u;
        __syncthreads();
        s_run[threadIdx.x] += v;
        __syncthreads();
    }
    uint32_t carry = s_base + s_run[threadIdx.x] - sum;
    for (int64_t t = t0; t < t1; t++) {
        const uint32_t v = tot[t];
        tot[t] = carry;
        carry += v;
    }
}

struct CarryAux {      // the tile carry of chunk c (tile = 32 chunks)
    const uint32_t* C;
    __device__ __forceinline__ int32_t operator()(int64_t c) const { return (int32_t)__ldg(C + (c >> 5)); }
};

template <typename OutT>
__global__ void __launch_bounds__(256, HSZG_WT_MINB_R) k_wt_prefix_stream(const uint8_t* __restrict__ payload, uint64_t len,
                                                          const uint64_t* __restrict__ offsets, int64_t n_chunks,
                                                          CarryAux aux, double two_eps, OutT* __restrict__ out,
                                                          uint32_t sb) {
    extern __shared__ __align__(16) uint8_t smem[];
    const int lane = threadIdx.x & 31;
    int32_t* tile = reinterpret_cast<int32_t*>(wt_scratch(smem, sb, WS_TILE_BYTES));
    warp_tiles(payload, len, offsets, n_chunks, smem + (threadIdx.x >> 5) * WT_NS * sb, sb, wt_bars(smem, sb),
               [&](int64_t c, const uint32_t* words, uint32_t rel, bool valid, int32_t C) {
        uint32_t run = 0;
        if (valid) run = decode32<true>(words, rel, tile + lane * kChunkStride, 0);
        uint32_t inc = run;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
            if (lane >= d) inc += o;
        }
        const uint32_t add = (uint32_t)C + inc - run;
        const int64_t c0 = c - lane;
        const int nv = n_chunks - c0 < 32 ? (int)(n_chunks - c0) : 32;
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 8; i++) {
            const int idx = 128 * i + 4 * lane;
            const uint32_t a = __shfl_sync(0xffffffffu, add, idx >> 5);
            if ((idx >> 5) < nv) {
                const int4 v = *reinterpret_cast<const int4*>(tile + (idx >> 5) * kChunkStride + (idx & 31));
                store4<OutT>(out + c0 * kChunkCap + idx,
                             make_int4((int)((uint32_t)v.x + a), (int)((uint32_t)v.y + a), (int)((uint32_t)v.z + a),
                                       (int)((uint32_t)v.w + a)),
                             two_eps);
            }
        }
        __syncwarp();
    }, aux);
}

inline size_t hszp_prefix_ws(int64_t n_chunks) {
    const int64_t tiles = (n_chunks + 31) / 32;
    return (((size_t)tiles * 4 + 255) & ~(size_t)255) + HCS_BLOCKS * 4 + 256;
}

template <typename OutT>
static bool launch_hszp_prefix(const HszgGeom* g, const HszgStream* s, OutT* out, void* ws, size_t ws_bytes,
                               cudaStream_t st) {
    if (ws_bytes < hszp_prefix_ws(g->n_chunks)) return false;
    const int64_t tiles = (g->n_chunks + 31) / 32;
    uint32_t* tot = reinterpret_cast<uint32_t*>(ws);
    uint32_t* bt = reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(ws) + (((size_t)tiles * 4 + 255) & ~(size_t)255));
    size_t sm;
    uint32_t sb;
    unsigned grid = wtile_grid(k_hszp_tile_totals, s->max_bitwidth, g->n_chunks, &sm, &sb);
    k_hszp_tile_totals<<<grid, 256, sm, st>>>(s->payload, s->payload_len, s->offsets, g->n_chunks, tot, sb);
    const int nb = (int)(tiles < HCS_BLOCKS ? tiles : HCS_BLOCKS);
    k_hszp_carry_blocks<<<nb, HCS_THREADS, 0, st>>>(tot, tiles, bt);
    k_hszp_carries<<<nb, HCS_THREADS, 0, st>>>(tot, tiles, bt);
    grid = wtile_grid(k_wt_prefix_stream<OutT>, s->max_bitwidth, g->n_chunks, &sm, &sb, WS_TILE_BYTES);
    k_wt_prefix_stream<OutT><<<grid, 256, sm, st>>>(s->payload, s->payload_len, s->offsets, g->n_chunks,
                                                    CarryAux{tot}, 2.0 * g->eps, out, sb);
    return true;
}

template <int Mode, typename OutT>
static void launch_stream_full(const HszgGeom* g, const HszgStream* s, const SegGeo& sg, OutT* out, cudaStream_t st) {
    static const char* wtb = getenv("HSZG_STREAM");
    if (Mode == 2 && !(wtb && wtb[0] == 'c')) {
        BlkGeo bg{ilog2_exact(sg.B[0]), ilog2_exact(sg.B[1]), ilog2_exact(sg.B[2]), 0, sg.G[1], sg.G[2], sg.n[1], sg.n[2]};
        if (bg.lb0 >= 0 && bg.lb1 >= 0 && bg.lb2 >= 2) {
            bg.lbs = bg.lb0 + bg.lb1 + bg.lb2;
            bg.pre = bg.lbs <= 10 && ((sg.B[0] - 1) * sg.n[1] + sg.B[1]) * sg.n[2] < ((int64_t)1 << 31);
            const int64_t cps = (sg.B[0] * sg.B[1] * sg.B[2]) / kChunkCap;
            MetaAux aux{s->metadata, cps, ilog2_exact(cps)};
            size_t sm;
            uint32_t sb;
            const unsigned grid = wtile_grid(k_wt_blocks<OutT>, s->max_bitwidth, g->n_chunks, &sm, &sb, WS_TILE_BYTES);
            k_wt_blocks<OutT><<<grid, 256, sm, st>>>(s->payload, s->payload_len, s->offsets, g->n_chunks, aux, bg,
                                                    2.0 * g->eps, out, sb);
            return;
        }
    }
    static const char* wt = getenv("HSZG_STREAM");           // 'c': the CTA-tile kernel below (A/B runs)
    if (Mode != 2 && !(wt && wt[0] == 'c')) {
        const int64_t cps = (sg.B[0] * sg.B[1] * sg.B[2]) / kChunkCap;
        MetaAux aux{s->metadata, cps > 0 ? cps : 1, -1};
        for (int k = 0; k < 40; k++)
            if (aux.cps == (int64_t)1 << k) aux.shift = k;
        size_t sm;
        uint32_t sb;
        const unsigned grid = wtile_grid(k_wt_stream<Mode, OutT>, s->max_bitwidth, g->n_chunks, &sm, &sb,
                                         WS_TILE_BYTES);
        k_wt_stream<Mode, OutT><<<grid, 256, sm, st>>>(s->payload, s->payload_len, s->offsets, g->n_chunks, aux,
                                                       2.0 * g->eps, out, sb);
        return;
    }
    const size_t smem = stage_bytes(s->max_bitwidth);
    allow_smem(k_stream_full<Mode, OutT>, smem);
    const int64_t tiles = (g->n_chunks + SF_THREADS - 1) / SF_THREADS;
    k_stream_full<Mode, OutT><<<(unsigned)tiles, SF_THREADS, smem, st>>>(
        s->payload, s->payload_len, s->offsets, g->n_chunks, s->metadata, (sg.B[0] * sg.B[1] * sg.B[2]) / kChunkCap,
        2.0 * g->eps, out, sg);
}

// ---- HSZP_ND: row scans along the last axis, then column scans -----------------------

constexpr int ROW_THREADS = 256, ROW_ITEMS = 8;

// short rows (L <= 32 * 4 * RW_VEC, 16-B aligned, L % 4 == 0): one warp per row, each lane a contiguous
// run of int4 groups (local prefix), a warp scan of the lane totals, then the offsets added
constexpr int RW_VEC = 8;     // int4 groups per lane: rows up to 1024 values
__global__ void __launch_bounds__(256) k_row_scan_warp(int32_t* buf, int64_t rows, int64_t L) {
    const int lane = threadIdx.x & 31;
    const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    if (row >= rows) return;
    int4* r = reinterpret_cast<int4*>(buf + row * L);
    const int ng = (int)(L >> 2);
    const int per = (ng + 31) / 32;                 // groups per lane
    const int g0 = lane * per;
    int4 v[RW_VEC];
    uint32_t run = 0;
#pragma unroll
    for (int k = 0; k < RW_VEC; k++) {
        if (k < per && g0 + k < ng) {
            v[k] = r[g0 + k];
            v[k].x = (int)(run += (uint32_t)v[k].x);
            v[k].y = (int)(run += (uint32_t)v[k].y);
            v[k].z = (int)(run += (uint32_t)v[k].z);
            v[k].w = (int)(run += (uint32_t)v[k].w);
        }
    }
    uint32_t inc = run;
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= d) inc += o;
    }
    const uint32_t add = inc - run;
#pragma unroll
    for (int k = 0; k < RW_VEC; k++)
        if (k < per && g0 + k < ng)
            r[g0 + k] = make_int4((int)((uint32_t)v[k].x + add), (int)((uint32_t)v[k].y + add),
                                  (int)((uint32_t)v[k].z + add), (int)((uint32_t)v[k].w + add));
}

__global__ void __launch_bounds__(ROW_THREADS) k_row_scan(int32_t* buf, int64_t L) {
    const int64_t row = blockIdx.x;
    int32_t* r = buf + row * L;
    uint32_t carry = 0;
    for (int64_t base = 0; base < L; base += ROW_THREADS * ROW_ITEMS) {
        const int64_t i0 = base + (int64_t)threadIdx.x * ROW_ITEMS;
        uint32_t v[ROW_ITEMS];
        uint32_t run = 0;
#pragma unroll
        for (int k = 0; k < ROW_ITEMS; k++) {
            v[k] = (i0 + k < L) ? (uint32_t)r[i0 + k] : 0u;
            run += v[k];
        }
        unsigned long long tot;
        const uint32_t ex = (uint32_t)block_exclusive_u64(run, &tot);
        uint32_t acc = carry + ex;
#pragma unroll
        for (int k = 0; k < ROW_ITEMS; k++) {
            acc += v[k];
            if (i0 + k < L) r[i0 + k] = (int32_t)acc;
        }
        carry += (uint32_t)tot;
    }
}

// view [A][M][Lc]; inclusive scan along M for every (a, l)
template <typename OutT>
__global__ void k_col_scan(const int32_t* src, int64_t A, int64_t M, int64_t Lc, double two_eps, OutT* dst) {
    const int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t a = blockIdx.y;
    if (l >= Lc) return;
    const int32_t* s = src + a * M * Lc + l;
    OutT* d = dst + a * M * Lc + l;
    uint32_t acc = 0;
    int64_t m = 0;
    for (; m + 4 <= M; m += 4) {
        const uint32_t v0 = (uint32_t)s[(m + 0) * Lc], v1 = (uint32_t)s[(m + 1) * Lc];
        const uint32_t v2 = (uint32_t)s[(m + 2) * Lc], v3 = (uint32_t)s[(m + 3) * Lc];
        acc += v0; d[(m + 0) * Lc] = Conv<OutT>::go((int32_t)acc, two_eps);
        acc += v1; d[(m + 1) * Lc] = Conv<OutT>::go((int32_t)acc, two_eps);
        acc += v2; d[(m + 2) * Lc] = Conv<OutT>::go((int32_t)acc, two_eps);
        acc += v3; d[(m + 3) * Lc] = Conv<OutT>::go((int32_t)acc, two_eps);
    }
    for (; m < M; m++) {
        acc += (uint32_t)s[m * Lc];
        d[m * Lc] = Conv<OutT>::go((int32_t)acc, two_eps);
    }
}

// z prefix of band-local prefixes: q[z][y][x] = sum_{z' <= z} (L[z'][y][x] + A[z'][y / BR][x]), A the
// exclusive band offsets of hszg_band_scan (an L2-resident n0 x nb x n2 table).  One column per
// thread (tried: several rows or planes per thread — fewer threads in flight, slower).
template <typename OutT>
__global__ void k_col_scan_bands(const int32_t* src, const int32_t* __restrict__ A, int64_t M, int64_t n1, int64_t n2,
                                 int64_t BR, int64_t nb, double two_eps, OutT* dst) {
    const int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t Lc = n1 * n2;
    if (l >= Lc) return;
    const int64_t y = l / n2, x = l - y * n2;
    const int32_t* a = A + (y / BR) * n2 + x;
    const int64_t as = nb * n2;
    const int32_t* s = src + l;
    OutT* d = dst + l;
    uint32_t acc = 0;
    int64_t m = 0;
    // src may be dst, but every element is read once, by the thread that later overwrites it, so the
    // non-coherent path is safe and frees the compiler to batch the loads across the stores
    for (; m + 8 <= M; m += 8) {
        uint32_t v[8], o[8];
#pragma unroll
        for (int k = 0; k < 8; k++) {
            v[k] = (uint32_t)__ldg(s + (m + k) * Lc);
            o[k] = (uint32_t)__ldg(a + (m + k) * as);
        }
#pragma unroll
        for (int k = 0; k < 8; k++) {
            acc += v[k] + o[k];
            d[(m + k) * Lc] = Conv<OutT>::go((int32_t)acc, two_eps);
        }
    }
    for (; m < M; m++) {
        acc += (uint32_t)s[m * Lc] + (uint32_t)__ldg(a + m * as);
        d[m * Lc] = Conv<OutT>::go((int32_t)acc, two_eps);
    }
}

// Vectorised z prefix (Lc % 4 == 0, 16-byte aligned planes): four adjacent columns per thread, so a
// warp reads 512 contiguous bytes per plane instead of 128 — fewer, longer DRAM bursts for the
// plane-strided walk.  A (optional) = the band offsets of k_col_scan_bands.  src may be dst: every
// element is read once, by the thread that later overwrites it, so the non-coherent path is safe.
template <typename OutT>
__device__ __forceinline__ void store4(OutT* d, const uint32_t (&v)[4], double two_eps) {
    if constexpr (sizeof(OutT) == 4) {
        typedef typename std::conditional<std::is_same<OutT, float>::value, float4, int4>::type V4;
        V4 o;
        o.x = Conv<OutT>::go((int32_t)v[0], two_eps);
        o.y = Conv<OutT>::go((int32_t)v[1], two_eps);
        o.z = Conv<OutT>::go((int32_t)v[2], two_eps);
        o.w = Conv<OutT>::go((int32_t)v[3], two_eps);
        *reinterpret_cast<V4*>(d) = o;
    } else {
#pragma unroll
        for (int j = 0; j < 4; j += 2)
            *reinterpret_cast<double2*>(d + j) =
                make_double2(Conv<OutT>::go((int32_t)v[j], two_eps), Conv<OutT>::go((int32_t)v[j + 1], two_eps));
    }
}

template <typename OutT, bool BANDS, typename SrcT = int32_t>
__global__ void __launch_bounds__(256) k_col_scan_v4(const SrcT* src, const int32_t* __restrict__ A, int64_t M,
                                                     int64_t n1, int64_t n2, int64_t BR, int64_t nb, double two_eps,
                                                     OutT* dst, const int32_t* __restrict__ carry = nullptr) {
    const int64_t Lc = n1 * n2;
    const int64_t l = 4 * (blockIdx.x * (int64_t)blockDim.x + threadIdx.x);
    if (l >= Lc) return;
    const SrcT* s = src + l;
    OutT* d = dst + l;
    const int32_t* a = A;
    int64_t as = 0;
    if constexpr (BANDS) {
        const int64_t y = l / n2, x = l - y * n2;
        a = A + (y / BR) * n2 + x;
        as = nb * n2;
    }
    uint32_t acc[4] = {0, 0, 0, 0};
    if (carry) {                                 // q of the plane before the stream's first (a slab's carry)
        const int4 c = __ldg(reinterpret_cast<const int4*>(carry + l));
        acc[0] = (uint32_t)c.x;
        acc[1] = (uint32_t)c.y;
        acc[2] = (uint32_t)c.z;
        acc[3] = (uint32_t)c.w;
    }
    constexpr int U = 4;
    int64_t m = 0;
    for (; m + U <= M; m += U) {
        int4 v[U], o[U];
#pragma unroll
        for (int k = 0; k < U; k++) {
            v[k] = ld_p2x4(s + (m + k) * Lc);
            if constexpr (BANDS) o[k] = __ldg(reinterpret_cast<const int4*>(a + (m + k) * as));
            else o[k] = make_int4(0, 0, 0, 0);
        }
#pragma unroll
        for (int k = 0; k < U; k++) {
            acc[0] += (uint32_t)v[k].x + (uint32_t)o[k].x;
            acc[1] += (uint32_t)v[k].y + (uint32_t)o[k].y;
            acc[2] += (uint32_t)v[k].z + (uint32_t)o[k].z;
            acc[3] += (uint32_t)v[k].w + (uint32_t)o[k].w;
            store4<OutT>(d + (m + k) * Lc, acc, two_eps);
        }
    }
    for (; m < M; m++) {
        const int4 v = ld_p2x4(s + m * Lc);
        int4 o = make_int4(0, 0, 0, 0);
        if constexpr (BANDS) o = __ldg(reinterpret_cast<const int4*>(a + m * as));
        acc[0] += (uint32_t)v.x + (uint32_t)o.x;
        acc[1] += (uint32_t)v.y + (uint32_t)o.y;
        acc[2] += (uint32_t)v.z + (uint32_t)o.z;
        acc[3] += (uint32_t)v.w + (uint32_t)o.w;
        store4<OutT>(d + m * Lc, acc, two_eps);
    }
}

// The same z prefix (no band offsets) with two columns per thread in 128-thread CTAs, eight planes in flight:
// planes with few int4 column groups (512^2: 65536 = 13 warps per SM) leave k_col_scan_v4 latency-bound
// (4.9 TB/s); twice the threads with half the columns each hide the load latency.
template <typename OutT, typename SrcT, bool BANDS = false>
__global__ void __launch_bounds__(128) k_col_scan_v2(const SrcT* src, int64_t M, int64_t Lc, double two_eps, OutT* dst,
                                                     const int32_t* __restrict__ carry,
                                                     const int32_t* __restrict__ A = nullptr, int64_t n2 = 1,
                                                     int64_t BR = 1, int64_t nb = 1) {
    const int64_t l = 2 * (blockIdx.x * (int64_t)blockDim.x + threadIdx.x);
    if (l >= Lc) return;
    const SrcT* s = src + l;
    OutT* d = dst + l;
    const int32_t* a = A;                        // BANDS: + the exclusive band offsets A[z][y / BR][x] per plane
    int64_t as = 0;
    if constexpr (BANDS) {
        const int64_t y = l / n2, x = l - y * n2;
        a = A + (y / BR) * n2 + x;
        as = nb * n2;
    }
    uint32_t acc[2] = {0, 0};
    if (carry) {
        const int2 c = __ldg(reinterpret_cast<const int2*>(carry + l));
        acc[0] = (uint32_t)c.x;
        acc[1] = (uint32_t)c.y;
    }
    auto put = [&](OutT* o) {
        if constexpr (sizeof(OutT) == 4) {
            OutT t[2] = {Conv<OutT>::go((int32_t)acc[0], two_eps), Conv<OutT>::go((int32_t)acc[1], two_eps)};
            *reinterpret_cast<uint2*>(o) = *reinterpret_cast<const uint2*>(t);
        } else {
            *reinterpret_cast<double2*>(o) =
                make_double2(Conv<OutT>::go((int32_t)acc[0], two_eps), Conv<OutT>::go((int32_t)acc[1], two_eps));
        }
    };
    constexpr int U = 8;
    int64_t m = 0;
    for (; m + U <= M; m += U) {
        int32_t v[U][2];
#pragma unroll
        for (int k = 0; k < U; k++) {
            P2Vec<2>::ld(s + (m + k) * Lc, v[k]);
            if constexpr (BANDS) {
                const int2 o = __ldg(reinterpret_cast<const int2*>(a + (m + k) * as));
                v[k][0] += o.x;
                v[k][1] += o.y;
            }
        }
#pragma unroll
        for (int k = 0; k < U; k++) {
            acc[0] += (uint32_t)v[k][0];
            acc[1] += (uint32_t)v[k][1];
            put(d + (m + k) * Lc);
        }
    }
    for (; m < M; m++) {
        int32_t v[2];
        P2Vec<2>::ld(s + m * Lc, v);
        if constexpr (BANDS) {
            const int2 o = __ldg(reinterpret_cast<const int2*>(a + m * as));
            v[0] += o.x;
            v[1] += o.y;
        }
        acc[0] += (uint32_t)v[0];
        acc[1] += (uint32_t)v[1];
        put(d + m * Lc);
    }
}

// small planes take the two-column kernel (HSZG_CS_V=4 forces the four-column one for A/B runs)
inline bool col_scan_narrow(int64_t Lc) {
    static const int force = getenv("HSZG_CS_V") ? atoi(getenv("HSZG_CS_V")) : 0;
    return force ? force == 2 : Lc / 4 < (int64_t)148 * 1024;
}

// Few, long columns (e.g. the y pass of a 2-D field: 3600 columns of 1800): S threads per column
// scan S segments — sums, an exclusive prefix across the segments in shared memory, then the
// segment rescans (re-read from L2) — so the launch has ~150k threads instead of one per column.
// src may be dst: every element is read in the first pass before any thread writes.
template <typename OutT>
__global__ void k_col_scan_seg(const int32_t* src, int64_t M, int64_t Lc, double two_eps, OutT* dst) {
    __shared__ uint32_t part[32][33];
    const int tx = threadIdx.x, sy = threadIdx.y, S = blockDim.y;
    const int64_t l = blockIdx.x * 32 + tx;
    const int64_t a = blockIdx.y;
    const bool act = l < Lc;
    const int64_t seg = (M + S - 1) / S;
    const int64_t m0 = sy * seg, m1 = m0 + seg < M ? m0 + seg : M;
    const int32_t* s = src + a * M * Lc + l;
    OutT* d = dst + a * M * Lc + l;
    uint32_t sum = 0;
    if (act) {
        int64_t m = m0;
        for (; m + 4 <= m1; m += 4)
            sum += (uint32_t)s[m * Lc] + (uint32_t)s[(m + 1) * Lc] + (uint32_t)s[(m + 2) * Lc] + (uint32_t)s[(m + 3) * Lc];
        for (; m < m1; m++) sum += (uint32_t)s[m * Lc];
    }
    part[sy][tx] = sum;
    __syncthreads();
    uint32_t acc = 0;
    for (int k = 0; k < sy; k++) acc += part[k][tx];
    if (!act) return;
    int64_t m = m0;
    for (; m + 4 <= m1; m += 4) {             // four loads in flight before the dependent stores
        const uint32_t v0 = (uint32_t)s[m * Lc], v1 = (uint32_t)s[(m + 1) * Lc];
        const uint32_t v2 = (uint32_t)s[(m + 2) * Lc], v3 = (uint32_t)s[(m + 3) * Lc];
        acc += v0; d[m * Lc] = Conv<OutT>::go((int32_t)acc, two_eps);
        acc += v1; d[(m + 1) * Lc] = Conv<OutT>::go((int32_t)acc, two_eps);
        acc += v2; d[(m + 2) * Lc] = Conv<OutT>::go((int32_t)acc, two_eps);
        acc += v3; d[(m + 3) * Lc] = Conv<OutT>::go((int32_t)acc, two_eps);
    }
    for (; m < m1; m++) {
        acc += (uint32_t)s[m * Lc];
        d[m * Lc] = Conv<OutT>::go((int32_t)acc, two_eps);
    }
}

template <typename OutT>
static void launch_col_scan(const int32_t* src, int64_t A, int64_t M, int64_t Lc, double two_eps, OutT* dst,
                            cudaStream_t st) {
    const int64_t cols = A * Lc;
    if (M >= 64 && cols < 148 * 1024 && A <= 65535) {
        int S = 1;
        while (S < 32 && cols * S < 148 * 2048 && S * 16 < M) S <<= 1;
        k_col_scan_seg<OutT><<<dim3((unsigned)((Lc + 31) / 32), (unsigned)A), dim3(32, S), 0, st>>>(src, M, Lc, two_eps,
                                                                                                   dst);
        return;
    }
    // grid.y is limited to 65535: fold A into chunks
    const int64_t ymax = 65535;
    for (int64_t a0 = 0; a0 < A; a0 += ymax) {
        const int64_t na = (A - a0) < ymax ? (A - a0) : ymax;
        dim3 grid((unsigned)((Lc + 255) / 256), (unsigned)na);
        k_col_scan<OutT><<<grid, 256, 0, st>>>(src + a0 * M * Lc, na, M, Lc, two_eps, dst + a0 * M * Lc);
    }
}

template <typename OutT>
__global__ void k_convert(const int32_t* q, int64_t n, double two_eps, OutT* out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = Conv<OutT>::go(__ldg(q + i), two_eps);
}

// flat inclusive int32 scan (device-wide, decoupled look-back); values wrap mod 2^32
__global__ void __launch_bounds__(SCAN_THREADS) k_scan_i32(const int32_t* in, int32_t* out, int64_t n, LBState st) {
    __shared__ unsigned int s_tile;
    __shared__ unsigned long long s_prefix;
    if (threadIdx.x == 0) s_tile = atomicAdd(st.ticket, 1u);
    __syncthreads();
    const int64_t tile = s_tile;
    const int64_t base = tile * SCAN_TILE + (int64_t)threadIdx.x * SCAN_ITEMS;
    uint32_t v[SCAN_ITEMS];
    uint32_t run = 0;
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; k++) {
        const int64_t i = base + k;
        v[k] = i < n ? (uint32_t)in[i] : 0u;
        run += v[k];
    }
    unsigned long long tot;
    const unsigned long long ex = block_exclusive_u64(run, &tot);
    if (threadIdx.x < 32) {
        const unsigned long long e = lookback_exclusive_warp32(st, tile, (uint32_t)tot);
        if (threadIdx.x == 0) s_prefix = e;
    }
    __syncthreads();
    uint32_t acc = (uint32_t)(s_prefix + ex);
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; k++) {
        const int64_t i = base + k;
        acc += v[k];
        if (i < n) out[i] = (int32_t)acc;
    }
}

__global__ void k_add_plane(int32_t* q, const int32_t* carry, int64_t plane, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        q[i] = (int32_t)((uint32_t)q[i] + (uint32_t)__ldg(carry + (i % plane)));
}

// ---- permutation helpers (HSZX_ND block-contiguous order) ------------------------------

template <typename Fn>
__device__ __forceinline__ void for_chunk_elements(const SegGeo& sg, int64_t c, Fn fn) {
    const ChunkLoc L = locate_chunk(sg, c);
    const int64_t b2 = L.seg % sg.G[2];
    const int64_t r = L.seg / sg.G[2];
    const int64_t b1 = r % sg.G[1];
    const int64_t b0 = r / sg.G[1];
    const int64_t s1 = seg_ext(sg, 1, b1), s2 = seg_ext(sg, 2, b2);
    int64_t l = (int64_t)L.j * kChunkCap;
    int64_t zl = l / (s1 * s2);
    int64_t rem = l - zl * s1 * s2;
    int64_t yl = rem / s2;
    int64_t xl = rem - yl * s2;
    for (int j = 0; j < L.count; j++) {
        const int64_t flat = ((b0 * sg.B[0] + zl) * sg.n[1] + (b1 * sg.B[1] + yl)) * sg.n[2] + b2 * sg.B[2] + xl;
        fn(L.start + j, flat, L.seg);
        if (++xl == s2) {
            xl = 0;
            if (++yl == s1) {
                yl = 0;
                ++zl;
            }
        }
    }
}

__global__ void k_stream_perm(SegGeo sg, int64_t* perm) {
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < sg.n_chunks;
         c += (int64_t)gridDim.x * blockDim.x)
        for_chunk_elements(sg, c, [&](int64_t pos, int64_t flat, int64_t) { perm[pos] = flat; });
}

__global__ void k_scatter_grid(SegGeo sg, const int32_t* src, const int32_t* meta, int add_meta, int32_t* out) {
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < sg.n_chunks;
         c += (int64_t)gridDim.x * blockDim.x)
        for_chunk_elements(sg, c, [&](int64_t pos, int64_t flat, int64_t seg) {
            out[flat] = src[pos] + (add_meta ? meta[seg] : 0);
        });
}

__global__ void k_metadata_grid(SegGeo sg, const int32_t* meta, int64_t* out) {
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < sg.n_chunks;
         c += (int64_t)gridDim.x * blockDim.x)
        for_chunk_elements(sg, c, [&](int64_t, int64_t flat, int64_t seg) { out[flat] = (int64_t)meta[seg]; });
}

}  // namespace hszg

using namespace hszg;

int hszg_set_cuda_error(HszgErr* err, cudaError_t e, const char* where);
int hszg_launch_decode(const HszgGeom* g, const HszgStream* s, int32_t* out, cudaStream_t st, HszgErr* err);

static inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

#define HSZG_CHECK_LAUNCH(where)                                           \
    do {                                                                   \
        cudaError_t _e = cudaGetLastError();                               \
        if (_e != cudaSuccess) return hszg_set_cuda_error(err, _e, where); \
    } while (0)

static bool blocks_fit_tile(const SegGeo& sg) { return sg.cpb[0] <= TILE_CHUNKS; }

// Stage 2 -> 3/4 on a stream-order int32 buffer `buf` (overwritten): the per-kind
// recorrelation (compressors.py:201-226) followed by the output conversion.
template <typename OutT>
static int transform_decoded(const HszgGeom* g, const SegGeo& sg, const int32_t* meta, int32_t* buf, OutT* out,
                             void* ws, size_t ws_bytes, cudaStream_t st, HszgErr* err) {
    const double two_eps = 2.0 * g->eps;
    const size_t need = (size_t)g->n * 4;
    if (g->kind == HSZG_HSZP_ND) {
        const int64_t N0 = sg.n[0], N1 = sg.n[1], N2 = sg.n[2];
        if (N2 % 4 == 0 && N2 <= 32 * 4 * RW_VEC && (reinterpret_cast<uintptr_t>(buf) & 15) == 0)
            k_row_scan_warp<<<(unsigned)((N0 * N1 + 7) / 8), 256, 0, st>>>(buf, N0 * N1, N2);
        else
            k_row_scan<<<(unsigned)(N0 * N1), ROW_THREADS, 0, st>>>(buf, N2);
        HSZG_CHECK_LAUNCH("row scan");
        const bool zpass = N0 > 1;
        if (N1 > 1) {
            if (zpass) launch_col_scan<int32_t>(buf, N0, N1, N2, two_eps, buf, st);
            else launch_col_scan<OutT>(buf, N0, N1, N2, two_eps, out, st);
            HSZG_CHECK_LAUNCH("col scan y");
        }
        if (zpass) {
            launch_col_scan<OutT>(buf, 1, N0, N1 * N2, two_eps, out, st);
            HSZG_CHECK_LAUNCH("col scan z");
        } else if (N1 <= 1) {
            launch_col_scan<OutT>(buf, 1, 1, N2, two_eps, out, st);  // conversion only
        }
        return HSZG_OK;
    }
    if (g->kind == HSZG_HSZP) {
        const int64_t tiles = (g->n + SCAN_TILE - 1) / SCAN_TILE;
        if (ws_bytes < lookback_ws_bytes(g->n)) {
            err->status = HSZG_INVALID_ARG;
            snprintf(err->message, sizeof(err->message), "workspace too small for the flat scan");
            return HSZG_INVALID_ARG;
        }
        LBState lb = lookback_carve(ws, tiles);
        cudaMemsetAsync(ws, 0, lookback_clear_bytes(tiles), st);
        k_scan_i32<<<(unsigned)tiles, SCAN_THREADS, 0, st>>>(buf, buf, g->n, lb);
        HSZG_CHECK_LAUNCH("flat scan");
        if (sizeof(OutT) != 4 || (void*)out != (void*)buf) launch_col_scan<OutT>(buf, 1, 1, g->n, two_eps, out, st);
        else launch_col_scan<OutT>(buf, 1, 1, g->n, two_eps, out, st);
        HSZG_CHECK_LAUNCH("convert");
        return HSZG_OK;
    }
    // HSZX / HSZX_ND: add metadata (and scatter block-contiguous -> row-major), then convert
    if (g->kind == HSZG_HSZX_ND) {
        if (ws_bytes < need) {
            err->status = HSZG_INVALID_ARG;
            snprintf(err->message, sizeof(err->message), "workspace too small for block scatter");
            return HSZG_INVALID_ARG;
        }
        int32_t* streamv = reinterpret_cast<int32_t*>(ws);
        cudaMemcpyAsync(streamv, buf, need, cudaMemcpyDeviceToDevice, st);
        k_scatter_grid<<<grid_for(g->n_chunks, 256, 148 * 64), 256, 0, st>>>(sg, streamv, meta, 1, buf);
    } else {
        k_scatter_grid<<<grid_for(g->n_chunks, 256, 148 * 64), 256, 0, st>>>(sg, buf, meta, 1, buf);
    }
    HSZG_CHECK_LAUNCH("scatter");
    launch_col_scan<OutT>(buf, 1, 1, g->n, two_eps, out, st);  // M=1: pure conversion
    HSZG_CHECK_LAUNCH("convert");
    return HSZG_OK;
}


// Narrow band-local prefixes for the API's 3-D HSZP_ND passes (stage 3 / 4, quantized sums): with one band per
// plane the band scan's L is P2 = q[z] - q[z-1], small for the reference's fields, so it is stored as int16 (half
// the write and the z scan's read of int32; hszg_band_scan l_mode 1) and its overflow flag is read back (a host
// sync, skipped under stream capture).  1: p16 holds every P2 value; 0: the caller runs the int32 path; < 0: error.
static int band_scan_narrow(const HszgGeom* g, const HszgStream* s, int64_t br, int16_t* p16, int32_t* A,
                            int32_t* flag, cudaStream_t st, HszgErr* err) {
    static const char* off = getenv("HSZG_P2_NARROW");       // "0": always int32 (A/B runs)
    if ((off && off[0] == '0') || g->dims[2] % 8) return 0;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
        cudaGetLastError();
        return 0;
    }
    if (cudaMemsetAsync(flag, 0, sizeof(int32_t), st) != cudaSuccess) return -HSZG_CUDA;
    const int rr = hszg_band_scan(g, s, br, p16, A, nullptr, 1, flag, 0, st, err);
    if (rr) return -rr;
    int32_t h = 0;
    if (cudaMemcpyAsync(&h, flag, sizeof(h), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
        return -HSZG_CUDA;
    return h == 0 ? 1 : 0;
}

template <typename OutT>
static int reconstruct_typed(const HszgGeom* g, const HszgStream* s, OutT* out, void* ws, size_t ws_bytes,
                             cudaStream_t st, HszgErr* err, const int32_t* carry = nullptr) {
    const SegGeo sg = make_seggeo(*g);
    const double two_eps = 2.0 * g->eps;
    if (g->n == 0) return HSZG_OK;
    const size_t smem = tile_smem_bytes(s->max_bitwidth);
    const int64_t tiles = (g->n_chunks + TILE_CHUNKS - 1) / TILE_CHUNKS;
    const bool fast = s->canonical != 0;
    // a carry plane (hszg_reconstruct_carry) is folded into the HSZP_ND band-scan z prefix only
    const bool band_path = fast && g->kind == HSZG_HSZP_ND && g->ndims == 3 && sg.n[2] % 32 == 0 &&
                           sg.n[2] <= 4096 && sg.n[0] <= 65535;
    if (carry && (!band_path || (reinterpret_cast<uintptr_t>(carry) & 15))) return HSZG_UNSUPPORTED_STAGE;
    switch (g->kind) {
        case HSZG_HSZX:
            if (fast && stream_full_ok(g, sg, out) && !sf_off()) {
                launch_stream_full<1, OutT>(g, s, sg, out, st);
                HSZG_CHECK_LAUNCH("reconstruct hszx");
                return HSZG_OK;
            }
            if (fast) {
                allow_smem(k_tile_stream<true, OutT>, smem);
                k_tile_stream<true, OutT><<<(unsigned)tiles, TILE_CHUNKS, smem, st>>>(
                    sg, s->payload, s->payload_len, s->offsets, s->metadata, two_eps, out);
                HSZG_CHECK_LAUNCH("reconstruct hszx");
                return HSZG_OK;
            }
            break;
        case HSZG_HSZP_ND:
            // 3-D with whole-chunk rows: one band per plane in hszg_band_scan (decode + x + y prefix in
            // one pass), then the z prefix (+ conversion) — instead of decode, row, y and z passes
            if (fast && g->ndims == 3 && sg.n[2] % 32 == 0 && sg.n[2] <= 4096 &&
                sg.n[0] <= 65535) {
                const size_t n4 = (size_t)g->n * 4;
                const int64_t br = recon_band_rows(sg.n[0], sg.n[1], sg.n[2]);
                const int64_t nb = (sg.n[1] + br - 1) / br;
                const size_t need = (sizeof(OutT) == 4 ? 0 : n4) + (size_t)sg.n[0] * nb * sg.n[2] * 4;
                // narrow first: int16 P2 in the workspace (n4 bytes for fp64 outputs, else n * 2), then A, flag
                const size_t p2b = sizeof(OutT) == 4 ? (((size_t)g->n * 2 + 255) & ~(size_t)255) : n4;
                const size_t abytes = (size_t)sg.n[0] * nb * sg.n[2] * 4;
                if (ws_bytes >= p2b + abytes + 256) {
                    int16_t* p16 = reinterpret_cast<int16_t*>(ws);
                    int32_t* A16 = reinterpret_cast<int32_t*>(reinterpret_cast<char*>(ws) + p2b);
                    int32_t* flag = reinterpret_cast<int32_t*>(reinterpret_cast<char*>(ws) + p2b + abytes);
                    const int nr_ = band_scan_narrow(g, s, br, p16, A16, flag, st, err);
                    if (nr_ < 0) return -nr_;
                    if (nr_ == 1) {
                        const unsigned cst = 256u;
                        const unsigned blocks = (unsigned)((sg.n[1] * sg.n[2] / 4 + 255) / 256);
                        if (nb == 1 && col_scan_narrow(sg.n[1] * sg.n[2]))
                            k_col_scan_v2<OutT, int16_t><<<(unsigned)((sg.n[1] * sg.n[2] / 2 + 127) / 128), 128, 0, st>>>(
                                p16, sg.n[0], sg.n[1] * sg.n[2], two_eps, out, carry);
                        else if (nb == 1)
                            k_col_scan_v4<OutT, false, int16_t><<<blocks, cst, 0, st>>>(
                                p16, nullptr, sg.n[0], sg.n[1], sg.n[2], br, nb, two_eps, out, carry);
                        else if (col_scan_narrow(sg.n[1] * sg.n[2]))
                            k_col_scan_v2<OutT, int16_t, true><<<(unsigned)((sg.n[1] * sg.n[2] / 2 + 127) / 128), 128, 0, st>>>(
                                p16, sg.n[0], sg.n[1] * sg.n[2], two_eps, out, carry, A16, sg.n[2], br, nb);
                        else
                            k_col_scan_v4<OutT, true, int16_t><<<blocks, cst, 0, st>>>(
                                p16, A16, sg.n[0], sg.n[1], sg.n[2], br, nb, two_eps, out, carry);
                        HSZG_CHECK_LAUNCH("z scan (int16)");
                        return HSZG_OK;
                    }
                }
                if (ws_bytes >= need) {
                    int32_t* buf = sizeof(OutT) == 4 ? reinterpret_cast<int32_t*>(out) : reinterpret_cast<int32_t*>(ws);
                    int32_t* A = reinterpret_cast<int32_t*>(reinterpret_cast<char*>(ws) + (sizeof(OutT) == 4 ? 0 : n4));
                    const int rr = hszg_band_scan(g, s, br, buf, A, nullptr, 0, nullptr, 0, st, err);
                    if (rr) return rr;
                    const int64_t Lc = sg.n[1] * sg.n[2];
                    static const int v4 = getenv("HSZG_COLSCAN_V4") ? atoi(getenv("HSZG_COLSCAN_V4")) : 1;
                    if (v4 || carry) {      // n2 % 32 == 0: whole int4 groups, 16-byte aligned planes
                        const unsigned cst = 256u;
                        const unsigned blocks = (unsigned)((Lc / 4 + 255) / 256);
                        if (nb == 1 && col_scan_narrow(Lc))
                            k_col_scan_v2<OutT, int32_t><<<(unsigned)((Lc / 2 + 127) / 128), 128, 0, st>>>(
                                buf, sg.n[0], Lc, two_eps, out, carry);
                        else if (nb == 1)
                            k_col_scan_v4<OutT, false><<<blocks, cst, 0, st>>>(buf, nullptr, sg.n[0], sg.n[1], sg.n[2],
                                                                               br, nb, two_eps, out, carry);
                        else if (col_scan_narrow(Lc))
                            k_col_scan_v2<OutT, int32_t, true><<<(unsigned)((Lc / 2 + 127) / 128), 128, 0, st>>>(
                                buf, sg.n[0], Lc, two_eps, out, carry, A, sg.n[2], br, nb);
                        else
                            k_col_scan_v4<OutT, true><<<blocks, cst, 0, st>>>(buf, A, sg.n[0], sg.n[1], sg.n[2], br,
                                                                              nb, two_eps, out, carry);
                    } else if (nb == 1) {   // one band per plane: A holds zeros, the plain z prefix
                        launch_col_scan<OutT>(buf, 1, sg.n[0], sg.n[1] * sg.n[2], two_eps, out, st);
                    } else {
                        k_col_scan_bands<OutT><<<(unsigned)((Lc + 255) / 256), 256, 0, st>>>(
                            buf, A, sg.n[0], sg.n[1], sg.n[2], br, nb, two_eps, out);
                    }
                    HSZG_CHECK_LAUNCH("z scan");
                    return HSZG_OK;
                }
            }
            if (carry) return HSZG_UNSUPPORTED_STAGE;     // workspace too small for the band path
            break;
        case HSZG_HSZX_ND:
            if (fast && stream_full_ok(g, sg, out) && sg.B[2] % 4 == 0 && 32 % sg.B[2] == 0 && !sf_off()) {
                launch_stream_full<2, OutT>(g, s, sg, out, st);
                HSZG_CHECK_LAUNCH("reconstruct hszx-nd");
                return HSZG_OK;
            }
            if (fast && blocks_fast_ok(sg)) {
                BlockTiles bt;
                bt.k = TILE_ELEMS / (sg.B[0] * sg.B[1] * sg.B[2]);
                bt.tpr = (sg.G[2] + bt.k - 1) / bt.k;
                const int64_t nt = sg.G[0] * sg.G[1] * bt.tpr;
                const size_t fsmem = kFastTileBytes + stage_bytes(s->max_bitwidth);
                allow_smem(k_tile_blocks_fast<OutT>, fsmem);
                k_tile_blocks_fast<OutT><<<(unsigned)nt, TILE_CHUNKS, fsmem, st>>>(
                    sg, bt, s->payload, s->payload_len, s->offsets, s->metadata, two_eps, out);
                HSZG_CHECK_LAUNCH("reconstruct hszx-nd");
                return HSZG_OK;
            }
            if (fast && blocks_fit_tile(sg)) {
                BlockTiles bt;
                // k full segments hold <= TILE_CHUNKS chunks, hence <= TILE_ELEMS values
                bt.k = TILE_CHUNKS / sg.cpb[0];
                bt.tpr = (sg.G[2] + bt.k - 1) / bt.k;
                const int64_t nt = sg.G[0] * sg.G[1] * bt.tpr;
                allow_smem(k_tile_blocks<OutT>, smem);
                k_tile_blocks<OutT><<<(unsigned)nt, TILE_CHUNKS, smem, st>>>(sg, bt, s->payload, s->payload_len,
                                                                               s->offsets, s->metadata, two_eps, out);
                HSZG_CHECK_LAUNCH("reconstruct hszx-nd");
                return HSZG_OK;
            }
            break;
        case HSZG_HSZP:
            if (fast && g->n_chunks * kChunkCap == g->n && (reinterpret_cast<uintptr_t>(out) & 15) == 0 && !sf_off() &&
                launch_hszp_prefix<OutT>(g, s, out, ws, ws_bytes, st)) {
                HSZG_CHECK_LAUNCH("reconstruct hszp");
                return HSZG_OK;
            }
            if (fast) {
                if (ws_bytes < lookback_ws_bytes(g->n_chunks)) break;
                LBState lb = lookback_carve(ws, tiles);
                cudaMemsetAsync(ws, 0, lookback_clear_bytes(tiles), st);
                if (g->n_chunks * kChunkCap == g->n && (reinterpret_cast<uintptr_t>(out) & 15) == 0) {
                    const size_t fsmem = kFastTileBytes + stage_bytes(s->max_bitwidth);
                    allow_smem(k_tile_scan_fast<OutT>, fsmem);
                    k_tile_scan_fast<OutT><<<(unsigned)tiles, TILE_CHUNKS, fsmem, st>>>(
                        s->payload, s->payload_len, s->offsets, g->n_chunks, lb, two_eps, out, nullptr);
                    HSZG_CHECK_LAUNCH("reconstruct hszp");
                    return HSZG_OK;
                }
                allow_smem(k_tile_scan<OutT>, smem);
                k_tile_scan<OutT><<<(unsigned)tiles, TILE_CHUNKS, smem, st>>>(sg, s->payload, s->payload_len,
                                                                               s->offsets, lb, two_eps, out);
                HSZG_CHECK_LAUNCH("reconstruct hszp");
                return HSZG_OK;
            }
            break;
        default:
            break;
    }
    // generic path: stage-2 decode into an int32 buffer, then the per-kind transform
    int32_t* buf;
    const size_t need = (size_t)g->n * 4;
    if (sizeof(OutT) == 4) {
        buf = reinterpret_cast<int32_t*>(out);   // in place: int32 and fp32 have the same footprint
    } else {
        if (ws_bytes < need) {
            err->status = HSZG_INVALID_ARG;
            snprintf(err->message, sizeof(err->message), "workspace too small for reconstruct (%zu < %zu)",
                     ws_bytes, need);
            return HSZG_INVALID_ARG;
        }
        buf = reinterpret_cast<int32_t*>(ws);
    }
    int r = hszg_launch_decode(g, s, buf, st, err);
    if (r) return r;
    char* rest = reinterpret_cast<char*>(ws) + (sizeof(OutT) == 4 ? 0 : need);
    const size_t rest_bytes = ws_bytes > (sizeof(OutT) == 4 ? 0 : need) ? ws_bytes - (sizeof(OutT) == 4 ? 0 : need) : 0;
    return transform_decoded<OutT>(g, sg, s->metadata, buf, out, rest, rest_bytes, st, err);
}

extern "C" int hszg_reconstruct(const HszgGeom* g, const HszgStream* s, void* out, int out_type, void* ws,
                                size_t ws_bytes, void* stream, HszgErr* err) {
    err->status = HSZG_OK;
    cudaStream_t st = as_stream(stream);
    switch (out_type) {
        case HSZG_I32: return reconstruct_typed<int32_t>(g, s, reinterpret_cast<int32_t*>(out), ws, ws_bytes, st, err);
        case HSZG_F32: return reconstruct_typed<float>(g, s, reinterpret_cast<float*>(out), ws, ws_bytes, st, err);
        case HSZG_F64: return reconstruct_typed<double>(g, s, reinterpret_cast<double*>(out), ws, ws_bytes, st, err);
        default:
            err->status = HSZG_INVALID_ARG;
            snprintf(err->message, sizeof(err->message), "unknown output type %d", out_type);
            return HSZG_INVALID_ARG;
    }
}

extern "C" int hszg_reconstruct_carry(const HszgGeom* g, const HszgStream* s, void* out, int out_type,
                                      const int32_t* carry, void* ws, size_t ws_bytes, void* stream, HszgErr* err) {
    err->status = HSZG_OK;
    cudaStream_t st = as_stream(stream);
    if (!carry) return hszg_reconstruct(g, s, out, out_type, ws, ws_bytes, stream, err);
    switch (out_type) {
        case HSZG_I32: return reconstruct_typed<int32_t>(g, s, reinterpret_cast<int32_t*>(out), ws, ws_bytes, st, err, carry);
        case HSZG_F32: return reconstruct_typed<float>(g, s, reinterpret_cast<float*>(out), ws, ws_bytes, st, err, carry);
        case HSZG_F64: return reconstruct_typed<double>(g, s, reinterpret_cast<double*>(out), ws, ws_bytes, st, err, carry);
        default:
            err->status = HSZG_INVALID_ARG;
            snprintf(err->message, sizeof(err->message), "unknown output type %d", out_type);
            return HSZG_INVALID_ARG;
    }
}

extern "C" int hszg_stream_perm(const HszgGeom* g, int64_t* perm, void* stream) {
    const SegGeo sg = make_seggeo(*g);
    if (g->n_chunks == 0) return HSZG_OK;
    k_stream_perm<<<grid_for(g->n_chunks, 256, 148 * 64), 256, 0, as_stream(stream)>>>(sg, perm);
    return cudaGetLastError() == cudaSuccess ? HSZG_OK : HSZG_CUDA;
}

extern "C" int hszg_scatter_grid(const HszgGeom* g, const int32_t* src, const int32_t* metadata, int add_meta,
                                 int32_t* out, void* stream) {
    const SegGeo sg = make_seggeo(*g);
    if (g->n_chunks == 0) return HSZG_OK;
    k_scatter_grid<<<grid_for(g->n_chunks, 256, 148 * 64), 256, 0, as_stream(stream)>>>(sg, src, metadata, add_meta,
                                                                                       out);
    return cudaGetLastError() == cudaSuccess ? HSZG_OK : HSZG_CUDA;
}

extern "C" int hszg_metadata_grid(const HszgGeom* g, const int32_t* metadata, int64_t* out, void* stream) {
    const SegGeo sg = make_seggeo(*g);
    if (g->n_chunks == 0) return HSZG_OK;
    k_metadata_grid<<<grid_for(g->n_chunks, 256, 148 * 64), 256, 0, as_stream(stream)>>>(sg, metadata, out);
    return cudaGetLastError() == cudaSuccess ? HSZG_OK : HSZG_CUDA;
}

extern "C" int hszg_dequantize(const int32_t* q, int64_t n, double two_eps, void* out, int out_type, void* stream) {
    if (n <= 0) return HSZG_OK;
    cudaStream_t st = as_stream(stream);
    const int grid = grid_for(n, 256 * 4, 148 * 32);
    if (out_type == HSZG_F32) k_convert<float><<<grid, 256, 0, st>>>(q, n, two_eps, reinterpret_cast<float*>(out));
    else if (out_type == HSZG_F64) k_convert<double><<<grid, 256, 0, st>>>(q, n, two_eps, reinterpret_cast<double*>(out));
    else return HSZG_INVALID_ARG;
    return cudaGetLastError() == cudaSuccess ? HSZG_OK : HSZG_CUDA;
}

template <typename OutT>
static int recorrelate_typed(const HszgGeom* g, const int32_t* p, const int32_t* meta, OutT* out, void* ws,
                             size_t ws_bytes, cudaStream_t st, HszgErr* err) {
    const SegGeo sg = make_seggeo(*g);
    const size_t need = (size_t)g->n * 4;
    if (g->n == 0) return HSZG_OK;
    int32_t* buf;
    size_t head = 0;
    if (sizeof(OutT) == 4) {
        buf = reinterpret_cast<int32_t*>(out);
    } else {
        if (ws_bytes < need) {
            err->status = HSZG_INVALID_ARG;
            snprintf(err->message, sizeof(err->message), "workspace too small for recorrelate");
            return HSZG_INVALID_ARG;
        }
        buf = reinterpret_cast<int32_t*>(ws);
        head = need;
    }
    if ((const void*)buf != (const void*)p) cudaMemcpyAsync(buf, p, need, cudaMemcpyDeviceToDevice, st);
    return transform_decoded<OutT>(g, sg, meta, buf, out, reinterpret_cast<char*>(ws) + head,
                                   ws_bytes > head ? ws_bytes - head : 0, st, err);
}

extern "C" int hszg_recorrelate(const HszgGeom* g, const int32_t* p, const int32_t* metadata, void* out, int out_type,
                                void* ws, size_t ws_bytes, void* stream, HszgErr* err) {
    err->status = HSZG_OK;
    cudaStream_t st = as_stream(stream);
    switch (out_type) {
        case HSZG_I32: return recorrelate_typed<int32_t>(g, p, metadata, reinterpret_cast<int32_t*>(out), ws, ws_bytes, st, err);
        case HSZG_F32: return recorrelate_typed<float>(g, p, metadata, reinterpret_cast<float*>(out), ws, ws_bytes, st, err);
        case HSZG_F64: return recorrelate_typed<double>(g, p, metadata, reinterpret_cast<double*>(out), ws, ws_bytes, st, err);
        default: return HSZG_INVALID_ARG;
    }
}

extern "C" int hszg_add_plane(int32_t* q, const int32_t* carry, int64_t plane, int64_t n, void* stream) {
    if (n <= 0) return HSZG_OK;
    k_add_plane<<<grid_for(n, 256 * 4, 148 * 32), 256, 0, as_stream(stream)>>>(q, carry, plane, n);
    return cudaGetLastError() == cudaSuccess ? HSZG_OK : HSZG_CUDA;
}

// ---- HSZP_ND shard carry: U[y,x] = sum_z p[z,y,x] over a stream's planes (wrap-around int32) ----
// the carry plane of a z-slab is the 2-D prefix of this plane sum (Lorenzo linearity).
namespace hszg {
__global__ void __launch_bounds__(TILE_CHUNKS) k_plane_sum(SegGeo sg, const uint8_t* payload, uint64_t len,
                                                          const uint64_t* offsets, int64_t plane,
                                                          unsigned int* U) {
    TileCtx t = tile_stage(sg, payload, len, offsets, blockIdx.x);
    const int64_t c = t.c0 + threadIdx.x;
    if (c < t.c1) {
        const ChunkLoc L = locate_chunk(sg, c);
        const int64_t base = L.start % plane;
        decode_chunk_words(t.words, (uint32_t)(offsets[c] - t.base), L.count, [&](int j, int32_t v) {
            if (v) atomicAdd(U + base + j, (unsigned int)v);
        });
    }
}
}  // namespace hszg

extern "C" int hszg_plane_sum(const HszgGeom* g, const HszgStream* s, int32_t* plane_out, void* stream, HszgErr* err) {
    err->status = HSZG_OK;
    cudaStream_t st = as_stream(stream);
    const SegGeo sg = make_seggeo(*g);
    if (g->kind != HSZG_HSZP_ND || g->ndims != 3 || !s->canonical) {
        err->status = HSZG_INVALID_ARG;
        snprintf(err->message, sizeof(err->message), "plane_sum needs a validated canonical 3-D HSZP_ND stream");
        return HSZG_INVALID_ARG;
    }
    const int64_t plane = sg.n[1] * sg.n[2];
    cudaMemsetAsync(plane_out, 0, (size_t)plane * 4, st);
    if (g->n_chunks == 0) return HSZG_OK;
    const int64_t tiles = (g->n_chunks + TILE_CHUNKS - 1) / TILE_CHUNKS;
    allow_smem(k_plane_sum, tile_smem_bytes(s->max_bitwidth));
    k_plane_sum<<<(unsigned)tiles, TILE_CHUNKS, tile_smem_bytes(s->max_bitwidth), st>>>(
        sg, s->payload, s->payload_len, s->offsets, plane, reinterpret_cast<unsigned int*>(plane_out));
    HSZG_CHECK_LAUNCH("plane sum");
    return HSZG_OK;
}

// In-place inclusive scan along the middle axis of an int32 view [A][M][L] (HSZP_ND y prefix of
// the windowed pipeline: A planes, M rows, L columns).
extern "C" int hszg_col_scan(int32_t* buf, int64_t A, int64_t M, int64_t L, void* stream) {
    if (A <= 0 || M <= 0 || L <= 0) return HSZG_OK;
    launch_col_scan<int32_t>(buf, A, M, L, 0.0, buf, as_stream(stream));
    return cudaGetLastError() == cudaSuccess ? HSZG_OK : HSZG_CUDA;
}

// stage-2 decode of a full-chunk canonical stream (codec.cu's hszg_decode fast path)
int hszg_decode_full(const HszgGeom* g, const HszgStream* s, int32_t* out, cudaStream_t st) {
    const SegGeo sg = make_seggeo(*g);
    if (!s->canonical || g->n_chunks * kChunkCap != g->n || (reinterpret_cast<uintptr_t>(out) & 15) || sf_off())
        return 1;
    launch_stream_full<0, int32_t>(g, s, sg, out, st);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

// ---- hszg_quantized_sums -------------------------------------------------------------------------
size_t hszg_reduce_ws_bytes(int64_t tiles);
int hszg_finalize_sums(HszgSums* partials, int64_t nparts, HszgSums* out, cudaStream_t st);

// 0 when the stream has no fused path (see include/hszg.h)
namespace hszg {
size_t hszp_tile_sums_ws(const HszgGeom* g, const HszgStream* s);
int hszp_tile_sums(const HszgGeom* g, const HszgStream* s, HszgSums* out_dev, void* ws, size_t ws_bytes,
                   cudaStream_t st);
}  // namespace hszg

size_t hszg_quantized_sums_ws(const HszgGeom* g, const HszgStream* s) {
    if (!s || !s->canonical || g->n == 0) return 0;
    if (const size_t t = hszg::hszp_tile_sums_ws(g, s)) return t;          // HSZP: tile algebra (ops.cu)
    const SegGeo sg = make_seggeo(*g);
    if (g->kind == HSZG_HSZP_ND && g->ndims == 3 && sg.n[2] % 32 == 0 && sg.n[2] <= 4096 && sg.n[0] <= 65535 &&
        recon_band_rows(sg.n[0], sg.n[1], sg.n[2]) >= sg.n[1]) {
        const int64_t Lc = sg.n[1] * sg.n[2];
        return (size_t)g->n * 4 + (size_t)sg.n[0] * sg.n[2] * 4 + hszg_reduce_ws_bytes((Lc + 255) / 256) + 512;
    }
    return 0;
}

extern "C" int hszg_quantized_sums(const HszgGeom* g, const HszgStream* s, HszgSums* out_dev, void* ws,
                                   size_t ws_bytes, void* stream, HszgErr* err) {
    err->status = HSZG_OK;
    cudaStream_t st = as_stream(stream);
    const size_t need = hszg_quantized_sums_ws(g, s);
    if (need == 0 || ws_bytes < need) {
        err->status = HSZG_INVALID_ARG;
        snprintf(err->message, sizeof(err->message), "quantized_sums: no fused path for this stream or workspace too small");
        return HSZG_INVALID_ARG;
    }
    const SegGeo sg = make_seggeo(*g);
    char* w = reinterpret_cast<char*>(ws);
    if (g->kind == HSZG_HSZP && hszg::hszp_tile_sums_ws(g, s)) {
        if (hszg::hszp_tile_sums(g, s, out_dev, ws, ws_bytes, st)) {
            err->status = HSZG_CUDA;
            snprintf(err->message, sizeof(err->message), "quantized sums hszp: launch failed");
            return HSZG_CUDA;
        }
        return HSZG_OK;
    }
    // HSZP_ND 3-D, one band per plane
    int32_t* L = reinterpret_cast<int32_t*>(w);
    int32_t* A = reinterpret_cast<int32_t*>(w + (size_t)g->n * 4);
    HszgSums* partials = reinterpret_cast<HszgSums*>(w + (((size_t)g->n * 4 + (size_t)sg.n[0] * sg.n[2] * 4 + 255) &
                                                          ~(size_t)255));
    const int64_t Lc = sg.n[1] * sg.n[2];
    if ((size_t)g->n >= 256) {   // int16 P2 in the first half of L's space, the flag after it (band_scan_narrow)
        int16_t* p16 = reinterpret_cast<int16_t*>(w);
        int32_t* flag = reinterpret_cast<int32_t*>(w + (((size_t)g->n * 2 + 255) & ~(size_t)255));
        const int nr_ = band_scan_narrow(g, s, sg.n[1], p16, A, flag, st, err);
        if (nr_ < 0) return -nr_;
        if (nr_ == 1) {
            const int64_t nb4 = launch_col_scan_sums(p16, sg.n[0], Lc, partials, st);   // n2 % 32 == 0: Lc % 4 == 0
            HSZG_CHECK_LAUNCH("quantized sums hszp-nd (int16)");
            return hszg_finalize_sums(partials, nb4, out_dev, st);
        }
    }
    const int rr = hszg_band_scan(g, s, sg.n[1], L, A, nullptr, 0, nullptr, 0, st, err);
    if (rr) return rr;
    const int64_t nb4 = launch_col_scan_sums(L, sg.n[0], Lc, partials, st);
    HSZG_CHECK_LAUNCH("quantized sums hszp-nd");
    return hszg_finalize_sums(partials, nb4, out_dev, st);
}
