// tile.cuh — the staged chunk-tile decoder used by every fused kernel (K-DEC).
//
// A CTA owns TILE_CHUNKS consecutive chunks [c0, c1).  With a canonical chunk
// index (the encoder's exclusive scan, validated once per upload) those
// chunks occupy the contiguous byte range [off[c0], off[c1]) of the payload
// and the contiguous stream range [e0, e1).  The CTA copies the byte range
// into shared memory with aligned 16-byte loads (coalesced, no per-chunk
// global traffic besides the 8-byte index entry), then every thread decodes
// one chunk lane-serially from shared memory (decode_chunk_words) into a
// bank-padded int32 value tile, which the epilogue consumes in stream order
// with coalesced stores.
#pragma once
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <unordered_map>
#include "common.cuh"

namespace hszg {

constexpr int TILE_CHUNKS = 256;                  // = blockDim.x of tile kernels
constexpr int TILE_ELEMS = TILE_CHUNKS * kChunkCap;
constexpr int TILE_VALS = TILE_ELEMS + TILE_ELEMS / 32 + 32;   // padded int32 slots

__device__ __forceinline__ int pad_idx(int i) { return i + (i >> 5); }

// shared-memory bytes of a tile kernel for a stream whose widest chunk has max_bw bits
inline size_t tile_smem_bytes(int max_bw) {
    size_t bytes = (size_t)TILE_CHUNKS * (size_t)chunk_bytes(kChunkCap, max_bw) + 64;
    bytes = (bytes + 15) & ~(size_t)15;
    return (size_t)TILE_VALS * 4 + bytes + 16;
}

// Opt a tile kernel into more dynamic shared memory than the default 48 KB minus its static shared
// memory (wide bit widths need ~69 KB).  The attribute is raised once per kernel to the largest
// size seen, so steady-state launches (and launches under CUDA-graph capture) make no runtime call.
inline void allow_smem_raw(const void* kernel, size_t bytes) {
    static std::mutex mu;
    static std::unordered_map<const void*, size_t> set;
    if (bytes <= 32 * 1024) return;              // below every kernel's default limit (static < 16 KB)
    std::lock_guard<std::mutex> lock(mu);
    size_t& cur = set[kernel];
    if (bytes <= cur) return;
    const size_t want = bytes < 96 * 1024 ? 96 * 1024 : bytes;
    const cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)want);
    if (e != cudaSuccess) {
        fprintf(stderr, "hszg: cudaFuncSetAttribute(%zu) failed: %s\n", want, cudaGetErrorString(e));
        cudaGetLastError();
        return;
    }
    // the maximum shared-memory carveout, so kernels on concurrent streams (the HSZP_ND band scans
    // under the z-sweeps) can co-reside on an SM without waiting for it to drain and reconfigure
    cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, (int)cudaSharedmemCarveoutMaxShared);
    cudaGetLastError();
    cur = want;
}
template <typename K>
inline void allow_smem(K kernel, size_t bytes) {
    allow_smem_raw(reinterpret_cast<const void*>(kernel), bytes);
}

// Band height of the stage-3 HSZP_ND band scan (recon.cu): one band per plane when there are planes
// enough for two waves of band-scan CTAs (then the z prefix needs no band offsets, which cost it
// ~60% more time); otherwise whole 256-chunk tiles and >= 16 bands-x-planes per SM.
inline int64_t recon_band_rows(int64_t n0, int64_t n1, int64_t n2) {
    if (const char* e = getenv("HSZG_RECON_BR")) {       // A/B runs: force the band height
        const int64_t v = atoll(e);
        if (v > 0) return v < n1 ? v : n1;
    }
    if (n0 >= 2 * 148) return n1 > 0 ? n1 : 1;
    const int64_t cpr = n2 / 32 > 0 ? n2 / 32 : 1;
    const int64_t rpt = TILE_CHUNKS / cpr > 0 ? TILE_CHUNKS / cpr : 1;
    const int64_t want = (16 * 148 + (n0 > 0 ? n0 : 1) - 1) / (n0 > 0 ? n0 : 1);   // bands per plane
    int64_t br = (n1 + want - 1) / want;
    br = (br + rpt - 1) / rpt * rpt;
    return br > 0 ? br : 1;
}

// ---- fast full-chunk decode (K-DEC fast path) -------------------------------------------------
// Tiles of the fused window kernels hold each 32-value chunk in kChunkStride words: 16-byte aligned,
// so a thread writes its chunk with 16-byte shared stores (8 threads of a store phase hit 8
// distinct 4-bank groups: conflict-free) and the row-major write-out reads 16-byte vectors.
constexpr int kChunkStride = 36;
constexpr size_t kFastTileBytes = (size_t)TILE_CHUNKS * kChunkStride * 4;

// Values of G = 4 / 2 / 1 per 32-bit funnel window (bw <= 8 / 16 / 32): one shift + mask per value,
// one bit-cursor advance per group instead of per value, fully unrolled over the chunk's 32 values.
template <int G, bool Prefix, typename Store>
__device__ __forceinline__ uint32_t decode32_g(const uint32_t* w, uint32_t rel, int bw, int32_t add, Store store) {
    const uint32_t smask = smem_u32(w, rel + 1);          // 4 sign bytes, value j <-> bit j
    const uint32_t bitpos = (rel + 5) * 8;
    uint32_t wi = bitpos >> 5, sh = bitpos & 31;
    uint32_t cur = w[wi], nxt = w[wi + 1];
    const uint32_t mask = bw >= 32 ? 0xffffffffu : (1u << bw) - 1u;
    const uint32_t adv = (uint32_t)(G * bw);
    uint32_t run = 0;
#pragma unroll
    for (int q = 0; q < 8; q++) {
        uint32_t v[4];
#pragma unroll
        for (int h = 0; h < 4; h += G) {
            const uint32_t grp = __funnelshift_r(cur, nxt, sh);
#pragma unroll
            for (int i = 0; i < G; i++) {
                const uint32_t mag = (grp >> (i * bw)) & mask;
                v[h + i] = ((smask >> (q * 4 + h + i)) & 1u) ? 0u - mag : mag;
            }
            sh += adv;
            if (sh >= 32) {
                sh -= 32;
                cur = nxt;
                wi++;
                nxt = w[wi + 1];
            }
        }
#pragma unroll
        for (int i = 0; i < 4; i++) {
            run += v[i];
            v[i] = Prefix ? run : v[i] + (uint32_t)add;
        }
        store(q, make_int4((int)v[0], (int)v[1], (int)v[2], (int)v[3]));
    }
    return run;
}

// Decode one validated FULL chunk (32 values) whose bytes start at byte `rel` of the staged words:
// store(g, int4) receives values 4g..4g+3 — the inclusive running sum (Prefix) or value + add.
// Returns the chunk sum mod 2^32.  Same bit layout as decode_chunk_words (_bitpack.pyx:124-143).
// The window width G is chosen per WARP (the widest chunk of the lanes calling it), so lanes with
// different bit-width classes never run two unrolled decodes one after the other; bw = 0 chunks go
// through the G = 4 decode (mask 0) unless the whole warp is zero.
template <bool Prefix, typename Store>
__device__ __forceinline__ uint32_t decode32s(const uint32_t* w, uint32_t rel, int32_t add, Store store) {
    const int bw = (int)smem_byte(w, rel);
    const unsigned act = __activemask();
    if (__all_sync(act, bw == 0)) {
        const int4 c = Prefix ? make_int4(0, 0, 0, 0) : make_int4(add, add, add, add);
#pragma unroll
        for (int q = 0; q < 8; q++) store(q, c);
        return 0;
    }
    if (__all_sync(act, bw <= 8)) return decode32_g<4, Prefix>(w, rel, bw, add, store);
    if (__all_sync(act, bw <= 16)) return decode32_g<2, Prefix>(w, rel, bw, add, store);
    if (bw <= 16) return decode32_g<2, Prefix>(w, rel, bw, add, store);
    return decode32_g<1, Prefix>(w, rel, bw, add, store);
}

// Values 8k .. 8k+7 of a validated FULL chunk (k = 0..3): the bit cursor starts at value 8k
// directly (the bit width is uniform in a chunk), so a chunk splits into 4 independent jobs.
template <int G>
__device__ __forceinline__ void decode8_g(const uint32_t* w, uint32_t rel, int bw, int k, int32_t add, int4& lo,
                                          int4& hi) {
    const uint32_t smask = smem_u32(w, rel + 1) >> (8 * k);
    const uint32_t bitpos = (rel + 5) * 8 + (uint32_t)(8 * k * bw);
    uint32_t wi = bitpos >> 5, sh = bitpos & 31;
    uint32_t cur = w[wi], nxt = w[wi + 1];
    const uint32_t mask = bw >= 32 ? 0xffffffffu : (1u << bw) - 1u;
    const uint32_t adv = (uint32_t)(G * bw);
    uint32_t v[8];
#pragma unroll
    for (int h = 0; h < 8; h += G) {
        const uint32_t grp = __funnelshift_r(cur, nxt, sh);
#pragma unroll
        for (int i = 0; i < G; i++) {
            const uint32_t mag = (grp >> (i * bw)) & mask;
            v[h + i] = (((smask >> (h + i)) & 1u) ? 0u - mag : mag) + (uint32_t)add;
        }
        if (h + G < 8) {
            sh += adv;
            if (sh >= 32) {
                sh -= 32;
                cur = nxt;
                wi++;
                nxt = w[wi + 1];
            }
        }
    }
    lo = make_int4((int)v[0], (int)v[1], (int)v[2], (int)v[3]);
    hi = make_int4((int)v[4], (int)v[5], (int)v[6], (int)v[7]);
}

__device__ __forceinline__ void decode8(const uint32_t* w, uint32_t rel, int k, int32_t add, int4& lo, int4& hi) {
    const int bw = (int)smem_byte(w, rel);
    const unsigned act = __activemask();                 // warp-uniform window width, as decode32s
    if (__all_sync(act, bw == 0)) {
        lo = hi = make_int4(add, add, add, add);
        return;
    }
    if (__all_sync(act, bw <= 8)) return decode8_g<4>(w, rel, bw, k, add, lo, hi);
    if (__all_sync(act, bw <= 16)) return decode8_g<2>(w, rel, bw, k, add, lo, hi);
    if (bw <= 16) return decode8_g<2>(w, rel, bw, k, add, lo, hi);
    return decode8_g<1>(w, rel, bw, k, add, lo, hi);
}

// decode32s into dst[0..32) (16-B aligned) with 16-byte shared stores
template <bool Prefix>
__device__ __forceinline__ uint32_t decode32(const uint32_t* w, uint32_t rel, int32_t* dst, int32_t add) {
    return decode32s<Prefix>(w, rel, add, [&](int q, int4 v) { *reinterpret_cast<int4*>(dst + 4 * q) = v; });
}

// staging bytes (after the fast tile) for a tile of chunks whose widest has max_bw bits
inline size_t stage_bytes(int max_bw) {
    size_t bytes = (size_t)TILE_CHUNKS * (size_t)chunk_bytes(kChunkCap, max_bw) + 64;
    return ((bytes + 15) & ~(size_t)15) + 16;
}

// Stage payload bytes [lo, hi) at 16-B granularity into sb (+ a zero vector after them, read by the
// bit cursor's look-ahead word).  Returns the payload byte mapped to sb[0].  All threads call it.
__device__ __forceinline__ uint64_t stage_range(const uint8_t* payload, uint64_t lo, uint64_t hi, uint4* sb) {
    const uint64_t base = lo & ~(uint64_t)15;
    const uint32_t nvec = (uint32_t)((hi - base + 15) >> 4);
    const uint4* g = reinterpret_cast<const uint4*>(payload + base);
    for (uint32_t i = threadIdx.x; i < nvec; i += blockDim.x) sb[i] = __ldg(g + i);
    if (threadIdx.x == 0) sb[nvec] = make_uint4(0, 0, 0, 0);
    return base;
}

struct TileCtx {
    int64_t c0, c1;      // chunk range
    int64_t e0, e1;      // stream range
    uint64_t base;       // payload byte mapped to smem byte 0 (16-B aligned)
    int32_t* vals;       // padded value tile
    const uint32_t* words;  // staged payload bytes
};

// Stage the tile's payload bytes.  Must be called by all threads of the CTA.
__device__ __forceinline__ TileCtx tile_stage(const SegGeo& sg, const uint8_t* payload, uint64_t len,
                                              const uint64_t* offsets, int64_t tile) {
    extern __shared__ __align__(16) uint8_t tile_smem[];
    __shared__ int64_t s_e0, s_e1;
    __shared__ uint64_t s_lo, s_hi;
    TileCtx t;
    t.c0 = tile * TILE_CHUNKS;
    t.c1 = t.c0 + TILE_CHUNKS < sg.n_chunks ? t.c0 + TILE_CHUNKS : sg.n_chunks;
    if (threadIdx.x == 0) {
        s_lo = offsets[t.c0];
        s_hi = t.c1 < sg.n_chunks ? offsets[t.c1] : payload_end(offsets, sg.n_chunks, len);
        s_e0 = locate_chunk(sg, t.c0).start;
        s_e1 = t.c1 < sg.n_chunks ? locate_chunk(sg, t.c1).start : sg.total;
    }
    __syncthreads();
    t.e0 = s_e0;
    t.e1 = s_e1;
    t.base = s_lo & ~(uint64_t)15;
    const uint64_t nvec = (s_hi - t.base + 15) >> 4;
    t.vals = reinterpret_cast<int32_t*>(tile_smem);
    uint4* sb = reinterpret_cast<uint4*>(tile_smem + (size_t)TILE_VALS * 4);
    const uint4* g = reinterpret_cast<const uint4*>(payload + t.base);
    for (uint64_t i = threadIdx.x; i < nvec; i += blockDim.x) sb[i] = __ldg(g + i);
    if (threadIdx.x == 0) sb[nvec] = make_uint4(0, 0, 0, 0);
    t.words = reinterpret_cast<const uint32_t*>(sb);
    __syncthreads();
    return t;
}

}  // namespace hszg
