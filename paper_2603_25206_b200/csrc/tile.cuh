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

// Opt a tile kernel into > 48 KB of dynamic shared memory (wide bit widths need ~69 KB).  The
// attribute is raised once per kernel to the largest size seen, so steady-state launches (and
// launches under CUDA-graph capture) make no runtime call here.
inline void allow_smem_raw(const void* kernel, size_t bytes) {
    static std::mutex mu;
    static std::unordered_map<const void*, size_t> set;
    if (bytes <= 48 * 1024) return;
    std::lock_guard<std::mutex> lock(mu);
    size_t& cur = set[kernel];
    if (bytes <= cur) return;
    const size_t want = bytes < 96 * 1024 ? 96 * 1024 : bytes;
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)want);
    cur = want;
}
template <typename K>
inline void allow_smem(K kernel, size_t bytes) {
    allow_smem_raw(reinterpret_cast<const void*>(kernel), bytes);
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
