// wtiles.cuh — warp-private staging of 32-chunk tiles for the fused reductions (K-STAT, K-REG).
//
// Each warp owns whole tiles of 32 consecutive chunks (one chunk per lane) and walks them grid-
// strided with no CTA-wide barrier: the tile's contiguous byte range [off[c0], off[c0+32]) (canonical
// index) is copied by one TMA bulk copy into the warp's own shared-memory ring of NS stages, NS - 1
// tiles ahead of the decode; the index entries (and one auxiliary word per chunk, e.g. its block mean)
// are loaded one further tile ahead, so neither the index nor the payload latency sits on the decode
// path, and the staging costs a handful of instructions per 32 values.
#pragma once
#include "async.cuh"
#include "common.cuh"
#include "tile.cuh"

namespace hszg {

#ifndef HSZG_WT_NS
#define HSZG_WT_NS 3
#endif
#ifndef HSZG_WT_MINB_R                    // min resident CTAs for the launch bounds of the warp-tile kernels
#define HSZG_WT_MINB_R 1                  // that stage a shared output tile (recon.cu) ...
#endif
#ifndef HSZG_WT_MINB_S
#define HSZG_WT_MINB_S 4                  // ... and of the reductions (ops.cu): 64 registers, 4 CTAs per SM
#endif
constexpr int WT_NS = HSZG_WT_NS;         // ring stages per warp

// per-warp stage bytes for a stream whose widest chunk has max_bw bits (32 full chunks + alignment
// slack + the bit cursor's zero look-ahead vector)
inline uint32_t wtile_stage_bytes(int max_bw) {
    size_t b = (size_t)32 * (size_t)chunk_bytes(kChunkCap, max_bw) + 16 + 16 + 16;
    return (uint32_t)((b + 15) & ~(size_t)15);
}

// this warp's WT_NS mbarriers, after the 8 warps' stage rings in a 256-thread CTA's dynamic smem
__device__ __forceinline__ uint64_t* wt_bars(uint8_t* smem, uint32_t stage_bytes) {
    return reinterpret_cast<uint64_t*>(smem + (size_t)8 * WT_NS * stage_bytes) + (threadIdx.x >> 5) * WT_NS;
}

struct WtNoAux {
    __device__ __forceinline__ int32_t operator()(int64_t) const { return 0; }
};

// body(c, words, rel, valid, aux): lane's chunk c of the current tile (valid = false past the end);
// all 32 lanes call it every tile.  smem: this warp's WT_NS * stage_bytes bytes (16-B aligned);
// bars: this warp's WT_NS mbarriers.  Lane 0 copies a tile's byte range with one 1-D TMA bulk copy
// (cp.async.bulk, completion on the stage's mbarrier); every lane loads its own index entry (and
// aux word) two tiles ahead.
template <typename Body, typename Aux = WtNoAux>
__device__ __forceinline__ void warp_tiles(const uint8_t* __restrict__ payload, uint64_t len,
                                           const uint64_t* __restrict__ offsets, int64_t n_chunks, uint8_t* smem,
                                           uint32_t stage_bytes, uint64_t* bars, Body body, Aux aux = Aux()) {
    const int lane = threadIdx.x & 31;
    const int64_t wpc = blockDim.x >> 5;
    const int64_t gw = blockIdx.x * wpc + (threadIdx.x >> 5);
    const int64_t nw = gridDim.x * wpc;
    const int64_t tiles = (n_chunks + 31) >> 5;
    struct Ent {
        uint64_t off;     // this lane's chunk start byte
        uint64_t hi;      // lane 0: end of the tile's last chunk
        int32_t aux;
    };
    auto load = [&](int64_t t) {
        Ent e{0, 0, 0};
        if (t < tiles) {
            const int64_t c = (t << 5) + lane;
            if (c < n_chunks) {
                e.off = __ldg(offsets + c);
                e.aux = aux(c);
            }
            if (lane == 0) {
                const int64_t ce = (t << 5) + 32;
                e.hi = ce < n_chunks ? __ldg(offsets + ce) : payload_end(offsets, n_chunks, len);
            }
        }
        return e;
    };
    auto issue = [&](int64_t t, const Ent& e, int stage) {
        if (t < tiles && lane == 0) {
            const uint64_t base = e.off & ~(uint64_t)15;
            const uint32_t bytes = (uint32_t)(((e.hi - base + 15) >> 4) << 4);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // earlier reads of the stage
            mbar_arrive_tx(&bars[stage], bytes);
            tma_load_1d(smem + (size_t)stage * stage_bytes, payload + base, bytes, &bars[stage]);
        }
    };
    int64_t t = gw;
    if (t >= tiles) return;
    // the stages' bytes past a tile are read (masked) by the bit cursor's look-ahead: start them defined
    for (uint32_t i = lane; i < WT_NS * stage_bytes / 16; i += 32)
        reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
    if (lane == 0)
        for (int k = 0; k < WT_NS; k++) mbar_init(&bars[k], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    Ent ring[WT_NS];
#pragma unroll
    for (int k = 0; k < WT_NS; k++) ring[k] = load(t + k * nw);
#pragma unroll
    for (int k = 0; k < WT_NS - 1; k++) issue(t + k * nw, ring[k], k);
    for (int i = 0; t < tiles; t += nw, i++) {
        const int stage = i % WT_NS;
        const Ent cur = ring[0];
        issue(t + (WT_NS - 1) * nw, ring[WT_NS - 1], (i + WT_NS - 1) % WT_NS);
#pragma unroll
        for (int k = 0; k < WT_NS - 1; k++) ring[k] = ring[k + 1];
        ring[WT_NS - 1] = load(t + WT_NS * nw);
        mbar_wait(&bars[stage], (uint32_t)((i / WT_NS) & 1));
        const int64_t c = (t << 5) + lane;
        const bool valid = c < n_chunks;
        const uint64_t base = __shfl_sync(0xffffffffu, cur.off, 0) & ~(uint64_t)15;
        body(c, reinterpret_cast<const uint32_t*>(smem + (size_t)stage * stage_bytes),
             valid ? (uint32_t)(cur.off - base) : 0u, valid, cur.aux);
        __syncwarp();                             // the stage may be refilled next iteration
    }
}

struct MetaAux {       // block mean of chunk c (every segment full: c / cps; cps a power of two: shift)
    const int32_t* meta;
    int64_t cps;
    int shift;         // >= 0: cps == 1 << shift
    __device__ __forceinline__ int32_t operator()(int64_t c) const {
        return __ldg(meta + (shift >= 0 ? (c >> shift) : c / cps));
    }
};

// warp_tiles launches: 256 threads, WT_NS stages per warp, as many CTAs per SM as fit
// (+ extra_per_warp bytes of per-warp scratch after the barriers)
template <typename K>
inline unsigned wtile_grid(K kernel, int max_bw, int64_t n_chunks, size_t* smem_out, uint32_t* stage_out,
                           size_t extra_per_warp = 0) {
    const uint32_t sb = wtile_stage_bytes(max_bw);
    const size_t smem = (size_t)8 * WT_NS * sb + 8 * WT_NS * 8 + 8 * extra_per_warp;
    allow_smem(kernel, smem);
    int per_sm = 1;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, 256, smem) != cudaSuccess || per_sm < 1)
        per_sm = 1;
    cudaGetLastError();
    const int64_t warps = (n_chunks + 31) / 32;
    int64_t grid = (int64_t)148 * per_sm;
    const int64_t need = (warps + 7) / 8;
    if (need < grid) grid = need > 0 ? need : 1;
    *smem_out = smem;
    *stage_out = sb;
    return (unsigned)grid;
}

// this warp's scratch (extra_per_warp bytes, 16-B aligned) after the rings and the barriers
__device__ __forceinline__ uint8_t* wt_scratch(uint8_t* smem, uint32_t stage_bytes, size_t extra_per_warp) {
    return smem + (size_t)8 * WT_NS * stage_bytes + 8 * WT_NS * 8 + (threadIdx.x >> 5) * extra_per_warp;
}

}  // namespace hszg
