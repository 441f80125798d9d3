// lookback.cuh — single-pass decoupled look-back prefix scan (device-wide).
//
// Used for (a) the encoder's exclusive scan of chunk byte sizes into the
// chunk index (_bitpack.pyx:24-51 does it serially) and (b) the HSZP
// stage-3 inclusive scan of residuals across tiles (compressors.py:212).
// Tiles take ids from an atomic ticket so every predecessor is already
// resident when a tile starts waiting on it (no scheduling deadlock).
#pragma once
#include "common.cuh"

namespace hszg {

struct LBState {
    unsigned long long* agg;
    unsigned long long* incl;
    int* flag;                 // 0 = empty, 1 = aggregate published, 2 = inclusive published
    unsigned int* ticket;
};

inline size_t lookback_ws_bytes(int64_t n_tiles_or_items) {
    // sized generously for either use: one state per 256 items is an upper bound on tiles
    const int64_t tiles = n_tiles_or_items / 256 + 2;
    size_t b = 64 + (size_t)tiles * (8 + 8 + 4);
    return (b + 255) & ~(size_t)255;
}

inline LBState lookback_carve(void* ws, int64_t tiles) {
    char* p = reinterpret_cast<char*>(ws);
    LBState s;
    s.ticket = reinterpret_cast<unsigned int*>(p);
    s.agg = reinterpret_cast<unsigned long long*>(p + 64);
    s.incl = s.agg + tiles;
    s.flag = reinterpret_cast<int*>(s.incl + tiles);
    return s;
}

inline size_t lookback_clear_bytes(int64_t tiles) { return 64 + (size_t)tiles * 20; }

// Called by ONE thread of the tile.  Returns the exclusive prefix of this tile.
__device__ __forceinline__ unsigned long long lookback_exclusive(const LBState& st, int64_t tile,
                                                                 unsigned long long agg) {
    volatile int* flag = st.flag;
    volatile unsigned long long* vagg = st.agg;
    volatile unsigned long long* vincl = st.incl;
    if (tile == 0) {
        vincl[0] = agg;
        __threadfence();
        flag[0] = 2;
        return 0ull;
    }
    vagg[tile] = agg;
    __threadfence();
    flag[tile] = 1;
    unsigned long long excl = 0;
    int64_t p = tile - 1;
    while (true) {
        int f;
        do {
            f = flag[p];
        } while (f == 0);
        __threadfence();
        if (f == 2) {
            excl += vincl[p];
            break;
        }
        excl += vagg[p];
        p--;
    }
    vincl[tile] = excl + agg;
    __threadfence();
    flag[tile] = 2;
    return excl;
}

// Called by ALL 32 lanes of one warp of the tile: the same result, but the look-back inspects 32
// predecessors per step (flags loaded in parallel, ballot for the nearest inclusive prefix, warp sum
// of the aggregates before it) instead of walking them one at a time.
__device__ __forceinline__ unsigned long long lookback_exclusive_warp(const LBState& st, int64_t tile,
                                                                      unsigned long long agg) {
    const int lane = threadIdx.x & 31;
    volatile int* flag = st.flag;
    volatile unsigned long long* vagg = st.agg;
    volatile unsigned long long* vincl = st.incl;
    if (tile == 0) {
        if (lane == 0) {
            vincl[0] = agg;
            __threadfence();
            flag[0] = 2;
        }
        return 0ull;
    }
    if (lane == 0) {
        vagg[tile] = agg;
        __threadfence();
        flag[tile] = 1;
    }
    unsigned long long excl = 0;
    int64_t p = tile - 1;
    while (true) {
        const int64_t idx = p - lane;
        const int f = idx >= 0 ? flag[idx] : 2;          // before tile 0: an inclusive prefix of 0
        const unsigned incl = __ballot_sync(0xffffffffu, f == 2);
        const unsigned zero = __ballot_sync(0xffffffffu, f == 0);
        const int k = incl ? __ffs(incl) - 1 : 31;      // nearest inclusive, else the whole window
        const unsigned need = (2u << k) - 1u;            // lanes 0..k (k = 31: all)
        if (zero & need) continue;                       // an aggregate in between is not out yet
        __threadfence();
        unsigned long long v = 0;
        if (lane <= k && idx >= 0) v = (lane == k && incl) ? vincl[idx] : vagg[idx];
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
        excl += v;
        if (incl) break;
        p -= 32;
    }
    if (lane == 0) {
        vincl[tile] = excl + agg;
        __threadfence();
        flag[tile] = 2;
    }
    return excl;
}

// 32-bit variant for scans mod 2^32 (the int32 q prefixes): the status flag and the value share one
// 64-bit word (bits 62-63 flag, low 32 bits value), published with a single 64-bit store, so readers
// need no fence between the flag and the value (the u64 version above fences every publication,
// which stalls behind the tile's streaming stores).  Uses st.agg as the word array.
__device__ __forceinline__ uint32_t lookback_exclusive_warp32(const LBState& st, int64_t tile, uint32_t agg) {
    const int lane = threadIdx.x & 31;
    volatile unsigned long long* w = st.agg;
    const unsigned long long AGG = 1ull << 62, INCL = 2ull << 62;
    if (lane == 0) w[tile] = (tile == 0 ? INCL : AGG) | agg;
    if (tile == 0) return 0u;
    uint32_t excl = 0;
    int64_t p = tile - 1;
    while (true) {
        const int64_t idx = p - lane;
        const unsigned long long v = idx >= 0 ? w[idx] : INCL;   // before tile 0: inclusive 0
        const unsigned f = (unsigned)(v >> 62);
        const unsigned incl = __ballot_sync(0xffffffffu, f == 2);
        const unsigned zero = __ballot_sync(0xffffffffu, f == 0);
        const int k = incl ? __ffs(incl) - 1 : 31;
        const unsigned need = (2u << k) - 1u;
        if (zero & need) continue;
        uint32_t x = lane <= k ? (uint32_t)v : 0u;
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) x += __shfl_xor_sync(0xffffffffu, x, d);
        excl += x;
        if (incl) break;
        p -= 32;
    }
    if (lane == 0) w[tile] = INCL | (uint32_t)(excl + agg);
    return excl;
}

// 62-bit variant (byte offsets): flag in bits 62-63, value in the low 62 bits, one 64-bit store per
// publication and no fences (the single-copy atomic word carries flag and value together).
__device__ __forceinline__ unsigned long long lookback_exclusive_warp62(const LBState& st, int64_t tile,
                                                                        unsigned long long agg) {
    const int lane = threadIdx.x & 31;
    volatile unsigned long long* w = st.agg;
    const unsigned long long AGG = 1ull << 62, INCL = 2ull << 62, VAL = (1ull << 62) - 1;
    if (lane == 0) w[tile] = (tile == 0 ? INCL : AGG) | agg;
    if (tile == 0) return 0ull;
    unsigned long long excl = 0;
    int64_t p = tile - 1;
    while (true) {
        const int64_t idx = p - lane;
        const unsigned long long v = idx >= 0 ? w[idx] : INCL;   // before tile 0: inclusive 0
        const unsigned f = (unsigned)(v >> 62);
        const unsigned incl = __ballot_sync(0xffffffffu, f == 2);
        const unsigned zero = __ballot_sync(0xffffffffu, f == 0);
        const int k = incl ? __ffs(incl) - 1 : 31;
        const unsigned need = (2u << k) - 1u;
        if (zero & need) continue;
        unsigned long long x = lane <= k ? (v & VAL) : 0ull;
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) x += __shfl_xor_sync(0xffffffffu, x, d);
        excl += x;
        if (incl) break;
        p -= 32;
    }
    if (lane == 0) w[tile] = INCL | (excl + agg);
    return excl;
}

// block-wide exclusive scan of one u64 per thread; returns exclusive value, *total = block sum
__device__ __forceinline__ unsigned long long block_exclusive_u64(unsigned long long v, unsigned long long* total) {
    __shared__ unsigned long long warp_tot[32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    unsigned long long x = v;
    for (int d = 1; d < 32; d <<= 1) {
        unsigned long long y = __shfl_up_sync(0xffffffffu, x, d);
        if (lane >= d) x += y;
    }
    if (lane == 31) warp_tot[wid] = x;
    __syncthreads();
    if (wid == 0) {
        const int nw = blockDim.x >> 5;
        unsigned long long t = lane < nw ? warp_tot[lane] : 0ull;
        for (int d = 1; d < 32; d <<= 1) {
            unsigned long long y = __shfl_up_sync(0xffffffffu, t, d);
            if (lane >= d) t += y;
        }
        if (lane < nw) warp_tot[lane] = t;  // inclusive warp totals
    }
    __syncthreads();
    const unsigned long long warp_excl = wid ? warp_tot[wid - 1] : 0ull;
    *total = warp_tot[(blockDim.x >> 5) - 1];
    __syncthreads();
    return warp_excl + x - v;
}

constexpr int SCAN_THREADS = 256;
constexpr int SCAN_ITEMS = 8;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;

static __global__ void __launch_bounds__(SCAN_THREADS) k_scan_u64(const uint64_t* in, uint64_t* out, int64_t n,
                                                           LBState st, uint64_t* total) {
    __shared__ unsigned int s_tile;
    __shared__ unsigned long long s_prefix;
    if (threadIdx.x == 0) s_tile = atomicAdd(st.ticket, 1u);
    __syncthreads();
    const int64_t tile = s_tile;
    const int64_t base = tile * SCAN_TILE + (int64_t)threadIdx.x * SCAN_ITEMS;
    unsigned long long v[SCAN_ITEMS];
    unsigned long long run = 0;
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; k++) {
        const int64_t i = base + k;
        v[k] = i < n ? in[i] : 0ull;
        run += v[k];
    }
    unsigned long long tot;
    const unsigned long long texcl = block_exclusive_u64(run, &tot);
    if (threadIdx.x < 32) {
        const unsigned long long e = lookback_exclusive_warp(st, tile, tot);
        if (threadIdx.x == 0) s_prefix = e;
    }
    __syncthreads();
    unsigned long long acc = s_prefix + texcl;
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; k++) {
        const int64_t i = base + k;
        if (i < n) out[i] = acc;
        acc += v[k];
    }
    if (total && base <= n - 1 && base + SCAN_ITEMS >= n) *total = acc;
}

// exclusive scan; `total` (device) receives the sum.  In-place allowed.
static inline int exclusive_scan_u64(const uint64_t* in, uint64_t* out, int64_t n, uint64_t* total, void* ws,
                              cudaStream_t st) {
    const int64_t tiles = (n + SCAN_TILE - 1) / SCAN_TILE;
    LBState s = lookback_carve(ws, tiles);
    cudaMemsetAsync(ws, 0, lookback_clear_bytes(tiles), st);
    if (tiles == 0) return 0;
    k_scan_u64<<<(unsigned)tiles, SCAN_THREADS, 0, st>>>(in, out, n, s, total);
    return cudaGetLastError() != cudaSuccess;
}

}  // namespace hszg
