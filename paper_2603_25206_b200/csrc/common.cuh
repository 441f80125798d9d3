// common.cuh — shared device code for libhszg (sm_100a).
//
// Stream geometry.  Every HSZ compressor kind streams its values as a
// sequence of "segments" (compressors.py:105-119): 1-D blocks (HSZP/HSZX),
// axis-0 rows/planes (HSZP_ND) or nd blocks (HSZX_ND); chunks of <= 32
// values restart at every segment (codec.py:96-106).  All four are the same
// object once the field is viewed as a 3-D box [n0][n1][n2] tiled by
// segments [B0][B1][B2] listed in row-major segment order with row-major
// elements inside each segment (grid.py:114-128):
//     HSZP, HSZX : box (1,1,N)       segments (1,1,S)
//     HSZP_ND    : box (n0,n1,n2)    segments (1,n1,n2)   (2-D: (1,n0,n1) / (1,1,n1))
//     HSZX_ND    : box (n0,n1,n2)    segments (B0,B1,B2)  (2-D: (1,n0,n1) / (1,B0,B1))
// Segment sizes only take two values per axis (full / edge), so chunk and
// element offsets of any segment are closed-form (SegGeo below): no span
// table is ever materialised on the device.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "../../include/hszg.h"

#define HSZG_HD __host__ __device__ __forceinline__

namespace hszg {

constexpr int kChunkCap = 32;                 // codec.py:20
constexpr int32_t kQmax = 2147483646;         // quant.py:19
constexpr int64_t kPmax = 2147483647LL;       // compressors.py:22

struct SegGeo {
    int64_t n[3];       // box dims
    int64_t B[3];       // full segment extents
    int64_t G[3];       // segment grid
    int64_t E[3];       // edge segment extents
    int64_t cpb[8];     // chunks per segment, index (c0<<2)|(c1<<1)|c2, c = "is edge"
    int64_t rowc[4];    // chunks per segment-row, index (c0<<1)|c1
    int64_t planec[2];  // chunks per segment-plane, index c0
    int64_t n_chunks;
    int64_t total;
};

HSZG_HD int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

inline SegGeo make_seggeo(const HszgGeom& g) {
    SegGeo s;
    for (int a = 0; a < 3; a++) {
        s.n[a] = g.sdims[a];
        s.B[a] = g.sblk[a];
        s.G[a] = g.sgrid[a];
        s.E[a] = s.n[a] - (s.G[a] - 1) * s.B[a];
    }
    for (int c0 = 0; c0 < 2; c0++)
        for (int c1 = 0; c1 < 2; c1++)
            for (int c2 = 0; c2 < 2; c2++) {
                int64_t sz = (c0 ? s.E[0] : s.B[0]) * (c1 ? s.E[1] : s.B[1]) * (c2 ? s.E[2] : s.B[2]);
                s.cpb[(c0 << 2) | (c1 << 1) | c2] = ceil_div(sz, kChunkCap);
            }
    for (int c0 = 0; c0 < 2; c0++)
        for (int c1 = 0; c1 < 2; c1++)
            s.rowc[(c0 << 1) | c1] = (s.G[2] - 1) * s.cpb[(c0 << 2) | (c1 << 1)] + s.cpb[(c0 << 2) | (c1 << 1) | 1];
    for (int c0 = 0; c0 < 2; c0++)
        s.planec[c0] = (s.G[1] - 1) * s.rowc[c0 << 1] + s.rowc[(c0 << 1) | 1];
    s.n_chunks = (s.G[0] - 1) * s.planec[0] + s.planec[1];
    s.total = s.n[0] * s.n[1] * s.n[2];
    return s;
}

HSZG_HD int64_t seg_ext(const SegGeo& s, int a, int64_t b) { return b == s.G[a] - 1 ? s.E[a] : s.B[a]; }

// element (stream) offset of segment (b0,b1,b2)
HSZG_HD int64_t seg_elem_start(const SegGeo& s, int64_t b0, int64_t b1, int64_t b2) {
    int64_t s0 = seg_ext(s, 0, b0), s1 = seg_ext(s, 1, b1);
    return b0 * s.B[0] * s.n[1] * s.n[2] + b1 * s0 * s.B[1] * s.n[2] + b2 * s0 * s1 * s.B[2];
}

// first chunk of segment (b0,b1,b2)
HSZG_HD int64_t seg_chunk_start(const SegGeo& s, int64_t b0, int64_t b1, int64_t b2) {
    int c0 = b0 == s.G[0] - 1, c1 = b1 == s.G[1] - 1;
    return b0 * s.planec[0] + b1 * s.rowc[c0 << 1] + b2 * s.cpb[(c0 << 2) | (c1 << 1)];
}

struct ChunkLoc {
    int64_t seg;     // linear segment index (row-major) = metadata index
    int64_t start;   // stream position of the chunk's first value
    int32_t count;   // values in the chunk
    int32_t j;       // chunk ordinal inside its segment
};

// chunk index -> segment, stream start and count (inverse of the prefix above)
HSZG_HD ChunkLoc locate_chunk(const SegGeo& s, int64_t c) {
    int64_t b0 = 0, r = c;
    if (s.G[0] > 1) {
        b0 = r / s.planec[0];
        if (b0 > s.G[0] - 1) b0 = s.G[0] - 1;
        r -= b0 * s.planec[0];
    }
    int c0 = b0 == s.G[0] - 1;
    int64_t b1 = 0;
    if (s.G[1] > 1) {
        int64_t rc = s.rowc[c0 << 1];
        b1 = r / rc;
        if (b1 > s.G[1] - 1) b1 = s.G[1] - 1;
        r -= b1 * rc;
    }
    int c1 = b1 == s.G[1] - 1;
    int64_t b2 = 0;
    if (s.G[2] > 1) {
        int64_t cb = s.cpb[(c0 << 2) | (c1 << 1)];
        b2 = r / cb;
        if (b2 > s.G[2] - 1) b2 = s.G[2] - 1;
        r -= b2 * cb;
    }
    int64_t size = seg_ext(s, 0, b0) * seg_ext(s, 1, b1) * seg_ext(s, 2, b2);
    ChunkLoc L;
    L.seg = (b0 * s.G[1] + b1) * s.G[2] + b2;
    L.j = (int32_t)r;
    L.start = seg_elem_start(s, b0, b1, b2) + r * kChunkCap;
    int64_t left = size - r * kChunkCap;
    L.count = (int32_t)(left < kChunkCap ? left : kChunkCap);
    return L;
}

// End of the stream's last chunk.  A plane view of a larger resident stream (sub-range of
// its chunk index) passes payload_len with the top bit set: the end is then the parent
// index entry just past the view, offsets[n_chunks] — no host round trip to look it up.
constexpr uint64_t kEndInIndex = 1ull << 63;
__device__ __forceinline__ uint64_t payload_end(const uint64_t* offsets, int64_t n_chunks, uint64_t len) {
    return (len & kEndInIndex) ? offsets[n_chunks] : len;
}

// byte size of a chunk (_fallback.py:52-55)
HSZG_HD int64_t chunk_bytes(int64_t count, int bw) {
    return bw == 0 ? 1 : 1 + (count + 7) / 8 + (count * bw + 7) / 8;
}

// ---- small helpers ---------------------------------------------------------

__device__ __forceinline__ uint32_t smem_byte(const uint32_t* w, uint32_t i) {
    return (w[i >> 2] >> ((i & 3) * 8)) & 0xffu;
}
// little-endian u32 starting at byte i of a word array
__device__ __forceinline__ uint32_t smem_u32(const uint32_t* w, uint32_t i) {
    return __funnelshift_r(w[i >> 2], w[(i >> 2) + 1], (i & 3) * 8);
}

// Lane-serial decode of one validated chunk whose bytes start at byte `rel`
// of the word array `w` (shared or global).  Calls emit(j, value) for
// j = 0..count-1.  Layout: _fallback.py:1-8; bit loop: _bitpack.pyx:124-143.
template <typename Emit>
__device__ __forceinline__ void decode_chunk_words(const uint32_t* w, uint32_t rel, int count, Emit emit) {
    const int bw = (int)smem_byte(w, rel);
    if (bw == 0) {
        for (int j = 0; j < count; j++) emit(j, 0);
        return;
    }
    uint32_t smask = smem_u32(w, rel + 1);
    const uint32_t sb = (uint32_t)((count + 7) >> 3);
    uint32_t bitpos = (rel + 1 + sb) * 8;
    uint32_t wi = bitpos >> 5;
    uint32_t sh = bitpos & 31;
    uint32_t cur = w[wi], nxt = w[wi + 1];
    const uint32_t mask = bw == 32 ? 0xffffffffu : ((1u << bw) - 1u);
    for (int j = 0; j < count; j++) {
        uint32_t mag = __funnelshift_r(cur, nxt, sh) & mask;
        sh += bw;
        if (sh >= 32) {
            sh -= 32;
            cur = nxt;
            wi++;
            nxt = w[wi + 1];
        }
        int32_t v = (int32_t)mag;
        v = ((smask >> j) & 1u) ? -v : v;
        emit(j, v);
    }
}

// ---- reductions ---------------------------------------------------------------

typedef __int128 i128;
typedef unsigned __int128 u128;

__device__ __forceinline__ i128 shfl_down_i128(i128 v, int d) {
    uint64_t lo = (uint64_t)v, hi = (uint64_t)((u128)v >> 64);
    lo = __shfl_down_sync(0xffffffffu, lo, d);
    hi = __shfl_down_sync(0xffffffffu, hi, d);
    return (i128)(((u128)hi << 64) | lo);
}

struct Acc {
    i128 s1, s2;
    int64_t count;
    int32_t vmin, vmax;
    double f1, f2;
    __device__ __forceinline__ void init() {
        s1 = 0; s2 = 0; count = 0; vmin = INT32_MAX; vmax = INT32_MIN; f1 = 0.0; f2 = 0.0;
    }
    __device__ __forceinline__ void merge(const Acc& o) {
        s1 += o.s1; s2 += o.s2; count += o.count;
        vmin = min(vmin, o.vmin); vmax = max(vmax, o.vmax);
        f1 += o.f1; f2 += o.f2;
    }
};

__device__ __forceinline__ void warp_reduce(Acc& a) {
    for (int d = 16; d > 0; d >>= 1) {
        Acc o;
        o.s1 = shfl_down_i128(a.s1, d);
        o.s2 = shfl_down_i128(a.s2, d);
        o.count = __shfl_down_sync(0xffffffffu, a.count, d);
        o.vmin = __shfl_down_sync(0xffffffffu, a.vmin, d);
        o.vmax = __shfl_down_sync(0xffffffffu, a.vmax, d);
        o.f1 = __shfl_down_sync(0xffffffffu, a.f1, d);
        o.f2 = __shfl_down_sync(0xffffffffu, a.f2, d);
        a.merge(o);
    }
}

// block-wide reduction; result valid in thread 0.  blockDim.x multiple of 32, <= 1024.
__device__ __forceinline__ void block_reduce(Acc& a) {
    __shared__ Acc part[32];
    warp_reduce(a);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) part[wid] = a;
    __syncthreads();
    if (wid == 0) {
        const int nw = blockDim.x >> 5;
        if (lane < nw) a = part[lane];
        else a.init();
        warp_reduce(a);
    }
}

__device__ __forceinline__ void store_sums(HszgSums* out, const Acc& a) {
    out->s1_lo = (uint64_t)a.s1;
    out->s1_hi = (int64_t)(a.s1 >> 64);
    out->s2_lo = (uint64_t)a.s2;
    out->s2_hi = (int64_t)(a.s2 >> 64);
    out->count = a.count;
    out->vmin = a.vmin;
    out->vmax = a.vmax;
    out->f1 = a.f1;
    out->f2 = a.f2;
}

__device__ __forceinline__ Acc load_sums(const HszgSums* in) {
    Acc a;
    a.s1 = (i128)(((u128)(uint64_t)in->s1_hi << 64) | in->s1_lo);
    a.s2 = (i128)(((u128)(uint64_t)in->s2_hi << 64) | in->s2_lo);
    a.count = in->count;
    a.vmin = in->vmin;
    a.vmax = in->vmax;
    a.f1 = in->f1;
    a.f2 = in->f2;
    return a;
}

inline int grid_for(int64_t work, int per_block, int cap = 148 * 32) {
    int64_t g = (work + per_block - 1) / per_block;
    if (g < 1) g = 1;
    if (g > cap) g = cap;
    return (int)g;
}

}  // namespace hszg
