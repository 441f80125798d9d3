// compress.cu — one-pass GPU compress (K-ENC fused, §8 rows E2–E5): fp32 field -> quantize
// (quant.py:69-82) -> decorrelate (compressors.py:149-198) -> chunk bit widths and sizes
// (_bitpack.pyx:24-51) -> chunk byte offsets (tile-local scan + decoupled look-back) -> packed chunk
// bytes (_bitpack.pyx:53-87), in ONE kernel: neither q nor p ever reaches HBM.  The multi-kernel path
// (encode.cu + codec.cu: quantize, decorrelate_sized, scan, pack) moves ≈ 20 + P B/value; this one
// reads the field once (4 B/value, the Lorenzo neighbour rows from L2) and writes P + I.
//
// A tile = 256 whole chunks of the stream (one per thread), its id drawn from an atomic ticket so every
// predecessor tile is already resident when it waits in the look-back (lookback.cuh):
//   front   the tile's values, quantized and decorrelated, into a shared p tile (chunk c = row c, stride 36
//           words) — per kind below;
//   sizes   each thread's chunk: bit width of max |p|, 1 + 4 + 4 bw bytes (1 if bw = 0);
//   offsets CTA exclusive scan of the sizes, warp 0 looks back for the tile's byte base; chunk index out;
//   pack    each thread packs its chunk (bw byte, sign bitmap, LSB-first magnitudes) into a shared staging
//           copy of the tile's byte range [base, base + total), which the CTA stores with aligned 16-B
//           vectors (byte stores only at the two edges it shares with its neighbours).
// Fronts (every chunk full: the stream is a sequence of 32-value groups):
//   CF_PREV     HSZP: p = diff(flat q, prepend 0); the value before a float4 group comes from the previous
//               lane (lane 0: quantized from the field).
//   CF_LORENZO  HSZP_ND (box n0 x n1 x n2, n2 % 32 == 0, n2 <= 8192): a tile = R = 8192 / n2 whole rows;
//               p = x-differences of the rows (z,y) - (z,y-1) - (z-1,y) + (z-1,y-1), each neighbour row
//               quantized again from the field (L2-resident: the previous plane was read a plane ago).
//   CF_BLOCKS   HSZX / HSZX_ND with full blocks (B0,B1,B2), B2 % 4 == 0, 32 | |block| <= 8192: a tile =
//               kb = 8192 / |block| blocks along x; q staged in stream order, the block's truncated integer
//               mean (compressors.py:134-138) from per-chunk partial sums (shared 64-bit atomics), p = q - M.
#include <cstdio>
#include "common.cuh"
#include "lookback.cuh"

namespace hszg {

#ifndef CF_TILE
#define CF_TILE 256
#endif
constexpr int CF_T = CF_TILE;                   // threads = chunks per tile
constexpr int CF_S = 36;                        // p tile row stride in words (conflict-free 16-B reads)
constexpr int CF_VALS = CF_T * kChunkCap;       // 8192 values per tile
constexpr int CF_MAXCB = 1 + 4 + 4 * 32;        // largest full chunk in bytes
constexpr size_t CF_PBYTES = (size_t)CF_T * CF_S * 4;
constexpr size_t CF_SMEM = CF_PBYTES + (size_t)CF_T * CF_MAXCB + 32;
enum { CF_PREV = 0, CF_LORENZO = 1, CF_BLOCKS = 2 };

struct CfArgs {
    const float* x;
    int64_t n;                                  // values
    double recip;                               // 1 / (2 eps)
    float vlim;                                 // |d| <= vlim => |d * recip + 0.5| < 2^28 (fast quantize)
    int64_t N0, N1, N2;                         // box dims
    int64_t rows_per_tile;                      // CF_LORENZO
    SegGeo sg;                                  // CF_BLOCKS
    int64_t tpr;                                // CF_BLOCKS: tiles per block row
    int kb;                                     // CF_BLOCKS: blocks per tile
    int64_t n_chunks, n_tiles;
    uint8_t* payload;
    uint64_t* offsets;
    int32_t* meta;
    LBState lb;
    unsigned int* flags;                        // bit 0 |index| > Qmax, bit 1 NaN, bit 2 residual overflow
    unsigned long long* total;                  // payload length (written by the last tile)
};

// quant.py:69-82: floor(d * recip + 0.5) in fp64, multiply and add rounded separately (no FMA); the floor is
// an add of 1.5 * 2^52 rounded toward -inf, whose low word is floor(t) mod 2^32 for |t| < 2^51.
//   cf_qf  fast form, valid when |d| <= vlim (the host's bound for |t| < 2^28): no range checks;
//   cf_q   exact form with the reference's range check (bit 0 |q| > QMAX / Inf, bit 1 NaN).
__device__ __forceinline__ int32_t cf_qf(float v, double recip) {
    return __double2loint(__dadd_rd(__dadd_rn(__dmul_rn((double)v, recip), 0.5), 6755399441055744.0));
}
__device__ __forceinline__ int32_t cf_q(float v, double recip, unsigned int& f) {
    const double t = __dadd_rn(__dmul_rn((double)v, recip), 0.5);
    const long long b = __double_as_longlong(__dadd_rd(t, 6755399441055744.0)) - 0x4338000000000000LL;
    if (b > kQmax || b < -(long long)kQmax) {
        f |= (v != v) ? 2u : 1u;
        return 0;
    }
    return (int32_t)b;
}
__device__ __forceinline__ int4 cf_q4(float4 v, double recip, unsigned int& f) {
    return make_int4(cf_q(v.x, recip, f), cf_q(v.y, recip, f), cf_q(v.z, recip, f), cf_q(v.w, recip, f));
}
__device__ __forceinline__ int4 cf_qf4(float4 v, double recip) {
    return make_int4(cf_qf(v.x, recip), cf_qf(v.y, recip), cf_qf(v.z, recip), cf_qf(v.w, recip));
}
// NaN-safe "outside the fast range": !(|v| <= vlim)
__device__ __forceinline__ bool cf_big(float4 v, float vlim) {
    return !(fabsf(v.x) <= vlim && fabsf(v.y) <= vlim && fabsf(v.z) <= vlim && fabsf(v.w) <= vlim);
}
__device__ __forceinline__ int32_t cf_res(int64_t d, unsigned int& f) {
    if (d > kPmax || d < -kPmax) f |= 4u;
    return (int32_t)d;
}
__device__ __forceinline__ int32_t* cf_slot(int32_t* P, int64_t e) {   // tile element e (stream order)
    return P + (e >> 5) * CF_S + (e & 31);
}

template <int FRONT>
__global__ void __launch_bounds__(CF_T, 768 / CF_T) k_compress_tiles(CfArgs a) {
    extern __shared__ __align__(16) uint8_t smem[];
    int32_t* P = reinterpret_cast<int32_t*>(smem);
    uint8_t* SB = smem + CF_PBYTES;
    __shared__ unsigned int s_tile;
    __shared__ unsigned long long s_base;
    __shared__ uint32_t s_wsum[CF_T / 32];
    __shared__ long long s_bsum[CF_T];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_tile = atomicAdd(a.lb.ticket, 1u);
    if (FRONT == CF_BLOCKS) s_bsum[threadIdx.x] = 0;
    for (int i = threadIdx.x; i < (int)((CF_SMEM - CF_PBYTES) / 16); i += CF_T)      // staging words are OR-ed
        reinterpret_cast<int4*>(SB)[i] = make_int4(0, 0, 0, 0);
    __syncthreads();
    const int64_t tile = s_tile;
    const double recip = a.recip;
    const float vlim = a.vlim;
    unsigned int f = 0;
    int64_t c0;                                  // first chunk of the tile
    int nch;                                     // chunks in the tile

    // ================================ front: p tile ================================
    if (FRONT == CF_PREV) {
        const int64_t e0 = tile * CF_VALS;
        const int64_t nv = a.n - e0 < CF_VALS ? a.n - e0 : CF_VALS;
        c0 = tile * CF_T;
        nch = (int)(nv >> 5);
        const int n4 = (int)(nv >> 2);
        const float4* x4 = reinterpret_cast<const float4*>(a.x + e0);
        constexpr int NI = CF_VALS / 4 / CF_T;                       // 8 float4 per thread, all in flight
        float4 vv[NI];
        float vps[NI];
#pragma unroll
        for (int j = 0; j < NI; j++) {
            const int i = (int)threadIdx.x + j * CF_T;
            vv[j] = i < n4 ? __ldg(x4 + i) : make_float4(0.f, 0.f, 0.f, 0.f);
            vps[j] = (lane == 0 && i < n4 && e0 + 4 * i > 0) ? __ldg(a.x + e0 + 4 * i - 1) : 0.f;
        }
#pragma unroll
        for (int j = 0; j < NI; j++) {
            const int i = (int)threadIdx.x + j * CF_T;
            const bool act = i < n4;
            const float4 v = vv[j];
            const float vp = vps[j];
            if (!__any_sync(0xffffffffu, cf_big(v, vlim) || !(fabsf(vp) <= vlim))) {
                const int4 q = cf_qf4(v, recip);                      // |q| < 2^28: int32 differences exact
                int prev = __shfl_up_sync(0xffffffffu, q.w, 1);
                if (lane == 0) prev = cf_qf(vp, recip);
                if (act)
                    *reinterpret_cast<int4*>(cf_slot(P, 4 * i)) = make_int4(q.x - prev, q.y - q.x, q.z - q.y, q.w - q.z);
            } else {                                                  // exact: range checks, int64 residuals
                const int4 q = act ? cf_q4(v, recip, f) : make_int4(0, 0, 0, 0);
                int prev = __shfl_up_sync(0xffffffffu, q.w, 1);
                if (lane == 0) prev = (act && e0 + 4 * i > 0) ? cf_q(vp, recip, f) : 0;
                if (act)
                    *reinterpret_cast<int4*>(cf_slot(P, 4 * i)) =
                        make_int4(cf_res((int64_t)q.x - prev, f), cf_res((int64_t)q.y - q.x, f),
                                  cf_res((int64_t)q.z - q.y, f), cf_res((int64_t)q.w - q.z, f));
            }
        }
    } else if (FRONT == CF_LORENZO) {
        // thread = one float4 column of a row segment, sliding down its rows: per row it quantizes (z, y)
        // and (z-1, y) and keeps their x-differences for the next row's (y-1) terms (~2.25 quantizations
        // per value: a segment's first row also needs row y-1 of both planes).  Fast rows (every value of
        // the warp's rows within vlim: |q| < 2^28) in int32; otherwise the row is recomputed exactly from
        // its four rows with range checks and int64 sums.
        const int64_t R = a.rows_per_tile, N1 = a.N1, N2 = a.N2;
        const int64_t NR = a.N0 * N1;
        const int64_t r0 = tile * R;
        const int nr = (int)(NR - r0 < R ? NR - r0 : R);
        const int cpr = (int)(N2 >> 5), G = (int)(N2 >> 2);
        c0 = r0 * cpr;
        nch = nr * cpr;
        const int64_t plane = N1 * N2;
        const int S = G >= CF_T ? 1 : CF_T / G;                    // row segments
        const int rps = (nr + S - 1) / S;                           // rows per segment (uniform)
        const int seg = G >= CF_T ? 0 : (int)threadIdx.x / G;
        const int col = G >= CF_T ? (int)threadIdx.x : (int)threadIdx.x - seg * G;
        const int rs = seg * rps;                                   // the segment's first tile row
        const int64_t z0 = r0 / N1, y0 = r0 - z0 * N1;              // once per tile
        const int4 z4 = make_int4(0, 0, 0, 0);
        const float4 f4 = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int cb = 0; cb < G; cb += CF_T) {                      // column blocks (G > 256: several)
            const int c = col + cb;
            const bool cact = seg < S && c < G;
            int4 dz_prev = z4, dzm_prev = z4;                        // x-diffs of rows (z, y-1), (z-1, y-1)
            bool prev_fast = false;
            // row k's (z, y), whether it exists, and its loads; issued one row ahead
            struct Row {
                int64_t z, y;
                bool act, rowok;
                const float* p;
                float4 va, vb;
                float la, lb;
            };
            auto fetch = [&](int k) {
                Row w;
                const int rr = rs + k;
                w.act = cact && rr < nr && r0 + rr >= 0;
                w.z = z0;
                w.y = y0 + rr;                                       // rr >= -1
                if (w.y < 0) {
                    w.z -= 1;
                    w.y += N1;
                } else if (w.y >= N1) {                              // the tile crosses a plane (rare)
                    const int64_t kk = w.y / N1;
                    w.z += kk;
                    w.y -= kk * N1;
                }
                w.rowok = w.act && w.z >= 0;
                const bool hz_ = w.z > 0;
                w.p = a.x + (w.z * N1 + w.y) * N2;
                w.va = w.rowok ? __ldg(reinterpret_cast<const float4*>(w.p) + c) : f4;
                w.vb = w.rowok && hz_ ? __ldg(reinterpret_cast<const float4*>(w.p - plane) + c) : f4;
                w.la = w.lb = 0.f;
                if (lane == 0 && c > 0 && w.rowok) {
                    w.la = __ldg(w.p + 4 * c - 1);
                    if (hz_) w.lb = __ldg(w.p - plane + 4 * c - 1);
                }
                return w;
            };
            Row nxt = fetch(-1);
            for (int k = -1; k < rps; k++) {                         // k = -1: the segment's halo row y-1
                const Row cur = nxt;
                if (k + 1 < rps) nxt = fetch(k + 1);
                const int rr = rs + k;
                const bool act = cur.act, rowok = cur.rowok, hz = cur.z > 0;
                const int64_t y = cur.y;
                const float* rowp = cur.p;
                const float4 va = cur.va, vb = cur.vb;
                const float la = cur.la, lb = cur.lb;
                const bool fast = !__any_sync(0xffffffffu, cf_big(va, vlim) || cf_big(vb, vlim) ||
                                                               !(fabsf(la) <= vlim) || !(fabsf(lb) <= vlim));
                int4 dz = z4, dzm = z4;
                if (fast) {
                    const int4 qa = cf_qf4(va, recip), qb = cf_qf4(vb, recip);
                    int pa = __shfl_up_sync(0xffffffffu, qa.w, 1), pb = __shfl_up_sync(0xffffffffu, qb.w, 1);
                    if (c == 0) pa = pb = 0;
                    else if (lane == 0) {
                        pa = cf_qf(la, recip);
                        pb = cf_qf(lb, recip);
                    }
                    dz = make_int4(qa.x - pa, qa.y - qa.x, qa.z - qa.y, qa.w - qa.z);
                    dzm = make_int4(qb.x - pb, qb.y - qb.x, qb.z - qb.y, qb.w - qb.z);
                }
                if (k >= 0) {
                    const bool hy = y > 0;
                    // warp-uniform (a warp may span row segments): |x-diff| < 2^29, the sum fits int32
                    if (fast && __all_sync(0xffffffffu, prev_fast || !hy)) {
                        if (act) {
                            const int4 pz = hy ? dz_prev : z4, pzm = hy ? dzm_prev : z4;
                            *reinterpret_cast<int4*>(cf_slot(P, (int64_t)rr * N2 + 4 * c)) =
                                make_int4(dz.x - pz.x - dzm.x + pzm.x, dz.y - pz.y - dzm.y + pzm.y,
                                          dz.z - pz.z - dzm.z + pzm.z, dz.w - pz.w - dzm.w + pzm.w);
                        }
                    } else {                                          // exact from the four rows
                        const float* rows[4] = {rowp, rowp - N2, rowp - plane, rowp - plane - N2};
                        const bool has[4] = {rowok, rowok && hy, rowok && hz, rowok && hy && hz};
                        int64_t acc[4] = {0, 0, 0, 0};
#pragma unroll
                        for (int t = 0; t < 4; t++) {
                            const int4 q = has[t] ? cf_q4(__ldg(reinterpret_cast<const float4*>(rows[t]) + c), recip, f) : z4;
                            int left = __shfl_up_sync(0xffffffffu, q.w, 1);
                            if (c == 0) left = 0;
                            else if (lane == 0) left = has[t] ? cf_q(__ldg(rows[t] + 4 * c - 1), recip, f) : 0;
                            const int64_t sg = (t == 0 || t == 3) ? 1 : -1;
                            acc[0] += sg * ((int64_t)q.x - left);
                            acc[1] += sg * ((int64_t)q.y - q.x);
                            acc[2] += sg * ((int64_t)q.z - q.y);
                            acc[3] += sg * ((int64_t)q.w - q.z);
                        }
                        if (act)
                            *reinterpret_cast<int4*>(cf_slot(P, (int64_t)rr * N2 + 4 * c)) =
                                make_int4(cf_res(acc[0], f), cf_res(acc[1], f), cf_res(acc[2], f), cf_res(acc[3], f));
                    }
                }
                dz_prev = dz;
                dzm_prev = dzm;
                prev_fast = fast;
            }
        }
    } else {                                                         // CF_BLOCKS
        const SegGeo& sg = a.sg;
        const int B0 = (int)sg.B[0], B1 = (int)sg.B[1], B2 = (int)sg.B[2];
        const int segsz = B0 * B1 * B2, cpb = segsz >> 5;
        const int64_t brow = tile / a.tpr;                           // block row (b0, b1)
        const int64_t b2a = (tile - brow * a.tpr) * a.kb;
        const int nseg = (int)(sg.G[2] - b2a < a.kb ? sg.G[2] - b2a : a.kb);
        const int64_t b0 = brow / sg.G[1], b1 = brow - b0 * sg.G[1];
        const int64_t n1 = sg.n[1], n2 = sg.n[2];
        const int64_t seg0 = brow * sg.G[2] + b2a;
        c0 = seg0 * cpb;
        nch = nseg * cpb;
        const int gpr = nseg * B2 / 4;                               // float4 columns of the box
        const int rows = B0 * B1;
        const float* xb = a.x + (b0 * B0 * n1 + b1 * B1) * n2 + b2a * B2;
        bool big = false;
        const int nit = rows * gpr;                                  // <= 2048 float4: <= 8 per thread
        float4 vv[8];
#pragma unroll
        for (int j = 0; j < 8; j++) {
            const int i = (int)threadIdx.x + j * CF_T;
            if (i < nit) {
                const int zy = i / gpr, g = i - zy * gpr;
                const int zl = zy / B1, yl = zy - zl * B1;
                vv[j] = __ldg(reinterpret_cast<const float4*>(xb + ((int64_t)zl * n1 + yl) * n2 + 4 * g));
            }
        }
#pragma unroll
        for (int j = 0; j < 8; j++) {
            const int i = (int)threadIdx.x + j * CF_T;
            if (i < nit) {
                const int zy = i / gpr, g = i - zy * gpr;
                const int xx = 4 * g, t = xx / B2, xl = xx - t * B2;
                const bool bg = cf_big(vv[j], vlim);
                big |= bg;
                int4 q;
                if (__any_sync(__activemask(), bg)) q = cf_q4(vv[j], recip, f);   // exact (range checks)
                else q = cf_qf4(vv[j], recip);
                *reinterpret_cast<int4*>(cf_slot(P, (int64_t)t * segsz + zy * B2 + xl)) = q;
            }
        }
        const bool exact = __syncthreads_or(big);                    // some |q| >= 2^28: int64 residual checks
        const int c = threadIdx.x;
        int32_t* row = P + c * CF_S;
        if (c < nch) {                                               // chunk partial sums -> block sums
            int64_t s = 0;
#pragma unroll
            for (int k = 0; k < 8; k++) {
                const int4 v = *reinterpret_cast<const int4*>(row + 4 * k);
                s += (int64_t)v.x + v.y + v.z + v.w;
            }
            if (cpb == 1) s_bsum[c] = s;
            else atomicAdd(reinterpret_cast<unsigned long long*>(&s_bsum[c / cpb]), (unsigned long long)s);
        }
        __syncthreads();
        if (c < nch) {
            const int blk = cpb == 1 ? c : c / cpb;
            const int64_t bs = s_bsum[blk];
            int64_t mean;                                            // truncation toward zero (C division)
            if ((segsz & (segsz - 1)) == 0) {
                const int lg = __ffs(segsz) - 1;
                mean = bs >= 0 ? (bs >> lg) : -((-bs) >> lg);
            } else {
                mean = bs / segsz;
            }
            if (c == blk * cpb) a.meta[seg0 + blk] = (int32_t)mean;
            if (!exact) {
                const int32_t m32 = (int32_t)mean;
#pragma unroll
                for (int k = 0; k < 8; k++) {
                    const int4 v = *reinterpret_cast<const int4*>(row + 4 * k);
                    *reinterpret_cast<int4*>(row + 4 * k) = make_int4(v.x - m32, v.y - m32, v.z - m32, v.w - m32);
                }
            } else {
#pragma unroll
                for (int k = 0; k < 8; k++) {
                    const int4 v = *reinterpret_cast<const int4*>(row + 4 * k);
                    *reinterpret_cast<int4*>(row + 4 * k) =
                        make_int4(cf_res((int64_t)v.x - mean, f), cf_res((int64_t)v.y - mean, f),
                                  cf_res((int64_t)v.z - mean, f), cf_res((int64_t)v.w - mean, f));
                }
            }
        }
    }
    __syncthreads();

    // ================================ sizes + offsets ================================
    const int c = threadIdx.x;
    const bool mine = c < nch;
    const int32_t* v = P + c * CF_S;
    uint32_t m = 0, sgn = 0;
#pragma unroll
    for (int k = 0; k < 8; k++) {
        const int4 w = mine ? *reinterpret_cast<const int4*>(v + 4 * k) : make_int4(0, 0, 0, 0);
        m |= (uint32_t)abs(w.x) | (uint32_t)abs(w.y) | (uint32_t)abs(w.z) | (uint32_t)abs(w.w);
        sgn |= ((uint32_t)w.x >> 31 | ((uint32_t)w.y >> 31) << 1 | ((uint32_t)w.z >> 31) << 2 |
                ((uint32_t)w.w >> 31) << 3) << (4 * k);
    }
    const int bw = m ? 32 - __clz(m) : 0;                            // bits of max |p| (OR has the same top bit)
    const uint32_t size = mine ? (bw ? 5u + 4u * (uint32_t)bw : 1u) : 0u;
    uint32_t inc = size;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= d) inc += o;
    }
    if (lane == 31) s_wsum[warp] = inc;
    __syncthreads();
    uint32_t before = 0, tot = 0;
#pragma unroll
    for (int w2 = 0; w2 < CF_T / 32; w2++) {
        const uint32_t t = s_wsum[w2];
        before += w2 < warp ? t : 0u;
        tot += t;
    }
    const uint32_t loc = before + inc - size;
    // warp 0 looks back for the tile's byte base while the other warps pack (the packed bytes do not depend
    // on the base: the staging copy starts at tile byte 0, the copy-out shifts it to the base's alignment)
    if (warp == 0) {
#ifdef CF_NO_LOOKBACK                                                 // timing probe only (wrong offsets)
        const unsigned long long base = (unsigned long long)tile * 20000ull;
#else
        const unsigned long long base = lookback_exclusive_warp62(a.lb, tile, (unsigned long long)tot);
#endif
        if (lane == 0) {
            s_base = base;
            if (tile == a.n_tiles - 1) *a.total = base + tot;
        }
    }

    // ================================ pack ================================
    // The chunk's bytes [bw][sign bitmap x4][magnitudes, bw bits each LSB-first] are the byte stream of the
    // word sequence X = (bw << 24, sgn, M_0 .. M_{bw-1}, 0) from byte 3 on; staged at tile byte loc of the
    // zeroed, word-aligned staging copy, word k of the chunk is funnel_r(X_k, X_k+1, 8(3 - loc%4)).  Its first
    // and last words are shared with the neighbouring chunks (atomicOr), the others are its own.
    if (mine && bw) {
        uint32_t* W = reinterpret_cast<uint32_t*>(SB) + (loc >> 2);
        const uint32_t r = 8u * (3u - (loc & 3u));
        uint32_t xa = (uint32_t)bw << 24, xb = sgn;
        atomicOr(W, __funnelshift_r(xa, xb, r));
        int k = 1;
        uint32_t cur = 0;
        int nb = 0;
#pragma unroll
        for (int g = 0; g < 8; g++) {
            const int4 w = *reinterpret_cast<const int4*>(v + 4 * g);
            const int32_t e4[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (int e = 0; e < 4; e++) {
                const uint32_t mg = (uint32_t)abs(e4[e]);
                cur |= mg << nb;
                nb += bw;
                if (nb >= 32) {                                       // M word complete
                    nb -= 32;
                    xa = xb;
                    xb = cur;
                    W[k++] = __funnelshift_r(xa, xb, r);
                    cur = __funnelshift_r(mg, 0u, (uint32_t)(bw - nb));   // the bits of mg past the word
                }
            }
        }
        atomicOr(W + k, __funnelshift_r(xb, 0u, r));                  // 32 bw bits: nothing left in cur
    }
    __syncthreads();
    const unsigned long long lo = s_base, hi = lo + tot;
    if (mine) a.offsets[c0 + c] = lo + loc;
    // copy-out: global byte g = staging byte g - lo; the aligned 16-B body from staging words shifted by
    // (a0 - lo) % 4 bytes, byte stores at the two edges shared with the neighbouring tiles
    const unsigned long long a0 = (lo + 15) & ~15ull, a1 = hi & ~15ull;
    if (a0 >= a1) {
        for (unsigned long long g = lo + threadIdx.x; g < hi; g += CF_T) a.payload[g] = SB[g - lo];
    } else {
        if (lo + threadIdx.x < a0) a.payload[lo + threadIdx.x] = SB[threadIdx.x];
        if (a1 + threadIdx.x < hi) a.payload[a1 + threadIdx.x] = SB[a1 - lo + threadIdx.x];
        const uint32_t d0 = (uint32_t)(a0 - lo);                      // staging byte of a0 (< 16)
        const uint32_t* sw = reinterpret_cast<const uint32_t*>(SB) + (d0 >> 2);
        const uint32_t rs = 8u * (d0 & 3u);
        uint4* gv = reinterpret_cast<uint4*>(a.payload + a0);
        const int nv16 = (int)((a1 - a0) >> 4);
        for (int i = threadIdx.x; i < nv16; i += CF_T) {
            const uint32_t* q = sw + 4 * i;
            const uint32_t w0 = q[0], w1 = q[1], w2 = q[2], w3 = q[3], w4 = q[4];
            gv[i] = make_uint4(__funnelshift_r(w0, w1, rs), __funnelshift_r(w1, w2, rs), __funnelshift_r(w2, w3, rs),
                               __funnelshift_r(w3, w4, rs));
        }
    }
    if (f) atomicOr(a.flags, f);
}

// Which front applies (0 = none: the multi-kernel path), and the tile grid
struct CfPlan {
    int front;
    int64_t tiles, rows_per_tile, tpr;
    int kb;
};

static CfPlan cf_plan(const HszgGeom* g) {
    CfPlan p{-1, 0, 0, 0, 0};
    if (g->n <= 0 || g->n_chunks * kChunkCap != g->n) return p;      // every chunk 32 values
    const SegGeo sg = make_seggeo(*g);
    switch (g->kind) {
        case HSZG_HSZP:
            p.front = CF_PREV;
            p.tiles = (g->n + CF_VALS - 1) / CF_VALS;
            break;
        case HSZG_HSZP_ND: {
            const int64_t n2 = sg.n[2];
            if (n2 % kChunkCap || n2 > CF_VALS) return p;
            p.front = CF_LORENZO;
            p.rows_per_tile = CF_VALS / n2;
            p.tiles = (sg.n[0] * sg.n[1] + p.rows_per_tile - 1) / p.rows_per_tile;
            break;
        }
        default: {
            const int64_t segsz = sg.B[0] * sg.B[1] * sg.B[2];
            if (sg.n[0] % sg.B[0] || sg.n[1] % sg.B[1] || sg.n[2] % sg.B[2] || sg.B[2] % 4 || segsz % kChunkCap ||
                segsz > CF_VALS || sg.n[2] % 4)
                return p;
            p.front = CF_BLOCKS;
            p.kb = (int)(CF_VALS / segsz);
            p.tpr = (sg.G[2] + p.kb - 1) / p.kb;
            p.tiles = sg.G[0] * sg.G[1] * p.tpr;
            break;
        }
    }
    return p;
}

// workspace: flags (4 B) | pad | total (8 B) at 8 | look-back state at 64
static size_t cf_ws_bytes(int64_t tiles) { return 64 + (size_t)tiles * 20 + 64 + 256; }

}  // namespace hszg

using namespace hszg;

int hszg_set_cuda_error(HszgErr* err, cudaError_t e, const char* where);

extern "C" int hszg_compress_plan(const HszgGeom* g, uint64_t* ws_bytes, uint64_t* payload_capacity) {
    const CfPlan p = cf_plan(g);
    if (p.front < 0) return 0;
    if (ws_bytes) *ws_bytes = cf_ws_bytes(p.tiles);
    if (payload_capacity) *payload_capacity = (uint64_t)g->n_chunks * CF_MAXCB + HSZG_PAYLOAD_PAD;
    return 1;
}

extern "C" int hszg_compress_fused(const HszgGeom* g, const float* field, double recip, uint8_t* payload,
                                   uint64_t capacity, uint64_t* offsets, int32_t* metadata, uint64_t* total_host,
                                   void* ws, size_t ws_bytes, void* stream, HszgErr* err) {
    err->status = HSZG_OK;
    const CfPlan p = cf_plan(g);
    const bool blocks = g->kind == HSZG_HSZX || g->kind == HSZG_HSZX_ND;
    if (p.front < 0 || ws_bytes < cf_ws_bytes(p.tiles) || capacity < (uint64_t)g->n_chunks * CF_MAXCB ||
        (reinterpret_cast<uintptr_t>(field) & 15) || (reinterpret_cast<uintptr_t>(payload) & 15) ||
        (blocks && !metadata) || !(recip > 0)) {
        err->status = HSZG_INVALID_ARG;
        snprintf(err->message, sizeof(err->message),
                 "compress_fused: unsupported geometry (hszg_compress_plan) or bad buffers");
        return HSZG_INVALID_ARG;
    }
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    char* w = reinterpret_cast<char*>(ws);
    CfArgs a;
    a.x = field;
    a.n = g->n;
    a.recip = recip;
    // the fast quantizer's range: |d| <= vlim keeps |t| below 2^28 with a wide margin for the roundings
    {
        const double lim = (268435456.0 - 4.0) / recip;
        float vl = (float)lim;
        if ((double)vl > lim) vl = nextafterf(vl, 0.0f);
        a.vlim = lim >= 3.0e38 ? 3.0e38f : vl;
    }
    a.sg = make_seggeo(*g);
    a.N0 = a.sg.n[0];
    a.N1 = a.sg.n[1];
    a.N2 = a.sg.n[2];
    a.rows_per_tile = p.rows_per_tile;
    a.tpr = p.tpr;
    a.kb = p.kb;
    a.n_chunks = g->n_chunks;
    a.n_tiles = p.tiles;
    a.payload = payload;
    a.offsets = offsets;
    a.meta = metadata;
    a.flags = reinterpret_cast<unsigned int*>(w);
    a.total = reinterpret_cast<unsigned long long*>(w + 8);
    a.lb = lookback_carve(w + 64, p.tiles);
    cudaMemsetAsync(w, 0, 64 + lookback_clear_bytes(p.tiles), st);
#define CF_LAUNCH(F)                                                                                     \
    do {                                                                                                 \
        cudaFuncSetAttribute(k_compress_tiles<F>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CF_SMEM); \
        k_compress_tiles<F><<<(unsigned)p.tiles, CF_T, CF_SMEM, st>>>(a);                               \
    } while (0)
    if (p.front == CF_PREV) CF_LAUNCH(CF_PREV);
    else if (p.front == CF_LORENZO) CF_LAUNCH(CF_LORENZO);
    else CF_LAUNCH(CF_BLOCKS);
#undef CF_LAUNCH
    {
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return hszg_set_cuda_error(err, e, "compress_fused");
    }
    unsigned long long h[2] = {0, 0};                                // flags word (low 32 bits), total
    cudaMemcpyAsync(h, w, 16, cudaMemcpyDeviceToHost, st);
    const cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return hszg_set_cuda_error(err, e, "compress_fused readback");
    const unsigned int fl = (unsigned int)(h[0] & 0xffffffffu);
    if (fl & 1u) {
        err->status = HSZG_EPS_TOO_SMALL;
        snprintf(err->message, sizeof(err->message), "quantization index exceeds %d; increase the error bound", kQmax);
        return HSZG_EPS_TOO_SMALL;
    }
    if (fl & 2u) {
        err->status = HSZG_VALUE;
        snprintf(err->message, sizeof(err->message), "field contains NaN or Inf; refusing to quantize");
        return HSZG_VALUE;
    }
    if (fl & 4u) {
        err->status = HSZG_EPS_TOO_SMALL;
        snprintf(err->message, sizeof(err->message),
                 "decorrelated residual overflows 32-bit range; increase the error bound");
        return HSZG_EPS_TOO_SMALL;
    }
    *total_host = h[1];
    // the HSZG_PAYLOAD_PAD bytes after the payload are zero (readers may touch them)
    cudaMemsetAsync(payload + h[1], 0, HSZG_PAYLOAD_PAD, st);
    {
        const cudaError_t e2 = cudaGetLastError();
        if (e2 != cudaSuccess) return hszg_set_cuda_error(err, e2, "compress_fused pad");
    }
    return HSZG_OK;
}
