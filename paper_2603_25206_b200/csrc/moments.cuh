// moments.cuh — lean per-chunk moments of a validated FULL chunk (32 values) straight from its
// staged bytes: the decode core of the fused statistics / regional reductions (K-STAT, K-REG).
//
// The layout is the reference chunk (_fallback.py:1-8, _bitpack.pyx:124-143): 1 bit-width byte,
// 4 sign bytes (value j <-> bit j), then 32 magnitudes of bw bits LSB-first.  Statistics never
// need the signed values one by one:
//     sum p   = sum |p| - 2 sum_{sign set} |p|      (a predicated add per value)
//     sum p^2 = sum |p|^2                            (sign-free: one IMAD per value)
//     sum j p = sum j|p| - 2 sum_{sign set} j|p|     (weighted means, stats.py:88/95-112)
// so a value costs a field extract, one add into |p|, a predicated add, one IMAD (+ two for the
// index-weighted sum, + a negate and a 3-input min/max when extrema are wanted).
//
// Field extraction reads G values per 32-bit funnel window (G = 4 for bw <= 8, G = 2 for bw <= 16):
// the bit cursor advances once per window.  The window width is chosen per WARP (all lanes <= 8:
// G = 4, all <= 16: G = 2), so lanes never diverge on it; chunks wider than 16 bits (rare: the
// reference encoder produces them only for |p| >= 2^16) take an exact 128-bit path.
#pragma once
#include "common.cuh"

namespace hszg {

struct ChunkMoments {
    int64_t sp;      // sum p
    u128 sq;         // sum p^2
    int64_t tp;      // sum j p (TSUM)
    int32_t mn, mx;  // min / max p (MINMAX)
};

// acc += v when (word & bit) != 0 (a predicated add: LOP3 -> P, @P IADD; bit is a constant after
// unrolling)
__device__ __forceinline__ void add_if_bit(uint32_t& acc, uint32_t word, uint32_t bit, uint32_t v) {
    asm("{\n .reg .pred p;\n .reg .b32 t;\n and.b32 t, %1, %2;\n setp.ne.b32 p, t, 0;\n @p add.u32 %0, %0, %3;\n}"
        : "+r"(acc)
        : "r"(word), "r"(bit), "r"(v));
}

template <int G, bool TSUM, bool MINMAX>
__device__ __forceinline__ void chunk_moments_g(const uint32_t* w, uint32_t rel, uint32_t bw, uint32_t smask,
                                                ChunkMoments& r) {
    const uint32_t bitpos = (rel + 5) * 8;
    uint32_t wi = bitpos >> 5, sh = bitpos & 31;
    uint32_t cur = w[wi], nxt = w[wi + 1];
    const uint32_t mask = (1u << bw) - 1u;          // bw <= 16 here
    const uint32_t adv = (uint32_t)G * bw;
    uint32_t sa = 0, sn = 0, ta = 0, tn = 0;
    uint32_t sq32 = 0;                               // G = 4: 32 squares of < 2^8 fit 21 bits
    uint64_t sq64 = 0;
    int32_t mn = INT32_MAX, mx = INT32_MIN;
#pragma unroll
    for (int k = 0; k < 32 / G; k++) {
        const uint32_t grp = __funnelshift_r(cur, nxt, sh);
#pragma unroll
        for (int i = 0; i < G; i++) {
            const int j = k * G + i;
            const uint32_t m = i == 0 ? (grp & mask) : ((grp >> (i * bw)) & mask);
            sa += m;
            add_if_bit(sn, smask, 1u << j, m);
            if (G == 4) sq32 += m * m;
            else sq64 += (uint64_t)m * m;
            if (TSUM) {
                ta += (uint32_t)j * m;
                add_if_bit(tn, smask, 1u << j, (uint32_t)j * m);
            }
            if (MINMAX) {
                const bool neg = (smask >> j) & 1u;
                const int32_t v = neg ? -(int32_t)m : (int32_t)m;
                mn = min(mn, v);
                mx = max(mx, v);
            }
        }
        if (k + 1 < 32 / G) {
            sh += adv;
            if (sh >= 32) {
                sh -= 32;
                cur = nxt;
                wi++;
                nxt = w[wi + 1];
            }
        }
    }
    r.sp = (int64_t)sa - 2 * (int64_t)sn;
    r.sq = G == 4 ? (u128)sq32 : (u128)sq64;
    r.tp = (int64_t)ta - 2 * (int64_t)tn;
    r.mn = mn;
    r.mx = mx;
}

// bw <= 8 without extrema, four values per IDP4A (SWAR): the four bw-bit fields of a 32-bit funnel window are
// spread into the bytes of a word (a shift + LOP3 each), the four sign bits into bytes of +1 / -1 (one
// magic multiply spreads bits 0-3 to bits 0, 8, 16, 24), and one dp4a each gives sum p, sum |p|^2 (and
// sum j p with per-byte signed indices): ~4 instructions per value instead of ~7.
__device__ __forceinline__ int32_t dp4a_us(uint32_t a, uint32_t b, int32_t c) {      // u8 x s8
    int32_t d;
    asm("dp4a.u32.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}
__device__ __forceinline__ uint32_t dp4a_uu(uint32_t a, uint32_t b, uint32_t c) {    // u8 x u8
    uint32_t d;
    asm("dp4a.u32.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

template <bool TSUM>
__device__ __forceinline__ void chunk_moments_b8(const uint32_t* w, uint32_t rel, uint32_t bw, uint32_t smask,
                                                 ChunkMoments& r) {
    const uint32_t bitpos = (rel + 5) * 8;
    uint32_t wi = bitpos >> 5, sh = bitpos & 31;
    uint32_t cur = w[wi], nxt = w[wi + 1];
    const uint32_t mask = (1u << bw) - 1u;          // bw <= 8
    const uint32_t adv = 4 * bw;
    const uint32_t s1 = 8 - bw, s2 = 16 - 2 * bw, s3 = 24 - 3 * bw;
    const uint32_t m1 = mask << 8, m2 = mask << 16, m3 = mask << 24;
    int32_t sp = 0, tp = 0;                          // |sum| <= 32 * 255, |sum j p| <= 31 * 32 * 255
    uint32_t sq = 0;                                 // <= 32 * 255^2
#pragma unroll
    for (int k = 0; k < 8; k++) {
        const uint32_t grp = __funnelshift_r(cur, nxt, sh);
        const uint32_t b = (grp & mask) | ((grp << s1) & m1) | ((grp << s2) & m2) | ((grp << s3) & m3);
        const uint32_t sb = (((smask >> (4 * k)) & 15u) * 0x00204081u) & 0x01010101u;   // sign bits -> bytes
        sp = dp4a_us(b, sb * 0xFEu + 0x01010101u, sp);                                  // bytes +1 / -1
        sq = dp4a_uu(b, b, sq);
        if (TSUM) {
            // signed byte indices j = 4k + i (negated where the sign is set; byte 0 of k = 0 is j = 0)
            const uint32_t sbt = k == 0 ? (sb & 0x01010100u) : sb;
            const uint32_t idx = 0x03020100u + 0x04040404u * (uint32_t)k;
            tp = dp4a_us(b, (idx ^ (sbt * 0xFFu)) + sbt, tp);
        }
        if (k + 1 < 8) {
            sh += adv;
            if (sh >= 32) {
                sh -= 32;
                cur = nxt;
                wi++;
                nxt = w[wi + 1];
            }
        }
    }
    r.sp = sp;
    r.sq = (u128)sq;
    r.tp = tp;
    r.mn = INT32_MAX;
    r.mx = INT32_MIN;
}

// bw 17..32: exact, value by value (int64 / u128)
template <bool TSUM, bool MINMAX>
__device__ __forceinline__ void chunk_moments_wide(const uint32_t* w, uint32_t rel, uint32_t bw, uint32_t smask,
                                                   ChunkMoments& r) {
    const uint32_t bitpos = (rel + 5) * 8;
    uint32_t wi = bitpos >> 5, sh = bitpos & 31;
    uint32_t cur = w[wi], nxt = w[wi + 1];
    const uint32_t mask = bw >= 32 ? 0xffffffffu : (1u << bw) - 1u;
    int64_t sp = 0, tp = 0;
    u128 sq = 0;
    int32_t mn = INT32_MAX, mx = INT32_MIN;
    for (int j = 0; j < 32; j++) {
        const uint32_t m = __funnelshift_r(cur, nxt, sh) & mask;    // <= 2^31 - 1 (validated)
        sh += bw;
        if (sh >= 32) {
            sh -= 32;
            cur = nxt;
            wi++;
            nxt = w[wi + 1];
        }
        const int64_t v = ((smask >> j) & 1u) ? -(int64_t)m : (int64_t)m;
        sp += v;
        sq += (u128)((uint64_t)m * m);
        if (TSUM) tp += (int64_t)j * v;
        if (MINMAX) {
            mn = min(mn, (int32_t)v);
            mx = max(mx, (int32_t)v);
        }
    }
    r.sp = sp;
    r.sq = sq;
    r.tp = tp;
    r.mn = mn;
    r.mx = mx;
}

// Moments of the full chunk whose bytes start at byte `rel` of the staged words.  All 32 lanes of
// the warp must call it (valid = false for lanes without a chunk); the window width is warp-uniform.
template <bool TSUM, bool MINMAX>
__device__ __forceinline__ ChunkMoments chunk_moments(const uint32_t* w, uint32_t rel, bool valid) {
    ChunkMoments r;
    uint32_t bw = valid ? smem_byte(w, rel) : 0u;
    const uint32_t smask = bw ? smem_u32(w, rel + 1) : 0u;
    const unsigned act = __activemask();
    if (__all_sync(act, bw <= 8)) {
        if (MINMAX) chunk_moments_g<4, TSUM, MINMAX>(w, rel, bw, smask, r);
        else chunk_moments_b8<TSUM>(w, rel, bw, smask, r);
    } else if (__all_sync(act, bw <= 16)) {
        chunk_moments_g<2, TSUM, MINMAX>(w, rel, bw, smask, r);
    } else if (bw <= 16) {
        chunk_moments_g<2, TSUM, MINMAX>(w, rel, bw, smask, r);
    } else {
        chunk_moments_wide<TSUM, MINMAX>(w, rel, bw, smask, r);
    }
    if (!valid) {
        r.sp = 0;
        r.sq = 0;
        r.tp = 0;
        r.mn = INT32_MAX;
        r.mx = INT32_MIN;
    }
    return r;
}

// Running-prefix moments of one full chunk (HSZP variance by tile algebra, ops.cu): with l_k the
// chunk-local inclusive prefix of p (l_31 = T, the chunk total), returns T, S1 = sum_k l_k and
// S2 = sum_k l_k^2.  Narrow chunks (bw <= 16: |l_k| < 2^21) run in int32 / one IMAD.WIDE per value; the
// window width is warp-uniform as in chunk_moments; wider chunks take int64 / u128.
struct PrefixMoments {
    int64_t T, S1;
    u128 S2;
    int64_t mn, mx;      // min / max of the l_k
};

template <int G>
__device__ __forceinline__ void prefix_moments_g(const uint32_t* w, uint32_t rel, uint32_t bw, uint32_t smask,
                                                 PrefixMoments& r) {
    const uint32_t bitpos = (rel + 5) * 8;
    uint32_t wi = bitpos >> 5, sh = bitpos & 31;
    uint32_t cur = w[wi], nxt = w[wi + 1];
    const uint32_t mask = (1u << bw) - 1u;
    const uint32_t adv = (uint32_t)G * bw;
    int32_t run = 0, s1 = 0, mn = INT32_MAX, mx = INT32_MIN;
    uint64_t s2 = 0;
#pragma unroll
    for (int k = 0; k < 32 / G; k++) {
        const uint32_t grp = __funnelshift_r(cur, nxt, sh);
#pragma unroll
        for (int i = 0; i < G; i++) {
            const int j = k * G + i;
            const int32_t m = (int32_t)(i == 0 ? (grp & mask) : ((grp >> (i * bw)) & mask));
            run += ((smask >> j) & 1u) ? -m : m;
            s1 += run;
            s2 += (uint64_t)((int64_t)run * run);
            mn = min(mn, run);
            mx = max(mx, run);
        }
        if (k + 1 < 32 / G) {
            sh += adv;
            if (sh >= 32) {
                sh -= 32;
                cur = nxt;
                wi++;
                nxt = w[wi + 1];
            }
        }
    }
    r.T = run;
    r.S1 = s1;
    r.S2 = s2;
    r.mn = mn;
    r.mx = mx;
}

__device__ __forceinline__ void prefix_moments_wide(const uint32_t* w, uint32_t rel, uint32_t bw, uint32_t smask,
                                                    PrefixMoments& r) {
    const uint32_t bitpos = (rel + 5) * 8;
    uint32_t wi = bitpos >> 5, sh = bitpos & 31;
    uint32_t cur = w[wi], nxt = w[wi + 1];
    const uint32_t mask = bw >= 32 ? 0xffffffffu : (1u << bw) - 1u;
    int64_t run = 0, s1 = 0, mn = INT64_MAX, mx = INT64_MIN;
    u128 s2 = 0;
    for (int j = 0; j < 32; j++) {
        const int64_t m = (int64_t)(__funnelshift_r(cur, nxt, sh) & mask);
        sh += bw;
        if (sh >= 32) {
            sh -= 32;
            cur = nxt;
            wi++;
            nxt = w[wi + 1];
        }
        run += ((smask >> j) & 1u) ? -m : m;
        s1 += run;
        s2 += (u128)(uint64_t)(run < 0 ? -run : run) * (u128)(uint64_t)(run < 0 ? -run : run);
        mn = min(mn, run);
        mx = max(mx, run);
    }
    r.T = run;
    r.S1 = s1;
    r.S2 = s2;
    r.mn = mn;
    r.mx = mx;
}

__device__ __forceinline__ PrefixMoments prefix_moments(const uint32_t* w, uint32_t rel, bool valid) {
    PrefixMoments r;
    const uint32_t bw = valid ? smem_byte(w, rel) : 0u;
    const uint32_t smask = bw ? smem_u32(w, rel + 1) : 0u;
    const unsigned act = __activemask();
    if (__all_sync(act, bw <= 8)) prefix_moments_g<4>(w, rel, bw, smask, r);
    else if (bw <= 16) prefix_moments_g<2>(w, rel, bw, smask, r);
    else prefix_moments_wide(w, rel, bw, smask, r);
    if (!valid) {
        r.T = 0;
        r.S1 = 0;
        r.S2 = 0;
        r.mn = INT64_MAX;
        r.mx = INT64_MIN;
    }
    return r;
}

}  // namespace hszg
