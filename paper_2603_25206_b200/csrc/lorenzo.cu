// lorenzo.cu — HSZP_ND in one pass: decode + Lorenzo inversion (x, y, z prefix) + gradient +
// Laplacian + exact statistics, q never in HBM.  compressors.py:201-226 (q = cumsum of p along
// every axis) fused with fields.py:34-80.
//
// Pre-pass (hszg_band_scan with bands of 16 rows, no L): per plane z, the exclusive band offsets
// A[z][b][x] = sum of the x-prefixed rows above band b (= P2 at the row above it), and per 128-wide
// strip s and row y the row prefix just left / right of the strip, E = R(128s-1), F = R(128s+128).
// Main kernel: a CTA owns x in [128s, 128s+128) by y in [16b, 16b+16) and slides along z over the
// whole slab.  Per plane:
//   warps 0-1   load (lane-parallel cp.async) the payload bytes of the 17 rows y0..y0+16 restricted to the strip's 4
//               chunks, the band-offset row A[z][b] and the strip edges (and writes the chunk
//               offsets, prefetched a plane ahead, into the staging slot);
//   warps 1-8   decode quarter-chunk jobs and prefix each row (half-warp scan + E) into R (double
//               buffered);
//   warps 9-13  run the column prefix from A[z][b] (y) and add the previous q plane (z):
//               P2[y][x] = A[b][x] + sum_{y0<=y'<=y} R[y'][x], q[z] = q[z-1] + P2[z]; the halo
//               columns x0-1 / x0+128 come from E / F, the halo row y0-1 from A alone;
//   warps 14-21 emit from the q ring (as fused.cu / zring.cu).
#include <cstdio>
#include "tile.cuh"
#include "stencil.cuh"
#include "async.cuh"

namespace hszg {

constexpr int LR_T = 736;
constexpr int LR_DT = 256;                  // decoders: warps 2-9
constexpr int LR_ST = 160;                  // scanners: warps 10-14 (130 columns)
constexpr int LR_CT = 256;                  // emitters: warps 15-22, 2 rows each
constexpr int LR_TX = 128, LR_TY = 16;
constexpr int LR_ROWS = LR_TY + 2;          // q ring rows y0-1 .. y0+16
constexpr int LR_DROWS = LR_TY + 1;         // decoded rows y0 .. y0+16
constexpr int LR_X0 = 8;
constexpr int LR_RW = 148;
constexpr int LR_PLANE = LR_ROWS * LR_RW;
constexpr int LR_NPL = 4;
constexpr int LR_D = 12;                    // staged planes in flight
constexpr int LR_AW = LR_TX + 8;            // staged band-offset row: x0-4 .. x0+132
constexpr int LR_EFN = 2 * (LR_DROWS + 1);  // staged strip edges (rows y0..y0+17), 144 B
constexpr int LR_OD = 16;                   // planes of chunk offsets in flight (loader-private ring)

struct LrArgs {
    const uint8_t* payload;
    uint64_t len;
    const uint64_t* offsets;
    int64_t n_chunks;
    int64_t nz, n1, n2, nb, nstrips;
    const int32_t* A;
    const int32_t* EF;
    const int32_t* carry;
    const int32_t* q_upper;
    int64_t gz0, gN0;
    double eps;
    float* o0;
    float* o1;
    float* o2;
    float* o3;
    HszgAcc* acc;
    uint32_t pr;                              // staged payload bytes per row
    uint32_t slot;                            // staging slot bytes
};

// staging slot: [payload 17 x pr][rel 17 x 4 u32][A row LR_AW i32][EF LR_EFN i32]
__host__ __device__ inline uint32_t lr_rel_off(uint32_t pr) { return LR_DROWS * pr; }
__host__ __device__ inline uint32_t lr_a_off(uint32_t pr) { return lr_rel_off(pr) + LR_DROWS * 16; }
__host__ __device__ inline uint32_t lr_ef_off(uint32_t pr) { return lr_a_off(pr) + LR_AW * 4; }
inline uint32_t lr_pr(int max_bw) { return (uint32_t)((4 * chunk_bytes(kChunkCap, max_bw) + 31 + 15) / 16 * 16); }
inline uint32_t lr_slot(int max_bw) { return (lr_ef_off(lr_pr(max_bw)) + LR_EFN * 4 + 127) / 128 * 128; }
inline size_t lr_smem(int max_bw) {
    return (size_t)LR_NPL * LR_PLANE * 4 + (size_t)LR_D * lr_slot(max_bw) + (size_t)2 * LR_DROWS * LR_TX * 4;
}

// strip-edge table rows per (plane, strip): even, so every (plane, strip) block starts 16-B aligned
__host__ __device__ inline int64_t ef_rows(int64_t n1) { return (n1 + 1) & ~(int64_t)1; }

template <bool Exact>
__global__ void __launch_bounds__(LR_T, 1) k_lorenzo_ring(LrArgs a) {
    extern __shared__ __align__(128) uint8_t lsm[];
    int32_t* Q = reinterpret_cast<int32_t*>(lsm);                         // [NPL][ROWS][RW]
    uint8_t* SL = lsm + (size_t)LR_NPL * LR_PLANE * 4;                    // [D][slot]
    int32_t* RB = reinterpret_cast<int32_t*>(SL + (size_t)LR_D * a.slot);  // [2][DROWS][TX]
    __shared__ __align__(8) uint64_t s_full[LR_D], s_empty[LR_D], q_full[LR_NPL], q_empty[LR_NPL], o_full[LR_OD],
        rb_full[2], rb_empty[2];
    __shared__ __align__(16) uint64_t OR[LR_OD * LR_DROWS * 6];        // offsets ring (loader only)
    const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
    const int64_t s = blockIdx.x, b = blockIdx.y;
    const int64_t x0 = s * LR_TX, y0 = b * LR_TY;
    const int64_t n1 = a.n1, n2 = a.n2, nz = a.nz;
    const int64_t plane = n1 * n2;
    const int cpr = (int)(n2 >> 5);                                       // chunks per row
    const int nch = (int)((n2 - x0) >> 5) < 4 ? (int)((n2 - x0) >> 5) : 4; // strip chunks
    const int nrow = (int)(n1 - y0) < LR_DROWS ? (int)(n1 - y0) : LR_DROWS;
    const int64_t xs = x0 >= 4 ? x0 - 4 : 0;
    const int64_t xe = x0 + LR_TX + 4 < n2 ? x0 + LR_TX + 4 : n2;

    for (int i = threadIdx.x; i < LR_NPL * LR_PLANE / 4; i += LR_T) reinterpret_cast<int4*>(Q)[i] = make_int4(0, 0, 0, 0);
    if (threadIdx.x == 0) {
        for (int i = 0; i < LR_D; i++) {
            mbar_init(&s_full[i], 65);                // 2 x 32 cp.async completions + the rel-table arrive
            mbar_init(&s_empty[i], LR_DT + LR_ST);
        }
        for (int i = 0; i < LR_NPL; i++) {
            mbar_init(&q_full[i], LR_ST);
            mbar_init(&q_empty[i], LR_CT);
        }
        for (int i = 0; i < LR_OD; i++) mbar_init(&o_full[i], 32);
        for (int i = 0; i < 2; i++) {
            mbar_init(&rb_full[i], LR_DT);
            mbar_init(&rb_empty[i], LR_ST);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (wp == 0) {
        // ================================ loader ================================
        const bool row_ok = lane < nrow;
        // Lane-parallel 16-B async copies (cp.async, completion tracked by the mbarriers): per plane
        // ~30 small pieces, which one elected lane would otherwise issue one TMA at a time.  All
        // addresses advance by a fixed stride per plane (no 64-bit index math in the loop).
        // Chunk offsets of this lane's row arrive LR_OD planes ahead (6 entries from an even chunk
        // index: the strip's 4 starts + the end; 4 entries for the index's last row, whose end is
        // the payload end).
        const int64_t ostride = n1 * cpr;                              // chunks per plane
        const uint64_t* osrc0 = a.offsets + (y0 + lane) * cpr + 4 * s;  // this lane's row, plane 0
        const bool tail = row_ok && (y0 + lane == n1 - 1) && (4 * s + nch == cpr);   // ends the index
        const uint64_t pay_end = payload_end(a.offsets, a.n_chunks, a.len);
        auto oissue = [&](int64_t zz) {
            const int os = (int)(zz % LR_OD);
            if (row_ok) {
                const uint64_t* src = osrc0 + zz * ostride;
                uint64_t* dst = OR + (os * LR_DROWS + lane) * 6;
                cp_async16(dst, src);
                cp_async16(dst + 2, src + 2);
                if (!(tail && zz == nz - 1)) cp_async16(dst + 4, src + 4);
            }
            cp_async_arrive_noinc(&o_full[os]);
        };
        for (int64_t zz = 0; zz < LR_OD && zz < nz; zz++) oissue(zz);
        const uint32_t rowoff = (uint32_t)lane * a.pr;
        for (int64_t zz = 0; zz < nz; zz++) {
            const int slot = (int)(zz % LR_D);
            if (zz >= LR_D) mbar_wait(&s_empty[slot], (uint32_t)((zz / LR_D - 1) & 1));
            const int os = (int)(zz % LR_OD);
            mbar_wait(&o_full[os], (uint32_t)((zz / LR_OD) & 1));
            uint8_t* sp = SL + (size_t)slot * a.slot;
            if (row_ok) {
                const uint64_t* ob = OR + (os * LR_DROWS + lane) * 6;
                const uint64_t o0 = ob[0];
                const uint64_t end = (tail && zz == nz - 1) ? pay_end : ob[nch];
                const uint64_t base = o0 & ~(uint64_t)15;
                const uint32_t b0 = (uint32_t)(o0 - base) + rowoff;
                uint4 rl;
                rl.x = b0;
                rl.y = (uint32_t)(ob[1] - o0) + b0;
                rl.z = (uint32_t)(ob[2] - o0) + b0;
                rl.w = (uint32_t)(ob[3] - o0) + b0;
                *reinterpret_cast<uint4*>(sp + lr_rel_off(a.pr) + 16 * lane) = rl;
                const int nv = (int)((uint32_t)(end - base + 15) >> 4);
                uint8_t* dst = sp + rowoff;
                const uint8_t* src = a.payload + base;
                for (int v = 0; v < nv; v++) cp_async16(dst + 16 * v, src + 16 * v);
            }
            cp_async_arrive_noinc(&s_full[slot]);
            __syncwarp();
            if (lane == 0) mbar_arrive(&s_full[slot]);        // publishes the rel table (generic stores)
            if (zz + LR_OD < nz) oissue(zz + LR_OD);         // refill the offsets slot just read
        }
        return;
    }

    if (wp == 1) {
        // ============================ loader, band offsets ============================
        // the band-offset row (x0-4 .. x0+132) and the strip edges of every plane
        const int anv = (int)(xe - xs) / 4;
        const int32_t* asrc = a.A + b * n2 + xs;
        const int64_t astride = a.nb * n2;
        const int32_t* esrc = a.EF + (s * ef_rows(n1) + y0) * 2;
        const int64_t estride = a.nstrips * ef_rows(n1) * 2;
        const uint32_t aoff = lr_a_off(a.pr) + (uint32_t)(xs - (x0 - 4)) * 4, eoff = lr_ef_off(a.pr);
        for (int64_t zz = 0; zz < nz; zz++) {
            const int slot = (int)(zz % LR_D);
            if (zz >= LR_D) mbar_wait(&s_empty[slot], (uint32_t)((zz / LR_D - 1) & 1));
            uint8_t* sp = SL + (size_t)slot * a.slot;
            const int32_t* as = asrc + zz * astride;
            int32_t* ad = reinterpret_cast<int32_t*>(sp + aoff);
            for (int v = lane; v < anv; v += 32) cp_async16(ad + 4 * v, as + 4 * v);
            if (lane < LR_EFN / 4) cp_async16(reinterpret_cast<int32_t*>(sp + eoff) + 4 * lane, esrc + zz * estride + 4 * lane);
            cp_async_arrive_noinc(&s_full[slot]);
        }
        return;
    }

    if (wp <= 1 + LR_DT / 32) {
        // ================================ decoders ================================
        // decode quarter-chunk jobs (a half-warp per row) and prefix the rows into RB[zz & 1]
        const int dt = threadIdx.x - 64;
        for (int64_t zz = 0; zz < nz; zz++) {
            const int slot = (int)(zz % LR_D);
            const int rb = (int)(zz & 1);
            mbar_wait(&s_full[slot], (uint32_t)((zz / LR_D) & 1));
            if (zz >= 2) mbar_wait(&rb_empty[rb], (uint32_t)(((zz >> 1) - 1) & 1));
            const uint8_t* sp = SL + (size_t)slot * a.slot;
            const uint32_t* pw = reinterpret_cast<const uint32_t*>(sp);
            const uint32_t* rel = reinterpret_cast<const uint32_t*>(sp + lr_rel_off(a.pr));
            const int32_t* EF = reinterpret_cast<const int32_t*>(sp + lr_ef_off(a.pr));
            int32_t* R = RB + rb * LR_DROWS * LR_TX;
#pragma unroll
            for (int pass = 0; pass < (LR_DROWS * 16 + LR_DT - 1) / LR_DT; pass++) {
                const int i = dt + pass * LR_DT;
                if (pass > 0 && (i & ~31) >= LR_DROWS * 16) break;        // warp-uniform: no jobs left
                const int r = i >> 4, qj = i & 15, kq = qj >> 2;
                const bool ok = r < nrow && kq < nch;
                uint32_t v[8];
                uint32_t t = 0;
                if (ok) {
                    int4 lo, hi;
                    decode8(pw, rel[4 * r + kq], qj & 3, 0, lo, hi);
                    v[0] = (uint32_t)lo.x;
                    v[1] = v[0] + (uint32_t)lo.y;
                    v[2] = v[1] + (uint32_t)lo.z;
                    v[3] = v[2] + (uint32_t)lo.w;
                    v[4] = v[3] + (uint32_t)hi.x;
                    v[5] = v[4] + (uint32_t)hi.y;
                    v[6] = v[5] + (uint32_t)hi.z;
                    v[7] = v[6] + (uint32_t)hi.w;
                    t = v[7];
                }
                uint32_t inc = t;
#pragma unroll
                for (int d = 1; d < 16; d <<= 1) {
                    const uint32_t w = __shfl_up_sync(0xffffffffu, inc, d, 16);
                    if ((lane & 15) >= d) inc += w;
                }
                if (ok) {
                    const uint32_t base = (uint32_t)EF[2 * r] + inc - t;   // row prefix before this job
                    int32_t* dst = R + r * LR_TX + 8 * qj;
                    *reinterpret_cast<int4*>(dst) = make_int4((int)(base + v[0]), (int)(base + v[1]),
                                                              (int)(base + v[2]), (int)(base + v[3]));
                    *reinterpret_cast<int4*>(dst + 4) = make_int4((int)(base + v[4]), (int)(base + v[5]),
                                                                  (int)(base + v[6]), (int)(base + v[7]));
                }
            }
            mbar_arrive(&s_empty[slot]);
            mbar_arrive(&rb_full[rb]);
        }
        return;
    }

    if (wp <= 1 + (LR_DT + LR_ST) / 32) {
        // ================================ scanners ================================
        // column prefix from the band offsets (y) + the previous q plane (z): thread st < 128 owns
        // column x0+st, st == 128 / 129 the halo columns x0-1 / x0+128 (their R comes from E / F)
        const int st = threadIdx.x - 64 - LR_DT;
        constexpr int C4 = LR_AW / 4;
        auto copy_plane = [&](const int32_t* g, int32_t* P) {
            for (int i = st; i < LR_ROWS * C4; i += LR_ST) {
                const int r = i / C4, j = 4 * (i - r * C4);
                const int64_t y = y0 - 1 + r, x = x0 - 4 + j;
                int4 v = make_int4(0, 0, 0, 0);
                if (g && y >= 0 && y < n1 && x >= 0 && x < n2) v = ld4(g + y * n2 + x);
                *reinterpret_cast<int4*>(P + r * LR_RW + LR_X0 - 4 + j) = v;
            }
        };
        copy_plane(a.carry, Q);                                        // plane -1 in slot 0
        mbar_arrive(&q_full[0]);
        const bool edge = st >= LR_TX;
        const int which = st - LR_TX;                                  // 0: left halo, 1: right halo
        bool colok;
        int col, jx;
        if (!edge) {
            colok = x0 + st < n2;
            col = LR_X0 + st;
            jx = 4 + st;
        } else {
            colok = which == 0 ? x0 > 0 : (which == 1 && x0 + LR_TX < n2);
            col = which == 0 ? LR_X0 - 1 : LR_X0 + LR_TX;
            jx = which == 0 ? 3 : 4 + LR_TX;
        }
        for (int64_t zz = 0; zz <= nz; zz++) {
            const int qs = (int)((zz + 1) % LR_NPL);
            const int64_t u = (zz + 1) / LR_NPL;
            if (u > 0) mbar_wait(&q_empty[qs], (uint32_t)((u - 1) & 1));
            int32_t* Pn = Q + qs * LR_PLANE;
            if (zz == nz) {                                             // the plane above the slab
                copy_plane(a.q_upper, Pn);
                mbar_arrive(&q_full[qs]);
                break;
            }
            const int slot = (int)(zz % LR_D);
            const int rb = (int)(zz & 1);
            mbar_wait(&rb_full[rb], (uint32_t)((zz >> 1) & 1));          // implies the slot's data landed
            const uint8_t* sp = SL + (size_t)slot * a.slot;
            const int32_t* SA = reinterpret_cast<const int32_t*>(sp + lr_a_off(a.pr));
            const int32_t* EF = reinterpret_cast<const int32_t*>(sp + lr_ef_off(a.pr));
            const int32_t* R = RB + rb * LR_DROWS * LR_TX;
            const int32_t* Pp = Q + (int)(zz % LR_NPL) * LR_PLANE;
            if (colok) {
                const uint32_t av = (uint32_t)SA[jx];
                if (y0 > 0) Pn[col] = (int)((uint32_t)Pp[col] + av);     // halo row y0-1: P2 = A
                uint32_t run = 0;
#pragma unroll
                for (int r = 0; r < LR_DROWS; r++) {
                    if (r < nrow) {
                        run += edge ? (uint32_t)EF[2 * r + which] : (uint32_t)R[r * LR_TX + st];
                        const int o = (r + 1) * LR_RW + col;
                        Pn[o] = (int)((uint32_t)Pp[o] + av + run);
                    }
                }
            }
            mbar_arrive(&rb_empty[rb]);
            mbar_arrive(&s_empty[slot]);
            mbar_arrive(&q_full[qs]);
        }
        return;
    }

    // ================================ emitters ================================
    const int cw = wp - 2 - (LR_DT + LR_ST) / 32;
    const float epsf = __double2float_rn(a.eps), two_epsf = 2.0f * epsf;
    const double two_eps = 2.0 * a.eps;
    WinStats st;
    st.init();
    int64_t count = 0;
    const int64_t x = x0 + 4 * lane;
    auto wait_q = [&](int64_t zz) {
        mbar_wait(&q_full[(int)((zz + 1) % LR_NPL)], (uint32_t)(((zz + 1) / LR_NPL) & 1));
    };
    wait_q(-1);
    wait_q(0);
    for (int64_t z = 0; z < nz; z++) {
        wait_q(z + 1);
        const int32_t* Pm = Q + (int)(z % LR_NPL) * LR_PLANE;
        const int32_t* Pc = Q + (int)((z + 1) % LR_NPL) * LR_PLANE;
        const int32_t* Pp = Q + (int)((z + 2) % LR_NPL) * LR_PLANE;
        const int64_t gz = a.gz0 + z;
        const bool zin = gz > 0 && gz < a.gN0 - 1;
#pragma unroll
        for (int k = 0; k < 2; k++) {
            const int r = 2 * cw + k;
            const int64_t y = y0 + r;
            const int so = (r + 1) * LR_RW + LR_X0 + 4 * lane;
            const int4 c = *reinterpret_cast<const int4*>(Pc + so);
            int left = __shfl_up_sync(0xffffffffu, c.w, 1);
            int right = __shfl_down_sync(0xffffffffu, c.x, 1);
            if (lane == 0) left = Pc[so - 1];
            if (lane == 31) right = Pc[so + 4];
            if (y < n1 && x < n2) {
                const bool yin = y > 0 && y < n1 - 1;
                const int4 ym = *reinterpret_cast<const int4*>(Pc + so - LR_RW);
                const int4 yp = *reinterpret_cast<const int4*>(Pc + so + LR_RW);
                const int4 zm = *reinterpret_cast<const int4*>(Pm + so);
                const int4 zp = *reinterpret_cast<const int4*>(Pp + so);
                const int64_t o = z * plane + y * n2 + x;
                if (Exact)
                    emit4(a.o0, a.o1, a.o2, a.o3, o, zin, yin, x, n2, zm, c, zp, ym, yp, left, right, a.eps,
                          two_eps);
                else if (zin && yin)
                    emit4f(a.o0, a.o1, a.o2, a.o3, o, true, true, x, n2, zm, c, zp, ym, yp, left, right, a.eps,
                           two_eps, epsf, two_epsf);
                else
                    emit4f(a.o0, a.o1, a.o2, a.o3, o, zin, yin, x, n2, zm, c, zp, ym, yp, left, right, a.eps,
                           two_eps, epsf, two_epsf);
                if (Exact) st.add4(c);                    // stats always kept (acc may be null)
                else st.add4f(c);
                count += 4;
            }
        }
        if (!Exact && (z & 15) == 15) st.fold();
        mbar_arrive(&q_empty[(int)(z % LR_NPL)]);
    }
    if (a.acc) st.flush(a.acc, count);
}

}  // namespace hszg

using namespace hszg;

int hszg_set_cuda_error(HszgErr* err, cudaError_t e, const char* where);

static bool al16l(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

extern "C" int hszg_lorenzo_onepass(const HszgGeom* g, const HszgStream* s, const int32_t* band_off,
                                    const int32_t* strip_edges, const int32_t* carry, const int32_t* q_upper,
                                    int64_t gz0, int64_t gN0, float* const* out, HszgAcc* acc, int exact,
                                    void* stream, HszgErr* err) {
    err->status = HSZG_OK;
    const int64_t nz = g->dims[0], n1 = g->dims[1], n2 = g->dims[2];
    const size_t smem = lr_smem(s->max_bitwidth);
    if (g->kind != HSZG_HSZP_ND || g->ndims != 3 || !s->canonical || n2 % 64 || n2 > 4096 || !al16l(s->offsets) ||
        smem > 227 * 1024 - 2048 || !al16l(s->payload) || !al16l(band_off) || !al16l(strip_edges) ||
        !al16l(out[0]) || !al16l(out[1]) || !al16l(out[2]) || !al16l(out[3]) || (carry && !al16l(carry)) ||
        (q_upper && !al16l(q_upper)) || !band_off || !strip_edges) {
        err->status = HSZG_INVALID_ARG;
        snprintf(err->message, sizeof(err->message),
                 "lorenzo_onepass: need canonical 3-D HSZP_ND, n2 %% 64 == 0, n2 <= 4096, band/edge tables, "
                 "16-B alignment (max bw %d)", s->max_bitwidth);
        return HSZG_INVALID_ARG;
    }
    if (g->n == 0) return HSZG_OK;
    LrArgs a;
    a.payload = s->payload;
    a.len = s->payload_len;
    a.offsets = s->offsets;
    a.n_chunks = g->n_chunks;
    a.nz = nz;
    a.n1 = n1;
    a.n2 = n2;
    a.nb = (n1 + LR_TY - 1) / LR_TY;
    a.nstrips = (n2 + LR_TX - 1) / LR_TX;
    a.A = band_off;
    a.EF = strip_edges;
    a.carry = carry;
    a.q_upper = q_upper;
    a.gz0 = gz0;
    a.gN0 = gN0;
    a.eps = g->eps;
    a.o0 = out[0];
    a.o1 = out[1];
    a.o2 = out[2];
    a.o3 = out[3];
    a.acc = acc;
    a.pr = lr_pr(s->max_bitwidth);
    a.slot = lr_slot(s->max_bitwidth);
    dim3 grid((unsigned)a.nstrips, (unsigned)a.nb);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (exact) {
        allow_smem(k_lorenzo_ring<true>, smem);
        k_lorenzo_ring<true><<<grid, LR_T, smem, st>>>(a);
    } else {
        allow_smem(k_lorenzo_ring<false>, smem);
        k_lorenzo_ring<false><<<grid, LR_T, smem, st>>>(a);
    }
    { const cudaError_t e_ = cudaGetLastError(); if (e_ != cudaSuccess) return hszg_set_cuda_error(err, e_, "lorenzo_onepass"); }
    return HSZG_OK;
}
