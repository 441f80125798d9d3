// lorenzo.cu — HSZP_ND in one pass: decode + Lorenzo inversion (x, y, z prefix) + gradient +
// Laplacian + exact statistics, q never in HBM.  compressors.py:201-226 (q = cumsum of p along
// every axis) fused with fields.py:34-80.
//
// Pre-pass (hszg_band_scan with bands of 16 rows, no L): per plane z, the exclusive band offsets
// A[z][b][x] = sum of the x-prefixed rows above band b (= P2 at the row above it), and per 128-wide
// strip s and row y the row prefix just left / right of the strip, E = R(128s-1), F = R(128s+128).
// Main kernel: a CTA owns x in [128s, 128s+128) by y in [16b, 16b+16) and slides along z over the
// whole slab.  Per plane:
//   warp 0      TMA-loads the payload bytes of the 17 rows y0..y0+16 restricted to the strip's 4
//               chunks, the band-offset row A[z][b] and the strip edges (and writes the chunk
//               offsets, prefetched a plane ahead, into the staging slot);
//   warps 1-8   decode quarter-chunk jobs and prefix each row (half-warp scan + E) into R, then
//               run the column prefix from A[z][b] (y) and add the previous q plane (z) —
//               P2[y][x] = A[b][x] + sum_{y0<=y'<=y} R[y'][x], q[z] = q[z-1] + P2[z]; the halo
//               columns x0-1 / x0+128 come from E / F, the halo row y0-1 from A alone;
//   warps 9-16  emit from the q ring (as fused.cu / zring.cu).
#include <cstdio>
#include "tile.cuh"
#include "stencil.cuh"
#include "async.cuh"

namespace hszg {

constexpr int LR_T = 544;
constexpr int LR_DT = 256;                  // decoders: warps 1-8
constexpr int LR_CT = 256;                  // emitters: warps 9-16, 2 rows each
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
    return (size_t)LR_NPL * LR_PLANE * 4 + (size_t)LR_D * lr_slot(max_bw) + (size_t)LR_DROWS * LR_TX * 4;
}

// strip-edge table rows per (plane, strip): even, so every (plane, strip) block starts 16-B aligned
__host__ __device__ inline int64_t ef_rows(int64_t n1) { return (n1 + 1) & ~(int64_t)1; }

__device__ __forceinline__ void decoder_sync() { asm volatile("bar.sync 1, %0;" ::"n"(LR_DT) : "memory"); }

template <bool Exact>
__global__ void __launch_bounds__(LR_T, 1) k_lorenzo_ring(LrArgs a) {
    extern __shared__ __align__(128) uint8_t lsm[];
    int32_t* Q = reinterpret_cast<int32_t*>(lsm);                         // [NPL][ROWS][RW]
    uint8_t* SL = lsm + (size_t)LR_NPL * LR_PLANE * 4;                    // [D][slot]
    int32_t* RB = reinterpret_cast<int32_t*>(SL + (size_t)LR_D * a.slot);  // [DROWS][TX]
    __shared__ __align__(8) uint64_t s_full[LR_D], s_empty[LR_D], q_full[LR_NPL], q_empty[LR_NPL], o_full[LR_OD];
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
            mbar_init(&s_full[i], 33);                // 32 cp.async completions + the rel-table arrive
            mbar_init(&s_empty[i], LR_DT);
        }
        for (int i = 0; i < LR_NPL; i++) {
            mbar_init(&q_full[i], LR_DT);
            mbar_init(&q_empty[i], LR_CT);
        }
        for (int i = 0; i < LR_OD; i++) mbar_init(&o_full[i], 32);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (wp == 0) {
        // ================================ loader ================================
        const bool row_ok = lane < nrow;
        // Lane-parallel 16-B async copies (cp.async, completion tracked by the mbarriers): per plane
        // ~30 small pieces, which one elected lane would otherwise issue one TMA at a time.
        // Chunk offsets of this lane's row arrive LR_OD planes ahead (6 entries from an even chunk
        // index: the strip's 4 starts + the end; 4 entries at the index's end, where the end is the
        // payload end).
        auto oissue = [&](int64_t zz) {
            const int os = (int)(zz % LR_OD);
            if (row_ok) {
                const int64_t c0 = (zz * n1 + y0 + lane) * cpr + 4 * s;
                const int nv = c0 + 6 <= a.n_chunks ? 3 : 2;
                uint64_t* dst = OR + (os * LR_DROWS + lane) * 6;
                for (int v = 0; v < nv; v++) cp_async16(dst + 2 * v, a.offsets + c0 + 2 * v);
            }
            cp_async_arrive_noinc(&o_full[os]);
        };
        for (int64_t zz = 0; zz < LR_OD && zz < nz; zz++) oissue(zz);
        const int anv = (int)(xe - xs) / 4;               // 16-B vectors of the band-offset row
        for (int64_t zz = 0; zz < nz; zz++) {
            const int slot = (int)(zz % LR_D);
            const int64_t u = zz / LR_D;
            if (u > 0) mbar_wait(&s_empty[slot], (uint32_t)((u - 1) & 1));
            const int os = (int)(zz % LR_OD);
            mbar_wait(&o_full[os], (uint32_t)((zz / LR_OD) & 1));
            uint64_t o[5];
#pragma unroll
            for (int k = 0; k < 5; k++) o[k] = OR[(os * LR_DROWS + lane) * 6 + k];
            uint8_t* sp = SL + (size_t)slot * a.slot;
            if (row_ok) {
                const int64_t c0 = (zz * n1 + y0 + lane) * cpr + 4 * s;
                const uint64_t end = c0 + nch < a.n_chunks
                                         ? (nch == 4 ? o[4] : nch == 3 ? o[3] : nch == 2 ? o[2] : o[1])
                                         : payload_end(a.offsets, a.n_chunks, a.len);
                const uint64_t base = o[0] & ~(uint64_t)15;
                const int nv = (int)((end - base + 15) >> 4);
                uint32_t* rel = reinterpret_cast<uint32_t*>(sp + lr_rel_off(a.pr)) + 4 * lane;
#pragma unroll
                for (int k = 0; k < 4; k++)
                    if (k < nch) rel[k] = (uint32_t)(o[k] - base) + (uint32_t)lane * a.pr;
                uint8_t* dst = sp + (size_t)lane * a.pr;
                const uint8_t* src = a.payload + base;
                for (int v = 0; v < nv; v++) cp_async16(dst + 16 * v, src + 16 * v);
            } else {
                // the other lanes: the band-offset row (x0-4 .. x0+132) and the strip edges
                const int l = lane - nrow, nl = 32 - nrow;
                const int32_t* asrc = a.A + (zz * a.nb + b) * n2 + xs;
                int32_t* adst = reinterpret_cast<int32_t*>(sp + lr_a_off(a.pr)) + (xs - (x0 - 4));
                for (int v = l; v < anv; v += nl) cp_async16(adst + 4 * v, asrc + 4 * v);
                const int32_t* esrc = a.EF + ((zz * a.nstrips + s) * ef_rows(n1) + y0) * 2;
                int32_t* edst = reinterpret_cast<int32_t*>(sp + lr_ef_off(a.pr));
                for (int v = l; v < LR_EFN / 4; v += nl) cp_async16(edst + 4 * v, esrc + 4 * v);
            }
            cp_async_arrive_noinc(&s_full[slot]);
            __syncwarp();
            if (lane == 0) mbar_arrive(&s_full[slot]);        // publishes the rel table (generic stores)
            if (zz + LR_OD < nz) oissue(zz + LR_OD);         // refill the offsets slot just read
        }
        return;
    }

    if (wp <= LR_DT / 32) {
        // ================================ decoders ================================
        const int dt = threadIdx.x - 32;
        constexpr int C4 = LR_AW / 4;
        auto copy_plane = [&](const int32_t* g, int32_t* P) {
            for (int i = dt; i < LR_ROWS * C4; i += LR_DT) {
                const int r = i / C4, j = 4 * (i - r * C4);
                const int64_t y = y0 - 1 + r, x = x0 - 4 + j;
                int4 v = make_int4(0, 0, 0, 0);
                if (g && y >= 0 && y < n1 && x >= 0 && x < n2) v = ld4(g + y * n2 + x);
                *reinterpret_cast<int4*>(P + r * LR_RW + LR_X0 - 4 + j) = v;
            }
        };
        copy_plane(a.carry, Q);                                        // plane -1 in slot 0
        mbar_arrive(&q_full[0]);
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
            mbar_wait(&s_full[slot], (uint32_t)((zz / LR_D) & 1));
            const uint8_t* sp = SL + (size_t)slot * a.slot;
            const uint32_t* pw = reinterpret_cast<const uint32_t*>(sp);
            const uint32_t* rel = reinterpret_cast<const uint32_t*>(sp + lr_rel_off(a.pr));
            const int32_t* SA = reinterpret_cast<const int32_t*>(sp + lr_a_off(a.pr));
            const int32_t* EF = reinterpret_cast<const int32_t*>(sp + lr_ef_off(a.pr));
            // -- 1. decode quarter-chunk jobs (a half-warp per row) and prefix the rows into RB
            decoder_sync();                                             // RB of the previous plane consumed
#pragma unroll
            for (int pass = 0; pass < (LR_DROWS * 16 + LR_DT - 1) / LR_DT; pass++) {
                const int i = dt + pass * LR_DT;
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
                    int32_t* dst = RB + r * LR_TX + 8 * qj;
                    *reinterpret_cast<int4*>(dst) = make_int4((int)(base + v[0]), (int)(base + v[1]),
                                                              (int)(base + v[2]), (int)(base + v[3]));
                    *reinterpret_cast<int4*>(dst + 4) = make_int4((int)(base + v[4]), (int)(base + v[5]),
                                                                  (int)(base + v[6]), (int)(base + v[7]));
                }
            }
            decoder_sync();
            // -- 2. column prefix from the band offsets (y) + previous plane (z), one column per thread
            const int32_t* Pp = Q + (int)(zz % LR_NPL) * LR_PLANE;
            // thread dt < 128: column x0+dt; dt == 128 / 129: the halo columns x0-1 / x0+128 (from E / F)
            const bool edge = dt >= LR_TX;
            const int which = dt - LR_TX;                          // 0: left halo, 1: right halo
            bool colok;
            int col, jx;
            if (!edge) {
                colok = x0 + dt < n2;
                col = LR_X0 + dt;
                jx = 4 + dt;
            } else {
                colok = which == 0 ? x0 > 0 : (which == 1 && x0 + LR_TX < n2);
                col = which == 0 ? LR_X0 - 1 : LR_X0 + LR_TX;
                jx = which == 0 ? 3 : 4 + LR_TX;
            }
            if (colok) {
                const uint32_t av = (uint32_t)SA[jx];
                if (y0 > 0) Pn[col] = (int)((uint32_t)Pp[col] + av);     // halo row y0-1: P2 = A
                uint32_t run = 0;
#pragma unroll
                for (int r = 0; r < LR_DROWS; r++) {
                    if (r < nrow) {
                        run += edge ? (uint32_t)EF[2 * r + which] : (uint32_t)RB[r * LR_TX + dt];
                        const int o = (r + 1) * LR_RW + col;
                        Pn[o] = (int)((uint32_t)Pp[o] + av + run);
                    }
                }
            }
            mbar_arrive(&s_empty[slot]);
            mbar_arrive(&q_full[qs]);
        }
        return;
    }

    // ================================ emitters ================================
    const int cw = wp - 1 - LR_DT / 32;
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
                if (a.acc) {
                    if (Exact) st.add4(c);
                    else st.add4f(c);
                }
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
    if (cudaGetLastError() != cudaSuccess) return hszg_set_cuda_error(err, cudaGetLastError(), "lorenzo_onepass");
    return HSZG_OK;
}
