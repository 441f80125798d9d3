// zring.cu — HSZP_ND z-sweep, warp-specialised (the default HSZP_ND analytics pass after
// hszg_band_scan).  Semantics of window.cu's k_zsweep: q[z] = q[z-1] + P2[z] with
// P2[z][y] = L[z][y] + A[z][y / BR] (band-local 2-D prefix + band offsets), gradient + Laplacian +
// exact statistics of planes [a, a+nout), q[a+nout-1] handed to the next window.
//
// A CTA owns 128 x by 16 y (+ halo rows y0-1, y0+16 and columns x0-1, x0+128) and slides along z:
//   warp 0      TMA-loads, ZR_D planes ahead, the 18 L rows and the <= 3 band-offset rows it needs;
//   warps 1-3   add them onto the previous q plane (ring of ZR_NPL q planes in shared memory);
//   warps 4-11  emit the 7-point stencils + stats from the ring (the same emitter as fused.cu).
// mbarriers: s_full / s_empty hand the staging slots between loader and adders, q_full / q_empty
// the q planes between adders and emitters.  q never goes to HBM (except the window carry).
#include <cstdio>
#include <type_traits>
#include "tile.cuh"
#include "stencil.cuh"
#include "async.cuh"

namespace hszg {

constexpr int ZR_T = 384;
constexpr int ZR_AT = 96;                   // adders: warps 1-3
constexpr int ZR_CT = 256;                  // emitters: warps 4-11, 2 rows each
constexpr int ZR_TY = 16;                   // output rows per CTA
constexpr int ZR_TX = 128;                  // output columns per CTA
constexpr int ZR_ROWS = ZR_TY + 2;          // q ring rows: y0-1 .. y0+16
constexpr int ZR_X0 = 8;                    // q ring column of x0
constexpr int ZR_RW = 148;                  // q ring row words (odd 16-B stride)
constexpr int ZR_PLANE = ZR_ROWS * ZR_RW;
constexpr int ZR_NPL = 4;                   // q planes in the ring
constexpr int ZR_D = 4;                     // staged P2 planes in flight
constexpr int ZR_SW = ZR_TX + 8;            // staged int32 row: x0-4 .. x0+132
constexpr int ZR_SW16 = ZR_TX + 16;         // staged int16 row: x0-8 .. x0+136 (16-B aligned ends)
constexpr int ZR_SW8 = ZR_TX + 32;          // staged int8 row: x0-16 .. x0+144 (16-B aligned ends)
constexpr int ZR_SROWS = ZR_ROWS + 3;       // 18 L rows + band-offset rows (above, tile, below)
// staged L row of width lw bytes per value: first column, value count, bytes
__host__ __device__ constexpr int zr_lead(int lw) { return lw == 4 ? 4 : (lw == 2 ? 8 : 16); }
__host__ __device__ constexpr int zr_row_vals(int lw) { return lw == 4 ? ZR_SW : (lw == 2 ? ZR_SW16 : ZR_SW8); }
__host__ __device__ constexpr int zr_lrow_bytes(int lw) { return zr_row_vals(lw) * lw; }
__host__ __device__ constexpr int zr_max(int a, int b) { return a > b ? a : b; }
// staging slot: 18 L rows (row stride = the wider of the L and lookahead rows) + 3 int32 band-offset rows
__host__ __device__ constexpr int zr_lb(int lw, int law) { return zr_max(zr_lrow_bytes(lw), zr_lrow_bytes(law)); }
__host__ __device__ constexpr int zr_slot_bytes(int lw, int law) { return ZR_ROWS * zr_lb(lw, law) + 3 * ZR_SW * 4; }
constexpr size_t zr_smem(int lw, int law, int em = EM_FAST) {
    return (size_t)ZR_NPL * ZR_PLANE * 4 + (size_t)ZR_D * zr_slot_bytes(lw, law) + (em == EM_TABLE ? XT_BYTES : 0);
}

struct ZrArgs {
    const void* L;                          // band-local 2-D prefixes: int32, int16 or int8 (LW bytes)
    const void* lookahead;
    const int32_t* carry;
    const int32_t* q_upper;
    int32_t* carry_out;
    const int32_t* A;
    const int32_t* lookA;
    int64_t n1, n2, nout, gz0, gN0, BR, nb;
    double eps;
    float* o0;
    float* o1;
    float* o2;
    float* o3;
    HszgAcc* acc;
};

// LW: bytes per L value of the window's planes, LAW: of the lookahead plane (the next window's first,
// which may be narrower: int16 window 0 + int8 rest)
// 64 registers (no spills): two sweep CTAs (2 x 12 warps x 2048 regs) leave exactly one k_band_scan
// CTA's 16 K registers free, so the side stream's band scans co-reside with the sweeps instead of
// waiting for a whole SM slot (at 72 registers they could not).
template <int EM, int LW, int LAW>
__global__ void __maxnreg__(64) k_zsweep_ring(ZrArgs a) {
    constexpr bool Exact = EM == EM_EXACT;
    extern __shared__ __align__(128) int32_t zsm[];
    int32_t* Q = zsm;                                     // [ZR_NPL][ZR_ROWS][ZR_RW]
    uint8_t* S = reinterpret_cast<uint8_t*>(zsm + ZR_NPL * ZR_PLANE);   // [ZR_D][slot]
    constexpr int LB = zr_lb(LW, LAW), SLOT = zr_slot_bytes(LW, LAW);
    __shared__ __align__(8) uint64_t s_full[ZR_D], s_empty[ZR_D], q_full[ZR_NPL], q_empty[ZR_NPL];
    const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
    const int64_t x0 = (int64_t)blockIdx.x * ZR_TX, y0 = (int64_t)blockIdx.y * ZR_TY;
    const int64_t n1 = a.n1, n2 = a.n2, nout = a.nout;
    const int64_t plane = n1 * n2;
    const int64_t xs = x0 >= 4 ? x0 - 4 : 0;
    const int64_t xe = x0 + ZR_TX + 4 < n2 ? x0 + ZR_TX + 4 : n2;
    const int scol = (int)(xs - (x0 - 4));                // staged column of xs
    // the tile rows share band y0 / BR (BR % 16 == 0); the halo rows may sit in the neighbours
    const int64_t band[3] = {y0 > 0 ? (y0 - 1) / a.BR : -1, y0 / a.BR, y0 + ZR_TY < n1 ? (y0 + ZR_TY) / a.BR : -1};
    const bool has_look = a.lookahead != nullptr && a.q_upper == nullptr;
    const int64_t nst = nout + (has_look ? 1 : 0);         // staged planes

    for (int i = threadIdx.x; i < (int)(zr_smem(LW, LAW) / 16); i += ZR_T) reinterpret_cast<int4*>(zsm)[i] = make_int4(0, 0, 0, 0);
    float* XT = reinterpret_cast<float*>(S + (size_t)ZR_D * SLOT);        // EM_TABLE: after the staging slots
    if (EM == EM_TABLE) xtable_fill(XT, a.eps, threadIdx.x, ZR_T);
    if (threadIdx.x == 0) {
        for (int i = 0; i < ZR_D; i++) {
            mbar_init(&s_full[i], 1);
            mbar_init(&s_empty[i], ZR_AT);
        }
        for (int i = 0; i < ZR_NPL; i++) {
            mbar_init(&q_full[i], ZR_AT);
            mbar_init(&q_empty[i], ZR_CT);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (wp == 0) {
        // ================================ loader ================================
        const uint32_t rbytes = (uint32_t)(xe - xs) * 4;
        const int64_t y = y0 - 1 + lane;                  // lanes 0..17: L rows; 18..20: band rows
        // one L row of width w bytes per value: source element offset, bytes, staging offset
        struct Row {
            int64_t off;
            uint32_t bytes, dst;
        };
        auto lrow = [&](int w) {
            const int lead = zr_lead(w);
            const int64_t s0 = x0 >= lead ? x0 - lead : 0;
            const int64_t s1 = x0 + ZR_TX + lead < n2 ? x0 + ZR_TX + lead : n2;
            return Row{y * n2 + s0, (uint32_t)(s1 - s0) * w, (uint32_t)lane * LB + (uint32_t)(s0 - (x0 - lead)) * w};
        };
        bool ok;
        Row rw, ra;                                       // the window's planes / the lookahead plane
        if (lane < ZR_ROWS) {
            ok = y >= 0 && y < n1;
            rw = lrow(LW);
            ra = lrow(LAW);
        } else if (lane < ZR_SROWS) {
            const int bi = lane - ZR_ROWS;                 // select, not a dynamically indexed array
            const int64_t bnd = bi == 0 ? band[0] : (bi == 1 ? band[1] : band[2]);
            ok = bnd >= 0;
            rw.off = bnd * n2 + xs;
            rw.bytes = rbytes;
            rw.dst = ZR_ROWS * LB + (lane - ZR_ROWS) * ZR_SW * 4 + (uint32_t)scol * 4;
            ra = rw;
        } else {
            ok = false;
            rw = ra = Row{0, 0, 0};
        }
        uint32_t txw = ok ? rw.bytes : 0, txa = ok ? ra.bytes : 0;
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
            txw += __shfl_xor_sync(0xffffffffu, txw, d);
            txa += __shfl_xor_sync(0xffffffffu, txa, d);
        }
        for (int64_t zz = 0; zz < nst; zz++) {
            const int slot = (int)(zz % ZR_D);
            const int64_t u = zz / ZR_D;
            const bool look = zz >= nout;
            if (u > 0) mbar_wait(&s_empty[slot], (uint32_t)((u - 1) & 1));
            if (lane == 0) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mbar_arrive_tx(&s_full[slot], look ? txa : txw);
            }
            __syncwarp();
            if (ok) {
                const int64_t roff = look ? ra.off : rw.off;       // by value: no stack copy of the rows
                const uint32_t rbytes_ = look ? ra.bytes : rw.bytes, rdst = look ? ra.dst : rw.dst;
                const uint8_t* src;
                if (lane < ZR_ROWS)
                    src = static_cast<const uint8_t*>(look ? a.lookahead : a.L) +
                          ((look ? 0 : zz * plane) + roff) * (look ? LAW : LW);
                else
                    src = reinterpret_cast<const uint8_t*>((look ? a.lookA : a.A + zz * a.nb * n2) + roff);
                tma_load_1d(S + (size_t)slot * SLOT + rdst, src, rbytes_, &s_full[slot]);
            }
        }
        return;
    }

    if (wp < 1 + ZR_AT / 32) {
        // ================================ adders ================================
        const int at = threadIdx.x - 32;
        constexpr int C4 = ZR_SW / 4;                      // int4 columns x0-4 .. x0+132
        // plane a-1 (the carry) into ring slot 0, planes zz = 0..nout into slot (zz + 1) % NPL
        auto copy_plane = [&](const int32_t* g, int32_t* P) {      // g: a q plane in HBM, or null
            for (int i = at; i < ZR_ROWS * C4; i += ZR_AT) {
                const int r = i / C4, j = 4 * (i - r * C4);
                const int64_t y = y0 - 1 + r, x = x0 - 4 + j;
                int4 v = make_int4(0, 0, 0, 0);
                if (g && y >= 0 && y < n1 && x >= 0 && x < n2) v = ld4(g + y * n2 + x);
                *reinterpret_cast<int4*>(P + r * ZR_RW + ZR_X0 - 4 + j) = v;
            }
        };
        copy_plane(a.carry, Q);
        mbar_arrive(&q_full[0]);
        for (int64_t zz = 0; zz <= nout; zz++) {
            const int qs = (int)((zz + 1) % ZR_NPL);
            const int64_t u = (zz + 1) / ZR_NPL;
            if (u > 0) mbar_wait(&q_empty[qs], (uint32_t)((u - 1) & 1));
            int32_t* P = Q + qs * ZR_PLANE;
            if (zz == nout && a.q_upper) {
                copy_plane(a.q_upper, P);
            } else if (zz < nst) {
                const int slot = (int)(zz % ZR_D);
                mbar_wait(&s_full[slot], (uint32_t)((zz / ZR_D) & 1));
                const int32_t* Pprev = Q + (int)(zz % ZR_NPL) * ZR_PLANE;
                const uint8_t* St = S + (size_t)slot * SLOT;
                const int32_t* Sa = reinterpret_cast<const int32_t*>(St + ZR_ROWS * LB);
                auto add_rows = [&](auto wtag) {
                    constexpr int W = decltype(wtag)::value;
                    for (int i = at; i < ZR_ROWS * C4; i += ZR_AT) {
                        const int r = i / C4, j = 4 * (i - r * C4);
                        const int br = r == 0 ? 0 : (r == ZR_ROWS - 1 ? 2 : 1);
                        int4 l;
                        if (W == 4) {
                            l = *reinterpret_cast<const int4*>(reinterpret_cast<const int32_t*>(St + r * LB) + j);
                        } else if (W == 2) {
                            const short4 h = *reinterpret_cast<const short4*>(
                                reinterpret_cast<const int16_t*>(St + r * LB) + j + 4);
                            l = make_int4(h.x, h.y, h.z, h.w);
                        } else {
                            const char4 h = *reinterpret_cast<const char4*>(
                                reinterpret_cast<const int8_t*>(St + r * LB) + j + 12);
                            l = make_int4(h.x, h.y, h.z, h.w);
                        }
                        const int4 b = *reinterpret_cast<const int4*>(Sa + br * ZR_SW + j);
                        const int4 q = *reinterpret_cast<const int4*>(Pprev + r * ZR_RW + ZR_X0 - 4 + j);
                        *reinterpret_cast<int4*>(P + r * ZR_RW + ZR_X0 - 4 + j) = add4(q, add4(l, b));
                    }
                };
                if (LAW != LW && zz >= nout) add_rows(std::integral_constant<int, LAW>());
                else add_rows(std::integral_constant<int, LW>());
                mbar_arrive(&s_empty[slot]);
            } else {
                copy_plane(nullptr, P);                     // q[a+nout] not needed (global last plane)
            }
            mbar_arrive(&q_full[qs]);
        }
        return;
    }

    // ================================ emitters ================================
    const int cw = wp - 1 - ZR_AT / 32;                   // rows 2cw, 2cw+1
    const float epsf = __double2float_rn(a.eps), two_epsf = 2.0f * epsf;
    const double two_eps = 2.0 * a.eps;
    WinStats st;
    st.init();
    int64_t count = 0;
    const int64_t x = x0 + 4 * lane;
    auto wait_q = [&](int64_t zz) {                       // q plane zz (zz = -1: the carry)
        mbar_wait(&q_full[(int)((zz + 1) % ZR_NPL)], (uint32_t)(((zz + 1) / ZR_NPL) & 1));
    };
    wait_q(-1);
    wait_q(0);
    for (int64_t z = 0; z < nout; z++) {
        wait_q(z + 1);
        const int32_t* Pm = Q + (int)(z % ZR_NPL) * ZR_PLANE;
        const int32_t* Pc = Q + (int)((z + 1) % ZR_NPL) * ZR_PLANE;
        const int32_t* Pp = Q + (int)((z + 2) % ZR_NPL) * ZR_PLANE;
        const int64_t gz = a.gz0 + z;
        const bool zin = gz > 0 && gz < a.gN0 - 1;
#pragma unroll
        for (int k = 0; k < 2; k++) {
            const int r = 2 * cw + k;
            const int64_t y = y0 + r;
            const int so = (r + 1) * ZR_RW + ZR_X0 + 4 * lane;
            const int4 c = *reinterpret_cast<const int4*>(Pc + so);
            int left = __shfl_up_sync(0xffffffffu, c.w, 1);
            int right = __shfl_down_sync(0xffffffffu, c.x, 1);
            if (lane == 0) left = Pc[so - 1];
            if (lane == 31) right = Pc[so + 4];
            if (y < n1 && x < n2) {
                const bool yin = y > 0 && y < n1 - 1;
                const int4 ym = *reinterpret_cast<const int4*>(Pc + so - ZR_RW);
                const int4 yp = *reinterpret_cast<const int4*>(Pc + so + ZR_RW);
                const int4 zm = *reinterpret_cast<const int4*>(Pm + so);
                const int4 zp = *reinterpret_cast<const int4*>(Pp + so);
                const int64_t o = z * plane + y * n2 + x;
                if (EM == EM_EXACT)
                    emit4(a.o0, a.o1, a.o2, a.o3, o, zin, yin, x, n2, zm, c, zp, ym, yp, left, right, a.eps,
                          two_eps);
                else if (EM == EM_TABLE)
                    emit4x<OM_ALL>(a.o0, a.o1, a.o2, a.o3, o, zin, yin, x, n2, zm, c, zp, ym, yp, left, right, a.eps,
                           XT + XT_R);
                else if (zin && yin)
                    emit4f(a.o0, a.o1, a.o2, a.o3, o, true, true, x, n2, zm, c, zp, ym, yp, left, right, a.eps,
                           two_eps, epsf, two_epsf);
                else
                    emit4f(a.o0, a.o1, a.o2, a.o3, o, zin, yin, x, n2, zm, c, zp, ym, yp, left, right, a.eps,
                           two_eps, epsf, two_epsf);
                if (Exact) st.add4(c);                    // stats always kept (acc may be null)
                else st.add4f(c);
                count += 4;
                if (z + 1 == nout && a.carry_out) *reinterpret_cast<int4*>(a.carry_out + y * n2 + x) = c;
            }
        }
        if (!Exact && (z & 15) == 15) st.fold();             // <= 32 add4f between folds
        mbar_arrive(&q_empty[(int)(z % ZR_NPL)]);             // plane z-1 retired
    }
    if (a.acc) st.flush(a.acc, count);
}

// launched by hszg_zsweep_grad_lap (window.cu) for band-split P2 with band_rows % 16 == 0
int launch_zsweep_ring(const int32_t* L, int64_t n1, int64_t n2, int64_t nout, const int32_t* lookahead,
                       const int32_t* carry, const int32_t* q_upper, int32_t* carry_out, int64_t gz0, int64_t gN0,
                       double eps, float* const* out, HszgAcc* acc, const int32_t* A, const int32_t* lookA,
                       int64_t BR, int64_t nb, int lmode, int lamode, int exact, cudaStream_t st) {
    ZrArgs a;
    a.L = L;
    a.lookahead = lookahead;
    a.carry = carry;
    a.q_upper = q_upper;
    a.carry_out = carry_out;
    a.A = A;
    a.lookA = lookA;
    a.n1 = n1;
    a.n2 = n2;
    a.nout = nout;
    a.gz0 = gz0;
    a.gN0 = gN0;
    a.BR = BR;
    a.nb = nb;
    a.eps = eps;
    a.o0 = out[0];
    a.o1 = out[1];
    a.o2 = out[2];
    a.o3 = out[3];
    a.acc = acc;
    dim3 grid((unsigned)((n2 + ZR_TX - 1) / ZR_TX), (unsigned)((n1 + ZR_TY - 1) / ZR_TY));
#define ZR_LAUNCH(E, W, WA)                                                           \
    do {                                                                              \
        allow_smem(k_zsweep_ring<E, W, WA>, zr_smem(W, WA, E));                       \
        k_zsweep_ring<E, W, WA><<<grid, ZR_T, zr_smem(W, WA, E), st>>>(a);            \
    } while (0)
#define ZR_WIDTHS(E)                                                                  \
    do {                                                                              \
        if (key == 0) ZR_LAUNCH(E, 4, 4);                                             \
        else if (key == 4) ZR_LAUNCH(E, 2, 2);                                        \
        else if (key == 8) ZR_LAUNCH(E, 1, 1);                                        \
        else if (key == 5) ZR_LAUNCH(E, 2, 1);                                        \
        else return 1;                                                                \
    } while (0)
    // width codes 0/1/2 = int32/int16/int8; supported pairs: equal, or int16 window + int8 lookahead
    const int key = lmode * 3 + lamode;
    // exact: 0 fast fp32, 1 exact (fp64 conversions), 2 exact by table (int32 stencils: |q| < 2^27)
    if (exact == 2) ZR_WIDTHS(EM_TABLE);
    else if (exact) ZR_WIDTHS(EM_EXACT);
    else ZR_WIDTHS(EM_FAST);
#undef ZR_WIDTHS
#undef ZR_LAUNCH
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

}  // namespace hszg
