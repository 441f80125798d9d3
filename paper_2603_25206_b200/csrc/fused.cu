// fused.cu — one-pass decode + analytics for the config-5 hot loop: the quantization indices q
// never reach HBM.  Each CTA owns an (x, y) column of the slab and slides along z, decoding the
// chunks it needs per plane from shared-memory-staged payload bytes into a 4-plane ring of q,
// then emits gradient (dz, dy, dx) + Laplacian (fields.py:34-80, via stencil.cuh) and the exact
// statistics of its planes.  HBM traffic per value: the compressed bytes + the 16 output bytes.
//
// HSZX_ND (8x8x8 blocks, compressors.py:170-199 / 214-218): q = p + M_b.  The CTA covers 16
// blocks along x (128 values) and 2 block rows (16 y); per block layer it stages the byte ranges
// of 4 block rows (top halo, 2 main, bottom halo), each extended by one block on both x sides,
// and decodes, per plane, the two chunks of every block that hold that plane (block-local order
// z, y, x: chunk 2*zl + h = rows 4h..4h+3 of plane zl) — halo rows only the half they need.
#include <cstdio>
#include "tile.cuh"
#include "stencil.cuh"

namespace hszg {

constexpr int FX_T = 256;                  // threads (8 warps)
constexpr int FX_BX = 16;                  // blocks along x per CTA
constexpr int FX_BY = 2;                   // block rows per CTA
constexpr int FX_ROWS = FX_BY * 8 + 2;     // smem rows: y0-1 .. y0+16
constexpr int FX_X0 = 8;                   // smem column of x0 (x0-8 .. x0+135 stored)
constexpr int FX_RW = 148;                 // words per smem row (144 + pad)
constexpr int FX_PLANE = FX_ROWS * FX_RW;  // words per ring plane
constexpr int FX_NPL = 4;                  // ring planes (z-1, z, z+1, loading z+2)
constexpr int FX_RANGES = FX_BY + 2;       // staged block rows per layer
constexpr int FX_RBLK = FX_BX + 2;         // blocks per staged block row

struct FxArgs {
    const uint8_t* payload;
    uint64_t len;
    const uint64_t* offsets;
    const int32_t* meta;
    int64_t n_chunks;
    int64_t nz, n1, n2, G1, G2;
    int64_t zlayers;                       // block layers per CTA (z segment)
    int64_t gz0, gN0;
    double eps;
    const int32_t* halo_lo;                // q plane below the slab (global z gz0-1) or null
    const int32_t* halo_hi;                // q plane above the slab or null
    float* o0;
    float* o1;
    float* o2;
    float* o3;
    HszgAcc* acc;
};

inline size_t fx_stage_bytes(int max_bw) {
    return (size_t)FX_RANGES * ((size_t)FX_RBLK * 16 * (size_t)chunk_bytes(kChunkCap, max_bw) + 48);
}
inline size_t fx_smem_bytes(int max_bw) {
    return (size_t)FX_NPL * FX_PLANE * 4 + (size_t)FX_RANGES * FX_RBLK * (16 * 8 + 4) + fx_stage_bytes(max_bw);
}

constexpr int FX_OSTR = FX_RBLK * 16;        // staged chunk offsets per range

template <bool Exact>
__global__ void __launch_bounds__(FX_T, 2) k_fused_blocks(FxArgs a) {
    extern __shared__ __align__(16) uint8_t smem[];
    int32_t* Q = reinterpret_cast<int32_t*>(smem);
    uint64_t* OFFS = reinterpret_cast<uint64_t*>(smem + (size_t)FX_NPL * FX_PLANE * 4);
    int32_t* MET = reinterpret_cast<int32_t*>(OFFS + FX_RANGES * FX_OSTR);
    uint4* SB = reinterpret_cast<uint4*>(MET + FX_RANGES * FX_RBLK);
    const uint32_t* SW = reinterpret_cast<const uint32_t*>(SB);
    __shared__ uint64_t s_gbase[FX_RANGES];
    __shared__ int64_t s_clo[FX_RANGES];
    __shared__ uint32_t s_vbase[FX_RANGES], s_nvec[FX_RANGES];
    __shared__ int s_ok[FX_RANGES], s_nblk[FX_RANGES];

    const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
    const int64_t bx0 = (int64_t)blockIdx.x * FX_BX, by0 = (int64_t)blockIdx.y * FX_BY;
    const int nby = (int)(a.G1 - by0 < FX_BY ? a.G1 - by0 : FX_BY);
    const int64_t x0 = bx0 * 8, y0 = by0 * 8;
    const int64_t nlay = a.nz >> 3;
    const int64_t L0 = (int64_t)blockIdx.z * a.zlayers;
    const int64_t L1 = L0 + a.zlayers < nlay ? L0 + a.zlayers : nlay;
    const int64_t Llast = L1 < nlay ? L1 : nlay - 1;          // last layer read (z halo included)
    const int64_t plane = a.n1 * a.n2;
    const float epsf = __double2float_rn(a.eps), two_epsf = 2.0f * epsf;
    const double two_eps = 2.0 * a.eps;
    const int64_t fbx = bx0 > 0 ? bx0 - 1 : 0;                 // first staged block column
    const int64_t lbx = bx0 + FX_BX < a.G2 ? bx0 + FX_BX : a.G2 - 1;

    for (int i = threadIdx.x; i < FX_NPL * FX_PLANE / 4; i += FX_T)
        reinterpret_cast<int4*>(Q)[i] = make_int4(0, 0, 0, 0);
    __syncthreads();

    // byte-range descriptor of block row r = threadIdx.x of a layer, loaded one layer ahead by
    // threads 0..3 so the offsets' latency is off the staging path
    int64_t d_L = -1, d_clo = 0;
    uint64_t d_lo = 0, d_hi = 0;
    int d_ok = 0;
    auto describe = [&](int64_t L) {
        const int64_t by = by0 - 1 + threadIdx.x;
        d_L = L;
        d_ok = by >= 0 && by < a.G1 && (int)threadIdx.x <= nby + 1;
        if (!d_ok) return;
        d_clo = ((L * a.G1 + by) * a.G2 + fbx) * 16;
        const int64_t c_hi = ((L * a.G1 + by) * a.G2 + lbx + 1) * 16;
        d_lo = __ldg(a.offsets + d_clo);
        d_hi = c_hi < a.n_chunks ? __ldg(a.offsets + c_hi) : payload_end(a.offsets, a.n_chunks, a.len);
    };
    int64_t staged = -1;
    auto stage = [&](int64_t L) {
        if (wp == 0) {
            uint32_t sz = 0;
            if (lane < FX_RANGES) {
                if (d_L != L) describe(L);
                if (d_ok) sz = (uint32_t)((d_hi - (d_lo & ~(uint64_t)15) + 15) >> 4) + 1;
            }
            uint32_t inc = sz;
#pragma unroll
            for (int d = 1; d < FX_RANGES; d <<= 1) {
                const uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
                if (lane >= d) inc += o;
            }
            if (lane < FX_RANGES) {
                s_ok[lane] = d_ok;
                s_gbase[lane] = d_lo & ~(uint64_t)15;
                s_vbase[lane] = inc - sz;
                s_nvec[lane] = sz ? sz - 1 : 0;
                s_clo[lane] = d_clo;
                s_nblk[lane] = (int)(lbx - fbx + 1);
            }
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < FX_RANGES; r++) {
            if (!s_ok[r]) continue;
            const uint4* g = reinterpret_cast<const uint4*>(a.payload + s_gbase[r]);
            uint4* d = SB + s_vbase[r];
            const uint32_t nv = s_nvec[r];
            for (uint32_t i = threadIdx.x; i < nv; i += FX_T) d[i] = __ldg(g + i);
            if (threadIdx.x == 0) d[nv] = make_uint4(0, 0, 0, 0);
            const int nc = s_nblk[r] * 16;
            const uint64_t* go = a.offsets + s_clo[r];
            for (int i = threadIdx.x; i < nc; i += FX_T) OFFS[r * FX_OSTR + i] = __ldg(go + i);
            if ((int)threadIdx.x < s_nblk[r]) MET[r * FX_RBLK + threadIdx.x] = __ldg(a.meta + s_clo[r] / 16 + threadIdx.x);
        }
        if (wp == 0 && lane < FX_RANGES && L + 1 <= Llast) describe(L + 1);
    };

    // fill ring slot (z & 3) with q of slab plane z, z in [-1, nz]
    auto load_plane = [&](int64_t z) {
        int32_t* P = Q + (int)(z & (FX_NPL - 1)) * FX_PLANE;
        if (z < 0 || z >= a.nz) {
            const int32_t* h = z < 0 ? a.halo_lo : a.halo_hi;
            for (int i = threadIdx.x; i < FX_ROWS * (FX_RW / 4); i += FX_T) {
                const int row = i / (FX_RW / 4), c4 = i - row * (FX_RW / 4);
                const int64_t y = y0 - 1 + row, x = x0 - FX_X0 + 4 * c4;
                int4 v = make_int4(0, 0, 0, 0);
                if (h && c4 < 36 && y >= 0 && y < a.n1 && x >= 0 && x < a.n2) v = ld4(h + y * a.n2 + x);
                *reinterpret_cast<int4*>(P + row * FX_RW + 4 * c4) = v;
            }
            return;
        }
        const int64_t L = z >> 3;
        const int zl = (int)(z & 7);
        if (L != staged) {
            __syncthreads();                       // previous layer's bytes fully consumed
            stage(L);
            staged = L;
            __syncthreads();
        }
        // one job = one 8-value row of one block in this plane (a quarter chunk): main block rows
        // all 8 rows, halo block rows only the row adjacent to the CTA
        const int nmain = FX_RBLK * 8 * nby;
        const int njobs = nmain + 2 * FX_RBLK;
        for (int i = threadIdx.x; i < njobs; i += FX_T) {
            int r, blk, yl;
            if (i < nmain) {
                r = 1 + i / (8 * FX_RBLK);
                const int rem = i - (r - 1) * 8 * FX_RBLK;
                blk = rem >> 3;
                yl = rem & 7;
            } else {
                const int j = i - nmain;
                const int side = j >= FX_RBLK;
                blk = j - side * FX_RBLK;
                r = side ? nby + 1 : 0;
                yl = side ? 0 : 7;
            }
            const int64_t bx = bx0 - 1 + blk;
            if (bx < 0 || bx >= a.G2 || !s_ok[r]) continue;
            const int rb = (int)(bx - fbx);
            const int cl = rb * 16 + zl * 2 + (yl >> 2);
            const uint32_t rel = (uint32_t)(OFFS[r * FX_OSTR + cl] - s_gbase[r]) + s_vbase[r] * 16;
            int4 lo, hi;
            decode8(SW, rel, yl & 3, MET[r * FX_RBLK + rb], lo, hi);
            const int row = r * 8 + yl - 7;        // (by0 - 1 + r) * 8 + yl - (y0 - 1)
            int32_t* dst = P + row * FX_RW + FX_X0 + (int)(bx * 8 - x0);
            *reinterpret_cast<int4*>(dst) = lo;
            *reinterpret_cast<int4*>(dst + 4) = hi;
        }
    };

    WinStats st;
    st.init();
    int64_t count = 0;
    const int64_t zb = L0 * 8, ze = L1 * 8;
    load_plane(zb - 1);
    load_plane(zb);
    const int64_t x = x0 + 4 * lane;
    for (int64_t z = zb; z < ze; z++) {
        load_plane(z + 1);
        __syncthreads();
        const int32_t* Pm = Q + (int)((z - 1) & (FX_NPL - 1)) * FX_PLANE;
        const int32_t* Pc = Q + (int)(z & (FX_NPL - 1)) * FX_PLANE;
        const int32_t* Pp = Q + (int)((z + 1) & (FX_NPL - 1)) * FX_PLANE;
        const int64_t gz = a.gz0 + z;
        const bool zin = gz > 0 && gz < a.gN0 - 1;
#pragma unroll
        for (int k = 0; k < 2; k++) {
            const int r = wp + 8 * k;                      // output row within the CTA
            const int64_t y = y0 + r;
            const int so = (r + 1) * FX_RW + FX_X0 + 4 * lane;
            const int4 c = *reinterpret_cast<const int4*>(Pc + so);
            int left = __shfl_up_sync(0xffffffffu, c.w, 1);
            int right = __shfl_down_sync(0xffffffffu, c.x, 1);
            if (lane == 0) left = Pc[so - 1];
            if (lane == 31) right = Pc[so + 4];
            if (r < 8 * nby && x < a.n2) {
                const bool yin = y > 0 && y < a.n1 - 1;
                const int4 ym = *reinterpret_cast<const int4*>(Pc + so - FX_RW);
                const int4 yp = *reinterpret_cast<const int4*>(Pc + so + FX_RW);
                const int4 zm = *reinterpret_cast<const int4*>(Pm + so);
                const int4 zp = *reinterpret_cast<const int4*>(Pp + so);
                const int64_t o = z * plane + y * a.n2 + x;
                if (Exact)
                    emit4(a.o0, a.o1, a.o2, a.o3, o, zin, yin, x, a.n2, zm, c, zp, ym, yp, left, right, a.eps,
                          two_eps);
                else
                    emit4f(a.o0, a.o1, a.o2, a.o3, o, zin, yin, x, a.n2, zm, c, zp, ym, yp, left, right, a.eps,
                           two_eps, epsf, two_epsf);
                if (a.acc) st.add4(c);
                count += 4;
            }
        }
    }
    if (a.acc) st.flush(a.acc, count);
}

}  // namespace hszg

using namespace hszg;

int hszg_set_cuda_error(HszgErr* err, cudaError_t e, const char* where);
static inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }
static bool al16f(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

extern "C" int hszg_fused_blocks(const HszgGeom* g, const HszgStream* s, int64_t gz0, int64_t gN0,
                                 const int32_t* halo_lo, const int32_t* halo_hi, float* const* out, HszgAcc* acc,
                                 int64_t zlayers, int exact, void* stream, HszgErr* err) {
    err->status = HSZG_OK;
    const int64_t nz = g->dims[0], n1 = g->dims[1], n2 = g->dims[2];
    const size_t smem = fx_smem_bytes(s->max_bitwidth);
    if (g->kind != HSZG_HSZX_ND || g->ndims != 3 || g->block_dims[0] != 8 || g->block_dims[1] != 8 ||
        g->block_dims[2] != 8 || nz % 8 || n1 % 8 || n2 % 8 || !s->canonical || !s->metadata || zlayers < 1 ||
        smem > 200 * 1024 || !al16f(out[0]) || !al16f(out[1]) || !al16f(out[2]) || !al16f(out[3]) ||
        (halo_lo && !al16f(halo_lo)) || (halo_hi && !al16f(halo_hi))) {
        err->status = HSZG_INVALID_ARG;
        snprintf(err->message, sizeof(err->message),
                 "fused_blocks needs a canonical 3-D HSZX_ND stream with 8x8x8 blocks dividing the box and "
                 "max bit width <= 16 (got %d)", s->max_bitwidth);
        return HSZG_INVALID_ARG;
    }
    if (g->n == 0) return HSZG_OK;
    FxArgs a;
    a.payload = s->payload;
    a.len = s->payload_len;
    a.offsets = s->offsets;
    a.meta = s->metadata;
    a.n_chunks = g->n_chunks;
    a.nz = nz;
    a.n1 = n1;
    a.n2 = n2;
    a.G1 = n1 / 8;
    a.G2 = n2 / 8;
    a.zlayers = zlayers;
    a.gz0 = gz0;
    a.gN0 = gN0;
    a.eps = g->eps;
    a.halo_lo = halo_lo;
    a.halo_hi = halo_hi;
    a.o0 = out[0];
    a.o1 = out[1];
    a.o2 = out[2];
    a.o3 = out[3];
    a.acc = acc;
    const int64_t nlay = nz / 8;
    dim3 grid((unsigned)((a.G2 + FX_BX - 1) / FX_BX), (unsigned)((a.G1 + FX_BY - 1) / FX_BY),
              (unsigned)((nlay + zlayers - 1) / zlayers));
    if (exact) {
        allow_smem(k_fused_blocks<true>, smem);
        k_fused_blocks<true><<<grid, FX_T, smem, as_stream(stream)>>>(a);
    } else {
        allow_smem(k_fused_blocks<false>, smem);
        k_fused_blocks<false><<<grid, FX_T, smem, as_stream(stream)>>>(a);
    }
    if (cudaGetLastError() != cudaSuccess) return hszg_set_cuda_error(err, cudaGetLastError(), "fused_blocks");
    return HSZG_OK;
}
