// fused.cu — one-pass decode + analytics for the config-5 hot loop: the quantization indices q
// never reach HBM.  Each CTA owns an (x, y) column of a z-slab and slides along z; the payload
// bytes it needs arrive in shared memory by TMA bulk copies one block layer ahead, producer warps
// decode them plane by plane into a ring of q planes, and consumer warps emit gradient (dz, dy, dx)
// + Laplacian (fields.py:34-80, via stencil.cuh) and the exact statistics of their planes.
// HBM traffic per value: the compressed bytes + the 16 output bytes.
//
// HSZX_ND (8x8x8 blocks, compressors.py:170-199 / 214-218): q = p + M_b.  The CTA covers 16
// blocks along x (128 values) and 2 block rows (16 y).  Per block layer it stages 4 block rows
// (top halo, 2 main, bottom halo), each extended by one block on both x sides: the payload range,
// the chunk offsets and the block means of each (contiguous in the block-row-major stream).  A
// decode job is one 8-value row of one block in one plane (a quarter chunk: block-local order z,
// y, x, so chunk 2*zl + h holds rows 4h..4h+3 of plane zl); halo block rows decode only the row
// next to the CTA.
//
// Pipeline (warp-specialised): warp 0 loads (TMA), warps 1-11 decode, warps 12-19 emit.  full[s] /
// empty[s] mbarriers hand ring slot s (plane z in slot z % NPL) between decoders and emitters;
// stage[b] carries the TMA transaction bytes of staging buffer b (layer L in buffer L & 1) to the
// decoders, free[b] hands the buffer back to the loader when the decoders moved past its layer.
#include <cstdio>
#include "tile.cuh"
#include "stencil.cuh"
#include "async.cuh"

namespace hszg {

constexpr int FX_T = 640;                  // threads
constexpr int FX_PT = 384;                 // producers: warp 0 loads, warps 1-11 decode
constexpr int FX_CT = FX_T - FX_PT;        // consumers: warps 12-19
constexpr int FX_DT = FX_PT - 32;          // decoders: warps 1-11 (warp 0 loads): 352 >= the 324 row
                                           // jobs of a plane, one job each (7 warps: two; 3.5% slower)
constexpr int FX_BX = 16;                  // blocks along x per CTA
constexpr int FX_BY = 2;                   // block rows per CTA
constexpr int FX_ROWS = FX_BY * 8 + 2;     // ring rows: y0-1 .. y0+16
constexpr int FX_RPW = FX_BY * 8 / (FX_CT / 32);   // output rows per consumer warp
constexpr int FX_X0 = 8;                   // ring column of x0 (x0-8 .. x0+135 stored)
constexpr int FX_RW = 148;                 // words per ring row (144 + pad: odd 16-B stride)
constexpr int FX_PLANE = FX_ROWS * FX_RW;  // words per ring plane
constexpr int FX_RANGES = FX_BY + 2;       // staged block rows per layer
constexpr int FX_RBLK = FX_BX + 2;         // blocks per staged block row
constexpr int FX_OSTR = FX_RBLK * 16;      // staged chunk offsets per range
constexpr int FX_JOBS = (FX_RBLK * 8 * FX_BY + 2 * FX_RBLK + FX_DT - 1) / FX_DT;   // decode jobs per thread
constexpr int FX_MSTR = FX_RBLK + 2;       // staged block means per range (16-B multiple of the buffer)


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

// staged bytes of one layer buffer: offsets, means, payload ranges (+1 spare vector each)
inline size_t fx_payload_bytes(int max_bw) {
    return (size_t)FX_RANGES * (((size_t)FX_OSTR * (size_t)chunk_bytes(kChunkCap, max_bw) + 15) / 16 * 16 + 32);
}
inline size_t fx_buffer_bytes(int max_bw) {
    return (size_t)FX_RANGES * (FX_OSTR * 8 + FX_MSTR * 4) + fx_payload_bytes(max_bw);
}
inline size_t fx_smem_bytes(int max_bw, int npl, int em = EM_FAST) {
    return (size_t)npl * FX_PLANE * 4 + 2 * fx_buffer_bytes(max_bw) + (em == EM_TABLE ? XT_BYTES : 0);
}

template <int EM, int NPL, int OM>
__global__ void __launch_bounds__(FX_T, 1) k_fused_blocks(FxArgs a, uint32_t buf_bytes) {
    constexpr bool Exact = EM == EM_EXACT;
    extern __shared__ __align__(128) uint8_t smem[];
    int32_t* Q = reinterpret_cast<int32_t*>(smem);
    uint8_t* BUF = smem + (size_t)NPL * FX_PLANE * 4;      // 2 layer buffers: [offsets | means | payload]
    __shared__ __align__(8) uint64_t bar_full[NPL], bar_empty[NPL], bar_stage[2], bar_free[2];
    __shared__ uint64_t s_gbase[2][FX_RANGES];
    __shared__ uint32_t s_vbase[2][FX_RANGES];
    __shared__ int s_ok[2][FX_RANGES];

    const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
    const int64_t bx0 = (int64_t)blockIdx.x * FX_BX, by0 = (int64_t)blockIdx.y * FX_BY;
    const int nby = (int)(a.G1 - by0 < FX_BY ? a.G1 - by0 : FX_BY);
    const int64_t x0 = bx0 * 8, y0 = by0 * 8;
    const int64_t nlay = a.nz >> 3;
    const int64_t L0 = (int64_t)blockIdx.z * a.zlayers;
    const int64_t L1 = L0 + a.zlayers < nlay ? L0 + a.zlayers : nlay;
    const int64_t zb = L0 * 8, ze = L1 * 8;                  // planes emitted
    const int64_t Lb = zb > 0 ? L0 - 1 : L0;                  // first / last layer read (z halos)
    const int64_t Llast = L1 < nlay ? L1 : nlay - 1;
    const int64_t fbx = bx0 > 0 ? bx0 - 1 : 0;                // staged block columns [fbx, lbx]
    const int64_t lbx = bx0 + FX_BX < a.G2 ? bx0 + FX_BX : a.G2 - 1;
    const int nblk = (int)(lbx - fbx + 1);

    for (int i = threadIdx.x; i < NPL * FX_PLANE / 4; i += FX_T) reinterpret_cast<int4*>(Q)[i] = make_int4(0, 0, 0, 0);
    float* XT = reinterpret_cast<float*>(BUF + 2 * (size_t)buf_bytes);      // EM_TABLE: after the layer buffers
    if (EM == EM_TABLE) xtable_fill(XT, a.eps, threadIdx.x, FX_T);
    if (threadIdx.x == 0) {
        for (int i = 0; i < NPL; i++) {
            mbar_init(&bar_full[i], FX_DT);
            mbar_init(&bar_empty[i], FX_CT);
        }
        mbar_init(&bar_stage[0], 1);
        mbar_init(&bar_stage[1], 1);
        mbar_init(&bar_free[0], FX_DT);
        mbar_init(&bar_free[1], FX_DT);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (wp < FX_PT / 32) {
        // ================================ producers ================================
        // descriptor of block row r = lane (< FX_RANGES) of a layer, loaded one layer ahead by warp 0
        int d_ok = 0;
        int64_t d_clo = 0;
        uint64_t d_lo = 0, d_hi = 0;
        int32_t d_m[3] = {0, 0, 0};          // block means: range lane >> 3, blocks (lane & 7) + 8k
        auto describe = [&](int64_t L) {
            const int64_t by = by0 - 1 + lane;
            const int mr = lane >> 3;
            const int64_t mby = by0 - 1 + mr;
            if (mr < FX_RANGES && mby >= 0 && mby < a.G1 && mr <= nby + 1) {
#pragma unroll
                for (int k = 0; k < 3; k++) {
                    const int idx = (lane & 7) + 8 * k;
                    if (idx < nblk) d_m[k] = __ldg(a.meta + (L * a.G1 + mby) * a.G2 + fbx + idx);
                }
            }
            d_ok = lane < FX_RANGES && by >= 0 && by < a.G1 && lane <= nby + 1;
            if (!d_ok) return;
            d_clo = ((L * a.G1 + by) * a.G2 + fbx) * 16;
            const int64_t c_hi = d_clo + (int64_t)nblk * 16;
            d_lo = __ldg(a.offsets + d_clo);
            d_hi = c_hi < a.n_chunks ? __ldg(a.offsets + c_hi) : payload_end(a.offsets, a.n_chunks, a.len);
        };
        // warp 0: TMA the layer described by d_* into buffer b
        auto issue = [&](int b) {
            uint8_t* buf = BUF + (size_t)b * buf_bytes;
            uint64_t* offs = reinterpret_cast<uint64_t*>(buf);
            int32_t* means = reinterpret_cast<int32_t*>(offs + FX_RANGES * FX_OSTR);
            uint4* pay = reinterpret_cast<uint4*>(means + FX_RANGES * FX_MSTR);
            const uint64_t base = d_lo & ~(uint64_t)15;
            const uint32_t nvec = d_ok ? (uint32_t)((d_hi - base + 15) >> 4) : 0;
            uint32_t inc = d_ok ? nvec + 1 : 0;
#pragma unroll
            for (int d = 1; d < FX_RANGES; d <<= 1) {
                const uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
                if (lane >= d) inc += o;
            }
            const uint32_t vbase = inc - (d_ok ? nvec + 1 : 0);
            const uint32_t obytes = (uint32_t)nblk * 16 * 8;
            uint32_t tx = d_ok ? nvec * 16 + obytes : 0;
#pragma unroll
            for (int d = 16; d > 0; d >>= 1) tx += __shfl_xor_sync(0xffffffffu, tx, d);
            if (lane < FX_RANGES) {
                s_ok[b][lane] = d_ok;
                s_gbase[b][lane] = base;
                s_vbase[b][lane] = vbase;
            }
#pragma unroll
            for (int k = 0; k < 3; k++) {                   // means: plain stores, published by the stage arrive
                const int idx = (lane & 7) + 8 * k;
                if ((lane >> 3) < FX_RANGES && idx < nblk) means[(lane >> 3) * FX_MSTR + idx] = d_m[k];
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            if (lane == 0) mbar_arrive_tx(&bar_stage[b], tx);
            __syncwarp();
            if (d_ok) {
                tma_load_1d(pay + vbase, a.payload + base, nvec * 16, &bar_stage[b]);
                tma_load_1d(offs + lane * FX_OSTR, a.offsets + d_clo, obytes, &bar_stage[b]);
            }
        };

        if (wp == 0) {
            // loader warp: TMA layer L into buffer L & 1 once the decoders released layer L-2
            describe(Lb);
            for (int64_t L = Lb; L <= Llast; L++) {
                const int b = (int)(L & 1);
                const int64_t u = (L - Lb) >> 1;
                if (u > 0) mbar_wait(&bar_free[b], (uint32_t)((u - 1) & 1));
                issue(b);
                if (L + 1 <= Llast) describe(L + 1);
            }
            return;
        }
        const int dt = threadIdx.x - 32;                // decoder thread (warps 1..7)
        // this thread's decode jobs, the same in every plane: job = one 8-value row of one block
        // (main block rows: all 8 rows; halo block rows: the row next to the CTA)
        int jr[FX_JOBS], jc[FX_JOBS], jq[FX_JOBS], jm[FX_JOBS], jd[FX_JOBS];
        bool jv[FX_JOBS];
        {
            const int nmain = FX_RBLK * 8 * nby;
            const int njobs = nmain + 2 * FX_RBLK;
#pragma unroll
            for (int k = 0; k < FX_JOBS; k++) {
                const int i = dt + k * FX_DT;
                int r = 0, blk = 0, yl = 0;
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
                const int64_t bx = bx0 - 1 + blk, by = by0 - 1 + r;
                jv[k] = i < njobs && bx >= 0 && bx < a.G2 && by >= 0 && by < a.G1;
                const int rb = jv[k] ? (int)(bx - fbx) : 0;
                jr[k] = r;
                jc[k] = rb * 16 + (yl >> 2);
                jq[k] = yl & 3;
                jm[k] = r * FX_MSTR + rb;
                jd[k] = (r * 8 + yl - 7) * FX_RW + FX_X0 + (int)(bx * 8 - x0);
            }
        }
        int64_t cur = -1;
        for (int64_t z = zb - 1; z <= ze; z++) {
            const int s = (int)(z & (NPL - 1));
            const int64_t use = (z - (zb - 1)) / NPL;
            if (use > 0) mbar_wait(&bar_empty[s], (uint32_t)((use - 1) & 1));
            int32_t* P = Q + s * FX_PLANE;
            if (z < 0 || z >= a.nz) {
                const int32_t* h = z < 0 ? a.halo_lo : a.halo_hi;
                for (int i = dt; i < FX_ROWS * (FX_RW / 4); i += FX_DT) {
                    const int row = i / (FX_RW / 4), c4 = i - row * (FX_RW / 4);
                    const int64_t y = y0 - 1 + row, x = x0 - FX_X0 + 4 * c4;
                    int4 v = make_int4(0, 0, 0, 0);
                    if (h && c4 < 36 && y >= 0 && y < a.n1 && x >= 0 && x < a.n2) v = ld4(h + y * a.n2 + x);
                    *reinterpret_cast<int4*>(P + row * FX_RW + 4 * c4) = v;
                }
            } else {
                const int64_t L = z >> 3;
                const int b = (int)(L & 1);
                if (L != cur) {
                    if (cur >= 0) mbar_arrive(&bar_free[(int)(cur & 1)]);   // layer cur's buffer released
                    mbar_wait(&bar_stage[b], (uint32_t)(((L - Lb) >> 1) & 1));
                    cur = L;
                }
                const uint8_t* buf = BUF + (size_t)b * buf_bytes;
                const uint64_t* offs = reinterpret_cast<const uint64_t*>(buf);
                const int32_t* means = reinterpret_cast<const int32_t*>(offs + FX_RANGES * FX_OSTR);
                const uint32_t* pw = reinterpret_cast<const uint32_t*>(means + FX_RANGES * FX_MSTR);
                const int zl = (int)(z & 7);
#pragma unroll
                for (int k = 0; k < FX_JOBS; k++) {
                    if (!jv[k]) continue;
                    const int r = jr[k];
                    const int cl = jc[k] + 2 * zl;
                    const uint32_t rel = (uint32_t)(offs[r * FX_OSTR + cl] - s_gbase[b][r]) + s_vbase[b][r] * 16;
                    int4 lo, hi;
                    decode8(pw, rel, jq[k], means[jm[k]], lo, hi);
                    int32_t* dst = P + jd[k];
                    *reinterpret_cast<int4*>(dst) = lo;
                    *reinterpret_cast<int4*>(dst + 4) = hi;
                }
            }
            mbar_arrive(&bar_full[s]);
        }
        return;
    }

    // ================================ consumers ================================
    const int cw = wp - FX_PT / 32;                               // rows FX_RPW*cw ..
    const int64_t plane = a.n1 * a.n2;
    const float epsf = __double2float_rn(a.eps), two_epsf = 2.0f * epsf;
    const double two_eps = 2.0 * a.eps;
    WinStats st;
    st.init();
    int64_t count = 0;
    const int64_t x = x0 + 4 * lane;
    auto wait_full = [&](int64_t z) {
        mbar_wait(&bar_full[(int)(z & (NPL - 1))], (uint32_t)(((z - (zb - 1)) / NPL) & 1));
    };
    wait_full(zb - 1);
    wait_full(zb);
    // loop-invariant parts hoisted: output offset = z * plane + (y * n2 + x)
    const int64_t ybase = y0 + FX_RPW * cw;
    const int64_t rowoff = ybase * a.n2 + x;
    const int so0 = (FX_RPW * cw + 1) * FX_RW + FX_X0 + 4 * lane;
    const int eo = lane == 0 ? -1 : 4;                            // lane 0: column x0-1; lane 31: x0+128
    int64_t zoff = zb * plane;
    for (int64_t z = zb; z < ze; z++, zoff += plane) {
        wait_full(z + 1);
        const int32_t* Pm = Q + (int)((z - 1) & (NPL - 1)) * FX_PLANE;
        const int32_t* Pc = Q + (int)(z & (NPL - 1)) * FX_PLANE;
        const int32_t* Pp = Q + (int)((z + 1) & (NPL - 1)) * FX_PLANE;
        const int64_t gz = a.gz0 + z;
        const bool zin = gz > 0 && gz < a.gN0 - 1;
#pragma unroll
        for (int k = 0; k < FX_RPW; k++) {
            const int r = FX_RPW * cw + k;                        // output row within the CTA
            const int64_t y = ybase + k;
            const int so = so0 + k * FX_RW;
            const int4 c = *reinterpret_cast<const int4*>(Pc + so);
            const int e = Pc[so + eo];                            // every lane loads: no branch
            int left = __shfl_up_sync(0xffffffffu, c.w, 1);
            int right = __shfl_down_sync(0xffffffffu, c.x, 1);
            left = lane == 0 ? e : left;
            right = lane == 31 ? e : right;
            if (r < 8 * nby && x < a.n2) {
                const bool yin = y > 0 && y < a.n1 - 1;
                const int4 ym = *reinterpret_cast<const int4*>(Pc + so - FX_RW);
                const int4 yp = *reinterpret_cast<const int4*>(Pc + so + FX_RW);
                const int4 zm = *reinterpret_cast<const int4*>(Pm + so);
                const int4 zp = *reinterpret_cast<const int4*>(Pp + so);
                const int64_t o = zoff + rowoff + k * a.n2;
                if (EM == EM_EXACT)
                    emit4<OM>(a.o0, a.o1, a.o2, a.o3, o, zin, yin, x, a.n2, zm, c, zp, ym, yp, left, right, a.eps,
                              two_eps);
                else if (EM == EM_TABLE)
                    emit4x<OM>(a.o0, a.o1, a.o2, a.o3, o, zin, yin, x, a.n2, zm, c, zp, ym, yp, left, right, a.eps,
                           XT + XT_R);
                else if (zin && yin)                          // interior rows: no boundary branches
                    emit4f(a.o0, a.o1, a.o2, a.o3, o, true, true, x, a.n2, zm, c, zp, ym, yp, left, right, a.eps,
                           two_eps, epsf, two_epsf);
                else
                    emit4f(a.o0, a.o1, a.o2, a.o3, o, zin, yin, x, a.n2, zm, c, zp, ym, yp, left, right, a.eps,
                           two_eps, epsf, two_epsf);
                if (OM == OM_ALL || a.acc) {              // the API's subsets pass no accumulator: no statistics
                    if (Exact) st.add4(c);
                    else st.add4f(c);
                    count += 4;
                }
            }
        }
        if (!Exact && (z & 15) == 15) st.fold();   // <= 32 add4f between folds
        mbar_arrive(&bar_empty[(int)((z - 1) & (NPL - 1))]);      // plane z-1 retired
    }
    if (a.acc) st.flush(a.acc, count);
}

}  // namespace hszg

using namespace hszg;

int hszg_set_cuda_error(HszgErr* err, cudaError_t e, const char* where);
static inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }
static bool al16f(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

template <int EM, int NPL, int OM>
static void launch_fused_blocks(const FxArgs& a, dim3 grid, size_t smem, uint32_t buf_bytes, cudaStream_t st) {
    allow_smem(k_fused_blocks<EM, NPL, OM>, smem);
    k_fused_blocks<EM, NPL, OM><<<grid, FX_T, smem, st>>>(a, buf_bytes);
}
template <int EM, int NPL>
static void launch_fused_om(int om, const FxArgs& a, dim3 grid, size_t smem, uint32_t bb, cudaStream_t st) {
    if (om == OM_ALL) launch_fused_blocks<EM, NPL, OM_ALL>(a, grid, smem, bb, st);
    else if (om == OM_GRAD) launch_fused_blocks<EM, NPL, OM_GRAD>(a, grid, smem, bb, st);
    else launch_fused_blocks<EM, NPL, OM_LAP>(a, grid, smem, bb, st);
}

static constexpr size_t kSmemLimit = 227 * 1024 - 2048;   // dynamic part (static barriers etc. aside)

extern "C" int hszg_fused_blocks(const HszgGeom* g, const HszgStream* s, int64_t gz0, int64_t gN0,
                                 const int32_t* halo_lo, const int32_t* halo_hi, float* const* out, HszgAcc* acc,
                                 int64_t zlayers, int exact, void* stream, HszgErr* err) {
    err->status = HSZG_OK;
    const int64_t nz = g->dims[0], n1 = g->dims[1], n2 = g->dims[2];
    // exact: 0 fast fp32, 1 exact (fp64 conversions), 2 exact by table (int32 stencils: |q| < 2^27)
    int em = exact == 2 ? EM_TABLE : (exact ? EM_EXACT : EM_FAST);
    if (em == EM_TABLE && fx_smem_bytes(s->max_bitwidth, 4, em) > kSmemLimit) em = EM_EXACT;   // wide bit widths
    // outputs: all four, the gradient only (laplacian null: the API's derivative) or the Laplacian only
    const bool has[4] = {out[0] != nullptr, out[1] != nullptr, out[2] != nullptr, out[3] != nullptr};
    const int om = (has[0] && has[1] && has[2]) ? (has[3] ? OM_ALL : OM_GRAD)
                                                : ((!has[0] && !has[1] && !has[2] && has[3]) ? OM_LAP : 0);
    const int npl = fx_smem_bytes(s->max_bitwidth, 8, em) <= kSmemLimit ? 8 : 4;
    const size_t smem = fx_smem_bytes(s->max_bitwidth, npl, em);
    if (g->kind != HSZG_HSZX_ND || g->ndims != 3 || g->block_dims[0] != 8 || g->block_dims[1] != 8 ||
        g->block_dims[2] != 8 || nz % 8 || n1 % 8 || n2 % 8 || !s->canonical || !s->metadata || zlayers < 1 ||
        smem > kSmemLimit || !om || !al16f(out[0]) || !al16f(out[1]) || !al16f(out[2]) || !al16f(out[3]) ||
        (halo_lo && !al16f(halo_lo)) || (halo_hi && !al16f(halo_hi)) || !al16f(s->offsets) ||
        !al16f(s->metadata) || !al16f(s->payload)) {
        err->status = HSZG_INVALID_ARG;
        snprintf(err->message, sizeof(err->message),
                 "fused_blocks: needs canonical 3-D HSZX_ND, 8^3 blocks dividing the box, 16-B aligned buffers, "
                 "outputs all / {dz,dy,dx} / {lap}, staging in smem (max bw %d)", s->max_bitwidth);
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
    const uint32_t bb = (uint32_t)fx_buffer_bytes(s->max_bitwidth);
    cudaStream_t st = as_stream(stream);
    if (em == EM_EXACT) {
        if (npl == 8) launch_fused_om<EM_EXACT, 8>(om, a, grid, smem, bb, st);
        else launch_fused_om<EM_EXACT, 4>(om, a, grid, smem, bb, st);
    } else if (em == EM_TABLE) {
        if (npl == 8) launch_fused_om<EM_TABLE, 8>(om, a, grid, smem, bb, st);
        else launch_fused_om<EM_TABLE, 4>(om, a, grid, smem, bb, st);
    } else {                                   // fast: all four outputs (the pipeline)
        if (om != OM_ALL) {
            err->status = HSZG_INVALID_ARG;
            snprintf(err->message, sizeof(err->message), "fused_blocks: output subsets need an exact emitter");
            return HSZG_INVALID_ARG;
        }
        if (npl == 8) launch_fused_blocks<EM_FAST, 8, OM_ALL>(a, grid, smem, bb, st);
        else launch_fused_blocks<EM_FAST, 4, OM_ALL>(a, grid, smem, bb, st);
    }
    { const cudaError_t e_ = cudaGetLastError(); if (e_ != cudaSuccess) return hszg_set_cuda_error(err, e_, "fused_blocks"); }
    return HSZG_OK;
}
