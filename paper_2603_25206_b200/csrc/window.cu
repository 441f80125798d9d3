// window.cu — the windowed 3-D analytics kernels of pipeline.py (config-5 hot loop).
//
// Default path (pipeline.py): HSZX_ND in one pass (fused.cu); HSZP_ND per window of W planes:
//   k_band_scan (here): decode + row (x) prefix + in-band column (y) prefix -> band-local L (int8 /
//             int16 / int32) and band totals, k_band_prefix -> exclusive band offsets A;
//   k_zsweep_ring (zring.cu): q[z] = q[z-1] + L + A in a shared ring + gradient + Laplacian + stats,
//             q never written, q[b-1] handed to the next window.
// Also here, for other shapes: k_zgrad_lap (HSZX_ND windows decoded by k_tile_blocks) and k_zsweep
// (per-column z prefix over int32 P2), each thread sliding along z.
// Integer stencils reproduce fields.py:34-80 exactly; fp32 outputs are either one rounding of the
// reference float64 (exact mode) or int32 stencil x fl32(eps) in fp32 (fast mode, <= 4 ulp, valid
// while |q| < 2^27 — the pipeline checks and redoes exactly), written with streaming stores.
// Statistics: exact int128 per thread, warp-reduced, added into 32-bit limbs with 64-bit
// atomics (HszgAcc) — order-independent and exact, finished on the host in Python ints.
#include <cstdio>
#include <cstdlib>
#include "tile.cuh"
#include "lookback.cuh"
#include "stencil.cuh"
#include "async.cuh"

namespace hszg {

constexpr int ZG_THREADS = 128;   // 512 x-points per CTA

// q window: box planes [0, np), outputs for planes [zlo, zhi) (plane zlo-1 and zhi are halos
// when they exist); the box plane 0 sits at global z = gz0 of a gN0-plane field.
template <bool Exact>
__global__ void __launch_bounds__(ZG_THREADS) k_zgrad_lap(const int32_t* __restrict__ q, int64_t n1, int64_t n2,
                                                          int64_t zlo, int64_t zhi, int64_t gz0, int64_t gN0,
                                                          double eps, double two_eps, float* __restrict__ o0,
                                                          float* __restrict__ o1, float* __restrict__ o2,
                                                          float* __restrict__ o3, HszgAcc* acc,
                                                          const int32_t* __restrict__ qprev,
                                                          const int32_t* __restrict__ qnext) {
    const int lane = threadIdx.x & 31;
    const float epsf = __double2float_rn(eps), two_epsf = 2.0f * epsf;
    const int64_t x = ((int64_t)blockIdx.x * ZG_THREADS + threadIdx.x) * 4;
    const int64_t y = blockIdx.y;
    const int64_t plane = n1 * n2;
    const bool active = x < n2;
    const int64_t xi = active ? x : 0;
    const bool yin = y > 0 && y < n1 - 1;
    const int64_t off = y * n2 + xi;
    const int32_t* col = q + off;
    WinStats st;
    st.init();
    const int4 z4 = make_int4(0, 0, 0, 0);
    // loads one iteration ahead (software pipelining): while plane z is computed, the centre row
    // of plane z+2 and the y+-1 rows / x edges of plane z+1 are already in flight
    auto centre = [&](int64_t z) -> int4 {   // plane z, row y (z == zhi may come from qnext)
        return (z == zhi && qnext) ? ld4(qnext + off) : ld4(col + z * plane);
    };
    int4 c = z4, zm = z4, zp = z4, ym = z4, yp = z4;
    int el = 0, er = 0;
    if (active) {
        c = ld4(col + zlo * plane);
        const int64_t gz = gz0 + zlo;
        if (gz > 0) zm = qprev ? ld4(qprev + off) : ld4(col + (zlo - 1) * plane);
        if (gz < gN0 - 1) zp = centre(zlo + 1);
        const int32_t* row = col + zlo * plane;
        if (yin) {
            ym = ld4(row - n2);
            yp = ld4(row + n2);
        }
        if (lane == 0 && xi > 0) el = __ldg(row - 1);
        if (lane == 31 && xi + 4 < n2) er = __ldg(row + 4);
    }
    for (int64_t z = zlo; z < zhi; z++) {
        const int64_t gz = gz0 + z;
        const bool zin = gz > 0 && gz < gN0 - 1;
        int4 zp2 = z4, ym2 = z4, yp2 = z4;
        int el2 = 0, er2 = 0;
        if (active && z + 1 < zhi) {
            if (gz + 1 < gN0 - 1) zp2 = centre(z + 2);
            const int32_t* row = col + (z + 1) * plane;
            if (yin) {
                ym2 = ld4(row - n2);
                yp2 = ld4(row + n2);
            }
            if (lane == 0 && xi > 0) el2 = __ldg(row - 1);
            if (lane == 31 && xi + 4 < n2) er2 = __ldg(row + 4);
        }
        int left = __shfl_up_sync(0xffffffffu, c.w, 1);
        int right = __shfl_down_sync(0xffffffffu, c.x, 1);
        if (lane == 0) left = el;
        if (lane == 31) right = er;
        if (active) {
            if (Exact)
                emit4(o0, o1, o2, o3, (z - zlo) * plane + off, zin, yin, xi, n2, zm, c, zp, ym, yp, left, right, eps,
                      two_eps);
            else if (zin && yin)                          // interior: no boundary branches
                emit4f(o0, o1, o2, o3, (z - zlo) * plane + off, true, true, xi, n2, zm, c, zp, ym, yp, left, right,
                       eps, two_eps, epsf, two_epsf);
            else
                emit4f(o0, o1, o2, o3, (z - zlo) * plane + off, zin, yin, xi, n2, zm, c, zp, ym, yp, left, right, eps,
                       two_eps, epsf, two_epsf);
            if (acc) {
                if (Exact) {
                    st.add4(c);
                } else {
                    st.add4f(c);
                    if ((z & 31) == 31) st.fold();
                }
            }
        }
        zm = c;
        c = zp;
        zp = zp2;
        ym = ym2;
        yp = yp2;
        el = el2;
        er = er2;
    }
    if (acc) st.flush(acc, active ? 4 * (zhi - zlo) : 0);
}

// HSZP_ND z-sweep.  P2: box planes [0, np) = planes [a, a+np) of 2-D prefixes (plane a+nout is the
// lookahead when present); carry = q[a-1] (NULL: a is the global first plane); q_upper = q[a+nout]
// from the next rank (NULL: use the lookahead P2 plane, or none at the global top).
template <bool Exact>
__global__ void __launch_bounds__(ZG_THREADS) k_zsweep(const int32_t* __restrict__ P2, int64_t n1, int64_t n2,
                                                       int64_t nout, const int32_t* lookahead, const int32_t* carry,
                                                       const int32_t* q_upper, int32_t* carry_out, int64_t gz0,
                                                       int64_t gN0, double eps, double two_eps,
                                                       float* __restrict__ o0, float* __restrict__ o1,
                                                       float* __restrict__ o2, float* __restrict__ o3, HszgAcc* acc,
                                                       const int32_t* __restrict__ A, const int32_t* lookA,
                                                       int64_t BR, int64_t nb) {
    const int lane = threadIdx.x & 31;
    const float epsf = __double2float_rn(eps), two_epsf = 2.0f * epsf;
    const int64_t x = ((int64_t)blockIdx.x * ZG_THREADS + threadIdx.x) * 4;
    const int64_t y = blockIdx.y;
    const int64_t plane = n1 * n2;
    const bool active = x < n2;
    const int64_t xi = active ? x : 0;
    const bool yin = y > 0 && y < n1 - 1;
    const int64_t off = y * n2 + xi;
    WinStats st;
    st.init();
    const int4 z4 = make_int4(0, 0, 0, 0);
    // running q at plane a-1 (rows y-1, y, y+1 and the x-edge neighbours)
    int4 qc = z4, qm = z4, qp = z4;
    int ql = 0, qr = 0;
    if (active && carry) {
        qc = ld4(carry + off);
        if (yin) {
            qm = ld4(carry + off - n2);
            qp = ld4(carry + off + n2);
        }
        if (lane == 0 && xi > 0) ql = __ldg(carry + off - 1);
        if (lane == 31 && xi + 4 < n2) qr = __ldg(carry + off + 4);
    }
    int4 prev = qc;                                     // q[a-1]
    // band offsets (k_band_scan): row y' of plane zz adds A[zz][y' / BR]
    const int64_t aplane = nb * n2;
    const int64_t ac = A ? (y / BR) * n2 + xi : 0;
    const int64_t am = (A && yin) ? ((y - 1) / BR) * n2 + xi : 0;
    const int64_t ap = (A && yin) ? ((y + 1) / BR) * n2 + xi : 0;
    // P2 rows of plane zz (zz == nout is the lookahead plane), loaded one iteration ahead so the
    // loads of plane z+2 are in flight while plane z is emitted (software pipelining)
    auto wanted = [&](int64_t zz) -> bool {       // will iteration zz-1 build q[zz] from P2[zz]?
        const bool avail = zz < nout || (zz == nout && lookahead != nullptr && !q_upper);
        return active && avail && gz0 + zz - 1 < gN0 - 1;
    };
    int4 pc = z4, pm = z4, pp = z4;
    int pl = 0, pr = 0;
    auto fetch = [&](int64_t zz, int4& c_, int4& m_, int4& p_, int& l_, int& r_) {
        const int32_t* p = (zz < nout ? P2 + zz * plane : lookahead) + off;
        c_ = ld4(p);
        if (yin) {
            m_ = ld4(p - n2);
            p_ = ld4(p + n2);
        }
        if (lane == 0 && xi > 0) l_ = __ldg(p - 1);
        if (lane == 31 && xi + 4 < n2) r_ = __ldg(p + 4);
        if (A) {
            const int32_t* a = zz < nout ? A + zz * aplane : lookA;
            const int4 av = ld4(a + ac);
            c_ = add4(c_, av);
            if (yin) {                              // rows y+-1 share y's band except at band edges
                m_ = add4(m_, am == ac ? av : ld4(a + am));
                p_ = add4(p_, ap == ac ? av : ld4(a + ap));
            }
            if (lane == 0 && xi > 0) l_ += __ldg(a + ac - 1);
            if (lane == 31 && xi + 4 < n2) r_ += __ldg(a + ac + 4);
        }
    };
    // advance to plane a
    if (active) {
        int4 t_c = z4, t_m = z4, t_p = z4;
        int t_l = 0, t_r = 0;
        fetch(0, t_c, t_m, t_p, t_l, t_r);
        qc = add4(qc, t_c);
        qm = add4(qm, t_m);
        qp = add4(qp, t_p);
        ql += t_l;
        qr += t_r;
    }
    if (wanted(1)) fetch(1, pc, pm, pp, pl, pr);
    for (int64_t z = 0; z < nout; z++) {
        const int64_t gz = gz0 + z;
        const bool zin = gz > 0 && gz < gN0 - 1;
        int4 pc2 = z4, pm2 = z4, pp2 = z4;
        int pl2 = 0, pr2 = 0;
        if (wanted(z + 2)) fetch(z + 2, pc2, pm2, pp2, pl2, pr2);
        // q[z+1] at the centre row (P2 plane z+1 / lookahead, or the upper neighbour's plane)
        int4 next = z4, nm = z4, np_ = z4;
        int nl = 0, nr = 0;
        if (active && gz < gN0 - 1) {
            if (z + 1 == nout && q_upper) {
                next = ld4(q_upper + off);
            } else if (wanted(z + 1)) {
                next = add4(qc, pc);
                nm = add4(qm, pm);
                np_ = add4(qp, pp);
                nl = ql + pl;
                nr = qr + pr;
            }
        }
        pc = pc2;
        pm = pm2;
        pp = pp2;
        pl = pl2;
        pr = pr2;
        int left = __shfl_up_sync(0xffffffffu, qc.w, 1);
        int right = __shfl_down_sync(0xffffffffu, qc.x, 1);
        if (lane == 0) left = ql;
        if (lane == 31) right = qr;
        if (active) {
            if (Exact)
                emit4(o0, o1, o2, o3, z * plane + off, zin, yin, xi, n2, prev, qc, next, qm, qp, left, right, eps,
                      two_eps);
            else if (zin && yin)                          // interior: no boundary branches
                emit4f(o0, o1, o2, o3, z * plane + off, true, true, xi, n2, prev, qc, next, qm, qp, left, right, eps,
                       two_eps, epsf, two_epsf);
            else
                emit4f(o0, o1, o2, o3, z * plane + off, zin, yin, xi, n2, prev, qc, next, qm, qp, left, right, eps,
                       two_eps, epsf, two_epsf);
            if (acc) {
                if (Exact) {
                    st.add4(qc);
                } else {
                    st.add4f(qc);
                    if ((z & 31) == 31) st.fold();
                }
            }
            if (z + 1 == nout && carry_out) *reinterpret_cast<int4*>(carry_out + off) = qc;
        }
        prev = qc;
        qc = next;
        qm = nm;
        qp = np_;
        ql = nl;
        qr = nr;
    }
    if (acc) st.flush(acc, active ? 4 * nout : 0);
}

// HSZP_ND decode fused with the in-row prefix: rows are whole chunks (n2 % 32 == 0) and a tile
// holds whole rows (256 % chunks_per_row == 0), so the row prefix is a segmented scan of the
// per-chunk sums across the tile's lanes.
__global__ void __launch_bounds__(TILE_CHUNKS) k_tile_rowscan(SegGeo sg, const uint8_t* payload, uint64_t len,
                                                             const uint64_t* offsets, int cpr, int32_t* out) {
    __shared__ unsigned long long ex[TILE_CHUNKS];
    TileCtx t = tile_stage(sg, payload, len, offsets, blockIdx.x);
    const int64_t c = t.c0 + threadIdx.x;
    uint32_t run = 0;
    int local = 0, count = 0;
    int32_t* vals = t.vals;
    if (c < t.c1) {
        const ChunkLoc L = locate_chunk(sg, c);
        local = (int)(L.start - t.e0);
        count = L.count;
        decode_chunk_words(t.words, (uint32_t)(offsets[c] - t.base), L.count, [&](int j, int32_t v) {
            run += (uint32_t)v;
            vals[pad_idx(local + j)] = (int32_t)run;
        });
    }
    unsigned long long tot;
    const unsigned long long e = block_exclusive_u64((unsigned long long)run, &tot);
    ex[threadIdx.x] = e;
    __syncthreads();
    const uint32_t add = (uint32_t)(e - ex[(threadIdx.x / cpr) * cpr]);
    for (int j = 0; j < count; j++) vals[pad_idx(local + j)] = (int32_t)((uint32_t)vals[pad_idx(local + j)] + add);
    __syncthreads();
    const int n = (int)(t.e1 - t.e0);
    for (int i = threadIdx.x; i < n; i += blockDim.x) out[t.e0 + i] = vals[pad_idx(i)];
}

// ---- HSZP_ND band scan: decode + x prefix + y prefix in one pass (replaces rowscan + col_scan) ----
// CTA (band b, plane z) walks the rows [b*BR, min((b+1)*BR, n1)) of plane z a tile at a time
// (256 chunks = 256/cpr whole rows): fast decode with the in-chunk running sum, a segmented scan of
// the chunk sums along each row (x prefix), then the row-major write-out adds each thread's running
// column sums (y prefix inside the band).  It writes L = the band-local 2-D prefix and the band's
// column totals A[z][b][:]; k_band_prefix makes A exclusive over the bands, so the 2-D prefix is
// P2[z][y][x] = L[z][y][x] + A[z][y / BR][x], added by k_zsweep as it loads rows.  All int32
// arithmetic wraps; every prefix is a q sum mod 2^32 (recon.cu header).
constexpr int BS_MAXG = 4;   // int4 column groups per thread: n2 <= 4 * 4 * TILE_CHUNKS = 4096
constexpr int SE_W = 128;    // strip width of the strip-edge table (the one-pass HSZP_ND kernel's x tile)


template <bool Edges, int LW, bool Full, int KM>
__global__ void __maxnreg__(56) k_band_scan(const uint8_t* __restrict__ payload, uint64_t len,
                                                          const uint64_t* __restrict__ offsets, int64_t n_chunks,
                                                          int n1, int n2, int BR, void* __restrict__ L,
                                                          int32_t* __restrict__ A, int32_t* __restrict__ EF,
                                                          int32_t* __restrict__ l_ovf, uint32_t sbytes, int nb,
                                                          int64_t np, int nbuf) {
    uint32_t rng16 = 0;                      // OR of (value + 2^15 / 2^7) over the values stored narrow
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ uint32_t s_off[TILE_CHUNKS];
    __shared__ uint32_t s_wt[TILE_CHUNKS / 32];
    __shared__ uint64_t s_base[2];
    __shared__ __align__(8) uint64_t bar[2];
    const int cpr = n2 >> 5;                 // chunks per row (<= 128)
    const int rpt = TILE_CHUNKS / cpr;       // rows per tile (whole rows: rpt * cpr <= 256 chunks)
    const int ng = n2 >> 2;
    // column groups per thread: KM = ceil(ng / 256) (launcher); this thread owns nk <= KM of them
    int nk = KM;
    if (!Full) nk = max(0, min(KM, (ng - (int)threadIdx.x + TILE_CHUNKS - 1) / TILE_CHUNKS));
    const int toff0 = (int)(threadIdx.x >> 3) * kChunkStride + (int)((threadIdx.x & 7) << 2);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int32_t* tile = reinterpret_cast<int32_t*>(smem);
    // nbuf = 2: two staging buffers of sbytes, tile u in buffer u & 1, loaded a tile ahead of the decode;
    // nbuf = 1: one buffer (a CTA more per SM for the one-CTA-per-item grid), tile u + 1 loaded as soon as
    // tile u is decoded, under its row scan and write-out
    uint8_t* SB = smem + kFastTileBytes;
    const uint32_t bmask = nbuf == 2 ? 1u : 0u, pshift = nbuf == 2 ? 1u : 0u;
    const uint32_t* words = reinterpret_cast<const uint32_t*>(SB);
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    // work items (band b, plane z), strided over the grid: one per CTA for the classic grid, or a
    // persistent grid small enough to co-reside with the z-sweep (hszg_band_scan); gt counts the
    // tiles this CTA consumed, so staging buffer and mbarrier phase of tile t are those of gt + t
    uint32_t gt = 0;
    for (int64_t item = blockIdx.x; item < (int64_t)nb * np; item += gridDim.x) {
        const int b = (int)(item % nb);
        const int64_t z = item / nb;
        const int y0 = b * BR;
        const int y1 = min(y0 + BR, n1);
        const int ntiles = (y1 - y0 + rpt - 1) / rpt;
        auto tile_c0 = [&](int t) { return (z * n1 + y0 + t * rpt) * (int64_t)cpr; };
        auto tile_nch = [&](int t) { return min(rpt, y1 - (y0 + t * rpt)) * cpr; };
        // thread 0: byte range of a tile (loaded a tile ahead) and its TMA into buffer (gt + t) & 1
        uint64_t n_lo = 0, n_hi = 0;
        auto range = [&](int t) {
            const int64_t c0 = tile_c0(t), c1 = c0 + tile_nch(t);
            n_lo = __ldg(offsets + c0);
            n_hi = c1 < n_chunks ? __ldg(offsets + c1) : payload_end(offsets, n_chunks, len);
        };
        auto issue = [&](int t) {
            const uint32_t u = (gt + (uint32_t)t) & bmask;
            const uint64_t base = n_lo & ~(uint64_t)15;
            const uint32_t bytes = (uint32_t)(((n_hi - base + 15) >> 4) << 4);
            s_base[u] = base;
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_arrive_tx(&bar[u], bytes);
            tma_load_1d(SB + (size_t)u * sbytes, payload + base, bytes, &bar[u]);
        };
        if (threadIdx.x == 0) {
            range(0);
            issue(0);
            if (ntiles > 1) range(1);
        }
        uint64_t my_off = (int)threadIdx.x < tile_nch(0) ? __ldg(offsets + tile_c0(0) + threadIdx.x) : 0;
        __syncthreads();
        int4 ysum[KM];
    #pragma unroll
        for (int k = 0; k < KM; k++) ysum[k] = make_int4(0, 0, 0, 0);
        for (int t = 0; t < ntiles; t++) {
            const int r0 = y0 + t * rpt;
            const int nr = min(rpt, y1 - r0);
            const int nch = nr * cpr;
            const uint32_t u = gt + (uint32_t)t;
            mbar_wait(&bar[u & bmask], (u >> pshift) & 1);
            if (nbuf == 2 && threadIdx.x == 0 && t + 1 < ntiles) {   // buffer (t+1)&1 was released at the end of t-1
                issue(t + 1);
                if (t + 2 < ntiles) range(t + 2);
            }
            const uint64_t cur_off = my_off;
            if (t + 1 < ntiles && (int)threadIdx.x < tile_nch(t + 1)) my_off = __ldg(offsets + tile_c0(t + 1) + threadIdx.x);
            uint32_t tot = 0;
            if ((int)threadIdx.x < nch) {
                const uint32_t rel = (uint32_t)(cur_off - s_base[u & bmask]) + (u & bmask) * sbytes;
                tot = decode32<true>(words, rel, tile + threadIdx.x * kChunkStride, 0);
            }
            // exclusive prefix of the chunk sums along each row
            uint32_t inc = tot;
            if ((cpr & (cpr - 1)) == 0) {            // rows align with warp segments: segmented shuffle scan
                const int wseg = cpr < 32 ? cpr : 32;
                if (wseg == 32) {                     // whole-warp rows (n2 >= 1024): unrolled
    #pragma unroll
                    for (int d = 1; d < 32; d <<= 1) {
                        const uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
                        if (lane >= d) inc += o;
                    }
                } else {
                    for (int d = 1; d < wseg; d <<= 1) {
                        const uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
                        if ((lane & (wseg - 1)) >= d) inc += o;
                    }
                }
                if (cpr > 32) {
                    if (lane == 31) s_wt[warp] = inc;
                    __syncthreads();
                    for (int w2 = warp & ~((cpr >> 5) - 1); w2 < warp; w2++) inc += s_wt[w2];
                }
                s_off[threadIdx.x] = inc - tot;
            } else {                                  // any cpr: tile-wide scan minus the row start's prefix
                for (int d = 1; d < 32; d <<= 1) {
                    const uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
                    if (lane >= d) inc += o;
                }
                if (lane == 31) s_wt[warp] = inc;
                __syncthreads();
                for (int w2 = 0; w2 < warp; w2++) inc += s_wt[w2];
                s_off[threadIdx.x] = inc;
                __syncthreads();
                const int rs = ((int)threadIdx.x / cpr) * cpr;
                const uint32_t before = rs > 0 ? s_off[rs - 1] : 0u;
                __syncthreads();
                s_off[threadIdx.x] = inc - tot - before;
            }
            __syncthreads();
            if (nbuf == 1 && threadIdx.x == 0 && t + 1 < ntiles) {   // every chunk of tile t is decoded
                issue(t + 1);
                if (t + 2 < ntiles) range(t + 2);
            }
            const int nstrips = (n2 + SE_W - 1) / SE_W;
            // rows of the tile.  Column group k of this thread is gi = tid + 256 k, i.e. chunk (tid >> 3) + 32 k,
            // words 4 (tid & 7) ..: a per-thread base plus compile-time offsets, advanced by uniform row
            // strides (the loop is unrolled over rows; threads without a column group skip it — there is
            // no barrier inside).  Narrow-range check by OR of v + 2^15 / 2^7 (bits >= 16 / 8 flag it).
            if (Full || nk > 0) {
                const int32_t* tp = tile + toff0;              // tile row rr: chunks rr*cpr ..
                const uint32_t* op = s_off + (threadIdx.x >> 3);
                uint8_t* Lp = static_cast<uint8_t*>(L) + ((z * n1 + r0) * (int64_t)n2 + 4 * (int)threadIdx.x) * LW;
    #pragma unroll 4
                for (int rr = 0; rr < nr; rr++, tp += cpr * kChunkStride, op += cpr, Lp += (int64_t)n2 * LW) {
    #pragma unroll
                    for (int k = 0; k < KM; k++) {
                        if (Full || k < nk) {
                            const int4 v = *reinterpret_cast<const int4*>(tp + 32 * k * kChunkStride);
                            const int4 rv = add4u(v, op[32 * k]);         // row prefix R at x = 4gi .. 4gi+3
                            ysum[k] = add4(ysum[k], rv);
                            uint8_t* Lk = Lp + (size_t)k * 4 * TILE_CHUNKS * LW;
                            if (L && LW == 4) *reinterpret_cast<int4*>(Lk) = ysum[k];
                            if (L && LW == 2) {
                                const int4 v4 = ysum[k];
                                rng16 |= ((uint32_t)v4.x + 0x8000u) | ((uint32_t)v4.y + 0x8000u) | ((uint32_t)v4.z + 0x8000u) |
                                         ((uint32_t)v4.w + 0x8000u);
                                uint2 pk;                                                  // low halves, 2 PRMTs
                                pk.x = __byte_perm((uint32_t)v4.x, (uint32_t)v4.y, 0x5410);
                                pk.y = __byte_perm((uint32_t)v4.z, (uint32_t)v4.w, 0x5410);
                                *reinterpret_cast<uint2*>(Lk) = pk;
                            }
                            if (L && LW == 1) {
                                const int4 v4 = ysum[k];
                                rng16 |= ((uint32_t)v4.x + 0x80u) | ((uint32_t)v4.y + 0x80u) | ((uint32_t)v4.z + 0x80u) |
                                         ((uint32_t)v4.w + 0x80u);
                                const uint32_t lo = __byte_perm((uint32_t)v4.x, (uint32_t)v4.y, 0x0040);   // low bytes
                                const uint32_t hi = __byte_perm((uint32_t)v4.z, (uint32_t)v4.w, 0x0040);
                                *reinterpret_cast<uint32_t*>(Lk) = __byte_perm(lo, hi, 0x5410);
                            }
                            if (Edges) {                                  // strip edges: E[s] = R(128s-1), F[s] = R(128s+128)
                                const int y = r0 + rr;
                                const int xg = 4 * ((int)threadIdx.x + k * TILE_CHUNKS);
                                const int64_t n1e = ((int64_t)n1 + 1) & ~(int64_t)1;   // even rows per strip block
                                int32_t* ef = EF + ((z * nstrips) * n1e + y) * 2;
                                if ((xg & (SE_W - 1)) == SE_W - 4 && (xg + 4) / SE_W < nstrips)
                                    ef[(int64_t)((xg + 4) / SE_W) * n1e * 2] = rv.w;
                                if ((xg & (SE_W - 1)) == 0) {
                                    const int s2 = xg / SE_W;
                                    if (s2 > 0) ef[(int64_t)(s2 - 1) * n1e * 2 + 1] = rv.x;
                                    else {
                                        ef[0] = 0;
                                        ef[(int64_t)(nstrips - 1) * n1e * 2 + 1] = 0;
                                    }
                                }
                            }
                        }
                    }
                }
            }
            __syncthreads();
        }
        int32_t* arow = A + (z * nb + b) * (int64_t)n2;
    #pragma unroll
        for (int k = 0; k < KM; k++) {
            const int gi = threadIdx.x + k * TILE_CHUNKS;
            if (gi < ng) *reinterpret_cast<int4*>(arow + 4 * gi) = ysum[k];
        }
        gt += (uint32_t)ntiles;
    }
    // a narrow L value did not fit: flag bit 1 (int8) or 2 (int16)
    const bool ovf = (rng16 & (LW == 1 ? 0xffffff00u : 0xffff0000u)) != 0;
    if (LW < 4 && __any_sync(0xffffffffu, ovf) && (threadIdx.x & 31) == 0) atomicOr(l_ovf, LW);
}

// A[z][b][:] band totals -> exclusive prefix over b (one thread per (plane, int4 column group));
// loads are issued 8 bands at a time so their latencies overlap
__global__ void k_band_prefix(int32_t* __restrict__ A, int nb, int64_t n2, int64_t np) {
    const int64_t ng = n2 >> 2;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= np * ng) return;
    const int64_t z = i / ng, g = i - z * ng;
    int4* p = reinterpret_cast<int4*>(A + z * nb * n2) + g;
    int4 run = make_int4(0, 0, 0, 0);
    for (int b0 = 0; b0 < nb; b0 += 8) {
        int4 t[8];
#pragma unroll
        for (int k = 0; k < 8; k++)
            if (b0 + k < nb) t[k] = p[(b0 + k) * ng];
#pragma unroll
        for (int k = 0; k < 8; k++)
            if (b0 + k < nb) {
                p[(b0 + k) * ng] = run;
                run = add4(run, t[k]);
            }
    }
}

__global__ void k_acc_reset(HszgAcc* acc) {
    if (threadIdx.x == 0) {
        for (int k = 0; k < 4; k++) {
            acc->s1_limb[k] = 0;
            acc->s2_limb[k] = 0;
        }
        acc->count = 0;
        acc->vmin = INT32_MAX;
        acc->vmax = INT32_MIN;
    }
}

}  // namespace hszg

using namespace hszg;

int hszg_set_cuda_error(HszgErr* err, cudaError_t e, const char* where);
static inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }
static bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

extern "C" int hszg_acc_reset(HszgAcc* acc, void* stream) {
    k_acc_reset<<<1, 32, 0, as_stream(stream)>>>(acc);
    return cudaGetLastError() == cudaSuccess ? HSZG_OK : HSZG_CUDA;
}

extern "C" int hszg_zgrad_lap(const int32_t* q, int64_t n1, int64_t n2, int64_t zlo, int64_t zhi, int64_t gz0,
                              int64_t gN0, double eps, float* const* out, HszgAcc* acc, const int32_t* qprev,
                              const int32_t* qnext, int exact, void* stream) {
    if (n2 % 4 || !al16(q) || !al16(out[0]) || !al16(out[1]) || !al16(out[2]) || !al16(out[3]) || n1 > 65535)
        return HSZG_INVALID_ARG;
    if (zhi <= zlo) return HSZG_OK;
    dim3 grid((unsigned)((n2 / 4 + ZG_THREADS - 1) / ZG_THREADS), (unsigned)n1);
    (exact ? k_zgrad_lap<true> : k_zgrad_lap<false>)<<<grid, ZG_THREADS, 0, as_stream(stream)>>>(q, n1, n2, zlo, zhi, gz0, gN0, eps, 2.0 * eps, out[0],
                                                            out[1], out[2], out[3], acc, qprev, qnext);
    return cudaGetLastError() == cudaSuccess ? HSZG_OK : HSZG_CUDA;
}

namespace hszg {
int launch_zsweep_ring(const int32_t* L, int64_t n1, int64_t n2, int64_t nout, const int32_t* lookahead,
                       const int32_t* carry, const int32_t* q_upper, int32_t* carry_out, int64_t gz0, int64_t gN0,
                       double eps, float* const* out, HszgAcc* acc, const int32_t* A, const int32_t* lookA,
                       int64_t BR, int64_t nb, int lmode, int lamode, int exact, cudaStream_t st);
}

extern "C" int hszg_zsweep_grad_lap(const int32_t* P2, int64_t n1, int64_t n2, int64_t nout, const int32_t* lookahead,
                                    const int32_t* carry, const int32_t* q_upper, int32_t* carry_out, int64_t gz0,
                                    int64_t gN0, double eps, float* const* out, HszgAcc* acc,
                                    const int32_t* band_off, const int32_t* look_band_off, int64_t band_rows,
                                    int p2_mode, int exact, void* stream) {
    // p2_mode: bits 0-3 the width code of P2 (0 int32, 1 int16, 2 int8), bits 4-7 that of the lookahead
    const int lmode = p2_mode & 15, lamode = lookahead ? (p2_mode >> 4) & 15 : lmode;
    const bool narrow = lmode != 0 || lamode != 0;
    if (n2 % 4 || !al16(P2) || !al16(out[0]) || !al16(out[1]) || !al16(out[2]) || !al16(out[3]) || n1 > 65535 ||
        (carry && !al16(carry)) || (q_upper && !al16(q_upper)) || (carry_out && !al16(carry_out)) ||
        (band_off && (band_rows < 1 || !al16(band_off) || (lookahead && (!look_band_off || !al16(look_band_off))))))
        return HSZG_INVALID_ARG;
    const int64_t nb = band_off ? (n1 + band_rows - 1) / band_rows : 0;
    if (nout <= 0) return HSZG_OK;
    dim3 grid((unsigned)((n2 / 4 + ZG_THREADS - 1) / ZG_THREADS), (unsigned)n1);
    static const char* zmode = getenv("HSZG_ZSWEEP");       // 'c': per-thread-column kernel (A/B runs)
    const bool modes_ok = lmode <= 2 && lamode <= 2 && (lmode == lamode || (lmode == 1 && lamode == 2)) &&
                          (!narrow || n2 % ((lmode == 2 || lamode == 2) ? 16 : 8) == 0);
    if (!modes_ok) return HSZG_INVALID_ARG;
    if (band_off && band_rows % 16 == 0 && !(zmode && zmode[0] == 'c') && al16(lookahead) &&
        al16(look_band_off)) {
        return launch_zsweep_ring(P2, n1, n2, nout, lookahead, carry, q_upper, carry_out, gz0, gN0, eps, out, acc,
                                  band_off, look_band_off, band_rows, nb, lmode, lamode, exact, as_stream(stream))
                   ? HSZG_CUDA
                   : HSZG_OK;
    }
    if (narrow) return HSZG_INVALID_ARG;                     // narrow band-local prefixes: ring sweep only
    (exact ? k_zsweep<true> : k_zsweep<false>)<<<grid, ZG_THREADS, 0, as_stream(stream)>>>(P2, n1, n2, nout, lookahead, carry, q_upper, carry_out,
                                                         gz0, gN0, eps, 2.0 * eps, out[0], out[1], out[2], out[3],
                                                         acc, band_off, look_band_off, band_rows, nb);
    return cudaGetLastError() == cudaSuccess ? HSZG_OK : HSZG_CUDA;
}

extern "C" int hszg_band_scan(const HszgGeom* g, const HszgStream* s, int64_t band_rows, void* L, int32_t* A,
                              int32_t* strip_edges, int l_mode, int32_t* l_overflow, int ctas_per_sm, void* stream,
                              HszgErr* err) {
    err->status = HSZG_OK;
    const int64_t n1 = g->dims[1], n2 = g->dims[2], np = g->dims[0];
    const int64_t cpr = n2 / kChunkCap;
    if (g->kind != HSZG_HSZP_ND || g->ndims != 3 || !s->canonical || n2 % kChunkCap || cpr < 1 ||
        n2 > 4 * BS_MAXG * TILE_CHUNKS || band_rows < 1 || n1 > INT32_MAX || np > 65535 ||
        !al16(L) || !al16(A) || !al16(s->payload) || (!L && !strip_edges) ||
        l_mode < 0 || l_mode > 2 || (l_mode && (!l_overflow || strip_edges || n2 % (l_mode == 2 ? 16 : 8)))) {
        err->status = HSZG_INVALID_ARG;
        snprintf(err->message, sizeof(err->message),
                 "band_scan needs a canonical 3-D HSZP_ND stream with whole-chunk rows (n2 %% 32 == 0, "
                 "n2 <= 4096, 16-B aligned buffers)");
        return HSZG_INVALID_ARG;
    }
    if (g->n_chunks == 0) return HSZG_OK;
    const int64_t nb = (n1 + band_rows - 1) / band_rows;
    const uint32_t sbytes = (uint32_t)((stage_bytes(s->max_bitwidth) + 15) / 16 * 16);
    // one staging buffer when that fits one more CTA per SM for the one-CTA-per-item grid (HSZG_BS_NBUF forces it)
    int nbuf = 2;
    if (ctas_per_sm == 0) {
        static const int force = getenv("HSZG_BS_NBUF") ? atoi(getenv("HSZG_BS_NBUF")) : 0;
        const size_t per_sm = 227 * 1024;
        const size_t s1 = kFastTileBytes + (size_t)sbytes + 16 + 2048, s2 = s1 + sbytes;   // + static and reserved
        if (force == 1 || (force == 0 && per_sm / s1 > per_sm / s2 && per_sm / s1 <= 4)) nbuf = 1;
    }
    const size_t smem = kFastTileBytes + (size_t)nbuf * sbytes + 16;
    // ctas_per_sm = 0: one CTA per (band, plane), the fastest grid alone; k > 0: a persistent grid of
    // k CTAs per SM, which leaves the z-sweep beside it its SM slots (pipeline.py runs the scans of
    // later windows on a high-priority side stream under the sweeps: config-5 HSZP_ND 32.5 -> 30.9 ms)
    const int64_t items = nb * np;
    int64_t nct = items;
    if (ctas_per_sm > 0) {
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        nct = items < (int64_t)ctas_per_sm * sms ? items : (int64_t)ctas_per_sm * sms;
    }
    const dim3 grid((unsigned)nct);
    cudaStream_t st = as_stream(stream);
    const int kmax = (int)((n2 / 4 + TILE_CHUNKS - 1) / TILE_CHUNKS);   // column groups per thread: 1, 2 or 4 (3 runs as 4)
    const bool full = n2 / 4 == (int64_t)(kmax == 3 ? 4 : kmax) * TILE_CHUNKS;   // every thread owns all its groups
#define HSZG_BS_K(E, LS, F, K)                                                                               \
    do {                                                                                                     \
        allow_smem(k_band_scan<E, LS, F, K>, smem);                                                          \
        k_band_scan<E, LS, F, K><<<grid, TILE_CHUNKS, smem, st>>>(s->payload, s->payload_len, s->offsets,     \
                                                                 g->n_chunks, (int)n1, (int)n2,              \
                                                                 (int)band_rows, L_, A,                      \
                                                                 E ? strip_edges : nullptr, l_overflow,      \
                                                                 sbytes, (int)nb, np, nbuf);                 \
    } while (0)
#define HSZG_BS(E, LS, F)                                                                                    \
    do {                                                                                                     \
        if (kmax == 1) HSZG_BS_K(E, LS, F, 1);                                                               \
        else if (kmax == 2) HSZG_BS_K(E, LS, F, 2);                                                          \
        else HSZG_BS_K(E, LS, F, 4);                                                                         \
    } while (0)
    void* L_ = L;
    if (strip_edges) {
        if (full) HSZG_BS(true, 4, true);
        else HSZG_BS(true, 4, false);
    } else if (l_mode == 1) {
        if (full) HSZG_BS(false, 2, true);
        else HSZG_BS(false, 2, false);
    } else if (l_mode == 2) {
        if (full) HSZG_BS(false, 1, true);
        else HSZG_BS(false, 1, false);
    } else {
        if (full) HSZG_BS(false, 4, true);
        else HSZG_BS(false, 4, false);
    }
#undef HSZG_BS
#undef HSZG_BS_K
    const int64_t threads = np * (n2 / 4);
    k_band_prefix<<<(unsigned)((threads + 255) / 256), 256, 0, as_stream(stream)>>>(A, (int)nb, n2, np);
    { const cudaError_t e_ = cudaGetLastError(); if (e_ != cudaSuccess) return hszg_set_cuda_error(err, e_, "band_scan"); }
    return HSZG_OK;
}

extern "C" int hszg_decode_rowscan(const HszgGeom* g, const HszgStream* s, int32_t* out, void* stream, HszgErr* err) {
    err->status = HSZG_OK;
    const SegGeo sg = make_seggeo(*g);
    const int64_t n2 = sg.n[2];
    const int64_t cpr = n2 / kChunkCap;
    if (g->kind != HSZG_HSZP_ND || !s->canonical || n2 % kChunkCap || cpr < 1 || TILE_CHUNKS % cpr) {
        err->status = HSZG_INVALID_ARG;
        snprintf(err->message, sizeof(err->message),
                 "decode_rowscan needs a canonical HSZP_ND stream whose rows are whole chunks dividing a tile");
        return HSZG_INVALID_ARG;
    }
    if (g->n_chunks == 0) return HSZG_OK;
    const int64_t tiles = (g->n_chunks + TILE_CHUNKS - 1) / TILE_CHUNKS;
    const size_t smem = tile_smem_bytes(s->max_bitwidth);
    allow_smem(k_tile_rowscan, smem);
    k_tile_rowscan<<<(unsigned)tiles, TILE_CHUNKS, smem, as_stream(stream)>>>(sg, s->payload, s->payload_len,
                                                                             s->offsets, (int)cpr, out);
    { const cudaError_t e_ = cudaGetLastError(); if (e_ != cudaSuccess) return hszg_set_cuda_error(err, e_, "decode_rowscan"); }
    return HSZG_OK;
}
