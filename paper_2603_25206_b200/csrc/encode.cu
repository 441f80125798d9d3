// encode.cu — the compress side (K-ENC): value range, quantization and decorrelation.
//
//   resolve_eps  quant.py:56-66         -> k_minmax (+ NaN/Inf count)
//   quantize     quant.py:69-82         -> k_quantize(_f32x4): floor(d*recip + 0.5) in fp64 with the
//                                          multiply and add rounded separately (no FMA, as numpy)
//   decorrelate  compressors.py:149-198 -> k_decor_prev(_x4) (HSZP), k_decor_lorenzo(_x4) (HSZP_ND),
//                                          k_decor_blockmean(_tiles, _b32, _1d) (HSZX, HSZX_ND; truncating
//                                          means 134-138)
// The chunk encoder proper (bit widths, scan, pack) lives in codec.cu.
#include <cstdio>
#include <cfloat>
#include <type_traits>
#include "common.cuh"

namespace hszg {

struct MinMaxPart {
    double mn, mx;
    unsigned long long nonfinite;
    unsigned long long pad;
};

template <typename T>
__global__ void k_minmax(const T* x, int64_t n, MinMaxPart* parts) {
    double mn = DBL_MAX, mx = -DBL_MAX;
    unsigned long long bad = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double v = (double)__ldg(x + i);
        if (!isfinite(v)) {
            bad++;
            continue;
        }
        mn = fmin(mn, v);
        mx = fmax(mx, v);
    }
    for (int d = 16; d > 0; d >>= 1) {
        mn = fmin(mn, __shfl_down_sync(0xffffffffu, mn, d));
        mx = fmax(mx, __shfl_down_sync(0xffffffffu, mx, d));
        bad += __shfl_down_sync(0xffffffffu, bad, d);
    }
    __shared__ MinMaxPart w[32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) w[wid] = MinMaxPart{mn, mx, bad, 0};
    __syncthreads();
    if (threadIdx.x == 0) {
        MinMaxPart r = w[0];
        for (int k = 1; k < (int)(blockDim.x >> 5); k++) {
            r.mn = fmin(r.mn, w[k].mn);
            r.mx = fmax(r.mx, w[k].mx);
            r.nonfinite += w[k].nonfinite;
        }
        parts[blockIdx.x] = r;
    }
}

__global__ void k_minmax_final(const MinMaxPart* parts, int np, double* out, int64_t* nonfinite) {
    if (threadIdx.x != 0) return;
    double mn = DBL_MAX, mx = -DBL_MAX;
    unsigned long long bad = 0;
    for (int i = 0; i < np; i++) {
        mn = fmin(mn, parts[i].mn);
        mx = fmax(mx, parts[i].mx);
        bad += parts[i].nonfinite;
    }
    out[0] = mn;
    out[1] = mx;
    *nonfinite = (int64_t)bad;
}

template <typename T>
__global__ void k_quantize(const T* x, int64_t n, double recip, int32_t* q, unsigned int* flags) {
    unsigned int f = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double d = (double)x[i];
        const double s = floor(__dadd_rn(__dmul_rn(d, recip), 0.5));
        if (fabs(s) > (double)kQmax) f |= 1u;       // quant.py:77-81 (also catches +-inf)
        if (s != s) f |= 2u;                         // NaN
        q[i] = (fabs(s) <= (double)kQmax) ? (int32_t)s : 0;
    }
    if (f) atomicOr(flags, f);
}

// HSZP: p = diff(flat q, prepend 0)  (compressors.py:149-157)
__global__ void k_decor_prev(const int32_t* q, int64_t n, int32_t* p, unsigned int* flags) {
    unsigned int f = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t d = (int64_t)q[i] - (i ? (int64_t)q[i - 1] : 0);
        if (d > kPmax || d < -kPmax) f |= 1u;
        p[i] = (int32_t)d;
    }
    if (f) atomicOr(flags, f);
}

// HSZP_ND: successive diffs along every axis with zero padding == inclusion-exclusion
// over the 2^nd lower corner (compressors.py:160-176).  Box view (N0,N1,N2).
__global__ void k_decor_lorenzo(const int32_t* q, int64_t N0, int64_t N1, int64_t N2, int32_t* p,
                                unsigned int* flags) {
    const int64_t i2 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i2 >= N2) return;
    const int64_t i1 = blockIdx.y, i0 = blockIdx.z;
    unsigned int f = 0;
    int64_t acc = 0;
#pragma unroll
    for (int s = 0; s < 8; s++) {
        const int d0 = (s >> 2) & 1, d1 = (s >> 1) & 1, d2 = s & 1;
        if ((d0 && i0 == 0) || (d1 && i1 == 0) || (d2 && i2 == 0)) continue;
        const int64_t v = q[((i0 - d0) * N1 + (i1 - d1)) * N2 + (i2 - d2)];
        acc += ((d0 + d1 + d2) & 1) ? -v : v;
    }
    if (acc > kPmax || acc < -kPmax) f |= 1u;
    p[(i0 * N1 + i1) * N2 + i2] = (int32_t)acc;
    if (f) atomicOr(flags, f);
}

// Fused encoder front (hszg_decorrelate_sized): the bit width of a full 32-value chunk from its
// lanes' magnitude maxima (a group of G aligned lanes, xor-reduced), recorded by the group's first lane
// as the encoder's per-chunk size (_bitpack.pyx:24-51), so hszg_encode_sizes' read of p is skipped.
template <int G>
__device__ __forceinline__ void chunk_size_out(uint32_t m, int lane, int64_t chunk, uint64_t* sizes, uint8_t* bws) {
#pragma unroll
    for (int d = 1; d < G; d <<= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, d));
    if ((lane & (G - 1)) == 0 && chunk >= 0) {
        const int bw = m ? 32 - __clz(m) : 0;
        bws[chunk] = (uint8_t)bw;
        sizes[chunk] = (uint64_t)chunk_bytes(kChunkCap, bw);
    }
}
__device__ __forceinline__ uint32_t mag4(int32_t a, int32_t b, int32_t c, int32_t d) {
    return max(max((uint32_t)abs(a), (uint32_t)abs(b)), max((uint32_t)abs(c), (uint32_t)abs(d)));
}

// HSZX 1-D with 32-value blocks (the default) and n % 32 == 0: a CTA stages 256 blocks with 16-B
// coalesced loads into shared memory (36-word stride: conflict-free per-thread 16-B reads), each
// thread reduces its block (sum, truncated mean, residuals, bit width / chunk size: one block = one
// chunk), and the residuals leave through shared memory with coalesced 16-B stores.
__global__ void __launch_bounds__(256) k_decor_blockmean_b32(const int4* __restrict__ q, int64_t nblk,
                                                             int4* __restrict__ p, int32_t* __restrict__ meta,
                                                             unsigned int* flags, uint64_t* sizes, uint8_t* bws) {
    __shared__ __align__(16) int32_t tile[256 * 36];
    const int64_t b0 = (int64_t)blockIdx.x * 256;
    const int nb = (int)(nblk - b0 < 256 ? nblk - b0 : 256);
    for (int i = threadIdx.x; i < nb * 8; i += 256)
        *reinterpret_cast<int4*>(tile + (i >> 3) * 36 + ((i & 7) << 2)) = __ldg(q + b0 * 8 + i);
    __syncthreads();
    unsigned int f = 0;
    if ((int)threadIdx.x < nb) {
        int32_t* t = tile + threadIdx.x * 36;
        int4 v[8];
        int64_t sum = 0;
#pragma unroll
        for (int k = 0; k < 8; k++) {
            v[k] = *reinterpret_cast<const int4*>(t + 4 * k);
            sum += (int64_t)v[k].x + v[k].y + v[k].z + v[k].w;
        }
        const int64_t mean = sum >= 0 ? (sum >> 5) : -((-sum) >> 5);     // truncation toward zero
        uint32_t m = 0;
#pragma unroll
        for (int k = 0; k < 8; k++) {
            const int64_t d0 = (int64_t)v[k].x - mean, d1 = (int64_t)v[k].y - mean;
            const int64_t d2 = (int64_t)v[k].z - mean, d3 = (int64_t)v[k].w - mean;
            if (d0 > kPmax || d0 < -kPmax || d1 > kPmax || d1 < -kPmax || d2 > kPmax || d2 < -kPmax || d3 > kPmax ||
                d3 < -kPmax)
                f |= 1u;
            const int4 o = make_int4((int32_t)d0, (int32_t)d1, (int32_t)d2, (int32_t)d3);
            m = max(m, mag4(o.x, o.y, o.z, o.w));
            *reinterpret_cast<int4*>(t + 4 * k) = o;
        }
        const int64_t b = b0 + threadIdx.x;
        meta[b] = (int32_t)mean;
        if (sizes) {
            const int bw = m ? 32 - __clz(m) : 0;
            bws[b] = (uint8_t)bw;
            sizes[b] = (uint64_t)chunk_bytes(kChunkCap, bw);
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < nb * 8; i += 256)
        p[b0 * 8 + i] = *reinterpret_cast<const int4*>(tile + (i >> 3) * 36 + ((i & 7) << 2));
    if (f) atomicOr(flags, f);
}

// HSZX 1-D with segments of B | 32 values (B a power of two): one value per lane, the B lanes of a
// segment reduce by xor-shuffles inside their aligned group (no per-segment index arithmetic); four
// 32-value groups per warp and step (loads in flight), 32-bit sums when every |q| < 2^26.
__device__ __forceinline__ int64_t trunc_div(int64_t s, int size, int lgB, bool full) {
    if (full) return s >= 0 ? (s >> lgB) : -((-s) >> lgB);       // truncation toward zero
    return (s >= INT32_MIN && s <= INT32_MAX) ? (int64_t)((int32_t)s / size) : s / size;
}

__global__ void k_decor_blockmean_1d(const int32_t* __restrict__ q, int64_t n, int lgB, int32_t* __restrict__ p,
                                     int32_t* __restrict__ meta, unsigned int* flags, uint64_t* sizes,
                                     uint8_t* bws) {
    constexpr int U = 4;
    const int lane = threadIdx.x & 31;
    const int B = 1 << lgB;
    unsigned int f = 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x * U;
    for (int64_t base = ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) & ~(int64_t)31) * U; base < n;
         base += stride) {
        int32_t v[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int64_t i = base + u * 32 + lane;
            v[u] = i < n ? __ldg(q + i) : 0;
        }
        bool narrow = true;
#pragma unroll
        for (int u = 0; u < U; u++) narrow = narrow && v[u] > -(1 << 26) && v[u] < (1 << 26);
        narrow = __all_sync(0xffffffffu, narrow);
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int64_t i = base + u * 32 + lane;
            int64_t sum;
            if (narrow) {
                int32_t s32 = v[u];
                for (int d = 1; d < B; d <<= 1) s32 += __shfl_xor_sync(0xffffffffu, s32, d);
                sum = s32;
            } else {
                sum = v[u];
                for (int d = 1; d < B; d <<= 1) sum += __shfl_xor_sync(0xffffffffu, sum, d);
            }
            if (i < n) {
                const int64_t seg0 = i - (lane & (B - 1));
                const bool full = seg0 + B <= n;
                const int64_t mean = trunc_div(sum, full ? B : (int)(n - seg0), lgB, full);
                if ((lane & (B - 1)) == 0) meta[seg0 >> lgB] = (int32_t)mean;
                const int64_t d = (int64_t)v[u] - mean;
                if (d > kPmax || d < -kPmax) f |= 1u;
                p[i] = (int32_t)d;
                v[u] = (int32_t)d;
            } else {
                v[u] = 0;
            }
            if (sizes)   // B == 32, n % 32 == 0: these 32 lanes are one chunk
                chunk_size_out<32>((uint32_t)abs(v[u]), lane, i < n ? i >> 5 : -1, sizes, bws);
        }
    }
    if (f) atomicOr(flags, f);
}

// ---- vectorised variants (16-B aligned arrays): four values per thread and step -----------------

__device__ __forceinline__ int32_t quant1(double d, double recip, unsigned int& f) {
    const double s = floor(__dadd_rn(__dmul_rn(d, recip), 0.5));
    if (fabs(s) > (double)kQmax) f |= 1u;
    if (s != s) f |= 2u;
    return (fabs(s) <= (double)kQmax) ? (int32_t)s : 0;
}

__global__ void k_quantize_f32x4(const float4* __restrict__ x, int64_t n4, double recip, int4* __restrict__ q,
                                 unsigned int* flags) {
    unsigned int f = 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    for (; i + stride < n4; i += 2 * stride) {                 // two 16-B loads in flight
        const float4 a = __ldg(x + i), b = __ldg(x + i + stride);
        q[i] = make_int4(quant1(a.x, recip, f), quant1(a.y, recip, f), quant1(a.z, recip, f), quant1(a.w, recip, f));
        q[i + stride] =
            make_int4(quant1(b.x, recip, f), quant1(b.y, recip, f), quant1(b.z, recip, f), quant1(b.w, recip, f));
    }
    for (; i < n4; i += stride) {
        const float4 a = __ldg(x + i);
        q[i] = make_int4(quant1(a.x, recip, f), quant1(a.y, recip, f), quant1(a.z, recip, f), quant1(a.w, recip, f));
    }
    if (f) atomicOr(flags, f);
}

__device__ __forceinline__ int32_t diff1(int64_t a, int64_t b, unsigned int& f) {
    const int64_t d = a - b;
    if (d > kPmax || d < -kPmax) f |= 1u;
    return (int32_t)d;
}

// HSZP on 4-value groups: the previous value of a group's first element is the previous lane's .w
__global__ void k_decor_prev_x4(const int4* __restrict__ q, int64_t n4, int4* __restrict__ p, unsigned int* flags,
                                uint64_t* sizes, uint8_t* bws) {
    unsigned int f = 0;
    const int lane = threadIdx.x & 31;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t base = blockIdx.x * (int64_t)blockDim.x; base < n4; base += stride) {
        const int64_t i = base + threadIdx.x;
        const bool act = i < n4;
        const int4 v = act ? __ldg(q + i) : make_int4(0, 0, 0, 0);
        int prev = __shfl_up_sync(0xffffffffu, v.w, 1);
        if (lane == 0) prev = (act && i > 0) ? __ldg(reinterpret_cast<const int32_t*>(q) + 4 * i - 1) : 0;
        int4 o = make_int4(0, 0, 0, 0);
        if (act) {
            o = make_int4(diff1(v.x, prev, f), diff1(v.y, v.x, f), diff1(v.z, v.y, f), diff1(v.w, v.z, f));
            p[i] = o;
        }
        if (sizes) chunk_size_out<8>(mag4(o.x, o.y, o.z, o.w), lane, act ? i >> 3 : -1, sizes, bws);
    }
    if (f) atomicOr(flags, f);
}

// HSZP_ND 3-D (box view) on 4 x-consecutive points: p = sum over the 2^3 lower corners with signs,
// written as the x-differences of the rows (z,y), (z,y-1), (z-1,y), (z-1,y-1); x-1 by shuffle
__global__ void k_decor_lorenzo_x4(const int32_t* __restrict__ q, int64_t N0, int64_t N1, int64_t N2,
                                   int32_t* __restrict__ p, unsigned int* flags, uint64_t* sizes, uint8_t* bws) {
    const int lane = threadIdx.x & 31;
    const int64_t x = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
    const int64_t i1 = blockIdx.y, i0 = blockIdx.z;
    const bool act = x < N2;
    const int64_t xi = act ? x : 0;
    const int64_t plane = N1 * N2;
    const int32_t* c = q + (i0 * N1 + i1) * N2 + xi;
    const int4 z4 = make_int4(0, 0, 0, 0);
    int4 r[4];                         // rows (z,y), (z,y-1), (z-1,y), (z-1,y-1)
    const bool hy = i1 > 0, hz = i0 > 0;
    r[0] = act ? __ldg(reinterpret_cast<const int4*>(c)) : z4;
    r[1] = act && hy ? __ldg(reinterpret_cast<const int4*>(c - N2)) : z4;
    r[2] = act && hz ? __ldg(reinterpret_cast<const int4*>(c - plane)) : z4;
    r[3] = act && hy && hz ? __ldg(reinterpret_cast<const int4*>(c - plane - N2)) : z4;
    int64_t d[4][4];                   // x-difference of each row at the 4 points
#pragma unroll
    for (int k = 0; k < 4; k++) {
        int left = __shfl_up_sync(0xffffffffu, r[k].w, 1);
        const int32_t* rowp = c - (k & 1 ? N2 : 0) - (k & 2 ? plane : 0);
        const bool has = act && (!(k & 1) || hy) && (!(k & 2) || hz);
        if (lane == 0) left = (has && xi > 0) ? __ldg(rowp - 1) : 0;
        d[k][0] = (int64_t)r[k].x - left;
        d[k][1] = (int64_t)r[k].y - r[k].x;
        d[k][2] = (int64_t)r[k].z - r[k].y;
        d[k][3] = (int64_t)r[k].w - r[k].z;
    }
    unsigned int f = 0;
    int32_t o[4];
#pragma unroll
    for (int j = 0; j < 4; j++) {
        const int64_t acc = d[0][j] - d[1][j] - d[2][j] + d[3][j];
        if (acc > kPmax || acc < -kPmax) f |= 1u;
        o[j] = act ? (int32_t)acc : 0;
    }
    if (sizes)   // n2 % 32 == 0: 8 lanes = one chunk of this row
        chunk_size_out<8>(mag4(o[0], o[1], o[2], o[3]), lane, act ? ((i0 * N1 + i1) * N2 + xi) >> 5 : -1, sizes,
                          bws);
    if (!act) return;
    *reinterpret_cast<int4*>(p + (i0 * N1 + i1) * N2 + xi) = make_int4(o[0], o[1], o[2], o[3]);
    if (f) atomicOr(flags, f);
}

// HSZX / HSZX_ND: one warp per segment; truncated integer mean; p in stream order.  Lane l walks the
// segment's values l, l+32, ... in stream (block row-major) order with incrementally advanced 32-bit
// (z, y, x) offsets — no per-value division; the second pass re-reads the segment from L1/L2.
// Full blocks (every n[a] % B[a] == 0, B2 % 4 == 0, 32 | B0*B1*B2 <= 8192): the mirror of recon.cu's
// k_tile_blocks_fast — a CTA loads a (B0, B1, k*B2) box of q with 16-B row-major loads into shared
// memory in stream (block-contiguous) order, then each warp reduces whole blocks from shared memory
// and stores p with 16-B stores.  k = 8192 / |block| blocks along x per tile.
constexpr int BT_THREADS = 256, BT_ELEMS = 8192;

__global__ void __launch_bounds__(BT_THREADS) k_decor_blockmean_tiles(SegGeo sg, int64_t tpr, int kb,
                                                                      const int32_t* __restrict__ q,
                                                                      int32_t* __restrict__ p,
                                                                      int32_t* __restrict__ meta, unsigned int* flags,
                                                                      uint64_t* sizes, uint8_t* bws) {
    __shared__ __align__(16) int32_t tile[BT_ELEMS];
    const int B0 = (int)sg.B[0], B1 = (int)sg.B[1], B2 = (int)sg.B[2];
    const int segsz = B0 * B1 * B2;
    const int64_t row = blockIdx.x / tpr;                      // block row (b0, b1)
    const int64_t b2a = (blockIdx.x - row * tpr) * kb;
    const int nseg = (int)(sg.G[2] - b2a < kb ? sg.G[2] - b2a : kb);
    const int64_t b0 = row / sg.G[1], b1 = row - b0 * sg.G[1];
    const int64_t n1 = sg.n[1], n2 = sg.n[2];
    const int gpr = nseg * B2 / 4;                             // int4 columns of the box
    const int rows = B0 * B1;
    const int32_t* qb = q + (b0 * B0 * n1 + b1 * B1) * n2 + b2a * B2;
    for (int i = threadIdx.x; i < rows * gpr; i += BT_THREADS) {
        const int zy = i / gpr, g = i - zy * gpr;
        const int zl = zy / B1, yl = zy - zl * B1;
        const int x = 4 * g, t = x / B2, xl = x - t * B2;
        const int4 v = __ldg(reinterpret_cast<const int4*>(qb + ((int64_t)zl * n1 + yl) * n2 + x));
        *reinterpret_cast<int4*>(tile + t * segsz + zy * B2 + xl) = v;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned int f = 0;
    const int64_t seg0 = row * sg.G[2] + b2a;                   // segment index of the tile's first block
    for (int t = warp; t < nseg; t += BT_THREADS / 32) {
        const int32_t* tb = tile + t * segsz;
        int64_t sum = 0;
        for (int j = lane; j < segsz / 4; j += 32) {
            const int4 v = *reinterpret_cast<const int4*>(tb + 4 * j);
            sum += (int64_t)v.x + v.y + v.z + v.w;
        }
        for (int d = 16; d > 0; d >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, d);
        const int64_t mean = (sum >= INT32_MIN && sum <= INT32_MAX) ? (int64_t)((int32_t)sum / segsz) : sum / segsz;
        if (lane == 0) meta[seg0 + t] = (int32_t)mean;
        int4* pb = reinterpret_cast<int4*>(p + (seg0 + t) * segsz);
        for (int j0 = 0; j0 < segsz / 4; j0 += 32) {          // every lane takes part (chunk shuffles)
            const int j = j0 + lane;
            const bool act = j < segsz / 4;
            int32_t o[4] = {0, 0, 0, 0};
            if (act) {
                const int4 v = *reinterpret_cast<const int4*>(tb + 4 * j);
                const int32_t a[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int e = 0; e < 4; e++) {
                    const int64_t d = (int64_t)a[e] - mean;
                    if (d > kPmax || d < -kPmax) f |= 1u;
                    o[e] = (int32_t)d;
                }
                pb[j] = make_int4(o[0], o[1], o[2], o[3]);
            }
            if (sizes)   // 8 lanes = one chunk of the block (32 | segsz)
                chunk_size_out<8>(mag4(o[0], o[1], o[2], o[3]), lane,
                                  act ? (seg0 + t) * (segsz / kChunkCap) + (j >> 3) : -1, sizes, bws);
        }
    }
    if (f) atomicOr(flags, f);
}

constexpr int BM_REG = 16;   // segments of <= 512 values (8^3, 8x8) are held in registers

__global__ void k_decor_blockmean(SegGeo sg, const int32_t* __restrict__ q, int32_t* __restrict__ p,
                                  int32_t* __restrict__ meta, unsigned int* flags) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t nb = sg.G[0] * sg.G[1] * sg.G[2];
    const int64_t n1 = sg.n[1], n2 = sg.n[2];
    unsigned int f = 0;
    const bool small = nb < INT32_MAX;                // 32-bit segment-index arithmetic
    const uint32_t G1 = (uint32_t)sg.G[1], G2 = (uint32_t)sg.G[2];
    for (int64_t b = warp; b < nb; b += nwarps) {
        int64_t b0, b1, b2;
        if (small) {
            const uint32_t bb = (uint32_t)b, r = bb / G2;
            b2 = bb - r * G2;
            b1 = r % G1;
            b0 = r / G1;
        } else {
            b2 = b % sg.G[2];
            const int64_t r = b / sg.G[2];
            b1 = r % sg.G[1];
            b0 = r / sg.G[1];
        }
        const int s0 = (int)seg_ext(sg, 0, b0), s1 = (int)seg_ext(sg, 1, b1), s2 = (int)seg_ext(sg, 2, b2);
        const int size = s0 * s1 * s2;
        const int32_t* qb = q + (b0 * sg.B[0] * n1 + b1 * sg.B[1]) * n2 + b2 * sg.B[2];
        // lane's first value and the per-step advance of 32 values, as (z, y, x) within the segment
        const int zl0 = lane / (s1 * s2), rem0 = lane - zl0 * s1 * s2;
        const int yl0 = rem0 / s2, xl0 = rem0 - yl0 * s2;
        auto walk = [&](auto&& body) {
            int zl = zl0, yl = yl0, xl = xl0;
            for (int l = lane; l < size; l += 32) {
                body(l, qb + ((int64_t)zl * n1 + yl) * n2 + xl);
                xl += 32;
                while (xl >= s2) {
                    xl -= s2;
                    if (++yl == s1) {
                        yl = 0;
                        ++zl;
                    }
                }
            }
        };
        int32_t* pb = p + seg_elem_start(sg, b0, b1, b2);
        if (size <= 32 * BM_REG && s2 <= 32 && !(s2 & (s2 - 1)) && !(s1 & (s1 - 1))) {
            // power-of-two rows (8^3, 8x8 blocks): the whole segment in registers, value l = lane + 32k at
            // (z, y, x) = (r >> lg1, r & (s1-1), l & (s2-1)) with r = l >> lg2 — BM_REG independent loads
            // in flight per lane, one read of q
            const int lg2 = __ffs(s2) - 1, lg1 = __ffs(s1) - 1;
            int32_t v[BM_REG];
#pragma unroll
            for (int k = 0; k < BM_REG; k++) {
                const int l = lane + 32 * k;
                const int r = l >> lg2;
                v[k] = l < size ? __ldg(qb + ((int64_t)(r >> lg1) * n1 + (r & (s1 - 1))) * n2 + (l & (s2 - 1))) : 0;
            }
            int64_t sum = 0;
#pragma unroll
            for (int k = 0; k < BM_REG; k++) sum += v[k];
            for (int d = 16; d > 0; d >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, d);
            const int64_t mean = (sum >= INT32_MIN && sum <= INT32_MAX) ? (int64_t)((int32_t)sum / size) : sum / size;
            if (lane == 0) meta[b] = (int32_t)mean;
#pragma unroll
            for (int k = 0; k < BM_REG; k++) {
                if (lane + 32 * k < size) {
                    const int64_t d = (int64_t)v[k] - mean;
                    if (d > kPmax || d < -kPmax) f |= 1u;
                    pb[lane + 32 * k] = (int32_t)d;
                }
            }
            continue;
        }
        int64_t sum = 0;
        walk([&](int, const int32_t* a) { sum += __ldg(a); });
        for (int d = 16; d > 0; d >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, d);
        // C division truncates toward zero (compressors.py:134-138); 32-bit when the sum fits
        const int64_t mean = (sum >= INT32_MIN && sum <= INT32_MAX) ? (int64_t)((int32_t)sum / size) : sum / size;
        if (lane == 0) meta[b] = (int32_t)mean;
        walk([&](int l, const int32_t* a) {
            const int64_t d = (int64_t)__ldg(a) - mean;
            if (d > kPmax || d < -kPmax) f |= 1u;
            pb[l] = (int32_t)d;
        });
    }
    if (f) atomicOr(flags, f);
}

}  // namespace hszg

using namespace hszg;

int hszg_set_cuda_error(HszgErr* err, cudaError_t e, const char* where);
static inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }
static bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

template <typename T>
static int minmax_impl(const T* field, int64_t n, double* out_dev, int64_t* nonfinite_dev, void* ws,
                       size_t ws_bytes, cudaStream_t st) {
    const int grid = grid_for(n, 256 * 8, 148 * 8);
    if (ws_bytes < (size_t)grid * sizeof(MinMaxPart)) return HSZG_INVALID_ARG;
    MinMaxPart* parts = reinterpret_cast<MinMaxPart*>(ws);
    k_minmax<T><<<grid, 256, 0, st>>>(field, n, parts);
    k_minmax_final<<<1, 32, 0, st>>>(parts, grid, out_dev, nonfinite_dev);
    return cudaGetLastError() == cudaSuccess ? HSZG_OK : HSZG_CUDA;
}

extern "C" int hszg_minmax_f32(const float* field, int64_t n, double* out_dev, int64_t* nonfinite_dev, void* ws,
                               size_t ws_bytes, void* stream) {
    return minmax_impl(field, n, out_dev, nonfinite_dev, ws, ws_bytes, as_stream(stream));
}

extern "C" int hszg_minmax_f64(const double* field, int64_t n, double* out_dev, int64_t* nonfinite_dev, void* ws,
                               size_t ws_bytes, void* stream) {
    return minmax_impl(field, n, out_dev, nonfinite_dev, ws, ws_bytes, as_stream(stream));
}

static int read_flags(unsigned int* flags_dev, unsigned int* h, cudaStream_t st, HszgErr* err) {
    cudaMemcpyAsync(h, flags_dev, 4, cudaMemcpyDeviceToHost, st);
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return hszg_set_cuda_error(err, e, "flag readback");
    return HSZG_OK;
}

template <typename T>
static int quantize_impl(const T* field, int64_t n, double recip, int32_t* q, void* ws, size_t ws_bytes,
                         cudaStream_t st, HszgErr* err) {
    err->status = HSZG_OK;
    if (ws_bytes < 4) return HSZG_INVALID_ARG;
    unsigned int* flags = reinterpret_cast<unsigned int*>(ws);
    cudaMemsetAsync(flags, 0, 4, st);
    const bool vec = std::is_same<T, float>::value && n % 4 == 0 && (reinterpret_cast<uintptr_t>(field) & 15) == 0 &&
                     (reinterpret_cast<uintptr_t>(q) & 15) == 0;
    if (n > 0 && vec)
        k_quantize_f32x4<<<grid_for(n / 4, 256 * 4, 148 * 16), 256, 0, st>>>(reinterpret_cast<const float4*>(field),
                                                                             n / 4, recip, reinterpret_cast<int4*>(q),
                                                                             flags);
    else if (n > 0)
        k_quantize<T><<<grid_for(n, 256 * 4, 148 * 32), 256, 0, st>>>(field, n, recip, q, flags);
    unsigned int h = 0;
    int r = read_flags(flags, &h, st, err);
    if (r) return r;
    if (h & 1u) {
        err->status = HSZG_EPS_TOO_SMALL;
        snprintf(err->message, sizeof(err->message), "quantization index exceeds %d; increase the error bound", kQmax);
        return HSZG_EPS_TOO_SMALL;
    }
    if (h & 2u) {
        err->status = HSZG_VALUE;
        snprintf(err->message, sizeof(err->message), "field contains NaN or Inf; refusing to quantize");
        return HSZG_VALUE;
    }
    return HSZG_OK;
}

extern "C" int hszg_quantize_f32(const float* field, int64_t n, double recip, int32_t* q, void* ws, size_t ws_bytes,
                                 void* stream, HszgErr* err) {
    return quantize_impl(field, n, recip, q, ws, ws_bytes, as_stream(stream), err);
}

extern "C" int hszg_quantize_f64(const double* field, int64_t n, double recip, int32_t* q, void* ws,
                                 size_t ws_bytes, void* stream, HszgErr* err) {
    return quantize_impl(field, n, recip, q, ws, ws_bytes, as_stream(stream), err);
}

static int decorrelate_impl(const HszgGeom* g, const int32_t* q, int32_t* p, int32_t* metadata, uint64_t* sizes,
                            uint8_t* bws, int* fused, void* ws, size_t ws_bytes, void* stream, HszgErr* err);

extern "C" int hszg_decorrelate(const HszgGeom* g, const int32_t* q, int32_t* p, int32_t* metadata, void* ws,
                                size_t ws_bytes, void* stream, HszgErr* err) {
    return decorrelate_impl(g, q, p, metadata, nullptr, nullptr, nullptr, ws, ws_bytes, stream, err);
}

extern "C" int hszg_decorrelate_sized(const HszgGeom* g, const int32_t* q, int32_t* p, int32_t* metadata,
                                      uint64_t* sizes, uint8_t* bitwidths, int* fused, void* ws, size_t ws_bytes,
                                      void* stream, HszgErr* err) {
    return decorrelate_impl(g, q, p, metadata, sizes, bitwidths, fused, ws, ws_bytes, stream, err);
}

static int decorrelate_impl(const HszgGeom* g, const int32_t* q, int32_t* p, int32_t* metadata, uint64_t* sizes,
                            uint8_t* bws, int* fused, void* ws, size_t ws_bytes, void* stream, HszgErr* err) {
    if (fused) *fused = 0;
    const bool full = sizes && bws && g->n_chunks * kChunkCap == g->n;   // every chunk 32 values
    err->status = HSZG_OK;
    cudaStream_t st = as_stream(stream);
    if (ws_bytes < 4) return HSZG_INVALID_ARG;
    unsigned int* flags = reinterpret_cast<unsigned int*>(ws);
    cudaMemsetAsync(flags, 0, 4, st);
    const SegGeo sg = make_seggeo(*g);
    if (g->n > 0) {
        switch (g->kind) {
            case HSZG_HSZP:
                if (g->n % 4 == 0 && al16(q) && al16(p)) {
                    k_decor_prev_x4<<<grid_for(g->n / 4, 256 * 4, 148 * 16), 256, 0, st>>>(
                        reinterpret_cast<const int4*>(q), g->n / 4, reinterpret_cast<int4*>(p), flags,
                        full ? sizes : nullptr, bws);
                    if (full) *fused = 1;
                } else
                    k_decor_prev<<<grid_for(g->n, 256 * 4, 148 * 32), 256, 0, st>>>(q, g->n, p, flags);
                break;
            case HSZG_HSZP_ND: {
                int64_t n[3] = {1, 1, 1};
                for (int k = 0; k < g->ndims; k++) n[3 - g->ndims + k] = g->dims[k];
                if (n[0] > 65535 || n[1] > 65535) {
                    err->status = HSZG_INVALID_ARG;
                    snprintf(err->message, sizeof(err->message), "grid too large for the Lorenzo launch");
                    return HSZG_INVALID_ARG;
                }
                if (n[2] % 4 == 0 && al16(q) && al16(p)) {
                    const bool fz = full && n[2] % kChunkCap == 0;
                    dim3 grid4((unsigned)((n[2] / 4 + 127) / 128), (unsigned)n[1], (unsigned)n[0]);
                    k_decor_lorenzo_x4<<<grid4, 128, 0, st>>>(q, n[0], n[1], n[2], p, flags, fz ? sizes : nullptr,
                                                              bws);
                    if (fz) *fused = 1;
                } else {
                    dim3 grid((unsigned)((n[2] + 255) / 256), (unsigned)n[1], (unsigned)n[0]);
                    k_decor_lorenzo<<<grid, 256, 0, st>>>(q, n[0], n[1], n[2], p, flags);
                }
                break;
            }
            default: {
                const int64_t nb = sg.G[0] * sg.G[1] * sg.G[2];
                const int64_t B = sg.B[2];
                if (sg.n[0] == 1 && sg.n[1] == 1 && B == 32 && g->n % 32 == 0 && al16(q) && al16(p)) {
                    const int64_t nblk = g->n / 32;
                    k_decor_blockmean_b32<<<(unsigned)((nblk + 255) / 256), 256, 0, st>>>(
                        reinterpret_cast<const int4*>(q), nblk, reinterpret_cast<int4*>(p), metadata, flags,
                        full ? sizes : nullptr, bws);
                    if (full) *fused = 1;
                    break;
                }
                if (sg.n[0] == 1 && sg.n[1] == 1 && B <= 32 && (32 % B) == 0) {
                    const int lgB = __builtin_ctzll((unsigned long long)B);
                    const bool fz = full && B == 32;
                    k_decor_blockmean_1d<<<grid_for(g->n, 256 * 4, 148 * 16), 256, 0, st>>>(
                        q, g->n, lgB, p, metadata, flags, fz ? sizes : nullptr, bws);
                    if (fz) *fused = 1;
                    break;
                }
                const int64_t segsz = sg.B[0] * sg.B[1] * sg.B[2];
                if (sg.n[0] % sg.B[0] == 0 && sg.n[1] % sg.B[1] == 0 && sg.n[2] % sg.B[2] == 0 && sg.B[2] % 4 == 0 &&
                    segsz % 32 == 0 && segsz <= BT_ELEMS && al16(q) && al16(p) && sg.n[2] % 4 == 0) {
                    const int kb = (int)(BT_ELEMS / segsz);
                    const int64_t tpr = (sg.G[2] + kb - 1) / kb;
                    k_decor_blockmean_tiles<<<(unsigned)(sg.G[0] * sg.G[1] * tpr), BT_THREADS, 0, st>>>(
                        sg, tpr, kb, q, p, metadata, flags, full ? sizes : nullptr, bws);
                    if (full) *fused = 1;
                    break;
                }
                k_decor_blockmean<<<grid_for(nb * 32, 256, 148 * 64), 256, 0, st>>>(sg, q, p, metadata, flags);
                break;
            }
        }
        { const cudaError_t e_ = cudaGetLastError(); if (e_ != cudaSuccess) return hszg_set_cuda_error(err, e_, "decorrelate"); }
    }
    unsigned int h = 0;
    int r = read_flags(flags, &h, st, err);
    if (r) return r;
    if (h) {
        err->status = HSZG_EPS_TOO_SMALL;
        snprintf(err->message, sizeof(err->message),
                 "decorrelated residual overflows 32-bit range; increase the error bound");
        return HSZG_EPS_TOO_SMALL;
    }
    return HSZG_OK;
}
