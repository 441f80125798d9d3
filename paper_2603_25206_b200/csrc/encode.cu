// encode.cu — the compress side (K-ENC): value range, quantization and decorrelation.
//
//   resolve_eps  quant.py:56-66         -> k_minmax (+ NaN/Inf count)
//   quantize     quant.py:69-82         -> k_quantize: floor(d*recip + 0.5) in fp64 with the
//                                          multiply and add rounded separately (no FMA, as numpy)
//   decorrelate  compressors.py:149-198 -> k_decor_prev (HSZP), k_decor_lorenzo (HSZP_ND),
//                                          k_decor_blockmean (HSZX, HSZX_ND; truncating means 134-138)
// The chunk encoder proper (bit widths, scan, pack) lives in codec.cu.
#include <cstdio>
#include <cfloat>
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

// HSZX / HSZX_ND: one warp per segment; truncated integer mean; p in stream order
__global__ void k_decor_blockmean(SegGeo sg, const int32_t* q, int32_t* p, int32_t* meta, unsigned int* flags) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t nb = sg.G[0] * sg.G[1] * sg.G[2];
    unsigned int f = 0;
    for (int64_t b = warp; b < nb; b += nwarps) {
        const int64_t b2 = b % sg.G[2];
        const int64_t r = b / sg.G[2];
        const int64_t b1 = r % sg.G[1];
        const int64_t b0 = r / sg.G[1];
        const int64_t s0 = seg_ext(sg, 0, b0), s1 = seg_ext(sg, 1, b1), s2 = seg_ext(sg, 2, b2);
        const int64_t size = s0 * s1 * s2;
        const int64_t z0 = b0 * sg.B[0], y0 = b1 * sg.B[1], x0 = b2 * sg.B[2];
        int64_t sum = 0;
        for (int64_t l = lane; l < size; l += 32) {
            const int64_t zl = l / (s1 * s2), rem = l - zl * s1 * s2, yl = rem / s2, xl = rem - yl * s2;
            sum += q[((z0 + zl) * sg.n[1] + (y0 + yl)) * sg.n[2] + x0 + xl];
        }
        for (int d = 16; d > 0; d >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, d);
        const int64_t mean = sum / size;   // C division truncates toward zero (compressors.py:134-138)
        if (lane == 0) meta[b] = (int32_t)mean;
        const int64_t e0 = seg_elem_start(sg, b0, b1, b2);
        for (int64_t l = lane; l < size; l += 32) {
            const int64_t zl = l / (s1 * s2), rem = l - zl * s1 * s2, yl = rem / s2, xl = rem - yl * s2;
            const int64_t d = (int64_t)q[((z0 + zl) * sg.n[1] + (y0 + yl)) * sg.n[2] + x0 + xl] - mean;
            if (d > kPmax || d < -kPmax) f |= 1u;
            p[e0 + l] = (int32_t)d;
        }
    }
    if (f) atomicOr(flags, f);
}

}  // namespace hszg

using namespace hszg;

int hszg_set_cuda_error(HszgErr* err, cudaError_t e, const char* where);
static inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

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
    if (n > 0) k_quantize<T><<<grid_for(n, 256 * 4, 148 * 32), 256, 0, st>>>(field, n, recip, q, flags);
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

extern "C" int hszg_decorrelate(const HszgGeom* g, const int32_t* q, int32_t* p, int32_t* metadata, void* ws,
                                size_t ws_bytes, void* stream, HszgErr* err) {
    err->status = HSZG_OK;
    cudaStream_t st = as_stream(stream);
    if (ws_bytes < 4) return HSZG_INVALID_ARG;
    unsigned int* flags = reinterpret_cast<unsigned int*>(ws);
    cudaMemsetAsync(flags, 0, 4, st);
    const SegGeo sg = make_seggeo(*g);
    if (g->n > 0) {
        switch (g->kind) {
            case HSZG_HSZP:
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
                dim3 grid((unsigned)((n[2] + 255) / 256), (unsigned)n[1], (unsigned)n[0]);
                k_decor_lorenzo<<<grid, 256, 0, st>>>(q, n[0], n[1], n[2], p, flags);
                break;
            }
            default: {
                const int64_t nb = sg.G[0] * sg.G[1] * sg.G[2];
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
