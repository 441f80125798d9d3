// gen.cu — synthetic input for BASELINE config 5 (2048^3), generated on the device.
//
// Not part of the decompression hot path: the config-5 field (32 GiB) takes
// hours to build on the host, so it is produced here, slab by
// slab, from a counter-based RNG (any z-range of any rank is reproducible):
//   field = sum_m A_m sin(2 pi (kz z/N0 + ky y/N1 + kx x/N2) + phi_m)
//         + scale * GaussianFilter_sigma(white noise)      (scipy "reflect" boundaries)
#include <cstdint>
#include <cuda_runtime.h>
#include "../../include/hszg.h"

namespace {

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

__global__ void k_gen_noise(float* out, int64_t e0, int64_t nz, int64_t N1, int64_t N2, uint64_t seed) {
    const int64_t n = nz * N1 * N2;
    const uint64_t key = splitmix64(seed * 0x632be59bd9b4e019ull + 12345);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t gidx = (uint64_t)(e0 * N1 * N2 + i);
        const uint64_t h = splitmix64(gidx ^ key);
        const float u1 = ((uint32_t)(h >> 40) + 1u) * (1.0f / 16777217.0f);   // (0, 1]
        const float u2 = (uint32_t)(h & 0xffffffu) * (1.0f / 16777216.0f);    // [0, 1)
        out[i] = sqrtf(-2.0f * logf(u1)) * cospif(2.0f * u2);
    }
}

__device__ __forceinline__ int64_t reflect(int64_t i, int64_t n) {
    if (i < 0) i = -i - 1;
    if (i >= n) i = 2 * n - i - 1;
    return i;
}

// x (axis 2) or y (axis 1) pass inside an extended slab holding whole planes
__global__ void k_gauss_xy(const float* in, float* out, int64_t nz, int64_t N1, int64_t N2, int axis, const float* w,
                           int r) {
    const int64_t n = nz * N1 * N2;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t x = i % N2;
        const int64_t y = (i / N2) % N1;
        const int64_t zb = i - y * N2 - x;   // plane base
        float acc = 0.f;
        if (axis == 2) {
            for (int k = -r; k <= r; k++) acc += w[k + r] * __ldg(in + zb + y * N2 + reflect(x + k, N2));
        } else {
            for (int k = -r; k <= r; k++) acc += w[k + r] * __ldg(in + zb + reflect(y + k, N1) * N2 + x);
        }
        out[i] = acc;
    }
}

__global__ void k_gauss_z(const float* in, float* out, int64_t e0, int64_t z0, int64_t nzout, int64_t N0, int64_t N1,
                          int64_t N2, const float* w, int r) {
    const int64_t plane = N1 * N2;
    const int64_t n = nzout * plane;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t zl = i / plane;
        const int64_t rem = i - zl * plane;
        const int64_t z = z0 + zl;
        float acc = 0.f;
        for (int k = -r; k <= r; k++) acc += w[k + r] * __ldg(in + (reflect(z + k, N0) - e0) * plane + rem);
        out[i] = acc;
    }
}

__global__ void k_gen_modes(float* out, int64_t z0, int64_t nz, int64_t N0, int64_t N1, int64_t N2,
                            const double* modes, int nmodes, double scale) {
    const int64_t n = nz * N1 * N2;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t x = i % N2;
        const int64_t y = (i / N2) % N1;
        const int64_t z = z0 + i / (N1 * N2);
        double acc = 0.0;
        for (int m = 0; m < nmodes; m++) {
            const double* p = modes + 5 * m;   // kz, ky, kx, A, phi
            double f = p[0] * (double)z / (double)N0 + p[1] * (double)y / (double)N1 + p[2] * (double)x / (double)N2;
            f -= floor(f);
            acc += p[3] * (double)sinpif((float)(2.0 * f + p[4] * 0.31830988618379067));
        }
        out[i] = (float)(acc + scale * (double)out[i]);
    }
}

inline int grid_of(int64_t n) {
    int64_t g = (n + 255) / 256;
    return (int)(g < 148 * 64 ? (g < 1 ? 1 : g) : 148 * 64);
}

}  // namespace

extern "C" int hszg_gen_noise(float* out, int64_t e0, int64_t nz, const int64_t* dims, uint64_t seed, void* stream) {
    k_gen_noise<<<grid_of(nz * dims[1] * dims[2]), 256, 0, (cudaStream_t)stream>>>(out, e0, nz, dims[1], dims[2], seed);
    return cudaGetLastError() == cudaSuccess ? HSZG_OK : HSZG_CUDA;
}

extern "C" int hszg_gauss_pass(const float* in, float* out, int64_t e0, int64_t nz, const int64_t* dims, int axis,
                               const float* w, int r, void* stream) {
    (void)e0;
    if (axis != 1 && axis != 2) return HSZG_INVALID_ARG;
    k_gauss_xy<<<grid_of(nz * dims[1] * dims[2]), 256, 0, (cudaStream_t)stream>>>(in, out, nz, dims[1], dims[2], axis,
                                                                                  w, r);
    return cudaGetLastError() == cudaSuccess ? HSZG_OK : HSZG_CUDA;
}

extern "C" int hszg_gauss_pass_z(const float* in, float* out, int64_t e0, int64_t nz, int64_t z0, int64_t nzout,
                                 const int64_t* dims, const float* w, int r, void* stream) {
    (void)nz;
    k_gauss_z<<<grid_of(nzout * dims[1] * dims[2]), 256, 0, (cudaStream_t)stream>>>(in, out, e0, z0, nzout, dims[0],
                                                                                    dims[1], dims[2], w, r);
    return cudaGetLastError() == cudaSuccess ? HSZG_OK : HSZG_CUDA;
}

extern "C" int hszg_gen_modes(float* out, int64_t z0, int64_t nz, const int64_t* dims, const double* modes, int nmodes,
                              double scale, void* stream) {
    k_gen_modes<<<grid_of(nz * dims[1] * dims[2]), 256, 0, (cudaStream_t)stream>>>(out, z0, nz, dims[0], dims[1],
                                                                                   dims[2], modes, nmodes, scale);
    return cudaGetLastError() == cudaSuccess ? HSZG_OK : HSZG_CUDA;
}
