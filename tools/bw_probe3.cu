// bw_probe3.cu — HBM write ceiling for the analytics emit pattern (4 fp32 output planes per input
// plane), by CTA tile shape and store instruction.  Standalone (no torch):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bw_probe3 tools/bw_probe3.cu && tools/bw_probe3
// Volume 2048 x 2048 x NZ planes, outputs o0..o3 (fp32), optional int8 input plane read (1 B/value).
// Patterns:
//   seq    grid-stride float4 streaming stores over the flat volume (the upper bound)
//   tile   CTA = TX columns x TY rows, sliding along z (k_zsweep_ring / k_fused_blocks shape),
//          st.global.cs float4 from registers
//   bulk   same tiles, values staged in shared memory and written by cp.async.bulk (1-D TMA) per row
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); return 1; } } while (0)

constexpr int N2 = 2048, N1 = 2048;

__global__ void k_seq(const int8_t* __restrict__ in, float4* o0, float4* o1, float4* o2, float4* o3, long n4) {
    for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (long)gridDim.x * blockDim.x) {
        float v = in ? (float)in[i * 4] : (float)i;
        float4 f = make_float4(v, v + 1, v + 2, v + 3);
        __stcs(o0 + i, f); __stcs(o1 + i, f); __stcs(o2 + i, f); __stcs(o3 + i, f);
    }
}

template <int TX, int TY>
__global__ void k_tile(const int8_t* __restrict__ in, float* o0, float* o1, float* o2, float* o3, int nz) {
    const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
    constexpr int G = TX / 4;                    // float4 per row
    for (int z = 0; z < nz; z++) {
        for (int e = threadIdx.x; e < G * TY; e += blockDim.x) {
            const int r = e / G, g = e - r * G;
            const long off = ((long)z * N1 + y0 + r) * N2 + x0 + 4 * g;
            float v = in ? (float)in[off] : (float)off;
            float4 f = make_float4(v, v + 1, v + 2, v + 3);
            __stcs(reinterpret_cast<float4*>(o0 + off), f);
            __stcs(reinterpret_cast<float4*>(o1 + off), f);
            __stcs(reinterpret_cast<float4*>(o2 + off), f);
            __stcs(reinterpret_cast<float4*>(o3 + off), f);
        }
    }
}

__device__ __forceinline__ void bulk_store(void* g, const void* s, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(g),
                 "r"((uint32_t)__cvta_generic_to_shared(s)), "r"(bytes) : "memory");
}

// staged: two buffers of 4 outputs x TY x TX floats; thread 0 issues TY*4 bulk stores per plane
template <int TX, int TY>
__global__ void k_bulk(const int8_t* __restrict__ in, float* o0, float* o1, float* o2, float* o3, int nz) {
    extern __shared__ __align__(128) float sm[];
    const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
    constexpr int G = TX / 4;
    constexpr int PB = 4 * TY * TX;              // floats per buffer
    float* outs[4] = {o0, o1, o2, o3};
    for (int z = 0; z < nz; z++) {
        float* buf = sm + (z & 1) * PB;
        if (threadIdx.x == 0 && z >= 2) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        __syncthreads();                         // buffer z&1 free again
        for (int e = threadIdx.x; e < G * TY; e += blockDim.x) {
            const int r = e / G, g = e - r * G;
            const long off = ((long)z * N1 + y0 + r) * N2 + x0 + 4 * g;
            float v = in ? (float)in[off] : (float)off;
            float4 f = make_float4(v, v + 1, v + 2, v + 3);
#pragma unroll
            for (int k = 0; k < 4; k++) reinterpret_cast<float4*>(buf + (k * TY + r) * TX)[g] = f;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int k = 0; k < 4; k++)
                for (int r = 0; r < TY; r++)
                    bulk_store(outs[k] + ((long)z * N1 + y0 + r) * N2 + x0, buf + (k * TY + r) * TX, TX * 4);
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
    }
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
    const int NZ = 64;
    const long n = (long)N2 * N1 * NZ;
    int8_t* in;
    float* o[4];
    CK(cudaMalloc(&in, n));
    CK(cudaMemset(in, 1, n));
    for (int k = 0; k < 4; k++) CK(cudaMalloc(&o[k], n * 4));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto run = [&](const char* name, auto launch) {
        launch();
        cudaDeviceSynchronize();
        float best = 1e9;
        for (int it = 0; it < 7; it++) {
            cudaEventRecord(a);
            launch();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (ms < best) best = ms;
        }
        cudaError_t e = cudaGetLastError();
        printf("%-34s %8.3f ms  write %6.0f GB/s  (+read: %6.0f)  %s\n", name, best, 16.0 * n / best / 1e6,
               17.0 * n / best / 1e6, e == cudaSuccess ? "" : cudaGetErrorString(e));
    };
    for (int rd = 0; rd < 2; rd++) {
        const int8_t* src = rd ? in : nullptr;
        printf("--- %s\n", rd ? "with int8 input read" : "write only");
        for (int blocks : {148 * 4, 148 * 16})
            run(rd ? "seq (read)" : "seq", [&] {
                k_seq<<<blocks, 256>>>(src, (float4*)o[0], (float4*)o[1], (float4*)o[2], (float4*)o[3], n / 4);
            });
#define TILE(TX, TY, T)                                                                                     \
        run("tile " #TX "x" #TY " thr " #T, [&] {                                                             \
            k_tile<TX, TY><<<dim3(N2 / TX, N1 / TY), T>>>(src, o[0], o[1], o[2], o[3], NZ);               \
        });
        TILE(128, 16, 256) TILE(128, 16, 512) TILE(256, 8, 256) TILE(512, 4, 256) TILE(2048, 1, 512)
        TILE(256, 16, 512) TILE(512, 8, 512)
#define BULK(TX, TY, T)                                                                                     \
        {                                                                                                   \
            const size_t sm = 2 * 4 * TY * TX * 4;                                                          \
            cudaFuncSetAttribute(k_bulk<TX, TY>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);     \
            run("bulk " #TX "x" #TY " thr " #T, [&] {                                                         \
                k_bulk<TX, TY><<<dim3(N2 / TX, N1 / TY), T, sm>>>(src, o[0], o[1], o[2], o[3], NZ);       \
            });                                                                                             \
        }
        BULK(128, 16, 256) BULK(256, 8, 256) BULK(512, 4, 256) BULK(2048, 1, 256) BULK(128, 8, 256)
    }
    return 0;
}
