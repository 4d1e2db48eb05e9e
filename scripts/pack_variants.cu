// pack_variants.cu -- design-space probe for the multi-tensor pack kernel
// (a1): b[base + k] = cast(g[k]) over ResNet-50-sized gradients cut into
// 4096-element items, fp32 (8 B/param) and fp16 (6 B/param).  Standalone;
// ranks items-per-CTA choices before csrc/cmn_kernels.cu adopts one.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o build/pack_variants scripts/pack_variants.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)
constexpr int64_t N = 25557056;
constexpr int ITEM = 4096;

template <int DT>
__device__ __forceinline__ void st(void *p, int64_t j, const float4 &x) {
    if constexpr (DT == 0) {
        __stcs(reinterpret_cast<float4 *>(static_cast<float *>(p) + j), x);
    } else {
        const uint32_t a = __half_as_ushort(__float2half_rn(x.x)) | (uint32_t(__half_as_ushort(__float2half_rn(x.y))) << 16);
        const uint32_t b = __half_as_ushort(__float2half_rn(x.z)) | (uint32_t(__half_as_ushort(__float2half_rn(x.w))) << 16);
        __stcs(reinterpret_cast<uint2 *>(static_cast<uint16_t *>(p) + j), make_uint2(a, b));
    }
}

template <int DT, int K, int THR>
__global__ void __launch_bounds__(THR) k_pack(const float *__restrict__ g, void *__restrict__ out, int items) {
    constexpr int U = ITEM / 4 / THR;
    const int ib = blockIdx.x * K;
    float4 x[K][U];
#pragma unroll
    for (int j = 0; j < K; ++j)
        if (ib + j < items) {
            const float4 *src = reinterpret_cast<const float4 *>(g + (int64_t)(ib + j) * ITEM);
#pragma unroll
            for (int u = 0; u < U; ++u) x[j][u] = __ldcs(src + threadIdx.x + u * THR);
        }
#pragma unroll
    for (int j = 0; j < K; ++j)
        if (ib + j < items) {
#pragma unroll
            for (int u = 0; u < U; ++u) st<DT>(out, (int64_t)(ib + j) * ITEM + 4 * (threadIdx.x + u * THR), x[j][u]);
        }
}

int main() {
    float *g; void *out;
    CK(cudaMalloc(&g, N * 4)); CK(cudaMalloc(&out, N * 4));
    CK(cudaMemset(g, 0, N * 4));
    const int items = (int)(N / ITEM);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto run = [&](const char *name, int dt, auto launch) {
        for (int r = 0; r < 20; ++r) launch();
        cudaDeviceSynchronize();
        cudaEventRecord(e0);
        for (int r = 0; r < 200; ++r) launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        const double us = ms * 1e3 / 200, bytes = (double)items * ITEM * (dt == 0 ? 8 : 6);
        printf("{\"variant\": \"%s\", \"dtype\": \"%s\", \"us\": %.2f, \"gbs\": %.1f}\n", name, dt ? "fp16" : "fp32",
               us, bytes / (us * 1e-6) / 1e9);
    };
#define V(DT, K, THR) run("items/CTA=" #K " thr=" #THR, DT, [&] { k_pack<DT, K, THR><<<(items + K - 1) / K, THR>>>(g, out, items); })
    V(0, 1, 256); V(0, 2, 256); V(0, 4, 256); V(0, 8, 256); V(0, 2, 512); V(0, 4, 512);
    V(1, 1, 256); V(1, 2, 256); V(1, 4, 256); V(1, 8, 256); V(1, 2, 512); V(1, 4, 512);
    CK(cudaGetLastError());
    return 0;
}
