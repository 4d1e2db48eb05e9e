// update_variants.cu -- design-space probe for the N = 1 fused step kernel
// (k_update_direct): v = fma(mu, v, g); w = fma(-lr, v, w) over 25.6M fp32
// elements (ResNet-50 size), 20 B/element.  Standalone (not the product):
// it ranks memory-access designs on B200 before one is adopted in
// csrc/cmn_kernels.cu.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o build/update_variants scripts/update_variants.cu
//   build/update_variants
//
// Variants:
//   A  one 4096-element item per CTA, 256 thr, 4 float4/thread/array, ld/st .cs   (current)
//   B  as A with default cache operators
//   C  2048-element items (2 float4/thread/array)
//   D  8192-element items, 512 threads
//   E  persistent grid (4 CTAs/SM), grid-stride over 4096-element items
//   F  TMA bulk copies: 3 x 16 KB cp.async.bulk loads into smem (mbarrier),
//      compute in smem, 2 bulk stores; one item per CTA
//   G  as F, persistent, 2-stage smem ring (loads of item i+1 under item i)
//   H  as A with the L2::256B prefetch-size hint on the loads
//   I  as H without .cs
//   J  8192-element items, 256 threads (8 float4 per thread per array in flight)
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int64_t N = 25557056;

__device__ __forceinline__ void upd(float g, float lr, float mu, float &w, float &v) {
    v = __fmaf_rn(mu, v, g);
    w = __fmaf_rn(-lr, v, w);
}
__device__ __forceinline__ void upd4(const float4 &g, float lr, float mu, float4 &w, float4 &v) {
    upd(g.x, lr, mu, w.x, v.x); upd(g.y, lr, mu, w.y, v.y);
    upd(g.z, lr, mu, w.z, v.z); upd(g.w, lr, mu, w.w, v.w);
}

template <int ITEM, int THR, bool CS>
__global__ void __launch_bounds__(THR) k_item(const float *__restrict__ g, float *__restrict__ w,
                                              float *__restrict__ v, float lr, float mu) {
    constexpr int U = ITEM / 4 / THR;
    const int64_t base = (int64_t)blockIdx.x * ITEM;
    const float4 *g4 = reinterpret_cast<const float4 *>(g + base);
    float4 *w4 = reinterpret_cast<float4 *>(w + base);
    float4 *v4 = reinterpret_cast<float4 *>(v + base);
    const int nv = (int)(int64_t)((ITEM) < (N - base) ? (ITEM) : (N - base)) / 4;
    float4 a[U], b[U], c[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int q = threadIdx.x + u * THR;
        if (q < nv) {
            if (CS) { a[u] = __ldcs(g4 + q); b[u] = __ldcs(w4 + q); c[u] = __ldcs(v4 + q); }
            else { a[u] = g4[q]; b[u] = w4[q]; c[u] = v4[q]; }
        }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int q = threadIdx.x + u * THR;
        if (q < nv) {
            upd4(a[u], lr, mu, b[u], c[u]);
            if (CS) { __stcs(w4 + q, b[u]); __stcs(v4 + q, c[u]); }
            else { w4[q] = b[u]; v4[q] = c[u]; }
        }
    }
}

// H / I: variant A with an L2 prefetch-size hint on the loads (256-B
// sectors fetched per miss), with (.cs) or without the streaming operator.
template <bool CS>
__device__ __forceinline__ float4 ld_hint(const float4 *p) {
    float4 r;
    if (CS)
        asm volatile("ld.global.cs.L2::256B.v4.f32 {%0,%1,%2,%3}, [%4];"
                     : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
    else
        asm volatile("ld.global.L2::256B.v4.f32 {%0,%1,%2,%3}, [%4];"
                     : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
    return r;
}
template <bool CS>
__global__ void __launch_bounds__(256) k_hint(const float *__restrict__ g, float *__restrict__ w,
                                              float *__restrict__ v, float lr, float mu) {
    constexpr int U = 4;
    const int64_t base = (int64_t)blockIdx.x * 4096;
    const float4 *g4 = reinterpret_cast<const float4 *>(g + base);
    float4 *w4 = reinterpret_cast<float4 *>(w + base);
    float4 *v4 = reinterpret_cast<float4 *>(v + base);
    const int nv = (int)(int64_t)((4096) < (N - base) ? (4096) : (N - base)) / 4;
    float4 a[U], b[U], c[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int q = threadIdx.x + u * 256;
        if (q < nv) { a[u] = ld_hint<CS>(g4 + q); b[u] = ld_hint<CS>(w4 + q); c[u] = ld_hint<CS>(v4 + q); }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int q = threadIdx.x + u * 256;
        if (q < nv) { upd4(a[u], lr, mu, b[u], c[u]); __stcs(w4 + q, b[u]); __stcs(v4 + q, c[u]); }
    }
}

__global__ void __launch_bounds__(256) k_persist(const float *__restrict__ g, float *__restrict__ w,
                                                 float *__restrict__ v, float lr, float mu, int items) {
    for (int it = blockIdx.x; it < items; it += gridDim.x) {
        const int64_t base = (int64_t)it * 4096;
        const float4 *g4 = reinterpret_cast<const float4 *>(g + base);
        float4 *w4 = reinterpret_cast<float4 *>(w + base);
        float4 *v4 = reinterpret_cast<float4 *>(v + base);
        const int nv = (int)(int64_t)((4096) < (N - base) ? (4096) : (N - base)) / 4;
        float4 a[4], b[4], c[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int q = threadIdx.x + u * 256;
            if (q < nv) { a[u] = __ldcs(g4 + q); b[u] = __ldcs(w4 + q); c[u] = __ldcs(v4 + q); }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int q = threadIdx.x + u * 256;
            if (q < nv) { upd4(a[u], lr, mu, b[u], c[u]); __stcs(w4 + q, b[u]); __stcs(v4 + q, c[u]); }
        }
    }
}

// ---------------------------------------------------------------- TMA bulk
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_load(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bulk_store(void *dst, const void *src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                 ::"l"(dst), "r"(smem_u32(src)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

constexpr int TI = 4096;               // elements per TMA item
constexpr uint32_t TB = TI * 4;        // 16 KB per array

__global__ void __launch_bounds__(256) k_tma(const float *__restrict__ g, float *__restrict__ w,
                                             float *__restrict__ v, float lr, float mu) {
    extern __shared__ __align__(128) float sm[];
    float *sg = sm, *sw = sm + TI, *sv = sm + 2 * TI;
    __shared__ __align__(8) uint64_t bar;
    const int64_t base = (int64_t)blockIdx.x * TI;
    const uint32_t bytes = (uint32_t)(int64_t)((TI) < (N - base) ? (TI) : (N - base)) * 4;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        mbar_expect_tx(&bar, 3 * bytes);
        bulk_load(sg, g + base, bytes, &bar);
        bulk_load(sw, w + base, bytes, &bar);
        bulk_load(sv, v + base, bytes, &bar);
    }
    mbar_wait(&bar, 0);
    const int nv = bytes / 16;
    for (int q = threadIdx.x; q < nv; q += 256) {
        float4 a = reinterpret_cast<float4 *>(sg)[q], b = reinterpret_cast<float4 *>(sw)[q],
               c = reinterpret_cast<float4 *>(sv)[q];
        upd4(a, lr, mu, b, c);
        reinterpret_cast<float4 *>(sw)[q] = b;
        reinterpret_cast<float4 *>(sv)[q] = c;
    }
    fence_async_smem();
    __syncthreads();
    if (threadIdx.x == 0) {
        bulk_store(w + base, sw, bytes);
        bulk_store(v + base, sv, bytes);
        bulk_commit();
        bulk_wait_read0();
    }
}

// Persistent, 2-stage ring: stage s holds g/w/v of one item (48 KB).
__global__ void __launch_bounds__(256) k_tma2(const float *__restrict__ g, float *__restrict__ w,
                                              float *__restrict__ v, float lr, float mu, int items) {
    extern __shared__ __align__(128) float sm[];
    __shared__ __align__(8) uint64_t bar[2];
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](int it, int s) {
        const int64_t base = (int64_t)it * TI;
        const uint32_t bytes = (uint32_t)(int64_t)((TI) < (N - base) ? (TI) : (N - base)) * 4;
        float *st = sm + s * 3 * TI;
        mbar_expect_tx(&bar[s], 3 * bytes);
        bulk_load(st, g + base, bytes, &bar[s]);
        bulk_load(st + TI, w + base, bytes, &bar[s]);
        bulk_load(st + 2 * TI, v + base, bytes, &bar[s]);
    };
    int it = blockIdx.x;
    if (threadIdx.x == 0 && it < items) issue(it, 0);
    uint32_t phase[2] = {0, 0};
    for (int k = 0; it < items; ++k, it += gridDim.x) {
        const int s = k & 1;
        const int nxt = it + gridDim.x;
        if (threadIdx.x == 0 && nxt < items) {
            bulk_wait_read0();                 // stage s^1's previous stores have read smem
            issue(nxt, s ^ 1);
        }
        mbar_wait(&bar[s], phase[s]);
        phase[s] ^= 1;
        const int64_t base = (int64_t)it * TI;
        const uint32_t bytes = (uint32_t)(int64_t)((TI) < (N - base) ? (TI) : (N - base)) * 4;
        float *st = sm + s * 3 * TI;
        const int nv = bytes / 16;
        for (int q = threadIdx.x; q < nv; q += 256) {
            float4 a = reinterpret_cast<float4 *>(st)[q], b = reinterpret_cast<float4 *>(st + TI)[q],
                   c = reinterpret_cast<float4 *>(st + 2 * TI)[q];
            upd4(a, lr, mu, b, c);
            reinterpret_cast<float4 *>(st + TI)[q] = b;
            reinterpret_cast<float4 *>(st + 2 * TI)[q] = c;
        }
        fence_async_smem();
        __syncthreads();
        if (threadIdx.x == 0) {
            bulk_store(w + base, st + TI, bytes);
            bulk_store(v + base, st + 2 * TI, bytes);
            bulk_commit();
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) bulk_wait_read0();
}

int main() {
    float *g, *w, *v, *w0, *v0;
    CK(cudaMalloc(&g, N * 4)); CK(cudaMalloc(&w, N * 4)); CK(cudaMalloc(&v, N * 4));
    CK(cudaMalloc(&w0, N * 4)); CK(cudaMalloc(&v0, N * 4));
    std::vector<float> h(N);
    for (int64_t i = 0; i < N; ++i) h[i] = (float)((i * 2654435761u) % 1000) * 1e-4f - 0.05f;
    CK(cudaMemcpy(g, h.data(), N * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(w, h.data(), N * 4, cudaMemcpyHostToDevice));
    CK(cudaMemset(v, 0, N * 4));
    int nsm = 0;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
    const int items4k = (int)((N + 4095) / 4096);
    CK(cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * TB));
    CK(cudaFuncSetAttribute(k_tma2, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * TB));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    // reference result for correctness: variant A one step from a saved state
    CK(cudaMemcpy(w0, w, N * 4, cudaMemcpyDeviceToDevice));
    CK(cudaMemcpy(v0, v, N * 4, cudaMemcpyDeviceToDevice));
    std::vector<float> ref_w(N), got(N);
    k_item<4096, 256, true><<<items4k, 256>>>(g, w, v, 0.1f, 0.9f);
    CK(cudaMemcpy(ref_w.data(), w, N * 4, cudaMemcpyDeviceToHost));

    struct V { const char *name; int grid; };
    auto launch = [&](int which) {
        switch (which) {
            case 0: k_item<4096, 256, true><<<items4k, 256>>>(g, w, v, 0.1f, 0.9f); break;
            case 1: k_item<4096, 256, false><<<items4k, 256>>>(g, w, v, 0.1f, 0.9f); break;
            case 2: k_item<2048, 256, true><<<(int)((N + 2047) / 2048), 256>>>(g, w, v, 0.1f, 0.9f); break;
            case 3: k_item<8192, 512, true><<<(int)((N + 8191) / 8192), 512>>>(g, w, v, 0.1f, 0.9f); break;
            case 4: k_persist<<<nsm * 4, 256>>>(g, w, v, 0.1f, 0.9f, items4k); break;
            case 5: k_tma<<<items4k, 256, 3 * TB>>>(g, w, v, 0.1f, 0.9f); break;
            case 6: k_tma2<<<nsm * 2, 256, 6 * TB>>>(g, w, v, 0.1f, 0.9f, items4k); break;
            case 7: k_hint<true><<<items4k, 256>>>(g, w, v, 0.1f, 0.9f); break;
            case 8: k_hint<false><<<items4k, 256>>>(g, w, v, 0.1f, 0.9f); break;
            case 9: k_item<8192, 256, true><<<(int)((N + 8191) / 8192), 256>>>(g, w, v, 0.1f, 0.9f); break;
        }
    };
    const char *names[] = {"A item4096 .cs", "B item4096 default-cache", "C item2048 .cs",
                           "D item8192 512thr", "E persistent 4/SM", "F TMA bulk 1 item/CTA",
                           "G TMA bulk persistent 2-stage", "H item4096 .cs + L2::256B prefetch",
                           "I item4096 L2::256B prefetch", "J item8192 256thr (8 float4/thread/array)"};
    for (int which = 0; which < 10; ++which) {
        // correctness: one step from the saved state must equal variant A's
        CK(cudaMemcpy(w, w0, N * 4, cudaMemcpyDeviceToDevice));
        CK(cudaMemcpy(v, v0, N * 4, cudaMemcpyDeviceToDevice));
        launch(which);
        CK(cudaGetLastError());
        CK(cudaMemcpy(got.data(), w, N * 4, cudaMemcpyDeviceToHost));
        int64_t bad = 0;
        for (int64_t i = 0; i < N; ++i) bad += got[i] != ref_w[i];
        for (int r = 0; r < 20; ++r) launch(which);
        CK(cudaDeviceSynchronize());
        const int iters = 200;
        cudaEventRecord(e0);
        for (int r = 0; r < iters; ++r) launch(which);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double us = ms * 1e3 / iters;
        printf("{\"variant\": \"%s\", \"us\": %.2f, \"gbs\": %.1f, \"mismatch\": %lld}\n", names[which], us,
               20.0 * N / (us * 1e-6) / 1e9, (long long)bad);
    }
    return 0;
}
