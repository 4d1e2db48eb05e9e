// pcie_probe.cu -- design probe for the host-buffer (e2e) step: how fast can
// one B200 move the step's 102 MB of gradients in and 102 MB of parameters
// out over PCIe, by copy engines vs by SM loads/stores on mapped pinned host
// memory (zero-copy), alone and concurrently?  Prints one JSON line per case.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/pcie_probe scripts/pcie_probe.cu -lcuda
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda.h>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
    std::printf("{\"error\": \"%s at %d\"}\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

// 16-B vector copy, grid-stride, `u` vectors per thread per iteration in flight
template <int U>
__global__ void k_copy(const uint4 *__restrict__ src, uint4 *__restrict__ dst, int64_t n) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x * U;
    for (int64_t base = (static_cast<int64_t>(blockIdx.x) * blockDim.x) * U + threadIdx.x; base < n;
         base += stride) {
        uint4 x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t i = base + static_cast<int64_t>(u) * blockDim.x;
            if (i < n) x[u] = src[i];
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t i = base + static_cast<int64_t>(u) * blockDim.x;
            if (i < n) dst[i] = x[u];
        }
    }
}

// The fused zero-copy update shape: read g (host), w, v (device); write w, v
// (device) and w (host).  Arithmetic is momentum SGD, as in the library.
__global__ void k_zc_update(const float4 *__restrict__ hg, float4 *__restrict__ w,
                            float4 *__restrict__ v, float4 *__restrict__ hw, int64_t n, float lr,
                            float mu) {
    constexpr int U = 4;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x * U;
    for (int64_t base = (static_cast<int64_t>(blockIdx.x) * blockDim.x) * U + threadIdx.x; base < n;
         base += stride) {
        float4 g[U], a[U], b[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t i = base + static_cast<int64_t>(u) * blockDim.x;
            if (i < n) { g[u] = hg[i]; a[u] = w[i]; b[u] = v[i]; }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t i = base + static_cast<int64_t>(u) * blockDim.x;
            if (i < n) {
                b[u].x = __fmaf_rn(mu, b[u].x, g[u].x); a[u].x = __fmaf_rn(-lr, b[u].x, a[u].x);
                b[u].y = __fmaf_rn(mu, b[u].y, g[u].y); a[u].y = __fmaf_rn(-lr, b[u].y, a[u].y);
                b[u].z = __fmaf_rn(mu, b[u].z, g[u].z); a[u].z = __fmaf_rn(-lr, b[u].z, a[u].z);
                b[u].w = __fmaf_rn(mu, b[u].w, g[u].w); a[u].w = __fmaf_rn(-lr, b[u].w, a[u].w);
                w[i] = a[u]; v[i] = b[u]; hw[i] = a[u];
            }
        }
    }
}

// Flag-driven pipeline: the copy engine's H2D of piece p is followed on its
// stream by cuStreamWriteValue32(in_flag[p] = seq); one persistent kernel
// waits on in_flag[p], processes piece p, and the last CTA to finish it
// publishes out_flag[p] = seq, which cuStreamWaitValue32 on the D2H stream
// waits for before copying piece p back.  No event round trips per piece.
__global__ void k_flag_pipe(const uint4 *__restrict__ src, uint4 *__restrict__ dst, int64_t nv,
                            int pieces, const unsigned *in_flag, unsigned *out_flag,
                            unsigned *counters, unsigned seq) {
    for (int p = 0; p < pieces; ++p) {
        const int64_t v0 = nv * p / pieces, v1 = nv * (p + 1) / pieces;
        if (threadIdx.x == 0) {
            unsigned f;
            do {
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(f) : "l"(in_flag + p) : "memory");
            } while ((int)(f - seq) < 0);
        }
        __syncthreads();
        for (int64_t i = v0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < v1;
             i += (int64_t)gridDim.x * blockDim.x)
            dst[i] = src[i];
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            const unsigned old = atomicAdd(counters + p, 1u);
            if (old + 1 == seq * gridDim.x)
                asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(out_flag + p), "r"(seq) : "memory");
        }
    }
}

struct Timer {
    cudaEvent_t a, b;
    Timer() { cudaEventCreate(&a); cudaEventCreate(&b); }
    void start(cudaStream_t s) { cudaEventRecord(a, s); }
    float stop(cudaStream_t s) { cudaEventRecord(b, s); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); return ms; }
};

int main() {
    const int64_t L = 25557056;            // ResNet-50 padded layout, fp32
    const size_t bytes = static_cast<size_t>(L) * 4;
    const int64_t nv = L / 4;
    int nsm = 0;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
    float *hg, *hw, *dg, *dw, *dv, *dx;
    CK(cudaHostAlloc(&hg, bytes, cudaHostAllocMapped));
    CK(cudaHostAlloc(&hw, bytes, cudaHostAllocMapped));
    CK(cudaMalloc(&dg, bytes)); CK(cudaMalloc(&dw, bytes)); CK(cudaMalloc(&dv, bytes)); CK(cudaMalloc(&dx, bytes));
    for (int64_t i = 0; i < L; ++i) { hg[i] = 1e-3f * (i % 97); hw[i] = 0.f; }
    CK(cudaMemset(dw, 0, bytes)); CK(cudaMemset(dv, 0, bytes));
    cudaStream_t s0, s1;
    CK(cudaStreamCreateWithFlags(&s0, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
    Timer t;
    const int reps = 5;
    auto report = [&](const char *name, float ms, double moved) {
        std::printf("{\"case\": \"%s\", \"ms\": %.4f, \"gbs\": %.2f}\n", name, ms, moved / (ms * 1e-3) / 1e9);
    };
    auto run = [&](const char *name, double moved, auto fn) {
        fn(); CK(cudaDeviceSynchronize());
        t.start(s0);
        for (int r = 0; r < reps; ++r) fn();
        // join s1 into s0
        cudaEvent_t j; cudaEventCreateWithFlags(&j, cudaEventDisableTiming);
        cudaEventRecord(j, s1); cudaStreamWaitEvent(s0, j, 0);
        float ms = t.stop(s0) / reps;
        cudaEventDestroy(j);
        report(name, ms, moved);
        return 0;
    };
    cudaEvent_t fork; cudaEventCreateWithFlags(&fork, cudaEventDisableTiming);
    auto forked = [&]() { cudaEventRecord(fork, s0); cudaStreamWaitEvent(s1, fork, 0); };
    auto join = [&]() { cudaEventRecord(fork, s1); cudaStreamWaitEvent(s0, fork, 0); };

    run("ce_h2d", bytes, [&] { cudaMemcpyAsync(dg, hg, bytes, cudaMemcpyHostToDevice, s0); });
    run("ce_d2h", bytes, [&] { cudaMemcpyAsync(hw, dw, bytes, cudaMemcpyDeviceToHost, s0); });
    run("ce_both_concurrent", 2.0 * bytes, [&] {
        forked();
        cudaMemcpyAsync(dg, hg, bytes, cudaMemcpyHostToDevice, s0);
        cudaMemcpyAsync(hw, dw, bytes, cudaMemcpyDeviceToHost, s1);
        join();
    });
    for (int mult : {1, 2, 4}) {
        const int grid = mult * nsm;
        char nm[64];
        std::snprintf(nm, sizeof nm, "sm_read_host_%dxSM", mult);
        run(nm, bytes, [&] { k_copy<4><<<grid, 256, 0, s0>>>(reinterpret_cast<const uint4 *>(hg), reinterpret_cast<uint4 *>(dx), nv); });
        std::snprintf(nm, sizeof nm, "sm_write_host_%dxSM", mult);
        run(nm, bytes, [&] { k_copy<4><<<grid, 256, 0, s0>>>(reinterpret_cast<const uint4 *>(dw), reinterpret_cast<uint4 *>(hw), nv); });
        std::snprintf(nm, sizeof nm, "sm_both_concurrent_%dxSM", mult);
        run(nm, 2.0 * bytes, [&] {
            forked();
            k_copy<4><<<grid, 256, 0, s0>>>(reinterpret_cast<const uint4 *>(hg), reinterpret_cast<uint4 *>(dx), nv);
            k_copy<4><<<grid, 256, 0, s1>>>(reinterpret_cast<const uint4 *>(dw), reinterpret_cast<uint4 *>(hw), nv);
            join();
        });
        std::snprintf(nm, sizeof nm, "zc_fused_update_%dxSM", mult);
        run(nm, 2.0 * bytes, [&] {
            k_zc_update<<<grid, 256, 0, s0>>>(reinterpret_cast<const float4 *>(hg), reinterpret_cast<float4 *>(dw),
                                              reinterpret_cast<float4 *>(dv), reinterpret_cast<float4 *>(hw), nv, 0.1f, 0.9f);
        });
    }
    run("ce_h2d_plus_sm_write", 2.0 * bytes, [&] {
        forked();
        cudaMemcpyAsync(dg, hg, bytes, cudaMemcpyHostToDevice, s0);
        k_copy<4><<<2 * nsm, 256, 0, s1>>>(reinterpret_cast<const uint4 *>(dw), reinterpret_cast<uint4 *>(hw), nv);
        join();
    });
    run("sm_read_plus_ce_d2h", 2.0 * bytes, [&] {
        forked();
        k_copy<4><<<2 * nsm, 256, 0, s0>>>(reinterpret_cast<const uint4 *>(hg), reinterpret_cast<uint4 *>(dx), nv);
        cudaMemcpyAsync(hw, dw, bytes, cudaMemcpyDeviceToHost, s1);
        join();
    });
    // The library's N = 1 e2e pipeline shape: H2D(p) on s1 -> update(p) on s0
    // -> D2H(p) on s2; dependency events without timing, total step time.
    cudaStream_t s2;
    CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
    const std::vector<std::vector<int>> plans = {
        {1}, {1, 1}, {1, 1, 1}, {1, 1, 1, 1}, {1, 1, 1, 1, 1, 1}, {1, 1, 1, 1, 1, 1, 1, 1},
        {1, 2, 4, 8, 8, 8, 8, 8, 8, 4, 2, 1}, {1, 4, 16, 16, 16, 4, 1}, {1, 8, 8, 8, 8, 1},
        {1, 16, 16, 1}, {1, 30, 1}, {1, 3, 12, 12, 3, 1}, {2, 16, 16, 2}};
    for (const auto &wts : plans) {
        const int np = static_cast<int>(wts.size());
        std::vector<cudaEvent_t> ein(np), eup(np);
        for (int p = 0; p < np; ++p) {
            cudaEventCreateWithFlags(&ein[p], cudaEventDisableTiming);
            cudaEventCreateWithFlags(&eup[p], cudaEventDisableTiming);
        }
        cudaEvent_t ent, done;
        cudaEventCreateWithFlags(&ent, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&done, cudaEventDisableTiming);
        int tot = 0;
        for (int w : wts) tot += w;
        auto step = [&]() {
            cudaEventRecord(ent, s0);
            cudaStreamWaitEvent(s1, ent, 0);
            cudaStreamWaitEvent(s2, ent, 0);
            int acc = 0;
            for (int p = 0; p < np; ++p) {
                const int64_t v0 = nv * acc / tot;
                acc += wts[p];
                const int64_t v1 = nv * acc / tot;
                cudaMemcpyAsync(dg + 4 * v0, hg + 4 * v0, (v1 - v0) * 16, cudaMemcpyHostToDevice, s1);
                cudaEventRecord(ein[p], s1);
                cudaStreamWaitEvent(s0, ein[p], 0);
                k_copy<4><<<2 * nsm, 256, 0, s0>>>(reinterpret_cast<const uint4 *>(dg + 4 * v0),
                                                   reinterpret_cast<uint4 *>(dw + 4 * v0), v1 - v0);
                cudaEventRecord(eup[p], s0);
                cudaStreamWaitEvent(s2, eup[p], 0);
                cudaMemcpyAsync(hw + 4 * v0, dw + 4 * v0, (v1 - v0) * 16, cudaMemcpyDeviceToHost, s2);
            }
            cudaEventRecord(done, s2);
            cudaStreamWaitEvent(s0, done, 0);
        };
        step();
        CK(cudaDeviceSynchronize());
        t.start(s0);
        for (int r = 0; r < reps; ++r) step();
        const float ms = t.stop(s0) / reps;
        std::printf("{\"case\": \"pipeline\", \"weights\": [");
        for (int p = 0; p < np; ++p) std::printf("%s%d", p ? ", " : "", wts[p]);
        std::printf("], \"ms\": %.4f}\n", ms);
    }
    // flag-driven pipeline (stream memory operations), P pieces
    {
        unsigned *flags;
        const int maxp = 128;
        CK(cudaMalloc(&flags, 3 * maxp * sizeof(unsigned)));
        CK(cudaMemset(flags, 0, 3 * maxp * sizeof(unsigned)));
        unsigned *in_flag = flags, *out_flag = flags + maxp, *counters = flags + 2 * maxp;
        unsigned seq = 0;
        for (int P : {8, 16, 32, 64, 128}) {
            CK(cudaMemset(flags, 0, 3 * maxp * sizeof(unsigned)));
            seq = 0;
            auto step = [&]() {
                ++seq;
                cudaEventRecord(fork, s0);
                cudaStreamWaitEvent(s1, fork, 0);
                cudaStreamWaitEvent(s2, fork, 0);
                k_flag_pipe<<<2 * nsm, 256, 0, s0>>>(reinterpret_cast<const uint4 *>(dg), reinterpret_cast<uint4 *>(dw),
                                                     nv, P, in_flag, out_flag, counters, seq);
                for (int p = 0; p < P; ++p) {
                    const int64_t v0 = nv * p / P, v1 = nv * (p + 1) / P;
                    cudaMemcpyAsync(dg + 4 * v0, hg + 4 * v0, (v1 - v0) * 16, cudaMemcpyHostToDevice, s1);
                    cuStreamWriteValue32(s1, reinterpret_cast<CUdeviceptr>(in_flag + p), seq, 0);
                    cuStreamWaitValue32(s2, reinterpret_cast<CUdeviceptr>(out_flag + p), seq, CU_STREAM_WAIT_VALUE_GEQ);
                    cudaMemcpyAsync(hw + 4 * v0, dw + 4 * v0, (v1 - v0) * 16, cudaMemcpyDeviceToHost, s2);
                }
                cudaEvent_t j1, j2;
                cudaEventCreateWithFlags(&j1, cudaEventDisableTiming);
                cudaEventCreateWithFlags(&j2, cudaEventDisableTiming);
                cudaEventRecord(j1, s1); cudaEventRecord(j2, s2);
                cudaStreamWaitEvent(s0, j1, 0); cudaStreamWaitEvent(s0, j2, 0);
                cudaEventDestroy(j1); cudaEventDestroy(j2);
            };
            step();
            CK(cudaDeviceSynchronize());
            t.start(s0);
            for (int r = 0; r < reps; ++r) step();
            const float ms = t.stop(s0) / reps;
            CK(cudaGetLastError());
            std::printf("{\"case\": \"flag_pipeline\", \"pieces\": %d, \"ms\": %.4f}\n", P, ms);
        }
    }
    CK(cudaDeviceSynchronize());
    return 0;
}
