// cmn_core.cpp -- communicator state of the host runtime: errors, the packed
// layout, work-item tables, library-owned communication regions (CUDA IPC
// peer mapping, double-buffered by call parity), validation, grid sizes.
#include "cmn_comm.h"

#include <dlfcn.h>

#include <cstdio>
#include <cstring>

namespace cmn::rt {

thread_local std::string g_last_error;

cmn_status fail(cmn_status st, const std::string &msg) {
    g_last_error = msg;
    return st;
}

cmn_status cuda_fail(cudaError_t e, const char *what) {
    return fail(CMN_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

uint64_t fnv1a(uint64_t h, const void *data, size_t n) {
    const unsigned char *p = static_cast<const unsigned char *>(data);
    for (size_t i = 0; i < n; ++i) {
        h ^= p[i];
        h *= 1099511628211ull;
    }
    return h;
}

int64_t align_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

size_t env_size(const char *name, size_t dflt) {
    const char *v = std::getenv(name);
    if (!v || !*v) return dflt;
    return static_cast<size_t>(std::strtoull(v, nullptr, 10));
}

NcclApi g_nccl;

bool NcclApi::load() {
    if (h) return true;
    const char *cands[] = {std::getenv("CMN_NCCL_LIB"), "libnccl.so.2", "libnccl.so"};
    for (const char *c : cands) {
        if (!c) continue;
        h = dlopen(c, RTLD_NOW | RTLD_GLOBAL);
        if (h) break;
    }
    if (!h) return false;
    GetUniqueId = reinterpret_cast<int (*)(NcclUniqueId *)>(dlsym(h, "ncclGetUniqueId"));
    CommInitRank = reinterpret_cast<int (*)(void **, int, NcclUniqueId, int)>(
        dlsym(h, "ncclCommInitRank"));
    AllReduce = reinterpret_cast<int (*)(const void *, void *, size_t, int, int, void *,
                                         cudaStream_t)>(dlsym(h, "ncclAllReduce"));
    CommDestroy = reinterpret_cast<int (*)(void *)>(dlsym(h, "ncclCommDestroy"));
    GetErrorString = reinterpret_cast<const char *(*)(int)>(dlsym(h, "ncclGetErrorString"));
    return GetUniqueId && CommInitRank && AllReduce && CommDestroy;
}

cmn_status check_async_error(cmn_comm *c) {
    if (!c->h_err) return CMN_OK;
    const int e = *reinterpret_cast<volatile int *>(c->h_err);
    if (e == 1) return fail(CMN_ERR_TIMEOUT, "device spin-wait on a peer timed out");
    if (e == 2) return fail(CMN_ERR_MISMATCH, "peer issued a different collective (dtype/algo/kind/range)");
    if (e == 3)
        return fail(CMN_ERR_TIMEOUT, "a peer rank's communicator failed earlier (timeout or call "
                                     "mismatch there); this rank stopped waiting for it");
    return CMN_OK;
}

cmn_status launched(cmn_comm *c, cudaError_t e, const char *what) {
    if (e != cudaSuccess) return cuda_fail(e, what);
    ++c->launches;
    return CMN_OK;
}

void free_regions(cmn_comm *c) {
    for (int r = 0; r < kMaxWorld; ++r) {
        RankBufs &b = c->rb[r];
        if (b.base) {
            if (b.mapped)
                cudaIpcCloseMemHandle(b.base);
            else
                cudaFree(b.base);
        }
        b = RankBufs{};
    }
}

void free_registration(cmn_comm *c) {
    nvls_teardown(c->nvls);
    free_regions(c);
    cudaFree(c->d_td);
    cudaFree(c->d_items);
    cudaFree(c->d_sitems);
    c->d_sitems = nullptr;
    cudaFree(c->d_mom);
    cudaFree(c->d_adam);
    cudaFree(c->d_staging);
    cudaFree(c->d_pstage);
    c->d_pstage = nullptr;
    c->d_td = nullptr;
    c->d_items = nullptr;
    c->d_mom = c->d_adam = c->d_staging = nullptr;
    c->T = 0;
    c->L = 0;
    c->fresh = false;
    c->buckets.clear();
    c->bucket_fresh.clear();
    c->bucket_res.clear();
}

// Elements per region buffer: L plus slack so that a fused-push inbox of N
// slots of max-chunk length (N * align64(ceil(L/N)) <= L + 64 N) fits one
// buffer at any payload dtype.
int64_t buf_elems(int64_t L) { return L + static_cast<int64_t>(kAlign) * kMaxWorld; }

void carve(RankBufs &b, char *base, int64_t L) {
    const size_t buf = static_cast<size_t>(buf_elems(L)) * 4;
    b.base = base;
    b.packed[0] = base;
    b.packed[1] = base + buf;
    b.reduced[0] = base + 2 * buf;
    b.reduced[1] = base + 3 * buf;
    b.flags = reinterpret_cast<uint32_t *>(base + 4 * buf);
    b.epoch = b.flags + static_cast<size_t>(kBarrierSlots) * kMaxBarrierBlocks * kMaxWorld;
}

size_t flags_bytes() {   // signal pad + per-CTA epoch counters
    return (static_cast<size_t>(kBarrierSlots) * kMaxBarrierBlocks * kMaxWorld + kMaxBarrierBlocks) *
           sizeof(uint32_t);
}

cmn_status plan_layout_impl(int T, const int *ndims, const int64_t *dims,
                            std::vector<int64_t> &numel, std::vector<int64_t> &off,
                            uint64_t &hash) {
    if (T <= 0) return fail(CMN_ERR_INVALID_ARG, "n_tensors must be >= 1");
    if (!ndims) return fail(CMN_ERR_INVALID_ARG, "ndims is NULL");
    numel.assign(T, 0);
    off.assign(T + 1, 0);
    hash = 1469598103934665603ull;
    hash = fnv1a(hash, &T, sizeof T);
    int64_t pos = 0;
    for (int t = 0; t < T; ++t) {
        const int nd = ndims[t];
        if (nd < 0 || nd > 8) return fail(CMN_ERR_INVALID_ARG, "ndims out of range [0, 8]");
        if (nd > 0 && !dims) return fail(CMN_ERR_INVALID_ARG, "dims is NULL");
        int64_t n = 1;
        for (int d = 0; d < nd; ++d) {
            const int64_t e = dims[pos + d];
            if (e < 0) return fail(CMN_ERR_INVALID_ARG, "negative dimension");
            n *= e;
        }
        hash = fnv1a(hash, &nd, sizeof nd);
        if (nd > 0) hash = fnv1a(hash, dims + pos, sizeof(int64_t) * nd);
        pos += nd;
        numel[t] = n;
        off[t + 1] = align_up(off[t] + n, kAlign);
    }
    return CMN_OK;
}

// Allgather `bytes` from every rank; returns false if the callback failed.
bool allgather(cmn_comm *c, const void *send, void *recv, size_t bytes) {
    if (c->world == 1) {
        std::memcpy(recv, send, bytes);
        return true;
    }
    return c->ag(send, recv, bytes, c->user) == 0;
}

struct BootstrapMsg {
    uint64_t hash;
    uint64_t region_bytes;
    cudaIpcMemHandle_t handle;
};

cmn_status alloc_regions(cmn_comm *c) {
    c->region_bytes = static_cast<size_t>(buf_elems(c->L)) * 4 * 4 + flags_bytes();
    const int own = c->simulated ? c->world : 1;
    for (int i = 0; i < own; ++i) {
        const int r = c->simulated ? i : c->rank;
        void *p = nullptr;
        cudaError_t e = cudaMalloc(&p, c->region_bytes);
        if (e != cudaSuccess) return fail(CMN_ERR_OOM, "cudaMalloc(comm region) failed");
        CMN_CUDA(cudaMemset(p, 0, c->region_bytes));
        carve(c->rb[r], static_cast<char *>(p), c->L);
    }
    return CMN_OK;
}

cmn_status exchange_and_map(cmn_comm *c) {
    BootstrapMsg mine{};
    mine.hash = c->hash;
    mine.region_bytes = c->region_bytes;
    CMN_CUDA(cudaIpcGetMemHandle(&mine.handle, c->rb[c->rank].base));
    std::vector<BootstrapMsg> all(c->world);
    if (!allgather(c, &mine, all.data(), sizeof(BootstrapMsg)))
        return fail(CMN_ERR_BOOTSTRAP, "allgather callback failed");
    for (int r = 0; r < c->world; ++r)
        if (all[r].hash != c->hash || all[r].region_bytes != c->region_bytes)
            return fail(CMN_ERR_MISMATCH, "ranks registered different model structures");
    for (int r = 0; r < c->world; ++r) {
        if (r == c->rank) continue;
        void *p = nullptr;
        CMN_CUDA(cudaIpcOpenMemHandle(&p, all[r].handle, cudaIpcMemLazyEnablePeerAccess));
        carve(c->rb[r], static_cast<char *>(p), c->L);
        c->rb[r].mapped = true;
    }
    return CMN_OK;
}

int ar_blocks_for(const cmn_comm *c) {
    if (c->ar_blocks > 0) return c->ar_blocks;
    // Real ranks: one CTA per SM is ~19 MB of 16-B NVLink loads in flight at
    // N = 8 (far above the ~1 MB bandwidth-delay product) and leaves room
    // for the pipelined packs/updates.  Simulated ranks read local HBM:
    // two CTAs per SM.
    const size_t env = env_size("CMN_CTAS", 0);
    int b = env ? static_cast<int>(env) : (c->simulated ? 2 : 1) * c->nsm;
    if (b > kMaxBarrierBlocks) b = kMaxBarrierBlocks;
    if (b < 1) b = 1;
    return b;
}

// Grid of the barrier-gated HBM-bound kernels that grid-stride over work
// items (k_update_gather, k_gather_params): they stream 20 B/param through
// HBM, which one CTA per SM cannot saturate (scripts/update_variants.cu:
// persistent 4 CTAs/SM reach 6.0 TB/s), so default to 4 per SM -- the
// register-limited residency of the 256-thread item kernels -- capped by
// the signal pad, and never more CTAs than items.
int upd_blocks_for(const cmn_comm *c, int items) {
    int b = c->upd_blocks > 0 ? c->upd_blocks : 4 * c->nsm;
    if (b > kMaxBarrierBlocks) b = kMaxBarrierBlocks;
    if (b > items) b = items;
    if (b < 1) b = 1;
    return b;
}

bool grads_ok(const cmn_comm *c, const float *const *g, int count, std::string &why) {
    if (!g) {
        why = "grads table is NULL";
        return false;
    }
    for (int i = 0; i < count; ++i) {
        const int t = i % c->T;
        if (c->numel[t] == 0) continue;
        if (!g[i]) {
            why = "grad pointer " + std::to_string(i) + " is NULL";
            return false;
        }
        if (reinterpret_cast<uintptr_t>(g[i]) % 16 != 0) {
            why = "grad pointer " + std::to_string(i) + " is not 16-byte aligned";
            return false;
        }
    }
    return true;
}

GradTab make_tab(const float *const *g, int lo, int hi) {
    GradTab tab{};
    for (int t = lo; t < hi; ++t) tab.p[t - lo] = g[t];
    return tab;
}

Barrier make_barrier(cmn_comm *c, int dtype, BarrierKind kind, int64_t e0, int64_t e1) {
    Barrier b{};
    for (int r = 0; r < c->world; ++r) b.flags[r] = c->rb[r].flags;
    b.epoch = c->rb[c->rank].epoch;
    b.rank = c->rank;
    b.enabled = c->simulated ? 0 : 1;
    // call tag: dtype | kind | 4-bit hash of the packed range (cmn_internal.h)
    const int64_t range[2] = {e0, e1};
    const uint32_t h = static_cast<uint32_t>(fnv1a(0xcbf29ce484222325ull, range, sizeof(range)));
    b.tag = (static_cast<uint32_t>(dtype) & 1u) | ((static_cast<uint32_t>(kind) & 7u) << 1) |
            (((h ^ (h >> 4) ^ (h >> 8) ^ (h >> 12)) & 15u) << 4);
    b.timeout_ns = static_cast<uint64_t>(c->timeout_ms) * 1000000ull;
    b.err = c->d_err;
    b.derr = c->d_errdev;
    b.test_delay_ns = c->test_delay_ns;
    b.emul_g = 0;                  // set by the emulated launchers
    for (int r = 0; r < c->world; ++r) b.epochs[r] = c->rb[r].epoch;
    b.test_absent_rank = c->emulated ? c->test_absent_rank : -1;
    b.test_mismatch_rank = c->emulated ? c->test_mismatch_rank : -1;
    b.test_slow_rank = c->emulated ? c->test_slow_rank : -1;
    b.test_skip_mid = c->emulated ? c->test_skip_mid : 0;
    return b;
}

cmn_algo choose_algo(const cmn_comm *c, size_t bytes) {
    if (c->algo != CMN_ALGO_AUTO) return c->algo;
    if (c->world <= 2 || bytes <= c->oneshot_max) return CMN_ALGO_ONESHOT;
    return CMN_ALGO_TWOSHOT;
}

void chunk_plan(int64_t e0, int64_t e1, int world, int64_t *s, int64_t *e) {
    const int64_t n = e1 - e0;
    const int64_t cs = align_up((n + world - 1) / world, kAlign);
    for (int r = 0; r < world; ++r) {
        int64_t a = e0 + cs * r, b = e0 + cs * (r + 1);
        if (a > e1) a = e1;
        if (b > e1) b = e1;
        s[r] = a;
        e[r] = b;
    }
}

cmn_status require_registered(const cmn_comm *c) {
    if (!c) return fail(CMN_ERR_INVALID_ARG, "comm is NULL");
    if (c->T == 0) return fail(CMN_ERR_STATE, "cmn_register_params has not been called");
    return CMN_OK;
}

cmn_status require_dtype(int dtype) {
    if (dtype != CMN_FP32 && dtype != CMN_FP16) return fail(CMN_ERR_INVALID_ARG, "unknown dtype");
    return CMN_OK;
}

cmn_status set_device(const cmn_comm *c) {
    int cur = -1;
    if (cudaGetDevice(&cur) == cudaSuccess && cur == c->device) return CMN_OK;
    CMN_CUDA(cudaSetDevice(c->device));
    return CMN_OK;
}

cmn_status init_common(int rank, int world, int dev, bool sim, cmn_allgather_fn ag, void *user,
                       cmn_comm **out) {
    if (!out) return fail(CMN_ERR_INVALID_ARG, "out is NULL");
    *out = nullptr;
    if (world < 1 || world > kMaxWorld) return fail(CMN_ERR_INVALID_ARG, "world_size must be in [1, 8]");
    if (rank < 0 || rank >= world) return fail(CMN_ERR_INVALID_ARG, "rank out of range");
    if (!sim && world > 1 && !ag) return fail(CMN_ERR_INVALID_ARG, "allgather callback required");
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0)
        return fail(CMN_ERR_CUDA, "no CUDA device available (this library has no CPU fallback)");
    if (dev < 0 || dev >= ndev) return fail(CMN_ERR_INVALID_ARG, "cuda_device out of range");
    cudaDeviceProp prop{};
    CMN_CUDA(cudaGetDeviceProperties(&prop, dev));
    if (prop.major != 10)
        return fail(CMN_ERR_CUDA, "device is not sm_100 (kernels are built for sm_100a only)");
    CMN_CUDA(cudaSetDevice(dev));
    cmn_comm *c = new cmn_comm();
    c->rank = rank;
    c->world = world;
    c->device = dev;
    c->simulated = sim;
    c->ag = ag;
    c->user = user;
    c->nsm = prop.multiProcessorCount;
    c->oneshot_max = env_size("CMN_ONESHOT_MAX_BYTES", c->oneshot_max);
    c->pipe_pieces = static_cast<int>(env_size("CMN_PIECES", static_cast<size_t>(c->pipe_pieces)));
    c->test_delay_ns = static_cast<uint32_t>(env_size("CMN_TEST_ONESHOT_DELAY_US", 0) * 1000u);
    c->test_no_end_barrier = env_size("CMN_TEST_NO_END_BARRIER", 0) != 0;
    if (cudaHostAlloc(&c->h_err, sizeof(int), cudaHostAllocMapped) != cudaSuccess ||
        cudaHostGetDevicePointer(reinterpret_cast<void **>(&c->d_err), c->h_err, 0) != cudaSuccess) {
        delete c;
        return fail(CMN_ERR_CUDA, "cannot allocate the mapped error word");
    }
    *c->h_err = 0;
    if (cudaMalloc(&c->d_errdev, 256) != cudaSuccess || cudaMemset(c->d_errdev, 0, 256) != cudaSuccess) {
        cudaFreeHost(c->h_err);
        delete c;
        return fail(CMN_ERR_CUDA, "cannot allocate the device error word");
    }
    if (const char *a = std::getenv("CMN_ALGO")) {
        if (!std::strcmp(a, "oneshot")) c->algo = CMN_ALGO_ONESHOT;
        if (!std::strcmp(a, "twoshot")) c->algo = CMN_ALGO_TWOSHOT;
    }
    *out = c;
    return CMN_OK;
}

// Per-tensor host<->device copies (no coalescing across tensors: separate
// host allocations may happen to be adjacent, and one cudaMemcpy may not span
// two of them).
cmn_status copy_tensors(cmn_comm *c, const float *const *src, float *const *dst, int ta, int tb,
                        cudaMemcpyKind kind, cudaStream_t s) {
    for (int t = ta; t < tb; ++t) {
        if (c->numel[t] == 0) continue;
        CMN_CUDA(cudaMemcpyAsync(dst[t], src[t], static_cast<size_t>(c->numel[t]) * 4, kind, s));
    }
    return CMN_OK;
}

// Are the registered params views of ONE device allocation laid out like the
// packed layout (params[t] == params[0] + off[t])?  Then host<->device copies
// of parameter ranges may be single cudaMemcpys.  Verified with the driver's
// cuMemGetAddressRange so adjacency by accident is not mistaken for it.
bool params_are_flat(const cmn_comm *c) {
    if (c->T == 0 || !c->params[0]) return false;
    for (int t = 0; t < c->T; ++t)
        if (c->numel[t] > 0 && c->params[t] != c->params[0] + c->off[t]) return false;
    using Fn = int (*)(unsigned long long *, size_t *, unsigned long long);
    void *fp = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fp, cudaEnableDefault, &q) != cudaSuccess ||
        !fp)
        return false;
    unsigned long long base = 0;
    size_t size = 0;
    if (reinterpret_cast<Fn>(fp)(&base, &size, reinterpret_cast<unsigned long long>(c->params[0])) != 0)
        return false;
    const unsigned long long lo = reinterpret_cast<unsigned long long>(c->params[0]);
    int last = c->T - 1;
    while (last > 0 && c->numel[last] == 0) --last;
    const unsigned long long hi =
        reinterpret_cast<unsigned long long>(c->params[last] + c->numel[last]);
    return lo >= base && hi <= base + size;
}

cmn_status ensure_staging(cmn_comm *c) {
    if (c->d_staging) return CMN_OK;
    const int nsim = c->simulated ? c->world : 1;
    const size_t b = static_cast<size_t>(c->L > 0 ? c->L : 1) * 4 * nsim;
    if (cudaMalloc(&c->d_staging, b) != cudaSuccess) return fail(CMN_ERR_OOM, "staging alloc");
    return CMN_OK;
}

cmn_status ensure_pstage(cmn_comm *c, cudaStream_t s) {
    if (c->d_pstage) return CMN_OK;
    const size_t b = static_cast<size_t>(c->L > 0 ? c->L : 1) * 4;
    if (cudaMalloc(&c->d_pstage, b) != cudaSuccess) return fail(CMN_ERR_OOM, "param staging alloc");
    CMN_CUDA(cudaMemsetAsync(c->d_pstage, 0, b, s));   // pads stay +0 (only items are packed)
    return CMN_OK;
}

cmn_status ensure_side_streams(cmn_comm *c) {
    if (c->h2d) return CMN_OK;
    CMN_CUDA(cudaStreamCreateWithFlags(&c->h2d, cudaStreamNonBlocking));
    CMN_CUDA(cudaStreamCreateWithFlags(&c->d2h, cudaStreamNonBlocking));
    c->ev.resize(3 * kE2EMaxPieces + 2);
    for (auto &e : c->ev) CMN_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    return CMN_OK;
}

}  // namespace cmn::rt
