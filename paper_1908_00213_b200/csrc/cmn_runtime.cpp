// cmn_runtime.cpp -- host runtime behind include/cmn.h: validation, the
// packed layout, work-item tables, communication buffers (CUDA IPC peer
// mapping, double-buffered by call parity), algorithm choice, the NCCL
// comparison path, buckets for overlap, and error reporting.
//
// Paper passages: the communicator, the
// multi_node_optimizer wrapping, the all-reduce step
// (PAPER.md:449-454), fp16 payload, overlap
// (PAPER.md:788-792).  Readings R1-R16 are listed in DESIGN.md §3.
#include "../../include/cmn.h"

#include <dlfcn.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <iterator>
#include <string>
#include <utility>
#include <vector>

#include <cuda_runtime.h>

#include "cmn_internal.h"
#include "cmn_nvls.h"

using namespace cmn;

namespace {

thread_local std::string g_last_error;

cmn_status fail(cmn_status st, const std::string &msg) {
    g_last_error = msg;
    return st;
}

cmn_status cuda_fail(cudaError_t e, const char *what) {
    return fail(CMN_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

#define CMN_CUDA(call)                                          \
    do {                                                        \
        cudaError_t e_ = (call);                                \
        if (e_ != cudaSuccess) return cuda_fail(e_, #call);     \
    } while (0)

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

// ---------------------------------------------------------------- NCCL
// The comparison backend is loaded with dlopen so the library has no hard
// dependency on libnccl (only CMN_ALGO_NCCL needs it).
struct NcclUniqueId {   // layout of ncclUniqueId (NCCL_UNIQUE_ID_BYTES = 128), passed BY VALUE
    char internal[128];
};
struct NcclApi {
    void *h = nullptr;
    int (*GetUniqueId)(NcclUniqueId *) = nullptr;
    int (*CommInitRank)(void **, int, NcclUniqueId, int) = nullptr;
    int (*AllReduce)(const void *, void *, size_t, int, int, void *, cudaStream_t) = nullptr;
    int (*CommDestroy)(void *) = nullptr;
    const char *(*GetErrorString)(int) = nullptr;
    bool load() {
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
};
NcclApi g_nccl;
constexpr int kNcclFloat16 = 6, kNcclFloat32 = 7, kNcclSum = 0;
// Host-buffer (e2e) step at N = 1: piece weights of the H2D || update ||
// D2H pipeline, in units of L/62, ramping up from and down to L/62 so the
// fill (H2D of the first piece) and drain (D2H of the last) are short.
// Measured (profiles/r1_pcie_probe.jsonl, bench e2e): 2.5-2.6 ms for the
// R50 step whatever the plan (4/8/16 equal pieces, this ramp, or the
// parameter read-back done by the update kernel's own stores into mapped
// host memory) -- the copy engines' concurrent H2D + D2H inside a
// dependent pipeline, not the plan, is the limit.
constexpr int kE2EWeights[] = {1, 2, 4, 8, 8, 8, 8, 8, 8, 4, 2, 1};
constexpr int kE2EMaxPieces = 64;   // CMN_E2E_PIECES=n (equal pieces) is capped here

}  // namespace

// One rank's library-owned communication region:
//   [packed0 | packed1 | reduced0 | reduced1 | signal pad]
struct RankBufs {
    char *base = nullptr;
    void *packed[2] = {nullptr, nullptr};
    void *reduced[2] = {nullptr, nullptr};
    uint32_t *flags = nullptr;
    uint32_t *epoch = nullptr;   // per-CTA call counters (read by own kernels only)
    bool mapped = false;  // IPC-opened peer region
};

// Where an all-reduce left its result: buffer parity, payload dtype, and
// whether the "reduced" buffer is the packed one (N == 1 identity).
struct ArResult {
    int parity = 0;
    int dtype = 0;
    bool alias_packed = false;
    bool nvls = false;      // result lives in the NVLS buffer (unicast view)
};

struct cmn_comm {
    int rank = 0, world = 1, device = 0;
    bool simulated = false;
    cmn_allgather_fn ag = nullptr;
    void *user = nullptr;
    int nsm = 148;

    // registration
    int T = 0;
    std::vector<int64_t> numel, off;
    int64_t L = 0;
    uint64_t hash = 0;
    std::vector<float *> params;
    std::vector<TensorDesc> h_td;
    TensorDesc *d_td = nullptr;
    std::vector<Item> h_items;
    std::vector<int> item_begin;  // T + 1
    Item *d_items = nullptr;
    float *d_mom = nullptr;       // L floats, tensor t at off[t]
    float *d_adam = nullptr;      // 2 L floats (m then v), lazily
    float *d_staging = nullptr;   // host e2e staging, world_sim * L floats
    size_t region_bytes = 0;
    RankBufs rb[kMaxWorld];

    // state
    uint32_t seq = 0;
    bool fresh = false;           // reduced buffer holds an unconsumed result
    ArResult last;                    // of the last whole-model or bucket all-reduce
    cmn_algo algo = CMN_ALGO_AUTO;
    size_t oneshot_max = 1u << 20;
    uint32_t timeout_ms = 30000;
    int ar_blocks = 0;            // cmn_set_ctas: collective grid (0 = default)
    int upd_blocks = 0;           // cmn_set_ctas: barrier-gated update grid (0 = default)
    int *h_err = nullptr, *d_err = nullptr;
    uint64_t launches = 0;
    // cmn_set_kernel_timing: CUDA events around every launch of the step's
    // dominant kernels (all-reduce, fused all-gather+update, the N = 1
    // direct update) on the stream each runs on; pairs [0, ktimed) in use.
    bool ktiming = false;
    std::vector<cudaEvent_t> kev;
    size_t ktimed = 0;
    std::vector<std::pair<int, int>> buckets;   // [t_begin, t_end), reverse order
    std::vector<char> bucket_fresh;
    std::vector<ArResult> bucket_res;
    void *nccl = nullptr;
    bool params_flat = false;             // params are views of one packed-layout allocation
    cudaStream_t h2d = nullptr, d2h = nullptr;   // e2e copy streams (lazily)
    std::vector<cudaEvent_t> ev;
    // pipelined N > 1 step: pack(p+1) and update(p-1) on the caller's stream
    // overlap all-reduce(p) on a high-priority communication stream.
    int pipe_pieces = 4;
    int fused_update = 0;         // N > 1 cmn_step: RS + fused all-gather/update (1 pull, 2 push)
    Nvls nvls;                    // NEXT-3 multicast resources (CMN_ALGO_NVLS)
    // NEXT-4 sharded update: items clipped to every rank's two-shot chunk
    // (Item.reserved = owner), rank r's list is [sitem_begin[r], sitem_begin[r+1]).
    std::vector<int> sitem_begin;
    Item *d_sitems = nullptr;
    cudaStream_t sc = nullptr;
    std::vector<cudaEvent_t> pev;
};

namespace {

cmn_status check_async_error(cmn_comm *c) {
    if (!c->h_err) return CMN_OK;
    const int e = *reinterpret_cast<volatile int *>(c->h_err);
    if (e == 1) return fail(CMN_ERR_TIMEOUT, "device spin-wait on a peer timed out");
    if (e == 2) return fail(CMN_ERR_MISMATCH, "peer issued a different collective (dtype/algo)");
    return CMN_OK;
}

cmn_status launched(cmn_comm *c, cudaError_t e, const char *what) {
    if (e != cudaSuccess) return cuda_fail(e, what);
    ++c->launches;
    return CMN_OK;
}

// Run `f` (kernel launches on stream s) between two timing events when
// kernel timing is on and s is not being captured into a graph.
template <typename F>
cmn_status timed(cmn_comm *c, cudaStream_t s, F &&f) {
    bool on = c->ktiming;
    if (on) {
        cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
        on = cudaStreamIsCapturing(s, &cap) == cudaSuccess && cap == cudaStreamCaptureStatusNone;
    }
    if (on) {
        while (c->kev.size() < 2 * (c->ktimed + 1)) {
            cudaEvent_t e;
            CMN_CUDA(cudaEventCreate(&e));
            c->kev.push_back(e);
        }
        CMN_CUDA(cudaEventRecord(c->kev[2 * c->ktimed], s));
    }
    const cmn_status st = f();
    if (on && st == CMN_OK) {
        CMN_CUDA(cudaEventRecord(c->kev[2 * c->ktimed + 1], s));
        ++c->ktimed;
    }
    return st;
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

// Iterate tensor groups of at most kGradCap tensors inside [ta, tb).
template <typename F>
cmn_status for_groups(cmn_comm *c, int ta, int tb, F &&f) {
    for (int lo = ta; lo < tb; lo += kGradCap) {
        const int hi = lo + kGradCap < tb ? lo + kGradCap : tb;
        cmn_status st = f(lo, hi, c->item_begin[lo], c->item_begin[hi]);
        if (st != CMN_OK) return st;
    }
    return CMN_OK;
}

GradTab make_tab(const float *const *g, int lo, int hi) {
    GradTab tab{};
    for (int t = lo; t < hi; ++t) tab.p[t - lo] = g[t];
    return tab;
}

Barrier make_barrier(cmn_comm *c, int tag) {
    Barrier b{};
    for (int r = 0; r < c->world; ++r) b.flags[r] = c->rb[r].flags;
    b.epoch = c->rb[c->rank].epoch;
    b.rank = c->rank;
    b.enabled = c->simulated ? 0 : 1;
    b.tag = static_cast<uint32_t>(tag & 3);
    b.timeout_ns = static_cast<uint64_t>(c->timeout_ms) * 1000000ull;
    b.err = c->d_err;
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

// a1: pack every (simulated) rank's gradients of tensors [ta, tb) into its
// packed buffer of parity `par`.
cmn_status pack_phase(cmn_comm *c, int ta, int tb, const float *const *grads, int dtype, int par,
                      cudaStream_t s, void *dst_override = nullptr) {
    const int nsim = c->simulated ? c->world : 1;
    for (int i = 0; i < nsim; ++i) {
        const int r = c->simulated ? i : c->rank;
        const float *const *g = grads + static_cast<size_t>(i) * c->T;
        void *dst = dst_override ? dst_override : c->rb[r].packed[par];
        cmn_status st = for_groups(c, ta, tb, [&](int lo, int hi, int i0, int i1) {
            return launched(c,
                            launch_pack(make_tab(g, lo, hi), hi - lo, lo, c->d_td, c->d_items, i0, i1, dtype,
                                        dst, s),
                            "pack");
        });
        if (st != CMN_OK) return st;
    }
    return CMN_OK;
}

// a2 over the packed range of tensors [ta, tb) for the collective call with
// sequence number `seq` (its buffers have parity seq & 1).
cmn_status reduce_phase_launch(cmn_comm *c, int ta, int tb, int dtype, uint32_t seq, cmn_algo algo,
                               cudaStream_t s) {
    const int par = static_cast<int>(seq & 1u);
    const int64_t e0 = c->off[ta], e1 = c->off[tb];
    const size_t esz = dtype == 0 ? 4 : 2;
    const int nsim = c->simulated ? c->world : 1;
    // identity at N = 1 (fp16 rounding done by the pack) -- except through
    // NCCL / NVLS, whose single-rank all-reduce exercises their plumbing
    if (c->world == 1 && algo != CMN_ALGO_NCCL && algo != CMN_ALGO_NVLS) return CMN_OK;
    if (algo == CMN_ALGO_NVLS) {
        int64_t cs[kMaxWorld], ce[kMaxWorld];
        chunk_plan(e0, e1, c->world, cs, ce);
        const Barrier bar = make_barrier(c, dtype | 2);
        return launched(c,
                        launch_nvls_allreduce(c->nvls.packed_mc(), c->nvls.reduced_mc(),
                                              cs[c->rank], ce[c->rank], c->world, dtype, bar,
                                              ar_blocks_for(c), s),
                        "nvls_allreduce");
    }
    if (algo == CMN_ALGO_NCCL) {
        void *src = static_cast<char *>(c->rb[c->rank].packed[par]) + e0 * esz;
        void *dst = static_cast<char *>(c->rb[c->rank].reduced[par]) + e0 * esz;
        const int rc = g_nccl.AllReduce(src, dst, static_cast<size_t>(e1 - e0),
                                        dtype == 0 ? kNcclFloat32 : kNcclFloat16, kNcclSum,
                                        c->nccl, s);
        if (rc != 0)
            return fail(CMN_ERR_NCCL, std::string("ncclAllReduce: ") +
                                          (g_nccl.GetErrorString ? g_nccl.GetErrorString(rc) : "?"));
        return CMN_OK;
    }
    PeerBufs in{}, red{};
    for (int r = 0; r < c->world; ++r) {
        in.p[r] = c->rb[r].packed[par];
        red.p[r] = c->rb[r].reduced[par];
    }
    const int blocks = ar_blocks_for(c);
    const int tag = dtype | (algo == CMN_ALGO_TWOSHOT ? 2 : 0);
    const Barrier bar = make_barrier(c, tag);
    if (algo == CMN_ALGO_ONESHOT) {
        for (int i = 0; i < nsim; ++i) {
            const int r = c->simulated ? i : c->rank;
            cmn_status st = launched(c,
                                     launch_allreduce_oneshot(in, c->world, c->rb[r].reduced[par],
                                                              e0, e1, dtype, bar, blocks, s),
                                     "allreduce_oneshot");
            if (st != CMN_OK) return st;
        }
        return CMN_OK;
    }
    int64_t cs[kMaxWorld], ce[kMaxWorld];
    chunk_plan(e0, e1, c->world, cs, ce);
    if (c->simulated) {
        for (int phase = 1; phase <= 2; ++phase)
            for (int r = 0; r < c->world; ++r) {
                cmn_status st = launched(c,
                                         launch_allreduce_twoshot(in, red, c->world, r, cs, ce, dtype,
                                                                  phase, bar, blocks, s),
                                         "allreduce_twoshot");
                if (st != CMN_OK) return st;
            }
        return CMN_OK;
    }
    return launched(c,
                    launch_allreduce_twoshot(in, red, c->world, c->rank, cs, ce, dtype, 3, bar,
                                             blocks, s),
                    "allreduce_twoshot");
}

cmn_status reduce_phase(cmn_comm *c, int ta, int tb, int dtype, uint32_t seq, cmn_algo algo,
                        cudaStream_t s) {
    if (c->world == 1 && algo != CMN_ALGO_NCCL && algo != CMN_ALGO_NVLS) return CMN_OK;
    return timed(c, s, [&] { return reduce_phase_launch(c, ta, tb, dtype, seq, algo, s); });
}

// Validate and choose the algorithm for one collective over [ta, tb).
// CUDA-graph policy.  Barrier values come from device-resident per-CTA
// epochs, so replays never pass a barrier early.  What a graph does freeze is
// the host-chosen packed-buffer parity: a single collective per step needs
// consecutive calls to alternate buffers (a peer may still be reading the
// previous call's packed buffer when the next pack starts), which a replayed
// graph with one call cannot do.  Schedules whose buffer safety does not
// depend on alternation -- the pipelined step (P >= 2 pieces: a region's
// previous reader is >= 2 calls back) and the sharded step (every overwrite
// is behind a start barrier) -- pass graph_safe = true and may be captured;
// the single-call schedules refuse capture loudly instead of racing.
// (N = 1 and simulated communicators have no cross-process state.)
cmn_status begin_collective(cmn_comm *c, int ta, int tb, int dtype, cmn_algo &algo,
                            cudaStream_t s, bool graph_safe) {
    if (cmn_status st = check_async_error(c); st != CMN_OK) return st;
    if (!c->simulated && c->world > 1 && !graph_safe) {
        cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
        CMN_CUDA(cudaStreamIsCapturing(s, &cap));
        if (cap != cudaStreamCaptureStatusNone)
            return fail(CMN_ERR_UNSUPPORTED,
                        "this collective schedule cannot be captured into a CUDA graph "
                        "(use cmn_step with cmn_set_pipeline >= 2, or cmn_step_sharded)");
    }
    const size_t esz = dtype == 0 ? 4 : 2;
    algo = choose_algo(c, static_cast<size_t>(c->off[tb] - c->off[ta]) * esz);
    if (algo == CMN_ALGO_NVLS && !c->nvls.ready())
        return fail(CMN_ERR_STATE, "NVLS algorithm requested but no multicast resources "
                                   "(cmn_set_algo(CMN_ALGO_NVLS) after registration, on every rank)");
    if (algo == CMN_ALGO_NCCL && (c->simulated || !c->nccl))
        return fail(CMN_ERR_STATE, "NCCL algorithm requested but no NCCL communicator "
                                   "(cmn_set_algo(CMN_ALGO_NCCL) on every rank of a cmn_init comm)");
    return CMN_OK;
}

// a1 + a2 over the tensor range [ta, tb) (whole model or one bucket).
cmn_status allreduce_range(cmn_comm *c, int ta, int tb, const float *const *grads, int dtype,
                           cudaStream_t s) {
    cmn_algo algo = CMN_ALGO_AUTO;
    // NVLS is single-buffered behind start + end barriers: graph-safe.
    const bool nvls = c->algo == CMN_ALGO_NVLS;
    if (cmn_status st = begin_collective(c, ta, tb, dtype, algo, s, nvls); st != CMN_OK) return st;
    const uint32_t seq = ++c->seq;
    const int par = static_cast<int>(seq & 1u);
    if (cmn_status st = pack_phase(c, ta, tb, grads, dtype, par, s, nvls ? c->nvls.packed_uc() : nullptr);
        st != CMN_OK)
        return st;
    if (cmn_status st = reduce_phase(c, ta, tb, dtype, seq, algo, s); st != CMN_OK) return st;
    c->last = ArResult{par, dtype, c->world == 1 && algo != CMN_ALGO_NCCL && !nvls, nvls};
    return CMN_OK;
}

const void *reduced_ptr(const cmn_comm *c, const ArResult &res, int rank) {
    if (res.nvls) return c->nvls.reduced_uc();
    const int r = c->simulated ? rank : c->rank;
    return res.alias_packed ? c->rb[r].packed[res.parity] : c->rb[r].reduced[res.parity];
}

cmn_status update_range(cmn_comm *c, int ta, int tb, const ArResult &res, float lr, float mu,
                        cudaStream_t s) {
    const float inv_n = 1.0f / static_cast<float>(c->world);
    return for_groups(c, ta, tb, [&](int, int, int i0, int i1) {
        return launched(c,
                        launch_update_sgd(c->d_td, c->d_items, i0, i1, reduced_ptr(c, res, 0),
                                          res.dtype, inv_n, lr, mu, s),
                        "update_sgd");
    });
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
    if (cudaHostAlloc(&c->h_err, sizeof(int), cudaHostAllocMapped) != cudaSuccess ||
        cudaHostGetDevicePointer(reinterpret_cast<void **>(&c->d_err), c->h_err, 0) != cudaSuccess) {
        delete c;
        return fail(CMN_ERR_CUDA, "cannot allocate the mapped error word");
    }
    *c->h_err = 0;
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

cmn_status ensure_side_streams(cmn_comm *c) {
    if (c->h2d) return CMN_OK;
    CMN_CUDA(cudaStreamCreateWithFlags(&c->h2d, cudaStreamNonBlocking));
    CMN_CUDA(cudaStreamCreateWithFlags(&c->d2h, cudaStreamNonBlocking));
    c->ev.resize(3 * kE2EMaxPieces + 2);
    for (auto &e : c->ev) CMN_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    return CMN_OK;
}

// Item ranges [i0, i1) of the N = 1 host-buffer pipeline (item = 4096
// elements of one tensor, so a tensor may straddle pieces), sized by
// kE2EWeights -- or CMN_E2E_PIECES equal pieces (measurement).
std::vector<std::pair<int, int>> e2e_item_pieces(const cmn_comm *c) {
    const int I = c->item_begin[c->T];
    std::vector<int> wts(std::begin(kE2EWeights), std::end(kE2EWeights));
    if (const size_t n = env_size("CMN_E2E_PIECES", 0); n > 0)
        wts.assign(n < static_cast<size_t>(kE2EMaxPieces) ? n : kE2EMaxPieces, 1);
    int64_t total = 0;
    for (int w : wts) total += w;
    std::vector<std::pair<int, int>> out;
    int i = 0;
    int64_t acc = 0;
    for (size_t p = 0; p < wts.size() && i < I; ++p) {
        acc += wts[p];
        int j = i;
        if (p + 1 == wts.size()) {
            j = I;
        } else {
            const int64_t bound = c->L * acc / total;
            while (j < I && c->h_items[j].base < bound) ++j;
        }
        if (j > i) out.emplace_back(i, j);
        i = j;
    }
    return out;
}

// Tensor ranges of roughly equal bytes, forward order (at most `n`).
std::vector<std::pair<int, int>> equal_ranges(const cmn_comm *c, int n) {
    std::vector<std::pair<int, int>> out;
    const int64_t target = (c->L + n - 1) / n;
    int t = 0;
    while (t < c->T) {
        int u = t;
        int64_t acc = 0;
        while (u < c->T && (acc < target || static_cast<int>(out.size()) + 1 == n)) {
            acc += c->numel[u];
            ++u;
        }
        out.emplace_back(t, u);
        t = u;
    }
    return out;
}

cmn_status ensure_comm_stream(cmn_comm *c, size_t n_events) {
    if (!c->sc) {
        int lo = 0, hi = 0;
        CMN_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        CMN_CUDA(cudaStreamCreateWithPriority(&c->sc, cudaStreamNonBlocking, hi));
    }
    while (c->pev.size() < n_events) {
        cudaEvent_t e;
        CMN_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        c->pev.push_back(e);
    }
    return CMN_OK;
}

// Pipelined a1-a3 for N > 1: the model is cut into P contiguous pieces; each
// piece is one collective call.  Caller stream s: pack(0..P-1), then
// update(p) after all-reduce(p); communication stream: all-reduce(p) after
// pack(p).  HBM-bound packs/updates overlap the NVLink-bound all-reduces.
// Buffer reuse is safe for P >= 2: a piece's next pack (seq + P) is issued
// after update(P-1), i.e. after our all-reduce at seq + P - 1 passed its
// start barrier, so every peer finished all-reduce calls <= seq + P - 2.
// Host buffers of the e2e step (cmn_step_host_packed): packed layout, L
// floats per (simulated) rank for the gradients; parameters out or NULL.
struct HostIO {
    const float *grads = nullptr;
    float *params = nullptr;
};

// Device->host copy of the parameters of tensors [ta, tb) into the packed
// host layout: one copy when the params are one flat allocation (stopping
// at the last tensor's end), else one per tensor.
cmn_status d2h_params(cmn_comm *c, int ta, int tb, float *host_params, cudaStream_t s) {
    if (c->params_flat) {
        int last = c->T - 1;
        while (last > 0 && c->numel[last] == 0) --last;
        const int64_t flat_end = c->off[last] + c->numel[last];
        const int64_t e0 = c->off[ta], e1 = c->off[tb] < flat_end ? c->off[tb] : flat_end;
        if (e1 > e0)
            CMN_CUDA(cudaMemcpyAsync(host_params + e0, c->params[0] + e0, static_cast<size_t>(e1 - e0) * 4,
                                     cudaMemcpyDeviceToHost, s));
        return CMN_OK;
    }
    std::vector<float *> hp(c->T);
    for (int t = 0; t < c->T; ++t) hp[t] = host_params + c->off[t];
    std::vector<const float *> src(c->params.begin(), c->params.end());
    return copy_tensors(c, src.data(), hp.data(), ta, tb, cudaMemcpyDeviceToHost, s);
}

// With `io`, the e2e form: H2D(piece p) on a copy stream feeds pack(p), and
// D2H(piece p) on a second copy stream follows update(p), so PCIe in both
// directions overlaps the packs, NVLink all-reduces and updates of the
// other pieces (gradients land in the library's staging buffer, whose
// pointers `grads` are).
cmn_status step_pipelined(cmn_comm *c, const float *const *grads, int dtype, float lr, float mu,
                          cudaStream_t s, const HostIO *io = nullptr) {
    const auto pieces = equal_ranges(c, c->pipe_pieces);
    const size_t P = pieces.size();
    if (cmn_status st = ensure_comm_stream(c, 2 * P + 1); st != CMN_OK) return st;
    if (io)
        if (cmn_status st = ensure_side_streams(c); st != CMN_OK) return st;
    const int nsim = c->simulated ? c->world : 1;
    std::vector<cmn_algo> algo(P);
    for (size_t p = 0; p < P; ++p)
        if (cmn_status st = begin_collective(c, pieces[p].first, pieces[p].second, dtype, algo[p], s,
                                             P >= 2);
            st != CMN_OK)
            return st;
    cudaEvent_t entry = c->pev[2 * P];
    CMN_CUDA(cudaEventRecord(entry, s));
    CMN_CUDA(cudaStreamWaitEvent(c->sc, entry, 0));
    if (io) {
        CMN_CUDA(cudaStreamWaitEvent(c->h2d, entry, 0));
        CMN_CUDA(cudaStreamWaitEvent(c->d2h, entry, 0));
    }
    // NVLS: one multicast buffer pair; a piece's region is reused only after
    // its previous all-reduce passed its end barrier (same ordering argument
    // as above), so no parity alternation is needed.
    const bool nvls = c->algo == CMN_ALGO_NVLS;
    std::vector<ArResult> res(P);
    for (size_t p = 0; p < P; ++p) {
        const uint32_t seq = ++c->seq;
        const int par = static_cast<int>(seq & 1u);
        res[p] = ArResult{par, dtype, false, nvls};
        if (io) {
            const int64_t e0 = c->off[pieces[p].first], e1 = c->off[pieces[p].second];
            for (int i = 0; i < nsim; ++i) {
                const size_t base = static_cast<size_t>(i) * c->L;
                CMN_CUDA(cudaMemcpyAsync(c->d_staging + base + e0, io->grads + base + e0,
                                         static_cast<size_t>(e1 - e0) * 4, cudaMemcpyHostToDevice,
                                         c->h2d));
            }
            CMN_CUDA(cudaEventRecord(c->ev[2 + 3 * p], c->h2d));
            CMN_CUDA(cudaStreamWaitEvent(s, c->ev[2 + 3 * p], 0));
        }
        if (cmn_status st = pack_phase(c, pieces[p].first, pieces[p].second, grads, dtype, par, s,
                                       nvls ? c->nvls.packed_uc() : nullptr);
            st != CMN_OK)
            return st;
        CMN_CUDA(cudaEventRecord(c->pev[2 * p], s));
        CMN_CUDA(cudaStreamWaitEvent(c->sc, c->pev[2 * p], 0));
        if (cmn_status st = reduce_phase(c, pieces[p].first, pieces[p].second, dtype, seq, algo[p],
                                         c->sc);
            st != CMN_OK)
            return st;
        CMN_CUDA(cudaEventRecord(c->pev[2 * p + 1], c->sc));
    }
    for (size_t p = 0; p < P; ++p) {
        CMN_CUDA(cudaStreamWaitEvent(s, c->pev[2 * p + 1], 0));
        if (cmn_status st = update_range(c, pieces[p].first, pieces[p].second, res[p], lr, mu, s);
            st != CMN_OK)
            return st;
        if (io && io->params) {
            CMN_CUDA(cudaEventRecord(c->ev[3 + 3 * p], s));
            CMN_CUDA(cudaStreamWaitEvent(c->d2h, c->ev[3 + 3 * p], 0));
            if (cmn_status st = d2h_params(c, pieces[p].first, pieces[p].second, io->params, c->d2h);
                st != CMN_OK)
                return st;
        }
    }
    if (io) {
        CMN_CUDA(cudaEventRecord(c->ev[1], c->d2h));
        CMN_CUDA(cudaStreamWaitEvent(s, c->ev[1], 0));
    }
    c->last = res[P - 1];
    c->fresh = false;
    return CMN_OK;
}

// NEXT-4: reduce-scatter -> update own chunk -> all-gather parameters.
// Per rank: pack (HBM) -> RS over NVLink (start barrier, call s) -> momentum
// SGD on the own chunk only (1/N of the update traffic), publishing w' into
// the fp32 exchange buffer -> gather of the other chunks' w' (start barrier,
// call s+1: every peer's chunk update has completed).  Every element gets
// exactly the arithmetic of the replicated update, so w is bitwise equal;
// momentum is sharded (valid on the owner rank only).
cmn_status step_sharded(cmn_comm *c, const float *const *grads, int dtype, float lr, float mu,
                        cudaStream_t s) {
    cmn_algo algo = CMN_ALGO_AUTO;
    if (cmn_status st = begin_collective(c, 0, c->T, dtype, algo, s, true); st != CMN_OK) return st;
    const int nsim = c->simulated ? c->world : 1;
    const uint32_t seq1 = ++c->seq;
    const int par = static_cast<int>(seq1 & 1u);
    if (cmn_status st = pack_phase(c, 0, c->T, grads, dtype, par, s); st != CMN_OK) return st;
    PeerBufs in{}, red{}, exch{};
    for (int r = 0; r < c->world; ++r) {
        in.p[r] = c->rb[r].packed[par];
        red.p[r] = c->rb[r].reduced[0];
        exch.p[r] = c->rb[r].reduced[1];
    }
    int64_t cs[kMaxWorld], ce[kMaxWorld];
    chunk_plan(0, c->L, c->world, cs, ce);
    const int blocks = ar_blocks_for(c);
    const Barrier bar = make_barrier(c, dtype | 2);
    for (int i = 0; i < nsim; ++i) {
        const int r = c->simulated ? i : c->rank;
        cmn_status st = launched(c,
                                 launch_allreduce_twoshot(in, red, c->world, r, cs, ce, dtype, 1, bar,
                                                          blocks, s),
                                 "reduce_scatter");
        if (st != CMN_OK) return st;
    }
    const float inv_n = 1.0f / static_cast<float>(c->world);
    for (int i = 0; i < nsim; ++i) {
        const int r = c->simulated ? i : c->rank;
        cmn_status st = launched(c,
                                 launch_update_chunk(c->d_td, c->d_sitems, c->sitem_begin[r],
                                                     c->sitem_begin[r + 1], c->rb[r].reduced[0], dtype,
                                                     static_cast<float *>(c->rb[r].reduced[1]), inv_n,
                                                     lr, mu, s),
                                 "update_chunk");
        if (st != CMN_OK) return st;
    }
    ++c->seq;
    const Barrier bar2 = make_barrier(c, 3);
    const int total = c->sitem_begin[c->world];
    const int gblocks = upd_blocks_for(c, total);
    for (int i = 0; i < nsim; ++i) {
        const int r = c->simulated ? i : c->rank;
        cmn_status st = launched(c,
                                 launch_gather_params(c->d_td, c->d_sitems, 0, total, c->sitem_begin[r],
                                                      c->sitem_begin[r + 1], exch, c->world, bar2,
                                                      gblocks, s),
                                 "gather_params");
        if (st != CMN_OK) return st;
    }
    c->fresh = false;
    return CMN_OK;
}

// Fused two-shot step: pack -> reduce-scatter (start barrier) -> fused
// all-gather + update reading every reduced chunk from its owner (start
// barrier).  Every buffer overwrite is behind a start barrier (as in the
// sharded step), so the schedule is graph-safe.
cmn_status step_fused(cmn_comm *c, const float *const *grads, int dtype, float lr, float mu,
                      cudaStream_t s) {
    cmn_algo algo = CMN_ALGO_AUTO;
    if (cmn_status st = begin_collective(c, 0, c->T, dtype, algo, s, true); st != CMN_OK) return st;
    const int nsim = c->simulated ? c->world : 1;
    const uint32_t seq1 = ++c->seq;
    const int par = static_cast<int>(seq1 & 1u);
    PeerBufs red{};
    for (int r = 0; r < c->world; ++r) red.p[r] = c->rb[r].reduced[0];
    int64_t cs[kMaxWorld], ce[kMaxWorld];
    chunk_plan(0, c->L, c->world, cs, ce);
    const int blocks = ar_blocks_for(c);
    const int total = c->sitem_begin[c->world];
    const Barrier bar = make_barrier(c, dtype | 2);
    // Push form (fused_update == 2, one grad table): owner o's inbox is its
    // packed[0] buffer, slot i (rank i's contribution to chunk o) at
    // i * cmax payload elements; view(o, i) + j addresses packed index j.
    const bool push = c->fused_update == 2 && c->T <= kGradCap;
    const size_t esz = dtype == 0 ? 4 : 2;
    const int64_t cmax = align_up((c->L + c->world - 1) / c->world, kAlign);
    auto inbox_view = [&](int owner, int slot) -> const void * {
        const intptr_t a = reinterpret_cast<intptr_t>(c->rb[owner].packed[0]) +
                           static_cast<intptr_t>((slot * cmax - cs[owner]) * static_cast<int64_t>(esz));
        return reinterpret_cast<const void *>(a);
    };
    cmn_status st = CMN_OK;
    if (push) {
        const Barrier bar0 = make_barrier(c, dtype | 2);
        st = timed(c, s, [&] {
            for (int i = 0; i < nsim; ++i) {
                const int r = c->simulated ? i : c->rank;
                PeerBufs dst{};
                for (int o = 0; o < c->world; ++o) dst.p[o] = inbox_view(o, r);
                cmn_status st2 = launched(
                    c,
                    launch_pack_push(make_tab(grads + static_cast<size_t>(i) * c->T, 0, c->T), 0,
                                     c->d_sitems, 0, total, dst, c->world, dtype, bar0,
                                     upd_blocks_for(c, total), s),
                    "pack_push");
                if (st2 != CMN_OK) return st2;
            }
            return CMN_OK;
        });
    } else {
        st = pack_phase(c, 0, c->T, grads, dtype, par, s);
    }
    if (st != CMN_OK) return st;
    st = timed(c, s, [&] {
        for (int i = 0; i < nsim; ++i) {
            const int r = c->simulated ? i : c->rank;
            PeerBufs in{};
            for (int p = 0; p < c->world; ++p)
                in.p[p] = push ? inbox_view(r, p) : c->rb[p].packed[par];
            cmn_status st2 = launched(c,
                                      launch_allreduce_twoshot(in, red, c->world, r, cs, ce, dtype, 1,
                                                               bar, blocks, s),
                                      "reduce_scatter");
            if (st2 != CMN_OK) return st2;
        }
        return CMN_OK;
    });
    if (st != CMN_OK) return st;
    ++c->seq;
    const Barrier bar2 = make_barrier(c, dtype);
    const int gblocks = upd_blocks_for(c, total);
    // simulated ranks share one parameter replica: one launch updates it all
    st = timed(c, s, [&] {
        return launched(c,
                        launch_update_gather(c->d_td, c->d_sitems, 0, total, red, c->world, dtype,
                                             1.0f / static_cast<float>(c->world), lr, mu, bar2,
                                             gblocks, s),
                        "update_gather");
    });
    if (st != CMN_OK) return st;
    c->last = ArResult{0, dtype, false, false};   // rank r's chunk of reduced[0] (test hook)
    c->fresh = false;
    return CMN_OK;
}

}  // namespace

// =====================================================================
extern "C" {

int cmn_version(void) { return CMN_VERSION; }

const char *cmn_last_error(void) { return g_last_error.c_str(); }

cmn_status cmn_init(int rank, int world_size, int cuda_device, cmn_allgather_fn ag, void *user,
                    cmn_comm **out) {
    try {
        return init_common(rank, world_size, cuda_device, false, ag, user, out);
    } catch (...) {
        return fail(CMN_ERR_OOM, "host allocation failed");
    }
}

cmn_status cmn_init_simulated(int world_size, int cuda_device, cmn_comm **out) {
    try {
        return init_common(0, world_size, cuda_device, true, nullptr, nullptr, out);
    } catch (...) {
        return fail(CMN_ERR_OOM, "host allocation failed");
    }
}

cmn_status cmn_finalize(cmn_comm *c) {
    if (!c) return CMN_OK;
    cudaSetDevice(c->device);
    cudaDeviceSynchronize();
    if (c->nccl && g_nccl.CommDestroy) g_nccl.CommDestroy(c->nccl);
    for (auto e : c->ev) cudaEventDestroy(e);
    for (auto e : c->pev) cudaEventDestroy(e);
    for (auto e : c->kev) cudaEventDestroy(e);
    if (c->sc) cudaStreamDestroy(c->sc);
    if (c->h2d) cudaStreamDestroy(c->h2d);
    if (c->d2h) cudaStreamDestroy(c->d2h);
    free_registration(c);
    if (c->h_err) cudaFreeHost(c->h_err);
    delete c;
    return CMN_OK;
}

static cmn_status register_impl(cmn_comm *c, int T, const int *ndims, const int64_t *dims,
                                float *const *params);

cmn_status cmn_register_params(cmn_comm *c, int T, const int *ndims, const int64_t *dims,
                               float *const *params) {
    if (!c) return fail(CMN_ERR_INVALID_ARG, "comm is NULL");
    const cmn_status st = register_impl(c, T, ndims, dims, params);
    // A failed (re-)registration leaves the communicator unregistered (every
    // later call returns CMN_ERR_STATE), never half-mapped.
    if (st != CMN_OK && st != CMN_ERR_INVALID_ARG && c->T > 0) {
        const std::string msg = g_last_error;
        free_registration(c);
        g_last_error = msg;
    }
    return st;
}

static cmn_status register_impl(cmn_comm *c, int T, const int *ndims, const int64_t *dims,
                                float *const *params) {
    try {
        std::vector<int64_t> numel, off;
        uint64_t hash = 0;
        if (cmn_status st = plan_layout_impl(T, ndims, dims, numel, off, hash); st != CMN_OK)
            return st;
        if (!params) return fail(CMN_ERR_INVALID_ARG, "params table is NULL");
        for (int t = 0; t < T; ++t) {
            if (numel[t] == 0) continue;
            if (!params[t]) return fail(CMN_ERR_INVALID_ARG, "param pointer is NULL");
            if (reinterpret_cast<uintptr_t>(params[t]) % 16 != 0)
                return fail(CMN_ERR_INVALID_ARG, "param pointer is not 16-byte aligned");
        }
        if (cmn_status st = set_device(c); st != CMN_OK) return st;
        CMN_CUDA(cudaDeviceSynchronize());
        if (c->T > 0 && !c->simulated && c->world > 1) {
            // Re-registration frees IPC-exported buffers that peers may still be
            // reading in their last collective: all ranks first drain their
            // devices, then meet here (allgather as a host barrier).
            int one = 1;
            std::vector<int> all(c->world);
            if (!allgather(c, &one, all.data(), sizeof(int)))
                return fail(CMN_ERR_BOOTSTRAP, "allgather callback failed");
        }
        free_registration(c);
        c->T = T;
        c->numel = numel;
        c->off = off;
        c->L = off[T];
        c->hash = hash;
        c->params.assign(params, params + T);
        c->params_flat = params_are_flat(c);
        c->seq = 0;

        // Work items: each tensor cut into kItemElems pieces.
        c->h_items.clear();
        c->item_begin.assign(T + 1, 0);
        for (int t = 0; t < T; ++t) {
            c->item_begin[t] = static_cast<int>(c->h_items.size());
            for (int64_t k0 = 0; k0 < numel[t]; k0 += kItemElems) {
                const int64_t len = numel[t] - k0 < kItemElems ? numel[t] - k0 : kItemElems;
                const bool last = k0 + len == numel[t];
                c->h_items.push_back(Item{t, static_cast<int32_t>(len), k0, off[t] + k0,
                                          last ? static_cast<int32_t>(off[t + 1] - off[t] - numel[t]) : 0,
                                          0});
            }
        }
        c->item_begin[T] = static_cast<int>(c->h_items.size());

        const size_t Lb = static_cast<size_t>(c->L > 0 ? c->L : 1) * 4;
        if (cudaMalloc(&c->d_mom, Lb) != cudaSuccess) return fail(CMN_ERR_OOM, "momentum alloc");
        CMN_CUDA(cudaMemset(c->d_mom, 0, Lb));
        c->h_td.assign(T, TensorDesc{});
        for (int t = 0; t < T; ++t) {
            TensorDesc &d = c->h_td[t];
            d.w = params[t];
            d.mom = c->d_mom + off[t];
            d.n = numel[t];
            d.off = off[t];
            d.off_next = off[t + 1];
        }
        CMN_CUDA(cudaMalloc(&c->d_td, sizeof(TensorDesc) * T));
        CMN_CUDA(cudaMemcpy(c->d_td, c->h_td.data(), sizeof(TensorDesc) * T, cudaMemcpyHostToDevice));
        const size_t ib = sizeof(Item) * (c->h_items.empty() ? 1 : c->h_items.size());
        CMN_CUDA(cudaMalloc(&c->d_items, ib));
        if (!c->h_items.empty())
            CMN_CUDA(cudaMemcpy(c->d_items, c->h_items.data(), sizeof(Item) * c->h_items.size(),
                                cudaMemcpyHostToDevice));

        // Sharded-update item lists: items clipped to each rank's chunk.
        {
            std::vector<Item> sit;
            int64_t cs[kMaxWorld], ce[kMaxWorld];
            chunk_plan(0, c->L, c->world, cs, ce);
            c->sitem_begin.assign(c->world + 1, 0);
            for (int r = 0; r < c->world; ++r) {
                c->sitem_begin[r] = static_cast<int>(sit.size());
                for (const Item &it : c->h_items) {
                    const int64_t lo = it.base > cs[r] ? it.base : cs[r];
                    const int64_t hi = it.base + it.len < ce[r] ? it.base + it.len : ce[r];
                    if (lo >= hi) continue;
                    // a tensor's pad never straddles a chunk boundary (boundaries
                    // are multiples of 64, pads end at one): keep it on the piece
                    // that ends the tensor
                    const int32_t pad = hi == it.base + it.len ? it.pad : 0;
                    sit.push_back(Item{it.t, static_cast<int32_t>(hi - lo), it.k0 + (lo - it.base), lo,
                                       pad, r});
                }
            }
            c->sitem_begin[c->world] = static_cast<int>(sit.size());
            CMN_CUDA(cudaMalloc(&c->d_sitems, sizeof(Item) * (sit.empty() ? 1 : sit.size())));
            if (!sit.empty())
                CMN_CUDA(cudaMemcpy(c->d_sitems, sit.data(), sizeof(Item) * sit.size(),
                                    cudaMemcpyHostToDevice));
        }
        if (cmn_status st = alloc_regions(c); st != CMN_OK) return st;
        if (!c->simulated) {
            if (c->world > 1) {
                if (cmn_status st = exchange_and_map(c); st != CMN_OK) return st;
            }
            if (c->algo == CMN_ALGO_NVLS) {   // collective: every rank re-registers
                std::string err;
                if (!nvls_setup(c->nvls, c->rank, c->world, c->device, static_cast<size_t>(c->L) * 4,
                                c->ag, c->user, err)) {
                    nvls_teardown(c->nvls);
                    c->algo = CMN_ALGO_AUTO;
                    return fail(CMN_ERR_CUDA, "NVLS setup: " + err);
                }
            }
        }
        CMN_CUDA(cudaDeviceSynchronize());
        return CMN_OK;
    } catch (...) {
        return fail(CMN_ERR_OOM, "host allocation failed");
    }
}

cmn_status cmn_get_layout(const cmn_comm *c, int64_t *offsets, int64_t *padded_len) {
    if (!c) return fail(CMN_ERR_INVALID_ARG, "comm is NULL");
    if (c->T == 0) return fail(CMN_ERR_STATE, "not registered");
    if (offsets) std::memcpy(offsets, c->off.data(), sizeof(int64_t) * (c->T + 1));
    if (padded_len) *padded_len = c->L;
    return CMN_OK;
}

cmn_status cmn_allreduce_grads(cmn_comm *c, const float *const *grads, cmn_dtype dtype,
                               void *stream) {
    if (cmn_status st = require_registered(c); st != CMN_OK) return st;
    if (cmn_status st = require_dtype(dtype); st != CMN_OK) return st;
    std::string why;
    if (!grads_ok(c, grads, c->T * (c->simulated ? c->world : 1), why))
        return fail(CMN_ERR_INVALID_ARG, why);
    if (cmn_status st = set_device(c); st != CMN_OK) return st;
    cmn_status st = allreduce_range(c, 0, c->T, grads, dtype, static_cast<cudaStream_t>(stream));
    if (st == CMN_OK) {
        c->fresh = true;
        c->bucket_fresh.assign(c->buckets.size(), 0);
    }
    return st;
}

cmn_status cmn_update_momentum_sgd(cmn_comm *c, float lr, float mu, void *stream) {
    if (cmn_status st = require_registered(c); st != CMN_OK) return st;
    if (!c->fresh) return fail(CMN_ERR_STATE, "no fresh all-reduce result to consume");
    if (cmn_status st = set_device(c); st != CMN_OK) return st;
    cmn_status st = update_range(c, 0, c->T, c->last, lr, mu, static_cast<cudaStream_t>(stream));
    if (st == CMN_OK) c->fresh = false;
    return st;
}

cmn_status cmn_step(cmn_comm *c, const float *const *grads, cmn_dtype dtype, float lr, float mu,
                    void *stream) {
    if (cmn_status st = require_registered(c); st != CMN_OK) return st;
    if (cmn_status st = require_dtype(dtype); st != CMN_OK) return st;
    if (c->world > 1 || c->algo == CMN_ALGO_NVLS) {
        const bool lib_collective = c->algo == CMN_ALGO_NVLS || c->algo == CMN_ALGO_NCCL;
        if (lib_collective && (c->world == 1 || c->fused_update || c->pipe_pieces < 2)) {
            // single-rank plumbing, or a schedule that needs the two-shot
            // reduce-scatter: serial step
            cmn_status st = cmn_allreduce_grads(c, grads, dtype, stream);
            if (st != CMN_OK) return st;
            return cmn_update_momentum_sgd(c, lr, mu, stream);
        }
        if (c->fused_update) {
            std::string why;
            if (!grads_ok(c, grads, c->T * (c->simulated ? c->world : 1), why))
                return fail(CMN_ERR_INVALID_ARG, why);
            if (cmn_status st = set_device(c); st != CMN_OK) return st;
            return step_fused(c, grads, dtype, lr, mu, static_cast<cudaStream_t>(stream));
        }
        if (c->pipe_pieces >= 2 && c->T >= 2) {
            std::string why;
            if (!grads_ok(c, grads, c->T * (c->simulated ? c->world : 1), why))
                return fail(CMN_ERR_INVALID_ARG, why);
            if (cmn_status st = set_device(c); st != CMN_OK) return st;
            return step_pipelined(c, grads, dtype, lr, mu, static_cast<cudaStream_t>(stream));
        }
        cmn_status st = cmn_allreduce_grads(c, grads, dtype, stream);
        if (st != CMN_OK) return st;
        return cmn_update_momentum_sgd(c, lr, mu, stream);
    }
    std::string why;
    if (!grads_ok(c, grads, c->T, why)) return fail(CMN_ERR_INVALID_ARG, why);
    if (cmn_status st = set_device(c); st != CMN_OK) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    c->fresh = false;
    return timed(c, s, [&] {
        return for_groups(c, 0, c->T, [&](int lo, int hi, int i0, int i1) {
            return launched(c,
                            launch_update_direct(make_tab(grads, lo, hi), make_tab(c->params.data(), lo, hi),
                                                 hi - lo, lo, c->d_mom, c->d_items, i0, i1, dtype, lr,
                                                 mu, s),
                            "update_direct");
        });
    });
}

cmn_status cmn_step_sharded(cmn_comm *c, const float *const *grads, cmn_dtype dtype, float lr,
                            float mu, void *stream) {
    if (cmn_status st = require_registered(c); st != CMN_OK) return st;
    if (cmn_status st = require_dtype(dtype); st != CMN_OK) return st;
    if (c->world == 1) return cmn_step(c, grads, dtype, lr, mu, stream);
    std::string why;
    if (!grads_ok(c, grads, c->T * (c->simulated ? c->world : 1), why))
        return fail(CMN_ERR_INVALID_ARG, why);
    if (cmn_status st = set_device(c); st != CMN_OK) return st;
    return step_sharded(c, grads, dtype, lr, mu, static_cast<cudaStream_t>(stream));
}

cmn_status cmn_step_host(cmn_comm *c, const float *const *host_grads, float *const *host_params,
                         cmn_dtype dtype, float lr, float mu, void *stream) {
    if (cmn_status st = require_registered(c); st != CMN_OK) return st;
    if (cmn_status st = require_dtype(dtype); st != CMN_OK) return st;
    const int nsim = c->simulated ? c->world : 1;
    if (!host_grads) return fail(CMN_ERR_INVALID_ARG, "host_grads is NULL");
    for (int i = 0; i < nsim * c->T; ++i)
        if (c->numel[i % c->T] > 0 && !host_grads[i])
            return fail(CMN_ERR_INVALID_ARG, "host grad pointer is NULL");
    if (cmn_status st = set_device(c); st != CMN_OK) return st;
    if (cmn_status st = ensure_staging(c); st != CMN_OK) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    std::vector<const float *> dg(static_cast<size_t>(nsim) * c->T);
    for (int i = 0; i < nsim; ++i) {
        std::vector<float *> dst(c->T);
        for (int t = 0; t < c->T; ++t) {
            dst[t] = c->d_staging + static_cast<size_t>(i) * c->L + c->off[t];
            dg[static_cast<size_t>(i) * c->T + t] = dst[t];
        }
        if (cmn_status st = copy_tensors(c, host_grads + static_cast<size_t>(i) * c->T, dst.data(),
                                         0, c->T, cudaMemcpyHostToDevice, s);
            st != CMN_OK)
            return st;
    }
    if (cmn_status st = cmn_step(c, dg.data(), dtype, lr, mu, stream); st != CMN_OK) return st;
    if (host_params) {
        std::vector<const float *> src(c->params.begin(), c->params.end());
        if (cmn_status st = copy_tensors(c, src.data(), host_params, 0, c->T,
                                         cudaMemcpyDeviceToHost, s);
            st != CMN_OK)
            return st;
    }
    return CMN_OK;
}

cmn_status cmn_step_host_packed(cmn_comm *c, const float *host_grads, float *host_params,
                                cmn_dtype dtype, float lr, float mu, void *stream) {
    if (cmn_status st = require_registered(c); st != CMN_OK) return st;
    if (cmn_status st = require_dtype(dtype); st != CMN_OK) return st;
    if (!host_grads) return fail(CMN_ERR_INVALID_ARG, "host_grads is NULL");
    if (cmn_status st = set_device(c); st != CMN_OK) return st;
    if (cmn_status st = ensure_staging(c); st != CMN_OK) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int nsim = c->simulated ? c->world : 1;
    std::vector<const float *> dg(static_cast<size_t>(nsim) * c->T);
    for (int i = 0; i < nsim; ++i)
        for (int t = 0; t < c->T; ++t)
            dg[static_cast<size_t>(i) * c->T + t] = c->d_staging + static_cast<size_t>(i) * c->L + c->off[t];
    std::string why;
    if (!grads_ok(c, dg.data(), nsim * c->T, why)) return fail(CMN_ERR_INVALID_ARG, why);

    if (c->world > 1 || c->simulated) {
        // The pipelined schedule carries the host copies piece by piece.
        if (c->world > 1 && c->pipe_pieces >= 2 && c->T >= 2 && !c->fused_update) {
            const HostIO io{host_grads, host_params};
            return step_pipelined(c, dg.data(), dtype, lr, mu, s, &io);
        }
        // Other schedules: the all-reduce needs every gradient first.
        CMN_CUDA(cudaMemcpyAsync(c->d_staging, host_grads, static_cast<size_t>(c->L) * 4 * nsim,
                                 cudaMemcpyHostToDevice, s));
        if (cmn_status st = cmn_step(c, dg.data(), dtype, lr, mu, stream); st != CMN_OK) return st;
        return host_params ? d2h_params(c, 0, c->T, host_params, s) : CMN_OK;
    }

    // N = 1: pipeline H2D(piece p+1) || update(piece p) || D2H(piece p-1) on
    // two copy engines and the caller's stream, over item ranges.
    if (cmn_status st = ensure_side_streams(c); st != CMN_OK) return st;
    const auto pieces = e2e_item_pieces(c);
    const int I = c->item_begin[c->T];
    int last = c->T - 1;                  // end of the last tensor's data: contiguous
    while (last > 0 && c->numel[last] == 0) --last;   // D2H copies stop there
    const int64_t flat_end = c->off[last] + c->numel[last];
    cudaEvent_t entry = c->ev[0], done_d2h = c->ev[1];
    CMN_CUDA(cudaEventRecord(entry, s));
    CMN_CUDA(cudaStreamWaitEvent(c->h2d, entry, 0));
    CMN_CUDA(cudaStreamWaitEvent(c->d2h, entry, 0));
    c->fresh = false;
    for (size_t p = 0; p < pieces.size(); ++p) {
        const int i0 = pieces[p].first, i1 = pieces[p].second;
        const int64_t e0 = i0 == 0 ? 0 : c->h_items[i0].base;
        const int64_t e1 = i1 == I ? c->L : c->h_items[i1].base;
        cudaEvent_t ev_in = c->ev[2 + 3 * p], ev_upd = c->ev[3 + 3 * p];
        CMN_CUDA(cudaMemcpyAsync(c->d_staging + e0, host_grads + e0, static_cast<size_t>(e1 - e0) * 4,
                                 cudaMemcpyHostToDevice, c->h2d));
        CMN_CUDA(cudaEventRecord(ev_in, c->h2d));
        CMN_CUDA(cudaStreamWaitEvent(s, ev_in, 0));
        cmn_status st = for_groups(c, 0, c->T, [&](int lo, int hi, int g0, int g1) {
            const int a = g0 > i0 ? g0 : i0, b = g1 < i1 ? g1 : i1;
            if (a >= b) return CMN_OK;
            return launched(c,
                            launch_update_direct(make_tab(dg.data(), lo, hi),
                                                 make_tab(c->params.data(), lo, hi), hi - lo, lo,
                                                 c->d_mom, c->d_items, a, b, dtype, lr, mu, s),
                            "update_direct");
        });
        if (st != CMN_OK) return st;
        if (host_params) {
            CMN_CUDA(cudaEventRecord(ev_upd, s));
            CMN_CUDA(cudaStreamWaitEvent(c->d2h, ev_upd, 0));
            if (c->params_flat) {
                const int64_t hi = e1 < flat_end ? e1 : flat_end;
                if (hi > e0)
                    CMN_CUDA(cudaMemcpyAsync(host_params + e0, c->params[0] + e0,
                                             static_cast<size_t>(hi - e0) * 4,
                                             cudaMemcpyDeviceToHost, c->d2h));
            } else {
                // per tensor: the elements of [i0, i1) that belong to it
                for (int i = i0; i < i1;) {
                    const Item &a = c->h_items[i];
                    int j = i;
                    while (j + 1 < i1 && c->h_items[j + 1].t == a.t) ++j;
                    const Item &b = c->h_items[j];
                    CMN_CUDA(cudaMemcpyAsync(host_params + c->off[a.t] + a.k0, c->params[a.t] + a.k0,
                                             static_cast<size_t>(b.k0 + b.len - a.k0) * 4,
                                             cudaMemcpyDeviceToHost, c->d2h));
                    i = j + 1;
                }
            }
        }
    }
    CMN_CUDA(cudaEventRecord(done_d2h, c->d2h));
    CMN_CUDA(cudaStreamWaitEvent(s, done_d2h, 0));
    // the H2D stream is joined through the per-piece waits already
    return CMN_OK;
}

cmn_status cmn_unpack_avg_grads(cmn_comm *c, float *const *out, void *stream) {
    if (cmn_status st = require_registered(c); st != CMN_OK) return st;
    if (!c->fresh) return fail(CMN_ERR_STATE, "no fresh all-reduce result");
    std::string why;
    if (!grads_ok(c, const_cast<const float *const *>(out), c->T, why))
        return fail(CMN_ERR_INVALID_ARG, why);
    if (cmn_status st = set_device(c); st != CMN_OK) return st;
    const float inv_n = 1.0f / static_cast<float>(c->world);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    return for_groups(c, 0, c->T, [&](int lo, int hi, int i0, int i1) {
        return launched(c,
                        launch_unpack_avg(make_tab(const_cast<const float *const *>(out), lo, hi),
                                          lo, c->d_td, c->d_items, i0, i1,
                                          reduced_ptr(c, c->last, 0), c->last.dtype, inv_n, s),
                        "unpack_avg");
    });
}

cmn_status cmn_update_adam(cmn_comm *c, float alpha, float beta1, float beta2, float eps,
                           int step, void *stream) {
    if (cmn_status st = require_registered(c); st != CMN_OK) return st;
    if (!c->fresh) return fail(CMN_ERR_STATE, "no fresh all-reduce result to consume");
    if (step < 1) return fail(CMN_ERR_INVALID_ARG, "step must be >= 1");
    if (cmn_status st = set_device(c); st != CMN_OK) return st;
    if (!c->d_adam) {
        const size_t b = static_cast<size_t>(c->L > 0 ? c->L : 1) * 4 * 2;
        if (cudaMalloc(&c->d_adam, b) != cudaSuccess) return fail(CMN_ERR_OOM, "adam state alloc");
        CMN_CUDA(cudaMemset(c->d_adam, 0, b));
        for (int t = 0; t < c->T; ++t) {
            c->h_td[t].adam_m = c->d_adam + c->off[t];
            c->h_td[t].adam_v = c->d_adam + c->L + c->off[t];
        }
        CMN_CUDA(cudaMemcpy(c->d_td, c->h_td.data(), sizeof(TensorDesc) * c->T,
                            cudaMemcpyHostToDevice));
    }
    // alpha_t = alpha * sqrt(1 - beta2^t) / (1 - beta1^t), evaluated in double.
    const double b1t = std::pow(static_cast<double>(beta1), static_cast<double>(step));
    const double b2t = std::pow(static_cast<double>(beta2), static_cast<double>(step));
    const float alpha_t = static_cast<float>(static_cast<double>(alpha) * std::sqrt(1.0 - b2t) / (1.0 - b1t));
    const float c1 = 1.0f - beta1, c2 = 1.0f - beta2;
    const float inv_n = 1.0f / static_cast<float>(c->world);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    cmn_status st = for_groups(c, 0, c->T, [&](int, int, int i0, int i1) {
        return launched(c,
                        launch_update_adam(c->d_td, c->d_items, i0, i1,
                                           reduced_ptr(c, c->last, 0), c->last.dtype, inv_n,
                                           alpha_t, beta1, beta2, c1, c2, eps, s),
                        "update_adam");
    });
    if (st == CMN_OK) c->fresh = false;
    return st;
}

namespace {
// Reverse-order greedy bucket plan over tensor sizes (host only).
std::vector<std::pair<int, int>> bucket_plan(const int64_t *numel, int T, size_t bucket_bytes) {
    std::vector<std::pair<int, int>> out;
    int end = T;
    while (end > 0) {
        int begin = end - 1;
        size_t acc = static_cast<size_t>(numel[begin]) * 4;
        while (begin > 0 && bucket_bytes > 0 &&
               acc + static_cast<size_t>(numel[begin - 1]) * 4 <= bucket_bytes) {
            --begin;
            acc += static_cast<size_t>(numel[begin]) * 4;
        }
        if (bucket_bytes == 0) begin = 0;
        out.emplace_back(begin, end);
        end = begin;
    }
    return out;
}
}  // namespace

cmn_status cmn_plan_bucket_ranges(int n_tensors, const int64_t *numel, size_t bucket_bytes,
                                  int *n_buckets_out, int *t_begin, int *t_end) {
    if (n_tensors <= 0 || !numel || !n_buckets_out)
        return fail(CMN_ERR_INVALID_ARG, "n_tensors must be >= 1; numel and n_buckets_out non-NULL");
    for (int t = 0; t < n_tensors; ++t)
        if (numel[t] < 0) return fail(CMN_ERR_INVALID_ARG, "negative numel");
    try {
        const auto plan = bucket_plan(numel, n_tensors, bucket_bytes);
        *n_buckets_out = static_cast<int>(plan.size());
        for (size_t b = 0; b < plan.size(); ++b) {
            if (t_begin) t_begin[b] = plan[b].first;
            if (t_end) t_end[b] = plan[b].second;
        }
        return CMN_OK;
    } catch (...) {
        return fail(CMN_ERR_OOM, "host allocation failed");
    }
}

cmn_status cmn_plan_buckets(cmn_comm *c, size_t bucket_bytes, int *n_out) {
    if (cmn_status st = require_registered(c); st != CMN_OK) return st;
    c->buckets = bucket_plan(c->numel.data(), c->T, bucket_bytes);
    c->bucket_fresh.assign(c->buckets.size(), 0);
    c->bucket_res.assign(c->buckets.size(), ArResult{});
    if (n_out) *n_out = static_cast<int>(c->buckets.size());
    return CMN_OK;
}

cmn_status cmn_get_bucket(const cmn_comm *c, int b, int *t_begin, int *t_end) {
    if (!c) return fail(CMN_ERR_INVALID_ARG, "comm is NULL");
    if (b < 0 || b >= static_cast<int>(c->buckets.size()))
        return fail(CMN_ERR_INVALID_ARG, "bucket index out of range");
    if (t_begin) *t_begin = c->buckets[b].first;
    if (t_end) *t_end = c->buckets[b].second;
    return CMN_OK;
}

cmn_status cmn_allreduce_bucket(cmn_comm *c, int b, const float *const *grads, cmn_dtype dtype,
                                void *stream) {
    if (cmn_status st = require_registered(c); st != CMN_OK) return st;
    if (cmn_status st = require_dtype(dtype); st != CMN_OK) return st;
    if (b < 0 || b >= static_cast<int>(c->buckets.size()))
        return fail(CMN_ERR_INVALID_ARG, "bucket index out of range");
    std::string why;
    if (!grads_ok(c, grads, c->T * (c->simulated ? c->world : 1), why))
        return fail(CMN_ERR_INVALID_ARG, why);
    if (cmn_status st = set_device(c); st != CMN_OK) return st;
    cmn_status st = allreduce_range(c, c->buckets[b].first, c->buckets[b].second, grads, dtype,
                                    static_cast<cudaStream_t>(stream));
    if (st == CMN_OK) {
        c->bucket_fresh[b] = 1;
        c->bucket_res[b] = c->last;
        c->fresh = false;
    }
    return st;
}

cmn_status cmn_update_bucket(cmn_comm *c, int b, float lr, float mu, void *stream) {
    if (cmn_status st = require_registered(c); st != CMN_OK) return st;
    if (b < 0 || b >= static_cast<int>(c->buckets.size()))
        return fail(CMN_ERR_INVALID_ARG, "bucket index out of range");
    if (!c->bucket_fresh[b]) return fail(CMN_ERR_STATE, "bucket has no fresh all-reduce result");
    if (cmn_status st = set_device(c); st != CMN_OK) return st;
    // The bucket's reduced values sit in the buffer of the parity its own
    // all-reduce call used (recorded per bucket).
    cmn_status st = update_range(c, c->buckets[b].first, c->buckets[b].second, c->bucket_res[b],
                                 lr, mu, static_cast<cudaStream_t>(stream));
    if (st == CMN_OK) c->bucket_fresh[b] = 0;
    return st;
}

cmn_status cmn_set_algo(cmn_comm *c, cmn_algo algo, size_t oneshot_max_bytes) {
    if (!c) return fail(CMN_ERR_INVALID_ARG, "comm is NULL");
    if (algo < CMN_ALGO_AUTO || algo > CMN_ALGO_NVLS) return fail(CMN_ERR_INVALID_ARG, "bad algo");
    if (oneshot_max_bytes) c->oneshot_max = oneshot_max_bytes;
    if (algo == CMN_ALGO_NVLS && !c->nvls.ready()) {
        if (c->simulated) return fail(CMN_ERR_UNSUPPORTED, "NVLS needs one process per GPU");
        if (c->T == 0) return fail(CMN_ERR_STATE, "register parameters before selecting NVLS");
        if (cmn_status st = set_device(c); st != CMN_OK) return st;
        std::string err;
        if (!nvls_setup(c->nvls, c->rank, c->world, c->device, static_cast<size_t>(c->L) * 4, c->ag,
                        c->user, err)) {
            nvls_teardown(c->nvls);
            return fail(err.find("support") != std::string::npos ? CMN_ERR_UNSUPPORTED : CMN_ERR_CUDA,
                        "NVLS setup: " + err);
        }
    }
    if (algo == CMN_ALGO_NCCL && !c->nccl) {
        if (c->simulated) return fail(CMN_ERR_UNSUPPORTED, "NCCL needs one process per GPU");
        if (cmn_status st = set_device(c); st != CMN_OK) return st;
        // Every rank joins the id exchange even after a local failure, with
        // its status alongside, so no rank is left blocked in a collective.
        struct IdMsg {
            int ok;
            NcclUniqueId id;
        } mine{};
        std::string why;
        if (!g_nccl.load())
            why = "cannot load libnccl (set CMN_NCCL_LIB)";
        else if (c->rank == 0 && g_nccl.GetUniqueId(&mine.id) != 0)
            why = "ncclGetUniqueId failed";
        mine.ok = why.empty() ? 1 : 0;
        std::vector<IdMsg> all(c->world);
        if (!allgather(c, &mine, all.data(), sizeof(IdMsg)))
            return fail(CMN_ERR_BOOTSTRAP, "allgather callback failed");
        for (int r = 0; r < c->world && why.empty(); ++r)
            if (!all[r].ok) why = "NCCL setup failed on rank " + std::to_string(r);
        if (!why.empty()) return fail(CMN_ERR_NCCL, why);
        void *comm = nullptr;
        const int rc = g_nccl.CommInitRank(&comm, c->world, all[0].id, c->rank);   // rank 0's id
        if (rc != 0)
            return fail(CMN_ERR_NCCL, std::string("ncclCommInitRank: ") +
                                          (g_nccl.GetErrorString ? g_nccl.GetErrorString(rc) : "?"));
        c->nccl = comm;
    }
    c->algo = algo;
    return CMN_OK;
}

cmn_status cmn_set_fused_update(cmn_comm *c, int mode) {
    if (!c) return fail(CMN_ERR_INVALID_ARG, "comm is NULL");
    if (mode < 0 || mode > 2) return fail(CMN_ERR_INVALID_ARG, "fused-update mode must be 0, 1 or 2");
    c->fused_update = mode;
    return CMN_OK;
}

cmn_status cmn_set_pipeline(cmn_comm *c, int pieces) {
    if (!c) return fail(CMN_ERR_INVALID_ARG, "comm is NULL");
    if (pieces < 0 || pieces > 64) return fail(CMN_ERR_INVALID_ARG, "pieces must be in [0, 64]");
    c->pipe_pieces = pieces;
    return CMN_OK;
}

cmn_status cmn_set_ctas(cmn_comm *c, int collective_ctas, int update_ctas) {
    if (!c) return fail(CMN_ERR_INVALID_ARG, "comm is NULL");
    if (collective_ctas < 0 || collective_ctas > kMaxBarrierBlocks || update_ctas < 0 ||
        update_ctas > kMaxBarrierBlocks)
        return fail(CMN_ERR_INVALID_ARG, "CTA counts must be in [0, 1024] (0 = default)");
    c->ar_blocks = collective_ctas;
    c->upd_blocks = update_ctas;
    return CMN_OK;
}

cmn_status cmn_set_kernel_timing(cmn_comm *c, int on) {
    if (!c) return fail(CMN_ERR_INVALID_ARG, "comm is NULL");
    c->ktiming = on != 0;
    c->ktimed = 0;
    return CMN_OK;
}

cmn_status cmn_get_kernel_timing(cmn_comm *c, double *total_ms, int *count) {
    if (!c || !total_ms || !count) return fail(CMN_ERR_INVALID_ARG, "NULL argument");
    double sum = 0.0;
    for (size_t i = 0; i < c->ktimed; ++i) {
        CMN_CUDA(cudaEventSynchronize(c->kev[2 * i + 1]));
        float ms = 0.f;
        CMN_CUDA(cudaEventElapsedTime(&ms, c->kev[2 * i], c->kev[2 * i + 1]));
        sum += ms;
    }
    *total_ms = sum;
    *count = static_cast<int>(c->ktimed);
    c->ktimed = 0;
    return CMN_OK;
}

cmn_status cmn_set_timeout(cmn_comm *c, uint32_t timeout_ms) {
    if (!c) return fail(CMN_ERR_INVALID_ARG, "comm is NULL");
    if (timeout_ms == 0) return fail(CMN_ERR_INVALID_ARG, "timeout must be > 0");
    c->timeout_ms = timeout_ms;
    return CMN_OK;
}

cmn_status cmn_get_momentum(cmn_comm *c, int t, float **p) {
    if (cmn_status st = require_registered(c); st != CMN_OK) return st;
    if (t < 0 || t >= c->T || !p) return fail(CMN_ERR_INVALID_ARG, "bad tensor index / out ptr");
    *p = c->d_mom + c->off[t];
    return CMN_OK;
}

cmn_status cmn_get_adam_state(cmn_comm *c, int t, float **m, float **v) {
    if (cmn_status st = require_registered(c); st != CMN_OK) return st;
    if (t < 0 || t >= c->T) return fail(CMN_ERR_INVALID_ARG, "bad tensor index");
    if (!c->d_adam) return fail(CMN_ERR_STATE, "no Adam state (call cmn_update_adam first)");
    if (m) *m = c->d_adam + c->off[t];
    if (v) *v = c->d_adam + c->L + c->off[t];
    return CMN_OK;
}

static cmn_status copy_buf(cmn_comm *c, int rank, void *dst, void *stream, bool reduced) {
    if (cmn_status st = require_registered(c); st != CMN_OK) return st;
    if (!dst) return fail(CMN_ERR_INVALID_ARG, "dst is NULL");
    if (c->seq == 0) return fail(CMN_ERR_STATE, "no all-reduce issued yet");
    if (c->simulated ? (rank < 0 || rank >= c->world) : rank != c->rank)
        return fail(CMN_ERR_INVALID_ARG, "rank not accessible from this process");
    if (cmn_status st = set_device(c); st != CMN_OK) return st;
    const int r = c->simulated ? rank : c->rank;
    const void *src = reduced ? reduced_ptr(c, c->last, r)
                              : (c->last.nvls ? c->nvls.packed_uc() : c->rb[r].packed[c->last.parity]);
    const size_t bytes = static_cast<size_t>(c->L) * (c->last.dtype == 0 ? 4 : 2);
    CMN_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice,
                             static_cast<cudaStream_t>(stream)));
    return CMN_OK;
}

cmn_status cmn_copy_packed(cmn_comm *c, int rank, void *dst, void *stream) {
    return copy_buf(c, rank, dst, stream, false);
}

cmn_status cmn_copy_reduced(cmn_comm *c, int rank, void *dst, void *stream) {
    return copy_buf(c, rank, dst, stream, true);
}

cmn_status cmn_poll_error(cmn_comm *c) {
    if (!c) return fail(CMN_ERR_INVALID_ARG, "comm is NULL");
    return check_async_error(c);
}

uint64_t cmn_kernel_launches(const cmn_comm *c) { return c ? c->launches : 0; }

// ------------------------------------------------------- host-only helpers

cmn_status cmn_plan_layout(int T, const int *ndims, const int64_t *dims, int64_t *offsets,
                           int64_t *padded_len, uint64_t *hash_out) {
    try {
        std::vector<int64_t> numel, off;
        uint64_t hash = 0;
        if (cmn_status st = plan_layout_impl(T, ndims, dims, numel, off, hash); st != CMN_OK)
            return st;
        if (offsets) std::memcpy(offsets, off.data(), sizeof(int64_t) * (T + 1));
        if (padded_len) *padded_len = off[T];
        if (hash_out) *hash_out = hash;
        return CMN_OK;
    } catch (...) {
        return fail(CMN_ERR_OOM, "host allocation failed");
    }
}

cmn_status cmn_plan_chunks(int64_t L, int world, int64_t *starts, int64_t *ends) {
    if (world < 1 || world > kMaxWorld) return fail(CMN_ERR_INVALID_ARG, "world out of range");
    if (L < 0 || !starts || !ends) return fail(CMN_ERR_INVALID_ARG, "bad arguments");
    chunk_plan(0, L, world, starts, ends);
    return CMN_OK;
}

cmn_status cmn_share_fd(int rank, int world, cmn_allgather_fn ag, void *user, int fd_in,
                        int *fd_out) {
    if (world < 1 || world > kMaxWorld || rank < 0 || rank >= world || !fd_out)
        return fail(CMN_ERR_INVALID_ARG, "bad arguments");
    if (world > 1 && !ag) return fail(CMN_ERR_INVALID_ARG, "allgather callback required");
    std::string err;
    if (!share_fd(rank, world, ag, user, fd_in, fd_out, err)) return fail(CMN_ERR_BOOTSTRAP, err);
    return CMN_OK;
}

cmn_status cmn_bootstrap_verify(int rank, int world, cmn_allgather_fn ag, void *user,
                                uint64_t hash) {
    if (world < 1 || world > kMaxWorld || rank < 0 || rank >= world)
        return fail(CMN_ERR_INVALID_ARG, "rank/world out of range");
    if (world > 1 && !ag) return fail(CMN_ERR_INVALID_ARG, "allgather callback required");
    std::vector<uint64_t> all(world);
    if (world == 1) return CMN_OK;
    if (ag(&hash, all.data(), sizeof(uint64_t), user) != 0)
        return fail(CMN_ERR_BOOTSTRAP, "allgather callback failed");
    for (int r = 0; r < world; ++r)
        if (all[r] != hash) return fail(CMN_ERR_MISMATCH, "ranks registered different model structures");
    return CMN_OK;
}

}  // extern "C"
