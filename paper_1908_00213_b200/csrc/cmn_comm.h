// cmn_comm.h -- the communicator object behind include/cmn.h and the host
// runtime's internal helpers, shared by
//   cmn_core.cpp       errors, layout, buffers, CUDA-IPC peer mapping,
//                      validation, grid sizes
//   cmn_schedules.cpp  the step schedules: pack / all-reduce / update
//                      phases, pipelined, fused (pull / push), sharded,
//                      host-buffer pieces
//   cmn_api.cpp        the extern "C" entry points
// Not part of the ABI.
//
// Paper passages: the communicator, the
// multi_node_optimizer wrapping, the all-reduce step
// (PAPER.md:449-454), fp16 payload, overlap
// (PAPER.md:788-792).  Readings R1-R17 are listed in DESIGN.md §3.
#pragma once

#include "../../include/cmn.h"

#include <cstdint>
#include <cstdlib>
#include <string>
#include <utility>
#include <vector>

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include "cmn_internal.h"
#include "cmn_nvls.h"

using namespace cmn;

#define CMN_CUDA(call)                                          \
    do {                                                        \
        cudaError_t e_ = (call);                                \
        if (e_ != cudaSuccess) return cmn::rt::cuda_fail(e_, #call); \
    } while (0)

namespace cmn::rt {

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
    bool load();   // dlopen libnccl (CMN_NCCL_LIB, libnccl.so.2, libnccl.so)
};
extern NcclApi g_nccl;
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

}  // namespace cmn::rt

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
    // cmn_init_emulated: a simulated world (every rank's buffers in this
    // process) whose one-shot / two-shot all-reduces run as ONE cooperative
    // launch over all ranks with the cross-rank barriers live
    bool emulated = false;
    int test_absent_rank = -1;     // CMN_TEST_EMUL_ABSENT_RANK (emulation fault injection)
    int test_mismatch_rank = -1;   // CMN_TEST_EMUL_MISMATCH_RANK
    int test_slow_rank = -1;       // CMN_TEST_EMUL_SLOW_RANK (with CMN_TEST_ONESHOT_DELAY_US)
    int test_skip_mid = 0;         // CMN_TEST_EMUL_SKIP_MID (negative control)
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
    float *d_pstage = nullptr;    // N = 1 e2e: params packed for one D2H per piece, L floats
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
    int stream_ctas = 0;          // cmn_set_stream_ctas: cap on pack/update grids (0 = none)
    int *h_err = nullptr, *d_err = nullptr;   // host-mapped error word (host view, device view)
    int *d_errdev = nullptr;      // the same code in device memory: later kernels skip their stores
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
    // fault injection, tests only: CMN_TEST_ONESHOT_DELAY_US stalls this
    // rank's one-shot CTAs after their start barrier; CMN_TEST_NO_END_BARRIER=1
    // drops the pipelined step's one-shot end barrier (negative control)
    uint32_t test_delay_ns = 0;
    bool test_no_end_barrier = false;
    int fused_update = 0;         // N > 1 cmn_step: RS + fused all-gather/update (1 pull, 2 push)
    Nvls nvls;                    // NEXT-3 multicast resources (CMN_ALGO_NVLS)
    // NEXT-4 sharded update: items clipped to every rank's two-shot chunk
    // (Item.reserved = owner), rank r's list is [sitem_begin[r], sitem_begin[r+1]).
    std::vector<int> sitem_begin;
    Item *d_sitems = nullptr;
    cudaStream_t sc = nullptr;
    std::vector<cudaEvent_t> pev;
};

namespace cmn::rt {

// Bias-corrected Adam constants of one step (NEXT-1): alpha_t evaluated in
// double on the host (reading R17), c1 = 1 - beta1, c2 = 1 - beta2.
struct AdamArgs {
    float alpha_t, beta1, beta2, c1, c2, eps;
};

// Host buffers of the e2e step (cmn_step_host_packed): packed layout, L
// floats per (simulated) rank for the gradients; parameters out or NULL.
struct HostIO {
    const float *grads = nullptr;
    float *params = nullptr;
};

// ---------------------------------------------------------------- errors
extern thread_local std::string g_last_error;
cmn_status fail(cmn_status st, const std::string &msg);
cmn_status cuda_fail(cudaError_t e, const char *what);

// ------------------------------------------------------------- utilities
uint64_t fnv1a(uint64_t h, const void *data, size_t n);
int64_t align_up(int64_t x, int64_t a);
size_t env_size(const char *name, size_t dflt);

// -------------------------------------- communicator state (cmn_core.cpp)
cmn_status check_async_error(cmn_comm *c);
cmn_status launched(cmn_comm *c, cudaError_t e, const char *what);
void free_regions(cmn_comm *c);
void free_registration(cmn_comm *c);
int64_t buf_elems(int64_t L);
void carve(RankBufs &b, char *base, int64_t L);
size_t flags_bytes();
cmn_status plan_layout_impl(int T, const int *ndims, const int64_t *dims,
                            std::vector<int64_t> &numel, std::vector<int64_t> &off,
                            uint64_t &hash);
bool allgather(cmn_comm *c, const void *send, void *recv, size_t bytes);
cmn_status alloc_regions(cmn_comm *c);
cmn_status exchange_and_map(cmn_comm *c);
int ar_blocks_for(const cmn_comm *c);
int upd_blocks_for(const cmn_comm *c, int items);
bool grads_ok(const cmn_comm *c, const float *const *g, int count, std::string &why);
GradTab make_tab(const float *const *g, int lo, int hi);
// Kernel kinds in the barrier call tag (a peer in another kind of collective
// at the same epoch is a call-sequence mismatch).
enum BarrierKind : int {
    kBarOneshot = 0, kBarTwoshot = 1, kBarNvls = 2, kBarUpdateGather = 3,
    kBarGatherParams = 4, kBarPackPush = 5
};
Barrier make_barrier(cmn_comm *c, int dtype, BarrierKind kind, int64_t e0 = 0, int64_t e1 = 0);
cmn_algo choose_algo(const cmn_comm *c, size_t bytes);
void chunk_plan(int64_t e0, int64_t e1, int world, int64_t *s, int64_t *e);
cmn_status require_registered(const cmn_comm *c);
cmn_status require_dtype(int dtype);
cmn_status set_device(const cmn_comm *c);
cmn_status init_common(int rank, int world, int dev, bool sim, cmn_allgather_fn ag, void *user,
                       cmn_comm **out);
cmn_status copy_tensors(cmn_comm *c, const float *const *src, float *const *dst, int ta, int tb,
                        cudaMemcpyKind kind, cudaStream_t s);
bool params_are_flat(const cmn_comm *c);
cmn_status ensure_staging(cmn_comm *c);
cmn_status ensure_pstage(cmn_comm *c, cudaStream_t s);
cmn_status ensure_side_streams(cmn_comm *c);

// ------------------------------------------ step schedules (cmn_schedules.cpp)
cmn_status pack_phase(cmn_comm *c, int ta, int tb, const float *const *grads, int dtype, int par,
                      cudaStream_t s, void *dst_override = nullptr);
cmn_status reduce_phase(cmn_comm *c, int ta, int tb, int dtype, uint32_t seq, cmn_algo algo,
                        cudaStream_t s, bool end_barrier = false);
cmn_status begin_collective(cmn_comm *c, int ta, int tb, int dtype, cmn_algo &algo,
                            cudaStream_t s, bool graph_safe);
cmn_status allreduce_range(cmn_comm *c, int ta, int tb, const float *const *grads, int dtype,
                           cudaStream_t s);
const void *reduced_ptr(const cmn_comm *c, const ArResult &res, int rank);
cmn_status update_range(cmn_comm *c, int ta, int tb, const ArResult &res, float lr, float mu,
                        cudaStream_t s);
std::vector<std::pair<int, int>> e2e_item_pieces(const cmn_comm *c);
std::vector<std::pair<int, int>> equal_ranges(const cmn_comm *c, int n);
cmn_status ensure_comm_stream(cmn_comm *c, size_t n_events);
cmn_status d2h_params(cmn_comm *c, int ta, int tb, float *host_params, cudaStream_t s);
cmn_status step_pipelined(cmn_comm *c, const float *const *grads, int dtype, float lr, float mu,
                          cudaStream_t s, const HostIO *io = nullptr,
                          const AdamArgs *adam = nullptr);
cmn_status ensure_adam(cmn_comm *c);
AdamArgs adam_args(float alpha, float beta1, float beta2, float eps, int step);
cmn_status update_range_adam(cmn_comm *c, int ta, int tb, const ArResult &res, const AdamArgs &a,
                             cudaStream_t s);
cmn_status step_sharded(cmn_comm *c, const float *const *grads, int dtype, float lr, float mu,
                        cudaStream_t s);
cmn_status step_fused(cmn_comm *c, const float *const *grads, int dtype, float lr, float mu,
                      cudaStream_t s);

// NVTX range over one phase's host-side enqueue (SURVEY §5 tracing): names
// "cmn.pack", "cmn.allreduce", "cmn.update", "cmn.step.*", so nsys / ncu
// --nvtx captures separate the phases.  Header-only NVTX3: without an
// attached tool each push/pop is a null-callback check.
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange &) = delete;
    NvtxRange &operator=(const NvtxRange &) = delete;
};

// ------------------------------------------------------------ templates
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

}  // namespace cmn::rt
