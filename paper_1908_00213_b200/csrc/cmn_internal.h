// cmn_internal.h -- types shared by the host runtime (cmn_comm.h and its .cpp files) and
// the sm_100a kernels (cmn_kernels.cu).  Not part of the public ABI.
#pragma once

#include <cstddef>
#include <cstdint>

#include <cuda_runtime.h>

namespace cmn {

constexpr int kMaxWorld = 8;          // == CMN_MAX_WORLD
constexpr int kAlign = 64;            // == CMN_ALIGN_ELEMS
#ifndef CMN_THREADS
#define CMN_THREADS 256
#endif
#ifndef CMN_ITEM_ELEMS
#define CMN_ITEM_ELEMS 4096
#endif
constexpr int kThreads = CMN_THREADS;       // threads per CTA, every kernel
constexpr int kItemElems = CMN_ITEM_ELEMS;  // elements per work item (tensor-indexed kernels)
constexpr int kMaxBarrierBlocks = 1024;
constexpr int kBarrierSlots = 2;      // 0: start (inputs ready), 1: mid (reduce-scatter done)
constexpr int kGradCap = 256;         // grad pointers carried per launch (kernel params)
// Barrier flag value = (per-CTA epoch << kTagBits) | call tag.  The tag
// (make_barrier): payload dtype (bit 0), kernel kind (bits 1-3) and a 4-bit
// hash of the packed element range (bits 4-7), so a peer that issued a
// different collective -- another dtype, algorithm or piece -- at the same
// epoch is reported as CMN_ERR_MISMATCH instead of being paired with it.
constexpr uint32_t kTagBits = 8;
constexpr uint32_t kTagMask = (1u << kTagBits) - 1u;
// Poison tag a failed rank posts instead of a call tag (kind bits 7: no real
// kernel kind), so waiting peers fail at once instead of timing out.
constexpr uint32_t kDeadTag = 0xFFu;

// One registered tensor (device-resident table built at registration).
struct TensorDesc {
    float *w;          // parameters (caller-owned)
    float *mom;        // momentum-SGD state v (library-owned)
    float *adam_m;     // Adam first moment (library-owned, lazily allocated)
    float *adam_v;     // Adam second moment
    int64_t n;         // numel
    int64_t off;       // packed offset (elements, multiple of kAlign)
    int64_t off_next;  // off of tensor t+1 (= end of this tensor's pad)
};

// A contiguous piece of one tensor: elements [k0, k0 + len) of tensor t,
// packed at [base, base + len) (base = off_t + k0).  len <= kItemElems, k0 is
// a multiple of kItemElems; pad > 0 only on a tensor's last item: the number
// of alignment-pad elements that follow it in the packed layout.
struct Item {
    int32_t t;
    int32_t len;
    int64_t k0;
    int64_t base;
    int32_t pad;
    int32_t reserved;   // sharded-update item lists: owner rank of the chunk
};

// Grad pointers for the tensors [t_lo, t_lo + kGradCap) of one launch.
struct GradTab {
    const float *p[kGradCap];
};

// Cross-rank signalling for the P2P all-reduce.  flags[r] points at rank r's
// signal pad (IPC-mapped for peers); pad layout:
//   uint32 [kBarrierSlots][kMaxBarrierBlocks][kMaxWorld]
// The value CTA b signals in a call is ((epoch[b] + 1) << kTagBits) | tag, where
// epoch[b] is a per-CTA call counter in the rank's own device memory that
// the kernel itself advances -- nothing call-specific is a kernel argument,
// so a captured CUDA graph replays with fresh values.  Every rank issues the
// same collectives with the same grids, so epoch[b] agrees across ranks.
struct Barrier {
    uint32_t *flags[kMaxWorld];
    uint32_t *epoch;    // kMaxBarrierBlocks per-CTA counters (own memory)
    int rank;
    int enabled;        // 0 in simulated mode: stream order replaces barriers
    uint32_t tag;       // kTagBits bits (dtype, kernel kind, range hash); a
                        // same-epoch different-tag peer is a call-sequence mismatch
    uint64_t timeout_ns;
    int *err;           // host-mapped error word: 0 ok, 1 timeout, 2 mismatch, 3 peer failed
    int *derr;          // the same code in device memory, read by every later
                        // kernel of the communicator (comm_failed) to skip its stores
    uint32_t test_delay_ns;   // fault injection (tests only, CMN_TEST_ONESHOT_DELAY_US):
                              // one-shot / two-shot CTAs stall this long after the start barrier
    // Emulated world (cmn_init_emulated): one COOPERATIVE launch plays every
    // rank -- CTA b of rank r is blockIdx.x = r * emul_g + b, all co-resident
    // by construction -- so the cross-rank barrier runs for real on one GPU
    // without separate launches that wait on one another.  0 = off.
    int emul_g;
    uint32_t *epochs[kMaxWorld];   // emulation: every rank's per-CTA epoch counters
    int test_absent_rank;     // emulation fault injection: this rank's CTAs never arrive (-1: none)
    int test_mismatch_rank;   // emulation fault injection: this rank posts another call tag (-1: none)
    int test_slow_rank;       // emulation: only this rank's blocks take test_delay_ns (-1: every block)
    int test_skip_mid;        // emulation negative control: two-shot skips its mid barrier
};

// Peer buffer table (packed or reduced) in 16-byte units.
struct PeerBufs {
    const void *p[kMaxWorld];
};

// ---------------------------------------------------------------- launchers
// All return cudaGetLastError() after the launch.  `dtype` 0 = fp32, 1 = fp16.

// a1: pack items [i0, i1) (tensors of those items lie in [t_lo, t_lo + ntab),
// ntab <= kGradCap: the table's used entries; small tables launch smaller).
// max_ctas > 0 caps the grid (CTAs then stride over the items; results do
// not depend on it) -- cmn_set_stream_ctas, for sharing SMs with compute.
cudaError_t launch_pack(const GradTab &g, int ntab, int t_lo, const TensorDesc *td,
                        const Item *items, int i0, int i1, int dtype, void *packed, cudaStream_t s,
                        int max_ctas = 0);

// a3: update from a reduced packed buffer (payload dtype), momentum SGD.
// derr: the communicator's device error word (NULL = unchecked); when set
// (an earlier collective failed) the kernel leaves w and v untouched.
cudaError_t launch_update_sgd(const TensorDesc *td, const Item *items, int i0, int i1,
                              const void *reduced, int dtype, float n_rep, float lr, float mu,
                              const int *derr, cudaStream_t s, int max_ctas = 0);

// a1'+a3 at N = 1: read g directly (cast through fp16 if dtype == 1).
// wt: the parameter pointers of the same tensors; mom: momentum base (tensor
// t at off_t, so element (t, k) at mom + off_t + k).
cudaError_t launch_update_direct(const GradTab &g, const GradTab &wt, int ntab, int t_lo,
                                 float *mom, const Item *items, int i0, int i1, int dtype, float lr,
                                 float mu, cudaStream_t s);

// write a = r / n_rep into out tensors (test hook / Chainer semantics).
cudaError_t launch_unpack_avg(const GradTab &out, int t_lo, const TensorDesc *td,
                              const Item *items, int i0, int i1, const void *reduced, int dtype,
                              float n_rep, const int *derr, cudaStream_t s);

// NEXT-1 Adam.
cudaError_t launch_update_adam(const TensorDesc *td, const Item *items, int i0, int i1,
                               const void *reduced, int dtype, float n_rep, float alpha_t,
                               float beta1, float beta2, float c1, float c2, float eps,
                               const int *derr, cudaStream_t s, int max_ctas = 0);

// NEXT-1 at N = 1: Adam straight from the gradients (no pack); m, v at
// adam_m / adam_v + packed index; programmatic dependent launch.
cudaError_t launch_adam_direct(const GradTab &g, const GradTab &wt, int ntab, int t_lo,
                               float *adam_m, float *adam_v, const Item *items, int i0, int i1,
                               int dtype, float alpha_t, float beta1, float beta2, float c1,
                               float c2, float eps, cudaStream_t s);

// a2 one-shot: out[j] = tree_i(in_i[j]) for j in [e0, e1) (elements; e0, e1
// multiples of kAlign).  Barrier slot 0 at entry when enabled; with
// end_barrier also slot 1 at exit (every peer finished reading `in`).
// Emulated world (bar.enabled, emulate = true): ONE cooperative launch of
// world x G CTAs plays every rank (G = min(blocks, co-resident capacity /
// world)), rank r writing outs.p[r]; `out` is then unused.
cudaError_t launch_allreduce_oneshot(const PeerBufs &in, int world, void *out, int64_t e0,
                                     int64_t e1, int dtype, bool end_barrier, const Barrier &bar,
                                     int blocks, cudaStream_t s, bool emulate = false,
                                     const PeerBufs *outs = nullptr);

// a2 two-shot.  phase bit 1: reduce-scatter of rank `rank`'s chunk from all
// `in` buffers into red[rank]; phase bit 2: all-gather of every other
// rank's chunk from red[p] into red[rank].  With the barrier enabled and
// both phases: start barrier, RS, mid barrier, AG in one kernel.
// chunk_start/chunk_end give every rank's element range (within [e0, e1)).
// emulate = true: one cooperative launch plays every rank (`rank` unused;
// phases 3, or 1 for the fused / sharded schedules' reduce-scatter).
// inbox_slot_elems > 0 (emulated push form, phases 1): rank r reduces its
// own inbox, slot i at in.p[r] + i * inbox_slot_elems payload elements.
cudaError_t launch_allreduce_twoshot(const PeerBufs &in, const PeerBufs &red, int world, int rank,
                                     const int64_t *chunk_start, const int64_t *chunk_end,
                                     int dtype, int phases, const Barrier &bar, int blocks,
                                     cudaStream_t s, bool emulate = false, int64_t inbox_slot_elems = 0);

// NEXT-4 sharded update: momentum SGD on the items of the own chunk, also
// writing w' into the fp32 exchange buffer (packed layout).
cudaError_t launch_update_chunk(const TensorDesc *td, const Item *items, int i0, int i1,
                                const void *reduced, int dtype, float *exch, float n_rep, float lr,
                                float mu, const int *derr, cudaStream_t s);

// NEXT-4 all-gather of parameters: start barrier, then copy items [i0, i1)
// minus [s0, s1) from the owner's exchange buffer (Item.reserved = owner).
// emulate = true: one cooperative launch over every rank (barrier live), the
// whole grid striding over the items of the shared replica.
cudaError_t launch_gather_params(const TensorDesc *td, const Item *items, int i0, int i1, int s0,
                                 int s1, const PeerBufs &exch, int world, const Barrier &bar,
                                 int blocks, cudaStream_t s, bool emulate = false);

// Fused all-gather + update: start barrier, then momentum SGD over the
// chunk-clipped items [i0, i1) reading r from red.p[Item.reserved].
// emulate = true: as launch_gather_params.
cudaError_t launch_update_gather(const TensorDesc *td, const Item *items, int i0, int i1,
                                 const PeerBufs &red, int world, int dtype, float n_rep, float lr,
                                 float mu, const Barrier &bar, int blocks, cudaStream_t s,
                                 bool emulate = false);

// Fused pack + reduce-scatter transfer (push): start barrier, then cast and
// store the elements of the chunk-clipped items [i0, i1) (Item.reserved =
// owner; all tensors in [t_lo, t_lo + kGradCap)) to dst.p[owner] + base.
// emulate = true: one cooperative launch over every rank: rank r's gradient
// of tensor t at g.p[r * tstride + t - t_lo], its slot in owner o's inbox at
// dst.p[o] + r * slot_bytes (dst = rank 0's view).
cudaError_t launch_pack_push(const GradTab &g, int t_lo, const Item *items, int i0, int i1,
                             const PeerBufs &dst, int world, int dtype, const Barrier &bar,
                             int blocks, cudaStream_t s, bool emulate = false, int tstride = 0,
                             int64_t slot_bytes = 0);

// NEXT-3 NVLS: this rank's chunk [e0, e1) (elements) reduced in the switch
// from the multicast packed buffer and multicast-stored into every rank's
// reduced buffer; start and end cross-rank barriers.
cudaError_t launch_nvls_allreduce(const void *mc_packed, void *mc_reduced, int64_t e0, int64_t e1,
                                  int world, int dtype, const Barrier &bar, int blocks,
                                  cudaStream_t s);

// test hook: p[0, n) = pattern (cmn_debug_fill_buffers)
cudaError_t launch_fill_u32(uint32_t *p, size_t n, uint32_t pattern, cudaStream_t s);

int num_sms(int device);

}  // namespace cmn
