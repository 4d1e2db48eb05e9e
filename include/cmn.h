/*
 * cmn.h -- C ABI of the B200-native ChainerMN data-parallel update step.
 *
 * The operation (arXiv 1908.00213 §6, "Synchronous vs.
 * Asynchronous"): "workers communicate with each other to obtain and
 * distribute the sum of gradients calculated by individual workers. Each
 * worker calculates the average of gradients by dividing the sum by the
 * number of replicas, and updates its own replica of the model".  The
 * communicator abstraction is PAPER.md:475-478 and 506 ("a communicator
 * component that controls all inter-process communication"); the wrapped
 * optimizer is multi_node_optimizer, PAPER.md:510-514 ("wraps the normal
 * optimizer and exchanges the gradient across processes using the all-reduce
 * operation before optimizing the model"); the half-precision payload is
 * PAPER.md:838-839 (App. A.1).
 *
 * One step, per rank r of N:
 *   a1  pack      b_r[off_t + k] = cast(g_t[k])      (cast: fp32 identity or fp16 RNE)
 *   a2  allreduce r[j] = tree_{i<N}(b_i[j])          (pairwise tree in rank order, fp32
 *                                                      accumulation, fp16 rounded once)
 *   a3  update    a = r / N; v = fma(mu, v, a); w = fma(-lr, v, w)   (in place)
 * Layout: off_0 = 0, off_{t+1} = align64(off_t + n_t); pads are zero.
 * Results are bitwise identical on every rank and bitwise equal to the CPU
 * oracle (oracle/cmn_oracle.c) for the hand-written algorithms.
 *
 * Conventions for every entry point:
 *   - Plain C types only.  `stream` is a cudaStream_t passed as void*
 *     (NULL = the legacy default stream).  Every device pointer refers to
 *     memory of the communicator's CUDA device.
 *   - Calls are asynchronous with respect to the host: GPU work is ordered on
 *     `stream`; completion is observed by synchronising the stream.
 *   - Arguments are validated synchronously (CMN_ERR_INVALID_ARG, nothing
 *     enqueued).  CUDA / NCCL failures map to CMN_ERR_CUDA / CMN_ERR_NCCL.
 *     A device-side timeout or call-sequence mismatch detected by a kernel
 *     surfaces as CMN_ERR_TIMEOUT / CMN_ERR_MISMATCH on the NEXT call on that
 *     communicator (or from cmn_poll_error).  The failed call itself leaves
 *     the parameters, the momentum / Adam state and its other outputs
 *     untouched: the detecting kernel and every later kernel of the
 *     communicator skip their stores (device error word).  One partial case:
 *     a peer slower than the timeout, arriving after some of a kernel's CTAs
 *     gave up -- the CTAs that met it apply their (correct) part.  A failed
 *     communicator stays failed (finalize it) and posts a poison flag in
 *     its later collectives, so its peers fail at once with CMN_ERR_TIMEOUT
 *     ("a peer rank's communicator failed") instead of waiting out the
 *     timeout.  Call-sequence mismatches are
 *     detected by a per-call tag (payload dtype, kernel kind, packed range);
 *     a rank skipping a WHOLE step pairs its next step with the peers' current
 *     one undetected and the last call then times out.  cmn_last_error()
 *     returns a thread-local text for the last non-OK status.
 *   - Handles are not thread-safe; one thread drives one communicator.
 *   - Every rank must issue the same sequence of collective calls
 *     (cmn_register_params, cmn_allreduce_*, cmn_step*) with the same layout
 *     and dtype ("model structures are
 *     identical between workers merely in a single iteration"), and a
 *     rank's collective calls must be ordered on the GPU: issue them on one
 *     stream, or join the streams with events between calls (their kernels
 *     advance shared per-CTA barrier epochs; two collectives of one
 *     communicator running concurrently on unjoined streams is undefined).
 *   - CUDA graphs: barrier values live in device-resident per-CTA epoch
 *     counters, so collectives replay correctly from a captured graph.  The
 *     schedules whose buffer reuse does not rely on host-chosen alternation
 *     -- cmn_step with cmn_set_pipeline >= 2 (the default) and
 *     cmn_step_sharded, cmn_set_fused_update on -- may be captured; the
 *     single-call schedules
 *     (cmn_allreduce_grads, buckets, unpipelined cmn_step) return
 *     CMN_ERR_UNSUPPORTED under capture instead of racing.  N == 1 and
 *     simulated communicators may always be captured.
 *   - There is no CPU fallback: if the CUDA device or the sm_100a kernels are
 *     unavailable every compute entry point fails with CMN_ERR_CUDA.
 */
#ifndef CMN_H
#define CMN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CMN_VERSION 1
#define CMN_ALIGN_ELEMS 64      /* packed-layout alignment (elements)          */
#define CMN_MAX_WORLD 8         /* ranks per communicator (one NVSwitch node)  */

typedef struct cmn_comm cmn_comm;   /* opaque, one per process/rank, library-owned */

typedef enum {
    CMN_OK = 0,
    CMN_ERR_INVALID_ARG = 1,  /* null / misaligned pointer, bad count, bad dtype     */
    CMN_ERR_CUDA = 2,         /* CUDA runtime error, or no usable sm_100 device      */
    CMN_ERR_NCCL = 3,         /* NCCL comparison path error (or libnccl missing)     */
    CMN_ERR_BOOTSTRAP = 4,    /* the caller's allgather callback failed              */
    CMN_ERR_MISMATCH = 5,     /* ranks disagree on layout / call sequence / dtype    */
    CMN_ERR_TIMEOUT = 6,      /* a device spin-wait on a peer exceeded the timeout   */
    CMN_ERR_STATE = 7,        /* call out of order (e.g. update without allreduce)   */
    CMN_ERR_OOM = 8,          /* device allocation failed                            */
    CMN_ERR_UNSUPPORTED = 9   /* valid request this build cannot serve               */
} cmn_status;

/* Communication (payload) dtype.  Gradients, parameters and optimizer state
 * are always fp32 ("Computations were generally performed in
 * single precision"); CMN_FP16 is the paper's compression. */
typedef enum { CMN_FP32 = 0, CMN_FP16 = 1 } cmn_dtype;

/* All-reduce algorithm for N >= 2 (step a2).
 *   ONESHOT  every rank reads all N packed buffers over NVLink and reduces
 *            the whole buffer locally (one barrier; latency-optimal).
 *   TWOSHOT  reduce-scatter (rank r tree-reduces chunk r from all N buffers)
 *            then all-gather (bandwidth-optimal, 2(N-1)/N * S per GPU).
 *   NCCL     ncclAllReduce(sum) over NVLink -- the measured comparison
 *            ("We adopted NCCL ... as a primary library");
 *            NCCL's summation order is its own, so results match the oracle
 *            within the tolerance gate, not bitwise.
 *   NVLS     NEXT-3, NVLink SHARP: rank r reduces chunk r inside the
 *            NVSwitch (multimem.ld_reduce on a multicast object spanning every
 *            rank's packed buffer) and multicast-stores the sum into every
 *            rank's reduced buffer (multimem.st): (N+1)/N S bytes per rank and
 *            direction (the switch reads each rank's copy of every chunk once
 *            and fans each sum out once) instead of 2(N-1)/N S; the NVLink
 *            time falls by ~1.6x at N = 8.  The switch's summation order is
 *            its own: tolerance-gate parity, not bitwise, for N > 1.  Selecting
 *            it (after registration, on every rank) creates the multicast
 *            resources; needs an NVSwitch system (CMN_ERR_UNSUPPORTED
 *            otherwise).  Also runs at N = 1 (the switch "reduces" one copy).
 *   AUTO     ONESHOT when payload bytes <= oneshot_max_bytes or N == 2,
 *            else TWOSHOT. */
typedef enum {
    CMN_ALGO_AUTO = 0,
    CMN_ALGO_ONESHOT = 1,
    CMN_ALGO_TWOSHOT = 2,
    CMN_ALGO_NCCL = 3,
    CMN_ALGO_NVLS = 4
} cmn_algo;

/* Bootstrap allgather supplied by the caller (the Python binding uses
 * torch.distributed on a CPU/gloo group).  Gathers `bytes` bytes from every
 * rank into recv (world_size * bytes, rank-major).  Returns 0 on success. */
typedef int (*cmn_allgather_fn)(const void *send, void *recv, size_t bytes, void *user);

/* ------------------------------------------------------------------------
 * Communicator lifecycle
 * ------------------------------------------------------------------------ */

/* cmn_init -- create rank `rank` of a `world_size`-rank communicator on
 * CUDA device `cuda_device` (Fig. 4 create_communicator).
 * Allocates the library-owned, IPC-exported communication buffers lazily at
 * register time, exchanges CUDA IPC handles through `ag`, and maps every
 * peer.  world_size == 1 needs no allgather (ag may be NULL).
 * Errors: INVALID_ARG (rank/world out of range, world > CMN_MAX_WORLD,
 * ag NULL with world > 1), CUDA (device missing / not sm_100), BOOTSTRAP. */
cmn_status cmn_init(int rank, int world_size, int cuda_device,
                    cmn_allgather_fn ag, void *user, cmn_comm **out);

/* cmn_init_simulated -- one process plays all `world_size` ranks on one
 * device (test and single-GPU measurement mode).  Each simulated rank owns
 * its own packed and reduced buffers; the all-reduce kernels are the same
 * code as in cmn_init mode, reading the other ranks' buffers through the
 * same peer-pointer table, launched once per simulated rank, with the
 * cross-rank barriers compiled in but disabled (stream order replaces them).
 * Parameters and optimizer state are one replica (ranks are identical by
 * construction; cmn_copy_reduced exposes every rank's reduced buffer). */
cmn_status cmn_init_simulated(int world_size, int cuda_device, cmn_comm **out);

/* cmn_init_emulated -- a simulated world (as cmn_init_simulated: one process,
 * every rank's buffers, rank-major grads) whose one-shot and two-shot
 * all-reduces run as ONE cooperative launch over
 * all ranks -- CTA b of rank r is block r * G + b, every block co-resident
 * -- with the cross-rank barriers LIVE: the same flag pads, per-rank per-CTA
 * epochs, call tags, timeouts and poison flags as cmn_init mode, exercised
 * on one GPU without separate launches that wait on one another.  G is the
 * collective grid (cmn_set_ctas) capped at the co-resident capacity / N.
 * The fused pull step's reduce-scatter and all-gather + update and the
 * sharded step's reduce-scatter and parameter all-gather run the same way
 * (their blocks of every rank striding together over the one shared
 * replica's items), and so does the push form while N * n_tensors <= 256
 * (one launch's gradient-pointer table); NVLS and NCCL behave as in
 * cmn_init_simulated.  Test mode; fault injection through the environment:
 * CMN_TEST_EMUL_ABSENT_RANK=r (rank r's blocks never arrive: the others time
 * out), CMN_TEST_EMUL_MISMATCH_RANK=r (rank r posts another call tag),
 * CMN_TEST_EMUL_SLOW_RANK=r with CMN_TEST_ONESHOT_DELAY_US=t (rank r's blocks
 * stall t us after the start barrier), CMN_TEST_EMUL_SKIP_MID=1 (negative
 * control: the two-shot skips its mid barrier).
 * Errors: as cmn_init_simulated. */
cmn_status cmn_init_emulated(int world_size, int cuda_device, cmn_comm **out);

/* cmn_finalize -- synchronise the device, unmap peers, free everything the
 * library owns.  NULL is a no-op.  With world_size > 1 peers read this
 * rank's exported buffers during collectives, so call it only after every
 * rank has finished its last collective (e.g. after a host barrier);
 * re-registration performs that barrier itself. */
cmn_status cmn_finalize(cmn_comm *comm);

/* ------------------------------------------------------------------------
 * Registration (step a0): model structure -> packed layout
 * ------------------------------------------------------------------------ */

/* cmn_register_params -- register the model's parameter tensors in
 * traversal order ("collected easily by traversing it").
 *   n_tensors  T >= 1
 *   ndims      T entries, 0 <= ndims[t] <= 8
 *   dims       concatenated shapes (sum ndims entries); numel = product
 *              (1 for ndims == 0); tensors with numel 0 are allowed
 *   params     T device pointers to contiguous fp32 parameters, each 16-byte
 *              aligned, caller-owned; they must stay valid and unmoved until
 *              finalize or re-registration.
 * Computes the packed layout (off_t aligned to CMN_ALIGN_ELEMS elements),
 * allocates and zeroes the momentum buffers (library-owned), and the
 * communication buffers.  With world_size > 1 the layout hash is allgathered
 * and every rank returns CMN_ERR_MISMATCH if any rank differs (PAPER.md:495
 * "only assuming that the model structures are identical between workers
 * merely in a single iteration").  May be called again whenever the model
 * structure changes; that resets the momentum state.
 * Synchronous w.r.t. the host (allocations). */
cmn_status cmn_register_params(cmn_comm *comm, int n_tensors, const int *ndims,
                               const int64_t *dims, float *const *params);

/* cmn_get_layout -- offsets (n_tensors + 1 entries, element units) and the
 * padded packed length L = offsets[T].  Either output may be NULL. */
cmn_status cmn_get_layout(const cmn_comm *comm, int64_t *offsets, int64_t *padded_len);

/* ------------------------------------------------------------------------
 * The step (a1-a3)
 * ------------------------------------------------------------------------ */

/* cmn_allreduce_grads -- steps a1 + a2.
 *   grads  device fp32 gradient pointers, read-only, contiguous, 16-byte
 *          aligned, in registration order: n_tensors entries
 *          (cmn_init mode) or world_size * n_tensors entries, rank-major
 *          (cmn_init_simulated mode: rank i's tensor t is grads[i*T + t]).
 *   dtype  payload dtype (CMN_FP32 / CMN_FP16).
 * Grads are not modified.  Leaves the reduced sum r (payload dtype, packed
 * layout) in library memory for cmn_update_momentum_sgd / cmn_update_adam /
 * cmn_unpack_avg_grads.  N == 1 is the identity (fp16 rounding still applies).
 * Errors: INVALID_ARG, STATE (no registration), CUDA, NCCL, TIMEOUT,
 * MISMATCH. */
cmn_status cmn_allreduce_grads(cmn_comm *comm, const float *const *grads,
                               cmn_dtype dtype, void *stream);

/* cmn_update_momentum_sgd -- step a3 on every registered tensor, in place:
 *   a = r[off_t+k] / N (one IEEE division, "dividing the sum by the number of
 *   replicas");  v = fmaf(mu, v, a);  w = fmaf(-lr, v, w).
 * Consumes the reduced buffer of the last allreduce; calling it twice, or
 * before any allreduce, returns CMN_ERR_STATE. */
cmn_status cmn_update_momentum_sgd(cmn_comm *comm, float lr, float mu, void *stream);

/* cmn_step -- a1 + a2 + a3 in one call (the hot path timed by bench.py).
 * At N == 1 the pack is skipped: one fused kernel reads g, w, v and writes
 * w, v (20 B/param), bitwise equal to the unfused path.  grads as in
 * cmn_allreduce_grads. */
cmn_status cmn_step(cmn_comm *comm, const float *const *grads, cmn_dtype dtype,
                    float lr, float mu, void *stream);

/* cmn_step_sharded -- NEXT-4: a1 + reduce-scatter + a3 on the own chunk only
 * + all-gather of the updated PARAMETERS (instead of the reduced gradients).
 * Rank r owns the two-shot chunk r (cmn_plan_chunks); it runs the update
 * (1/N of the replicated update's HBM traffic) and publishes w' in fp32;
 * peers copy it over NVLink.  w is bitwise equal to cmn_step's on every
 * rank; the momentum state becomes sharded: after this call tensor t's
 * momentum (cmn_get_momentum) is current only on the elements the calling
 * rank owns.  Do not mix with cmn_step on the same communicator unless the
 * momentum is re-synchronised.  N == 1 is cmn_step.  grads as in
 * cmn_allreduce_grads. */
cmn_status cmn_step_sharded(cmn_comm *comm, const float *const *grads, cmn_dtype dtype,
                            float lr, float mu, void *stream);

/* cmn_step_host -- cmn_step with HOST buffers (end-to-end measurement):
 *   host_grads    n_tensors (or world*n_tensors, simulated) host fp32 pointers;
 *                 pinned memory gives asynchronous copies
 *   host_params   NULL, or n_tensors host fp32 pointers that receive the
 *                 updated parameters
 * Copies the gradients host->device into library-owned staging, runs
 * cmn_step, copies the parameters device->host, all on `stream`. */
cmn_status cmn_step_host(cmn_comm *comm, const float *const *host_grads,
                         float *const *host_params, cmn_dtype dtype,
                         float lr, float mu, void *stream);

/* cmn_step_host_packed -- cmn_step_host with each side given as ONE host
 * buffer in the packed layout: host_grads holds L floats per (simulated)
 * rank (gradient t at offset off_t, pads ignored), host_params (NULL or L
 * floats) receives the updated parameters at the same offsets.  At N == 1
 * the call pipelines the host->device copy, the update and the
 * device->host copy over 12 ranges of 4096-element work items (sizes ramp
 * up from and down to L/62 so the pipeline's fill and drain are short;
 * env CMN_E2E_PIECES=n selects n equal ranges) on two internal copy
 * streams joined back into `stream`, so the step costs about one
 * full-duplex PCIe transfer instead of two.  If the registered params are
 * views of one allocation in the packed layout, the device->host copies
 * are contiguous (they stop at the last tensor's last element); separate
 * parameter tensors are first packed (fp32, 8 B/param of HBM) into a
 * library-owned device staging buffer of L floats, allocated on first use
 * and freed at re-registration, so each range still leaves in one copy
 * (env CMN_E2E_PER_TENSOR_D2H=1: one copy per tensor instead; measured
 * 3.92 -> 2.44 ms for ResNet-50 at N = 1).  Pad positions of host_params
 * are unspecified. */
cmn_status cmn_step_host_packed(cmn_comm *comm, const float *host_grads, float *host_params,
                                cmn_dtype dtype, float lr, float mu, void *stream);

/* cmn_unpack_avg_grads -- writes the averaged gradient a = r / N
 * back into `out` (n_tensors device fp32 pointers; may alias the grads),
 * which is Chainer's own semantics of "updates its own replica ... with the
 * gradient obtained through the all-reduce".  Does not
 * consume the reduced buffer. */
cmn_status cmn_unpack_avg_grads(cmn_comm *comm, float *const *out, void *stream);

/* cmn_update_adam -- NEXT-1: step a3 with bias-corrected Adam (the optimizer
 * of the paper's own example, Fig. 4), state m, v library-owned
 * and zeroed at registration; `step` >= 1 is the 1-based update count t:
 *   m = b1 m + (1-b1) a;  v = b2 v + (1-b2) a^2;
 *   w = w - alpha_t * m / (sqrt(v) + eps),  alpha_t = alpha sqrt(1-b2^t)/(1-b1^t).
 * Consumes the reduced buffer like cmn_update_momentum_sgd. */
cmn_status cmn_update_adam(cmn_comm *comm, float alpha, float beta1, float beta2,
                           float eps, int step, void *stream);

/* cmn_step_adam -- the whole step (a1-a3) with the Adam update of
 * cmn_update_adam, same arguments as cmn_allreduce_grads for grads/dtype.
 * N == 1: one kernel straight from the gradients (no pack; 28 B/param).
 * N > 1: the pipelined schedule of cmn_step (cmn_set_pipeline >= 2, the
 * default; per-piece Adam updates overlap the all-reduces), else all-reduce
 * then update.  Bitwise identical to cmn_allreduce_grads + cmn_update_adam.
 * Errors as cmn_allreduce_grads; INVALID_ARG for step < 1. */
cmn_status cmn_step_adam(cmn_comm *comm, const float *const *grads, cmn_dtype dtype,
                         float alpha, float beta1, float beta2, float eps, int step,
                         void *stream);

/* ------------------------------------------------------------------------
 * Overlap with backward (a4): contiguous buckets of the layout
 * ------------------------------------------------------------------------ */

/* cmn_plan_buckets -- split the registered tensors into contiguous ranges
 * of at most ~bucket_bytes fp32 gradient bytes each (a tensor is never
 * split), numbered in REVERSE registration order: bucket 0 holds the last
 * tensors, whose gradients backward produces first ("starting
 * all-reduce as soon as the backward computation of a layer is completed").
 * bucket_bytes == 0 means one bucket. */
cmn_status cmn_plan_buckets(cmn_comm *comm, size_t bucket_bytes, int *n_buckets_out);

/* cmn_plan_bucket_ranges -- the same plan, host only, from tensor sizes
 * (numel[n_tensors]); writes the bucket count and, when non-NULL, each
 * bucket's [t_begin[b], t_end[b]) (arrays of >= n_tensors entries, the
 * maximum bucket count).  No communicator or GPU needed. */
cmn_status cmn_plan_bucket_ranges(int n_tensors, const int64_t *numel, size_t bucket_bytes,
                                  int *n_buckets_out, int *t_begin, int *t_end);

/* cmn_get_bucket -- tensor range [t_begin, t_end) of bucket b. */
cmn_status cmn_get_bucket(const cmn_comm *comm, int bucket, int *t_begin, int *t_end);

/* cmn_allreduce_bucket / cmn_update_bucket -- a1+a2 / a3 restricted to the
 * bucket's tensors (grads as in cmn_allreduce_grads, full n_tensors table).
 * Every element is packed, reduced and updated by the same arithmetic as the
 * unbucketed path, so the result is bitwise identical (reading R15). */
cmn_status cmn_allreduce_bucket(cmn_comm *comm, int bucket, const float *const *grads,
                                cmn_dtype dtype, void *stream);
cmn_status cmn_update_bucket(cmn_comm *comm, int bucket, float lr, float mu, void *stream);

/* ------------------------------------------------------------------------
 * Configuration, state access, test hooks
 * ------------------------------------------------------------------------ */

/* cmn_set_algo -- choose the all-reduce algorithm and the AUTO threshold
 * (payload bytes; 0 keeps the default).  Takes effect on the next call. */
cmn_status cmn_set_algo(cmn_comm *comm, cmn_algo algo, size_t oneshot_max_bytes);

/* cmn_set_pipeline -- N > 1 cmn_step schedule: `pieces` >= 2 cuts the model
 * into that many contiguous, equal-byte tensor ranges, each its own
 * collective call; packs and updates run on `stream` while the all-reduces
 * run on an internal high-priority stream, so HBM work overlaps NVLink
 * transfer (results are bitwise identical: every element's arithmetic is
 * unchanged).  0 or 1 = unpipelined (pack, all-reduce, update in sequence).
 * Default 4 (env CMN_PIECES).  Every rank must use the same value. */
cmn_status cmn_set_pipeline(cmn_comm *comm, int pieces);

/* cmn_set_fused_update -- N > 1 cmn_step schedule (takes precedence over
 * the pipeline when on), `mode`:
 *   0  off (default)
 *   1  pack -> reduce-scatter (each owner pulls its chunk of every rank's
 *      packed buffer) -> ONE kernel that updates every parameter reading
 *      each reduced chunk directly from its owner rank over NVLink (no
 *      all-gather copy through local HBM)
 *   2  as 1, but pack and the reduce-scatter transfer are ONE kernel: each
 *      rank casts its gradients and stores them straight into the chunk
 *      owners' inboxes (NVLink stores overlapping the gradient reads; no
 *      local packed buffer); the owner then reduces its inbox locally.
 *      Needs n_tensors <= 256 (one kernel-parameter grad table), else
 *      mode 1 runs.
 * Bitwise identical to the other schedules; graph-capturable.  Every rank
 * must use the same setting.  Other values: CMN_ERR_INVALID_ARG. */
cmn_status cmn_set_fused_update(cmn_comm *comm, int mode);

/* cmn_set_ctas -- grid sizes of the cross-rank kernels (takes effect on the
 * next call; 0 restores the default).  `collective_ctas`: one-shot, two-shot
 * and NVLS all-reduce kernels (default one CTA per SM; two per SM for a
 * simulated communicator).  `update_ctas`: the barrier-gated, item-striding
 * update kernels of the fused and sharded schedules (default 4 per SM).
 * Both at most 1024 (the signal pad's per-CTA cells), else
 * CMN_ERR_INVALID_ARG.  Results do not depend on them.  Collective: every
 * rank must use the same values (CTA b of every rank pairs with CTA b of
 * its peers). */
cmn_status cmn_set_ctas(cmn_comm *comm, int collective_ctas, int update_ctas);

/* cmn_set_stream_ctas -- cap on the grid of the stream-local item kernels
 * (pack, update from the reduced buffer, Adam update): 0 (default) launches
 * one CTA per 4096-element work item; max_ctas > 0 launches at most that many
 * CTAs, which stride over the items.  For overlapping the bucketed
 * exchange with a concurrent backward: an uncapped
 * kernel takes every free SM slot and the next GEMM waits for it to drain.
 * Local to this rank (no cross-rank pairing); results do not depend on it.
 * max_ctas < 0 gives CMN_ERR_INVALID_ARG. */
cmn_status cmn_set_stream_ctas(cmn_comm *comm, int max_ctas);

/* cmn_set_kernel_timing -- on: bracket every launch of the step's dominant
 * kernels (the all-reduce kernels -- one-shot / two-shot / NVLS / NCCL --,
 * the reduce-scatter and fused all-gather+update kernels of the fused
 * schedule, the N = 1 direct update) with CUDA events on the stream that
 * launch runs on (internal streams included); launches being captured into
 * a CUDA graph are not timed.  Setting it (on or off) clears the record.
 * cmn_get_kernel_timing -- waits for the recorded launches, returns their
 * summed device time (ms) and count, and clears the record.  Used by
 * bench.py for the roofline of the dominant kernel. */
cmn_status cmn_set_kernel_timing(cmn_comm *comm, int on);
cmn_status cmn_get_kernel_timing(cmn_comm *comm, double *total_ms, int *count);

/* cmn_set_timeout -- device spin-wait timeout in milliseconds (default
 * 30000). */
cmn_status cmn_set_timeout(cmn_comm *comm, uint32_t timeout_ms);

/* cmn_get_momentum -- device pointer of tensor t's momentum buffer
 * (library-owned, fp32, numel(t) elements; read/write for checkpointing). */
cmn_status cmn_get_momentum(cmn_comm *comm, int tensor, float **dev_ptr);

/* cmn_get_adam_state -- device pointers of tensor t's Adam m and v. */
cmn_status cmn_get_adam_state(cmn_comm *comm, int tensor, float **m_ptr, float **v_ptr);

/* cmn_copy_packed / cmn_copy_reduced -- copy rank `rank`'s packed buffer
 * (a1 output) / reduced buffer (a2 output), L elements of the last call's
 * payload dtype, into device memory `dst`.  In cmn_init mode only
 * rank == own rank is accepted. */
cmn_status cmn_copy_packed(cmn_comm *comm, int rank, void *dst, void *stream);
cmn_status cmn_copy_reduced(cmn_comm *comm, int rank, void *dst, void *stream);

/* cmn_debug_fill_buffers -- test hook ("poisoned receive
 * buffers"): fill this rank's library-owned packed and reduced buffers (every
 * simulated / emulated rank's in those modes; both parities, the whole
 * allocation incl. the push-form inbox slack, NOT the signal pad) with the
 * 32-bit `pattern`, stream-ordered on `stream`.  With 0x7FC07FC0 -- a NaN
 * as fp32 and as each fp16 half -- any later read of a location no kernel of
 * the step wrote propagates NaN into the result, so a bit-exact step after
 * the fill proves the step reads only what it wrote.  Discards any
 * unconsumed all-reduce result (a following update returns STATE).
 * Errors: INVALID_ARG (comm NULL), STATE (no registration), CUDA. */
cmn_status cmn_debug_fill_buffers(cmn_comm *comm, uint32_t pattern, void *stream);

/* cmn_poll_error -- non-blocking check of the device error word (timeouts,
 * sequence mismatches) without issuing work. */
cmn_status cmn_poll_error(cmn_comm *comm);

/* cmn_kernel_launches -- number of kernels this communicator has launched
 * since creation (bench.py reports the count inside its timed region). */
uint64_t cmn_kernel_launches(const cmn_comm *comm);

/* cmn_last_error -- thread-local message for the last non-OK status. */
const char *cmn_last_error(void);

/* cmn_version -- CMN_VERSION of the loaded library. */
int cmn_version(void);

/* ------------------------------------------------------------------------
 * Host-only plan helpers (no CUDA; usable on a machine without a GPU)
 * ------------------------------------------------------------------------ */

/* cmn_plan_layout -- the packed layout for the given shapes (same inputs as
 * cmn_register_params minus the pointers): offsets (T+1) and L.  Returns the
 * 64-bit structure hash in *hash_out (may be NULL). */
cmn_status cmn_plan_layout(int n_tensors, const int *ndims, const int64_t *dims,
                           int64_t *offsets, int64_t *padded_len, uint64_t *hash_out);

/* cmn_plan_chunks -- two-shot partition of L elements over N ranks: chunk
 * size c = align64(ceil(L/N)); rank r owns [min(r c, L), min((r+1) c, L)).
 * starts/ends have N entries. */
cmn_status cmn_plan_chunks(int64_t padded_len, int world_size, int64_t *starts, int64_t *ends);

/* cmn_bootstrap_verify -- allgather `hash` through `ag` and return CMN_OK
 * if all ranks agree, CMN_ERR_MISMATCH (on every rank) otherwise.  This is
 * the registration-time structure check, exposed for host-only tests. */
cmn_status cmn_bootstrap_verify(int rank, int world_size, cmn_allgather_fn ag, void *user,
                                uint64_t hash);

/* cmn_share_fd -- the file-descriptor hand-off CMN_ALGO_NVLS uses to give
 * every rank rank 0's multicast-object handle: rank 0 listens on an
 * abstract Unix-domain socket whose name goes through `ag`, every other
 * rank connects and receives `fd_in` via SCM_RIGHTS into *fd_out (rank 0:
 * *fd_out = fd_in).  Host-only; exposed for tests. */
cmn_status cmn_share_fd(int rank, int world_size, cmn_allgather_fn ag, void *user, int fd_in,
                        int *fd_out);

#ifdef __cplusplus
}
#endif
#endif /* CMN_H */
