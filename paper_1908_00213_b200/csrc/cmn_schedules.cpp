// cmn_schedules.cpp -- the data-parallel update step (arXiv 1908.00213 §6.1.2,
// PAPER.md:449-454) as schedules of the sm_100a kernels: pack (a1), all-reduce
// (a2: one-shot / two-shot P2P, NVLS, NCCL), update (a3); the pipelined N > 1
// step, the fused all-gather + update (pull or push reduce-scatter), the
// sharded update (NEXT-4) and the host-buffer pipeline of the e2e step.
#include "cmn_comm.h"

#include <cmath>
#include <cstdlib>
#include <iterator>

namespace cmn::rt {

// a1: pack every (simulated) rank's gradients of tensors [ta, tb) into its
// packed buffer of parity `par`.
cmn_status pack_phase(cmn_comm *c, int ta, int tb, const float *const *grads, int dtype, int par,
                      cudaStream_t s, void *dst_override) {
    NvtxRange nv("cmn.pack");
    const int nsim = c->simulated ? c->world : 1;
    for (int i = 0; i < nsim; ++i) {
        const int r = c->simulated ? i : c->rank;
        const float *const *g = grads + static_cast<size_t>(i) * c->T;
        void *dst = dst_override ? dst_override : c->rb[r].packed[par];
        cmn_status st = for_groups(c, ta, tb, [&](int lo, int hi, int i0, int i1) {
            return launched(c,
                            launch_pack(make_tab(g, lo, hi), hi - lo, lo, c->d_td, c->d_items, i0, i1, dtype,
                                        dst, s, c->stream_ctas),
                            "pack");
        });
        if (st != CMN_OK) return st;
    }
    return CMN_OK;
}

// a2 over the packed range of tensors [ta, tb) for the collective call with
// sequence number `seq` (its buffers have parity seq & 1).
cmn_status reduce_phase_launch(cmn_comm *c, int ta, int tb, int dtype, uint32_t seq, cmn_algo algo,
                               cudaStream_t s, bool end_barrier) {
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
        const Barrier bar = make_barrier(c, dtype, kBarNvls, e0, e1);
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
    Barrier bar = make_barrier(c, dtype, algo == CMN_ALGO_TWOSHOT ? kBarTwoshot : kBarOneshot, e0, e1);
    int64_t cs[kMaxWorld], ce[kMaxWorld];
    chunk_plan(e0, e1, c->world, cs, ce);
    if (c->emulated) {
        // one cooperative launch plays every rank, barriers live
        bar.enabled = 1;
        if (algo == CMN_ALGO_ONESHOT)
            return launched(c,
                            launch_allreduce_oneshot(in, c->world, nullptr, e0, e1, dtype, end_barrier, bar,
                                                     blocks, s, true, &red),
                            "allreduce_oneshot (emulated world)");
        return launched(c,
                        launch_allreduce_twoshot(in, red, c->world, 0, cs, ce, dtype, 3, bar, blocks, s,
                                                 true),
                        "allreduce_twoshot (emulated world)");
    }
    if (algo == CMN_ALGO_ONESHOT) {
        for (int i = 0; i < nsim; ++i) {
            const int r = c->simulated ? i : c->rank;
            cmn_status st = launched(c,
                                     launch_allreduce_oneshot(in, c->world, c->rb[r].reduced[par],
                                                              e0, e1, dtype, end_barrier, bar, blocks, s),
                                     "allreduce_oneshot");
            if (st != CMN_OK) return st;
        }
        return CMN_OK;
    }
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
                        cudaStream_t s, bool end_barrier) {
    if (c->world == 1 && algo != CMN_ALGO_NCCL && algo != CMN_ALGO_NVLS) return CMN_OK;
    NvtxRange nv("cmn.allreduce");
    return timed(c, s, [&] { return reduce_phase_launch(c, ta, tb, dtype, seq, algo, s, end_barrier); });
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
    NvtxRange nv("cmn.update");
    const float n_rep = static_cast<float>(c->world);   // a = r / N (reading R3)
    return for_groups(c, ta, tb, [&](int, int, int i0, int i1) {
        return launched(c,
                        launch_update_sgd(c->d_td, c->d_items, i0, i1, reduced_ptr(c, res, 0),
                                          res.dtype, n_rep, lr, mu, c->d_errdev, s, c->stream_ctas),
                        "update_sgd");
    });
}

// NEXT-1 state: m and v, L floats each in the packed layout, zeroed on
// first use after a registration.
cmn_status ensure_adam(cmn_comm *c) {
    if (c->d_adam) return CMN_OK;
    const size_t b = static_cast<size_t>(c->L > 0 ? c->L : 1) * 4 * 2;
    if (cudaMalloc(&c->d_adam, b) != cudaSuccess) return fail(CMN_ERR_OOM, "adam state alloc");
    CMN_CUDA(cudaMemset(c->d_adam, 0, b));
    for (int t = 0; t < c->T; ++t) {
        c->h_td[t].adam_m = c->d_adam + c->off[t];
        c->h_td[t].adam_v = c->d_adam + c->L + c->off[t];
    }
    CMN_CUDA(cudaMemcpy(c->d_td, c->h_td.data(), sizeof(TensorDesc) * c->T, cudaMemcpyHostToDevice));
    return CMN_OK;
}

// alpha_t = alpha * sqrt(1 - beta2^t) / (1 - beta1^t), evaluated in double.
AdamArgs adam_args(float alpha, float beta1, float beta2, float eps, int step) {
    const double b1t = std::pow(static_cast<double>(beta1), static_cast<double>(step));
    const double b2t = std::pow(static_cast<double>(beta2), static_cast<double>(step));
    const float alpha_t =
        static_cast<float>(static_cast<double>(alpha) * std::sqrt(1.0 - b2t) / (1.0 - b1t));
    return AdamArgs{alpha_t, beta1, beta2, 1.0f - beta1, 1.0f - beta2, eps};
}

cmn_status update_range_adam(cmn_comm *c, int ta, int tb, const ArResult &res, const AdamArgs &a,
                             cudaStream_t s) {
    NvtxRange nv("cmn.update_adam");
    const float n_rep = static_cast<float>(c->world);   // a = r / N (reading R3)
    return for_groups(c, ta, tb, [&](int, int, int i0, int i1) {
        return launched(c,
                        launch_update_adam(c->d_td, c->d_items, i0, i1, reduced_ptr(c, res, 0),
                                           res.dtype, n_rep, a.alpha_t, a.beta1, a.beta2, a.c1,
                                           a.c2, a.eps, c->d_errdev, s, c->stream_ctas),
                        "update_adam");
    });
}

// Item ranges [i0, i1) of the N = 1 host-buffer pipeline (item = 4096
// elements of one tensor, so a tensor may straddle pieces), sized by
// kE2EWeights -- or CMN_E2E_PIECES equal pieces, or CMN_E2E_WEIGHTS="w0,w1,..."
// (measurement switches).
std::vector<std::pair<int, int>> e2e_item_pieces(const cmn_comm *c) {
    const int I = c->item_begin[c->T];
    std::vector<int> wts(std::begin(kE2EWeights), std::end(kE2EWeights));
    if (const size_t n = env_size("CMN_E2E_PIECES", 0); n > 0)
        wts.assign(n < static_cast<size_t>(kE2EMaxPieces) ? n : kE2EMaxPieces, 1);
    if (const char *e = std::getenv("CMN_E2E_WEIGHTS"); e && *e) {
        std::vector<int> w;
        for (const char *q = e; *q && static_cast<int>(w.size()) < kE2EMaxPieces;) {
            char *end = nullptr;
            const long v = std::strtol(q, &end, 10);
            if (end == q) break;
            if (v > 0) w.push_back(static_cast<int>(v));
            q = *end == ',' ? end + 1 : end;
        }
        if (!w.empty()) wts = w;
    }
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

// Device->host copy of the parameters of tensors [ta, tb) into the packed
// host layout: one copy when the params are one flat allocation (stopping
// at the last tensor's end); separate tensors are first packed into the
// staging buffer d_pstage on `s` and leave in one copy as well (per-tensor
// copies with CMN_E2E_PER_TENSOR_D2H=1, measurement switch).
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
    if (tb <= ta) return CMN_OK;
    std::vector<const float *> src(c->params.begin(), c->params.end());
    if (!env_size("CMN_E2E_PER_TENSOR_D2H", 0)) {
        // separate tensors: pack them (fp32, on `s`) into the staging buffer
        // in the packed layout, then ONE copy for the whole range
        if (cmn_status st = ensure_pstage(c, s); st != CMN_OK) return st;
        if (cmn_status st = for_groups(c, ta, tb, [&](int lo, int hi, int i0, int i1) {
                return launched(c,
                                launch_pack(make_tab(src.data(), lo, hi), hi - lo, lo, c->d_td,
                                            c->d_items, i0, i1, CMN_FP32, c->d_pstage, s),
                                "pack_params");
            });
            st != CMN_OK)
            return st;
        int last = tb - 1;
        while (last > ta && c->numel[last] == 0) --last;
        const int64_t e0 = c->off[ta], e1 = c->off[last] + c->numel[last];
        if (e1 > e0)
            CMN_CUDA(cudaMemcpyAsync(host_params + e0, c->d_pstage + e0, static_cast<size_t>(e1 - e0) * 4,
                                     cudaMemcpyDeviceToHost, s));
        return CMN_OK;
    }
    std::vector<float *> hp(c->T);
    for (int t = 0; t < c->T; ++t) hp[t] = host_params + c->off[t];
    return copy_tensors(c, src.data(), hp.data(), ta, tb, cudaMemcpyDeviceToHost, s);
}

// Pipelined a1-a3 for N > 1: the model is cut into P contiguous pieces; each
// piece is one collective call.  Caller stream s: pack(0..P-1), then
// update(p) after all-reduce(p); communication stream: all-reduce(p) after
// pack(p).  HBM-bound packs/updates overlap the NVLink-bound all-reduces.
// Buffer reuse: a piece's next pack (next step, or the next replay of a
// captured step) is issued after update(P-1), i.e. after our all-reduce of
// the last piece passed its start barrier, so every peer finished the
// all-reduces of pieces 0..P-2.  The last piece itself is covered by that
// all-reduce's own end: two-shot's mid barrier (every peer finished its
// reduce-scatter reads of our packed buffer) or NVLS's end barrier, and for
// one-shot -- which reads every packed buffer to the end and has no later
// barrier -- an explicit end barrier on the last piece (slot 1).
// With `io`, the e2e form: H2D(piece p) on a copy stream feeds pack(p), and
// D2H(piece p) on a second copy stream follows update(p), so PCIe in both
// directions overlaps the packs, NVLink all-reduces and updates of the
// other pieces (gradients land in the library's staging buffer, whose
// pointers `grads` are).
cmn_status step_pipelined(cmn_comm *c, const float *const *grads, int dtype, float lr, float mu,
                          cudaStream_t s, const HostIO *io, const AdamArgs *adam) {
    NvtxRange nv("cmn.step.pipelined");
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
                                         c->sc, p + 1 == P && !c->test_no_end_barrier);
            st != CMN_OK)
            return st;
        CMN_CUDA(cudaEventRecord(c->pev[2 * p + 1], c->sc));
    }
    for (size_t p = 0; p < P; ++p) {
        CMN_CUDA(cudaStreamWaitEvent(s, c->pev[2 * p + 1], 0));
        if (cmn_status st = adam ? update_range_adam(c, pieces[p].first, pieces[p].second, res[p],
                                                     *adam, s)
                                 : update_range(c, pieces[p].first, pieces[p].second, res[p], lr, mu, s);
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
    NvtxRange nv("cmn.step.sharded");
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
    Barrier bar = make_barrier(c, dtype, kBarTwoshot, 0, c->L);
    if (c->emulated) {          // one cooperative reduce-scatter over every rank, barrier live
        bar.enabled = 1;
        cmn_status st = launched(c,
                                 launch_allreduce_twoshot(in, red, c->world, 0, cs, ce, dtype, 1, bar,
                                                          blocks, s, true),
                                 "reduce_scatter (emulated world)");
        if (st != CMN_OK) return st;
    }
    for (int i = 0; i < (c->emulated ? 0 : nsim); ++i) {
        const int r = c->simulated ? i : c->rank;
        cmn_status st = launched(c,
                                 launch_allreduce_twoshot(in, red, c->world, r, cs, ce, dtype, 1, bar,
                                                          blocks, s),
                                 "reduce_scatter");
        if (st != CMN_OK) return st;
    }
    const float n_rep = static_cast<float>(c->world);   // a = r / N (reading R3)
    for (int i = 0; i < nsim; ++i) {
        const int r = c->simulated ? i : c->rank;
        cmn_status st = launched(c,
                                 launch_update_chunk(c->d_td, c->d_sitems, c->sitem_begin[r],
                                                     c->sitem_begin[r + 1], c->rb[r].reduced[0], dtype,
                                                     static_cast<float *>(c->rb[r].reduced[1]), n_rep,
                                                     lr, mu, c->d_errdev, s),
                                 "update_chunk");
        if (st != CMN_OK) return st;
    }
    ++c->seq;
    Barrier bar2 = make_barrier(c, dtype, kBarGatherParams);
    const int total = c->sitem_begin[c->world];
    const int gblocks = upd_blocks_for(c, total);
    if (c->emulated) {
        // every rank's blocks in one cooperative grid, barrier live; the
        // shared replica's items are each copied once from their owner's
        // exchange buffer (the owner's own chunk included: the same values)
        bar2.enabled = 1;
        cmn_status st = launched(c,
                                 launch_gather_params(c->d_td, c->d_sitems, 0, total, 0, 0, exch, c->world,
                                                      bar2, gblocks, s, true),
                                 "gather_params (emulated world)");
        if (st != CMN_OK) return st;
        c->fresh = false;
        return CMN_OK;
    }
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
    NvtxRange nv("cmn.step.fused");
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
    const Barrier bar = make_barrier(c, dtype, kBarTwoshot, 0, c->L);
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
    // Emulated world: the barrier kernels as cooperative launches over every
    // rank, barriers live -- the pull form always, the push form while every
    // rank's gradient pointers fit one launch's table (N * T <= kGradCap)
    const bool emul_push = c->emulated && push && c->world * c->T <= kGradCap && cmax > 0;
    const bool emul = c->emulated && (!push || emul_push);
    if (emul_push) {
        Barrier bar0 = make_barrier(c, dtype, kBarPackPush);
        bar0.enabled = 1;
        PeerBufs dst0{};
        for (int o = 0; o < c->world; ++o) dst0.p[o] = inbox_view(o, 0);
        st = timed(c, s, [&] {
            return launched(c,
                            launch_pack_push(make_tab(grads, 0, c->world * c->T), 0, c->d_sitems, 0, total,
                                             dst0, c->world, dtype, bar0, upd_blocks_for(c, total), s, true,
                                             c->T, cmax * static_cast<int64_t>(esz)),
                            "pack_push (emulated world)");
        });
    } else if (push) {
        const Barrier bar0 = make_barrier(c, dtype, kBarPackPush);
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
        if (emul) {
            // pull: every rank's packed buffer; push: every rank reduces its
            // own inbox (rank p's packed[0], slot i at + i * cmax elements)
            PeerBufs in{};
            for (int p = 0; p < c->world; ++p) in.p[p] = push ? c->rb[p].packed[0] : c->rb[p].packed[par];
            Barrier b = bar;
            b.enabled = 1;
            return launched(c,
                            launch_allreduce_twoshot(in, red, c->world, 0, cs, ce, dtype, 1, b, blocks, s,
                                                     true, push ? cmax : 0),
                            "reduce_scatter (emulated world)");
        }
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
    Barrier bar2 = make_barrier(c, dtype, kBarUpdateGather);
    if (emul) bar2.enabled = 1;
    const int gblocks = upd_blocks_for(c, total);
    // simulated ranks share one parameter replica: one launch updates it all
    // (emulated: one cooperative launch whose blocks of every rank stride
    // over the replica's items together, each item once)
    st = timed(c, s, [&] {
        return launched(c,
                        launch_update_gather(c->d_td, c->d_sitems, 0, total, red, c->world, dtype,
                                             static_cast<float>(c->world), lr, mu, bar2,
                                             gblocks, s, emul),
                        emul ? "update_gather (emulated world)" : "update_gather");
    });
    if (st != CMN_OK) return st;
    c->last = ArResult{0, dtype, false, false};   // rank r's chunk of reduced[0] (test hook)
    c->fresh = false;
    return CMN_OK;
}

}  // namespace cmn::rt
