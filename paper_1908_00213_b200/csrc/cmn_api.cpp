// cmn_api.cpp -- the extern "C" entry points of include/cmn.h (argument
// validation, dispatch to the schedules, state access, host-only helpers).
#include "cmn_comm.h"

#include <cmath>
#include <cstring>

using namespace cmn::rt;

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

cmn_status cmn_init_emulated(int world_size, int cuda_device, cmn_comm **out) {
    try {
        const cmn_status st = init_common(0, world_size, cuda_device, true, nullptr, nullptr, out);
        if (st != CMN_OK) return st;
        cmn_comm *c = *out;
        c->emulated = true;
        const auto env_rank = [](const char *name) {
            const char *v = std::getenv(name);
            return v && *v ? std::atoi(v) : -1;
        };
        c->test_absent_rank = env_rank("CMN_TEST_EMUL_ABSENT_RANK");
        c->test_mismatch_rank = env_rank("CMN_TEST_EMUL_MISMATCH_RANK");
        c->test_slow_rank = env_rank("CMN_TEST_EMUL_SLOW_RANK");
        c->test_skip_mid = env_size("CMN_TEST_EMUL_SKIP_MID", 0) != 0 ? 1 : 0;
        return CMN_OK;
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
    if (c->d_errdev) cudaFree(c->d_errdev);
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
    NvtxRange nv("cmn.step.direct");
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
    NvtxRange nv("cmn.step.host_packed");
    if (cmn_status st = ensure_side_streams(c); st != CMN_OK) return st;
    // Separate parameter tensors: each piece's updated params are first
    // packed (fp32, on the caller's stream, 8 B/param of HBM) into a staging
    // buffer in the packed layout, so the piece leaves in ONE device->host
    // copy instead of one per tensor (every extra pinned copy costs ~15-30 us
    // of copy-engine time while the other direction is busy).
    const bool stage_params = host_params && !c->params_flat && !env_size("CMN_E2E_PER_TENSOR_D2H", 0);
    if (stage_params)
        if (cmn_status st = ensure_pstage(c, s); st != CMN_OK) return st;
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
        if (stage_params) {
            st = for_groups(c, 0, c->T, [&](int lo, int hi, int g0, int g1) {
                const int a = g0 > i0 ? g0 : i0, b = g1 < i1 ? g1 : i1;
                if (a >= b) return CMN_OK;
                return launched(c,
                                launch_pack(make_tab(const_cast<const float *const *>(c->params.data()),
                                                     lo, hi),
                                            hi - lo, lo, c->d_td, c->d_items, a, b, CMN_FP32,
                                            c->d_pstage, s),
                                "pack_params");
            });
            if (st != CMN_OK) return st;
        }
        if (host_params) {
            CMN_CUDA(cudaEventRecord(ev_upd, s));
            CMN_CUDA(cudaStreamWaitEvent(c->d2h, ev_upd, 0));
            if (c->params_flat || stage_params) {
                const float *src = stage_params ? c->d_pstage : c->params[0];
                const int64_t hi = e1 < flat_end ? e1 : flat_end;
                if (hi > e0)
                    CMN_CUDA(cudaMemcpyAsync(host_params + e0, src + e0,
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
    const float n_rep = static_cast<float>(c->world);   // a = r / N (reading R3)
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    return for_groups(c, 0, c->T, [&](int lo, int hi, int i0, int i1) {
        return launched(c,
                        launch_unpack_avg(make_tab(const_cast<const float *const *>(out), lo, hi),
                                          lo, c->d_td, c->d_items, i0, i1,
                                          reduced_ptr(c, c->last, 0), c->last.dtype, n_rep,
                                          c->d_errdev, s),
                        "unpack_avg");
    });
}

cmn_status cmn_update_adam(cmn_comm *c, float alpha, float beta1, float beta2, float eps,
                           int step, void *stream) {
    if (cmn_status st = require_registered(c); st != CMN_OK) return st;
    if (!c->fresh) return fail(CMN_ERR_STATE, "no fresh all-reduce result to consume");
    if (step < 1) return fail(CMN_ERR_INVALID_ARG, "step must be >= 1");
    if (cmn_status st = set_device(c); st != CMN_OK) return st;
    if (cmn_status st = ensure_adam(c); st != CMN_OK) return st;
    cmn_status st = update_range_adam(c, 0, c->T, c->last, adam_args(alpha, beta1, beta2, eps, step),
                                      static_cast<cudaStream_t>(stream));
    if (st == CMN_OK) c->fresh = false;
    return st;
}

cmn_status cmn_step_adam(cmn_comm *c, const float *const *grads, cmn_dtype dtype, float alpha,
                         float beta1, float beta2, float eps, int step, void *stream) {
    if (cmn_status st = require_registered(c); st != CMN_OK) return st;
    if (cmn_status st = require_dtype(dtype); st != CMN_OK) return st;
    if (step < 1) return fail(CMN_ERR_INVALID_ARG, "step must be >= 1");
    std::string why;
    if (!grads_ok(c, grads, c->T * (c->simulated ? c->world : 1), why))
        return fail(CMN_ERR_INVALID_ARG, why);
    if (cmn_status st = set_device(c); st != CMN_OK) return st;
    if (cmn_status st = ensure_adam(c); st != CMN_OK) return st;
    const AdamArgs a = adam_args(alpha, beta1, beta2, eps, step);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (c->world == 1 && c->algo != CMN_ALGO_NVLS && c->algo != CMN_ALGO_NCCL) {
        // N = 1: the all-reduce is the identity; Adam straight from g.
        c->fresh = false;
        return timed(c, s, [&] {
            return for_groups(c, 0, c->T, [&](int lo, int hi, int i0, int i1) {
                return launched(c,
                                launch_adam_direct(make_tab(grads, lo, hi),
                                                   make_tab(c->params.data(), lo, hi), hi - lo, lo,
                                                   c->d_adam, c->d_adam + c->L, c->d_items, i0, i1,
                                                   dtype, a.alpha_t, a.beta1, a.beta2, a.c1, a.c2,
                                                   a.eps, s),
                                "adam_direct");
            });
        });
    }
    if (c->world > 1 && c->pipe_pieces >= 2 && c->T >= 2)
        return step_pipelined(c, grads, dtype, 0.0f, 0.0f, s, nullptr, &a);
    if (cmn_status st = cmn_allreduce_grads(c, grads, dtype, stream); st != CMN_OK) return st;
    cmn_status st = update_range_adam(c, 0, c->T, c->last, a, s);
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

cmn_status cmn_set_stream_ctas(cmn_comm *c, int max_ctas) {
    if (!c) return fail(CMN_ERR_INVALID_ARG, "comm is NULL");
    if (max_ctas < 0) return fail(CMN_ERR_INVALID_ARG, "max_ctas must be >= 0 (0 = one CTA per item)");
    c->stream_ctas = max_ctas;
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

cmn_status cmn_debug_fill_buffers(cmn_comm *c, uint32_t pattern, void *stream) {
    if (cmn_status st = require_registered(c); st != CMN_OK) return st;
    if (cmn_status st = set_device(c); st != CMN_OK) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const size_t words = static_cast<size_t>(buf_elems(c->L)) * 4;   // packed0..reduced1, fp32 words
    const int own = c->simulated ? c->world : 1;
    for (int i = 0; i < own; ++i) {
        const int r = c->simulated ? i : c->rank;
        CMN_CUDA(launch_fill_u32(static_cast<uint32_t *>(c->rb[r].packed[0]), words, pattern, s));
    }
    c->fresh = false;
    return CMN_OK;
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
