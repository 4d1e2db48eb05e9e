// cmn_device.cuh -- device helpers for the sm_100a kernels: fp16 payload
// conversion, the fixed pairwise reduction tree, streaming vector memory
// ops, and the cross-GPU release/acquire barrier.
#pragma once

#include <cstdint>

#include <cuda_fp16.h>

#include "cmn_internal.h"

namespace cmn {

// ------------------------------------------------------------ fp16 payload
// fp32 -> fp16 is cvt.rn.f16.f32 (IEEE round-to-nearest-even, subnormals
// kept: the library is built without --use_fast_math / -ftz), reading R4.
__device__ __forceinline__ uint32_t pack_half2(float lo, float hi) {
    const uint32_t a = __half_as_ushort(__float2half_rn(lo));
    const uint32_t b = __half_as_ushort(__float2half_rn(hi));
    return a | (b << 16);
}
__device__ __forceinline__ float half_lo(uint32_t h2) {
    return __half2float(__ushort_as_half(static_cast<unsigned short>(h2 & 0xffffu)));
}
__device__ __forceinline__ float half_hi(uint32_t h2) {
    return __half2float(__ushort_as_half(static_cast<unsigned short>(h2 >> 16)));
}
__device__ __forceinline__ float round_through_half(float x) {
    return __half2float(__float2half_rn(x));
}

// ----------------------------------------------------- the reduction tree
// tree(x_lo..x_hi) = tree(x_lo..x_m) + tree(x_m+1..x_hi), low half holds
// ceil(n/2) inputs, IEEE fp32 round-to-nearest additions (reading R2).
// __fadd_rn is never contracted into an FMA.
template <int LO, int HI>
struct Tree {
    static constexpr int kN = HI - LO + 1;
    static constexpr int kM = LO + (kN + 1) / 2 - 1;
    __device__ __forceinline__ static float sum(const float *x) {
        return __fadd_rn(Tree<LO, kM>::sum(x), Tree<kM + 1, HI>::sum(x));
    }
};
template <int I>
struct Tree<I, I> {
    __device__ __forceinline__ static float sum(const float *x) { return x[I]; }
};

// ------------------------------------------------------------- memory ops
// Streaming (evict-first) 16-byte accesses for data touched exactly once.
// Built with -DCMN_NO_STREAMING_HINTS they become plain accesses (a
// measurement switch for scripts/gpu_hints_ab.sh).
#ifndef CMN_NO_STREAMING_HINTS
__device__ __forceinline__ float4 ld_cs_f4(const float *p) {
    return __ldcs(reinterpret_cast<const float4 *>(p));
}
__device__ __forceinline__ void st_cs_f4(float *p, const float4 &v) {
    __stcs(reinterpret_cast<float4 *>(p), v);
}
__device__ __forceinline__ uint2 ld_cs_u2(const void *p) {
    return __ldcs(reinterpret_cast<const uint2 *>(p));
}
__device__ __forceinline__ void st_cs_u2(void *p, const uint2 &v) {
    __stcs(reinterpret_cast<uint2 *>(p), v);
}
#else
__device__ __forceinline__ float4 ld_cs_f4(const float *p) {
    return *reinterpret_cast<const float4 *>(p);
}
__device__ __forceinline__ void st_cs_f4(float *p, const float4 &v) {
    *reinterpret_cast<float4 *>(p) = v;
}
__device__ __forceinline__ uint2 ld_cs_u2(const void *p) {
    return *reinterpret_cast<const uint2 *>(p);
}
__device__ __forceinline__ void st_cs_u2(void *p, const uint2 &v) {
    *reinterpret_cast<uint2 *>(p) = v;
}
#endif

// 32-byte (256-bit, LDG/STG.E.ENL2.256 on sm_100a) streaming accesses; the
// address must be 32-byte aligned.
struct F8 {
    float4 lo, hi;
};
__device__ __forceinline__ F8 ld_cs_f8(const float *p) {
    F8 r;
    asm volatile("ld.global.cs.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(r.lo.x), "=f"(r.lo.y), "=f"(r.lo.z), "=f"(r.lo.w), "=f"(r.hi.x), "=f"(r.hi.y),
                   "=f"(r.hi.z), "=f"(r.hi.w)
                 : "l"(p));
    return r;
}
__device__ __forceinline__ void st_cs_f8(float *p, const F8 &v) {
    asm volatile("st.global.cs.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(v.lo.x),
                 "f"(v.lo.y), "f"(v.lo.z), "f"(v.lo.w), "f"(v.hi.x), "f"(v.hi.y), "f"(v.hi.z),
                 "f"(v.hi.w)
                 : "memory");
}

__device__ __forceinline__ F8 ld_f8(const float *p) {
    F8 r;
    asm volatile("ld.global.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(r.lo.x), "=f"(r.lo.y), "=f"(r.lo.z), "=f"(r.lo.w), "=f"(r.hi.x), "=f"(r.hi.y),
                   "=f"(r.hi.z), "=f"(r.hi.w)
                 : "l"(p));
    return r;
}
__device__ __forceinline__ void st_f8(float *p, const F8 &v) {
    asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(v.lo.x),
                 "f"(v.lo.y), "f"(v.lo.z), "f"(v.lo.w), "f"(v.hi.x), "f"(v.hi.y), "f"(v.hi.z),
                 "f"(v.hi.w)
                 : "memory");
}
__device__ __forceinline__ bool aligned32(const void *p) {
    return (reinterpret_cast<uintptr_t>(p) & 31u) == 0;
}

// 16-byte load that may target a peer GPU's memory (UVA / IPC mapping) and
// data published by a peer during this kernel: weak load, no L1 allocation
// (never the non-coherent .nc path).
__device__ __forceinline__ uint4 ld_peer_u4(const void *p) {
    uint4 r;
    asm volatile("ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p)
                 : "memory");
    return r;
}
__device__ __forceinline__ uint2 ld_peer_u2(const void *p) {
    uint2 r;
    asm volatile("ld.global.L1::no_allocate.v2.u32 {%0,%1}, [%2];"
                 : "=r"(r.x), "=r"(r.y)
                 : "l"(p)
                 : "memory");
    return r;
}
__device__ __forceinline__ void st_u2(void *p, const uint2 &v) {
    asm volatile("st.global.v2.u32 [%0], {%1,%2};" ::"l"(p), "r"(v.x), "r"(v.y) : "memory");
}
__device__ __forceinline__ void st_u4(void *p, const uint4 &v) {
    asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
                 "r"(v.w)
                 : "memory");
}

// ----------------------------------------------------------- the barrier
__device__ __forceinline__ void st_release_sys(uint32_t *p, uint32_t v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t ld_relaxed_sys(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void fence_acq_rel_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }
__device__ __forceinline__ void st_relaxed_sys(uint32_t *p, uint32_t v) {
    asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Barrier memory ordering (CMN_BARRIER_VARIANT; 3 is the default since
// round 2, session 3, the others stay as measurement switches):
//   0: every polling thread: __threadfence_system, st.release.sys, spin on
//      ld.acquire.sys (the round-1/2 form: TWO MEMBAR.SYS per flag)
//   1: every polling thread: st.release.sys, spin on ld.acquire.sys
//   3: thread 0: ONE fence.acq_rel.sys for the CTA, then every peer's flag
//      as st.relaxed.sys (release pattern: fence + strong store, same
//      thread; bar.sync before it ordered every thread's writes); the
//      polling threads spin on ld.acquire.sys
//   4: as 3, but spin on ld.relaxed.sys and take one ld.acquire.sys of the
//      cell once it is satisfied
// Measured in the emulated world (profiles/r2s3_barrier_ab*.jsonl, tiny
// all-reduce, graph replay): a system-scope fence costs ~6-8 us here; 0 ->
// 3 takes the N = 2 two-shot from 36 to 20.5 us per call (7.8 us with
// gpu-scope fences, which are not valid across GPUs), the R50 N = 8 fp32
// two-shot from 385 to 370 us.  1, 3 and 4 are within 0.5 us of each other.
#ifndef CMN_BARRIER_VARIANT
#define CMN_BARRIER_VARIANT 3
#endif

__device__ __forceinline__ uint64_t global_timer_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Has a collective of this communicator failed (timeout or mismatch)?  The
// device-memory error word is set by the barrier that detected it; every
// later kernel of the step checks it and leaves its outputs untouched.
__device__ __forceinline__ bool comm_failed(const int *derr) {
    return derr && *reinterpret_cast<const volatile int *>(derr) != 0;
}

__device__ __forceinline__ void record_failure(const Barrier &bar, int code) {
    *reinterpret_cast<volatile int *>(bar.derr) = code;
    __threadfence();
    *reinterpret_cast<volatile int *>(bar.err) = code;
}

// Fault injection for tests: stall the calling thread for `ns` nanoseconds.
__device__ __forceinline__ void stall_ns(uint32_t ns) {
    const uint64_t t0 = global_timer_ns();
    while (global_timer_ns() - t0 < ns) {
    }
}

// This call's barrier value for the calling CTA: reads and advances the
// CTA's epoch counter (one increment per collective kernel; the next kernel
// on the stream starts after this one completes, so reads see the update).
//
// When an earlier kernel of this communicator already failed (device error
// word) the value carries the reserved tag kDeadTag instead of the call tag:
// cross_rank_barrier then posts it as a poison flag and returns false.  A
// failed rank that posted a normal value would overwrite its cell with a
// later epoch, which a peer still waiting on an earlier barrier reads as
// "passed" (flags only grow) -- pairing it with a collective that never
// happened (scripts/diag_piece_mismatch.py saw a TIMEOUT at the next
// barrier instead of the MISMATCH); the poison instead makes every waiting
// peer fail at once.  The error word is loaded together with the epoch
// counter, so the check costs no latency.
// Which rank and which of its CTAs this block plays: itself on a real rank;
// under emulation (bar.emul_g > 0, one cooperative launch for the whole
// world) block r * emul_g + b plays CTA b of rank r.
struct CtaRank {
    int b;      // CTA index within the rank's grid
    int n;      // the rank's grid size
    int rank;
};
__device__ __forceinline__ CtaRank cta_rank(const Barrier &bar) {
    if (bar.emul_g > 0)
        return CtaRank{static_cast<int>(blockIdx.x) % bar.emul_g, bar.emul_g,
                       static_cast<int>(blockIdx.x) / bar.emul_g};
    return CtaRank{static_cast<int>(blockIdx.x), static_cast<int>(gridDim.x), bar.rank};
}

__device__ __forceinline__ uint32_t barrier_value(const Barrier &bar) {
    __shared__ uint32_t s_val;
    if (!bar.enabled) return 0;
    if (threadIdx.x == 0) {
        const CtaRank cr = cta_rank(bar);
        uint32_t *epoch = bar.emul_g > 0 ? bar.epochs[cr.rank] : bar.epoch;
        const bool dead = comm_failed(bar.derr);
        const uint32_t e = epoch[cr.b] + 1u;
        epoch[cr.b] = e;
        const uint32_t tag = cr.rank == bar.test_mismatch_rank ? (bar.tag ^ 0x2u) : bar.tag;
        s_val = (e << kTagBits) | (dead ? kDeadTag : (tag & kTagMask));
    }
    __syncthreads();
    return s_val;
}

// Fault injection (tests only): a slow peer.  Every CTA of this rank on a
// real rank; under emulation only the blocks of bar.test_slow_rank (or all
// of them when it is -1).
__device__ __forceinline__ void test_stall(const Barrier &bar, const CtaRank &cr) {
    if (bar.test_delay_ns && (bar.emul_g == 0 || bar.test_slow_rank < 0 || cr.rank == bar.test_slow_rank))
        stall_ns(bar.test_delay_ns);
}

// Emulation fault injection: the CTAs of bar.test_absent_rank never arrive
// (they return before touching anything), so their peers' barriers time out.
__device__ __forceinline__ bool emulated_absent(const Barrier &bar) {
    return bar.emul_g > 0 && static_cast<int>(blockIdx.x) / bar.emul_g == bar.test_absent_rank;
}

// Pairwise per-CTA barrier across ranks: CTA b of rank r tells CTA b of
// every rank "my inputs for this phase are published" and waits for the
// same from all of them.  Flag values only grow, so no reset is needed; a
// peer at the same epoch with another tag (payload dtype, algorithm, kernel
// kind or packed range) is a call-sequence mismatch.  Spins are bounded by
// %globaltimer (default 30 s).  Because a kernel starts only
// after the previous kernel on its stream completed, passing the barrier
// also proves every peer finished all its earlier collective kernels.
//
// Returns false when the CTA must not touch data: an earlier kernel of this
// communicator already failed (barrier_value carried kDeadTag: the poison
// is posted to every peer's cells of both slots, nothing else happens), a
// peer posted the poison, this wait timed out or saw a mismatch, or another
// CTA of this rank recorded a failure while we spun (polled every 64 spins,
// so one CTA's timeout stops the others at once).  Callers return immediately, so a
// failed call leaves its outputs (and, through comm_failed, the parameters
// and optimizer state the update kernels would write) untouched.  Within one
// kernel a CTA that passed its start barrier still posts its later barrier
// (mid / end) even if another CTA failed meanwhile: its peer CTA passed the
// same start barrier, so the pair stays consistent.
__device__ __forceinline__ bool cross_rank_barrier(const Barrier &bar, uint32_t value, int world,
                                                   int slot) {
    if (!bar.enabled) return true;
    const int tid = threadIdx.x;
    const CtaRank cr = cta_rank(bar);
    if ((value & kTagMask) == kDeadTag) {  // uniform across the CTA (shared value)
        if (tid < world) {
            for (int sl = 0; sl < kBarrierSlots; ++sl)
                st_release_sys(bar.flags[tid] +
                                   (static_cast<size_t>(sl) * kMaxBarrierBlocks + cr.b) * kMaxWorld +
                                   cr.rank,
                               value);
        }
        return false;
    }
    __syncthreads();
    int bad = 0;
    const size_t cell = (static_cast<size_t>(slot) * kMaxBarrierBlocks + cr.b) * kMaxWorld;
#if CMN_BARRIER_VARIANT >= 3
    if (tid == 0) {
        // release: one fence for the whole CTA (bar.sync above ordered every
        // thread's writes before it), then the flags as plain strong stores
        fence_acq_rel_sys();
        for (int p = 0; p < world; ++p) st_relaxed_sys(bar.flags[p] + cell + cr.rank, value);
    }
#endif
    if (tid < world) {
#if CMN_BARRIER_VARIANT == 0
        __threadfence_system();
#endif
#if CMN_BARRIER_VARIANT < 3
        st_release_sys(bar.flags[tid] + cell + cr.rank, value);
#endif
        const uint32_t *mine = bar.flags[cr.rank] + cell + tid;
        uint64_t t0 = 0;
        for (uint32_t spin = 1;; ++spin) {
#if CMN_BARRIER_VARIANT == 4
            uint32_t v = ld_relaxed_sys(mine);
#else
            uint32_t v = ld_acquire_sys(mine);
#endif
            if ((v & kTagMask) == kDeadTag) {   // the peer's communicator failed earlier
                record_failure(bar, 3);
                bad = 1;
                break;
            }
            if ((v >> kTagBits) == (value >> kTagBits) && v != value) {
                record_failure(bar, 2);
                bad = 1;
                break;
            }
            if (static_cast<int32_t>(v - value) >= 0) {
#if CMN_BARRIER_VARIANT == 4
                v = ld_acquire_sys(mine);   // acquire: synchronises with the peer's release
                (void)v;
#endif
                break;
            }
            if ((spin & 63u) == 0 && comm_failed(bar.derr)) {   // failed elsewhere: stop waiting
                bad = 1;
                break;
            }
            if ((spin & 1023u) == 0) {
                const uint64_t t = global_timer_ns();
                if (t0 == 0) {
                    t0 = t;
                } else if (t - t0 > bar.timeout_ns) {
                    record_failure(bar, 1);
                    bad = 1;
                    break;
                }
            }
        }
    }
    return __syncthreads_or(bad) == 0;
}

}  // namespace cmn
