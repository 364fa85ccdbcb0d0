// device_utils.cuh — small device helpers shared by the CUDA sources of libgalois.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "galois_internal.h"

namespace galois {

// Bounds checks of the staged kernels for a checking build (-DGALOIS_BOUNDS_CHECK: a failed
// check traps the kernel, the launch returns an error); compiled out otherwise.
#ifdef GALOIS_BOUNDS_CHECK
#define GALOIS_DEV_CHECK(cond) \
    do {                       \
        if (!(cond)) __trap(); \
    } while (0)
#else
#define GALOIS_DEV_CHECK(cond) \
    do {                       \
    } while (0)
#endif

// Member-in-word layout of every bit plane (X, R, E): member i (0..31) of a 32-member word
// sits at bit 8 (i mod 4) + i / 4, i.e. member j of quad q' (i = 4 q' + j) at bit 8 j + q'.
// A thread owning quad q' reads its 4 members as (w >> q') & 0x01010101 — already one
// per byte, ready for SWAR counting — and 8 lanes pack their quads by 4 ballots + 3 PRMT.
__device__ __forceinline__ int bitpos(int i) { return ((i & 3) << 3) | (i >> 2); }
__device__ __forceinline__ int member_of_bit(int p) { return ((p & 7) << 2) | (p >> 3); }
// smem counter index (32-member word, bit position) -> member offset
__device__ __forceinline__ int member_of_slot(int i) { return (i & ~31) | member_of_bit(i & 31); }
__device__ __forceinline__ uint32_t quad_bits(uint32_t w, int qp) { return (w >> qp) & 0x01010101u; }

// The 32-bit word of the 8-lane group of this lane from each lane's 4-bit quad (bit j =
// member j); mask = the active lanes (whole 8-lane groups).
__device__ __forceinline__ uint32_t pack_quads(uint32_t nib, int lane, uint32_t mask = 0xffffffffu)
{
    const uint32_t b0 = __ballot_sync(mask, nib & 1u), b1 = __ballot_sync(mask, nib & 2u);
    const uint32_t b2 = __ballot_sync(mask, nib & 4u), b3 = __ballot_sync(mask, nib & 8u);
    const uint32_t k = (uint32_t)(lane >> 3) & 3u;
    const uint32_t sel = k | ((k + 4u) << 4);                 // byte k of x, byte k of y
    return __byte_perm(__byte_perm(b0, b1, sel), __byte_perm(b2, b3, sel), 0x5410);
}

__device__ __forceinline__ int pinned_bit(const StepParams &p, int32_t v, int64_t b_global)
{
    if (p.pin_rank == nullptr) return -1;
    const int r = p.pin_rank[v];
    return r < 0 ? -1 : (int)((b_global >> r) & 1);
}

__device__ __forceinline__ float exp_neg_abs(float z)            // exp(-|z|), one MUFU.EX2
{
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(-1.4426950408889634f * fabsf(z)));
    return y;
}

__device__ __forceinline__ float sqrt_approx(float x)            // MUFU.SQRT, rel err ~2^-23
{
    float y;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Best record after a check (reading R10): the key (u << 32 | global b) is the
// minimum over the members (and, with NCCL, over the ranks); the record improves only on
// a strictly smaller count, so ties keep the earlier step and then the lower member.
__device__ __forceinline__ void finalize_best(Ctrl *ctrl, unsigned long long key, int64_t b0, int32_t b_loc)
{
    const int64_t u = (int64_t)(key >> 32);         // 2^32 - 1 when no rank has members
    const int64_t b = (int64_t)(key & 0xFFFFFFFFull);
    ctrl->improved = 0;
    if (u < (int64_t)ctrl->best_u) {
        ctrl->best_u = (int32_t)u;
        ctrl->best_t = ctrl->t;
        ctrl->best_b = b;
        ctrl->improved = (b >= b0 && b < b0 + b_loc) ? 1 : 0;
    }
    ctrl->last_check_t = ctrl->t;
    if (ctrl->best_u == 0) ctrl->stopped = 1;
}

// Block-wide argmin of (unsat[i] << 32 | b0 + i) over the local members; keeps a copy of
// the counts in unsat_last; thread 0 stores key_local and (one rank) finalizes.
__device__ __forceinline__ void block_best(const int32_t *unsat, int32_t *unsat_last, int32_t b_loc, int64_t b0,
                                           Ctrl *ctrl, bool finalize)
{
    __shared__ unsigned long long s_min[32];
    unsigned long long best = ~0ull;
#pragma unroll 8
    for (int32_t i = threadIdx.x; i < b_loc; i += blockDim.x) {
        const int32_t u = __ldcg(unsat + i);
        unsat_last[i] = u;
        const unsigned long long key = ((unsigned long long)(uint32_t)u << 32) | (unsigned long long)(b0 + i);
        best = key < best ? key : best;
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        const unsigned long long o = __shfl_xor_sync(0xffffffffu, best, d);
        best = o < best ? o : best;
    }
    if ((threadIdx.x & 31) == 0) s_min[threadIdx.x >> 5] = best;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) best = s_min[w] < best ? s_min[w] : best;
        ctrl->key_local = best;
        if (finalize) finalize_best(ctrl, best, b0, b_loc);
    }
}

// End of an update kernel: the last CTA to finish advances the step counter. Every CTA
// read ctrl->t at its start, and the last CTA finishes after all of them started, so
// no CTA can observe the new value. Call with the whole CTA (contains __syncthreads).
__device__ __forceinline__ void last_cta_tick(Ctrl *ctrl)
{
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const uint32_t total = gridDim.x * gridDim.y * gridDim.z;
        if (atomicAdd(&ctrl->done_ctas, 1u) == total - 1u) {
            ctrl->done_ctas = 0;
            ctrl->t += 1;
            __threadfence();
        }
    }
}

// --------------------------------------------------------------- mbarrier + TMA bulk copy
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init()
{
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

// Wait for the phase with the given parity. The suspend-time hint lets the hardware park
// the warp until the phase completes (instead of re-issuing try_wait + branch in a tight
// loop, which steals issue slots from the compute warps of the same SM sub-partition).
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase)
{
#ifdef GALOIS_MBAR_NOHINT
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
#else
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(phase), "r"(0x989680u)
        : "memory");
#endif
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// 1-D TMA bulk copy global -> shared (cp.async.bulk; SASS UBLKCP), completion counted in
// bytes on the mbarrier. dst/src 16-B aligned, bytes a multiple of 16.
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// The same operations on precomputed shared-window addresses (smem_u32 once per kernel:
// the generic -> shared conversion otherwise repeats at every call inside the loops).
__device__ __forceinline__ void mbar_wait_s(uint32_t bar, uint32_t phase)
{
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(bar),
        "r"(phase), "r"(0x989680u)
        : "memory");
}

__device__ __forceinline__ void mbar_arrive_s(uint32_t bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx_s(uint32_t bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}

__device__ __forceinline__ void bulk_g2s_s(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}

// Order this thread's earlier generic-proxy smem accesses before later async-proxy ones.
__device__ __forceinline__ void fence_proxy_async_smem()
{
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

}  // namespace galois
