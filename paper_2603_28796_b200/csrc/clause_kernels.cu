// clause_kernels.cu — rows a5 (clause-polynomial forward) and a8 (exact checker) in ONE
// sweep over the clauses, vectorised: each lane owns 4 consecutive batch words
// (16 B = 128 members) of a row.
//
// For clause c and a lane's 4 words, with S_i = X[v_i] xor negmask_i (literal true):
//   any = OR_i S_i, two = OR_{i<j} (S_i AND S_j)   (>= 1 / >= 2 literals true)
//   U   = ~any                      = prod_i (1 - s_i)          (Eq.2, clause unsatisfied)
//   E_i = ~any | (S_i & ~two)       = prod_{j != i} (1 - s_j)   (exclusive products)
// E is written in CSC order into the chunk-major layout E[chunk][pos][CW] that the update
// kernel reads with one TMA bulk copy per (variable, chunk). Per-member counts of U —
// the ST loss Lambda of the sample X (kForward) and the exact unsat counts of the
// rounding R (kCheck) — are accumulated in shared memory and added to global memory
// once per block (integer, deterministic). Step s runs forward(X_s) fused with the check
// of R_{s-1} (the rounding of the previous update): one pass over the clause indices, two
// independent row gathers per slot.
//
// Lane layout: LPC = min(W/4, 32) lanes per clause (16 B each, 128 B per 8 lanes:
// coalesced row segments), CPW = 32 / LPC clauses in flight per warp (width-sorted
// order), blockIdx.y selects 128-word column chunks. Requires W % 4 == 0.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "device_utils.cuh"
#include "galois_internal.h"

namespace galois {

namespace {
constexpr int kCached = 3;   // slots kept in registers between the two passes (rest re-gathered)

__device__ __forceinline__ void count_bits_smem4(int32_t *s_cnt, int vl, uint4 U)
{
    const uint32_t w[4] = {U.x, U.y, U.z, U.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        uint32_t u = w[k];
        while (u) {
            const int j = __ffs(u) - 1;
            atomicAdd(&s_cnt[((vl << 2) + k) * 32 + j], 1);
            u &= u - 1;
        }
    }
}

// B: this lane's X (or R) vector of row 0; rows are RS uint4 apart (interleaved X/R rows)
__device__ __forceinline__ uint4 lit4(const uint4 *B, int RS, int32_t code)
{
    const uint32_t neg = 0u - (uint32_t)(code & 1);
    uint4 s = B[(size_t)(code >> 1) * RS];
    s.x ^= neg; s.y ^= neg; s.z ^= neg; s.w ^= neg;
    return s;
}

#ifndef GALOIS_SWEEP_XR256
#define GALOIS_SWEEP_XR256 1   // fused forward + check: X and R of a literal in one 256-bit load
#endif
// X and R vectors of literal `code` (16 B each, adjacent: R = X + 4 words) in ONE 256-bit
// load with an L2 evict-last priority (the X/R rows are the sweep's reused working set;
// E and the index stream past them), sign applied to both
__device__ __forceinline__ void lit_xr(const uint4 *BX, int RS, int32_t code, uint4 &x, uint4 &r)
{
    const uint4 *p = BX + (size_t)(code >> 1) * RS;
    asm("ld.global.nc.L2::evict_last.v8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
        : "=r"(x.x), "=r"(x.y), "=r"(x.z), "=r"(x.w), "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
        : "l"(p));
    const uint32_t neg = 0u - (uint32_t)(code & 1);
    x.x ^= neg; x.y ^= neg; x.z ^= neg; x.w ^= neg;
    r.x ^= neg; r.y ^= neg; r.z ^= neg; r.w ^= neg;
}

__device__ __forceinline__ void acc2(uint4 &any, uint4 &two, uint4 s)
{
    two.x |= any.x & s.x; two.y |= any.y & s.y; two.z |= any.z & s.z; two.w |= any.w & s.w;
    any.x |= s.x; any.y |= s.y; any.z |= s.z; any.w |= s.w;
}

__device__ __forceinline__ void or4(uint4 &any, uint4 s)
{
    any.x |= s.x; any.y |= s.y; any.z |= s.z; any.w |= s.w;
}

// X and R vectors (16 B each, adjacent) of one literal: one 256-bit load (LDG.E.ENL2.256)
__device__ __forceinline__ void ld_xr(const uint4 *p, uint4 &x, uint4 &r)
{
    asm("ld.global.nc.v8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
        : "=r"(x.x), "=r"(x.y), "=r"(x.z), "=r"(x.w), "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
        : "l"(p));
}

__device__ __forceinline__ uint64_t l2_policy(bool evict_first)
{
    uint64_t pol;
    if (evict_first)
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    else
        asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

__device__ __forceinline__ void st_e(uint32_t *p, uint4 e, uint64_t pol)
{
    asm volatile("st.global.L2::cache_hint.v4.b32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "r"(e.x), "r"(e.y),
                 "r"(e.z), "r"(e.w), "l"(pol)
                 : "memory");
}

__device__ __forceinline__ void bulk_g2s_hint(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar,
                                              uint64_t pol)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], "
        "%4;" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(bar), "l"(pol)
        : "memory");
}

}  // namespace

template <bool kForward, bool kCheck>
__global__ void __launch_bounds__(256) k_clauses_v4(DevCnf c, int32_t W, int32_t b_pad,
                                                    const uint32_t *__restrict__ X, const uint32_t *__restrict__ R,
                                                    uint32_t *__restrict__ E, int32_t *__restrict__ lam,
                                                    int32_t *__restrict__ unsat, Ctrl *__restrict__ ctrl,
                                                    BestArgs ba)
{
    __shared__ int32_t s_lam[kForward ? 4096 : 1];   // members of this block's 128-word chunk
    __shared__ int32_t s_uns[kCheck ? 4096 : 1];
    if (ctrl->stopped) return;
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) {
        if (kForward) s_lam[i] = 0;
        if (kCheck) s_uns[i] = 0;
    }
    __syncthreads();

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int VW = W >> 2;                    // 16-B vector words per row
    const int RS = 2 * VW;                    // uint4 per interleaved X/R row
    const int LPC = VW < 32 ? VW : 32;
    const int CPW = 32 / LPC;
    const int sub = lane / LPC, vl = lane - sub * LPC;
    const int vw = blockIdx.y * 32 + vl;      // this lane's vector word
    const bool lane_ok = sub < CPW && vw < VW;
    const int64_t ngroups = ((int64_t)c.m + CPW - 1) / CPW;
    const int64_t stride = (int64_t)gridDim.x * (blockDim.x >> 5);
    // E chunk plane and offset of words 4vw..4vw+3 (chunk width CW = min(W, 32) words)
    const int CW = W < 32 ? W : 32;
    const int ch = (vw << 2) / CW, wi = (vw << 2) - ch * CW;
    uint32_t *Ecol = kForward ? E + (size_t)ch * c.L * CW + wi : nullptr;
    const uint4 *BX = reinterpret_cast<const uint4 *>(X) + 2 * vw;   // interleaved rows: X, R groups alternate
    const uint4 *BR = reinterpret_cast<const uint4 *>(R) + 2 * vw;

    for (int64_t g = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp; g < ngroups; g += stride) {
        const int64_t ci = g * CPW + sub;
        if (!lane_ok || ci >= c.m) continue;
        // sweep order (width-sorted, the CSR regrouped: no clause_perm -> clause_off hop);
        // forward + check: a literal's X and R vectors in one 256-bit load
        const int32_t lo = c.sweep_off[ci], width = c.sweep_off[ci + 1] - lo;
        uint4 any = make_uint4(0, 0, 0, 0), two = make_uint4(0, 0, 0, 0), anyR = make_uint4(0, 0, 0, 0);
        uint4 S[kCached];
        int2 si[kCached];
#pragma unroll
        for (int i = 0; i < kCached; ++i)
            if (i < width) si[i] = c.sweep_slot[lo + i];
#pragma unroll
        for (int i = 0; i < kCached; ++i) {
            if (i < width) {
                if (kForward && kCheck) {
                    uint4 r;
                    lit_xr(BX, RS, si[i].x, S[i], r);
                    acc2(any, two, S[i]);
                    or4(anyR, r);
                } else {
                    if (kForward) {
                        S[i] = lit4(BX, RS, si[i].x);
                        acc2(any, two, S[i]);
                    }
                    if (kCheck) or4(anyR, lit4(BR, RS, si[i].x));
                }
            }
        }
        for (int i = kCached; i < width; ++i) {
            const int2 sj = c.sweep_slot[lo + i];
            if (kForward && kCheck) {
                uint4 x, r;
                lit_xr(BX, RS, sj.x, x, r);
                acc2(any, two, x);
                or4(anyR, r);
            } else {
                if (kForward) acc2(any, two, lit4(BX, RS, sj.x));
                if (kCheck) or4(anyR, lit4(BR, RS, sj.x));
            }
        }
        if (kForward) {
#pragma unroll
            for (int i = 0; i < kCached; ++i)
                if (i < width) {
                    const uint4 s = S[i];
                    const uint32_t nm = 0u - (uint32_t)(si[i].x & 1);   // negative: stored complemented
                    const uint4 e = make_uint4((~any.x | (s.x & ~two.x)) ^ nm, (~any.y | (s.y & ~two.y)) ^ nm,
                                               (~any.z | (s.z & ~two.z)) ^ nm, (~any.w | (s.w & ~two.w)) ^ nm);
                    *reinterpret_cast<uint4 *>(Ecol + (size_t)si[i].y * CW) = e;
                }
            for (int i = kCached; i < width; ++i) {
                const int2 sj = c.sweep_slot[lo + i];
                const uint4 s = lit4(BX, RS, sj.x);
                const uint32_t nm = 0u - (uint32_t)(sj.x & 1);
                const uint4 e = make_uint4((~any.x | (s.x & ~two.x)) ^ nm, (~any.y | (s.y & ~two.y)) ^ nm,
                                           (~any.z | (s.z & ~two.z)) ^ nm, (~any.w | (s.w & ~two.w)) ^ nm);
                *reinterpret_cast<uint4 *>(Ecol + (size_t)sj.y * CW) = e;
            }
            count_bits_smem4(s_lam, vl, make_uint4(~any.x, ~any.y, ~any.z, ~any.w));
        }
        if (kCheck) count_bits_smem4(s_uns, vl, make_uint4(~anyR.x, ~anyR.y, ~anyR.z, ~anyR.w));
    }
    __syncthreads();
    const int base = blockIdx.y * 4096;
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) {
        const int mb = base + member_of_slot(i);       // i = word * 32 + bit position
        if (mb >= b_pad) continue;
        if (kForward && s_lam[i] != 0) atomicAdd(&lam[mb], s_lam[i]);
        if (kCheck && s_uns[i] != 0) atomicAdd(&unsat[mb], s_uns[i]);
    }
    if (kCheck) {
        // the last CTA to finish reduces the complete counts to the best key (a8) and, on
        // a single rank, updates the best record and the stop flag (no extra launch)
        __shared__ bool s_last;
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            s_last = atomicAdd(&ctrl->done_ctas, 1u) == gridDim.x * gridDim.y - 1u;
        }
        __syncthreads();
        if (s_last) {
            __threadfence();
            block_best(unsat, ba.unsat_last, ba.b_loc, ba.b0, ctrl, ba.finalize != 0);
            if (threadIdx.x == 0) ctrl->done_ctas = 0;
            if (ba.extract_n > 0) {          // small n: the winner's bits of R, in this CTA
                __syncthreads();
                if (__ldcg(&ctrl->improved)) {
                    const int64_t lb = ctrl->best_b - ba.b0;
#pragma unroll 8
                    for (int32_t v = threadIdx.x; v < ba.extract_n; v += blockDim.x)
                        ba.best_bits[v] =
                            (uint8_t)((R[xr_at(v, (int32_t)(lb >> 5), ba.W)] >> bitpos((int)(lb & 31))) & 1u);
                }
            }
        }
    }
}

// ---------------------------------------------------------------------------------------
// k_sweep: the same sweep for W % 32 == 0 (1024-member chunks, blockIdx.y = chunk) with
// bit-sliced per-member counters instead of one shared atomic per set bit.
//
// Lane = (sub, vl): 8 lanes (vl) cover one clause's 1024-member chunk (16 B each), 4 clauses
// (sub) per warp. Lanes with equal vl hold the same 128 members of 4 different clauses, so
// a two-round butterfly (shfl_xor 8, 16) adds their 4 U words and leaves lane (sub, vl)
// with the 3-bit counts of word 4 vl + sub (a reduce-scatter of a 4 x 4 bit-word block).
// Each lane adds that into a vertical counter of 8 (or 6) planes (one full adder per plane);
// every 63 (15) groups, before a count can reach 2^planes, they are flushed into shared counters
// with weight 2^k. At dense unsat patterns (C4: ~7% of clause-member pairs) this replaces
// ~40 instructions per U word by ~10.
namespace {

__device__ __forceinline__ uint32_t sel(uint32_t m, uint32_t a, uint32_t b) { return (a & m) | (b & ~m); }

// U: this lane's 4 words; bm/cm: all-ones masks of sub bit 0 / bit 1. Adds the butterfly
// counts of word (sub) into planes P[0..7].
template <int kPlanes>
__device__ __forceinline__ void butterfly_add(uint32_t (&P)[kPlanes], uint4 U, uint32_t bm, uint32_t cm)
{
    // round 1 (partner sub ^ 1): keep words {b, b + 2}, send {1 - b, 3 - b}
    const uint32_t k0 = sel(bm, U.y, U.x), s0 = sel(bm, U.x, U.y);
    const uint32_t k1 = sel(bm, U.w, U.z), s1 = sel(bm, U.z, U.w);
    const uint32_t r0 = __shfl_xor_sync(0xffffffffu, s0, 8);
    const uint32_t r1 = __shfl_xor_sync(0xffffffffu, s1, 8);
    const uint32_t a00 = k0 ^ r0, a10 = k0 & r0;      // 2-bit count of word b
    const uint32_t a01 = k1 ^ r1, a11 = k1 & r1;      // 2-bit count of word b + 2
    // round 2 (partner sub ^ 2): keep word b + 2c, send the other
    const uint32_t q0 = sel(cm, a01, a00), q1 = sel(cm, a11, a10);
    const uint32_t o0 = __shfl_xor_sync(0xffffffffu, sel(cm, a00, a01), 16);
    const uint32_t o1 = __shfl_xor_sync(0xffffffffu, sel(cm, a10, a11), 16);
    const uint32_t t0 = q0 ^ o0, c0 = q0 & o0;
    const uint32_t t1 = q1 ^ o1 ^ c0;
    const uint32_t t2 = (q1 & o1) | (c0 & (q1 ^ o1));
    // P += t (ripple through 8 planes)
    uint32_t carry = P[0] & t0;
    P[0] ^= t0;
    uint32_t nc = (P[1] & t1) | (carry & (P[1] ^ t1));
    P[1] ^= t1 ^ carry;
    carry = nc;
    nc = (P[2] & t2) | (carry & (P[2] ^ t2));
    P[2] ^= t2 ^ carry;
    carry = nc;
#pragma unroll
    for (int k = 3; k < kPlanes; ++k) {
        nc = P[k] & carry;
        P[k] ^= carry;
        carry = nc;
    }
}

template <int kPlanes>
__device__ __forceinline__ void flush_planes(uint32_t (&P)[kPlanes], int32_t *s_cnt, int word)
{
    int32_t *dst = s_cnt + word * 32;
#pragma unroll
    for (int k = 0; k < kPlanes; ++k) {
        uint32_t u = P[k];
        while (u) {
            const int j = __ffs(u) - 1;
            atomicAdd(dst + j, 1 << k);
            u &= u - 1;
        }
        P[k] = 0;
    }
}

}  // namespace

// Two shapes: kWide (average clause width >= 4.5: many gathers per clause, L2-resident
// rows) trades register caching and counter planes for a 4th resident CTA per SM.
#ifndef GALOIS_SWEEP_CACHED
#define GALOIS_SWEEP_CACHED 2
#endif
#ifndef GALOIS_SWEEP_CTAS
#define GALOIS_SWEEP_CTAS 3
#endif
template <bool kWide>
struct SweepShape {
    static constexpr int kPlanes = kWide ? 6 : 8;            // counts < 2^kPlanes between flushes
    static constexpr int kFlushGroups = ((1 << kPlanes) - 1) / 4;   // a group adds <= 4 per member
    static constexpr int kCached = kWide ? 0 : GALOIS_SWEEP_CACHED;   // slots kept in registers for the E pass
    static constexpr int kMinBlocks = kWide ? 4 : GALOIS_SWEEP_CTAS;
};

template <bool kForward, bool kCheck, bool kWide, bool kLoop>
__global__ void __launch_bounds__(256, SweepShape<kWide>::kMinBlocks) k_sweep(DevCnf c, int32_t W, int32_t b_pad, const uint32_t *__restrict__ X,
                                               const uint32_t *__restrict__ R, uint32_t *__restrict__ E,
                                               int32_t *__restrict__ lam, int32_t *__restrict__ unsat,
                                               Ctrl *__restrict__ ctrl, BestArgs ba, int32_t stream_hint)
{
    __shared__ int32_t s_lam[kForward ? 1024 : 1];   // members of the current 1024-member chunk
    __shared__ int32_t s_uns[kCheck ? 1024 : 1];
    if (ctrl->stopped) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int sub = lane >> 3, vl = lane & 7;
    const uint32_t bm = 0u - (uint32_t)(sub & 1), cm = 0u - (uint32_t)((sub >> 1) & 1);
    const int VW = W >> 2;
    const int RS = 2 * VW;                            // uint4 per interleaved X/R row
    const int32_t ngroups = (c.m + 3) / 4;
    const int32_t stride = gridDim.x * (blockDim.x >> 5);
    constexpr int kPlanes = SweepShape<kWide>::kPlanes;
    constexpr int kSweepCached = SweepShape<kWide>::kCached;
    uint32_t PL[kPlanes], PU[kPlanes];
#pragma unroll
    for (int k = 0; k < kPlanes; ++k) PL[k] = PU[k] = 0;
    // Chunks blockIdx.y, blockIdx.y + gridDim.y, ...: the launcher sizes gridDim.y so that
    // the X and R slices of the chunks in flight stay L2-resident (C5: one 1024-member chunk
    // of all 100k rows at a time instead of all 64 chunks' 1.6 GB).
    const int chunk_end = kLoop ? W / 32 : (int)blockIdx.y + 1;   // !kLoop: one chunk per CTA
    for (int chunk = blockIdx.y; chunk < chunk_end; chunk += gridDim.y) {
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) {
        if (kForward) s_lam[i] = 0;
        if (kCheck) s_uns[i] = 0;
    }
    __syncthreads();
    const int vw = chunk * 8 + vl;                    // this lane's 16-B vector word of a row
    uint32_t *Ecol = kForward ? E + (size_t)chunk * c.L * 32 + vl * 4 : nullptr;
    const uint4 *BX = reinterpret_cast<const uint4 *>(X) + 2 * vw;   // interleaved rows: X, R groups alternate
    const uint4 *BR = reinterpret_cast<const uint4 *>(R) + 2 * vw;
    const uint64_t pol = l2_policy(stream_hint != 0);
    int since = 0;

    // the offsets of the next group are loaded one iteration ahead (sweep order: no
    // clause_perm -> clause_off indirection on the critical path)
    int32_t g = blockIdx.x * (blockDim.x >> 5) + warp;
    int32_t nlo = 0, nhi = 0;
    if (g < ngroups && g * 4 + sub < c.m) {
        nlo = c.sweep_off[g * 4 + sub];
        nhi = c.sweep_off[g * 4 + sub + 1];
    }
    for (; g < ngroups; g += stride) {
        const int32_t ci = g * 4 + sub;
        const int32_t lo = nlo, width = nhi - nlo;
        {
            const int32_t cn = ci + stride * 4;
            if (cn < c.m) {
                nlo = c.sweep_off[cn];
                nhi = c.sweep_off[cn + 1];
            }
        }
        uint4 any = make_uint4(0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu), anyR = any;
        if (ci < c.m) {
            uint4 two = make_uint4(0, 0, 0, 0);
            any = make_uint4(0, 0, 0, 0);
            anyR = any;
            uint4 S[kSweepCached > 0 ? kSweepCached : 1];
            int2 si[kSweepCached > 0 ? kSweepCached : 1];
#pragma unroll
            for (int i = 0; i < kSweepCached; ++i)
                if (i < width) si[i] = c.sweep_slot[lo + i];
#pragma unroll
            for (int i = 0; i < kSweepCached; ++i) {
                if (i < width) {
                    if (kForward && kCheck && GALOIS_SWEEP_XR256) {
                        uint4 r;
                        lit_xr(BX, RS, si[i].x, S[i], r);
                        acc2(any, two, S[i]);
                        or4(anyR, r);
                    } else {
                        if (kForward) {
                            S[i] = lit4(BX, RS, si[i].x);
                            acc2(any, two, S[i]);
                        }
                        if (kCheck) or4(anyR, lit4(BR, RS, si[i].x));
                    }
                }
            }
            for (int i = kSweepCached; i < width; ++i) {
                const int2 sj = c.sweep_slot[lo + i];
                if (kForward && kCheck && GALOIS_SWEEP_XR256) {
                    uint4 x, r;
                    lit_xr(BX, RS, sj.x, x, r);
                    acc2(any, two, x);
                    or4(anyR, r);
                } else {
                    if (kForward) acc2(any, two, lit4(BX, RS, sj.x));
                    if (kCheck) or4(anyR, lit4(BR, RS, sj.x));
                }
            }
            if (kForward) {
#pragma unroll
                for (int i = 0; i < kSweepCached; ++i)
                    if (i < width) {
                        const uint4 s = S[i];
                        const uint32_t nm = 0u - (uint32_t)(si[i].x & 1);   // negative: stored complemented
                        const uint4 e = make_uint4((~any.x | (s.x & ~two.x)) ^ nm, (~any.y | (s.y & ~two.y)) ^ nm,
                                                   (~any.z | (s.z & ~two.z)) ^ nm, (~any.w | (s.w & ~two.w)) ^ nm);
                        st_e(Ecol + (size_t)si[i].y * 32, e, pol);
                    }
                for (int i = kSweepCached; i < width; ++i) {
                    const int2 sj = c.sweep_slot[lo + i];
                    const uint4 s = lit4(BX, RS, sj.x);
                    const uint32_t nm = 0u - (uint32_t)(sj.x & 1);
                    const uint4 e = make_uint4((~any.x | (s.x & ~two.x)) ^ nm, (~any.y | (s.y & ~two.y)) ^ nm,
                                               (~any.z | (s.z & ~two.z)) ^ nm, (~any.w | (s.w & ~two.w)) ^ nm);
                    st_e(Ecol + (size_t)sj.y * 32, e, pol);
                }
            }
        }
        // U = ~any (clause unsatisfied); an absent clause (ci >= m) contributes 0
        if (kForward) butterfly_add(PL, make_uint4(~any.x, ~any.y, ~any.z, ~any.w), bm, cm);
        if (kCheck) butterfly_add(PU, make_uint4(~anyR.x, ~anyR.y, ~anyR.z, ~anyR.w), bm, cm);
        if (++since == SweepShape<kWide>::kFlushGroups) {                // warp-uniform: counts stay below 2^kPlanes
            if (kForward) flush_planes(PL, s_lam, vl * 4 + sub);
            if (kCheck) flush_planes(PU, s_uns, vl * 4 + sub);
            since = 0;
        }
    }
    if (kForward) flush_planes(PL, s_lam, vl * 4 + sub);
    if (kCheck) flush_planes(PU, s_uns, vl * 4 + sub);
    __syncthreads();
    const int base = chunk * 1024;
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) {
        const int mb = base + member_of_slot(i);       // i = word * 32 + bit position
        if (mb >= b_pad) continue;
        if (kForward && s_lam[i] != 0) atomicAdd(&lam[mb], s_lam[i]);
        if (kCheck && s_uns[i] != 0) atomicAdd(&unsat[mb], s_uns[i]);
    }
    if (kLoop) __syncthreads();                       // s_lam / s_uns are reused by the next chunk
    }                                                 // chunk loop
    if (kCheck) {
        __shared__ bool s_last;
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            s_last = atomicAdd(&ctrl->done_ctas, 1u) == gridDim.x * gridDim.y - 1u;
        }
        __syncthreads();
        if (s_last) {
            __threadfence();
            block_best(unsat, ba.unsat_last, ba.b_loc, ba.b0, ctrl, ba.finalize != 0);
            if (threadIdx.x == 0) ctrl->done_ctas = 0;
            if (ba.extract_n > 0) {
                __syncthreads();
                if (__ldcg(&ctrl->improved)) {
                    const int64_t lb = ctrl->best_b - ba.b0;
#pragma unroll 8
                    for (int32_t v = threadIdx.x; v < ba.extract_n; v += blockDim.x)
                        ba.best_bits[v] =
                            (uint8_t)((R[xr_at(v, (int32_t)(lb >> 5), ba.W)] >> bitpos((int)(lb & 31))) & 1u);
                }
            }
        }
    }
}

// ---------------------------------------------------------------------------------------
// k_sweep_tma: the same sweep (W % 32 == 0) with the clause index staged in shared memory.
//
// The grid-stride k_sweep chains two dependent global loads per literal (slot index ->
// X/R row gather); on C4 (sweep index 124 MB, X/R 256 MB: neither L2-resident) the first
// one is a DRAM round trip on the critical path of every group. Here a producer warp
// bulk-copies (cp.async.bulk, TMA) each 32-clause tile's offsets (33 of the sweep-ordered
// CSR) and its slots {code, CSC position} into a ring of kSwStages shared-memory stages,
// kSwStages tiles ahead of the 8 consumer warps (full / empty mbarriers); a consumer
// warp takes one 4-clause group of each tile (8 lanes x 32 B per clause: the X and R
// vectors of 128 members of a literal are one 32-B sector, fetched by ONE 256-bit load)
// and issues the row gathers of up to 4 literals back to back. Tiles whose slots exceed
// a stage (clauses wider than 16 on average) read their slots from global memory.
// E is stored with an L2 evict-first policy when it cannot stay L2-resident for the update
// (C4: 2 GB), so the streaming E and index traffic does not displace the X/R rows.
#ifndef GALOIS_SWEEP_TMA
#define GALOIS_SWEEP_TMA 1      // 0: k_sweep everywhere; 1: k_sweep_tma for the chunk loop; 2: always
#endif
#ifndef GALOIS_SWEEP_HINT
#define GALOIS_SWEEP_HINT 1
#endif
namespace {
#ifndef GALOIS_SW_WARPS
#define GALOIS_SW_WARPS 8
#endif
constexpr int kSwWarps = GALOIS_SW_WARPS;   // consumer warps (one 4-clause group per tile each)
constexpr int kSwTile = 4 * kSwWarps;       // clauses per staged tile
#ifndef GALOIS_SW_STAGES
#define GALOIS_SW_STAGES 6
#endif
#ifndef GALOIS_SW_CTAS
#define GALOIS_SW_CTAS 2
#endif
constexpr int kSwStages = GALOIS_SW_STAGES;
constexpr int kSwCap = 512;                 // slots per stage
constexpr int kSwOffBytes = ((kSwTile + 1) * 4 + 15) & ~15;   // the tile's kSwTile + 1 offsets
static_assert(kSwOffBytes / 4 <= kSweepOffPad, "sweep_off padding must cover a whole tile copy");
constexpr int kSwStageBytes = kSwOffBytes + kSwCap * 8;
constexpr int kSwSmem = kSwStages * kSwStageBytes;
static_assert(kSwStageBytes % 16 == 0, "bulk copy destinations must stay 16-B aligned");

__device__ __forceinline__ uint4 exclusive4(uint4 s, uint4 any, uint4 two, uint32_t nm)
{
    return make_uint4((~any.x | (s.x & ~two.x)) ^ nm, (~any.y | (s.y & ~two.y)) ^ nm,
                      (~any.z | (s.z & ~two.z)) ^ nm, (~any.w | (s.w & ~two.w)) ^ nm);
}

__device__ __forceinline__ void neg4(uint4 &s, uint32_t nm)
{
    s.x ^= nm; s.y ^= nm; s.z ^= nm; s.w ^= nm;
}

// literal values (row xor sign mask), zeroed for an absent literal (keep = 0)
__device__ __forceinline__ void mask4(uint4 &s, uint32_t nm, uint32_t keep)
{
    s.x = (s.x ^ nm) & keep; s.y = (s.y ^ nm) & keep; s.z = (s.z ^ nm) & keep; s.w = (s.w ^ nm) & keep;
}

__device__ __forceinline__ int32_t ld_volatile_pos(const int2 *p)
{
    return *reinterpret_cast<const volatile int32_t *>(&p->y);
}

// One batch of up to 4 literals of a clause (`left` >= 1 remain from sl): their X/R rows
// gathered back to back (indices clamped to the last literal, values of absent ones masked
// to 0), accumulated into any / two (forward) and anyR (check). x / code return the batch.
template <bool kForward, bool kCheck>
__device__ __forceinline__ void sweep_batch(const int2 *sl, int32_t left, const uint4 *BX, const uint4 *BR, int RS,
                                            uint4 &any, uint4 &two, uint4 &anyR, uint4 (&x)[4], int32_t (&code)[4])
{
    uint4 r[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) code[j] = sl[min(j, left - 1)].x;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const size_t row = (size_t)(code[j] >> 1) * RS;
        if (kForward && kCheck)
            ld_xr(BX + row, x[j], r[j]);
        else if (kForward)
            x[j] = __ldg(BX + row);
        else
            r[j] = __ldg(BR + row);
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const uint32_t keep = j < left ? 0xffffffffu : 0u, nm = 0u - (uint32_t)(code[j] & 1);
        if (kForward) {
            mask4(x[j], nm, keep);
            acc2(any, two, x[j]);
        }
        if (kCheck) {
            mask4(r[j], nm, keep);
            or4(anyR, r[j]);
        }
    }
}
}  // namespace

template <bool kForward, bool kCheck, bool kWide, bool kLoop>
__global__ void __launch_bounds__(32 * (kSwWarps + 1), GALOIS_SW_CTAS)
    k_sweep_tma(DevCnf c, int32_t W, int32_t b_pad, const uint32_t *__restrict__ X, const uint32_t *__restrict__ R,
                uint32_t *__restrict__ E, int32_t *__restrict__ lam, int32_t *__restrict__ unsat,
                Ctrl *__restrict__ ctrl, BestArgs ba, int32_t stream_hint)
{
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ uint64_t full[kSwStages], empty[kSwStages];
    __shared__ int32_t s_lam[kForward ? 1024 : 1];
    __shared__ int32_t s_uns[kCheck ? 1024 : 1];
    if (ctrl->stopped) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int32_t ntiles = (c.m + kSwTile - 1) / kSwTile;
    const int chunk_end = kLoop ? W / 32 : (int)blockIdx.y + 1;
    const uint32_t full_s = smem_u32(full), empty_s = smem_u32(empty), stage_s = smem_u32(smem);
    if (tid == 0) {
        for (int i = 0; i < kSwStages; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 32 * kSwWarps);   // every consumer thread releases the stage
        }
        fence_mbar_init();
    }
    __syncthreads();

    if (warp == kSwWarps) {                // ----------------------------------- producer warp
        const uint64_t pol = l2_policy(stream_hint != 0);
        uint32_t slot = 0;
        for (int chunk = blockIdx.y; chunk < chunk_end; chunk += gridDim.y) {
            for (int32_t t0 = blockIdx.x; t0 < ntiles; t0 += 32 * (int32_t)gridDim.x) {
                // lane j holds the slot range of this CTA's (t0 / gridDim.x + j)-th tile
                const int32_t tl = t0 + lane * (int32_t)gridDim.x;
                int32_t mylo = 0, myhi = 0;
                if (tl < ntiles) {
                    mylo = __ldg(c.sweep_off + (size_t)tl * kSwTile);
                    myhi = __ldg(c.sweep_off + (size_t)tl * kSwTile + kSwTile);
                }
                const int32_t cnt = min(32, (ntiles - t0 + (int32_t)gridDim.x - 1) / (int32_t)gridDim.x);
                for (int32_t j = 0; j < cnt; ++j, ++slot) {
                    const int32_t lo = __shfl_sync(0xffffffffu, mylo, j), hi = __shfl_sync(0xffffffffu, myhi, j);
                    if (lane == 0) {
                        const int32_t t = t0 + j * (int32_t)gridDim.x;
                        const int st = (int)(slot % kSwStages);
                        if (slot >= (uint32_t)kSwStages) {
                            mbar_wait_s(empty_s + 8u * st, ((slot / kSwStages) - 1u) & 1u);
                            fence_proxy_async_smem();
                        }
                        const int32_t a0 = lo & ~1, a1 = (hi + 1) & ~1;
                        const uint32_t nb = (a1 - a0 <= kSwCap) ? (uint32_t)(a1 - a0) * 8u : 0u;
                        const uint32_t fb = full_s + 8u * st, sb = stage_s + (uint32_t)(st * kSwStageBytes);
                        mbar_arrive_expect_tx_s(fb, (uint32_t)kSwOffBytes + nb);
                        bulk_g2s_s(sb, c.sweep_off + (size_t)t * kSwTile, (uint32_t)kSwOffBytes, fb);
                        if (nb) bulk_g2s_hint(sb + kSwOffBytes, c.sweep_slot + a0, nb, fb, pol);
                    }
                    __syncwarp();
                }
            }
        }
    } else {                               // -------------------------------- consumer warps
        const uint64_t pol = l2_policy(stream_hint != 0);
        const int sub = lane >> 3, vl = lane & 7;
        const uint32_t bm = 0u - (uint32_t)(sub & 1), cm = 0u - (uint32_t)((sub >> 1) & 1);
        const int RS = 2 * (W >> 2);                       // uint4 per interleaved X/R row
        constexpr int kPlanes = SweepShape<kWide>::kPlanes;
        uint32_t PL[kPlanes], PU[kPlanes];
#pragma unroll
        for (int k = 0; k < kPlanes; ++k) PL[k] = PU[k] = 0;
        uint32_t slot = 0;
        for (int chunk = blockIdx.y; chunk < chunk_end; chunk += gridDim.y) {
            for (int i = tid; i < 1024; i += 32 * kSwWarps) {
                if (kForward) s_lam[i] = 0;
                if (kCheck) s_uns[i] = 0;
            }
            asm volatile("bar.sync 1, %0;" ::"n"(kSwWarps * 32) : "memory");
            const int vw = chunk * 8 + vl;                 // this lane's 16-B vector word of a row
            uint32_t *Ecol = kForward ? E + (size_t)chunk * c.L * 32 + vl * 4 : nullptr;
            const uint4 *BX = reinterpret_cast<const uint4 *>(X) + 2 * vw;   // X vector; R = BX + 1
            const uint4 *BR = reinterpret_cast<const uint4 *>(R) + 2 * vw;   // R = X + 4 words
            int since = 0;
#pragma unroll 1
            for (int32_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++slot) {
                const int st = (int)(slot % kSwStages);
                mbar_wait_s(full_s + 8u * st, (slot / kSwStages) & 1u);
                const uint8_t *sb = smem + st * kSwStageBytes;
                const int32_t *so = reinterpret_cast<const int32_t *>(sb);
                const int32_t a0 = so[0] & ~1;
                const bool staged = ((so[kSwTile] + 1) & ~1) - a0 <= kSwCap;
                const int2 *sl = staged ? reinterpret_cast<const int2 *>(sb + kSwOffBytes) - a0 : c.sweep_slot;
                const int32_t ci = t * kSwTile + warp * 4 + sub;
                const int32_t lo = so[warp * 4 + sub], width = so[warp * 4 + sub + 1] - lo;
                uint4 any = make_uint4(0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu), anyR = any;
                if (ci < c.m) {
                    uint4 two = make_uint4(0, 0, 0, 0);
                    any = two;
                    anyR = two;
                    // batch 0: literals 0..3 (absent ones masked to 0); their X vectors are
                    // kept for E when the clause has at most 4 literals
                    uint4 x[4];
                    int32_t code[4];
                    sweep_batch<kForward, kCheck>(sl + lo, width, BX, BR, RS, any, two, anyR, x, code);
                    if (width <= 4) {
                        if (kForward) {
#pragma unroll
                            for (int j = 0; j < 4; ++j)
                                if (j < width)
                                    st_e(Ecol + (size_t)ld_volatile_pos(sl + lo + j) * 32,
                                         exclusive4(x[j], any, two, 0u - (uint32_t)(code[j] & 1)), pol);
                        }
                    } else {
#pragma unroll 1
                        for (int32_t i0 = 4; i0 < width; i0 += 4)
                            sweep_batch<kForward, kCheck>(sl + lo + i0, width - i0, BX, BR, RS, any, two, anyR, x,
                                                          code);
                        if (kForward) {
                            // E pass: the rows were just fetched (L1 hits); re-read in batches
#pragma unroll 1
                            for (int32_t i0 = 0; i0 < width; i0 += 4) {
                                int2 sj[4];
#pragma unroll
                                for (int j = 0; j < 4; ++j) sj[j] = sl[lo + min(i0 + j, width - 1)];
#pragma unroll
                                for (int j = 0; j < 4; ++j) x[j] = __ldg(BX + (size_t)(sj[j].x >> 1) * RS);
#pragma unroll
                                for (int j = 0; j < 4; ++j)
                                    if (i0 + j < width) {
                                        const uint32_t nm = 0u - (uint32_t)(sj[j].x & 1);
                                        neg4(x[j], nm);
                                        st_e(Ecol + (size_t)sj[j].y * 32, exclusive4(x[j], any, two, nm), pol);
                                    }
                            }
                        }
                    }
                }
                mbar_arrive_s(empty_s + 8u * st);   // this thread is done with the stage
                // U = ~any (clause unsatisfied); an absent clause (ci >= m) contributes 0
                if (kForward) butterfly_add(PL, make_uint4(~any.x, ~any.y, ~any.z, ~any.w), bm, cm);
                if (kCheck) butterfly_add(PU, make_uint4(~anyR.x, ~anyR.y, ~anyR.z, ~anyR.w), bm, cm);
                if (++since == SweepShape<kWide>::kFlushGroups) {   // warp-uniform
                    if (kForward) flush_planes(PL, s_lam, vl * 4 + sub);
                    if (kCheck) flush_planes(PU, s_uns, vl * 4 + sub);
                    since = 0;
                }
            }
            if (kForward) flush_planes(PL, s_lam, vl * 4 + sub);
            if (kCheck) flush_planes(PU, s_uns, vl * 4 + sub);
            asm volatile("bar.sync 1, %0;" ::"n"(kSwWarps * 32) : "memory");
            const int base = chunk * 1024;
            for (int i = tid; i < 1024; i += 32 * kSwWarps) {
                const int mb = base + member_of_slot(i);   // i = word * 32 + bit position
                if (mb >= b_pad) continue;
                if (kForward && s_lam[i] != 0) atomicAdd(&lam[mb], s_lam[i]);
                if (kCheck && s_uns[i] != 0) atomicAdd(&unsat[mb], s_uns[i]);
            }
            if (kLoop) asm volatile("bar.sync 1, %0;" ::"n"(kSwWarps * 32) : "memory");
        }
    }
    if (kCheck) {
        __shared__ bool s_last;
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            s_last = atomicAdd(&ctrl->done_ctas, 1u) == gridDim.x * gridDim.y - 1u;
        }
        __syncthreads();
        if (s_last) {
            __threadfence();
            block_best(unsat, ba.unsat_last, ba.b_loc, ba.b0, ctrl, ba.finalize != 0);
            if (threadIdx.x == 0) ctrl->done_ctas = 0;
            if (ba.extract_n > 0) {
                __syncthreads();
                if (__ldcg(&ctrl->improved)) {
                    const int64_t lb = ctrl->best_b - ba.b0;
#pragma unroll 8
                    for (int32_t v = threadIdx.x; v < ba.extract_n; v += blockDim.x)
                        ba.best_bits[v] =
                            (uint8_t)((R[xr_at(v, (int32_t)(lb >> 5), ba.W)] >> bitpos((int)(lb & 31))) & 1u);
                }
            }
        }
    }
}

namespace launch {

static dim3 clause_grid_v4(const DevCnf &c, int32_t W)
{
    const int VW = W / 4;
    const int LPC = VW < 32 ? VW : 32;
    const int CPW = 32 / LPC;
    const int64_t groups = ((int64_t)c.m + CPW - 1) / CPW;
    const unsigned chunks = (unsigned)((VW + 31) / 32);
    const int64_t want = (groups + 7) / 8;
    unsigned bx = (unsigned)(want < 1 ? 1 : want);
    // one resident wave (3 CTAs per SM): each warp sweeps many clause groups, so the
    // per-CTA shared-counter clear and flush (4096 members) is amortised
    const unsigned cap = (148u * 3u + chunks - 1) / chunks;
    if (bx > cap) bx = cap;
    return dim3(bx, chunks);
}

bool use_v4_clauses(int32_t W) { return W % 4 == 0; }



// X != null: forward of the sample X (E, lam); R != null: exact check of R (unsat).
void clauses_v4(const DevCnf &c, int32_t W, int32_t b_pad, const uint32_t *X, const uint32_t *R, uint32_t *E,
                int32_t *lam, int32_t *unsat, Ctrl *ctrl, const BestArgs &ba, cudaStream_t st)
{
    if (W % 32 == 0) {
        const bool wide = (int64_t)c.L >= (int64_t)c.m * 9 / 2;      // average width >= 4.5
        const unsigned chunks = (unsigned)(W / 32);
        // chunks in flight: their X and R slices (2 n 128 B each) within ~48 MB of L2
        const int64_t slice = 2 * (int64_t)c.n * 128;
        int64_t gy = (48ll << 20) / (slice > 0 ? slice : 1);
        if (gy < 1) gy = 1;
        if (gy > (int64_t)chunks) gy = chunks;
        const int64_t groups = ((int64_t)c.m + 3) / 4;
        int64_t bx = (groups + 7) / 8;
        const int64_t cap = ((wide ? 4 : GALOIS_SWEEP_CTAS) * 148 + gy - 1) / gy;
        if (bx > cap) bx = cap;
        if (bx < 1) bx = 1;
        const bool loop = gy < (int64_t)chunks;
        // E (and the staged sweep's index) stream through L2 with evict-first when E cannot
        // stay L2-resident until the update reads it (C4: 2 GB); a small E stays cached
        const int32_t hint = GALOIS_SWEEP_HINT && (int64_t)c.L * 128 * (int64_t)chunks > (64ll << 20) ? 1 : 0;
        if (GALOIS_SWEEP_TMA == 2 || (GALOIS_SWEEP_TMA == 1 && loop)) {
            // a 32-clause tile per consumer warp group; one resident wave of CTAs
            const int64_t tiles = ((int64_t)c.m + kSwTile - 1) / kSwTile;
            int64_t tx = (GALOIS_SW_CTAS * 148 + gy - 1) / gy;
            if (tx > tiles) tx = tiles;
            if (tx < 1) tx = 1;
            const dim3 tgrid((unsigned)tx, (unsigned)gy);
#define GALOIS_SWEEP_T(F, C)                                                                                       \
    (wide ? (loop ? k_sweep_tma<F, C, true, true><<<tgrid, 32 * (kSwWarps + 1), kSwSmem, st>>>(                    \
                        c, W, b_pad, X, R, E, lam, unsat, ctrl, ba, hint)                                          \
                  : k_sweep_tma<F, C, true, false><<<tgrid, 32 * (kSwWarps + 1), kSwSmem, st>>>(                   \
                        c, W, b_pad, X, R, E, lam, unsat, ctrl, ba, hint))                                         \
          : (loop ? k_sweep_tma<F, C, false, true><<<tgrid, 32 * (kSwWarps + 1), kSwSmem, st>>>(                   \
                        c, W, b_pad, X, R, E, lam, unsat, ctrl, ba, hint)                                          \
                  : k_sweep_tma<F, C, false, false><<<tgrid, 32 * (kSwWarps + 1), kSwSmem, st>>>(                  \
                        c, W, b_pad, X, R, E, lam, unsat, ctrl, ba, hint)))
            if (X && R)
                GALOIS_SWEEP_T(true, true);
            else if (X)
                GALOIS_SWEEP_T(true, false);
            else if (R)
                GALOIS_SWEEP_T(false, true);
#undef GALOIS_SWEEP_T
            return;
        }
        const dim3 grid((unsigned)bx, (unsigned)gy);
#define GALOIS_SWEEP(F, C)                                                                                \
    (wide ? (loop ? k_sweep<F, C, true, true><<<grid, 256, 0, st>>>(c, W, b_pad, X, R, E, lam, unsat, ctrl, ba, hint)  \
                  : k_sweep<F, C, true, false><<<grid, 256, 0, st>>>(c, W, b_pad, X, R, E, lam, unsat, ctrl, ba, hint)) \
          : (loop ? k_sweep<F, C, false, true><<<grid, 256, 0, st>>>(c, W, b_pad, X, R, E, lam, unsat, ctrl, ba, hint) \
                  : k_sweep<F, C, false, false><<<grid, 256, 0, st>>>(c, W, b_pad, X, R, E, lam, unsat, ctrl, ba, hint)))
        if (X && R)
            GALOIS_SWEEP(true, true);
        else if (X)
            GALOIS_SWEEP(true, false);
        else if (R)
            GALOIS_SWEEP(false, true);
#undef GALOIS_SWEEP
        return;
    }
    const dim3 grid = clause_grid_v4(c, W);
    if (X && R)
        k_clauses_v4<true, true><<<grid, 256, 0, st>>>(c, W, b_pad, X, R, E, lam, unsat, ctrl, ba);
    else if (X)
        k_clauses_v4<true, false><<<grid, 256, 0, st>>>(c, W, b_pad, X, R, E, lam, unsat, ctrl, ba);
    else if (R)
        k_clauses_v4<false, true><<<grid, 256, 0, st>>>(c, W, b_pad, X, R, E, lam, unsat, ctrl, ba);
}

}  // namespace launch
}  // namespace galois
