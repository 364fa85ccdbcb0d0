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

__device__ __forceinline__ void acc2(uint4 &any, uint4 &two, uint4 s)
{
    two.x |= any.x & s.x; two.y |= any.y & s.y; two.z |= any.z & s.z; two.w |= any.w & s.w;
    any.x |= s.x; any.y |= s.y; any.z |= s.z; any.w |= s.w;
}

__device__ __forceinline__ void or4(uint4 &any, uint4 s)
{
    any.x |= s.x; any.y |= s.y; any.z |= s.z; any.w |= s.w;
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
        const int32_t cl = c.clause_perm[ci];     // width-sorted order
        const int32_t lo = c.clause_off[cl], width = c.clause_off[cl + 1] - lo;
        uint4 any = make_uint4(0, 0, 0, 0), two = make_uint4(0, 0, 0, 0), anyR = make_uint4(0, 0, 0, 0);
        uint4 S[kCached];
        int2 si[kCached];
#pragma unroll
        for (int i = 0; i < kCached; ++i)
            if (i < width) si[i] = c.slot_info[lo + i];
#pragma unroll
        for (int i = 0; i < kCached; ++i) {
            if (i < width) {
                if (kForward) {
                    S[i] = lit4(BX, RS, si[i].x);
                    acc2(any, two, S[i]);
                }
                if (kCheck) or4(anyR, lit4(BR, RS, si[i].x));
            }
        }
        for (int i = kCached; i < width; ++i) {
            const int2 sj = c.slot_info[lo + i];
            if (kForward) acc2(any, two, lit4(BX, RS, sj.x));
            if (kCheck) or4(anyR, lit4(BR, RS, sj.x));
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
                const int2 sj = c.slot_info[lo + i];
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
                                               Ctrl *__restrict__ ctrl, BestArgs ba)
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
                    if (kForward) {
                        S[i] = lit4(BX, RS, si[i].x);
                        acc2(any, two, S[i]);
                    }
                    if (kCheck) or4(anyR, lit4(BR, RS, si[i].x));
                }
            }
            for (int i = kSweepCached; i < width; ++i) {
                const int2 sj = c.sweep_slot[lo + i];
                if (kForward) acc2(any, two, lit4(BX, RS, sj.x));
                if (kCheck) or4(anyR, lit4(BR, RS, sj.x));
            }
            if (kForward) {
#pragma unroll
                for (int i = 0; i < kSweepCached; ++i)
                    if (i < width) {
                        const uint4 s = S[i];
                        const uint32_t nm = 0u - (uint32_t)(si[i].x & 1);   // negative: stored complemented
                        const uint4 e = make_uint4((~any.x | (s.x & ~two.x)) ^ nm, (~any.y | (s.y & ~two.y)) ^ nm,
                                                   (~any.z | (s.z & ~two.z)) ^ nm, (~any.w | (s.w & ~two.w)) ^ nm);
                        *reinterpret_cast<uint4 *>(Ecol + (size_t)si[i].y * 32) = e;
                    }
                for (int i = kSweepCached; i < width; ++i) {
                    const int2 sj = c.sweep_slot[lo + i];
                    const uint4 s = lit4(BX, RS, sj.x);
                    const uint32_t nm = 0u - (uint32_t)(sj.x & 1);
                    const uint4 e = make_uint4((~any.x | (s.x & ~two.x)) ^ nm, (~any.y | (s.y & ~two.y)) ^ nm,
                                               (~any.z | (s.z & ~two.z)) ^ nm, (~any.w | (s.w & ~two.w)) ^ nm);
                    *reinterpret_cast<uint4 *>(Ecol + (size_t)sj.y * 32) = e;
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
        const dim3 grid((unsigned)bx, (unsigned)gy);
        const bool loop = gy < (int64_t)chunks;
#define GALOIS_SWEEP(F, C)                                                                                   \
    (wide ? (loop ? k_sweep<F, C, true, true><<<grid, 256, 0, st>>>(c, W, b_pad, X, R, E, lam, unsat, ctrl, ba)  \
                  : k_sweep<F, C, true, false><<<grid, 256, 0, st>>>(c, W, b_pad, X, R, E, lam, unsat, ctrl, ba)) \
          : (loop ? k_sweep<F, C, false, true><<<grid, 256, 0, st>>>(c, W, b_pad, X, R, E, lam, unsat, ctrl, ba) \
                  : k_sweep<F, C, false, false><<<grid, 256, 0, st>>>(c, W, b_pad, X, R, E, lam, unsat, ctrl, ba)))
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
