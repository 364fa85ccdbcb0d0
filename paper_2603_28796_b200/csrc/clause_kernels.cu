// clause_kernels.cu — rows a5 (clause-polynomial forward) and a8 (exact checker),
// vectorised: each lane owns 4 consecutive batch words (16 B = 128 members) of a row.
//
// For clause c and a lane's 4 words, with S_i = X[v_i] xor negmask_i (literal true):
//   any = OR_i S_i, two = OR_{i<j} (S_i AND S_j)   (>= 1 / >= 2 literals true)
//   U   = ~any                      = prod_i (1 - s_i)          (Eq.2, clause unsatisfied)
//   E_i = ~any | (S_i & ~two)       = prod_{j != i} (1 - s_j)   (exclusive products)
// E is written in CSC order into the chunk-major layout E[chunk][pos][32] that the update
// kernel reads with one TMA bulk copy per (variable, chunk). Per-member counts of U (the
// ST loss Lambda in the forward, the exact unsat counts in the checker) are accumulated in
// shared memory and added to global memory once per block (integer, deterministic).
//
// Lane layout: LPC = min(W/4, 32) lanes per clause (16 B each, 128 B per 8 lanes:
// coalesced row segments), CPW = 32 / LPC clauses in flight per warp, blockIdx.y selects
// 128-word column chunks. Requires W % 4 == 0.
#include <cuda_runtime.h>

#include <cstdint>

#include "device_utils.cuh"
#include "galois_internal.h"

namespace galois {

namespace {
constexpr int kCached = 3;   // slots kept in registers between the two passes (rest re-gathered)
}

template <bool kForward>
__global__ void __launch_bounds__(256, 4) k_clauses_v4(DevCnf c, int32_t W, int32_t b_pad,
                                                    const uint32_t *__restrict__ bits, uint32_t *__restrict__ E,
                                                    int32_t *__restrict__ cnt, Ctrl *__restrict__ ctrl)
{
    __shared__ int32_t s_cnt[4096];          // members of this block's 128-word chunk
    if (ctrl->stopped) return;
    if (kForward && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) ctrl->t += 1;
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) s_cnt[i] = 0;
    __syncthreads();

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int VW = W >> 2;                    // 16-B vector words per row
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
    uint32_t *Ecol = E ? E + (size_t)ch * c.L * CW + wi : nullptr;
    const uint4 *B = reinterpret_cast<const uint4 *>(bits) + vw;

    for (int64_t g = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp; g < ngroups; g += stride) {
        const int64_t ci = g * CPW + sub;
        if (!lane_ok || ci >= c.m) continue;
        const int32_t cl = c.clause_perm[ci];     // width-sorted order
        const int32_t lo = c.clause_off[cl], width = c.clause_off[cl + 1] - lo;
        uint4 any = make_uint4(0, 0, 0, 0), two = make_uint4(0, 0, 0, 0);
        uint4 S[kCached];
        int2 si[kCached];
#pragma unroll
        for (int i = 0; i < kCached; ++i)
            if (i < width) si[i] = c.slot_info[lo + i];
#pragma unroll
        for (int i = 0; i < kCached; ++i) {
            if (i < width) {
                const uint32_t neg = 0u - (uint32_t)(si[i].x & 1);
                uint4 s = B[(size_t)(si[i].x >> 1) * VW];
                s.x ^= neg; s.y ^= neg; s.z ^= neg; s.w ^= neg;
                S[i] = s;
                two.x |= any.x & s.x; two.y |= any.y & s.y; two.z |= any.z & s.z; two.w |= any.w & s.w;
                any.x |= s.x; any.y |= s.y; any.z |= s.z; any.w |= s.w;
            }
        }
        for (int i = kCached; i < width; ++i) {
            if (!kForward && (any.x & any.y & any.z & any.w) == 0xFFFFFFFFu) break;   // all satisfied
            const int2 sj = c.slot_info[lo + i];
            const uint32_t neg = 0u - (uint32_t)(sj.x & 1);
            uint4 s = B[(size_t)(sj.x >> 1) * VW];
            s.x ^= neg; s.y ^= neg; s.z ^= neg; s.w ^= neg;
            two.x |= any.x & s.x; two.y |= any.y & s.y; two.z |= any.z & s.z; two.w |= any.w & s.w;
            any.x |= s.x; any.y |= s.y; any.z |= s.z; any.w |= s.w;
        }
        if (kForward) {
#pragma unroll
            for (int i = 0; i < kCached; ++i)
                if (i < width) {
                    const uint4 s = S[i];
                    const uint4 e = make_uint4(~any.x | (s.x & ~two.x), ~any.y | (s.y & ~two.y),
                                               ~any.z | (s.z & ~two.z), ~any.w | (s.w & ~two.w));
                    *reinterpret_cast<uint4 *>(Ecol + (size_t)si[i].y * CW) = e;
                }
            for (int i = kCached; i < width; ++i) {
                const int2 sj = c.slot_info[lo + i];
                const uint32_t neg = 0u - (uint32_t)(sj.x & 1);
                uint4 s = B[(size_t)(sj.x >> 1) * VW];
                s.x ^= neg; s.y ^= neg; s.z ^= neg; s.w ^= neg;
                const uint4 e = make_uint4(~any.x | (s.x & ~two.x), ~any.y | (s.y & ~two.y),
                                           ~any.z | (s.z & ~two.z), ~any.w | (s.w & ~two.w));
                *reinterpret_cast<uint4 *>(Ecol + (size_t)sj.y * CW) = e;
            }
        }
        const uint32_t U[4] = {~any.x, ~any.y, ~any.z, ~any.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            uint32_t u = U[k];
            while (u) {
                const int j = __ffs(u) - 1;
                atomicAdd(&s_cnt[((vl << 2) + k) * 32 + j], 1);
                u &= u - 1;
            }
        }
    }
    __syncthreads();
    const int base = blockIdx.y * 4096;
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) {
        const int32_t v = s_cnt[i];
        if (v != 0 && base + i < b_pad) atomicAdd(&cnt[base + i], v);
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
    const unsigned cap = (148u * 8u * 4u + chunks - 1) / chunks;   // ~4 waves of 8 blocks/SM
    if (bx > cap) bx = cap;
    return dim3(bx, chunks);
}

bool use_v4_clauses(int32_t W) { return W % 4 == 0; }

void forward_v4(const DevCnf &c, int32_t W, int32_t b_pad, const uint32_t *X, uint32_t *E, int32_t *lam,
                Ctrl *ctrl, cudaStream_t st)
{
    k_clauses_v4<true><<<clause_grid_v4(c, W), 256, 0, st>>>(c, W, b_pad, X, E, lam, ctrl);
}

void check_v4(const DevCnf &c, int32_t W, int32_t b_pad, const uint32_t *R, int32_t *unsat, Ctrl *ctrl,
              cudaStream_t st)
{
    k_clauses_v4<false><<<clause_grid_v4(c, W), 256, 0, st>>>(c, W, b_pad, R, nullptr, unsat, ctrl);
}

}  // namespace launch
}  // namespace galois
