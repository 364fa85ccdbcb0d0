// step_kernels.cu — rows a3, a5/a8 (small batches) and a8-a9 of SURVEY §8 (straight-
// through mode, the paper's).
//
//   k_init        a3  theta ~ N(0,1) -> z0 = theta_1 - theta_0 (Box-Muller, fp32), first
//                     sample X_1 and rounding R_0
//   k_resample        R_t and X_{t+1} from an injected iterate (set_iterate test hook)
//   k_clauses_st  a5/a8 the scalar clause sweep for batches whose word count W is not a
//                     multiple of 4 (b_pad < 1024 padded to 32): U = AND of false-literal
//                     words, exclusive products E = ~any | (S_i & ~atleast2) in CSC order
//                     (negative occurrences complemented), per-member counts of U; the
//                     forward of X and the check of R in one pass over the sweep order
//   k_best / k_gfinalize / k_extract  a8-a9 best tracking (local, over ranks) and the winner's bits
// (the sweep for b_pad >= 1024 is k_sweep in clause_kernels.cu, the update in
// update_kernels.cu)
//
// Thread mapping of the per-variable kernels: one thread per QUAD = 4 consecutive members
// of one variable row (float4 state loads, one Philox call per quad); 8 quads form one
// 32-bit word of the packed bits (member-in-word layout: device_utils.cuh bitpos).
#include <cuda_runtime.h>

#include <cstdint>

#include "device_utils.cuh"
#include "galois_internal.h"
#include "philox.cuh"

namespace galois {

// --------------------------------------------------------------------------- a3: init
__global__ void __launch_bounds__(256) k_init(StepParams p, float4 *__restrict__ z4, float4 *__restrict__ m4,
                                              float4 *__restrict__ v4, uint32_t *__restrict__ X,
                                              uint32_t *__restrict__ R)
{
    const int lane = threadIdx.x & 31;
    const uint32_t QW = (uint32_t)p.b_pad / 4u;               // a multiple of 8: whole words per 8 lanes
    // A CTA pass covers rpc rows: one row's quads across the CTA (QW >= 256, a multiple of
    // 256), or 256 / QW whole rows of QW quads (small sub-batch windows: b_pad = 32 would
    // otherwise leave 248 of 256 threads idle). Every lane runs the same passes (ballots).
    const uint32_t rpc = QW >= 256u ? 1u : 256u / QW;
    const uint32_t r_t = QW >= 256u ? 0u : threadIdx.x / QW;
    const uint32_t q_t = threadIdx.x - r_t * (QW >= 256u ? 0u : QW);
    for (int64_t base = (int64_t)blockIdx.x * rpc; base < p.n; base += (int64_t)gridDim.x * rpc)
    for (uint32_t q = q_t; q < (QW >= 256u ? QW : q_t + 1u); q += blockDim.x) {
        const int32_t v = (int32_t)base + (int32_t)r_t;
        const bool valid = r_t < rpc && v < p.n;            // uniform over each 8-lane group
        const int64_t bq = p.b0 + 4 * (int64_t)q;           // global index of member 0 of the quad
        float zz[4];
#pragma unroll
        for (int h = 0; h < 2; ++h) {                        // init counter (v, b/2, 0, 0)
            const uint4 w = philox4x32_10(make_uint4((uint32_t)v, (uint32_t)((bq >> 1) + h), 0u, 0u), p.keys);
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                // Box-Muller theta_0 = rho cos(2 pi u1), theta_1 = rho sin(2 pi u1), rho =
                // sqrt(-2 ln u0); z0 = theta_1 - theta_0 = sqrt(-4 ln u0) sin(pi (2 u1 - 1/4))
                // (sin a - cos a = sqrt2 sin(a - pi/4)): one sinpi, no cancellation, so fp32
                // keeps a few ulps of relative error (u0, 2 u1 - 1/4 are exact in binary32)
                const float u0 = uniform_f32(j ? w.z : w.x);
                const float u1 = uniform_f32(j ? w.w : w.y);
                zz[2 * h + j] = sqrtf(-4.0f * logf(u0)) * sinpif(fmaf(2.0f, u1, -0.25f));
            }
        }
        const uint4 wn = philox4x32_10(make_uint4((uint32_t)v, (uint32_t)(bq >> 2), 1u, 1u), p.keys);
        const uint32_t wv[4] = {wn.x, wn.y, wn.z, wn.w};
        uint32_t xn = 0, rn = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int pb = valid ? pinned_bit(p, v, bq + j) : -1;
            // X_1 = [z0 + logit u >= 0] (the sign of a = (z0 + ell) / tau does not depend on
            // tau > 0), without a logarithm: with e = exp(-|z0|), u - ub e >= 0 (z0 >= 0)
            // or u e - ub >= 0 (z0 < 0), as one FMA (the update's rewrite, update_kernels.cu)
            const float2 uu = unif_pair(wv[j]);
            const float e = exp_neg_abs(zz[j]);
            const bool r0 = zz[j] >= 0.0f;
            const float g = fmaf(-e, r0 ? uu.y : uu.x, r0 ? uu.x : uu.y);
            const uint32_t xb = pb >= 0 ? (uint32_t)pb : ((r0 ? g : -g) >= 0.0f ? 1u : 0u);
            const uint32_t rb = pb >= 0 ? (uint32_t)pb : (r0 ? 1u : 0u);
            xn |= xb << j;
            rn |= rb << j;
        }
        if (valid) {
            const size_t idx = (size_t)v * QW + q;
            GALOIS_DEV_CHECK(q < QW && v < p.n);
            z4[idx] = make_float4(zz[0], zz[1], zz[2], zz[3]);
            m4[idx] = make_float4(0.f, 0.f, 0.f, 0.f);
            v4[idx] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
        // every lane of the warp is here (same passes); groups of 8 lanes never straddle rows
        const uint32_t xw = pack_quads(xn, lane), rw = pack_quads(rn, lane);
        if (valid && (lane & 7) == 0) {
            X[xr_at(v, (int32_t)(q >> 3), p.W)] = xw;
            R[xr_at(v, (int32_t)(q >> 3), p.W)] = rw;
        }
    }
}

// Recompute R_t = [z >= 0] and X_{t+1} from the current z (after set_iterate).
__global__ void __launch_bounds__(256) k_resample(StepParams p, const float4 *__restrict__ z4,
                                                  uint32_t *__restrict__ X, uint32_t *__restrict__ R,
                                                  int32_t t_next)
{
    const int lane = threadIdx.x & 31;
    const uint32_t QW = (uint32_t)p.b_pad / 4u;               // a multiple of 8: whole words per 8 lanes
    // rows blockIdx.x, blockIdx.x + gridDim.x, ...; quads of a row across the CTA (no division)
    for (int32_t v = blockIdx.x; v < p.n; v += gridDim.x)
    for (uint32_t q = threadIdx.x; q < QW; q += blockDim.x) {
        const int64_t bq = p.b0 + 4 * (int64_t)q;
        const float4 z = z4[(size_t)v * QW + q];
        const float zz[4] = {z.x, z.y, z.z, z.w};
        const uint4 wn = philox4x32_10(make_uint4((uint32_t)v, (uint32_t)(bq >> 2), (uint32_t)t_next, 1u), p.keys);
        const uint32_t wv[4] = {wn.x, wn.y, wn.z, wn.w};
        uint32_t xn = 0, rn = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int pb = pinned_bit(p, v, bq + j);
            const float ell = logistic_from_word(wv[j]);
            xn |= (pb >= 0 ? (uint32_t)pb : (zz[j] + ell >= 0.0f ? 1u : 0u)) << j;
            rn |= (pb >= 0 ? (uint32_t)pb : (zz[j] >= 0.0f ? 1u : 0u)) << j;
        }
        // active lanes: whole 8-lane groups with q < QW (QW is a multiple of 8)
        const uint32_t qb = q & ~31u;
        const uint32_t act = QW - qb >= 32u ? 0xffffffffu : ((1u << (QW - qb)) - 1u);
        const uint32_t xw = pack_quads(xn, lane, act), rw = pack_quads(rn, lane, act);
        if ((lane & 7) == 0) {
            X[xr_at(v, (int32_t)(q >> 3), p.W)] = xw;
            R[xr_at(v, (int32_t)(q >> 3), p.W)] = rw;
        }
    }
}

// ------------------------------------------------------------- a5 / a8: clause kernels
template <bool kForward, bool kCheck>
__global__ void __launch_bounds__(256) k_clauses_st(DevCnf c, int32_t W, int32_t b_pad,
                                                    const uint32_t *__restrict__ X, const uint32_t *__restrict__ R,
                                                    uint32_t *__restrict__ E, int32_t *__restrict__ lam,
                                                    int32_t *__restrict__ unsat, Ctrl *__restrict__ ctrl)
{
    __shared__ int32_t s_lam[kForward ? 1024 : 1];
    __shared__ int32_t s_uns[kCheck ? 1024 : 1];
    if (ctrl->stopped) return;
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) {
        if (kForward) s_lam[i] = 0;
        if (kCheck) s_uns[i] = 0;
    }
    __syncthreads();

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int LW = W < 32 ? W : 32;
    const int CPW = 32 / LW;
    const int sub = lane / LW, wl = lane - sub * LW;
    const int word = blockIdx.y * 32 + wl;
    const bool lane_ok = sub < CPW && word < W;
    const int64_t ngroups = ((int64_t)c.m + CPW - 1) / CPW;
    const int64_t stride = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t g = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp; g < ngroups; g += stride) {
        const int64_t ci = g * CPW + sub;
        if (!lane_ok || ci >= c.m) continue;
        uint32_t Ux = 0, Ur = 0;         // U words of this lane's clause
        const int32_t lo = c.sweep_off[ci], width = c.sweep_off[ci + 1] - lo;
        uint32_t any = 0, two = 0;       // per member bit: >= 1 / >= 2 literals of X true
        uint32_t anyR = 0;               // >= 1 literal of R true
        // literals in batches of 4, loads issued back to back (index clamped to the last
        // literal, an absent literal masked to 0): under `if (i < width)` each gather waited
        // for the previous one; the first batch's X words are kept for E
        uint32_t S[4];
        int2 s0[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) s0[j] = c.sweep_slot[lo + min(j, width - 1)];
        {
            uint32_t xv[4], rv[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const size_t at = xr_at(s0[j].x >> 1, word, W);
                if (kForward) xv[j] = X[at];
                if (kCheck) rv[j] = R[at];
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint32_t keep = j < width ? 0xFFFFFFFFu : 0u, nm = 0u - (uint32_t)(s0[j].x & 1);
                if (kForward) {
                    const uint32_t sv = (xv[j] ^ nm) & keep;
                    S[j] = sv;
                    two |= any & sv;
                    any |= sv;
                }
                if (kCheck) anyR |= (rv[j] ^ nm) & keep;
            }
        }
        for (int i0 = 4; i0 < width; i0 += 4) {
            if (!kForward && anyR == 0xFFFFFFFFu) break;   // every member already satisfied
            int2 sj[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) sj[j] = c.sweep_slot[lo + min(i0 + j, width - 1)];
            uint32_t xv[4], rv[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const size_t at = xr_at(sj[j].x >> 1, word, W);
                if (kForward) xv[j] = X[at];
                if (kCheck) rv[j] = R[at];
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint32_t keep = i0 + j < width ? 0xFFFFFFFFu : 0u, nm = 0u - (uint32_t)(sj[j].x & 1);
                if (kForward) {
                    const uint32_t sv = (xv[j] ^ nm) & keep;
                    two |= any & sv;
                    any |= sv;
                }
                if (kCheck) anyR |= (rv[j] ^ nm) & keep;
            }
        }
        if (kForward) {
            // E_i = prod_{j != i} (1 - s_j): all other literals false <=> none true, or
            // exactly one true and it is i. Chunk-major layout E[chunk][csc position][LW];
            // rows of negative occurrences are stored complemented (galois_internal.h).
            uint32_t *Ec = E + (size_t)blockIdx.y * c.L * LW + wl;
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (j < width) Ec[(size_t)s0[j].y * LW] = (~any | (S[j] & ~two)) ^ (0u - (uint32_t)(s0[j].x & 1));
            for (int i0 = 4; i0 < width; i0 += 4) {
                int2 sj[4];
                uint32_t xv[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) sj[j] = c.sweep_slot[lo + min(i0 + j, width - 1)];
#pragma unroll
                for (int j = 0; j < 4; ++j) xv[j] = X[xr_at(sj[j].x >> 1, word, W)];
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (i0 + j < width) {
                        const uint32_t nm = 0u - (uint32_t)(sj[j].x & 1);
                        Ec[(size_t)sj[j].y * LW] = (~any | ((xv[j] ^ nm) & ~two)) ^ nm;
                    }
            }
            Ux = ~any;                      // U = prod_i (1 - s_i): clause unsatisfied
        }
        if (kCheck) Ur = ~anyR;
        if (kForward)
            for (uint32_t U = Ux; U; U &= U - 1) atomicAdd(&s_lam[wl * 32 + __ffs(U) - 1], 1);
        if (kCheck)
            for (uint32_t U = Ur; U; U &= U - 1) atomicAdd(&s_uns[wl * 32 + __ffs(U) - 1], 1);
    }
    __syncthreads();
    const int base = blockIdx.y * 1024;
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) {
        const int mb = member_of_slot(i);                 // i = word * 32 + bit position
        if (base + mb >= b_pad) continue;
        if (kForward && s_lam[i] != 0) atomicAdd(&lam[base + mb], s_lam[i]);
        if (kCheck && s_uns[i] != 0) atomicAdd(&unsat[base + mb], s_uns[i]);
    }
}

// ------------------------------------------------------------------- a8/a9: best
// Single block: min over local members of (u << 32 | global b), and this rank's best record.
__global__ void __launch_bounds__(1024) k_best(const int32_t *__restrict__ unsat, int32_t *__restrict__ unsat_last,
                                               int32_t b_loc, int64_t b0, Ctrl *__restrict__ ctrl, int32_t finalize)
{
    if (ctrl->stopped) return;
    block_best(unsat, unsat_last, b_loc, b0, ctrl, finalize != 0);
}

// NCCL exchange (a9), on the engine's exchange stream after the MIN all-reduce of check
// t's key: the global record improves only on a strictly smaller count (ties keep the
// earlier check, and within a check the key orders by global member), and a global count
// of 0 stops every rank. Never returns early: a rank stopped by its own SAT must still
// fold that check into the global record.
__global__ void k_gfinalize(Ctrl *__restrict__ ctrl)
{
    const unsigned long long key = ctrl->key_global;
    const int64_t u = (int64_t)(key >> 32);         // 2^32 - 1 when no rank has members
    if (u < (int64_t)ctrl->g_u) {
        ctrl->g_u = (int32_t)u;
        ctrl->g_t = ctrl->last_check_t;
        ctrl->g_b = (int64_t)(key & 0xFFFFFFFFull);
    }
    if (ctrl->g_u == 0) ctrl->stopped = 1;
}

// Copy the rounding column of the new best member (only when it improved on this rank).
__global__ void k_extract(const uint32_t *__restrict__ R, int32_t n, int32_t W, int64_t b0,
                          const Ctrl *__restrict__ ctrl, uint8_t *__restrict__ best_bits)
{
    if (!ctrl->improved) return;
    const int64_t lb = ctrl->best_b - b0;
    for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
        best_bits[v] = (uint8_t)((R[xr_at(v, (int32_t)(lb >> 5), W)] >> bitpos((int)(lb & 31))) & 1u);
}

// One member's sample and rounding bits (test hook galois_engine_get_member).
__global__ void k_member_bits(const uint32_t *__restrict__ X, int32_t n, int32_t W, int32_t lb,
                              uint8_t *__restrict__ x_out, uint8_t *__restrict__ r_out)
{
    const size_t w = (size_t)(lb >> 5);
    const int bit = bitpos(lb & 31);
    for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
        const size_t at = xr_at(v, (int32_t)w, W);
        if (x_out) x_out[v] = (uint8_t)((X[at] >> bit) & 1u);
        if (r_out) r_out[v] = (uint8_t)((X[at + xr_roff(W)] >> bit) & 1u);   // R = X + xr_roff(W) words
    }
}

// ------------------------------------------------------------------ launch wrappers
namespace launch {

void member_bits(const uint32_t *X, int32_t n, int32_t W, int32_t lb, uint8_t *x_out, uint8_t *r_out, cudaStream_t st)
{
    k_member_bits<<<(n + 255) / 256 < 4096 ? (n + 255) / 256 : 4096, 256, 0, st>>>(X, n, W, lb, x_out, r_out);
}

static unsigned grid_cap(uint64_t work, unsigned threads, unsigned cap)
{
    uint64_t g = (work + threads - 1) / threads;
    if (g < 1) g = 1;
    if (g > cap) g = cap;
    return (unsigned)g;
}

void init(const StepParams &p, float *z, float *m, float *v, uint32_t *X, uint32_t *R, cudaStream_t st)
{
    const uint32_t QW = (uint32_t)p.b_pad / 4u, rpc = QW >= 256u ? 1u : 256u / QW;
    const int64_t passes = ((int64_t)p.n + rpc - 1) / rpc;
    const unsigned grid = (unsigned)(passes < 148 * 16 ? (passes > 0 ? passes : 1) : 148 * 16);
    k_init<<<grid, 256, 0, st>>>(p, (float4 *)z, (float4 *)m, (float4 *)v, X, R);
}

void resample(const StepParams &p, const float *z, uint32_t *X, uint32_t *R, int32_t t_next, cudaStream_t st)
{
    const uint64_t total = (uint64_t)p.n * (p.b_pad / 4);
    k_resample<<<grid_cap(total, 256, 148 * 16), 256, 0, st>>>(p, (const float4 *)z, X, R, t_next);
}

static dim3 clause_grid(const DevCnf &c, int32_t W)
{
    const int LW = W < 32 ? W : 32;
    const int CPW = 32 / LW;
    const int64_t groups = ((int64_t)c.m + CPW - 1) / CPW;
    const unsigned chunks = (unsigned)((W + 31) / 32);
    const int64_t want_blocks = (groups + 7) / 8;
    unsigned bx = (unsigned)(want_blocks < 1 ? 1 : want_blocks);
    const unsigned cap = (148u * 8u + chunks - 1) / chunks * 2;   // ~2 waves of 8 blocks/SM
    if (bx > cap) bx = cap;
    return dim3(bx, chunks);
}

bool use_v4_clauses(int32_t W);
void clauses_v4(const DevCnf &c, int32_t W, int32_t b_pad, const uint32_t *X, const uint32_t *R, uint32_t *E,
                int32_t *lam, int32_t *unsat, Ctrl *ctrl, const BestArgs &ba, cudaStream_t st);

// One sweep over the clauses: forward of the sample X (E, Lambda) when X != null and the
// exact check of the rounding R (unsat counts) when R != null. Returns true when the
// sweep also did the best tracking of the check in its last CTA (vectorised path);
// otherwise the caller launches k_best.
bool clauses(const DevCnf &c, int32_t W, int32_t b_pad, const uint32_t *X, const uint32_t *R, uint32_t *E,
             int32_t *lam, int32_t *unsat, Ctrl *ctrl, const BestArgs &ba, cudaStream_t st)
{
    if (use_v4_clauses(W)) {
        clauses_v4(c, W, b_pad, X, R, E, lam, unsat, ctrl, ba, st);
        return R != nullptr;
    }
    const dim3 grid = clause_grid(c, W);
    if (X && R)
        k_clauses_st<true, true><<<grid, 256, 0, st>>>(c, W, b_pad, X, R, E, lam, unsat, ctrl);
    else if (X)
        k_clauses_st<true, false><<<grid, 256, 0, st>>>(c, W, b_pad, X, nullptr, E, lam, nullptr, ctrl);
    else if (R)
        k_clauses_st<false, true><<<grid, 256, 0, st>>>(c, W, b_pad, nullptr, R, nullptr, nullptr, unsat, ctrl);
    return false;
}

void best(const int32_t *unsat, int32_t *unsat_last, int32_t b_loc, int64_t b0, Ctrl *ctrl, bool finalize,
          cudaStream_t st)
{
    k_best<<<1, 1024, 0, st>>>(unsat, unsat_last, b_loc, b0, ctrl, finalize ? 1 : 0);
}

void gfinalize(Ctrl *ctrl, cudaStream_t st)
{
    k_gfinalize<<<1, 1, 0, st>>>(ctrl);
}

void extract(const uint32_t *R, int32_t n, int32_t W, int64_t b0, const Ctrl *ctrl, uint8_t *best_bits,
             cudaStream_t st)
{
    k_extract<<<grid_cap((uint64_t)n, 256, 148 * 4), 256, 0, st>>>(R, n, W, b0, ctrl, best_bits);
}

}  // namespace launch
}  // namespace galois
