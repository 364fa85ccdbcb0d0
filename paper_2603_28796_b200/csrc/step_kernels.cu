// step_kernels.cu — rows a3-a8 of SURVEY §8 (straight-through mode, the paper's).
//
//   k_init        a3  theta ~ N(0,1) -> z0 = theta_1 - theta_0 (fp64 Box-Muller), first
//                     sample X_1 and rounding R_0
//   k_forward_st  a5  clause polynomial on bit-packed samples: U = AND of false-literal
//                     words, exclusive products E = ~any | (S_i & ~atleast2) written in CSC
//                     order, Lambda_b = popcount of U per member
//   k_hub_partial a6  deterministic chunked partial sums of the signal for hub variables
//   k_update_st   a6+a7 fused: per-variable segmented reduction of the signal G from E
//                     (no atomics), straight-through gradient, Adam, rounding R_t, next
//                     sample X_{t+1}
//   k_check       a8  exact checker on R: per-member unsat counts
//   k_best / k_finalize / k_extract  a8-a9 best tracking and the winner's bits
//
// Thread mapping of the per-variable kernels: one thread per QUAD = 4 consecutive members
// of one variable row (float4 state loads, one Philox call per quad); 8 quads form one
// 32-bit word of the packed bits. Clause kernels: one lane per (clause, batch word), the
// lanes of a warp reading consecutive words of the same variable row (128 B coalesced).
#include <cuda_runtime.h>

#include <cstdint>

#include "galois_internal.h"
#include "philox.cuh"

namespace galois {

namespace {

__device__ __forceinline__ uint32_t group8_mask(int lane) { return 0xFFu << (lane & 24); }

// OR the 4-bit nibbles of the 8 lanes that share one 32-bit word.
__device__ __forceinline__ uint32_t gather_word(uint32_t nib, int lane)
{
    const uint32_t mask = group8_mask(lane);
    uint32_t w = nib << (4 * (lane & 7));
    w |= __shfl_xor_sync(mask, w, 1);
    w |= __shfl_xor_sync(mask, w, 2);
    w |= __shfl_xor_sync(mask, w, 4);
    return w;
}

// 4 bits -> four 8-bit counters (bit i -> byte i).
__device__ __forceinline__ uint32_t spread4(uint32_t nib) { return (nib * 0x00204081u) & 0x01010101u; }

__device__ __forceinline__ int pinned_bit(const StepParams &p, int32_t v, int64_t b_global)
{
    if (p.pin_rank == nullptr) return -1;
    const int r = p.pin_rank[v];
    return r < 0 ? -1 : (int)((b_global >> r) & 1);
}

}  // namespace

// --------------------------------------------------------------------------- a3: init
__global__ void __launch_bounds__(256) k_init(StepParams p, float4 *__restrict__ z4, float4 *__restrict__ m4,
                                              float4 *__restrict__ v4, uint32_t *__restrict__ X,
                                              uint32_t *__restrict__ R)
{
    const int lane = threadIdx.x & 31;
    const uint32_t QW = (uint32_t)p.b_pad / 4u;
    const uint64_t total = (uint64_t)p.n * QW;
    const uint2 key = make_uint2((uint32_t)p.seed, (uint32_t)(p.seed >> 32));
    for (uint64_t flat = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; flat < total;
         flat += (uint64_t)gridDim.x * blockDim.x) {
        const int32_t v = (int32_t)(flat / QW);
        const uint32_t q = (uint32_t)(flat - (uint64_t)v * QW);
        const int64_t bq = p.b0 + 4 * (int64_t)q;           // global index of member 0 of the quad
        float zz[4];
#pragma unroll
        for (int h = 0; h < 2; ++h) {                        // init counter (v, b/2, 0, 0)
            const uint4 w = philox4x32_10(make_uint4((uint32_t)v, (uint32_t)((bq >> 1) + h), 0u, 0u), key);
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const double u0 = uniform_f64(j ? w.z : w.x);
                const double u1 = uniform_f64(j ? w.w : w.y);
                const double rho = sqrt(-2.0 * log(u0));
                double s, c;
                sincospi(2.0 * u1, &s, &c);
                zz[2 * h + j] = (float)(rho * s - rho * c);  // theta_1 - theta_0
            }
        }
        const uint4 wn = philox4x32_10(make_uint4((uint32_t)v, (uint32_t)(bq >> 2), 1u, 1u), key);
        const uint32_t wv[4] = {wn.x, wn.y, wn.z, wn.w};
        uint32_t xn = 0, rn = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int pb = pinned_bit(p, v, bq + j);
            const float ell = logistic_from_word(wv[j]);
            const uint32_t xb = pb >= 0 ? (uint32_t)pb : (zz[j] + ell >= 0.0f ? 1u : 0u);
            const uint32_t rb = pb >= 0 ? (uint32_t)pb : (zz[j] >= 0.0f ? 1u : 0u);
            xn |= xb << j;
            rn |= rb << j;
        }
        const size_t idx = (size_t)v * QW + q;
        z4[idx] = make_float4(zz[0], zz[1], zz[2], zz[3]);
        m4[idx] = make_float4(0.f, 0.f, 0.f, 0.f);
        v4[idx] = make_float4(0.f, 0.f, 0.f, 0.f);
        const uint32_t xw = gather_word(xn, lane), rw = gather_word(rn, lane);
        if ((lane & 7) == 0) {
            X[(size_t)v * p.W + (q >> 3)] = xw;
            R[(size_t)v * p.W + (q >> 3)] = rw;
        }
    }
}

// Recompute R_t = [z >= 0] and X_{t+1} from the current z (after set_iterate).
__global__ void __launch_bounds__(256) k_resample(StepParams p, const float4 *__restrict__ z4,
                                                  uint32_t *__restrict__ X, uint32_t *__restrict__ R,
                                                  int32_t t_next)
{
    const int lane = threadIdx.x & 31;
    const uint32_t QW = (uint32_t)p.b_pad / 4u;
    const uint64_t total = (uint64_t)p.n * QW;
    const uint2 key = make_uint2((uint32_t)p.seed, (uint32_t)(p.seed >> 32));
    for (uint64_t flat = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; flat < total;
         flat += (uint64_t)gridDim.x * blockDim.x) {
        const int32_t v = (int32_t)(flat / QW);
        const uint32_t q = (uint32_t)(flat - (uint64_t)v * QW);
        const int64_t bq = p.b0 + 4 * (int64_t)q;
        const float4 z = z4[(size_t)v * QW + q];
        const float zz[4] = {z.x, z.y, z.z, z.w};
        const uint4 wn = philox4x32_10(make_uint4((uint32_t)v, (uint32_t)(bq >> 2), (uint32_t)t_next, 1u), key);
        const uint32_t wv[4] = {wn.x, wn.y, wn.z, wn.w};
        uint32_t xn = 0, rn = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int pb = pinned_bit(p, v, bq + j);
            const float ell = logistic_from_word(wv[j]);
            xn |= (pb >= 0 ? (uint32_t)pb : (zz[j] + ell >= 0.0f ? 1u : 0u)) << j;
            rn |= (pb >= 0 ? (uint32_t)pb : (zz[j] >= 0.0f ? 1u : 0u)) << j;
        }
        const uint32_t xw = gather_word(xn, lane), rw = gather_word(rn, lane);
        if ((lane & 7) == 0) {
            X[(size_t)v * p.W + (q >> 3)] = xw;
            R[(size_t)v * p.W + (q >> 3)] = rw;
        }
    }
}

// ------------------------------------------------------------- a5 / a8: clause kernels
// Lane layout: LW = min(W, 32) lanes per clause cover 32-word chunk blockIdx.y of the batch
// words; CPW = 32 / LW clauses per warp row. kForward: write E and count U of the sample
// X into cnt (Lambda). !kForward: count U of the rounding into cnt (exact unsat counts).
template <bool kForward>
__global__ void __launch_bounds__(256) k_clauses_st(DevCnf c, int32_t W, int32_t b_pad,
                                                    const uint32_t *__restrict__ bits,
                                                    uint32_t *__restrict__ E, int32_t *__restrict__ cnt,
                                                    Ctrl *__restrict__ ctrl)
{
    __shared__ int32_t s_cnt[1024];
    if (ctrl->stopped) return;
    if (kForward && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) ctrl->t += 1;
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) s_cnt[i] = 0;
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
        const int64_t cl = g * CPW + sub;
        if (!lane_ok || cl >= c.m) continue;
        const int32_t lo = c.clause_off[cl], width = c.clause_off[cl + 1] - lo;
        uint32_t any = 0, two = 0;       // per member bit: >= 1 / >= 2 literals true
        uint32_t S[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (i < width) {
                const int2 si = c.slot_info[lo + i];
                const uint32_t s = bits[(size_t)(si.x >> 1) * W + word] ^ (0u - (uint32_t)(si.x & 1));
                S[i] = s;
                two |= any & s;
                any |= s;
            }
        }
        for (int i = 8; i < width; ++i) {
            if (!kForward && any == 0xFFFFFFFFu) break;   // every member already satisfied
            const int2 si = c.slot_info[lo + i];
            const uint32_t s = bits[(size_t)(si.x >> 1) * W + word] ^ (0u - (uint32_t)(si.x & 1));
            two |= any & s;
            any |= s;
        }
        if (kForward) {
            // E_i = prod_{j != i} (1 - s_j): all other literals false <=> none true, or
            // exactly one true and it is i.
#pragma unroll
            for (int i = 0; i < 8; ++i)
                if (i < width) {
                    const int2 si = c.slot_info[lo + i];
                    E[(size_t)si.y * W + word] = ~any | (S[i] & ~two);
                }
            for (int i = 8; i < width; ++i) {
                const int2 si = c.slot_info[lo + i];
                const uint32_t s = bits[(size_t)(si.x >> 1) * W + word] ^ (0u - (uint32_t)(si.x & 1));
                E[(size_t)si.y * W + word] = ~any | (s & ~two);
            }
        }
        uint32_t U = ~any;                  // U = prod_i (1 - s_i): clause unsatisfied
        while (U) {
            const int j = __ffs(U) - 1;
            atomicAdd(&s_cnt[wl * 32 + j], 1);
            U &= U - 1;
        }
    }
    __syncthreads();
    const int base = blockIdx.y * 1024;
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) {
        const int32_t v = s_cnt[i];
        if (v != 0 && base + i < b_pad) atomicAdd(&cnt[base + i], v);
    }
}

// ------------------------------------------------ per-variable kernels: shared pieces
namespace {

constexpr int kBatch = 8;   // independent E loads in flight per thread

// Count the E bits of one quad (4 members: bits sh..sh+3 of word column `col`) over the
// occurrences [k0, k1), into four counters. Loads are issued kBatch at a time
// (predicated, independent) so one memory round trip covers a whole batch; four 8-bit
// counters live in one register (spread4) and are flushed before they can overflow.
__device__ __forceinline__ void count_bits(const uint32_t *__restrict__ col, int32_t W, int32_t k0, int32_t k1,
                                           int sh, int32_t sign, int32_t G[4])
{
    const uint32_t *ptr = col + (size_t)k0 * W;
    int32_t left = k1 - k0;
    while (left > 0) {
        int32_t blk = min(left, 248);              // 8-bit counters: <= 255 adds per flush
        left -= blk;
        uint32_t acc = 0;
        for (; blk >= kBatch; blk -= kBatch) {     // full batches: no predication
            uint32_t e[kBatch];
#pragma unroll
            for (int i = 0; i < kBatch; ++i) e[i] = __ldg(ptr + i * W);
            ptr += kBatch * W;
#pragma unroll
            for (int i = 0; i < kBatch; ++i) acc += spread4((e[i] >> sh) & 15u);
        }
        if (blk > 0) {                             // remainder, predicated
            uint32_t e[kBatch - 1];
#pragma unroll
            for (int i = 0; i < kBatch - 1; ++i) e[i] = i < blk ? __ldg(ptr + i * W) : 0u;
            ptr += blk * W;
#pragma unroll
            for (int i = 0; i < kBatch - 1; ++i) acc += spread4((e[i] >> sh) & 15u);
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) G[j] += sign * (int32_t)((acc >> (8 * j)) & 255u);
    }
}

struct ItemPos {
    uint32_t row;    // variable (or hub chunk)
    uint32_t q;      // quad within the row
    bool valid;
};

__device__ __forceinline__ ItemPos item_pos(const RowMap &rm, uint32_t item, uint32_t r_t, uint32_t q_t)
{
    const uint32_t grp = (uint32_t)(((uint64_t)__umulhi(item, rm.div_mul) + item) >> rm.div_shift);
    const uint32_t chunk = item - grp * rm.cpr;
    ItemPos ip;
    ip.row = grp * rm.R + r_t;
    ip.q = chunk * 256u + q_t;
    ip.valid = r_t < rm.R && ip.row < rm.rows && ip.q < rm.QW;
    return ip;
}

// Helpers of the tau = 1 path: with (u, ub = 1 - u) from unif_pair and e = exp(-|z|),
// sigma(z + logit(u)) sigma(-(z + logit(u))) = u ub e / (A + B e)^2 where
// (A, B) = (u, ub) if z >= 0 else (ub, u); and [z + logit(u) >= 0] <=> A >= B e (z >= 0)
// or B e >= A (z < 0). Exact rewrites of Eq.3 at tau = 1 with no logarithm.
__device__ __forceinline__ bool sample_bit_tau1(float z, float2 uu, float e)
{
    return z >= 0.0f ? (uu.x >= uu.y * e) : (uu.x * e >= uu.y);
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

}  // namespace

// --------------------------------------------------------------- a6: hub partial sums
// Row = hub chunk of <= kHubChunk occurrences of one variable; per quad, the signed count
// of E bits over the chunk (|value| <= 128 -> int16). Fixed chunk order = deterministic.
__global__ void __launch_bounds__(256) k_hub_partial(DevCnf c, int32_t W, RowMap rm, const uint32_t *__restrict__ E,
                                                     short4 *__restrict__ partial, const Ctrl *__restrict__ ctrl)
{
    if (ctrl->stopped) return;
    const uint32_t r_t = rm.QW >= 256 ? 0u : threadIdx.x / rm.QW;
    const uint32_t q_t = rm.QW >= 256 ? threadIdx.x : threadIdx.x - r_t * rm.QW;
    for (uint32_t item = blockIdx.x; item < rm.items; item += gridDim.x) {
        const ItemPos ip = item_pos(rm, item, r_t, q_t);
        if (!ip.valid) continue;
        const int2 info = c.hub_chunk[ip.row];                 // {variable, first CSC position}
        const int32_t split = c.code_off[2 * info.x + 1], end = c.code_off[2 * info.x + 2];
        const int32_t k1 = min(info.y + kHubChunk, end);
        const uint32_t *col = E + (ip.q >> 3);
        const int sh = 4 * (ip.q & 7);
        int32_t G[4] = {0, 0, 0, 0};
        count_bits(col, W, info.y, min(split, k1), sh, 1, G);
        count_bits(col, W, max(split, info.y), k1, sh, -1, G);
        partial[(size_t)ip.row * rm.QW + ip.q] = make_short4((short)G[0], (short)G[1], (short)G[2], (short)G[3]);
    }
}

// ------------------------------------------------------------ a6 + a7: fused update
// Per quad: G = sum over occurrences of sigma * E (CSC: positive codes, then negative),
// g1 = -G p q / tau (straight-through), Adam on the reduced iterate
// z = theta_1 - theta_0, rounding R_t = [z >= 0], next sample X_{t+1}.
template <bool kDebug, bool kTau1, bool kAdam, bool kPins>
__global__ void __launch_bounds__(256) k_update_st(DevCnf c, StepParams p, RowMap rm, float4 *__restrict__ z4,
                                                   float4 *__restrict__ m4, float4 *__restrict__ v4,
                                                   uint32_t *__restrict__ X, uint32_t *__restrict__ R,
                                                   const uint32_t *__restrict__ E,
                                                   const short4 *__restrict__ partial, Ctrl *__restrict__ ctrl,
                                                   int4 *__restrict__ dbg_G, float4 *__restrict__ dbg_g1)
{
    if (ctrl->stopped) return;
    const int32_t s = ctrl->t;                       // this step's index (t-1 -> t)
    const float2 ac = p.adam_consts[s];              // {2 lr / bc1, 1 / sqrt(bc2)}
    const int lane = threadIdx.x & 31;
    const uint32_t r_t = rm.QW >= 256 ? 0u : threadIdx.x / rm.QW;
    const uint32_t q_t = rm.QW >= 256 ? threadIdx.x : threadIdx.x - r_t * rm.QW;
    bool bad = false;
    for (uint32_t item = blockIdx.x; item < rm.items; item += gridDim.x) {
        const ItemPos ip = item_pos(rm, item, r_t, q_t);
        const int32_t v = (int32_t)ip.row;
        const uint32_t q = ip.q;
        uint32_t xn = 0, rn = 0;
        if (ip.valid) {
            const int64_t bq = p.b0 + 4 * (int64_t)q;
            const size_t idx = (size_t)v * rm.QW + q;
            const float4 z = z4[idx], m = m4[idx], vv = v4[idx];

            // --- a6: signal G of the 4 members
            int32_t G[4] = {0, 0, 0, 0};
            const int32_t hub = c.num_hubs > 0 ? c.hub_of_var[v] : -1;
            if (hub >= 0) {
                const int32_t c0 = c.hub_chunk_off[hub], c1 = c.hub_chunk_off[hub + 1];
                for (int32_t ch = c0; ch < c1; ++ch) {
                    const short4 pp = partial[(size_t)ch * rm.QW + q];
                    G[0] += pp.x; G[1] += pp.y; G[2] += pp.z; G[3] += pp.w;
                }
            } else {
                const int32_t k0 = c.code_off[2 * v], k1 = c.code_off[2 * v + 1], k2 = c.code_off[2 * v + 2];
                const uint32_t *col = E + (q >> 3);
                const int sh = 4 * (q & 7);
                count_bits(col, p.W, k0, k1, sh, 1, G);
                count_bits(col, p.W, k1, k2, sh, -1, G);
            }

            // --- a7: straight-through gradient, optimiser, rounding, next sample
            const uint4 wn4 = philox4x32_10(make_uint4((uint32_t)v, (uint32_t)(bq >> 2), (uint32_t)s, 1u), p.keys);
            const uint4 wx4 = philox4x32_10(make_uint4((uint32_t)v, (uint32_t)(bq >> 2), (uint32_t)(s + 1), 1u), p.keys);
            const uint32_t wn[4] = {wn4.x, wn4.y, wn4.z, wn4.w};
            const uint32_t wx[4] = {wx4.x, wx4.y, wx4.z, wx4.w};
            float zz[4] = {z.x, z.y, z.z, z.w}, mm[4] = {m.x, m.y, m.z, m.w}, ww[4] = {vv.x, vv.y, vv.z, vv.w};
            float g1o[4];
            const int pin_r = kPins ? (int)p.pin_rank[v] : -1;   // cube pin of this variable
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                float g1;
                if (kTau1) {
                    const float2 uu = unif_pair(wn[j]);
                    const float e = exp_neg_abs(zz[j]);
                    const bool pos = zz[j] >= 0.0f;
                    const float d = pos ? fmaf(uu.y, e, uu.x) : fmaf(uu.x, e, uu.y);
                    const float pq = __fdividef(uu.x * uu.y * e, d * d);   // sigma(a) sigma(-a)
                    g1 = -(float)G[j] * pq;                // dL/dtheta_1 (straight-through), tau = 1
                } else {
                    const float a = (zz[j] + logistic_from_word(wn[j])) * p.inv_tau;
                    const float e = exp_neg_abs(a);
                    const float d = 1.0f + e;
                    g1 = -(float)G[j] * __fdividef(e, d * d) * p.inv_tau;
                }
                if (kPins && pin_r >= 0) g1 = 0.0f;
                float zn;
                if (kAdam) {
                    const float mn = fmaf(p.beta1, mm[j], p.omb1 * g1);
                    const float wv = fmaf(p.beta2, ww[j], p.omb2 * g1 * g1);
                    zn = zz[j] - ac.x * __fdividef(mn, fmaf(sqrt_approx(wv), ac.y, p.eps));
                    if (!kPins || pin_r < 0) { mm[j] = mn; ww[j] = wv; }
                } else {
                    zn = zz[j] - 2.0f * p.lr * g1;
                }
                if (!kPins || pin_r < 0) zz[j] = zn;
                bad |= !isfinite(zz[j]);
                g1o[j] = g1;
                uint32_t xb, rb;
                if (kPins && pin_r >= 0) {
                    xb = rb = (uint32_t)((bq + j) >> pin_r) & 1u;
                } else {
                    rb = zz[j] >= 0.0f ? 1u : 0u;
                    if (kTau1)
                        xb = sample_bit_tau1(zz[j], unif_pair(wx[j]), exp_neg_abs(zz[j])) ? 1u : 0u;
                    else
                        xb = zz[j] + logistic_from_word(wx[j]) >= 0.0f ? 1u : 0u;
                }
                rn |= rb << j;
                xn |= xb << j;
            }
            z4[idx] = make_float4(zz[0], zz[1], zz[2], zz[3]);
            m4[idx] = make_float4(mm[0], mm[1], mm[2], mm[3]);
            v4[idx] = make_float4(ww[0], ww[1], ww[2], ww[3]);
            if (kDebug) {
                dbg_G[idx] = make_int4(G[0], G[1], G[2], G[3]);
                dbg_g1[idx] = make_float4(g1o[0], g1o[1], g1o[2], g1o[3]);
            }
        }
        // 8 lanes = one 32-bit word; validity is uniform within each group of 8 lanes
        const uint32_t xw = gather_word(xn, lane), rw = gather_word(rn, lane);
        if (ip.valid && (lane & 7) == 0) {
            X[(size_t)v * p.W + (q >> 3)] = xw;
            R[(size_t)v * p.W + (q >> 3)] = rw;
        }
    }
    if (bad) atomicOr(&ctrl->nonfinite, 1);
}

// ------------------------------------------------------------------- a8/a9: best
// Single block: min over local members of (u << 32 | global b). world == 1 finalizes too.
__device__ void finalize_best(Ctrl *ctrl, unsigned long long key, int64_t b0, int32_t b_loc)
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

__global__ void __launch_bounds__(1024) k_best(const int32_t *__restrict__ unsat, int32_t b_loc, int64_t b0,
                                               Ctrl *__restrict__ ctrl, int32_t finalize)
{
    __shared__ unsigned long long s_min[32];
    if (ctrl->stopped) return;
    unsigned long long best = ~0ull;
    for (int32_t i = threadIdx.x; i < b_loc; i += blockDim.x) {
        const unsigned long long key = ((unsigned long long)(uint32_t)unsat[i] << 32) | (unsigned long long)(b0 + i);
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

__global__ void k_finalize(Ctrl *__restrict__ ctrl, int64_t b0, int32_t b_loc)
{
    if (ctrl->stopped) return;
    finalize_best(ctrl, ctrl->key_global, b0, b_loc);
}

// Copy the rounding column of the new best member (only when it improved on this rank).
__global__ void k_extract(const uint32_t *__restrict__ R, int32_t n, int32_t W, int64_t b0,
                          const Ctrl *__restrict__ ctrl, uint8_t *__restrict__ best_bits)
{
    if (!ctrl->improved) return;
    const int64_t lb = ctrl->best_b - b0;
    for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
        best_bits[v] = (uint8_t)((R[(size_t)v * W + (lb >> 5)] >> (lb & 31)) & 1u);
}

// ------------------------------------------------------------------ launch wrappers
namespace launch {

static unsigned grid_cap(uint64_t work, unsigned threads, unsigned cap)
{
    uint64_t g = (work + threads - 1) / threads;
    if (g < 1) g = 1;
    if (g > cap) g = cap;
    return (unsigned)g;
}

void init(const StepParams &p, float *z, float *m, float *v, uint32_t *X, uint32_t *R, cudaStream_t st)
{
    const uint64_t total = (uint64_t)p.n * (p.b_pad / 4);
    k_init<<<grid_cap(total, 256, 148 * 16), 256, 0, st>>>(p, (float4 *)z, (float4 *)m, (float4 *)v, X, R);
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

void forward_st(const DevCnf &c, int32_t W, int32_t b_pad, const uint32_t *X, uint32_t *E, int32_t *lam,
                Ctrl *ctrl, cudaStream_t st)
{
    k_clauses_st<true><<<clause_grid(c, W), 256, 0, st>>>(c, W, b_pad, X, E, lam, ctrl);
}

void check(const DevCnf &c, int32_t W, int32_t b_pad, const uint32_t *R, int32_t *unsat, Ctrl *ctrl,
           cudaStream_t st)
{
    k_clauses_st<false><<<clause_grid(c, W), 256, 0, st>>>(c, W, b_pad, R, nullptr, unsat, ctrl);
}

RowMap make_rowmap(uint32_t rows, uint32_t b_pad)
{
    RowMap rm;
    rm.QW = b_pad / 4u;
    rm.rows = rows;
    if (rm.QW >= 256) {
        rm.cpr = (rm.QW + 255u) / 256u;
        rm.R = 1;
    } else {
        rm.cpr = 1;
        rm.R = 256u / rm.QW;
    }
    rm.items = (rows + rm.R - 1) / rm.R * rm.cpr;
    // q = (umulhi(x, mul) + x) >> shift == x / cpr for all 32-bit x (64-bit add)
    uint32_t l = 0;
    while ((1ull << l) < rm.cpr) ++l;
    rm.div_shift = l;
    rm.div_mul = (uint32_t)((((1ull << l) - rm.cpr) << 32) / rm.cpr + 1ull);
    if (rm.cpr == 1) rm.div_mul = 0;
    return rm;
}

static unsigned item_grid(const RowMap &rm, unsigned ctas_per_sm)
{
    unsigned g = 148u * ctas_per_sm;
    if (rm.items < g) g = rm.items;
    return g < 1 ? 1 : g;
}

void hub_partial(const DevCnf &c, int32_t W, int32_t b_pad, const uint32_t *E, short4 *partial,
                 const Ctrl *ctrl, cudaStream_t st)
{
    if (c.num_hub_chunks == 0) return;
    const RowMap rm = make_rowmap((uint32_t)c.num_hub_chunks, (uint32_t)b_pad);
    k_hub_partial<<<item_grid(rm, 8), 256, 0, st>>>(c, W, rm, E, partial, ctrl);
}

void update_st(const DevCnf &c, const StepParams &p, float *z, float *m, float *v, uint32_t *X, uint32_t *R,
               const uint32_t *E, const short4 *partial, Ctrl *ctrl, int32_t *dbg_G, float *dbg_g1,
               cudaStream_t st)
{
    const RowMap rm = make_rowmap((uint32_t)p.n, (uint32_t)p.b_pad);
    const unsigned grid = item_grid(rm, 8);
    const int variant = (dbg_G ? 8 : 0) | (p.inv_tau == 1.0f ? 4 : 0) | (p.optimizer == 0 ? 2 : 0) |
                        (p.pin_rank ? 1 : 0);
    using K = void (*)(DevCnf, StepParams, RowMap, float4 *, float4 *, float4 *, uint32_t *, uint32_t *,
                       const uint32_t *, const short4 *, Ctrl *, int4 *, float4 *);
    static const K table[16] = {
        k_update_st<false, false, false, false>, k_update_st<false, false, false, true>,
        k_update_st<false, false, true, false>,  k_update_st<false, false, true, true>,
        k_update_st<false, true, false, false>,  k_update_st<false, true, false, true>,
        k_update_st<false, true, true, false>,   k_update_st<false, true, true, true>,
        k_update_st<true, false, false, false>,  k_update_st<true, false, false, true>,
        k_update_st<true, false, true, false>,   k_update_st<true, false, true, true>,
        k_update_st<true, true, false, false>,   k_update_st<true, true, false, true>,
        k_update_st<true, true, true, false>,    k_update_st<true, true, true, true>,
    };
    table[variant]<<<grid, 256, 0, st>>>(c, p, rm, (float4 *)z, (float4 *)m, (float4 *)v, X, R, E, partial, ctrl,
                                          (int4 *)dbg_G, (float4 *)dbg_g1);
}

void best(const int32_t *unsat, int32_t b_loc, int64_t b0, Ctrl *ctrl, bool finalize, cudaStream_t st)
{
    k_best<<<1, 1024, 0, st>>>(unsat, b_loc, b0, ctrl, finalize ? 1 : 0);
}

void finalize(Ctrl *ctrl, int64_t b0, int32_t b_loc, cudaStream_t st)
{
    k_finalize<<<1, 1, 0, st>>>(ctrl, b0, b_loc);
}

void extract(const uint32_t *R, int32_t n, int32_t W, int64_t b0, const Ctrl *ctrl, uint8_t *best_bits,
             cudaStream_t st)
{
    k_extract<<<grid_cap((uint64_t)n, 256, 148 * 4), 256, 0, st>>>(R, n, W, b0, ctrl, best_bits);
}

}  // namespace launch
}  // namespace galois
