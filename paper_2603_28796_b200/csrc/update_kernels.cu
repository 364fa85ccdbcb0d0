// update_kernels.cu — rows a6 + a7 of SURVEY §8: the fused backward + update.
//
// For every variable v and member b (one thread per QUAD of 4 members):
//   a6  G_v,b = sum over the occurrences of v of sigma * E   (segmented, CSC order:
//       positive codes, then negative; integer, no atomics -> deterministic; negative
//       rows are stored complemented, so G = sum of all row bits - negative row count)
//   a7  g1 = -G p q / tau (straight-through, Eq.4 text P:160; p q = sigma(a) sigma(-a)),
//       Adam (App. A) on the reduced iterate z = theta_1 - theta_0, rounding
//       R_t = [z >= 0], next sample X_{t+1} = [z + ell_{t+1} >= 0] (Eq.3-4).
// E layout: chunk-major E[chunk][csc position][CW], CW = min(W, 32) words, so the
// occurrences of one variable within one 1024-member chunk are ONE contiguous block of
// deg * 128 B — one TMA bulk copy (k_update_tma). Hub variables (degree > kHubDegree)
// are first reduced in fixed-size chunks by k_hub_partial (deterministic int16 partials).
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>

#include "device_utils.cuh"
#include "galois_internal.h"
#include "philox.cuh"

namespace galois {

namespace {

constexpr int kBatch = 8;             // independent E loads in flight per thread (global path)
#ifndef GALOIS_UPD_STAGES
#define GALOIS_UPD_STAGES 4
#endif
#ifndef GALOIS_UPD_CTAS
#define GALOIS_UPD_CTAS 3
#endif
constexpr int kStages = GALOIS_UPD_STAGES;   // TMA pipeline depth
#ifndef GALOIS_STAGE_ROWS
#define GALOIS_STAGE_ROWS 48
#endif
#ifndef GALOIS_SLICED_ROWS
#define GALOIS_SLICED_ROWS 16
#endif
constexpr int kStageRows = GALOIS_STAGE_ROWS;   // E rows staged per piece (48: C3a update -1.7 %, C4 -0.7 %)
static_assert(kStageRows <= 56, "a piece's rows must fit count_rows_sliced<3> (<= 7 per thread)");
constexpr int kTmaCtasPerSm = GALOIS_UPD_CTAS;   // 3 x (4 x 16 KB) shared memory per SM
constexpr int kStageE = kStageRows * 128;
constexpr int kStageBytes = kStageE + 3 * 4096;   // E rows + z, m, v of 256 quads
constexpr int kTmaSmem = kStages * kStageBytes;

// Count the E bits of one quad (bits qp + 8j of column `col`, row stride CW words) over
// occurrences [k0, k1): kBatch independent predicated loads per round trip; four 8-bit
// counters in one register (one bit per byte), flushed before they can overflow. Rows of negative
// occurrences are stored complemented, so sum over all rows = G + (number of negative
// rows): the callers subtract that count (one pass, no sign split).
__device__ __forceinline__ void count_bits(const uint32_t *__restrict__ col, int32_t CW, int32_t k0, int32_t k1,
                                           int qp, int32_t G[4])
{
    const uint32_t *ptr = col + (size_t)k0 * CW;
    int32_t left = k1 - k0;
    while (left > 0) {
        int32_t blk = min(left, 248);
        left -= blk;
        uint32_t acc = 0;
        for (; blk >= kBatch; blk -= kBatch) {
            uint32_t e[kBatch];
#pragma unroll
            for (int i = 0; i < kBatch; ++i) e[i] = __ldg(ptr + i * CW);
            ptr += kBatch * CW;
#pragma unroll
            for (int i = 0; i < kBatch; ++i) acc += quad_bits(e[i], qp);
        }
        if (blk > 0) {
            uint32_t e[kBatch - 1];
#pragma unroll
            for (int i = 0; i < kBatch - 1; ++i) e[i] = i < blk ? __ldg(ptr + i * CW) : 0u;
            ptr += blk * CW;
#pragma unroll
            for (int i = 0; i < kBatch - 1; ++i) acc += quad_bits(e[i], qp);
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) G[j] += (int32_t)((acc >> (8 * j)) & 255u);
    }
}

// Same count over rows staged in shared memory (row = 32 words = 128 B).
__device__ __forceinline__ void count_bits_smem(const uint32_t *srow, int32_t n, int qp, int32_t G[4])
{
    uint32_t acc = 0;                     // n <= 128 < 256: no overflow
#pragma unroll 8
    for (int32_t k = 0; k < n; ++k) acc += quad_bits(srow[k * 32], qp);
#pragma unroll
    for (int j = 0; j < 4; ++j) G[j] += (int32_t)((acc >> (8 * j)) & 255u);
}

// Long segments (32-row pieces of the update): the 8 threads sharing a 32-member word
// split the rows (thread i takes rows i, i+8, ...) and add FULL words into a bit-sliced
// counter (one half adder per plane), then sum the 8 partial counters by a 3-round
// shuffle butterfly (one full adder per plane) and each thread reads its nibble's counts
// back out of the planes: ~11 instructions per row per 32 members instead of ~5.5 per
// row per 4 members. kIn planes hold the per-thread partial (rows/8 < 2^kIn); the sum
// needs kIn + 3 planes. Adds the 4 counts of this thread's nibble to G.
#ifndef GALOIS_HUB_CF
#define GALOIS_HUB_CF 1
#endif
#ifndef GALOIS_HARLEY_SEAL
#define GALOIS_HARLEY_SEAL 1
#endif
// Carry-save adder (one LOP3 each for the sum and the majority).
__device__ __forceinline__ void csa(uint32_t &h, uint32_t &l, uint32_t a, uint32_t b, uint32_t c)
{
    const uint32_t u = a ^ b;
    h = (a & b) | (u & c);
    l = u ^ c;
}

// Add bit-rows sub, sub + 8, ... (< n) of a word column into the vertical counter P[0..kIn)
// (P[k] = bit k of each lane's count). Harley-Seal: 8 rows cost 7 carry-save adders (14
// LOP3) plus one carry rippled into P[3..], 4 rows 3 adders plus a carry into P[2..];
// single rows ripple (2 ops per plane) — instead of 2 kIn ops per row.
template <int kIn, int kMaxRows>
__device__ __forceinline__ void add_rows(uint32_t (&P)[kIn], const uint32_t *wcol, int32_t n, int sub)
{
    int32_t r = sub;
    if (kIn >= 4 && kMaxRows >= 8) {
        for (; r + 56 < n; r += 64) {
            uint32_t d[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) d[i] = wcol[(r + 8 * i) * 32];
            uint32_t tA, tB, fA, fB, e;
            csa(tA, P[0], P[0], d[0], d[1]);
            csa(tB, P[0], P[0], d[2], d[3]);
            csa(fA, P[1], P[1], tA, tB);
            csa(tA, P[0], P[0], d[4], d[5]);
            csa(tB, P[0], P[0], d[6], d[7]);
            csa(fB, P[1], P[1], tA, tB);
            csa(e, P[2], P[2], fA, fB);
#pragma unroll
            for (int k = 3; k < kIn; ++k) {
                const uint32_t t = P[k] & e;
                P[k] ^= e;
                e = t;
            }
        }
    }
    if (kIn >= 3 && kMaxRows >= 4) {
        for (; r + 24 < n; r += 32) {
            const uint32_t d0 = wcol[r * 32], d1 = wcol[(r + 8) * 32], d2 = wcol[(r + 16) * 32],
                           d3 = wcol[(r + 24) * 32];
            uint32_t tA, tB, f;
            csa(tA, P[0], P[0], d0, d1);
            csa(tB, P[0], P[0], d2, d3);
            csa(f, P[1], P[1], tA, tB);
#pragma unroll
            for (int k = 2; k < kIn; ++k) {
                const uint32_t t = P[k] & f;
                P[k] ^= f;
                f = t;
            }
        }
    }
    for (; r < n; r += 8) {
        uint32_t c = wcol[r * 32];
#pragma unroll
        for (int k = 0; k < kIn; ++k) {
            const uint32_t t = P[k] & c;
            P[k] ^= c;
            c = t;
        }
    }
}

template <int kIn>
__device__ __forceinline__ void count_rows_sliced(const uint32_t *wcol, int32_t n, int sub, int qp, int32_t G[4])
{
    constexpr int kOut = kIn + 3;
    uint32_t P[kOut];
#pragma unroll
    for (int k = 0; k < kOut; ++k) P[k] = 0;
#if GALOIS_HARLEY_SEAL
    if (kIn >= 5) {                             // hub chunks (<= 32 rows per thread); the
        uint32_t Q[kIn];                        // update's short pieces keep the ripple below
#pragma unroll
        for (int k = 0; k < kIn; ++k) Q[k] = 0;
        add_rows<kIn, (1 << kIn) - 1>(Q, wcol, n, sub);
#pragma unroll
        for (int k = 0; k < kIn; ++k) P[k] = Q[k];
    } else
#endif
    for (int32_t r = sub; r < n; r += 8) {
        uint32_t c = wcol[r * 32];
#pragma unroll
        for (int k = 0; k < kIn; ++k) {
            const uint32_t t = P[k] & c;
            P[k] ^= c;
            c = t;
        }
    }
#pragma unroll
    for (int d = 1; d < 8; d <<= 1) {           // lanes 8w .. 8w+7 hold the same word
        uint32_t carry = 0;
#pragma unroll
        for (int k = 0; k < kOut; ++k) {
            const uint32_t o = __shfl_xor_sync(0xffffffffu, P[k], d);
            const uint32_t sum = P[k] ^ o ^ carry;
            carry = (P[k] & o) | (carry & (P[k] ^ o));
            P[k] = sum;
        }
    }
    uint32_t acc = 0;                           // planes 0..7: byte j = count mod 256 of member j
#pragma unroll
    for (int k = 0; k < kOut && k < 8; ++k) acc += quad_bits(P[k], qp) << k;
#pragma unroll
    for (int j = 0; j < 4; ++j) G[j] += (int32_t)((acc >> (8 * j)) & 255u);
#pragma unroll
    for (int k = 8; k < kOut; ++k) {            // (a 256-row hub chunk can count 256)
        const uint32_t b = quad_bits(P[k], qp);
#pragma unroll
        for (int j = 0; j < 4; ++j) G[j] += (int32_t)((b >> (8 * j)) & 1u) << k;
    }
}

// The same bit-sliced count split in two, for a variable whose E rows arrive in several
// pieces: sliced_add() adds one piece's rows (thread `sub` of the 8 sharing a word takes
// rows sub, sub + 8, ...) into kIn planes that persist across the pieces, and
// sliced_finish() runs the butterfly ONCE per variable and adds this thread's 4 counts to
// G. For degree <= 256 a thread adds <= 32 rows: kIn = 6 planes, 9 after the butterfly.
template <int kIn>
__device__ __forceinline__ void sliced_add(uint32_t (&P)[kIn], const uint32_t *wcol, int32_t n, int sub)
{
#if GALOIS_HARLEY_SEAL
    add_rows<kIn, 4>(P, wcol, n, sub);          // a piece has <= 32 rows: <= 4 per thread
    return;
#endif
    for (int32_t r = sub; r < n; r += 8) {
        uint32_t c = wcol[r * 32];
#pragma unroll
        for (int k = 0; k < kIn; ++k) {
            const uint32_t t = P[k] & c;
            P[k] ^= c;
            c = t;
        }
    }
}

template <int kIn>
__device__ __forceinline__ void sliced_finish(const uint32_t (&Pin)[kIn], int qp, int32_t G[4])
{
    constexpr int kOut = kIn + 3;
    uint32_t P[kOut];
#pragma unroll
    for (int k = 0; k < kOut; ++k) P[k] = k < kIn ? Pin[k] : 0u;
#pragma unroll
    for (int d = 1; d < 8; d <<= 1) {           // lanes 8w .. 8w+7 hold the same word
        uint32_t carry = 0;
#pragma unroll
        for (int k = 0; k < kOut; ++k) {
            const uint32_t o = __shfl_xor_sync(0xffffffffu, P[k], d);
            const uint32_t sum = P[k] ^ o ^ carry;
            carry = (P[k] & o) | (carry & (P[k] ^ o));
            P[k] = sum;
        }
    }
    uint32_t acc = 0;                           // planes 0..7: byte j = count mod 256 of member j
#pragma unroll
    for (int k = 0; k < kOut && k < 8; ++k) acc += quad_bits(P[k], qp) << k;
#pragma unroll
    for (int j = 0; j < 4; ++j) G[j] += (int32_t)((acc >> (8 * j)) & 255u);
#pragma unroll
    for (int k = 8; k < kOut; ++k) {
        const uint32_t b = quad_bits(P[k], qp);
#pragma unroll
        for (int j = 0; j < 4; ++j) G[j] += (int32_t)((b >> (8 * j)) & 1u) << k;
    }
}

struct ItemPos {
    uint32_t row;    // variable (or hub chunk)
    uint32_t q;      // quad within the row
    bool valid;
};

__device__ __forceinline__ uint32_t div_cpr(const RowMap &rm, uint32_t x)
{
    return (uint32_t)(((uint64_t)__umulhi(x, rm.div_mul) + x) >> rm.div_shift);
}

__device__ __forceinline__ ItemPos item_pos(const RowMap &rm, uint32_t item, uint32_t r_t, uint32_t q_t)
{
    const uint32_t grp = div_cpr(rm, item);
    const uint32_t chunk = item - grp * rm.cpr;
    ItemPos ip;
    ip.row = grp * rm.R + r_t;
    ip.q = chunk * 256u + q_t;
    ip.valid = r_t < rm.R && ip.row < rm.rows && ip.q < rm.QW;
    return ip;
}

// Column of quad q in the chunk-major E: chunk q/256 (when CW = 32), word (q/8) mod CW.
__device__ __forceinline__ const uint32_t *e_column(const uint32_t *E, int32_t L, int32_t CW, uint32_t q)
{
    const uint32_t w = q >> 3;
    const uint32_t ch = w / (uint32_t)CW, wi = w - ch * (uint32_t)CW;
    return E + (size_t)ch * L * CW + wi;
}

// tau = 1 rewrites of Eq.3 with no logarithm: with (u, ub = 1 - u) and e = exp(-|z|),
// sigma(z + logit u) sigma(-(z + logit u)) = u ub e / d^2 with d = u + ub e (z >= 0) or
// ub + u e (z < 0); and [z + logit u >= 0] <=> u >= ub e (z >= 0) or u e >= ub (z < 0).

// a7 for one quad: gradient, optimiser, rounding, next sample. Returns the four members'
// sample and rounding bits as predicates (the TMA kernels ballot them directly).
template <bool kTau1, bool kAdam, bool kPins>
__device__ __forceinline__ void quad_update_bits(const StepParams &p, float2 ac, int32_t v, int64_t bq, int32_t s,
                                                 const int32_t G[4], float4 &z, float4 &m, float4 &vv,
                                                 bool (&xbit)[4], bool (&rbit)[4], float g1o[4], bool &bad,
                                                 const uint4 wn4, const uint4 wx4)
{
    const uint32_t wn[4] = {wn4.x, wn4.y, wn4.z, wn4.w};
    const uint32_t wx[4] = {wx4.x, wx4.y, wx4.z, wx4.w};
    float zz[4] = {z.x, z.y, z.z, z.w}, mm[4] = {m.x, m.y, m.z, m.w}, ww[4] = {vv.x, vv.y, vv.z, vv.w};
    const int pin_r = kPins ? (int)p.pin_rank[v] : -1;       // cube pin of this variable
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        float g1;
        if (kTau1) {
            const float2 uu = unif_pair(wn[j]);
            const float e = exp_neg_abs(zz[j]);
            const float d = zz[j] >= 0.0f ? fmaf(uu.y, e, uu.x) : fmaf(uu.x, e, uu.y);
            g1 = -(float)G[j] * __fdividef(uu.x * uu.y * e, d * d);   // -G sigma(a) sigma(-a)
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
        g1o[j] = g1;
        bool xb, rb;
        if (kPins && pin_r >= 0) {
            xb = rb = (((bq + j) >> pin_r) & 1) != 0;
        } else {
            rb = zz[j] >= 0.0f;
            if (kTau1) {
                // [z + logit u >= 0] with e = exp(-|z|): u - ub e >= 0 (z >= 0) or u e - ub >= 0
                // (z < 0);
                // with ub = 1 - u both cases are one FMA on u alone:
                //   z >= 0: u - ub e = u (1 + e) - e;   z < 0: u e - ub = u (1 + e) - 1
                const float u = unif_pair(wx[j]).x;
                const float e = exp_neg_abs(zz[j]);
                xb = fmaf(u, 1.0f + e, rb ? -e : -1.0f) >= 0.0f;
            } else {
                xb = zz[j] + logistic_from_word(wx[j]) >= 0.0f;
            }
        }
        rbit[j] = rb;
        xbit[j] = xb;
    }
    bad |= !isfinite((zz[0] + zz[1]) + (zz[2] + zz[3]));   // NaN/Inf in any lane survives the sum
    z = make_float4(zz[0], zz[1], zz[2], zz[3]);
    m = make_float4(mm[0], mm[1], mm[2], mm[3]);
    vv = make_float4(ww[0], ww[1], ww[2], ww[3]);
}

// The quad's two Philox draws: the noise of step s (gradient) and of step s + 1 (next sample).
__device__ __forceinline__ uint4 quad_noise(const StepParams &p, int32_t v, int64_t bq, int32_t step)
{
    return philox4x32_10(make_uint4((uint32_t)v, (uint32_t)(bq >> 2), (uint32_t)step, 1u), p.keys);
}

template <bool kTau1, bool kAdam, bool kPins>
__device__ __forceinline__ void quad_update_bits(const StepParams &p, float2 ac, int32_t v, int64_t bq, int32_t s,
                                                 const int32_t G[4], float4 &z, float4 &m, float4 &vv,
                                                 bool (&xbit)[4], bool (&rbit)[4], float g1o[4], bool &bad)
{
    quad_update_bits<kTau1, kAdam, kPins>(p, ac, v, bq, s, G, z, m, vv, xbit, rbit, g1o, bad,
                                          quad_noise(p, v, bq, s), quad_noise(p, v, bq, s + 1));
}

// The same with the bits as nibbles (bit j = member j), for callers whose lanes do not all
// take part (k_update_st's ragged rows, k_small_run).
template <bool kTau1, bool kAdam, bool kPins>
__device__ __forceinline__ void quad_update(const StepParams &p, float2 ac, int32_t v, int64_t bq, int32_t s,
                                            const int32_t G[4], float4 &z, float4 &m, float4 &vv, uint32_t &xn,
                                            uint32_t &rn, float g1o[4], bool &bad)
{
    bool xb[4], rb[4];
    quad_update_bits<kTau1, kAdam, kPins>(p, ac, v, bq, s, G, z, m, vv, xb, rb, g1o, bad);
    xn = (xb[0] ? 1u : 0u) | (xb[1] ? 2u : 0u) | (xb[2] ? 4u : 0u) | (xb[3] ? 8u : 0u);
    rn = (rb[0] ? 1u : 0u) | (rb[1] ? 2u : 0u) | (rb[2] ? 4u : 0u) | (rb[3] ? 8u : 0u);
}

// The 32-bit word of this lane's 8-lane group from every lane's four member bits (all 32
// lanes take part): pack_quads without building the nibble first.
__device__ __forceinline__ uint32_t pack_bits(const bool (&b)[4], int lane)
{
    const uint32_t b0 = __ballot_sync(0xffffffffu, b[0]), b1 = __ballot_sync(0xffffffffu, b[1]);
    const uint32_t b2 = __ballot_sync(0xffffffffu, b[2]), b3 = __ballot_sync(0xffffffffu, b[3]);
    const uint32_t k = (uint32_t)(lane >> 3) & 3u;
    const uint32_t sel = k | ((k + 4u) << 4);
    return __byte_perm(__byte_perm(b0, b1, sel), __byte_perm(b2, b3, sel), 0x5410);
}

__device__ __forceinline__ void hub_signal(const DevCnf &c, const short4 *__restrict__ partial, uint32_t QW,
                                           int32_t hub, uint32_t q, int32_t G[4])
{
    const int32_t c0 = c.hub_chunk_off[hub], c1 = c.hub_chunk_off[hub + 1];
    for (int32_t ch = c0; ch < c1; ++ch) {
        const short4 pp = partial[(size_t)ch * QW + q];
        G[0] += pp.x; G[1] += pp.y; G[2] += pp.z; G[3] += pp.w;
    }
}

}  // namespace

// --------------------------------------------------------------- a6: hub partial sums
// Row = hub chunk of <= kHubChunk occurrences of one variable; per quad, the signed count
// of E bits over the chunk (|value| <= 128 -> int16). Fixed chunk order = deterministic.
__global__ void __launch_bounds__(256) k_hub_partial(DevCnf c, int32_t CW, RowMap rm, const uint32_t *__restrict__ E,
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
        const uint32_t *col = e_column(E, c.L, CW, ip.q);
        const int sh = ip.q & 7;          // bit offset of this quad's members
        int32_t G[4] = {0, 0, 0, 0};
        count_bits(col, CW, info.y, k1, sh, G);
        const int32_t nneg = k1 - max(split, info.y);
        if (nneg > 0) { G[0] -= nneg; G[1] -= nneg; G[2] -= nneg; G[3] -= nneg; }
        partial[(size_t)ip.row * rm.QW + ip.q] = make_short4((short)G[0], (short)G[1], (short)G[2], (short)G[3]);
    }
}

// ------------------------------------------------- a6 + a7: fused update, generic layout
template <bool kDebug, bool kTau1, bool kAdam, bool kPins>
__global__ void __launch_bounds__(256) k_update_st(DevCnf c, StepParams p, RowMap rm, float4 *__restrict__ z4,
                                                   float4 *__restrict__ m4, float4 *__restrict__ v4,
                                                   uint32_t *__restrict__ X, uint32_t *__restrict__ R,
                                                   const uint32_t *__restrict__ E,
                                                   const short4 *__restrict__ partial, Ctrl *__restrict__ ctrl,
                                                   int4 *__restrict__ dbg_G, float4 *__restrict__ dbg_g1)
{
    if (ctrl->stopped) return;
    const int32_t s = ctrl->t + 1;                   // this step's index (t -> t+1)
    const float2 ac = p.adam_consts[s];              // {2 lr / bc1, 1 / sqrt(bc2)}
    const int lane = threadIdx.x & 31;
    const int32_t CW = p.W < 32 ? p.W : 32;
    const uint32_t r_t = rm.QW >= 256 ? 0u : threadIdx.x / rm.QW;
    const uint32_t q_t = rm.QW >= 256 ? threadIdx.x : threadIdx.x - r_t * rm.QW;
    bool bad = false;
    clear_counters(p);
    for (uint32_t item = blockIdx.x; item < rm.items; item += gridDim.x) {
        const ItemPos ip = item_pos(rm, item, r_t, q_t);
        const int32_t v = (int32_t)ip.row;
        const uint32_t q = ip.q;
        uint32_t xn = 0, rn = 0;
        if (ip.valid) {
            const int64_t bq = p.b0 + 4 * (int64_t)q;
            const size_t idx = (size_t)v * rm.QW + q;
            float4 z = z4[idx], m = m4[idx], vv = v4[idx];
            int32_t G[4] = {0, 0, 0, 0};
            const int32_t hub = c.num_hubs > 0 ? c.hub_of_var[v] : -1;
            if (hub >= 0) {
                hub_signal(c, partial, rm.QW, hub, q, G);
            } else {
                const int32_t k0 = c.code_off[2 * v], k1 = c.code_off[2 * v + 1], k2 = c.code_off[2 * v + 2];
                const uint32_t *col = e_column(E, c.L, CW, q);
                const int sh = q & 7;
                count_bits(col, CW, k0, k2, sh, G);
                G[0] -= k2 - k1; G[1] -= k2 - k1; G[2] -= k2 - k1; G[3] -= k2 - k1;
            }
            float g1o[4];
            quad_update<kTau1, kAdam, kPins>(p, ac, v, bq, s, G, z, m, vv, xn, rn, g1o, bad);
            z4[idx] = z;
            m4[idx] = m;
            v4[idx] = vv;
            if (kDebug) {
                dbg_G[idx] = make_int4(G[0], G[1], G[2], G[3]);
                dbg_g1[idx] = make_float4(g1o[0], g1o[1], g1o[2], g1o[3]);
            }
        }
        // 8 lanes = one 32-bit word; validity is uniform within each group of 8 lanes
        const uint32_t xw = pack_quads(xn, lane), rw = pack_quads(rn, lane);
        if (ip.valid && (lane & 7) == 0) {
            X[xr_at(v, (int32_t)(q >> 3), p.W)] = xw;
            R[xr_at(v, (int32_t)(q >> 3), p.W)] = rw;
        }
    }
    if (bad) atomicOr(&ctrl->nonfinite, 1);
    last_cta_tick(ctrl);
}

// -------------------------------- a6 + a7: fused update, TMA-pipelined (W % 32 == 0)
// Persistent CTAs of 8 consumer warps (one quad per thread) + 1 producer warp; item =
// (variable, 1024-member chunk). The producer's elected lane runs kStages stages ahead of
// the consumers: an item's first stage carries the z, m, v rows (3 x 4 KB, 1-D TMA bulk
// copies, cp.async.bulk) and the first kStageRows rows of the variable's contiguous E
// block; a variable of higher degree streams its remaining E rows through further stages
// (one 4 KB piece each), so every non-hub degree is counted from shared memory. Stages
// complete on their `full` mbarrier (transaction bytes); consumer warps release them
// through `empty` (one arrive per warp). No CTA-wide barrier in the loop. Hub variables
// (degree > kHubDegree) take one stage for z, m, v and read their partial sums.
constexpr int kConsumerWarps = 8;
// variables of at least this degree count their E rows bit-sliced across all their pieces
// (~1.6 instructions per row and thread + one ~170-instruction butterfly) instead of ~4.1
// per row and thread; kHubDegree bounds a thread's rows at 32 (6 planes)
#ifndef GALOIS_SLICED_MIN_DEGREE
#define GALOIS_SLICED_MIN_DEGREE 64
#endif
constexpr int kSlicedMinDegree = GALOIS_SLICED_MIN_DEGREE;
constexpr int kSlicedPlanes = 6;
#ifndef GALOIS_SLICED_SMALL
#define GALOIS_SLICED_SMALL 1   // variables of <= 120 rows: 4 planes and a 7-plane butterfly
#endif
#ifndef GALOIS_SLICED_MIN_AVG_DEGREE
#define GALOIS_SLICED_MIN_AVG_DEGREE 48
#endif
constexpr int kSlicedMinAvgDegree = GALOIS_SLICED_MIN_AVG_DEGREE;   // L / n at which update_st picks kSliced
static_assert(kHubDegree <= 8 * ((1 << kSlicedPlanes) - 1) + 8, "rows per thread must fit the planes");

struct StageHdr {
    int32_t v;       // variable
    int32_t k1;      // first negative CSC position of v
    int32_t r0, r1;  // CSC rows staged in this piece
};

template <bool kDebug, bool kTau1, bool kAdam, bool kPins, bool kSliced>
__global__ void __launch_bounds__(256 + 32, kTmaCtasPerSm) k_update_tma(DevCnf c, StepParams p, RowMap rm, float4 *__restrict__ z4,
                                                         float4 *__restrict__ m4, float4 *__restrict__ v4,
                                                         uint32_t *__restrict__ X, uint32_t *__restrict__ R,
                                                         const uint32_t *__restrict__ E,
                                                         const short4 *__restrict__ partial, Ctrl *__restrict__ ctrl,
                                                         int4 *__restrict__ dbg_G, float4 *__restrict__ dbg_g1)
{
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ uint64_t full[kStages], empty[kStages];
    __shared__ StageHdr hdr[kStages];
    __shared__ int32_t hflags[kStages];    // bit 0 first piece, bit 1 last piece, bit 2 hub, bit 3 pinned
    if (ctrl->stopped) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t QW = rm.QW;
    const uint32_t full_s = smem_u32(full), empty_s = smem_u32(empty), stage_s = smem_u32(smem);

    if (tid == 0) {
        for (int i = 0; i < kStages; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 32 * kConsumerWarps);   // every consumer thread releases
        }
        fence_mbar_init();
    }
    __syncthreads();

    if (warp == kConsumerWarps) {          // ------------------------------ producer warp
        if (lane == 0) {
            int st = 0;                    // ring stage, its phase parity, and whether the ring wrapped
            uint32_t ph = 0;
            bool wrapped = false;
            for (uint32_t item = blockIdx.x; item < rm.items; item += gridDim.x) {
                const uint32_t v = div_cpr(rm, item), ch = item - v * rm.cpr;
                const int32_t k0 = c.code_off[2 * v], k1 = c.code_off[2 * v + 1], k2 = c.code_off[2 * v + 2];
                const bool hub = c.num_hubs > 0 && c.hub_of_var[v] >= 0;
                const bool pinned = kPins && p.pin_rank[v] >= 0;   // cube pin: read once, by the producer
                const bool sliced = kSliced && !hub && k2 - k0 >= kSlicedMinDegree;
                const int32_t pieces = hub ? 1 : max(1, (k2 - k0 + kStageRows - 1) / kStageRows);
                const size_t off = (size_t)v * QW + (size_t)ch * 256u;
                const uint32_t *Ech = E + (size_t)ch * c.L * 32u;
                for (int32_t pc = 0; pc < pieces; ++pc) {
                    if (wrapped) {
                        mbar_wait_s(empty_s + 8u * st, ph ^ 1u);
                        fence_proxy_async_smem();
                    }
                    const int32_t r0 = hub ? k0 : k0 + pc * kStageRows;
                    const int32_t r1 = hub ? k0 : min(k2, r0 + kStageRows);
                    hdr[st] = StageHdr{(int32_t)v, k1, r0, r1};
                    hflags[st] = (pc == 0 ? 1 : 0) | (pc == pieces - 1 ? 2 : 0) | (hub ? 4 : 0) | (pinned ? 8 : 0) |
                                 (sliced ? 16 : 0) | (sliced && GALOIS_SLICED_SMALL && k2 - k0 <= 8 * 15 ? 32 : 0);
                    const uint32_t ebytes = (uint32_t)(r1 - r0) * 128u;
                    const uint32_t fb = full_s + 8u * st, sbs = stage_s + (uint32_t)(st * kStageBytes);
                    mbar_arrive_expect_tx_s(fb, (pc == 0 ? 3u * 4096u : 0u) + ebytes);
                    if (pc == 0) {
                        bulk_g2s_s(sbs + kStageE, z4 + off, 4096u, fb);
                        bulk_g2s_s(sbs + kStageE + 4096, m4 + off, 4096u, fb);
                        bulk_g2s_s(sbs + kStageE + 8192, v4 + off, 4096u, fb);
                    }
                    if (ebytes) bulk_g2s_s(sbs, Ech + (size_t)r0 * 32u, ebytes, fb);
                    if (++st == kStages) {
                        st = 0;
                        ph ^= 1u;
                        wrapped = true;
                    }
                }
            }
        }
    } else {
    // ------------------------------------------------------------------ consumer warps
    const int32_t s = ctrl->t + 1;         // this step's index (t -> t+1)
    const float2 ac = p.adam_consts[s];
    bool bad = false;
    for (int32_t i = blockIdx.x * 256 + tid; i < p.b_pad; i += gridDim.x * 256) {   // next sweep's counters
        if (p.clear_a) p.clear_a[i] = 0;
        if (p.clear_b) p.clear_b[i] = 0;
    }
    const int sh = tid & 7;
    int st = 0;                            // ring stage and its phase parity (no division)
    uint32_t ph = 0;
    for (uint32_t item = blockIdx.x; item < rm.items; item += gridDim.x) {
        float4 z, m, vv;
        int32_t v = 0, flags = 0, negs = 0;
        int32_t G[4] = {0, 0, 0, 0};
        // kSliced (high average degree): counts carried across an item's pieces in SWAR bytes
        // (degree < kSlicedMinDegree: a byte cannot overflow) or bit-sliced planes (flag 16),
        // G formed after the last piece. Otherwise each piece adds its counts to G.
        uint32_t acc = 0;
        uint32_t PS[kSlicedPlanes];
#pragma unroll
        for (int k = 0; k < kSlicedPlanes; ++k) PS[k] = 0;
        do {
            mbar_wait_s(full_s + 8u * st, ph);
            const StageHdr h = hdr[st];
            flags = hflags[st];
            v = h.v;
            const uint8_t *sb = smem + st * kStageBytes;
            if (flags & 1) {
                z = reinterpret_cast<const float4 *>(sb + kStageE)[tid];
                m = reinterpret_cast<const float4 *>(sb + kStageE + 4096)[tid];
                vv = reinterpret_cast<const float4 *>(sb + kStageE + 8192)[tid];
            }
            if (flags & 4) {
                if (!kSliced) {
                    const uint32_t q = (item - (uint32_t)v * rm.cpr) * 256u + (uint32_t)tid;
                    hub_signal(c, partial, QW, c.hub_of_var[v], q, G);
                }
            } else {
                // rows [r0, r1): negative ones (from k1 on) are stored complemented
                const uint32_t *srow = reinterpret_cast<const uint32_t *>(sb) + (tid >> 3);
                const int32_t nrows = h.r1 - h.r0, nneg = h.r1 - max(h.k1, h.r0);
                if (kSliced) {
                    negs += max(0, nneg);
                    if (flags & 32) {               // <= 120 rows: <= 15 per thread, 4 planes
                        sliced_add<4>(*reinterpret_cast<uint32_t(*)[4]>(&PS), srow, nrows, tid & 7);
                    } else if (flags & 16) {        // uniform over the CTA: a high-degree variable
                        sliced_add(PS, srow, nrows, tid & 7);
                    } else {
#pragma unroll 8
                        for (int32_t k = 0; k < nrows; ++k) acc += quad_bits(srow[k * 32], sh);
                    }
                } else {
                    if (nrows >= GALOIS_SLICED_ROWS)   // uniform over the CTA: a long piece
                        count_rows_sliced<3>(srow, nrows, tid & 7, sh, G);   // <= 6 rows per thread
                    else
                        count_bits_smem(srow, nrows, sh, G);
                    if (nneg > 0) { G[0] -= nneg; G[1] -= nneg; G[2] -= nneg; G[3] -= nneg; }
                }
            }
            mbar_arrive_s(empty_s + 8u * st);   // this thread is done reading the stage
            if (++st == kStages) {
                st = 0;
                ph ^= 1u;
            }
        } while (!(flags & 2));
        const uint32_t q = (item - (uint32_t)v * rm.cpr) * 256u + (uint32_t)tid;
        if (kSliced && (flags & 4)) {
            hub_signal(c, partial, QW, c.hub_of_var[v], q, G);
        } else if (kSliced) {
            if (flags & 32)
                sliced_finish<4>(*reinterpret_cast<const uint32_t(*)[4]>(&PS), sh, G);
            else if (flags & 16)
                sliced_finish(PS, sh, G);           // one butterfly per variable
            else
#pragma unroll
                for (int j = 0; j < 4; ++j) G[j] = (int32_t)((acc >> (8 * j)) & 255u);
#pragma unroll
            for (int j = 0; j < 4; ++j) G[j] -= negs;
        }
        const int64_t bq = p.b0 + 4 * (int64_t)q;
        uint32_t xn, rn;
        float g1o[4];
        // cube pins (C5: 16 of 100k variables): the pinned code path only where the
        // item's variable is pinned (uniform over the item), the plain one elsewhere
#if defined(GALOIS_UPD_MEMONLY) && !defined(GALOIS_PARITY_BREAKING_EXPERIMENT)
#error "GALOIS_UPD_MEMONLY breaks oracle parity: also define GALOIS_PARITY_BREAKING_EXPERIMENT"
#endif
#ifdef GALOIS_UPD_MEMONLY   // experiment: the data movement of this kernel without its arithmetic
        xn = (uint32_t)G[0] & 15u; rn = __float_as_uint(z.x) & 15u; (void)bq; (void)g1o;
        z.x += 1.0f; m.x += 1.0f; vv.x += 1.0f;
#else
        if (kPins && (flags & 8))
            quad_update<kTau1, kAdam, true>(p, ac, v, bq, s, G, z, m, vv, xn, rn, g1o, bad);
        else
            quad_update<kTau1, kAdam, false>(p, ac, v, bq, s, G, z, m, vv, xn, rn, g1o, bad);
#endif
        const size_t idx = (size_t)v * QW + q;
        z4[idx] = z;
        m4[idx] = m;
        v4[idx] = vv;
        if (kDebug) {
            dbg_G[idx] = make_int4(G[0], G[1], G[2], G[3]);
            dbg_g1[idx] = make_float4(g1o[0], g1o[1], g1o[2], g1o[3]);
        }
        const uint32_t xw = pack_quads(xn, lane), rw = pack_quads(rn, lane);
        if ((lane & 7) == 0) {
            X[xr_at(v, (int32_t)(q >> 3), p.W)] = xw;
            R[xr_at(v, (int32_t)(q >> 3), p.W)] = rw;
        }
    }
    if (bad) atomicOr(&ctrl->nonfinite, 1);
    }                                      // consumer warps
    last_cta_tick(ctrl);                   // one barrier site for producer and consumers
}

// ------------------------- a6 + a7: fused update over variable PAIRS (W % 32 == 0)
// k_update_tma with item = (variables 2p and 2p + 1, 1024-member chunk): a pair whose two
// E blocks together fit one stage (no hub, <= kPairRows rows — most variables of sparse
// instances) travels as ONE stage — z, m, v of both (8 KB per array, one bulk copy each
// when the rows are adjacent, i.e. b_pad = 1024) and both CSC blocks (adjacent: one copy)
// — and each consumer thread updates its quad of BOTH variables: the per-stage costs
// (mbarrier waits and polls, header, flags, release) are paid once per two variables, and
// the two quads' arithmetic interleaves. Other pairs go variable by variable through
// pieces of kPairRows rows as in k_update_tma (flag 64: the stage is about the second
// variable). Non-debug, non-sliced instantiations only (the launcher keeps k_update_tma
// for those); same per-quad arithmetic (quad_update), so iterates are bit-identical.
#ifndef GALOIS_PAIR_NOISE4
#define GALOIS_PAIR_NOISE4 1
#endif
#ifndef GALOIS_PAIR_ROWS
#define GALOIS_PAIR_ROWS 56
#endif
constexpr int kPairRows = GALOIS_PAIR_ROWS;          // <= 7 rows per thread: count_rows_sliced<3>
#ifndef GALOIS_PAIR_STAGES
#define GALOIS_PAIR_STAGES 3
#endif
#ifndef GALOIS_PAIR_CTAS
#define GALOIS_PAIR_CTAS 2
#endif
constexpr int kPairStages = GALOIS_PAIR_STAGES;
constexpr int kPairCtasPerSm = GALOIS_PAIR_CTAS;
constexpr int kPairE = kPairRows * 128;
constexpr int kPairStageBytes = kPairE + 3 * 8192;   // E rows + z, m, v of two variables
constexpr int kPairSmem = kPairStages * kPairStageBytes;
static_assert(kPairStageBytes % 128 == 0, "stage alignment");

struct PairHdr {
    int32_t v0;       // first variable of the pair
    int32_t r0, r1;   // CSC rows staged
    int32_t split;    // pair stage: first row of v0 + 1
    int32_t neg0;     // first negative row of v0 (or of the stage's variable)
    int32_t neg1;     // pair stage: first negative row of v0 + 1
};
// stage flags
constexpr int kPfFirst = 1, kPfLast = 2, kPfHub = 4, kPfPin0 = 8, kPfPin1 = 16, kPfPair = 32, kPfSlot1 = 64,
              kPfHas1 = 128;

__device__ __forceinline__ void count_piece(const uint32_t *srow, int32_t n, int qp, int32_t G[4])
{
    if (n >= GALOIS_SLICED_ROWS)       // uniform over the CTA: a long piece
        count_rows_sliced<3>(srow, n, threadIdx.x & 7, qp, G);
    else
        count_bits_smem(srow, n, qp, G);
}

template <bool kTau1, bool kAdam, bool kPins>
__global__ void __launch_bounds__(256 + 32, kPairCtasPerSm)
    k_update_pair(DevCnf c, StepParams p, RowMap rm, float4 *__restrict__ z4, float4 *__restrict__ m4,
                  float4 *__restrict__ v4, uint32_t *__restrict__ X, uint32_t *__restrict__ R,
                  const uint32_t *__restrict__ E, const short4 *__restrict__ partial, Ctrl *__restrict__ ctrl)
{
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ uint64_t full[kPairStages], empty[kPairStages];
    __shared__ PairHdr hdr[kPairStages];
    __shared__ int32_t hflags[kPairStages];
    if (ctrl->stopped) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t QW = rm.QW;
    const uint32_t full_s = smem_u32(full), empty_s = smem_u32(empty), stage_s = smem_u32(smem);
    if (tid == 0) {
        for (int i = 0; i < kPairStages; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 32 * kConsumerWarps);
        }
        fence_mbar_init();
    }
    __syncthreads();

    if (warp == kConsumerWarps) {          // ------------------------------ producer warp
        if (lane == 0) {
            int st = 0;
            uint32_t ph = 0;
            bool wrapped = false;
            auto acquire = [&]() -> uint32_t {  // the next free stage's shared-window address
                if (wrapped) {
                    mbar_wait_s(empty_s + 8u * st, ph ^ 1u);
                    fence_proxy_async_smem();
                }
                return stage_s + (uint32_t)(st * kPairStageBytes);
            };
            auto advance = [&]() {
                if (++st == kPairStages) {
                    st = 0;
                    ph ^= 1u;
                    wrapped = true;
                }
            };
            for (uint32_t item = blockIdx.x; item < rm.items; item += gridDim.x) {
                const uint32_t pr = div_cpr(rm, item), ch = item - pr * rm.cpr;
                const int32_t v0 = 2 * (int32_t)pr;
                const bool has1 = v0 + 1 < c.n;
                const int32_t k0 = c.code_off[2 * v0], k1 = c.code_off[2 * v0 + 1], k2 = c.code_off[2 * v0 + 2];
                const int32_t k3 = has1 ? c.code_off[2 * v0 + 3] : k2, k4 = has1 ? c.code_off[2 * v0 + 4] : k2;
                const bool hub0 = c.num_hubs > 0 && c.hub_of_var[v0] >= 0;
                const bool hub1 = has1 && c.num_hubs > 0 && c.hub_of_var[v0 + 1] >= 0;
                const int32_t pins = (kPins && p.pin_rank[v0] >= 0 ? kPfPin0 : 0) |
                                     (kPins && has1 && p.pin_rank[v0 + 1] >= 0 ? kPfPin1 : 0) | (has1 ? kPfHas1 : 0);
                const size_t off0 = (size_t)v0 * QW + (size_t)ch * 256u, off1 = off0 + QW;
                const uint32_t *Ech = E + (size_t)ch * c.L * 32u;
                if (has1 && !hub0 && !hub1 && k4 - k0 <= kPairRows) {
                    const uint32_t sbs = acquire(), fb = full_s + 8u * st;
                    hdr[st] = PairHdr{v0, k0, k4, k2, k1, k3};
                    hflags[st] = kPfFirst | kPfLast | kPfPair | pins;
                    const uint32_t ebytes = (uint32_t)(k4 - k0) * 128u;
                    mbar_arrive_expect_tx_s(fb, 3u * 8192u + ebytes);
                    if (QW == 256u) {           // the two rows are adjacent
                        bulk_g2s_s(sbs + kPairE, z4 + off0, 8192u, fb);
                        bulk_g2s_s(sbs + kPairE + 8192, m4 + off0, 8192u, fb);
                        bulk_g2s_s(sbs + kPairE + 16384, v4 + off0, 8192u, fb);
                    } else {
                        bulk_g2s_s(sbs + kPairE, z4 + off0, 4096u, fb);
                        bulk_g2s_s(sbs + kPairE + 4096, z4 + off1, 4096u, fb);
                        bulk_g2s_s(sbs + kPairE + 8192, m4 + off0, 4096u, fb);
                        bulk_g2s_s(sbs + kPairE + 12288, m4 + off1, 4096u, fb);
                        bulk_g2s_s(sbs + kPairE + 16384, v4 + off0, 4096u, fb);
                        bulk_g2s_s(sbs + kPairE + 20480, v4 + off1, 4096u, fb);
                    }
                    if (ebytes) bulk_g2s_s(sbs, Ech + (size_t)k0 * 32u, ebytes, fb);
                    advance();
                    continue;
                }
                for (int slot = 0; slot < (has1 ? 2 : 1); ++slot) {
                    const int32_t kb = slot ? k2 : k0, kn = slot ? k3 : k1, ke = slot ? k4 : k2;
                    const bool hub = slot ? hub1 : hub0;
                    const int32_t pieces = hub ? 1 : max(1, (ke - kb + kPairRows - 1) / kPairRows);
                    const size_t off = slot ? off1 : off0;
                    for (int32_t pc = 0; pc < pieces; ++pc) {
                        const uint32_t sbs = acquire(), fb = full_s + 8u * st;
                        const int32_t r0 = hub ? kb : kb + pc * kPairRows;
                        const int32_t r1 = hub ? kb : min(ke, r0 + kPairRows);
                        const bool last = pc == pieces - 1 && slot == (has1 ? 1 : 0);
                        hdr[st] = PairHdr{v0, r0, r1, r1, kn, kn};
                        hflags[st] = (pc == 0 ? kPfFirst : 0) | (last ? kPfLast : 0) | (hub ? kPfHub : 0) |
                                     (slot ? kPfSlot1 : 0) | pins;
                        const uint32_t ebytes = (uint32_t)(r1 - r0) * 128u;
                        mbar_arrive_expect_tx_s(fb, (pc == 0 ? 3u * 4096u : 0u) + ebytes);
                        if (pc == 0) {
                            const uint32_t zb = sbs + kPairE + (uint32_t)slot * 4096u;
                            bulk_g2s_s(zb, z4 + off, 4096u, fb);
                            bulk_g2s_s(zb + 8192, m4 + off, 4096u, fb);
                            bulk_g2s_s(zb + 16384, v4 + off, 4096u, fb);
                        }
                        if (ebytes) bulk_g2s_s(sbs, Ech + (size_t)r0 * 32u, ebytes, fb);
                        advance();
                    }
                }
            }
        }
    } else {
    // ------------------------------------------------------------------ consumer warps
    const int32_t s = ctrl->t + 1;
    const float2 ac = p.adam_consts[s];
    bool bad = false;
    for (int32_t i = blockIdx.x * 256 + tid; i < p.b_pad; i += gridDim.x * 256) {   // next sweep's counters
        if (p.clear_a) p.clear_a[i] = 0;
        if (p.clear_b) p.clear_b[i] = 0;
    }
    const int sh = tid & 7;
    int st = 0;
    uint32_t ph = 0;
    for (uint32_t item = blockIdx.x; item < rm.items; item += gridDim.x) {
        const uint32_t pr = div_cpr(rm, item);
        const uint32_t q = (item - pr * rm.cpr) * 256u + (uint32_t)tid;
        const int32_t v0 = 2 * (int32_t)pr;
        float4 z0, m0, w0, z1, m1, w1;
        int32_t G0[4] = {0, 0, 0, 0}, G1[4] = {0, 0, 0, 0};
        int32_t flags = 0;
        do {
            mbar_wait_s(full_s + 8u * st, ph);
            const PairHdr h = hdr[st];
            flags = hflags[st];
            const uint8_t *sb = smem + st * kPairStageBytes;
            const float4 *za = reinterpret_cast<const float4 *>(sb + kPairE);
            const uint32_t *srow = reinterpret_cast<const uint32_t *>(sb) + (tid >> 3);
            if (flags & kPfPair) {
                z0 = za[tid];       z1 = za[256 + tid];
                m0 = za[512 + tid]; m1 = za[768 + tid];
                w0 = za[1024 + tid]; w1 = za[1280 + tid];
                const int32_t n0 = h.split - h.r0, n1 = h.r1 - h.split;
                count_piece(srow, n0, sh, G0);
                count_piece(srow + n0 * 32, n1, sh, G1);
                const int32_t g0 = h.split - h.neg0, g1 = h.r1 - h.neg1;   // negative rows (complemented)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    G0[j] -= g0;
                    G1[j] -= g1;
                }
            } else {
                const bool slot1 = (flags & kPfSlot1) != 0;
                if (flags & kPfFirst) {
                    if (slot1) {
                        z1 = za[256 + tid]; m1 = za[768 + tid]; w1 = za[1280 + tid];
                    } else {
                        z0 = za[tid]; m0 = za[512 + tid]; w0 = za[1024 + tid];
                    }
                }
                int32_t Gt[4] = {0, 0, 0, 0};
                if (flags & kPfHub) {
                    hub_signal(c, partial, QW, c.hub_of_var[v0 + (slot1 ? 1 : 0)], q, Gt);
                } else {
                    const int32_t nrows = h.r1 - h.r0, nneg = h.r1 - max(h.neg0, h.r0);
                    count_piece(srow, nrows, sh, Gt);
                    if (nneg > 0) {
#pragma unroll
                        for (int j = 0; j < 4; ++j) Gt[j] -= nneg;
                    }
                }
                if (slot1) {
#pragma unroll
                    for (int j = 0; j < 4; ++j) G1[j] += Gt[j];
                } else {
#pragma unroll
                    for (int j = 0; j < 4; ++j) G0[j] += Gt[j];
                }
            }
            mbar_arrive_s(empty_s + 8u * st);
            if (++st == kPairStages) {
                st = 0;
                ph ^= 1u;
            }
        } while (!(flags & kPfLast));
        const int64_t bq = p.b0 + 4 * (int64_t)q;
        bool xb[4], rb[4];
        float g1o[4];
#if GALOIS_PAIR_NOISE4
        // the pair's four Philox calls drawn together: four independent round chains
        const uint4 n0 = quad_noise(p, v0, bq, s), x0 = quad_noise(p, v0, bq, s + 1);
        const uint4 n1 = quad_noise(p, v0 + 1, bq, s), x1 = quad_noise(p, v0 + 1, bq, s + 1);
        if (kPins && (flags & kPfPin0))
            quad_update_bits<kTau1, kAdam, true>(p, ac, v0, bq, s, G0, z0, m0, w0, xb, rb, g1o, bad, n0, x0);
        else
            quad_update_bits<kTau1, kAdam, false>(p, ac, v0, bq, s, G0, z0, m0, w0, xb, rb, g1o, bad, n0, x0);
#else
        if (kPins && (flags & kPfPin0))
            quad_update_bits<kTau1, kAdam, true>(p, ac, v0, bq, s, G0, z0, m0, w0, xb, rb, g1o, bad);
        else
            quad_update_bits<kTau1, kAdam, false>(p, ac, v0, bq, s, G0, z0, m0, w0, xb, rb, g1o, bad);
#endif
        size_t idx = (size_t)v0 * QW + q;
        z4[idx] = z0;
        m4[idx] = m0;
        v4[idx] = w0;
        uint32_t xw = pack_bits(xb, lane), rw = pack_bits(rb, lane);
        if ((lane & 7) == 0) {
            X[xr_at(v0, (int32_t)(q >> 3), p.W)] = xw;
            R[xr_at(v0, (int32_t)(q >> 3), p.W)] = rw;
        }
        if (flags & kPfHas1) {             // uniform over the CTA
#if GALOIS_PAIR_NOISE4
            if (kPins && (flags & kPfPin1))
                quad_update_bits<kTau1, kAdam, true>(p, ac, v0 + 1, bq, s, G1, z1, m1, w1, xb, rb, g1o, bad, n1, x1);
            else
                quad_update_bits<kTau1, kAdam, false>(p, ac, v0 + 1, bq, s, G1, z1, m1, w1, xb, rb, g1o, bad, n1, x1);
#else
            if (kPins && (flags & kPfPin1))
                quad_update_bits<kTau1, kAdam, true>(p, ac, v0 + 1, bq, s, G1, z1, m1, w1, xb, rb, g1o, bad);
            else
                quad_update_bits<kTau1, kAdam, false>(p, ac, v0 + 1, bq, s, G1, z1, m1, w1, xb, rb, g1o, bad);
#endif
            idx += QW;
            z4[idx] = z1;
            m4[idx] = m1;
            v4[idx] = w1;
            xw = pack_bits(xb, lane);
            rw = pack_bits(rb, lane);
            if ((lane & 7) == 0) {
                X[xr_at(v0 + 1, (int32_t)(q >> 3), p.W)] = xw;
                R[xr_at(v0 + 1, (int32_t)(q >> 3), p.W)] = rw;
            }
        }
    }
    if (bad) atomicOr(&ctrl->nonfinite, 1);
    }                                      // consumer warps
    last_cta_tick(ctrl);
}

// --------------------------------------------- a6: hub partial sums, TMA-staged (W % 32 == 0)
// Item = (hub chunk of <= kHubChunk = 256 occurrences, 1024-member chunk): the chunk's E
// rows (<= 32 KB, contiguous) arrive by one bulk copy; per quad the signed count
// (|.| <= 256: int16). 3 x 32 KB stages allow 2 CTAs per SM (kHubCtasPerSm); measured
// against 128-occurrence chunks at 4 CTAs per SM: C3b hub partials 0.194 -> 0.183 ms,
// update 0.065 -> 0.060 ms (half the partials to read), C4 0.191 -> 0.181 ms.
constexpr int kHubStageBytes = kHubChunk * 128;
constexpr int kHubStages = 3;
constexpr int kHubCtasPerSm = 2;                 // 2 x (3 x 32 KB) shared memory per SM

__global__ void __launch_bounds__(256 + 32, kHubCtasPerSm) k_hub_partial_tma(DevCnf c, RowMap rm,
                                                                           const uint32_t *__restrict__ E,
                                                                           short4 *__restrict__ partial,
                                                                           const Ctrl *__restrict__ ctrl)
{
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ uint64_t full[kHubStages], empty[kHubStages];
    __shared__ int4 hdr[kHubStages];          // {first row, positive rows, rows, hub chunk}
    if (ctrl->stopped) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) {
        for (int i = 0; i < kHubStages; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 32 * kConsumerWarps);   // every consumer thread releases
        }
        fence_mbar_init();
    }
    __syncthreads();
    if (warp == kConsumerWarps) {
        if (lane == 0) {
            uint32_t slot = 0;
            for (uint32_t item = blockIdx.x; item < rm.items; item += gridDim.x, ++slot) {
                const int st = (int)(slot % kHubStages);
                if (slot >= (uint32_t)kHubStages) {
                    mbar_wait(&empty[st], ((slot / kHubStages) - 1u) & 1u);
                    fence_proxy_async_smem();
                }
                const uint32_t hc = div_cpr(rm, item), ch = item - hc * rm.cpr;
                const int2 info = c.hub_chunk[hc];             // {variable, first CSC position}
                const int32_t split = c.code_off[2 * info.x + 1], end = c.code_off[2 * info.x + 2];
                const int32_t k1 = min(info.y + kHubChunk, end);
                const int32_t npos = min(max(split - info.y, 0), k1 - info.y);
                hdr[st] = make_int4(info.y, npos, k1 - info.y, (int32_t)hc);
                const uint32_t bytes = (uint32_t)(k1 - info.y) * 128u;
                mbar_arrive_expect_tx(&full[st], bytes);
                bulk_g2s(smem + st * kHubStageBytes, E + ((size_t)ch * c.L + info.y) * 32u, bytes, &full[st]);
            }
        }
    } else {
        const int sh = tid & 7;
        uint32_t slot = 0;
#if GALOIS_HUB_CF
        // Row pass with lane = word and warp = row subset (rows warp, warp + 8, ...): the 32
        // lanes of an LDS read 32 different banks (the quad mapping below would put the 8
        // row-sharing lanes of a word on one bank: 8-way conflicts). The 8 warps' partial
        // counters meet in shared memory (double-buffered by item parity, one named barrier
        // of the 256 consumer threads per item); thread (word tid / 8, quad tid % 8) sums
        // its 4 members' counts over them.
        constexpr int kHP = kHubChunk <= 248 ? 5 : 6;
        __shared__ uint32_t sP[2][kConsumerWarps][kHP][32];
        for (uint32_t item = blockIdx.x; item < rm.items; item += gridDim.x, ++slot) {
            const int st = (int)(slot % kHubStages);
            mbar_wait(&full[st], (slot / kHubStages) & 1u);
            const int4 h = hdr[st];
            uint32_t Q[kHP];
#pragma unroll
            for (int k = 0; k < kHP; ++k) Q[k] = 0;
            add_rows<kHP, (1 << kHP) - 1>(Q, reinterpret_cast<const uint32_t *>(smem + st * kHubStageBytes) + lane, h.z,
                                         warp);
            mbar_arrive(&empty[st]);                           // this thread is done with the stage
            const int pb = (int)(slot & 1u);
#pragma unroll
            for (int k = 0; k < kHP; ++k) sP[pb][warp][k][lane] = Q[k];
            asm volatile("bar.sync 1, %0;" ::"n"(kConsumerWarps * 32) : "memory");
            int32_t G[4] = {0, 0, 0, 0};
            const int w2 = tid >> 3;
#pragma unroll
            for (int k = 0; k < kHP; ++k) {
                uint32_t acc = 0;                               // bytes: <= 8 per member
#pragma unroll
                for (int wp = 0; wp < kConsumerWarps; ++wp) acc += quad_bits(sP[pb][wp][k][w2], sh);
#pragma unroll
                for (int j = 0; j < 4; ++j) G[j] += (int32_t)((acc >> (8 * j)) & 255u) << k;
            }
            const int32_t nneg = h.z - h.y;
            G[0] -= nneg; G[1] -= nneg; G[2] -= nneg; G[3] -= nneg;
            const uint32_t ch = item - (uint32_t)h.w * rm.cpr;
            partial[(size_t)h.w * rm.QW + ch * 256u + tid] = make_short4((short)G[0], (short)G[1], (short)G[2], (short)G[3]);
        }
#else
        for (uint32_t item = blockIdx.x; item < rm.items; item += gridDim.x, ++slot) {
            const int st = (int)(slot % kHubStages);
            mbar_wait(&full[st], (slot / kHubStages) & 1u);
            const int4 h = hdr[st];
            const uint32_t *srow = reinterpret_cast<const uint32_t *>(smem + st * kHubStageBytes) + (tid >> 3);
            int32_t G[4] = {0, 0, 0, 0};
            // h.z <= kHubChunk rows (the last h.z - h.y negative): per-thread share <= kHubChunk / 8
            count_rows_sliced<kHubChunk <= 248 ? 5 : 6>(reinterpret_cast<const uint32_t *>(smem + st * kHubStageBytes) + (tid >> 3), h.z,
                                 tid & 7, sh, G);
            const int32_t nneg = h.z - h.y;
            G[0] -= nneg; G[1] -= nneg; G[2] -= nneg; G[3] -= nneg;
            mbar_arrive(&empty[st]);
            const uint32_t ch = item - (uint32_t)h.w * rm.cpr;
            partial[(size_t)h.w * rm.QW + ch * 256u + tid] = make_short4((short)G[0], (short)G[1], (short)G[2], (short)G[3]);
        }
#endif
    }
}

// ------------------------------------ small instances: a whole run() in ONE launch (a3-a8)
// One CTA per 32-member word keeps its members' whole state in shared memory — z, m, v
// (n x 32 fp32 each), the X and R words of every variable and one E word per literal slot
// — and runs the steps itself: the clause pass (forward of X_s into E, Lambda, and the
// exact check of R_{s-1}), then the fused update of every (variable, quad) with the SAME
// quad_update() as k_update_tma, so every member's trajectory is bit-identical to the
// per-step kernels'. Members never interact, so CTAs meet only at check steps: each keeps
// its own best record (lexicographic (u, t, b); the winner's bits snapshotted on
// improvement), publishes a SAT at t* by atomicMin, and after a grid barrier (cooperative
// launch: all CTAs co-resident) every CTA stops before update(t* + 1), exactly where the
// per-step engine stops. The last CTA merges the records into the control block. Used by
// run() when the state fits shared memory (C1-sized instances, which the per-step path
// runs at ~12 us per step of launch latency).
struct SmallRec {
    int32_t u, t;
    int64_t b;
};

// Grid-wide barrier of a cooperative launch (all CTAs co-resident): a monotonic arrival
// counter, release add + acquire polls; the k-th barrier waits for k * gridDim.x arrivals
// (the last CTA zeroes the counter after the run).
__device__ __forceinline__ void grid_barrier(SmallScratch *gs, uint32_t target)
{
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(&gs->arrive) : "memory");
        uint32_t seen;
        for (;;) {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(&gs->arrive) : "memory");
            if (seen >= target) break;
            __nanosleep(8);
        }
    }
    __syncthreads();
}

template <bool kTau1, bool kAdam, bool kPins>
__global__ void __launch_bounds__(512) k_small_run(DevCnf c, StepParams p, int32_t T, int32_t K, int32_t pending0,
                                                   float4 *__restrict__ z4, float4 *__restrict__ m4,
                                                   float4 *__restrict__ v4, uint32_t *__restrict__ X,
                                                   uint32_t *__restrict__ R, int32_t *__restrict__ unsat_last,
                                                   int32_t *__restrict__ lam, SmallScratch *__restrict__ gs,
                                                   SmallRec *__restrict__ recs, uint8_t *__restrict__ snap,
                                                   uint8_t *__restrict__ best_bits, Ctrl *__restrict__ ctrl)
{
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ int32_t cntU[32], cntL[32];
    __shared__ int32_t s_bu, s_bt, s_flag, s_improved;
    __shared__ int64_t s_bb;
    if (ctrl->stopped) return;
    const int32_t n = c.n;
    const int tid = threadIdx.x, lane = tid & 31;
    const int w = blockIdx.x;                           // this CTA's 32-member word
    const uint32_t QW = (uint32_t)p.b_pad / 4u;
    const int64_t bw = p.b0 + 32 * (int64_t)w;         // global index of the word's member 0
    const int32_t nvalid = min(32, p.b_loc - 32 * w);   // existing members of the word
    float4 *sz = reinterpret_cast<float4 *>(smem);
    float4 *sm = sz + (size_t)n * 8;
    float4 *sv = sm + (size_t)n * 8;
    uint32_t *sX = reinterpret_cast<uint32_t *>(sv + (size_t)n * 8);
    uint32_t *sR = sX + n;
    uint32_t *sE = sR + n;                              // [L] in CSC order, plain (not complemented)
    for (int32_t i = tid; i < n * 8; i += blockDim.x) {
        const size_t idx = (size_t)(i >> 3) * QW + (size_t)w * 8 + (i & 7);
        sz[i] = z4[idx];
        sm[i] = m4[idx];
        sv[i] = v4[idx];
    }
    for (int32_t v = tid; v < n; v += blockDim.x) {
        sX[v] = X[xr_at(v, w, p.W)];
        sR[v] = R[xr_at(v, w, p.W)];
    }
    if (tid == 0) {
        s_bu = INT32_MAX;
        s_bt = -1;
        s_bb = -1;
    }
    const int32_t t0 = ctrl->t;
    bool pending = pending0 != 0, bad = false;
    int32_t s = t0 + 1;
    uint32_t barriers = 0;                              // arrivals the next barrier waits for
    for (;;) {
        const bool fwd = s <= T;
        if (!fwd && !pending) break;
        if (tid < 32) {
            cntU[tid] = 0;
            cntL[tid] = 0;
        }
        __syncthreads();
        // clause pass: thread per clause (sweep order); lane p of a warp then owns bit p
        int32_t myU = 0, myL = 0;
        for (int32_t base = 0; base < c.m; base += blockDim.x) {
            const int32_t ci = base + tid;
            uint32_t U = 0, UR = 0;
            if (ci < c.m) {
                const int32_t lo = c.sweep_off[ci], hi = c.sweep_off[ci + 1];
                uint32_t any = 0, two = 0, anyR = 0;
                for (int32_t k = lo; k < hi; ++k) {
                    const int2 si = c.sweep_slot[k];
                    const uint32_t neg = 0u - (uint32_t)(si.x & 1);
                    if (fwd) {
                        const uint32_t sl = sX[si.x >> 1] ^ neg;
                        two |= any & sl;
                        any |= sl;
                    }
                    if (pending) anyR |= sR[si.x >> 1] ^ neg;
                }
                if (fwd) {
                    for (int32_t k = lo; k < hi; ++k) {       // E_i = no OTHER literal true
                        const int2 si = c.sweep_slot[k];
                        const uint32_t sl = sX[si.x >> 1] ^ (0u - (uint32_t)(si.x & 1));
                        sE[si.y] = ~any | (sl & ~two);
                    }
                    U = ~any;
                }
                if (pending) UR = ~anyR;
            }
            for (int b = 0; b < 32; ++b) {
                if (fwd) {
                    const uint32_t bl = __ballot_sync(0xffffffffu, (U >> b) & 1u);
                    if (lane == b) myL += __popc(bl);
                }
                if (pending) {
                    const uint32_t bl = __ballot_sync(0xffffffffu, (UR >> b) & 1u);
                    if (lane == b) myU += __popc(bl);
                }
            }
        }
        if (fwd && myL) atomicAdd(&cntL[lane], myL);
        if (pending && myU) atomicAdd(&cntU[lane], myU);
        __syncthreads();
        if (pending) {                                   // exact check of R_{s-1}
            if (tid < 32) {
                const int32_t u = cntU[bitpos(tid)];
                if (tid < nvalid) unsat_last[32 * w + tid] = u;
                unsigned long long key = tid < nvalid ? ((unsigned long long)(uint32_t)u << 32) |
                                                            (unsigned long long)(bw + tid)
                                                      : ~0ull;
#pragma unroll
                for (int d = 16; d > 0; d >>= 1) {
                    const unsigned long long o = __shfl_xor_sync(0xffffffffu, key, d);
                    key = o < key ? o : key;
                }
                if (tid == 0) {
                    s_improved = 0;
                    if (key != ~0ull && (int64_t)(key >> 32) < (int64_t)s_bu) {
                        s_bu = (int32_t)(key >> 32);
                        s_bt = s - 1;
                        s_bb = (int64_t)(key & 0xFFFFFFFFull);
                        s_improved = 1;
                        if (s_bu == 0) atomicMin(&gs->tstar, s - 1);
                    }
                }
            }
            __syncthreads();
            if (s_improved) {                           // the new best member's rounding
                const int jb = bitpos((int)(s_bb - bw));
                for (int32_t v = tid; v < n; v += blockDim.x) snap[(size_t)w * n + v] = (uint8_t)((sR[v] >> jb) & 1u);
            }
        }
        if (!fwd) break;
        if (tid < nvalid) lam[(size_t)(s & 1) * p.b_pad + 32 * w + tid] = cntL[bitpos(tid)];
        if (pending) {
            // every CTA has checked R_{s-1}: a SAT anywhere stops all of them before update(s),
            // exactly where the per-step engine stops
            barriers += gridDim.x;
            grid_barrier(gs, barriers);
            if (tid == 0) s_flag = __ldcg(&gs->tstar) <= s - 1;
            __syncthreads();
            if (s_flag) break;
        }
        // fused update of step s: signal, gradient, Adam, R_s, X_{s+1}
        const float2 ac = p.adam_consts[s];
        for (int32_t base = 0; base < n * 8; base += blockDim.x) {
            const int32_t i = base + tid;
            const bool valid = i < n * 8;
            uint32_t xn = 0, rn = 0;
            if (valid) {
                const int32_t v = i >> 3, q = i & 7;
                const int32_t k0 = c.code_off[2 * v], k1 = c.code_off[2 * v + 1], k2 = c.code_off[2 * v + 2];
                int32_t G[4] = {0, 0, 0, 0};
                for (int32_t k = k0; k < k2; ++k) {
                    const uint32_t b = quad_bits(sE[k], q);
                    const int32_t sg = k < k1 ? 1 : -1;
#pragma unroll
                    for (int j = 0; j < 4; ++j) G[j] += sg * (int32_t)((b >> (8 * j)) & 1u);
                }
                const int64_t bq = p.b0 + 4 * ((int64_t)w * 8 + q);
                float4 z = sz[i], m = sm[i], vv = sv[i];
                float g1o[4];
                quad_update<kTau1, kAdam, kPins>(p, ac, v, bq, s, G, z, m, vv, xn, rn, g1o, bad);
                sz[i] = z;
                sm[i] = m;
                sv[i] = vv;
            }
            const uint32_t xw = pack_quads(xn, lane), rw = pack_quads(rn, lane);
            if (valid && (lane & 7) == 0) {
                sX[i >> 3] = xw;
                sR[i >> 3] = rw;
            }
        }
        __syncthreads();
        pending = (s % K) == 0 || s == T;
        ++s;
    }
    if (bad) atomicOr(&ctrl->nonfinite, 1);
    __syncthreads();
    for (int32_t i = tid; i < n * 8; i += blockDim.x) {
        const size_t idx = (size_t)(i >> 3) * QW + (size_t)w * 8 + (i & 7);
        z4[idx] = sz[i];
        m4[idx] = sm[i];
        v4[idx] = sv[i];
    }
    for (int32_t v = tid; v < n; v += blockDim.x) {
        X[xr_at(v, w, p.W)] = sX[v];
        R[xr_at(v, w, p.W)] = sR[v];
    }
    // the last CTA merges the records (lexicographic (u, t, b), with the record of earlier runs)
    if (tid == 0) {
        recs[w] = SmallRec{s_bu, s_bt, s_bb};
        __threadfence();
        s_flag = atomicAdd(&gs->done, 1u) == gridDim.x - 1u;
    }
    __syncthreads();
    if (!s_flag) return;
    __threadfence();
    if (tid == 0) {
        int32_t bu = ctrl->best_u, bt = ctrl->best_t;
        int64_t bb = ctrl->best_b;
        int win = -1;
        for (int k = 0; k < (int)gridDim.x; ++k) {
            SmallRec r;                                  // written by other CTAs: bypass L1
            r.u = __ldcg(&recs[k].u);
            r.t = __ldcg(&recs[k].t);
            r.b = __ldcg(&recs[k].b);
            if (r.b < 0) continue;
            if (r.u < bu || (r.u == bu && (r.t < bt || (r.t == bt && r.b < bb)))) {
                bu = r.u;
                bt = r.t;
                bb = r.b;
                win = k;
            }
        }
        ctrl->improved = win >= 0 ? 1 : 0;
        ctrl->best_u = bu;
        ctrl->best_t = bt;
        ctrl->best_b = bb;
        const int32_t tstar = *(volatile int32_t *)&gs->tstar;
        ctrl->stopped = bu == 0 ? 1 : 0;
        ctrl->t = bu == 0 ? tstar : T;
        ctrl->last_check_t = ctrl->t;
        gs->tstar = 0x7f7f7f7f;                         // ready for the next run
        gs->done = 0;
        gs->arrive = 0;
        s_bu = win;
    }
    __syncthreads();
    if (s_bu >= 0)
        for (int32_t v = tid; v < n; v += blockDim.x) best_bits[v] = snap[(size_t)s_bu * n + v];
}

// ------------------------------------------------------------------ launch wrappers
// ---------------- a6 + a7: fused update for sub-1024 windows, TMA-pipelined (32 % W == 0)
// Batches of 32, 64, 128, 256 or 512 members (W = b_pad / 32 in {1, 2, 4, 8, 16}: f4's
// sub-batch windows on instances too large for 1024 resident members). E rows are
// W words (E[L][W], CSC order), so an item is a GROUP of R = 32 / W consecutive variables
// x all their members — 256 quads, one per consumer thread — and its z, m, v are 3 x 4 KB
// contiguous, its E rows one contiguous CSC range. The producer warp bulk-copies z, m, v
// and the group's rows (minus hub variables' rows, which come from the hub partials) into
// kSwStages-deep ring stages of kSwE bytes, splitting long ranges into pieces; a consumer
// thread counts the rows of its own variable that fall in each piece. Same per-quad
// arithmetic (quad_update) as k_update_st, so iterates are bit-identical to it.
#ifndef GALOIS_UPD_SMALLW
#define GALOIS_UPD_SMALLW 1
#endif
#ifndef GALOIS_SMALLW_STAGES
#define GALOIS_SMALLW_STAGES 3
#endif
#ifndef GALOIS_SMALLW_E
#define GALOIS_SMALLW_E 8192
#endif
#ifndef GALOIS_SMALLW_CTAS
#define GALOIS_SMALLW_CTAS 3
#endif
constexpr int kSwStages = GALOIS_SMALLW_STAGES;
constexpr int kSwCtasPerSm = GALOIS_SMALLW_CTAS;
constexpr int kSwE = GALOIS_SMALLW_E;                     // E bytes per stage
constexpr int kSwStageBytes = kSwE + 3 * 4096;
constexpr int kSwSmem = kSwStages * kSwStageBytes;

struct SwHdr {
    int32_t r0, r1;    // CSC rows [r0, r1) of this piece
    int32_t ra;        // first row copied (r0 rounded down to a 16-byte boundary)
};

template <bool kTau1, bool kAdam, bool kPins>
__global__ void __launch_bounds__(256 + 32, kSwCtasPerSm)
    k_update_smallw(DevCnf c, StepParams p, int32_t W, uint32_t groups, float4 *__restrict__ z4,
                    float4 *__restrict__ m4, float4 *__restrict__ v4, uint32_t *__restrict__ X,
                    uint32_t *__restrict__ R, const uint32_t *__restrict__ E, const short4 *__restrict__ partial,
                    Ctrl *__restrict__ ctrl)
{
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ uint64_t full[kSwStages], empty[kSwStages];
    __shared__ SwHdr hdr[kSwStages];
    __shared__ int32_t hflags[kSwStages];   // bit 0: z, m, v in this stage; bit 1: the group's last stage
    __shared__ int4 vinfo[kSwStages][32];   // first stage of a group: {k0, k1, k2, hub} per variable
    if (ctrl->stopped) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t QW = 8u * (uint32_t)W;    // quads per variable row
    const int32_t RG = 32 / W;               // variables per group
    const uint32_t full_s = smem_u32(full), empty_s = smem_u32(empty), stage_s = smem_u32(smem);
    if (tid == 0) {
        for (int i = 0; i < kSwStages; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 32 * kConsumerWarps);
        }
        fence_mbar_init();
    }
    __syncthreads();

    if (warp == kConsumerWarps) {          // ------------------------------ producer warp
        const int32_t rpa = W >= 4 ? 1 : 4 / W;             // rows per 16 bytes
        const int32_t cap = kSwE / (4 * W);                  // rows per stage (a multiple of rpa)
        int st = 0;
        uint32_t ph = 0;
        bool wrapped = false;
        for (uint32_t g = blockIdx.x; g < groups; g += gridDim.x) {
            const int32_t v0 = (int32_t)g * RG, nv = min(RG, c.n - v0);
            // lane j: variable v0 + j's CSC range and whether it is a hub
            int32_t kb = 0, kn = 0, ke = 0, hubi = -1;
            bool hub = false;
            if (lane < nv) {
                kb = c.code_off[2 * (v0 + lane)];
                kn = c.code_off[2 * (v0 + lane) + 1];
                ke = c.code_off[2 * (v0 + lane) + 2];
                hubi = c.num_hubs > 0 ? c.hub_of_var[v0 + lane] : -1;
                hub = hubi >= 0;
            }
            uint32_t hm = __ballot_sync(0xffffffffu, hub);
            const int32_t end = __shfl_sync(0xffffffffu, ke, nv - 1);
            int32_t a = __shfl_sync(0xffffffffu, kb, 0);
            bool first = true;
            // pieces of [a, b) (the last one of the group flagged when `fin`)
            auto pieces = [&](int32_t lo, int32_t hi, bool fin) {
                while (true) {
                    const int32_t ra = lo / rpa * rpa;
                    const int32_t r1 = min(hi, ra + cap);
                    const bool last = fin && r1 >= hi;
                    if (r1 > lo || last || first) {
                        if (lane == 0 && wrapped) {
                            mbar_wait_s(empty_s + 8u * st, ph ^ 1u);
                            fence_proxy_async_smem();
                        }
                        __syncwarp();
                        // the group's variable table travels with its first stage (the
                        // consumers read it from shared memory instead of global)
                        if (first && lane < nv) vinfo[st][lane] = make_int4(kb, kn, ke, hubi);
                        __syncwarp();
                        if (lane == 0) {
                            hdr[st] = SwHdr{lo, max(lo, r1), ra};
                            hflags[st] = (first ? 1 : 0) | (last ? 2 : 0);
                            const int32_t rb = r1 > lo ? (r1 + rpa - 1) / rpa * rpa : ra;
                            const uint32_t ebytes = (uint32_t)(rb - ra) * 4u * (uint32_t)W;
                            GALOIS_DEV_CHECK(ra >= 0 && ra <= lo && rb >= ra && ebytes <= (uint32_t)kSwE &&
                                             (int64_t)rb * W <= (int64_t)c.L * W + 4);
                            const uint32_t zb = (uint32_t)nv * QW * 16u;
                            const uint32_t fb = full_s + 8u * st, sbs = stage_s + (uint32_t)(st * kSwStageBytes);
                            mbar_arrive_expect_tx_s(fb, (first ? 3u * zb : 0u) + ebytes);
                            if (first) {
                                const size_t off = (size_t)v0 * QW;
                                bulk_g2s_s(sbs + kSwE, z4 + off, zb, fb);
                                bulk_g2s_s(sbs + kSwE + 4096, m4 + off, zb, fb);
                                bulk_g2s_s(sbs + kSwE + 8192, v4 + off, zb, fb);
                            }
                            if (ebytes) bulk_g2s_s(sbs, E + (size_t)ra * W, ebytes, fb);
                        }
                        __syncwarp();
                        first = false;
                        if (++st == kSwStages) {
                            st = 0;
                            ph ^= 1u;
                            wrapped = true;
                        }
                    }
                    if (r1 >= hi) break;
                    lo = r1;
                }
            };
            while (hm) {                                     // skip the hub variables' rows
                const int j = __ffs(hm) - 1;
                hm &= hm - 1;
                pieces(a, __shfl_sync(0xffffffffu, kb, j), false);
                a = __shfl_sync(0xffffffffu, ke, j);
            }
            pieces(a, max(a, end), true);
        }
    } else {
    // ------------------------------------------------------------------ consumer warps
    const int32_t s = ctrl->t + 1;
    const float2 ac = p.adam_consts[s];
    bool bad = false;
    for (int32_t i = blockIdx.x * 256 + tid; i < p.b_pad; i += gridDim.x * 256) {   // next sweep's counters
        if (p.clear_a) p.clear_a[i] = 0;
        if (p.clear_b) p.clear_b[i] = 0;
    }
    const uint32_t r_t = (uint32_t)tid / QW, q = (uint32_t)tid - r_t * QW;   // variable in group, quad
    const int sh = tid & 7;                  // quad within its 32-member word (QW % 8 == 0)
    const uint32_t wq = q >> 3;              // word within the row
    int st = 0;
    uint32_t ph = 0;
    for (uint32_t g = blockIdx.x; g < groups; g += gridDim.x) {
        const int32_t v = (int32_t)g * RG + (int32_t)r_t;
        const bool valid = v < c.n;
        int32_t k0 = 0, k1 = 0, k2 = 0, hub = -1;
        float4 z = make_float4(0.f, 0.f, 0.f, 0.f), m = z, vv = z;
        int32_t G[4] = {0, 0, 0, 0};
        int32_t flags = 0;
        do {
            mbar_wait_s(full_s + 8u * st, ph);
            const SwHdr h = hdr[st];
            flags = hflags[st];
            const uint8_t *sb = smem + st * kSwStageBytes;
            if ((flags & 1) && valid) {
                const int4 vi = vinfo[st][r_t];
                k0 = vi.x;
                k1 = vi.y;
                k2 = vi.z;
                hub = vi.w;
                z = reinterpret_cast<const float4 *>(sb + kSwE)[tid];
                m = reinterpret_cast<const float4 *>(sb + kSwE + 4096)[tid];
                vv = reinterpret_cast<const float4 *>(sb + kSwE + 8192)[tid];
            }
            if (valid && hub < 0) {
                const int32_t a = max(h.r0, k0), b = min(h.r1, k2);
                if (b > a) {
                    GALOIS_DEV_CHECK(a >= h.ra && (b - h.ra) * W <= kSwE / 4 && b - a <= 256);
                    const uint32_t *srow = reinterpret_cast<const uint32_t *>(sb) + (a - h.ra) * W + wq;
                    static_assert(kHubDegree <= 256, "one SWAR pass + one row");
                    // SWAR bytes: a non-hub variable has <= kHubDegree = 256 rows, so 255 of
                    // them fit a byte and at most one more is added on its own
                    const int32_t nr = b - a, n1 = min(nr, 255);
                    uint32_t acc = 0;
#pragma unroll 8
                    for (int32_t k = 0; k < n1; ++k) acc += quad_bits(srow[k * W], sh);
#pragma unroll
                    for (int j = 0; j < 4; ++j) G[j] += (int32_t)((acc >> (8 * j)) & 255u);
                    if (nr > 255) {
                        const uint32_t last = quad_bits(srow[255 * W], sh);
#pragma unroll
                        for (int j = 0; j < 4; ++j) G[j] += (int32_t)((last >> (8 * j)) & 1u);
                    }
                    const int32_t nneg = b - max(a, k1);          // negative rows are complemented
                    if (nneg > 0) { G[0] -= nneg; G[1] -= nneg; G[2] -= nneg; G[3] -= nneg; }
                }
            }
            mbar_arrive_s(empty_s + 8u * st);
            if (++st == kSwStages) {
                st = 0;
                ph ^= 1u;
            }
        } while (!(flags & 2));
        uint32_t xn = 0, rn = 0;
        if (valid) {
            if (hub >= 0) hub_signal(c, partial, QW, hub, q, G);
            const int64_t bq = p.b0 + 4 * (int64_t)q;
            float g1o[4];
            quad_update<kTau1, kAdam, kPins>(p, ac, v, bq, s, G, z, m, vv, xn, rn, g1o, bad);
            const size_t idx = (size_t)v * QW + q;
            z4[idx] = z;
            m4[idx] = m;
            v4[idx] = vv;
        }
        const uint32_t xw = pack_quads(xn, lane), rw = pack_quads(rn, lane);   // 8-lane groups stay in a row
        if (valid && (lane & 7) == 0) {
            X[xr_at(v, (int32_t)wq, p.W)] = xw;
            R[xr_at(v, (int32_t)wq, p.W)] = rw;
        }
    }
    if (bad) atomicOr(&ctrl->nonfinite, 1);
    }                                      // consumer warps
    last_cta_tick(ctrl);
}

namespace launch {

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
    // x / cpr == (umulhi(x, mul) + x) >> shift for all 32-bit x (64-bit add)
    uint32_t l = 0;
    while ((1ull << l) < rm.cpr) ++l;
    rm.div_shift = l;
    rm.div_mul = rm.cpr == 1 ? 0u : (uint32_t)((((1ull << l) - rm.cpr) << 32) / rm.cpr + 1ull);
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
    if (W % 32 == 0)
        k_hub_partial_tma<<<item_grid(rm, kHubCtasPerSm), 256 + 32, kHubStages * kHubStageBytes, st>>>(c, rm, E, partial,
                                                                                                   ctrl);
    else
        k_hub_partial<<<item_grid(rm, 8), 256, 0, st>>>(c, W < 32 ? W : 32, rm, E, partial, ctrl);
}

using UpdKernel = void (*)(DevCnf, StepParams, RowMap, float4 *, float4 *, float4 *, uint32_t *, uint32_t *,
                           const uint32_t *, const short4 *, Ctrl *, int4 *, float4 *);

template <template <bool, bool, bool, bool> class Sel>
static UpdKernel pick(int variant)
{
    static const UpdKernel table[16] = {
        Sel<false, false, false, false>::k, Sel<false, false, false, true>::k, Sel<false, false, true, false>::k,
        Sel<false, false, true, true>::k,   Sel<false, true, false, false>::k,  Sel<false, true, false, true>::k,
        Sel<false, true, true, false>::k,   Sel<false, true, true, true>::k,    Sel<true, false, false, false>::k,
        Sel<true, false, false, true>::k,   Sel<true, false, true, false>::k,   Sel<true, false, true, true>::k,
        Sel<true, true, false, false>::k,   Sel<true, true, false, true>::k,    Sel<true, true, true, false>::k,
        Sel<true, true, true, true>::k,
    };
    return table[variant];
}

template <bool a, bool b, bool c, bool d>
struct SelGeneric {
    static constexpr UpdKernel k = k_update_st<a, b, c, d>;
};
template <bool a, bool b, bool c, bool d>
struct SelTma {
    static constexpr UpdKernel k = k_update_tma<a, b, c, d, false>;
};
using PairKernel = void (*)(DevCnf, StepParams, RowMap, float4 *, float4 *, float4 *, uint32_t *, uint32_t *,
                            const uint32_t *, const short4 *, Ctrl *);
static PairKernel pick_pair(int variant)   // variant bits: 4 tau1, 2 adam, 1 pins
{
    static const PairKernel table[8] = {k_update_pair<false, false, false>, k_update_pair<false, false, true>,
                                        k_update_pair<false, true, false>,  k_update_pair<false, true, true>,
                                        k_update_pair<true, false, false>,  k_update_pair<true, false, true>,
                                        k_update_pair<true, true, false>,   k_update_pair<true, true, true>};
    return table[variant & 7];
}
#ifndef GALOIS_UPD_PAIR
#define GALOIS_UPD_PAIR 1
#endif
using SmallWKernel = void (*)(DevCnf, StepParams, int32_t, uint32_t, float4 *, float4 *, float4 *, uint32_t *,
                              uint32_t *, const uint32_t *, const short4 *, Ctrl *);
static SmallWKernel pick_smallw(int variant)   // variant bits: 4 tau1, 2 adam, 1 pins
{
    static const SmallWKernel table[8] = {k_update_smallw<false, false, false>, k_update_smallw<false, false, true>,
                                          k_update_smallw<false, true, false>,  k_update_smallw<false, true, true>,
                                          k_update_smallw<true, false, false>,  k_update_smallw<true, false, true>,
                                          k_update_smallw<true, true, false>,   k_update_smallw<true, true, true>};
    return table[variant & 7];
}

template <bool a, bool b, bool c, bool d>
struct SelTmaSliced {
    static constexpr UpdKernel k = k_update_tma<a, b, c, d, true>;
};
// high average degree (5-SAT-like): E rows counted bit-sliced across a variable's pieces
static bool use_sliced(const DevCnf &c) { return (int64_t)c.L >= (int64_t)kSlicedMinAvgDegree * c.n; }

bool use_tma_update(int32_t W) { return W % 32 == 0; }

// Function attributes (dynamic shared memory of the TMA kernels) for the current device;
// called once per engine before any launch (and so never during CUDA-graph capture).
size_t small_run_smem(int32_t n, int32_t L) { return (size_t)n * 8 * 16 * 3 + (size_t)n * 8 + (size_t)L * 4; }

cudaError_t small_run(const DevCnf &c, const StepParams &p, int32_t T, int32_t K, bool pending, float *z, float *m,
                      float *v, uint32_t *X, uint32_t *R, int32_t *unsat_last, int32_t *lam, SmallScratch *gs,
                      void *recs, uint8_t *snap, uint8_t *best_bits, Ctrl *ctrl, cudaStream_t st)
{
    using K_t = void (*)(DevCnf, StepParams, int32_t, int32_t, int32_t, float4 *, float4 *, float4 *, uint32_t *,
                         uint32_t *, int32_t *, int32_t *, SmallScratch *, SmallRec *, uint8_t *, uint8_t *, Ctrl *);
    static const K_t ks[8] = {k_small_run<false, false, false>, k_small_run<false, false, true>,
                              k_small_run<false, true, false>,  k_small_run<false, true, true>,
                              k_small_run<true, false, false>,  k_small_run<true, false, true>,
                              k_small_run<true, true, false>,   k_small_run<true, true, true>};
    const int variant = (p.inv_tau == 1.0f ? 4 : 0) | (p.optimizer == 0 ? 2 : 0) | (p.pin_rank ? 1 : 0);
    const K_t k = ks[variant];
    const size_t smem = small_run_smem(c.n, c.L);
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    // cooperative launch: every CTA must be resident for the grid barrier (else the caller
    // takes the per-step path)
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, 512, smem);
    if (e != cudaSuccess) return e;
    const unsigned grid = (unsigned)(p.b_pad / 32);
    if ((int64_t)per_sm * sms < (int64_t)grid) return cudaErrorCooperativeLaunchTooLarge;
    int32_t pend = pending ? 1 : 0;
    float4 *z4 = (float4 *)z, *m4 = (float4 *)m, *v4 = (float4 *)v;
    SmallRec *rc = (SmallRec *)recs;
    DevCnf cc = c;
    StepParams pp = p;
    void *args[] = {&cc, &pp, &T, &K, &pend, &z4, &m4, &v4, &X, &R, &unsat_last, &lam, &gs, &rc, &snap, &best_bits, &ctrl};
    return cudaLaunchCooperativeKernel((const void *)k, dim3(grid), dim3(512), args, smem, st);
}

cudaError_t configure_kernels()
{
    static std::atomic<uint64_t> done{0};
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 64 && (done.load() >> dev) & 1ull) return cudaSuccess;
    for (int v = 0; v < 16; ++v) {
        e = cudaFuncSetAttribute((const void *)pick<SelTma>(v), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 kTmaSmem);
        if (e != cudaSuccess) return e;
        e = cudaFuncSetAttribute((const void *)pick<SelTmaSliced>(v), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 kTmaSmem);
        if (e != cudaSuccess) return e;
    }
    for (int v = 0; v < 8; ++v) {
        e = cudaFuncSetAttribute((const void *)pick_pair(v), cudaFuncAttributeMaxDynamicSharedMemorySize, kPairSmem);
        if (e != cudaSuccess) return e;
    }
    for (int v = 0; v < 8; ++v) {
        e = cudaFuncSetAttribute((const void *)pick_smallw(v), cudaFuncAttributeMaxDynamicSharedMemorySize, kSwSmem);
        if (e != cudaSuccess) return e;
    }
    e = cudaFuncSetAttribute((const void *)k_hub_partial_tma, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             kHubStages * kHubStageBytes);
    if (e != cudaSuccess) return e;
    if (dev < 64) done.fetch_or(1ull << dev);
    return cudaSuccess;
}

void update_st(const DevCnf &c, const StepParams &p, float *z, float *m, float *v, uint32_t *X, uint32_t *R,
               const uint32_t *E, const short4 *partial, Ctrl *ctrl, int32_t *dbg_G, float *dbg_g1,
               cudaStream_t st)
{
    const RowMap rm = make_rowmap((uint32_t)p.n, (uint32_t)p.b_pad);
    const int variant = (dbg_G ? 8 : 0) | (p.inv_tau == 1.0f ? 4 : 0) | (p.optimizer == 0 ? 2 : 0) |
                        (p.pin_rank ? 1 : 0);
    if (GALOIS_UPD_PAIR && use_tma_update(p.W) && !dbg_G && !use_sliced(c)) {
        const RowMap rp = make_rowmap(((uint32_t)p.n + 1u) / 2u, (uint32_t)p.b_pad);
        pick_pair(variant)<<<item_grid(rp, kPairCtasPerSm), 256 + 32, kPairSmem, st>>>(
            c, p, rp, (float4 *)z, (float4 *)m, (float4 *)v, X, R, E, partial, ctrl);
    } else if (use_tma_update(p.W)) {
        // smem attribute set by configure_kernels()
        const UpdKernel k = use_sliced(c) ? pick<SelTmaSliced>(variant) : pick<SelTma>(variant);
        k<<<item_grid(rm, kTmaCtasPerSm), 256 + 32, kTmaSmem, st>>>(c, p, rm, (float4 *)z, (float4 *)m, (float4 *)v, X, R, E,
                                                   partial, ctrl, (int4 *)dbg_G, (float4 *)dbg_g1);
    } else if (GALOIS_UPD_SMALLW && !dbg_G && p.W < 32 && 32 % p.W == 0) {
        const uint32_t RG = 32u / (uint32_t)p.W, groups = ((uint32_t)p.n + RG - 1u) / RG;
        unsigned grid = 148u * kSwCtasPerSm;
        if (groups < grid) grid = groups < 1 ? 1 : groups;
        pick_smallw(variant)<<<grid, 256 + 32, kSwSmem, st>>>(c, p, p.W, groups, (float4 *)z, (float4 *)m,
                                                             (float4 *)v, X, R, E, partial, ctrl);
    } else {
        const UpdKernel k = pick<SelGeneric>(variant);
        k<<<item_grid(rm, 8), 256, 0, st>>>(c, p, rm, (float4 *)z, (float4 *)m, (float4 *)v, X, R, E, partial,
                                            ctrl, (int4 *)dbg_G, (float4 *)dbg_g1);
    }
}

}  // namespace launch
}  // namespace galois
