// philox.cuh — the CUDA path's counter-based RNG (reading R2 of DESIGN.md).
//
// Philox4x32-10 (Salmon et al., SC'11). One call yields four 32-bit words, which is
// exactly one "quad" of four consecutive batch members in the noise layout
// (counter (v, b/4, t, 1), word b mod 4), or two members of the init layout
// (counter (v, b/2, 0, 0), words 2(b mod 2), 2(b mod 2)+1).
#pragma once
#include <cstdint>

namespace galois {

__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k)
{
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint64_t p0 = (uint64_t)0xD2511F53u * c.x;   // one IMAD.WIDE.U32 each
        const uint64_t p1 = (uint64_t)0xCD9E8D57u * c.z;
        c = make_uint4((uint32_t)(p1 >> 32) ^ c.y ^ k.x, (uint32_t)p1, (uint32_t)(p0 >> 32) ^ c.w ^ k.y, (uint32_t)p0);
        k.x += 0x9E3779B9u;
        k.y += 0xBB67AE85u;
    }
    return c;
}

// Same generator with the 10 round keys precomputed on the host (key + r * W for
// r = 0..9) and passed as kernel parameters: each round is then two IMAD.WIDE and two
// LOP3 whose key operand comes straight from the constant bank.
struct PhiloxKeys {
    uint32_t k0[10];
    uint32_t k1[10];
};

inline PhiloxKeys philox_round_keys(uint64_t seed)
{
    PhiloxKeys pk;
    uint32_t a = (uint32_t)seed, b = (uint32_t)(seed >> 32);
    for (int r = 0; r < 10; ++r) {
        pk.k0[r] = a;
        pk.k1[r] = b;
        a += 0x9E3779B9u;
        b += 0xBB67AE85u;
    }
    return pk;
}

#ifndef GALOIS_PHILOX_ROUNDS_EXPERIMENT
#define GALOIS_PHILOX_ROUNDS_EXPERIMENT 10   // timing experiment only: results differ from the oracle
#endif
#if GALOIS_PHILOX_ROUNDS_EXPERIMENT != 10 && !defined(GALOIS_PARITY_BREAKING_EXPERIMENT)
#error "GALOIS_PHILOX_ROUNDS_EXPERIMENT breaks oracle parity: also define GALOIS_PARITY_BREAKING_EXPERIMENT"
#endif
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, const PhiloxKeys &pk)
{
#pragma unroll
    for (int r = 0; r < GALOIS_PHILOX_ROUNDS_EXPERIMENT; ++r) {
        const uint64_t p0 = (uint64_t)0xD2511F53u * c.x;
        const uint64_t p1 = (uint64_t)0xCD9E8D57u * c.z;
        c = make_uint4((uint32_t)(p1 >> 32) ^ c.y ^ pk.k0[r], (uint32_t)p1, (uint32_t)(p0 >> 32) ^ c.w ^ pk.k1[r],
                       (uint32_t)p0);
    }
    return c;
}

// Open-interval uniform pair (u, 1 - u) from the low 23 bits k of a word (reading R2):
// f = 1 + k 2^-23 is built by OR-ing k into the mantissa of 1.0f, and
// u = f - (1 - 2^-24) = (2k+1) 2^-24, 1 - u = (2^24 - 1 - 2k) 2^-24 are both exact in
// binary32 (24 significant bits; Sterbenz), so the pair costs one LOP3 and two FADDs.
__device__ __forceinline__ float2 unif_pair(uint32_t w)
{
    uint32_t b;                             // (w & 0x7FFFFF) | 0x3F800000 in ONE LOP3
    asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(b) : "r"(w), "r"(0x7FFFFFu), "r"(0x3F800000u));
    const float f = __uint_as_float(b);
    const float u = f - 0.999999940395355224609375f;
    return make_float2(u, 1.0f - u);
}

// Logistic(0,1) draw ell = ln u - ln(1 - u) = g_1 - g_0 (Eq.3).
// lg2.approx has absolute error <= 2^-22.6 for arguments in [0.5, 2] and relative error
// 2^-22 elsewhere, so |d ell| <~ 2.3e-7 + 2.4e-7 |ell|.
__device__ __forceinline__ float logistic_from_word(uint32_t w)
{
    const float2 uu = unif_pair(w);
    return (__log2f(uu.x) - __log2f(uu.y)) * 0.69314718055994531f;
}

// Init uniform (2k+1) 2^-24, k = the low 23 bits of the word: exact in binary32.
__device__ __forceinline__ float uniform_f32(uint32_t w)
{
    return (float)(((w & 0x7FFFFFu) << 1) | 1u) * (1.0f / 16777216.0f);
}

}  // namespace galois
