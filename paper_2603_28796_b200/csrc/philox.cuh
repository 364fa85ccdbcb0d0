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
        const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
        const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
        c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
        k.x += 0x9E3779B9u;
        k.y += 0xBB67AE85u;
    }
    return c;
}

// Logistic(0,1) draw ell = ln u - ln(1 - u) = g_1 - g_0 (Eq.3) from the top
// 23 bits k of a word: u = (2k+1) 2^-24 and 1 - u = (2^24 - 1 - 2k) 2^-24 are exact in
// binary32. lg2.approx has absolute error <= 2^-22.6 for arguments in [0.5, 2] and
// relative error 2^-22 elsewhere, so |d ell| <~ 2.3e-7 + 2.4e-7 |ell|.
__device__ __forceinline__ float logistic_from_word(uint32_t w)
{
    const uint32_t k2 = (w >> 9) << 1;
    const float u = __uint2float_rn(k2 + 1u) * 5.9604644775390625e-8f;       // (2k+1) 2^-24
    const float ub = __uint2float_rn(16777215u - k2) * 5.9604644775390625e-8f; // 1 - u, exact
    return (__log2f(u) - __log2f(ub)) * 0.69314718055994531f;
}

// Same draw in fp64 (init path only).
__device__ __forceinline__ double uniform_f64(uint32_t w)
{
    return (double)(((w >> 9) << 1) | 1u) * (1.0 / 16777216.0);  // (2k+1) 2^-24
}

}  // namespace galois
