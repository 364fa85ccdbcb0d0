// select_kernels.cu — NEXT rows f1 and f3 of SURVEY §8(f): what the CPU stage consumes.
//
//   k_select    theta_sel ("the batch with the minimal clause loss"; "the one
//               with the highest loss value"): arg min / arg max of the exact unsat counts
//               of the last check, ties to the lower member
//   k_gather_z  the selected member's reduced logits z_v = theta_{v,1} - theta_{v,0}
//   k_pool      candidate pool (Eq.10): N Gumbel samples of theta_sel,
//               x^(k)_v = [z_v + ell^(k)_v >= 0], confidence c^(k)_v = max(y0, y1)
//               = sigma(|a|), a = (z_v + ell^(k)_v) / tau; ell from Philox counter
//               (v, k/4, 0, 2) word k mod 4 under the pool seed
//   k_topk      per candidate, the |S| most confident variables (Eq.11): exact
//               radix select over the unique 64-bit keys (conf bits, ~v) — descending
//               confidence, ties to the lower index — emitted as unit literals
//   k_lowconf   the d least confident variables of theta_sel (Lemma 1 branching):
//               radix select of the d smallest (|z| bits, v), i.e. noise-free confidence
//               sigma(|z|/tau) ascending, ties to the lower index
#include <cuda_runtime.h>

#include <cstdint>

#include "device_utils.cuh"
#include "galois_internal.h"
#include "philox.cuh"

namespace galois {

namespace {
constexpr int kSelThreads = 1024;
constexpr int kMaxSorted = 4096;    // largest |S| / d the per-CTA selection sorts

// Exact selection of the `want` largest 64-bit keys among key_of(0..n-1) by one CTA
// (8 radix passes of 8 bits over the candidates sharing the current prefix). Returns the
// threshold key: the selected set is exactly { i : key_of(i) >= threshold } (keys unique).
template <typename KeyOf>
__device__ uint64_t select_threshold(int32_t n, int32_t want, KeyOf key_of)
{
    __shared__ int32_t hist[256];
    __shared__ uint64_t s_prefix;
    __shared__ int32_t s_remaining;
    if (threadIdx.x == 0) {
        s_prefix = 0;
        s_remaining = want;
    }
    __syncthreads();
    uint64_t mask = 0;
    for (int p = 7; p >= 0; --p) {
        for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
        __syncthreads();
        const uint64_t prefix = s_prefix;
        for (int32_t i = threadIdx.x; i < n; i += blockDim.x) {
            const uint64_t k = key_of(i);
            if ((k & mask) == prefix) atomicAdd(&hist[(k >> (8 * p)) & 255u], 1);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            int32_t rem = s_remaining, cum = 0;
            for (int b = 255; b >= 0; --b) {
                if (cum + hist[b] >= rem) {
                    s_prefix = prefix | ((uint64_t)b << (8 * p));
                    s_remaining = rem - cum;
                    break;
                }
                cum += hist[b];
            }
        }
        mask |= (uint64_t)255u << (8 * p);
        __syncthreads();
    }
    return s_prefix;
}

// Collect the keys >= thr (exactly `count` of them) and sort them descending (bitonic) in
// s_keys: shared memory up to kMaxSorted keys, else a global scratch row of the block
// (__syncthreads orders the block's global accesses as it does its shared ones).
template <typename KeyOf>
__device__ void collect_sorted_desc(int32_t n, int32_t count, uint64_t thr, KeyOf key_of, uint64_t *s_keys)
{
    __shared__ int32_t s_n;
    int32_t P = 1;
    while (P < count) P <<= 1;
    for (int i = threadIdx.x; i < P; i += blockDim.x) s_keys[i] = 0;   // padding sorts last
    if (threadIdx.x == 0) s_n = 0;
    __syncthreads();
    for (int32_t i = threadIdx.x; i < n; i += blockDim.x) {
        const uint64_t k = key_of(i);
        if (k >= thr) s_keys[atomicAdd(&s_n, 1)] = k;
    }
    __syncthreads();
    for (int size = 2; size <= P; size <<= 1)
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = threadIdx.x; i < P; i += blockDim.x) {
                const int j = i ^ stride;
                if (j > i) {
                    const bool desc = (i & size) == 0;
                    const uint64_t a = s_keys[i], b = s_keys[j];
                    if ((a < b) == desc) {
                        s_keys[i] = b;
                        s_keys[j] = a;
                    }
                }
            }
            __syncthreads();
        }
}
}  // namespace

// rule 0: arg min, 1: arg max of the counts; ties to the lower global member.
__global__ void __launch_bounds__(kSelThreads) k_select(const int32_t *__restrict__ counts, int32_t b_loc, int64_t b0,
                                                        int32_t rule, unsigned long long *__restrict__ out)
{
    __shared__ unsigned long long s_min[32];
    unsigned long long best = ~0ull;
    for (int32_t i = threadIdx.x; i < b_loc; i += blockDim.x) {
        const uint32_t u = (uint32_t)counts[i];
        const unsigned long long key = ((unsigned long long)(rule ? ~u : u) << 32) | (unsigned long long)(b0 + i);
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
        *out = best;
    }
}

__global__ void k_gather_z(const float *__restrict__ z, int32_t n, int32_t b_pad, int32_t lb, float *__restrict__ out)
{
    for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
        out[v] = z[(size_t)v * b_pad + lb];
}

// Candidates k0 .. k0 + N - 1 over the variables 0 .. n - 1 (rows of n, candidate k0 first).
__global__ void __launch_bounds__(256) k_pool(const float *__restrict__ zsel, int32_t n, int32_t k0, int32_t N,
                                              float inv_tau, PhiloxKeys keys, uint8_t *__restrict__ x,
                                              float *__restrict__ conf)
{
    const int64_t total = (int64_t)N * n;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t kr = (int32_t)(i / n), v = (int32_t)(i - (int64_t)kr * n), k = k0 + kr;
        const uint4 w = philox4x32_10(make_uint4((uint32_t)v, (uint32_t)(k >> 2), 0u, 2u), keys);
        const uint32_t wk = (k & 3) == 0 ? w.x : (k & 3) == 1 ? w.y : (k & 3) == 2 ? w.z : w.w;
        const float a = (zsel[v] + logistic_from_word(wk)) * inv_tau;
        x[i] = a >= 0.0f ? 1 : 0;
        conf[i] = 1.0f / (1.0f + __expf(-fabsf(a)));     // max(y0, y1)
    }
}

// One CTA per candidate: the S most confident variables as unit literals, descending
// confidence, ties to the lower index.
__global__ void __launch_bounds__(kSelThreads) k_topk(const uint8_t *__restrict__ x, const float *__restrict__ conf,
                                                      int32_t n, int32_t n_sel, int32_t S,
                                                      int32_t *__restrict__ units, uint64_t *__restrict__ gkeys,
                                                      int32_t gstride)
{
    // rows of n variables; the units come from the first n_sel (the original variables of
    // a normalised CNF: P:214 excludes the auxiliaries). |S| > kMaxSorted: the block sorts
    // in its row of the global scratch gkeys (gstride keys, a power of two >= S)
    __shared__ uint64_t s_keys[kMaxSorted];
    const int32_t k = blockIdx.x;
    const float *c = conf + (size_t)k * n;
    auto key_of = [&](int32_t v) -> uint64_t {
        return ((uint64_t)__float_as_uint(c[v]) << 32) | (uint64_t)(0xFFFFFFFFu - (uint32_t)v);
    };
    GALOIS_DEV_CHECK(S <= kMaxSorted || (gkeys != nullptr && gstride >= S));
    uint64_t *keys = S <= kMaxSorted ? s_keys : gkeys + (size_t)k * gstride;
    const uint64_t thr = select_threshold(n_sel, S, key_of);
    collect_sorted_desc(n_sel, S, thr, key_of, keys);
    for (int32_t j = threadIdx.x; j < S; j += blockDim.x) {
        const int32_t v = (int32_t)(0xFFFFFFFFu - (uint32_t)(keys[j] & 0xFFFFFFFFull));
        units[(size_t)k * S + j] = x[(size_t)k * n + v] ? v + 1 : -(v + 1);
    }
}

// The d least confident variables of z (smallest |z|, ties to the lower index), ascending.
__global__ void __launch_bounds__(kSelThreads) k_lowconf(const float *__restrict__ zsel, int32_t n, int32_t d,
                                                         int32_t *__restrict__ vars)
{
    __shared__ uint64_t s_keys[kMaxSorted];
    // largest of the complemented keys == smallest (|z|, v)
    auto key_of = [&](int32_t v) -> uint64_t {
        return ~(((uint64_t)__float_as_uint(fabsf(zsel[v])) << 32) | (uint64_t)(uint32_t)v);
    };
    const uint64_t thr = select_threshold(n, d, key_of);
    // collect as variable-index keys, sorted descending, then emitted ascending
    auto vkey = [&](int32_t v) -> uint64_t { return key_of(v) >= thr ? (uint64_t)(uint32_t)v + 1 : 0; };
    collect_sorted_desc(n, d, 1, vkey, s_keys);
    for (int32_t j = threadIdx.x; j < d; j += blockDim.x) vars[j] = (int32_t)s_keys[d - 1 - j];   // 1-based
}

namespace launch {

void select_member(const int32_t *counts, int32_t b_loc, int64_t b0, int32_t rule, unsigned long long *out,
                   cudaStream_t st)
{
    k_select<<<1, kSelThreads, 0, st>>>(counts, b_loc, b0, rule, out);
}

void gather_z(const float *z, int32_t n, int32_t b_pad, int32_t lb, float *out, cudaStream_t st)
{
    k_gather_z<<<(n + 255) / 256 < 4096 ? (n + 255) / 256 : 4096, 256, 0, st>>>(z, n, b_pad, lb, out);
}

void pool(const float *zsel, int32_t n, int32_t k0, int32_t N, float inv_tau, uint64_t pool_seed, uint8_t *x,
          float *conf, cudaStream_t st)
{
    const int64_t total = (int64_t)N * n;
    int64_t g = (total + 255) / 256;
    if (g > 148 * 16) g = 148 * 16;
    k_pool<<<(unsigned)(g < 1 ? 1 : g), 256, 0, st>>>(zsel, n, k0, N, inv_tau, philox_round_keys(pool_seed), x,
                                                       conf);
}

void topk(const uint8_t *x, const float *conf, int32_t n, int32_t n_sel, int32_t N, int32_t S, int32_t *units,
          uint64_t *gkeys, int32_t gstride, cudaStream_t st)
{
    k_topk<<<N, kSelThreads, 0, st>>>(x, conf, n, n_sel, S, units, gkeys, gstride);
}

void lowconf(const float *zsel, int32_t n, int32_t d, int32_t *vars, cudaStream_t st)
{
    k_lowconf<<<1, kSelThreads, 0, st>>>(zsel, n, d, vars);
}

int max_sorted() { return kMaxSorted; }

}  // namespace launch
}  // namespace galois
