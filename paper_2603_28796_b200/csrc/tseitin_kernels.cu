// tseitin_kernels.cu — NEXT row f2 of SURVEY §8(f): clause normalisation to a fixed width k
// (the paper's GPU preprocessing, §2.2 "Clause Normalization for Vectorization",
// Eq.6-9; k = 3 in the experiments, App. A).
//
// A clause (l_1 ... l_u) with u > k becomes the chain (Eq.7 for k = 3)
//     (l_1 .. l_{k-1} f_1) (-f_1 l_k .. l_{2k-4} f_2) ... (-f_{q-1} l_.. .. l_u [pad])
// with fresh auxiliaries f_j (equisatisfiable, Eq.9); a clause with u <= k is padded by
// duplicating its last literal (Appendix B: (-x1 x3) -> (-x1 x3 x3)). Auxiliary
// j of clause c is variable n + aux_off[c] + j (1-based), in clause order.
// Two passes: shape (output clauses q_c, auxiliaries a_c) + exclusive scans, then writes.
#include <cuda_runtime.h>

#include <cstdint>

#include "galois_internal.h"

namespace galois {

namespace {

__device__ __forceinline__ void chain_shape(int32_t u, int32_t k, int32_t &q, int32_t &a)
{
    if (u <= k) {
        q = 1;
        a = 0;
        return;
    }
    const int32_t rem = u - (k - 1);               // literals after the first clause
    const int32_t mid = rem <= k - 1 ? 0 : (rem - (k - 1) + (k - 3)) / (k - 2);   // ceil(.. / (k-2))
    q = 2 + mid;
    a = q - 1;
}

__device__ __forceinline__ int32_t lit_of(int2 si) { return (si.x & 1) ? -((si.x >> 1) + 1) : (si.x >> 1) + 1; }

__global__ void k_tseitin_shape(const int32_t *__restrict__ clause_off, int64_t m, int32_t k, int32_t *__restrict__ q,
                                int32_t *__restrict__ a)
{
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c <= m; c += (int64_t)gridDim.x * blockDim.x) {
        int32_t qc = 0, ac = 0;
        if (c < m) chain_shape(clause_off[c + 1] - clause_off[c], k, qc, ac);
        q[c] = qc;                                  // entry m is 0: the scans give the totals
        a[c] = ac;
    }
}

__global__ void k_tseitin_write(const int32_t *__restrict__ clause_off, const int2 *__restrict__ slot_info, int64_t m,
                                int32_t n, int32_t k, const int32_t *__restrict__ q_off,
                                const int32_t *__restrict__ a_off, int32_t *__restrict__ out)
{
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < m; c += (int64_t)gridDim.x * blockDim.x) {
        const int32_t lo = clause_off[c], u = clause_off[c + 1] - lo;
        int32_t *dst = out + (int64_t)q_off[c] * k;
        if (u <= k) {
            for (int32_t i = 0; i < k; ++i) dst[i] = lit_of(slot_info[lo + (i < u ? i : u - 1)]);
            continue;
        }
        int32_t qc, ac;
        chain_shape(u, k, qc, ac);
        const int32_t f0 = n + a_off[c];            // f_j = f0 + j
        int32_t pos = 0;                            // next original literal
        for (int32_t j = 0; j < qc; ++j) {
            int32_t *cl = dst + (int64_t)j * k;
            int32_t w = 0;
            if (j > 0) cl[w++] = -(f0 + j);         // -f_j continues the chain
            const int32_t take = (j == 0) ? k - 1 : (j == qc - 1 ? u - pos : k - 2);
            for (int32_t i = 0; i < take; ++i) cl[w++] = lit_of(slot_info[lo + pos + i]);
            pos += take;
            if (j < qc - 1) cl[w++] = f0 + j + 1;   // +f_{j+1}
            while (w < k) { cl[w] = cl[w - 1]; ++w; }   // last clause: duplicate to width k
        }
    }
}

__global__ void k_fixed_offsets(int64_t m2, int32_t k, int64_t *__restrict__ off)
{
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c <= m2; c += (int64_t)gridDim.x * blockDim.x)
        off[c] = c * k;
}

unsigned grid_of(int64_t work)
{
    int64_t g = (work + 255) / 256;
    if (g < 1) g = 1;
    if (g > 148 * 16) g = 148 * 16;
    return (unsigned)g;
}

}  // namespace

namespace launch {

// Normalise to width k: allocates *d_off_out [m2 + 1] (int64) and *d_lits_out [m2 * k].
cudaError_t tseitin(const int32_t *clause_off, const int2 *slot_info, int64_t m, int32_t n, int32_t k,
                    int64_t **d_off_out, int32_t **d_lits_out, int64_t *m_out, int32_t *aux_out, cudaStream_t st)
{
    *d_off_out = nullptr;
    *d_lits_out = nullptr;
    int32_t *q = nullptr, *a = nullptr, *scratch = nullptr;
    cudaError_t e = cudaMallocAsync((void **)&q, sizeof(int32_t) * (size_t)(m + 1), st);
    if (e == cudaSuccess) e = cudaMallocAsync((void **)&a, sizeof(int32_t) * (size_t)(m + 1), st);
    if (e == cudaSuccess)
        e = cudaMallocAsync((void **)&scratch, sizeof(int32_t) * device_scan_scratch_elems(m + 1), st);
    if (e != cudaSuccess) return e;
    k_tseitin_shape<<<grid_of(m + 1), 256, 0, st>>>(clause_off, m, k, q, a);
    device_exclusive_scan(q, q, m + 1, scratch, st);
    device_exclusive_scan(a, a, m + 1, scratch, st);
    int32_t tot[2] = {0, 0};
    e = cudaMemcpyAsync(&tot[0], q + m, 4, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(&tot[1], a + m, 4, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    const int64_t m2 = tot[0];
    if (e == cudaSuccess && m2 * (int64_t)k >= INT32_MAX) e = cudaErrorInvalidValue;
    if (e == cudaSuccess) e = cudaMallocAsync((void **)d_off_out, sizeof(int64_t) * (size_t)(m2 + 1), st);
    if (e == cudaSuccess) e = cudaMallocAsync((void **)d_lits_out, sizeof(int32_t) * (size_t)(m2 * k > 0 ? m2 * k : 1), st);
    if (e == cudaSuccess) {
        k_fixed_offsets<<<grid_of(m2 + 1), 256, 0, st>>>(m2, k, *d_off_out);
        if (m > 0) k_tseitin_write<<<grid_of(m), 256, 0, st>>>(clause_off, slot_info, m, n, k, q, a, *d_lits_out);
        e = cudaGetLastError();
    }
    cudaFreeAsync(q, st);
    cudaFreeAsync(a, st);
    cudaFreeAsync(scratch, st);
    *m_out = m2;
    *aux_out = tot[1];
    return e;
}

}  // namespace launch
}  // namespace galois
