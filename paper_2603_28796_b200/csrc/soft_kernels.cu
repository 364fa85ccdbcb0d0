// soft_kernels.cu — SOFT mode of rows a5-a7 (the fully relaxed polynomial;
// the debug mode the survey uses for finite-difference checks).
//
// Literal values are the fp32 probabilities p = sigma((z + ell)/tau) instead of the hard
// bits, so E and G are fp32 and every reduction runs in a FIXED order (deterministic,
// no atomics): clauses in order within a chunk, chunks in order; occurrences of a
// variable in CSC order (positive codes then negative, each in ascending slot order).
// One thread per member: lanes of a warp touch 32 consecutive members of one row.
#include <cuda_runtime.h>

#include <cstdint>

#include "device_utils.cuh"
#include "galois_internal.h"
#include "philox.cuh"

namespace galois {

namespace {
constexpr int kSoftChunks = 64;   // clause chunks of the soft forward (partial Lambda rows)

__device__ __forceinline__ int soft_pinned_bit(const StepParams &p, int32_t v, int64_t b_global)
{
    if (p.pin_rank == nullptr) return -1;
    const int r = p.pin_rank[v];
    return r < 0 ? -1 : (int)((b_global >> r) & 1);
}
}  // namespace

// P[v][b] = sigma((z + ell_s)/tau) for the step s = t + 1 (increments t).
__global__ void __launch_bounds__(256) k_soft_sample(StepParams p, const float *__restrict__ z,
                                                     float *__restrict__ P, Ctrl *__restrict__ ctrl)
{
    if (ctrl->stopped) return;
    const int32_t s = ctrl->t + 1;
    const uint64_t total = (uint64_t)p.n * p.b_pad;
    const uint2 key = make_uint2((uint32_t)p.seed, (uint32_t)(p.seed >> 32));
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const int32_t v = (int32_t)(i / (uint32_t)p.b_pad);
        const int32_t b = (int32_t)(i - (uint64_t)v * p.b_pad);
        const int64_t bg = p.b0 + b;
        const uint4 w = philox4x32_10(make_uint4((uint32_t)v, (uint32_t)(bg >> 2), (uint32_t)s, 1u), key);
        const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
        const int pb = soft_pinned_bit(p, v, bg);
        const float a = (z[i] + logistic_from_word(ws[bg & 3])) * p.inv_tau;
        P[i] = pb >= 0 ? (float)pb : 1.0f / (1.0f + __expf(-a));
    }
}


// Clause chunk blockIdx.y, member b: E (prefix then suffix products, as Eq.2 in slot
// order) written to Es[csc position][b]; partial Lambda of the chunk to lam_part.
__global__ void __launch_bounds__(256) k_soft_clauses(DevCnf c, int32_t b_pad, const float *__restrict__ P,
                                                      float *__restrict__ Es, float *__restrict__ lam_part,
                                                      const Ctrl *__restrict__ ctrl)
{
    if (ctrl->stopped) return;
    const int32_t b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= b_pad) return;
    const int64_t per = ((int64_t)c.m + gridDim.y - 1) / gridDim.y;
    const int64_t c0 = per * blockIdx.y, c1 = min((int64_t)c.m, c0 + per);
    float lam = 0.0f;
    for (int64_t cl = c0; cl < c1; ++cl) {
        const int32_t lo = c.clause_off[cl], hi = c.clause_off[cl + 1];
        float prefix = 1.0f;
        for (int32_t k = lo; k < hi; ++k) {
            const int2 si = c.slot_info[k];
            const float pv = P[(size_t)(si.x >> 1) * b_pad + b];
            const float s = (si.x & 1) ? 1.0f - pv : pv;
            Es[(size_t)si.y * b_pad + b] = prefix;
            prefix *= (1.0f - s);
        }
        lam += prefix;                                   // U_c
        float suffix = 1.0f;
        for (int32_t k = hi - 1; k >= lo; --k) {
            const int2 si = c.slot_info[k];
            const float pv = P[(size_t)(si.x >> 1) * b_pad + b];
            const float s = (si.x & 1) ? 1.0f - pv : pv;
            Es[(size_t)si.y * b_pad + b] *= suffix;
            suffix *= (1.0f - s);
        }
    }
    lam_part[(size_t)blockIdx.y * b_pad + b] = lam;
}

__global__ void k_soft_lam(int32_t b_pad, int32_t chunks, const float *__restrict__ lam_part,
                           float *__restrict__ lam, const Ctrl *__restrict__ ctrl)
{
    if (ctrl->stopped) return;
    const int32_t b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= b_pad) return;
    float acc = 0.0f;
    for (int32_t ch = 0; ch < chunks; ++ch) acc += lam_part[(size_t)ch * b_pad + b];
    lam[b] = acc;
}

// Fused a6 + a7 in SOFT mode: G = sum sigma * E in CSC order, then the same update as ST.
__global__ void __launch_bounds__(256) k_update_soft(DevCnf c, StepParams p, float *__restrict__ z,
                                                     float *__restrict__ m, float *__restrict__ vv,
                                                     uint32_t *__restrict__ X, uint32_t *__restrict__ R,
                                                     const float *__restrict__ Es, Ctrl *__restrict__ ctrl,
                                                     float *__restrict__ dbg_G, float *__restrict__ dbg_g1)
{
    if (ctrl->stopped) return;
    const int32_t s = ctrl->t + 1;                   // this step's index (t -> t+1)
    const float2 ac = p.adam_consts[s];
    const int lane = threadIdx.x & 31;
    const uint64_t total = (uint64_t)p.n * p.b_pad;
    const uint2 key = make_uint2((uint32_t)p.seed, (uint32_t)(p.seed >> 32));
    bool bad = false;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const int32_t v = (int32_t)(i / (uint32_t)p.b_pad);
        const int32_t slot = (int32_t)(i - (uint64_t)v * p.b_pad);
        // lane l of a 32-member word handles the member stored at bit l (device_utils.cuh)
        const int32_t b = (slot & ~31) | member_of_bit(slot & 31);
        const size_t ii = (size_t)v * p.b_pad + b;
        const int64_t bg = p.b0 + b;
        const int32_t k0 = c.code_off[2 * v], k1 = c.code_off[2 * v + 1], k2 = c.code_off[2 * v + 2];
        float G = 0.0f;
        for (int32_t k = k0; k < k1; ++k) G += Es[(size_t)k * p.b_pad + b];
        for (int32_t k = k1; k < k2; ++k) G -= Es[(size_t)k * p.b_pad + b];
        const uint4 wn = philox4x32_10(make_uint4((uint32_t)v, (uint32_t)(bg >> 2), (uint32_t)s, 1u), key);
        const uint4 wx = philox4x32_10(make_uint4((uint32_t)v, (uint32_t)(bg >> 2), (uint32_t)(s + 1), 1u), key);
        const uint32_t wna[4] = {wn.x, wn.y, wn.z, wn.w}, wxa[4] = {wx.x, wx.y, wx.z, wx.w};
        const int pb = soft_pinned_bit(p, v, bg);
        float zz = z[ii], mm = m[ii], w2 = vv[ii], g1 = 0.0f;
        if (pb < 0) {
            const float a = (zz + logistic_from_word(wna[bg & 3])) * p.inv_tau;
            const float e = __expf(-fabsf(a));
            const float d = 1.0f + e;
            g1 = -G * __fdividef(e, d * d) * p.inv_tau;
            if (p.optimizer == 0) {
                mm = p.beta1 * mm + p.omb1 * g1;
                w2 = p.beta2 * w2 + p.omb2 * g1 * g1;
                zz = zz - ac.x * __fdividef(mm, sqrtf(w2) * ac.y + p.eps);   // ac.x = 2 lr / bc1
            } else {
                zz = zz - 2.0f * p.lr * g1;
            }
            bad |= !isfinite(zz);
            z[ii] = zz;
            m[ii] = mm;
            vv[ii] = w2;
        }
        if (dbg_G) {
            dbg_G[ii] = G;
            dbg_g1[ii] = g1;
        }
        const bool rb = pb >= 0 ? pb != 0 : zz >= 0.0f;
        const bool xb = pb >= 0 ? pb != 0 : zz + logistic_from_word(wxa[bg & 3]) >= 0.0f;
        // 32 consecutive members of one row form one word (b_pad is a multiple of 32)
        const uint32_t rw = __ballot_sync(0xffffffffu, rb), xw = __ballot_sync(0xffffffffu, xb);
        if (lane == 0) {
            R[xr_at(v, b >> 5, p.W)] = rw;
            X[xr_at(v, b >> 5, p.W)] = xw;
        }
    }
    if (bad) atomicOr(&ctrl->nonfinite, 1);
    last_cta_tick(ctrl);
}

namespace launch {

static unsigned cap_grid(uint64_t work, unsigned cap)
{
    uint64_t g = (work + 255) / 256;
    if (g < 1) g = 1;
    if (g > cap) g = cap;
    return (unsigned)g;
}

void forward_soft(const DevCnf &c, const StepParams &p, const float *z, float *P, float *Es, float *lam,
                  Ctrl *ctrl, cudaStream_t st)
{
    // lam holds b_pad floats followed by kSoftChunks * b_pad partials (allocated by the engine)
    float *lam_part = lam + p.b_pad;
    k_soft_sample<<<cap_grid((uint64_t)p.n * p.b_pad, 148 * 8), 256, 0, st>>>(p, z, P, ctrl);
    dim3 grid((unsigned)((p.b_pad + 255) / 256), kSoftChunks);
    k_soft_clauses<<<grid, 256, 0, st>>>(c, p.b_pad, P, Es, lam_part, ctrl);
    k_soft_lam<<<(unsigned)((p.b_pad + 255) / 256), 256, 0, st>>>(p.b_pad, kSoftChunks, lam_part, lam, ctrl);
}

void update_soft(const DevCnf &c, const StepParams &p, float *z, float *m, float *v, uint32_t *X, uint32_t *R,
                 const float *Es, Ctrl *ctrl, float *dbg_G, float *dbg_g1, cudaStream_t st)
{
    k_update_soft<<<cap_grid((uint64_t)p.n * p.b_pad, 148 * 8), 256, 0, st>>>(c, p, z, m, v, X, R, Es, ctrl, dbg_G,
                                                                               dbg_g1);
}

int soft_chunks() { return kSoftChunks; }

}  // namespace launch
}  // namespace galois
