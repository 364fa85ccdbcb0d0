// galois_internal.h — device data layout shared by the CUDA sources of libgalois.
//
// HBM layout. n variables, m clauses, L literal slots, a rank's
// b_pad members (b_loc valid, padded to a multiple of 32), W = b_pad / 32 words:
//   CSR  clause_off[m+1] int32, slot_info[L] int2 = {lit code (v<<1)|neg, CSC position}
//   CSC  code_off[2n+1] int32: occurrences of literal code c are CSC positions
//        [code_off[c], code_off[c+1]), ascending slot order (stable counting sort)
//   state z, m, v float [n][b_pad]  (reduced iterate z = theta_1 - theta_0)
//   bits  X, R interleaved in one array: row v = 2 WP words (WP = W rounded up to 4),
//         16-byte groups alternating X words 4g..4g+3 and R words 4g..4g+3, R = X + 4 words
//         (xr_at); a sweep lane's X and R vectors of a literal are one 32-byte sector.
//         W < 4 (windows of 32-96 members): compact rows of 2W words, the W X words then
//         the W R words, R = X + W words — four variables' rows per sector at W = 1.
//         Word w holds members 32w..32w+31; member 32w + i at bit 8 (i mod 4) + i / 4
//         (device_utils.cuh bitpos)
//   E     uint32 [L][W] in CSC order (exclusive products of each occurrence); the row of a
//         NEGATIVE occurrence is stored complemented, so the signed signal of a variable is
//         (sum of all its row bits) - (number of its negative rows) — one count pass
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "philox.cuh"

namespace galois {

constexpr int kHubDegree = 256;      // variables with more occurrences use the hub path
constexpr int kSweepOffPad = 128;    // sweep_off entries past m (all = L): whole-tile copies

// word w of row v of the interleaved X/R array (apply to X for X words, to R = X + xr_roff(W)
// for R)
__host__ __device__ __forceinline__ int32_t xr_pad(int32_t W) { return W < 4 ? W : (W + 3) & ~3; }
__host__ __device__ __forceinline__ int32_t xr_roff(int32_t W) { return W < 4 ? W : 4; }
// (one formula for both layouts: below W = 4 the word index w < 4 adds just w)
__host__ __device__ __forceinline__ size_t xr_at(int32_t v, int32_t w, int32_t W)
{
    return (size_t)v * 2 * (size_t)xr_pad(W) + ((size_t)(w >> 2) << 3) + (size_t)(w & 3);
}
#ifndef GALOIS_HUB_CHUNK
#define GALOIS_HUB_CHUNK 256
#endif
constexpr int kHubChunk = GALOIS_HUB_CHUNK;   // occurrences per hub partial item (|partial| <= 256: int16)

// Device-side control block (one per engine, device memory).
struct Ctrl {
    int32_t t;            // steps done (incremented by the last CTA of each update kernel)
    int32_t stopped;      // 1 once the best member satisfies the CNF
    int32_t best_u;       // best unsat count so far (INT32_MAX = none)
    int32_t best_t;       // step of the best
    int64_t best_b;       // global member index of the best
    int32_t improved;     // last finalize improved the best AND this rank owns it
    int32_t nonfinite;    // sticky: an iterate became NaN/Inf
    unsigned long long key_local;   // (u << 32) | global b, min over local members
    unsigned long long key_global;  // same, min over ranks (NCCL MIN)
    int32_t last_check_t; // step of the last check
    uint32_t done_ctas;   // CTAs of the running update kernel that finished (last one ticks t)
    // NCCL (world > 1): the best record over ALL ranks, kept by k_gfinalize on the engine's
    // exchange stream from the MIN all-reduced key of every check; best_* above is then this
    // rank's own record (whose rounding bits best_bits hold)
    int32_t g_u;
    int32_t g_t;
    int64_t g_b;
};

struct DevCnf {
    int32_t n;
    int32_t m;
    int32_t L;
    const int32_t *clause_off;   // [m+1]
    const int32_t *clause_perm;  // [m] clauses in stable width order (warp-uniform widths)
    const int32_t *sweep_off;    // [m+1+kSweepOffPad] CSR offsets in clause_perm order (tail = L)
    const int2 *sweep_slot;      // [L+2] slot_info in clause_perm order (sweep c = clause_perm[c])
    const int2 *slot_info;       // [L] {code, csc position}
    const int32_t *code_off;     // [2n+1]
    const int32_t *occ_slot;     // [L]
    // hub path
    int32_t num_hubs;
    int32_t num_hub_chunks;
    const int32_t *hub_of_var;   // [n] hub index or -1
    const int32_t *hub_chunk_off;// [num_hubs+1] first chunk of each hub
    const int2 *hub_chunk;       // [num_hub_chunks] {var, first CSC position}
};

// Work layout of the per-variable kernels: one thread per QUAD (4 members) of a row; a
// 256-thread CTA covers one 256-quad chunk of a row (QW >= 256) or R = 256 / QW whole
// rows (QW < 256). Item i = (row group i / cpr, chunk i % cpr). No per-quad division.
struct RowMap {
    uint32_t QW;        // quads per row = b_pad / 4 (a multiple of 8)
    uint32_t cpr;       // 256-quad chunks per row (1 when QW < 256)
    uint32_t R;         // rows per item (1 when QW >= 256)
    uint32_t rows;      // number of rows (variables, or hub chunks)
    uint32_t items;     // ceil(rows / R) * cpr
    uint32_t div_mul;   // fast division by cpr: q = (umulhi(x, mul) + x) >> shift
    uint32_t div_shift;
};

struct StepParams {
    int32_t n;
    int32_t b_pad;
    int32_t W;
    int32_t b_loc;
    int64_t b0;               // global index of local member 0
    uint64_t seed;
    float tau, inv_tau;
    float beta1, beta2, eps;
    float omb1, omb2;         // 1 - beta1, 1 - beta2 (rounded from fp64)
    int32_t optimizer;        // 0 Adam, 1 SGD
    float lr;
    const float2 *adam_consts;// [steps+2] {2 lr / (1 - beta1^t), 1 / sqrt(1 - beta2^t)}
    int32_t num_pins;
    const int8_t *pin_rank;   // [n] r or -1 (NULL if no pins)
    PhiloxKeys keys;          // round keys of the seed (philox.cuh)
    // counters the update kernel zeroes for the next clause sweep (b_pad ints each, may be
    // null); an update that returns early (engine stopped) leaves them untouched
    int32_t *clear_a;
    int32_t *clear_b;
};

// Scratch of one single-launch small-instance run (k_small_run): the earliest SAT step
// over the CTAs and the count of finished CTAs ({0x7f7f7f7f, 0}: set at prepare, reset by
// the last CTA of every run).
struct SmallScratch {
    int32_t tstar;
    uint32_t done;
    uint32_t arrive;        // grid-barrier arrivals of the cooperative launch (0 between runs)
    uint32_t pad;
};
constexpr size_t kSmallRecBytes = 16;   // per-CTA record {u, t, b}

// Best tracking done by the last CTA of a checking clause sweep.
struct BestArgs {
    int32_t *unsat_last;   // copy of the counts of this check
    int32_t b_loc;
    int64_t b0;
    int32_t finalize;      // 1: single rank — update the best record and stop flag in-kernel
    uint8_t *best_bits;    // with finalize and extract_n = n: copy the winner's rounding bits
    int32_t extract_n;     //   in the same CTA (small n); 0: the engine launches k_extract
    int32_t W;
};

// Zero the next sweep's counters (grid-stride over the CTAs of an update kernel).
__device__ __forceinline__ void clear_counters(const StepParams &p)
{
    const int32_t stride = gridDim.x * blockDim.x;
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < p.b_pad; i += stride) {
        if (p.clear_a) p.clear_a[i] = 0;
        if (p.clear_b) p.clear_b[i] = 0;
    }
}

// kernels (launch wrappers in kernels.cu)
cudaError_t launch_build_cnf(int32_t n, int64_t m, int64_t L, const int64_t *d_offsets64,
                             const int32_t *d_lits, int32_t *d_clause_off, int2 *d_slot_info,
                             int32_t *d_code_off, int32_t *d_occ_slot, int32_t *d_err,
                             int32_t *d_max_width, int32_t *d_clause_perm, void *d_scratch,
                             size_t scratch_bytes, cudaStream_t st);
size_t build_cnf_scratch_bytes(int32_t n, int64_t L);
// sweep order: sweep_off = scan of the widths in clause_perm order, sweep_slot = slot_info
// regrouped so that the clauses of one sweep are contiguous (scratch: device_scan_scratch_elems(m+1))
cudaError_t launch_sweep_order(int64_t m, const int32_t *d_clause_off, const int32_t *d_clause_perm,
                               const int2 *d_slot_info, int32_t *d_sweep_off, int2 *d_sweep_slot, int32_t *d_scratch,
                               cudaStream_t st);
// out[i] = sum_{j < i} in[j] (int32, in-place allowed); scratch of device_scan_scratch_elems(N)
void device_exclusive_scan(const int32_t *in, int32_t *out, int64_t N, int32_t *scratch, cudaStream_t st);
size_t device_scan_scratch_elems(int64_t N);

}  // namespace galois
