// cnf_build.cu — rows a1 (CSR build + validation) and a2 (CSC transpose) of SURVEY §8.
//
// a1: validate the DIMACS CSR on the device (clauses of signed literals; empty
//     clause = trivially UNSAT) and encode every slot as code = (v << 1) | neg.
// a2: the variable-major transpose as a STABLE counting sort of the slots by code, i.e.
//     by (variable, sign, slot): an LSD radix sort with 8-bit digits, per-tile digit
//     histograms, a device exclusive scan, and a rank-preserving scatter that uses
//     __match_any_sync inside each warp. No float work; bit-exact and deterministic.
#include <cuda_runtime.h>

#include <cstdint>

#include "galois_internal.h"

namespace galois {

namespace {

constexpr int kThreads = 256;
constexpr int kItems = 16;                   // keys per thread per radix tile
constexpr int kTile = kThreads * kItems;     // 4096 keys per tile
constexpr int kScanBlock = 1024;             // elements per scan block (256 threads x 4)

enum : int32_t { kErrOffsets = 1, kErrVarRange = 2, kErrEmpty = 4 };

__global__ void k_validate_clauses(int64_t m, int64_t L, const int64_t *__restrict__ off64,
                                   int32_t *__restrict__ clause_off, int32_t *__restrict__ err,
                                   int32_t *__restrict__ max_width)
{
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c <= m;
         c += (int64_t)gridDim.x * blockDim.x) {
        const int64_t lo = off64[c];
        if (c == 0 && lo != 0) atomicOr(err, kErrOffsets);
        if (lo < 0 || lo > L) atomicOr(err, kErrOffsets);
        clause_off[c] = (int32_t)lo;
        if (c < m) {
            const int64_t hi = off64[c + 1];
            if (hi < lo) {
                atomicOr(err, kErrOffsets);
                atomicMin(err + 1, (int32_t)c);
            } else if (hi == lo) {
                atomicOr(err, kErrEmpty);
                atomicMin(err + 2, (int32_t)c);
            } else {
                atomicMax(max_width, (int32_t)(hi - lo));
            }
        }
    }
}

__global__ void k_encode_slots(int32_t n, int64_t L, const int32_t *__restrict__ lits,
                               uint32_t *__restrict__ keys, int32_t *__restrict__ vals,
                               int32_t *__restrict__ err)
{
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < L;
         s += (int64_t)gridDim.x * blockDim.x) {
        const int32_t lit = lits[s];
        const int64_t a = lit < 0 ? -(int64_t)lit : (int64_t)lit;
        if (lit == 0 || a > n) {
            atomicOr(err, kErrVarRange);
            atomicMin(err + 3, (int32_t)s);
            keys[s] = 0;
        } else {
            keys[s] = ((uint32_t)(a - 1) << 1) | (lit < 0 ? 1u : 0u);
        }
        vals[s] = (int32_t)s;
    }
}

// ---------------------------------------------------------------- exclusive scan (int32)
__global__ void k_scan_local(const int32_t *__restrict__ in, int32_t *__restrict__ out, int64_t N,
                             int32_t *__restrict__ block_sums)
{
    __shared__ int32_t s_warp[kThreads / 32];
    const int64_t base = (int64_t)blockIdx.x * kScanBlock + threadIdx.x * 4;
    int32_t v[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] = (base + i < N) ? in[base + i] : 0;
    int32_t local = v[0] + v[1] + v[2] + v[3];
    // inclusive warp scan of the per-thread totals
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int32_t incl = local;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int32_t y = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += y;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    int32_t warp_off = 0;
    for (int w = 0; w < warp; ++w) warp_off += s_warp[w];
    int32_t run = warp_off + incl - local;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        if (base + i < N) out[base + i] = run;
        run += v[i];
    }
    if (threadIdx.x == kThreads - 1 && block_sums) block_sums[blockIdx.x] = run;
}

__global__ void k_scan_add(int32_t *__restrict__ out, int64_t N, const int32_t *__restrict__ block_off)
{
    const int64_t base = (int64_t)blockIdx.x * kScanBlock + threadIdx.x * 4;
    const int32_t add = block_off[blockIdx.x];
#pragma unroll
    for (int i = 0; i < 4; ++i)
        if (base + i < N) out[base + i] += add;
}

size_t scan_scratch_elems(int64_t N)
{
    size_t total = 0;
    while (N > kScanBlock) {
        N = (N + kScanBlock - 1) / kScanBlock;
        total += (size_t)N * 2;
    }
    return total + 2;
}

// out[i] = sum_{j<i} in[i]; in and out may alias.
void exclusive_scan(const int32_t *in, int32_t *out, int64_t N, int32_t *scratch, cudaStream_t st)
{
    if (N <= 0) return;
    const int64_t blocks = (N + kScanBlock - 1) / kScanBlock;
    if (blocks == 1) {
        k_scan_local<<<1, kThreads, 0, st>>>(in, out, N, nullptr);
        return;
    }
    int32_t *sums = scratch;
    int32_t *sums_scanned = scratch + blocks;
    k_scan_local<<<(unsigned)blocks, kThreads, 0, st>>>(in, out, N, sums);
    exclusive_scan(sums, sums_scanned, blocks, scratch + 2 * blocks, st);
    k_scan_add<<<(unsigned)blocks, kThreads, 0, st>>>(out, N, sums_scanned);
}

// ------------------------------------------------------------------------ radix sort
__global__ void k_radix_hist(const uint32_t *__restrict__ keys, int64_t L, int shift, int64_t tiles,
                             int32_t *__restrict__ hist)
{
    __shared__ int32_t s_cnt[256];
    s_cnt[threadIdx.x] = 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * kTile;
#pragma unroll 4
    for (int i = 0; i < kItems; ++i) {
        const int64_t idx = base + (int64_t)i * kThreads + threadIdx.x;
        if (idx < L) atomicAdd(&s_cnt[(keys[idx] >> shift) & 255u], 1);
    }
    __syncthreads();
    hist[(int64_t)threadIdx.x * tiles + blockIdx.x] = s_cnt[threadIdx.x];
}

__global__ void k_radix_scatter(const uint32_t *__restrict__ keys_in, const int32_t *__restrict__ vals_in,
                                uint32_t *__restrict__ keys_out, int32_t *__restrict__ vals_out,
                                int64_t L, int shift, int64_t tiles, const int32_t *__restrict__ hist_off)
{
    __shared__ int32_t s_base[256];                  // global offset of each digit for this tile
    __shared__ int32_t s_wcnt[kThreads / 32][256];   // per-warp digit counts -> prefix
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    s_base[threadIdx.x] = hist_off[(int64_t)threadIdx.x * tiles + blockIdx.x];
    const int64_t base = (int64_t)blockIdx.x * kTile;
    const uint32_t lt_mask = (1u << lane) - 1u;
    for (int i = 0; i < kItems; ++i) {
        for (int w = 0; w < kThreads / 32; ++w) s_wcnt[w][threadIdx.x] = 0;
        __syncthreads();
        const int64_t idx = base + (int64_t)i * kThreads + threadIdx.x;
        const bool valid = idx < L;
        uint32_t key = 0;
        int32_t val = 0;
        int digit = 256 + lane;                      // unique sentinel for invalid lanes
        if (valid) {
            key = keys_in[idx];
            val = vals_in[idx];
            digit = (int)((key >> shift) & 255u);
        }
        const uint32_t peers = __match_any_sync(0xffffffffu, digit);
        const int rank = __popc(peers & lt_mask);
        if (valid && rank == 0) s_wcnt[warp][digit] = __popc(peers);
        __syncthreads();
        {   // per digit: exclusive prefix over warps, then advance the tile base
            const int d = threadIdx.x;
            int32_t run = 0;
            for (int w = 0; w < kThreads / 32; ++w) {
                const int32_t c = s_wcnt[w][d];
                s_wcnt[w][d] = run;
                run += c;
            }
            __syncthreads();
            if (valid) {
                const int32_t pos = s_base[digit] + s_wcnt[warp][digit] + rank;
                keys_out[pos] = key;
                vals_out[pos] = val;
            }
            __syncthreads();
            s_base[d] += run;
        }
        __syncthreads();
    }
}

__global__ void k_width_keys(int64_t m, const int32_t *__restrict__ clause_off, uint32_t *__restrict__ keys,
                             int32_t *__restrict__ vals)
{
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < m; c += (int64_t)gridDim.x * blockDim.x) {
        const int32_t w = clause_off[c + 1] - clause_off[c];
        keys[c] = (uint32_t)(w < 0 ? 0 : (w > 255 ? 255 : w));
        vals[c] = (int32_t)c;
    }
}

// Sweep-order key of a clause: width (8 bits) above its HIGHEST variable scaled to 24 bits
// (stable sort: clause order within a bucket). Consecutive clauses
// then share that variable's X/R row; on a Tseitin-normalised formula the highest variable
// of a chain clause is its auxiliary f_j (numbered in chain order), so the sweep
// walks each chain in order and clause j + 1 finds f_j's row just loaded (the lowest
// variable — an original one — scattered the chains: normalised C4 forward -36 % at 32
// members, -13 % at 256; neutral on C2 / C4).
__global__ void k_width_maxvar_keys(int64_t m, int32_t n, const int32_t *__restrict__ clause_off,
                                    const int32_t *__restrict__ lits, uint32_t *__restrict__ keys,
                                    int32_t *__restrict__ vals)
{
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < m; c += (int64_t)gridDim.x * blockDim.x) {
        const int32_t a = clause_off[c], b = clause_off[c + 1], w = b - a;
        int32_t mv = -1;
        for (int32_t k = a; k < b; ++k) mv = max(mv, abs(lits[k]) - 1);
        const uint32_t bucket = (uint32_t)(((uint64_t)(mv < 0 ? 0 : mv) << 24) / (uint64_t)(n > 0 ? n : 1));
        keys[c] = ((uint32_t)(w < 0 ? 0 : (w > 255 ? 255 : w)) << 24) | (bucket & 0xFFFFFFu);
        vals[c] = (int32_t)c;
    }
}

__global__ void k_code_hist(const uint32_t *__restrict__ keys, int64_t L, int32_t *__restrict__ cnt)
{
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < L;
         s += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(&cnt[keys[s]], 1);
}

__global__ void k_slot_info(const uint32_t *__restrict__ codes, const int32_t *__restrict__ occ_slot,
                            int64_t L, int2 *__restrict__ slot_info)
{
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < L;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int32_t s = occ_slot[k];
        slot_info[s] = make_int2((int32_t)codes[k], (int32_t)k);
    }
}

__global__ void k_sweep_widths(int64_t m, const int32_t *__restrict__ clause_off, const int32_t *__restrict__ perm,
                               int32_t *__restrict__ w)
{
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c <= m + kSweepOffPad;
         c += (int64_t)gridDim.x * blockDim.x) {
        int32_t x = 0;
        if (c < m) {
            const int32_t cl = perm[c];
            x = clause_off[cl + 1] - clause_off[cl];
        }
        w[c] = x;
    }
}

__global__ void k_sweep_slots(int64_t m, const int32_t *__restrict__ clause_off, const int32_t *__restrict__ perm,
                              const int2 *__restrict__ slot_info, const int32_t *__restrict__ sweep_off,
                              int2 *__restrict__ sweep_slot)
{
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < m; c += (int64_t)gridDim.x * blockDim.x) {
        const int32_t cl = perm[c];
        const int32_t lo = clause_off[cl], w = clause_off[cl + 1] - lo, dst = sweep_off[c];
        for (int32_t i = 0; i < w; ++i) sweep_slot[dst + i] = slot_info[lo + i];
    }
}

unsigned grid_for(int64_t work, int threads = kThreads)
{
    int64_t g = (work + threads - 1) / threads;
    if (g < 1) g = 1;
    if (g > 148 * 32) g = 148 * 32;
    return (unsigned)g;
}

}  // namespace

void device_exclusive_scan(const int32_t *in, int32_t *out, int64_t N, int32_t *scratch, cudaStream_t st)
{
    exclusive_scan(in, out, N, scratch, st);
}

size_t device_scan_scratch_elems(int64_t N) { return scan_scratch_elems(N); }

cudaError_t launch_sweep_order(int64_t m, const int32_t *d_clause_off, const int32_t *d_clause_perm,
                               const int2 *d_slot_info, int32_t *d_sweep_off, int2 *d_sweep_slot, int32_t *d_scratch,
                               cudaStream_t st)
{
    k_sweep_widths<<<grid_for(m + 1 + kSweepOffPad), kThreads, 0, st>>>(m, d_clause_off, d_clause_perm, d_sweep_off);
    exclusive_scan(d_sweep_off, d_sweep_off, m + 1 + kSweepOffPad, d_scratch, st);
    if (m > 0)
        k_sweep_slots<<<grid_for(m), kThreads, 0, st>>>(m, d_clause_off, d_clause_perm, d_slot_info, d_sweep_off,
                                                       d_sweep_slot);
    return cudaGetLastError();
}

size_t build_cnf_scratch_bytes(int32_t n, int64_t L)
{
    const int64_t tiles = (L + kTile - 1) / kTile;
    const int64_t hist = 256 * (tiles > 0 ? tiles : 1);
    const int64_t codes = 2 * (int64_t)n + 1;
    const int64_t scan_n = hist > codes ? hist : codes;
    size_t bytes = 0;
    bytes += (size_t)L * 4 * 3;            // keys a/b, vals b  (vals a = occ_slot output)
    bytes += (size_t)hist * 4;             // histogram / offsets
    bytes += scan_scratch_elems(scan_n) * 4;
    return bytes + 256;
}

#ifndef GALOIS_SWEEP_LOCALITY
#define GALOIS_SWEEP_LOCALITY 1
#endif
cudaError_t launch_build_cnf(int32_t n, int64_t m, int64_t L, const int64_t *d_off64,
                             const int32_t *d_lits, int32_t *d_clause_off, int2 *d_slot_info,
                             int32_t *d_code_off, int32_t *d_occ_slot, int32_t *d_err,
                             int32_t *d_max_width, int32_t *d_clause_perm, void *d_scratch,
                             size_t scratch_bytes, cudaStream_t st)
{
    (void)scratch_bytes;
    // scratch is sized by build_cnf_scratch_bytes(n, max(L, m)): with empty clauses m > L
    const int64_t NB = L > m ? L : m;
    const int64_t tiles = (L + kTile - 1) / kTile;
    const int64_t tiles_nb = (NB + kTile - 1) / kTile;
    char *p = (char *)d_scratch;
    uint32_t *keys_a = (uint32_t *)p; p += (size_t)NB * 4;
    uint32_t *keys_b = (uint32_t *)p; p += (size_t)NB * 4;
    int32_t *vals_b = (int32_t *)p;   p += (size_t)NB * 4;
    int32_t *hist = (int32_t *)p;     p += (size_t)256 * (tiles_nb > 0 ? tiles_nb : 1) * 4;
    int32_t *scan_scratch = (int32_t *)p;
    int32_t *vals_a = d_occ_slot;

    k_validate_clauses<<<grid_for(m + 1), kThreads, 0, st>>>(m, L, d_off64, d_clause_off, d_err, d_max_width);
    if (L > 0)
        k_encode_slots<<<grid_for(L), kThreads, 0, st>>>(n, L, d_lits, keys_a, vals_a, d_err);

    // LSD radix passes over the bits of the largest code 2n-1 (results land in *_a)
    int bits = 1;
    while (bits < 32 && ((uint64_t)1 << bits) < (uint64_t)(2 * (int64_t)n)) ++bits;
    const int passes = (bits + 7) / 8;
    uint32_t *kin = keys_a, *kout = keys_b;
    int32_t *vin = vals_a, *vout = vals_b;
    for (int ps = 0; ps < passes && L > 0; ++ps) {
        k_radix_hist<<<(unsigned)tiles, kThreads, 0, st>>>(kin, L, 8 * ps, tiles, hist);
        exclusive_scan(hist, hist, 256 * tiles, scan_scratch, st);
        k_radix_scatter<<<(unsigned)tiles, kThreads, 0, st>>>(kin, vin, kout, vout, L, 8 * ps, tiles, hist);
        uint32_t *tk = kin; kin = kout; kout = tk;
        int32_t *tv = vin; vin = vout; vout = tv;
    }
    if (vin != d_occ_slot && L > 0) {
        cudaMemcpyAsync(d_occ_slot, vin, (size_t)L * 4, cudaMemcpyDeviceToDevice, st);
    }
    // code_off = exclusive scan of the code histogram (2n + 1 entries)
    const int64_t ncodes = 2 * (int64_t)n;
    cudaMemsetAsync(d_code_off, 0, (size_t)(ncodes + 1) * 4, st);
    if (L > 0) k_code_hist<<<grid_for(L), kThreads, 0, st>>>(kin, L, d_code_off);
    exclusive_scan(d_code_off, d_code_off, ncodes + 1, scan_scratch, st);
    if (L > 0) k_slot_info<<<grid_for(L), kThreads, 0, st>>>(kin, d_occ_slot, L, d_slot_info);

    // clause processing order: stable sort of the clauses by width (one 8-bit radix pass;
    // widths >= 255 share the last bucket) so that the clauses a warp handles together
    // have similar widths — no divergence on mixed-width (industrial) CNFs
    if (m > 0 && GALOIS_SWEEP_LOCALITY) {
        // (width, highest variable): four stable 8-bit passes, LSD first
        const int64_t mt = (m + kTile - 1) / kTile;
        k_width_maxvar_keys<<<grid_for(m), kThreads, 0, st>>>(m, n, d_clause_off, d_lits, keys_a, vals_b);
        uint32_t *kin = keys_a, *kout = keys_b;
        int32_t *vin = vals_b, *vout = d_clause_perm;
        for (int ps = 0; ps < 4; ++ps) {
            k_radix_hist<<<(unsigned)mt, kThreads, 0, st>>>(kin, m, 8 * ps, mt, hist);
            exclusive_scan(hist, hist, 256 * mt, scan_scratch, st);
            k_radix_scatter<<<(unsigned)mt, kThreads, 0, st>>>(kin, vin, kout, vout, m, 8 * ps, mt, hist);
            uint32_t *tk = kin; kin = kout; kout = tk;
            int32_t *tv = vin; vin = vout; vout = tv;
        }
        if (vin != d_clause_perm) cudaMemcpyAsync(d_clause_perm, vin, (size_t)m * 4, cudaMemcpyDeviceToDevice, st);
    } else if (m > 0) {
        const int64_t mt = (m + kTile - 1) / kTile;
        k_width_keys<<<grid_for(m), kThreads, 0, st>>>(m, d_clause_off, keys_a, vals_b);
        k_radix_hist<<<(unsigned)mt, kThreads, 0, st>>>(keys_a, m, 0, mt, hist);
        exclusive_scan(hist, hist, 256 * mt, scan_scratch, st);
        k_radix_scatter<<<(unsigned)mt, kThreads, 0, st>>>(keys_a, vals_b, keys_b, d_clause_perm, m, 0, mt, hist);
    }
    return cudaGetLastError();
}

}  // namespace galois
