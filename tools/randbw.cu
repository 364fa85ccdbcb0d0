// randbw.cu — DRAM ceiling probe for the sweep's access pattern (not product code).
//
// The C4 sweep gathers random 256-B X/R rows (256 MB table) and writes random 128-B E rows
// (2 GB, CSC order). This probe times, on one B200, each pattern alone and mixed, with
// 8 lanes per row segment exactly as k_sweep issues them, to bound what the sweep can reach.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/randbw tools/randbw.cu && /tmp/randbw
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x)                                                                        \
    do {                                                                             \
        cudaError_t e = (x);                                                         \
        if (e != cudaSuccess) {                                                      \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
            return 1;                                                                \
        }                                                                            \
    } while (0)

__global__ void k_copy(const uint4 *__restrict__ a, uint4 *__restrict__ b, size_t n)
{
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        b[i] = a[i];
}

// mode bit 0: gather rows (256 B: 8 lanes x 32 B) of tab at idx_r; bit 1: scatter 128-B rows
// (8 lanes x 16 B) of out at idx_w. One "slot" per 8-lane group per iteration; `seq_w`
// writes sequential rows instead (the E-in-slot-order alternative).
__global__ void k_rand(const uint4 *__restrict__ tab, const int32_t *__restrict__ idx_r, uint4 *__restrict__ out,
                       const int32_t *__restrict__ idx_w, int64_t slots, int mode, int seq_w, uint32_t *sink)
{
    const int vl = threadIdx.x & 7;
    uint32_t acc = 0;
    for (int64_t s = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 3; s < slots;
         s += ((int64_t)gridDim.x * blockDim.x) >> 3) {
        uint4 x = make_uint4(0, 0, 0, 0), r = x;
        if (mode & 1) {
            const uint4 *p = tab + (size_t)__ldg(idx_r + s) * 16 + vl * 2;
            x = __ldg(p);
            r = __ldg(p + 1);
        }
        if (mode & 2) {
            const size_t row = seq_w ? (size_t)s : (size_t)__ldg(idx_w + s);
            uint4 *q = out + row * 8 + vl;
            *q = make_uint4(x.x ^ r.x ^ (uint32_t)s, x.y ^ r.y, x.z ^ r.z, x.w ^ r.w);
        } else {
            acc ^= x.x ^ r.y ^ x.z ^ r.w;
        }
    }
    if (acc == 0x12345678u) *sink = acc;
}

// random 128-B row reads (8 lanes x 16 B) of a 2 GB array, rows in idx order (the update's
// E reads if E were stored in sweep order); `unroll` rows in flight per lane group
template <int kUnroll>
__global__ void k_rread(const uint4 *__restrict__ src, const int32_t *__restrict__ idx, int64_t slots, uint32_t *sink)
{
    const int vl = threadIdx.x & 7;
    uint32_t acc = 0;
    const int64_t step = ((int64_t)gridDim.x * blockDim.x) >> 3;
    for (int64_t s = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 3; s < slots; s += step * kUnroll) {
        uint4 x[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const int64_t t = s + u * step;
            x[u] = t < slots ? __ldg(src + (size_t)__ldg(idx + t) * 8 + vl) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) acc ^= x[u].x ^ x[u].y ^ x[u].z ^ x[u].w;
    }
    if (acc == 0x12345678u) *sink = acc;
}

// L2-resident gathers: random 256-B rows (8 lanes x 32 B, one 256-bit load each) of a table
// of `rows` rows that fits L2 (C3b's X/R: 500 rows x 4 KB); `iters` gathers per lane group
__global__ void k_l2gather(const uint4 *__restrict__ tab, int64_t rows, int64_t iters, uint32_t *sink)
{
    const int vl = threadIdx.x & 7;
    const int64_t g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 3;
    uint32_t h = (uint32_t)g * 2654435761u + 12345u, acc = 0;
    for (int64_t i = 0; i < iters; i += 4) {
        uint4 x[4], r[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            h = h * 1664525u + 1013904223u;
            const uint4 *p = tab + (size_t)(h % (uint32_t)rows) * 16 + vl * 2;
            asm volatile("ld.global.nc.v8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                         : "=r"(x[u].x), "=r"(x[u].y), "=r"(x[u].z), "=r"(x[u].w), "=r"(r[u].x), "=r"(r[u].y),
                           "=r"(r[u].z), "=r"(r[u].w)
                         : "l"(p));
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) acc ^= x[u].x ^ r[u].w;
    }
    if (acc == 0x12345678u) *sink = acc;
}

int main()
{
    const int64_t rows_r = 1 << 20;                // 1M rows x 256 B = 256 MB (C4's X/R)
    const int64_t slots = 15548079;                // C4's L: 2 GB of 128-B E rows
    uint4 *tab, *out, *a, *b;
    int32_t *idx_r, *idx_w;
    uint32_t *sink;
    CK(cudaMalloc(&tab, rows_r * 256));
    CK(cudaMalloc(&out, slots * 128));
    CK(cudaMalloc(&idx_r, slots * 4));
    CK(cudaMalloc(&idx_w, slots * 4));
    CK(cudaMalloc(&sink, 4));
    CK(cudaMemset(tab, 1, rows_r * 256));
    std::vector<int32_t> h(slots);
    uint64_t st = 88172645463325252ull;
    auto rnd = [&]() { st ^= st << 13; st ^= st >> 7; st ^= st << 17; return st; };
    // gathers: power-law (C4: P(i) ~ i^-0.8, permuted ids) approximated by u^(1/0.2)
    for (int64_t i = 0; i < slots; ++i) {
        const double u = (double)(rnd() >> 11) * (1.0 / 9007199254740992.0);
        int64_t v = (int64_t)(rows_r * __builtin_pow(u, 5.0));
        h[i] = (int32_t)((v * 2654435761ull) % rows_r);   // scramble ids
    }
    CK(cudaMemcpy(idx_r, h.data(), slots * 4, cudaMemcpyHostToDevice));
    // scatter: a random permutation of the E rows (each written once)
    for (int64_t i = 0; i < slots; ++i) h[i] = (int32_t)i;
    for (int64_t i = slots - 1; i > 0; --i) {
        const int64_t j = (int64_t)(rnd() % (uint64_t)(i + 1));
        std::swap(h[i], h[j]);
    }
    CK(cudaMemcpy(idx_w, h.data(), slots * 4, cudaMemcpyHostToDevice));
    const size_t cn = (size_t)1 << 26;             // 1 GiB copy
    CK(cudaMalloc(&a, cn * 16));
    CK(cudaMalloc(&b, cn * 16));
    CK(cudaMemset(a, 2, cn * 16));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto timeit = [&](auto fn, int reps) {
        fn();
        cudaEventRecord(e0);
        for (int i = 0; i < reps; ++i) fn();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        return ms / reps;
    };
    float ms = timeit([&] { k_copy<<<148 * 8, 256>>>(a, b, cn); }, 10);
    printf("copy 1 GiB: %.3f ms  %.0f GB/s (read+write)\n", ms, 2.0 * cn * 16 / ms / 1e6);
    for (int blocks : {148 * 3, 148 * 6, 148 * 8}) {
        for (int mode = 1; mode <= 3; ++mode) {
            for (int seq = 0; seq < (mode & 2 ? 2 : 1); ++seq) {
                ms = timeit([&] { k_rand<<<blocks, 256>>>(tab, idx_r, out, idx_w, slots, mode, seq, sink); }, 5);
                const double bytes = (mode & 1 ? slots * 256.0 : 0) + (mode & 2 ? slots * 128.0 : 0) + slots * 4.0 * ((mode & 1) + (mode & 2 && !seq ? 1 : 0));
                printf("blocks %4d %s%s%s: %.3f ms  %.0f GB/s algorithmic\n", blocks, mode & 1 ? "gather256 " : "",
                       mode & 2 ? "scatter128" : "", mode & 2 ? (seq ? "(seq)" : "(rand)") : "", ms, bytes / ms / 1e6);
            }
        }
    }
    for (int blocks : {148 * 4, 148 * 8}) {
        ms = timeit([&] { k_rread<1><<<blocks, 256>>>(out, idx_w, slots, sink); }, 5);
        printf("blocks %4d rand-read128 x1: %.3f ms  %.0f GB/s\n", blocks, ms, slots * 132.0 / ms / 1e6);
        ms = timeit([&] { k_rread<4><<<blocks, 256>>>(out, idx_w, slots, sink); }, 5);
        printf("blocks %4d rand-read128 x4: %.3f ms  %.0f GB/s\n", blocks, ms, slots * 132.0 / ms / 1e6);
    }
    for (int64_t rows : {(int64_t)8192, (int64_t)131072}) {       // 2 MB (C3b X/R) and 32 MB tables
        for (int blocks : {148 * 4, 148 * 8}) {
            const int64_t iters = 4096;
            ms = timeit([&] { k_l2gather<<<blocks, 256>>>(tab, rows, iters, sink); }, 5);
            const double bytes = (double)blocks * 256 / 8 * iters * 256;
            printf("L2 gather256 table %5.1f MB blocks %4d: %.3f ms  %.0f GB/s\n", rows * 256 / 1e6, blocks, ms,
                   bytes / ms / 1e6);
        }
    }
    CK(cudaGetLastError());
    return 0;
}
