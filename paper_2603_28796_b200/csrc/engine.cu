// engine.cu — the C ABI (include/galois.h) and the engine orchestration.
//
// One engine = one rank's slice of the batch on one GPU. Step s enqueues, on the
// engine's stream:
//   clause sweep: forward of X_s (a5) [+ exact check of R_{s-1} if it is a check point (a8)]
//   [best | NCCL MIN (a9) | finalize | extract]   (when R_{s-1} was checked)
//   [hub partials (a6)] | fused update (a6+a7; its last CTA advances t)
// A check left pending at the end (t = T, or before any result is read) runs alone.
// Every kernel reads the device control block first and returns immediately once the
// best member satisfies the CNF, so the host only polls the control block per chunk.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/galois.h"
#include "comm.h"
#include "galois_internal.h"

namespace galois {
namespace launch {
void init(const StepParams &p, float *z, float *m, float *v, uint32_t *X, uint32_t *R, cudaStream_t st);
void resample(const StepParams &p, const float *z, uint32_t *X, uint32_t *R, int32_t t_next, cudaStream_t st);
bool clauses(const DevCnf &c, int32_t W, int32_t b_pad, const uint32_t *X, const uint32_t *R, uint32_t *E,
             int32_t *lam, int32_t *unsat, Ctrl *ctrl, const BestArgs &ba, cudaStream_t st);
void hub_partial(const DevCnf &c, int32_t W, int32_t b_pad, const uint32_t *E, short4 *partial,
                 const Ctrl *ctrl, cudaStream_t st);
size_t small_run_smem(int32_t n, int32_t L);
cudaError_t small_run(const DevCnf &c, const StepParams &p, int32_t T, int32_t K, bool pending, float *z, float *m,
                      float *v, uint32_t *X, uint32_t *R, int32_t *unsat_last, int32_t *lam, SmallScratch *gs,
                      void *recs, uint8_t *snap, uint8_t *best_bits, Ctrl *ctrl, cudaStream_t st);
void update_st(const DevCnf &c, const StepParams &p, float *z, float *m, float *v, uint32_t *X, uint32_t *R,
               const uint32_t *E, const short4 *partial, Ctrl *ctrl, int32_t *dbg_G, float *dbg_g1,
               cudaStream_t st);
void best(const int32_t *unsat, int32_t *unsat_last, int32_t b_loc, int64_t b0, Ctrl *ctrl, bool finalize,
          cudaStream_t st);
void gfinalize(Ctrl *ctrl, cudaStream_t st);
void extract(const uint32_t *R, int32_t n, int32_t W, int64_t b0, const Ctrl *ctrl, uint8_t *best_bits,
             cudaStream_t st);
void member_bits(const uint32_t *X, int32_t n, int32_t W, int32_t lb, uint8_t *x_out, uint8_t *r_out, cudaStream_t st);
// SOFT mode (soft_kernels.cu)
void forward_soft(const DevCnf &c, const StepParams &p, const float *z, float *P, float *Es, float *lam,
                  Ctrl *ctrl, cudaStream_t st);
void update_soft(const DevCnf &c, const StepParams &p, float *z, float *m, float *v, uint32_t *X, uint32_t *R,
                 const float *Es, Ctrl *ctrl, float *dbg_G, float *dbg_g1, cudaStream_t st);
int soft_chunks();
cudaError_t configure_kernels();
// selection (select_kernels.cu)
void select_member(const int32_t *counts, int32_t b_loc, int64_t b0, int32_t rule, unsigned long long *out,
                   cudaStream_t st);
void gather_z(const float *z, int32_t n, int32_t b_pad, int32_t lb, float *out, cudaStream_t st);
void pool(const float *zsel, int32_t n, int32_t k0, int32_t N, float inv_tau, uint64_t pool_seed, uint8_t *x,
          float *conf, cudaStream_t st);
void topk(const uint8_t *x, const float *conf, int32_t n, int32_t n_sel, int32_t N, int32_t S, int32_t *units,
          uint64_t *gkeys, int32_t gstride, cudaStream_t st);
void lowconf(const float *zsel, int32_t n, int32_t d, int32_t *vars, cudaStream_t st);
int max_sorted();
}  // namespace launch
}  // namespace galois

using namespace galois;

// ------------------------------------------------------------------------ errors
static thread_local std::string g_last_error;
constexpr size_t kSmallRunSmem = 200 * 1024;   // dynamic shared memory of one k_small_run CTA (max)

static int fail(int code, const std::string &msg)
{
    g_last_error = msg;
    return code;
}

#define CUDA_TRY(expr)                                                                         \
    do {                                                                                       \
        cudaError_t _e = (expr);                                                               \
        if (_e != cudaSuccess) {                                                               \
            return fail(_e == cudaErrorMemoryAllocation ? GALOIS_E_OOM : GALOIS_E_CUDA,        \
                        std::string(#expr) + ": " + cudaGetErrorString(_e));                   \
        }                                                                                      \
    } while (0)

static int check_device(int *dev)
{
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0)
        return fail(GALOIS_E_CUDA, std::string("no CUDA device: ") +
                                       (e != cudaSuccess ? cudaGetErrorString(e) : "device count is 0"));
    CUDA_TRY(cudaGetDevice(dev));
    return GALOIS_OK;
}

// ------------------------------------------------------------------------ CNF
struct galois_cnf {
    std::atomic<int> refs{1};
    int device = 0;
    int32_t n = 0;
    int32_t n_orig = 0;      // variables of the CNF before normalisation (= n unless normalised)
    int64_t m = 0;
    int64_t L = 0;
    int32_t max_width = 0;
    int32_t max_degree = 0;
    int32_t *clause_off = nullptr;
    int32_t *clause_perm = nullptr;
    int32_t *sweep_off = nullptr;
    int2 *slot_info = nullptr;
    int2 *sweep_slot = nullptr;
    int32_t *code_off = nullptr;
    int32_t *occ_slot = nullptr;
    int32_t *hub_of_var = nullptr;
    int32_t *hub_chunk_off = nullptr;
    int2 *hub_chunk = nullptr;
    int32_t num_hubs = 0;
    int32_t num_hub_chunks = 0;

    DevCnf view() const
    {
        DevCnf d;
        d.n = n;
        d.m = (int32_t)m;
        d.L = (int32_t)L;
        d.clause_off = clause_off;
        d.clause_perm = clause_perm;
        d.sweep_off = sweep_off;
        d.sweep_slot = sweep_slot;
        d.slot_info = slot_info;
        d.code_off = code_off;
        d.occ_slot = occ_slot;
        d.num_hubs = num_hubs;
        d.num_hub_chunks = num_hub_chunks;
        d.hub_of_var = hub_of_var;
        d.hub_chunk_off = hub_chunk_off;
        d.hub_chunk = hub_chunk;
        return d;
    }
    ~galois_cnf()
    {
        int cur = 0;
        cudaGetDevice(&cur);
        cudaSetDevice(device);
        cudaFreeAsync(clause_off, 0);
        cudaFreeAsync(clause_perm, 0);
        cudaFreeAsync(sweep_off, 0);
        cudaFreeAsync(sweep_slot, 0);
        cudaFreeAsync(slot_info, 0);
        cudaFreeAsync(code_off, 0);
        cudaFreeAsync(occ_slot, 0);
        cudaFreeAsync(hub_of_var, 0);
        cudaFreeAsync(hub_chunk_off, 0);
        cudaFreeAsync(hub_chunk, 0);
        cudaSetDevice(cur);
    }
};

static void cnf_release(galois_cnf *c)
{
    if (c && c->refs.fetch_sub(1) == 1) delete c;
}

// Sub-allocation plan of one contiguous device block (256-B aligned pieces).
struct Slab {
    std::vector<std::pair<void **, size_t>> items;
    template <typename T>
    void add(T **p, size_t count)
    {
        items.push_back({reinterpret_cast<void **>(p), (count ? count : 1) * sizeof(T)});
    }
    static size_t up(size_t x) { return (x + 255) / 256 * 256; }
    size_t total() const
    {
        size_t t = 0;
        for (const auto &it : items) t += up(it.second);
        return t;
    }
    void assign(void *base) const
    {
        char *p = static_cast<char *>(base);
        for (const auto &it : items) {
            *it.first = p;
            p += up(it.second);
        }
    }
};

// Pinned host mirrors of the control block (2 slots per engine) come from one process-wide
// pinned page: page-locking memory costs ~ms, an engine should not pay it.

// Non-blocking streams are reused across engines and CNF loads (creating one costs ~50 us,
// as much as the rest of an engine's preparation): released streams are synchronised and
// parked per device, up to 64.
static std::mutex g_stream_mu;
static std::vector<std::pair<int, cudaStream_t>> g_stream_pool;

static cudaError_t stream_acquire(cudaStream_t *out)
{
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    {
        std::lock_guard<std::mutex> lock(g_stream_mu);
        for (size_t i = 0; i < g_stream_pool.size(); ++i)
            if (g_stream_pool[i].first == dev) {
                *out = g_stream_pool[i].second;
                g_stream_pool.erase(g_stream_pool.begin() + (std::ptrdiff_t)i);
                return cudaSuccess;
            }
    }
    return cudaStreamCreateWithFlags(out, cudaStreamNonBlocking);
}

static void stream_release(cudaStream_t s)
{
    if (!s) return;
    int dev = 0;
    if (cudaStreamSynchronize(s) != cudaSuccess || cudaGetDevice(&dev) != cudaSuccess) {
        cudaGetLastError();
        cudaStreamDestroy(s);
        return;
    }
    std::lock_guard<std::mutex> lock(g_stream_mu);
    if (g_stream_pool.size() < 64)
        g_stream_pool.emplace_back(dev, s);
    else
        cudaStreamDestroy(s);
}

static std::mutex g_pin_mu;
static Ctrl *g_pin_base = nullptr;
static std::vector<int> g_pin_free;
constexpr int kPinSlots = 256;

static cudaError_t pinned_ctrl_acquire(Ctrl **out)
{
    std::lock_guard<std::mutex> lock(g_pin_mu);
    if (!g_pin_base) {
        cudaError_t e = cudaMallocHost((void **)&g_pin_base, sizeof(Ctrl) * 2 * kPinSlots);
        if (e != cudaSuccess) return e;
        for (int i = kPinSlots - 1; i >= 0; --i) g_pin_free.push_back(i);
    }
    if (g_pin_free.empty()) return cudaMallocHost((void **)out, 2 * sizeof(Ctrl));   // overflow: own block
    *out = g_pin_base + 2 * g_pin_free.back();
    g_pin_free.pop_back();
    return cudaSuccess;
}

static void pinned_ctrl_release(Ctrl *p)
{
    std::lock_guard<std::mutex> lock(g_pin_mu);
    if (g_pin_base && p >= g_pin_base && p < g_pin_base + 2 * kPinSlots)
        g_pin_free.push_back((int)((p - g_pin_base) / 2));
    else
        cudaFreeHost(p);
}

// Keep freed blocks in the device's default memory pool (no release to the OS between
// engines), so repeated create/free is a pool hit.
static cudaError_t use_pool_for_device(int device)
{
    static std::atomic<uint64_t> done{0};
    if (device < 64 && (done.load() >> device) & 1ull) return cudaSuccess;
    cudaMemPool_t pool;
    cudaError_t e = cudaDeviceGetDefaultMemPool(&pool, device);
    if (e != cudaSuccess) return e;
    uint64_t threshold = UINT64_MAX;
    e = cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold);
    if (e == cudaSuccess && device < 64) done.fetch_or(1ull << device);
    return e;
}

// CNF buffers come from the device's stream-ordered pool (cudaMallocAsync on the build
// stream; freed with cudaFreeAsync): repeated load / normalise / free is a pool hit instead
// of a driver allocation with an implicit device synchronisation.
template <typename T>
static cudaError_t dmalloc(T **p, size_t count, cudaStream_t st)
{
    *p = nullptr;
    if (count == 0) count = 1;
    return cudaMallocAsync((void **)p, count * sizeof(T), st);
}

// Build a device CNF from device-resident DIMACS CSR arrays (d_off64 [m+1], d_lits [L]),
// which this function takes over (frees): validation (a1), literal codes, CSC (a2),
// width order, hub table. Work is ordered on the caller's stream st.
static int cnf_build_device(int dev, int32_t num_vars, int64_t num_clauses, int64_t L, int64_t *d_off64,
                            int32_t *d_lits, cudaStream_t st, galois_cnf **out)
{
    galois_cnf *c = new galois_cnf();
    c->device = dev;
    c->n = num_vars;
    c->n_orig = num_vars;
    c->m = num_clauses;
    c->L = L;
    const int64_t m = num_clauses;
    int32_t *d_err = nullptr;
    void *d_scratch = nullptr;
    auto cleanup = [&]() {
        cudaFreeAsync(d_off64, st);
        cudaFreeAsync(d_lits, st);
        cudaFreeAsync(d_err, st);
        cudaFreeAsync(d_scratch, st);
        cudaStreamSynchronize(st);
    };
    auto bail = [&](int code, const std::string &msg) {
        cleanup();
        cnf_release(c);
        return fail(code, msg);
    };
#define LOAD_TRY(expr)                                                                                   \
    do {                                                                                                 \
        cudaError_t _e = (expr);                                                                         \
        if (_e != cudaSuccess)                                                                           \
            return bail(_e == cudaErrorMemoryAllocation ? GALOIS_E_OOM : GALOIS_E_CUDA,                  \
                        std::string(#expr) + ": " + cudaGetErrorString(_e));                             \
    } while (0)

    LOAD_TRY(dmalloc(&d_err, 8, st));
    LOAD_TRY(dmalloc(&c->clause_off, (size_t)m + 1, st));
    LOAD_TRY(dmalloc(&c->clause_perm, (size_t)m, st));
    LOAD_TRY(dmalloc(&c->slot_info, (size_t)L, st));
    LOAD_TRY(dmalloc(&c->code_off, 2 * (size_t)num_vars + 1, st));
    LOAD_TRY(dmalloc(&c->occ_slot, (size_t)L, st));
    const size_t scratch = build_cnf_scratch_bytes(num_vars, std::max<int64_t>(L, m));
    LOAD_TRY(cudaMallocAsync(&d_scratch, scratch, st));
    const int32_t h_err_init[8] = {0, INT32_MAX, INT32_MAX, INT32_MAX, 0, 0, 0, 0};
    LOAD_TRY(cudaMemcpyAsync(d_err, h_err_init, sizeof(h_err_init), cudaMemcpyHostToDevice, st));
    LOAD_TRY(launch_build_cnf(num_vars, m, L, d_off64, d_lits, c->clause_off, c->slot_info, c->code_off,
                              c->occ_slot, d_err, d_err + 4, c->clause_perm, d_scratch, scratch, st));
    int32_t h_err[8];
    LOAD_TRY(cudaMemcpyAsync(h_err, d_err, sizeof(h_err), cudaMemcpyDeviceToHost, st));
    LOAD_TRY(cudaStreamSynchronize(st));
    if (h_err[0] & 1) {
        char buf[160];
        snprintf(buf, sizeof buf, "clause offsets are not a valid CSR (first bad clause %d)", h_err[1]);
        return bail(GALOIS_E_OFFSETS, buf);
    }
    if (h_err[0] & 4) {
        char buf[160];
        snprintf(buf, sizeof buf, "clause %d is empty: the CNF is trivially UNSAT", h_err[2]);
        return bail(GALOIS_E_EMPTY_CLAUSE, buf);
    }
    if (h_err[0] & 2) {
        char buf[160];
        snprintf(buf, sizeof buf, "literal at slot %d is 0 or exceeds num_vars=%d", h_err[3], num_vars);
        return bail(GALOIS_E_VAR_RANGE, buf);
    }
    c->max_width = h_err[4];
    // padded for the staged sweep's tile copies (k_sweep_tma): offsets past m hold L, and a
    // 16-B aligned slot copy may read one int2 past L
    LOAD_TRY(dmalloc(&c->sweep_off, (size_t)m + 1 + kSweepOffPad, st));
    LOAD_TRY(dmalloc(&c->sweep_slot, (size_t)L + 2, st));
    LOAD_TRY(launch_sweep_order(m, c->clause_off, c->clause_perm, c->slot_info, c->sweep_off, c->sweep_slot,
                                (int32_t *)d_scratch, st));

    // hub table: variables with more than kHubDegree occurrences are reduced in chunks
    std::vector<int32_t> code_off(2 * (size_t)num_vars + 1);
    LOAD_TRY(cudaMemcpyAsync(code_off.data(), c->code_off, code_off.size() * 4, cudaMemcpyDeviceToHost, st));
    LOAD_TRY(cudaStreamSynchronize(st));
    std::vector<int32_t> hub_of_var(num_vars, -1), hub_chunk_off(1, 0);
    std::vector<int2> hub_chunk;
    for (int32_t v = 0; v < num_vars; ++v) {
        const int32_t a = code_off[2 * (size_t)v], e = code_off[2 * (size_t)v + 2];
        const int32_t deg = e - a;
        c->max_degree = std::max(c->max_degree, deg);
        if (deg > kHubDegree) {
            hub_of_var[v] = c->num_hubs++;
            for (int32_t k = a; k < e; k += kHubChunk) hub_chunk.push_back(make_int2(v, k));
            hub_chunk_off.push_back((int32_t)hub_chunk.size());
        }
    }
    c->num_hub_chunks = (int32_t)hub_chunk.size();
    if (c->num_hubs > 0) {
        LOAD_TRY(dmalloc(&c->hub_of_var, (size_t)num_vars, st));
        LOAD_TRY(dmalloc(&c->hub_chunk_off, hub_chunk_off.size(), st));
        LOAD_TRY(dmalloc(&c->hub_chunk, hub_chunk.size(), st));
        LOAD_TRY(cudaMemcpyAsync(c->hub_of_var, hub_of_var.data(), hub_of_var.size() * 4, cudaMemcpyHostToDevice, st));
        LOAD_TRY(cudaMemcpyAsync(c->hub_chunk_off, hub_chunk_off.data(), hub_chunk_off.size() * 4,
                                 cudaMemcpyHostToDevice, st));
        LOAD_TRY(cudaMemcpyAsync(c->hub_chunk, hub_chunk.data(), hub_chunk.size() * sizeof(int2), cudaMemcpyHostToDevice,
                                 st));
        LOAD_TRY(cudaStreamSynchronize(st));   // the host vectors go out of scope
    }
#undef LOAD_TRY
    cleanup();
    *out = c;
    return GALOIS_OK;
}

extern "C" int galois_cnf_load(int32_t num_vars, int64_t num_clauses, const int64_t *clause_offsets,
                               const int32_t *literals, galois_cnf **out)
{
    if (!out) return fail(GALOIS_E_ARG, "out is NULL");
    *out = nullptr;
    if (num_vars < 1 || num_vars >= (1 << 30)) return fail(GALOIS_E_ARG, "num_vars must be in [1, 2^30)");
    if (num_clauses < 0 || num_clauses >= INT32_MAX) return fail(GALOIS_E_ARG, "num_clauses must be in [0, 2^31-1)");
    if (!clause_offsets) return fail(GALOIS_E_ARG, "clause_offsets is NULL");
    const int64_t L = clause_offsets[num_clauses];
    if (clause_offsets[0] != 0) return fail(GALOIS_E_OFFSETS, "clause_offsets[0] != 0");
    if (L < 0 || L >= INT32_MAX) return fail(GALOIS_E_OFFSETS, "literal count L must be in [0, 2^31-1)");
    if (L > 0 && !literals) return fail(GALOIS_E_ARG, "literals is NULL");
    int dev = 0;
    if (int rc = check_device(&dev)) return rc;
    cudaStream_t st = nullptr;
    int64_t *d_off64 = nullptr;
    int32_t *d_lits = nullptr;
    CUDA_TRY(use_pool_for_device(dev));
    CUDA_TRY(stream_acquire(&st));
    cudaError_t ce = dmalloc(&d_off64, (size_t)num_clauses + 1, st);
    if (ce == cudaSuccess) ce = dmalloc(&d_lits, (size_t)L, st);
    if (ce == cudaSuccess)
        ce = cudaMemcpyAsync(d_off64, clause_offsets, sizeof(int64_t) * (size_t)(num_clauses + 1),
                             cudaMemcpyHostToDevice, st);
    if (ce == cudaSuccess && L > 0)
        ce = cudaMemcpyAsync(d_lits, literals, sizeof(int32_t) * (size_t)L, cudaMemcpyHostToDevice, st);
    if (ce != cudaSuccess) {
        cudaFreeAsync(d_off64, st);
        cudaFreeAsync(d_lits, st);
        cudaStreamSynchronize(st);
        stream_release(st);
        return fail(ce == cudaErrorMemoryAllocation ? GALOIS_E_OOM : GALOIS_E_CUDA,
                    std::string("cnf upload: ") + cudaGetErrorString(ce));
    }
    const int rc = cnf_build_device(dev, num_vars, num_clauses, L, d_off64, d_lits, st, out);
    stream_release(st);
    return rc;
}

namespace galois {
namespace launch {
cudaError_t tseitin(const int32_t *clause_off, const int2 *slot_info, int64_t m, int32_t n, int32_t k,
                    int64_t **d_off_out, int32_t **d_lits_out, int64_t *m_out, int32_t *aux_out, cudaStream_t st);
}
}  // namespace galois

extern "C" int galois_cnf_normalize(const galois_cnf *in, int32_t k, galois_cnf **out, int32_t *num_aux)
{
    if (!out) return fail(GALOIS_E_ARG, "out is NULL");
    *out = nullptr;
    if (!in) return fail(GALOIS_E_ARG, "cnf is NULL");
    if (k < 3 || k > 32) return fail(GALOIS_E_ARG, "k must be in [3, 32]");
    CUDA_TRY(cudaSetDevice(in->device));
    cudaStream_t st = nullptr;
    CUDA_TRY(stream_acquire(&st));
    int64_t *d_off = nullptr, m2 = 0;
    int32_t *d_lits = nullptr, aux = 0;
    cudaError_t ce = launch::tseitin(in->clause_off, in->slot_info, in->m, in->n, k, &d_off, &d_lits, &m2, &aux, st);
    if (ce == cudaSuccess && (int64_t)in->n + aux >= (1 << 30)) ce = cudaErrorInvalidValue;
    if (ce != cudaSuccess) {
        cudaFreeAsync(d_off, st);
        cudaFreeAsync(d_lits, st);
        cudaStreamSynchronize(st);
        stream_release(st);
        return fail(ce == cudaErrorMemoryAllocation ? GALOIS_E_OOM : GALOIS_E_CUDA,
                    std::string("normalize: ") + cudaGetErrorString(ce));
    }
    if (num_aux) *num_aux = aux;
    const int rc = cnf_build_device(in->device, in->n + aux, m2, m2 * k, d_off, d_lits, st, out);
    if (rc == GALOIS_OK) (*out)->n_orig = in->n_orig;   // auxiliaries are not candidates
    stream_release(st);
    return rc;
}

extern "C" int galois_cnf_get_csr(const galois_cnf *c, int64_t *clause_offsets, int32_t *literals)
{
    if (!c) return fail(GALOIS_E_ARG, "cnf is NULL");
    CUDA_TRY(cudaSetDevice(c->device));
    if (clause_offsets) {
        std::vector<int32_t> off((size_t)c->m + 1);
        CUDA_TRY(cudaMemcpy(off.data(), c->clause_off, off.size() * 4, cudaMemcpyDeviceToHost));
        for (size_t i = 0; i < off.size(); ++i) clause_offsets[i] = off[i];
    }
    if (literals && c->L > 0) {
        std::vector<int2> si((size_t)c->L);
        CUDA_TRY(cudaMemcpy(si.data(), c->slot_info, si.size() * sizeof(int2), cudaMemcpyDeviceToHost));
        for (size_t i = 0; i < si.size(); ++i) {
            const int32_t v = (si[i].x >> 1) + 1;
            literals[i] = (si[i].x & 1) ? -v : v;
        }
    }
    return GALOIS_OK;
}

extern "C" int galois_cnf_info(const galois_cnf *c, int32_t *n, int64_t *m, int64_t *L, int32_t *max_width,
                               int32_t *max_degree, int32_t *num_hubs)
{
    if (!c) return fail(GALOIS_E_ARG, "cnf is NULL");
    if (n) *n = c->n;
    if (m) *m = c->m;
    if (L) *L = c->L;
    if (max_width) *max_width = c->max_width;
    if (max_degree) *max_degree = c->max_degree;
    if (num_hubs) *num_hubs = c->num_hubs;
    return GALOIS_OK;
}

extern "C" int galois_cnf_original_vars(const galois_cnf *c, int32_t *n_orig)
{
    if (!c || !n_orig) return fail(GALOIS_E_ARG, "cnf and n_orig are required");
    *n_orig = c->n_orig;
    return GALOIS_OK;
}

// Eq.11: |S| = max(1, ceil(rho n)) over the original variables.
constexpr int32_t kMaxUnits = 1 << 20;   // |S| per candidate (paper rho = 0.0005: n < 2^31)

static int32_t units_per_candidate(const galois_cnf *c, double rho)
{
    return std::max<int32_t>(1, (int32_t)std::ceil(rho * (double)c->n_orig - 1e-9));
}

extern "C" int galois_candidate_pool_size(const galois_cnf *c, double rho, int32_t *S)
{
    if (!c || !S) return fail(GALOIS_E_ARG, "cnf and S are required");
    if (!(rho > 0.0 && rho <= 1.0)) return fail(GALOIS_E_ARG, "need 0 < rho <= 1");
    *S = units_per_candidate(c, rho);
    return GALOIS_OK;
}

extern "C" int galois_cnf_get_csc(const galois_cnf *c, int32_t *code_off, int32_t *occ_slot)
{
    if (!c) return fail(GALOIS_E_ARG, "cnf is NULL");
    CUDA_TRY(cudaSetDevice(c->device));
    if (code_off) CUDA_TRY(cudaMemcpy(code_off, c->code_off, (2 * (size_t)c->n + 1) * 4, cudaMemcpyDeviceToHost));
    if (occ_slot && c->L > 0) CUDA_TRY(cudaMemcpy(occ_slot, c->occ_slot, (size_t)c->L * 4, cudaMemcpyDeviceToHost));
    return GALOIS_OK;
}

extern "C" void galois_cnf_free(galois_cnf *c) { cnf_release(c); }

// ------------------------------------------------------------------------ engine
struct galois_engine {
    galois_cnf *cnf = nullptr;
    int device = 0;
    // configuration
    int64_t B = 0;
    int32_t T = 0;
    double lr = 0.5, tau = 1.0, beta1 = 0.9, beta2 = 0.999, eps = 1e-8;
    int32_t optimizer = 0, mode = 0, K = 1;
    uint64_t seed = 0;
    std::vector<int32_t> pins;   // 0-based, ascending
    int32_t rank = 0, world = 1;
    unsigned char nccl_id[128] = {0};
    bool use_comm = false;         // NCCL path (world > 1, or a 1-rank communicator for tests)
    // NCCL exchange off the critical path: the MIN all-reduce of a check runs on `xstream`
    // (forked after the checking sweep by ev_chk) while the update runs; the main stream
    // joins ev_x and runs k_gfinalize before its next sweep or result read (x_pending)
    cudaStream_t xstream = nullptr;
    cudaEvent_t ev_chk = nullptr, ev_x = nullptr;
    bool x_pending = false;
    bool debug = false, profiling = false;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    // state
    bool prepared = false, poisoned = false;
    bool pending_check = false;  // the rounding in R still has to be checked
    int32_t steps_enqueued = 0;
    int64_t b_per = 0, b0 = 0;
    int32_t b_loc = 0, b_pad = 0, W = 0;
    // sub-batching (f4): `windows` consecutive windows of `sub` members over the local
    // slice [slice_b0, slice_b0 + slice_loc); b0 / b_loc describe the resident window
    int32_t sub = 0, windows = 1;
    int64_t slice_b0 = 0, slice_loc = 0;
    struct Agg {
        int32_t u = INT32_MAX, t = -1, steps = 0;
        int64_t b = -1;
        bool sat = false, ran = false;
    } agg;
    std::vector<uint8_t> agg_bits;     // winner's rounding over all windows
    std::vector<int32_t> agg_counts;   // each local member's last check
    // theta_sel over the windows (rule 0 min / rule 1 max of each member's last count):
    // key as k_select, and that member's iterate at the end of its window (device [2][n])
    unsigned long long sel_key[2] = {~0ull, ~0ull};
    float *sel_z = nullptr;
    unsigned long long *sel_dkey = nullptr;
    // lanes: the local slice split into `lane.size()` engines over consecutive member ranges
    // (1024-member multiples), each with its own stream and control block, stepped
    // concurrently so one lane's clause sweep overlaps another lane's update. Members never
    // interact, so every member's trajectory is the one the undivided engine gives it; the
    // aggregate (agg, sel_*) is formed over the lanes as over f4's windows.
    int32_t lanes_req = 1;
    std::vector<galois_engine *> lane;
    int64_t lane_size = 0;
    bool fixed_slice = false;          // a lane: b0 / b_loc set by the parent
    cudaEvent_t fork_ev = nullptr;
    std::vector<cudaEvent_t> join_ev;
    Comm comm;
    // device buffers
    float *z = nullptr, *m = nullptr, *v = nullptr;
    uint32_t *X = nullptr, *R = nullptr, *E = nullptr;
    void *slab = nullptr;          // one pooled allocation holding every device buffer below
    short4 *partial = nullptr;
    int32_t *lam = nullptr, *unsat = nullptr, *unsat_last = nullptr;   // lam: 2 x b_pad (step parity)
    Ctrl *ctrl = nullptr;
    uint8_t *best_bits = nullptr;
    // single-launch run of small instances (k_small_run): scratch, per-CTA records, snapshots
    SmallScratch *small_gs = nullptr;
    unsigned long long *small_recs = nullptr;
    uint8_t *small_snap = nullptr;
    int8_t *pin_rank = nullptr;
    float2 *adam_consts = nullptr;
    int32_t *dbg_G = nullptr;
    float *dbg_g1 = nullptr;
    float *P = nullptr, *Es = nullptr, *lam_f = nullptr, *dbg_Gf = nullptr;   // SOFT mode
    Ctrl *h_ctrl = nullptr;     // pinned mirror (2 slots)
    cudaEvent_t poll_ev[2] = {nullptr, nullptr};
    // CUDA graph of kGraphSteps consecutive steps (run(); not while profiling)
    cudaGraphExec_t graph = nullptr;
    int32_t graph_steps = 0;
    bool graph_failed = false;
    int32_t graphs_mode = 0;     // galois_engine_set_graphs: -1 never, 0 auto, 1 always
    // profiling
    struct Rec {
        int cls;
        cudaEvent_t a, b;
    };
    std::vector<Rec> recs;
    std::vector<cudaEvent_t> ev_pool;

    StepParams params() const
    {
        StepParams p;
        p.n = cnf->n;
        p.b_pad = b_pad;
        p.W = W;
        p.b_loc = b_loc;
        p.b0 = b0;
        p.seed = seed;
        p.tau = (float)tau;
        p.inv_tau = (float)(1.0 / tau);
        p.beta1 = (float)beta1;
        p.beta2 = (float)beta2;
        p.eps = (float)eps;
        p.omb1 = (float)(1.0 - beta1);
        p.omb2 = (float)(1.0 - beta2);
        p.optimizer = optimizer;
        p.lr = (float)lr;
        p.adam_consts = adam_consts;
        p.num_pins = (int32_t)pins.size();
        p.pin_rank = pins.empty() ? nullptr : pin_rank;
        p.keys = philox_round_keys(seed);
        p.clear_a = nullptr;
        p.clear_b = nullptr;
        return p;
    }

    cudaEvent_t take_event()
    {
        if (!ev_pool.empty()) {
            cudaEvent_t e = ev_pool.back();
            ev_pool.pop_back();
            return e;
        }
        cudaEvent_t e = nullptr;
        cudaEventCreate(&e);
        return e;
    }
    template <typename F>
    void timed(int cls, F &&f, cudaStream_t on = nullptr)
    {
        if (!profiling) {
            f();
            return;
        }
        Rec r{cls, take_event(), take_event()};
        cudaEventRecord(r.a, on ? on : stream);
        f();
        cudaEventRecord(r.b, on ? on : stream);
        recs.push_back(r);
    }
};

static void engine_free_buffers(galois_engine *e)
{
    if (e->sel_z) cudaFreeAsync(e->sel_z, e->stream);
    if (e->sel_dkey) cudaFreeAsync(e->sel_dkey, e->stream);
    e->sel_z = nullptr;
    e->sel_dkey = nullptr;
    if (e->slab) {
        cudaFreeAsync(e->slab, e->stream);
        cudaStreamSynchronize(e->stream);
    }
    e->slab = nullptr;
    if (e->h_ctrl) pinned_ctrl_release(e->h_ctrl);
    e->h_ctrl = nullptr;
    e->z = e->m = e->v = nullptr;
}

extern "C" int galois_engine_create(const galois_cnf *cnf, int64_t batch, int32_t steps, double lr, uint64_t seed,
                                    galois_engine **out)
{
    if (!out) return fail(GALOIS_E_ARG, "out is NULL");
    *out = nullptr;
    if (!cnf) return fail(GALOIS_E_ARG, "cnf is NULL");
    if (batch < 1 || batch > (int64_t(1) << 32)) return fail(GALOIS_E_ARG, "batch must be in [1, 2^32]");
    if (steps < 0 || steps > (1 << 30)) return fail(GALOIS_E_ARG, "steps must be in [0, 2^30]");
    if (!(lr > 0.0f) || !std::isfinite(lr)) return fail(GALOIS_E_ARG, "lr must be a positive finite number");
    galois_engine *e = new galois_engine();
    const_cast<galois_cnf *>(cnf)->refs.fetch_add(1);
    e->cnf = const_cast<galois_cnf *>(cnf);
    e->device = cnf->device;
    e->B = batch;
    e->T = steps;
    e->lr = lr;
    e->seed = seed;
    *out = e;
    return GALOIS_OK;
}

#define ENGINE_ENTRY(e)                                                                        \
    do {                                                                                       \
        if (!(e)) return fail(GALOIS_E_ARG, "engine is NULL");                                 \
        if ((e)->poisoned) return fail(GALOIS_E_STATE, "engine is poisoned by an earlier error"); \
    } while (0)

#define WHOLE_SLICE_ONLY(e)                                                                                  \
    do {                                                                                                     \
        if ((e)->windows > 1) return fail(GALOIS_E_STATE, "not available on a sub-batched engine (run only)"); \
        if (!(e)->lane.empty()) return fail(GALOIS_E_STATE, "not available on an engine split into lanes");   \
    } while (0)

// results formed over several sub-engines / windows (f4 windows, lanes)
static bool aggregated(const galois_engine *e) { return e->windows > 1 || !e->lane.empty(); }

// Test hooks on a split engine: f(lane, offset of the lane's first member in the slice) for
// every lane holding members (host arrays are [local member][...], so lane rows follow each
// other).
template <typename F>
static int for_each_lane(galois_engine *e, F &&f)
{
    for (galois_engine *l : e->lane) {
        if (l->b_loc == 0) continue;
        if (int rc = f(l, (size_t)(l->b0 - e->b0))) return rc;
    }
    return GALOIS_OK;
}

#define NO_WINDOWS(e)                                                                                        \
    do {                                                                                                     \
        if ((e)->windows > 1) return fail(GALOIS_E_STATE, "not available on a sub-batched engine (run only)"); \
    } while (0)

#define SETTER_ENTRY(e)                                                                        \
    do {                                                                                       \
        ENGINE_ENTRY(e);                                                                       \
        if ((e)->prepared) return fail(GALOIS_E_STATE, "setters are valid only before the first step"); \
    } while (0)

extern "C" int galois_engine_set_mode(galois_engine *e, int32_t mode)
{
    SETTER_ENTRY(e);
    if (mode != GALOIS_MODE_ST && mode != GALOIS_MODE_SOFT) return fail(GALOIS_E_ARG, "mode must be 0 or 1");
    e->mode = mode;
    return GALOIS_OK;
}

extern "C" int galois_engine_set_hparams(galois_engine *e, double tau, double beta1, double beta2, double eps,
                                         int32_t optimizer)
{
    SETTER_ENTRY(e);
    if (!(tau > 0.0f) || !std::isfinite(tau)) return fail(GALOIS_E_ARG, "tau must be > 0");
    if (!(beta1 >= 0.0f && beta1 < 1.0f) || !(beta2 >= 0.0f && beta2 < 1.0f))
        return fail(GALOIS_E_ARG, "betas must be in [0, 1)");
    if (!(eps > 0.0f) || !std::isfinite(eps)) return fail(GALOIS_E_ARG, "eps must be > 0");
    if (optimizer != GALOIS_ADAM && optimizer != GALOIS_SGD) return fail(GALOIS_E_ARG, "optimizer must be 0 or 1");
    e->tau = tau;
    e->beta1 = beta1;
    e->beta2 = beta2;
    e->eps = eps;
    e->optimizer = optimizer;
    return GALOIS_OK;
}

extern "C" int galois_engine_set_check_interval(galois_engine *e, int32_t k)
{
    SETTER_ENTRY(e);
    if (k < 1) return fail(GALOIS_E_ARG, "check interval must be >= 1");
    e->K = k;
    return GALOIS_OK;
}

extern "C" int galois_engine_set_cubes(galois_engine *e, int32_t d, const int32_t *vars)
{
    SETTER_ENTRY(e);
    if (d < 0 || d > 30) return fail(GALOIS_E_ARG, "d must be in [0, 30]");
    if (d > 0 && !vars) return fail(GALOIS_E_ARG, "vars is NULL");
    std::vector<int32_t> p(vars, vars + d);
    for (int32_t &x : p) {
        if (x < 1 || x > e->cnf->n) return fail(GALOIS_E_VAR_RANGE, "cube variable out of range");
        x -= 1;
    }
    std::sort(p.begin(), p.end());
    if (std::adjacent_find(p.begin(), p.end()) != p.end()) return fail(GALOIS_E_ARG, "cube variables must be distinct");
    e->pins = p;
    return GALOIS_OK;
}

extern "C" int galois_engine_set_comm(galois_engine *e, int32_t rank, int32_t world, const void *id)
{
    SETTER_ENTRY(e);
    if (world < 1 || rank < 0 || rank >= world) return fail(GALOIS_E_ARG, "need 0 <= rank < world");
    e->rank = rank;
    e->world = world;
    if (id) memcpy(e->nccl_id, id, 128);
    // id: the NCCL path (world = 1 with an id: on one GPU); no id: rank's slice alone
    e->use_comm = id != nullptr;
    return GALOIS_OK;
}

extern "C" int galois_engine_set_subbatch(galois_engine *e, int32_t sub_batch)
{
    SETTER_ENTRY(e);
    if (sub_batch < 0 || sub_batch % 32 != 0) return fail(GALOIS_E_ARG, "sub_batch must be 0 or a positive multiple of 32");
    e->sub = sub_batch;
    return GALOIS_OK;
}

extern "C" int galois_engine_bytes_per_member(const galois_cnf *c, int32_t mode, int64_t *bytes)
{
    if (!c || !bytes) return fail(GALOIS_E_ARG, "cnf and bytes are required");
    if (mode != GALOIS_MODE_ST && mode != GALOIS_MODE_SOFT) return fail(GALOIS_E_ARG, "mode must be 0 or 1");
    // mirrors prepare(): z, m, v fp32 + X, R bits + unsat, unsat_last (+ mode buffers)
    int64_t b = 12 * (int64_t)c->n + ((int64_t)c->n + 3) / 4 + 8;
    if (mode == GALOIS_MODE_ST)
        b += ((int64_t)c->L + 7) / 8 + 8 + 2 * (int64_t)c->num_hub_chunks;   // E bits, lam x 2, hub partials
    else
        b += 4 * (int64_t)c->n + 4 * (int64_t)c->L + 4 * (1 + launch::soft_chunks());   // P, Es, lam_f
    *bytes = b;
    return GALOIS_OK;
}

static void engine_layout(Slab &slab, galois_engine *e);

static int32_t padded_members(int64_t resident)   // prepare's b_pad for `resident` members
{
    return resident <= 1024 ? (int32_t)std::max<int64_t>(32, (resident + 31) / 32 * 32)
                            : (int32_t)((resident + 1023) / 1024 * 1024);
}

static int64_t window_bytes(const galois_cnf *c, int32_t mode, int64_t members, int32_t steps, bool cubes)
{
    galois_engine tmp;
    tmp.cnf = const_cast<galois_cnf *>(c);
    tmp.mode = mode;
    tmp.T = steps;
    tmp.b_pad = padded_members(members);
    tmp.W = tmp.b_pad / 32;
    if (cubes) tmp.pins.assign(1, 1);
    Slab slab;
    engine_layout(slab, &tmp);
    tmp.cnf = nullptr;
    return (int64_t)slab.total();
}

extern "C" int galois_engine_window_bytes(const galois_cnf *c, int32_t mode, int32_t members, int32_t steps,
                                          int32_t with_cubes, int64_t *bytes)
{
    if (!c || !bytes) return fail(GALOIS_E_ARG, "cnf and bytes are required");
    if (mode != GALOIS_MODE_ST && mode != GALOIS_MODE_SOFT) return fail(GALOIS_E_ARG, "mode must be 0 or 1");
    if (members < 1 || steps < 0) return fail(GALOIS_E_ARG, "need members >= 1 and steps >= 0");
    *bytes = window_bytes(c, mode, members, steps, with_cubes != 0);
    return GALOIS_OK;
}

extern "C" int galois_engine_max_sub_batch(const galois_cnf *c, int32_t mode, int32_t steps, int32_t with_cubes,
                                           int64_t budget_bytes, int32_t *sub_batch)
{
    if (!c || !sub_batch) return fail(GALOIS_E_ARG, "cnf and sub_batch are required");
    if (mode != GALOIS_MODE_ST && mode != GALOIS_MODE_SOFT) return fail(GALOIS_E_ARG, "mode must be 0 or 1");
    if (steps < 0) return fail(GALOIS_E_ARG, "steps must be >= 0");
    const bool cubes = with_cubes != 0;
    if (window_bytes(c, mode, 32, steps, cubes) > budget_bytes)
        return fail(GALOIS_E_OOM, "a 32-member window does not fit the budget");
    int64_t lo = 1, hi = (int64_t)(INT32_MAX - 1024) / 32;   // multiples of 32 members: lo fits
    while (lo < hi) {
        const int64_t mid = (lo + hi + 1) / 2;
        if (window_bytes(c, mode, 32 * mid, steps, cubes) <= budget_bytes)
            lo = mid;
        else
            hi = mid - 1;
    }
    *sub_batch = (int32_t)(32 * lo);
    return GALOIS_OK;
}

extern "C" int galois_device_free_bytes(int32_t device, int64_t *bytes)
{
    if (!bytes) return fail(GALOIS_E_ARG, "bytes is NULL");
    int cur = 0;
    CUDA_TRY(cudaGetDevice(&cur));
    CUDA_TRY(cudaSetDevice(device));
    size_t free_b = 0, total_b = 0;
    cudaError_t ce = cudaMemGetInfo(&free_b, &total_b);
    cudaMemPool_t pool;
    uint64_t reserved = 0, used = 0;
    if (ce == cudaSuccess) ce = cudaDeviceGetDefaultMemPool(&pool, device);
    if (ce == cudaSuccess) ce = cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved);
    if (ce == cudaSuccess) ce = cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used);
    cudaSetDevice(cur);
    CUDA_TRY(ce);
    *bytes = (int64_t)free_b + (int64_t)(reserved > used ? reserved - used : 0);
    return GALOIS_OK;
}

extern "C" int galois_engine_set_stream(galois_engine *e, void *s)
{
    SETTER_ENTRY(e);
    e->stream = (cudaStream_t)s;
    e->own_stream = false;
    return GALOIS_OK;
}

extern "C" int galois_engine_set_debug(galois_engine *e, int32_t enable)
{
    SETTER_ENTRY(e);
    e->debug = enable != 0;
    return GALOIS_OK;
}

extern "C" int galois_engine_set_profiling(galois_engine *e, int32_t enable)
{
    ENGINE_ENTRY(e);
    e->profiling = enable != 0;
    for (galois_engine *l : e->lane) l->profiling = e->profiling;
    return GALOIS_OK;
}

extern "C" int galois_engine_set_lanes(galois_engine *e, int32_t lanes)
{
    SETTER_ENTRY(e);
    if (lanes < 1 || lanes > 16) return fail(GALOIS_E_ARG, "lanes must be in [1, 16]");
    e->lanes_req = lanes;
    return GALOIS_OK;
}

extern "C" int galois_engine_set_graphs(galois_engine *e, int32_t mode)
{
    SETTER_ENTRY(e);
    if (mode < -1 || mode > 1) return fail(GALOIS_E_ARG, "graphs mode must be -1, 0 or 1");
    e->graphs_mode = mode;
    return GALOIS_OK;
}

extern "C" int galois_comm_unique_id(void *out128)
{
    if (!out128) return fail(GALOIS_E_ARG, "out is NULL");
    std::string why;
    if (!nccl_unique_id(out128, &why)) return fail(GALOIS_E_NCCL, why);
    return GALOIS_OK;
}

static int poison(galois_engine *e, int code, const std::string &msg)
{
    e->poisoned = true;
    return fail(code, msg);
}

#define ENG_CUDA(e, expr)                                                                      \
    do {                                                                                       \
        cudaError_t _e = (expr);                                                               \
        if (_e != cudaSuccess)                                                                 \
            return poison((e), _e == cudaErrorMemoryAllocation ? GALOIS_E_OOM : GALOIS_E_CUDA, \
                          std::string(#expr) + ": " + cudaGetErrorString(_e));                 \
    } while (0)

static bool is_check_step(const galois_engine *e, int32_t s) { return (s % e->K) == 0 || s == e->T; }

// Best tracking after the unsat counts of the rounding R_t are in e->unsat (t = ctrl->t):
// local argmin, [NCCL MIN over ranks, finalize], winner's bits. One timing record per
// kernel, so the launch counts of galois_engine_kernel_times are exact.
static BestArgs best_args(const galois_engine *e)
{
    BestArgs ba;
    ba.unsat_last = e->unsat_last;
    ba.b_loc = e->b_loc;
    ba.b0 = e->b0;
    ba.finalize = 1;                  // this rank's record (with NCCL the global one follows at the join)
    // small instances: the sweep's last CTA also copies the winner's bits (n loads in one
    // CTA); large ones launch the grid-wide k_extract instead
    ba.best_bits = e->best_bits;
    ba.W = e->W;
    ba.extract_n = e->cnf->n <= 32768 ? e->cnf->n : 0;
    return ba;
}

// The main stream waits for the exchange of the last check (before anything that rewrites
// key_local, reads the control block, or ends a graph capture). One step of lag at most:
// a rank that did not hold the SAT member may run the update right after the deciding check.
static int exchange_join(galois_engine *e)
{
    if (!e->x_pending) return GALOIS_OK;
    ENG_CUDA(e, cudaStreamWaitEvent(e->stream, e->ev_x, 0));
    // the global record and stop flag are folded in on the MAIN stream: the update kernels
    // that overlapped the all-reduce read ctrl->stopped, so no other stream may write it
    // while they run (a flag flipping mid-launch would stop only part of a grid)
    e->timed(3, [&] { launch::gfinalize(e->ctrl, e->stream); });
    e->x_pending = false;
    return GALOIS_OK;
}

// a9 with NCCL: fork the check's key to the exchange stream and MIN all-reduce it over the
// ranks there; the main stream continues with the update and folds the result into the
// global record (k_gfinalize) when it joins, before its next sweep or result read.
static int exchange_fork(galois_engine *e)
{
    ENG_CUDA(e, cudaEventRecord(e->ev_chk, e->stream));
    ENG_CUDA(e, cudaStreamWaitEvent(e->xstream, e->ev_chk, 0));
    std::string why;
    if (!e->comm.allreduce_min_u64(&e->ctrl->key_local, &e->ctrl->key_global, e->xstream, &why))
        return poison(e, GALOIS_E_NCCL, why);
    ENG_CUDA(e, cudaEventRecord(e->ev_x, e->xstream));
    e->x_pending = true;
    return GALOIS_OK;
}

// After the counts of a check are complete. best_done: the sweep's last CTA already
// reduced them into this rank's record. extract: launch k_extract for the record's bits
// (false when the sweep's last CTA already copied them). With NCCL the exchange follows
// on its own stream.
static int enqueue_best(galois_engine *e, bool best_done, bool extract)
{
    if (!best_done)
        e->timed(3, [&] { launch::best(e->unsat, e->unsat_last, e->b_loc, e->b0, e->ctrl, true, e->stream); });
    if (extract)
        e->timed(3, [&] { launch::extract(e->R, e->cnf->n, e->W, e->b0, e->ctrl, e->best_bits, e->stream); });
    ENG_CUDA(e, cudaGetLastError());
    if (e->use_comm)
        if (int rc = exchange_fork(e)) return rc;
    return GALOIS_OK;
}

// Check of the pending rounding alone (t = 0 after init, or the last step before results
// are read): check-only sweep + best tracking.
static int flush_check(galois_engine *e)
{
    if (!e->pending_check) return GALOIS_OK;
    if (int rc = exchange_join(e)) return rc;
    const DevCnf c = e->cnf->view();
    ENG_CUDA(e, cudaMemsetAsync(e->unsat, 0, sizeof(int32_t) * (size_t)e->b_pad, e->stream));
    bool done = false;
    e->timed(2, [&] {
        done = launch::clauses(c, e->W, e->b_pad, nullptr, e->R, nullptr, nullptr, e->unsat, e->ctrl, best_args(e),
                               e->stream);
    });
    e->pending_check = false;
    if (int rc = enqueue_best(e, done, !(done && best_args(e).extract_n > 0))) return rc;
    ENG_CUDA(e, cudaGetLastError());
    return GALOIS_OK;
}

// Step s = steps_enqueued + 1. ST mode: one clause sweep does the forward of X_s and, if
// the previous step was a check point, the exact check of R_{s-1}; then best tracking
// for R_{s-1} (so a SAT rounding stops the engine before the update of step s), the hub
// partials, and the fused update (which ticks t at its end).
static int enqueue_step(galois_engine *e)
{
    const DevCnf c = e->cnf->view();
    StepParams p = e->params();
    const int32_t s = e->steps_enqueued + 1;
    if (int rc = exchange_join(e)) return rc;
    if (e->mode == GALOIS_MODE_ST) {
        const bool chk = e->pending_check;
        // Lambda of step s goes to lam[s & 1]; the update of step s zeroes lam[(s+1) & 1]
        // and unsat for the next sweep (and does nothing once the engine has stopped, so
        // the counters of the deciding check survive)
        int32_t *lam_s = e->lam + (size_t)(s & 1) * e->b_pad;
        p.clear_a = e->lam + (size_t)((s + 1) & 1) * e->b_pad;
        p.clear_b = e->unsat;
        bool done = false;
        e->timed(0, [&] {
            done = launch::clauses(c, e->W, e->b_pad, e->X, chk ? e->R : nullptr, e->E, lam_s, e->unsat, e->ctrl,
                                   best_args(e), e->stream);
        });
        if (chk) {
            e->pending_check = false;
            if (int rc = enqueue_best(e, done, !(done && best_args(e).extract_n > 0))) return rc;
        }
        if (c.num_hub_chunks > 0)
            e->timed(4, [&] { launch::hub_partial(c, e->W, e->b_pad, e->E, e->partial, e->ctrl, e->stream); });
        e->timed(1, [&] {
            launch::update_st(c, p, e->z, e->m, e->v, e->X, e->R, e->E, e->partial, e->ctrl,
                              e->debug ? e->dbg_G : nullptr, e->debug ? e->dbg_g1 : nullptr, e->stream);
        });
    } else {
        if (int rc = flush_check(e)) return rc;
        ENG_CUDA(e, cudaMemsetAsync(e->lam_f, 0, sizeof(float) * (size_t)e->b_pad, e->stream));
        e->timed(0, [&] { launch::forward_soft(c, p, e->z, e->P, e->Es, e->lam_f, e->ctrl, e->stream); });
        e->timed(1, [&] {
            launch::update_soft(c, p, e->z, e->m, e->v, e->X, e->R, e->Es, e->ctrl,
                                e->debug ? e->dbg_Gf : nullptr, e->debug ? e->dbg_g1 : nullptr, e->stream);
        });
    }
    ENG_CUDA(e, cudaGetLastError());
    e->steps_enqueued = s;
    e->pending_check = is_check_step(e, s);
    return GALOIS_OK;
}

static int prepare(galois_engine *e);

// Lanes of ls members (the last one shorter) over the local slice; each lane is a complete
// engine (own buffers, stream, control block, CUDA graph) with the parent's configuration.
static int prepare_lanes(galois_engine *e, int64_t ls, int64_t lspan)
{
    if (!e->stream) {
        ENG_CUDA(e, stream_acquire(&e->stream));
        e->own_stream = true;
    }
    e->lane_size = ls;
    for (int64_t off = 0; off < lspan; off += ls) {
        galois_engine *l = new galois_engine();
        e->cnf->refs.fetch_add(1);
        l->cnf = e->cnf;
        l->device = e->device;
        l->B = e->B;
        l->T = e->T;
        l->lr = e->lr;
        l->tau = e->tau;
        l->beta1 = e->beta1;
        l->beta2 = e->beta2;
        l->eps = e->eps;
        l->optimizer = e->optimizer;
        l->mode = e->mode;
        l->K = e->K;
        l->seed = e->seed;
        l->pins = e->pins;
        l->profiling = e->profiling;
        l->graphs_mode = e->graphs_mode;
        l->fixed_slice = true;
        l->b0 = e->b0 + off;
        l->b_loc = (int32_t)std::max<int64_t>(0, std::min<int64_t>(ls, e->b_loc - off));
        l->b_per = e->b_per;
        e->lane.push_back(l);
        if (int rc = prepare(l)) {
            e->poisoned = true;
            return rc;
        }
        cudaEvent_t ev = nullptr;
        ENG_CUDA(e, cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        e->join_ev.push_back(ev);
    }
    ENG_CUDA(e, cudaEventCreateWithFlags(&e->fork_ev, cudaEventDisableTiming));
    e->prepared = true;
    return GALOIS_OK;
}

// The engine's device buffers (ONE slab, see prepare): shared by prepare and the sizing
// calls (galois_engine_window_bytes), so a window's size is exactly what prepare allocates.
static void engine_layout(Slab &slab, galois_engine *e)
{
    const galois_cnf *c = e->cnf;
    const int32_t n = c->n;
    const size_t nb = (size_t)n * (size_t)e->b_pad;
    slab.add(&e->z, nb);
    slab.add(&e->m, nb);
    slab.add(&e->v, nb);
    slab.add(&e->X, (size_t)n * 2 * xr_pad(e->W));   // interleaved X/R rows (galois_internal.h)
    slab.add(&e->unsat, (size_t)e->b_pad);
    slab.add(&e->unsat_last, (size_t)e->b_pad);
    slab.add(&e->ctrl, 1);
    slab.add(&e->best_bits, (size_t)n);
    slab.add(&e->adam_consts, (size_t)e->T + 2);
    if (!e->pins.empty()) slab.add(&e->pin_rank, (size_t)n);
    if (e->mode == GALOIS_MODE_ST && launch::small_run_smem(n, (int32_t)c->L) <= kSmallRunSmem) {
        slab.add(&e->small_gs, 1);
        slab.add(&e->small_recs, 2 * (size_t)e->W);
        slab.add(&e->small_snap, (size_t)e->W * (size_t)n);
    }
    if (e->mode == GALOIS_MODE_ST) {
        slab.add(&e->E, (size_t)c->L * e->W + 4);   // + 16 B: the small-window update copies whole 16-B units
        slab.add(&e->lam, 2 * (size_t)e->b_pad);
        if (c->num_hub_chunks > 0) slab.add(&e->partial, (size_t)c->num_hub_chunks * (e->b_pad / 4));
        if (e->debug) {
            slab.add(&e->dbg_G, nb);
            slab.add(&e->dbg_g1, nb);
        }
    } else {
        slab.add(&e->P, nb);
        slab.add(&e->Es, (size_t)c->L * e->b_pad);
        slab.add(&e->lam_f, (size_t)e->b_pad * (1 + launch::soft_chunks()));
        if (e->debug) {
            slab.add(&e->dbg_Gf, nb);
            slab.add(&e->dbg_g1, nb);
        }
    }
}

static int prepare(galois_engine *e)
{
    if (e->prepared) return GALOIS_OK;
    ENG_CUDA(e, cudaSetDevice(e->device));
    ENG_CUDA(e, launch::configure_kernels());
    galois_cnf *c = e->cnf;
    const int32_t n = c->n;
    // batch slice: b_per = roundup(ceil(B / world), 32); pad the local slice to 32
    if (e->fixed_slice) {                // a lane: b0 / b_loc (/ b_per) were set by its parent
        if (!e->b_per) e->b_per = e->b_loc;
    } else {
        int64_t per = (e->B + e->world - 1) / e->world;
        per = (per + 31) / 32 * 32;
        e->b_per = per;
        e->b0 = per * e->rank;
        if (per > INT32_MAX - 1024) return poison(e, GALOIS_E_ARG, "local batch slice must be < 2^31 - 1024 members");
        const int64_t left = e->B - e->b0;
        e->b_loc = (int32_t)std::max<int64_t>(0, std::min<int64_t>(per, left));
    }
    e->slice_b0 = e->b0;
    e->slice_loc = e->b_loc;
    // f4: windows of sub members; with NCCL every rank runs the same number of windows
    const int64_t span = e->use_comm ? e->b_per : e->slice_loc;
    if (e->sub > 0 && e->sub < span) {
        e->windows = (int32_t)((span + e->sub - 1) / e->sub);
        e->b_loc = (int32_t)std::min<int64_t>(e->sub, e->slice_loc);
    }
    if (e->lanes_req > 1 && e->windows == 1 && e->mode == GALOIS_MODE_ST && !e->debug && !e->use_comm) {
        const int64_t lspan = e->b_loc;
        const int64_t per_lane = (lspan + e->lanes_req - 1) / e->lanes_req;
        const int64_t ls = (per_lane + 1023) / 1024 * 1024;
        if (lspan > ls) return prepare_lanes(e, ls, lspan);
    }
    const int32_t resident = e->windows > 1 ? e->sub : e->b_loc;
    // pad to 32 members (one bit word) up to 1024, then to whole 1024-member chunks, so that
    // W <= 32 or W % 32 == 0 (chunk-major E, TMA-staged update)
    e->b_pad = padded_members(resident);
    e->W = e->b_pad / 32;
    if ((uint64_t)n * (uint64_t)e->b_pad / 4 >= (1ull << 40))
        return poison(e, GALOIS_E_ARG, "n * local batch too large");
    if (!e->stream) {
        ENG_CUDA(e, stream_acquire(&e->stream));
        e->own_stream = true;
    }
    const size_t nb = (size_t)n * (size_t)e->b_pad;
    // all device buffers of the engine live in ONE stream-ordered allocation from the
    // device's memory pool (cheap to create and free repeatedly, e.g. time-to-SAT runs)
    Slab slab;
    engine_layout(slab, e);
    ENG_CUDA(e, use_pool_for_device(e->device));
    ENG_CUDA(e, cudaMallocAsync(&e->slab, slab.total(), e->stream));
    slab.assign(e->slab);
    e->R = e->X + xr_roff(e->W);
    ENG_CUDA(e, cudaMemsetAsync(e->unsat, 0, sizeof(int32_t) * (size_t)e->b_pad, e->stream));
    ENG_CUDA(e, cudaMemsetAsync(e->unsat_last, 0, sizeof(int32_t) * (size_t)e->b_pad, e->stream));
    ENG_CUDA(e, cudaMemsetAsync(e->best_bits, 0, (size_t)n, e->stream));
    if (e->lam) ENG_CUDA(e, cudaMemsetAsync(e->lam, 0, 2 * sizeof(int32_t) * (size_t)e->b_pad, e->stream));
    if (e->small_gs) {                   // {tstar = "no SAT", done = 0, arrive = 0}; the last CTA resets them
        ENG_CUDA(e, cudaMemsetAsync(e->small_gs, 0, sizeof(SmallScratch), e->stream));
        ENG_CUDA(e, cudaMemsetAsync(&e->small_gs->tstar, 0x7f, sizeof(int32_t), e->stream));
    }
    // Adam step constants in fp64, per step index: 2 lr / (1 - beta1^t), 1 / sqrt(1 - beta2^t)
    // (the factor 2: z = theta_1 - theta_0 moves by twice the per-logit step)
    std::vector<float2> consts((size_t)e->T + 2);
    for (size_t t = 0; t < consts.size(); ++t) {
        const double bc1 = 1.0 - std::pow(e->beta1, (double)t);
        const double bc2 = 1.0 - std::pow(e->beta2, (double)t);
        consts[t] = make_float2(t ? (float)(2.0 * e->lr / bc1) : 0.f, t ? (float)(1.0 / std::sqrt(bc2)) : 0.f);
    }
    ENG_CUDA(e, cudaMemcpyAsync(e->adam_consts, consts.data(), consts.size() * sizeof(float2), cudaMemcpyHostToDevice,
                                e->stream));
    std::vector<int8_t> pr;
    if (!e->pins.empty()) {
        pr.assign((size_t)n, -1);
        for (size_t r = 0; r < e->pins.size(); ++r) pr[e->pins[r]] = (int8_t)r;
        ENG_CUDA(e, cudaMemcpyAsync(e->pin_rank, pr.data(), (size_t)n, cudaMemcpyHostToDevice, e->stream));
    }
    Ctrl h{};
    h.t = 0;
    h.stopped = 0;
    h.best_u = h.g_u = INT32_MAX;
    h.best_t = h.g_t = -1;
    h.best_b = h.g_b = -1;
    ENG_CUDA(e, pinned_ctrl_acquire(&e->h_ctrl));
    e->h_ctrl[0] = h;
    // (no sync: later D2H copies into h_ctrl are ordered after this one on the stream, and
    // the host writes h_ctrl[0] again only after a stream synchronisation)
    ENG_CUDA(e, cudaMemcpyAsync(e->ctrl, &e->h_ctrl[0], sizeof(Ctrl), cudaMemcpyHostToDevice, e->stream));
    for (auto &ev : e->poll_ev) ENG_CUDA(e, cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    if (e->use_comm) {
        std::string why;
        if (!e->comm.init(e->rank, e->world, e->nccl_id, &why)) return poison(e, GALOIS_E_NCCL, why);
        ENG_CUDA(e, stream_acquire(&e->xstream));
        ENG_CUDA(e, cudaEventCreateWithFlags(&e->ev_chk, cudaEventDisableTiming));
        ENG_CUDA(e, cudaEventCreateWithFlags(&e->ev_x, cudaEventDisableTiming));
    }
    e->prepared = true;
    // a3: initial logits, first sample, and the check at t = 0
    const StepParams p = e->params();
    e->timed(5, [&] { launch::init(p, e->z, e->m, e->v, e->X, e->R, e->stream); });
    ENG_CUDA(e, cudaGetLastError());
    e->pending_check = true;             // the t = 0 check runs with the first sweep
    return GALOIS_OK;
}

// Enqueue G steps as one CUDA graph. The first call captures enqueue_step() G times (the
// host-side state advances during capture exactly as every replay must) and launches
// the instantiated graph; later calls replay it. Kernels read the step index from the
// device control block, so one graph serves every chunk that starts at a multiple of G.
static int launch_graph_chunk(galois_engine *e, int32_t G)
{
    if (e->graph && e->graph_steps == G) {
        ENG_CUDA(e, cudaGraphLaunch(e->graph, e->stream));
        e->steps_enqueued += G;
        e->pending_check = is_check_step(e, e->steps_enqueued);
        return GALOIS_OK;
    }
    if (e->graph) {
        cudaGraphExecDestroy(e->graph);
        e->graph = nullptr;
    }
    if (int rc = exchange_join(e)) return rc;        // (no event from outside the capture)
    const int32_t s0 = e->steps_enqueued;
    const bool pend0 = e->pending_check;
    cudaGraph_t g = nullptr;
    bool ok = cudaStreamBeginCapture(e->stream, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
    int rc = GALOIS_OK;
    for (int32_t i = 0; ok && i < G && rc == GALOIS_OK; ++i) rc = enqueue_step(e);
    if (ok && rc == GALOIS_OK) rc = exchange_join(e);   // the exchange stream rejoins inside the graph
    if (ok) ok = cudaStreamEndCapture(e->stream, &g) == cudaSuccess && rc == GALOIS_OK;
    if (ok) ok = cudaGraphInstantiate(&e->graph, g, 0) == cudaSuccess;
    if (g) cudaGraphDestroy(g);
    if (!ok) {                                  // fall back to plain launches for good
        cudaGetLastError();
        e->graph = nullptr;
        e->graph_failed = true;
        e->poisoned = false;
        e->steps_enqueued = s0;
        e->pending_check = pend0;
        e->x_pending = false;
        for (int32_t i = 0; i < G; ++i)
            if (int r2 = enqueue_step(e)) return r2;
        return GALOIS_OK;
    }
    e->graph_steps = G;
    ENG_CUDA(e, cudaGraphLaunch(e->graph, e->stream));
    return GALOIS_OK;
}

// The reported best record (u*, t*, b*): this rank's own on one rank, the global one (over
// all ranks, k_gfinalize) with NCCL.
struct Record {
    int32_t u, t;
    int64_t b;
};
static Record record_of(const galois_engine *e, const Ctrl &h)
{
    if (e->use_comm) return Record{h.g_u, h.g_t, h.g_b};
    return Record{h.best_u, h.best_t, h.best_b};
}

static int read_ctrl(galois_engine *e, Ctrl *out)
{
    if (int rc = exchange_join(e)) return rc;
    ENG_CUDA(e, cudaMemcpyAsync(&e->h_ctrl[0], e->ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, e->stream));
    ENG_CUDA(e, cudaStreamSynchronize(e->stream));
    *out = e->h_ctrl[0];
    if (out->nonfinite) return poison(e, GALOIS_E_NONFINITE, "an iterate became NaN/Inf");
    return GALOIS_OK;
}

// Run the pending check (if any) and read the control block: every result read goes
// through here so the last rounding is always checked before it is reported.
static int settle(galois_engine *e, Ctrl *out)
{
    if (int rc = flush_check(e)) return rc;
    return read_ctrl(e, out);
}

static int lanes_enqueue(galois_engine *e, int32_t max_steps);
static int lanes_refresh(galois_engine *e);

extern "C" int galois_engine_step(galois_engine *e)
{
    ENGINE_ENTRY(e);
    if (int rc = prepare(e)) return rc;
    if (!e->lane.empty()) {
        if (int rc = lanes_refresh(e)) return rc;
        if (e->agg.sat) return GALOIS_SAT;
        if (e->steps_enqueued >= e->T) return GALOIS_BUDGET;
        if (int rc = lanes_enqueue(e, 1)) return rc;
        if (int rc = lanes_refresh(e)) return rc;
        return e->agg.sat ? GALOIS_SAT : GALOIS_OK;
    }
    WHOLE_SLICE_ONLY(e);
    Ctrl h;
    if (int rc = read_ctrl(e, &h)) return rc;
    if (h.stopped) return GALOIS_SAT;
    if (e->steps_enqueued >= e->T) return GALOIS_BUDGET;
    if (int rc = enqueue_step(e)) return rc;
    if (int rc = settle(e, &h)) return rc;
    return h.stopped ? GALOIS_SAT : GALOIS_OK;
}

extern "C" int galois_engine_enqueue(galois_engine *e, int32_t max_steps)
{
    ENGINE_ENTRY(e);
    if (int rc = prepare(e)) return rc;
    if (!e->lane.empty()) {
        if (e->steps_enqueued >= e->T) return GALOIS_BUDGET;
        return lanes_enqueue(e, max_steps);
    }
    WHOLE_SLICE_ONLY(e);
    if (e->steps_enqueued >= e->T) return GALOIS_BUDGET;
    for (int32_t i = 0; i < max_steps && e->steps_enqueued < e->T; ++i)
        if (int rc = enqueue_step(e)) return rc;
    return GALOIS_OK;
}

static int run_windows(galois_engine *e);
static int run_lanes(galois_engine *e);

// Small instances: the remaining steps of run() as ONE launch of k_small_run (state in
// shared memory, one CTA per 32 members; update_kernels.cu). Bypassed while profiling (its
// per-kernel records need the per-step kernels), in debug mode and with NCCL.
static bool small_run_ok(const galois_engine *e)
{
    return e->small_gs && e->mode == GALOIS_MODE_ST && !e->use_comm && e->windows == 1 && e->lane.empty() &&
           !e->debug && !e->profiling && e->graphs_mode != 1 && e->steps_enqueued < e->T;
}

static int run_steps(galois_engine *e);

// CUDA graphs of G-step chunks: forced on / off by galois_engine_set_graphs, else used when
// the capture + instantiation (~ms) is amortised over many chunks (short time-to-SAT runs
// launch directly)
static bool use_graphs(const galois_engine *e, int32_t left, int32_t G)
{
    if (e->graphs_mode != 0) return e->graphs_mode > 0;
    return left >= 32 * G;
}

static int run_small(galois_engine *e)
{
    Ctrl h;
    const StepParams p = e->params();     // (a stopped engine: the kernel returns at once)
    const cudaError_t le = launch::small_run(e->cnf->view(), p, e->T, e->K, e->pending_check, e->z, e->m, e->v, e->X,
                                             e->R, e->unsat_last, e->lam, e->small_gs, e->small_recs, e->small_snap,
                                             e->best_bits, e->ctrl, e->stream);
    if (le == cudaErrorCooperativeLaunchTooLarge) {   // not all CTAs fit at once: per-step path
        cudaGetLastError();
        e->small_gs = nullptr;
        return run_steps(e);
    }
    ENG_CUDA(e, le);
    e->steps_enqueued = e->T;
    e->pending_check = false;
    if (int rc = read_ctrl(e, &h)) return rc;
    return h.stopped ? GALOIS_SAT : GALOIS_BUDGET;
}

// Steps of the resident members until SAT or e->T (see galois_engine_run).
static int run_steps(galois_engine *e)
{
    if (small_run_ok(e)) return run_small(e);
    // chunks of G steps (G even and a multiple of K, so every chunk that starts at a
    // multiple of G has the same kernel sequence and Lambda parity): replayed as one CUDA
    // graph; the stop flag of chunk i-1 is polled while chunk i is queued
    const int32_t KK = e->K % 2 == 0 ? e->K : 2 * e->K;
    const int32_t G = KK * std::max<int32_t>(1, 8 / KK);
    // graphs only pay off when the capture + instantiation (~ms) is amortised over many
    // chunks; short runs (time-to-SAT) launch directly
    const bool graphs = !e->profiling && e->stream != nullptr && e->mode == GALOIS_MODE_ST && !e->graph_failed &&
                        use_graphs(e, e->T - e->steps_enqueued, G);
    int iter = 0;
    while (e->steps_enqueued < e->T) {
        const int32_t s0 = e->steps_enqueued;
        if (graphs && s0 % G == 0 && s0 + G < e->T) {
            if (int rc = launch_graph_chunk(e, G)) return rc;
        } else {
            const int32_t end = std::min<int32_t>(e->T, (s0 / G + 1) * G);
            while (e->steps_enqueued < end)
                if (int rc = enqueue_step(e)) return rc;
        }
        if (int rc = exchange_join(e)) return rc;   // every rank polls the same global decision
        Ctrl *slot = &e->h_ctrl[iter & 1];
        ENG_CUDA(e, cudaMemcpyAsync(slot, e->ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, e->stream));
        ENG_CUDA(e, cudaEventRecord(e->poll_ev[iter & 1], e->stream));
        if (iter >= 1) {
            ENG_CUDA(e, cudaEventSynchronize(e->poll_ev[(iter - 1) & 1]));
            if (e->h_ctrl[(iter - 1) & 1].stopped) break;
        }
        ++iter;
    }
    Ctrl h;
    if (int rc = settle(e, &h)) return rc;
    return h.stopped ? GALOIS_SAT : GALOIS_BUDGET;
}

extern "C" int galois_engine_run(galois_engine *e)
{
    ENGINE_ENTRY(e);
    if (int rc = prepare(e)) return rc;
    if (!e->lane.empty()) return run_lanes(e);
    return e->windows > 1 ? run_windows(e) : run_steps(e);
}

// f4: put window w of the local slice into the resident buffers and initialise it at t = 0
// (the same init, RNG counters and best record a full-batch engine gives those members).
static int reseat(galois_engine *e, int32_t w)
{
    e->b0 = e->slice_b0 + (int64_t)w * e->sub;
    e->b_loc = (int32_t)std::max<int64_t>(0, std::min<int64_t>(e->sub, e->slice_loc - (int64_t)w * e->sub));
    if (e->graph) {                     // captured kernels carry b0 / b_loc in their parameters
        ENG_CUDA(e, cudaGraphExecDestroy(e->graph));
        e->graph = nullptr;
    }
    ENG_CUDA(e, cudaStreamSynchronize(e->stream));
    Ctrl h{};
    h.best_u = h.g_u = INT32_MAX;
    h.best_t = h.g_t = -1;
    h.best_b = h.g_b = -1;
    e->h_ctrl[0] = h;
    ENG_CUDA(e, cudaMemcpyAsync(e->ctrl, &e->h_ctrl[0], sizeof(Ctrl), cudaMemcpyHostToDevice, e->stream));
    ENG_CUDA(e, cudaMemsetAsync(e->unsat, 0, sizeof(int32_t) * (size_t)e->b_pad, e->stream));
    ENG_CUDA(e, cudaMemsetAsync(e->unsat_last, 0, sizeof(int32_t) * (size_t)e->b_pad, e->stream));
    ENG_CUDA(e, cudaMemsetAsync(e->best_bits, 0, (size_t)e->cnf->n, e->stream));
    if (e->lam) ENG_CUDA(e, cudaMemsetAsync(e->lam, 0, 2 * sizeof(int32_t) * (size_t)e->b_pad, e->stream));
    e->steps_enqueued = 0;
    const StepParams p = e->params();
    e->timed(5, [&] { launch::init(p, e->z, e->m, e->v, e->X, e->R, e->stream); });
    ENG_CUDA(e, cudaGetLastError());
    ENG_CUDA(e, cudaStreamSynchronize(e->stream));   // h_ctrl[0] is reused by the polls
    e->pending_check = true;
    return GALOIS_OK;
}

// f4: every window runs from t = 0 (after a SAT at t*, at most t* steps); the best is the
// lexicographic (u, t, b) minimum over the windows' records, the full-batch result.
static int run_windows(galois_engine *e)
{
    if (e->agg.ran) return e->agg.sat ? GALOIS_SAT : GALOIS_BUDGET;
    const int32_t T = e->T;
    e->agg_bits.assign((size_t)e->cnf->n, 0);
    e->agg_counts.assign((size_t)e->slice_loc, 0);
    for (int32_t w = 0; w < e->windows; ++w) {
        if (w > 0)
            if (int rc = reseat(e, w)) return rc;
        e->T = e->agg.sat ? e->agg.t : T;
        const int rc = run_steps(e);
        e->T = T;
        if (rc != GALOIS_SAT && rc != GALOIS_BUDGET) return rc;
        Ctrl h;
        if (int r2 = read_ctrl(e, &h)) return r2;
        const galois_engine::Agg &a = e->agg;
        const Record rec = record_of(e, h);
        const bool better = rec.b >= 0 && (rec.u != a.u ? rec.u < a.u : rec.t != a.t ? rec.t < a.t : rec.b < a.b);
        if (better) {
            if (e->use_comm) {           // every rank takes the same decision (global record)
                std::string why;
                if (!e->comm.broadcast_bytes(e->best_bits, (size_t)e->cnf->n, (int)(rec.b / e->b_per), e->stream, &why))
                    return poison(e, GALOIS_E_NCCL, why);
            }
            ENG_CUDA(e, cudaMemcpyAsync(e->agg_bits.data(), e->best_bits, (size_t)e->cnf->n, cudaMemcpyDeviceToHost,
                                        e->stream));

            e->agg.u = rec.u;
            e->agg.t = rec.t;
            e->agg.b = rec.b;
        }
        if (e->b_loc > 0) {
            ENG_CUDA(e, cudaMemcpyAsync(e->agg_counts.data() + (size_t)w * e->sub, e->unsat_last,
                                        sizeof(int32_t) * (size_t)e->b_loc, cudaMemcpyDeviceToHost, e->stream));
            // theta_sel candidates of this window (f1): keep the iterate of a new min / max
            if (!e->sel_z) {
                ENG_CUDA(e, cudaMallocAsync((void **)&e->sel_z, 2 * (size_t)e->cnf->n * 4, e->stream));
                ENG_CUDA(e, cudaMallocAsync((void **)&e->sel_dkey, 2 * sizeof(unsigned long long), e->stream));
            }
            for (int r = 0; r < 2; ++r) launch::select_member(e->unsat_last, e->b_loc, e->b0, r, e->sel_dkey + r, e->stream);
            unsigned long long k[2];
            ENG_CUDA(e, cudaMemcpyAsync(k, e->sel_dkey, sizeof(k), cudaMemcpyDeviceToHost, e->stream));
            ENG_CUDA(e, cudaStreamSynchronize(e->stream));
            for (int r = 0; r < 2; ++r)
                if (k[r] < e->sel_key[r]) {
                    e->sel_key[r] = k[r];
                    launch::gather_z(e->z, e->cnf->n, e->b_pad, (int32_t)((int64_t)(k[r] & 0xFFFFFFFFull) - e->b0),
                                     e->sel_z + (size_t)r * e->cnf->n, e->stream);
                }
        }
        ENG_CUDA(e, cudaStreamSynchronize(e->stream));
        e->agg.steps = std::max(e->agg.steps, (e->use_comm && h.stopped) ? rec.t : h.t);
        if (h.stopped) e->agg.sat = true;
    }
    e->agg.ran = true;
    return e->agg.sat ? GALOIS_SAT : GALOIS_BUDGET;
}

// ------------------------------------------------------------------------- lanes
// The lanes' streams wait for the work queued so far on the engine's stream (fork); the
// engine's stream waits for everything queued on the lanes (join).
static int lanes_fork(galois_engine *e)
{
    ENG_CUDA(e, cudaEventRecord(e->fork_ev, e->stream));
    for (galois_engine *l : e->lane) ENG_CUDA(e, cudaStreamWaitEvent(l->stream, e->fork_ev, 0));
    return GALOIS_OK;
}

static int lanes_join(galois_engine *e)
{
    for (size_t i = 0; i < e->lane.size(); ++i) {
        ENG_CUDA(e, cudaEventRecord(e->join_ev[i], e->lane[i]->stream));
        ENG_CUDA(e, cudaStreamWaitEvent(e->stream, e->join_ev[i], 0));
    }
    return GALOIS_OK;
}

static int lane_fail(galois_engine *e, int rc)
{
    e->poisoned = true;
    return rc;
}

// Up to max_steps steps on every lane, interleaved step by step across the lanes.
static int lanes_enqueue(galois_engine *e, int32_t max_steps)
{
    if (int rc = lanes_fork(e)) return rc;
    for (int32_t i = 0; i < max_steps; ++i)
        for (galois_engine *l : e->lane)
            if (l->steps_enqueued < l->T)
                if (int rc = enqueue_step(l)) return lane_fail(e, rc);
    if (int rc = lanes_join(e)) return rc;
    int32_t s = 0;
    for (galois_engine *l : e->lane) s = std::max(s, l->steps_enqueued);
    e->steps_enqueued = s;
    e->agg.ran = false;                   // the aggregate is formed again on the next query
    return GALOIS_OK;
}

// Best record, last-check counts and theta_sel candidates over the lanes, exactly as
// run_windows() forms them over windows: the best is the lexicographic (u, t, b) minimum of
// the lanes' records, which is the undivided engine's record (a lane that stops at its
// first SAT t* has run every step <= t*; records of steps after another lane's t* can
// never precede it).
static int lanes_refresh(galois_engine *e)
{
    if (e->lane.empty() || e->agg.ran) return GALOIS_OK;
    const int32_t n = e->cnf->n;
    galois_engine::Agg a;
    e->agg_bits.assign((size_t)n, 0);
    e->agg_counts.assign((size_t)e->slice_loc, 0);
    e->sel_key[0] = e->sel_key[1] = ~0ull;
    if (!e->sel_z) {
        ENG_CUDA(e, cudaMallocAsync((void **)&e->sel_z, 2 * (size_t)n * 4, e->stream));
        ENG_CUDA(e, cudaMallocAsync((void **)&e->sel_dkey, 2 * sizeof(unsigned long long), e->stream));
        ENG_CUDA(e, cudaStreamSynchronize(e->stream));
    }
    for (size_t i = 0; i < e->lane.size(); ++i) {
        galois_engine *l = e->lane[i];
        Ctrl h;
        if (int rc = settle(l, &h)) return lane_fail(e, rc);
        const bool better = h.best_b >= 0 &&
                            (h.best_u != a.u ? h.best_u < a.u : h.best_t != a.t ? h.best_t < a.t : h.best_b < a.b);
        if (better) {
            ENG_CUDA(e, cudaMemcpyAsync(e->agg_bits.data(), l->best_bits, (size_t)n, cudaMemcpyDeviceToHost, l->stream));
            a.u = h.best_u;
            a.t = h.best_t;
            a.b = h.best_b;
        }
        if (l->b_loc > 0) {
            ENG_CUDA(e, cudaMemcpyAsync(e->agg_counts.data() + (size_t)i * e->lane_size, l->unsat_last,
                                        sizeof(int32_t) * (size_t)l->b_loc, cudaMemcpyDeviceToHost, l->stream));
            for (int r = 0; r < 2; ++r) launch::select_member(l->unsat_last, l->b_loc, l->b0, r, e->sel_dkey + r, l->stream);
            unsigned long long k[2];
            ENG_CUDA(e, cudaMemcpyAsync(k, e->sel_dkey, sizeof(k), cudaMemcpyDeviceToHost, l->stream));
            ENG_CUDA(e, cudaStreamSynchronize(l->stream));
            for (int r = 0; r < 2; ++r)
                if (k[r] < e->sel_key[r]) {
                    e->sel_key[r] = k[r];
                    launch::gather_z(l->z, n, l->b_pad, (int32_t)((int64_t)(k[r] & 0xFFFFFFFFull) - l->b0),
                                     e->sel_z + (size_t)r * n, l->stream);
                }
        }
        ENG_CUDA(e, cudaStreamSynchronize(l->stream));
        a.steps = std::max(a.steps, h.t);
        if (h.stopped) a.sat = true;
    }
    a.ran = true;
    e->agg = a;
    return GALOIS_OK;
}

// run() on lanes: every lane runs run_steps()' chunks (CUDA graphs of G steps) in lockstep
// with the others; the stop flags are polled one chunk behind and a stop in any lane ends
// the run of all (they have all completed at least the steps of the deciding check).
static int run_lanes(galois_engine *e)
{
    const int32_t KK = e->K % 2 == 0 ? e->K : 2 * e->K;
    const int32_t G = KK * std::max<int32_t>(1, 8 / KK);
    if (int rc = lanes_refresh(e)) return rc;
    if (e->agg.sat) return GALOIS_SAT;
    if (int rc = lanes_fork(e)) return rc;
    const size_t NL = e->lane.size();
    std::vector<int> polled(NL, -1);
    bool stop = false;
    for (int iter = 0; !stop; ++iter) {
        bool any = false;
        for (size_t i = 0; i < NL; ++i) {
            galois_engine *l = e->lane[i];
            if (l->steps_enqueued >= l->T) continue;
            const int32_t s0 = l->steps_enqueued;
            const bool graphs = !l->profiling && !l->graph_failed && use_graphs(l, l->T - s0, G);
            if (graphs && s0 % G == 0 && s0 + G < l->T) {
                if (int rc = launch_graph_chunk(l, G)) return lane_fail(e, rc);
            } else {
                const int32_t end = std::min<int32_t>(l->T, (s0 / G + 1) * G);
                while (l->steps_enqueued < end)
                    if (int rc = enqueue_step(l)) return lane_fail(e, rc);
            }
            Ctrl *slot = &l->h_ctrl[iter & 1];
            ENG_CUDA(e, cudaMemcpyAsync(slot, l->ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, l->stream));
            ENG_CUDA(e, cudaEventRecord(l->poll_ev[iter & 1], l->stream));
            polled[i] = iter;
            any = true;
        }
        if (!any) break;
        for (size_t i = 0; i < NL && iter >= 1; ++i) {
            galois_engine *l = e->lane[i];
            if (polled[i] < iter - 1) continue;
            const int j = polled[i] == iter ? (iter - 1) & 1 : polled[i] & 1;
            ENG_CUDA(e, cudaEventSynchronize(l->poll_ev[j]));
            if (l->h_ctrl[j].stopped) stop = true;
        }
    }
    if (int rc = lanes_join(e)) return rc;
    int32_t s = 0;
    for (galois_engine *l : e->lane) s = std::max(s, l->steps_enqueued);
    e->steps_enqueued = s;
    e->agg.ran = false;
    if (int rc = lanes_refresh(e)) return rc;
    return e->agg.sat ? GALOIS_SAT : GALOIS_BUDGET;
}

extern "C" int galois_engine_info(galois_engine *e, int64_t *local_batch, int64_t *first_global_b,
                                  int32_t *steps_done, int32_t *stopped)
{
    ENGINE_ENTRY(e);
    if (int rc = prepare(e)) return rc;
    if (aggregated(e)) {
        if (int rc = lanes_refresh(e)) return rc;
        if (local_batch) *local_batch = e->slice_loc;
        if (first_global_b) *first_global_b = e->slice_b0;
        if (steps_done) *steps_done = e->agg.sat ? e->agg.t : e->agg.steps;   // what the full batch did
        if (stopped) *stopped = e->agg.sat;
        return GALOIS_OK;
    }
    Ctrl h;
    if (int rc = settle(e, &h)) return rc;
    if (local_batch) *local_batch = e->b_loc;
    if (first_global_b) *first_global_b = e->b0;
    // with NCCL a rank may have run one update past the deciding check (exchange_join)
    if (steps_done) *steps_done = (e->use_comm && h.stopped) ? record_of(e, h).t : h.t;
    if (stopped) *stopped = h.stopped;
    return GALOIS_OK;
}

extern "C" int galois_best_assignment(galois_engine *e, uint8_t *values, int32_t *unsat, int64_t *global_b,
                                      int32_t *step)
{
    ENGINE_ENTRY(e);
    if (int rc = prepare(e)) return rc;
    if (aggregated(e)) {
        if (int rc = lanes_refresh(e)) return rc;
        if (values && e->agg.ran) memcpy(values, e->agg_bits.data(), (size_t)e->cnf->n);
        else if (values) memset(values, 0, (size_t)e->cnf->n);
        if (unsat) *unsat = e->agg.u;
        if (global_b) *global_b = e->agg.b;
        if (step) *step = e->agg.t;
        return GALOIS_OK;
    }
    Ctrl h;
    if (!e->use_comm) {                   // one round trip: the control block and the bits together
        if (int rc = flush_check(e)) return rc;
        ENG_CUDA(e, cudaMemcpyAsync(&e->h_ctrl[0], e->ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, e->stream));
        if (values)
            ENG_CUDA(e, cudaMemcpyAsync(values, e->best_bits, (size_t)e->cnf->n, cudaMemcpyDeviceToHost, e->stream));
        ENG_CUDA(e, cudaStreamSynchronize(e->stream));
        h = e->h_ctrl[0];
        if (h.nonfinite) return poison(e, GALOIS_E_NONFINITE, "an iterate became NaN/Inf");
    } else {
        // the owner's own record is the global winner (a rank owns the global record only
        // through a strictly smaller local count, so its best_bits were extracted at that
        // check): broadcast them from there
        if (int rc = settle(e, &h)) return rc;
        if (h.g_b >= 0) {
            const int root = (int)(h.g_b / e->b_per);
            std::string why;
            if (!e->comm.broadcast_bytes(e->best_bits, (size_t)e->cnf->n, root, e->stream, &why))
                return poison(e, GALOIS_E_NCCL, why);
        }
        if (values)
            ENG_CUDA(e, cudaMemcpyAsync(values, e->best_bits, (size_t)e->cnf->n, cudaMemcpyDeviceToHost, e->stream));
        ENG_CUDA(e, cudaStreamSynchronize(e->stream));
    }
    const Record rec = record_of(e, h);
    if (unsat) *unsat = rec.u;
    if (global_b) *global_b = rec.b;
    if (step) *step = rec.t;
    return GALOIS_OK;
}

extern "C" int galois_unsat_counts(galois_engine *e, int32_t *counts, int64_t *first_global_b)
{
    ENGINE_ENTRY(e);
    if (int rc = prepare(e)) return rc;
    if (aggregated(e)) {
        if (int rc = lanes_refresh(e)) return rc;
        if (counts && e->agg.ran) memcpy(counts, e->agg_counts.data(), sizeof(int32_t) * (size_t)e->slice_loc);
        else if (counts) memset(counts, 0, sizeof(int32_t) * (size_t)e->slice_loc);
        if (first_global_b) *first_global_b = e->slice_b0;
        return GALOIS_OK;
    }
    Ctrl h;
    if (int rc = settle(e, &h)) return rc;
    if (counts && e->b_loc > 0)
        ENG_CUDA(e, cudaMemcpyAsync(counts, e->unsat_last, sizeof(int32_t) * (size_t)e->b_loc,
                                    cudaMemcpyDeviceToHost, e->stream));
    ENG_CUDA(e, cudaStreamSynchronize(e->stream));
    if (first_global_b) *first_global_b = e->b0;
    return GALOIS_OK;
}

// [n][b_pad] device -> [b_loc][n] host
template <typename T>
static int copy_transposed_out(galois_engine *e, const T *dev, T *host)
{
    const int32_t n = e->cnf->n;
    std::vector<T> tmp((size_t)n * e->b_pad);
    ENG_CUDA(e, cudaMemcpyAsync(tmp.data(), dev, tmp.size() * sizeof(T), cudaMemcpyDeviceToHost, e->stream));
    ENG_CUDA(e, cudaStreamSynchronize(e->stream));
    for (int32_t b = 0; b < e->b_loc; ++b)
        for (int32_t v = 0; v < n; ++v) host[(size_t)b * n + v] = tmp[(size_t)v * e->b_pad + b];
    return GALOIS_OK;
}

// ----------------------------------------------------------- selection (f1, f3)
// Scratch for the selection calls: temporary stream-ordered allocations (not hot path).
template <typename T>
static int tmp_alloc(galois_engine *e, T **p, size_t count)
{
    ENG_CUDA(e, cudaMallocAsync((void **)p, std::max<size_t>(count, 1) * sizeof(T), e->stream));
    return GALOIS_OK;
}

extern "C" int galois_select_member(galois_engine *e, int32_t rule, int64_t *global_b, int32_t *unsat, float *z)
{
    ENGINE_ENTRY(e);
    if (rule != 0 && rule != 1) return fail(GALOIS_E_ARG, "rule must be 0 (min loss) or 1 (max loss)");
    if (int rc = prepare(e)) return rc;
    if (aggregated(e)) {                  // sub-batched: tracked over the windows by run(); lanes: refreshed
        if (int rc = lanes_refresh(e)) return rc;
        if (!e->agg.ran || e->sel_key[rule] == ~0ull)
            return fail(GALOIS_E_STATE, "sub-batched engine: call run() first (this rank has members)");
        const unsigned long long key = e->sel_key[rule];
        const uint32_t u = (uint32_t)(key >> 32);
        if (global_b) *global_b = (int64_t)(key & 0xFFFFFFFFull);
        if (unsat) *unsat = (int32_t)(rule ? ~u : u);
        if (z) {
            ENG_CUDA(e, cudaMemcpyAsync(z, e->sel_z + (size_t)rule * e->cnf->n, (size_t)e->cnf->n * 4,
                                        cudaMemcpyDeviceToHost, e->stream));
            ENG_CUDA(e, cudaStreamSynchronize(e->stream));
        }
        return GALOIS_OK;
    }
    Ctrl h;
    if (int rc = settle(e, &h)) return rc;
    if (e->b_loc == 0) return fail(GALOIS_E_STATE, "this rank has no members");
    unsigned long long *d_key = nullptr;
    if (int rc = tmp_alloc(e, &d_key, 1)) return rc;
    launch::select_member(e->unsat_last, e->b_loc, e->b0, rule, d_key, e->stream);
    unsigned long long key = 0;
    ENG_CUDA(e, cudaMemcpyAsync(&key, d_key, 8, cudaMemcpyDeviceToHost, e->stream));
    ENG_CUDA(e, cudaFreeAsync(d_key, e->stream));
    ENG_CUDA(e, cudaStreamSynchronize(e->stream));
    const int64_t b = (int64_t)(key & 0xFFFFFFFFull);
    const uint32_t u = (uint32_t)(key >> 32);
    if (global_b) *global_b = b;
    if (unsat) *unsat = (int32_t)(rule ? ~u : u);
    if (z) {
        float *d_z = nullptr;
        if (int rc = tmp_alloc(e, &d_z, (size_t)e->cnf->n)) return rc;
        launch::gather_z(e->z, e->cnf->n, e->b_pad, (int32_t)(b - e->b0), d_z, e->stream);
        ENG_CUDA(e, cudaMemcpyAsync(z, d_z, (size_t)e->cnf->n * 4, cudaMemcpyDeviceToHost, e->stream));
        ENG_CUDA(e, cudaFreeAsync(d_z, e->stream));
        ENG_CUDA(e, cudaStreamSynchronize(e->stream));
    }
    return GALOIS_OK;
}

static int local_member(galois_engine *e, int64_t global_b, int32_t *lb)
{
    if (global_b < e->b0 || global_b >= e->b0 + e->b_loc)
        return fail(GALOIS_E_ARG, "member is not local to this rank");
    *lb = (int32_t)(global_b - e->b0);
    return GALOIS_OK;
}

// The iterate of member global_b into d_z: a resident member, or on a sub-batched engine
// the retained winner of run() (theta_sel; other members' windows are gone).
static int member_z(galois_engine *e, int64_t global_b, float *d_z)
{
    for (galois_engine *l : e->lane)       // lanes: every member stays resident in its lane
        if (global_b >= l->b0 && global_b < l->b0 + l->b_loc) {
            if (int rc = lanes_refresh(e)) return rc;    // the lane's pending check is settled
            launch::gather_z(l->z, e->cnf->n, l->b_pad, (int32_t)(global_b - l->b0), d_z, l->stream);
            ENG_CUDA(e, cudaStreamSynchronize(l->stream));
            return GALOIS_OK;
        }
    if (!e->lane.empty()) return fail(GALOIS_E_ARG, "member is not local to this rank");
    if (e->windows > 1) {
        for (int r = 0; r < 2 && e->agg.ran; ++r)
            if (e->sel_key[r] != ~0ull && (int64_t)(e->sel_key[r] & 0xFFFFFFFFull) == global_b) {
                ENG_CUDA(e, cudaMemcpyAsync(d_z, e->sel_z + (size_t)r * e->cnf->n, (size_t)e->cnf->n * 4,
                                            cudaMemcpyDeviceToDevice, e->stream));
                return GALOIS_OK;
            }
        return fail(GALOIS_E_STATE, "sub-batched engine: only the theta_sel members (after run) are retained");
    }
    int32_t lb = 0;
    if (int rc = local_member(e, global_b, &lb)) return rc;
    launch::gather_z(e->z, e->cnf->n, e->b_pad, lb, d_z, e->stream);
    return GALOIS_OK;
}

extern "C" int galois_candidate_pool(galois_engine *e, int64_t global_b, int32_t N, double rho, uint64_t pool_seed,
                                     uint8_t *values, float *confidence, int32_t *units, int32_t *S_out)
{
    ENGINE_ENTRY(e);
    if (N < 1 || !(rho > 0.0 && rho <= 1.0)) return fail(GALOIS_E_ARG, "need N >= 1 and 0 < rho <= 1");
    if (int rc = prepare(e)) return rc;
    const int32_t n = e->cnf->n, n_sel = e->cnf->n_orig;
    const int32_t S = units_per_candidate(e->cnf, rho);
    if (S > kMaxUnits) return fail(GALOIS_E_ARG, "|S| exceeds 2^20 units per candidate");
    const bool full = values || confidence;          // the [N][n] arrays go to the host
    if (full && (int64_t)N * n > (int64_t(1) << 31)) return fail(GALOIS_E_ARG, "N * n too large");
    if (S_out) *S_out = S;
    // Units only: the pool is drawn over the original variables alone (the units come from
    // them; counters are per variable, so the values are those of the full draw) in
    // groups of candidates whose scratch stays within ~1.25 GB.
    const int32_t row = full ? n : n_sel;
    const int32_t grp = full ? N : (int32_t)std::max<int64_t>(1, std::min<int64_t>(N, (int64_t(1) << 28) / row));
    int32_t gstride = 1;                             // bitonic width >= S for the global-memory sort
    while (gstride < S) gstride <<= 1;
    const bool gsort = S > launch::max_sorted();
    ENG_CUDA(e, cudaStreamSynchronize(e->stream));
    float *d_z = nullptr, *d_c = nullptr;
    uint8_t *d_x = nullptr;
    int32_t *d_u = nullptr;
    uint64_t *d_k = nullptr;
    auto release = [&]() {
        for (void *p : {(void *)d_z, (void *)d_c, (void *)d_x, (void *)d_u, (void *)d_k})
            if (p) cudaFreeAsync(p, e->stream);
    };
    if (int rc = tmp_alloc(e, &d_z, (size_t)n)) return rc;
    if (int rc = tmp_alloc(e, &d_c, (size_t)grp * row)) return release(), rc;
    if (int rc = tmp_alloc(e, &d_x, (size_t)grp * row)) return release(), rc;
    if (int rc = tmp_alloc(e, &d_u, (size_t)N * S)) return release(), rc;
    if (gsort && units)
        if (int rc = tmp_alloc(e, &d_k, (size_t)grp * gstride)) return release(), rc;
    if (int rc = member_z(e, global_b, d_z)) return release(), rc;
    for (int32_t k0 = 0; k0 < N; k0 += grp) {
        const int32_t g = std::min(grp, N - k0);
        launch::pool(d_z, row, k0, g, (float)(1.0 / e->tau), pool_seed, d_x, d_c, e->stream);
        if (units) launch::topk(d_x, d_c, row, n_sel, g, S, d_u + (size_t)k0 * S, d_k, gstride, e->stream);
    }
    ENG_CUDA(e, cudaGetLastError());
    if (values) ENG_CUDA(e, cudaMemcpyAsync(values, d_x, (size_t)N * n, cudaMemcpyDeviceToHost, e->stream));
    if (confidence) ENG_CUDA(e, cudaMemcpyAsync(confidence, d_c, (size_t)N * n * 4, cudaMemcpyDeviceToHost, e->stream));
    if (units) ENG_CUDA(e, cudaMemcpyAsync(units, d_u, (size_t)N * S * 4, cudaMemcpyDeviceToHost, e->stream));
    release();
    ENG_CUDA(e, cudaStreamSynchronize(e->stream));
    return GALOIS_OK;
}

extern "C" int galois_cube_variables(galois_engine *e, int64_t global_b, int32_t d, int32_t *vars)
{
    ENGINE_ENTRY(e);
    if (!vars) return fail(GALOIS_E_ARG, "vars is NULL");
    if (int rc = prepare(e)) return rc;
    const int32_t n = e->cnf->n, n_orig = e->cnf->n_orig;   // cubes over the original variables
    if (d < 1 || d > n_orig || d > launch::max_sorted()) return fail(GALOIS_E_ARG, "need 1 <= d <= min(n, 4096)");
    ENG_CUDA(e, cudaStreamSynchronize(e->stream));
    float *d_z = nullptr;
    int32_t *d_v = nullptr;
    if (int rc = tmp_alloc(e, &d_z, (size_t)n)) return rc;
    if (int rc = tmp_alloc(e, &d_v, (size_t)d)) return rc;
    if (int rc = member_z(e, global_b, d_z)) {
        cudaFreeAsync(d_z, e->stream);
        cudaFreeAsync(d_v, e->stream);
        return rc;
    }
    launch::lowconf(d_z, n_orig, d, d_v, e->stream);
    ENG_CUDA(e, cudaGetLastError());
    ENG_CUDA(e, cudaMemcpyAsync(vars, d_v, (size_t)d * 4, cudaMemcpyDeviceToHost, e->stream));
    ENG_CUDA(e, cudaFreeAsync(d_z, e->stream));
    ENG_CUDA(e, cudaFreeAsync(d_v, e->stream));
    ENG_CUDA(e, cudaStreamSynchronize(e->stream));
    return GALOIS_OK;
}

extern "C" int galois_engine_get_iterate(galois_engine *e, float *z, float *m, float *v, int32_t *t)
{
    ENGINE_ENTRY(e);
    if (int rc = prepare(e)) return rc;
    NO_WINDOWS(e);
    if (!e->lane.empty()) {
        const size_t n = (size_t)e->cnf->n;
        int32_t tmax = 0;
        const int rc = for_each_lane(e, [&](galois_engine *l, size_t off) {
            int32_t tl = 0;
            const int r = galois_engine_get_iterate(l, z ? z + off * n : nullptr, m ? m + off * n : nullptr,
                                                    v ? v + off * n : nullptr, &tl);
            tmax = std::max(tmax, tl);
            return r;
        });
        if (t) *t = tmax;
        return rc;
    }
    if (z) if (int rc = copy_transposed_out(e, e->z, z)) return rc;
    if (m) if (int rc = copy_transposed_out(e, e->m, m)) return rc;
    if (v) if (int rc = copy_transposed_out(e, e->v, v)) return rc;
    if (t) {
        Ctrl h;
        if (int rc = read_ctrl(e, &h)) return rc;
        *t = h.t;
    }
    return GALOIS_OK;
}

extern "C" int galois_engine_set_iterate(galois_engine *e, const float *z, const float *m, const float *v, int32_t t)
{
    ENGINE_ENTRY(e);
    if (!z || !m || !v) return fail(GALOIS_E_ARG, "z, m and v are required");
    if (t < 0 || t > e->T) return fail(GALOIS_E_ARG, "t must be in [0, steps]");
    if (int rc = prepare(e)) return rc;
    NO_WINDOWS(e);
    if (!e->lane.empty()) {
        const size_t n = (size_t)e->cnf->n;
        const int rc = for_each_lane(e, [&](galois_engine *l, size_t off) {
            return galois_engine_set_iterate(l, z + off * n, m + off * n, v + off * n, t);
        });
        if (rc) return rc;
        for (galois_engine *l : e->lane) l->steps_enqueued = t;
        e->steps_enqueued = t;
        e->agg.ran = false;
        return GALOIS_OK;
    }
    const int32_t n = e->cnf->n;
    const float *src[3] = {z, m, v};
    float *dst[3] = {e->z, e->m, e->v};
    std::vector<float> tmp((size_t)n * e->b_pad);
    ENG_CUDA(e, cudaStreamSynchronize(e->stream));
    for (int a = 0; a < 3; ++a) {
        ENG_CUDA(e, cudaMemcpy(tmp.data(), dst[a], tmp.size() * 4, cudaMemcpyDeviceToHost));  // keep padding
        for (int32_t b = 0; b < e->b_loc; ++b)
            for (int32_t x = 0; x < n; ++x) tmp[(size_t)x * e->b_pad + b] = src[a][(size_t)b * n + x];
        ENG_CUDA(e, cudaMemcpy(dst[a], tmp.data(), tmp.size() * 4, cudaMemcpyHostToDevice));
    }
    Ctrl h;
    if (int rc = read_ctrl(e, &h)) return rc;
    h.t = t;
    h.stopped = 0;
    h.nonfinite = 0;
    e->h_ctrl[0] = h;
    ENG_CUDA(e, cudaMemcpyAsync(e->ctrl, &e->h_ctrl[0], sizeof(Ctrl), cudaMemcpyHostToDevice, e->stream));
    launch::resample(e->params(), e->z, e->X, e->R, t + 1, e->stream);
    ENG_CUDA(e, cudaGetLastError());
    if (e->lam) ENG_CUDA(e, cudaMemsetAsync(e->lam, 0, 2 * sizeof(int32_t) * (size_t)e->b_pad, e->stream));
    ENG_CUDA(e, cudaMemsetAsync(e->unsat, 0, sizeof(int32_t) * (size_t)e->b_pad, e->stream));
    ENG_CUDA(e, cudaStreamSynchronize(e->stream));
    e->steps_enqueued = t;
    e->pending_check = false;            // the injected iterate is not a check point
    return GALOIS_OK;
}

// One member's state read in place on the device (column lb of the [n][b_pad] arrays), so
// full-size engines (C4: 4 GB per state array) can be compared member by member.
extern "C" int galois_engine_get_member(galois_engine *e, int64_t global_b, float *z, float *m, float *v,
                                        uint8_t *x_next, uint8_t *r, int32_t *G, float *g1, int32_t *t,
                                        int32_t *unsat, int32_t *check_t)
{
    ENGINE_ENTRY(e);
    if (int rc = prepare(e)) return rc;
    if (e->windows > 1) return fail(GALOIS_E_STATE, "not available on a sub-batched engine (run only)");
    galois_engine *x = e;
    for (galois_engine *l : e->lane)
        if (global_b >= l->b0 && global_b < l->b0 + l->b_loc) x = l;
    if (x == e && !e->lane.empty()) return fail(GALOIS_E_ARG, "member is not local to this rank");
    int32_t lb = 0;
    if (int rc = local_member(x, global_b, &lb)) return rc;
    if ((G || g1) && !x->debug) return fail(GALOIS_E_STATE, "G / g1 need set_debug(1) before the first step");
    if ((G || g1) && x->mode != GALOIS_MODE_ST) return fail(GALOIS_E_STATE, "G / g1 of one member: ST mode only");
    const int32_t n = x->cnf->n;
    ENG_CUDA(e, cudaStreamSynchronize(x->stream));
    char *d = nullptr;
    ENG_CUDA(e, cudaMallocAsync((void **)&d, (size_t)n * 22 + 256, x->stream));
    float *dz = (float *)d, *dm = dz + n, *dv = dm + n, *dg1 = dv + n;
    int32_t *dG = (int32_t *)(dg1 + n);
    uint8_t *dx = (uint8_t *)(dG + n), *dr = dx + n;
    const float *src[5] = {x->z, x->m, x->v, x->dbg_g1, (const float *)x->dbg_G};
    float *dst[5] = {dz, dm, dv, dg1, (float *)dG};
    void *host[5] = {z, m, v, g1, G};
    for (int a = 0; a < 5; ++a)
        if (host[a]) launch::gather_z(src[a], n, x->b_pad, lb, dst[a], x->stream);   // (a bit copy)
    if (x_next || r) launch::member_bits(x->X, n, x->W, lb, x_next ? dx : nullptr, r ? dr : nullptr, x->stream);
    for (int a = 0; a < 5; ++a)
        if (host[a]) ENG_CUDA(e, cudaMemcpyAsync(host[a], dst[a], (size_t)n * 4, cudaMemcpyDeviceToHost, x->stream));
    if (x_next) ENG_CUDA(e, cudaMemcpyAsync(x_next, dx, (size_t)n, cudaMemcpyDeviceToHost, x->stream));
    if (r) ENG_CUDA(e, cudaMemcpyAsync(r, dr, (size_t)n, cudaMemcpyDeviceToHost, x->stream));
    if (unsat) ENG_CUDA(e, cudaMemcpyAsync(unsat, x->unsat_last + lb, 4, cudaMemcpyDeviceToHost, x->stream));
    ENG_CUDA(e, cudaFreeAsync(d, x->stream));
    if (t || check_t) {
        if (int rc = exchange_join(x)) return rc;
        ENG_CUDA(e, cudaMemcpyAsync(&x->h_ctrl[0], x->ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, x->stream));
        ENG_CUDA(e, cudaStreamSynchronize(x->stream));
        if (t) *t = x->h_ctrl[0].t;
        if (check_t) *check_t = x->h_ctrl[0].last_check_t;
    }
    ENG_CUDA(e, cudaStreamSynchronize(x->stream));
    return GALOIS_OK;
}

extern "C" int galois_engine_get_grad(galois_engine *e, int32_t *G, float *g1)
{
    ENGINE_ENTRY(e);
    if (!e->debug) return fail(GALOIS_E_STATE, "get_grad needs set_debug(1) before the first step");
    if (int rc = prepare(e)) return rc;
    WHOLE_SLICE_ONLY(e);
    if (G) {
        if (e->mode == GALOIS_MODE_ST) {
            if (int rc = copy_transposed_out(e, e->dbg_G, G)) return rc;
        } else {
            std::vector<float> tmp((size_t)e->b_loc * e->cnf->n);
            if (int rc = copy_transposed_out(e, e->dbg_Gf, tmp.data())) return rc;
            for (size_t i = 0; i < tmp.size(); ++i) G[i] = (int32_t)lrintf(tmp[i]);
        }
    }
    if (g1) if (int rc = copy_transposed_out(e, e->dbg_g1, g1)) return rc;
    return GALOIS_OK;
}

extern "C" int galois_engine_get_loss(galois_engine *e, double *lambda)
{
    ENGINE_ENTRY(e);
    if (!lambda) return fail(GALOIS_E_ARG, "lambda is NULL");
    if (int rc = prepare(e)) return rc;
    NO_WINDOWS(e);
    if (!e->lane.empty())
        return for_each_lane(e, [&](galois_engine *l, size_t off) { return galois_engine_get_loss(l, lambda + off); });
    if (e->mode == GALOIS_MODE_ST) {
        // Lambda of the last completed step t lives in lam[t & 1] (see enqueue_step)
        Ctrl h;
        if (int rc = read_ctrl(e, &h)) return rc;
        std::vector<int32_t> tmp((size_t)e->b_pad);
        ENG_CUDA(e, cudaMemcpyAsync(tmp.data(), e->lam + (size_t)(h.t & 1) * e->b_pad, tmp.size() * 4,
                                    cudaMemcpyDeviceToHost, e->stream));
        ENG_CUDA(e, cudaStreamSynchronize(e->stream));
        for (int32_t b = 0; b < e->b_loc; ++b) lambda[b] = (double)tmp[b];   // exact: counts reach 2^24 on P:559's sizes
    } else {
        std::vector<float> tmp((size_t)e->b_loc);
        ENG_CUDA(e, cudaMemcpyAsync(tmp.data(), e->lam_f, (size_t)e->b_loc * 4, cudaMemcpyDeviceToHost, e->stream));
        ENG_CUDA(e, cudaStreamSynchronize(e->stream));
        for (int32_t b = 0; b < e->b_loc; ++b) lambda[b] = (double)tmp[b];
    }
    return GALOIS_OK;
}

extern "C" int galois_engine_get_bits(galois_engine *e, uint8_t *x_next, uint8_t *r)
{
    ENGINE_ENTRY(e);
    if (int rc = prepare(e)) return rc;
    NO_WINDOWS(e);
    if (!e->lane.empty()) {
        const size_t n = (size_t)e->cnf->n;
        return for_each_lane(e, [&](galois_engine *l, size_t off) {
            return galois_engine_get_bits(l, x_next ? x_next + off * n : nullptr, r ? r + off * n : nullptr);
        });
    }
    const int32_t n = e->cnf->n;
    std::vector<uint32_t> tmp((size_t)n * 2 * xr_pad(e->W));
    ENG_CUDA(e, cudaMemcpyAsync(tmp.data(), e->X, tmp.size() * 4, cudaMemcpyDeviceToHost, e->stream));
    ENG_CUDA(e, cudaStreamSynchronize(e->stream));
    uint8_t *outs[2] = {x_next, r};
    for (int a = 0; a < 2; ++a) {
        if (!outs[a]) continue;
        const uint32_t *base = tmp.data() + (size_t)xr_roff(e->W) * a;   // R = X + xr_roff(W) words
        for (int32_t b = 0; b < e->b_loc; ++b)
            for (int32_t v = 0; v < n; ++v)
                outs[a][(size_t)b * n + v] =   // member i of a word at bit 8 (i mod 4) + i / 4
                    (uint8_t)((base[xr_at(v, b >> 5, e->W)] >> (((b & 3) << 3) | ((b & 31) >> 2))) & 1u);
    }
    return GALOIS_OK;
}

extern "C" int galois_engine_kernel_times(galois_engine *e, double *ms, int64_t *launches)
{
    ENGINE_ENTRY(e);
    if (ms) std::fill(ms, ms + GALOIS_NUM_KERNEL_CLASSES, 0.0);
    if (launches) std::fill(launches, launches + GALOIS_NUM_KERNEL_CLASSES, 0);
    for (galois_engine *l : e->lane) {     // lanes: summed over the lanes (their launches overlap)
        double lm[GALOIS_NUM_KERNEL_CLASSES];
        int64_t lc[GALOIS_NUM_KERNEL_CLASSES];
        if (int rc = galois_engine_kernel_times(l, lm, lc)) return rc;
        for (int k = 0; k < GALOIS_NUM_KERNEL_CLASSES; ++k) {
            if (ms) ms[k] += lm[k];
            if (launches) launches[k] += lc[k];
        }
    }
    if (e->stream) ENG_CUDA(e, cudaStreamSynchronize(e->stream));
    for (auto &r : e->recs) {
        float t = 0.f;
        ENG_CUDA(e, cudaEventElapsedTime(&t, r.a, r.b));
        if (ms) ms[r.cls] += t;
        if (launches) launches[r.cls] += 1;
        e->ev_pool.push_back(r.a);
        e->ev_pool.push_back(r.b);
    }
    e->recs.clear();
    return GALOIS_OK;
}

extern "C" void galois_engine_free(galois_engine *e)
{
    if (!e) return;
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(e->device);
    if (e->stream) cudaStreamSynchronize(e->stream);
    for (galois_engine *l : e->lane) galois_engine_free(l);
    for (auto ev : e->join_ev) cudaEventDestroy(ev);
    if (e->fork_ev) cudaEventDestroy(e->fork_ev);
    e->comm.destroy(e->poisoned);
    if (e->xstream) stream_release(e->xstream);
    if (e->ev_chk) cudaEventDestroy(e->ev_chk);
    if (e->ev_x) cudaEventDestroy(e->ev_x);
    engine_free_buffers(e);
    for (auto &r : e->recs) {
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
    }
    for (auto ev : e->ev_pool) cudaEventDestroy(ev);
    for (auto ev : e->poll_ev)
        if (ev) cudaEventDestroy(ev);
    if (e->graph) cudaGraphExecDestroy(e->graph);
    if (e->own_stream && e->stream) stream_release(e->stream);
    cnf_release(e->cnf);
    cudaSetDevice(cur);
    delete e;
}

extern "C" const char *galois_last_error(void) { return g_last_error.c_str(); }
