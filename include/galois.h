/*
 * galois.h — C ABI of the B200-native GaloisSAT GPU stage (arxiv 2603.28796).
 *
 * The library runs the paper's differentiable SAT engine on one GPU per process:
 * every CNF clause is the polynomial C = 1 - prod_i (1 - s_i) of its literal values
 * (Eq.1-2); a batch of independent relaxed assignments (restarts or
 * Shannon cubes, Lemma 1) is sampled with Gumbel noise and a
 * straight-through argmax (Eq.3-4), scored by the MaxSAT loss
 * L = -sum_t C_t (Eq.5), updated by Adam (App. A), rounded and
 * checked exactly against the CNF. The best member (minimal unsat count)
 * is tracked on the device and, with several GPUs, min-reduced over NCCL.
 *
 * Conventions (all functions):
 *  - Status codes only (enum galois_status); no exception crosses the ABI. The message
 *    of the last failure on the calling thread is galois_last_error().
 *  - Input arrays are BORROWED for the duration of the call and copied; output arrays
 *    are caller-allocated HOST memory unless stated otherwise.
 *  - Handles are not thread-safe; distinct handles may be used concurrently.
 *  - An engine binds to the CUDA device current at galois_engine_create and uses a
 *    library-owned stream unless galois_engine_set_stream is called.
 *  - After a CUDA / NCCL error or a non-finite iterate the engine is poisoned: every
 *    later call on it returns GALOIS_E_STATE until it is freed.
 *  - Host layouts of per-member arrays are member-major: [local member][variable].
 *  - Member indices in outputs are GLOBAL: rank r owns members
 *    [r * b_per, min(B, (r+1) * b_per)) with b_per = roundup(ceil(B / world), 32).
 */
#ifndef GALOIS_H
#define GALOIS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct galois_cnf galois_cnf;       /* device-resident CSR + CSC of one CNF, refcounted */
typedef struct galois_engine galois_engine; /* one rank's slice of the batch                   */

enum galois_status {
    GALOIS_OK = 0,
    GALOIS_BUDGET = 1,           /* step budget spent, no satisfying member found            */
    GALOIS_SAT = 10,             /* the best member satisfies every clause (u* = 0)           */
    GALOIS_E_ARG = -1,           /* invalid argument (null pointer, bad size, bad hparam)     */
    GALOIS_E_VAR_RANGE = -2,     /* a literal is 0 or |lit| > num_vars                        */
    GALOIS_E_OFFSETS = -3,       /* offsets[0] != 0, decreasing offsets, or L >= 2^31         */
    GALOIS_E_EMPTY_CLAUSE = -4,  /* a clause has no literal: the CNF is trivially UNSAT       */
    GALOIS_E_OOM = -5,           /* device allocation failed                                   */
    GALOIS_E_CUDA = -6,          /* CUDA runtime error (incl. no device)                       */
    GALOIS_E_NCCL = -7,          /* NCCL unavailable or failed                                 */
    GALOIS_E_NONFINITE = -8,     /* an iterate became NaN/Inf                                  */
    GALOIS_E_STATE = -9          /* wrong call order, or handle poisoned by an earlier error   */
};

enum galois_mode { GALOIS_MODE_ST = 0, GALOIS_MODE_SOFT = 1 };
enum galois_optimizer { GALOIS_ADAM = 0, GALOIS_SGD = 1 };

/* ------------------------------------------------------------------------------ CNF */

/* Load a CNF given as clause-major CSR (a conjunction of clauses, each a
 * disjunction of literals): clause c holds literals[clause_offsets[c] ..
 * clause_offsets[c+1]-1], each a DIMACS signed 1-based variable (+v = x_v, -v = not x_v).
 *   num_vars       n >= 1
 *   num_clauses    m >= 0
 *   clause_offsets m+1 int64, host, borrowed; offsets[0] = 0, non-decreasing, L = offsets[m] < 2^31
 *   literals       L int32, host, borrowed; 1 <= |lit| <= n
 * Duplicate literals and tautologies are kept verbatim (per-slot polynomial semantics).
 * Builds on the device: the literal codes, the variable-major transpose (CSC, stable in
 * the slot order within (variable, sign)) and the hub table of high-degree variables.
 * Errors: E_ARG, E_OFFSETS, E_VAR_RANGE, E_EMPTY_CLAUSE (validated on the device),
 * E_OOM, E_CUDA. On error *out is NULL. */
int galois_cnf_load(int32_t num_vars, int64_t num_clauses, const int64_t *clause_offsets,
                    const int32_t *literals, galois_cnf **out);

/* Sizes of a loaded CNF (any pointer may be NULL). */
int galois_cnf_info(const galois_cnf *cnf, int32_t *num_vars, int64_t *num_clauses,
                    int64_t *num_slots, int32_t *max_width, int32_t *max_degree, int32_t *num_hubs);

/* Copy the device CSC back (test hook): var_off[2n+1] gives, for code 2v+neg, the range
 * [var_off[code], var_off[code+1]) of occ_slot[L] holding the slots of literal code in
 * ascending slot order. Any pointer may be NULL. */
int galois_cnf_get_csc(const galois_cnf *cnf, int32_t *code_off, int32_t *occ_slot);

/* Fixed-width normalisation on the device (§2.2 "Clause Normalization for Vectorization",
 * Eq.6-9; the paper uses k = 3, App. A): every clause longer than k
 * becomes the equisatisfiable chain (l_1 .. l_{k-1} f_1)(-f_1 l_k .. f_2)...(-f_q ... l_u)
 * with fresh auxiliaries f_j = variables n+1, n+2, ... in clause order; shorter clauses are
 * padded by repeating their last literal (Appendix B: (-x1 x3) -> (-x1 x3 x3)).
 * *out is a new CNF over n + *num_aux variables, every clause of width k; the first n
 * bits of any model of *out are a model of the input. 3 <= k <= 32. */
int galois_cnf_normalize(const galois_cnf *cnf, int32_t k, galois_cnf **out, int32_t *num_aux);

/* Copy the CSR back in DIMACS form (test hook): offsets m+1 int64, literals L int32. */
int galois_cnf_get_csr(const galois_cnf *cnf, int64_t *clause_offsets, int32_t *literals);

/* Variables of the CNF before normalisation (= num_vars unless made by galois_cnf_normalize,
 * whose auxiliaries f_j are variables n_orig+1 ..; P:214 excludes them from the candidate
 * literals, and cubes branch on original variables only). */
int galois_cnf_original_vars(const galois_cnf *cnf, int32_t *n_orig);

/* Drop the caller's reference (engines hold their own). NULL is a no-op. */
void galois_cnf_free(galois_cnf *cnf);

/* --------------------------------------------------------------------------- engine */

/* Create an engine for a global batch of B >= 1 independent members, a budget of
 * steps >= 0 optimiser steps ("epochs", one full-batch step each), learning
 * rate lr > 0 (paper 0.5) and RNG seed. Defaults: ST mode, tau = 1, Adam (0.9, 0.999,
 * 1e-8), check interval 1, no cubes, world = 1. Device memory is allocated and the
 * logits initialised lazily at the first step/run/get (so setters may follow create);
 * a local slice b_per >= 2^31 - 1024 members is rejected there (E_ARG). */
int galois_engine_create(const galois_cnf *cnf, int64_t batch, int32_t steps, double lr,
                         uint64_t seed, galois_engine **out);

/* One optimiser step t -> t+1 (sample, clause forward, straight-through gradient,
 * update, round, and the exact check if t+1 is a check point). Returns GALOIS_OK,
 * GALOIS_SAT once the best member satisfies the CNF (further steps are no-ops), or
 * GALOIS_BUDGET if the step budget is already spent. Synchronises the stream. */
int galois_engine_step(galois_engine *eng);

/* Run steps until SAT (GALOIS_SAT) or until the budget is spent (GALOIS_BUDGET). The
 * host polls an 8-byte device flag once per chunk of steps; kernels of steps enqueued
 * after the stop are no-ops, so the recorded best and step count are exact.
 * Small instances (32 members' z, m, v, bit planes and one E word per slot within 200 KB
 * of shared memory, ST mode, no NCCL / sub-batching / lanes / debug / profiling) run all
 * remaining steps in ONE kernel launch, one CTA per 32 members, with the same arithmetic
 * (bit-identical iterates, best record and counts; a grid barrier at each check stops
 * every CTA exactly where the per-step engine stops). Needs all W CTAs co-resident
 * (cooperative launch); otherwise the per-step path runs. */
int galois_engine_run(galois_engine *eng);

/* Like run, but enqueues at most max_steps further steps and does not synchronise the
 * stream (the caller times / synchronises, e.g. with events on the same stream).
 * Returns OK (or BUDGET if nothing was left to enqueue). */
int galois_engine_enqueue(galois_engine *eng, int32_t max_steps);

/* Best member over all check points so far, min over (unsat, step, global member)
 * lexicographically ("minimal clause loss"): its noise-free rounding (n bytes
 * 0/1, host; may be NULL), unsat count, global member index and step. With world > 1
 * this is collective (all ranks must call it; the winner's bits are broadcast). */
int galois_best_assignment(galois_engine *eng, uint8_t *values, int32_t *unsat,
                           int64_t *global_b, int32_t *step);

/* Exact unsat counts of the local members at the last check point (b_loc int32, host),
 * and the global index of the first local member (may be NULL). */
int galois_unsat_counts(galois_engine *eng, int32_t *counts, int64_t *first_global_b);

/* Local slice and progress: number of local members, first global member, steps done,
 * whether the engine stopped on SAT. Any pointer may be NULL. */
int galois_engine_info(galois_engine *eng, int64_t *local_batch, int64_t *first_global_b,
                       int32_t *steps_done, int32_t *stopped);

void galois_engine_free(galois_engine *eng);

/* Thread-local message of the last failure ("" if none). */
const char *galois_last_error(void);

/* ------------------------------------------- setters (before the first step, else E_STATE) */

/* 0 = straight-through (paper, Eq.4), 1 = fully soft forward (debug mode for
 * finite-difference checks; ~10x more memory traffic). */
int galois_engine_set_mode(galois_engine *eng, int32_t mode);

/* tau > 0 (Eq.3; paper 1.0), Adam beta1, beta2 in [0,1), eps > 0, optimizer
 * 0 = Adam (App. A), 1 = plain gradient step theta -= lr g. */
int galois_engine_set_hparams(galois_engine *eng, double tau, double beta1, double beta2, double eps,
                              int32_t optimizer);

/* Check (round + exact count + best update) at t = 0, every k >= 1 steps, and at the
 * last step of the budget. */
int galois_engine_set_check_interval(galois_engine *eng, int32_t k);

/* Cube pins (Lemma 1): d variables (1-based, distinct, 0 <= d <= 30); member b
 * fixes variable vars[r] to bit r of alpha = b mod 2^d (sorted ascending by variable
 * index). Pinned variables are frozen (no update) and forced in every sample/rounding. */
int galois_engine_set_cubes(galois_engine *eng, int32_t d, const int32_t *vars);

/* Join an NCCL communicator of `world` ranks (one per GPU) created from a 128-byte
 * ncclUniqueId produced by galois_comm_unique_id on one rank and shared by the caller.
 * The communicator is initialised (collectively) at the first step.
 * Exchange (row a9; mechanism ours, the paper's 2 -> 8 GPU split is Table 3):
 * every rank keeps its own best record and the winner's bits exactly as on one rank; after
 * each check an 8-byte MIN all-reduce of (u << 32 | global member) runs on an engine-owned
 * exchange stream, overlapping the update of the same step; the main stream joins it and
 * folds it into the global record before the next sweep. The global record (u*, t*, b*), its bits
 * (broadcast from the owner rank, b* / b_per), the unsat counts and steps_done are exactly
 * the single-GPU result; a rank that did not hold the SAT member may run one update past t*
 * (its iterate then is one step ahead; no further check runs). All ranks must make the same
 * sequence of step / enqueue / run / info / unsat_counts / best_assignment calls: each may
 * run the pending check and its collective exchange.
 * nccl_unique_id = NULL: no communicator — the engine runs rank `rank`'s slice of the
 * world-rank split alone (same slice, global member indices and RNG counters as with NCCL)
 * and its best record, bits and stop decision are the slice's own; the caller combines the
 * ranks' records (lexicographic minimum of (u, t, b), the key the exchange reduces). */
int galois_engine_set_comm(galois_engine *eng, int32_t rank, int32_t world, const void *nccl_unique_id);

/* Use the caller's CUDA stream (a cudaStream_t, e.g. torch.cuda.current_stream()). */
int galois_engine_set_stream(galois_engine *eng, void *cuda_stream);

/* Sub-batching for memory ("the batch is divided into sub-batches ... due to
 * memory limits"). sub_batch = 0 (default) keeps every local member
 * resident; a multiple of 32 smaller than the local slice makes the engine hold only
 * sub_batch members in HBM and galois_engine_run process the slice in consecutive
 * windows of sub_batch members, each run from t = 0 (members are independent: the
 * straight-through loss is a sum over members and every member's RNG counters use its
 * global index, so each member's trajectory is unchanged). A window after a SAT at step
 * t* runs at most t* steps. The best record is the lexicographic (unsat, step, member)
 * minimum over all windows — exactly the full-batch result; unsat_counts reports each
 * member's last check, info the slice and the full batch's step count. Only run() drives a
 * sub-batched engine (step/enqueue/set_iterate and the test hooks return E_STATE); run()
 * also keeps the theta_sel members (rule 0 and 1 of galois_select_member over every
 * member's last count) with their final iterates, so select_member, candidate_pool and
 * cube_variables work for those two members as on a resident batch.
 * With world > 1 every rank runs ceil(b_per / sub_batch) windows in lock step. */
int galois_engine_set_subbatch(galois_engine *eng, int32_t sub_batch);

/* Split the local slice into `lanes` (1..16) concurrent engines over consecutive member
 * ranges of ceil(b_loc / lanes) members rounded up to a multiple of 1024, each with its own
 * buffers, CUDA stream and control block; step(), enqueue() and run() drive them
 * interleaved, so one lane's clause sweep (a5 + a8, latency-bound) overlaps another lane's
 * fused update (a6 + a7, HBM-bound). Members never interact (the batch is a set of
 * independent restarts; RNG counters use the global member index), so every
 * member's trajectory is the undivided engine's, and the best record (u*, t*, b*) and its
 * assignment are identical (lexicographic minimum over the lanes' records). After a SAT,
 * lanes other than the winner's may have run up to two CUDA-graph chunks (16 steps) past t*;
 * unsat_counts then reports their members' counts at their own last check. Applies only
 * when the slice spans more than one lane, in ST mode, WITHOUT an NCCL communicator
 * (set_comm: concurrent collectives on several communicators of one device are not
 * guaranteed to progress), without sub-batching or debug; otherwise the engine is
 * undivided. get_iterate / set_iterate / get_loss / get_bits / get_member act on every lane
 * (set_iterate: each lane from the same step t); kernel_times sums over the lanes.
 * Setter: valid only before the first step. */
int galois_engine_set_lanes(galois_engine *eng, int32_t lanes);

/* CUDA graphs for run(): -1 never, 0 automatic (graphs of 8-step chunks when the run has
 * >= 32 chunks left), 1 always (also bypasses the single-launch small-instance run). The
 * result is identical in every mode (kernels read the step index from the device). */
int galois_engine_set_graphs(galois_engine *eng, int32_t mode);

/* Device bytes one member costs in the given mode (z, m, v, bit planes, E or soft
 * buffers, counters), for sizing sub_batch to a memory budget. */
int galois_engine_bytes_per_member(const galois_cnf *cnf, int32_t mode, int64_t *bytes);

/* Exact device bytes of an engine (or f4 window) of `members` resident members for
 * `steps` steps in the given mode, with_cubes != 0 if it holds cube pins: the allocation
 * prepare makes (members padded to 32, or to 1024-member chunks above 1024, plus E, hub
 * partials and counters: a window's bytes are not its members times bytes_per_member). */
int galois_engine_window_bytes(const galois_cnf *cnf, int32_t mode, int32_t members, int32_t steps,
                               int32_t with_cubes, int64_t *bytes);

/* The largest multiple of 32 members whose window_bytes fit budget_bytes (f4's
 * sub_batch for a memory budget, e.g. galois_device_free_bytes minus a margin).
 * E_OOM if not even 32 members fit. */
int galois_engine_max_sub_batch(const galois_cnf *cnf, int32_t mode, int32_t steps, int32_t with_cubes,
                                int64_t budget_bytes, int32_t *sub_batch);

/* Device memory available to a new engine on `device`: the driver's free bytes plus what
 * the library's stream-ordered pool holds unused (freed engines and CNFs stay reserved in
 * it for reuse). Divide by bytes_per_member for the largest resident sub_batch (f4). */
int galois_device_free_bytes(int32_t device, int64_t *bytes);

/* Test hook: also store the per-step clause signal G and gradient g1 (see get_grad). */
int galois_engine_set_debug(galois_engine *eng, int32_t enable);

/* Record CUDA events around every kernel launch (see galois_engine_kernel_times). */
int galois_engine_set_profiling(galois_engine *eng, int32_t enable);

/* Produce a 128-byte ncclUniqueId into out (on one rank). E_NCCL if NCCL is absent. */
int galois_comm_unique_id(void *out128);

/* ------------------------------------- what the CPU stage consumes */

/* theta_sel ("we select the logits theta_sel from the batch with the minimal clause
 * loss"; "the one with the highest loss value"): rule 0 = the local member with the
 * fewest unsatisfied clauses at the last check, rule 1 = the most; ties to the lower member.
 * Outputs its global index, its count and (z may be NULL) its reduced logits
 * z_v = theta_{v,1} - theta_{v,0} (n floats, host). Local to this rank. */
int galois_select_member(galois_engine *eng, int32_t rule, int64_t *global_b, int32_t *unsat, float *z);

/* |S| = max(1, ceil(rho * n_orig)) of galois_candidate_pool (Eq.11), for sizing
 * its units array. E_ARG unless 0 < rho <= 1. */
int galois_candidate_pool_size(const galois_cnf *cnf, double rho, int32_t *S);

/* Candidate pool (Eq.10) of member `global_b` (local to this rank): N samples
 * x^(k)_v = [z_v + ell^(k)_v >= 0] with fresh logistic noise (Philox counter (v, k/4, 0, 2),
 * word k mod 4, key pool_seed) and confidences c^(k)_v = max(y_0, y_1) = sigma(|z_v + ell|/tau)
 * over all n variables; and per candidate the S = max(1, ceil(rho * n_orig)) most confident
 * ORIGINAL variables (Eq.11, auxiliaries excluded as P:214 states; paper
 * rho = 0.0005) as DIMACS unit literals (+v if x = 1, else -v), ordered by descending
 * confidence, ties to the lower index.
 *   values [N][n] uint8 (may be NULL), confidence [N][n] float (may be NULL),
 *   units [N][S] int32 (may be NULL; S <= 2^20), *S_out = S. E_ARG on bad sizes
 *   (N * n > 2^31 when values or confidence is requested).
 * With values = confidence = NULL the pool is drawn over the n_orig original variables
 * only (the same per-variable counters, so the same draws) in groups of candidates whose
 * device scratch stays near 1.3 GB — the form for instances of the paper's largest size
 * (P:559), where |S| = ceil(0.0005 n_orig) exceeds one CTA's shared-memory sort (4096
 * keys) and is sorted in global memory instead. */
int galois_candidate_pool(galois_engine *eng, int64_t global_b, int32_t N, double rho, uint64_t pool_seed,
                          uint8_t *values, float *confidence, int32_t *units, int32_t *S_out);

/* Confidence-guided branching (Lemma 1: "identify d variables with the lowest
 * confidence"): the d original variables (1..n_orig) of member global_b with the lowest
 * noise-free confidence sigma(|z_v|/tau) (= smallest |z_v|), ties to the lower index,
 * 1-based ascending — ready for galois_engine_set_cubes. 1 <= d <= min(n_orig, 4096). */
int galois_cube_variables(galois_engine *eng, int64_t global_b, int32_t d, int32_t *vars);

/* ------------------------------------------------------ test hooks (parity / resume) */

/* Reduced iterate of the local members, host [b_loc][n] float each (NULL to skip):
 * z = theta_1 - theta_0, m = Adam first moment of theta_1, v = second moment; t = steps. */
int galois_engine_get_iterate(galois_engine *eng, float *z, float *m, float *v, int32_t *t);

/* Overwrite the iterate (same layout) and the step counter; recomputes the rounding R_t
 * and the next sample X_{t+1}; clears the stop flag (the best record is kept). */
int galois_engine_set_iterate(galois_engine *eng, const float *z, const float *m, const float *v,
                              int32_t t);

/* One member's state, read in place on the device (works on lanes and at full size) and
 * WITHOUT running a pending check (unlike unsat_counts): reduced iterate z, m, v (n floats
 * each), the sample bits X_{t+1} the next forward uses and the rounding R_t (n bytes 0/1
 * each), with set_debug(1) the last step's signal G (n int32) and g1 (n floats); t = the
 * steps of the engine (or lane) holding the member; unsat = its count at the last check
 * that ran, check_t = that check's step. Any output may be NULL. E_ARG if global_b is not
 * local; E_STATE on a sub-batched engine. */
int galois_engine_get_member(galois_engine *eng, int64_t global_b, float *z, float *m, float *v,
                             uint8_t *x_next, uint8_t *r, int32_t *G, float *g1, int32_t *t,
                             int32_t *unsat, int32_t *check_t);

/* Of the last step (requires set_debug(1) before the first step): the clause signal
 * G = sum over occurrences of sigma * E (int32; ST mode) and dL/dtheta_1 = -G p q / tau
 * (float), host [b_loc][n] each (NULL to skip). */
int galois_engine_get_grad(galois_engine *eng, int32_t *G, float *g1);

/* Of the last forward: Lambda_b = sum_c U_c (= L_b + m; the unsat count of the sample
 * in ST mode, exact: double holds every count up to 2^53), host b_loc doubles. */
int galois_engine_get_loss(galois_engine *eng, double *lambda);

/* The sample bits X_{t+1} the next forward will use and the rounding R_t of the last
 * update, host [b_loc][n] bytes 0/1 each (NULL to skip). */
int galois_engine_get_bits(galois_engine *eng, uint8_t *x_next, uint8_t *r);

/* Kernel times accumulated since the last call (profiling mode): for kernel class
 * k in {0 forward, 1 update, 2 check, 3 best/extract, 4 hub-partial, 5 init}:
 * ms[k] total milliseconds and launches[k] count (arrays of GALOIS_NUM_KERNEL_CLASSES). */
#define GALOIS_NUM_KERNEL_CLASSES 6
int galois_engine_kernel_times(galois_engine *eng, double *ms, int64_t *launches);

#ifdef __cplusplus
}
#endif
#endif /* GALOIS_H */
