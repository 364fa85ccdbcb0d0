/*
 * oracle.c — plain, slow, fp64 CPU reference of GaloisSAT's GPU stage.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library. The product path
 * (paper_2603_28796_b200/) never imports, links or executes anything under oracle/,
 * and this file shares no code, header, table or constant generator with the CUDA
 * path (it carries its own Philox).
 *
 * Every function follows one passage of the paper, cited as P:<line> of PAPER.md
 * (arxiv 2603.28796) with its equation / section, or a reading listed in DESIGN.md
 * ("R<k>"). The arithmetic is the definition written out, one batch member at a
 * time, with no blocking, fusion or reordering:
 *
 *   Eq.1  not x = 1-x, x and y = xy, x or y = x+y-xy
 *   Eq.2  C = 1 - prod_i (1 - s_i)
 *   Eq.3  y_ij = softmax_j((theta_ij + g_ij)/tau), g iid Gumbel(0,1)
 *   Eq.4  x_hat = argmax_j y_ij; backward dL/dx_hat ~ dL/dy (straight-through)
 *   Eq.5  L = - sum_t C_t
 *   App. A     Adam, lr 0.5, tau 1
 *   P:59               a CNF is satisfied iff every clause has a true literal
 *   P:102              theta_sel from the batch member with the minimal clause loss
 *
 * Pins (tests/test_oracle_*.py): Philox KATs (Random123), logistic/normal
 * statistics, exhaustive Boolean tables, the paper's printed numbers (P:144,
 * P:766), brute force over all 2^n assignments, the flip-delta identity,
 * central finite differences, torch.optim.Adam and a torch-autograd transcription
 * of Eq.3-5. No function here is "parity unpinned".
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------------- */
/* Random numbers (reading R2 in DESIGN.md).                                  */
/* Philox4x32-10, Salmon, Moraes, Dror, Shaw, SC'11 ("Random123").            */
/* ------------------------------------------------------------------------- */

#define PHILOX_M0 0xD2511F53u
#define PHILOX_M1 0xCD9E8D57u
#define PHILOX_W0 0x9E3779B9u
#define PHILOX_W1 0xBB67AE85u

void oracle_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4])
{
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int round = 0; round < 10; round++) {
        uint64_t p0 = (uint64_t)PHILOX_M0 * (uint64_t)c0;
        uint64_t p1 = (uint64_t)PHILOX_M1 * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        k0 += PHILOX_W0;
        k1 += PHILOX_W1;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* Open-interval uniform from the low 23 bits of a 32-bit word (reading R2):
 * u = (k + 1/2) 2^-23 with k = w mod 2^23, so u and 1-u are both exact binary
 * fractions with 24 significant bits. */
double oracle_uniform(uint32_t w)
{
    uint32_t k = w & 0x7FFFFFu;
    return ((double)k + 0.5) / 8388608.0;
}

double oracle_uniform_complement(uint32_t w)
{
    uint32_t k = w & 0x7FFFFFu;
    return ((double)(8388607u - k) + 0.5) / 8388608.0;
}

/* theta_{b,v,j} ~ N(0,1) i.i.d. ("each batch is independently and randomly
 * initialized"; reading R1): Box-Muller on Philox counter (v, b/2, 0, 0), key =
 * seed; member b uses words 2(b mod 2) and 2(b mod 2)+1. */
void oracle_init_logits(int32_t n, int64_t b0, int64_t nb, uint64_t seed, double *theta /* [nb][n][2] */)
{
    const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    for (int64_t bi = 0; bi < nb; bi++) {
        int64_t b = b0 + bi;
        for (int32_t v = 0; v < n; v++) {
            uint32_t ctr[4] = {(uint32_t)v, (uint32_t)(b >> 1), 0u, 0u};
            uint32_t w[4];
            oracle_philox4x32_10(ctr, key, w);
            int j = (int)(b & 1);
            double u0 = oracle_uniform(w[2 * j]);
            double u1 = oracle_uniform(w[2 * j + 1]);
            double rho = sqrt(-2.0 * log(u0));
            theta[(bi * n + v) * 2 + 0] = rho * cos(2.0 * M_PI * u1);
            theta[(bi * n + v) * 2 + 1] = rho * sin(2.0 * M_PI * u1);
        }
    }
}

/* Gumbel difference at step t >= 1 (Eq.3; reading R2):
 * ell = g_1 - g_0 ~ Logistic(0,1), drawn as ell = ln u - ln(1-u) from Philox counter
 * (v, b/4, t, 1), word b mod 4. The 2-class softmax of Eq.3 depends on the g's
 * only through g_1 - g_0, which is exactly Logistic(0,1)-distributed. */
double oracle_logistic_noise(int32_t v, int64_t b, int32_t t, uint64_t seed)
{
    const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint32_t ctr[4] = {(uint32_t)v, (uint32_t)(b >> 2), (uint32_t)t, 1u};
    uint32_t w[4];
    oracle_philox4x32_10(ctr, key, w);
    uint32_t word = w[b & 3];
    return log(oracle_uniform(word)) - log(oracle_uniform_complement(word));
}

void oracle_noise(int32_t n, int64_t b0, int64_t nb, uint64_t seed, int32_t t, double *ell /* [nb][n] */)
{
    for (int64_t bi = 0; bi < nb; bi++)
        for (int32_t v = 0; v < n; v++)
            ell[bi * n + v] = oracle_logistic_noise(v, b0 + bi, t, seed);
}

/* ------------------------------------------------------------------------- */
/* CNF: clause c holds slots offsets[c] .. offsets[c+1]-1, each a DIMACS literal */
/* (+v or -v, 1-based), P:59 and the SPEC's cnf-core.                          */
/* ------------------------------------------------------------------------- */

typedef struct {
    int32_t n;                /* variables */
    int64_t m;                /* clauses */
    const int64_t *offsets;   /* m+1 */
    const int32_t *lits;      /* offsets[m] */
} oracle_cnf;

/* Eq.2 on the literal values s of each slot: U_c = prod_i (1 - s_{c,i})
 * (1 iff the clause is unsatisfied on Boolean inputs), C_c = 1 - U_c. Also the
 * exclusive products E_{c,i} = prod_{j != i} (1 - s_{c,j}), formed from prefix and
 * suffix products in slot order (never by dividing U by 1 - s_i, reading R23). */
void oracle_clause_products(const oracle_cnf *f, const double *s /* [L] */,
                            double *U /* [m] */, double *E /* [L] */)
{
    for (int64_t c = 0; c < f->m; c++) {
        int64_t lo = f->offsets[c], hi = f->offsets[c + 1];
        double prefix = 1.0;
        for (int64_t k = lo; k < hi; k++) {     /* E_k <- prod_{j<k} (1 - s_j) */
            E[k] = prefix;
            prefix *= (1.0 - s[k]);
        }
        U[c] = prefix;                          /* prod over all slots */
        double suffix = 1.0;
        for (int64_t k = hi - 1; k >= lo; k--) { /* E_k *= prod_{j>k} (1 - s_j) */
            E[k] *= suffix;
            suffix *= (1.0 - s[k]);
        }
    }
}

/* Literal value s of slot k given variable values xval (s = x for a positive
 * literal, 1 - x for a negated one; Eq.1's "not x = 1 - x"). */
static double literal_value(int32_t lit, const double *xval)
{
    int32_t v = (lit > 0 ? lit : -lit) - 1;
    return lit > 0 ? xval[v] : 1.0 - xval[v];
}

/* The straight-through clause signal of one member (Eq.4 text; Eq.5):
 * with L = -sum_c C_c = sum_c U_c - m,  dL/ds_{c,i} = dU_c/ds_{c,i} = -E_{c,i} and
 * ds/dx = sigma (+1 positive, -1 negated), so dL/dx_v = -G_v with
 * G_v = sum over the slots of v, in ascending slot order, of sigma * E.
 * Returns Lambda = sum_c U_c (= L + m, the loss that is zero iff all clauses hold). */
double oracle_member_signal(const oracle_cnf *f, const double *xval /* [n] */,
                            double *s_scratch /* [L] */, double *U /* [m] */,
                            double *E /* [L] */, double *G /* [n] */)
{
    int64_t L = f->offsets[f->m];
    for (int64_t k = 0; k < L; k++)
        s_scratch[k] = literal_value(f->lits[k], xval);
    oracle_clause_products(f, s_scratch, U, E);
    for (int32_t v = 0; v < f->n; v++)
        G[v] = 0.0;
    for (int64_t k = 0; k < L; k++) {
        int32_t lit = f->lits[k];
        int32_t v = (lit > 0 ? lit : -lit) - 1;
        G[v] += (lit > 0 ? 1.0 : -1.0) * E[k];
    }
    double lambda = 0.0;
    for (int64_t c = 0; c < f->m; c++)
        lambda += U[c];
    return lambda;
}

/* Exact Boolean check (SPEC cnf-core.verify_model): the number of clauses in
 * which no literal is true under the 0/1 assignment r. A separate code path from
 * the polynomial: a plain OR over the literals. */
int64_t oracle_unsat_count(const oracle_cnf *f, const uint8_t *r /* [n] */)
{
    int64_t unsat = 0;
    for (int64_t c = 0; c < f->m; c++) {
        int satisfied = 0;
        for (int64_t k = f->offsets[c]; k < f->offsets[c + 1]; k++) {
            int32_t lit = f->lits[k];
            int32_t v = (lit > 0 ? lit : -lit) - 1;
            int value = r[v] ? 1 : 0;
            if ((lit > 0 && value) || (lit < 0 && !value)) {
                satisfied = 1;
                break;
            }
        }
        if (!satisfied)
            unsat++;
    }
    return unsat;
}

/* ------------------------------------------------------------------------- */
/* One optimiser step for a slice of members (C.1 steps 2-12 of SURVEY §8(c)). */
/* ------------------------------------------------------------------------- */

typedef struct {
    int32_t mode;        /* 0 = straight-through (paper), 1 = fully soft (debug) */
    int32_t optimizer;   /* 0 = Adam (App. A), 1 = plain gradient step */
    double lr;           /* 0.5 */
    double tau;          /* 1.0 */
    double beta1, beta2, eps;  /* 0.9, 0.999, 1e-8 (reading R7) */
    uint64_t seed;
    int32_t num_pins;    /* d (Lemma 1); 0 = none */
    const int32_t *pin_vars; /* d variables, 0-based, ascending; member b takes bit r of (b mod 2^d) */
} oracle_config;

/* Pinned value of variable v for member b, or -1 when v is free (Lemma 1, P:247:
 * cube alpha in {0,1}^d; reading R14: alpha = b mod 2^d, little-endian). */
static int pin_value(const oracle_config *cfg, int32_t v, int64_t b)
{
    for (int32_t r = 0; r < cfg->num_pins; r++)
        if (cfg->pin_vars[r] == v) {
            uint64_t alpha = (uint64_t)b & ((cfg->num_pins >= 64) ? ~0ull : ((1ull << cfg->num_pins) - 1ull));
            return (int)((alpha >> r) & 1ull);
        }
    return -1;
}

/* Per-member outputs of one step, all optional (NULL = not wanted). */
typedef struct {
    double *a;       /* [nb][n] (theta_1 - theta_0 + ell)/tau, the argument of the 2-class softmax */
    uint8_t *xhat;   /* [nb][n] hard sample used by the forward */
    double *lambda;  /* [nb]    sum_c U_c of the forward */
    double *G;       /* [nb][n] clause signal */
    double *grad1;   /* [nb][n] dL_b/dtheta_{b,v,1} */
    uint8_t *r;      /* [nb][n] noise-free rounding after the update */
    int64_t *unsat;  /* [nb]    exact unsat count of r */
} oracle_step_out;

/* One step t >= 1 for members b0 .. b0+nb-1, in place on theta/mom/vel [nb][n][2]
 * (the paper's Theta in R^{B x n x 2}, with Adam's two moment tensors). */
void oracle_step(const oracle_cnf *f, const oracle_config *cfg, int64_t b0, int64_t nb, int32_t t,
                 double *theta, double *mom, double *vel, oracle_step_out *out)
{
    const int32_t n = f->n;
    const int64_t L = f->offsets[f->m];
#pragma omp parallel
    {
        double *xval = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
        double *p = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
        double *q = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
        double *G = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
        double *s = (double *)malloc(sizeof(double) * (size_t)(L > 0 ? L : 1));
        double *E = (double *)malloc(sizeof(double) * (size_t)(L > 0 ? L : 1));
        double *U = (double *)malloc(sizeof(double) * (size_t)(f->m > 0 ? f->m : 1));
        uint8_t *r = (uint8_t *)malloc((size_t)(n > 0 ? n : 1));
#pragma omp for schedule(static)
        for (int64_t bi = 0; bi < nb; bi++) {
            int64_t b = b0 + bi;
            double *th = theta + bi * n * 2, *m1 = mom + bi * n * 2, *v1 = vel + bi * n * 2;
            /* Eq.3: y = softmax((theta + g)/tau); for two classes y_1 = sigma(a) with
             * a = (theta_1 + g_1 - theta_0 - g_0)/tau. q = y_0 = sigma(-a) is computed
             * directly rather than as 1 - p (reading R23). Eq.4: x_hat = argmax_j y_j,
             * ties to class 1 (reading R3). */
            for (int32_t v = 0; v < n; v++) {
                double ell = oracle_logistic_noise(v, b, t, cfg->seed);
                double a = (th[2 * v + 1] - th[2 * v + 0] + ell) / cfg->tau;
                p[v] = 1.0 / (1.0 + exp(-a));
                q[v] = 1.0 / (1.0 + exp(a));
                int pv = pin_value(cfg, v, b);
                int hard = (pv >= 0) ? pv : (a >= 0.0 ? 1 : 0);
                if (pv >= 0) { p[v] = (double)pv; q[v] = 1.0 - (double)pv; }
                xval[v] = (cfg->mode == 0) ? (double)hard : p[v];
                if (out && out->a) out->a[bi * n + v] = a;
                if (out && out->xhat) out->xhat[bi * n + v] = (uint8_t)hard;
            }
            /* Eq.2 + Eq.5 on the hard (ST) or soft values, and the clause signal G. */
            double lambda = oracle_member_signal(f, xval, s, U, E, G);
            if (out && out->lambda) out->lambda[bi] = lambda;
            for (int32_t v = 0; v < n; v++) {
                int pv = pin_value(cfg, v, b);
                /* Straight-through: dL/dp_v = dL/dx_v = -G_v; the softmax
                 * Jacobian at fixed noise gives dp/dtheta_1 = p q / tau = -dp/dtheta_0. */
                double g1 = (pv >= 0) ? 0.0 : -G[v] * p[v] * q[v] / cfg->tau;
                double g0 = -g1;
                if (out && out->G) out->G[bi * n + v] = G[v];
                if (out && out->grad1) out->grad1[bi * n + v] = g1;
                if (pv >= 0)
                    continue;   /* pinned variables are frozen (reading R14) */
                double g[2] = {g0, g1};
                for (int j = 0; j < 2; j++) {
                    if (cfg->optimizer == 0) {
                        /* Adam (App. A) in PyTorch's formulation (reading R7):
                         * m <- b1 m + (1-b1) g ; v <- b2 v + (1-b2) g^2 ;
                         * theta <- theta - (lr / (1-b1^t)) m / (sqrt(v)/sqrt(1-b2^t) + eps) */
                        m1[2 * v + j] = cfg->beta1 * m1[2 * v + j] + (1.0 - cfg->beta1) * g[j];
                        v1[2 * v + j] = cfg->beta2 * v1[2 * v + j] + (1.0 - cfg->beta2) * g[j] * g[j];
                        double bc1 = 1.0 - pow(cfg->beta1, (double)t);
                        double bc2 = 1.0 - pow(cfg->beta2, (double)t);
                        double denom = sqrt(v1[2 * v + j]) / sqrt(bc2) + cfg->eps;
                        th[2 * v + j] -= (cfg->lr / bc1) * m1[2 * v + j] / denom;
                    } else {
                        th[2 * v + j] -= cfg->lr * g[j];
                    }
                }
            }
            /* Noise-free rounding r = argmax_j theta_j (reading R11) and exact check. */
            for (int32_t v = 0; v < n; v++) {
                int pv = pin_value(cfg, v, b);
                r[v] = (uint8_t)((pv >= 0) ? pv : (th[2 * v + 1] >= th[2 * v + 0] ? 1 : 0));
                if (out && out->r) out->r[bi * n + v] = r[v];
            }
            if (out && out->unsat) out->unsat[bi] = oracle_unsat_count(f, r);
        }
        free(xval); free(p); free(q); free(G); free(s); free(E); free(U); free(r);
    }
}

/* Rounding and check of the initial logits (the t = 0 check point, reading R22). */
void oracle_round_and_check(const oracle_cnf *f, const oracle_config *cfg, int64_t b0, int64_t nb,
                            const double *theta, uint8_t *r_out /* [nb][n] or NULL */,
                            int64_t *unsat /* [nb] */)
{
    const int32_t n = f->n;
#pragma omp parallel
    {
        uint8_t *r = (uint8_t *)malloc((size_t)(n > 0 ? n : 1));
#pragma omp for schedule(static)
        for (int64_t bi = 0; bi < nb; bi++) {
            const double *th = theta + bi * n * 2;
            for (int32_t v = 0; v < n; v++) {
                int pv = pin_value(cfg, v, b0 + bi);
                r[v] = (uint8_t)((pv >= 0) ? pv : (th[2 * v + 1] >= th[2 * v + 0] ? 1 : 0));
                if (r_out) r_out[bi * n + v] = r[v];
            }
            unsat[bi] = oracle_unsat_count(f, r);
        }
        free(r);
    }
}

/* The whole GPU-stage loop for members b0 .. b0+nb-1: init, then
 * steps t = 1..T, checking the noise-free rounding at t = 0, every K steps and at
 * t = T (reading R22); the best record is the lexicographic minimum of
 * (unsat, t, b) (reading R10); the loop stops when the best is 0 (SAT).
 * Returns the number of steps executed. best_r receives the n bits of the best. */
int32_t oracle_run(const oracle_cnf *f, const oracle_config *cfg, int64_t b0, int64_t nb,
                   int32_t T, int32_t K, double *theta, double *mom, double *vel,
                   int64_t *best_unsat, int32_t *best_t, int64_t *best_b, uint8_t *best_r,
                   int64_t *last_unsat /* [nb] counts of the last check */)
{
    const int32_t n = f->n;
    uint8_t *r = (uint8_t *)malloc((size_t)nb * (size_t)(n > 0 ? n : 1));
    int64_t *unsat = (int64_t *)malloc(sizeof(int64_t) * (size_t)(nb > 0 ? nb : 1));
    oracle_init_logits(n, b0, nb, cfg->seed, theta);
    memset(mom, 0, sizeof(double) * (size_t)nb * (size_t)n * 2);
    memset(vel, 0, sizeof(double) * (size_t)nb * (size_t)n * 2);
    *best_unsat = INT64_MAX; *best_t = -1; *best_b = -1;
    oracle_round_and_check(f, cfg, b0, nb, theta, r, unsat);
    int32_t t = 0;
    for (;;) {
        int is_check = (t == 0) || (K > 0 && t % K == 0) || (t == T);
        if (is_check) {
            for (int64_t bi = 0; bi < nb; bi++) {
                if (unsat[bi] < *best_unsat) {   /* strict: earlier t, then lower b, wins ties */
                    *best_unsat = unsat[bi]; *best_t = t; *best_b = b0 + bi;
                    if (best_r) memcpy(best_r, r + bi * n, (size_t)n);
                }
            }
            if (last_unsat) memcpy(last_unsat, unsat, sizeof(int64_t) * (size_t)nb);
            if (*best_unsat == 0)
                break;
        }
        if (t == T)
            break;
        t++;
        oracle_step_out out = {0};
        out.r = r;
        out.unsat = unsat;
        oracle_step(f, cfg, b0, nb, t, theta, mom, vel, &out);
    }
    free(r); free(unsat);
    return t;
}

/* Candidate pool (Eq.10; SPEC sat-pool.sample_pool): N Gumbel samples of the
 * selected member's logits, here in reduced form z_v = theta_{v,1} - theta_{v,0}. Sample k
 * draws ell^(k)_v = ln u - ln(1-u) from Philox counter (v, k/4, 0, 2), word k mod 4, key =
 * pool_seed (reading R2's layout in a separate counter domain); a = (z_v + ell)/tau;
 * x^(k)_v = [a >= 0] (Eq.4, ties to 1); c^(k)_v = max(y_0, y_1) = sigma(|a|). */
void oracle_pool(const double *z, int32_t n, int32_t N, double tau, uint64_t pool_seed,
                 uint8_t *x /* [N][n] */, double *conf /* [N][n] */)
{
    const uint32_t key[2] = {(uint32_t)pool_seed, (uint32_t)(pool_seed >> 32)};
    for (int32_t k = 0; k < N; k++)
        for (int32_t v = 0; v < n; v++) {
            uint32_t ctr[4] = {(uint32_t)v, (uint32_t)(k >> 2), 0u, 2u};
            uint32_t w[4];
            oracle_philox4x32_10(ctr, key, w);
            uint32_t word = w[k & 3];
            double ell = log(oracle_uniform(word)) - log(oracle_uniform_complement(word));
            double a = (z[v] + ell) / tau;
            x[(int64_t)k * n + v] = (uint8_t)(a >= 0.0 ? 1 : 0);
            conf[(int64_t)k * n + v] = 1.0 / (1.0 + exp(-fabs(a)));
        }
}

int32_t oracle_num_threads(void)
{
#ifdef _OPENMP
    return (int32_t)omp_get_max_threads();
#else
    return 1;
#endif
}

void oracle_set_num_threads(int32_t k)
{
#ifdef _OPENMP
    if (k > 0) omp_set_num_threads(k);
#else
    (void)k;
#endif
}
