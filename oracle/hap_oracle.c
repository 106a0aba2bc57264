/*
 * hap_oracle.c — plain, slow, obviously-correct fp64 CPU oracle.
 *
 * TEST INFRASTRUCTURE ONLY (see hap_oracle.h).  It is never linked into, loaded
 * by, or called from the product path; it shares no code with it.
 *
 * Everything is fp64, plain loops, no blocking/fusion/reordering beyond what the
 * paper's Algorithm 1 states.  Readings where the paper is
 * silent are listed in DESIGN.md ("Readings"), R-numbers cited inline.
 */
#include "hap_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------- */
/* Philox4x32-10 — Salmon, Moraes, Dror, Shaw, "Parallel random numbers: as   */
/* easy as 1, 2, 3" (SC'11).  Round: (c0,c1,c2,c3) -> (hi(M1 c2)^c1^k0,       */
/* lo(M1 c2), hi(M0 c0)^c3^k1, lo(M0 c0)); key bumped by the Weyl constants   */
/* between rounds.  Pinned by the Random123 known-answer vectors in           */
/* tests/golden/philox_kat.txt.                                               */
/* ------------------------------------------------------------------------- */
void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    uint32_t k0 = key[0], k1 = key[1];
    for (int round = 0; round < 10; ++round) {
        uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* word number `idx` of the Philox stream with counter words (c1, c2, c3):     */
/* block q = idx/4 is philox((q, c1, c2, c3), key), word idx%4 of that block. */
static uint32_t stream_word(const uint32_t key[2], uint32_t c1, uint32_t c2, uint32_t c3,
                            uint64_t idx) {
    uint32_t ctr[4] = {(uint32_t)(idx / 4), c1, c2, c3};
    uint32_t out[4];
    orc_philox4x32_10(ctr, key, out);
    return out[idx % 4];
}

/* ------------------------------------------------------------------------- */
/* PERM-SPEC v1 (R6).  "Randomly partition Z into     */
/* (X^(b), Y^(b)) with sizes (n, m)" (Alg. 1) realised as the     */
/* partial forward Fisher–Yates shuffle:                                       */
/*   a = [0..N-1];  for i = 0..n_x-1:  j = i + U(N-i);  swap(a[i], a[j]);      */
/*   group 1 = {a[0..n_x-1]}.                                                  */
/* U(k): Lemire's exact bounded draw on word w_i of the main stream            */
/* (counter (i/4, b, s, 0)); a rejected word is replaced by the next word of   */
/* the side stream (counter (q', b, s, 1+i), q' = 0, 1, ...).                  */
/* ------------------------------------------------------------------------- */
int orc_perm_set(uint64_t seed, uint32_t s, uint32_t b, int64_t N, int64_t n_x,
                 uint8_t* in_g1) {
    if (N < 1 || n_x < 0 || n_x > N || N > 0xFFFFFFFFll || !in_g1) return -1;
    const uint32_t key[2] = {(uint32_t)(seed & 0xFFFFFFFFu), (uint32_t)(seed >> 32)};
    int64_t* a = (int64_t*)malloc(sizeof(int64_t) * (size_t)N);
    if (!a) return -1;
    for (int64_t p = 0; p < N; ++p) a[p] = p;
    int redraws = 0;
    for (int64_t i = 0; i < n_x; ++i) {
        uint32_t k = (uint32_t)(N - i);
        uint32_t x = stream_word(key, b, s, 0u, (uint64_t)i);
        uint64_t m = (uint64_t)x * (uint64_t)k;
        uint32_t l = (uint32_t)m;
        if (l < k) {
            uint32_t t = (uint32_t)(0u - k) % k; /* (2^32 - k) mod k */
            uint64_t side = 0;
            while (l < t) {
                x = stream_word(key, b, s, (uint32_t)(1 + i), side++);
                m = (uint64_t)x * (uint64_t)k;
                l = (uint32_t)m;
                ++redraws;
            }
        }
        int64_t j = i + (int64_t)(m >> 32);
        int64_t tmp = a[i];
        a[i] = a[j];
        a[j] = tmp;
    }
    memset(in_g1, 0, (size_t)N);
    for (int64_t p = 0; p < n_x; ++p) in_g1[a[p]] = 1;
    free(a);
    return redraws;
}

/* ------------------------------------------------------------------------- */
/* Alignment, §3.1 / Alg. 1 steps 1-3.                                */
/* ------------------------------------------------------------------------- */
static double dot(const double* a, const double* b, int64_t d) {
    double s = 0.0;
    for (int64_t c = 0; c < d; ++c) s += a[c] * b[c];
    return s;
}

int orc_align(const float* X, int64_t n_x, const float* Y, int64_t n_y, int64_t d, int mode,
              double* Z, double* u, double* info) {
    if (n_x < 1 || n_y < 1 || d < 2 || !X || !Y || !Z || !u || !info) return ORC_E_ARG;
    const int64_t N = n_x + n_y;
    info[0] = info[1] = info[2] = 0.0;
    info[3] = -1.0;
    /* Eq. 2: x = h / ||h||_2 ; rows of Z are X then Y. */
    for (int64_t i = 0; i < N; ++i) {
        const float* h = (i < n_x) ? (X + i * d) : (Y + (i - n_x) * d);
        double nrm2 = 0.0;
        for (int64_t c = 0; c < d; ++c) nrm2 += (double)h[c] * (double)h[c];
        double nrm = sqrt(nrm2);
        if (nrm < 1e-12) { /* ZeroVector (R3) */
            info[3] = (double)i;
            return ORC_E_ZERO_VECTOR;
        }
        for (int64_t c = 0; c < d; ++c) Z[i * d + c] = (double)h[c] / nrm;
    }
    /* means xbar, ybar (Alg. 1), ascending order */
    double* xbar = (double*)calloc((size_t)d, sizeof(double));
    double* ybar = (double*)calloc((size_t)d, sizeof(double));
    double* v = (double*)calloc((size_t)d, sizeof(double));
    for (int64_t i = 0; i < n_x; ++i)
        for (int64_t c = 0; c < d; ++c) xbar[c] += Z[i * d + c];
    for (int64_t i = n_x; i < N; ++i)
        for (int64_t c = 0; c < d; ++c) ybar[c] += Z[i * d + c];
    for (int64_t c = 0; c < d; ++c) { xbar[c] /= (double)n_x; ybar[c] /= (double)n_y; }
    double nx = sqrt(dot(xbar, xbar, d)), ny = sqrt(dot(ybar, ybar, d));
    info[0] = nx;
    info[1] = ny;
    int rc = ORC_OK;
    if (nx < 1e-12 || ny < 1e-12) { /* DegenerateMean (R3) */
        rc = ORC_E_DEGENERATE_MEAN;
        goto done;
    }
    for (int64_t c = 0; c < d; ++c) u[c] = 0.0;
    if (mode == 0) {
        /* Eq. 5: u = (mu_x - mu_y)/||mu_x - mu_y|| ; identity if
         * mu_x == mu_y (tolerance 1e-9, R3). */
        for (int64_t c = 0; c < d; ++c) v[c] = xbar[c] / nx - ybar[c] / ny;
        double nv = sqrt(dot(v, v, d));
        if (nv < 1e-9) {
            info[2] = 1.0;
        } else {
            for (int64_t c = 0; c < d; ++c) u[c] = v[c] / nv;
            /* Eq. 7 with Eq. householder_fast (Alg. 1
             * PAPER.md:667-670): x' = x - 2 u (u^T x), X only; Y unchanged. */
            for (int64_t i = 0; i < n_x; ++i) {
                double* x = Z + i * d;
                double ux = dot(u, x, d);
                for (int64_t c = 0; c < d; ++c) x[c] = x[c] - 2.0 * u[c] * ux;
            }
        }
    } else {
        info[2] = 1.0; /* naive baseline: no reflection */
    }
done:
    free(xbar);
    free(ybar);
    free(v);
    return rc;
}

/* ------------------------------------------------------------------------- */
/* Dispersion, PAPER.md:164-180 (Eqs. 8-10) with g_d = Banerjee's kappa-hat    */
/* (R1): L(r) = log kappa-hat(r) = -log v.              */
/* ------------------------------------------------------------------------- */
double orc_logkappa(double r, int64_t d) {
    if (r > 1.0 - 1e-9) r = 1.0 - 1e-9; /* SPEC.md:132, R4 */
    if (r <= 0.0) return -INFINITY;
    double r2 = r * r;
    return log(r) + log((double)d - r2) - log(1.0 - r2);
}

/* T = log v(G1) - log v(G2) = L(r2) - L(r1) (Eq. 10/11).
 * Both r = 0: T := 0 (R4). */
static double stat_T(double L1, double L2) {
    if (isinf(L1) && isinf(L2)) return 0.0;
    return L2 - L1;
}

void orc_group_stats(const double* Z, int64_t N, int64_t d, int64_t n_x, const uint8_t* in_g1,
                     double* out) {
    double* s1 = (double*)calloc((size_t)d, sizeof(double));
    double* s2 = (double*)calloc((size_t)d, sizeof(double));
    for (int64_t i = 0; i < N; ++i) { /* direct group sums, ascending i */
        double* s = in_g1[i] ? s1 : s2;
        for (int64_t c = 0; c < d; ++c) s[c] += Z[i * d + c];
    }
    const int64_t n_y = N - n_x;
    double r1 = sqrt(dot(s1, s1, d)) / (double)n_x; /* Eq. 8 on the permuted groups */
    double r2 = sqrt(dot(s2, s2, d)) / (double)n_y;
    double L1 = orc_logkappa(r1, d), L2 = orc_logkappa(r2, d);
    out[0] = r1;
    out[1] = r2;
    out[2] = L1;
    out[3] = L2;
    out[4] = stat_T(L1, L2);
    free(s1);
    free(s2);
}

/* one comparison against the observed value (Eq. pvalue uses >=, PAPER.md:189;
 * two-sided |T_b| >= |T_obs| is DESIGN.md R5).  The near-tie flag (R8) marks a
 * permutation within tau of either decision boundary: T_obs (one-sided) or |T_obs|
 * (two-sided). */
static void tally(double T, double t_obs, double tau, uint64_t* c) {
    if (T >= t_obs) c[0]++;
    if (fabs(T) >= fabs(t_obs)) c[1]++;
    if (T == t_obs || fabs(T - t_obs) <= tau || fabs(T) == fabs(t_obs) ||
        fabs(fabs(T) - fabs(t_obs)) <= tau)
        c[2]++;
}

/* ------------------------------------------------------------------------- */
/* Permutation loop, Alg. 1 step 5.                        */
/* ------------------------------------------------------------------------- */
typedef struct {
    const double* Z;
    int64_t N, d, n_x;
    uint64_t seed;
    uint32_t s;
    uint64_t b0, b1, b_base;
    double t_obs, tau;
    uint64_t counts[3];
    double* stats;
} perm_job;

static void* perm_worker(void* arg) {
    perm_job* jb = (perm_job*)arg;
    uint8_t* g = (uint8_t*)malloc((size_t)jb->N);
    double st[5];
    for (uint64_t b = jb->b0; b < jb->b1; ++b) {
        orc_perm_set(jb->seed, jb->s, (uint32_t)b, jb->N, jb->n_x, g);
        orc_group_stats(jb->Z, jb->N, jb->d, jb->n_x, g, st);
        tally(st[4], jb->t_obs, jb->tau, jb->counts);
        if (jb->stats) {
            double* o = jb->stats + 3 * (b - jb->b_base);
            o[0] = st[0];
            o[1] = st[1];
            o[2] = st[4];
        }
    }
    free(g);
    return NULL;
}

void orc_permtest(const double* Z, int64_t N, int64_t d, int64_t n_x, uint64_t seed, uint32_t s,
                  uint64_t b_begin, uint64_t b_end, double t_obs, double tau, int nthreads,
                  uint64_t* counts, double* stats) {
    if (b_end <= b_begin) return;
    if (nthreads < 1) nthreads = 1;
    uint64_t nb = b_end - b_begin;
    if ((uint64_t)nthreads > nb) nthreads = (int)nb;
    perm_job* jobs = (perm_job*)calloc((size_t)nthreads, sizeof(perm_job));
    pthread_t* th = (pthread_t*)calloc((size_t)nthreads, sizeof(pthread_t));
    for (int t = 0; t < nthreads; ++t) {
        perm_job* jb = &jobs[t];
        jb->Z = Z; jb->N = N; jb->d = d; jb->n_x = n_x; jb->seed = seed; jb->s = s;
        jb->b0 = b_begin + nb * (uint64_t)t / (uint64_t)nthreads;
        jb->b1 = b_begin + nb * (uint64_t)(t + 1) / (uint64_t)nthreads;
        jb->b_base = b_begin;
        jb->t_obs = t_obs; jb->tau = tau; jb->stats = stats;
        pthread_create(&th[t], NULL, perm_worker, jb);
    }
    for (int t = 0; t < nthreads; ++t) {
        pthread_join(th[t], NULL);
        for (int k = 0; k < 3; ++k) counts[k] += jobs[t].counts[k];
    }
    free(jobs);
    free(th);
}

/* ------------------------------------------------------------------------- */
/* Exhaustive enumeration of all C(N, n_x) relabelings.      */
/* Lexicographic combinations idx[0] < ... < idx[n_x-1].                       */
/* ------------------------------------------------------------------------- */
int64_t orc_exhaustive(const double* Z, int64_t N, int64_t d, int64_t n_x, double t_obs,
                       double tau, uint64_t* counts) {
    if (n_x < 1 || n_x >= N || N > 40) return 0;
    double comb = 1.0;
    for (int64_t k = 0; k < n_x; ++k) comb = comb * (double)(N - k) / (double)(k + 1);
    if (comb > 2147483647.0) return 0;
    int64_t* idx = (int64_t*)malloc(sizeof(int64_t) * (size_t)n_x);
    uint8_t* g = (uint8_t*)malloc((size_t)N);
    for (int64_t k = 0; k < n_x; ++k) idx[k] = k;
    int64_t total = 0;
    double st[5];
    for (;;) {
        memset(g, 0, (size_t)N);
        for (int64_t k = 0; k < n_x; ++k) g[idx[k]] = 1;
        orc_group_stats(Z, N, d, n_x, g, st);
        tally(st[4], t_obs, tau, counts);
        ++total;
        int64_t k = n_x - 1;
        while (k >= 0 && idx[k] == N - n_x + k) --k;
        if (k < 0) break;
        ++idx[k];
        for (int64_t q = k + 1; q < n_x; ++q) idx[q] = idx[q - 1] + 1;
    }
    free(idx);
    free(g);
    return total;
}

double orc_pvalue(uint64_t exceed, uint64_t B) {
    return (1.0 + (double)exceed) / ((double)B + 1.0);
}
