/*
 * hap_oracle.h — fp64 CPU ORACLE for the Householder-aligned permutation test
 * (arXiv 2605.08048).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load this library.  It shares no code,
 * header, table or constant generator with the CUDA path (paper_2605_08048_b200/csrc).
 *
 * Every function follows the paper step by step in its own notation; "PAPER.md:L"
 * cites a line of the paper's LaTeX source, "SPEC.md:L" the third-party spec,
 * "SURVEY.md §8c" the PERM-SPEC v1 reading recorded in DESIGN.md.
 *
 * Pins (tests/test_oracle.py): Random123 KATs (philox), SURVEY golden sets (perm_set,
 * main stream) and sets decided by Lemire rejections from an independent pure-Python
 * generator, with their rejection counts (perm_set side stream, the redraw count;
 * tests/golden/gen_permspec_rejections.py), FY chi^2 uniformity, Householder identities +
 * App. D closed form (align), SPEC worked numbers + brute-force exhaustive enumeration
 * (stats, exhaustive), MC-vs-exhaustive within 3 SE (permtest), and the near-tie counter
 * on a pool whose ties are fixed by combinatorics (tally's `flagged`, tests/tiecase.py).
 * No function is "parity unpinned".
 */
#ifndef HAP_ORACLE_H
#define HAP_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (same meaning as the product's, own numbering) */
#define ORC_OK 0
#define ORC_E_ARG 1
#define ORC_E_ZERO_VECTOR 2
#define ORC_E_DEGENERATE_MEAN 3

/* Philox4x32-10 (Salmon et al. 2011): out = philox(ctr, key). */
void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);

/* PERM-SPEC v1 (DESIGN.md "Readings" R6): partial forward
 * Fisher–Yates over n_x steps keyed by Philox.  Writes in_g1[0..N-1] (1 = row
 * assigned to group 1, i.e. the X side) and returns the number of side-stream
 * redraws that happened (>= 0), or -1 on bad arguments. */
int orc_perm_set(uint64_t seed, uint32_t s, uint32_t b, int64_t N, int64_t n_x,
                 uint8_t* in_g1);

/* Householder alignment, PAPER.md:115-161 (§3.1 Eqs. 2,5,6,7) + Alg. 1 steps 1-3
 * (PAPER.md:660-670).  X: n_x*d fp32 raw rows, Y: n_y*d.  mode 0 = Householder,
 * 1 = none (naive baseline).  Writes Z ((n_x+n_y)*d, rows 0..n_x-1 = X'),
 * u (d; zero if identity) and info[] = {norm_xbar, norm_ybar, is_identity,
 * bad_row}. Returns ORC_OK / ORC_E_ZERO_VECTOR / ORC_E_DEGENERATE_MEAN. */
int orc_align(const float* X, int64_t n_x, const float* Y, int64_t n_y, int64_t d, int mode,
              double* Z, double* u, double* info);

/* log kappa-hat(r) with kappa-hat = r(d-r^2)/(1-r^2) (Banerjee),
 * r clamped to [0, 1-1e-9]. L(0) = -inf. */
double orc_logkappa(double r, int64_t d);

/* Group statistic of one split, PAPER.md:164-186 (Eqs. 8-11) / Alg. 1 lines
 * sigma1 = sum_{i in G} z_i, sigma2 = sum_{i not in G} z_i, both
 * summed directly in ascending i; r = ||sigma||/n; T = L(r2) - L(r1) (= log v(G1) -
 * log v(G2)).  out[5] = {r1, r2, L1, L2, T}. */
void orc_group_stats(const double* Z, int64_t N, int64_t d, int64_t n_x, const uint8_t* in_g1,
                     double* out);

/* Monte Carlo permutation loop, Alg. 1 step 5 with PERM-SPEC v1
 * sets for b in [b_begin, b_end), on nthreads host threads.  counts[3] +=
 * {#[T_b >= t_obs], #[|T_b| >= |t_obs|], #[near-tie]} with near-tie =
 * |T_b - t_obs| <= tau or ||T_b| - |t_obs|| <= tau (R8).  stats
 * (optional, may be NULL): (b_end-b_begin)*3 doubles {r1, r2, T}. */
void orc_permtest(const double* Z, int64_t N, int64_t d, int64_t n_x, uint64_t seed, uint32_t s,
                  uint64_t b_begin, uint64_t b_end, double t_obs, double tau, int nthreads,
                  uint64_t* counts, double* stats);

/* Exhaustive enumeration of all C(N, n_x) splits: counts[3] as
 * above, returns C(N, n_x) (or 0 if it exceeds 2^31). */
int64_t orc_exhaustive(const double* Z, int64_t N, int64_t d, int64_t n_x, double t_obs,
                       double tau, uint64_t* counts);

/* p = (1 + c)/(B + 1), PAPER.md:187-191 (Eq. pvalue). */
double orc_pvalue(uint64_t exceed, uint64_t B);

#ifdef __cplusplus
}
#endif
#endif
