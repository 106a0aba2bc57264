/*
 * hap.h — C ABI of libhap.so, the B200 (sm_100a) implementation of the hot path of the
 * Householder-aligned permutation test (Kato et al., arXiv 2605.08048).
 *
 * Citations: "PAPER.md:L" = line L of the paper's LaTeX source (section / equation /
 * algorithm named alongside); "DESIGN.md Rk" = reading k recorded in DESIGN.md where the
 * paper is silent.
 *
 * Conventions (all entry points):
 *  - Plain C types only.  `stream` is a cudaStream_t passed as void* (NULL = legacy
 *    default stream).  Every call validates its arguments on the host, enqueues its work
 *    on `stream` and returns without synchronising.
 *  - Pointers marked [device] must be device (or managed) memory, [host] host memory,
 *    [any] either (host memory is copied in on `stream` by the library).  The caller owns
 *    every pointer it passes; the library owns only its context workspace.
 *  - Errors: argument / shape errors are returned synchronously as hap_status; data
 *    errors found on the device (ZeroVector, DegenerateMean) are written to the device
 *    hap_align_info.status, make every later kernel of that test a no-op, and are
 *    returned by hap_sync().  No C++ exception crosses the ABI.  hap_last_error() gives
 *    a message for the last non-OK status of a context.
 *  - A context is bound to one device and is not thread-safe; use one per host thread.
 *  - The alignment kernel (hap_align and the batch's alignment waves) is a cooperative grid
 *    with a software grid barrier; two such grids sharing a device could each hold part of
 *    the SMs and wait for the other.  Every alignment launch of the PROCESS on a device is
 *    therefore ordered after the previous one (an event chain across all contexts and
 *    streams): a hap_align on one stream also waits for the alignments already issued on
 *    other streams, and the calls cannot be captured into a CUDA graph.
 *  - Requires sm_100 (B200).  There is no CPU fallback: hap_create fails with
 *    HAP_E_UNSUPPORTED_ARCH elsewhere.
 */
#ifndef HAP_H
#define HAP_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HAP_ABI_VERSION 1

#if defined(__GNUC__)
#define HAP_API __attribute__((visibility("default")))
#else
#define HAP_API
#endif

typedef struct hap_ctx_s* hap_ctx;

typedef enum {
    HAP_OK = 0,
    HAP_E_INVALID_ARG = 1,
    HAP_E_DIM_MISMATCH = 2,
    HAP_E_ZERO_VECTOR = 3,      /* a raw row has ||h|| < 1e-12 (R3) */
    HAP_E_DEGENERATE_MEAN = 4,  /* ||xbar|| or ||ybar|| < 1e-12 (R3) */
    HAP_E_MIXED_SHAPES = 5,
    HAP_E_OOM = 6,
    HAP_E_CUDA = 7,
    HAP_E_UNSUPPORTED_ARCH = 8, /* device is not sm_100 */
    HAP_E_NOT_ALIGNED = 9       /* hap_permtest before any successful hap_align */
} hap_status;

typedef enum {
    HAP_ALIGN_HOUSEHOLDER = 0, /* x' = x - 2u(u^T x) on X */
    HAP_ALIGN_NONE = 1         /* naive baseline: pool the normalised clouds unreflected */
} hap_align_mode;

/* Result of hap_align, written to DEVICE memory (sizeof(hap_align_info) bytes, 8-byte
 * aligned) so that hap_permtest can consume it without a host round trip. */
typedef struct {
    int64_t n_x, n_y, d;      /* n, m, d of PAPER.md:121-128 */
    int64_t n_pad, d_pad;     /* padded GEMM extents (K = n_pad rows, d_pad columns) */
    int32_t is_identity;      /* 1 if ||mu_x - mu_y|| < 1e-9 (no reflection; R3) or mode NONE */
    int32_t status;           /* hap_status of the device-side data checks */
    int64_t bad_row;          /* pooled row index of a ZeroVector error, else -1 */
    double r_x, r_y;          /* MRLs ||xbar||, ||ybar|| in fp64 (Eq. 8; r(X') = r(X), :161) */
    double logk_x, logk_y;    /* L(r) = log kappa-hat(r) = -log v (Eq. 9; R1, R4) */
    double t_obs;             /* T_obs = log v(X') - log v(Y) = logk_y - logk_x (Eq. 10), fp64 */
    /* the observed split evaluated through the mask-GEMM + epilogue path (row 0 of every
     * tile, D7): the value hap_permtest compares each T_b against, so that a
     * permutation that redraws the observed split ties it bit-exactly.  Written by
     * hap_permtest (NaN until then). */
    double gemm_r_x, gemm_r_y, gemm_t_obs;
} hap_align_info;

/* One test's permutation configuration (PERM-SPEC v1, R6). */
typedef struct {
    uint64_t seed;      /* Philox key = (lo32(seed), hi32(seed)) */
    uint64_t B;         /* permutations of the whole test (informational; p uses it) */
    uint64_t b_begin;   /* this call's shard [b_begin, b_end) of [0, B); b < 2^32 */
    uint64_t b_end;
    uint32_t stream_id; /* s: third Philox counter word (pair id by default) */
    uint32_t block;     /* B0 permutations per generator/GEMM block; perf only, 0 = auto */
    int32_t pair_mode;  /* K3 CTA grouping: 0 = auto (2), 1 = cta_group::1, 2 = cta_group::2 */
    int32_t wave;       /* hap_permtest_batch: tests per alignment/generator/GEMM launch, 1..4;
                         * perf only; 0 = auto (4 with HAP_FLAG_SHARED_MASK or when every
                         * pair of the batch has N <= 2048, else 3) */
    double tie_rel;     /* tie band tau = tie_rel * (|logk_x| + |logk_y|) (R8); <= 0 -> 1e-6 */
    uint32_t flags;     /* HAP_FLAG_* */
    uint32_t reserved;
} hap_perm_cfg;

/* hap_permtest_batch only: every pair uses the SAME permutations, generator stream
 * s = cfg->stream_id (SPEC.md "shared mode").  Consecutive selected pairs
 * with equal (n_x, n_y) then share one generated mask block per launch: the generator runs
 * once per wave instead of once per pair.  Each pair is still an exact permutation test;
 * the tests are no longer independent of each other. */
#define HAP_FLAG_SHARED_MASK 1u

/* hap_permtest only: EXHAUSTIVE enumeration.  b
 * indexes the C(N, n_x) splits in colex order (b -> the combination {c_1 < .. < c_nx} with
 * b = sum_i C(c_i, i)) instead of PERM-SPEC draws; seed and stream_id are ignored.  Needs
 * C(N, n_x) < 2^32 (N <= 34) and b_end <= C(N, n_x).  Over [0, C(N, n_x)) the counts are
 * those of the exact permutation distribution, the observed split included:
 * p_exact = exceed_ge / C(N, n_x).  HAP_E_INVALID_ARG otherwise. */
#define HAP_FLAG_EXHAUSTIVE 2u

/* K3 arithmetic:
 * the statistic needs only S1 = ||sigma1||^2 and S2 = ||sigma2||^2 of the group sums, and
 * with the centred pooled rows z'_i, ||sum_{i in G_b} z'_i||^2 = m_b^T (Z' Z'^T) m_b is a
 * quadratic form in the N x N Gram matrix.  The GRAM form multiplies the mask block by
 * Z' Z'^T (bf16 hi/lo of fp64-combined sums, N_pad x N_pad) instead of Z' (N_pad x d_pad):
 * 4 N_pad^2 instead of 4 N_pad d_pad issued tensor FLOP per permutation, for N << d.
 * By default hap_permtest / hap_permtest_batch choose it per test from (n_pad, d_pad,
 * cfg->B) when it saves time (never for 2 n_pad > d_pad); HAP_FLAG_GRAM forces it
 * (needs n_pad <= 4096), HAP_FLAG_NO_GRAM forbids it.  Both forms meet the same parity
 * bar; their statistics differ in rounding only, so flag a test consistently over its
 * shards (the automatic choice uses cfg->B, the whole test's permutation count). */
#define HAP_FLAG_GRAM 4u
#define HAP_FLAG_NO_GRAM 8u

/* Exceedance counters of one test, DEVICE memory, ADDED into (caller zeroes them), so
 * shards and resumed ranges compose by summation (Eq. pvalue). */
typedef struct {
    uint64_t exceed_ge;  /* #[T_b >= T_obs]      one-sided "greater" */
    uint64_t exceed_abs; /* #[|T_b| >= |T_obs|]  two-sided (R5) */
    uint64_t flagged;    /* #[|T_b - T_obs| <= tau] near-ties (R8) */
} hap_counts;

/* ---- context ------------------------------------------------------------------- */
HAP_API int hap_abi_version(void);
/* Create a context on CUDA device `device` (fails unless it is sm_100). */
HAP_API hap_status hap_create(int device, hap_ctx* out);
HAP_API hap_status hap_destroy(hap_ctx ctx);
/* Synchronise the context's last stream; returns the first deferred error (CUDA error or
 * the device status of the last hap_align). */
HAP_API hap_status hap_sync(hap_ctx ctx);
HAP_API const char* hap_last_error(hap_ctx ctx);

/* ---- S1-S6: normalise, means, Householder axis, reflect, pool, T_obs ------------ */
/* PAPER.md §3.1 (lines 115-180) and Alg. 1 steps 1-4.
 *   X [any]  n_x*d fp32 row-major raw embeddings h (unnormalised)
 *   Y [any]  n_y*d fp32 row-major
 *   info [device] hap_align_info, written.
 * Builds, in the context workspace, the pooled aligned cloud Z = [X'; Y]
 * as the transposed bf16 hi/lo planes Zt_hi, Zt_lo (d_pad x n_pad, K contiguous) with
 * hi = bf16(z), lo = bf16(z - hi) (PAPER.md:258 precision note; R9), the total
 * t = 1^T Z (Eq. gemm) and the observed statistic r_x, r_y, logk_x,
 * logk_y, t_obs in fp64 (Alg. 1 step 4).
 * Constraints: 1 <= n_x, n_y; n_x + n_y <= 65535; 2 <= d <= 16384.
 * Kernels: pairs with d % 4 == 0, d <= 4096 and 16-byte aligned X, Y take the streaming
 * alignment (K1s: three bandwidth kernels); the others one cooperative kernel, and those
 * cooperative launches are ordered one after the other on a device across all contexts and
 * streams (an event chain; concurrent cooperative grids could wait on each other's SMs). */
HAP_API hap_status hap_align(hap_ctx ctx, const float* X, int64_t n_x, const float* Y, int64_t n_y,
                     int64_t d, hap_align_mode mode, hap_align_info* info, void* stream);

/* ---- S7-S9: permutation masks, mask-GEMM, statistic, exceedance counts ----------- */
/* PAPER.md §3.2 (lines 201-243), Alg. 2: for each b in
 * [cfg->b_begin, cfg->b_end) draws the PERM-SPEC v1 group-1 set G_b, forms sigma1 =
 * sum_{i in G_b} z_i with the tcgen05 mask-GEMM, sigma2 = t - sigma1,
 * r1 = ||sigma1||/n_x, r2 = ||sigma2||/n_y, T_b = L(r2) - L(r1) and ADDS
 * the three comparisons against T_obs into *counts, T_obs being evaluated through the
 * same GEMM path on the observed split (written to info->gemm_*).  Uses the Z from the
 * last hap_align on this context; `info` must be that call's info (device, updated).
 *   counts [device] hap_counts, added into.
 *   stats  [device] optional (NULL = none): (b_end-b_begin)*3 doubles {r1, r2, T_b}. */
HAP_API hap_status hap_permtest(hap_ctx ctx, hap_align_info* info, const hap_perm_cfg* cfg,
                        hap_counts* counts, double* stats, void* stream);

/* ---- many word pairs ------------------------------------------------------------ */
/* Varlen batch of P independent tests (configs 4/5): pair p has X rows
 * X_packed[cu_nx[p] .. cu_nx[p+1]) and Y rows Y_packed[cu_ny[p] .. cu_ny[p+1]).
 * The selected pairs are processed largest first (equal shapes adjacent; the results do not
 * depend on the order) and grouped into waves of cfg->wave tests (see hap_perm_cfg)
 * that share one generator and one mask-GEMM launch; waves alternate between two internal
 * lanes (own workspaces and streams, forked from and joined back to `stream`), so one
 * wave's alignment and mask generation overlap the previous wave's mask-GEMM.  Pair p uses
 * generator stream cfg->stream_id + p (cfg->stream_id for all with HAP_FLAG_SHARED_MASK).  Shape errors of any selected pair
 * are returned before anything is enqueued.
 *   X_packed, Y_packed [device, or both host]: host inputs (pinned for overlap) are copied
 *            per pair into the wave's workspaces on internal copy streams, so the copies of
 *            one wave overlap the other lane's kernels (the end-to-end path of bench.py); the
 *            host buffers must stay valid and unchanged until the work enqueued on `stream`
 *            has completed (the copies are asynchronous);
 *   cu_nx, cu_ny [host] int64[P+1] prefix offsets.
 *   pair_sel [host] optional list of the pairs this call handles (NULL = all P); the
 *            others' infos/counts are left untouched (used for multi-GPU sharding).
 *   cfg->stream_id is the base s; pair p uses s = stream_id + p.
 *   infos [device] P hap_align_info; counts [device] P hap_counts (added into).
 * A pair with a data error has its own infos[p].status set; the batch continues. */
HAP_API hap_status hap_permtest_batch(hap_ctx ctx, int64_t P, const float* X_packed, const int64_t* cu_nx,
                              const float* Y_packed, const int64_t* cu_ny, int64_t d,
                              hap_align_mode mode, const hap_perm_cfg* cfg,
                              const int64_t* pair_sel, int64_t n_sel, hap_align_info* infos,
                              hap_counts* counts, void* stream);

/* p = (1 + c)/(B + 1)  (Eq. pvalue). */
HAP_API double hap_pvalue(uint64_t exceed, uint64_t B);
/* Exact p-value of an exhaustive enumeration (HAP_FLAG_EXHAUSTIVE over all `total` =
 * C(N, n_x) splits, the observed one included): p = c / total.
 * NaN when total = 0. */
HAP_API double hap_p_exact(uint64_t exceed, uint64_t total);

/* ---- live profiling (bench.py) ---------------------------------------------------- */
/* Phases of the hot path, for per-kernel timing and launch counting. */
typedef enum {
    HAP_PHASE_ALIGN = 0,     /* K1 kernels (S1-S5) */
    HAP_PHASE_OBSERVED = 1,  /* reserved (S6 runs inside K1 and, through the GEMM, in K3) */
    HAP_PHASE_PERMGEN = 2,   /* K2 permutation generator (S7) */
    HAP_PHASE_MASKGEMM = 3,  /* K3 mask-GEMM + statistic epilogue (S8-S9) */
    HAP_NUM_PHASES = 4
} hap_phase;
/* enable != 0: every later launch of the context is bracketed by CUDA events recorded on
 * its own stream (adds host work; leave off when timing whole steps).  enable >= 2 also
 * serialises the generator onto the caller's stream so the phase times do not overlap. */
HAP_API hap_status hap_profile(hap_ctx ctx, int enable);
/* Synchronises the recorded events and returns, per phase, the summed device time (ms,
 * [host] double[HAP_NUM_PHASES]) of the launches timed since the last reset and the number
 * of kernel launches issued ([host] int64_t[HAP_NUM_PHASES], counted whether or not timing
 * is enabled).  reset != 0 clears both. */
HAP_API hap_status hap_profile_read(hap_ctx ctx, double* ms, int64_t* launches, int reset);

/* Timeline of the launches timed since the last read/reset (profiling on): out [host]
 * max_n * 3 doubles {phase, start_us, end_us} relative to the first recorded launch, in
 * record order; *n receives the count.  Consumes the records (like hap_profile_read). */
HAP_API hap_status hap_profile_timeline(hap_ctx ctx, double* out, int64_t max_n, int64_t* n);

/* Kernel spans: with enable != 0 every kernel launched afterwards (by this context and its
 * batch lanes) records {first CTA entry, last CTA exit} with the device's global timer, so
 * concurrent launches on different streams can be laid on one timeline without the event
 * records of hap_profile between them.  hap_profile_spans_read synchronises the device and
 * writes, per launch in issue order, [host] out[3k] = phase + HAP_NUM_PHASES * lane (lane 0
 * = this context, 1 and 2 = batch lanes), out[3k+1], out[3k+2] = start, end in us relative
 * to the earliest start (-1 for a kernel that returned before the exit stamp); *n = number
 * of launches recorded (at most 8192 per read), then resets. */
HAP_API hap_status hap_profile_spans(hap_ctx ctx, int enable);
HAP_API hap_status hap_profile_spans_read(hap_ctx ctx, double* out, int64_t max_n, int64_t* n);

/* ---- introspection for parity tests (same kernels as the hot path) -------------- */
/* PERM-SPEC v1 sets for b in [b_begin, b_begin+count): out [device] count*N uint8
 * membership (1 = group 1), produced by the product's generator kernel. */
HAP_API hap_status hap_perm_sets(hap_ctx ctx, uint64_t seed, uint32_t stream_id, uint64_t b_begin,
                         int64_t count, int64_t N, int64_t n_x, uint8_t* out, void* stream);
/* Parity introspection of HAP_FLAG_EXHAUSTIVE: out [device] count*N uint8, row r = the
 * indicator of combination b_begin + r of C(N, n_x) (colex unranking); N <= 64,
 * b_begin + count <= C(N, n_x) < 2^32. */
HAP_API hap_status hap_comb_sets(hap_ctx ctx, uint64_t b_begin, int64_t count, int64_t N, int64_t n_x,
                                 uint8_t* out, void* stream);
/* C(N, k) as uint64 (0 when it exceeds 2^64 - 1 or k > N). */
HAP_API uint64_t hap_n_choose_k(int64_t N, int64_t k);
/* Copy out the pooled workspace of the last hap_align: zhi, zlo [device] d_pad*n_pad
 * uint16, the transposed bf16 planes Zt of the CENTRED cloud (row c holds column c of
 * Z - 1 m^T over the n_pad pooled rows, zero padded), so z[i][c] ~ hi + lo + m[c];
 * t [device] d_pad fp64 = N m + column sums of (hi + lo);  m [device] d_pad fp64 centre
 * (DESIGN.md "Numerics"). */
HAP_API hap_status hap_export_pooled(hap_ctx ctx, uint16_t* zhi, uint16_t* zlo, double* t, double* m,
                                     void* stream);

#ifdef __cplusplus
}
#endif
#endif /* HAP_H */
