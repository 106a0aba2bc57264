// k_maskgemm.cu — K3: tcgen05/TMEM mask-GEMM with the statistic epilogue
// (DESIGN.md "Kernels" K3; S8 + S9 of SURVEY.md §8a).
//
//   sigma1_b = sum_{i in G_b} z_i  as one row of  U' = M_blk Z  (0/1 mask instead of the
//   paper's +-1 signs, PAPER.md:205-220 Eq. gemm; R7).  Z is held centred as
//   Z - 1 m^T in two bf16 planes (hi, lo), so the accumulator is
//       acc[b, c] = sum_k M[b,k] Zhi[k,c] + sum_k M[b,k] Zlo[k,c]        (fp32, TMEM)
//   and sigma1 = a + acc, sigma2 = t - sigma1 = b - acc  with a = n_x m, b = t - a
//   ("without a second GEMM").
//   r1 = ||sigma1||/n_x, r2 = ||sigma2||/n_y
//   T_b = L(r2) - L(r1)                       (Alg. 2)
//   counts += [T_b >= T_obs], [|T_b| >= |T_obs|], near-tie   (R8)
// No B x d intermediate reaches HBM: acc lives in TMEM; only 8 bytes per (row, d-chunk)
// of fp32 partial sums are exchanged between the CTAs that share a tile.
//
// Work: a launch covers `ntiles` tiles of R = 128*kPair mask rows; row 0 of every tile is
// the OBSERVED split {0..n_x-1}, so T_obs is evaluated through exactly the same MMA +
// epilogue path as every permutation (D7) with no extra launch or dependency.
// Schedule: the (tile, column) space is cut into one equal contiguous range per CTA pair
// (multiples of 32 columns), each range into pieces at tile boundaries and at 256 columns
// (the accumulator width); MMA time is proportional to the width, so the pairs finish
// together.  A pair walks its pieces in order; every piece runs the full K loop.
//
// kPair = 2 (default): a 2-CTA cluster runs tcgen05.mma.cta_group::2 with M = 256: each CTA
// holds 128 mask rows (A) and half of the chunk's columns (B), so each SM streams half of
// the Z~ tile; 3-stage TMA ring of 48 KB (the rest of the SM's smem is left to K2).  kPair = 1: one CTA, M = 128, 2 stages of 80 KB.
// Warps: 0 TMA producer, 1 MMA issuer (leader CTA) + TMEM owner, 2-5 epilogue (thread =
// TMEM lane = one mask row).  The accumulator is double-buffered in TMEM (2 x 256 columns)
// so unit i+1's MMAs overlap unit i's epilogue.  The last CTA to finish a unit of a tile
// (atomic ticket) sums the tile's piece partials in column order (deterministic), forms the
// statistics and counts.
#include <cmath>

#define HAP_CHECK_TU 3
#include "hap_device.cuh"
#include "hap_internal.h"

namespace hap {
namespace {

constexpr int kThreads = 192;
constexpr uint32_t kTmemCols = 512;
constexpr int kStageA = kTileM * 128;  // 16 KB: 128 rows x 64 bf16
constexpr int kQ = 6;                    // piece queue: the leader's producer publishes the
                                         // pair's pieces to every role of both CTAs

#ifndef HAP_K3_STAGES
#define HAP_K3_STAGES 3
#endif
template <int kPair>
struct Cfg {
    // 3 x 48 KB leaves room for the generator (K2) CTAs to co-reside on every SM
    static constexpr int kStages = kPair == 2 ? HAP_K3_STAGES : 2;
    static constexpr int kBRows = kChunkN / kPair;   // B rows (d-columns) held per CTA
    static constexpr int kStageB = kBRows * 128;     // one plane
    static constexpr int kStageBytes = kStageA + 2 * kStageB;
    static constexpr size_t kSmem = (size_t)kStages * kStageBytes + 1024 + 2048;
};


// timing-only switches exist only in the development build (-DHAP_EXPERIMENTS); in the
// release library they are the constant 0 and the skipped-work paths are compiled out
#ifdef HAP_EXPERIMENTS
#define K3_EXP(g) ((g).exp)
#else
#define K3_EXP(g) 0
#endif

__device__ __forceinline__ long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return (long long)t;
}
// EXPERIMENT (exp bit 16): per (CTA, local unit i, event) timestamps
#define K3_STAMP(i, ev)                                                                      \
    do {                                                                                     \
        if ((K3_EXP(g) & 16) && g.stamps && (i) < 8)                                             \
            g.stamps[((size_t)blockIdx.x * 8 + (i)) * 8 + (ev)] = gtimer();                  \
    } while (0)

struct RowStat {
    double r1, r2, T, e;  // e: error bound of T (R14)
};

// q(r) = kappa-hat(r) = r (d - r^2)/(1 - r^2) with r clamped (R1, R4); L = log q
__device__ __forceinline__ double kappa_hat(double r, double d) {
    if (r > 1.0 - 1e-9) r = 1.0 - 1e-9;
    if (r <= 0.0) return 0.0;
    const double r2 = r * r;
    return r * (d - r2) / (1.0 - r2);
}

// log(q2/q1) = L(r2) - L(r1): near 1 the ratio goes through log1p of q2/q1 - 1 (formed in
// fp64) in fp32 - its error, ~1e-7 of T's natural scale, is far below the tie band, and it
// keeps the finalize off the fp64 pipe, which the running MMAs slow down; a ratio far from
// 1 (|T| > 0.4) takes the fp64 log (fp32 would round q2/q1 - 1 to -1 once |T| > 16)
// the rare far-from-1 ratio: an out-of-line fp64 log, so the common path does not evaluate
// it under a predicate
__device__ __noinline__ double log_far(double q1, double q2) { return log(q2 / q1); }
__device__ __forceinline__ double log_ratio(double q1, double q2) {
    if (q1 == 0.0) return q2 == 0.0 ? 0.0 : INFINITY;  // r1 = 0: T = +inf; both 0: T := 0 (R4)
    const double x = (q2 - q1) / q1;
    if (fabs(x) < 0.5) return (double)log1pf((float)x);
    return log_far(q1, q2);
}

// Half-width of the interval that holds L(r) of the exact statistic, given the GPU's
// estimate r and its error bound delta (R14): 2 delta |L'(r)| (twice the linear
// term, L' = 1/r + 2r/(1 - r^2) - 2r/(d - r^2) <= 1/r + 2r/(1 - r^2)), formed in fp32 with a
// 1 % allowance; unbounded (every decision flagged) when the interval reaches r = 0 or the
// clamp at 1 - 1e-9; groups of one are exact (delta = 0).  Branch-free: the finalize runs
// beside the MMAs, and a data-dependent branch to an exact near-clamp interval cost ~6 % of
// the mask-GEMM (profiles/r02_experiments/e31_eb.log).
__device__ __forceinline__ double l_width(double r, float delta) {
    const float rf = (float)r;
    const float w = 2.02f * delta * (__frcp_rn(rf) + 2.f * rf * __frcp_rn(1.f - rf * rf));
    const bool unbounded = r <= 2.0 * (double)delta || r + 2.0 * (double)delta >= 1.0 - 1e-9;
    return delta == 0.f ? 0.0 : (unbounded ? (double)INFINITY : (double)w);
}

// Gram form (k_gram.cu): error of r from the form's own roundings, on top of the planes'
// representation error that both forms share (R14).  Both S1 and S2 are sums over the MASKED
// group's entries (S_g = S_gc + sum_j m_bj (U_bj +- 2 alpha/beta_j), U_bj = sum_k m_bk G'_jk),
// so both carry the error of n^2 Gram entries with n = n_x, the mask's group: the bf16 hi/lo
// rounding (2^-17 relative, independent signs: ~ sqrt of the sum of squares, entries <=
// |z'|^2 <= 4, off-diagonal ones ~ 1/sqrt(d) of that) and the fp32 accumulation of each U_bj
// over n terms (2^-24 per add); 8x margin as in R14; dr_g = dS / (2 n_g^2 r_g) (the complement
// group's r inherits the masked group's dS: a small Y next to a large X is wide).
__device__ __forceinline__ float gram_delta(float n_mask, float n_g, float d, double r) {
    const float dS = 8.f * 4.f * sqrtf(1.f + n_mask / d) * (0x1p-17f * sqrtf(n_mask) + 0x1p-22f * n_mask);
    return 1.01f * dS / (2.f * n_g * n_g * fmaxf((float)r, 1e-6f));
}

// statistic of a tile row from its accumulated sums S1 = |sigma1|^2, S2 = |sigma2|^2;
// T = L(r2) - L(r1) = log(q(r2)/q(r1)); eps = the test's representation-error scale
__device__ __forceinline__ RowStat row_stat(const GemmArgs& g, const GemmTest& T, double S1, double S2,
                                            double eps) {
    RowStat s;
    // a group of one unit vector has MRL exactly 1 (Eq. 8); the GEMM's
    // 1 +- 1e-7 would fall on either side of the clamp at 1 - 1e-9 (R4)
    s.r1 = T.n_x == 1 ? 1.0 : sqrt(fmax(S1, 0.0)) / (double)T.n_x;
    s.r2 = T.n_y == 1 ? 1.0 : sqrt(fmax(S2, 0.0)) / (double)T.n_y;
    const double d = (double)g.d;
    s.T = log_ratio(kappa_hat(s.r1, d), kappa_hat(s.r2, d));
    // |r_gpu - r| <= 8 eps / sqrt(n d) per group (R14: the row errors average over the n
    // rows and the d coordinates; measured <= 1/4 of this bound at every tested shape)
    const float k = 1.01f * 8.f * (float)eps * rsqrtf((float)d);
    float d1 = k * rsqrtf((float)T.n_x), d2 = k * rsqrtf((float)T.n_y);
    if (T.gram) {  // + the Gram form's own rounding
        d1 += gram_delta((float)T.n_x, (float)T.n_x, (float)d, s.r1);
        d2 += gram_delta((float)T.n_x, (float)T.n_y, (float)d, s.r2);
    } else {
        // + the fp32 accumulation of the masked sums (R14b): sigma1 = a + acc and, through
        // the complement, sigma2 = b - acc carry the accumulator's rounding over the n_x
        // masked rows (2 n_x / 16 MMA steps, |acc_c| ~ sqrt(n_x / d)): 8x margin ->
        // |dr_g| <= 2^-22 n_x / (sqrt(d) n_g), which matters for a small group beside a large one
        const float ka = 1.01f * 0x1p-22f * (float)T.n_x * rsqrtf((float)d);
        d1 += ka / (float)T.n_x;
        d2 += ka / (float)T.n_y;
    }
    s.e = l_width(s.r1, T.n_x == 1 ? 0.f : d1) + l_width(s.r2, T.n_y == 1 ? 0.f : d2);
    return s;
}

// Last CTA of a tile: every thread evaluates the observed row (row 0, identical result in
// all threads: same partials, same order) and its own permutation rows etid, etid + 128.
// All partial loads of the three rows are issued together (one L2 round trip per 8 pieces);
// the piece partials are summed in ascending slot order (deterministic).
__device__ void finalize_tile(const GemmArgs& g, const GemmTest& T, int tile, int lt, int np, int etid,
                              unsigned* s_cnt, double S1c, double S2c, double tau, double eps, int unit = -1) {
#define FIN_STAMP(ev) do { if (unit == 3 && etid == 0) K3_STAMP(6, ev); } while (0)
    FIN_STAMP(0);
    const int R = g.rows_per_tile;
    if (etid < 3) s_cnt[etid] = 0u;
    constexpr int kRows = 3;  // row 0, etid, etid + 128 (R <= 256)
    const int rows[kRows] = {0, etid, etid + 128};
    double S1[kRows], S2[kRows];
#pragma unroll
    for (int k = 0; k < kRows; ++k) {
        S1[k] = S1c;
        S2[k] = S2c;
    }
    const float2* p = g.part + (size_t)tile * g.max_slots * R;
    for (int c0 = 0; c0 < np; c0 += 8) {
        float2 v[kRows][8];
#pragma unroll
        for (int c = 0; c < 8; ++c)
#pragma unroll
            for (int k = 0; k < kRows; ++k)
                v[k][c] = (c0 + c < np && rows[k] < R) ? __ldcg(p + (size_t)(c0 + c) * R + rows[k])
                                                        : make_float2(0.f, 0.f);
#pragma unroll
        for (int c = 0; c < 8; ++c)
#pragma unroll
            for (int k = 0; k < kRows; ++k) {
                S1[k] += (double)v[k][c].x;
                S2[k] += (double)v[k][c].y;
            }
    }
    FIN_STAMP(1);
    const RowStat o = row_stat(g, T, S1[0], S2[0], eps);
    FIN_STAMP(2);
    if (lt == 0 && etid == 0) {
        T.info->gemm_r_x = o.r1;
        T.info->gemm_r_y = o.r2;
        T.info->gemm_t_obs = o.T;
    }
    const double t_obs = o.T;
    const int lane = etid & 31;
    named_bar_sync(1, 128);  // s_cnt cleared
    FIN_STAMP(3);
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        const int row = rows[1 + j];
        const int perm = lt * (R - 1) + row - 1;
        const bool valid = row >= 1 && row < R && perm < T.count;
        const RowStat st = row_stat(g, T, S1[1 + j], S2[1 + j], eps);
        const double Tb = st.T;
        const bool ge = valid && (Tb >= t_obs);
        const bool ab = valid && (fabs(Tb) >= fabs(t_obs));
        // near-ties (R8), the band widened by both statistics' error bounds (R14): every
        // permutation whose decision the kernel's precision cannot certify is flagged
        const double band = tau + st.e + o.e;
        const bool fl = valid && (Tb == t_obs || fabs(Tb - t_obs) <= band || fabs(Tb) == fabs(t_obs) ||
                                  fabs(fabs(Tb) - fabs(t_obs)) <= band);
        const uint32_t bge = __ballot_sync(0xffffffffu, ge);
        const uint32_t bab = __ballot_sync(0xffffffffu, ab);
        const uint32_t bfl = __ballot_sync(0xffffffffu, fl);
        if (lane == 0) {  // per-CTA totals first: 3 global atomics per tile
            if (bge) atomicAdd(s_cnt + 0, (unsigned)__popc(bge));
            if (bab) atomicAdd(s_cnt + 1, (unsigned)__popc(bab));
            if (bfl) atomicAdd(s_cnt + 2, (unsigned)__popc(bfl));
        }
        if (T.stats && valid) {
            double* out = T.stats + 3 * (int64_t)perm;
            out[0] = st.r1;
            out[1] = st.r2;
            out[2] = Tb;
        }
    }
    FIN_STAMP(4);
    named_bar_sync(1, 128);
    FIN_STAMP(5);
    if (etid < 3 && s_cnt[etid])
        atomicAdd(reinterpret_cast<unsigned long long*>(T.counts) + etid, (unsigned long long)s_cnt[etid]);
    if (etid == 0) g.tile_done[tile] = 0;  // ready for the next launch
    FIN_STAMP(6);
#undef FIN_STAMP
}

// finalize queue (GemmArgs::fq): [0] pop counter, [1] push counter, [2] exit counter,
// [4 + k] the k-th published entry: tile + 1, or -(tile + 1) for a failed test's tile
__device__ __forceinline__ void fq_push(const GemmArgs& g, int v) {
    __threadfence();  // the tile's partials (all pieces, fenced before their tickets) first
    const int pos = atomicAdd(g.fq + 1, 1);
    atomicExch(g.fq + 4 + pos, v);
}

// test of a wave tile (the tests' tiles are contiguous, in test order)
__device__ __forceinline__ int test_of(const GemmArgs& g, int tile) {
    int ti = 0;
    while (ti + 1 < g.G && tile >= g.t[ti + 1].tile0) ++ti;
    return ti;
}
// a test whose data failed (ZeroVector, DegenerateMean) is skipped by every role alike
__device__ __forceinline__ bool test_failed(const GemmTest& T) {
    return *reinterpret_cast<const volatile int*>(&T.info->status) != HAP_OK;
}

#ifndef HAP_K3_MAXNREG
#define HAP_K3_MAXNREG 168
#endif
template <int kPair>
__global__ void __maxnreg__(HAP_K3_MAXNREG)
    k3_maskgemm(const __grid_constant__ GemmMaps maps, const GemmArgs g) {
    using C = Cfg<kPair>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::kStages * C::kStageBytes);
    uint64_t* empty = full + C::kStages;
    uint64_t* tfull = empty + C::kStages;
    uint64_t* tempty = tfull + 2;
    uint64_t* qfull = tempty + 2;   // [kQ] piece index published (both CTAs)
    uint64_t* qempty = qfull + kQ;  // [kQ] every consumer has read it (leader)
    int* s_q = reinterpret_cast<int*>(qempty + kQ);  // [kQ] piece indices (-1: no more)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(s_q + kQ);
    int* s_last = reinterpret_cast<int*>(tmem_slot + 1);
    unsigned* s_cnt = tmem_slot + 4;  // [3] per-tile counts of the finalize
    double* s_tc = reinterpret_cast<double*>(tmem_slot + 8);  // [kMaxWave][4] S1c, S2c, tau, eps

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) K3_STAMP(7, 0);  // kernel entry
    if (threadIdx.x == 0) span_enter(g.span);
    const uint32_t rank = kPair == 2 ? cluster_ctarank() : 0u;
    const bool leader = rank == 0;
    const int pair_id = blockIdx.x / kPair;
    const int R = g.rows_per_tile;
    // static schedule: this pair's pieces are a contiguous, equal-cost range of the (tile,
    // column) space; dynamic: pairs claim the next piece from a global counter, so pairs
    // that start late (their SM still busy with another lane's kernels) take fewer
    const int pc_begin = g.dyn ? 0 : g.piece_off[pair_id], pc_end = g.dyn ? 0 : g.piece_off[pair_id + 1];
    constexpr uint32_t kQConsumers = 1 + 4 * kPair + (kPair - 1);  // MMA, epilogue warps, peer TMA
    // consumer side of the piece queue: the piece of position `cur` (-1 = no more)
    auto q_take = [&](int cur) -> int {
        mbar_wait(&qfull[cur % kQ], (uint32_t)(cur / kQ) & 1u);
        return *reinterpret_cast<volatile int*>(&s_q[cur % kQ]);
    };
    auto q_release = [&](int cur) {  // one thread per consumer unit, after it read the slot
        if constexpr (kPair == 2) {
            if (leader) mbar_arrive(&qempty[cur % kQ]);
            else mbar_arrive_remote(mapa_shared(smem_u32(&qempty[cur % kQ]), 0));
        } else {
            mbar_arrive(&qempty[cur % kQ]);
        }
    };

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < C::kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 4 * kPair);  // one arrival per epilogue warp of the pair
        }
        for (int s = 0; s < kQ; ++s) {
            mbar_init(&qfull[s], 1);
            mbar_init(&qempty[s], kQConsumers);
        }
        fence_barrier_init();
        for (int ti = 0; ti < g.G; ++ti) {
            tma_prefetch_desc(&maps.a[ti]);
            tma_prefetch_desc(&maps.bhi[ti]);
            tma_prefetch_desc(&maps.blo[ti]);
        }
    }
    if (threadIdx.x >= 64 && threadIdx.x < 64 + g.G) {  // finalize constants per test
        const GemmTest& T = g.t[threadIdx.x - 64];
        s_tc[4 * (threadIdx.x - 64) + 0] = T.sconst[0];
        s_tc[4 * (threadIdx.x - 64) + 1] = T.sconst[1];
        s_tc[4 * (threadIdx.x - 64) + 2] = g.tie_rel * (fabs(T.info->logk_x) + fabs(T.info->logk_y));
        s_tc[4 * (threadIdx.x - 64) + 3] = T.sconst[2];
    }
    if (warp == 1) {
        if constexpr (kPair == 2) tmem_alloc_pair<kTmemCols>(tmem_slot);
        else tmem_alloc<kTmemCols>(tmem_slot);
    }
    tc_fence_before();
    __syncthreads();
    if constexpr (kPair == 2) cluster_sync();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    if (threadIdx.x == 0) K3_STAMP(7, 2);  // setup done

    if (warp == 0) {
        // ---------------- TMA producer (both CTAs load their own A rows and B half)
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            // the leader claims a piece and publishes it (queue entry e) to both CTAs; entry
            // cur + 1 is published while piece cur is still being loaded, so the claim's
            // atomic and the cross-CTA publish stay off the stage ring's critical path
            auto claim_publish = [&](int e) -> int {
                int pc;
                if (g.dyn) {
                    pc = atomicAdd(g.claim, 1);
                    pc = pc < g.npieces ? pc : -1;
                } else {
                    pc = pc_begin + e < pc_end ? pc_begin + e : -1;
                }
                const int slot = e % kQ;
                mbar_wait(&qempty[slot], ((uint32_t)(e / kQ) & 1u) ^ 1u);
                s_q[slot] = pc;
                if constexpr (kPair == 2) {  // the peer's slot: an async store that completes its barrier
                    const uint32_t rb = mapa_shared(smem_u32(&qfull[slot]), 1);
                    mbar_arrive_expect_tx_cluster_relaxed(rb, 4u);
                    st_async_u32(mapa_shared(smem_u32(&s_q[slot]), 1), (uint32_t)pc, rb);
                }
                mbar_arrive(&qfull[slot]);
                return pc;
            };
            int pc_cur = leader ? claim_publish(0) : 0, pc_nxt = -2;  // -2: not yet published
            for (int cur = 0;; ++cur) {
                int pc;
                if (leader) {
                    pc = pc_cur;
                } else {
                    pc = q_take(cur);
                    q_release(cur);
                }
                if (pc < 0) break;
                const int4 pd = g.pieces[pc];  // {wave tile, col0, width, slot}
                const int tile = pd.x, width = pd.z;
                const int ti = test_of(g, tile);
                HAP_CHECK(tile >= 0 && tile < g.ntiles && pd.w >= 0 && pd.w < g.max_slots);
                HAP_CHECK(width > 0 && width <= kChunkN && width % 32 == 0 && pd.y % 32 == 0 &&
                          pd.y + width <= g.t[ti].ncols);
                HAP_CHECK(pd.w < g.tile_npieces[tile]);
                if (!test_failed(g.t[ti])) {
                    const int nkb = g.t[ti].n_pad / kKBlock;
                    const CUtensorMap* tmA = &maps.a[ti];
                    const CUtensorMap* tmBhi = &maps.bhi[ti];
                    const CUtensorMap* tmBlo = &maps.blo[ti];
                    const int arow = (tile - g.t[ti].tile0) * R + (int)rank * kTileM;
                    const int brow = pd.y + (int)rank * (width / kPair);
                    const int ui = cur;
                    for (int kb = 0; kb < nkb; ++kb) {
                        mbar_wait(&empty[stage], phase ^ 1u);
                        if (kb == 0) K3_STAMP(ui, 0);
                        if (kb == nkb - 1) K3_STAMP(ui, 1);
                        uint8_t* sA = smem + stage * C::kStageBytes;
                        if constexpr (kPair == 2) {
                            // EXPERIMENT (timing only): bit0 skips A loads, bit1 skips B lo loads
                            const uint32_t bytes = (uint32_t)C::kStageBytes - ((K3_EXP(g) & 1) ? kStageA : 0) -
                                                   ((K3_EXP(g) & 2) ? C::kStageB : 0);
                            if (leader) mbar_arrive_expect_tx(&full[stage], 2u * bytes);
                            const uint32_t fb = mapa_shared(smem_u32(&full[stage]), 0);
                            if (!(K3_EXP(g) & 1)) tma_load_2d_pair(tmA, fb, sA, kb * kKBlock, arow);
                            tma_load_2d_pair(tmBhi, fb, sA + kStageA, kb * kKBlock, brow);
                            if (!(K3_EXP(g) & 2))
                                tma_load_2d_pair(tmBlo, fb, sA + kStageA + C::kStageB, kb * kKBlock, brow);
                        } else {
                            mbar_arrive_expect_tx(&full[stage], (uint32_t)C::kStageBytes);
                            tma_load_2d(tmA, &full[stage], sA, kb * kKBlock, arow);
                            tma_load_2d(tmBhi, &full[stage], sA + kStageA, kb * kKBlock, brow);
                            tma_load_2d(tmBlo, &full[stage], sA + kStageA + C::kStageB, kb * kKBlock,
                                        brow);
                        }
                        if (++stage == C::kStages) { stage = 0; phase ^= 1u; }
                        if (leader && kb == (nkb >> 1) && pc_nxt == -2) pc_nxt = claim_publish(cur + 1);
                    }
                }
                if (leader) {
                    if (pc_nxt == -2) pc_nxt = claim_publish(cur + 1);
                    pc_cur = pc_nxt;
                    pc_nxt = -2;
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer: one thread of the leader CTA
        if (leader && lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            int i = 0;
            for (int cur = 0;; ++cur) {
                const int pc = q_take(cur);
                q_release(cur);
                if (pc < 0) break;
                const int width = g.pieces[pc].z;
                const int ti = test_of(g, g.pieces[pc].x);
                if (test_failed(g.t[ti])) continue;
                const int nkb = g.t[ti].n_pad / kKBlock;
                const uint32_t idesc = idesc_bf16_f32(kTileM * kPair, (uint32_t)width);
                const int a = i & 1;
                mbar_wait(&tempty[a], (((uint32_t)i >> 1) & 1u) ^ 1u);
                tc_fence_after();
                K3_STAMP(i, 2);
                const uint32_t dtm = tmem + (uint32_t)(a * kChunkN);
                for (int kb = 0; kb < nkb; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint32_t aBase = smem_u32(smem + stage * C::kStageBytes);
                    const uint32_t hBase = aBase + kStageA, lBase = hBase + C::kStageB;
#pragma unroll
                    for (int k = 0; k < kKBlock / 16; ++k) {
                        const uint64_t ad = smem_desc_k_sw128(aBase + 32u * k);
                        const uint64_t hd = smem_desc_k_sw128(hBase + 32u * k);
                        const uint64_t ld = smem_desc_k_sw128(lBase + 32u * k);
                        if constexpr (kPair == 2) {
                            umma_bf16_ss_pair(dtm, ad, hd, idesc, (kb | k) != 0 ? 1u : 0u);
                            if (!(K3_EXP(g) & 4)) umma_bf16_ss_pair(dtm, ad, ld, idesc, 1u);
                        } else {
                            umma_bf16_ss(dtm, ad, hd, idesc, (kb | k) != 0 ? 1u : 0u);
                            umma_bf16_ss(dtm, ad, ld, idesc, 1u);
                        }
                    }
                    if constexpr (kPair == 2) umma_commit_pair(&empty[stage], 0x3);
                    else umma_commit(&empty[stage]);
                    if (++stage == C::kStages) { stage = 0; phase ^= 1u; }
                }
                if constexpr (kPair == 2) umma_commit_pair(&tfull[a], 0x3);
                else umma_commit(&tfull[a]);
                K3_STAMP(i, 3);
                ++i;
            }
        }
    } else {
        // ---------------- epilogue: thread = TMEM lane = one mask row of this CTA
        const int q = warp & 3;
        const int trow = (int)rank * kTileM + 32 * q + lane;  // row within the tile
        const int etid = threadIdx.x - 64;
        uint32_t tempty_c[2] = {0, 0};
        if constexpr (kPair == 2) {
            tempty_c[0] = mapa_shared(smem_u32(&tempty[0]), 0);
            tempty_c[1] = mapa_shared(smem_u32(&tempty[1]), 0);
        }
        int i = 0;
        for (int cur = 0;; ++cur) {
            const int pc = q_take(cur);
            __syncwarp();
            if (lane == 0) q_release(cur);
            if (pc < 0) break;
            const int4 pd = g.pieces[pc];
            const int tile = pd.x, width = pd.z;
            const int ti = test_of(g, tile);
            const GemmTest& T = g.t[ti];
            if (test_failed(T)) {
                // no MMA ran for it; the tile still takes part in the finalize queue (as a
                // skip entry) so that every queue position is filled exactly once
                named_bar_sync(1, 128);
                if (etid == 0) {
                    const unsigned old = atomicAdd(g.tile_done + tile, 1u);
                    if (old == (unsigned)(kPair * g.tile_npieces[tile] - 1)) {
                        g.tile_done[tile] = 0;
                        fq_push(g, -(tile + 1));
                    }
                }
                continue;
            }
            const int np_tile = g.tile_npieces[tile];
            HAP_CHECK(np_tile >= 1 && np_tile <= g.max_slots && trow < R);
            HAP_CHECK(!T.gram || (T.mbits != nullptr &&
                                  tile - T.tile0 < (ti + 1 < g.G ? g.t[ti + 1].tile0 : g.ntiles) - T.tile0));
            const int a = i & 1;
            // Gram form: this row's mask bits for the piece's columns, loaded before the
            // accumulator wait (width <= 256: at most 8 words)
            uint32_t mw[8];
            if (T.gram) {
                const uint32_t* mb =
                    T.mbits + (size_t)((tile - T.tile0) * R + trow) * (size_t)(T.n_pad >> 5) + (pd.y >> 5);
#pragma unroll
                for (int w = 0; w < 8; ++w) mw[w] = w < (width >> 5) ? __ldcg(mb + w) : 0u;
            }
            mbar_wait(&tfull[a], ((uint32_t)i >> 1) & 1u);
            tc_fence_after();
            if (etid == 0) K3_STAMP(i, 4);
            // sigma1 = a + acc, sigma2 = b - acc:  |sigma1|^2 - |a|^2 = sum acc (acc + 2a), ...
            float s1 = 0.f, s2 = 0.f;
            const float4* abp = reinterpret_cast<const float4*>(T.ab + pd.y);
            const uint32_t tbase = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(a * kChunkN);
            const int nblk = (K3_EXP(g) & 8) ? 0 : width / 32;
            if (T.gram) {
                // s1 = sum_j m_bj (U_bj + 2 alpha_j), s2 = sum_j m_bj (U_bj - 2 beta_j)
#pragma unroll
                for (int cb = 0; cb < 8; cb += 2) {
                    if (cb >= nblk) break;
                    uint32_t r[2][32];
                    tmem_ld_32x32b_x32(tbase + (uint32_t)(32 * cb), r[0]);
                    if (cb + 1 < nblk) tmem_ld_32x32b_x32(tbase + (uint32_t)(32 * cb + 32), r[1]);
                    tmem_ld_wait();
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        if (cb + h >= nblk) break;
                        const uint32_t bits = mw[cb + h];
#pragma unroll
                        for (int j2 = 0; j2 < 16; ++j2) {
                            const float4 k4 = __ldg(abp + (cb + h) * 16 + j2);  // {2al, 2be} x 2 columns
                            const float x0 = __uint_as_float(r[h][2 * j2]), x1 = __uint_as_float(r[h][2 * j2 + 1]);
                            const bool m0 = (bits >> (2 * j2)) & 1u, m1 = (bits >> (2 * j2 + 1)) & 1u;
                            s1 += m0 ? x0 + k4.x : 0.f;
                            s2 += m0 ? x0 - k4.y : 0.f;
                            s1 += m1 ? x1 + k4.z : 0.f;
                            s2 += m1 ? x1 - k4.w : 0.f;
                        }
                    }
                }
            }
            for (int cb = 0; cb < (T.gram ? 0 : nblk); cb += 2) {  // two 32-column loads in flight per wait
                uint32_t r[2][32];
                tmem_ld_32x32b_x32(tbase + (uint32_t)(32 * cb), r[0]);
                if (cb + 1 < nblk) tmem_ld_32x32b_x32(tbase + (uint32_t)(32 * cb + 32), r[1]);
                tmem_ld_wait();
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    if (cb + h >= nblk) break;
#pragma unroll
                    for (int j2 = 0; j2 < 16; ++j2) {
                        const float4 k4 = __ldg(abp + (cb + h) * 16 + j2);  // {2a, 2b} of two columns
                        const float x0 = __uint_as_float(r[h][2 * j2]), x1 = __uint_as_float(r[h][2 * j2 + 1]);
                        s1 = fmaf(x0, x0 + k4.x, s1);
                        s2 = fmaf(x0, x0 - k4.y, s2);
                        s1 = fmaf(x1, x1 + k4.z, s1);
                        s2 = fmaf(x1, x1 - k4.w, s2);
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {  // accumulator buffer free again
                if constexpr (kPair == 2) mbar_arrive_cluster(tempty_c[a]);
                else mbar_arrive(&tempty[a]);
            }
            if (etid == 0) K3_STAMP(i, 5);
            g.part[((size_t)tile * g.max_slots + pd.w) * R + trow] = make_float2(s1, s2);
            __threadfence();
            named_bar_sync(1, 128);
            if (etid == 0) {
                const unsigned old = atomicAdd(g.tile_done + tile, 1u);
                *s_last = (old == (unsigned)(kPair * np_tile - 1)) ? 1 : 0;
            }
            named_bar_sync(1, 128);
            // The last arriving CTA publishes the tile in the launch's finalize queue; the
            // finalizes run after the CTAs' pieces (mid-kernel the partial loads queue behind
            // the operand streams: 12-16 us instead of ~1 us), taken from the queue by
            // whichever CTAs are done, so the tail is shared by all of them instead of each
            // CTA finalizing the tiles it happened to complete (up to ~3 x 5 us).
            if (*s_last && etid == 0) fq_push(g, tile + 1);
            named_bar_sync(1, 128);
            ++i;
        }
        for (int f = 0;; ++f) {
            if (etid == 0) {
                const int pos = atomicAdd(g.fq, 1);
                int v = 0;
                if (pos < g.ntiles) {
                    volatile int* slot = g.fq + 4 + pos;
                    for (uint32_t spins = 0; (v = *slot) == 0; ++spins) {
                        __nanosleep(64);
                        if (spins > (1u << 27)) __trap();  // never wait forever
                    }
                    *slot = 0;  // ready for the next launch
                    __threadfence();
                }
                *s_last = v;  // 0: queue drained
            }
            named_bar_sync(1, 128);
            const int v = *s_last;
            named_bar_sync(1, 128);
            if (v == 0) break;
            if (v < 0) continue;  // a failed test's tile: nothing to count
            const int tile = v - 1;
            const int ti = test_of(g, tile);
            const GemmTest& T = g.t[ti];
            __threadfence();
            if (etid == 0) K3_STAMP(f & 7, 6);
            finalize_tile(g, T, tile, tile - T.tile0, g.tile_npieces[tile], etid, s_cnt, s_tc[4 * ti],
                          s_tc[4 * ti + 1], s_tc[4 * ti + 2], s_tc[4 * ti + 3], f);
            if (etid == 0) K3_STAMP(f & 7, 7);
            named_bar_sync(1, 128);
        }
    }
    tc_fence_before();
    __syncthreads();
    if constexpr (kPair == 2) cluster_sync();
    if (threadIdx.x == 0) {  // the last CTA out resets the claim and finalize-queue counters
        __threadfence();
        if (atomicAdd(g.fq + 2, 1) == (int)gridDim.x - 1) {
            if (g.dyn) {
                g.claim[0] = 0;
                g.claim[1] = 0;
            }
            g.fq[0] = 0;
            g.fq[1] = 0;
            g.fq[2] = 0;
        }
    }
    if (threadIdx.x == 0) K3_STAMP(7, 1);  // all roles done
    if (threadIdx.x == 0) span_exit(g.span);
    if (warp == 1) {
        tc_fence_after();
        if constexpr (kPair == 2) tmem_dealloc_pair<kTmemCols>(tmem);
        else tmem_dealloc<kTmemCols>(tmem);
    }
}

template <int kPair>
cudaError_t launch_impl(const GemmMaps& maps, const GemmArgs& g, cudaStream_t st) {
    using C = Cfg<kPair>;
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(k3_maskgemm<kPair>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::kSmem);
        // the whole unified L1/shared array as shared memory: with the default (smallest
        // sufficient) carveout an SM running a mask-GEMM CTA has no room left for the
        // generator / alignment CTAs of the next block, which then wait for it to finish
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(k3_maskgemm<kPair>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                     cudaSharedmemCarveoutMaxShared);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)(g.npairs * kPair));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = C::kSmem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = kPair;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k3_maskgemm<kPair>, maps, g);
}

}  // namespace

int maskgemm_b_rows(int pair_mode) { return kChunkN / pair_mode; }

cudaError_t launch_maskgemm(const GemmMaps& maps, const GemmArgs& g, int pair_mode, cudaStream_t st) {
    if (g.ntiles <= 0) return cudaSuccess;
    return pair_mode == 2 ? launch_impl<2>(maps, g, st) : launch_impl<1>(maps, g, st);
}

HAP_CHECK_ACCESSOR(check_word_gemm)

}  // namespace hap
