// k_align.cu — K1: S1-S6 of the hot path as ONE cooperative kernel (DESIGN.md "Kernels" K1).
//
//   S1 normalise   x = h/||h||               PAPER.md:115-118 (§3.1 Eq. 2)
//   S2 means       xbar, ybar, mu_x, mu_y    PAPER.md:143-148; Alg. 1
//   S3 axis        u = (mu_x-mu_y)/||.||     PAPER.md:149-156 (Eqs. 5-6); Alg. 1 :664
//   S4 reflect     x' = x - 2u(u^T x)        PAPER.md:157-161, 245-255 (Eq. householder_fast)
//   S5 pool+split  Z = [X';Y] -> centred bf16 hi/lo planes (transposed, K contiguous),
//                  t = 1^T Z                 PAPER.md:183, 215-218 (Eq. gemm), 258
//   S6 observed    r_X = ||xbar|| (= r(X')), r_Y, T_obs (Eq. 10), fp64
//
// The problem is small (C2: 6 MB) and a chain of dependent reductions, so the cost is
// latency, not bandwidth.  One persistent cooperative grid (one CTA of 512 threads per SM)
// works on ITEMS of R consecutive pooled rows x all d columns, held as an fp32 tile in
// shared memory, and needs ONE software grid barrier:
//   P1 items  : load tile; row norms (ZeroVector check); column sums of x over the CTA's
//               items, added as fixed-point int64 into global accumulators   | barrier
//   P3 (local): every CTA forms xbar, ybar from the accumulators and reduces ||xbar||,
//               ||ybar||, ||v||, v.xbar itself (same order in every CTA, so identical
//               bits), CTA 0 writes info
//   P4 items  : the tile of P1 is still resident: row dots -> reflection coefficients,
//               z' = x - coef u - m, bf16 hi/lo split, transposed writes of both planes,
//               fixed-point column sums of t' = sum (hi + lo)
//   P5 (last CTA by ticket): t, epilogue constants {2a, 2b}, sum a^2, sum b^2; clears the
//               accumulators
// Cross-CTA sums are exact integer sums of per-CTA fixed-order partials, so Z~ and t are
// bit-identical across runs and ranks.
#include <cuda_bf16.h>

#include <cfloat>
#include <climits>
#include <mutex>
#include <cstdlib>
#include <algorithm>
#include <utility>

#define HAP_CHECK_TU 1
#include "hap_device.cuh"
#include "hap_internal.h"

namespace hap {
namespace {

#ifndef HAP_K1_THREADS
#define HAP_K1_THREADS 512
#endif
constexpr int kThreads = HAP_K1_THREADS;  // 64 registers per thread: 2 (or 4) CTAs fit per SM
constexpr int kWarps = kThreads / 32;
constexpr int kMaxItemRows = 16;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// block-wide fixed-order fp64 sums of two values
__device__ double2 block_sum2(double v0, double v1, double* red) {
    v0 = warp_sum(v0);
    v1 = warp_sum(v1);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) {
        red[w] = v0;
        red[kWarps + w] = v1;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double s0 = 0.0, s1 = 0.0;
        for (int i = 0; i < kWarps; ++i) {
            s0 += red[i];
            s1 += red[kWarps + i];
        }
        red[2 * kWarps] = s0;
        red[2 * kWarps + 1] = s1;
    }
    __syncthreads();
    return make_double2(red[2 * kWarps], red[2 * kWarps + 1]);
}

// the same for a block of NT threads (streaming kernels)
template <int NT>
__device__ double2 block_sum2_n(double v0, double v1, double* red) {
    constexpr int W = NT / 32;
    v0 = warp_sum(v0);
    v1 = warp_sum(v1);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) {
        red[w] = v0;
        red[W + w] = v1;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double s0 = 0.0, s1 = 0.0;
        for (int i = 0; i < W; ++i) {
            s0 += red[i];
            s1 += red[W + i];
        }
        red[2 * W] = s0;
        red[2 * W + 1] = s1;
    }
    __syncthreads();
    return make_double2(red[2 * W], red[2 * W + 1]);
}


__device__ __forceinline__ void stamp(const AlignArgs& a, int k) {
    if (a.stamps && blockIdx.x == 0 && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        a.stamps[k] = (long long)t;
    }
}

// per-CTA stamps (profiling level 3): stamps[8 + 8 cta + k]
__device__ __forceinline__ void cstamp(const AlignArgs& a, int k) {
    if (a.stamps && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        a.stamps[8 + 8 * blockIdx.x + k] = (long long)t;
    }
}

// development build only: KS1 per-CTA phase stamps (stamps[8 + 8 cta + k], grid <= 4 SMs)
#ifdef HAP_EXPERIMENTS
#define KS1_STAMP(k) cstamp(a, k)
#else
#define KS1_STAMP(k) do { } while (0)
#endif

// Software grid barrier (all CTAs are co-resident: cooperative launch): one release-add
// per CTA on a counter that only grows within a launch, then acquire-polling until every
// CTA has arrived.  The counter is cleared for the next launch by the last CTA of P5 (all
// CTAs have passed the barrier by then).
__device__ __forceinline__ void grid_sync(unsigned* bar) {
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
        unsigned v = 0;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
        } while (v < gridDim.x);
    }
    __syncthreads();
}

// L(r) = log kappa-hat(r), r clamped to [0, 1-1e-9] (Eq. 9; R1, R4)
__device__ __forceinline__ double logkappa64(double r, double d) {
    if (r > 1.0 - 1e-9) r = 1.0 - 1e-9;
    if (r <= 0.0) return -INFINITY;
    const double r2 = r * r;
    return log(r) + log(d - r2) - log(1.0 - r2);
}

__device__ __forceinline__ const float* row_ptr(const AlignPair& q, int64_t i) {
    return i < q.n_x ? q.X + i * q.d : q.Y + (i - q.n_x) * q.d;
}

// raw rows [r0, r0 + R) -> tile[r * P + c] (zero rows beyond N); all loads in flight first
__device__ __forceinline__ void load_tile(const AlignPair& q, float* tile, int64_t r0, int R, int P) {
    const int64_t N = q.n_x + q.n_y;
    if ((q.d & 3) == 0) {
        const int nq = (int)(q.d >> 2);
        const int total = R * nq;
        for (int b = threadIdx.x; b < total; b += 4 * kThreads) {
            float4 v[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int idx = b + k * kThreads;
                const int r = idx / nq, c4 = idx - r * nq;
                v[k] = (idx < total && r0 + r < N)
                           ? __ldg(reinterpret_cast<const float4*>(row_ptr(q, r0 + r)) + c4)
                           : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int idx = b + k * kThreads;
                if (idx < total) {
                    const int r = idx / nq, c4 = idx - r * nq;
                    float2* t2 = reinterpret_cast<float2*>(tile + (size_t)r * P + 4 * c4);
                    t2[0] = make_float2(v[k].x, v[k].y);
                    t2[1] = make_float2(v[k].z, v[k].w);
                }
            }
        }
    } else {
        const int d = (int)q.d;
        for (int idx = threadIdx.x; idx < R * d; idx += kThreads) {
            const int r = idx / d, c = idx - r * d;
            tile[(size_t)r * P + c] = r0 + r < N ? __ldg(row_ptr(q, r0 + r) + c) : 0.f;
        }
    }
}

// Deterministic cross-CTA sums: every CTA adds its fixed-order fp64 partial, rounded to a
// multiple of 2^-kFixS, into an int64 accumulator; integer addition is exact and commutes,
// so the sum is the same bits in every run whatever the arrival order.  Column sums of x
// are < 2^16 in magnitude (N <= 65535, |x_c| <= 1) and those of z' < 2^18, so 2^-44
// resolution keeps them below 2^62; the rounding error (<= 2^-45 per CTA partial) is far
// below the fp64 parity bar of the observed statistic (DESIGN.md D-K1).
constexpr double kFixScale = 17592186044416.0;  // 2^44
constexpr double kFixInv = 1.0 / 17592186044416.0;
__device__ __forceinline__ void fix_add(long long* acc, double v) {
    atomicAdd(reinterpret_cast<unsigned long long*>(acc), (unsigned long long)__double2ll_rn(v * kFixScale));
}
__device__ __forceinline__ double fix_get(const long long* acc) {
    return (double)__ldcg(acc) * kFixInv;
}

// scalars of one pair that every CTA working on it derives itself (P3)
struct PairScalars {
    double rnx, rny, rnv, ux, rN, rnX, rnY;
    bool identity;
};

__device__ __forceinline__ int pair_of(const AlignArgs& a, int64_t item) {
    int g = 0;
    while (g + 1 < a.G && item >= a.item_off[g + 1]) ++g;
    return g;
}

// Items of CTA `cta` (of G): the CTAs are split among the pairs in proportion to their items
// (at least one each) and a pair's items evenly among its CTAs, so a CTA works on ONE pair
// (its scalars are formed once) and on contiguous items.  Every partial sum is flushed per
// item, so the bits do not depend on this assignment (a pair alone or in any wave).
__device__ __forceinline__ void cta_items(const AlignArgs& a, int cta, int G, int64_t& i0, int64_t& i1) {
    const int64_t items = a.item_off[a.G];
    int c0 = 0;
    i0 = i1 = 0;
    for (int g = 0; g < a.G; ++g) {
        const int64_t ng = a.item_off[g + 1] - a.item_off[g];
        int cg = g == a.G - 1 ? G - c0 : (int)((ng * (int64_t)G) / (items > 0 ? items : 1));
        cg = cg < 1 ? 1 : cg;
        const int rest = G - c0 - (a.G - 1 - g);  // leave one CTA for each later pair
        cg = cg > rest ? rest : cg;
        if (cta < c0 + cg) {
            const int64_t j = cta - c0;
            i0 = a.item_off[g] + (j * ng) / cg;
            i1 = a.item_off[g] + ((j + 1) * ng) / cg;
            return;
        }
        c0 += cg;
    }
}

// W consecutive u32 words (W = R/2 <= 8) to a 4W-byte aligned address
template <int W>
__device__ __forceinline__ void store_words(uint32_t* dst, const uint32_t (&w)[W]) {
    if constexpr (W == 8) {
        reinterpret_cast<uint4*>(dst)[0] = make_uint4(w[0], w[1], w[2], w[3]);
        reinterpret_cast<uint4*>(dst)[1] = make_uint4(w[4], w[5], w[6], w[7]);
    } else if constexpr (W == 4) {
        reinterpret_cast<uint4*>(dst)[0] = make_uint4(w[0], w[1], w[2], w[3]);
    } else if constexpr (W == 2) {
        reinterpret_cast<uint2*>(dst)[0] = make_uint2(w[0], w[1]);
    } else {
        dst[0] = w[0];
    }
}

// P5 (the last CTA of an alignment launch, by ticket): per pair t = N m + t', a = n_x m,
// b = t - a (fp32) for the GEMM epilogue, {sum a^2, sum b^2} in fixed order; then the
// accumulators and flags are cleared for the next launch.  Shared by the fused K1 and the
// streaming K1s transform kernel.
template <int NT = kThreads>
__device__ void finish_pair(const AlignArgs& a, int g, double* red) {
    const int tid = threadIdx.x;
    const int d = (int)a.d;
    {
        const AlignPair& q = a.p[g];
        const int64_t N = q.n_x + q.n_y;
        double sa = 0.0, sb = 0.0, sm = 0.0;
        constexpr int kC = 8;  // loads of kC columns in flight per thread (ascending c)
        for (int64_t c0 = tid; c0 < a.d_pad; c0 += kC * NT) {
          double ts[kC], ms[kC];
#pragma unroll
          for (int u = 0; u < kC; ++u) {
            const int64_t c = c0 + u * NT;
            ts[u] = c < a.d_pad ? fix_get(q.acc + 2 * d + c) : 0.0;
            ms[u] = c < a.d_pad ? __ldcg(q.m + c) : 0.0;
          }
#pragma unroll
          for (int u = 0; u < kC; ++u) {
            const int64_t c = c0 + u * NT;
            if (c >= a.d_pad) break;
            const double tsum = ts[u];
            const double m = ms[u];
            sm += m * m;
            q.t64[c] = (double)N * m + tsum;
            const float af = (float)((double)q.n_x * m);
            const float bf = (float)((double)q.n_y * m + tsum);
            q.ab[c] = make_float2(2.0f * af, 2.0f * bf);
            sa += (double)af * (double)af;
            sb += (double)bf * (double)bf;
          }
        }
        const double2 sab = block_sum2_n<NT>(sa, sb, red);
        const double smm = block_sum2_n<NT>(sm, 0.0, red).x;
        for (int64_t c = tid; c < 2 * (int64_t)d + a.d_pad; c += NT) q.acc[c] = 0;
        if (tid == 0) {
            q.sconst[0] = sab.x;
            q.sconst[1] = sab.y;
            // representation-error scale of a pooled row (R14): the planes keep
            // z' = z - m to 2^-17 relative (bf16 hi + lo) after an fp32 evaluation of z
            // (2^-23 of |z| = 1); E||z'||^2 = 1 - ||m||^2
            q.sconst[2] = 0x1p-17 * sqrt(fmax(1.0 - smm, 0.0)) + 0x1p-23;
            *q.bad = LLONG_MAX;  // reset the pair's ZeroVector word
        }
    }
}
template <int NT = kThreads>
__device__ void finish_pairs(const AlignArgs& a, double* red) {
    for (int g = 0; g < a.G; ++g) finish_pair<NT>(a, g, red);
    if (threadIdx.x == 0) {  // reset the ticket and the barrier
        reinterpret_cast<unsigned*>(a.scratch + 1)[0] = 0u;
        reinterpret_cast<unsigned*>(a.scratch + 2)[0] = 0u;
    }
}

// Per-pair completion tickets of the streaming kernels: the CTA that completes a pair's last
// work unit runs that pair's scalar pass, so the pairs of a wave finish in parallel on
// different CTAs instead of in series on the launch's last one.  Word 4 (warp-per-row KS1
// items: P3) / 5 (KS3 tiles: P5) of the pair's own scratch; reset by the finishing CTA.
__device__ __forceinline__ bool pair_ticket(const AlignPair& q, int word, unsigned units, unsigned total, int* s_flag) {
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned* t = reinterpret_cast<unsigned*>(q.bad + word);
        const unsigned old = atomicAdd(t, units);
        *s_flag = old + units == total;
        if (old + units == total) *t = 0u;
    }
    __syncthreads();
    const bool last = *s_flag != 0;
    if (last) __threadfence();
    return last;
}

// dynamic smem: tile f32 [R][P] | (u_c, m_c) f32 [d_pad] (stage_umc) | xs, ys f64 [d]
// (stage_means) | t' partials f64 [d_pad] (stage_umc); R <= 16.
// <= 64 registers/thread (launch bound 2): a K1 CTA then fits beside a mask-GEMM CTA on
// one SM, so the next test's alignment overlaps the current test's GEMM.
// Items of all pairs of the launch (a wave) form one list; a CTA's column sums are flushed
// to a pair's accumulators whenever its next item belongs to another pair.
template <int R>
__global__ void __launch_bounds__(kThreads, 65536 / (kThreads * 64)) k1_align_fused(AlignArgs a, int P, int stage_umc,
                                                              int stage_means) {
    extern __shared__ __align__(16) uint8_t k1_smem[];
    __shared__ double red[2 * kWarps + 2];
    __shared__ double s_inv[kMaxItemRows];
    __shared__ float s_invf[kMaxItemRows], s_cff[kMaxItemRows];
    __shared__ int s_last;
    float* tile = reinterpret_cast<float*>(k1_smem);
    float2* umc = reinterpret_cast<float2*>(k1_smem + (size_t)R * P * 4);  // [d_pad] (u_c, m_c)
    double* xs = reinterpret_cast<double*>(umc + (stage_umc ? a.d_pad : 0));
    double* ys = xs + a.d;
    double* s_t = stage_means ? ys + a.d : xs;  // [d_pad] t' partials (with stage_umc)
    const int G = gridDim.x, cta = blockIdx.x;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int d = (int)a.d;
    unsigned* bar = reinterpret_cast<unsigned*>(a.scratch + 2);
    if (tid == 0) span_enter(a.span);
    stamp(a, 0);
    cstamp(a, 0);

    // ---------------- P1: norms + column sums of x over this CTA's items -> accumulators
    int64_t resident = -1;
    {
        double sx0 = 0.0, sy0 = 0.0, sx1 = 0.0, sy1 = 0.0;  // columns tid, tid + kThreads
        int cur = -1;  // pair of the partial sums held in registers
        auto flush = [&]() {
            if (cur < 0) return;
            long long* acc = a.p[cur].acc;
            if (tid < d) {
                fix_add(acc + tid, sx0);
                fix_add(acc + d + tid, sy0);
            }
            if (tid + kThreads < d) {
                fix_add(acc + tid + kThreads, sx1);
                fix_add(acc + d + tid + kThreads, sy1);
            }
            sx0 = sy0 = sx1 = sy1 = 0.0;
        };
        int64_t i0, i1;
        cta_items(a, cta, G, i0, i1);
        for (int64_t item = i0; item < i1; ++item) {
            const int g = pair_of(a, item);
            const AlignPair& q = a.p[g];
            const int64_t N = q.n_x + q.n_y;
            const int64_t r0 = (item - a.item_off[g]) * R;
            flush();  // per item (see cta_items)
            cur = g;
            if (resident >= 0) __syncthreads();  // previous tile fully consumed
            load_tile(q, tile, r0, R, P);
            __syncthreads();
            for (int rw = warp; rw < R; rw += kWarps) {
                const int64_t i = r0 + rw;
                double s4[4] = {0.0, 0.0, 0.0, 0.0};  // independent chains (latency)
                const float* tr = tile + (size_t)rw * P;
                int c = lane;
                for (; c + 96 < d; c += 128) {
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const double v = (double)tr[c + 32 * u];
                        s4[u] += v * v;
                    }
                }
                for (; c < d; c += 32) {
                    const double v = (double)tr[c];
                    s4[0] += v * v;
                }
                double s = (s4[0] + s4[1]) + (s4[2] + s4[3]);
                s = warp_sum(s);
                if (lane == 0) {
                    const double nrm = sqrt(s);
                    const double iv = (i < N && nrm >= 1e-12) ? 1.0 / nrm : 0.0;
                    s_inv[rw] = iv;
                    if (i < N) {
                        q.inv[i] = iv;
                        if (nrm < 1e-12) atomicMin(q.bad, (long long)i);
                    }
                }
            }
            __syncthreads();
            const int64_t nxr64 = q.n_x - r0;  // X rows of the item
            const int nxr = nxr64 <= 0 ? 0 : (nxr64 >= R ? R : (int)nxr64);
            for (int c = tid, k = 0; c < d; c += kThreads, ++k) {
                double px0 = 0.0, py0 = 0.0, px1 = 0.0, py1 = 0.0;  // two chains per group
#pragma unroll
                for (int r = 0; r < R; r += 2) {
                    const double v0 = (double)tile[(size_t)r * P + c] * s_inv[r];
                    const double v1 = (double)tile[(size_t)(r + 1) * P + c] * s_inv[r + 1];
                    if (r < nxr) px0 += v0;
                    else py0 += v0;
                    if (r + 1 < nxr) px1 += v1;
                    else py1 += v1;
                }
                const double px = px0 + px1, py = py0 + py1;
                if (k == 0) {
                    sx0 += px;
                    sy0 += py;
                } else if (k == 1) {
                    sx1 += px;
                    sy1 += py;
                } else {  // d > 2 kThreads: straight to the accumulators
                    fix_add(q.acc + c, px);
                    fix_add(q.acc + d + c, py);
                }
            }
            resident = item;
        }
        flush();
    }
    cstamp(a, 1);
    grid_sync(bar);
    stamp(a, 1);
    cstamp(a, 2);
    stamp(a, 2);
    cstamp(a, 3);

    // ---------------- P3 (per pair, CTA-local, identical in every CTA that needs it):
    // means, their norms, axis, centre; the CTA holding a pair's item 0 writes its info
    PairScalars sc{};
    auto pair_scalars = [&](int g, bool writer) {
        const AlignPair& q = a.p[g];
        const long long* acc_x = q.acc;
        const long long* acc_y = q.acc + d;
        const int64_t N = q.n_x + q.n_y;
        sc.rnX = 1.0 / (double)q.n_x;
        sc.rnY = 1.0 / (double)q.n_y;
        double sxx = 0.0, syy = 0.0;
        for (int c = tid; c < d; c += kThreads) {
            const double xb = fix_get(acc_x + c) * sc.rnX, yb = fix_get(acc_y + c) * sc.rnY;
            if (stage_means) {
                xs[c] = xb;
                ys[c] = yb;
            }
            if (writer) {
                q.xbar[c] = xb;
                q.ybar[c] = yb;
            }
            sxx += xb * xb;
            syy += yb * yb;
        }
        const double2 sq = block_sum2(sxx, syy, red);
        const double nx = sqrt(sq.x), ny = sqrt(sq.y);
        const bool degenerate = nx < 1e-12 || ny < 1e-12;
        sc.rnx = degenerate ? 0.0 : 1.0 / nx;
        sc.rny = degenerate ? 0.0 : 1.0 / ny;
        double sv = 0.0, svx = 0.0;
        for (int c = tid; c < d; c += kThreads) {
            const double xb = stage_means ? xs[c] : fix_get(acc_x + c) * sc.rnX;
            const double yb = stage_means ? ys[c] : fix_get(acc_y + c) * sc.rnY;
            const double v = xb * sc.rnx - yb * sc.rny;
            sv += v * v;
            svx += v * xb;
        }
        const double2 vv = block_sum2(sv, svx, red);
        const double nv0 = sqrt(vv.x);
        sc.identity = (a.mode == HAP_ALIGN_NONE) || degenerate || nv0 < 1e-9;  // R3
        sc.rnv = sc.identity ? 0.0 : 1.0 / nv0;
        sc.ux = vv.y * sc.rnv;  // u . xbar
        sc.rN = 4096.0 / (double)N;
        if (stage_umc || writer)
            for (int c = tid; c < (int)a.d_pad; c += kThreads) {
                double ud = 0.0, md = 0.0;
                if (c < d) {  // axis u_c; centre m_c = t_c/N quantised to 2^-12, t = n_x (xbar -
                              // 2u(u.xbar)) + n_y ybar
                    const double xb = stage_means ? xs[c] : fix_get(acc_x + c) * sc.rnX;
                    const double yb = stage_means ? ys[c] : fix_get(acc_y + c) * sc.rnY;
                    ud = (xb * sc.rnx - yb * sc.rny) * sc.rnv;
                    const double t = (double)q.n_x * (xb - 2.0 * ud * sc.ux) + (double)q.n_y * yb;
                    md = rint(t * sc.rN) * (1.0 / 4096.0);
                }
                if (stage_umc) umc[c] = make_float2((float)ud, (float)md);
                if (writer) {  // export copies (read in P5 and by hap_export_pooled)
                    q.u[c] = ud;
                    q.m[c] = md;
                }
            }
        if (writer && tid == 0) {
            hap_align_info* f = q.info;
            const long long bad = *reinterpret_cast<volatile long long*>(q.bad);
            f->n_x = q.n_x;
            f->n_y = q.n_y;
            f->d = a.d;
            f->n_pad = q.n_pad;
            f->d_pad = a.d_pad;
            f->is_identity = sc.identity ? 1 : 0;
            f->status = bad < N ? HAP_E_ZERO_VECTOR : (degenerate ? HAP_E_DEGENERATE_MEAN : HAP_OK);
            f->bad_row = bad < N ? bad : -1;
            // observed statistic in fp64 (Alg. 1 step 4): r(X') = ||xbar||
            // since H is orthogonal; T_obs = L(r_Y) - L(r_X) (Eq. 10)
            f->r_x = nx;
            f->r_y = ny;
            const double lx = logkappa64(nx, (double)a.d), ly = logkappa64(ny, (double)a.d);
            f->logk_x = lx;
            f->logk_y = ly;
            f->t_obs = (isinf(lx) && isinf(ly)) ? 0.0 : ly - lx;
            const double qnan = __longlong_as_double(0x7ff8000000000000ll);
            f->gemm_r_x = f->gemm_r_y = f->gemm_t_obs = qnan;
        }
        __syncthreads();  // umc / xs / ys ready
    };
    // axis and centre of a column on the fly (wide d: not staged)
    auto axis_centre = [&](const AlignPair& q, int c, double& ud, double& md) {
        ud = 0.0;
        md = 0.0;
        if (c < d) {
            const double xb = fix_get(q.acc + c) * sc.rnX, yb = fix_get(q.acc + d + c) * sc.rnY;
            ud = (xb * sc.rnx - yb * sc.rny) * sc.rnv;
            const double t = (double)q.n_x * (xb - 2.0 * ud * sc.ux) + (double)q.n_y * yb;
            md = rint(t * sc.rN) * (1.0 / 4096.0);
        }
    };
    // pairs whose item 0 falls to another CTA still need no scalars here; the writer of
    // each pair is the CTA of its item 0 (handled in the item loop below)
    stamp(a, 3);
    cstamp(a, 4);

    // ---------------- P4: this CTA's items again, last one first (still resident)
    int sp = -1;  // pair whose scalars / t' partials are current
    auto flush_t = [&]() {
        if (sp < 0 || !stage_umc) return;
        __syncthreads();
        for (int c = tid; c < (int)a.d_pad; c += kThreads) fix_add(a.p[sp].acc + 2 * d + c, s_t[c]);
    };
    if (resident >= 0) {
        int64_t i0, i1;
        cta_items(a, cta, G, i0, i1);
        for (int64_t item = i1 - 1; item >= i0; --item) {
            const int g = pair_of(a, item);
            const AlignPair& q = a.p[g];
            const int64_t N = q.n_x + q.n_y;
            const int64_t li = item - a.item_off[g];
            const int64_t r0 = li * R;
            flush_t();  // per item (see cta_items)
            if (g != sp) {
                // the CTA that holds the pair's item 0 writes its info and exports
                pair_scalars(g, i0 == a.item_off[g]);
                sp = g;
            }
            if (stage_umc) {
                __syncthreads();
                for (int c = tid; c < (int)a.d_pad; c += kThreads) s_t[c] = 0.0;
            }
            if (item != resident) {
                __syncthreads();
                load_tile(q, tile, r0, R, P);
                if (tid < R) s_inv[tid] = r0 + tid < N ? __ldcg(q.inv + r0 + tid) : 0.0;
                __syncthreads();
            }
            // reflection coefficients 2 u^T x_i = 2 (xbar.h_i/||xbar|| - ybar.h_i/||ybar||)
            // / (||v|| ||h_i||) of the X rows (Y is not reflected)
            for (int rw = warp; rw < R; rw += kWarps) {
                const int64_t i = r0 + rw;
                double cf = 0.0;
                if (i < q.n_x && !sc.identity) {
                    double dx = 0.0, dy = 0.0;
                    for (int c = lane; c < d; c += 32) {
                        const double hv = (double)tile[(size_t)rw * P + c];
                        dx += hv * (stage_means ? xs[c] : fix_get(q.acc + c) * sc.rnX);
                        dy += hv * (stage_means ? ys[c] : fix_get(q.acc + d + c) * sc.rnY);
                    }
                    dx = warp_sum(dx);
                    dy = warp_sum(dy);
                    cf = 2.0 * ((dx * sc.rnx - dy * sc.rny) * s_inv[rw]) * sc.rnv;
                }
                if (lane == 0) {
                    s_cff[rw] = (float)cf;
                    s_invf[rw] = (float)s_inv[rw];
                }
            }
            __syncthreads();
            if (item == i1 - 1) cstamp(a, 5);
            // z' = x - coef u - m in fp32 (the value is then kept to 16 bits), hi/lo split;
            // thread = column: the item's R rows of the column -> 2R contiguous bytes per plane
            // (16-byte stores), and the column's t' partial summed in fp64 without any
            // cross-lane reduction (hi + lo is exact in fp32 with <= 16 significant bits, so the
            // fp64 sum of the R values is exact: t = N m + t' is the exact sum of the planes)
            for (int c = tid; c < (int)a.d_pad; c += kThreads) {
                float2 um;  // (0, 0) for pad columns
                if (stage_umc) {
                    um = umc[c];
                } else {
                    double ud, md;
                    axis_centre(q, c, ud, md);
                    um = make_float2((float)ud, (float)md);
                }
                uint32_t hw[R / 2], lw[R / 2];
                double tv = 0.0;
#pragma unroll
                for (int r = 0; r < R; r += 2) {
                    const bool v0 = r0 + r < N && c < d, v1 = r0 + r + 1 < N && c < d;
                    const float z0 = v0 ? fmaf(-s_cff[r], um.x, tile[(size_t)r * P + c] * s_invf[r]) - um.y : 0.f;
                    const float z1 =
                        v1 ? fmaf(-s_cff[r + 1], um.x, tile[(size_t)(r + 1) * P + c] * s_invf[r + 1]) - um.y : 0.f;
                    const __nv_bfloat16 h0 = __float2bfloat16_rn(z0), h1 = __float2bfloat16_rn(z1);
                    const float fh0 = __bfloat162float(h0), fh1 = __bfloat162float(h1);
                    const __nv_bfloat16 l0 = __float2bfloat16_rn(z0 - fh0), l1 = __float2bfloat16_rn(z1 - fh1);
                    hw[r / 2] = (uint32_t)__bfloat16_as_ushort(h0) | ((uint32_t)__bfloat16_as_ushort(h1) << 16);
                    lw[r / 2] = (uint32_t)__bfloat16_as_ushort(l0) | ((uint32_t)__bfloat16_as_ushort(l1) << 16);
                    tv += (double)(fh0 + __bfloat162float(l0)) + (double)(fh1 + __bfloat162float(l1));
                }
                const size_t off = ((size_t)c * (size_t)q.n_pad + (size_t)r0) >> 1;  // u32 words
                store_words<R / 2>(reinterpret_cast<uint32_t*>(q.zt_hi) + off, hw);
                store_words<R / 2>(reinterpret_cast<uint32_t*>(q.zt_lo) + off, lw);
                if (stage_umc) s_t[c] += tv;  // the column's owner thread
                else fix_add(q.acc + 2 * d + c, tv);
            }
        }
        flush_t();
    }
    // ---------------- P4b (optional): the generator draws of the wave (K2a's work, see
    // k_perm.cu k2_draws), staged in each permutation's mask row.  Register-only work in
    // this latency-bound kernel's idle issue slots; K2b then skips the draws.
    if (a.do_draws) {
        const PermArgs& pd = a.draws;
        const int64_t ditems = pd.item_off[pd.G];
        for (int64_t pi = (int64_t)cta * kWarps + warp; pi < ditems; pi += (int64_t)G * kWarps) {
            int ti = 0;
            while (ti + 1 < pd.G && pi >= pd.item_off[ti + 1]) ++ti;
            const PermTest& T = pd.t[ti];
            const int64_t li = pi - pd.item_off[ti];
            if (li >= T.count) continue;  // observed-split rows: K2b
            const uint32_t Nn = (uint32_t)T.N, nxx = (uint32_t)T.n_x;
            const uint32_t key0 = (uint32_t)(T.seed & 0xFFFFFFFFu), key1 = (uint32_t)(T.seed >> 32);
            const uint32_t b = (uint32_t)(T.b_begin + (uint64_t)li);
            const int64_t R1 = pd.rows_per_tile - 1;
            const int64_t orow = (li / R1) * pd.rows_per_tile + 1 + li % R1;
            uint16_t* jrow = static_cast<uint16_t*>(T.out) + orow * T.n_pad;
            for (uint32_t k0 = 4u * (uint32_t)lane; k0 < nxx; k0 += 128u) {
                uint32_t j[4];
                draw_targets(k0, nxx, Nn, b, T.s, key0, key1, j);
                *reinterpret_cast<uint2*>(jrow + k0) = make_uint2(j[0] | (j[1] << 16), j[2] | (j[3] << 16));
            }
        }
    }
    cstamp(a, 6);
    stamp(a, 4);

    // ---------------- P5 (last CTA to finish, ticket): per pair t = N m + t', a = n_x m,
    // b = t - a (fp32) for the GEMM epilogue, {sum a^2, sum b^2} in fixed order; then the
    // accumulators and flags are cleared for the next launch
    __threadfence();
    __syncthreads();
    if (tid == 0) {
        unsigned* ticket = reinterpret_cast<unsigned*>(a.scratch + 1);
        s_last = atomicAdd(ticket, 1u) == (unsigned)G - 1;
    }
    __syncthreads();
    if (s_last) {
        __threadfence();
        finish_pairs(a, red);
    }
    stamp(a, 5);
    cstamp(a, 7);
    __syncthreads();
    if (tid == 0) span_exit(a.span);
}


// ==========================================================================================
// K1s — STREAMING alignment for large pairs (n_pad * d >= kStreamMinElems).
// The fused kernel above is latency-shaped (one CTA per SM, a grid barrier, reloads); at
// LLM sizes (C3: 164 MB of fp32 input) the alignment is a bandwidth problem, so it runs as
// three bandwidth passes over HBM, each with many loads in flight:
//   KS1 k1s_stats : items of R rows -> a 3-stage shared-memory ring filled by cp.async.bulk
//                   (one bulk copy per row); row norms -> inv (ZeroVector check); fp64
//                   column partials of x = h/||h|| per item, rounded per item to fixed point
//                   and summed as int64 in registers (exact, order-free), one atomic per
//                   column per CTA; the last CTA (ticket) forms every pair's means, axis,
//                   centre and observed statistic (the P3 arithmetic of the fused kernel)
//   KS2 k1s_coef  : reflection coefficients 2 u.x_i of the X rows (fp64 dot, 4 rows per
//                   warp so each u load serves 4 rows); {coef, 1/||h||} per row
//   KS3 k1s_xform : tiled transpose, 64 rows x 64 columns per tile: z' = x - coef u - m
//                   (fp32, as the fused kernel), bf16 hi/lo split, 128-byte column runs per
//                   plane; per-column t' partials per tile in fixed point; the last CTA
//                   (ticket) runs P5 (finish_pairs).
// Algorithmic bytes: read 4Nd (KS1) + 4 n_x d (KS2) + 4Nd (KS3), write 4 n_pad d_pad (KS3).
// Deterministic: every cross-CTA sum is an integer sum of per-item / per-tile roundings and
// the CTA -> work assignment depends only on the shapes.
constexpr int kSStages = 3;
#ifndef HAP_K1S_MIN_ELEMS
#define HAP_K1S_MIN_ELEMS (8ll << 20)
#endif
constexpr int64_t kStreamMinElems = HAP_K1S_MIN_ELEMS;  // n_pad * d: 32 MB of fp32 input
constexpr int kXfRows = 128, kXfCols = 64;  // KS3 tile: 128 rows x 64 columns

__device__ __forceinline__ void bulk_load_row(float* dst, const float* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// expect_tx + arrive WITHOUT release semantics: a release arrive waits (MEMBAR) for the
// issuing thread's earlier global stores and atomics, which stalled the whole CTA once per
// item; the stage's readers are ordered before the refill by the __syncthreads before it
__device__ __forceinline__ void mbar_arrive_expect_tx_relaxed(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.relaxed.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

// P3 of one pair from its (complete) accumulators, written to global memory (xbar, ybar, axis
// u, centre m, info), with every column's accumulators loaded ONCE into registers (kC >= d /
// NT columns per thread, all loads in flight together: one L2 round trip).  The warp-per-row
// KS1 (d <= 1024) runs it on the CTA that completes the pair's last item (per-pair ticket,
// word 4 of the pair's scratch), after its main loop, when registers are free; for d > 1024
// every KS2 CTA derives P3 itself (k1s_coef<true>) instead of one CTA holding up the pass.
template <int NT, int kC>
__device__ void stream_pair_scalars_cached(const AlignArgs& a, int g, double* red) {
    const AlignPair& q = a.p[g];
    const int tid = threadIdx.x;
    const int d = (int)a.d;
    const long long* acc_x = q.acc;
    const long long* acc_y = q.acc + d;
    const int64_t N = q.n_x + q.n_y;
    const double rnX = 1.0 / (double)q.n_x, rnY = 1.0 / (double)q.n_y;
    double xb[kC], yb[kC];
#pragma unroll
    for (int u = 0; u < kC; ++u) {
        const int c = tid + u * NT;
        xb[u] = c < d ? fix_get(acc_x + c) * rnX : 0.0;
        yb[u] = c < d ? fix_get(acc_y + c) * rnY : 0.0;
    }
    double sxx = 0.0, syy = 0.0;
#pragma unroll
    for (int u = 0; u < kC; ++u) {
        const int c = tid + u * NT;
        if (c < d) {
            q.xbar[c] = xb[u];
            q.ybar[c] = yb[u];
            sxx += xb[u] * xb[u];
            syy += yb[u] * yb[u];
        }
    }
    const double2 sq = block_sum2_n<NT>(sxx, syy, red);
    const double nx = sqrt(sq.x), ny = sqrt(sq.y);
    const bool degenerate = nx < 1e-12 || ny < 1e-12;
    const double rnx = degenerate ? 0.0 : 1.0 / nx;
    const double rny = degenerate ? 0.0 : 1.0 / ny;
    double sv = 0.0, svx = 0.0;
#pragma unroll
    for (int u = 0; u < kC; ++u) {
        if (tid + u * NT < d) {
            const double v = xb[u] * rnx - yb[u] * rny;
            sv += v * v;
            svx += v * xb[u];
        }
    }
    const double2 vv = block_sum2_n<NT>(sv, svx, red);
    const double nv0 = sqrt(vv.x);
    const bool identity = (a.mode == HAP_ALIGN_NONE) || degenerate || nv0 < 1e-9;  // R3
    const double rnv = identity ? 0.0 : 1.0 / nv0;
    const double ux = vv.y * rnv;
    const double rN = 4096.0 / (double)N;
#pragma unroll
    for (int u = 0; u < kC; ++u) {
        const int c = tid + u * NT;
        double ud = 0.0, md = 0.0;
        if (c < d) {
            ud = (xb[u] * rnx - yb[u] * rny) * rnv;
            const double t = (double)q.n_x * (xb[u] - 2.0 * ud * ux) + (double)q.n_y * yb[u];
            md = rint(t * rN) * (1.0 / 4096.0);
        }
        if (c < (int)a.d_pad) {
            q.u[c] = ud;
            q.m[c] = md;
        }
    }
    for (int c = tid + kC * NT; c < (int)a.d_pad; c += NT) {  // padding columns beyond kC NT
        q.u[c] = 0.0;
        q.m[c] = 0.0;
    }
    if (tid == 0) {
        hap_align_info* f = q.info;
        const long long bad = *reinterpret_cast<volatile long long*>(q.bad);
        f->n_x = q.n_x;
        f->n_y = q.n_y;
        f->d = a.d;
        f->n_pad = q.n_pad;
        f->d_pad = a.d_pad;
        f->is_identity = identity ? 1 : 0;
        f->status = bad < N ? HAP_E_ZERO_VECTOR : (degenerate ? HAP_E_DEGENERATE_MEAN : HAP_OK);
        f->bad_row = bad < N ? bad : -1;
        f->r_x = nx;  // r(X') = ||xbar||
        f->r_y = ny;
        const double lx = logkappa64(nx, (double)a.d), ly = logkappa64(ny, (double)a.d);
        f->logk_x = lx;
        f->logk_y = ly;
        f->t_obs = (isinf(lx) && isinf(ly)) ? 0.0 : ly - lx;  // Eq. 10
        const double qnan = __longlong_as_double(0x7ff8000000000000ll);
        f->gemm_r_x = f->gemm_r_y = f->gemm_t_obs = qnan;
    }
    __syncthreads();
}

// KS1.  a.item_off: items of R rows (R = 8 / G4), ceil(N/R) per pair.  CTA c takes items
// [I c / grid, I (c+1) / grid); 256 threads, two CTAs per SM.  Thread t owns the float4
// column groups t + 256 k (k < G4) of every row of an item: it widens each fp32 value to
// fp64 ONCE (registers), forms its partial squares per row (reduced in fixed order ->
// 1/||h||) and then the item's column partials of x = h/||h||.  Column sums of pair g, side
// X (0) / Y (1) are held as int64 in registers and flushed (one atomic per column) when the
// (pair, side) changes.
// kRing = false (K1s-lean, pairs below kStreamMinElems): no shared-memory ring; every
// thread loads its own float4 groups of the item's rows straight into registers and the
// NEXT item's rows are in flight while the current one is reduced - the same arithmetic in
// the same order (identical bits), < 1 KB of shared memory, so the CTAs fit beside a
// mask-GEMM CTA and generator CTAs on one SM.
constexpr int kS1Threads = 256;
constexpr int kS1LeanThreads = 128;  // lean: one warp per SM sub-partition (registers beside K3)
template <int G4, bool kRing = true, int NT = kS1Threads>
__global__ void __launch_bounds__(NT, 512 / NT) k1s_stats(AlignArgs a) {
    constexpr int R = 8 / G4;
    constexpr int W = NT / 32;
    extern __shared__ __align__(128) uint8_t ks_smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(ks_smem);
    float* ring = reinterpret_cast<float*>(ks_smem + 128);
    __shared__ double s_part[2][W][R];  // by item parity: one barrier per item
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int d = (int)a.d;
    const int d4 = d >> 2;
    const int64_t items = a.item_off[a.G];
    const int64_t i0 = items * blockIdx.x / gridDim.x, i1 = items * (blockIdx.x + 1) / gridDim.x;
    const size_t stage_floats = (size_t)R * d;
    KS1_STAMP(0);
    if (tid == 0) {
        span_enter(a.span);
        if constexpr (kRing) {
            for (int k = 0; k < kSStages; ++k) mbar_init(&full[k], 1);
            fence_barrier_init();
        }
    }
    __syncthreads();
    // lean mode: this thread's float4 groups of an item's rows, straight from global memory
    auto load_regs = [&](int64_t item, float4 (&f)[R][G4]) {
        const int g = pair_of(a, item);
        const AlignPair& q = a.p[g];
        const int64_t N = q.n_x + q.n_y;
        const int64_t r0 = (item - a.item_off[g]) * R;
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
            for (int kk = 0; kk < G4; ++kk) {
                const int c4 = tid + kk * NT;
                f[r][kk] = (r0 + r < N && c4 < d4) ? __ldcs(reinterpret_cast<const float4*>(row_ptr(q, r0 + r)) + c4)
                                                   : make_float4(0.f, 0.f, 0.f, 0.f);
            }
    };
    float4 nxt[R][G4];
    if constexpr (!kRing)
        if (i0 < i1) load_regs(i0, nxt);
    auto issue = [&](int64_t item, int st) {  // one thread
        const int g = pair_of(a, item);
        const AlignPair& q = a.p[g];
        const int64_t N = q.n_x + q.n_y;
        const int64_t r0 = (item - a.item_off[g]) * R;
        const int nr = (int)(N - r0 < R ? N - r0 : R);
        mbar_arrive_expect_tx_relaxed(&full[st], (uint32_t)nr * (uint32_t)d * 4u);
        for (int r = 0; r < nr; ++r)
            bulk_load_row(ring + st * stage_floats + (size_t)r * d, row_ptr(q, r0 + r), (uint32_t)d * 4u, &full[st]);
    };
    if constexpr (kRing)
        if (tid == 0)
            for (int k = 0; k < kSStages && i0 + k < i1; ++k) issue(i0 + k, k);
    long long acc[G4][4];
#pragma unroll
    for (int k = 0; k < G4; ++k)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[k][e] = 0;
    int cur = -1;  // 2 * pair + side of the register sums
    auto flush = [&]() {
        if (cur < 0) return;
        long long* dst = a.p[cur >> 1].acc + (cur & 1) * d;
#pragma unroll
        for (int k = 0; k < G4; ++k) {
            const int c4 = tid + k * NT;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                if (c4 < d4 && acc[k][e] != 0)
                    atomicAdd(reinterpret_cast<unsigned long long*>(dst + 4 * c4 + e), (unsigned long long)acc[k][e]);
                acc[k][e] = 0;
            }
        }
    };
    // (the pairs' scalars P3 are derived by every KS2 CTA from the complete column sums, so
    // no CTA here waits for the others: a CTA issues its last atomics and exits)
    for (int64_t item = i0; item < i1; ++item) {
        const int64_t k = item - i0;
        const int st = (int)(k % kSStages);
        const int g = pair_of(a, item);
        const AlignPair& q = a.p[g];
        const int64_t N = q.n_x + q.n_y;
        const int64_t r0 = (item - a.item_off[g]) * R;
        HAP_CHECK(g < a.G && r0 >= 0 && r0 < N && item < a.item_off[a.G]);
        const int nr = (int)(N - r0 < R ? N - r0 : R);
        double v[R][G4][4];
        if constexpr (kRing) {
            const float4* tile = reinterpret_cast<const float4*>(ring + st * stage_floats);
            mbar_wait(&full[st], (uint32_t)((k / kSStages) & 1));
            if (k == 0) KS1_STAMP(1);
#pragma unroll
            for (int r = 0; r < R; ++r)
#pragma unroll
                for (int kk = 0; kk < G4; ++kk) {
                    const int c4 = tid + kk * NT;
                    float4 f = make_float4(0.f, 0.f, 0.f, 0.f);
                    if (r < nr && c4 < d4) f = tile[(size_t)r * d4 + c4];
                    v[r][kk][0] = (double)f.x;
                    v[r][kk][1] = (double)f.y;
                    v[r][kk][2] = (double)f.z;
                    v[r][kk][3] = (double)f.w;
                }
        } else {
#pragma unroll
            for (int r = 0; r < R; ++r)
#pragma unroll
                for (int kk = 0; kk < G4; ++kk) {
                    v[r][kk][0] = (double)nxt[r][kk].x;
                    v[r][kk][1] = (double)nxt[r][kk].y;
                    v[r][kk][2] = (double)nxt[r][kk].z;
                    v[r][kk][3] = (double)nxt[r][kk].w;
                }
            if (item + 1 < i1) load_regs(item + 1, nxt);  // in flight during this item
        }
        // row norms: per-thread partial squares, warp tree, then the warps in order.  ONE
        // barrier per item: it also frees the ring stage (every thread holds the item in
        // registers), and every warp forms the rows' 1/||h|| itself (lane r: row r, the same
        // fixed-order sum in every warp), so no second barrier hands them out; s_part is
        // double-buffered by item parity (a warp reaches item k + 2 only after every warp
        // has passed item k + 1's barrier, i.e. finished reading item k's partials).
        double (*sp)[R] = s_part[k & 1];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            double sq0 = 0.0, sq1 = 0.0;
#pragma unroll
            for (int kk = 0; kk < G4; ++kk) {
                sq0 += v[r][kk][0] * v[r][kk][0] + v[r][kk][1] * v[r][kk][1];
                sq1 += v[r][kk][2] * v[r][kk][2] + v[r][kk][3] * v[r][kk][3];
            }
            const double sq = warp_sum(sq0 + sq1);
            if (lane == 0) sp[warp][r] = sq;
        }
        __syncthreads();
        if constexpr (kRing)
            if (tid == 0 && item + kSStages < i1) issue(item + kSStages, st);
        double my_iv = 0.0;
        if (lane < nr) {
            double ss = 0.0;
#pragma unroll
            for (int w = 0; w < W; ++w) ss += sp[w][lane];
            const double nrm = sqrt(ss);
            my_iv = nrm >= 1e-12 ? 1.0 / nrm : 0.0;
            if (warp == 0) {
                q.inv[r0 + lane] = my_iv;
                if (nrm < 1e-12) atomicMin(q.bad, (long long)(r0 + lane));
            }
        }
        double iv[R];
#pragma unroll
        for (int r = 0; r < R; ++r) iv[r] = __shfl_sync(0xffffffffu, my_iv, r);  // 0 beyond nr
        const int64_t nxr64 = q.n_x - r0;
        const int nxr = nxr64 <= 0 ? 0 : (nxr64 >= nr ? nr : (int)nxr64);
        if (nxr == 0 || nxr == nr) {  // the whole item on one side (all but <= 1 item per pair)
            const int code = 2 * g + (nxr == 0 ? 1 : 0);
            if (code != cur) {
                flush();
                cur = code;
            }
#pragma unroll
            for (int kk = 0; kk < G4; ++kk)
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    double p0 = 0.0, p1 = 0.0;
#pragma unroll
                    for (int r = 0; r < R; r += 2) {
                        p0 += v[r][kk][e] * iv[r];
                        if (r + 1 < R) p1 += v[r + 1][kk][e] * iv[r + 1];
                    }
                    acc[kk][e] += __double2ll_rn((p0 + p1) * kFixScale);
                }
        } else {
#pragma unroll
            for (int side = 0; side < 2; ++side) {
                const int lo = side ? nxr : 0, hi = side ? nr : nxr;
                const int code = 2 * g + side;
                if (code != cur) {
                    flush();
                    cur = code;
                }
#pragma unroll
                for (int kk = 0; kk < G4; ++kk)
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        double p = 0.0;
#pragma unroll
                        for (int r = 0; r < R; ++r)
                            if (r >= lo && r < hi) p += v[r][kk][e] * iv[r];
                        acc[kk][e] += __double2ll_rn(p * kFixScale);
                    }
            }
        }
    }
    KS1_STAMP(2);
    pdl_trigger();  // the coefficient pass may launch (it waits for this grid to complete)
    flush();
    KS1_STAMP(4);
    if (tid == 0) span_exit(a.span);
}

// KS1-lean for d <= 1024 (C1, C2, C4, C5): WARP per row, no block-wide barrier per item.
// A CTA takes a contiguous run of ONE pair's items (cta_items) of kSWRows = 4 rows; its 4 warps take
// the items in turn.  A warp streams an item's rows (lane = float4 column groups l + 32 k,
// the next row in flight), forms the row norm with a butterfly (identical bits in every
// lane) -> 1/||h|| (ZeroVector check), and adds x = h/||h|| into fp64 register partials of
// its columns; each (item, side) segment is rounded to fixed point and added into the CTA's
// int64 shared-memory column sums (exact, order-free), flushed once per CTA.  Bits depend on
// the pair's shape only (rounding per item), not on the grid.  The per-pair ticket runs P3.
constexpr int kSWRows = 4;
template <int G>
__global__ void __launch_bounds__(kS1LeanThreads, 4) k1s_stats_warp(AlignArgs a) {
    constexpr int W = kS1LeanThreads / 32;
    extern __shared__ __align__(16) long long sw_acc[];  // [2][d] X / Y column sums
    __shared__ double red[2 * W + 2];
    __shared__ int s_last;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int d = (int)a.d, d4 = d >> 2;
    if (tid == 0) span_enter(a.span);
    int64_t i0, i1;
    cta_items(a, blockIdx.x, gridDim.x, i0, i1);
    if (i0 >= i1) {
        if (tid == 0) span_exit(a.span);
        return;
    }
    const int g = pair_of(a, i0);
    const AlignPair& q = a.p[g];
    const int64_t N = q.n_x + q.n_y;
    for (int c = tid; c < 2 * d; c += kS1LeanThreads) sw_acc[c] = 0;
    __syncthreads();
    auto load_row = [&](int64_t i, float4 (&f)[G]) {
        const float4* rp = reinterpret_cast<const float4*>(row_ptr(q, i));
#pragma unroll
        for (int k = 0; k < G; ++k) {
            const int c4 = lane + 32 * k;
            f[k] = c4 < d4 ? __ldcs(rp + c4) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
    };
    for (int64_t item = i0 + warp; item < i1; item += W) {
        const int64_t r0 = (item - a.item_off[g]) * kSWRows;
        const int nr = (int)(N - r0 < kSWRows ? N - r0 : kSWRows);
        HAP_CHECK(r0 >= 0 && nr >= 1);
        double p[G][4];
#pragma unroll
        for (int k = 0; k < G; ++k) p[k][0] = p[k][1] = p[k][2] = p[k][3] = 0.0;
        int side = r0 < q.n_x ? 0 : 1;
        auto flush = [&]() {  // this (item, side) segment -> fixed point -> CTA sums
            long long* dst = sw_acc + side * d;
#pragma unroll
            for (int k = 0; k < G; ++k) {
                const int c4 = lane + 32 * k;
                if (c4 < d4)
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const long long v = __double2ll_rn(p[k][e] * kFixScale);
                        if (v) atomicAdd(reinterpret_cast<unsigned long long*>(dst + 4 * c4 + e), (unsigned long long)v);
                        p[k][e] = 0.0;
                    }
            }
        };
        float4 nxt[G];
        load_row(r0, nxt);
        for (int r = 0; r < nr; ++r) {
            float4 cur[G];
#pragma unroll
            for (int k = 0; k < G; ++k) cur[k] = nxt[k];
            if (r + 1 < nr) load_row(r0 + r + 1, nxt);
            const int rs = r0 + r < q.n_x ? 0 : 1;
            if (rs != side) {
                flush();
                side = rs;
            }
            double sq0 = 0.0, sq1 = 0.0;
#pragma unroll
            for (int k = 0; k < G; ++k) {
                const double x0 = cur[k].x, x1 = cur[k].y, x2 = cur[k].z, x3 = cur[k].w;
                sq0 += x0 * x0 + x1 * x1;
                sq1 += x2 * x2 + x3 * x3;
            }
            const double ss = warp_sum(sq0 + sq1);
            const double nrm = sqrt(ss);
            const double iv = nrm >= 1e-12 ? 1.0 / nrm : 0.0;
            if (lane == 0) {
                q.inv[r0 + r] = iv;
                if (nrm < 1e-12) atomicMin(q.bad, (long long)(r0 + r));
            }
#pragma unroll
            for (int k = 0; k < G; ++k) {
                p[k][0] += (double)cur[k].x * iv;
                p[k][1] += (double)cur[k].y * iv;
                p[k][2] += (double)cur[k].z * iv;
                p[k][3] += (double)cur[k].w * iv;
            }
        }
        flush();
    }
    pdl_trigger();
    __syncthreads();
    for (int c = tid; c < 2 * d; c += kS1LeanThreads) {
        const long long v = sw_acc[c];
        if (v) atomicAdd(reinterpret_cast<unsigned long long*>(q.acc + c), (unsigned long long)v);
    }
    const unsigned total = (unsigned)(a.item_off[g + 1] - a.item_off[g]);
    if (pair_ticket(q, 4, (unsigned)(i1 - i0), total, &s_last))
        stream_pair_scalars_cached<kS1LeanThreads, (32 * G + kS1LeanThreads - 1) / kS1LeanThreads * 4>(a, g, red);
    if (tid == 0) span_exit(a.span);
}

// KS2: {2 u.x_i, 1/||h_i||} per pooled row (Y rows and identity pairs: coefficient 0).  The
// CTAs (no more than fit on the GPU at once, so there is no second wave) are split among the
// pairs in proportion to their X rows; a warp takes X rows in turn (fp64 dot with u staged in
// shared memory, lane = columns l, l + 32, ... in that order) with 8 column steps of 16 bytes
// in flight per lane; 64 registers and (kP3) 2 d_pad doubles of shared memory, u written over
// xbar, let 3 CTAs share an SM (KS2 36.7 -> 33 us at C3 against 16 steps and 3 d_pad).
constexpr int kCoefInFlight = 8;
constexpr int kCoefThreads = 256;
template <bool kP3>
__global__ void __launch_bounds__(kCoefThreads) k1s_coef(AlignArgs a, int ctas_per_pair0, int ctas_per_pair1,
                                                         int ctas_per_pair2, int ctas_per_pair3) {
    if constexpr (kP3) {  // the X rows are inputs, not KS1 results: toward L2 while KS1 finishes
        const int cpp[4] = {ctas_per_pair0, ctas_per_pair1, ctas_per_pair2, ctas_per_pair3};
        int g = 0, c0 = 0;
        while (g < a.G - 1 && (int)blockIdx.x >= c0 + cpp[g]) c0 += cpp[g++];
        const AlignPair& q = a.p[g];
        const int nw = blockDim.x >> 5;
        if ((threadIdx.x & 31) == 0)
            for (int64_t i = (int64_t)(blockIdx.x - c0) * nw + (threadIdx.x >> 5); i < q.n_x; i += (int64_t)cpp[g] * nw)
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(q.X + i * a.d), "r"((uint32_t)a.d * 4u)
                             : "memory");
    }
    pdl_wait();  // KS1 (column sums, 1/||h||, ZeroVector rows) complete and visible
    extern __shared__ __align__(16) uint8_t kc_smem[];
    double* su = reinterpret_cast<double*>(kc_smem);  // [d_pad] axis u
    double* sxb = su;                                   // [d_pad] xbar (kP3 only; the axis u
                                                        // overwrites it column by column)
    double* syb = su + a.d_pad;                         // [d_pad] ybar
    __shared__ double red[2 * (kCoefThreads / 32) + 2];
    const int cpp[4] = {ctas_per_pair0, ctas_per_pair1, ctas_per_pair2, ctas_per_pair3};
    int g = 0, c0 = 0;
    while (g < a.G - 1 && (int)blockIdx.x >= c0 + cpp[g]) c0 += cpp[g++];
    const int nct = cpp[g], cta = blockIdx.x - c0;
    const AlignPair& q = a.p[g];
    const int d = (int)a.d, tid = threadIdx.x;
    const int64_t N = q.n_x + q.n_y;
    if (tid == 0) span_enter(a.span);
    bool identity;
    if constexpr (kP3) {
        // ---- P3, derived by EVERY CTA of the pair from the complete column sums (all loads in
        // flight together: one L2 round trip; identical arithmetic and order in every CTA, so
        // every CTA holds the same bits): xbar, ybar (Eq. 8 means), r, the axis u and centre m
        // (Eq. householder_fast), the observed statistic; CTA 0 of the pair publishes u, m and
        // the pair's info for KS3, K3 and the host.  (d <= 4096 on this path: kPC columns per
        // thread cover it.)
        // (xbar, ybar of this thread's own columns are kept in shared memory: no barrier needed
        // between the passes, registers stay free for the coefficient loop)
        constexpr int kPC = 4096 / kCoefThreads;
        const double rnX = 1.0 / (double)q.n_x, rnY = 1.0 / (double)q.n_y;
        double sxx = 0.0, syy = 0.0;
        {
            long long ax[kPC], ay[kPC];
    #pragma unroll
            for (int u = 0; u < kPC; ++u) {
                const int c = tid + u * kCoefThreads;
                ax[u] = c < d ? __ldcg(q.acc + c) : 0;
                ay[u] = c < d ? __ldcg(q.acc + d + c) : 0;
            }
    #pragma unroll
            for (int u = 0; u < kPC; ++u) {
                const int c = tid + u * kCoefThreads;
                const double xb = (double)ax[u] * kFixInv * rnX, yb = (double)ay[u] * kFixInv * rnY;
                sxx += xb * xb;
                syy += yb * yb;
                if (c < (int)a.d_pad) {
                    sxb[c] = xb;
                    syb[c] = yb;
                }
            }
        }
        const double2 sq = block_sum2_n<kCoefThreads>(sxx, syy, red);
        const double nx = sqrt(sq.x), ny = sqrt(sq.y);
        const bool degenerate = nx < 1e-12 || ny < 1e-12;
        const double rnx = degenerate ? 0.0 : 1.0 / nx;
        const double rny = degenerate ? 0.0 : 1.0 / ny;
        double sv = 0.0, svx = 0.0;
    #pragma unroll
        for (int u = 0; u < kPC; ++u) {
            const int c = tid + u * kCoefThreads;
            if (c < d) {
                const double v = sxb[c] * rnx - syb[c] * rny;
                sv += v * v;
                svx += v * sxb[c];
            }
        }
        const double2 vv = block_sum2_n<kCoefThreads>(sv, svx, red);
        const double nv0 = sqrt(vv.x);
        const bool identity_ = (a.mode == HAP_ALIGN_NONE) || degenerate || nv0 < 1e-9;  // R3
        const double rnv = identity_ ? 0.0 : 1.0 / nv0;
        const double ux = vv.y * rnv;
        const double rN = 4096.0 / (double)N;
    #pragma unroll
        for (int u = 0; u < kPC; ++u) {
            const int c = tid + u * kCoefThreads;
            double ud = 0.0, md = 0.0;
            if (c < d) {
                const double xb = sxb[c], yb = syb[c];
                ud = (xb * rnx - yb * rny) * rnv;
                const double t = (double)q.n_x * (xb - 2.0 * ud * ux) + (double)q.n_y * yb;
                md = rint(t * rN) * (1.0 / 4096.0);
            }
            if (c < (int)a.d_pad) {
                su[c] = ud;
                if (cta == 0) {
                    q.u[c] = ud;
                    q.m[c] = md;
                }
            }
        }
        if (cta == 0 && tid == 0) {
            hap_align_info* f = q.info;
            const long long bad = __ldcg(q.bad);
            f->n_x = q.n_x;
            f->n_y = q.n_y;
            f->d = a.d;
            f->n_pad = q.n_pad;
            f->d_pad = a.d_pad;
            f->is_identity = identity_ ? 1 : 0;
            f->status = bad < N ? HAP_E_ZERO_VECTOR : (degenerate ? HAP_E_DEGENERATE_MEAN : HAP_OK);
            f->bad_row = bad < N ? bad : -1;
            f->r_x = nx;  // r(X') = ||xbar||
            f->r_y = ny;
            const double lx = logkappa64(nx, (double)a.d), ly = logkappa64(ny, (double)a.d);
            f->logk_x = lx;
            f->logk_y = ly;
            f->t_obs = (isinf(lx) && isinf(ly)) ? 0.0 : ly - lx;  // Eq. 10
            const double qnan = __longlong_as_double(0x7ff8000000000000ll);
            f->gemm_r_x = f->gemm_r_y = f->gemm_t_obs = qnan;
        }
        identity = identity_;
    } else {  // P3 ran in KS1 (warp-per-row variant, d <= 1024): stage u
        identity = q.info->is_identity != 0;
        for (int c = tid; c < (int)a.d_pad; c += kCoefThreads) su[c] = q.u[c];
    }
    __syncthreads();  // su complete
    // ---- S4 coefficients: rows without a reflection {0, 1/||h||}
    for (int64_t i = (int64_t)cta * blockDim.x + tid; i < N; i += (int64_t)nct * blockDim.x)
        if (identity || i >= q.n_x) q.coef[i] = make_float2(0.f, (float)__ldcg(q.inv + i));
    if (!identity) {
        const int warp = tid >> 5, lane = tid & 31, nw = blockDim.x >> 5;
        const int n4 = d / 4;
        const double2* su2 = reinterpret_cast<const double2*>(su);
        for (int64_t i = (int64_t)cta * nw + warp; i < q.n_x; i += (int64_t)nct * nw) {
            const float4* rp = reinterpret_cast<const float4*>(q.X + i * d);
            double dot0 = 0.0, dot1 = 0.0;
            // (d <= 1024: 8 steps cover a row, and fewer registers leave room beside K3)
            constexpr int kIF = kP3 ? kCoefInFlight : 8;
#pragma unroll 1
            for (int c4b = 0; c4b < n4; c4b += 32 * kIF) {
                float4 h[kIF];
#pragma unroll
                for (int u = 0; u < kIF; ++u) {
                    const int c4 = c4b + 32 * u + lane;
                    h[u] = c4 < n4 ? __ldcs(rp + c4) : make_float4(0.f, 0.f, 0.f, 0.f);
                }
#pragma unroll
                for (int u = 0; u < kIF; ++u) {
                    const int c4 = c4b + 32 * u + lane;
                    if (c4 < n4) {
                        const double2 ua = su2[2 * c4], ub = su2[2 * c4 + 1];
                        dot0 += (double)h[u].x * ua.x + (double)h[u].y * ua.y;
                        dot1 += (double)h[u].z * ub.x + (double)h[u].w * ub.y;
                    }
                }
            }
            const double dot = warp_sum(dot0 + dot1);
            if (lane == 0) {
                const double iv = __ldcg(q.inv + i);
                q.coef[i] = make_float2((float)(2.0 * dot * iv), (float)iv);
            }
        }
    }
    pdl_trigger();
    __syncthreads();
    if (tid == 0) span_exit(a.span);
}

// KS3: tiles (pair, column strip of 64, row block of 128) in that order; CTA c takes tiles
// [T c / grid, T (c+1) / grid).  The raw fp32 tiles stream into a 3-stage shared-memory
// ring with cp.async (two tiles in flight per CTA); 512 threads.  Transform thread = (row
// pair 2p, 2p + 1; columns 4 q .. 4 q + 3) x 2 row pairs: z' = x - coef u - m (fp32), bf16
// hi/lo, each column's two rows packed into one 32-bit word of a TRANSPOSED staging tile
// [column][row]; writing thread = (column, 16 rows): two 16-byte shared loads per plane and
// two 16-byte global stores (8 threads cover a column's 256-byte run per plane).  t' per
// column and tile in fp64 (exact: hi + lo has <= 16 significant bits), rounded per tile to
// fixed point, summed as int64 over the CTA's tiles of one strip, one atomic per column per
// strip run.
constexpr int kXfStages = 3;
constexpr int kXfTP = kXfRows + 2;  // u16 pitch of the transposed staging (65 words)
constexpr size_t kXfSmem = (size_t)kXfStages * kXfRows * kXfCols * 4 + (size_t)kXfStages * kXfRows * 8 +
                           2 * (size_t)kXfCols * kXfTP * 2;

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem_dst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// the fields of one pair that KS3 touches per tile, cached in registers
struct XfPair {
    const float* X;
    const float* Y;
    const float2* coef;
    uint16_t* zhi;
    uint16_t* zlo;
    long long* tacc;
    int n_x, N, n_pad, rtiles;
};

__global__ void __launch_bounds__(kThreads, 1) k1s_xform(AlignArgs a, int64_t tile_off1, int64_t tile_off2,
                                                         int64_t tile_off3, int64_t tiles_total) {
    pdl_wait();  // KS2 (coefficients) complete and visible
    KS1_STAMP(7);
    extern __shared__ __align__(16) uint8_t xf_smem[];
    float* raw = reinterpret_cast<float*>(xf_smem);  // [kXfStages][128][64]
    float2* rcoef = reinterpret_cast<float2*>(raw + kXfStages * kXfRows * kXfCols);  // [kXfStages][128]
    uint16_t* sh_hi = reinterpret_cast<uint16_t*>(rcoef + kXfStages * kXfRows);  // [64][kXfTP]
    uint16_t* sh_lo = sh_hi + kXfCols * kXfTP;
    __shared__ double red[2 * kWarps + 2];
    __shared__ int s_last;
    const int tid = threadIdx.x;
    const int d = (int)a.d, d_pad = (int)a.d_pad;
    const int64_t t0 = tiles_total * blockIdx.x / gridDim.x, t1 = tiles_total * (blockIdx.x + 1) / gridDim.x;
    if (tid == 0) span_enter(a.span);
    // copy role: rows lr + 32 k (k < 4), columns 4 lc4 .. 4 lc4 + 3
    const int lc4 = tid & 15, lr = tid >> 4;
    // transform role: row pairs (2 tp, 2 tp + 1) and (64 + 2 tp, 65 + 2 tp), columns 4 tq ..
    const int tq = tid & 15, tp = tid >> 4;
    // write role: column wc, rows 8 wg .. 8 wg + 7 and 64 + 8 wg .. 64 + 8 wg + 7
    const int wg = tid & 7, wc = tid >> 3;
    const int strips = (d_pad + kXfCols - 1) / kXfCols;
    auto pair_fields = [&](int g) {
        const AlignPair& q = a.p[g];
        XfPair P;
        P.X = q.X;
        P.Y = q.Y;
        P.coef = q.coef;
        P.zhi = q.zt_hi;
        P.zlo = q.zt_lo;
        P.tacc = q.acc + 2 * d;
        P.n_x = (int)q.n_x;
        P.N = (int)(q.n_x + q.n_y);
        P.n_pad = (int)q.n_pad;
        P.rtiles = (int)((q.n_pad + kXfRows - 1) / kXfRows);
        return P;
    };
    struct TileAt {
        int g, strip, rt;
    };
    auto locate = [&](int64_t t) {  // once per CTA (offsets of absent pairs are tiles_total)
        TileAt L;
        L.g = (t >= tile_off1) + (t >= tile_off2) + (t >= tile_off3);
        const int64_t lt = t - (L.g == 0 ? 0 : L.g == 1 ? tile_off1 : L.g == 2 ? tile_off2 : tile_off3);
        const int64_t rtiles = (a.p[L.g].n_pad + kXfRows - 1) / kXfRows;
        L.strip = (int)(lt / rtiles);
        L.rt = (int)(lt % rtiles);
        return L;
    };
    TileAt Ld = locate(t0);  // the loader's position and its pair
    XfPair Pl = pair_fields(Ld.g);
    auto load = [&](int64_t t, int slot) {  // this thread's 4 pieces of tile t (+ coefficients)
        if (t < t1) {
            const int r0 = Ld.rt * kXfRows, c = Ld.strip * kXfCols + 4 * lc4;
            float* dst = raw + (size_t)slot * kXfRows * kXfCols + 4 * lc4;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int i = r0 + lr + 32 * k;
                if (i < Pl.N && c < d) {
                    const float* src = i < Pl.n_x ? Pl.X + (size_t)i * d : Pl.Y + (size_t)(i - Pl.n_x) * d;
                    cp_async16(dst + (lr + 32 * k) * kXfCols, src + c);
                }
            }
            if (tid < kXfRows / 2 && r0 + 2 * tid < Pl.n_pad)  // {coef, 1/||h||} of the rows (n_pad long)
                cp_async16(rcoef + slot * kXfRows + 2 * tid, Pl.coef + r0 + 2 * tid);
            if (++Ld.rt == Pl.rtiles) {  // advance
                Ld.rt = 0;
                if (++Ld.strip == strips) {
                    Ld.strip = 0;
                    if (++Ld.g < a.G) Pl = pair_fields(Ld.g);
                }
            }
        }
        cp_async_commit();
    };
#pragma unroll
    for (int k = 0; k < kXfStages - 1; ++k) load(t0 + k, k);
    long long tacc = 0;  // fixed-point t' of column wc of the current strip (wg == 0 lanes)
    TileAt L = locate(t0);
    XfPair P = pair_fields(L.g);
    int cur_g = -1, cur_strip = -1;
    float4 u4 = make_float4(0.f, 0.f, 0.f, 0.f), m4 = u4;
    auto flush = [&]() {
        const int c = cur_strip * kXfCols + wc;
        if (cur_g >= 0 && wg == 0 && c < d_pad && tacc != 0)
            atomicAdd(reinterpret_cast<unsigned long long*>(P.tacc + c), (unsigned long long)tacc);
        tacc = 0;
    };
    int slot = 0;
    // a pair's P5 runs on the CTA that completes its last tile (per-pair ticket)
    int pg = L.g;
    unsigned pcnt = 0;
    auto pair_done = [&]() {
        flush();
        cur_g = -1;  // (flushed)
        const unsigned total = (unsigned)(strips * ((a.p[pg].n_pad + kXfRows - 1) / kXfRows));
        if (pair_ticket(a.p[pg], 5, pcnt, total, &s_last)) {
            finish_pair(a, pg, red);
            KS1_STAMP(6);
        }
        pcnt = 0;
    };
    for (int64_t t = t0; t < t1; ++t) {
        if (L.g != pg) {
            pair_done();
            pg = L.g;
        }
        ++pcnt;
        if (L.g != cur_g || L.strip != cur_strip) {
            flush();
            if (L.g != cur_g) P = pair_fields(L.g);
            cur_g = L.g;
            cur_strip = L.strip;
            const AlignPair& q = a.p[L.g];
            float uu[4], mm[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int c = L.strip * kXfCols + 4 * tq + k;
                uu[k] = c < d ? (float)__ldcg(q.u + c) : 0.f;
                mm[k] = c < d ? (float)__ldcg(q.m + c) : 0.f;
            }
            u4 = make_float4(uu[0], uu[1], uu[2], uu[3]);
            m4 = make_float4(mm[0], mm[1], mm[2], mm[3]);
        }
        const int r0 = L.rt * kXfRows, cb = L.strip * kXfCols;
        cp_async_wait<kXfStages - 2>();  // this thread's pieces of tile t have landed
        __syncthreads();                 // ... and every thread's (rows, coefficients)
        const float* rt_raw = raw + (size_t)slot * kXfRows * kXfCols;
        const bool cvalid = cb + 4 * tq < d;
#pragma unroll
        for (int hp = 0; hp < 2; ++hp) {  // row pairs (2 tp, 2 tp + 1) + 64 hp
            const int ra = 64 * hp + 2 * tp;
            float z[2][4];
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const int rr = ra + k;
                if (r0 + rr < P.N && cvalid) {
                    const float4 h = *reinterpret_cast<const float4*>(rt_raw + rr * kXfCols + 4 * tq);
                    const float2 cv = rcoef[slot * kXfRows + rr];  // {coef, 1/||h||}
                    z[k][0] = fmaf(-cv.x, u4.x, h.x * cv.y) - m4.x;
                    z[k][1] = fmaf(-cv.x, u4.y, h.y * cv.y) - m4.y;
                    z[k][2] = fmaf(-cv.x, u4.z, h.z * cv.y) - m4.z;
                    z[k][3] = fmaf(-cv.x, u4.w, h.w * cv.y) - m4.w;
                } else {
                    z[k][0] = z[k][1] = z[k][2] = z[k][3] = 0.f;
                }
            }
#pragma unroll
            for (int e = 0; e < 4; ++e) {  // column 4 tq + e: rows ra, ra + 1 in one word
                const __nv_bfloat162 hh = __floats2bfloat162_rn(z[0][e], z[1][e]);
                const float2 hf = __bfloat1622float2(hh);
                const __nv_bfloat162 ll = __floats2bfloat162_rn(z[0][e] - hf.x, z[1][e] - hf.y);
                const int w = (4 * tq + e) * (kXfTP / 2) + (ra >> 1);
                reinterpret_cast<uint32_t*>(sh_hi)[w] = *reinterpret_cast<const uint32_t*>(&hh);
                reinterpret_cast<uint32_t*>(sh_lo)[w] = *reinterpret_cast<const uint32_t*>(&ll);
            }
        }
        __syncthreads();  // planes staged (transposed); the ring slot of tile t is free
        load(t + kXfStages - 1, slot == 0 ? kXfStages - 1 : slot - 1);
        {
            const int col = cb + wc;
            double tv = 0.0;
#pragma unroll
            for (int hb = 0; hb < 2; ++hb) {
                const int rb = 64 * hb + 8 * wg;
                if (r0 + rb < P.n_pad) {  // (the last row block of a pair may be half: n_pad % 128 = 64)
                    // 8 rows = 16 bytes per plane; the staging rows are 4-byte aligned (65-word
                    // pitch), so two 8-byte loads
                    const uint32_t* hs = reinterpret_cast<const uint32_t*>(sh_hi) + wc * (kXfTP / 2) + (rb >> 1);
                    const uint32_t* ls = reinterpret_cast<const uint32_t*>(sh_lo) + wc * (kXfTP / 2) + (rb >> 1);
                    const uint4 hv = make_uint4(hs[0], hs[1], hs[2], hs[3]);
                    const uint4 lv = make_uint4(ls[0], ls[1], ls[2], ls[3]);
                    const uint32_t hw[4] = {hv.x, hv.y, hv.z, hv.w}, lw[4] = {lv.x, lv.y, lv.z, lv.w};
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        tv += (double)(__uint_as_float(hw[j] << 16) + __uint_as_float(lw[j] << 16));
                        tv += (double)(__uint_as_float(hw[j] & 0xFFFF0000u) + __uint_as_float(lw[j] & 0xFFFF0000u));
                    }
                    if (col < d_pad) {
                        const size_t off = (size_t)col * (size_t)P.n_pad + (size_t)(r0 + rb);  // u16 elements
                        *reinterpret_cast<uint4*>(P.zhi + off) = hv;
                        *reinterpret_cast<uint4*>(P.zlo + off) = lv;
                    }
                }
            }
            // fixed-order sum of the column's 8 row groups (adjacent lanes)
            tv += __shfl_xor_sync(0xffffffffu, tv, 1);
            tv += __shfl_xor_sync(0xffffffffu, tv, 2);
            tv += __shfl_xor_sync(0xffffffffu, tv, 4);
            tacc += __double2ll_rn(tv * kFixScale);
        }
        __syncthreads();  // the plane staging is free
        slot = slot + 1 == kXfStages ? 0 : slot + 1;
        if (++L.rt == P.rtiles) {
            L.rt = 0;
            if (++L.strip == strips) {
                L.strip = 0;
                ++L.g;
            }
        }
    }
    cp_async_wait<0>();
    KS1_STAMP(3);
    if (t0 < t1) pair_done();
    KS1_STAMP(5);
    if (tid == 0) span_exit(a.span);
}

// KS3-lean (pairs below kStreamMinElems): tiles of 64 rows x 64 columns in the same (pair,
// strip, row block) order, 128 threads (one warp per SM sub-partition, so the CTA's
// registers fit beside a mask-GEMM CTA's), NO raw-tile ring: thread (row pair p, column
// group q) loads rows 2p + 16k, 2p + 1 + 16k (k < 4) x columns 4q..4q+3 (float4, 256
// coalesced bytes per row) and their {coef, 1/||h||} straight into registers, the next
// tile's in flight while the current one is transformed; z' = x - coef u - m (fp32, the
// arithmetic of KS3), bf16 hi/lo, two rows per 32-bit word into a TRANSPOSED staging tile
// [column][row] (17 KB for both planes); write thread = (column, 32 rows): 64 contiguous
// bytes per plane.  t' per column and tile in fp64, rounded per tile to fixed point,
// summed as int64 per strip run; the last CTA (ticket) runs P5.
constexpr int kXlRows = 64;
constexpr int kXlThreads = 128;
constexpr int kXlTW = kXlRows / 2 + 1;  // u32 words per staging column (33: conflict-free reads)

__global__ void __launch_bounds__(kXlThreads, 4) k1s_xform_lean(AlignArgs a, int64_t tile_off1, int64_t tile_off2,
                                                               int64_t tile_off3, int64_t tiles_total) {
    pdl_wait();  // KS2 (coefficients) complete and visible
    KS1_STAMP(7);
    __shared__ uint32_t sh_hi[kXfCols * kXlTW];
    __shared__ uint32_t sh_lo[kXfCols * kXlTW];
    __shared__ double red[2 * (kXlThreads / 32) + 2];
    __shared__ int s_last;
    const int tid = threadIdx.x;
    const int d = (int)a.d, d_pad = (int)a.d_pad;
    const int64_t t0 = tiles_total * blockIdx.x / gridDim.x, t1 = tiles_total * (blockIdx.x + 1) / gridDim.x;
    if (tid == 0) span_enter(a.span);
    const int q = tid & 15, p = tid >> 4;     // transform role: column group, row pair (0..7)
    const int wg = tid & 1, wc = tid >> 1;    // write role: 32-row half, column
    const int strips = (d_pad + kXfCols - 1) / kXfCols;
    struct TileAt {
        int g, strip, rt;
    };
    auto locate = [&](int64_t t) {
        TileAt L;
        L.g = (t >= tile_off1) + (t >= tile_off2) + (t >= tile_off3);
        const int64_t lt = t - (L.g == 0 ? 0 : L.g == 1 ? tile_off1 : L.g == 2 ? tile_off2 : tile_off3);
        const int64_t rtiles = (a.p[L.g].n_pad + kXlRows - 1) / kXlRows;
        L.strip = (int)(lt / rtiles);
        L.rt = (int)(lt % rtiles);
        return L;
    };
    auto advance = [&](TileAt& L) {
        const int64_t rtiles = (a.p[L.g].n_pad + kXlRows - 1) / kXlRows;
        if (++L.rt == rtiles) {
            L.rt = 0;
            if (++L.strip == strips) {
                L.strip = 0;
                ++L.g;
            }
        }
    };
    // row k (k < 8) of this thread: pair block k / 2, row 2p + (k & 1) + 16 (k / 2)
    auto row_of = [&](int k) { return 2 * p + (k & 1) + 16 * (k >> 1); };
    auto load = [&](const TileAt& L, float4 (&h)[8], float2 (&cv)[8]) {
        const AlignPair& qp = a.p[L.g];
        const int N = (int)(qp.n_x + qp.n_y);
        const int r0 = L.rt * kXlRows, c = L.strip * kXfCols + 4 * q;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int i = r0 + row_of(k);
            h[k] = (i < N && c < d) ? __ldcs(reinterpret_cast<const float4*>(row_ptr(qp, i) + c))
                                    : make_float4(0.f, 0.f, 0.f, 0.f);
            cv[k] = i < N ? __ldcg(qp.coef + i) : make_float2(0.f, 0.f);
        }
    };
    float4 hn[8];
    float2 cn[8];
    TileAt Ld = locate(t0);
    if (t0 < t1) load(Ld, hn, cn);
    TileAt L = Ld;
    long long tacc = 0;  // fixed-point t' of column wc of the current strip (wg == 0 lanes)
    int cur_g = -1, cur_strip = -1;
    float4 u4 = make_float4(0.f, 0.f, 0.f, 0.f), m4 = u4;
    auto flush = [&]() {
        const int c = cur_strip * kXfCols + wc;
        if (cur_g >= 0 && wg == 0 && c < d_pad && tacc != 0)
            atomicAdd(reinterpret_cast<unsigned long long*>(a.p[cur_g].acc + 2 * d + c), (unsigned long long)tacc);
        tacc = 0;
    };
    // a pair's P5 runs on the CTA that completes its last tile (per-pair ticket)
    int pg = L.g;
    unsigned pcnt = 0;
    auto pair_done = [&]() {
        flush();
        cur_g = -1;  // (flushed)
        const unsigned total = (unsigned)(strips * ((a.p[pg].n_pad + kXlRows - 1) / kXlRows));
        if (pair_ticket(a.p[pg], 5, pcnt, total, &s_last)) finish_pair<kXlThreads>(a, pg, red);
        pcnt = 0;
    };
    for (int64_t t = t0; t < t1; ++t) {
        if (L.g != pg) {
            pair_done();
            pg = L.g;
        }
        ++pcnt;
        float4 h[8];
        float2 cv[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            h[k] = hn[k];
            cv[k] = cn[k];
        }
        if (t + 1 < t1) {  // the next tile's rows in flight during this one
            advance(Ld);
            load(Ld, hn, cn);
        }
        if (L.g != cur_g || L.strip != cur_strip) {
            flush();
            cur_g = L.g;
            cur_strip = L.strip;
            const AlignPair& qp = a.p[L.g];
            float uu[4], mm[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int c = L.strip * kXfCols + 4 * q + k;
                uu[k] = c < d ? (float)__ldcg(qp.u + c) : 0.f;
                mm[k] = c < d ? (float)__ldcg(qp.m + c) : 0.f;
            }
            u4 = make_float4(uu[0], uu[1], uu[2], uu[3]);
            m4 = make_float4(mm[0], mm[1], mm[2], mm[3]);
        }
        const AlignPair& qp = a.p[L.g];
        const int N = (int)(qp.n_x + qp.n_y), n_pad = (int)qp.n_pad;
        const int r0 = L.rt * kXlRows, cb = L.strip * kXfCols;
        HAP_CHECK(L.g < a.G && r0 < n_pad && cb < d_pad && N <= n_pad);
        const bool cvalid = cb + 4 * q < d;
#pragma unroll
        for (int hp = 0; hp < 4; ++hp) {  // row pair (2p, 2p+1) + 16 hp
            float z[2][4];
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const int kk = 2 * hp + k;
                if (r0 + row_of(kk) < N && cvalid) {
                    z[k][0] = fmaf(-cv[kk].x, u4.x, h[kk].x * cv[kk].y) - m4.x;
                    z[k][1] = fmaf(-cv[kk].x, u4.y, h[kk].y * cv[kk].y) - m4.y;
                    z[k][2] = fmaf(-cv[kk].x, u4.z, h[kk].z * cv[kk].y) - m4.z;
                    z[k][3] = fmaf(-cv[kk].x, u4.w, h[kk].w * cv[kk].y) - m4.w;
                } else {
                    z[k][0] = z[k][1] = z[k][2] = z[k][3] = 0.f;
                }
            }
#pragma unroll
            for (int e = 0; e < 4; ++e) {  // column 4q + e: rows 2p + 16hp, +1 in one word
                const __nv_bfloat162 hh = __floats2bfloat162_rn(z[0][e], z[1][e]);
                const float2 hf = __bfloat1622float2(hh);
                const __nv_bfloat162 ll = __floats2bfloat162_rn(z[0][e] - hf.x, z[1][e] - hf.y);
                const int w = (4 * q + e) * kXlTW + p + 8 * hp;
                sh_hi[w] = *reinterpret_cast<const uint32_t*>(&hh);
                sh_lo[w] = *reinterpret_cast<const uint32_t*>(&ll);
            }
        }
        __syncthreads();  // planes staged (transposed)
        {
            const int col = cb + wc;
            const int rb = 32 * wg;
            double tv = 0.0;
            if (r0 + rb < n_pad) {
                uint32_t hw[16], lw[16];
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    hw[j] = sh_hi[wc * kXlTW + (rb >> 1) + j];
                    lw[j] = sh_lo[wc * kXlTW + (rb >> 1) + j];
                }
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    tv += (double)(__uint_as_float(hw[j] << 16) + __uint_as_float(lw[j] << 16));
                    tv += (double)(__uint_as_float(hw[j] & 0xFFFF0000u) + __uint_as_float(lw[j] & 0xFFFF0000u));
                }
                if (col < d_pad) {
                    const size_t off = (size_t)col * (size_t)n_pad + (size_t)(r0 + rb);  // u16 elements
                    uint4* dh = reinterpret_cast<uint4*>(qp.zt_hi + off);
                    uint4* dl = reinterpret_cast<uint4*>(qp.zt_lo + off);
#pragma unroll
                    for (int v = 0; v < 4; ++v) {
                        dh[v] = make_uint4(hw[4 * v], hw[4 * v + 1], hw[4 * v + 2], hw[4 * v + 3]);
                        dl[v] = make_uint4(lw[4 * v], lw[4 * v + 1], lw[4 * v + 2], lw[4 * v + 3]);
                    }
                }
            }
            tv += __shfl_xor_sync(0xffffffffu, tv, 1);  // the column's two halves, fixed order
            tacc += __double2ll_rn(tv * kFixScale);
        }
        __syncthreads();  // the staging is free
        advance(L);
    }
    if (t0 < t1) pair_done();
    if (tid == 0) span_exit(a.span);
}
}  // namespace

AlignGeom align_geometry(int64_t d) {
    // EXPERIMENT HAP_K1_SMEM_KB: cap K1's shared memory (so it fits beside a deeper K3 ring)
    static const char* cap_env = getenv("HAP_K1_SMEM_KB");
    const size_t cap = cap_env ? (size_t)atoi(cap_env) * 1024u : 220u * 1024u;
    AlignGeom g{};
    g.pitch = (int)(round_up(d, 16) + 2);  // = 2 (mod 16): conflict-free (column, row-pair) reads
    g.rows = kMaxItemRows;
    const size_t umc = (size_t)8 * round_up(d, 32), means = (size_t)16 * d;
    while (g.rows > 2 && (size_t)g.rows * g.pitch * 4 + std::min<size_t>(2 * umc, cap / 2) > std::min<size_t>(cap, 200u * 1024u))
        g.rows >>= 1;
    const size_t tile = (size_t)g.rows * g.pitch * 4;
    g.stage_umc = tile + 2 * umc <= cap;
    g.stage_means = g.stage_umc && tile + 2 * umc + means <= cap;
    g.smem = tile + (g.stage_umc ? 2 * umc : 0) + (g.stage_means ? means : 0);  // + t' partials
    return g;
}


// ---- K1s host side -------------------------------------------------------------------
// every pipeline kernel asks for the whole unified L1/shared array as shared memory, so the
// SM's carveout leaves room for the other lane's / next block's CTAs (see k_maskgemm.cu)
static cudaError_t max_carveout(const void* fn) {
    return cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
}
int align_path(int64_t N, int64_t d) {
    if (d % 4 != 0 || d > 4096) return kAlignFused;
    return round_up(N, kKBlock) * d >= kStreamMinElems ? kAlignRing : kAlignLean;
}

bool align_uses_stream(const AlignArgs& a) {
#ifdef HAP_EXPERIMENTS
    if (a.do_draws) return false;  // development build: KS1 writes per-CTA stamps (ks1_stamp)
#else
    if (a.do_draws || a.stamps) return false;  // experiments / K1 phase stamps: fused kernel only
#endif
    for (int g = 0; g < a.G; ++g) {
        const AlignPair& q = a.p[g];
        if (align_path(q.n_x + q.n_y, a.d) == kAlignFused) return false;
        if ((reinterpret_cast<uintptr_t>(q.X) | reinterpret_cast<uintptr_t>(q.Y)) & 15u) return false;
    }
    return true;
}

int align_launch_count(const AlignArgs& a) { return align_uses_stream(a) ? 3 : 1; }

static cudaError_t launch_align_ks23(AlignArgs a, int sm_count, cudaStream_t st, bool lean);

// launch with programmatic stream serialization: the kernel may start while the previous
// kernel on `st` finishes (its griddepcontrol.wait orders the reads); HAP_PDL=0 turns it off
template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*fn)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
    static const char* env = getenv("HAP_PDL");
    static const bool on = !(env && atoi(env) == 0);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = on ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, fn, std::forward<Args>(args)...);
}

static cudaError_t launch_align_stream(AlignArgs a, int sm_count, cudaStream_t st) {
    const int d = (int)a.d;
    // every pair of a launch takes the same variant (the callers form waves so)
    const bool lean = align_path(a.p[0].n_x + a.p[0].n_y, a.d) == kAlignLean;
    cudaError_t e;
    if (lean && d <= 1024) {  // KS1 warp-per-row variant (items of 8 rows)
        a.item_off[0] = 0;
        for (int g = 0; g < a.G; ++g)
            a.item_off[g + 1] = a.item_off[g] + ceil_div(a.p[g].n_x + a.p[g].n_y, kSWRows);
        const int G = (int)ceil_div(d, 128);
        const void* fw[8] = {(const void*)k1s_stats_warp<1>, (const void*)k1s_stats_warp<2>,
                             (const void*)k1s_stats_warp<3>, (const void*)k1s_stats_warp<4>,
                             (const void*)k1s_stats_warp<5>, (const void*)k1s_stats_warp<6>,
                             (const void*)k1s_stats_warp<7>, (const void*)k1s_stats_warp<8>};
        const void* fn = fw[G - 1];
        static bool sw_configured[8] = {};
        if (!sw_configured[G - 1]) {
            e = max_carveout(fn);
            if (e != cudaSuccess) return e;
            sw_configured[G - 1] = true;
        }
        const int64_t items = a.item_off[a.G];
        // ~4 items per CTA (one per warp), at least one CTA per pair
        const int grid = (int)std::max<int64_t>(a.G, std::min<int64_t>(ceil_div(items, 4), 4ll * sm_count));
        void* args[] = {&a};
        e = cudaLaunchKernel(fn, dim3(grid), dim3(kS1LeanThreads), args, (size_t)2 * d * 8, st);
        if (e != cudaSuccess) return e;
        return launch_align_ks23(a, sm_count, st, lean);
    }
    const int nt1 = lean ? kS1LeanThreads : kS1Threads;
    const int g4 = (int)ceil_div(d / 4, nt1);           // float4 column groups per thread
    const int G4t = g4 <= 1 ? 1 : g4 <= 2 ? 2 : g4 <= 4 ? 4 : 8;  // template instance
    const int R = 8 / G4t;                              // rows per item (= the kernel's)
    a.item_off[0] = 0;
    for (int g = 0; g < a.G; ++g) a.item_off[g + 1] = a.item_off[g] + ceil_div(a.p[g].n_x + a.p[g].n_y, R);
    const int64_t items = a.item_off[a.G];
    const size_t smem1 = lean ? 0 : 128 + (size_t)kSStages * R * d * 4;
    const void* fn = lean ? (G4t == 1   ? (const void*)k1s_stats<1, false, kS1LeanThreads>
                             : G4t == 2 ? (const void*)k1s_stats<2, false, kS1LeanThreads>
                             : G4t == 4 ? (const void*)k1s_stats<4, false, kS1LeanThreads>
                                        : (const void*)k1s_stats<8, false, kS1LeanThreads>)
                          : (G4t == 1 ? (const void*)k1s_stats<1>
                             : G4t == 2 ? (const void*)k1s_stats<2>
                                        : (const void*)k1s_stats<4>);
    static size_t configured[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // dynamic smem configured + 1
    const int fi = (G4t == 1 ? 0 : G4t == 2 ? 1 : G4t == 4 ? 2 : 3) + (lean ? 4 : 0);
    if (smem1 + 1 > configured[fi]) {
        e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem1);
        if (e == cudaSuccess) e = max_carveout(fn);
        if (e != cudaSuccess) return e;
        configured[fi] = smem1 + 1;
    }
    {
        const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(items, (lean ? 4ll : 2ll) * sm_count));
        void* args[] = {&a};
        e = cudaLaunchKernel(fn, dim3(grid), dim3(nt1), args, smem1, st);
        if (e != cudaSuccess) return e;
    }
    return launch_align_ks23(a, sm_count, st, lean);
}

static cudaError_t launch_align_ks23(AlignArgs a, int sm_count, cudaStream_t st, bool lean) {
    cudaError_t e;
    // KS2 derives P3 itself unless KS1 was the warp-per-row variant (lean, d <= 1024), whose
    // ticketed P3 is a single short round trip (and whose waves run beside the mask-GEMM)
    const bool p3 = !(lean && a.d <= 1024);
    {  // KS2: CTAs in proportion to the pairs' X rows (kP3: at most what is resident at once)
        const size_t smem2 = (size_t)a.d_pad * 8 * (p3 ? 2 : 1);  // u (= xbar) (+ ybar)
        int cpp[kMaxWave] = {0, 0, 0, 0}, total = 0;
        if (p3) {
            static int per_sm[2] = {0, 0};  // resident CTAs per SM for d_pad <= / > 2048
            const int big = a.d_pad > 2048;
            if (per_sm[big] == 0) {
                e = cudaFuncSetAttribute(k1s_coef<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4096 * 8 * 2);
                if (e == cudaSuccess) e = max_carveout((const void*)k1s_coef<true>);
                if (e == cudaSuccess)
                    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[big], k1s_coef<true>, kCoefThreads,
                                                                      (big ? 4096 : 2048) * 8 * 2);
                if (e != cudaSuccess) return e;
                per_sm[big] = std::max(per_sm[big], 1);
            }
            const int64_t cap = (int64_t)per_sm[big] * sm_count;
            int64_t rows = 0;
            for (int g = 0; g < a.G; ++g) rows += a.p[g].n_x;
            for (int g = 0; g < a.G; ++g) {  // one warp per X row at a time (8 warps per CTA)
                const int64_t want = ceil_div(a.p[g].n_x, 8);
                const int64_t share = rows > 0 ? ceil_div(cap * a.p[g].n_x, rows) : 1;
                cpp[g] = (int)std::max<int64_t>(1, std::min(want, share));
                total += cpp[g];
            }
            e = launch_pdl(k1s_coef<true>, dim3(total), dim3(kCoefThreads), smem2, st, a, cpp[0], cpp[1], cpp[2],
                           cpp[3]);
        } else {
            for (int g = 0; g < a.G; ++g) {  // one warp per X row (8 warps per CTA)
                cpp[g] = (int)std::max<int64_t>(1, ceil_div(a.p[g].n_x, 8));
                total += cpp[g];
            }
            e = launch_pdl(k1s_coef<false>, dim3(total), dim3(kCoefThreads), smem2, st, a, cpp[0], cpp[1], cpp[2],
                           cpp[3]);
        }
        if (e != cudaSuccess) return e;
    }
    if (lean) {  // KS3-lean: 64-row tiles, two CTAs per SM at most
        const int64_t strips = ceil_div(a.d_pad, kXfCols);
        int64_t off[kMaxWave + 1] = {0, 0, 0, 0, 0};
        for (int g = 0; g < a.G; ++g) off[g + 1] = off[g] + strips * ceil_div(a.p[g].n_pad, kXlRows);
        for (int g = a.G + 1; g <= kMaxWave; ++g) off[g] = off[a.G];
        const int64_t total = off[a.G];
        const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(total, 4ll * sm_count));
        static bool xl_configured = false;
        if (!xl_configured) {
            e = max_carveout((const void*)k1s_xform_lean);
            if (e == cudaSuccess) e = max_carveout((const void*)k1s_coef<false>);
            if (e != cudaSuccess) return e;
            xl_configured = true;
        }
        return launch_pdl(k1s_xform_lean, dim3(grid), dim3(kXlThreads), 0, st, a, off[1], off[2], off[3], total);
    }
    {  // KS3
        const int64_t strips = ceil_div(a.d_pad, kXfCols);
        int64_t off[kMaxWave + 1] = {0, 0, 0, 0, 0};
        for (int g = 0; g < a.G; ++g) off[g + 1] = off[g] + strips * ceil_div(a.p[g].n_pad, kXfRows);
        for (int g = a.G + 1; g <= kMaxWave; ++g) off[g] = off[a.G];
        const int64_t total = off[a.G];
        const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(total, sm_count));
        static bool xf_configured = false;
        if (!xf_configured) {
            e = cudaFuncSetAttribute(k1s_xform, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kXfSmem);
            if (e == cudaSuccess) e = max_carveout((const void*)k1s_xform);
            if (e != cudaSuccess) return e;
            xf_configured = true;
        }
        e = launch_pdl(k1s_xform, dim3(grid), dim3(kThreads), kXfSmem, st, a, off[1], off[2], off[3], total);
    }
    return e;
}

// Cooperative grids of different streams could each be partly resident and wait for each
// other's SMs at their grid barriers; every K1 launch of the process is therefore ordered
// after the previous one on the device (an event chain; K1 is latency-bound and short).
static std::mutex g_k1_mu;
static cudaEvent_t g_k1_last[64] = {};

void align_items(AlignArgs& a) {
    const AlignGeom g = align_geometry(a.d);
    a.item_off[0] = 0;
    for (int k = 0; k < a.G; ++k) a.item_off[k + 1] = a.item_off[k] + a.p[k].n_pad / g.rows;
}

cudaError_t launch_align(const AlignArgs& a, int grid, cudaStream_t st) {
    if (align_uses_stream(a)) return launch_align_stream(a, grid, st);
    const AlignGeom g = align_geometry(a.d);
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(g_k1_mu);
    cudaEvent_t& last = g_k1_last[dev & 63];
    if (!last) {
        cudaError_t e = cudaEventCreateWithFlags(&last, cudaEventDisableTiming);
        if (e != cudaSuccess) return e;
    } else {
        cudaError_t e = cudaStreamWaitEvent(st, last, 0);
        if (e != cudaSuccess) return e;
    }
    const void* fn = g.rows == 16 ? (const void*)k1_align_fused<16>
                     : g.rows == 8 ? (const void*)k1_align_fused<8>
                     : g.rows == 4 ? (const void*)k1_align_fused<4>
                                   : (const void*)k1_align_fused<2>;
    static size_t configured[5] = {0, 0, 0, 0, 0};
    const int fi = g.rows == 16 ? 4 : g.rows == 8 ? 3 : g.rows == 4 ? 2 : 1;
    if (g.smem > configured[fi]) {
        cudaError_t e = g.smem > 48 * 1024
                            ? cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g.smem)
                            : cudaSuccess;
        if (e == cudaSuccess) e = max_carveout(fn);
        if (e != cudaSuccess) return e;
        configured[fi] = g.smem;
    }
    AlignArgs copy = a;
    int P = g.pitch, su = g.stage_umc ? 1 : 0, sm = g.stage_means ? 1 : 0;
    void* args[] = {&copy, &P, &su, &sm};
    // no more CTAs than items: small pairs (C1, the small tests of a C4 batch) then pay a
    // grid barrier and a ticket over few CTAs
    const int64_t items = a.item_off[a.G];
    const int g_ctas = (int)std::max<int64_t>(1, std::min<int64_t>(grid, items));
    cudaError_t e = cudaLaunchCooperativeKernel(fn, dim3(g_ctas), dim3(kThreads), args, g.smem, st);
    if (e != cudaSuccess) return e;
    return cudaEventRecord(last, st);
}

HAP_CHECK_ACCESSOR(check_word_align)

}  // namespace hap
