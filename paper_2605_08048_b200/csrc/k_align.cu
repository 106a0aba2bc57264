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
// latency, not bandwidth: one persistent cooperative grid (one CTA per SM) runs the five
// phases below separated by four software grid barriers.  Every reduction is fixed-order
// (per-CTA partials combined in ascending CTA order by a warp xor-tree or a block tree), so
// Z~ and t are bit-identical across runs and ranks; scalars needed by every CTA are reduced
// redundantly by every CTA from the same partials (identical results, no broadcast).
//   P1 rows   : norms (ZeroVector check) + per-CTA fp64 column partials of X and of Y
//   P2 columns: xbar, ybar (warp per column over the CTA partials); partials of |xbar|^2..
//   P3 columns: ||xbar||, ||ybar||; partials of ||v||^2, v.xbar (v = mu_x - mu_y); rows:
//               xbar.h_i, ybar.h_i for the reflection coefficients
//   P4 tiles  : info; 32x64 tiles: axis u and centre m per column, coef from the P3 dots,
//               reflect, centre, bf16 hi/lo split, transpose, t partials
//   P5 columns: t, epilogue constants {2a, 2b}; the last CTA (ticket) forms sum a^2, sum b^2
#include <cuda_bf16.h>

#include <cfloat>
#include <climits>

#include "hap_device.cuh"
#include "hap_internal.h"

namespace hap {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kSpartStride = 8;  // doubles per CTA in spart: P2 [0,1], P3 [2,3], P6 [4,5]

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// block-wide fixed-order fp64 sum
__device__ double block_sum(double v, double* red) {
    v = warp_sum(v);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int i = 0; i < kWarps; ++i) s += red[i];
        red[32] = s;
    }
    __syncthreads();
    return red[32];
}

// sum over CTAs p of spart[p*kSpartStride + k], fixed order (same in every CTA)
__device__ double cta_partials_sum(const double* spart, int k, double* red) {
    double v = 0.0;
    for (int p = threadIdx.x; p < (int)gridDim.x; p += kThreads)
        v += __ldcg(spart + (size_t)p * kSpartStride + k);
    return block_sum(v, red);
}

__device__ __forceinline__ void stamp(const AlignArgs& a, int k) {
    if (a.stamps && blockIdx.x == 0 && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        a.stamps[k] = (long long)t;
    }
}

// Software grid barrier (all CTAs are co-resident: cooperative launch).  bar[0] counts
// arrivals, bar[1] is the generation; the last arriver resets the count before bumping
// the generation, so a CTA that sees the new generation also sees the reset.
__device__ __forceinline__ void grid_sync(unsigned* bar) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned* vb = bar;
        const unsigned gen = vb[1];
        __threadfence();
        if (atomicAdd(bar, 1u) == gridDim.x - 1) {
            vb[0] = 0u;
            __threadfence();
            atomicAdd(bar + 1, 1u);
        } else {
            while (vb[1] == gen) __nanosleep(32);
        }
        __threadfence();
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

__device__ __forceinline__ const float* row_ptr(const AlignArgs& a, int64_t i) {
    return i < a.n_x ? a.X + i * a.d : a.Y + (i - a.n_x) * a.d;
}

constexpr int kSP = 33;  // padded smem pitch (32-bit words) of a 64-row bf16 column

__global__ void __launch_bounds__(kThreads, 1) k1_align_fused(AlignArgs a) {
    __shared__ double red[33];
    __shared__ double s_inv[512];
    __shared__ uint32_t s_hi[64 * kSP];
    __shared__ uint32_t s_lo[64 * kSP];
    const int G = gridDim.x, cta = blockIdx.x;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t N = a.n_x + a.n_y;
    const bool vec = (a.d & 3) == 0;
    unsigned* bar = reinterpret_cast<unsigned*>(a.scratch + 2);
    stamp(a, 0);

    // ---------------- P1: norms + per-CTA column partials (X slice and Y slice)
    for (int q = 0; q < 2; ++q) {
        const int64_t n = q ? a.n_y : a.n_x;
        const int64_t r0 = n * cta / G, r1 = n * (cta + 1) / G;  // <= 443 rows (N <= 65535)
        const int64_t base = q ? a.n_x : 0;
        for (int64_t r = r0 + warp; r < r1; r += kWarps) {
            const float* h = row_ptr(a, base + r);
            double s = 0.0;
            if (vec) {
                const float4* h4 = reinterpret_cast<const float4*>(h);
#pragma unroll 4
                for (int64_t c = lane; c < a.d / 4; c += 32) {
                    const float4 v = __ldg(h4 + c);
                    s += (double)v.x * v.x + (double)v.y * v.y + (double)v.z * v.z +
                         (double)v.w * v.w;
                }
            } else {
                for (int64_t c = lane; c < a.d; c += 32) {
                    const double v = (double)__ldg(h + c);
                    s += v * v;
                }
            }
            s = warp_sum(s);
            if (lane == 0) {
                const double nrm = sqrt(s);
                const double iv = nrm < 1e-12 ? 0.0 : 1.0 / nrm;
                a.inv[base + r] = iv;
                s_inv[r - r0] = iv;
                if (nrm < 1e-12)
                    atomicMin(reinterpret_cast<long long*>(a.scratch), (long long)(base + r));
            }
        }
        __syncthreads();
        double* part = a.part + (size_t)(2 * cta + q) * a.d;
        const int nr = (int)(r1 - r0);
        if (vec) {
            for (int64_t c4 = tid; c4 < a.d / 4; c4 += kThreads) {
                double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
#pragma unroll 8
                for (int r = 0; r < nr; ++r) {
                    const float4 v =
                        __ldg(reinterpret_cast<const float4*>(row_ptr(a, base + r0 + r)) + c4);
                    const double iv = s_inv[r];
                    s0 += (double)v.x * iv;
                    s1 += (double)v.y * iv;
                    s2 += (double)v.z * iv;
                    s3 += (double)v.w * iv;
                }
                part[4 * c4 + 0] = s0;
                part[4 * c4 + 1] = s1;
                part[4 * c4 + 2] = s2;
                part[4 * c4 + 3] = s3;
            }
        } else {
            for (int64_t c = tid; c < a.d; c += kThreads) {
                double acc = 0.0;
                for (int r = 0; r < nr; ++r)
                    acc += (double)__ldg(row_ptr(a, base + r0 + r) + c) * s_inv[r];
                part[c] = acc;
            }
        }
        __syncthreads();
    }
    grid_sync(bar);
    stamp(a, 1);

    // ---------------- P2: xbar_c, ybar_c = (sum over CTA partials, lane-strided + xor tree)/n
    {
        double sxx = 0.0, syy = 0.0;
        for (int64_t it = (int64_t)cta * kWarps + warp; it < 2 * a.d; it += (int64_t)G * kWarps) {
            const int q = (int)(it / a.d);
            const int64_t c = it % a.d;
            double v = 0.0;
#pragma unroll 8
            for (int p = lane; p < G; p += 32) v += __ldcg(a.part + (size_t)(2 * p + q) * a.d + c);
            v = warp_sum(v) / (double)(q ? a.n_y : a.n_x);
            if (lane == 0) {
                (q ? a.ybar : a.xbar)[c] = v;
                if (q) syy += v * v;
                else sxx += v * v;
            }
        }
        sxx = block_sum(sxx, red);
        syy = block_sum(syy, red);
        if (tid == 0) {
            a.spart[(size_t)cta * kSpartStride + 0] = sxx;
            a.spart[(size_t)cta * kSpartStride + 1] = syy;
        }
    }
    grid_sync(bar);
    stamp(a, 2);

    // ---------------- P3: norms; partials of ||v||^2 and v.xbar
    const double nx = sqrt(cta_partials_sum(a.spart, 0, red));
    const double ny = sqrt(cta_partials_sum(a.spart, 1, red));
    const bool degenerate = nx < 1e-12 || ny < 1e-12;
    const double rnx = degenerate ? 0.0 : 1.0 / nx, rny = degenerate ? 0.0 : 1.0 / ny;
    {
        double sv = 0.0, svx = 0.0;
        for (int64_t c = (int64_t)cta * kThreads + tid; c < a.d; c += (int64_t)G * kThreads) {
            const double xb = __ldcg(a.xbar + c), yb = __ldcg(a.ybar + c);
            const double v = xb * rnx - yb * rny;
            sv += v * v;
            svx += v * xb;
        }
        sv = block_sum(sv, red);
        svx = block_sum(svx, red);
        if (tid == 0) {
            a.spart[(size_t)cta * kSpartStride + 2] = sv;
            a.spart[(size_t)cta * kSpartStride + 3] = svx;
        }
        // row dots for the reflection coefficients (they do not need ||v||):
        // coef_i = 2 u^T x_i = 2 (xbar.h_i / ||xbar|| - ybar.h_i / ||ybar||) / (||v|| ||h_i||)
        if (a.mode != HAP_ALIGN_NONE && !degenerate) {
            for (int64_t i = (int64_t)cta * kWarps + warp; i < a.n_x; i += (int64_t)G * kWarps) {
                const float* h = a.X + i * a.d;
                double dx = 0.0, dy = 0.0;
#pragma unroll 8
                for (int64_t c = lane; c < a.d; c += 32) {
                    const double hv = (double)__ldg(h + c);
                    dx += hv * __ldcg(a.xbar + c);
                    dy += hv * __ldcg(a.ybar + c);
                }
                dx = warp_sum(dx);
                dy = warp_sum(dy);
                if (lane == 0) a.coef[i] = (dx * rnx - dy * rny) * __ldcg(a.inv + i);
            }
        }
    }
    grid_sync(bar);
    stamp(a, 3);

    // ---------------- P4: identity, info; then 32-row tiles, each CTA self-contained:
    // coefficients coef_i = 2 u^T x_i of its rows, axis u_c and centre m_c per column (both
    // from the means), z' = h/||h|| - coef u - m (fp32 is ample: the value is then kept to
    // 16 significant bits), hi/lo split, transpose, fixed-order t partial per column
    const double nv0 = sqrt(cta_partials_sum(a.spart, 2, red));
    const double vx = cta_partials_sum(a.spart, 3, red);
    const bool identity = (a.mode == HAP_ALIGN_NONE) || degenerate || nv0 < 1e-9;  // R3
    const double rnv = identity ? 0.0 : 1.0 / nv0;
    const double ux = vx * rnv;  // u . xbar
    const double rN = 4096.0 / (double)N;
    if (cta == 0 && tid == 0) {
        hap_align_info* f = a.info;
        const long long bad = *reinterpret_cast<volatile long long*>(a.scratch);
        f->n_x = a.n_x;
        f->n_y = a.n_y;
        f->d = a.d;
        f->n_pad = a.n_pad;
        f->d_pad = a.d_pad;
        f->is_identity = identity ? 1 : 0;
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
    {
        // 2-D tiles (32 rows x 64 columns); P3 stored (u^T x_i) * ||v|| in coef[i]
        double* s_cf = s_inv;         // [32] 2 u^T x_i of the tile rows
        double* s_iv = s_inv + 64;    // [32] 1/||h_i||
        uint16_t* sh16 = reinterpret_cast<uint16_t*>(s_hi);
        uint16_t* sl16 = reinterpret_cast<uint16_t*>(s_lo);
        const int64_t ntr = a.n_pad / kRowTile, ntc = (a.d_pad + 63) / 64;
        for (int64_t tile = cta; tile < ntr * ntc; tile += G) {
            const int64_t rt = tile / ntc, c0 = (tile % ntc) * 64;
            const int64_t r0 = rt * kRowTile;
            if (tid < kRowTile) {
                const int64_t i = r0 + tid;
                s_cf[tid] = (i < a.n_x && !identity) ? 2.0 * __ldcg(a.coef + i) * rnv : 0.0;
                s_iv[tid] = i < N ? __ldcg(a.inv + i) : 0.0;
            }
            const int tc = tid & 63, tr = tid >> 6;  // 64 columns x 4 row groups of 8
            const int64_t c = c0 + tc;
            float hv[kRowTile / 4];
#pragma unroll
            for (int j = 0; j < kRowTile / 4; ++j) {  // issue all loads first
                const int64_t i = r0 + tr + 4 * j;
                hv[j] = (i < N && c < a.d) ? __ldg(row_ptr(a, i) + c) : 0.f;
            }
            double ud = 0.0, md = 0.0;
            if (c < a.d) {
                const double xb = __ldcg(a.xbar + c), yb = __ldcg(a.ybar + c);
                ud = (xb * rnx - yb * rny) * rnv;
                // centre m = t/N quantised to 2^-12, t = n_x (xbar - 2u(u.xbar)) + n_y ybar
                const double t = (double)a.n_x * (xb - 2.0 * ud * ux) + (double)a.n_y * yb;
                md = rint(t * rN) * (1.0 / 4096.0);
            }
            if (rt == 0 && tr == 0 && c < a.d_pad) {  // export copies (read in P5)
                a.u[c] = ud;
                a.m[c] = md;
            }
            __syncthreads();
            const float uc = (float)ud, mc = (float)md;
#pragma unroll
            for (int j = 0; j < kRowTile / 4; ++j) {
                const int rl = tr + 4 * j;
                const float z = (r0 + rl < N && c < a.d)
                                    ? fmaf(-(float)s_cf[rl], uc, hv[j] * (float)s_iv[rl]) - mc
                                    : 0.f;
                const __nv_bfloat16 hi = __float2bfloat16_rn(z);
                const __nv_bfloat16 lo = __float2bfloat16_rn(z - __bfloat162float(hi));
                sh16[tc * (2 * kSP) + rl] = __bfloat16_as_ushort(hi);
                sl16[tc * (2 * kSP) + rl] = __bfloat16_as_ushort(lo);
            }
            __syncthreads();
            // 32 rows = 16 words per column: half-warps write one column each
            const int hw = lane >> 4, hl = lane & 15;
            for (int cc = 2 * warp + hw; cc < 64; cc += 2 * kWarps) {
                const int64_t col = c0 + cc;
                double v = 0.0;
                if (col < a.d_pad) {
                    const uint32_t vh = s_hi[cc * kSP + hl], vl = s_lo[cc * kSP + hl];
                    reinterpret_cast<uint32_t*>(a.zt_hi + col * a.n_pad + r0)[hl] = vh;
                    reinterpret_cast<uint32_t*>(a.zt_lo + col * a.n_pad + r0)[hl] = vl;
                    v = (double)__bfloat162float(__ushort_as_bfloat16((uint16_t)(vh & 0xFFFF))) +
                        (double)__bfloat162float(__ushort_as_bfloat16((uint16_t)(vl & 0xFFFF))) +
                        (double)__bfloat162float(__ushort_as_bfloat16((uint16_t)(vh >> 16))) +
                        (double)__bfloat162float(__ushort_as_bfloat16((uint16_t)(vl >> 16)));
                }
#pragma unroll
                for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                if (hl == 0 && col < a.d_pad) a.tpart[rt * a.d_pad + col] = v;
            }
            __syncthreads();
        }
    }
    grid_sync(bar);
    stamp(a, 4);

    // ---------------- P5: t = N m + sum of tile partials (lane-strided + xor tree);
    // a = n_x m, b = t - a (fp32) for the GEMM epilogue; partials of sum a^2, sum b^2;
    // the last CTA to finish (ticket) forms {sum a^2, sum b^2} in fixed order
    {
        __shared__ int s_last;
        const int64_t ntr = a.n_pad / kRowTile;
        double sa = 0.0, sb = 0.0;
        for (int64_t c = (int64_t)cta * kWarps + warp; c < a.d_pad; c += (int64_t)G * kWarps) {
            double tp = 0.0;
#pragma unroll 4
            for (int64_t t = lane; t < ntr; t += 32) tp += __ldcg(a.tpart + t * a.d_pad + c);
            tp = warp_sum(tp);
            if (lane == 0) {
                const double m = __ldcg(a.m + c);
                a.t64[c] = (double)N * m + tp;
                const float af = (float)((double)a.n_x * m);
                const float bf = (float)((double)a.n_y * m + tp);
                a.ab[c] = make_float2(2.0f * af, 2.0f * bf);
                sa += (double)af * (double)af;
                sb += (double)bf * (double)bf;
            }
        }
        sa = block_sum(sa, red);
        sb = block_sum(sb, red);
        if (tid == 0) {
            a.spart[(size_t)cta * kSpartStride + 4] = sa;
            a.spart[(size_t)cta * kSpartStride + 5] = sb;
            __threadfence();
            unsigned* ticket = reinterpret_cast<unsigned*>(a.scratch + 1);
            s_last = atomicAdd(ticket, 1u) == (unsigned)G - 1;
        }
        __syncthreads();
        if (s_last) {
            __threadfence();
            const double SA = cta_partials_sum(a.spart, 4, red);
            const double SB = cta_partials_sum(a.spart, 5, red);
            if (tid == 0) {
                a.sconst[0] = SA;
                a.sconst[1] = SB;
                a.scratch[0] = LLONG_MAX;  // reset the ZeroVector word and the ticket
                reinterpret_cast<unsigned*>(a.scratch + 1)[0] = 0u;
            }
        }
    }
    stamp(a, 5);
}

}  // namespace

cudaError_t launch_align(const AlignArgs& a, int grid, cudaStream_t st) {
    AlignArgs copy = a;
    void* args[] = {&copy};
    return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k1_align_fused), dim3(grid),
                                       dim3(kThreads), args, 0, st);
}

}  // namespace hap
