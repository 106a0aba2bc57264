// k_align.cu — K1: S1-S6 of the hot path (DESIGN.md "Kernels" K1a-K1e).
//
//   S1 normalise   x = h/||h||               PAPER.md:115-118 (§3.1 Eq. 2)
//   S2 means       xbar, ybar, mu_x, mu_y    PAPER.md:143-148; Alg. 1
//   S3 axis        u = (mu_x-mu_y)/||.||     PAPER.md:149-156 (Eqs. 5-6); Alg. 1 :664
//   S4 reflect     x' = x - 2u(u^T x)        PAPER.md:157-161, 245-255 (Eq. householder_fast)
//   S5 pool+split  Z = [X';Y] -> centred bf16 hi/lo planes (transposed, K contiguous),
//                  t = 1^T Z                 PAPER.md:183, 215-218 (Eq. gemm), 258
//   S6 observed    r_X = ||xbar|| (= r(X')), r_Y, T_obs (Eq. 10), fp64
//
// Five grid-wide kernels, none single-CTA: per-row-block partials (K1a), per-column means
// with a last-arriving-CTA scalar finalize (K1b), per-row reflection coefficients (K1c),
// reflect/centre/split/transpose tiles (K1d), per-column totals with a last-CTA finalize of
// the epilogue constants (K1e).  All reductions are fixed-order (partials summed in
// ascending block order), so Z~ and t are bit-identical across runs and ranks.
#include <cuda_bf16.h>

#include <cfloat>
#include <climits>

#include "hap_device.cuh"
#include "hap_internal.h"

namespace hap {
namespace {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// block-wide fixed-order fp64 sum (blockDim.x multiple of 32, <= 1024)
__device__ double block_sum(double v, double* red) {
    v = warp_sum(v);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += red[i];
        red[32] = s;
    }
    __syncthreads();
    return red[32];
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

// ---------------------------------------------------------------------------------
// K1a (S1 + S2 partials): one CTA per block of kRowBlock rows of X or of Y.
// Phase 1: warp-per-row fp64 norms ||h_i|| (ZeroVector check).
// Phase 2: fp64 column partial sums of the normalised rows h_i/||h_i||.
__global__ void __launch_bounds__(256) k1a_norm_colsum(AlignArgs a, int nblk_x) {
    __shared__ double s_inv[kRowBlock];
    const bool isx = (int)blockIdx.x < nblk_x;
    const int64_t blk = isx ? blockIdx.x : blockIdx.x - nblk_x;
    const int64_t nrows = isx ? a.n_x : a.n_y;
    const int64_t r0 = blk * kRowBlock;
    const int rn = (int)((nrows - r0 < kRowBlock) ? (nrows - r0) : (int64_t)kRowBlock);
    const int64_t base = isx ? r0 : a.n_x + r0;  // pooled row index of local row 0
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    const bool vec = (a.d & 3) == 0;
    for (int r = w; r < rn; r += 8) {
        const float* h = row_ptr(a, base + r);
        double s = 0.0;
        if (vec) {
            const float4* h4 = reinterpret_cast<const float4*>(h);
            for (int64_t c = l; c < a.d / 4; c += 32) {
                const float4 v = __ldg(h4 + c);
                s += (double)v.x * v.x + (double)v.y * v.y + (double)v.z * v.z + (double)v.w * v.w;
            }
        } else {
            for (int64_t c = l; c < a.d; c += 32) {
                const double v = (double)h[c];
                s += v * v;
            }
        }
        s = warp_sum(s);
        if (l == 0) {
            const double nrm = sqrt(s);
            a.nrm[base + r] = nrm;
            a.inv[base + r] = nrm < 1e-12 ? 0.0 : 1.0 / nrm;
            if (nrm < 1e-12) atomicMin(reinterpret_cast<long long*>(a.scratch), (long long)(base + r));
            s_inv[r] = nrm < 1e-12 ? 0.0 : 1.0 / nrm;
        }
    }
    __syncthreads();
    double* part = a.part + (int64_t)blockIdx.x * a.d;
    if (vec) {
        for (int64_t c4 = threadIdx.x; c4 < a.d / 4; c4 += blockDim.x) {
            double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
            for (int r = 0; r < rn; ++r) {
                const float4 v = __ldg(reinterpret_cast<const float4*>(row_ptr(a, base + r)) + c4);
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
        for (int64_t c = threadIdx.x; c < a.d; c += blockDim.x) {
            double acc = 0.0;
            for (int r = 0; r < rn; ++r) acc += (double)row_ptr(a, base + r)[c] * s_inv[r];
            part[c] = acc;
        }
    }
}

// ---------------------------------------------------------------------------------
// K1b (S2 finish + S3 + S6): CTA per 256 columns: xbar_c, ybar_c from the block partials
// (ascending block order), per-CTA partial sums of ||xbar||^2, ||ybar||^2.  The last CTA
// to finish (atomic ticket) finalises the scalars in fixed order: norms, DegenerateMean,
// v = mu_x - mu_y (||v|| and v.xbar summed directly), identity test, r, L, T_obs, info.
constexpr int kMeanCols = 64;   // columns per CTA in K1b / K1e
constexpr int kMeanGroups = 4;  // threads per column, each summing a contiguous block range
__device__ __forceinline__ double grouped_colsum(const double* base, int64_t stride, int nblk,
                                                int g, double* s_grp, int col) {
    // fixed order: group g sums blocks [g*q, (g+1)*q) ascending; groups combined 0..3
    const int q = (nblk + kMeanGroups - 1) / kMeanGroups;
    const int b0 = g * q, b1 = min(nblk, b0 + q);
    double acc = 0.0;
#pragma unroll 8
    for (int b = b0; b < b1; ++b) acc += __ldcg(base + (int64_t)b * stride);
    s_grp[g * kMeanCols + col] = acc;
    __syncthreads();
    double tot = 0.0;
#pragma unroll
    for (int gg = 0; gg < kMeanGroups; ++gg) tot += s_grp[gg * kMeanCols + col];
    __syncthreads();
    return tot;
}

__global__ void __launch_bounds__(kMeanCols * kMeanGroups) k1b_means(AlignArgs a, int nblk_x, int nblk_y) {
    __shared__ double red[33];
    __shared__ double s_grp[kMeanGroups * kMeanCols];
    __shared__ int s_last;
    const int col = threadIdx.x % kMeanCols, g = threadIdx.x / kMeanCols;
    const int64_t c = (int64_t)blockIdx.x * kMeanCols + col;
    const int64_t cc0 = c < a.d ? c : 0;
    const double xs = grouped_colsum(a.part + cc0, a.d, nblk_x, g, s_grp, col);
    const double ys = grouped_colsum(a.part + (int64_t)nblk_x * a.d + cc0, a.d, nblk_y, g, s_grp, col);
    double sxx = 0.0, syy = 0.0;
    if (c < a.d && g == 0) {
        const double xb = xs / (double)a.n_x, yb = ys / (double)a.n_y;
        a.xbar[c] = xb;
        a.ybar[c] = yb;
        sxx = xb * xb;
        syy = yb * yb;
    }
    sxx = block_sum(sxx, red);
    syy = block_sum(syy, red);
    if (threadIdx.x == 0) {
        a.spart[2 * blockIdx.x + 0] = sxx;
        a.spart[2 * blockIdx.x + 1] = syy;
        __threadfence();
        const unsigned t = atomicAdd(reinterpret_cast<unsigned*>(a.scratch + 1), 1u);
        s_last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    // ---- last CTA: scalars (fixed order), then u (S3)
    double SX = 0.0, SY = 0.0;
    if (threadIdx.x < gridDim.x) {
        SX = __ldcg(a.spart + 2 * threadIdx.x);
        SY = __ldcg(a.spart + 2 * threadIdx.x + 1);
    }
    SX = block_sum(SX, red);
    SY = block_sum(SY, red);
    const double nx = sqrt(SX), ny = sqrt(SY);
    const bool degenerate = nx < 1e-12 || ny < 1e-12;
    bool identity = (a.mode == HAP_ALIGN_NONE) || degenerate;
    double nv = 0.0, vx = 0.0;
    const double rnx = degenerate ? 0.0 : 1.0 / nx, rny = degenerate ? 0.0 : 1.0 / ny;
    if (!identity) {
        double sv = 0.0, svx = 0.0;
        for (int64_t cc = threadIdx.x; cc < a.d; cc += blockDim.x) {
            const double xb = __ldcg(a.xbar + cc), yb = __ldcg(a.ybar + cc);
            const double v = xb * rnx - yb * rny;
            sv += v * v;
            svx += v * xb;
        }
        nv = sqrt(block_sum(sv, red));
        vx = block_sum(svx, red);
        identity = nv < 1e-9;  // coincident mean directions (R3)
    }
    const double rnv = identity ? 0.0 : 1.0 / nv;
    const double ux = vx * rnv;  // u . xbar
    const double rN = 4096.0 / (double)(a.n_x + a.n_y);
    for (int64_t cc = threadIdx.x; cc < a.d_pad; cc += blockDim.x) {
        double u = 0.0, m = 0.0;
        if (cc < a.d) {
            const double xb = __ldcg(a.xbar + cc), yb = __ldcg(a.ybar + cc);
            u = (xb * rnx - yb * rny) * rnv;
            // centre m = t/N quantised to 2^-12 with t = n_x (xbar - 2u(u.xbar)) + n_y ybar
            const double t = (double)a.n_x * (xb - 2.0 * u * ux) + (double)a.n_y * yb;
            m = rint(t * rN) * (1.0 / 4096.0);
        }
        a.u[cc] = u;
        a.m[cc] = m;
    }
    if (threadIdx.x == 0) {
        double* sc = a.scal;
        sc[0] = nx;
        sc[1] = ny;
        sc[2] = identity ? 0.0 : nv;
        sc[3] = ux;
        sc[4] = identity ? 1.0 : 0.0;
        hap_align_info* f = a.info;
        const long long bad = *reinterpret_cast<volatile long long*>(a.scratch);
        f->n_x = a.n_x;
        f->n_y = a.n_y;
        f->d = a.d;
        f->n_pad = a.n_pad;
        f->d_pad = a.d_pad;
        f->is_identity = identity ? 1 : 0;
        f->status = bad < a.n_x + a.n_y ? HAP_E_ZERO_VECTOR
                                        : (degenerate ? HAP_E_DEGENERATE_MEAN : HAP_OK);
        f->bad_row = bad < a.n_x + a.n_y ? bad : -1;
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
        // reset the scratch words for the next call
        a.scratch[0] = LLONG_MAX;
        reinterpret_cast<unsigned*>(a.scratch + 1)[0] = 0u;
    }
}

// ---------------------------------------------------------------------------------
// K1c (S4 coefficient): warp per X row, coef_i = 2 u^T x_i = 2 (u^T h_i)/||h_i||.
__global__ void __launch_bounds__(256) k1c_rowdot(AlignArgs a) {
    const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int l = threadIdx.x & 31;
    if (i >= a.n_x) return;
    if (a.scal[4] != 0.0) {
        if (l == 0) a.coef[i] = 0.0;
        return;
    }
    const float* h = a.X + i * a.d;
    double s = 0.0;
    if ((a.d & 3) == 0) {
        const float4* h4 = reinterpret_cast<const float4*>(h);
        const double2* u2 = reinterpret_cast<const double2*>(a.u);
#pragma unroll 2
        for (int64_t c = l; c < a.d / 4; c += 32) {
            const float4 v = __ldg(h4 + c);
            const double2 u0 = __ldg(u2 + 2 * c), u1 = __ldg(u2 + 2 * c + 1);
            s += (double)v.x * u0.x + (double)v.y * u0.y + (double)v.z * u1.x + (double)v.w * u1.y;
        }
    } else {
        for (int64_t c = l; c < a.d; c += 32) s += (double)__ldg(h + c) * __ldg(a.u + c);
    }
    s = warp_sum(s);
    if (l == 0) a.coef[i] = 2.0 * s * a.inv[i];
}

// ---------------------------------------------------------------------------------
// K1d (S4 reflect + S5 centre/split/transpose + t partials): CTA per (64 rows, 64 cols).
// z = h/||h|| - coef * u  (fp64), centred z' = z - m with m = t/N quantised to 2^-12, where
// t = n_x (xbar - 2u(u^T xbar)) + n_y ybar follows from the means;
// hi = bf16(z'), lo = bf16(z' - hi)  (R9, "Numerics"); written transposed into
// Zt_hi/Zt_lo [d_pad][n_pad].  t partial of the tile: fixed-order fp64 sum of (hi + lo).
constexpr int kSP = 33;  // padded smem row pitch in 32-bit words (64 bf16 + pad)
__global__ void __launch_bounds__(256) k1d_reflect_split(AlignArgs a) {
    __shared__ uint32_t s_hi[64 * kSP];
    __shared__ uint32_t s_lo[64 * kSP];
    const int64_t N = a.n_x + a.n_y;
    const int64_t r0 = (int64_t)blockIdx.x * kRowTile;
    const int64_t c0 = (int64_t)blockIdx.y * 64;
    const int tc = threadIdx.x & 63, tr = threadIdx.x >> 6;  // 64 cols x 4 rows per pass
    uint16_t* sh16 = reinterpret_cast<uint16_t*>(s_hi);
    uint16_t* sl16 = reinterpret_cast<uint16_t*>(s_lo);
    const int64_t c = c0 + tc;
    // fp32 is ample here: the value is then represented with 16 mantissa bits (hi + lo)
    const float uc = c < a.d_pad ? (float)a.u[c] : 0.f;
    const float mc = c < a.d_pad ? (float)a.m[c] : 0.f;
#pragma unroll 4
    for (int j = 0; j < 16; ++j) {
        const int rl = tr + 4 * j;
        const int64_t i = r0 + rl;
        float z = 0.f;
        if (i < N && c < a.d) {
            const float h = __ldg(row_ptr(a, i) + c);
            const float cf = i < a.n_x ? (float)a.coef[i] : 0.f;
            z = fmaf(-cf, uc, h * (float)a.inv[i]) - mc;
        }
        const __nv_bfloat16 hi = __float2bfloat16_rn(z);
        const __nv_bfloat16 lo = __float2bfloat16_rn(z - __bfloat162float(hi));
        sh16[tc * (2 * kSP) + rl] = __bfloat16_as_ushort(hi);
        sl16[tc * (2 * kSP) + rl] = __bfloat16_as_ushort(lo);
    }
    __syncthreads();
    // write out: warp w handles column rows cc = w, w+8, ...; lane writes 2 bf16 (4 bytes)
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    for (int cc = w; cc < 64; cc += 8) {
        const int64_t col = c0 + cc;
        if (col >= a.d_pad) break;
        const uint32_t vh = s_hi[cc * kSP + l], vl = s_lo[cc * kSP + l];
        uint32_t* dh = reinterpret_cast<uint32_t*>(a.zt_hi + col * a.n_pad + r0);
        uint32_t* dl = reinterpret_cast<uint32_t*>(a.zt_lo + col * a.n_pad + r0);
        dh[l] = vh;
        dl[l] = vl;
        const double v = (double)__bfloat162float(__ushort_as_bfloat16((uint16_t)(vh & 0xFFFF))) +
                         (double)__bfloat162float(__ushort_as_bfloat16((uint16_t)(vl & 0xFFFF))) +
                         (double)__bfloat162float(__ushort_as_bfloat16((uint16_t)(vh >> 16))) +
                         (double)__bfloat162float(__ushort_as_bfloat16((uint16_t)(vl >> 16)));
        const double s = warp_sum(v);
        if (l == 0) a.tpart[(int64_t)blockIdx.x * a.d_pad + col] = s;
    }
}

// ---------------------------------------------------------------------------------
// K1e (S5 finish + epilogue constants): CTA per 256 columns.  t'[c] = sum of the row-tile
// partials (ascending); t = N m + t'.  With a = n_x m and b = t - a = n_y m + t' (fp32),
// the GEMM epilogue forms S1 = SA + sum acc (acc + 2a), S2 = SB + sum acc (acc - 2b) with
// SA = sum a^2, SB = sum b^2 (fp64; last CTA sums the per-CTA partials in fixed order).
__global__ void __launch_bounds__(kMeanCols * kMeanGroups) k1e_tfinal(AlignArgs a, int ntiles) {
    __shared__ double red[33];
    __shared__ double s_grp[kMeanGroups * kMeanCols];
    __shared__ int s_last;
    const int col = threadIdx.x % kMeanCols, g = threadIdx.x / kMeanCols;
    const int64_t c = (int64_t)blockIdx.x * kMeanCols + col;
    const double tp = grouped_colsum(a.tpart + (c < a.d_pad ? c : 0), a.d_pad, ntiles, g, s_grp, col);
    double sa = 0.0, sb = 0.0;
    if (c < a.d_pad && g == 0) {
        const double m = a.m[c];
        a.t64[c] = (double)(a.n_x + a.n_y) * m + tp;
        const float af = (float)((double)a.n_x * m);
        const float bf = (float)((double)a.n_y * m + tp);
        a.ab[c] = make_float2(2.0f * af, 2.0f * bf);
        sa = (double)af * (double)af;
        sb = (double)bf * (double)bf;
    }
    sa = block_sum(sa, red);
    sb = block_sum(sb, red);
    if (threadIdx.x == 0) {
        a.spart[2 * blockIdx.x + 0] = sa;
        a.spart[2 * blockIdx.x + 1] = sb;
        __threadfence();
        const unsigned t = atomicAdd(reinterpret_cast<unsigned*>(a.scratch + 1) + 1, 1u);
        s_last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    double SA = 0.0, SB = 0.0;
    if (threadIdx.x < gridDim.x) {
        SA = __ldcg(a.spart + 2 * threadIdx.x);
        SB = __ldcg(a.spart + 2 * threadIdx.x + 1);
    }
    SA = block_sum(SA, red);
    SB = block_sum(SB, red);
    if (threadIdx.x == 0) {
        a.sconst[0] = SA;
        a.sconst[1] = SB;
        reinterpret_cast<unsigned*>(a.scratch + 1)[1] = 0u;
    }
}

}  // namespace

cudaError_t launch_align(const AlignArgs& a, cudaStream_t st) {
    const int64_t N = a.n_x + a.n_y;
    const int nbx = (int)ceil_div(a.n_x, kRowBlock), nby = (int)ceil_div(a.n_y, kRowBlock);
    k1a_norm_colsum<<<nbx + nby, 256, 0, st>>>(a, nbx);
    k1b_means<<<(unsigned)ceil_div(a.d, kMeanCols), kMeanCols * kMeanGroups, 0, st>>>(a, nbx, nby);
    k1c_rowdot<<<(unsigned)ceil_div(a.n_x * 32, 256), 256, 0, st>>>(a);
    const int ntiles = (int)(a.n_pad / kRowTile);
    dim3 grid((unsigned)ntiles, (unsigned)ceil_div(a.d_pad, 64));
    k1d_reflect_split<<<grid, 256, 0, st>>>(a);
    k1e_tfinal<<<(unsigned)ceil_div(a.d_pad, kMeanCols), kMeanCols * kMeanGroups, 0, st>>>(a, ntiles);
    (void)N;
    return cudaGetLastError();
}

}  // namespace hap
