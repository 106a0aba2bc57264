// k_align.cu — K1: S1-S5 of the hot path (DESIGN.md "Kernels" K1a-K1e).
//
//   S1 normalise   x = h/||h||               PAPER.md:115-118 (§3.1 Eq. 2)
//   S2 means       xbar, ybar, mu_x, mu_y    PAPER.md:143-148; Alg. 1
//   S3 axis        u = (mu_x-mu_y)/||.||     PAPER.md:149-156 (Eqs. 5-6); Alg. 1 :664
//   S4 reflect     x' = x - 2u(u^T x)        PAPER.md:157-161, 245-255 (Eq. householder_fast)
//   S5 pool+split  Z = [X';Y] -> bf16 hi/lo planes (transposed, K contiguous), t = 1^T Z
//                                             PAPER.md:183, 215-218 (Eq. gemm), 258
//
// All reductions are fixed-order (per-block fp64 partials summed in ascending block
// order), so Z~ and t are bit-identical across runs and ranks.
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
    double s = 0.0;
    if (threadIdx.x == 0) {
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += red[i];
        red[32] = s;
    }
    __syncthreads();
    return red[32];
}

__device__ __forceinline__ double logkappa64(double r, double d) {
    if (r > 1.0 - 1e-9) r = 1.0 - 1e-9;
    if (r <= 0.0) return -INFINITY;
    const double r2 = r * r;
    return log(r) + log(d - r2) - log(1.0 - r2);
}

__device__ __forceinline__ const float* row_ptr(const AlignArgs& a, int64_t i) {
    return i < a.n_x ? a.X + i * a.d : a.Y + (i - a.n_x) * a.d;
}

// K1 init: shape fields and a clean status
__global__ void k1_init(AlignArgs a) {
    hap_align_info* f = a.info;
    f->n_x = a.n_x;
    f->n_y = a.n_y;
    f->d = a.d;
    f->n_pad = a.n_pad;
    f->d_pad = a.d_pad;
    f->is_identity = 0;
    f->status = HAP_OK;
    f->bad_row = LLONG_MAX;
    f->r_x = f->r_y = f->logk_x = f->logk_y = f->t_obs = 0.0;
    f->gemm_r_x = f->gemm_r_y = f->gemm_t_obs = __longlong_as_double(0x7ff8000000000000ll);  // NaN
}

// K1a (S1+S2 partials): one CTA per block of kRowBlock rows of X or of Y.
// Phase 1: warp-per-row fp64 norms ||h_i|| (ZeroVector check).
// Phase 2: fp64 column partial sums of the normalised rows h_i/||h_i||.
__global__ void __launch_bounds__(256) k1_norm_colsum(AlignArgs a, int nblk_x) {
    __shared__ double s_inv[kRowBlock];
    const bool isx = (int)blockIdx.x < nblk_x;
    const int64_t blk = isx ? blockIdx.x : blockIdx.x - nblk_x;
    const int64_t nrows = isx ? a.n_x : a.n_y;
    const int64_t r0 = blk * kRowBlock;
    const int64_t rn = (nrows - r0 < kRowBlock) ? (nrows - r0) : (int64_t)kRowBlock;
    const int64_t base = isx ? r0 : a.n_x + r0;  // pooled row index of local row 0
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    for (int r = w; r < rn; r += 8) {
        const float* h = row_ptr(a, base + r);
        double s = 0.0;
        for (int64_t c = l; c < a.d; c += 32) {
            const double v = (double)h[c];
            s += v * v;
        }
        s = warp_sum(s);
        if (l == 0) {
            const double nrm = sqrt(s);
            a.nrm[base + r] = nrm;
            if (nrm < 1e-12) {
                a.info->status = HAP_E_ZERO_VECTOR;
                atomicMin(reinterpret_cast<long long*>(&a.info->bad_row), (long long)(base + r));
                s_inv[r] = 0.0;
            } else {
                s_inv[r] = 1.0 / nrm;
            }
        }
    }
    __syncthreads();
    double* part = a.part + (int64_t)blockIdx.x * a.d;
    for (int64_t c = threadIdx.x; c < a.d; c += blockDim.x) {
        double acc = 0.0;
        for (int r = 0; r < rn; ++r) acc += (double)row_ptr(a, base + r)[c] * s_inv[r];
        part[c] = acc;
    }
}

// K1b (S2 finish + S3): one CTA.  xbar, ybar from the partials in ascending block order,
// norms, DegenerateMean check, mean directions, Householder axis u (fp64).
__global__ void __launch_bounds__(1024) k1_finalize(AlignArgs a, int nblk_x, int nblk_y) {
    __shared__ double red[33];
    double sx = 0.0, sy = 0.0;
    for (int64_t c = threadIdx.x; c < a.d; c += blockDim.x) {
        double xs = 0.0, ys = 0.0;
        for (int b = 0; b < nblk_x; ++b) xs += a.part[(int64_t)b * a.d + c];
        for (int b = 0; b < nblk_y; ++b) ys += a.part[(int64_t)(nblk_x + b) * a.d + c];
        const double xb = xs / (double)a.n_x, yb = ys / (double)a.n_y;
        a.xbar[c] = xb;
        a.ybar[c] = yb;
        sx += xb * xb;
        sy += yb * yb;
    }
    const double nx = sqrt(block_sum(sx, red));
    const double ny = sqrt(block_sum(sy, red));
    const bool degenerate = nx < 1e-12 || ny < 1e-12;
    bool identity = (a.mode == HAP_ALIGN_NONE) || degenerate;
    double nv = 0.0;
    if (!identity) {
        double sv = 0.0;
        for (int64_t c = threadIdx.x; c < a.d; c += blockDim.x) {
            const double v = a.xbar[c] / nx - a.ybar[c] / ny;
            sv += v * v;
        }
        nv = sqrt(block_sum(sv, red));
        identity = nv < 1e-9;  // coincident mean directions (R3)
    }
    double sux = 0.0;
    for (int64_t c = threadIdx.x; c < a.d; c += blockDim.x) {
        const double uc = identity ? 0.0 : (a.xbar[c] / nx - a.ybar[c] / ny) / nv;
        a.u[c] = uc;
        sux += uc * a.xbar[c];
    }
    // Centre m = t/N, quantised to a multiple of 2^-12 (exact shift,
    // since every mask row has exactly n_x ones).  t follows from the means without the
    // reflected rows: t = n_x (xbar - 2u(u^T xbar)) + n_y ybar.
    const double ux = block_sum(sux, red);
    const double Nd = (double)(a.n_x + a.n_y);
    for (int64_t c = threadIdx.x; c < a.d_pad; c += blockDim.x) {
        double m = 0.0;
        if (c < a.d) {
            const double t = (double)a.n_x * (a.xbar[c] - 2.0 * a.u[c] * ux) + (double)a.n_y * a.ybar[c];
            m = rint(t / Nd * 4096.0) / 4096.0;
        }
        a.m[c] = m;
    }
    if (threadIdx.x == 0) {
        hap_align_info* f = a.info;
        // observed statistic in fp64 (Alg. 1 step 4): r(X') = ||xbar|| since
        // H is orthogonal; T_obs = L(r_Y) - L(r_X) (Eq. 10; R1, R4)
        f->r_x = nx;
        f->r_y = ny;
        const double lx = logkappa64(nx, (double)a.d), ly = logkappa64(ny, (double)a.d);
        f->logk_x = lx;
        f->logk_y = ly;
        f->t_obs = (isinf(lx) && isinf(ly)) ? 0.0 : ly - lx;
        f->is_identity = identity ? 1 : 0;
        if (f->status == HAP_OK && degenerate) f->status = HAP_E_DEGENERATE_MEAN;
        if (f->bad_row == LLONG_MAX) f->bad_row = -1;
    }
}

// K1c (S4 coefficient): warp per pooled row, coef_i = 2 u^T x_i = 2 (u^T h_i)/||h_i||
// for X rows (0 for Y rows and the identity).
__global__ void __launch_bounds__(256) k1_rowdot(AlignArgs a) {
    const int64_t N = a.n_x + a.n_y;
    const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int l = threadIdx.x & 31;
    if (i >= N) return;
    if (i >= a.n_x || a.info->is_identity) {
        if (l == 0) a.coef[i] = 0.0;
        return;
    }
    const float* h = a.X + i * a.d;
    double s = 0.0;
    for (int64_t c = l; c < a.d; c += 32) s += (double)h[c] * a.u[c];
    s = warp_sum(s);
    if (l == 0) a.coef[i] = a.nrm[i] > 0.0 ? 2.0 * s / a.nrm[i] : 0.0;
}

// K1d (S4 reflect + S5 split/transpose + t partials): CTA per (64-row tile, 64-col tile).
// z = h/||h|| - coef * u  (fp64), centred z' = z - m;  hi = bf16(z'), lo = bf16(z' - hi)
// (R9 and "Numerics");
// written transposed into Zt_hi/Zt_lo [d_pad][n_pad] (GEMM K contiguous).
// t partial of the tile: sum over its 64 rows of (hi + lo) in fp64, fixed order.
constexpr int kSP = 33;  // padded smem row pitch in 32-bit words (64 bf16 + pad)
__global__ void __launch_bounds__(256) k1_reflect_split(AlignArgs a) {
    __shared__ uint32_t s_hi[64 * kSP];
    __shared__ uint32_t s_lo[64 * kSP];
    const int64_t N = a.n_x + a.n_y;
    const int64_t r0 = (int64_t)blockIdx.x * kRowTile;
    const int64_t c0 = (int64_t)blockIdx.y * 64;
    const int tc = threadIdx.x & 63, tr = threadIdx.x >> 6;  // 64 cols x 4 rows per pass
    uint16_t* sh16 = reinterpret_cast<uint16_t*>(s_hi);
    uint16_t* sl16 = reinterpret_cast<uint16_t*>(s_lo);
    const int64_t c = c0 + tc;
    const double uc = (c < a.d) ? a.u[c] : 0.0;
    const double mc = (c < a.d) ? a.m[c] : 0.0;
#pragma unroll 4
    for (int j = 0; j < 16; ++j) {
        const int rl = tr + 4 * j;
        const int64_t i = r0 + rl;
        double z = 0.0;
        if (i < N && c < a.d) {
            const double nrm = a.nrm[i];
            const double h = (double)row_ptr(a, i)[c];
            z = (nrm > 0.0 ? h / nrm : 0.0) - a.coef[i] * uc - mc;
        }
        const __nv_bfloat16 hi = __double2bfloat16(z);
        const __nv_bfloat16 lo = __double2bfloat16(z - (double)__bfloat162float(hi));
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
        // t partial for column `col` over these 64 rows (fixed order: pairs, then xor tree)
        const double v = (double)__bfloat162float(__ushort_as_bfloat16((uint16_t)(vh & 0xFFFF))) +
                         (double)__bfloat162float(__ushort_as_bfloat16((uint16_t)(vl & 0xFFFF))) +
                         (double)__bfloat162float(__ushort_as_bfloat16((uint16_t)(vh >> 16))) +
                         (double)__bfloat162float(__ushort_as_bfloat16((uint16_t)(vl >> 16)));
        const double s = warp_sum(v);
        if (l == 0) a.tpart[(int64_t)blockIdx.x * a.d_pad + col] = s;
    }
}

// K1e (S5 finish + epilogue constants), one CTA.  t'[c] = sum of the row-tile partials
// (ascending tile order) of the centred planes; t = N m + t'.  With a = n_x m and
// b = t - a = n_y m + t' (both rounded to fp32), the epilogue forms
//   S1 = ||a + acc||^2 = SA + sum acc (acc + 2a),   S2 = ||b - acc||^2 = SB + sum acc (acc - 2b)
// with SA = sum a^2, SB = sum b^2 in fp64.
__global__ void __launch_bounds__(1024) k1_tfinal(AlignArgs a, int ntiles) {
    __shared__ double red[33];
    double sa = 0.0, sb = 0.0;
    for (int64_t c = threadIdx.x; c < a.d_pad; c += blockDim.x) {
        double tp = 0.0;
        for (int t = 0; t < ntiles; ++t) tp += a.tpart[(int64_t)t * a.d_pad + c];
        const double m = a.m[c];
        a.t64[c] = (double)(a.n_x + a.n_y) * m + tp;
        const float af = (float)((double)a.n_x * m);
        const float bf = (float)((double)a.n_y * m + tp);
        a.ab[c] = make_float2(2.0f * af, 2.0f * bf);
        sa += (double)af * (double)af;
        sb += (double)bf * (double)bf;
    }
    sa = block_sum(sa, red);
    sb = block_sum(sb, red);
    if (threadIdx.x == 0) {
        a.sconst[0] = sa;
        a.sconst[1] = sb;
    }
}

}  // namespace

cudaError_t launch_align(const AlignArgs& a, cudaStream_t st) {
    const int64_t N = a.n_x + a.n_y;
    const int nbx = (int)ceil_div(a.n_x, kRowBlock), nby = (int)ceil_div(a.n_y, kRowBlock);
    k1_init<<<1, 1, 0, st>>>(a);
    k1_norm_colsum<<<nbx + nby, 256, 0, st>>>(a, nbx);
    k1_finalize<<<1, 1024, 0, st>>>(a, nbx, nby);
    k1_rowdot<<<(unsigned)ceil_div(N * 32, 256), 256, 0, st>>>(a);
    const int ntiles = (int)(a.n_pad / kRowTile);
    dim3 grid((unsigned)ntiles, (unsigned)ceil_div(a.d_pad, 64));
    k1_reflect_split<<<grid, 256, 0, st>>>(a);
    k1_tfinal<<<1, 1024, 0, st>>>(a, ntiles);
    return cudaGetLastError();
}

}  // namespace hap
