// k_gram.cu — the Gram form of the mask-GEMM operand (
// DESIGN.md "Gram form").
//
// The statistic needs only S1 = ||sigma1||^2 and S2 = ||sigma2||^2 of the group sums
// (PAPER.md:221-237).  With the centred planes z'_i = z_i - m,
// acc_b = sum_{i in G_b} z'_i, a = n_x m, b = t - a:
//     S1 = |a|^2 + 2 a.acc + |acc|^2,   S2 = |b|^2 - 2 b.acc + |acc|^2,
//     |acc|^2 = sum_{j,k in G_b} G'_jk  (the quadratic form m_b^T G' m_b),  G' = Z' Z'^T,
//     a.acc   = sum_{j in G_b} alpha_j,  alpha_j = a.z'_j,   b.acc = sum_{j in G_b} beta_j.
// So for N << d the mask-GEMM can multiply the mask block by the N_pad x N_pad matrix G'
// instead of the N_pad x d_pad planes: U = M G' (K = N_pad, N = N_pad columns), and the
// epilogue forms sum_j m_bj (U_bj + 2 alpha_j) and sum_j m_bj (U_bj - 2 beta_j), which are
// exactly the two per-row partials of the plane form (sum_c acc_c (acc_c + 2 a_c) and
// sum_c acc_c (acc_c - 2 b_c)); the finalize is shared.  Issued tensor work per
// permutation 4 N_pad^2 instead of 4 N_pad d_pad.
//
//   k1g_gram     : G' from the planes the alignment wrote (z' = hi + lo, exact in fp32):
//                  CTA = (64 x 64 upper-triangle tile, 256 columns of d); fp32 products
//                  per 32-column chunk, chunks in fp64, the CTA's partial as fixed point
//                  into int64 accumulators (exact, order-free); diagonal tiles also form
//                  {2 alpha_j, 2 beta_j} in fp64 with the fp32 a, b the plane epilogue uses
//                  ({2a, 2b} = ab).
//   k1g_finish   : accumulators -> G' as bf16 hi/lo planes [j][k] (symmetric, so the
//                  K-major B operand is G' itself) and {2 alpha, 2 beta}; zeroes them.
//   k2_pack_bits : the generator's bf16 mask rows -> one bit per pooled row (the Gram
//                  epilogue reads m_bj for the columns of its piece: 32 bytes per row and
//                  256 columns instead of 512).
#include <cuda_bf16.h>

#include <algorithm>

#define HAP_CHECK_TU 4
#include "hap_device.cuh"
#include "hap_internal.h"

namespace hap {
namespace {

constexpr int kGT = 64;          // output tile kGT x kGT (thread = 4 x 4 outputs)
constexpr int kGC = 32;          // columns c per shared-memory chunk
constexpr int kGSplit = 256;     // columns c per CTA (split-K; partials summed exactly)
constexpr int kGThreads = 256;
constexpr double kGFix = 1099511627776.0;  // 2^40: |G'| <= 4, sums of <= 64 splits < 2^48

__device__ __forceinline__ float bf16_bits(uint32_t b) { return __uint_as_float(b << 16); }

// CTA = (upper-triangle tile jb <= kb, split of 256 columns c).  z' = hi + lo is exact in
// fp32; the products are summed in fp32 per 32-column chunk (unbiased round-to-nearest),
// the chunks in fp64, and the CTA's partial is rounded to a multiple of 2^-40 and added
// into int64 accumulators: exact integer sums in any order, so G' has the same bits in
// every run.  Diagonal tiles also accumulate {2 a.z'_j, 2 b.z'_j} (fp64 -> fixed point).
__global__ void __launch_bounds__(kGThreads) k1g_gram(GramArgs g) {
    __shared__ __align__(16) float sJ[kGC][kGT];
    __shared__ __align__(16) float sK[kGC][kGT];
    const int tid = threadIdx.x;
    const int T = g.n_pad / kGT;
    const int split = blockIdx.y;
    int jb = 0, rem = blockIdx.x;  // blockIdx.x -> (jb, kb), jb <= kb, row-major
    while (rem >= T - jb) {
        rem -= T - jb;
        ++jb;
    }
    const int kb = jb + rem;
    const int j0 = jb * kGT, k0 = kb * kGT;
    const bool diag = jb == kb;
    HAP_CHECK(kb < T && k0 + kGT <= g.n_pad && split * kGSplit < g.d_pad);
    if (tid == 0 && blockIdx.x == 0 && split == 0) span_enter(g.span);
    const int ty = tid >> 4, tx = tid & 15;  // outputs (j0 + 4 ty + u, k0 + 4 tx + v)
    // staging role: column cc = tid / 8, rows 8 (tid % 8) .. + 7 (one 16-byte load per plane)
    const int sc = tid >> 3, sr = 8 * (tid & 7);
    double acc[4][4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = 0.0;
    double al = 0.0, be = 0.0;  // diagonal tiles: row j0 + tid (tid < 64)
    const int c_end = min(g.d_pad, (split + 1) * kGSplit);
    for (int c0 = split * kGSplit; c0 < c_end; c0 += kGC) {
        {
            const int c = c0 + sc;
            float zj[8], zk[8];
            if (c < g.d_pad) {
                const size_t oj = (size_t)c * g.n_pad + j0 + sr, ok = (size_t)c * g.n_pad + k0 + sr;
                const uint4 hj = __ldg(reinterpret_cast<const uint4*>(g.zt_hi + oj));
                const uint4 lj = __ldg(reinterpret_cast<const uint4*>(g.zt_lo + oj));
                const uint4 hk = __ldg(reinterpret_cast<const uint4*>(g.zt_hi + ok));
                const uint4 lk = __ldg(reinterpret_cast<const uint4*>(g.zt_lo + ok));
                const uint32_t hjw[4] = {hj.x, hj.y, hj.z, hj.w}, ljw[4] = {lj.x, lj.y, lj.z, lj.w};
                const uint32_t hkw[4] = {hk.x, hk.y, hk.z, hk.w}, lkw[4] = {lk.x, lk.y, lk.z, lk.w};
#pragma unroll
                for (int w = 0; w < 4; ++w) {
                    zj[2 * w] = bf16_bits(hjw[w] & 0xFFFFu) + bf16_bits(ljw[w] & 0xFFFFu);
                    zj[2 * w + 1] = bf16_bits(hjw[w] >> 16) + bf16_bits(ljw[w] >> 16);
                    zk[2 * w] = bf16_bits(hkw[w] & 0xFFFFu) + bf16_bits(lkw[w] & 0xFFFFu);
                    zk[2 * w + 1] = bf16_bits(hkw[w] >> 16) + bf16_bits(lkw[w] >> 16);
                }
            } else {
#pragma unroll
                for (int e = 0; e < 8; ++e) zj[e] = zk[e] = 0.f;
            }
            float4* dj = reinterpret_cast<float4*>(&sJ[sc][sr]);
            float4* dk = reinterpret_cast<float4*>(&sK[sc][sr]);
            dj[0] = make_float4(zj[0], zj[1], zj[2], zj[3]);
            dj[1] = make_float4(zj[4], zj[5], zj[6], zj[7]);
            dk[0] = make_float4(zk[0], zk[1], zk[2], zk[3]);
            dk[1] = make_float4(zk[4], zk[5], zk[6], zk[7]);
        }
        __syncthreads();
        float p[4][4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v) p[u][v] = 0.f;
#pragma unroll 8
        for (int cc = 0; cc < kGC; ++cc) {
            const float4 a = *reinterpret_cast<const float4*>(&sJ[cc][4 * ty]);
            const float4 b = *reinterpret_cast<const float4*>(&sK[cc][4 * tx]);
            const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int v = 0; v < 4; ++v) p[u][v] = fmaf(av[u], bv[v], p[u][v]);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v) acc[u][v] += (double)p[u][v];
        if (diag && tid < kGT) {
            for (int cc = 0; cc < kGC && c0 + cc < g.d_pad; ++cc) {
                const float2 ab = __ldg(g.ab + c0 + cc);
                const double z = (double)sJ[cc][tid];
                al += (double)ab.x * z;
                be += (double)ab.y * z;
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            const long long q = __double2ll_rn(acc[u][v] * kGFix);
            if (q) atomicAdd(reinterpret_cast<unsigned long long*>(g.gacc + (size_t)(j0 + 4 * ty + u) * g.n_pad + k0 + 4 * tx + v),
                             (unsigned long long)q);
        }
    if (diag && tid < kGT) {
        atomicAdd(reinterpret_cast<unsigned long long*>(g.gabacc + 2 * (j0 + tid)), (unsigned long long)__double2ll_rn(al * kGFix));
        atomicAdd(reinterpret_cast<unsigned long long*>(g.gabacc + 2 * (j0 + tid) + 1),
                  (unsigned long long)__double2ll_rn(be * kGFix));
    }
}

// G' (upper triangle of the accumulators) -> bf16 hi/lo planes [j][k] and [k][j];
// {2 alpha, 2 beta}; the accumulators are zeroed for the next alignment.
__global__ void __launch_bounds__(256) k1g_finish(GramArgs g) {
    const int64_t n = g.n_pad;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n * n; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = e / n, k = e % n;
        if ((j / kGT) > (k / kGT)) continue;  // lower-triangle tiles: written from their mirror
        long long* a = g.gacc + e;
        const float gv = (float)((double)*a * (1.0 / kGFix));
        *a = 0;
        const __nv_bfloat16 h = __float2bfloat16_rn(gv);
        const __nv_bfloat16 l = __float2bfloat16_rn(gv - __bfloat162float(h));
        const uint16_t hb = *reinterpret_cast<const uint16_t*>(&h), lb = *reinterpret_cast<const uint16_t*>(&l);
        g.g_hi[j * n + k] = hb;
        g.g_lo[j * n + k] = lb;
        if ((j / kGT) != (k / kGT)) {
            g.g_hi[k * n + j] = hb;
            g.g_lo[k * n + j] = lb;
        }
    }
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        long long* a = g.gabacc + 2 * j;
        g.gab[j] = make_float2((float)((double)a[0] * (1.0 / kGFix)), (float)((double)a[1] * (1.0 / kGFix)));
        a[0] = a[1] = 0;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) span_exit(g.span);
}

// bit (j % 32) of word j / 32 of row r = mask[r][j] (bf16 1.0 or 0): thread = one word
__global__ void __launch_bounds__(256) k2_pack_bits(const uint16_t* __restrict__ mask, uint32_t* __restrict__ bits,
                                                   int64_t rows, int n_pad) {
    const int wpr = n_pad / 32;
    const int64_t total = rows * wpr;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / wpr;
        const int w = (int)(i % wpr);
        const uint4* src = reinterpret_cast<const uint4*>(mask + r * n_pad + 32 * w);
        uint32_t out = 0;
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            const uint4 q = __ldcg(src + v);
            const uint32_t x[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                out |= ((x[e] & 0xFFFFu) ? 1u : 0u) << (8 * v + 2 * e);
                out |= ((x[e] >> 16) ? 1u : 0u) << (8 * v + 2 * e + 1);
            }
        }
        bits[i] = out;
    }
}

}  // namespace

cudaError_t launch_gram(const GramArgs& g, int sm_count, cudaStream_t st) {
    if (g.n_pad % kGT) return cudaErrorInvalidValue;
    const int T = g.n_pad / kGT;
    const dim3 grid(T * (T + 1) / 2, (g.d_pad + kGSplit - 1) / kGSplit);
    k1g_gram<<<grid, kGThreads, 0, st>>>(g);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const int64_t n2 = (int64_t)g.n_pad * g.n_pad;
    k1g_finish<<<(int)std::min<int64_t>((n2 + 255) / 256, 4ll * sm_count), 256, 0, st>>>(g);
    return cudaGetLastError();
}

cudaError_t launch_pack_bits(const uint16_t* mask, uint32_t* bits, int64_t rows, int n_pad, int sm_count,
                             cudaStream_t st) {
    if (rows <= 0) return cudaSuccess;
    const int64_t total = rows * (n_pad / 32);
    const int grid = (int)std::min<int64_t>((total + 255) / 256, 8ll * sm_count);
    k2_pack_bits<<<grid, 256, 0, st>>>(mask, bits, rows, n_pad);
    return cudaGetLastError();
}

HAP_CHECK_ACCESSOR(check_word_gram)

}  // namespace hap
