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
//   k1g_gram     : G' from the planes the alignment wrote (z' = hi + lo, exact in fp32),
//                  fp32 products summed per 64-column chunk, chunks in fp64; G' -> bf16
//                  hi/lo planes [j][k] (symmetric, so the K-major B operand is G' itself);
//                  diagonal tiles also form {2 alpha_j, 2 beta_j} in fp64 with the fp32 a, b
//                  the plane epilogue uses ({2a, 2b} = ab).
//   k2_pack_bits : the generator's bf16 mask rows -> one bit per pooled row (the Gram
//                  epilogue reads m_bj for the columns of its piece: 32 bytes per row and
//                  256 columns instead of 512).
#include <cuda_bf16.h>

#include <algorithm>

#include "hap_device.cuh"
#include "hap_internal.h"

namespace hap {
namespace {

constexpr int kGT = 32;       // output tile kGT x kGT
constexpr int kGC = 64;       // columns c per smem chunk
constexpr int kGThreads = 256;  // thread = 2 x 2 outputs

__device__ __forceinline__ float bf16_bits(uint16_t b) { return __uint_as_float((uint32_t)b << 16); }

// CTA = one upper-triangle tile (jb <= kb) of G'; writes the tile and its transpose
__global__ void __launch_bounds__(kGThreads) k1g_gram(GramArgs g) {
    __shared__ float sJ[kGC][kGT + 1];
    __shared__ float sK[kGC][kGT + 1];
    const int tid = threadIdx.x;
    const int T = g.n_pad / kGT;
    // blockIdx -> (jb, kb) with jb <= kb, row-major over the upper triangle
    int jb = 0, rem = blockIdx.x;
    while (rem >= T - jb) {
        rem -= T - jb;
        ++jb;
    }
    const int kb = jb + rem;
    const int j0 = jb * kGT, k0 = kb * kGT;
    const bool diag = jb == kb;
    if (tid == 0) span_enter(g.span);
    const int ty = tid >> 4, tx = tid & 15;  // outputs (j0 + 2 ty + {0,1}, k0 + 2 tx + {0,1})
    double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
    double al = 0.0, be = 0.0;  // diagonal tiles: 2 alpha, 2 beta of row j0 + tid (tid < 32)
    for (int c0 = 0; c0 < g.d_pad; c0 += kGC) {
        // stage z' = hi + lo of columns c0 .. c0 + 63 for rows j0.. and k0.. (fp32, exact)
        for (int e = tid; e < kGC * kGT; e += kGThreads) {
            const int cc = e / kGT, r = e % kGT;
            const int c = c0 + cc;
            float zj = 0.f, zk = 0.f;
            if (c < g.d_pad) {
                const size_t oj = (size_t)c * g.n_pad + j0 + r, ok = (size_t)c * g.n_pad + k0 + r;
                zj = bf16_bits(g.zt_hi[oj]) + bf16_bits(g.zt_lo[oj]);
                zk = bf16_bits(g.zt_hi[ok]) + bf16_bits(g.zt_lo[ok]);
            }
            sJ[cc][r] = zj;
            sK[cc][r] = zk;
        }
        __syncthreads();
        float p[2][2] = {{0.f, 0.f}, {0.f, 0.f}};
#pragma unroll 8
        for (int cc = 0; cc < kGC; ++cc) {
            const float a0 = sJ[cc][2 * ty], a1 = sJ[cc][2 * ty + 1];
            const float b0 = sK[cc][2 * tx], b1 = sK[cc][2 * tx + 1];
            p[0][0] = fmaf(a0, b0, p[0][0]);
            p[0][1] = fmaf(a0, b1, p[0][1]);
            p[1][0] = fmaf(a1, b0, p[1][0]);
            p[1][1] = fmaf(a1, b1, p[1][1]);
        }
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
            for (int v = 0; v < 2; ++v) acc[u][v] += (double)p[u][v];
        if (diag && tid < kGT) {
            for (int cc = 0; cc < kGC && c0 + cc < g.d_pad; ++cc) {
                const float2 ab = g.ab[c0 + cc];
                const double z = (double)sJ[cc][tid];
                al += (double)ab.x * z;
                be += (double)ab.y * z;
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int v = 0; v < 2; ++v) {
            const int j = j0 + 2 * ty + u, k = k0 + 2 * tx + v;
            const float gv = (float)acc[u][v];
            const __nv_bfloat16 h = __float2bfloat16_rn(gv);
            const __nv_bfloat16 l = __float2bfloat16_rn(gv - __bfloat162float(h));
            const uint16_t hb = *reinterpret_cast<const uint16_t*>(&h), lb = *reinterpret_cast<const uint16_t*>(&l);
            g.g_hi[(size_t)j * g.n_pad + k] = hb;
            g.g_lo[(size_t)j * g.n_pad + k] = lb;
            if (!diag) {
                g.g_hi[(size_t)k * g.n_pad + j] = hb;
                g.g_lo[(size_t)k * g.n_pad + j] = lb;
            }
        }
    if (diag && tid < kGT) g.gab[j0 + tid] = make_float2((float)al, (float)be);
    if (tid == 0) span_exit(g.span);
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

cudaError_t launch_gram(const GramArgs& g, cudaStream_t st) {
    if (g.n_pad % kGT) return cudaErrorInvalidValue;
    const int T = g.n_pad / kGT;
    k1g_gram<<<T * (T + 1) / 2, kGThreads, 0, st>>>(g);
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

}  // namespace hap
