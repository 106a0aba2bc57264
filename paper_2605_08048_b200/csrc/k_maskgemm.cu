// k_maskgemm.cu — K3: tcgen05/TMEM mask-GEMM with the statistic epilogue
// (DESIGN.md "Kernels" K3; S8 + S9 of SURVEY.md §8a).
//
//   sigma1_b = sum_{i in G_b} z_i  as one row of  U' = M_blk Z  (0/1 mask instead of the
//   paper's +-1 signs, PAPER.md:205-220 Eq. gemm; R7), Z~ = hi + lo bf16 planes:
//       D[b, c] = sum_k M[b,k] Zhi[k,c] + sum_k M[b,k] Zlo[k,c]   (fp32 in TMEM)
//   sigma2 = t - sigma1            ("without a second GEMM")
//   r1 = ||sigma1||/n_x, r2 = ||sigma2||/n_y
//   T_b = L(r2) - L(r1)             (Alg. 2)
//   counts += [T_b >= T_obs], [|T_b| >= |T_obs|], [|T_b - T_obs| <= tau]
// No B x d intermediate reaches HBM: sigma1 lives only in TMEM.
//
// v1 structure: one CTA per 128-permutation tile (M = 128, cta_group::1), 6 warps:
//   warp 0  TMA producer   (A = mask tile 128x64, B = Zt_hi / Zt_lo tiles 256x64; SW128)
//   warp 1  MMA issuer + TMEM owner (512 columns = 2 accumulator buffers of 256)
//   warps 2-5 epilogue: thread = TMEM lane = one permutation; loops over d-chunks of 256
//            with the accumulator double-buffered so chunk c+1's MMAs overlap chunk c's
//            epilogue.
#include <cmath>

#include "hap_device.cuh"
#include "hap_internal.h"

namespace hap {
namespace {

constexpr int kStages = 2;
constexpr int kStageA = kTileM * 128;              // 16 KB: 128 rows x 64 bf16
constexpr int kStageB = kChunkN * 128;             // 32 KB: 256 rows x 64 bf16
constexpr int kStageBytes = kStageA + 2 * kStageB; // 80 KB
constexpr int kThreads = 192;
constexpr uint32_t kTmemCols = 512;

// L(r) = log kappa-hat(r), kappa-hat = r(d - r^2)/(1 - r^2), r clamped to [0, 1-1e-9]
// (Eq. 9 with DESIGN.md R1, R4).
__device__ __forceinline__ double logkappa(double r, double d) {
    if (r > 1.0 - 1e-9) r = 1.0 - 1e-9;
    if (r <= 0.0) return -INFINITY;
    const double r2 = r * r;
    return log(r) + log(d - r2) - log(1.0 - r2);
}

__global__ void __launch_bounds__(kThreads, 1)
    k3_maskgemm(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmBhi,
                const __grid_constant__ CUtensorMap tmBlo, GemmArgs g) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    if (g.info->status != HAP_OK) return;  // deferred data error: whole test is a no-op
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
    uint64_t* empty = full + kStages;
    uint64_t* tfull = empty + kStages;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nkb = g.n_pad / kKBlock;
    const int nchunks = (g.d_pad + kChunkN - 1) / kChunkN;
    const int row0 = blockIdx.x * kTileM;

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 4 * 32);
        }
        fence_barrier_init();
        tma_prefetch_desc(&tmA);
        tma_prefetch_desc(&tmBhi);
        tma_prefetch_desc(&tmBlo);
    }
    if (warp == 1) tmem_alloc<kTmemCols>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ---------------- TMA producer
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            const uint32_t bytes = (uint32_t)(kTileM + 2 * g.box_n) * 128u;
            for (int c = 0; c < nchunks; ++c) {
                for (int kb = 0; kb < nkb; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1u);
                    uint8_t* sA = smem + stage * kStageBytes;
                    mbar_arrive_expect_tx(&full[stage], bytes);
                    tma_load_2d(&tmA, &full[stage], sA, kb * kKBlock, row0);
                    tma_load_2d(&tmBhi, &full[stage], sA + kStageA, kb * kKBlock, c * kChunkN);
                    tma_load_2d(&tmBlo, &full[stage], sA + kStageA + kStageB, kb * kKBlock,
                                c * kChunkN);
                    if (++stage == kStages) { stage = 0; phase ^= 1u; }
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer (single thread)
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int c = 0; c < nchunks; ++c) {
                const int a = c & 1;
                const int width = min(kChunkN, g.d_pad - c * kChunkN);
                const uint32_t idesc = idesc_bf16_f32(kTileM, (uint32_t)width);
                mbar_wait(&tempty[a], (((uint32_t)c >> 1) & 1u) ^ 1u);
                tc_fence_after();
                const uint32_t dtm = tmem + (uint32_t)(a * kChunkN);
                for (int kb = 0; kb < nkb; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint32_t aBase = smem_u32(smem + stage * kStageBytes);
                    const uint32_t hBase = aBase + kStageA, lBase = hBase + kStageB;
#pragma unroll
                    for (int k = 0; k < kKBlock / 16; ++k) {
                        const uint64_t ad = smem_desc_k_sw128(aBase + 32u * k);
                        umma_bf16_ss(dtm, ad, smem_desc_k_sw128(hBase + 32u * k), idesc,
                                     (kb | k) != 0 ? 1u : 0u);
                        umma_bf16_ss(dtm, ad, smem_desc_k_sw128(lBase + 32u * k), idesc, 1u);
                    }
                    umma_commit(&empty[stage]);  // frees the smem slot when these MMAs retire
                    if (++stage == kStages) { stage = 0; phase ^= 1u; }
                }
                umma_commit(&tfull[a]);  // accumulator chunk ready for the epilogue
            }
        }
    } else {
        // ---------------- epilogue: one thread per TMEM lane (= permutation row)
        const int q = warp & 3;
        const int row = 32 * q + lane;
        const int perm = row0 + row;
        // sigma1 = a + acc, sigma2 = b - acc  (centred accumulator acc)
        double S1 = g.sconst[0], S2 = g.sconst[1];
        for (int c = 0; c < nchunks; ++c) {
            const int a = c & 1;
            const int width = min(kChunkN, g.d_pad - c * kChunkN);
            mbar_wait(&tfull[a], ((uint32_t)c >> 1) & 1u);
            tc_fence_after();
            float s1 = 0.f, s2 = 0.f;
            const float4* abp = reinterpret_cast<const float4*>(g.ab + c * kChunkN);
            for (int cb = 0; cb < width / 32; ++cb) {
                uint32_t r[32];
                tmem_ld_32x32b_x32(tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(a * kChunkN + 32 * cb),
                                   r);
                tmem_ld_wait();
#pragma unroll
                for (int j2 = 0; j2 < 16; ++j2) {
                    const float4 k4 = __ldg(abp + cb * 16 + j2);  // {2a, 2b} of two columns
                    const float x0 = __uint_as_float(r[2 * j2]), x1 = __uint_as_float(r[2 * j2 + 1]);
                    s1 = fmaf(x0, x0 + k4.x, s1);
                    s2 = fmaf(x0, x0 - k4.y, s2);
                    s1 = fmaf(x1, x1 + k4.z, s1);
                    s2 = fmaf(x1, x1 - k4.w, s2);
                }
            }
            tc_fence_before();
            mbar_arrive(&tempty[a]);
            S1 += (double)s1;
            S2 += (double)s2;
        }
        S1 = fmax(S1, 0.0);
        S2 = fmax(S2, 0.0);
        const double r1 = sqrt(S1) / (double)g.n_x;
        const double r2 = sqrt(S2) / (double)g.n_y;
        const double L1 = logkappa(r1, (double)g.d), L2 = logkappa(r2, (double)g.d);
        const double T = (isinf(L1) && isinf(L2)) ? 0.0 : L2 - L1;
        if (g.observed) {
            if (row == 0 && blockIdx.x == 0) {
                hap_align_info* f = g.info;
                f->r_x = r1;
                f->r_y = r2;
                f->logk_x = L1;
                f->logk_y = L2;
                f->t_obs = T;
            }
        } else {
            const double t_obs = g.info->t_obs;
            const double tau = g.tie_rel * (fabs(g.info->logk_x) + fabs(g.info->logk_y));
            const bool valid = perm < g.count;
            const bool ge = valid && (T >= t_obs);
            const bool ab = valid && (fabs(T) >= fabs(t_obs));
            // near-tie of either decision (R8)
            const bool fl = valid && (T == t_obs || fabs(T - t_obs) <= tau ||
                                      fabs(T) == fabs(t_obs) || fabs(fabs(T) - fabs(t_obs)) <= tau);
            const uint32_t bge = __ballot_sync(0xffffffffu, ge);
            const uint32_t bab = __ballot_sync(0xffffffffu, ab);
            const uint32_t bfl = __ballot_sync(0xffffffffu, fl);
            if (lane == 0) {
                unsigned long long* cnt = reinterpret_cast<unsigned long long*>(g.counts);
                if (bge) atomicAdd(cnt + 0, (unsigned long long)__popc(bge));
                if (bab) atomicAdd(cnt + 1, (unsigned long long)__popc(bab));
                if (bfl) atomicAdd(cnt + 2, (unsigned long long)__popc(bfl));
            }
            if (g.stats && valid) {
                double* o = g.stats + 3 * (int64_t)perm;
                o[0] = r1;
                o[1] = r2;
                o[2] = T;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<kTmemCols>(tmem);
    }
}

}  // namespace

size_t maskgemm_smem_bytes() { return (size_t)kStages * kStageBytes + 1024 + 128; }

cudaError_t launch_maskgemm(const CUtensorMap* tmA, const CUtensorMap* tmBhi,
                            const CUtensorMap* tmBlo, const GemmArgs& g, cudaStream_t st) {
    if (g.count <= 0) return cudaSuccess;
    static bool configured = false;
    const size_t smem = maskgemm_smem_bytes();
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(k3_maskgemm, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    const int grid = (int)ceil_div(g.count, kTileM);
    k3_maskgemm<<<grid, kThreads, smem, st>>>(*tmA, *tmBhi, *tmBlo, g);
    return cudaGetLastError();
}

}  // namespace hap
