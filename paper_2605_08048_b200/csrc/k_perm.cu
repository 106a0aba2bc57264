// k_perm.cu — K2: PERM-SPEC v1 permutation generator (DESIGN.md "Kernels" K2, R6).
//
// "Randomly partition Z into (X^(b), Y^(b)) with sizes (n, m)" (Alg. 1);
// "S_blk <- random {+1,-1}^{B0 x N} with exactly n entries +1 per row" (Alg. 2,
// PAPER.md:710).  PERM-SPEC v1 fixes the law as the partial forward Fisher-Yates
// shuffle over n_x steps with Philox4x32-10 words and Lemire bounded draws:
//     a = [0..N-1]; for k < n_x: j_k = k + U(N-k); swap(a[k], a[j_k]);  G_b = a[0..n_x).
//
// GPU formulation (one warp per permutation, no serial swap chain).  With
//   LT[q] = 1 + max{k : j_k = q, k != q}  (0 if no such step)       "last writer of q",
// the final contents satisfy (K2 derivation):
//   * a high position p >= n_x keeps value p unless written; if written, its final value
//     is the value position k* = LT[p]-1 held just before step k*, i.e. chain(k*) with
//     chain(k) = LT[k] ? chain(LT[k]-1) : k;
//   * hence G_b = ([0, n_x) \ E) U {p >= n_x : LT[p] != 0},  E = {chain(LT[p]-1)}.
// Phase A draws all j_k in parallel (lanes own Philox blocks) and scatters LT with
// last-writer-wins in step order; phase B follows the (short, disjoint) chains; phase C
// emits the exact 0/1 mask row.  Bit-exact against oracle/orc_perm_set (tests).
#include <cuda_bf16.h>

#include "hap_device.cuh"
#include "hap_internal.h"

namespace hap {
namespace {

constexpr int kPermWarps = 4;
constexpr uint16_t kExiled = 0xFFFF;

// U(N-k) for step k: Lemire on the main-stream word x; rejected words are replaced by
// the side stream (counter (q', b, s, 1+k)) in order.
__device__ __forceinline__ uint32_t fy_target(uint32_t x, uint32_t k, uint32_t N, uint32_t b,
                                              uint32_t s, uint32_t k0, uint32_t k1) {
    const uint32_t bound = N - k;
    uint64_t m = (uint64_t)x * bound;
    uint32_t lo = (uint32_t)m;
    if (lo < bound) {
        const uint32_t t = (0u - bound) % bound;
        uint32_t side = 0;
        while (lo < t) {
            const u32x4 w = philox4x32_10(u32x4{side >> 2, b, s, 1u + k}, k0, k1);
            x = u32x4_get(w, side & 3u);
            ++side;
            m = (uint64_t)x * bound;
            lo = (uint32_t)m;
        }
    }
    return k + (uint32_t)(m >> 32);
}

__global__ void __launch_bounds__(kPermWarps * 32) k2_perm_fy(PermArgs a, int lt_pitch) {
    extern __shared__ __align__(16) uint8_t smem[];
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    uint16_t* LT = reinterpret_cast<uint16_t*>(smem) + (size_t)w * (lt_pitch + 128);
    uint16_t* stage = LT + lt_pitch;
    const uint32_t N = (uint32_t)a.N, nx = (uint32_t)a.n_x, s = a.s;
    const uint32_t key0 = (uint32_t)(a.seed & 0xFFFFFFFFu), key1 = (uint32_t)(a.seed >> 32);
    const int nw = (int)(blockDim.x >> 5);
    const int64_t wstride = (int64_t)gridDim.x * nw;
    const int64_t items = a.count + (a.out_kind == kMaskBf16Row ? a.ntiles : 0);
    for (int64_t pi = (int64_t)blockIdx.x * nw + w; pi < items; pi += wstride) {
        if (pi >= a.count) {  // observed split: row 0 of tile (pi - count)
            const int64_t t = pi - a.count;
            uint4* row = reinterpret_cast<uint4*>(static_cast<uint16_t*>(a.out) +
                                                  t * a.rows_per_tile * a.n_pad);
            for (int64_t v8 = l; v8 < a.n_pad / 8; v8 += 32) {
                uint32_t wds[4];
#pragma unroll
                for (int e2 = 0; e2 < 4; ++e2) {
                    const int64_t v = 8 * v8 + 2 * e2;
                    wds[e2] = (v < a.n_x ? 0x3F80u : 0u) | ((v + 1 < a.n_x ? 0x3F80u : 0u) << 16);
                }
                row[v8] = make_uint4(wds[0], wds[1], wds[2], wds[3]);
            }
            continue;
        }
        const uint32_t b = (uint32_t)(a.b_begin + (uint64_t)pi);
        uint4* LT4 = reinterpret_cast<uint4*>(LT);
        for (int q = l; q < lt_pitch / 8; q += 32) LT4[q] = make_uint4(0, 0, 0, 0);
        __syncwarp();
        // ---- phase A: draws + last-writer scatter, 128 steps per round
        for (uint32_t k0 = 0; k0 < nx; k0 += 128) {
            if (k0 + 4u * l < nx) {
                const u32x4 wd = philox4x32_10(u32x4{(k0 >> 2) + (uint32_t)l, b, s, 0u}, key0, key1);
                uint32_t j[4];
#pragma unroll
                for (uint32_t e = 0; e < 4; ++e) {
                    const uint32_t k = k0 + 4u * l + e;
                    j[e] = k < nx ? fy_target(u32x4_get(wd, e), k, N, b, s, key0, key1) : 0u;
                }
                *reinterpret_cast<uint2*>(stage + 4 * l) =
                    make_uint2(j[0] | (j[1] << 16), j[2] | (j[3] << 16));
            }
            __syncwarp();
            // scatter in 4 rounds of 32 consecutive steps (round r has larger k than r-1,
            // so rounds resolve in step order); a collision inside a round is fixed below
            uint32_t jr[4], kr[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const uint32_t k = k0 + 32u * r + l;
                const uint32_t j = k < nx ? (uint32_t)stage[32 * r + l] : k;
                // self-targets never move a value (k != q in LT); idle lanes act as such
                jr[r] = j;
                kr[r] = (j != k) ? k + 1u : 0u;  // value to store, 0 = no write
                if (kr[r]) LT[j] = (uint16_t)kr[r];
                __syncwarp();
            }
            // last writer (largest k) must win: a step that lost a same-round collision to
            // a smaller k rewrites; repeat until no step is short-changed (rarely > 1 pass)
            for (;;) {
                uint32_t lost = 0u;
#pragma unroll
                for (int r = 0; r < 4; ++r) lost |= (uint32_t)(LT[jr[r]] < kr[r]) << r;
                if (!__any_sync(0xffffffffu, lost)) break;
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    if ((lost >> r) & 1u) LT[jr[r]] = (uint16_t)kr[r];
                    __syncwarp();
                }
            }
        }
        // ---- phase B: each written high position exiles the end of its chain.  Per lane a
        // two-state machine (scan the lane's high positions / walk a chain), one LDS per
        // iteration, so lanes with short chains keep scanning while others walk.  In both
        // states the step ends on t == 0 (unwritten position / chain end); high positions
        // are never marked, chain nodes never exiled, so one test serves both states.
        {
            const uint32_t Nm1 = N - 1u;
            uint32_t pn = nx + l;          // next high position of this lane to scan
            uint32_t cur = min(pn, Nm1);   // LT index read this iteration
            uint32_t walking = 0u;
            while (__any_sync(0xffffffffu, pn < N)) {
#pragma unroll
                for (int rep = 0; rep < 2; ++rep) {  // dead lanes only read (store is gated)
                    const uint32_t t = LT[cur];
                    const uint32_t stop = (t == 0u) | (t == (uint32_t)kExiled);
                    if (walking & stop & (pn < N)) LT[cur] = kExiled;  // chain end: exiled
                    pn += stop ? 32u : 0u;
                    cur = stop ? min(pn, Nm1) : t - 1u;
                    walking = stop ^ 1u;
                }
            }
        }
        __syncwarp();
        // ---- phase C: exact 0/1 row
        if (a.out_kind == kMaskBf16Row) {
            const int64_t R1 = a.rows_per_tile - 1;
            const int64_t orow = (pi / R1) * a.rows_per_tile + 1 + pi % R1;
            uint4* row = reinterpret_cast<uint4*>(static_cast<uint16_t*>(a.out) + orow * a.n_pad);
            const uint4* L4 = reinterpret_cast<const uint4*>(LT);
            for (int64_t v8 = l; v8 < a.n_pad / 8; v8 += 32) {
                const uint4 q = L4[v8];
                const uint32_t w[4] = {q.x, q.y, q.z, q.w};
                uint32_t o[4];
                const int64_t v0 = 8 * v8;
                if (v0 + 8 <= (int64_t)nx) {  // low block: selected unless exiled
#pragma unroll
                    for (int e = 0; e < 4; ++e) o[e] = ~__vcmpeq2(w[e], 0xFFFFFFFFu) & 0x3F803F80u;
                } else if (v0 >= (int64_t)nx) {  // high block: selected iff written
#pragma unroll
                    for (int e = 0; e < 4; ++e) o[e] = __vcmpne2(w[e], 0u) & 0x3F803F80u;
                } else {
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        uint32_t pack = 0;
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const int64_t v = v0 + 2 * e + h;
                            const uint32_t t = (w[e] >> (16 * h)) & 0xFFFFu;
                            const bool sel = v < (int64_t)nx ? (t != kExiled) : (t != 0);
                            pack |= (sel ? 0x3F80u : 0u) << (16 * h);
                        }
                        o[e] = pack;
                    }
                }
                row[v8] = make_uint4(o[0], o[1], o[2], o[3]);
            }
        } else {
            uint8_t* row = static_cast<uint8_t*>(a.out) + pi * a.N;
            for (uint32_t v = l; v < N; v += 32) {
                const uint16_t t = LT[v];
                row[v] = (v < nx) ? (t != kExiled) : (t != 0);
            }
        }
        __syncwarp();
    }
}

}  // namespace

cudaError_t launch_perm(const PermArgs& a, int sm_count, cudaStream_t st) {
    if (a.count <= 0) return cudaSuccess;
    const int lt_pitch = (int)round_up(a.N, 64);  // uint16 entries, 128-byte multiple
    const size_t per_warp = (size_t)(lt_pitch + 128) * sizeof(uint16_t);
    const int nw = (int)std::max<size_t>(1, std::min<size_t>(kPermWarps, (200u * 1024u) / per_warp));
    const size_t smem = (size_t)nw * per_warp;
    static size_t configured = 0;
    if (smem > 48 * 1024 && smem > configured) {
        cudaError_t e = cudaFuncSetAttribute(k2_perm_fy, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
        configured = smem;
    }
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k2_perm_fy, nw * 32, smem);
    // at most 4 resident CTAs per SM: the generator for the next block runs beside the
    // persistent mask-GEMM, which keeps one CTA per SM
    per_sm = std::max(1, std::min(per_sm, a.max_ctas_per_sm > 0 ? a.max_ctas_per_sm : per_sm));
    const int64_t need = ceil_div(a.count + (a.out_kind == kMaskBf16Row ? a.ntiles : 0), nw);
    const int grid = (int)std::min<int64_t>(need, (int64_t)sm_count * per_sm);
    k2_perm_fy<<<grid, nw * 32, smem, st>>>(a, lt_pitch);
    return cudaGetLastError();
}

}  // namespace hap
