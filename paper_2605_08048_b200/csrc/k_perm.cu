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

#include <cstdlib>

#define HAP_CHECK_TU 2
#include "hap_device.cuh"
#include "hap_internal.h"

namespace hap {
namespace {

constexpr uint16_t kExiled = 0xFFFF;

// kPW warps share one permutation's table (more warps per SM for the same shared memory);
// warp w draws and scatters steps k0 + 128 w .. of each block of 128 kPW steps.
template <int kPW>
__device__ __forceinline__ void perm_sync() {
    if constexpr (kPW == 1) __syncwarp(); else __syncthreads();
}

template <int kPW>
__global__ void __launch_bounds__(kPW * 32) k2_perm_fy(PermArgs a, int lt_pitch) {
    extern __shared__ __align__(16) uint8_t smem[];
    constexpr uint32_t kT = 32u * kPW;
    const int tid = threadIdx.x, w = tid >> 5, l = tid & 31;
    uint16_t* LT = reinterpret_cast<uint16_t*>(smem);
    uint16_t* stage = LT + lt_pitch + 128 * w;
    const int64_t items = a.item_off[a.G];
    if (tid == 0) span_enter(a.span);
    for (int64_t pi = blockIdx.x; pi < items; pi += gridDim.x) {
        int ti = 0;  // test of this item (the tests' items are contiguous, in test order)
        while (ti + 1 < a.G && pi >= a.item_off[ti + 1]) ++ti;
        const PermTest& T = a.t[ti];
        const int64_t li = pi - a.item_off[ti];
        const uint32_t N = (uint32_t)T.N, nx = (uint32_t)T.n_x, s = T.s;
        const uint32_t key0 = (uint32_t)(T.seed & 0xFFFFFFFFu), key1 = (uint32_t)(T.seed >> 32);
        if (li >= T.count) {  // observed split: row 0 of tile (li - count)
            const int64_t t = li - T.count;
            uint4* row = reinterpret_cast<uint4*>(static_cast<uint16_t*>(T.out) +
                                                  t * a.rows_per_tile * T.n_pad);
            for (int64_t v8 = tid; v8 < T.n_pad / 8; v8 += kT) {
                uint32_t wds[4];
#pragma unroll
                for (int e2 = 0; e2 < 4; ++e2) {
                    const int64_t v = 8 * v8 + 2 * e2;
                    wds[e2] = (v < T.n_x ? 0x3F80u : 0u) | ((v + 1 < T.n_x ? 0x3F80u : 0u) << 16);
                }
                row[v8] = make_uint4(wds[0], wds[1], wds[2], wds[3]);
            }
            continue;
        }
        const uint32_t b = (uint32_t)(T.b_begin + (uint64_t)li);
        uint4* LT4 = reinterpret_cast<uint4*>(LT);
        for (int q = tid; q < lt_pitch / 8; q += kT) LT4[q] = make_uint4(0, 0, 0, 0);
        perm_sync<kPW>();
        // ---- phase A: draws + last-writer scatter, 128 steps per warp and round
        for (uint32_t k00 = 0; k00 < nx; k00 += 128u * kPW) {
            const uint32_t k0 = k00 + 128u * (uint32_t)w;
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
            // so rounds resolve in step order); a collision inside a round (or, kPW > 1,
            // with another warp's steps) is fixed below
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
            // last writer (largest k) must win: a step that lost a collision to a smaller k
            // rewrites; repeat until no step is short-changed (rarely > 1 pass)
            for (;;) {
                if constexpr (kPW > 1) __syncthreads();
                uint32_t lost = 0u;
#pragma unroll
                for (int r = 0; r < 4; ++r) lost |= (uint32_t)(LT[jr[r]] < kr[r]) << r;
                bool again;
                if constexpr (kPW == 1) again = __any_sync(0xffffffffu, lost);
                else again = __syncthreads_or(lost != 0u);
                if (!again) break;
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    if ((lost >> r) & 1u) LT[jr[r]] = (uint16_t)kr[r];
                    __syncwarp();
                }
            }
        }
        if constexpr (kPW > 1) __syncthreads();
        // ---- phase B: each written high position exiles the end of its chain.  Per lane a
        // two-state machine (scan the lane's high positions / walk a chain), one LDS per
        // iteration, so lanes with short chains keep scanning while others walk.  In both
        // states the step ends on t == 0 (unwritten position / chain end); high positions
        // are never marked, chain nodes never exiled, so one test serves both states.
        {
            const uint32_t Nm1 = N - 1u;
            uint32_t pn = nx + (uint32_t)tid;  // next high position of this thread to scan
            uint32_t cur = min(pn, Nm1);   // LT index read this iteration
            uint32_t walking = 0u;
            while (__any_sync(0xffffffffu, pn < N)) {
#pragma unroll
                for (int rep = 0; rep < 2; ++rep) {  // dead lanes only read (store is gated)
                    const uint32_t t = LT[cur];
                    const uint32_t stop = (t == 0u) | (t == (uint32_t)kExiled);
                    if (walking & stop & (pn < N)) LT[cur] = kExiled;  // chain end: exiled
                    pn += stop ? kT : 0u;
                    cur = stop ? min(pn, Nm1) : t - 1u;
                    walking = stop ^ 1u;
                }
            }
        }
        perm_sync<kPW>();
        // ---- phase C: exact 0/1 row
        if (a.out_kind == kMaskBf16Row) {
            const int64_t R1 = a.rows_per_tile - 1;
            const int64_t orow = (li / R1) * a.rows_per_tile + 1 + li % R1;
            uint4* row = reinterpret_cast<uint4*>(static_cast<uint16_t*>(T.out) + orow * T.n_pad);
            const uint4* L4 = reinterpret_cast<const uint4*>(LT);
            for (int64_t v8 = tid; v8 < T.n_pad / 8; v8 += kT) {
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
            uint8_t* row = static_cast<uint8_t*>(T.out) + li * T.N;
            for (uint32_t v = tid; v < N; v += kT) {
                const uint16_t t = LT[v];
                row[v] = (v < nx) ? (t != kExiled) : (t != 0);
            }
        }
        perm_sync<kPW>();
    }
    if (tid == 0) span_exit(a.span);
}


// ---------------------------------------------------------------------------------------
// Wide-table variant (N <= kWideMaxN): LT as uint32 so the last-writer scatter is one
// shared atomicMax per step (any order, no rounds / verification), and phase B first
// compacts the chain starts of the written high positions into a per-warp list, then
// walks the chains lane-balanced.  Same result bits as k2_perm_fy (tests).
constexpr uint32_t kExiled32 = 0xFFFFFFFFu;

// K2a (split generator): the draws only, register-resident, no shared memory, so it can
// run beside the smem-bandwidth-bound mask-GEMM without slowing it (measured); the targets
// (u16, n_x per permutation) are staged in the permutation's own mask row, which K2b reads
// before overwriting it with the mask.
__global__ void __launch_bounds__(128) k2_draws(PermArgs a) {
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    const int nw = (int)(blockDim.x >> 5);
    const int64_t items = a.item_off[a.G];
    if (threadIdx.x == 0) span_enter(a.span);
    for (int64_t pi = (int64_t)blockIdx.x * nw + w; pi < items; pi += (int64_t)gridDim.x * nw) {
        int ti = 0;
        while (ti + 1 < a.G && pi >= a.item_off[ti + 1]) ++ti;
        const PermTest& T = a.t[ti];
        const int64_t li = pi - a.item_off[ti];
        if (li >= T.count) continue;  // observed-split rows: K2b
        const uint32_t N = (uint32_t)T.N, nx = (uint32_t)T.n_x;
        const uint32_t key0 = (uint32_t)(T.seed & 0xFFFFFFFFu), key1 = (uint32_t)(T.seed >> 32);
        const uint32_t b = (uint32_t)(T.b_begin + (uint64_t)li);
        const int64_t R1 = a.rows_per_tile - 1;
        const int64_t orow = (li / R1) * a.rows_per_tile + 1 + li % R1;
        uint16_t* jrow = static_cast<uint16_t*>(T.out) + orow * T.n_pad;
        for (uint32_t k0 = 4u * (uint32_t)l; k0 < nx; k0 += 128u) {
            uint32_t j[4];
            draw_targets(k0, nx, N, b, T.s, key0, key1, j);
            *reinterpret_cast<uint2*>(jrow + k0) = make_uint2(j[0] | (j[1] << 16), j[2] | (j[3] << 16));
        }
    }
    if (threadIdx.x == 0) span_exit(a.span);
}

__device__ __forceinline__ void emit_row_u32(const PermArgs& a, const PermTest& T, const uint32_t* LT,
                                             int64_t li, uint32_t nx, int l, int nthreads) {
    const int64_t R1 = a.rows_per_tile - 1;
    const int64_t orow = (li / R1) * a.rows_per_tile + 1 + li % R1;
    HAP_CHECK(orow < (int64_t)T.ntiles * a.rows_per_tile && (T.n_pad & 3) == 0);
    // lane = 4 consecutive entries per step (contiguous 512 B per warp: conflict-free
    // LDS/STS.128), 8-byte stores of 4 bf16 (256 B per warp)
    uint2* row = reinterpret_cast<uint2*>(static_cast<uint16_t*>(T.out) + orow * T.n_pad);
    uint4* L4 = reinterpret_cast<uint4*>(const_cast<uint32_t*>(LT));
    const uint4 z = make_uint4(0, 0, 0, 0);
    for (int v4 = l; v4 < (int)(T.n_pad >> 2); v4 += nthreads) {
        const uint4 q = L4[v4];
        L4[v4] = z;  // leave the table zeroed for the next permutation
        const uint32_t t[4] = {q.x, q.y, q.z, q.w};
        const uint32_t v0 = 4u * (uint32_t)v4;
        uint32_t o[2];
        // low position: selected unless exiled (t + 1 != 0); high: iff written (t != 0)
        if (v0 + 4u <= nx || v0 >= nx) {  // all four on one side of n_x (all but one group)
            const uint32_t k = v0 < nx ? 1u : 0u;
            o[0] = (t[0] + k ? 0x3F80u : 0u) | (t[1] + k ? 0x3F800000u : 0u);
            o[1] = (t[2] + k ? 0x3F80u : 0u) | (t[3] + k ? 0x3F800000u : 0u);
        } else {
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const uint32_t va = v0 + 2 * e, vb = va + 1;
                const bool sa = t[2 * e] + (va < nx ? 1u : 0u) != 0u;
                const bool sb = t[2 * e + 1] + (vb < nx ? 1u : 0u) != 0u;
                o[e] = (sa ? 0x3F80u : 0u) | (sb ? 0x3F800000u : 0u);
            }
        }
        row[v4] = make_uint2(o[0], o[1]);
    }
}

// kPW warps share one permutation's table (as k2_perm_fy): the atomics of phase A and the
// mask emit split the steps / positions; each warp compacts and walks the chains of its own
// high positions (chains are disjoint) in its own start list.
template <int kPW>
__global__ void __launch_bounds__(kPW * 32) k2_perm_fy32(PermArgs a, int lt_pitch) {
    extern __shared__ __align__(16) uint8_t smem[];
    constexpr uint32_t kT = 32u * kPW;
    const int tid = threadIdx.x, w = tid >> 5, l = tid & 31;
    // per CTA: LT u32[lt_pitch] | sink u32[32 kPW] | kPW x starts u16[lt_pitch / 2 + 16]
    uint32_t* LT = reinterpret_cast<uint32_t*>(smem);
    uint32_t* sink = LT + lt_pitch + tid;  // per-thread target of the atomics of no-op steps
    uint16_t* starts = reinterpret_cast<uint16_t*>(LT + lt_pitch + kT) + (size_t)w * (lt_pitch / 2 + 16);
    const uint32_t lane_lt = (1u << l) - 1u;
    const int64_t items = a.item_off[a.G];
    if (tid == 0) span_enter(a.span);
    {
        uint4* L4 = reinterpret_cast<uint4*>(LT);
        for (int q = tid; q < lt_pitch / 4; q += kT) L4[q] = make_uint4(0, 0, 0, 0);
    }
    perm_sync<kPW>();
    for (int64_t pi = blockIdx.x; pi < items; pi += gridDim.x) {
        int ti = 0;  // test of this item (the tests' items are contiguous, in test order)
        while (ti + 1 < a.G && pi >= a.item_off[ti + 1]) ++ti;
        const PermTest& T = a.t[ti];
        const int64_t li = pi - a.item_off[ti];
        const uint32_t N = (uint32_t)T.N, nx = (uint32_t)T.n_x, s = T.s;
        const uint32_t key0 = (uint32_t)(T.seed & 0xFFFFFFFFu), key1 = (uint32_t)(T.seed >> 32);
        if (li >= T.count) {  // observed split: row 0 of tile (li - count)
            const int64_t t = li - T.count;
            uint4* row = reinterpret_cast<uint4*>(static_cast<uint16_t*>(T.out) +
                                                  t * a.rows_per_tile * T.n_pad);
            for (int64_t v8 = tid; v8 < T.n_pad / 8; v8 += kT) {
                uint32_t wds[4];
#pragma unroll
                for (int e2 = 0; e2 < 4; ++e2) {
                    const int64_t v = 8 * v8 + 2 * e2;
                    wds[e2] = (v < T.n_x ? 0x3F80u : 0u) | ((v + 1 < T.n_x ? 0x3F80u : 0u) << 16);
                }
                row[v8] = make_uint4(wds[0], wds[1], wds[2], wds[3]);
            }
            continue;
        }
        const uint32_t b = (uint32_t)(T.b_begin + (uint64_t)li);
        const int64_t R1 = a.rows_per_tile - 1;
        const int64_t orow = (li / R1) * a.rows_per_tile + 1 + li % R1;
        const uint16_t* jrow = static_cast<const uint16_t*>(T.out) + orow * T.n_pad;
        // ---- phase A: draws (or the targets K2a staged in this row) + last-writer scatter
        // (atomicMax = largest step wins)
        if (a.split == 2) {
            for (uint32_t kc = 4u * (uint32_t)tid; kc < nx; kc += 8u * 4u * kT) {
                uint2 jj[8];  // 8 blocks of 4 targets in flight (one L2 round trip)
#pragma unroll
                for (int it = 0; it < 8; ++it) {
                    const uint32_t k0 = kc + 4u * kT * it;
                    jj[it] = k0 < nx ? *reinterpret_cast<const uint2*>(jrow + k0) : make_uint2(0, 0);
                }
#pragma unroll
                for (int it = 0; it < 8; ++it) {
                    const uint32_t k0 = kc + 4u * kT * it;
                    const uint32_t j[4] = {jj[it].x & 0xFFFFu, jj[it].x >> 16, jj[it].y & 0xFFFFu,
                                           jj[it].y >> 16};
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const uint32_t k = k0 + e;
                        atomicMax((k < nx && j[e] != k) ? LT + j[e] : sink, k + 1u);
                    }
                }
            }
        } else {
            const PhiloxKeys K = philox_keys(key0, key1);
            for (uint32_t k0 = 4u * (uint32_t)tid; k0 < nx; k0 += 4u * kT) {
                uint32_t j[4];
                draw_targets(k0, nx, N, b, s, key0, key1, j, &K);
#pragma unroll
                for (int e = 0; e < 4; ++e) {  // unconditional: no-op steps hit the lane's sink
                    const uint32_t k = k0 + e;
                    HAP_CHECK(k >= nx || (j[e] >= k && j[e] < N));
                    atomicMax((k < nx && j[e] != k) ? LT + j[e] : sink, k + 1u);
                }
            }
        }
        perm_sync<kPW>();
        // ---- phase B1: chain starts LT[p]-1 of the written high positions, 8 per lane per
        // pass.  A chain that ends at its start (position k* not written before step k*,
        // ~70 % of them) is exiled right here; the others enter the list at their second
        // node, at offsets from a warp prefix sum of the per-lane counts (4 ballots).
        uint32_t nst = 0;
        for (uint32_t base = (nx & ~3u) + 256u * (uint32_t)w; __any_sync(0xffffffffu, base + 4u * (uint32_t)l < N);
             base += 256u * kPW) {
            // entries base + 4l .. +3 and base + 128 + 4l .. +3: each half is a contiguous
            // 512 B per warp (conflict-free LDS.128); beyond N the table is 0
            const uint32_t pa = base + 4u * (uint32_t)l, pb = pa + 128u;
            uint4 q0 = make_uint4(0, 0, 0, 0), q1 = q0;
            if (pa < N) q0 = *reinterpret_cast<const uint4*>(LT + pa);
            if (pb < N) q1 = *reinterpret_cast<const uint4*>(LT + pb);
            uint32_t t[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
            if (pa < nx) {  // positions below n_x only occur in the first pass (lane 0)
#pragma unroll
                for (int e = 0; e < 4; ++e) t[e] = pa + e >= nx ? t[e] : 0u;
            }
            uint32_t u[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) u[e] = t[e] ? LT[t[e] - 1u] : 0u;  // all in flight
            uint32_t cnt = 0;
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                if (t[e] != 0u && u[e] == 0u) LT[t[e] - 1u] = kExiled32;
                cnt += (t[e] != 0u && u[e] != 0u) ? 1u : 0u;
            }
            uint32_t at = nst;  // + exclusive prefix of cnt over the lanes below
#pragma unroll
            for (int bit = 0; bit < 4; ++bit)
                at += (uint32_t)__popc(__ballot_sync(0xffffffffu, (cnt >> bit) & 1u) & lane_lt) << bit;
            const uint32_t tot = __reduce_add_sync(0xffffffffu, cnt);
            HAP_CHECK(at + 8u <= (uint32_t)(lt_pitch / 2 + 16));
#pragma unroll
            for (int e = 0; e < 8; ++e)
                if (t[e] != 0u && u[e] != 0u) starts[at++] = (uint16_t)(u[e] - 1u);
            nst += tot;
        }
        __syncwarp();
        // ---- phase B2: walk each chain to its end (an unwritten low position) and exile it;
        // two cursors per lane (starts l, l+64, ... and l+32, l+96, ...) keep two table
        // reads in flight (chains are disjoint, so the cursors never meet)
        {
            uint32_t i0 = (uint32_t)l, i1 = (uint32_t)l + 32u;
            uint32_t c0 = i0 < nst ? starts[i0] : 0u, c1 = i1 < nst ? starts[i1] : 0u;
            while (__any_sync(0xffffffffu, (i0 < nst) | (i1 < nst))) {
                const uint32_t t0 = LT[c0], t1 = LT[c1];  // inactive cursors re-read entry 0
                const bool e0 = (i0 < nst) & (t0 == 0u), e1 = (i1 < nst) & (t1 == 0u);
                if (e0) LT[c0] = kExiled32;
                if (e1) LT[c1] = kExiled32;
                i0 += e0 ? 64u : 0u;
                i1 += e1 ? 64u : 0u;
                const uint32_t n0 = starts[min(i0, nst)], n1 = starts[min(i1, nst)];  // in bounds
                c0 = i0 < nst ? (e0 ? n0 : t0 - 1u) : 0u;
                c1 = i1 < nst ? (e1 ? n1 : t1 - 1u) : 0u;
            }
        }
        perm_sync<kPW>();
        // ---- phase C: exact 0/1 row (re-zeroes the table)
        if (a.out_kind == kMaskBf16Row) {
            emit_row_u32(a, T, LT, li, nx, tid, (int)kT);
        } else {
            uint8_t* row = static_cast<uint8_t*>(T.out) + li * T.N;
            for (uint32_t v = tid; v < N; v += kT) {
                const uint32_t t = LT[v];
                LT[v] = 0u;
                row[v] = (v < nx) ? (t != kExiled32) : (t != 0u);
            }
        }
        perm_sync<kPW>();
    }
    if (tid == 0) span_exit(a.span);
}

// ---------------------------------------------------------------------------------------
// Exhaustive mode (HAP_FLAG_EXHAUSTIVE): thread = one combination, b is
// its colex rank: b = sum_{i=1..n_x} C(c_i, i) with c_1 < .. < c_nx, unranked greedily from
// the largest element down with a shared binomial table.  N <= 64 (n_pad = 64).
constexpr int kCombMaxN = 64;

__global__ void __launch_bounds__(128) k2_comb_unrank(PermArgs a) {
    constexpr int kK = kCombMaxN / 2 + 1;  // k <= 32 (the smaller side of the split)
    __shared__ unsigned long long binom[kCombMaxN + 1][kK + 1];
    if (threadIdx.x == 0) {  // Pascal's triangle, saturating (only values < 2^32 are used)
        const unsigned long long sat = 1ull << 62;
        for (int n = 0; n <= kCombMaxN; ++n)
            for (int k = 0; k <= kK; ++k) {
                unsigned long long c;
                if (k == 0) c = 1;
                else if (n == 0) c = 0;
                else c = binom[n - 1][k - 1] + binom[n - 1][k];
                binom[n][k] = c > sat ? sat : c;
            }
    }
    __syncthreads();
    if (threadIdx.x == 0) span_enter(a.span);
    const int64_t items = a.item_off[a.G];
    for (int64_t pi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; pi < items;
         pi += (int64_t)gridDim.x * blockDim.x) {
        int ti = 0;
        while (ti + 1 < a.G && pi >= a.item_off[ti + 1]) ++ti;
        const PermTest& T = a.t[ti];
        const int64_t li = pi - a.item_off[ti];
        const int N = (int)T.N, nx = (int)T.n_x;
        const unsigned long long all = N >= 64 ? ~0ull : ((1ull << N) - 1ull);
        unsigned long long sel = 0;  // bit c = element c in group 1
        if (li >= T.count) {
            sel = nx >= 64 ? ~0ull : ((1ull << nx) - 1ull);  // observed split {0..n_x-1}
        } else {
            // enumerate the smaller side (k = min(n_x, n_y)); complement when n_x > n_y
            const int k = nx <= N - nx ? nx : N - nx;
            unsigned long long r = T.b_begin + (uint64_t)li;
            int c = N - 1;
            for (int i = k; i >= 1; --i) {  // largest c with C(c, i) <= r
                while (binom[c][i] > r) --c;
                r -= binom[c][i];
                sel |= 1ull << c;
                --c;
            }
            if (k != nx) sel = ~sel & all;
        }
        if (a.out_kind == kMaskBf16Row) {
            const int64_t R1 = a.rows_per_tile - 1;
            const int64_t orow = li >= T.count ? (li - T.count) * a.rows_per_tile
                                               : (li / R1) * a.rows_per_tile + 1 + li % R1;
            uint4* row = reinterpret_cast<uint4*>(static_cast<uint16_t*>(T.out) + orow * T.n_pad);
            for (int v8 = 0; v8 < (int)(T.n_pad >> 3); ++v8) {
                const uint32_t byte = (uint32_t)(v8 < 8 ? (sel >> (8 * v8)) & 0xFFu : 0u);
                uint32_t o[4];
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    o[e] = (((byte >> (2 * e)) & 1u) | (((byte >> (2 * e + 1)) & 1u) << 16)) * 0x3F80u;
                row[v8] = make_uint4(o[0], o[1], o[2], o[3]);
            }
        } else {
            uint8_t* row = static_cast<uint8_t*>(T.out) + li * T.N;
            for (int v = 0; v < N; ++v) row[v] = (uint8_t)((sel >> v) & 1ull);
        }
    }
    if (threadIdx.x == 0) span_exit(a.span);
}

// Development aid (scheduling experiments): a register-only Philox loop, no shared memory.
__global__ void k_debug_alu_burn(uint32_t iters, uint32_t* sink) {
    u32x4 c{threadIdx.x, blockIdx.x, 0u, 0u};
    for (uint32_t i = 0; i < iters; ++i) {
        c = philox4x32_10(c, 0x12345678u, 0x9abcdef0u);
        c.z = i;
    }
    if (c.x == 0x7fffffffu) sink[0] = c.y;  // keep the loop alive
}

}  // namespace

cudaError_t launch_debug_alu_burn(uint32_t iters, int ctas, int threads, uint32_t* sink, cudaStream_t st) {
    k_debug_alu_burn<<<ctas, threads, 0, st>>>(iters, sink);
    return cudaGetLastError();
}

bool perm_can_split(const PermArgs& a) {
    static const char* nar = getenv("HAP_K2_NARROW");
    if (a.out_kind != kMaskBf16Row || (nar && atoi(nar))) return false;
    int64_t maxN = 0;
    for (int g = 0; g < a.G; ++g) {
        if (a.t[g].exhaustive) return false;
        maxN = std::max<int64_t>(maxN, a.t[g].N);
    }
    const int lt_pitch = (int)round_up(maxN, 64);
    return (size_t)lt_pitch * 5u + 160u <= (200u * 1024u) / 4u;  // the wide table path
}

void perm_items(PermArgs& a) {
    a.item_off[0] = 0;
    for (int g = 0; g < a.G; ++g)
        a.item_off[g + 1] = a.item_off[g] + a.t[g].count + (a.out_kind == kMaskBf16Row ? a.t[g].ntiles : 0);
}

cudaError_t launch_perm(const PermArgs& a, int sm_count, cudaStream_t st) {
    const int64_t items = a.item_off[a.G];
    if (items <= 0) return cudaSuccess;
    if (a.t[0].exhaustive) {  // a wave is all-exhaustive or not at all
        const int64_t grid = std::min<int64_t>(ceil_div(items, 128), (int64_t)sm_count * 8);
        k2_comb_unrank<<<(int)grid, 128, 0, st>>>(a);
        return cudaGetLastError();
    }
    int64_t maxN = 0;
    for (int g = 0; g < a.G; ++g) maxN = std::max<int64_t>(maxN, a.t[g].N);
    const int lt_pitch = (int)round_up(maxN, 64);  // entries, 128-byte multiple; >= every n_pad
    // wide (uint32) table + start list when 4 warps fit in the budget, else uint16 table
    static const char* nar = getenv("HAP_K2_NARROW");  // EXPERIMENT: force the u16 table
    // the u32 table + start list take 5 bytes per pooled row and warp: for large N the u16
    // table doubles the warps per SM, which wins over the wide kernel's cheaper scatter
    // (batches of equal pairs: N = 2400 wide 100.7 vs 103.6 us/test, N = 3000 125.5 vs 124.1,
    // N = 4000 169.7 vs 164.9; C4 115.2 -> 110-112, C3 13.9 -> 13.7 ms); cut-over at
    // HAP_K2_WIDE_MAX_N (default 2560 pooled rows)
    static const char* wmax_env = getenv("HAP_K2_WIDE_MAX_N");
    const int64_t wide_max_n = wmax_env ? atoll(wmax_env) : 2560;
    const bool wide = (size_t)lt_pitch * 5u + 160u <= (200u * 1024u) / 4u && !(nar && atoi(nar)) &&
                      maxN <= wide_max_n;
    // narrow: kPW warps per permutation share its table, so latency-bound warps are not
    // limited by tables per SM (N = 5000 / 10^4 pairs: 216 -> 206 / 499 -> 408 us per test
    // with 2 / 4 warps); HAP_K2_PW = 1, 2 or 4 overrides
    static const char* pw_env = getenv("HAP_K2_PW");
    const int pw = pw_env ? std::max(1, std::min(4, atoi(pw_env))) : maxN >= 6144 ? 4 : 2;
    static const char* wpw_env = getenv("HAP_K2_WIDE_PW");  // the same for the u32 table
    const int wpw = wpw_env ? std::max(1, std::min(4, atoi(wpw_env))) : 1;
    const int kpw = wide ? (wpw >= 4 ? 4 : wpw >= 2 ? 2 : 1) : (pw >= 4 ? 4 : pw >= 2 ? 2 : 1);
    // per CTA (one permutation at a time): u32 table + sinks + a start list per warp, or
    // u16 table + a staging row per warp
    const size_t smem = wide ? (size_t)lt_pitch * (4u + kpw) + 160u * kpw
                             : (size_t)(lt_pitch + 128 * kpw) * sizeof(uint16_t);
    const int nw = kpw;
    const void* fn = wide ? (kpw == 4 ? (const void*)k2_perm_fy32<4>
                             : kpw == 2 ? (const void*)k2_perm_fy32<2>
                                        : (const void*)k2_perm_fy32<1>)
                     : kpw == 4 ? (const void*)k2_perm_fy<4>
                     : kpw == 2 ? (const void*)k2_perm_fy<2>
                                : (const void*)k2_perm_fy<1>;
    const int fi = (wide ? 5 : 0) + kpw;
    static size_t configured[10] = {};
    if (smem > 48 * 1024 && smem > configured[fi]) {
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        configured[fi] = smem;
    }
    static bool carve[10] = {};
    if (!carve[fi]) {  // max shared carveout, so generator CTAs fit beside a mask-GEMM CTA
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout,
                                             cudaSharedmemCarveoutMaxShared);
        if (e != cudaSuccess) return e;
        carve[fi] = true;
    }
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, nw * 32, smem);
    per_sm = std::max(1, std::min(per_sm, a.max_ctas_per_sm > 0 ? a.max_ctas_per_sm : per_sm));
    const int64_t need = items;  // one permutation per CTA at a time
    const int grid = (int)std::min<int64_t>(need, (int64_t)sm_count * per_sm);
    if (a.split == 1) {  // K2a: draws into the rows, register-only (wide path only)
        const int64_t g2 = std::min<int64_t>(ceil_div(items, 4), (int64_t)sm_count * 4);
        k2_draws<<<(int)g2, 128, 0, st>>>(a);
    } else if (wide) {
        if (kpw == 4) k2_perm_fy32<4><<<grid, 128, smem, st>>>(a, lt_pitch);
        else if (kpw == 2) k2_perm_fy32<2><<<grid, 64, smem, st>>>(a, lt_pitch);
        else k2_perm_fy32<1><<<grid, 32, smem, st>>>(a, lt_pitch);
    } else {
        if (kpw == 4) k2_perm_fy<4><<<grid, 128, smem, st>>>(a, lt_pitch);
        else if (kpw == 2) k2_perm_fy<2><<<grid, 64, smem, st>>>(a, lt_pitch);
        else k2_perm_fy<1><<<grid, 32, smem, st>>>(a, lt_pitch);
    }
    return cudaGetLastError();
}

HAP_CHECK_ACCESSOR(check_word_perm)

}  // namespace hap
