// hap_device.cuh — sm_100a device helpers for libhap: mbarrier, TMA, tcgen05/TMEM
// inline PTX, and the product's Philox4x32-10.  (Independent of oracle/: nothing here is
// shared with the checker.)
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#define HAP_DEV __device__ __forceinline__

namespace hap {

// --------------------------------------------------------------------------- basics
HAP_DEV uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// kernel span profiling: {min entry, max exit} %globaltimer over CTAs (one clock for all
// kernels and streams, so concurrent launches can be laid on one timeline)
HAP_DEV unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
HAP_DEV void span_enter(unsigned long long* span) {
    if (span) atomicMin(span, global_ns());
}
HAP_DEV void span_exit(unsigned long long* span) {
    if (span) atomicMax(span + 1, global_ns());
}

// ---- device checks (the checked build, -DHAP_DEVICE_CHECKS: libhap_checked.so).  A
// failed HAP_CHECK records {translation unit, source line} of the FIRST failure in a
// per-translation-unit word (read and cleared by hap_debug_check_status) and execution
// continues; the release library compiles every check out.  The stand-in for
// compute-sanitizer, which this GPU pool refuses.
#ifdef HAP_DEVICE_CHECKS
static __device__ unsigned long long g_hap_check = 0ull;
#define HAP_CHECK(cond)                                                                         \
    do {                                                                                       \
        if (!(cond))                                                                           \
            atomicCAS(&g_hap_check, 0ull, ((unsigned long long)HAP_CHECK_TU << 32) | __LINE__); \
    } while (0)
// host side: read and clear this translation unit's word
#define HAP_CHECK_ACCESSOR(fn)                                                   \
    unsigned long long fn() {                                                   \
        unsigned long long v = 0ull, z = 0ull;                                   \
        cudaMemcpyFromSymbol(&v, g_hap_check, sizeof v);                        \
        cudaMemcpyToSymbol(g_hap_check, &z, sizeof z);                          \
        return v;                                                               \
    }
#else
#define HAP_CHECK(cond) \
    do {                \
    } while (0)
#define HAP_CHECK_ACCESSOR(fn) \
    unsigned long long fn() { return 0ull; }
#endif

// programmatic dependent launch: a kernel launched with programmatic stream serialization
// may start while its predecessor finishes; griddepcontrol.wait blocks until the predecessor
// grid has completed and its memory is visible (a no-op without the launch attribute)
HAP_DEV void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
HAP_DEV void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

HAP_DEV uint32_t lane_id() { return threadIdx.x & 31u; }
HAP_DEV uint32_t warp_id() { return __shfl_sync(0xffffffffu, threadIdx.x >> 5, 0); }
HAP_DEV bool elect_one() {
    uint32_t pred = 0;
    asm volatile(
        "{\n\t.reg .pred P;\n\t"
        "elect.sync _|P, 0xffffffff;\n\t"
        "selp.u32 %0, 1, 0, P;\n\t}\n"
        : "=r"(pred));
    return pred != 0;
}

// --------------------------------------------------------------------------- mbarrier
HAP_DEV void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
HAP_DEV void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
HAP_DEV void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
HAP_DEV void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(
                     smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
HAP_DEV bool mbar_try_wait(uint32_t addr, uint32_t parity) {
    uint32_t ok = 0;
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2, 1000000;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t}\n"
        : "=r"(ok)
        : "r"(addr), "r"(parity)
        : "memory");
    return ok != 0;
}
// Blocking wait on the phase with the given parity.  A wait that never completes (a
// pipeline bug) traps after ~2^35 cycles (~20 s) instead of hanging the GPU.
HAP_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
    const uint32_t addr = smem_u32(bar);
    uint32_t n = 0;
    long long t0 = 0;
    while (!mbar_try_wait(addr, parity)) {
        if ((++n & 1023u) == 0) {
            const long long now = clock64();
            if (t0 == 0) t0 = now;
            else if (now - t0 > (1ll << 35)) __trap();
        }
    }
}

// --------------------------------------------------------------------------- TMA
HAP_DEV void tma_prefetch_desc(const void* desc) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(desc)) : "memory");
}
// 2-D tiled load: coordinates (c0 = innermost element index, c1 = row)
HAP_DEV void tma_load_2d(const void* desc, uint64_t* bar, void* smem_dst, int32_t c0, int32_t c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(smem_dst)),
        "l"(reinterpret_cast<uint64_t>(desc)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}

// --------------------------------------------------------------------------- tcgen05
HAP_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
HAP_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

template <uint32_t kCols>
HAP_DEV void tmem_alloc(uint32_t* smem_dst) {  // whole warp
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(smem_dst)),
                 "n"(kCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
template <uint32_t kCols>
HAP_DEV void tmem_dealloc(uint32_t taddr) {  // whole warp
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols)
                 : "memory");
}

// D[tmem] (+)= A[smem] * B[smem]^T, kind::f16 (bf16 x bf16 -> fp32), issued by one thread.
HAP_DEV void umma_bf16_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                          uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// mbarrier arrives when all prior tcgen05 async ops of this thread complete
HAP_DEV void umma_commit(uint64_t* bar) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(bar))
        : "memory");
}

// Shared-memory matrix descriptor, K-major operand, 128-byte swizzle (canonical
// layout: rows of 128 B, 8-row groups 1024 B apart).  Bits: start>>4 [0,14), LBO>>4
// [16,30) (unused for swizzled K-major, =1), SBO>>4 [32,46), version=1 [46,48),
// base offset 0, layout type SWIZZLE_128B = 2 at [61,64).
HAP_DEV uint64_t smem_desc_k_sw128(uint32_t smem_addr) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((smem_addr >> 4) & 0x3FFFu);
    d |= static_cast<uint64_t>(1u) << 16;
    d |= static_cast<uint64_t>(1024u >> 4) << 32;
    d |= static_cast<uint64_t>(1u) << 46;
    d |= static_cast<uint64_t>(2u) << 61;
    return d;
}

// Instruction descriptor, kind::f16: D fp32, A/B bf16, both K-major, shape M x N.
HAP_DEV constexpr uint32_t idesc_bf16_f32(uint32_t M, uint32_t N) {
    return (1u << 4)            // D format F32
           | (1u << 7)          // A format BF16
           | (1u << 10)         // B format BF16
           | ((N >> 3) << 17)   // N >> 3
           | ((M >> 4) << 24);  // M >> 4
}

// 32 lanes x 32 bit, 32 consecutive columns -> 32 registers per thread
HAP_DEV void tmem_ld_32x32b_x32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
          "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
          "=r"(r[31])
        : "r"(taddr));
}
HAP_DEV void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// --------------------------------------------------------------------------- clusters / 2-SM
HAP_DEV uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
HAP_DEV void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                     : "memory");
}
// shared::cluster address of the same smem offset in CTA `rank` of the cluster
HAP_DEV uint32_t mapa_shared(uint32_t local_addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local_addr), "r"(rank));
    return r;
}
HAP_DEV void mbar_arrive_cluster(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
                 : "memory");
}
// remote arrive with the default (release, CTA-scope) semantics, as CUTLASS's cluster
// barriers use for peer-CTA signalling
HAP_DEV void mbar_arrive_remote(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// arrive on a (possibly remote) mbarrier and expect `bytes` of transaction data, relaxed
HAP_DEV void mbar_arrive_expect_tx_cluster_relaxed(uint32_t cluster_bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.relaxed.cluster.shared::cluster.b64 _, [%0], %1;" ::"r"(cluster_bar),
                 "r"(bytes)
                 : "memory");
}
// asynchronous store into a (possibly remote) CTA's shared memory; completes `bytes` on the
// mbarrier at `cluster_bar` (same CTA as the destination) when the data has landed
HAP_DEV void st_async_u32(uint32_t cluster_addr, uint32_t v, uint32_t cluster_bar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.u32 [%0], %1, [%2];" ::"r"(cluster_addr),
                 "r"(v), "r"(cluster_bar)
                 : "memory");
}
HAP_DEV void st_shared_cluster_u32(uint32_t cluster_addr, uint32_t v) {
    asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(cluster_addr), "r"(v) : "memory");
}
// 2-SM TMA: data lands in this CTA's smem, completion bytes are counted on the mbarrier at
// the shared::cluster address `bar_cluster` (the leader CTA's barrier).
HAP_DEV void tma_load_2d_pair(const void* desc, uint32_t bar_cluster, void* smem_dst, int32_t c0,
                              int32_t c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(smem_dst)),
        "l"(reinterpret_cast<uint64_t>(desc)), "r"(bar_cluster), "r"(c0), "r"(c1)
        : "memory");
}
template <uint32_t kCols>
HAP_DEV void tmem_alloc_pair(uint32_t* smem_dst) {  // whole warp, same warp id in both CTAs
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(smem_dst)),
                 "n"(kCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
template <uint32_t kCols>
HAP_DEV void tmem_dealloc_pair(uint32_t taddr) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols)
                 : "memory");
}
// D[tmem of both CTAs] (+)= A[smem of both CTAs] * B[smem of both CTAs]^T, M = 256; issued by
// one thread of the leader CTA.
HAP_DEV void umma_bf16_ss_pair(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                               uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// arrive on the barrier at the same offset in every CTA of `cta_mask` when this thread's
// prior tcgen05 ops complete
HAP_DEV void umma_commit_pair(uint64_t* bar, uint16_t cta_mask) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
        " [%0], %1;" ::"r"(smem_u32(bar)),
        "h"(cta_mask)
        : "memory");
}
HAP_DEV void named_bar_sync(uint32_t id, uint32_t nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// --------------------------------------------------------------------------- Philox
// Philox4x32-10 (Salmon et al., SC'11): the product's own implementation.
struct u32x4 {
    uint32_t x, y, z, w;
};
HAP_DEV u32x4 philox4x32_10(u32x4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
        const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
        c = u32x4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return c;
}
// the ten round keys of a (seed) key, computed once per permutation instead of once per
// block (2 adds per round otherwise)
struct PhiloxKeys {
    uint32_t a[10], b[10];
};
HAP_DEV PhiloxKeys philox_keys(uint32_t k0, uint32_t k1) {
    PhiloxKeys K;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        K.a[r] = k0;
        K.b[r] = k1;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return K;
}
HAP_DEV u32x4 philox4x32_10(u32x4 c, const PhiloxKeys& K) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
        const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
        c = u32x4{hi1 ^ c.y ^ K.a[r], lo1, hi0 ^ c.w ^ K.b[r], lo0};
    }
    return c;
}
HAP_DEV uint32_t u32x4_get(const u32x4& v, uint32_t e) {
    return e == 0 ? v.x : e == 1 ? v.y : e == 2 ? v.z : v.w;
}

// ---- PERM-SPEC v1 draws (R6), shared by K2 and K1's staged-draw pass
// U(N-k) for step k: Lemire on the main-stream word x; rejected words are replaced by
// the side stream (counter (q', b, s, 1+k)) in order.
HAP_DEV uint32_t fy_target(uint32_t x, uint32_t k, uint32_t N, uint32_t b,
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

// targets j_k = k + U(N - k) of steps k0 .. k0+3 (one Philox block; Lemire, exact slow path)
HAP_DEV void draw_targets(uint32_t k0, uint32_t nx, uint32_t N, uint32_t b,
                                             uint32_t s, uint32_t key0, uint32_t key1, uint32_t j[4],
                                             const PhiloxKeys* K = nullptr) {
    const u32x4 wd = K ? philox4x32_10(u32x4{k0 >> 2, b, s, 0u}, *K)
                       : philox4x32_10(u32x4{k0 >> 2, b, s, 0u}, key0, key1);
    const uint32_t x[4] = {wd.x, wd.y, wd.z, wd.w};
    bool slow = false;
#pragma unroll
    for (int e = 0; e < 4; ++e) {  // Lemire fast path; rejection needs lo < bound
        const uint32_t k = k0 + e, bound = N - k;
        const uint64_t m = (uint64_t)x[e] * bound;
        slow |= (uint32_t)m < bound;
        j[e] = k + (uint32_t)(m >> 32);
    }
    if (slow) {
#pragma unroll
        for (int e = 0; e < 4; ++e)
            if (k0 + e < nx) j[e] = fy_target(x[e], k0 + e, N, b, s, key0, key1);
    }
}


}  // namespace hap
