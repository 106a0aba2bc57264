// hap_internal.h — declarations shared by the libhap translation units (host side).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/hap.h"
#include "../../include/hap_debug.h"

namespace hap {

// checked build (-DHAP_DEVICE_CHECKS): first failed device check per translation unit,
// {unit << 32 | line}, 0 = none; read and cleared (0 in the release library)
unsigned long long check_word_align();
unsigned long long check_word_perm();
unsigned long long check_word_gemm();
unsigned long long check_word_gram();

constexpr int kKBlock = 64;     // GEMM K-block: 64 bf16 = one 128-byte swizzle atom
constexpr int kTileM = 128;     // permutations per CTA tile (TMEM lanes)
#ifndef HAP_CHUNK_N
#define HAP_CHUNK_N 256
#endif
constexpr int kChunkN = HAP_CHUNK_N;  // d-columns per accumulator chunk (UMMA N <= 256, % 32 == 0)

inline int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }
inline int64_t ceil_div(int64_t x, int64_t m) { return (x + m - 1) / m; }

constexpr int kMaxWave = 4;  // tests per launch of a wave (K1, K2, K3)

// A WAVE is up to kMaxWave independent tests (each aligned in its own workspace) whose
// rows go through ONE K1 launch, whose generator rows go through ONE K2 launch and whose
// tiles go through ONE K3 launch.

// ---- K2: PERM-SPEC v1 generator (k_perm.cu) ----------------------------------------
enum MaskOut { kMaskBf16Row = 0, kMaskU8Set = 1 };
struct PermTest {
    uint64_t seed;
    uint32_t s;              // generator stream id
    uint64_t b_begin;
    int64_t count;           // permutations b_begin .. b_begin + count
    int64_t N, n_x, n_pad;
    void* out;               // bf16 rows (tile layout) or uint8 [count][N]
    int ntiles;              // bf16 mode: tiles (each also gets its observed-split row 0)
    int exhaustive;          // 1: b = colex rank of the combination (HAP_FLAG_EXHAUSTIVE)
};
struct PermArgs {
    int G;                   // tests in this launch
    PermTest t[kMaxWave];
    int64_t item_off[kMaxWave + 1];  // warp items of test g: [item_off[g], item_off[g+1])
    int out_kind;            // MaskOut
    int rows_per_tile;       // bf16 mode: R; perm p -> row (p/(R-1))*R + 1 + p%(R-1),
                             // row t*R = observed split {0..n_x-1} for t < ntiles
    int max_ctas_per_sm;     // 0 = occupancy limit
    int split;               // 0 = fused; 1 = K2a: draws staged in the rows (register-only);
                             // 2 = K2b: table, chains and rows from the staged draws
    unsigned long long* span;  // optional {first CTA entry, last CTA exit} globaltimer
};
// fills item_off from the tests (count + ntiles rows each in bf16 mode)
void perm_items(PermArgs& a);
// whether a launch may be split into K2a + K2b (bf16 rows, wide table, not exhaustive)
bool perm_can_split(const PermArgs& a);
cudaError_t launch_perm(const PermArgs& a, int sm_count, cudaStream_t st);
cudaError_t launch_debug_alu_burn(uint32_t iters, int ctas, int threads, uint32_t* sink, cudaStream_t st);

// ---- K1: alignment (k_align.cu) ----------------------------------------------------

// One word pair of a K1 launch (its own workspace buffers)
struct AlignPair {
    const float* X;
    const float* Y;
    int64_t n_x, n_y, d, n_pad;
    hap_align_info* info;    // device
    double* inv;             // [N]    1/||h_i|| (0 for a zero row)
    float2* coef;            // [N]    {2 u.x_i, 1/||h_i||} (streaming path, K1s)
    double* u;               // [d_pad] Householder axis (0 for the identity)
    double* xbar;            // [d]
    double* ybar;            // [d]
    uint16_t* zt_hi;         // [>=d_pad][n_pad] bf16 bits
    uint16_t* zt_lo;         // [>=d_pad][n_pad]
    double* m;               // [d_pad] centre (multiple of 2^-12): planes hold z - m
    double* t64;             // [d_pad] t = N m + t'
    float2* ab;              // [d_pad] epilogue constants {2a, 2b}, a = n_x m, b = t - a
    double* sconst;          // [3]     {sum a^2, sum b^2, eps_rep (R14)}
    long long* acc;          // [2 d + d_pad] fixed-point column sums (zero between launches)
    long long* bad;          // min ZeroVector row (LLONG_MAX = none; reset by the launch)
};
struct AlignArgs {
    int G;                   // pairs in this launch (same d)
    AlignPair p[kMaxWave];
    int64_t item_off[kMaxWave + 1];  // items (R-row blocks) of pair g: [item_off[g], item_off[g+1])
    int64_t d, d_pad;
    int mode;                // hap_align_mode
    long long* scratch;      // [1] ticket, [2] grid barrier of the launch
    long long* stamps;       // optional [8 + 8 grid] globaltimer stamps (profiling)
    unsigned long long* span;  // optional {first CTA entry, last CTA exit} globaltimer
    int do_draws;            // 1: also stage the generator draws of `draws` (K2a's work)
    PermArgs draws;          // split = 1 job, run in K1's idle issue slots
};
// item geometry of K1: R pooled rows x all d columns as an fp32 smem tile of pitch P
struct AlignGeom {
    int rows, pitch;
    bool stage_umc;    // per-column (u_c, m_c) staged in smem
    bool stage_means;  // xbar, ybar also staged in smem
    size_t smem;       // dynamic smem bytes
};
AlignGeom align_geometry(int64_t d);
// fills item_off (n_pad / R items per pair) for the geometry of d
void align_items(AlignArgs& a);
// Alignment path of a pair, a function of its shape only (so a pair gets the same bits
// alone, in any batch wave and on every rank; a wave's pairs all take one path):
//   kAlignRing  d % 4 == 0, d <= 4096, n_pad d >= 8 Mi elements: K1s, three bandwidth
//               kernels with shared-memory rings (LLM-sized clouds, C3);
//   kAlignLean  the same constraints below 8 Mi elements: K1s-lean, the same three passes
//               with register-prefetched loads and < 18 KB of shared memory per CTA, so
//               they run beside a mask-GEMM CTA (C1, C2, C4, C5);
//   kAlignFused otherwise (d % 4 != 0 or d > 4096; also inputs not 16-byte aligned): ONE
//               cooperative kernel of `grid` CTAs whose scratch[2] holds its grid barrier.
enum { kAlignFused = 0, kAlignLean = 1, kAlignRing = 2 };
int align_path(int64_t N, int64_t d);
bool align_uses_stream(const AlignArgs& a);
int align_launch_count(const AlignArgs& a);  // kernels issued by launch_align
cudaError_t launch_align(const AlignArgs& a, int grid, cudaStream_t st);

// ---- K3: tcgen05 mask-GEMM + statistic epilogue (k_maskgemm.cu) --------------------
struct GemmTest {
    int n_pad, n_x, n_y;
    int ncols;               // GEMM output columns: d_pad (planes) or n_pad (Gram form)
    int gram;                // 1: B = the Gram planes G' (k_gram.cu), epilogue reads mbits
    const uint32_t* mbits;   // Gram form: the launch's mask rows, one bit per pooled row
    int count;               // valid permutations of this test in the launch
    int tile0;               // first wave tile of this test (its tiles are contiguous)
    hap_align_info* info;
    hap_counts* counts;
    double* stats;           // optional, [count][3]
    const float2* ab;        // [d_pad] {2a, 2b}
    const double* sconst;    // {sum a^2, sum b^2, eps_rep}
};
struct GemmArgs {
    int d_pad, d;            // shared by the tests of a wave
    int G;
    GemmTest t[kMaxWave];
    int ntiles;              // wave tiles of rows_per_tile mask rows (row 0 = observed split)
    int npairs;              // CTA pairs (grid / pair_mode)
    const int4* pieces;      // {wave tile, col0, width, slot} in (tile, col0) order
    const int* piece_off;    // [npairs + 1] piece range of each pair
    const int* tile_npieces; // [ntiles] pieces (= partial slots) per tile
    int max_slots;           // partial slots per tile (stride)
    int rows_per_tile;       // 128 * pair_mode
    double tie_rel;
    float2* part;            // [ntiles][max_slots][rows_per_tile] piece partials {s1, s2}
    unsigned* tile_done;     // [ntiles] arrival tickets (zero between launches)
    int dyn;                 // 1: CTA pairs claim pieces from a global counter (dynamic)
    int npieces;             // pieces in the launch (dynamic mode: every kChunkN chunk)
    int* claim;              // [2] claim / exit counters (zero between launches)
    int* fq;                 // [4 + ntiles] finalize queue (zero between launches)
    int exp;                 // timing experiments only (HAP_K3_EXPERIMENT), 0 in production
    long long* stamps;       // exp bit 16: [grid][8 units][8 events] globaltimer
    unsigned long long* span;  // optional {first CTA entry, last CTA exit} globaltimer
};
// ---- Gram form (k_gram.cu) -----------------------------------
struct GramArgs {
    const uint16_t* zt_hi;   // [d_pad][n_pad] planes of hap_align
    const uint16_t* zt_lo;
    const float2* ab;        // [d_pad] {2a, 2b} of the plane epilogue
    int n_pad, d_pad;
    uint16_t* g_hi;          // [n_pad][n_pad] bf16 hi / lo of G' = Z' Z'^T
    uint16_t* g_lo;
    float2* gab;             // [n_pad] {2 a.z'_j, 2 b.z'_j}
    long long* gacc;         // [n_pad][n_pad] fixed-point accumulators (zero between uses)
    long long* gabacc;       // [n_pad][2]
    unsigned long long* span;
};
cudaError_t launch_gram(const GramArgs& g, int sm_count, cudaStream_t st);
// bf16 mask rows [rows][n_pad] -> bits [rows][n_pad / 32] (bit j % 32 of word j / 32)
cudaError_t launch_pack_bits(const uint16_t* mask, uint32_t* bits, int64_t rows, int n_pad, int sm_count,
                             cudaStream_t st);

// TMA descriptors of the wave's tests: mask (A), Zt hi / lo planes (B)
struct GemmMaps {
    CUtensorMap a[kMaxWave], bhi[kMaxWave], blo[kMaxWave];
};
int maskgemm_b_rows(int pair_mode);  // B tile rows per CTA (TMA box)
cudaError_t launch_maskgemm(const GemmMaps& maps, const GemmArgs& g, int pair_mode, cudaStream_t st);

}  // namespace hap
