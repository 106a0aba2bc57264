// hap_api.cu — host side of the C ABI declared in include/hap.h: context, workspace,
// TMA tensor maps, argument validation and the launch sequence of the hot path.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "hap_internal.h"

using namespace hap;

// batch lanes: two by default (HAP_LANES: 1..kMaxLanes, experiments)
constexpr int kMaxLanes = 3;

struct hap_ctx_s {
    int device = 0;
    int sm_count = 0;
    std::string err;
    cudaStream_t last_stream = nullptr;
    const hap_align_info* last_info = nullptr;
    // ---- workspace (grow-only)
    void* buf[40] = {};
    size_t cap[40] = {};
    size_t req[40] = {};  // checked build: bytes requested (guard bytes beyond, up to cap)
    // ---- state of the last successful hap_align
    bool aligned = false;
    bool gram_ok = false;  // the Gram planes of the current alignment are built (k_gram.cu)
    int last_gram = -1;    // K3 form of the last test planned on this context (1 = Gram)
    int64_t n_x = 0, n_y = 0, d = 0, n_pad = 0, d_pad = 0;
    // ---- TMA descriptors (valid for the current buffers/shape); tmA per mask slot
    CUtensorMap tmA[2]{}, tmBhi{}, tmBlo{};
    CUtensorMap tmGhi{}, tmGlo{};  // Gram planes (B operand of the Gram form)
    const void* tmg_key[2] = {};
    int64_t tmg_shape[2] = {};
    const void* tm_key[4] = {};
    int64_t tm_shape[5] = {};
    // ---- generator side stream: K2 only depends on (seed, s, b, N, n_x), so it runs on
    // `side` with no dependency on the caller's stream except the mask-GEMM that last read
    // the mask slot it overwrites; K3 joins it with an event wait
    cudaStream_t side = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_ready[2] = {}, ev_free[2] = {};
    // hap_permtest's mask-GEMM stream (highest priority): when a mask-GEMM ends, the next
    // block's mask-GEMM and the generator of the block after it become ready together, and
    // the block scheduler must place the GEMM's CTAs first
    cudaStream_t hi = nullptr;
    cudaEvent_t ev_hi[2] = {};
    int slot = 0;
    bool used[2] = {false, false};
    // batch pipeline: two lanes (internal streams forked from / joined to the caller's
    // stream), each with kMaxWave sub-contexts (own workspaces + generator streams)
    hap_ctx sub[kMaxLanes][kMaxWave] = {};
    cudaStream_t sub_stream[kMaxLanes] = {};
    cudaEvent_t ev_sub[kMaxLanes] = {};
    // host inputs: per lane a copy stream that stages a wave's rows as soon as the lane's
    // previous K1 (the last reader of the staging buffers) is done
    // (two staging buffers per workspace, alternating over the lane's waves)
    cudaStream_t cp_stream[kMaxLanes] = {};
    cudaEvent_t ev_k1done[kMaxLanes][2] = {}, ev_copied[kMaxLanes] = {};
    bool k1_recorded[kMaxLanes][2] = {};
    int lane_waves[kMaxLanes] = {};
    // cached K3 schedules: key {d_pad, npairs, (ntiles, n_pad) per test} -> offset (ints)
    // in buf[kSched]; new ones are staged in pinned host memory and copied on the stream
    struct Sched { std::vector<int64_t> key; int64_t off; int max_slots; };
    std::vector<Sched> sched;
    int64_t sched_used = 0;
    int* sched_host = nullptr;  // pinned staging, same size as buf[kSched]
    // ---- profiling
    bool prof = false;
    bool serial = false;  // profiling level 2: generator on the caller's stream
    bool stamp_k1 = false;  // profiling level 3: K1 phase timestamps
    struct Mark { cudaEvent_t a, b; int phase; };
    std::vector<Mark> marks;
    std::vector<cudaEvent_t> pool;
    int64_t launches[HAP_NUM_PHASES] = {};
    double ms[HAP_NUM_PHASES] = {};
    // kernel spans (hap_profile_spans): device {entry, exit} pairs, phase of each slot
    bool spans = false;
    std::vector<int> span_phase;
};

namespace {

enum Buf {
    kX = 0, kY, kNrm, kCoef, kPart, kXbar, kYbar, kU, kZhi, kZlo, kTpart, kT64, kAB, kMask,
    kM, kSconst, kGemmPart, kTileDone, kScal, kSpart, kScratch, kMask1, kInv, kStamps, kK3Stamps,
    kSched, kSpans, kX2, kY2, kClaim, kGhi, kGlo, kGab, kMbits, kMbits1, kGacc, kFinQ, kNumBufs
};

hap_status fail(hap_ctx c, hap_status s, const std::string& msg) {
    if (c) c->err = msg;
    return s;
}

hap_status cuda_fail(hap_ctx c, cudaError_t e, const char* what) {
    return fail(c, HAP_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// grow-only device buffer
hap_status ensure(hap_ctx c, int which, size_t bytes) {
    bytes = std::max<size_t>(bytes, 256);
    if (c->cap[which] >= bytes) {
#ifdef HAP_DEVICE_CHECKS
        c->req[which] = std::max(c->req[which], bytes);  // the guard starts past the largest request
#endif
        return HAP_OK;
    }
    if (c->buf[which]) {
        if (c->last_stream) cudaStreamSynchronize(c->last_stream);
        if (c->side) cudaStreamSynchronize(c->side);
        cudaFree(c->buf[which]);
        c->buf[which] = nullptr;
        c->cap[which] = 0;
    }
    size_t alloc = bytes + bytes / 4;
    cudaError_t e = cudaMalloc(&c->buf[which], alloc);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(c, HAP_E_OOM, std::string("cudaMalloc failed: ") + cudaGetErrorString(e));
    }
    // zero it and wait: the consumers run on non-blocking streams (lanes, generator, copies),
    // which the legacy-stream memset does not order (allocation is a slow path anyway)
    e = cudaMemset(c->buf[which], 0, alloc);
#ifdef HAP_DEVICE_CHECKS
    // guard bytes past the request: a kernel that writes beyond what its buffer was sized
    // for is reported by hap_debug_check_status
    if (e == cudaSuccess) e = cudaMemset(static_cast<char*>(c->buf[which]) + bytes, 0xA5, alloc - bytes);
    c->req[which] = bytes;
#endif
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return fail(c, HAP_E_CUDA, std::string("workspace zeroing: ") + cudaGetErrorString(e));
    c->cap[which] = alloc;
    return HAP_OK;
}

template <typename T>
T* B(hap_ctx c, int which) { return static_cast<T*>(c->buf[which]); }

bool is_device_ptr(const void* p) {
    cudaPointerAttributes at{};
    cudaError_t e = cudaPointerGetAttributes(&at, p);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q{};
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

// 2-D bf16 tensor map: inner dim `inner` (contiguous), `rows` rows, box {64, box_rows},
// 128-byte swizzle, out-of-bounds elements read as zero.
bool make_map(CUtensorMap* m, const void* base, uint64_t inner, uint64_t rows, uint32_t box_rows) {
    auto fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[2] = {inner, rows};
    cuuint64_t strides[1] = {inner * 2};
    cuuint32_t box[2] = {64, box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                    box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

int64_t mask_rows_cap(hap_ctx c) {
    return (int64_t)(std::min(c->cap[kMask], c->cap[kMask1]) / (size_t)(c->n_pad * 2));
}
// Zt planes are allocated with at least kChunkN rows so every TMA box fits the tensor
int64_t zt_rows(int64_t d_pad) { return std::max<int64_t>(d_pad, kChunkN); }

hap_status refresh_maps(hap_ctx c, int pair_mode) {
    const void* keys[4] = {c->buf[kMask], c->buf[kMask1], c->buf[kZhi], c->buf[kZlo]};
    const int64_t shape[5] = {c->n_pad, c->d_pad, mask_rows_cap(c), pair_mode, 0};
    if (std::equal(keys, keys + 4, c->tm_key) && std::equal(shape, shape + 5, c->tm_shape))
        return HAP_OK;
    const uint32_t box_b = (uint32_t)maskgemm_b_rows(pair_mode);
    const uint64_t zr = (uint64_t)zt_rows(c->d_pad);
    const uint64_t mr = (uint64_t)mask_rows_cap(c);
    if (!make_map(&c->tmA[0], c->buf[kMask], (uint64_t)c->n_pad, mr, kTileM) ||
        !make_map(&c->tmA[1], c->buf[kMask1], (uint64_t)c->n_pad, mr, kTileM) ||
        !make_map(&c->tmBhi, c->buf[kZhi], (uint64_t)c->n_pad, zr, box_b) ||
        !make_map(&c->tmBlo, c->buf[kZlo], (uint64_t)c->n_pad, zr, box_b))
        return fail(c, HAP_E_CUDA, "cuTensorMapEncodeTiled failed");
    std::copy(keys, keys + 4, c->tm_key);
    std::copy(shape, shape + 5, c->tm_shape);
    return HAP_OK;
}

// ---- Gram form (k_gram.cu) -----------
// The mask-GEMM multiplies the masks by the N_pad x N_pad Gram matrix of the centred cloud
// instead of the N_pad x d_pad planes.  Forced by HAP_FLAG_GRAM (n_pad <= kGramMaxNpad),
// refused by HAP_FLAG_NO_GRAM; otherwise chosen when the tensor time it saves (4 n_pad
// (d_pad - n_pad) FLOP per permutation at ~1.3 PFLOP/s) exceeds twice its set-up (the Gram
// kernel, ~n_pad^2 d_pad / 10^7 us, plus ~10 us).  The choice depends only on the test's
// shape, cfg->B (the whole test, not this call's shard) and the flags, so every shard of a
// test takes the same form.
constexpr int64_t kGramMaxNpad = 4096;

bool use_gram(hap_ctx w, const hap_perm_cfg* cfg) {
    if (cfg->flags & HAP_FLAG_NO_GRAM) return false;
    if (cfg->flags & HAP_FLAG_EXHAUSTIVE) return false;
    if (cfg->flags & HAP_FLAG_GRAM) return w->n_pad <= kGramMaxNpad;
    if (2 * w->n_pad > w->d_pad) return false;
    const double B = (double)(cfg->B ? cfg->B : cfg->b_end - cfg->b_begin);
    const double np = (double)w->n_pad, dp = (double)w->d_pad;
    const double save_us = B * 4.0 * np * (dp - np) / 1.3e9;
    const double cost_us = 10.0 + np * np * dp / 1e7;
    return save_us > 2.0 * cost_us;
}

// Gram planes of `w` (buffers and TMA descriptors; plan time) and their contents for the
// current alignment (built once per hap_align, on the wave's stream after the alignment)
hap_status ensure_gram(hap_ctx w, int pair_mode);
hap_status build_gram(hap_ctx w, cudaStream_t st);

// dynamic piece claiming (default): CTA pairs that start late beside the other lane's
// kernels take fewer pieces (C2 bench +2.7 %, C4 +3.6 % vs the static split);
// HAP_K3_DYNAMIC=0 restores the static balanced split (scheduling knob, same results)
int k3_dynamic() {
    static const char* dy = getenv("HAP_K3_DYNAMIC");
    return dy ? atoi(dy) : 1;
}
// dynamic mode piece width (HAP_K3_PIECE_COLS, scheduling knob; 256 = one accumulator chunk)
int64_t k3_piece_cols() {
    static const char* pw = getenv("HAP_K3_PIECE_COLS");
    return pw ? std::max<int64_t>(32, atoi(pw)) : kChunkN;
}
// partial slots per tile: one per piece (dynamic: d_pad / piece width; static: pieces are cut
// at multiples of 32 columns)
int64_t part_slots(hap_ctx, int64_t d_pad) {
    return std::max<int64_t>(1, ceil_div(d_pad, k3_dynamic() ? k3_piece_cols() : 32));
}

GemmArgs gemm_args(hap_ctx c) {
    GemmArgs g{};
    g.d_pad = (int)c->d_pad;
    g.d = (int)c->d;
    g.tie_rel = 1e-6;
#ifdef HAP_EXPERIMENTS
    // development build only (-DHAP_EXPERIMENTS): HAP_K3_EXPERIMENT bits 1, 2, 4, 8 skip
    // mask-GEMM work (timing only, the counts are then invalid), bit 16 records per-unit
    // timestamps; the release library has no such switch
    static const char* ex = getenv("HAP_K3_EXPERIMENT");
    g.exp = ex ? atoi(ex) : 0;
    static bool warned = false;
    if ((g.exp & 15) && !warned) {
        fprintf(stderr, "libhap: HAP_K3_EXPERIMENT=%d skips mask-GEMM work: timing only, results are invalid\n",
                g.exp);
        warned = true;
    }
#else
    g.exp = 0;
#endif
    g.dyn = k3_dynamic();
    g.claim = nullptr;
    if (g.dyn && ensure(c, kClaim, 64) == HAP_OK) g.claim = B<int>(c, kClaim);
    if (!g.claim) g.dyn = 0;
    g.stamps = nullptr;
    if ((g.exp & 16) && ensure(c, kK3Stamps, (size_t)c->sm_count * 64 * 8) == HAP_OK)
        g.stamps = B<long long>(c, kK3Stamps);
    return g;
}

// Balanced K3 schedule (see k_maskgemm.cu): every pair gets an equal contiguous range of
// the tile-major column space (multiples of 32), cut into pieces at tile boundaries and at
// 256 columns; slot = index of the piece within its tile.  Cached per shape; the device
// copy is stream-ordered after earlier launches on the same stream.
// A piece's K loop cannot run faster than the stage round trip (TMA + barrier latency over
// the 3-stage ring): measured ~0.49 us per stage, i.e. the MMA time of a ~196-column piece
// (K3 piece durations on B200: 15.7 us for widths 32..128, 20.5 us for 256).
constexpr double kPieceFloor = 4.0 * 196.0;

constexpr int64_t kSchedInts = 1 << 20;  // 4 MB schedule ring (device + pinned host staging)

hap_status reserve_schedule(hap_ctx c) {
    if (c->sched_host) return HAP_OK;
    hap_status s = ensure(c, kSched, (size_t)kSchedInts * sizeof(int));
    if (s) return s;
    if (cudaMallocHost(&c->sched_host, (size_t)kSchedInts * sizeof(int)) != cudaSuccess)
        return fail(c, HAP_E_OOM, "pinned schedule staging");
    return HAP_OK;
}

hap_status get_schedule(hap_ctx c, const GemmArgs& w, int np, cudaStream_t st, GemmArgs& g);

// stage a schedule blob in the pinned ring and copy it to the device on `st`
hap_status upload_schedule(hap_ctx c, const std::vector<int64_t>& key, const std::vector<int>& blob,
                           int max_slots, cudaStream_t st) {
    const int64_t need = (int64_t)blob.size();
    if (need > kSchedInts) return fail(c, HAP_E_INVALID_ARG, "K3 schedule too large");
    if (hap_status s = reserve_schedule(c)) return s;
    if (c->sched_used + need > kSchedInts) {  // wrap: the ring's old copies must have run
        if (c->last_stream) cudaStreamSynchronize(c->last_stream);
        cudaStreamSynchronize(st);
        c->sched.clear();
        c->sched_used = 0;
    }
    const int64_t at = c->sched_used;
    std::copy(blob.begin(), blob.end(), c->sched_host + at);
    cudaError_t e = cudaMemcpyAsync(B<int>(c, kSched) + at, c->sched_host + at, blob.size() * sizeof(int),
                                    cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return cuda_fail(c, e, "schedule upload");
    c->sched.push_back({key, at, max_slots});
    c->sched_used = at + round_up(need, 4);
    return HAP_OK;
}

hap_status get_schedule(hap_ctx c, const GemmArgs& w, int np, cudaStream_t st, GemmArgs& g) {
    std::vector<int64_t> key = {w.d_pad, np, w.dyn};
    for (int k = 0; k < w.G; ++k) {
        const int64_t nt = (k + 1 < w.G ? w.t[k + 1].tile0 : w.ntiles) - w.t[k].tile0;
        key.push_back(nt);
        key.push_back(w.t[k].n_pad);
        key.push_back(w.t[k].ncols);
    }
    const int64_t nt_all = w.ntiles;
    for (auto& e : c->sched)
        if (e.key == key) {
            const int* base = B<int>(c, kSched) + e.off;
            g.piece_off = base;
            g.tile_npieces = base + (np + 1);
            g.pieces = reinterpret_cast<const int4*>(base + round_up(np + 1 + nt_all, 4));
            g.max_slots = e.max_slots;
            return HAP_OK;  // (dyn: g.npieces is set by the caller)
        }
    // Piece cost model (cycles, measured on B200): per K-stage tensor-bound 4w (8 MMAs of
    // 128 x w/256 cycles) but never below the stage round-trip floor; a piece runs
    // n_pad/64 stages.  The 256-column chunks of every tile (test-major, tile-major) are cut
    // into np consecutive parts of cost <= M (a chunk is split at a multiple of 32 columns
    // only where a part ends inside it); M is the smallest feasible makespan (binary search).
    struct Chunk { int64_t width, nkb, tile, c0; };
    std::vector<Chunk> chunks;
    for (int k = 0; k < w.G; ++k) {
        const int64_t nt = (k + 1 < w.G ? w.t[k + 1].tile0 : w.ntiles) - w.t[k].tile0;
        for (int64_t t = 0; t < nt; ++t)
            for (int64_t c0 = 0; c0 < w.t[k].ncols; c0 += kChunkN)
                chunks.push_back({std::min<int64_t>(kChunkN, w.t[k].ncols - c0), w.t[k].n_pad / kKBlock,
                                  w.t[k].tile0 + t, c0});
    }
    auto cost = [](int64_t wd, int64_t nkb) { return (double)nkb * std::max(4.0 * (double)wd, kPieceFloor); };
    if (w.dyn) {  // dynamic: every chunk is a piece, claimed in (test, tile, column) order
        std::vector<int> npc(nt_all, 0), pcs;
        const int64_t pwidth = k3_piece_cols();
        for (const Chunk& ch : chunks)
            for (int64_t o = 0; o < ch.width; o += pwidth)
                pcs.insert(pcs.end(), {(int)ch.tile, (int)(ch.c0 + o), (int)std::min<int64_t>(pwidth, ch.width - o),
                                       npc[ch.tile]++});
        // claim order column-major inside groups of G tiles: the pairs running at once share
        // the B-plane columns in L2 while a group's mask tiles stay there for all its columns
        // (C3: B planes of 164 MB re-read ~76x per launch in tile order; 12.4 -> 12.0 ms per
        // test at G = 16, 12.1 at 8 and 32, 12.65 at 64; C2 / C4 unchanged).
        // HAP_K3_TILE_GROUP overrides (0: plain tile order)
        static const char* tg = getenv("HAP_K3_TILE_GROUP");
        const int G = tg ? atoi(tg) : 16;
        if (G > 0) {
            const size_t n4 = pcs.size() / 4;
            std::vector<size_t> idx(n4);
            for (size_t i = 0; i < n4; ++i) idx[i] = i;
            std::stable_sort(idx.begin(), idx.end(), [&](size_t x, size_t y) {
                const int gx = pcs[4 * x] / G, gy = pcs[4 * y] / G;
                if (gx != gy) return gx < gy;
                return pcs[4 * x + 1] < pcs[4 * y + 1];
            });
            std::vector<int> re;
            re.reserve(pcs.size());
            for (size_t i : idx) re.insert(re.end(), pcs.begin() + 4 * i, pcs.begin() + 4 * i + 4);
            pcs.swap(re);
        }
        std::vector<int> blob(round_up(np + 1 + nt_all, 4), 0);
        std::copy(npc.begin(), npc.end(), blob.begin() + (np + 1));
        blob.insert(blob.end(), pcs.begin(), pcs.end());
        int max_slots = 1;
        for (int v : npc) max_slots = std::max(max_slots, v);
        if (hap_status s = upload_schedule(c, key, blob, max_slots, st)) return s;
        return get_schedule(c, w, np, st, g);
    }
    auto fill = [&](double M, std::vector<int>* out_pcs, std::vector<int>* out_off,
                    std::vector<int>* out_npc) {
        size_t ci = 0;
        int64_t done = 0;
        for (int p = 0; p < np; ++p) {
            if (out_off) (*out_off)[p] = (int)(out_pcs->size() / 4);
            double used = 0.0;
            while (ci < chunks.size()) {
                const Chunk& ch = chunks[ci];
                const int64_t left = ch.width - done;
                int64_t wd = left;
                if (used + cost(left, ch.nkb) > M) {
                    wd = 0;
                    for (int64_t cand = 32; cand < left; cand += 32)
                        if (used + cost(cand, ch.nkb) <= M) wd = cand;
                    if (wd == 0) break;
                }
                if (out_pcs)
                    out_pcs->insert(out_pcs->end(), {(int)ch.tile, (int)(ch.c0 + done), (int)wd,
                                                     (*out_npc)[ch.tile]++});
                used += cost(wd, ch.nkb);
                done += wd;
                if (done == ch.width) {
                    ++ci;
                    done = 0;
                }
            }
        }
        return ci == chunks.size();
    };
    double lo = 0.0, hi = 1.0;
    for (const Chunk& ch : chunks) hi += cost(ch.width, ch.nkb);
    for (int it = 0; it < 40; ++it) {
        const double mid = 0.5 * (lo + hi);
        if (fill(mid, nullptr, nullptr, nullptr)) hi = mid;
        else lo = mid;
    }
    std::vector<int> off(np + 1, 0), npc(nt_all, 0), pcs;
    // EXPERIMENT: list schedule of the whole chunks in (test, tile, chunk) order, each to the
    // least loaded pair (round-robin for equal costs: a tile's chunks run at the same time on
    // neighbouring pairs).  It reads the masks from DRAM exactly once even from a cold L2,
    // but measured 19 % slower than the contiguous balanced schedule (the default below).
    std::vector<double> load(np, 0.0);
    std::vector<std::vector<int>> per(np);
    for (const Chunk& ch : chunks) {
        int best = 0;
        for (int p = 1; p < np; ++p)
            if (load[p] < load[best]) best = p;
        load[best] += cost(ch.width, ch.nkb);
        per[best].push_back((int)(&ch - chunks.data()));
    }
    const double list_ms = *std::max_element(load.begin(), load.end());
    static const char* rr = getenv("HAP_K3_ROUND_ROBIN");  // measured slower on B200 (kept
    if (rr && atoi(rr) && list_ms <= 1.05 * hi) {           // for experiments only)
        for (int p = 0; p < np; ++p) {
            off[p] = (int)(pcs.size() / 4);
            for (int ci : per[p]) {
                const Chunk& ch = chunks[ci];
                pcs.insert(pcs.end(), {(int)ch.tile, (int)ch.c0, (int)ch.width, 0});
            }
        }
        // slots: index of the piece within its tile, in (tile, column) order
        std::vector<std::pair<int64_t, int>> order;  // (tile * d_pad + c0, piece index)
        for (size_t k = 0; k < pcs.size() / 4; ++k)
            order.push_back({(int64_t)pcs[4 * k] * 65536 + pcs[4 * k + 1], (int)k});
        std::sort(order.begin(), order.end());
        for (auto& o : order) pcs[4 * o.second + 3] = npc[pcs[4 * o.second]]++;
    } else {
        fill(hi, &pcs, &off, &npc);
    }
    off[np] = (int)(pcs.size() / 4);
    int max_slots = 1;
    for (int v : npc) max_slots = std::max(max_slots, v);
    std::vector<int> blob(round_up(np + 1 + nt_all, 4), 0);
    std::copy(off.begin(), off.end(), blob.begin());
    std::copy(npc.begin(), npc.end(), blob.begin() + (np + 1));
    blob.insert(blob.end(), pcs.begin(), pcs.end());
    if (hap_status s = upload_schedule(c, key, blob, max_slots, st)) return s;
    return get_schedule(c, w, np, st, g);
}

// bytes of bf16 mask per launch: large enough that a C4-sized test (N = 10^4, B = 10^4)
// is one block and joins a wave (C4 sample 121.9 -> 117.5 us/test vs 64 MB), and that a
// C3 block gives every K3 pair ~45 pieces, so the last-piece tail is short (C3 12.9 /
// 12.5 / 12.4 / 12.45 ms per test at 256 / 512 / 1024 / 2048 MB); K3 streams the masks
// with TMA and is not DRAM-bound, so they need not stay in L2.  A worker holds two such
// blocks (2 GB) only when a test's masks are that large.
constexpr int64_t kMaskBudget = 1024ll << 20;
constexpr int64_t kMaxBlockTiles = 4096;

cudaEvent_t take_event(hap_ctx c) {
    if (!c->pool.empty()) {
        cudaEvent_t e = c->pool.back();
        c->pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

// Brackets the launches issued in its scope: counts them and, when profiling is on,
// records a start/stop event pair on the launching stream.
struct PhaseScope {
    hap_ctx c;
    int phase;
    int nlaunch;
    cudaStream_t st;
    cudaEvent_t a = nullptr;
    PhaseScope(hap_ctx c_, int phase_, int nlaunch_, cudaStream_t st_)
        : c(c_), phase(phase_), nlaunch(nlaunch_), st(st_) {
        if (c->prof) {
            a = take_event(c);
            cudaEventRecord(a, st);
        }
    }
    ~PhaseScope() {
        c->launches[phase] += nlaunch;
        if (a) {
            cudaEvent_t b = take_event(c);
            cudaEventRecord(b, st);
            c->marks.push_back({a, b, phase});
        }
    }
};

constexpr int64_t kMaxSpans = 8192;

hap_status reset_spans(hap_ctx c) {
    hap_status s = ensure(c, kSpans, (size_t)kMaxSpans * 16);
    if (s) return s;
    std::vector<unsigned long long> init(2 * kMaxSpans);
    for (int64_t i = 0; i < kMaxSpans; ++i) {
        init[2 * i] = ~0ull;
        init[2 * i + 1] = 0ull;
    }
    cudaError_t e = cudaMemcpy(c->buf[kSpans], init.data(), init.size() * 8, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return cuda_fail(c, e, "span reset");
    c->span_phase.clear();
    return HAP_OK;
}

// device slot for the next launch of `phase` (nullptr when span profiling is off / full)
unsigned long long* next_span(hap_ctx c, int phase) {
    if (!c->spans || (int64_t)c->span_phase.size() >= kMaxSpans) return nullptr;
    c->span_phase.push_back(phase);
    return B<unsigned long long>(c, kSpans) + 2 * (c->span_phase.size() - 1);
}

}  // namespace

extern "C" {

int hap_abi_version(void) { return HAP_ABI_VERSION; }

hap_status hap_create(int device, hap_ctx* out) {
    if (!out) return HAP_E_INVALID_ARG;
    *out = nullptr;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || device < 0 || device >= n) {
        cudaGetLastError();
        return HAP_E_INVALID_ARG;
    }
    cudaDeviceProp prop{};
    if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return HAP_E_CUDA;
    if (prop.major != 10 || prop.minor != 0) return HAP_E_UNSUPPORTED_ARCH;
    hap_ctx c = new (std::nothrow) hap_ctx_s();
    if (!c) return HAP_E_OOM;
    c->device = device;
    c->sm_count = prop.multiProcessorCount;
    cudaSetDevice(device);
    // K1 scratch words: no ZeroVector row seen yet, tickets at zero
    if (ensure(c, kScratch, 64) != HAP_OK) {
        delete c;
        return HAP_E_OOM;
    }
    if (cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming) != cudaSuccess) {
        hap_destroy(c);
        return HAP_E_CUDA;
    }
    for (int i = 0; i < 2; ++i)
        if (cudaEventCreateWithFlags(&c->ev_ready[i], cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&c->ev_free[i], cudaEventDisableTiming) != cudaSuccess) {
            hap_destroy(c);
            return HAP_E_CUDA;
        }
    const long long init[2] = {0x7fffffffffffffffll, 0};
    if (cudaMemcpy(c->buf[kScratch], init, sizeof init, cudaMemcpyHostToDevice) != cudaSuccess) {
        hap_destroy(c);
        return HAP_E_CUDA;
    }
    *out = c;
    return HAP_OK;
}

hap_status hap_destroy(hap_ctx c) {
    if (!c) return HAP_E_INVALID_ARG;
    cudaSetDevice(c->device);
    if (c->last_stream) cudaStreamSynchronize(c->last_stream);
    for (void* p : c->buf)
        if (p) cudaFree(p);
    for (auto& m : c->marks) {
        cudaEventDestroy(m.a);
        cudaEventDestroy(m.b);
    }
    for (auto e : c->pool) cudaEventDestroy(e);
    if (c->side) {
        cudaStreamSynchronize(c->side);
        cudaStreamDestroy(c->side);
    }
    if (c->sched_host) cudaFreeHost(c->sched_host);
    for (int i = 0; i < kMaxLanes; ++i) {
        for (int k = 0; k < kMaxWave; ++k)
            if (c->sub[i][k]) hap_destroy(c->sub[i][k]);
        if (c->sub_stream[i]) cudaStreamDestroy(c->sub_stream[i]);
        if (c->ev_sub[i]) cudaEventDestroy(c->ev_sub[i]);
        if (c->cp_stream[i]) cudaStreamDestroy(c->cp_stream[i]);
        for (int b = 0; b < 2; ++b)
            if (c->ev_k1done[i][b]) cudaEventDestroy(c->ev_k1done[i][b]);
        if (c->ev_copied[i]) cudaEventDestroy(c->ev_copied[i]);
    }
    if (c->ev_fork) cudaEventDestroy(c->ev_fork);
    if (c->hi) cudaStreamDestroy(c->hi);
    for (auto e : c->ev_hi)
        if (e) cudaEventDestroy(e);
    for (int i = 0; i < 2; ++i) {
        if (c->ev_ready[i]) cudaEventDestroy(c->ev_ready[i]);
        if (c->ev_free[i]) cudaEventDestroy(c->ev_free[i]);
    }
    delete c;
    return HAP_OK;
}

const char* hap_last_error(hap_ctx c) { return c ? c->err.c_str() : "null context"; }

hap_status hap_sync(hap_ctx c) {
    if (!c) return HAP_E_INVALID_ARG;
    cudaSetDevice(c->device);
    cudaError_t e = c->last_stream ? cudaStreamSynchronize(c->last_stream) : cudaDeviceSynchronize();
    if (e != cudaSuccess) return cuda_fail(c, e, "hap_sync");
    if (c->last_info) {
        hap_align_info h{};
        e = cudaMemcpy(&h, c->last_info, sizeof(h), cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) return cuda_fail(c, e, "hap_sync info");
        if (h.status != HAP_OK) {
            char msg[160];
            snprintf(msg, sizeof msg, "data error %d (bad_row %lld)", h.status, (long long)h.bad_row);
            return fail(c, (hap_status)h.status, msg);
        }
    }
    return HAP_OK;
}

double hap_pvalue(uint64_t exceed, uint64_t Bn) { return (1.0 + (double)exceed) / ((double)Bn + 1.0); }

double hap_p_exact(uint64_t exceed, uint64_t total) {
    return total ? (double)exceed / (double)total : __builtin_nan("");
}

}  // extern "C"

namespace {

// Workspace of one pair in `c` (grow-only), host inputs staged on the stream; fills the
// pair's K1 arguments and records the pair's shape in the context.
// Grow-only workspace for pairs of up to N pooled rows in d dimensions and waves of up to
// `tiles` mask tiles of R rows (owner buffers included): allocating (and zeroing) buffers
// synchronises, so the batch reserves every workspace before its first launch.
hap_status ensure_gram(hap_ctx w, int pair_mode) {
    const int64_t n_pad = w->n_pad, rows = zt_rows(n_pad);
    hap_status s;
    if ((s = ensure(w, kGhi, (size_t)rows * n_pad * 2)) || (s = ensure(w, kGlo, (size_t)rows * n_pad * 2)) ||
        (s = ensure(w, kGab, (size_t)n_pad * 8)) ||
        (s = ensure(w, kGacc, (size_t)n_pad * n_pad * 8 + (size_t)n_pad * 16)))
        return s;
    const void* keys[2] = {w->buf[kGhi], w->buf[kGlo]};
    const int64_t shape[2] = {n_pad, pair_mode};
    if (!std::equal(keys, keys + 2, w->tmg_key) || !std::equal(shape, shape + 2, w->tmg_shape)) {
        const uint32_t box_b = (uint32_t)maskgemm_b_rows(pair_mode);
        if (!make_map(&w->tmGhi, w->buf[kGhi], (uint64_t)n_pad, (uint64_t)rows, box_b) ||
            !make_map(&w->tmGlo, w->buf[kGlo], (uint64_t)n_pad, (uint64_t)rows, box_b))
            return fail(w, HAP_E_CUDA, "cuTensorMapEncodeTiled failed (Gram planes)");
        std::copy(keys, keys + 2, w->tmg_key);
        std::copy(shape, shape + 2, w->tmg_shape);
    }
    return HAP_OK;
}

hap_status build_gram(hap_ctx w, cudaStream_t st) {
    const int64_t n_pad = w->n_pad;
    if (!w->gram_ok) {
        GramArgs ga{};
        ga.zt_hi = B<uint16_t>(w, kZhi);
        ga.zt_lo = B<uint16_t>(w, kZlo);
        ga.ab = B<float2>(w, kAB);
        ga.n_pad = (int)n_pad;
        ga.d_pad = (int)w->d_pad;
        ga.g_hi = B<uint16_t>(w, kGhi);
        ga.g_lo = B<uint16_t>(w, kGlo);
        ga.gab = B<float2>(w, kGab);
        ga.gacc = B<long long>(w, kGacc);
        ga.gabacc = ga.gacc + n_pad * n_pad;
        ga.span = next_span(w, HAP_PHASE_ALIGN);
        cudaError_t e;
        {
            PhaseScope ps(w, HAP_PHASE_ALIGN, 2, st);
            e = launch_gram(ga, w->sm_count, st);
        }
        if (e != cudaSuccess) return cuda_fail(w, e, "Gram kernel");
        w->gram_ok = true;
    }
    return HAP_OK;
}

hap_status reserve_pair(hap_ctx c, int64_t N, int64_t d, int64_t tiles, int64_t R, bool owner) {
    const int64_t n_pad = round_up(N, kKBlock), d_pad = round_up(d, 32);
    hap_status s;
    if (owner &&  // only a wave's owner (its first workspace) holds the launch's piece partials
        ((s = ensure(c, kGemmPart, (size_t)kMaxWave * tiles * part_slots(c, d_pad) * R * sizeof(float2))) ||
         (s = ensure(c, kTileDone, (size_t)kMaxWave * tiles * sizeof(unsigned)))))
        return s;
    if ((s = ensure(c, kXbar, d * 8)) || (s = ensure(c, kYbar, d * 8)) ||
        (s = ensure(c, kInv, N * 8)) || (s = ensure(c, kCoef, n_pad * 8)) ||
        (s = ensure(c, kU, d_pad * 8)) ||
        (s = ensure(c, kZhi, (size_t)zt_rows(d_pad) * n_pad * 2)) ||
        (s = ensure(c, kZlo, (size_t)zt_rows(d_pad) * n_pad * 2)) ||
        (s = ensure(c, kTpart, (size_t)(2 * d + d_pad) * 8)) ||
        (s = ensure(c, kT64, d_pad * 8)) || (s = ensure(c, kAB, d_pad * 8)) ||
        (s = ensure(c, kM, d_pad * 8)) || (s = ensure(c, kSconst, 32)) ||
        (s = ensure(c, kMask, (size_t)std::max<int64_t>(2, tiles) * R * n_pad * 2)) ||
        (s = ensure(c, kMask1, (size_t)std::max<int64_t>(2, tiles) * R * n_pad * 2)) ||
        (s = reserve_schedule(c)))
        return s;
    return HAP_OK;
}

// host inputs are copied on `cp` (default: st)
hap_status prepare_pair_cp(hap_ctx c, const float* X, int64_t n_x, const float* Y, int64_t n_y, int64_t d,
                           hap_align_info* info, cudaStream_t st, AlignPair& q, cudaStream_t cp = nullptr,
                           int buf = 0) {
    const int bX = buf ? kX2 : kX, bY = buf ? kY2 : kY;
    if (!X || !Y || !info) return fail(c, HAP_E_INVALID_ARG, "null pointer");
    if (n_x < 1 || n_y < 1 || n_x + n_y > 65535)
        return fail(c, HAP_E_INVALID_ARG, "need 1 <= n_x, n_y and n_x + n_y <= 65535");
    if (d < 2 || d > 16384) return fail(c, HAP_E_DIM_MISMATCH, "need 2 <= d <= 16384");
    if (!is_device_ptr(info)) return fail(c, HAP_E_INVALID_ARG, "info must be device memory");
    const int64_t N = n_x + n_y;
    const int64_t n_pad = round_up(N, kKBlock);
    const int64_t d_pad = round_up(d, 32);
    hap_status s;
    if ((s = ensure(c, kXbar, d * 8)) || (s = ensure(c, kYbar, d * 8)) ||
        (s = ensure(c, kInv, N * 8)) || (s = ensure(c, kCoef, n_pad * 8)) ||
        (s = ensure(c, kU, d_pad * 8)) ||
        (s = ensure(c, kZhi, (size_t)zt_rows(d_pad) * n_pad * 2)) ||
        (s = ensure(c, kZlo, (size_t)zt_rows(d_pad) * n_pad * 2)) ||
        (s = ensure(c, kTpart, (size_t)(2 * d + d_pad) * 8)) ||
        (s = ensure(c, kT64, d_pad * 8)) || (s = ensure(c, kAB, d_pad * 8)) ||
        (s = ensure(c, kM, d_pad * 8)) || (s = ensure(c, kSconst, 32)) ||
        (s = ensure(c, kMask, (size_t)2 * kTileM * n_pad * 2)))
        return s;
    // host inputs are staged into the context (copied on `stream`)
    const float* dX = X;
    const float* dY = Y;
    if (!is_device_ptr(X)) {
        if ((s = ensure(c, bX, (size_t)n_x * d * 4))) return s;
        cudaError_t e = cudaMemcpyAsync(c->buf[bX], X, (size_t)n_x * d * 4, cudaMemcpyHostToDevice, cp ? cp : st);
        if (e != cudaSuccess) return cuda_fail(c, e, "H2D X");
        dX = B<float>(c, bX);
    }
    if (!is_device_ptr(Y)) {
        if ((s = ensure(c, bY, (size_t)n_y * d * 4))) return s;
        cudaError_t e = cudaMemcpyAsync(c->buf[bY], Y, (size_t)n_y * d * 4, cudaMemcpyHostToDevice, cp ? cp : st);
        if (e != cudaSuccess) return cuda_fail(c, e, "H2D Y");
        dY = B<float>(c, bY);
    }
    c->n_x = n_x;
    c->n_y = n_y;
    c->d = d;
    c->n_pad = n_pad;
    c->d_pad = d_pad;
    q = AlignPair{};
    q.X = dX;
    q.Y = dY;
    q.n_x = n_x;
    q.n_y = n_y;
    q.d = d;
    q.n_pad = n_pad;
    q.info = info;
    q.inv = B<double>(c, kInv);
    q.coef = B<float2>(c, kCoef);
    q.u = B<double>(c, kU);
    q.xbar = B<double>(c, kXbar);
    q.ybar = B<double>(c, kYbar);
    q.zt_hi = B<uint16_t>(c, kZhi);
    q.zt_lo = B<uint16_t>(c, kZlo);
    q.m = B<double>(c, kM);
    q.t64 = B<double>(c, kT64);
    q.ab = B<float2>(c, kAB);
    q.sconst = B<double>(c, kSconst);
    q.acc = B<long long>(c, kTpart);
    q.bad = B<long long>(c, kScratch);  // word 0 of the pair's own scratch
    return HAP_OK;
}

hap_status prepare_pair(hap_ctx c, const float* X, int64_t n_x, const float* Y, int64_t n_y, int64_t d,
                        hap_align_info* info, cudaStream_t st, AlignPair& q) {
    return prepare_pair_cp(c, X, n_x, Y, n_y, d, info, st, q);
}
// ONE K1 launch aligning G pairs (each in its own workspace ws[k]); `owner` (= ws[0])
// provides the launch's barrier / ticket words and the profiling records.
hap_status align_wave(hap_ctx owner, int G, hap_ctx* ws, const AlignPair* pairs, hap_align_mode mode,
                      cudaStream_t st, const PermArgs* draws = nullptr) {
    AlignArgs a{};
    if (draws) {
        a.do_draws = 1;
        a.draws = *draws;
        a.draws.split = 1;
    }
    a.G = G;
    for (int k = 0; k < G; ++k) {
        a.p[k] = pairs[k];
        if (pairs[k].d != pairs[0].d) return fail(owner, HAP_E_DIM_MISMATCH, "wave pairs differ in d");
    }
    a.d = pairs[0].d;
    a.d_pad = round_up(a.d, 32);
    a.mode = mode;
    a.scratch = B<long long>(owner, kScratch);
    a.stamps = nullptr;
    if (owner->stamp_k1 && ensure(owner, kStamps, (size_t)(8 + 8 * 4 * owner->sm_count) * 8) == HAP_OK)
        a.stamps = B<long long>(owner, kStamps);
    align_items(a);
    a.span = next_span(owner, HAP_PHASE_ALIGN);
    cudaError_t e;
    {
        PhaseScope ps(owner, HAP_PHASE_ALIGN, align_launch_count(a), st);
        e = launch_align(a, owner->sm_count, st);
    }
    if (e != cudaSuccess) return cuda_fail(owner, e, "align kernel");
    for (int k = 0; k < G; ++k) {
        ws[k]->aligned = true;
        ws[k]->gram_ok = false;
        ws[k]->last_stream = st;
        ws[k]->last_info = pairs[k].info;
    }
    return HAP_OK;
}

}  // namespace

extern "C" {

hap_status hap_align(hap_ctx c, const float* X, int64_t n_x, const float* Y, int64_t n_y, int64_t d,
                     hap_align_mode mode, hap_align_info* info, void* stream) {
    if (!c) return HAP_E_INVALID_ARG;
    if (mode != HAP_ALIGN_HOUSEHOLDER && mode != HAP_ALIGN_NONE)
        return fail(c, HAP_E_INVALID_ARG, "bad mode");
    cudaSetDevice(c->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    AlignPair q;
    hap_status s = prepare_pair(c, X, n_x, Y, n_y, d, info, st, q);
    if (s) return s;
    return align_wave(c, 1, &c, &q, mode, st);
}

}  // extern "C"

namespace {

// One test's share of a wave: permutations [b_begin, b_begin + cnt) of an aligned workspace.
struct WaveTest {
    hap_ctx w;
    hap_align_info* info;
    const hap_perm_cfg* cfg;
    hap_counts* counts;
    double* stats;       // rows of this block (already offset), or null
    uint64_t b_begin;
    int64_t cnt;
};

// ONE generator launch (K2) and ONE mask-GEMM launch (K3) for G tests.  `owner` holds the
// wave buffers (piece partials, tile tickets, schedule) and the generator side stream; each
// test's masks go to the next mask slot of its own workspace, which K2 rewrites only after
// the K3 that last read it (event), so K2 can overlap earlier work of other streams.
// Arguments of a wave's K2 and K3 launches; picks (and toggles) each test's mask slot.
struct WavePlan {
    GemmArgs g;
    GemmMaps maps;
    PermArgs pa;
    int slots[kMaxWave];
    int npairs;
};

hap_status plan_wave(hap_ctx owner, int G, const WaveTest* T, int pair, bool shared, WavePlan& P) {
    const int64_t R = (int64_t)kTileM * pair;  // mask rows per tile; row 0 = observed split
    P.npairs = owner->sm_count / pair;
    P.g = gemm_args(owner);
    P.pa = PermArgs{};
    GemmArgs& g = P.g;
    PermArgs& pa = P.pa;
    pa.G = G;
    pa.out_kind = kMaskBf16Row;
    pa.rows_per_tile = (int)R;
    {
        static const char* cap = getenv("HAP_K2_MAX_CTAS");  // scheduling experiments
        pa.max_ctas_per_sm = cap ? atoi(cap) : 0;
    }
    g.G = G;
    g.rows_per_tile = (int)R;
    g.tie_rel = T[0].cfg->tie_rel > 0 ? T[0].cfg->tie_rel : 1e-6;
    int64_t tiles = 0, max_cols = 0;
    hap_status s;
    for (int k = 0; k < G; ++k) {
        hap_ctx w = T[k].w;
        if (w->d_pad != owner->d_pad) return fail(owner, HAP_E_DIM_MISMATCH, "wave tests differ in d");
        const int64_t nt = std::max<int64_t>(1, ceil_div(T[k].cnt, R - 1));
        if ((s = ensure(w, kMask, (size_t)nt * R * w->n_pad * 2)) ||
            (s = ensure(w, kMask1, (size_t)nt * R * w->n_pad * 2)) || (s = refresh_maps(w, pair)))
            return s == HAP_OK ? s : fail(owner, s, w->err);
        // shared masks: every test reads test 0's block (same N, n_x, stream, b-range)
        P.slots[k] = (shared && k > 0) ? P.slots[0] : w->slot;
        if (!(shared && k > 0)) w->slot ^= 1;
        PermTest& pt = pa.t[k];
        pt.seed = T[k].cfg->seed;
        pt.s = T[k].cfg->stream_id;
        pt.b_begin = T[k].b_begin;
        pt.count = T[k].cnt;
        pt.N = w->n_x + w->n_y;
        pt.n_x = w->n_x;
        pt.n_pad = w->n_pad;
        pt.out = w->buf[P.slots[k] ? kMask1 : kMask];
        pt.ntiles = (int)nt;
        pt.exhaustive = (T[k].cfg->flags & HAP_FLAG_EXHAUSTIVE) ? 1 : 0;
        GemmTest& gt = g.t[k];
        gt.gram = use_gram(w, T[k].cfg) ? 1 : 0;
        w->last_gram = gt.gram;
        gt.ncols = gt.gram ? (int)w->n_pad : (int)w->d_pad;
        gt.mbits = nullptr;
        if (gt.gram) {
            // the mask owner's bit rows (test 0's with shared masks), packed after K2
            hap_ctx mo = (shared && k > 0) ? T[0].w : w;
            const int mb = P.slots[k] ? kMbits1 : kMbits;
            if ((s = ensure(mo, mb, (size_t)nt * R * (mo->n_pad / 8))) || (s = ensure_gram(w, pair)))
                return s == HAP_OK ? s : fail(owner, s, w->err + mo->err);
            gt.mbits = B<uint32_t>(mo, mb);
        }
        gt.n_pad = (int)w->n_pad;
        gt.n_x = (int)w->n_x;
        gt.n_y = (int)w->n_y;
        gt.count = (int)T[k].cnt;
        gt.tile0 = (int)tiles;
        gt.info = T[k].info;
        gt.counts = T[k].counts;
        gt.stats = T[k].stats;
        gt.ab = B<float2>(w, gt.gram ? kGab : kAB);
        gt.sconst = B<double>(w, kSconst);
        P.maps.a[k] = shared ? T[0].w->tmA[P.slots[0]] : w->tmA[P.slots[k]];
        P.maps.bhi[k] = gt.gram ? w->tmGhi : w->tmBhi;
        P.maps.blo[k] = gt.gram ? w->tmGlo : w->tmBlo;
        max_cols = std::max<int64_t>(max_cols, gt.ncols);
        tiles += nt;
    }
    if (shared) pa.G = 1;  // one generated block serves the whole wave
    perm_items(pa);
    g.ntiles = (int)tiles;
    g.npairs = P.npairs;
    {  // dynamic mode: every piece (a chunk, or HAP_K3_PIECE_COLS columns of it)
        const int64_t pwidth = k3_piece_cols();
        int64_t np_all = 0;
        for (int k = 0; k < G; ++k) {
            int64_t per_tile = 0;
            for (int64_t c0 = 0; c0 < g.t[k].ncols; c0 += kChunkN)
                per_tile += ceil_div(std::min<int64_t>(kChunkN, g.t[k].ncols - c0), pwidth);
            np_all += (int64_t)pa.t[k].ntiles * per_tile;
        }
        g.npieces = (int)np_all;
        // dynamic claiming needs no fixed split: a small wave launches only as many CTA
        // pairs as it has pieces (less setup and teardown for C1-sized tests)
        if (g.dyn && g.npieces < P.npairs) P.npairs = g.npairs = std::max(1, g.npieces);
    }
    if ((s = ensure(owner, kGemmPart, (size_t)tiles * part_slots(owner, max_cols) * R * sizeof(float2))) ||
        (s = ensure(owner, kTileDone, (size_t)tiles * sizeof(unsigned))) ||
        (s = ensure(owner, kFinQ, (size_t)(4 + tiles) * sizeof(int))))
        return s;
    g.fq = B<int>(owner, kFinQ);
    g.part = B<float2>(owner, kGemmPart);
    g.tile_done = B<unsigned>(owner, kTileDone);
    return HAP_OK;
}

// K2 (fused, split over `light`, or - `staged` - only the table pass after K1 staged the
// draws on `st`) and K3 of a planned wave.
hap_status launch_wave(hap_ctx owner, const WaveTest* T, int pair, cudaStream_t st, WavePlan& P,
                       cudaStream_t light = nullptr, bool staged = false) {
    PermArgs& pa = P.pa;
    GemmArgs& g = P.g;
    const int* slots = P.slots;
    hap_status s;
    cudaError_t e = cudaSuccess;
    if (staged) {
        // K1 (on st) staged the draws: the table pass waits for it on the side stream
        cudaStream_t gs = owner->serial ? st : owner->side;
        if (gs != st) {
            e = cudaEventRecord(owner->ev_ready[1], st);
            if (e == cudaSuccess) e = cudaStreamWaitEvent(gs, owner->ev_ready[1], 0);
        }
        if (e == cudaSuccess) {
            pa.split = 2;
            pa.span = next_span(owner, HAP_PHASE_PERMGEN);
            PhaseScope ps(owner, HAP_PHASE_PERMGEN, 1, gs);
            e = launch_perm(pa, owner->sm_count, gs);
        }
        if (e == cudaSuccess && gs != st) e = cudaEventRecord(owner->ev_ready[0], gs);
        if (e == cudaSuccess && gs != st) e = cudaStreamWaitEvent(st, owner->ev_ready[0], 0);
        if (e != cudaSuccess) return cuda_fail(owner, e, "perm generator");
    } else if (light && light != st && perm_can_split(pa)) {
        // split generator: K2a (draws, register-only) on the light stream, where it runs
        // beside the other wave's mask-GEMM for free; K2b (table, chains, rows) on `st`,
        // i.e. never beside a mask-GEMM (both lean on shared-memory bandwidth)
        for (int k = 0; k < pa.G && e == cudaSuccess; ++k)
            if (T[k].w->used[slots[k]]) e = cudaStreamWaitEvent(light, T[k].w->ev_free[slots[k]], 0);
        PermArgs d = pa;
        d.split = 1;
        if (e == cudaSuccess) e = launch_perm(d, owner->sm_count, light);
        if (e == cudaSuccess) e = cudaEventRecord(owner->ev_ready[0], light);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(st, owner->ev_ready[0], 0);
        if (e == cudaSuccess) {
            pa.split = 2;
            pa.span = next_span(owner, HAP_PHASE_PERMGEN);
            PhaseScope ps(owner, HAP_PHASE_PERMGEN, 2, st);
            e = launch_perm(pa, owner->sm_count, st);
        }
        if (e != cudaSuccess) return cuda_fail(owner, e, "perm generator");
    } else {
        // K2 on the side stream: each test's slot is rewritten only after the K3 that read it
        // (on `st` itself when serialised or when the caller passed its light stream as st)
        cudaStream_t gs = (owner->serial || (light && light == st)) ? st : owner->side;
        for (int k = 0; k < pa.G && e == cudaSuccess && !owner->serial; ++k)
            if (T[k].w->used[slots[k]]) e = cudaStreamWaitEvent(gs, T[k].w->ev_free[slots[k]], 0);
        if (e == cudaSuccess) {
            pa.span = next_span(owner, HAP_PHASE_PERMGEN);
            PhaseScope ps(owner, HAP_PHASE_PERMGEN, 1, gs);
            e = launch_perm(pa, owner->sm_count, gs);
        }
        if (e == cudaSuccess) e = cudaEventRecord(owner->ev_ready[0], gs);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(st, owner->ev_ready[0], 0);  // join
        if (e != cudaSuccess) return cuda_fail(owner, e, "perm generator");
    }
    for (int k = 0; k < g.G; ++k)  // Gram form: G' of each test's current alignment
        if (g.t[k].gram && (s = build_gram(T[k].w, st))) return fail(owner, s, T[k].w->err);
    for (int k = 0; k < pa.G && e == cudaSuccess; ++k) {  // Gram form: bit rows of the masks
        if (!g.t[k].gram) continue;
        PhaseScope ps(owner, HAP_PHASE_PERMGEN, 1, st);
        e = launch_pack_bits(static_cast<const uint16_t*>(pa.t[k].out), const_cast<uint32_t*>(g.t[k].mbits),
                             (int64_t)pa.t[k].ntiles * P.g.rows_per_tile, (int)pa.t[k].n_pad, owner->sm_count, st);
    }
    if (e != cudaSuccess) return cuda_fail(owner, e, "mask bits");
    if ((s = get_schedule(owner, g, P.npairs, st, g))) return s;
    {
        g.span = next_span(owner, HAP_PHASE_MASKGEMM);
        PhaseScope ps(owner, HAP_PHASE_MASKGEMM, 1, st);
        e = launch_maskgemm(P.maps, g, pair, st);
    }
    for (int k = 0; k < pa.G && e == cudaSuccess; ++k) {
        e = cudaEventRecord(T[k].w->ev_free[slots[k]], st);
        T[k].w->used[slots[k]] = true;
    }
    if (e != cudaSuccess) return cuda_fail(owner, e, "mask-GEMM");
    return HAP_OK;
}


hap_status run_wave(hap_ctx owner, int G, const WaveTest* T, int pair, cudaStream_t st,
                    bool shared = false, cudaStream_t light = nullptr) {
    WavePlan P;
    hap_status s = plan_wave(owner, G, T, pair, shared, P);
    if (s) return s;
    return launch_wave(owner, T, pair, st, P, light);
}

hap_status check_cfg(hap_ctx c, const hap_perm_cfg* cfg) {
    if (cfg->b_end < cfg->b_begin || cfg->b_end > (1ull << 32))
        return fail(c, HAP_E_INVALID_ARG, "need b_begin <= b_end <= 2^32");
    if (cfg->pair_mode < 0 || cfg->pair_mode > 2) return fail(c, HAP_E_INVALID_ARG, "bad pair_mode");
    return HAP_OK;
}

// tiles of one launch for a test of n_pad pooled rows: the block's bf16 mask stays within
// the L2-resident budget, or cfg->block permutations when set
int64_t block_tiles(const hap_perm_cfg* cfg, int64_t n_pad, int64_t R) {
    static const char* mb = getenv("HAP_MASK_BUDGET_MB");  // EXPERIMENT: block size
    const int64_t budget = mb ? (int64_t)atoi(mb) << 20 : kMaskBudget;
    // at most kMaxBlockTiles tiles (~10^6 permutations) per launch: small pools would
    // otherwise fill the byte budget with tens of thousands of tiles per workspace
    int64_t t = std::max<int64_t>(1, std::min<int64_t>(kMaxBlockTiles, budget / (R * n_pad * 2)));
    if (cfg->block) t = std::max<int64_t>(1, ceil_div((int64_t)cfg->block, R - 1));
    return t;
}

}  // namespace

extern "C" {

hap_status hap_permtest(hap_ctx c, hap_align_info* info, const hap_perm_cfg* cfg,
                        hap_counts* counts, double* stats, void* stream) {
    if (!c) return HAP_E_INVALID_ARG;
    if (!c->aligned) return fail(c, HAP_E_NOT_ALIGNED, "hap_permtest before hap_align");
    if (!info || !cfg || !counts) return fail(c, HAP_E_INVALID_ARG, "null pointer");
    hap_status s = check_cfg(c, cfg);
    if (s) return s;
    if (!is_device_ptr(counts) || (stats && !is_device_ptr(stats)))
        return fail(c, HAP_E_INVALID_ARG, "counts/stats must be device memory");
    if (cfg->flags & HAP_FLAG_EXHAUSTIVE) {
        const uint64_t total = hap_n_choose_k(c->n_x + c->n_y, c->n_x);
        if (c->n_x + c->n_y > 64 || total == 0 || total >= (1ull << 32) || cfg->b_end > total)
            return fail(c, HAP_E_INVALID_ARG, "exhaustive mode needs C(N, n_x) < 2^32 and b_end <= C(N, n_x)");
    }
    cudaSetDevice(c->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int pair = cfg->pair_mode ? cfg->pair_mode : 2;
    const int64_t R = (int64_t)kTileM * pair;
    const int64_t total = (int64_t)(cfg->b_end - cfg->b_begin);
    const int64_t max_tiles = block_tiles(cfg, c->n_pad, R);
    const int64_t total_tiles = ceil_div(std::max<int64_t>(total, 1), R - 1);
    // Block schedule: the generator of block i+1 runs beside the mask-GEMM of block i (side
    // stream, two mask slots), but block 0's generator and the alignment have nothing to hide
    // behind.  A long test therefore starts with a small block and grows it geometrically
    // (x1.75: the generator, slowed ~2x beside a mask-GEMM, still finishes within the
    // previous block's GEMM) up to the L2-sized maximum; an explicit cfg->block is kept as
    // given.  Results do not depend on the blocking (PERM-SPEC v1 is addressed by b).
    int64_t tiles = max_tiles;
    const bool grow = !cfg->block && total_tiles >= 16;
    if (grow) tiles = std::min<int64_t>(max_tiles, std::max<int64_t>(4, total_tiles / 12));
    // the blocks' mask-GEMMs run on the context's high-priority stream, forked from and
    // joined back to `st`
    cudaStream_t ks = st;
    if (total_tiles > tiles) {
        if (!c->hi) {
            int lo_p = 0, hi_p = 0;
            cudaDeviceGetStreamPriorityRange(&lo_p, &hi_p);
            if (cudaStreamCreateWithPriority(&c->hi, cudaStreamNonBlocking, hi_p) != cudaSuccess ||
                cudaEventCreateWithFlags(&c->ev_hi[0], cudaEventDisableTiming) != cudaSuccess ||
                cudaEventCreateWithFlags(&c->ev_hi[1], cudaEventDisableTiming) != cudaSuccess)
                return fail(c, HAP_E_CUDA, "mask-GEMM stream");
        }
        cudaError_t e = cudaEventRecord(c->ev_hi[0], st);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(c->hi, c->ev_hi[0], 0);
        if (e != cudaSuccess) return cuda_fail(c, e, "fork");
        ks = c->hi;
    }
    for (int64_t off = 0; off < total;) {
        const int64_t blk = tiles * (R - 1);
        const WaveTest t{c, info, cfg, counts, stats ? stats + 3 * off : nullptr,
                         cfg->b_begin + (uint64_t)off, std::min<int64_t>(blk, total - off)};
        if ((s = run_wave(c, 1, &t, pair, ks))) return s;
        off += blk;
        if (grow) tiles = std::min<int64_t>(max_tiles, (tiles * 7 + 3) / 4);
    }
    if (ks != st) {
        cudaError_t e = cudaEventRecord(c->ev_hi[1], ks);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(st, c->ev_hi[1], 0);
        if (e != cudaSuccess) return cuda_fail(c, e, "join");
    }
    c->last_stream = st;
    return HAP_OK;
}

hap_status hap_permtest_batch(hap_ctx c, int64_t P, const float* X_packed, const int64_t* cu_nx,
                              const float* Y_packed, const int64_t* cu_ny, int64_t d,
                              hap_align_mode mode, const hap_perm_cfg* cfg, const int64_t* pair_sel,
                              int64_t n_sel, hap_align_info* infos, hap_counts* counts, void* stream) {
    if (!c) return HAP_E_INVALID_ARG;
    if (P < 0 || !X_packed || !Y_packed || !cu_nx || !cu_ny || !cfg || !infos || !counts)
        return fail(c, HAP_E_INVALID_ARG, "null pointer / negative P");
    if (pair_sel && n_sel < 0) return fail(c, HAP_E_INVALID_ARG, "n_sel < 0");
    if (mode != HAP_ALIGN_HOUSEHOLDER && mode != HAP_ALIGN_NONE)
        return fail(c, HAP_E_INVALID_ARG, "bad mode");
    if (cfg->flags & HAP_FLAG_EXHAUSTIVE)
        return fail(c, HAP_E_INVALID_ARG, "exhaustive mode: use hap_permtest per pair");
    hap_status s = check_cfg(c, cfg);
    if (s) return s;
    // inputs in device memory, or both in host memory (pinned for overlap): each wave then
    // copies its pairs' rows on its lane stream, overlapping the other lane's kernels
    const bool host_in = !is_device_ptr(X_packed);
    if (host_in != !is_device_ptr(Y_packed))
        return fail(c, HAP_E_INVALID_ARG, "X_packed and Y_packed must both be device or both host memory");
    const int64_t n = pair_sel ? n_sel : P;
    // shape checks are synchronous: validate every selected pair before enqueuing anything
    std::vector<char> seen(pair_sel ? (size_t)P : 0, 0);
    for (int64_t i = 0; i < n; ++i) {
        const int64_t p = pair_sel ? pair_sel[i] : i;
        if (p < 0 || p >= P) return fail(c, HAP_E_INVALID_ARG, "pair_sel out of range");
        if (pair_sel && seen[(size_t)p]++)  // a repeated pair would add its counts twice
            return fail(c, HAP_E_INVALID_ARG, "pair_sel lists pair " + std::to_string(p) + " twice");
        const int64_t nx = cu_nx[p + 1] - cu_nx[p], ny = cu_ny[p + 1] - cu_ny[p];
        if (nx < 1 || ny < 1 || nx + ny > 65535)
            return fail(c, HAP_E_INVALID_ARG, "pair " + std::to_string(p) + ": bad n_x / n_y");
    }
    if (d < 2 || d > 16384) return fail(c, HAP_E_DIM_MISMATCH, "need 2 <= d <= 16384");
    cudaSetDevice(c->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    static const char* lanes_env = getenv("HAP_LANES");  // EXPERIMENT: number of lanes
    const int nlanes = std::max(1, std::min(kMaxLanes, lanes_env ? atoi(lanes_env) : 2));
    for (int k = 0; k < nlanes; ++k) {
        for (int j = 0; j < kMaxWave; ++j)
            if (!c->sub[k][j]) {
                s = hap_create(c->device, &c->sub[k][j]);
                if (s) return fail(c, s, "sub-context");
                hap_profile(c->sub[k][j], c->serial ? 2 : c->prof ? 1 : 0);
                if (c->spans) hap_profile_spans(c->sub[k][j], 1);
            }
        // lane streams (alignment + mask-GEMM) at the highest priority, the generator side
        // streams at the default (lowest): pending alignment / mask-GEMM CTAs are placed before
        // the generator's (HAP_LANE_PRIO=0: all at the default, experiments)
        static const char* lp = getenv("HAP_LANE_PRIO");
        int prio_lo = 0, prio_hi = 0;
        cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
        const int lane_prio = (lp && atoi(lp) == 0) ? prio_lo : prio_hi;
        if (!c->sub_stream[k] &&
            (cudaStreamCreateWithPriority(&c->sub_stream[k], cudaStreamNonBlocking, lane_prio) != cudaSuccess ||
             cudaEventCreateWithFlags(&c->ev_sub[k], cudaEventDisableTiming) != cudaSuccess))
            return fail(c, HAP_E_CUDA, "batch streams");
        if (host_in && !c->cp_stream[k] &&
            (cudaStreamCreateWithFlags(&c->cp_stream[k], cudaStreamNonBlocking) != cudaSuccess ||
             cudaEventCreateWithFlags(&c->ev_k1done[k][0], cudaEventDisableTiming) != cudaSuccess ||
             cudaEventCreateWithFlags(&c->ev_k1done[k][1], cudaEventDisableTiming) != cudaSuccess ||
             cudaEventCreateWithFlags(&c->ev_copied[k], cudaEventDisableTiming) != cudaSuccess))
            return fail(c, HAP_E_CUDA, "batch copy streams");
    }
    const int pair = cfg->pair_mode ? cfg->pair_mode : 2;
    const int64_t R = (int64_t)kTileM * pair;
    const int64_t B = (int64_t)(cfg->b_end - cfg->b_begin);
    int64_t maxN = 0, maxnx = 0, maxny = 0;
    for (int64_t i = 0; i < n; ++i) {
        const int64_t p = pair_sel ? pair_sel[i] : i;
        maxN = std::max<int64_t>(maxN, (cu_nx[p + 1] - cu_nx[p]) + (cu_ny[p + 1] - cu_ny[p]));
        maxnx = std::max<int64_t>(maxnx, cu_nx[p + 1] - cu_nx[p]);
        maxny = std::max<int64_t>(maxny, cu_ny[p + 1] - cu_ny[p]);
    }
    // wave size: tests whose whole b-range is one block are grouped (cfg->wave, else
    // HAP_WAVE, else 4 with shared masks or when every pair has N <= 2048, else 3: measured on
    // B200, profiles/r02_experiments/e50_wave.log: C2 73.0 -> 72.0 and C5 40.2 -> 39.2 us per
    // test with 4, the varlen C4 batch (N up to 10^4) 92.4 vs 93.9 with 3); others run alone
    // with their blocks in sequence
    const bool shared = (cfg->flags & HAP_FLAG_SHARED_MASK) != 0;
    static const char* wv = getenv("HAP_WAVE");
    const int wave_auto = (shared || maxN <= 2048) ? kMaxWave : 3;
    const int wave_max = std::max(1, std::min(kMaxWave, cfg->wave > 0 ? cfg->wave : wv ? atoi(wv) : wave_auto));
    {  // reserve every workspace the waves can use before the first launch
        if (maxN > 0) {
            const int64_t n_pad = round_up(maxN, kKBlock);
            const int64_t tiles = std::min(std::max<int64_t>(1, ceil_div(std::max<int64_t>(B, 1), R - 1)),
                                           block_tiles(cfg, n_pad, R));
            for (int k = 0; k < nlanes && !s; ++k)
                for (int j = 0; j < wave_max && !s; ++j) {
                    s = reserve_pair(c->sub[k][j], maxN, d, tiles, R, j == 0);
                    for (int b = 0; b < 2 && host_in; ++b) {  // (the owner's: a whole wave's rows)
                        const int64_t f = j == 0 ? wave_max : 1;
                        if (!s) s = ensure(c->sub[k][j], b ? kX2 : kX, (size_t)f * maxnx * d * 4);
                        if (!s) s = ensure(c->sub[k][j], b ? kY2 : kY, (size_t)f * maxny * d * 4);
                    }
                }
            if (s) return fail(c, s, "batch workspace");
        }
    }
    // fork: the two lanes start after the work already on the caller's stream
    cudaError_t e = cudaEventRecord(c->ev_fork, st);
    for (int k = 0; k < nlanes && e == cudaSuccess; ++k) {
        // (the copy streams need no fork: their only hazard, the K1 that last read a staging
        // buffer, is tracked across calls, so the next call's copies start at once)
        e = cudaStreamWaitEvent(c->sub_stream[k], c->ev_fork, 0);
    }
    if (e != cudaSuccess) return cuda_fail(c, e, "batch fork");
    std::vector<hap_perm_cfg> pcs((size_t)n);
    // processing order: largest pairs first, equal shapes adjacent (results do not depend on
    // the order: every pair has its own generator stream and workspace); waves of similar
    // sizes balance the mask-GEMM and keep shared-mask waves full (C4: 134 -> 122 us/test)
    std::vector<int64_t> order((size_t)n);
    for (int64_t i = 0; i < n; ++i) order[(size_t)i] = pair_sel ? pair_sel[i] : i;
    std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) {
        const int64_t na = cu_nx[a + 1] - cu_nx[a], nb = cu_nx[b + 1] - cu_nx[b];
        const int64_t Na = na + cu_ny[a + 1] - cu_ny[a], Nb = nb + cu_ny[b + 1] - cu_ny[b];
        return Na != Nb ? Na > Nb : na > nb;
    });
    int64_t i = 0, wave = 0;
    while (i < n && !s) {
        const int k = (int)(wave % nlanes);  // consecutive waves rotate over the lanes
        cudaStream_t ls = c->sub_stream[k];
        WaveTest T[kMaxWave];
        AlignPair Q[kMaxWave];
        hap_ctx W[kMaxWave];
        // the wave's pairs (decided on their shapes before anything is enqueued)
        int64_t mem[kMaxWave];
        int Gm = 0;
        for (int64_t j = i; j < n && Gm < wave_max;) {
            const int64_t p = order[(size_t)j];
            const int64_t nx = cu_nx[p + 1] - cu_nx[p], ny = cu_ny[p + 1] - cu_ny[p];
            const bool one_block = ceil_div(std::max<int64_t>(B, 1), R - 1) <= block_tiles(cfg, round_up(nx + ny, kKBlock), R);
            if (Gm > 0) {
                const int64_t p0 = mem[0], nx0 = cu_nx[p0 + 1] - cu_nx[p0], ny0 = cu_ny[p0 + 1] - cu_ny[p0];
                if (!one_block) break;  // a multi-block test starts its own wave
                if (shared && (nx != nx0 || ny != ny0)) break;  // same masks
                // one alignment path per wave (the path is a function of the pair's shape)
                if (align_path(nx + ny, d) != align_path(nx0 + ny0, d)) break;
            }
            mem[Gm++] = p;
            ++j;
            if (!one_block) break;
        }
        const int sb = c->lane_waves[k] & 1;  // staging buffers of this wave
        if (host_in && Gm > 0 && c->k1_recorded[k][sb])  // their last reader: the K1 two waves back
            cudaStreamWaitEvent(c->cp_stream[k], c->ev_k1done[k][sb], 0);
        // host inputs of consecutive packed pairs: ONE copy of the wave's X rows and one of its
        // Y rows into the wave owner's staging buffers (a copy per pair paid ~5 us of DMA set-up
        // per 3 MB at C2, ~9 % of the H2D time); the pairs then read their rows from there
        const float* dXw = nullptr;
        const float* dYw = nullptr;
        if (host_in && Gm > 1) {
            bool contiguous = true;
            for (int j = 1; j < Gm; ++j) contiguous &= mem[j] == mem[j - 1] + 1;
            if (contiguous) {
                hap_ctx w0 = c->sub[k][0];
                const int bX = sb ? kX2 : kX, bY = sb ? kY2 : kY;
                const int64_t rx = cu_nx[mem[Gm - 1] + 1] - cu_nx[mem[0]], ry = cu_ny[mem[Gm - 1] + 1] - cu_ny[mem[0]];
                if (!(s = ensure(w0, bX, (size_t)rx * d * 4)) && !(s = ensure(w0, bY, (size_t)ry * d * 4))) {
                    cudaError_t e2 = cudaMemcpyAsync(w0->buf[bX], X_packed + cu_nx[mem[0]] * d, (size_t)rx * d * 4,
                                                     cudaMemcpyHostToDevice, c->cp_stream[k]);
                    if (e2 == cudaSuccess)
                        e2 = cudaMemcpyAsync(w0->buf[bY], Y_packed + cu_ny[mem[0]] * d, (size_t)ry * d * 4,
                                             cudaMemcpyHostToDevice, c->cp_stream[k]);
                    if (e2 != cudaSuccess) s = cuda_fail(c, e2, "H2D wave rows");
                    dXw = static_cast<const float*>(w0->buf[bX]);
                    dYw = static_cast<const float*>(w0->buf[bY]);
                }
                if (s) break;
            }
        }
        int G = 0;
        for (; G < Gm; ++G) {
            const int64_t p = mem[G];
            const int64_t nx = cu_nx[p + 1] - cu_nx[p], ny = cu_ny[p + 1] - cu_ny[p];
            hap_ctx w = c->sub[k][G];
            const float* Xp = dXw ? dXw + (cu_nx[p] - cu_nx[mem[0]]) * d : X_packed + cu_nx[p] * d;
            const float* Yp = dYw ? dYw + (cu_ny[p] - cu_ny[mem[0]]) * d : Y_packed + cu_ny[p] * d;
            s = prepare_pair_cp(w, Xp, nx, Yp, ny, d, infos + p, ls, Q[G],
                                host_in && !dXw ? c->cp_stream[k] : nullptr, sb);
            if (s) {
                c->err = "pair " + std::to_string(p) + ": " + w->err;
                break;
            }
            W[G] = w;
            pcs[i] = *cfg;
            pcs[i].stream_id = shared ? cfg->stream_id : cfg->stream_id + (uint32_t)p;
            T[G] = WaveTest{w, infos + p, &pcs[i], counts + p, nullptr, cfg->b_begin, B};
            ++i;
        }
        const bool multi = G == 1 && ceil_div(std::max<int64_t>(B, 1), R - 1) > block_tiles(cfg, Q[0].n_pad, R);
        WavePlan P;
        bool staged = false;
        if (!s && G > 0 && !multi && B > 0) {
            s = plan_wave(W[0], G, T, pair, shared, P);
            // EXPERIMENT (HAP_K1_DRAWS=1): the wave's generator draws ride in K1's idle issue
            // slots and K2 keeps only its table pass; bit-exact, but the lane then runs
            // K1 -> K2b -> K3 in series and measured 106 vs 85 us per C2 test, so off
            static const char* kd = getenv("HAP_K1_DRAWS");
            staged = !s && kd && atoi(kd) != 0 && perm_can_split(P.pa) &&
                     align_path(Q[0].n_x + Q[0].n_y, d) == kAlignFused;
        }
        if (!s && G > 0 && host_in) {  // K1 waits for the wave's rows
            cudaEventRecord(c->ev_copied[k], c->cp_stream[k]);
            cudaStreamWaitEvent(ls, c->ev_copied[k], 0);
        }
        if (!s && G > 0) {
            s = align_wave(W[0], G, W, Q, mode, ls, staged ? &P.pa : nullptr);  // one K1 launch
            if (s) c->err = "wave " + std::to_string(wave) + ": " + W[0]->err;
        }
        if (!s && G > 0 && host_in) {
            const int sb = c->lane_waves[k] & 1;
            cudaEventRecord(c->ev_k1done[k][sb], ls);
            c->k1_recorded[k][sb] = true;
        }
        ++c->lane_waves[k];
        if (s || G == 0) break;
        if (multi) {
            s = hap_permtest(T[0].w, T[0].info, T[0].cfg, T[0].counts, nullptr, ls);  // blocks
        } else if (B > 0) {
            static const char* sp = getenv("HAP_BATCH_SPLIT");  // K2a on the side stream
            const bool split = sp && atoi(sp) != 0;
            s = launch_wave(T[0].w, T, pair, ls, P, split ? T[0].w->side : nullptr, staged);
        }
        if (s) c->err = "wave " + std::to_string(wave) + ": " + T[0].w->err;
        ++wave;
    }
    // join: the caller's stream waits for both lanes (also on error, to keep ordering sane)
    for (int k = 0; k < nlanes; ++k) {
        if (cudaEventRecord(c->ev_sub[k], c->sub_stream[k]) == cudaSuccess)
            cudaStreamWaitEvent(st, c->ev_sub[k], 0);
    }
    c->last_stream = st;
    c->last_info = nullptr;  // per-pair data errors are reported in infos[p].status
    return s;
}

hap_status hap_profile_spans(hap_ctx c, int enable) {
    if (!c) return HAP_E_INVALID_ARG;
    cudaSetDevice(c->device);
    if (enable) {
        hap_status s = reset_spans(c);
        if (s) return s;
    }
    c->spans = enable != 0;
    for (auto& lane : c->sub)
        for (hap_ctx w : lane)
            if (w) {
                hap_status s = hap_profile_spans(w, enable);
                if (s) return s;
            }
    return HAP_OK;
}

hap_status hap_profile_spans_read(hap_ctx c, double* out, int64_t max_n, int64_t* n) {
    if (!c || !n) return HAP_E_INVALID_ARG;
    cudaSetDevice(c->device);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return cuda_fail(c, e, "span read");
    std::vector<std::pair<hap_ctx, int>> lanes = {{c, 0}};
    for (int k = 0; k < kMaxLanes; ++k)
        for (hap_ctx w : c->sub[k])
            if (w) lanes.push_back({w, k + 1});
    struct Rec { int code; unsigned long long a, b; };
    std::vector<Rec> recs;
    for (auto& lw : lanes) {
        hap_ctx w = lw.first;
        const int lane = lw.second;
        if (!w || !w->spans || w->span_phase.empty()) continue;
        std::vector<unsigned long long> h(2 * w->span_phase.size());
        e = cudaMemcpy(h.data(), w->buf[kSpans], h.size() * 8, cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) return cuda_fail(c, e, "span read");
        for (size_t i = 0; i < w->span_phase.size(); ++i)
            recs.push_back({w->span_phase[i] + HAP_NUM_PHASES * lane, h[2 * i], h[2 * i + 1]});
        hap_status s = reset_spans(w);
        if (s) return s;
    }
    unsigned long long t0 = ~0ull;
    for (auto& r : recs)
        if (r.b) t0 = std::min(t0, r.a);
    int64_t k = 0;
    for (auto& r : recs) {
        if (out && k < max_n) {
            out[3 * k + 0] = r.code;
            out[3 * k + 1] = r.b ? 1e-3 * (double)(r.a - t0) : -1.0;  // -1: kernel exited early
            out[3 * k + 2] = r.b ? 1e-3 * (double)(r.b - t0) : -1.0;
        }
        ++k;
    }
    *n = k;
    return HAP_OK;
}

hap_status hap_profile(hap_ctx c, int enable) {
    if (!c) return HAP_E_INVALID_ARG;
    c->prof = enable != 0;
    c->serial = enable >= 2;
    c->stamp_k1 = enable >= 3;
    for (auto& lane : c->sub)
        for (hap_ctx w : lane)
            if (w) hap_profile(w, enable);
    return HAP_OK;
}

hap_status hap_debug_k3_stamps(hap_ctx c, long long* out, int64_t n) {
    if (c && !c->buf[kK3Stamps] && c->sub[0][0]) c = c->sub[0][0];  // a batch: lane 0's owner
    if (!c || !out || !c->buf[kK3Stamps]) return HAP_E_INVALID_ARG;
    cudaDeviceSynchronize();
    const size_t bytes = std::min<size_t>((size_t)n * 8, (size_t)c->sm_count * 64 * 8);
    if (cudaMemcpy(out, c->buf[kK3Stamps], bytes, cudaMemcpyDeviceToHost) != cudaSuccess)
        return HAP_E_CUDA;
    return HAP_OK;
}

hap_status hap_debug_k1_stamps(hap_ctx c, long long* out, int64_t n) {
    if (c && !c->buf[kStamps] && c->sub[0][0]) c = c->sub[0][0];  // a batch: lane 0's owner
    if (!c || !out || !c->buf[kStamps]) return HAP_E_INVALID_ARG;
    cudaDeviceSynchronize();
    const size_t bytes = std::min<size_t>((size_t)n * 8, c->cap[kStamps]);
    if (cudaMemcpy(out, c->buf[kStamps], bytes, cudaMemcpyDeviceToHost) != cudaSuccess)
        return HAP_E_CUDA;
    return HAP_OK;
}

hap_status hap_profile_k1_phases(hap_ctx c, double* us) {
    if (!c || !us) return HAP_E_INVALID_ARG;
    if (!c->buf[kStamps]) return fail(c, HAP_E_INVALID_ARG, "K1 stamps not enabled (hap_profile 3)");
    long long t[8];
    cudaError_t e = cudaDeviceSynchronize();
    if (e == cudaSuccess) e = cudaMemcpy(t, c->buf[kStamps], sizeof t, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_fail(c, e, "k1 phases");
    for (int k = 0; k < 5; ++k) us[k] = 1e-3 * (double)(t[k + 1] - t[k]);
    us[5] = us[6] = 0.0;
    return HAP_OK;
}

hap_status hap_profile_read(hap_ctx c, double* ms, int64_t* launches, int reset) {
    if (!c) return HAP_E_INVALID_ARG;
    cudaSetDevice(c->device);
    for (auto& m : c->marks) {
        float t = 0.f;
        cudaError_t e = cudaEventSynchronize(m.b);
        if (e == cudaSuccess) e = cudaEventElapsedTime(&t, m.a, m.b);
        if (e != cudaSuccess) return cuda_fail(c, e, "profile events");
        c->ms[m.phase] += t;
        c->pool.push_back(m.a);
        c->pool.push_back(m.b);
    }
    c->marks.clear();
    double sub_ms[HAP_NUM_PHASES] = {}, sub_sum_ms[HAP_NUM_PHASES] = {};
    int64_t sub_n[HAP_NUM_PHASES] = {}, sub_sum_n[HAP_NUM_PHASES] = {};
    for (auto& lane : c->sub)
        for (hap_ctx w : lane) {
            if (!w) continue;
            hap_profile_read(w, sub_ms, sub_n, reset);
            for (int p = 0; p < HAP_NUM_PHASES; ++p) {
                sub_sum_ms[p] += sub_ms[p];
                sub_sum_n[p] += sub_n[p];
            }
        }
    for (int p = 0; p < HAP_NUM_PHASES; ++p) {
        if (ms) ms[p] = c->ms[p] + sub_sum_ms[p];
        if (launches) launches[p] = c->launches[p] + sub_sum_n[p];
        if (reset) {
            c->ms[p] = 0.0;
            c->launches[p] = 0;
        }
    }
    return HAP_OK;
}

hap_status hap_profile_timeline(hap_ctx c, double* out, int64_t max_n, int64_t* n) {
    if (!c || !n) return HAP_E_INVALID_ARG;
    cudaSetDevice(c->device);
    // lane 0 = this context, lanes 1, 2 = the batch lanes' sub-contexts; one time base
    std::vector<std::pair<hap_ctx, int>> lanes = {{c, 0}};
    for (int k = 0; k < kMaxLanes; ++k)
        for (hap_ctx w : c->sub[k])
            if (w) lanes.push_back({w, k + 1});
    cudaEvent_t t0 = nullptr;
    for (auto& lw : lanes)
        if (!lw.first->marks.empty() && !t0) t0 = lw.first->marks.front().a;
    int64_t k = 0;
    double tmin = 0.0;
    for (auto& lw : lanes) {
        hap_ctx w = lw.first;
        const int lane = lw.second;
        for (auto& m : w->marks) {
            float ta = 0.f, tb = 0.f;
            cudaError_t e = cudaEventSynchronize(m.b);
            if (e == cudaSuccess) e = cudaEventElapsedTime(&ta, t0, m.a);
            if (e == cudaSuccess) e = cudaEventElapsedTime(&tb, t0, m.b);
            if (e != cudaSuccess) return cuda_fail(c, e, "profile timeline");
            if (out && k < max_n) {
                out[3 * k + 0] = m.phase + HAP_NUM_PHASES * lane;
                out[3 * k + 1] = 1e3 * ta;
                out[3 * k + 2] = 1e3 * tb;
            }
            tmin = std::min(tmin, 1e3 * (double)ta);
            ++k;
            w->ms[m.phase] += tb - ta;
        }
        for (auto& m : w->marks) {
            w->pool.push_back(m.a);
            w->pool.push_back(m.b);
        }
        w->marks.clear();
    }
    if (out)
        for (int64_t i = 0; i < std::min(k, max_n); ++i) {
            out[3 * i + 1] -= tmin;
            out[3 * i + 2] -= tmin;
        }
    *n = k;
    return HAP_OK;
}

hap_status hap_perm_sets(hap_ctx c, uint64_t seed, uint32_t stream_id, uint64_t b_begin, int64_t count,
                         int64_t N, int64_t n_x, uint8_t* out, void* stream) {
    if (!c) return HAP_E_INVALID_ARG;
    if (!out || count < 0 || N < 1 || N > 65535 || n_x < 0 || n_x > N)
        return fail(c, HAP_E_INVALID_ARG, "bad perm_sets arguments");
    if (b_begin + (uint64_t)count > (1ull << 32)) return fail(c, HAP_E_INVALID_ARG, "b >= 2^32");
    cudaSetDevice(c->device);
    PermArgs pa{};
    pa.G = 1;
    pa.t[0].seed = seed;
    pa.t[0].s = stream_id;
    pa.t[0].b_begin = b_begin;
    pa.t[0].count = count;
    pa.t[0].N = N;
    pa.t[0].n_x = n_x;
    pa.t[0].n_pad = round_up(N, kKBlock);
    pa.t[0].out = out;
    pa.t[0].ntiles = 0;
    pa.out_kind = kMaskU8Set;
    pa.rows_per_tile = 0;
    perm_items(pa);
    cudaError_t e = launch_perm(pa, c->sm_count, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(c, e, "perm generator");
    return HAP_OK;
}

hap_status hap_debug_last_form(hap_ctx c, int32_t* gram) {
    if (!c || !gram) return HAP_E_INVALID_ARG;
    *gram = c->last_gram;
    return HAP_OK;
}

hap_status hap_debug_check_status(hap_ctx c, uint64_t* word) {
    if (!c || !word) return HAP_E_INVALID_ARG;
    *word = 0;
#ifdef HAP_DEVICE_CHECKS
    cudaSetDevice(c->device);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return cuda_fail(c, e, "check sync");
    const unsigned long long w[4] = {check_word_align(), check_word_perm(), check_word_gemm(), check_word_gram()};
    for (unsigned long long v : w)
        if (v && !*word) *word = v;
    std::vector<hap_ctx> all = {c};
    for (auto& lane : c->sub)
        for (hap_ctx s : lane)
            if (s) all.push_back(s);
    std::vector<unsigned char> tail;
    for (hap_ctx s : all)
        for (int b = 0; b < kNumBufs; ++b) {
            if (!s->buf[b] || s->cap[b] <= s->req[b]) continue;
            tail.resize(s->cap[b] - s->req[b]);
            if (cudaMemcpy(tail.data(), static_cast<char*>(s->buf[b]) + s->req[b], tail.size(),
                           cudaMemcpyDeviceToHost) != cudaSuccess)
                return fail(c, HAP_E_CUDA, "guard readback");
            for (unsigned char x : tail)
                if (x != 0xA5)
                    return fail(c, HAP_E_CUDA, "guard bytes of workspace buffer " + std::to_string(b) +
                                                   " overwritten");
        }
    return HAP_OK;
#else
    return fail(c, HAP_E_INVALID_ARG, "release library: no device checks compiled in");
#endif
}

hap_status hap_debug_alu_burn(hap_ctx c, uint32_t iters, int ctas, int threads, void* stream) {
    if (!c) return HAP_E_INVALID_ARG;
    if (ensure(c, kStamps, 64) != HAP_OK) return HAP_E_OOM;
    cudaError_t e = launch_debug_alu_burn(iters, ctas, threads, B<uint32_t>(c, kStamps),
                                          static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? HAP_OK : cuda_fail(c, e, "alu burn");
}

uint64_t hap_n_choose_k(int64_t N, int64_t k) {
    if (k < 0 || N < 0 || k > N) return 0;
    if (k > N - k) k = N - k;
    unsigned __int128 c = 1;
    for (int64_t i = 1; i <= k; ++i) {
        c = c * (unsigned __int128)(N - k + i) / (unsigned __int128)i;  // exact at every step
        if (c > (unsigned __int128)UINT64_MAX) return 0;
    }
    return (uint64_t)c;
}

hap_status hap_comb_sets(hap_ctx c, uint64_t b_begin, int64_t count, int64_t N, int64_t n_x, uint8_t* out,
                         void* stream) {
    if (!c) return HAP_E_INVALID_ARG;
    const uint64_t total = hap_n_choose_k(N, n_x);
    if (!out || count < 0 || N < 1 || N > 64 || n_x < 0 || n_x > N || total == 0 ||
        total >= (1ull << 32) || b_begin + (uint64_t)count > total)
        return fail(c, HAP_E_INVALID_ARG, "bad comb_sets arguments");
    cudaSetDevice(c->device);
    PermArgs pa{};
    pa.G = 1;
    pa.t[0].b_begin = b_begin;
    pa.t[0].count = count;
    pa.t[0].N = N;
    pa.t[0].n_x = n_x;
    pa.t[0].n_pad = round_up(N, kKBlock);
    pa.t[0].out = out;
    pa.t[0].exhaustive = 1;
    pa.out_kind = kMaskU8Set;
    perm_items(pa);
    cudaError_t e = launch_perm(pa, c->sm_count, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(c, e, "comb generator");
    return HAP_OK;
}

hap_status hap_export_pooled(hap_ctx c, uint16_t* zhi, uint16_t* zlo, double* t, double* m,
                             void* stream) {
    if (!c) return HAP_E_INVALID_ARG;
    if (!c->aligned) return fail(c, HAP_E_NOT_ALIGNED, "no pooled cloud yet");
    if (!zhi || !zlo || !t || !m) return fail(c, HAP_E_INVALID_ARG, "null pointer");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const size_t bytes = (size_t)c->d_pad * c->n_pad * 2;  // the first d_pad rows of the planes
    cudaError_t e = cudaMemcpyAsync(zhi, c->buf[kZhi], bytes, cudaMemcpyDeviceToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(zlo, c->buf[kZlo], bytes, cudaMemcpyDeviceToDevice, st);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(t, c->buf[kT64], (size_t)c->d_pad * 8, cudaMemcpyDeviceToDevice, st);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(m, c->buf[kM], (size_t)c->d_pad * 8, cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) return cuda_fail(c, e, "export");
    return HAP_OK;
}

}  // extern "C"
