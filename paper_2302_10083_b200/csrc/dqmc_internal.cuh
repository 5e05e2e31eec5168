// dqmc_internal.cuh — shared declarations of libdqmc's translation units.
//
// libdqmc.so is the B200 (sm_100a) dense prime-implicant engine behind the C
// ABI of include/dqmc.h. It replaces the reference dense path
// (/root/reference/pkg/src/implicants/dense.py:340-418): load -> MERGE all
// dims -> REDUCE all dims -> extract. Design: the 3^(n-5)
// blocks of the reference layout are swept in a handful of HBM passes
// instead of the reference's 2(n-5)+1:
//
//   pass A  k_c0_merge           (dqmc_merge.cu)  truth table -> blocks, in-block
//                                 MERGE + the C0 block axes (contiguous 3^g-block
//                                 tiles in smem); only top-binary tiles are produced.
//   pass B  k_strided            (dqmc_merge.cu)  one group of <= 6 higher block
//                                 axes, reads the group's binary rows, writes its
//                                 star rows.
//   pass C  k_merge_reduce_pipe  (dqmc_reduce.cu) last group: MERGE then REDUCE of
//                                 the group (+ in-block axes); TMA gather of the
//                                 binary rows, TMA stores of every row.
//   pass D  k_strided_pipe       (dqmc_reduce.cu) REDUCE of the other groups +
//                                 in-block axes; TMA tiles, one producer warp.
//   pass E  k_c0_final           (dqmc_final.cu)  REDUCE of the C0 axes,
//                                 popcounts, per-tile scratch range and
//                                 ordered compaction; then a scan + k_reorder.
// The n = 24 plan (Plan::nz) adds zero-skip flags: pass C records which D
// items and E tiles can be nonzero, D and E skip the others.
// Small n (<= 12): one CTA does A+E on a single smem tile (k_small).
// dqmc_engine.cu holds the plan, the workspace and the C ABI; dqmc_input.cu
// the input conversion and generators; dqmc_shard.cu the sharded path's
// building blocks; dqmc_state.cu the per-dimension DenseState API.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <cmath>
#include <deque>
#include <atomic>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/dqmc.h"
#include "dqmc_device.cuh"

namespace dqmc {

constexpr int kC0Max = 7;           // block axes in the contiguous tile (3^7 blocks = 68.3 KiB)
constexpr int kC0MaxBlocks = 2187;  // 3^kC0Max
constexpr int kGroupMax = 6;        // block axes per strided pass (3^6 rows x 128 B = 91 KiB)
constexpr int kRowBlocks = 4;       // blocks per strided row (128 B)
constexpr int kStridedThreads = 288;  // 9 warps: 27 sub-cube tasks per round divide evenly
constexpr int kTileThreads = 224;   // 7 warps: the 4+3 C0 rounds divide into 1 and 3 tasks/thread
// pass E: 12 warps x 3 CTAs (smem-limited) = 36 warps/SM to hide LDS/shuffle
// latency; 56 registers/thread is the most that still fits 3 CTAs.
constexpr int kFinalThreads = 384;  // (224 and 288 measured slower: 9.46 / 9.14 vs 8.98 ms)
constexpr int kMaxKill = 8;         // parent bitmaps one final pass can clear (sharded path)

enum Mode { MERGE_ONLY = 0, MERGE_REDUCE = 1, REDUCE_ONLY = 2 };

__host__ __device__ inline int64_t pow3l(int k) {
    int64_t r = 1;
    for (int i = 0; i < k; i++) r *= 3;
    return r;
}

__device__ __forceinline__ int64_t bin_to_tern_rt(uint64_t b) {
    int64_t r = 0, p = 1;
    while (b) {
        if (b & 1) r += p;
        b >>= 1;
        p *= 3;
    }
    return r;
}

struct FinalArgs {
    int64_t *out;               // final ranks (single tile); null = scratch output or count only
    uint32_t *out32 = nullptr;  // multi-tile: tile-relative cell offsets (< 3^12) into the scratch;
                                // k_reorder adds the tile's first rank (tile_rank0) on the way out
    int64_t *tile_rank0 = nullptr;
    int64_t cap;                // capacity of out
    int64_t rank_add;           // added to every rank (dummy-variable padding < 0, top-block offset > 0)
    // sharded path: the state is nslots consecutive super-blocks (tiles_per_slot
    // tiles each); per slot up to kMaxKill parent super-block addresses (null
    // padded; local or peer memory) whose OR is cleared, and the rank added
    // to the slot's cells (rank_add_tab; null: rank_add for every tile)
    const uint64_t *kill_tab = nullptr;
    const int64_t *rank_add_tab = nullptr;
    int64_t tiles_per_slot = 1;
    int skip_c0 = 0;            // the C0 axes are already reduced (sharded extract pass)
    uint32_t ib_mask;           // in-block axes reduced in this pass
    uint32_t *bitmap_out;       // write final bitmap here (null: do not)
    unsigned long long *alloc;  // running scratch allocation counter
    int64_t *tile_base;         // per tile: offset of its ranks in out
    int32_t *tile_cnt;          // per tile: prime count
    int64_t tile0;              // first tile of this launch (chunked final stage)
    int prefetch = 0;           // L2 prefetch distance in tiles (0: off)
    int64_t pitch = 0;          // storage blocks per tile (0: 3^G, the reference layout)
    int pm_nr = 0;              // piece-major group 0 (make_plan): its 3^r rows; 0 = contiguous tiles
    int pm_np = 0;              // pieces (128 B) per tile
    const uint32_t *nz_e = nullptr;  // zero-tile flags (Plan::nz): bit u of row l = tile (u, l) may be nonzero
    int slot = 0;                    // per-tile scratch slot (entries); 0: every tile reserves with an atomic
    int64_t ovf0 = 0;                // first entry of the overflow pool (after the slots)
    // gather finish (Plan::nz, sparse states): pass D is not run; the group-0
    // parents of every block that survives the C0 reduce are read from the
    // state itself (piece-major: the same D item, (2 - d_j) 3^j rows up)
    // It is chosen on the device: pass C counts the nonzero blocks it wrote
    // (g0_cnt); the gather runs when they are at most g0_limit, else pass D ran.
    const uint32_t *g0 = nullptr;
    const unsigned long long *g0_cnt = nullptr;
    unsigned long long g0_limit = 0;
    uint32_t ib_gather = 0;  // in-block axes pass D would have reduced
};
// device-side choice between pass D and the gather finish (both kernels evaluate it)
__device__ __forceinline__ bool gather_chosen(const unsigned long long *cnt, unsigned long long limit) {
    return cnt != nullptr && __ldg(cnt) <= limit;
}

// ---------------------------------------------------------------------------
// TMA bulk copies (cp.async.bulk, SASS UBLKCP) with an mbarrier

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t *mbar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(mbar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *mbar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(mbar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, uint64_t *mbar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(mbar))
        : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *mbar, unsigned phase) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(mbar)),
        "r"(phase)
        : "memory");
}

// At n = 24 about four in five blocks of the state are zero (a block is
// nonzero only when its 19 block digits hold few stars: M(c) = AND over 2^stars
// completions), and reducing a zero cell is a no-op. The reduce rounds skip
// the work of a warp whose words are all zero (one vote per task).
template <int N>
__device__ __forceinline__ bool warp_any(const uint32_t (&v)[N]) {
    uint32_t a = 0;
#pragma unroll
    for (int x = 0; x < N; x++) a |= v[x];
    return __any_sync(0xffffffffu, a != 0u);
}

// ---------------------------------------------------------------------------
// TMA tensor copies (cp.async.bulk.tensor, SASS UTMALDG/UTMASTG)

__device__ __forceinline__ void tma_store_3d(const CUtensorMap *map, int c0, int c1, int c2, const void *src) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(map), "r"(c0),
                 "r"(c1), "r"(c2), "r"(smem_u32(src))
                 : "memory");
}

__device__ __forceinline__ void tma_load_4d(void *dst, const CUtensorMap *map, int c0, int c1, int c2, int c3,
                                            uint64_t *mbar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::
            "r"(smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(mbar))
        : "memory");
}

__device__ __forceinline__ void tma_store_4d(const CUtensorMap *map, int c0, int c1, int c2, int c3, const void *src) {
    asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];" ::"l"(map),
                 "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(src))
                 : "memory");
}

__device__ __forceinline__ void tma_prefetch_4d(const CUtensorMap *map, int c0, int c1, int c2, int c3) {
    asm volatile("cp.async.bulk.prefetch.tensor.4d.L2.global [%0, {%1, %2, %3, %4}];" ::"l"(map), "r"(c0), "r"(c1),
                 "r"(c2), "r"(c3)
                 : "memory");
}

__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ void mbar_arrive(uint64_t *mbar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(mbar)) : "memory");
}

__device__ __forceinline__ void bar_compute(int nthreads) {
    asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}

// Columns per tile: a group of 3^r rows with r < 6 packs CC adjacent 128-B
// columns into one tile, so tiles stay ~90 KB (enough bytes in flight per SM)
// and rows are written CC x 128 B wide (far-stride rows stream at ~4.1 TB/s in
// 128-B pieces, ~5.9 TB/s in 256-B and wider pieces; tools/probes/). The TMA
// box limit (256 elements) caps CC at 8.
template <int R1, int R2>
__host__ __device__ constexpr int pipe_cols() {
    constexpr int nr = P3<R1>::v * P3<R2>::v;
    return nr >= 729 ? 1 : (729 / nr > 8 ? 8 : 729 / nr);
}

template <int R1, int R2, int CC = pipe_cols<R1, R2>()>
struct PipeSmem {
    static constexpr int N1 = P3<R1>::v, N2 = P3<R2>::v;
    static constexpr int NR = N1 * N2;
    static constexpr int PITCH = 32 * CC;  // words per tile row
    static constexpr int TILE_WORDS = NR * PITCH;
    static constexpr int STAGE_WORDS = (1 << R1) * (1 << R2) * PITCH;
    static constexpr int BOXR = NR > 243 ? 243 : NR;  // TMA box rows (<= 256)
    static constexpr int NBOX = NR / BOXR;
    // compute warps: one register sub-cube task per warp per round (up to 27)
    static constexpr int TASKS = (N1 > N2 ? N1 : N2) * CC;
    static constexpr int CW = TASKS < 4 ? 4 : (TASKS > 27 ? 27 : TASKS);
    static constexpr int THREADS = (CW + 1) * 32;
    static constexpr int SMEM = (2 * TILE_WORDS + 2 * STAGE_WORDS) * 4;
};

__device__ __forceinline__ void tma_load_5d(void *dst, const CUtensorMap *map, int c0, int c1, int c2, int c3, int c4,
                                            uint64_t *mbar) {
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, "
        "%6}], [%7];" ::"r"(smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(smem_u32(mbar))
        : "memory");
}

// In-block REDUCE of a smem tile, thread per 32-B block (plain LDS.128 pairs:
// a 2-way bank conflict costs MIO wavefronts, which have slack, where a lane
// half-swap would cost 16 ALU selects per block). Warp-uniform iterations so
// an all-zero warp can skip (sparse).
// blkmask (optional, shared): bit j of word w = block 32w + j is nonzero after
// the round (every word written, zero for skipped warps).
__device__ __forceinline__ void inblock_round(uint32_t *tile, int nblocks, uint32_t ib_mask, int nct, int sparse,
                                              uint32_t *blkmask = nullptr) {
    const int lane = threadIdx.x & 31;
    for (int t0 = (int)(threadIdx.x & ~31u); t0 < nblocks; t0 += nct) {
        const int t = t0 + lane;
        const bool in = t < nblocks;
        uint4 *p = reinterpret_cast<uint4 *>(tile + (in ? t : 0) * 8);
        uint4 x0 = make_uint4(0, 0, 0, 0), x1 = x0;
        if (in) x0 = p[0], x1 = p[1];
        if (sparse && !__any_sync(0xffffffffu, (x0.x | x0.y | x0.z | x0.w | x1.x | x1.y | x1.z | x1.w) != 0u)) {
            if (blkmask && lane == 0) blkmask[t0 >> 5] = 0u;
            continue;
        }
        uint32_t v[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
        inblock_reduce(v, ib_mask);
        if (in) {
            p[0] = make_uint4(v[0], v[1], v[2], v[3]);
            p[1] = make_uint4(v[4], v[5], v[6], v[7]);
        }
        if (blkmask) {
            const uint32_t nzb =
                __ballot_sync(0xffffffffu, in && (v[0] | v[1] | v[2] | v[3] | v[4] | v[5] | v[6] | v[7]) != 0u);
            if (lane == 0) blkmask[t0 >> 5] = nzb;
        }
    }
}

// 4:1 OR-compaction of a 32-bit block mask: bit k of the result = any of bits 4k..4k+3
__device__ __forceinline__ uint32_t or4_compact(uint32_t w) {
    uint32_t m = w | (w >> 1);
    m = (m | (m >> 2)) & 0x11111111u;
    m = (m | (m >> 3)) & 0x03030303u;
    m = (m | (m >> 6)) & 0x000F000Fu;
    return (m | (m >> 12)) & 0xFFu;
}

// ---------------------------------------------------------------------------
// contiguous C0 tile: 3^g blocks x 8 words in shared memory

// MERGE of the C0 block axes on a tile whose 2^g binary blocks are loaded:
// minimal-work order, each star block computed once (3^g - 2^g ANDs).
inline __device__ void tile_merge_c0(uint32_t *sm, int g) {
    for (int j = 0; j < g; j++) {
        const int sj = (int)pow3l(j);
        const int nhi = 1 << (g - 1 - j);
        const int ntask = sj * nhi * 8;
        for (int t = threadIdx.x; t < ntask; t += blockDim.x) {
            const int w = t & 7, q = t >> 3;
            const int lo = q % sj, hi = q / sj;
            const int blk = lo + (int)bin_to_tern_rt(hi) * 3 * sj;
            sm[(blk + 2 * sj) * 8 + w] = sm[blk * 8 + w] & sm[(blk + sj) * 8 + w];
        }
        __syncthreads();
    }
}

// Load the binary blocks of a C0 tile from the truth table and merge it.
// Tile index tb (binary over the top digits) selects 32-bit TT words
// [tb << g, (tb+1) << g): point x = x_low5 + 32*(C0 bits) + 2^(5+g)*(top bits).
inline __device__ void tile_build(uint32_t *sm, const uint32_t *__restrict__ tt32, int g, int64_t tb) {
    const int nbin = 1 << g;
    for (int e = threadIdx.x; e < nbin; e += blockDim.x) {
        const uint32_t w = tt32[(tb << g) + e];
        uint32_t v[8];
        lm5(w, v);
        const int pos = (int)bin_to_tern_rt((uint64_t)e);
        uint4 *p = reinterpret_cast<uint4 *>(sm + pos * 8);
        p[0] = make_uint4(v[0], v[1], v[2], v[3]);
        p[1] = make_uint4(v[4], v[5], v[6], v[7]);
    }
    __syncthreads();
    tile_merge_c0(sm, g);
}

// ---------------------------------------------------------------------------
// host side

// ---------------------------------------------------------------------------
// host side

struct Plan {
    int n = 0, ne = 0;  // requested / effective (>= 5) variable count
    int H = 0, g = 0, T = 0, m = 0;
    int r[8] = {0}, a[8] = {0};
    uint32_t ib_C = 0, ib_E = 0, ib_D[8] = {0};
    int64_t rank_sub = 0;
    int64_t nblocks = 0;
    int64_t pitch = 0;   // storage blocks per C0 tile (3^g, or 3^g rounded up to 128 B)
    uint64_t sbytes = 0; // storage bytes of the state
    bool pm = false;     // piece-major storage of group 0 (see make_plan)
    bool nz = false;     // pass C records which D items / E tiles can be nonzero (see make_plan)
};

// Zero-skip flags of the n = 24 plan (Plan::nz): pass C ORs, per item (piece
// x, group-0 row l), the 729-bit mask of its nonzero rows u into row (x, l/243)
// of nz_b (box l/243 of D item (x, u)) and row l of nz_e (E tile (u, l)); rows
// are kNzWords words. REDUCE only clears bits, so a zero flag is exact for D
// and E.
constexpr int kNzWords = 24;
constexpr int kGatherPermille = 600;  // default dqmc_gather_threshold
// Flag layout in g_eng.nzflags (npiece = pieces per C0 tile, nr = 3^6 group-0
// rows): nz_b [npiece][3 boxes of 243 rows][kNzWords] (pass D's items (x, u)
// per box), nz_e [nr][kNzWords] (pass E's tiles (u, l)), then a zero page of
// one 243-row box (128-B aligned) that pass D loads its all-zero boxes from.
inline size_t nz_e_offset(size_t npiece) { return npiece * 3 * kNzWords; }
// ... then pass C's count of nonzero blocks (one unsigned long long)
inline size_t nz_count_offset(size_t npiece, size_t nr) {
    return (((npiece * 3 + nr) * kNzWords + 31) & ~(size_t)31) + (nr / 3) * 32;
}
inline size_t nz_zero_page(size_t npiece, size_t nr) { return ((npiece * 3 + nr) * kNzWords + 31) & ~(size_t)31; }

Plan make_plan(int n, bool padded = true);

extern thread_local std::string g_err;
extern const bool g_debug;  // DQMC_DEBUG: sync + report after every pass
extern std::mutex g_mu;

inline int set_err(int code, const std::string &msg) {
    g_err = msg;
    return code;
}

#define CK(call)                                                                                         \
    do {                                                                                                 \
        cudaError_t e_ = (call);                                                                         \
        if (e_ != cudaSuccess) return set_err(DQMC_ERR_CUDA, std::string(#call ": ") + cudaGetErrorString(e_)); \
    } while (0)

// every kernel launch of the dense, sharded, sparse and input paths is
// checked through this macro and counted (dqmc_launch_count: the bench line's
// gpu_launches)
extern std::atomic<uint64_t> g_launches;
#define CK_LAUNCH()                                  \
    do {                                             \
        g_launches.fetch_add(1, std::memory_order_relaxed); \
        CK(cudaGetLastError());                      \
    } while (0)

struct PinnedBuf {
    int64_t *ptr = nullptr;  // mapped pinned host memory (UVA: also the device address)
    size_t cap = 0;          // entries
};

typedef CUresult (*AddrRangeFn)(CUdeviceptr *, size_t *, CUdeviceptr);

// a submitted host-API job (dqmc_submit_* / dqmc_collect)
struct Job {
    int64_t id = 0;
    int slot = -1;        // -1: ran synchronously at submit, result in `res`
    dqmc_result_t res{};  // sync jobs only
    const void *in = nullptr;
    int kind = 0, n = 0;
    uint32_t flags = 0;
    // packed rank transfer (large results): the slot holds 4-byte tile offsets
    // in rank order and the tiles' positions; collect widens them on the host
    bool packed = false;
    int64_t ntiles = 0, tile_cells = 0, rank_add = 0;
};

// Jobs in flight on the host API stream: with three, the next call's passes are
// always queued behind the current one while the oldest call's ranks are being
// copied out, so the engine never idles between calls (two left a gap of the
// host's submit latency per call: 35.9 ms per n=24 step for ~32 ms of passes
// and ~32 ms of D2H).
constexpr int kJobSlots = 3;

struct Engine {
    int device = -1;
    cudaStream_t stream = nullptr;
    uint32_t *state = nullptr;
    size_t state_cap = 0;  // bytes
    int64_t *tile_base = nullptr, *tile_pos = nullptr;
    int32_t *tile_cnt = nullptr;
    size_t tile_cap = 0, tile_pos_cap = 0, tile_cnt_cap = 0;  // entries
    uint32_t *scratch = nullptr;               // tile-relative offsets of the final stage
    size_t scratch_cap = 0, scratch_want = 0;  // entries
    int64_t *tile_rank0 = nullptr;             // per tile: rank of its first cell
    size_t tile_rank0_cap = 0;                 // entries
    unsigned long long *alloc = nullptr;
    int64_t *total = nullptr;
    void *cub_tmp = nullptr;
    size_t cub_tmp_cap = 0;
    cudaStream_t stream2 = nullptr;   // copy-out stream of the pipelined host API
    cudaEvent_t chunk_ev[17] = {};
    cudaEvent_t copy_ev[17] = {};     // packed rank transfer: chunk c's D2H has landed
    uint32_t *stage32 = nullptr;      // pinned host staging of the packed offsets
    size_t stage32_cap = 0;           // entries
    int64_t *stage_pos = nullptr;     // pinned host copy of the tile positions
    size_t stage_pos_cap = 0;         // entries
    int64_t *chunk_base = nullptr;    // device running bases of the chunked final stage
    int64_t *hbase = nullptr;         // mapped pinned host mirror of chunk_base
    int hint_n = -1;
    int64_t hint_count = 0;           // prime count of the last host call (sizes the pinned output)
    uint32_t *tt_tmp = nullptr;
    size_t tt_tmp_cap = 0;  // bytes
    uint32_t *nzflags = nullptr;  // Plan::nz flags: nz_d rows then nz_e rows
    size_t nzflags_cap = 0;       // words
    void *in_tmp = nullptr;
    size_t in_tmp_cap = 0;
    int64_t *ranks = nullptr;
    size_t ranks_cap = 0;  // entries
    std::vector<PinnedBuf> free_pinned;
    // timings of the last DQMC_FLAG_TIMING call
    std::vector<std::string> pass_names;
    std::vector<float> pass_ms;
    std::vector<uint64_t> pass_bytes;
    int state_n = -1;  // n whose final bitmap is held in `state` (KEEP_BITMAP)
    uint64_t held_need = 0;  // largest device need a finished call has allocated (check_cap skips the query)
    bool attrs_set = false;
    int num_sms = 148;
    PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    AddrRangeFn addr_range = nullptr;  // cuMemGetAddressRange (IPC offsets)
    // submit/collect: at most kJobSlots jobs in flight, one slot each
    std::deque<Job> jobs;
    int64_t next_job = 0;
    void *jin[kJobSlots] = {};
    size_t jin_cap[kJobSlots] = {};  // bytes
    int64_t *jranks[kJobSlots] = {};
    size_t jranks_cap[kJobSlots] = {};  // entries
    int64_t *jpos[kJobSlots] = {};      // packed jobs: the slot's copy of the tile positions
    size_t jpos_cap[kJobSlots] = {};    // entries
    int64_t *jcount_host = nullptr;  // pinned, one count per slot
    cudaEvent_t jev[kJobSlots] = {};
    // ordering between entry points: every call that enqueues work on the
    // engine's workspace waits for this event first and records it after, so
    // the host API stream, caller streams and graph replays never overlap on
    // the shared buffers (state, scratch, tile arrays, counters)
    cudaEvent_t last_use = nullptr;
    // bumped whenever a workspace buffer is (re)allocated or released:
    // captured CUDA graphs hold raw pointers and must not replay across it
    uint64_t generation = 1;
    // gather finish (Plan::nz): taken when pass C wrote at most this many
    // nonzero blocks per 1000 (dqmc_gather_threshold; 0 = never, 1000 = always)
    int gather_permille = kGatherPermille;
    int gather_n = -1;                         // n of the last call whose pass C counted blocks
    unsigned long long gather_limit_last = 0;  // its limit
};

extern Engine g_eng;

template <typename T>
int grow(T *&ptr, size_t &cap, size_t need, size_t elem) {
    if (need <= cap && ptr) return DQMC_OK;
    if (ptr) {
        cudaFree(ptr);
        ptr = nullptr;
        cap = 0;
    }
    cudaError_t e = cudaMalloc((void **)&ptr, need * elem);
    if (e != cudaSuccess) {
        (void)cudaGetLastError();
        ptr = nullptr;
        char buf[256];
        snprintf(buf, sizeof buf, "device allocation of %llu bytes failed: %s", (unsigned long long)(need * elem),
                 cudaGetErrorString(e));
        return set_err(DQMC_ERR_RESOURCE, buf);
    }
    cap = need;
    g_eng.generation++;
    return DQMC_OK;
}

struct Timer {
    bool on;
    cudaStream_t s;
    std::vector<cudaEvent_t> ev;
    std::vector<std::string> names;
    std::vector<uint64_t> bytes;
    void mark(const char *name, uint64_t b) {
        if (g_debug) {
            cudaError_t e = cudaStreamSynchronize(s);
            if (e != cudaSuccess) {
                fprintf(stderr, "[dqmc debug] %s failed: %s\n", name, cudaGetErrorString(e));
                fflush(stderr);
            }
        }
        if (!on) return;
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, s);
        ev.push_back(e);
        names.push_back(name);
        bytes.push_back(b);
    }
    void begin() {
        if (!on) return;
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, s);
        ev.push_back(e);
    }
    void finish() {
        if (!on) return;
        cudaEventSynchronize(ev.back());
        g_eng.pass_names.clear();
        g_eng.pass_ms.clear();
        g_eng.pass_bytes.clear();
        for (size_t i = 1; i < ev.size(); i++) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, ev[i - 1], ev[i]);
            g_eng.pass_ms.push_back(ms);
            g_eng.pass_names.push_back(names[i - 1]);
            g_eng.pass_bytes.push_back(bytes[i - 1]);
        }
        for (auto e : ev) cudaEventDestroy(e);
        ev.clear();
    }
};

// engine (dqmc_engine.cu)
int ensure_device();
int ensure_attrs();
int ensure_encode();
uint64_t state_bytes_ref(int n, int h);
int validate(int n, int h);
// serialise `s` behind every earlier use of the engine workspace; call
// engine_done(s) after the last enqueue that touches it
int engine_begin(cudaStream_t s);
int engine_done(cudaStream_t s);

int alloc_pinned(size_t entries, PinnedBuf &out);  // pinned host pool (dqmc_free_result returns to it)
void sparse_release();                              // the sparse engine's buffers (dqmc_sparse.cu)

// input (dqmc_input.cu)
int input_words(const void *in, int kind, int n, const uint32_t **tt32, cudaStream_t s);

// merge passes A, B (dqmc_merge.cu)
int merge_set_attrs();
int run_merge(const Plan &p, const uint32_t *tt32, uint32_t *state, bool full, Timer &tm, cudaStream_t s);

// reduce passes C, D (dqmc_reduce.cu)
int reduce_set_attrs();
// nbatch: that many consecutive independent states of this plan (reduce-only)
int run_reduce(const Plan &p, uint32_t *state, bool fused, Timer &tm, cudaStream_t s, int64_t nbatch = 1);
// timing mode: bytes of the zero-skip passes D and E as really moved
int nz_account(const Plan &p, Timer &tm, cudaStream_t s);

// final stage E (dqmc_final.cu)
int final_set_attrs();
unsigned long long gather_limit(const Plan &p);
struct FinalOpts {
    uint32_t *bitmap_out = nullptr;         // write the final bitmap (reference layout)
    int64_t *count_dev = nullptr;           // DQMC_FLAG_ASYNC: publish the count here, no host sync
    int64_t nbatch = 1;                     // consecutive independent states (sharded super-blocks)
    const uint64_t *kill_tab = nullptr;     // per state: kMaxKill parent addresses (FinalArgs.kill_tab)
    const int64_t *rank_add_tab = nullptr;  // per state: rank of its first cell
    bool skip_c0 = false;                   // the C0 axes are already reduced
    uint32_t *packed32 = nullptr;           // multi-tile: write rank-ordered 4-byte tile offsets here (cap entries)
                                            // instead of int64 ranks (the host widens them, dqmc_hostpack.cpp)
    int64_t *slot_start = nullptr;          // per state: offset / count of its ranks in the output
    int64_t *slot_count = nullptr;
};
int run_final(const Plan &p, const uint32_t *tt32, const uint32_t *state, uint32_t ib_mask, int64_t rank_add,
              int64_t *ranks, int64_t cap, bool count_only, const FinalOpts &o, int64_t *count, Timer &tm,
              cudaStream_t s);
int run_final_retry(const Plan &p, const uint32_t *tt32, const uint32_t *state, uint32_t ib_mask, int64_t rank_add,
                    int64_t *ranks, int64_t cap, bool count_only, const FinalOpts &o, int64_t *count, Timer &tm,
                    cudaStream_t s);
int run_final_pipelined(const Plan &p, const uint32_t *state, int64_t *host, int64_t host_cap, int64_t *count,
                        bool *host_ok, cudaStream_t s);

// results of at least this many ranks (32 MB of int64) take the chunked,
// packed host paths; smaller ones one plain int64 copy
constexpr int64_t kPackedMinRanks = (int64_t)1 << 22;
int grow_pinned(void **ptr, size_t &cap, size_t need, size_t elem);  // pinned host staging (kept until release)
// dqmc_hostpack.cpp: widen packed tile offsets to int64 ranks on the host thread pool
void host_widen(const uint32_t *off32, int64_t *out, const int64_t *pos, int64_t add, int64_t end, int64_t t0,
                int64_t t1, int64_t tile_cells, int64_t rank_add);
int host_widen_threads(int n);

}  // namespace dqmc
