// dqmc.cu — B200 (sm_100a) dense prime-implicant engine + C ABI (include/dqmc.h).
//
// Replaces the reference dense path (/root/reference/pkg/src/implicants/
// dense.py:340-418): load -> MERGE all dims -> REDUCE all dims -> extract.
// Design: the 3^(n-5) blocks of the reference layout are
// swept in a handful of HBM passes instead of the reference's 2(n-5)+1:
//
//   pass A  k_c0_merge          : truth table -> blocks, in-block MERGE + the C0
//                                 block axes (contiguous 3^g-block tiles in smem);
//                                 only top-binary tiles are produced.
//   pass B  k_strided<MERGE_ONLY>: one group of <= 6 higher block axes, reads the
//                                 group's binary rows, writes its star rows.
//   pass C  k_merge_reduce_pipe  : last group: MERGE then REDUCE of the group
//                                 (+ an in-block axis); TMA gather of the binary
//                                 rows, TMA stores of every row (load / compute /
//                                 store warps).
//   pass D  k_strided_pipe<REDUCE_ONLY>: REDUCE of the other groups + 4 in-block
//                                 axes; TMA tiles, one producer warp.
//   pass E  k_c0_final           : REDUCE of the C0 axes, popcounts, per-tile
//                                 scratch reservation and ordered compaction;
//                                 then a CUB scan + k_reorder place the ranks.
// Groups under 6 axes pack several adjacent 128-B columns per tile (pipe_cols).
// Small n (<= 12): one CTA does A+E on a single smem tile (k_small).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
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
#include <mutex>
#include <string>
#include <vector>

#include "../../include/dqmc.h"
#include "dqmc_device.cuh"

using namespace dqmc;

namespace {

constexpr int kC0Max = 7;        // block axes in the contiguous tile (3^7 blocks = 68.3 KiB)
constexpr int kC0MaxBlocks = 2187;  // 3^kC0Max
constexpr int kGroupMax = 6;     // block axes per strided pass (3^6 rows x 128 B = 91 KiB)
constexpr int kRowBlocks = 4;    // blocks per strided row (128 B)
constexpr int kStridedThreads = 288;  // 9 warps: 27 sub-cube tasks per round divide evenly
constexpr int kTileThreads = 224;  // 7 warps: the 4+3 C0 rounds divide into 1 and 3 tasks/thread
// pass E: 12 warps x 3 CTAs (smem-limited) = 36 warps/SM to hide LDS/shuffle
// latency; 56 registers/thread is the most that still fits 3 CTAs.
constexpr int kFinalThreads = 384;

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

// ---------------------------------------------------------------------------
// input conversion

// DQMC_IN_U8 -> 32-bit truth-table words (on ∪ dc, ternary.py:210-218), n >= 5
__global__ void k_u8_to_words(const uint8_t *__restrict__ v, uint32_t *__restrict__ out, int64_t nwords) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = (gridDim.x * (int64_t)blockDim.x) >> 5;
    for (int64_t w = warp; w < nwords; w += nwarps) {
        const unsigned bits = __ballot_sync(0xffffffffu, v[w * 32 + lane] != 0);
        if (lane == 0) out[w] = bits;
    }
}

// n < 5: pad with dummy variables n+1..5 (primes of f' = primes of f with '*'
// appended, rank shifted by 3^5 - 3^n): the 2^n-bit table is replicated.
__global__ void k_pad_small(const void *in, int kind, int n, uint32_t *out) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    uint32_t pat = 0;
    const int npts = 1 << n;
    for (int x = 0; x < npts; x++) {
        int bit;
        if (kind == DQMC_IN_U8)
            bit = ((const uint8_t *)in)[x] != 0;
        else
            bit = (int)((((const uint64_t *)in)[0] >> x) & 1ull);
        pat |= (uint32_t)bit << x;
    }
    uint32_t w = 0;
    for (int p = 0; p < 32; p++) w |= ((pat >> (p % npts)) & 1u) << p;
    out[0] = w;
}

// splitmix64 finaliser (ttio.py:331-338)
__device__ __forceinline__ uint64_t mix64(uint64_t x) {
    x ^= x >> 30;
    x *= 0xBF58476D1CE4E5B9ull;
    x ^= x >> 27;
    x *= 0x94D049BB133111EBull;
    x ^= x >> 31;
    return x;
}

// three-way generator: value of point x from the frozen
// counter generator mix(seed + (x+1)*GAMMA) >> 11 (ttio.py:341-343, 365-374)
__global__ void k_gen3(uint8_t *__restrict__ out, int64_t x0, int64_t npts, uint64_t seed, uint64_t t_on,
                       uint64_t t_any) {
    const int64_t stride = gridDim.x * (int64_t)blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < npts; i += stride) {
        const uint64_t x = (uint64_t)(x0 + i);
        const uint64_t u = mix64(seed + (x + 1) * 0x9E3779B97F4A7C15ull) >> 11;
        out[i] = u < t_on ? 1 : (u < t_any ? 2 : 0);
    }
}

// config 3 S-box table: one CTA of 1024 threads ranks the 1024 generator
// values (stable: ties by index), P[rank(i)] = i, then clears v[x | P(x) << 10]
// (the table was set to 1 beforehand).
__global__ void __launch_bounds__(1024) k_sbox(uint8_t *__restrict__ v, uint64_t seed) {
    __shared__ uint64_t val[1024];
    __shared__ uint16_t perm[1024];
    const int i = threadIdx.x;
    val[i] = mix64(seed + ((uint64_t)i + 1) * 0x9E3779B97F4A7C15ull);
    __syncthreads();
    const uint64_t me = val[i];
    int rank = 0;
    for (int j = 0; j < 1024; j++) {
        const uint64_t o = val[j];
        rank += (o < me) || (o == me && j < i);
    }
    perm[rank] = (uint16_t)i;
    __syncthreads();
    v[i | ((int)perm[i] << 10)] = 0;
}

// ---------------------------------------------------------------------------
// contiguous C0 tile: 3^g blocks x 8 words in shared memory

// MERGE of the C0 block axes on a tile whose 2^g binary blocks are loaded:
// minimal-work order, each star block computed once (3^g - 2^g ANDs).
__device__ void tile_merge_c0(uint32_t *sm, int g) {
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

// REDUCE along C0 axes [j0, j0+K) with register sub-cubes, lane = word.
template <int K>
__device__ void tile_reduce_axes(uint32_t *sm, int g, int j0) {
    constexpr int N = P3<K>::v;
    const int sj = (int)pow3l(j0);
    const int span = sj * N;
    const int nhi = (int)pow3l(g) / span;
    const int ntask = sj * nhi * 8;
    for (int t = threadIdx.x; t < ntask; t += blockDim.x) {
        const int w = t & 7, q = t >> 3;
        const int lo = q % sj, hi = q / sj;
        const int blk = lo + hi * span;
        uint32_t v[N];
#pragma unroll
        for (int i = 0; i < N; i++) v[i] = sm[(blk + i * sj) * 8 + w];
        cube_reduce_par<K>(v);
#pragma unroll
        for (int i = 0; i < N; i++) sm[(blk + i * sj) * 8 + w] = v[i];
    }
    __syncthreads();
}

__device__ void tile_reduce_c0(uint32_t *sm, int g) {
    int j = 0;
    while (g - j >= 3) {
        tile_reduce_axes<3>(sm, g, j);
        j += 3;
    }
    if (g - j == 2) tile_reduce_axes<2>(sm, g, j);
    if (g - j == 1) tile_reduce_axes<1>(sm, g, j);
}

struct FinalArgs {
    int64_t *out;               // scratch (multi-tile) or final ranks (single tile); null = count only
    int64_t cap;                // capacity of out
    int64_t rank_add;           // added to every rank (dummy-variable padding < 0, top-block offset > 0)
    const uint32_t *kill;       // optional: cells to clear after the low reduce (kills from top parents)
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
};


// In-block reduce, popcount and ordered compaction of one tile
// (dense.py:376-397 extract_ranks: rank = block*243 + bit; memory order is
// rank order, so the output needs no sort). Warp w owns the contiguous block
// range [b0, b1); lane l takes blocks b0+l, b0+l+32, ... (group j = the j-th
// 32 blocks). Block counts stay in registers, two 16-bit fields per word, so
// one packed warp scan serves every group: the phases are short latency
// chains, which is what bounds this pass (3 CTAs/SM, smem-limited).
template <int NT>
__device__ void tile_finish(uint32_t *sm, int nb, int64_t tile, int64_t blk0, const FinalArgs &fa) {
    constexpr int kMaxIter = ((kC0MaxBlocks + NT / 32 - 1) / (NT / 32) + 31) / 32;  // ceil(max warp range / 32)
    constexpr int kPk = (kMaxIter + 1) / 2;
    __shared__ int64_t s_warp_off[NT / 32];
    __shared__ int64_t s_tile_off;
    __shared__ uint16_t s_cnt[NT / 32][kMaxIter][32];  // slow-path block popcounts, then the emission list
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nwarps = blockDim.x >> 5;
    const int b0 = (int)((int64_t)nb * warp / nwarps), b1 = (int)((int64_t)nb * (warp + 1) / nwarps);
    const int h = (lane >> 2) & 1;  // half-swap: conflict-free LDS.128 at 32-B lane stride

    // (1) lane = block: popcount (+ in-block axes, kills, bitmap on the slow path)
    uint32_t pk[kPk];
#pragma unroll
    for (int i = 0; i < kPk; i++) pk[i] = 0;
    if (!fa.ib_mask && !fa.kill && !fa.bitmap_out) {  // count only: word order does not matter
#pragma unroll
        for (int j = 0; j < kMaxIter; j++) {
            const int b = b0 + 32 * j + lane;
            if (b < b1) {
                const uint4 *p = reinterpret_cast<const uint4 *>(sm + b * 8);
                const uint4 x0 = p[h], x1 = p[h ^ 1];
                const uint32_t cj = __popc(x0.x) + __popc(x0.y) + __popc(x0.z) + __popc(x0.w) + __popc(x1.x) +
                                    __popc(x1.y) + __popc(x1.z) + __popc(x1.w);
                pk[j >> 1] |= cj << (16 * (j & 1));
            }
        }
    } else {
        // rolled (the in-block code is large: the kernel must stay inside the instruction cache)
#pragma unroll 1
        for (int j = 0; j < kMaxIter; j++) {
            const int b = b0 + 32 * j + lane;
            int cj = 0;
            if (b < b1) {
                uint4 *p = reinterpret_cast<uint4 *>(sm + b * 8);
                const uint4 ya = p[h], yb = p[h ^ 1];
                uint4 x0 = h ? yb : ya, x1 = h ? ya : yb;
                if (fa.ib_mask) {
                    uint32_t v[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
                    inblock_reduce(v, fa.ib_mask);
                    x0 = make_uint4(v[0], v[1], v[2], v[3]);
                    x1 = make_uint4(v[4], v[5], v[6], v[7]);
                }
                if (fa.kill) {
                    const uint4 *kq = reinterpret_cast<const uint4 *>(fa.kill + (blk0 + b) * 8);
                    const uint4 k0 = kq[0], k1 = kq[1];
                    x0 = make_uint4(x0.x & ~k0.x, x0.y & ~k0.y, x0.z & ~k0.z, x0.w & ~k0.w);
                    x1 = make_uint4(x1.x & ~k1.x, x1.y & ~k1.y, x1.z & ~k1.z, x1.w & ~k1.w);
                }
                if (fa.ib_mask || fa.kill) {
                    p[h] = h ? x1 : x0;
                    p[h ^ 1] = h ? x0 : x1;
                }
                if (fa.bitmap_out) {
                    uint4 *q = reinterpret_cast<uint4 *>(fa.bitmap_out + (blk0 + b) * 8);
                    q[0] = x0;
                    q[1] = x1;
                }
                cj = __popc(x0.x) + __popc(x0.y) + __popc(x0.z) + __popc(x0.w) + __popc(x1.x) + __popc(x1.y) +
                     __popc(x1.z) + __popc(x1.w);
            }
            s_cnt[warp][j][lane] = (uint16_t)cj;
        }
        __syncwarp();
#pragma unroll
        for (int j = 0; j < kMaxIter; j++) pk[j >> 1] |= (uint32_t)s_cnt[warp][j][lane] << (16 * (j & 1));
    }

    // (2) packed inclusive warp scan (fields <= 32 * 243 < 2^16: no carries
    //     between fields), group bases, the warp's total
    uint32_t inc[kPk];
#pragma unroll
    for (int i = 0; i < kPk; i++) inc[i] = pk[i];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
        for (int i = 0; i < kPk; i++) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, inc[i], o);
            if (lane >= o) inc[i] += y;
        }
    }
    int gbase[kMaxIter];
    int wsum = 0;
#pragma unroll
    for (int i = 0; i < kPk; i++) {
        const uint32_t t = __shfl_sync(0xffffffffu, inc[i], 31);
        gbase[2 * i] = wsum;
        wsum += (int)(t & 0xffffu);
        if (2 * i + 1 < kMaxIter) {
            gbase[2 * i + 1] = wsum;
            wsum += (int)(t >> 16);
        }
    }
    if (lane == 0) s_warp_off[warp] = wsum;
    __syncthreads();

    // (3) reserve this tile's range in the scratch output with one atomic (no
    //     waiting on other tiles); k_scan_tiles + k_reorder restore rank order.
    if (threadIdx.x == 0) {
        int64_t acc = 0;
        for (int w = 0; w < nwarps; w++) {
            const int64_t c = s_warp_off[w];
            s_warp_off[w] = acc;
            acc += c;
        }
        const int64_t base = acc ? (int64_t)atomicAdd(fa.alloc, (unsigned long long)acc) : 0;
        fa.tile_base[tile] = base;
        fa.tile_cnt[tile] = (int32_t)acc;
        s_tile_off = base;
    }
    __syncthreads();
    if (fa.out == nullptr) return;

    // (4) ordered emission. Primes are sparse (~0.2 per block at n = 24, ~5
    //     nonzero blocks per 32-block group), so the nonzero blocks of the
    //     warp's range are first compacted into a list (ballot + prefix;
    //     s_cnt is free again), then processed 32 at a time with every lane
    //     busy: reload the block, popcount, one warp scan for the positions,
    //     walk the set bits. Stores of one step ascend with the lane and coalesce.
    const int64_t off = s_tile_off + s_warp_off[warp];
    uint16_t *lst = &s_cnt[warp][0][0];  // kMaxIter * 32 entries >= the warp's range
    const uint32_t lt = (1u << lane) - 1u;
    int n = 0;
#pragma unroll
    for (int j = 0; j < kMaxIter; j++) {
        const uint32_t c = (pk[j >> 1] >> (16 * (j & 1))) & 0xffffu;
        const uint32_t m = __ballot_sync(0xffffffffu, c != 0);
        if (c) lst[n + __popc(m & lt)] = (uint16_t)(32 * j + lane);
        n += __popc(m);
    }
    __syncwarp();
    int64_t run = off;
#pragma unroll 1
    for (int e0 = 0; e0 < n; e0 += 32) {
        const int e = e0 + lane;
        uint32_t wv[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
        int cnt = 0, b = 0;
        if (e < n) {
            b = b0 + lst[e];
            const uint4 *p = reinterpret_cast<const uint4 *>(sm + b * 8);
            const uint4 x0 = p[0], x1 = p[1];
            wv[0] = x0.x, wv[1] = x0.y, wv[2] = x0.z, wv[3] = x0.w;
            wv[4] = x1.x, wv[5] = x1.y, wv[6] = x1.z, wv[7] = x1.w;
#pragma unroll
            for (int k = 0; k < 8; k++) cnt += __popc(wv[k]);
        }
        int incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        int64_t pos = run + (incl - cnt);
        run += __shfl_sync(0xffffffffu, incl, 31);
        const int64_t rbase = (blk0 + b) * 243 + fa.rank_add;
        int64_t *o = fa.out + pos;
        if (pos + cnt <= fa.cap) {
            // walk only the nonzero words (most blocks hold one or two): their
            // mask from the registers, the words themselves re-read from smem
            uint32_t nz = 0;
#pragma unroll
            for (int k = 0; k < 8; k++) nz |= (wv[k] != 0u ? 1u : 0u) << k;
            const uint32_t *bw = sm + b * 8;
            while (nz) {
                const int k = __ffs(nz) - 1;
                nz &= nz - 1;
                uint32_t w = bw[k];
                do {
                    *o++ = rbase + k * 32 + (__ffs(w) - 1);
                    w &= w - 1;
                } while (w);
            }
        } else {  // the scratch is too small: write what fits (the host grows it and reruns)
#pragma unroll
            for (int k = 0; k < 8; k++) {
                uint32_t w = wv[k];
                while (w) {
                    if (pos < fa.cap) fa.out[pos] = rbase + k * 32 + (__ffs(w) - 1);
                    pos++;
                    w &= w - 1;
                }
            }
        }
    }
}

// Exclusive scan of the per-tile counts (one CTA) -> rank-order positions and
// the total prime count.
__global__ void __launch_bounds__(1024) k_scan_tiles(const int32_t *__restrict__ cnt, int64_t *__restrict__ pos,
                                                     int64_t n, int64_t *total) {
    __shared__ int64_t s_part[1024];
    const int t = threadIdx.x;
    const int64_t per = (n + blockDim.x - 1) / blockDim.x;
    const int64_t lo = min(n, t * per), hi = min(n, lo + per);
    int64_t acc = 0;
    for (int64_t i = lo; i < hi; i++) acc += cnt[i];
    s_part[t] = acc;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {
        const int64_t y = t >= o ? s_part[t - o] : 0;
        __syncthreads();
        s_part[t] += y;
        __syncthreads();
    }
    int64_t run = s_part[t] - acc;
    for (int64_t i = lo; i < hi; i++) {
        pos[i] = run;
        run += cnt[i];
    }
    if (t == blockDim.x - 1) *total = s_part[t];
}

// chunk pipeline: next = cur + pos[last] + cnt[last] (device-side running base)
__global__ void k_chunk_advance(const int32_t *__restrict__ cnt_last, const int64_t *__restrict__ pos_last,
                                int64_t *base, volatile int64_t *host_mirror) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        const int64_t b0 = base[0], b1 = b0 + *pos_last + *cnt_last;
        base[1] = b1;
        host_mirror[0] = b0;  // mapped pinned memory: the host reads it after the chunk event
        host_mirror[1] = b1;
    }
}

// total = pos[n-1] + cnt[n-1] after the exclusive scan
__global__ void k_scan_total(const int32_t *__restrict__ cnt, const int64_t *__restrict__ pos, int64_t n,
                             int64_t *total) {
    if (threadIdx.x == 0 && blockIdx.x == 0) *total = n ? pos[n - 1] + cnt[n - 1] : 0;
}

// Copy every tile's ranks from its scratch range to its rank-order position
// (one warp per tile, coalesced 8-B copies).
// DQMC_FLAG_ASYNC: publish the count in stream order; -(count + 1) flags an
// incomplete rank list (output or scratch too small).
__global__ void k_publish_count(const int64_t *__restrict__ total, int64_t limit, int64_t *__restrict__ dst) {
    const int64_t t = *total;
    *dst = t <= limit ? t : -(t + 1);
}

__global__ void __launch_bounds__(256) k_reorder(const int64_t *__restrict__ scratch, const int64_t *__restrict__ base,
                                                 const int32_t *__restrict__ cnt, const int64_t *__restrict__ pos,
                                                 int64_t *__restrict__ out, int64_t cap, int64_t ntiles,
                                                 int64_t scap, const int64_t *__restrict__ dbase = nullptr) {
    const int lane = threadIdx.x & 31;
    const int64_t add = dbase ? *dbase : 0;
    const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = (gridDim.x * (int64_t)blockDim.x) >> 5;
    for (int64_t t = w; t < ntiles; t += nw) {
        const int c = cnt[t];
        const int64_t src = base[t], dst = pos[t] + add;
        // a tile whose range overflowed the scratch is skipped: the host sees
        // total > scratch capacity, grows the scratch and reruns the final stage
        if (c < 0 || src < 0 || src + c > scap) continue;
        int i = lane;
        if (dst + c <= cap) {
            // four independent loads in flight per lane (the copy is latency-bound)
            for (; i + 96 < c; i += 128) {
                const int64_t a0 = __ldcs(scratch + src + i), a1 = __ldcs(scratch + src + i + 32);
                const int64_t a2 = __ldcs(scratch + src + i + 64), a3 = __ldcs(scratch + src + i + 96);
                out[dst + i] = a0;
                out[dst + i + 32] = a1;
                out[dst + i + 64] = a2;
                out[dst + i + 96] = a3;
            }
        }
        for (; i < c; i += 32)
            if (dst + i < cap) out[dst + i] = __ldcs(scratch + src + i);
    }
}

// wildcard count of every rank (ternary.py:139-146), stored as the sort key
// n - weight so an ascending stable radix sort yields weight-descending order
// with ranks ascending inside each weight (cli.py:134-135 ordering).
__global__ void k_weight_keys(const int64_t *__restrict__ ranks, int64_t count, int n, uint8_t *__restrict__ keys) {
    const int64_t stride = gridDim.x * (int64_t)blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += stride) {
        uint64_t r = (uint64_t)ranks[i];
        int w = 0;
        for (int k = 0; k < n; k++) {
            const uint64_t q = __umul64hi(r, 0xAAAAAAAAAAAAAAABull) >> 1;  // r / 3
            w += (r - 3 * q) == 2;
            r = q;
        }
        keys[i] = (uint8_t)(n - w);
    }
}

// dst = a & b (op 0) or a | b (op 1), 16 B per thread: the top-axis block
// ANDs of the sharded path (M_t = AND over completions) and kill accumulation.
__global__ void k_bitop(uint4 *__restrict__ dst, const uint4 *__restrict__ a, const uint4 *__restrict__ b, int64_t n16,
                        int op) {
    const int64_t stride = gridDim.x * (int64_t)blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16; i += stride) {
        const uint4 x = __ldcs(a + i), y = __ldcs(b + i);
        dst[i] = op == 0 ? make_uint4(x.x & y.x, x.y & y.y, x.z & y.z, x.w & y.w)
                         : make_uint4(x.x | y.x, x.y | y.y, x.z | y.z, x.w | y.w);
    }
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

// REDUCE along C0 axes [J0, J0+K) of a 3^G-block tile, compile-time shape.
template <int K, int G, int J0>
__device__ __forceinline__ void tile_reduce_axes_t(uint32_t *sm) {
    constexpr int N = P3<K>::v;
    constexpr int SJ = pow3i(J0);
    constexpr int SPAN = SJ * N;
    constexpr int NHI = pow3i(G) / SPAN;
    constexpr int NTASK = SJ * NHI * 8;
    // warp-uniform iterations: an all-zero warp skips its reduce (see warp_any)
    for (int t0 = (int)(threadIdx.x & ~31u); t0 < NTASK; t0 += blockDim.x) {
        const int t = t0 + (int)(threadIdx.x & 31u);
        const bool in = t < NTASK;
        const int w = t & 7, q = in ? t >> 3 : 0;
        const int lo = q % SJ, hi = q / SJ;
        const int blk = lo + hi * SPAN;
        uint32_t v[N];
#pragma unroll
        for (int i = 0; i < N; i++) v[i] = sm[(blk + i * SJ) * 8 + w];
        if (K <= 3) {  // 81-register cubes (K = 4) would spill with the vote
            if (!warp_any(v) || !in) continue;
        } else if (!in) {
            continue;
        }
        cube_reduce_par<K>(v);
#pragma unroll
        for (int i = 0; i < N; i++) sm[(blk + i * SJ) * 8 + w] = v[i];
    }
    __syncthreads();
}

template <int G, int J0>
__device__ __forceinline__ void tile_reduce_c0_t(uint32_t *sm) {
    if constexpr (G - J0 == 7) {
        tile_reduce_axes_t<4, G, J0>(sm);
        tile_reduce_c0_t<G, J0 + 4>(sm);
    } else if constexpr (G - J0 >= 3) {
        tile_reduce_axes_t<3, G, J0>(sm);
        tile_reduce_c0_t<G, J0 + 3>(sm);
    } else if constexpr (G - J0 == 2) {
        tile_reduce_axes_t<2, G, J0>(sm);
    } else if constexpr (G - J0 == 1) {
        tile_reduce_axes_t<1, G, J0>(sm);
    }
}

// Load the binary blocks of a C0 tile from the truth table and merge it.
// Tile index tb (binary over the top digits) selects 32-bit TT words
// [tb << g, (tb+1) << g): point x = x_low5 + 32*(C0 bits) + 2^(5+g)*(top bits).
__device__ void tile_build(uint32_t *sm, const uint32_t *__restrict__ tt32, int g, int64_t tb) {
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

// pass A: top-binary tiles (2^T of them), merged over in-block + C0 axes
__global__ void __launch_bounds__(kTileThreads) k_c0_merge(const uint32_t *__restrict__ tt32,
                                                           uint32_t *__restrict__ state, int g, int T, int pitch,
                                                           int pm_r) {
    extern __shared__ __align__(16) uint32_t sm[];
    const int64_t ntiles = 1ll << T;
    const int nb = (int)pow3l(g);
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        int64_t base = 0, p = pitch;  // storage block of the tile: ternary index of its top digits x pitch
        for (int k = 0; k < T; k++, p *= 3)
            if ((tile >> k) & 1) base += p;
        tile_build(sm, tt32, g, tile);
        const uint4 *src = reinterpret_cast<const uint4 *>(sm);
        if (pm_r) {
            // piece-major group 0 (make_plan): piece x of the tile lives at
            // ((upper * npieces + x) * 3^r + row0) pieces, row0 = the group-0 digits
            const int64_t nr = pow3l(pm_r), np = pitch / kRowBlocks;
            const int64_t row0 = (int64_t)bin_to_tern_rt((uint64_t)(tile & ((1ll << pm_r) - 1)));
            const int64_t upper = (int64_t)bin_to_tern_rt((uint64_t)(tile >> pm_r));
            uint4 *dst = reinterpret_cast<uint4 *>(state) + ((upper * np) * nr + row0) * 8;
            for (int t = threadIdx.x; t < pitch * 2; t += blockDim.x)
                dst[(int64_t)(t >> 3) * nr * 8 + (t & 7)] = t < nb * 2 ? src[t] : make_uint4(0, 0, 0, 0);
        } else {
            uint4 *dst = reinterpret_cast<uint4 *>(state + base * 8);
            for (int t = threadIdx.x; t < pitch * 2; t += blockDim.x) dst[t] = t < nb * 2 ? src[t] : make_uint4(0, 0, 0, 0);
        }
        __syncthreads();
    }
}

// pass E: one CTA per C0 tile (3^G blocks), tiles taken in rank order by
// ticket; the tile arrives in shared memory with one TMA bulk copy.
__device__ __forceinline__ void tma_load_4d(void *dst, const CUtensorMap *map, int c0, int c1, int c2, int c3,
                                            uint64_t *mbar);
__device__ __forceinline__ void tma_prefetch_4d(const CUtensorMap *map, int c0, int c1, int c2, int c3);

template <int G>
__global__ void __launch_bounds__(kFinalThreads, 3)
    k_c0_final(const uint32_t *__restrict__ state, FinalArgs fa, const __grid_constant__ CUtensorMap ma,
               const __grid_constant__ CUtensorMap mb) {
    extern __shared__ __align__(128) uint32_t sm_raw[];
    __shared__ __align__(8) uint64_t mbar;
    constexpr int NB = pow3i(G);
    // tensor-map destinations need 128-B alignment; the dynamic window follows
    // this kernel's static arrays (the launch reserves 128 B for the shift)
    uint32_t *sm = sm_raw + (fa.pm_nr ? ((128u - (smem_u32(sm_raw) & 127u)) & 127u) >> 2 : 0u);
    const int64_t tile = blockIdx.x + fa.tile0;
    const int64_t blk0 = tile * NB;  // logical (rank) block
    const int64_t pitch = fa.pitch ? fa.pitch : NB;
    const uint32_t *src = state + tile * pitch * 8;
    if (threadIdx.x == 0 && fa.pm_nr) {
        // piece-major group 0: the tile is pm_np pieces 3^r pieces apart; boxes
        // of 256 pieces (map ma) and one remainder box (map mb)
        mbar_init(&mbar, 1);
        mbar_expect_tx(&mbar, fa.pm_np * 128);
        const int nfull = fa.pm_np >> 8, rem = fa.pm_np & 255;
        const int q1 = (int)(tile % fa.pm_nr), up = (int)(tile / fa.pm_nr);
        for (int j = 0; j < nfull; j++) tma_load_4d(sm + j * 256 * 32, &ma, 0, 256 * j, q1, up, &mbar);
        if (rem) tma_load_4d(sm + nfull * 256 * 32, &mb, 0, 256 * nfull, q1, up, &mbar);
        const int pf = (int)blockIdx.x + fa.prefetch;
        if (fa.prefetch > 0 && pf < (int)gridDim.x) {
            const int64_t t2 = tile + fa.prefetch;
            const int q1b = (int)(t2 % fa.pm_nr), upb = (int)(t2 / fa.pm_nr);
            for (int j = 0; j < nfull; j++) tma_prefetch_4d(&ma, 0, 256 * j, q1b, upb);
            if (rem) tma_prefetch_4d(&mb, 0, 256 * nfull, q1b, upb);
        }
    } else if (threadIdx.x == 0) {
        mbar_init(&mbar, 1);
        mbar_expect_tx(&mbar, NB * 32);
        bulk_g2s(sm, src, NB * 32, &mbar);
        // warm L2 for the CTA that will take this slot a generation later
        // (CTAs start roughly in tile order, ~3 per SM resident)
        const int pf = (int)blockIdx.x + fa.prefetch;
        if (fa.prefetch > 0 && pf < (int)gridDim.x)
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src + (int64_t)fa.prefetch * pitch * 8),
                         "r"(NB * 32)
                         : "memory");
    }
    __syncthreads();
    mbar_wait(&mbar, 0);
    tile_reduce_c0_t<G, 0>(sm);
    tile_finish<kFinalThreads>(sm, NB, tile, blk0, fa);
}

// n <= 12: the whole problem is one tile; one CTA does A and E.
__global__ void __launch_bounds__(kTileThreads) k_small(const uint32_t *__restrict__ tt32, int g, FinalArgs fa) {
    extern __shared__ __align__(16) uint32_t sm[];
    tile_build(sm, tt32, g, 0);
    tile_reduce_c0(sm, g);
    tile_finish<kTileThreads>(sm, (int)pow3l(g), 0, 0, fa);
}

// ---------------------------------------------------------------------------
// strided group pass: R = R1 + R2 block axes at block stride Q = 3^a.
// Tile = 3^R rows x 4 blocks (128 B); row rho = rho1 + 3^R1 * rho2.
// Work item = (outer, column); lane = word within the 128-B row.

template <int R1, int R2, int MODE>
__global__ void __launch_bounds__(kStridedThreads) k_strided(uint32_t *__restrict__ state, int64_t Q, int64_t ncol,
                                                             int64_t nitems, uint32_t ib_mask, int64_t rs, int64_t cs,
                                                             int64_t os) {
    constexpr int N1 = P3<R1>::v, N2 = P3<R2>::v, B1 = 1 << R1, B2 = 1 << R2;
    constexpr int NR = N1 * N2;
    extern __shared__ __align__(16) uint32_t sm[];  // NR rows x 32 words
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nwarps = blockDim.x >> 5;
    // strides in blocks: row rs, column cs, outer os (reference layout: Q, 4,
    // 3^R Q; piece-major group 0: 4, 3^R 4, pitch 3^R)
    const int64_t Qw = rs * 8;  // row stride in words

    for (int64_t item = blockIdx.x; item < nitems; item += gridDim.x) {
        const int64_t col = item % ncol;
        const int64_t outer = item / ncol;
        const int64_t ob = (MODE == MERGE_ONLY) ? bin_to_tern_rt((uint64_t)outer) : outer;
        const int64_t c0 = col * kRowBlocks;
        const int valid = (int)min((int64_t)kRowBlocks, Q - c0) * 8;
        const bool act = lane < valid;
        uint32_t *g0 = state + (ob * os + col * cs) * 8 + lane;  // word of row 0
        // in-block round needed?
        const bool ib = (MODE != MERGE_ONLY) && ib_mask != 0;

        if (MODE == MERGE_ONLY || MODE == MERGE_REDUCE) {
            // round 1: for each binary rho2, merge the R1 axes
            for (int t2 = warp; t2 < B2; t2 += nwarps) {
                const int r2 = (int)bin_to_tern_rt((uint64_t)t2);
                uint32_t v[N1];
#pragma unroll
                for (int i = 0; i < N1; i++) v[i] = 0;
#pragma unroll
                for (int b = 0; b < B1; b++) {
                    const int r1 = bin_to_tern(b);
                    v[r1] = act ? g0[(int64_t)(r1 + N1 * r2) * Qw] : 0u;
                }
                cube_merge<R1>(v);
                if (MODE == MERGE_REDUCE && R2 == 0) {
                    cube_reduce_par<R1>(v);
#pragma unroll
                    for (int i = 0; i < N1; i++) {
                        if (ib)
                            sm[(i + N1 * r2) * 32 + lane] = v[i];
                        else if (act)
                            g0[(int64_t)(i + N1 * r2) * Qw] = v[i];
                    }
                } else {
#pragma unroll
                    for (int i = 0; i < N1; i++) {
                        if (MODE == MERGE_ONLY && has_star(i, R1) && act) g0[(int64_t)(i + N1 * r2) * Qw] = v[i];
                        if (R2 > 0) sm[(i + N1 * r2) * 32 + lane] = v[i];
                    }
                }
            }
            __syncthreads();
            if (R2 > 0) {
                // round 2: for each rho1, merge the R2 axes (+ reduce them)
                for (int t1 = warp; t1 < N1; t1 += nwarps) {
                    uint32_t v[N2];
#pragma unroll
                    for (int i = 0; i < N2; i++) v[i] = 0;
#pragma unroll
                    for (int b = 0; b < B2; b++) {
                        const int r2 = bin_to_tern(b);
                        v[r2] = sm[(t1 + N1 * r2) * 32 + lane];
                    }
                    cube_merge<R2>(v);
                    if (MODE == MERGE_ONLY) {
#pragma unroll
                        for (int i = 0; i < N2; i++)
                            if (has_star(i, R2) && act) g0[(int64_t)(t1 + N1 * i) * Qw] = v[i];
                    } else {
                        cube_reduce_par<R2>(v);
                        __syncwarp();
#pragma unroll
                        for (int i = 0; i < N2; i++) sm[(t1 + N1 * i) * 32 + lane] = v[i];
                    }
                }
                __syncthreads();
                if (MODE == MERGE_REDUCE) {
                    // round 3: reduce the R1 axes
                    for (int t2 = warp; t2 < N2; t2 += nwarps) {
                        uint32_t v[N1];
#pragma unroll
                        for (int i = 0; i < N1; i++) v[i] = sm[(i + N1 * t2) * 32 + lane];
                        cube_reduce_par<R1>(v);
#pragma unroll
                        for (int i = 0; i < N1; i++) {
                            if (ib)
                                sm[(i + N1 * t2) * 32 + lane] = v[i];
                            else if (act)
                                g0[(int64_t)(i + N1 * t2) * Qw] = v[i];
                        }
                    }
                    __syncthreads();
                }
            }
        } else {  // REDUCE_ONLY
            // round 1: reduce the R1 axes, rows straight from HBM
            for (int t2 = warp; t2 < N2; t2 += nwarps) {
                uint32_t v[N1];
#pragma unroll
                for (int i = 0; i < N1; i++) v[i] = act ? __ldcs(g0 + (int64_t)(i + N1 * t2) * Qw) : 0u;
                cube_reduce_par<R1>(v);
#pragma unroll
                for (int i = 0; i < N1; i++) {
                    if (R2 > 0 || ib)
                        sm[(i + N1 * t2) * 32 + lane] = v[i];
                    else if (act)
                        g0[(int64_t)(i + N1 * t2) * Qw] = v[i];
                }
            }
            __syncthreads();
            if (R2 > 0) {
                for (int t1 = warp; t1 < N1; t1 += nwarps) {
                    uint32_t v[N2];
#pragma unroll
                    for (int i = 0; i < N2; i++) v[i] = sm[(t1 + N1 * i) * 32 + lane];
                    cube_reduce_par<R2>(v);
                    __syncwarp();
#pragma unroll
                    for (int i = 0; i < N2; i++) {
                        if (ib)
                            sm[(t1 + N1 * i) * 32 + lane] = v[i];
                        else if (act)
                            g0[(int64_t)(t1 + N1 * i) * Qw] = v[i];
                    }
                }
                __syncthreads();
            }
        }

        if (ib) {
            // in-block axes: thread per (row, block); 32-B stores
            const int nblk_valid = valid / 8;
            for (int t = threadIdx.x; t < NR * kRowBlocks; t += blockDim.x) {
                const int row = t >> 2, b = t & 3;
                if (b >= nblk_valid) continue;
                uint4 *p = reinterpret_cast<uint4 *>(sm + row * 32 + b * 8);
                const uint4 x0 = p[0], x1 = p[1];
                uint32_t v[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
                inblock_reduce(v, ib_mask);
                uint4 *q = reinterpret_cast<uint4 *>(state + (ob * os + (int64_t)row * rs + col * cs + b) * 8);
                q[0] = make_uint4(v[0], v[1], v[2], v[3]);
                q[1] = make_uint4(v[4], v[5], v[6], v[7]);
            }
            __syncthreads();
        }
    }
}

// ---------------------------------------------------------------------------
// Pipelined strided pass D (REDUCE_ONLY): persistent CTAs, two tile buffers,
// one producer warp that streams tiles in and out with TMA (3-D tensor map:
// words x rows x outer; zero-fill / clipping handle the ragged last column
// group) while the compute warps work on the other buffer. Pass C
// (k_merge_reduce_pipe, below) gathers only the 2^R binary rows.

__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *map, int c0, int c1, int c2, uint64_t *mbar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
            "r"(smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(mbar))
        : "memory");
}

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

__device__ __forceinline__ void cp_async16(void *dst, const void *src, bool valid) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(valid ? 16 : 0)
                 : "memory");
}

__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t *mbar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(mbar)) : "memory");
}

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

// Sparse mode: see warp_any.

// In-block REDUCE of a smem tile, thread per 32-B block (plain LDS.128 pairs:
// a 2-way bank conflict costs MIO wavefronts, which have slack, where a lane
// half-swap would cost 16 ALU selects per block). Warp-uniform iterations so
// an all-zero warp can skip (sparse).
__device__ __forceinline__ void inblock_round(uint32_t *tile, int nblocks, uint32_t ib_mask, int nct, int sparse) {
    const int lane = threadIdx.x & 31;
    for (int t0 = (int)(threadIdx.x & ~31u); t0 < nblocks; t0 += nct) {
        const int t = t0 + lane;
        const bool in = t < nblocks;
        uint4 *p = reinterpret_cast<uint4 *>(tile + (in ? t : 0) * 8);
        uint4 x0 = make_uint4(0, 0, 0, 0), x1 = x0;
        if (in) x0 = p[0], x1 = p[1];
        if (sparse && !__any_sync(0xffffffffu, (x0.x | x0.y | x0.z | x0.w | x1.x | x1.y | x1.z | x1.w) != 0u)) continue;
        uint32_t v[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
        inblock_reduce(v, ib_mask);
        if (in) {
            p[0] = make_uint4(v[0], v[1], v[2], v[3]);
            p[1] = make_uint4(v[4], v[5], v[6], v[7]);
        }
    }
}

// inblock_round that also records which 128-B rows (4 blocks) of a one-column
// tile are nonzero afterwards: bit r of rowbits (smem, cleared by the caller).
__device__ __forceinline__ void inblock_round_bits(uint32_t *tile, int nblocks, uint32_t ib_mask, int nct,
                                                   uint32_t *rowbits) {
    const int lane = threadIdx.x & 31;
    for (int t0 = (int)(threadIdx.x & ~31u); t0 < nblocks; t0 += nct) {
        const int t = t0 + lane;
        const bool in = t < nblocks;
        uint4 *p = reinterpret_cast<uint4 *>(tile + (in ? t : 0) * 8);
        uint4 x0 = make_uint4(0, 0, 0, 0), x1 = x0;
        if (in) x0 = p[0], x1 = p[1];
        if (!__any_sync(0xffffffffu, (x0.x | x0.y | x0.z | x0.w | x1.x | x1.y | x1.z | x1.w) != 0u)) continue;
        uint32_t v[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
        inblock_reduce(v, ib_mask);
        if (in) {
            p[0] = make_uint4(v[0], v[1], v[2], v[3]);
            p[1] = make_uint4(v[4], v[5], v[6], v[7]);
        }
        const bool nz = (v[0] | v[1] | v[2] | v[3] | v[4] | v[5] | v[6] | v[7]) != 0u;
        const uint32_t m = __ballot_sync(0xffffffffu, in && nz);
        // lanes 4j..4j+3 hold row t0/4 + j (t0 is a multiple of 32: 8 whole rows)
        uint32_t rb = 0;
#pragma unroll
        for (int j = 0; j < 8; j++) rb |= ((m >> (4 * j)) & 0xFu) ? (1u << j) : 0u;
        const int r0 = t0 >> 2;  // multiple of 8
        if (lane == 0 && rb) atomicOr(&rowbits[r0 >> 5], rb << (r0 & 31));
    }
}

template <int R1, int R2, int MODE>
__global__ void __launch_bounds__(PipeSmem<R1, R2>::THREADS, 1)
    k_strided_pipe(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ CUtensorMap gmap,
                   int64_t ncol, int64_t nitems, uint32_t ib_mask, int pm, int sparse) {
    using SM = PipeSmem<R1, R2>;
    constexpr int N1 = SM::N1, N2 = SM::N2, B1 = 1 << R1, B2 = 1 << R2;
    constexpr int NR = SM::NR;
    constexpr int CW = SM::CW;
    constexpr int CC = pipe_cols<R1, R2>(), PITCH = SM::PITCH;
    extern __shared__ __align__(128) uint32_t smem[];
    __shared__ __align__(8) uint64_t full[2], computed[2];
    // 4-D map coordinates of an item: reference layout {col words, row, outer, 0};
    // piece-major group 0 (pm, CC = 1) {0, row, col, outer} (make_group_map4)
    auto crd = [&](int64_t it, int &c0, int &c2, int &c3) {
        const int64_t col = it % ncol, outer = it / ncol;
        c0 = pm ? 0 : (int)(col * 32 * CC);
        c2 = (int)(pm ? col : outer);
        c3 = pm ? (int)outer : 0;
    };
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // items strided over the grid: the CTAs work on adjacent columns at the same
    // time (a contiguous range per CTA measured 16.0 vs 13.9 ms at n = 24)
    const int64_t L = nitems > blockIdx.x ? (nitems - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
    auto item = [&](int64_t i) { return blockIdx.x + i * gridDim.x; };

    if (threadIdx.x == 0) {
        for (int b = 0; b < 2; b++) {
            mbar_init(&full[b], 1);
            mbar_init(&computed[b], CW);
        }
    }
    __syncthreads();

    if (warp == CW) {
        // ------------------------------ producer warp (one elected lane)
        if (lane == 0) {
            for (int64_t i = 0; i < L + 2; i++) {
                const int b = (int)(i & 1);
                uint32_t *tile = smem + b * SM::TILE_WORDS;
                const bool st = i >= 2;
                if (st) {
                    const int64_t it = item(i - 2);
                    mbar_wait(&computed[b], (unsigned)(((i - 2) >> 1) & 1));
                    int c0, c2, c3;
                    crd(it, c0, c2, c3);
#pragma unroll
                    for (int x = 0; x < SM::NBOX; x++) {  // one bulk group per box
                        tma_store_4d(&tmap, c0, x * SM::BOXR, c2, c3, tile + x * SM::BOXR * PITCH);
                        bulk_commit();
                    }
                }
                if (i < L) {
                    const int64_t it = item(i);
                    int c0, c2, c3;
                    crd(it, c0, c2, c3);
                    // each box is reloaded as soon as its store has read it out of
                    // smem: the next tile's load overlaps the previous tile's store
                    mbar_expect_tx(&full[b], SM::TILE_WORDS * 4);
                    static_assert(SM::NBOX <= 3, "box-wise store/load overlap handles <= 3 boxes");
#pragma unroll
                    for (int x = 0; x < SM::NBOX; x++) {
                        if (st) {
                            if (SM::NBOX - 1 - x == 2) bulk_wait_read<2>();
                            else if (SM::NBOX - 1 - x == 1) bulk_wait_read<1>();
                            else bulk_wait_read<0>();
                        }
                        tma_load_4d(tile + x * SM::BOXR * PITCH, &tmap, c0, x * SM::BOXR, c2, c3, &full[b]);
                    }
                }
                if (st) bulk_wait_read<0>();  // buffer b is rewritten by compute only after `full`
            }
            bulk_wait0();
        }
        return;
    }

    // ---------------------------------- compute warps
    constexpr int NCT = CW * 32;
    for (int64_t i = 0; i < L; i++) {
        const int b = (int)(i & 1);
        const int tb = b * SM::TILE_WORDS;
        mbar_wait(&full[b], (unsigned)((i >> 1) & 1));
        // round 1: reduce the R1 axes
        for (int tt = warp; tt < N2 * CC; tt += CW) {
            const int t2 = tt % N2, h = tt / N2;
            uint32_t v[N1];
#pragma unroll
            for (int x = 0; x < N1; x++) v[x] = smem[tb + (x + N1 * t2) * PITCH + 32 * h + lane];
            if (sparse && !warp_any(v)) continue;
            cube_reduce_par<R1>(v);
#pragma unroll
            for (int x = 0; x < N1; x++) smem[tb + (x + N1 * t2) * PITCH + 32 * h + lane] = v[x];
        }
        if (R2 > 0) {
            bar_compute(NCT);
            for (int tt = warp; tt < N1 * CC; tt += CW) {
                const int t1 = tt % N1, h = tt / N1;
                uint32_t v[N2];
#pragma unroll
                for (int x = 0; x < N2; x++) v[x] = smem[tb + (t1 + N1 * x) * PITCH + 32 * h + lane];
                if (sparse && !warp_any(v)) continue;
                cube_reduce_par<R2>(v);
#pragma unroll
                for (int x = 0; x < N2; x++) smem[tb + (t1 + N1 * x) * PITCH + 32 * h + lane] = v[x];
            }
        }
        if (ib_mask) {
            bar_compute(NCT);
            // in-block axes, thread per block; plain LDS.128 pairs (a 2-way bank
            // conflict costs MIO wavefronts, which have slack here; a lane
            // half-swap would cost 16 ALU selects per block on the saturated ALU pipe)
            inblock_round(&smem[tb], NR * kRowBlocks * CC, ib_mask, NCT, sparse);
        }
        fence_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&computed[b]);
    }
}

// MERGE_REDUCE pass with decoupled resources: the 2^R binary-row gathers land
// in two small stage buffers (load warp), the finished 3^R-row tiles leave
// from two tile buffers (store warp). A gather never waits for a tile store,
// so the compute warps always find the next item's rows ready.
template <int R1, int R2>
__global__ void __launch_bounds__(PipeSmem<R1, R2>::THREADS + 32, 1)
    k_merge_reduce_pipe(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ CUtensorMap gmap,
                        int64_t ncol, int64_t nitems, uint32_t ib_mask, int sparse, uint32_t *__restrict__ nzmap) {
    using SM = PipeSmem<R1, R2>;
    constexpr int N1 = SM::N1, N2 = SM::N2, B1 = 1 << R1, B2 = 1 << R2;
    constexpr int NR = SM::NR;
    constexpr int CW = SM::CW;
    constexpr int CC = pipe_cols<R1, R2>(), PITCH = SM::PITCH;
    extern __shared__ __align__(128) uint32_t smem[];
    __shared__ __align__(8) uint64_t stage_full[2], stage_free[2], tile_done[2], tile_free[2];
    __shared__ uint32_t s_rowbits[2][24];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t L = nitems > blockIdx.x ? (nitems - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;

    if (threadIdx.x < 48) s_rowbits[threadIdx.x / 24][threadIdx.x % 24] = 0u;
    if (threadIdx.x == 0) {
        for (int b = 0; b < 2; b++) {
            mbar_init(&stage_full[b], 1);
            mbar_init(&stage_free[b], CW);
            mbar_init(&tile_done[b], CW);
            mbar_init(&tile_free[b], 1);
        }
    }
    __syncthreads();

    if (warp == CW) {  // ---------------------------------- load warp
        if (lane == 0) {
            for (int64_t i = 0; i < L; i++) {
                const int b = (int)(i & 1);
                if (i >= 2) mbar_wait(&stage_free[b], (unsigned)(((i - 2) >> 1) & 1));
                const int64_t it = blockIdx.x + i * gridDim.x;
                const int c0 = (int)((it % ncol) * 32 * CC);
                uint32_t *st = smem + 2 * SM::TILE_WORDS + b * SM::STAGE_WORDS;
                mbar_expect_tx(&stage_full[b], SM::STAGE_WORDS * 4);
#pragma unroll
                for (int b2 = 0; b2 < B2; b2++)
                    tma_load_5d(st + b2 * B1 * PITCH, &gmap, c0, 0, 0, 0, bin_to_tern(b2), &stage_full[b]);
            }
        }
        return;
    }
    if (warp == CW + 1) {  // ------------------------------ store warp
        if (lane == 0) {
            for (int64_t i = 0; i < L; i++) {
                const int b = (int)(i & 1);
                const int64_t it = blockIdx.x + i * gridDim.x;
                mbar_wait(&tile_done[b], (unsigned)((i >> 1) & 1));
                const uint32_t *tile = smem + b * SM::TILE_WORDS;
                const int c0 = (int)((it % ncol) * 32 * CC);
#pragma unroll
                for (int x = 0; x < SM::NBOX; x++) tma_store_3d(&tmap, c0, x * SM::BOXR, 0, tile + x * SM::BOXR * PITCH);
                bulk_commit();
                bulk_wait_read0();
                mbar_arrive(&tile_free[b]);
            }
            bulk_wait0();
        }
        return;
    }

    // ---------------------------------------------- compute warps
    constexpr int NCT = CW * 32;
    for (int64_t i = 0; i < L; i++) {
        const int b = (int)(i & 1);
        const int tb = b * SM::TILE_WORDS;
        const int sb = 2 * SM::TILE_WORDS + b * SM::STAGE_WORDS;
        mbar_wait(&stage_full[b], (unsigned)((i >> 1) & 1));
        if (i >= 2) mbar_wait(&tile_free[b], (unsigned)(((i - 2) >> 1) & 1));
        // round 1: merge the R1 axes for each binary rho2 (stage -> tile)
        for (int tt = warp; tt < B2 * CC; tt += CW) {
                const int t2 = tt % B2, h = tt / B2;
            const int r2 = bin_to_tern(t2);
            uint32_t v[N1];
#pragma unroll
            for (int x = 0; x < N1; x++) v[x] = 0;
#pragma unroll
            for (int b1 = 0; b1 < B1; b1++) v[bin_to_tern(b1)] = smem[sb + (b1 + B1 * t2) * PITCH + 32 * h + lane];
            cube_merge<R1>(v);
            if (R2 == 0) cube_reduce_par<R1>(v);
#pragma unroll
            for (int x = 0; x < N1; x++) smem[tb + (x + N1 * r2) * PITCH + 32 * h + lane] = v[x];
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&stage_free[b]);
        if (R2 > 0) {
            bar_compute(NCT);
            for (int tt = warp; tt < N1 * CC; tt += CW) {
                const int t1 = tt % N1, h = tt / N1;
                uint32_t v[N2];
#pragma unroll
                for (int x = 0; x < N2; x++) v[x] = 0;
#pragma unroll
                for (int b2 = 0; b2 < B2; b2++) v[bin_to_tern(b2)] = smem[tb + (t1 + N1 * bin_to_tern(b2)) * PITCH + 32 * h + lane];
                cube_merge<R2>(v);
                cube_reduce_par<R2>(v);
#pragma unroll
                for (int x = 0; x < N2; x++) smem[tb + (t1 + N1 * x) * PITCH + 32 * h + lane] = v[x];
            }
        }
        if (R2 > 0) {
            bar_compute(NCT);
            for (int tt = warp; tt < N2 * CC; tt += CW) {
                const int t2 = tt % N2, h = tt / N2;
                uint32_t v[N1];
#pragma unroll
                for (int x = 0; x < N1; x++) v[x] = smem[tb + (x + N1 * t2) * PITCH + 32 * h + lane];
                if ((sparse & 1) && !warp_any(v)) continue;
                cube_reduce_par<R1>(v);
#pragma unroll
                for (int x = 0; x < N1; x++) smem[tb + (x + N1 * t2) * PITCH + 32 * h + lane] = v[x];
            }
        }
        if (ib_mask) {
            bar_compute(NCT);
            // thread per block; plain LDS.128 pairs (a 2-way bank conflict costs
            // MIO wavefronts, which have slack here; a lane half-swap would cost
            // 16 ALU selects per block on the saturated ALU pipe)
            if (nzmap)
                inblock_round_bits(&smem[tb], NR * kRowBlocks * CC, ib_mask, NCT, s_rowbits[b]);
            else
                inblock_round(&smem[tb], NR * kRowBlocks * CC, ib_mask, NCT, sparse & 1);
        }
        if (nzmap) {
            // nonzero-row bits of this item (one column: CC = 1) in item-major
            // order, nzmap[item * 24 + w]; k_bits_transpose reorders them for pass D
            bar_compute(NCT);
            if (warp == 0 && lane < 24) {
                const int64_t it = blockIdx.x + i * gridDim.x;
                nzmap[it * 24 + lane] = s_rowbits[b][lane];
                s_rowbits[b][lane] = 0u;
            }
        }
        fence_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tile_done[b]);
    }
}

__global__ void k_popc_sum(const uint32_t *__restrict__ w, int64_t n, unsigned long long *out) {
    unsigned long long acc = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        acc += __popc(w[i]);
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0 && acc) atomicAdd(out, acc);
}

// Row bits of pass C, item-major (src[p * 24 + w], bit r of the 729-bit row
// set of column p) -> row-major for pass D: bit q*PPR + p of dst (PPR = ppr
// rounded up to 256). One CTA per 256 columns: the 256 x 24 source words in
// smem, each thread builds output words (row q, 32 columns).
__global__ void __launch_bounds__(256) k_bits_transpose(const uint32_t *__restrict__ src, uint32_t *__restrict__ dst,
                                                        int64_t ppr, int nrows, int64_t ppr_pad) {
    __shared__ uint32_t sb[256 * 24];
    const int64_t p0 = (int64_t)blockIdx.x * 256;
    for (int t = threadIdx.x; t < 256 * 24; t += blockDim.x) {
        const int64_t p = p0 + t / 24;
        sb[t] = p < ppr ? src[p0 * 24 + t] : 0u;
    }
    __syncthreads();
    const int64_t wpr = ppr_pad / 32;  // words per output row
    for (int t = threadIdx.x; t < nrows * 8; t += blockDim.x) {
        const int q = t >> 3, w = t & 7;  // row q, output word w of this CTA's 8
        uint32_t o = 0;
#pragma unroll 8
        for (int i = 0; i < 32; i++) o |= ((sb[(32 * w + i) * 24 + (q >> 5)] >> (q & 31)) & 1u) << i;
        dst[(int64_t)q * wpr + p0 / 32 + w] = o;
    }
}

// Sparse reduce-only pass D over piece-major group 0. Pass C flagged the
// nonzero 128-B rows of its output (k_bits_transpose puts the bits in D's
// order); at n = 24 one row in four is nonzero. Only flagged rows are read
// (cp.async) and written back (STG); the others are zero in memory already.
// One CTA per SM, two tile buffers; every warp issues the loads of the next
// item and the stores of the current one for the rows of its 32-row mask
// word (warp k <-> rows 32k..32k+31), four rows per pass (8 lanes x 16 B).
// Invariant: a buffer is zero outside the flagged rows of its last item
// (zeroed at start; reduce keeps zero rows zero; the write-back zeroes them).
template <int R1, int R2>
__global__ void __launch_bounds__(PipeSmem<R1, R2>::THREADS, 1)
    k_reduce_sparse(uint32_t *__restrict__ state, const uint32_t *__restrict__ nzmap, int64_t nitems,
                    uint32_t ib_mask, int64_t ncol, int64_t ppr_pad) {
    using SM = PipeSmem<R1, R2>;
    static_assert(pipe_cols<R1, R2>() == 1, "one 128-B column per tile");
    constexpr int N1 = SM::N1, N2 = SM::N2, NR = SM::NR, CW = SM::CW, PITCH = SM::PITCH;
    constexpr int NWB = (NR + 31) / 32;
    static_assert(NWB <= CW, "one mask word per warp");
    extern __shared__ __align__(128) uint32_t smem[];
    __shared__ uint32_t msk[3][32];  // row masks of items i, i+1, i+2 (slot = item % 3)
    __shared__ uint32_t rlist[32][16];  // per warp: the rows of its mask word (uint16)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 3, q16 = lane & 7;
    constexpr int NCT = CW * 32;
    const int64_t L = nitems > blockIdx.x ? (nitems - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
    auto item = [&](int64_t i) { return (int64_t)blockIdx.x + i * (int64_t)gridDim.x; };

    // warp 0: the 729 row flags of item i as 23 mask words in msk[b]; the
    // bitmap words of item i+1 are fetched now (their latency hides under an item)
    uint32_t Wn = 0;
    auto fetch = [&](int64_t i) {
        if (warp == 0 && i < L) {
            const int64_t it = item(i);
            const int64_t B0 = (it / ncol) * ppr_pad + (it % ncol) * NR;
            Wn = lane <= NWB ? __ldg(&nzmap[(B0 >> 5) + lane]) : 0u;
        }
    };
    auto masks = [&](int64_t i) {
        const int b = (int)(i % 3);
        if (warp == 0) {
            const int64_t it = item(i);
            const int64_t B0 = (it / ncol) * ppr_pad + (it % ncol) * NR;
            const int sh = (int)(B0 & 31);
            const uint32_t W = Wn;
            fetch(i + 1);
            const uint32_t hi = __shfl_down_sync(0xffffffffu, W, 1);
            uint32_t m = sh ? __funnelshift_r(W, hi, sh) : W;  // bits 32*lane .. 32*lane+31 of the span
            const int r0 = 32 * lane;
            if (r0 + 32 > NR) m &= r0 >= NR ? 0u : ((1u << (NR - r0)) - 1u);
            if (lane < NWB) msk[b][lane] = m;
        }
    };
    // warp k: cp.async of the flagged rows of mask word k of item i into buffer b
    auto load = [&](int64_t i, int b) {
        if (warp < NWB) {
            const int64_t base = item(i) * NR;
            uint32_t *tile = smem + b * SM::TILE_WORDS;
            uint32_t mm = msk[i % 3][warp];
            while (mm) {
                uint32_t mg = mm;  // the g-th set bit of mm (g = 0..3)
                if (g > 0) mg &= mg - 1;
                if (g > 1) mg &= mg - 1;
                if (g > 2) mg &= mg - 1;
                const uint32_t j = (uint32_t)__ffs(mg) - 1u;
                if (mg) {
                    const int r = 32 * warp + (int)j;
                    cp_async16(tile + r * PITCH + q16 * 4, state + (base + r) * 32 + q16 * 4, true);
                }
#pragma unroll
                for (int c = 0; c < 4; c++) mm &= mm - 1;
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };

    for (int t = threadIdx.x; t < 2 * SM::TILE_WORDS / 4; t += blockDim.x)
        reinterpret_cast<uint4 *>(smem)[t] = make_uint4(0, 0, 0, 0);
    fetch(0);
    if (L > 0) masks(0);
    if (L > 1) masks(1);
    __syncthreads();
    if (L > 0) load(0, 0);
    for (int64_t i = 0; i < L; i++) {
        const int b = (int)(i & 1);
        const int tb = b * SM::TILE_WORDS;
        if (i + 2 < L) masks(i + 2);
        __syncthreads();  // msk of i+2 visible; buffer b^1's previous write-back (zeroing) done
        if (i + 1 < L) load(i + 1, b ^ 1);
        else asm volatile("cp.async.commit_group;" ::: "memory");
        asm volatile("cp.async.wait_group 1;" ::: "memory");  // this thread's copies of item i
        __syncthreads();                                       // everyone's
        for (int t2 = warp; t2 < N2; t2 += CW) {
            uint32_t v[N1];
#pragma unroll
            for (int x = 0; x < N1; x++) v[x] = smem[tb + (x + N1 * t2) * PITCH + lane];
            if (!warp_any(v)) continue;
            cube_reduce_par<R1>(v);
#pragma unroll
            for (int x = 0; x < N1; x++) smem[tb + (x + N1 * t2) * PITCH + lane] = v[x];
        }
        if (R2 > 0) {
            __syncthreads();
            for (int t1 = warp; t1 < N1; t1 += CW) {
                uint32_t v[N2];
#pragma unroll
                for (int x = 0; x < N2; x++) v[x] = smem[tb + (t1 + N1 * x) * PITCH + lane];
                if (!warp_any(v)) continue;
                cube_reduce_par<R2>(v);
#pragma unroll
                for (int x = 0; x < N2; x++) smem[tb + (t1 + N1 * x) * PITCH + lane] = v[x];
            }
        }
        if (ib_mask) {
            // in-block axes on the flagged rows only (the others are zero):
            // warp k compacts the rows of mask word k, 8 rows x 4 blocks per pass
            __syncthreads();
            if (warp < NWB) {
                const uint32_t mm = msk[i % 3][warp];
                const int nrow = __popc(mm);
                uint16_t *rl = reinterpret_cast<uint16_t *>(&rlist[warp][0]);
                if ((mm >> lane) & 1u) rl[__popc(mm & ((1u << lane) - 1u))] = (uint16_t)(32 * warp + lane);
                __syncwarp();
                for (int e0 = 0; e0 < nrow; e0 += 8) {
                    const int e = e0 + (lane >> 2);
                    if (e < nrow) {
                        uint4 *p = reinterpret_cast<uint4 *>(&smem[tb + rl[e] * PITCH + (lane & 3) * 8]);
                        const uint4 x0 = p[0], x1 = p[1];
                        uint32_t v[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
                        inblock_reduce(v, ib_mask);
                        p[0] = make_uint4(v[0], v[1], v[2], v[3]);
                        p[1] = make_uint4(v[4], v[5], v[6], v[7]);
                    }
                }
            }
        }
        __syncthreads();
        // write back (and zero) the flagged rows of item i
        if (warp < NWB) {
            const int64_t base = item(i) * NR;
            uint32_t *tile = smem + tb;
            uint32_t mm = msk[i % 3][warp];
            while (mm) {
                uint32_t mg = mm;  // the g-th set bit of mm (g = 0..3)
                if (g > 0) mg &= mg - 1;
                if (g > 1) mg &= mg - 1;
                if (g > 2) mg &= mg - 1;
                const uint32_t j = (uint32_t)__ffs(mg) - 1u;
                if (mg) {
                    const int r = 32 * warp + (int)j;
                    uint4 *sp = reinterpret_cast<uint4 *>(tile + r * PITCH) + q16;
                    const uint4 x = *sp;
                    *sp = make_uint4(0, 0, 0, 0);
                    reinterpret_cast<uint4 *>(state + (base + r) * 32)[q16] = x;
                }
#pragma unroll
                for (int c = 0; c < 4; c++) mm &= mm - 1;
            }
        }
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
}

// Block-sparse pass D (piece-major group 0, 3^6 rows, one column): the tile's
// 729 rows are 27 sub-blocks of 27 consecutive rows (one value of the three
// high group-0 digits). Pass C's row bits (k_bits_transpose order) say which
// sub-blocks hold a nonzero row: at n = 24 about half of them
// (tools/sparsity.py). Only those are loaded and stored, each as one TMA box
// of 27 rows x 128 B; the compute warps zero-fill the others in shared memory.
template <int R1, int R2>
__global__ void __launch_bounds__(PipeSmem<R1, R2>::THREADS, 1)
    k_reduce_blocks(const __grid_constant__ CUtensorMap smap, const uint32_t *__restrict__ nzmap, int64_t ncol,
                    int64_t nitems, uint32_t ib_mask, int64_t ppr_pad) {
    using SM = PipeSmem<R1, R2>;
    static_assert(pipe_cols<R1, R2>() == 1 && SM::NR == 729, "3^6 rows, one column");
    constexpr int N1 = SM::N1, N2 = SM::N2, NR = SM::NR, CW = SM::CW, PITCH = SM::PITCH;
    constexpr int SB = 27, NSB = NR / SB, SBW = SB * PITCH;  // sub-block rows, count, words
    constexpr int NWB = (NR + 31) / 32;
    extern __shared__ __align__(128) uint32_t smem[];
    __shared__ __align__(8) uint64_t full[2], computed[2];
    __shared__ uint32_t s_F[2];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t L = nitems > blockIdx.x ? (nitems - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
    auto item = [&](int64_t i) { return (int64_t)blockIdx.x + i * (int64_t)gridDim.x; };
    if (threadIdx.x == 0) {
        for (int b = 0; b < 2; b++) {
            mbar_init(&full[b], 1);
            mbar_init(&computed[b], CW);
        }
    }
    __syncthreads();

    if (warp == CW) {  // ------------------------------ producer warp
        uint32_t Fb[2] = {0u, 0u};
        for (int64_t i = 0; i < L + 2; i++) {
            const int b = (int)(i & 1);
            uint32_t *tile = smem + b * SM::TILE_WORDS;
            if (i >= 2) {  // store the loaded sub-blocks of item i-2
                mbar_wait(&computed[b], (unsigned)(((i - 2) >> 1) & 1));
                const int64_t it = item(i - 2);
                if (lane == 0) {
                    uint32_t F = Fb[b];
                    while (F) {
                        const int k = __ffs(F) - 1;
                        F &= F - 1;
                        tma_store_4d(&smap, 0, SB * k, (int)(it % ncol), (int)(it / ncol), tile + k * SBW);
                    }
                    bulk_commit();
                    bulk_wait_read<0>();  // buffer b is reloaded next
                }
                __syncwarp();
            }
            if (i < L) {
                const int64_t it = item(i);
                // sub-block flags from the 729 row bits (lane k < 27: rows 27k..27k+26)
                const int64_t B0 = (it / ncol) * ppr_pad + (it % ncol) * NR;
                const int sh = (int)(B0 & 31);
                const uint32_t W = lane <= NWB ? __ldg(&nzmap[(B0 >> 5) + lane]) : 0u;
                const int q = sh + SB * (lane < NSB ? lane : 0);
                const uint32_t w0 = __shfl_sync(0xffffffffu, W, (q >> 5) & 31);
                const uint32_t w1 = __shfl_sync(0xffffffffu, W, ((q >> 5) + 1) & 31);
                const uint32_t bits = __funnelshift_r(w0, w1, q & 31) & ((1u << SB) - 1u);
                const uint32_t F = __ballot_sync(0xffffffffu, lane < NSB && bits != 0u);
                Fb[b] = F;
                if (lane == 0) {
                    s_F[b] = F;
                    mbar_expect_tx(&full[b], (unsigned)(__popc(F) * SB * 128));
                    uint32_t G = F;
                    while (G) {
                        const int k = __ffs(G) - 1;
                        G &= G - 1;
                        tma_load_4d(tile + k * SBW, &smap, 0, SB * k, (int)(it % ncol), (int)(it / ncol), &full[b]);
                    }
                }
                __syncwarp();
            }
        }
        if (lane == 0) bulk_wait0();
        return;
    }

    // ---------------------------------- compute warps
    constexpr int NCT = CW * 32;
    for (int64_t i = 0; i < L; i++) {
        const int b = (int)(i & 1);
        const int tb = b * SM::TILE_WORDS;
        mbar_wait(&full[b], (unsigned)((i >> 1) & 1));
        const uint32_t F = s_F[b];
        if (F) {
            if (F != (1u << NSB) - 1u) {  // zero the sub-blocks that were not loaded
                for (int t = threadIdx.x; t < NSB * (SBW / 4); t += NCT) {
                    const int k = t / (SBW / 4);
                    if (!((F >> k) & 1u)) reinterpret_cast<uint4 *>(smem + tb)[t] = make_uint4(0, 0, 0, 0);
                }
                bar_compute(NCT);
            }
            for (int t2 = warp; t2 < N2; t2 += CW) {
                uint32_t v[N1];
#pragma unroll
                for (int x = 0; x < N1; x++) v[x] = smem[tb + (x + N1 * t2) * PITCH + lane];
                if (!warp_any(v)) continue;
                cube_reduce_par<R1>(v);
#pragma unroll
                for (int x = 0; x < N1; x++) smem[tb + (x + N1 * t2) * PITCH + lane] = v[x];
            }
            bar_compute(NCT);
            for (int t1 = warp; t1 < N1; t1 += CW) {
                uint32_t v[N2];
#pragma unroll
                for (int x = 0; x < N2; x++) v[x] = smem[tb + (t1 + N1 * x) * PITCH + lane];
                if (!warp_any(v)) continue;
                cube_reduce_par<R2>(v);
#pragma unroll
                for (int x = 0; x < N2; x++) smem[tb + (t1 + N1 * x) * PITCH + lane] = v[x];
            }
            if (ib_mask) {  // zero sub-blocks are skipped warp by warp
                bar_compute(NCT);
                inblock_round(&smem[tb], NR * kRowBlocks, ib_mask, NCT, 1);
            }
        }
        fence_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&computed[b]);
    }
}

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
};

// padded: each C0 tile of 3^g blocks is stored at a pitch rounded up to a
// multiple of 4 blocks (128 B; 2187 -> 2188 blocks at g = 7) so that every
// 128-B row piece the strided passes move is 128-B aligned (TMA load+store of
// misaligned 32-B-granular rows measured 24% slower, tools/probes/layout_probe.cu).
// The pad block is zero and stays zero (MERGE: 0 & 0, REDUCE: 0 & ~x). Only the
// fused single-GPU plan uses it; the bitmap-keeping and sharded entry points
// keep the reference layout (dense.py:1-23).
Plan make_plan(int n, bool padded = true) {
    Plan p;
    p.n = n;
    p.ne = n < 5 ? 5 : n;
    p.rank_sub = n < 5 ? (243 - pow3l(n)) : 0;
    p.H = p.ne - 5;
    p.g = std::min(p.H, kC0Max);
    p.T = p.H - p.g;
    p.nblocks = pow3l(p.H);
    p.pitch = pow3l(p.g);
    if (padded && p.T > 0) p.pitch = (p.pitch + kRowBlocks - 1) / kRowBlocks * kRowBlocks;
    p.sbytes = (uint64_t)pow3l(p.T) * (uint64_t)p.pitch * 32;
    if (p.T > 0) {
        p.m = (p.T + kGroupMax - 1) / kGroupMax;
        int a = p.g;
        for (int k = 0; k < p.m; k++) {
            const int rk = p.T / p.m + (k < p.T % p.m ? 1 : 0);
            p.r[k] = rk;
            p.a[k] = a;
            a += rk;
        }
    }
    // piece-major group 0: the state is stored as [upper digits][piece x of the
    // C0 tile][group-0 row][128 B] instead of [upper][group-0 row][C0 tile], so
    // the tile of pass D (group 0 reduce, the read+write pass) is one
    // contiguous 93 KB range instead of 729 pieces 70 KB apart, and pass E reads
    // its C0 tile as pieces 93 KB apart (tools/probes/layout_probe.cu: in-place
    // R+W of contiguous tiles 11.8 vs 15.6 ms; the E read 5.9 vs 5.1 ms).
    // Groups above 0 see the same rows/columns as before (columns enumerate the
    // pieces). Needs one 128-B column per tile (3^6 rows) and a separate D pass.
    p.pm = padded && p.T > 0 && p.m >= 2 && p.r[0] == kGroupMax && !getenv("DQMC_NO_PM");
    // distribute the five in-block REDUCE axes over the passes that hold whole
    // blocks: pass C (write-only) takes axes 1 and 4, the read+write passes D
    // share the rest, the final pass E takes none when a D pass exists (it is
    // latency-bound by the C0 axes + compaction). With the sparse skip, D runs
    // at the HBM copy rate with three axes (n = 24: C 9.8 / D 11.6 ms; axes
    // 1 / 2-5 gave 10.8 / 12.5, 1-2 / 3-5 10.0 / 11.5, none / all 11.9 / 11.8
    // — tools/ab_ib.sh).
    if (p.T == 0) {
        p.ib_E = 31u;
    } else if (p.m == 1) {
        p.ib_C = 3u;   // axes 1,2
        p.ib_E = 28u;  // axes 3,4,5
    } else {
        p.ib_C = 9u;
        const int rest[3] = {1, 2, 4};  // 0-based axes 2, 3, 5
        int i = 0;
        const int nd = p.m - 1;
        for (int q = 0; q < nd; q++) {
            const int take = (3 - i) / (nd - q);
            for (int c = 0; c < take; c++) p.ib_D[p.m - 2 - q] |= 1u << rest[i++];
        }
        if (const char *e = getenv("DQMC_IB_C")) {  // experiment: C's in-block axes; the first D pass takes the rest
            p.ib_C = (uint32_t)strtoul(e, nullptr, 0) & 31u;
            for (int k = 0; k < 8; k++) p.ib_D[k] = 0;
            p.ib_D[p.m - 2] = 31u & ~p.ib_C;
        }
    }
    return p;
}

thread_local std::string g_err;
const bool g_debug = getenv("DQMC_DEBUG") != nullptr;  // sync + report after every pass
const int g_sparse = getenv("DQMC_NO_SPARSE") ? 0 : 1;  // skip all-zero warps in the reduce rounds
std::mutex g_mu;

int set_err(int code, const std::string &msg) {
    g_err = msg;
    return code;
}

#define CK(call)                                                                                         \
    do {                                                                                                 \
        cudaError_t e_ = (call);                                                                         \
        if (e_ != cudaSuccess) return set_err(DQMC_ERR_CUDA, std::string(#call ": ") + cudaGetErrorString(e_)); \
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
    uint32_t *nzmap = nullptr;  // nonzero-piece bitmap of pass C (sparse pass D)
    size_t nzmap_cap = 0;       // bytes
    int64_t *tile_base = nullptr, *tile_pos = nullptr;
    int32_t *tile_cnt = nullptr;
    size_t tile_cap = 0, tile_pos_cap = 0, tile_cnt_cap = 0;  // entries
    int64_t *scratch = nullptr;
    size_t scratch_cap = 0, scratch_want = 0;  // entries
    unsigned long long *alloc = nullptr;
    int64_t *total = nullptr;
    void *cub_tmp = nullptr;
    size_t cub_tmp_cap = 0;
    cudaStream_t stream2 = nullptr;   // copy-out stream of the pipelined host API
    cudaEvent_t chunk_ev[17] = {};
    int64_t *chunk_base = nullptr;    // device running bases of the chunked final stage
    int64_t *hbase = nullptr;         // mapped pinned host mirror of chunk_base
    int hint_n = -1;
    int64_t hint_count = 0;           // prime count of the last host call (sizes the pinned output)
    uint32_t *tt_tmp = nullptr;
    size_t tt_tmp_cap = 0;  // bytes
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
    int64_t *jcount_host = nullptr;  // pinned, one count per slot
    cudaEvent_t jev[kJobSlots] = {};
};

Engine g_eng;

int ensure_device() {
    if (g_eng.device >= 0) return DQMC_OK;
    int cnt = 0;
    cudaError_t e = cudaGetDeviceCount(&cnt);
    if (e != cudaSuccess || cnt == 0)
        return set_err(DQMC_ERR_NODEVICE, "no CUDA device visible: libdqmc has no CPU fallback");
    int dev = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaSetDevice(dev));
    g_eng.device = dev;
    CK(cudaStreamCreateWithFlags(&g_eng.stream, cudaStreamNonBlocking));
    CK(cudaMalloc(&g_eng.alloc, 256));
    CK(cudaStreamCreateWithFlags(&g_eng.stream2, cudaStreamNonBlocking));
    for (int i = 0; i < 16; i++) CK(cudaEventCreateWithFlags(&g_eng.chunk_ev[i], cudaEventDisableTiming));
    CK(cudaMalloc(&g_eng.chunk_base, 17 * sizeof(int64_t)));
    CK(cudaHostAlloc((void **)&g_eng.hbase, 17 * sizeof(int64_t), cudaHostAllocMapped));
    CK(cudaMalloc(&g_eng.total, 256));
    return DQMC_OK;
}

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
    return DQMC_OK;
}

template <int R1, int R2, int MODE>
int set_strided_attr() {
    constexpr int smem = P3<R1>::v * P3<R2>::v * 32 * 4;
    CK(cudaFuncSetAttribute(k_strided<R1, R2, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    return DQMC_OK;
}

template <int R1, int R2, int MODE>
int set_pipe_attr() {
    using SM = PipeSmem<R1, R2>;
    CK(cudaFuncSetAttribute(k_strided_pipe<R1, R2, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, SM::SMEM));
    return DQMC_OK;
}

template <int R1, int R2>
int set_mr_attr() {
    using SM = PipeSmem<R1, R2>;
    CK(cudaFuncSetAttribute(k_merge_reduce_pipe<R1, R2>, cudaFuncAttributeMaxDynamicSharedMemorySize, SM::SMEM));
    return DQMC_OK;
}

template <int MODE>
int set_pipe_attrs() {
    int rc;
    if ((rc = set_pipe_attr<1, 0, MODE>())) return rc;
    if ((rc = set_pipe_attr<2, 0, MODE>())) return rc;
    if ((rc = set_pipe_attr<3, 0, MODE>())) return rc;
    if ((rc = set_pipe_attr<2, 2, MODE>())) return rc;
    if ((rc = set_pipe_attr<3, 2, MODE>())) return rc;
    if ((rc = set_pipe_attr<3, 3, MODE>())) return rc;
    return DQMC_OK;
}

template <int MODE>
int set_mode_attrs() {
    int rc;
    if ((rc = set_strided_attr<1, 0, MODE>())) return rc;
    if ((rc = set_strided_attr<2, 0, MODE>())) return rc;
    if ((rc = set_strided_attr<3, 0, MODE>())) return rc;
    if ((rc = set_strided_attr<2, 2, MODE>())) return rc;
    if ((rc = set_strided_attr<3, 2, MODE>())) return rc;
    if ((rc = set_strided_attr<3, 3, MODE>())) return rc;
    return DQMC_OK;
}

int ensure_attrs() {
    if (g_eng.attrs_set) return DQMC_OK;
    const int tile_smem = (int)pow3l(kC0Max) * 32;
    CK(cudaFuncSetAttribute(k_c0_merge, cudaFuncAttributeMaxDynamicSharedMemorySize, tile_smem));
    // + one 128-B piece (the padded pitch of a piece-major tile, make_plan) + 128 B of alignment
    CK(cudaFuncSetAttribute(k_c0_final<kC0Max>, cudaFuncAttributeMaxDynamicSharedMemorySize, tile_smem + 256));
    CK(cudaFuncSetAttribute(k_small, cudaFuncAttributeMaxDynamicSharedMemorySize, tile_smem));
    int rc;
    if ((rc = set_mode_attrs<MERGE_ONLY>())) return rc;  // pass B (k_strided)
    if ((rc = set_pipe_attrs<REDUCE_ONLY>())) return rc;  // pass D (k_strided_pipe)
    {
        using SMD = PipeSmem<3, 3>;
        CK(cudaFuncSetAttribute(k_reduce_sparse<3, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMD::SMEM));
        CK(cudaFuncSetAttribute(k_reduce_blocks<3, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMD::SMEM));
    }
    if ((rc = set_mr_attr<1, 0>()) || (rc = set_mr_attr<2, 0>()) || (rc = set_mr_attr<3, 0>()) ||
        (rc = set_mr_attr<2, 2>()) || (rc = set_mr_attr<3, 2>()) || (rc = set_mr_attr<3, 3>()))
        return rc;
    CK(cudaDeviceGetAttribute(&g_eng.num_sms, cudaDevAttrMultiProcessorCount, g_eng.device));
    g_eng.attrs_set = true;
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

// 3-D tensor map over the state for a strided group: dim0 = words of the
// inner extent (8*Q), dim1 = the 3^R rows (stride Q blocks), dim2 = outer
// index (stride 3^R*Q blocks); box = 32 words x BOXR rows x 1.
int ensure_encode() {
    if (!g_eng.encode) {
        cudaDriverEntryPointQueryResult q;
        void *fn = nullptr;
        CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
        if (!fn || q != cudaDriverEntryPointSuccess) return set_err(DQMC_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
        g_eng.encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    }
    return DQMC_OK;
}

int make_group_map(CUtensorMap *map, uint32_t *state, int64_t Q, int nr, int64_t nouter, int boxr, int box0 = 32) {
    int rc;
    if ((rc = ensure_encode())) return rc;
    cuuint64_t dims[3] = {(cuuint64_t)(8 * Q), (cuuint64_t)nr, (cuuint64_t)nouter};
    cuuint64_t strides[2] = {(cuuint64_t)(Q * 32), (cuuint64_t)(Q * 32 * nr)};
    cuuint32_t box[3] = {(cuuint32_t)box0, (cuuint32_t)boxr, 1};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = g_eng.encode(map, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, state, dims, strides, box, es,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return set_err(DQMC_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
    return DQMC_OK;
}

// 4-D map for the reduce-only pipe: the reference layout as {8Q words, rows,
// outer, 1}; piece-major group 0 (pm) as {32 words, rows (128 B apart),
// columns (3^R pieces apart), outer (Q/4 * 3^R pieces apart)}.
int make_group_map4(CUtensorMap *map, uint32_t *state, int64_t Q, int nr, int64_t nouter, int boxr, int box0, bool pm) {
    int rc;
    if ((rc = ensure_encode())) return rc;
    cuuint64_t dims[4], strides[3];
    if (pm) {
        const int64_t ncol = Q / kRowBlocks;
        dims[0] = 32, dims[1] = (cuuint64_t)nr, dims[2] = (cuuint64_t)ncol, dims[3] = (cuuint64_t)nouter;
        strides[0] = 128, strides[1] = (cuuint64_t)nr * 128, strides[2] = (cuuint64_t)(ncol * nr * 128);
    } else {
        dims[0] = (cuuint64_t)(8 * Q), dims[1] = (cuuint64_t)nr, dims[2] = (cuuint64_t)nouter, dims[3] = 1;
        strides[0] = (cuuint64_t)(Q * 32), strides[1] = (cuuint64_t)(Q * 32 * nr),
        strides[2] = (cuuint64_t)(Q * 32 * nr * nouter);
    }
    cuuint32_t box[4] = {(cuuint32_t)box0, (cuuint32_t)boxr, 1, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = g_eng.encode(map, CU_TENSOR_MAP_DATA_TYPE_UINT32, 4, state, dims, strides, box, es,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return set_err(DQMC_ERR_CUDA, "cuTensorMapEncodeTiled (4-D) failed: " + std::to_string((int)r));
    return DQMC_OK;
}

// 5-D map for the binary-row gather of a MERGE_REDUCE group: dims {8Q words,
// 3 x R1 digit dims (strides Q, 3Q, 9Q blocks), 3^R2}; box {32, 2, .., 2, 1}.
int make_gather_map(CUtensorMap *map, uint32_t *state, int64_t Q, int r1, int r2, int box0 = 32) {
    cuuint64_t dims[5];
    cuuint64_t strides[4];
    cuuint32_t box[5], es[5];
    int rank = 0;
    dims[rank] = (cuuint64_t)(8 * Q);
    box[rank] = (cuuint32_t)box0;
    es[rank++] = 1;
    int64_t st = Q * 32;
    for (int k = 0; k < r1; k++) {
        dims[rank] = 3;
        strides[rank - 1] = (cuuint64_t)st;
        box[rank] = 2;
        es[rank++] = 1;
        st *= 3;
    }
    while (rank < 4) {  // pad to a fixed 5-D layout with unit dims
        dims[rank] = 1;
        strides[rank - 1] = (cuuint64_t)st;
        box[rank] = 1;
        es[rank++] = 1;
    }
    dims[rank] = (cuuint64_t)pow3l(r2);
    strides[rank - 1] = (cuuint64_t)st;
    box[rank] = 1;
    es[rank++] = 1;
    CUresult r = g_eng.encode(map, CU_TENSOR_MAP_DATA_TYPE_UINT32, 5, state, dims, strides, box, es,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return set_err(DQMC_ERR_CUDA, "cuTensorMapEncodeTiled (gather) failed: " + std::to_string((int)r));
    return DQMC_OK;
}

template <int R1, int R2, int MODE>
int launch_pipe(uint32_t *state, int64_t Q, int64_t ncol, int64_t nouter, uint32_t ib, bool pm, cudaStream_t s,
                uint32_t *nzmap) {
    using SM = PipeSmem<R1, R2>;
    constexpr int CC = pipe_cols<R1, R2>();  // 128-B columns per tile
    CUtensorMap map, gmap;
    int rc;
    if (pm && (CC != 1 || MODE == MERGE_REDUCE)) return set_err(DQMC_ERR_INVALID, "internal: piece-major needs CC = 1");
    if (MODE == MERGE_REDUCE) {
        if ((rc = make_group_map(&map, state, Q, SM::NR, nouter, SM::BOXR, 32 * CC))) return rc;
    } else {
        if ((rc = make_group_map4(&map, state, Q, SM::NR, nouter, SM::BOXR, 32 * CC, pm))) return rc;
    }
    if (MODE == MERGE_REDUCE) {
        if ((rc = make_gather_map(&gmap, state, Q, R1, R2, 32 * CC))) return rc;
    } else {
        gmap = map;
    }
    const int64_t ncolg = (ncol + CC - 1) / CC;  // column groups: one tile each per outer index
    const int64_t nitems = ncolg * nouter;
    const int grid = (int)std::min<int64_t>(nitems, g_eng.num_sms);
    if (MODE == MERGE_REDUCE)
        k_merge_reduce_pipe<R1, R2><<<grid, SM::THREADS + 32, SM::SMEM, s>>>(
            map, gmap, ncolg, nitems, ib, g_sparse, nzmap);
    else
        k_strided_pipe<R1, R2, MODE><<<grid, SM::THREADS, SM::SMEM, s>>>(map, gmap, ncolg, nitems, ib, pm ? 1 : 0,
                                                                          g_sparse);
    CK(cudaGetLastError());
    return DQMC_OK;
}

template <int MODE>
int launch_pipe_mode(int r, uint32_t *state, int64_t Q, int64_t ncol, int64_t nouter, uint32_t ib, cudaStream_t s,
                     bool pm = false, uint32_t *nzmap = nullptr) {
    switch (r) {
        case 1: return launch_pipe<1, 0, MODE>(state, Q, ncol, nouter, ib, pm, s, nzmap);
        case 2: return launch_pipe<2, 0, MODE>(state, Q, ncol, nouter, ib, pm, s, nzmap);
        case 3: return launch_pipe<3, 0, MODE>(state, Q, ncol, nouter, ib, pm, s, nzmap);
        case 4: return launch_pipe<2, 2, MODE>(state, Q, ncol, nouter, ib, pm, s, nzmap);
        case 5: return launch_pipe<3, 2, MODE>(state, Q, ncol, nouter, ib, pm, s, nzmap);
        default: return launch_pipe<3, 3, MODE>(state, Q, ncol, nouter, ib, pm, s, nzmap);
    }
}

template <int MODE>
void launch_strided_mode(int r, uint32_t *state, int64_t Q, int64_t ncol, int64_t nitems, uint32_t ib, bool pm,
                         cudaStream_t s) {
    const int grid = (int)std::min<int64_t>(nitems, 148ll * 16);
#define LS(R1, R2)                                                                             \
    k_strided<R1, R2, MODE><<<grid, kStridedThreads, P3<R1>::v * P3<R2>::v * 32 * 4, s>>>(                 \
        state, Q, ncol, nitems, ib, pm ? kRowBlocks : Q, pm ? P3<R1>::v * P3<R2>::v * kRowBlocks : kRowBlocks, \
        pm ? Q * P3<R1>::v * P3<R2>::v : P3<R1>::v * P3<R2>::v * Q)
    switch (r) {
        case 1: LS(1, 0); break;
        case 2: LS(2, 0); break;
        case 3: LS(3, 0); break;
        case 4: LS(2, 2); break;
        case 5: LS(3, 2); break;
        default: LS(3, 3); break;
    }
#undef LS
}

uint64_t state_bytes_ref(int n, int h) {
    // dense.py:56-63
    uint64_t used = (uint64_t)pow3l(h), b = 1;
    while (b < used) b <<= 1;
    if (b < 64) b = 64;
    return (uint64_t)pow3l(n - h) * b / 8;
}

void note_held(const Plan &p, bool keep);

uint64_t engine_device_bytes(const Plan &p, bool keep) {
    if (p.T == 0 && !keep) return 0;
    return p.sbytes + (uint64_t)pow3l(p.T) * 20;
}

// E's tensor maps for piece-major group 0: dims {32 words, pieces (3^r x 128 B
// apart), group-0 rows (128 B apart), upper (pieces x 3^r x 128 B apart)}
int make_final_maps(const Plan &p, const uint32_t *state, CUtensorMap *ma, CUtensorMap *mb, FinalArgs &fa) {
    memset(ma, 0, sizeof *ma);
    memset(mb, 0, sizeof *mb);
    fa.pm_nr = 0;
    fa.pm_np = 0;
    if (!p.pm) return DQMC_OK;
    int rc;
    if ((rc = ensure_encode())) return rc;
    const int64_t nr = pow3l(p.r[0]), np = p.pitch / kRowBlocks, nu = pow3l(p.T - p.r[0]);
    cuuint64_t dims[4] = {32, (cuuint64_t)np, (cuuint64_t)nr, (cuuint64_t)nu};
    cuuint64_t strides[3] = {(cuuint64_t)(nr * 128), 128, (cuuint64_t)(np * nr * 128)};
    cuuint32_t es[4] = {1, 1, 1, 1};
    for (int k = 0; k < 2; k++) {
        const int rows = k == 0 ? 256 : (int)(np & 255);
        if (rows == 0) continue;
        cuuint32_t box[4] = {32, (cuuint32_t)rows, 1, 1};
        CUresult r = g_eng.encode(k == 0 ? ma : mb, CU_TENSOR_MAP_DATA_TYPE_UINT32, 4, (void *)state, dims, strides, box,
                                  es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return set_err(DQMC_ERR_CUDA, "cuTensorMapEncodeTiled (final) failed: " + std::to_string((int)r));
    }
    fa.pm_nr = (int)nr;
    fa.pm_np = (int)np;
    return DQMC_OK;
}

int launch_c0_final(int g, int64_t ntiles, const uint32_t *state, const FinalArgs &fa, const CUtensorMap &ma,
                    const CUtensorMap &mb, cudaStream_t s) {
    const int smem = fa.pm_nr ? fa.pm_np * 128 + 128 : (int)pow3l(g) * 32;
    switch (g) {
#define CASE(G)                                                                         \
    case G:                                                                             \
        k_c0_final<G><<<(unsigned)ntiles, kFinalThreads, smem, s>>>(state, fa, ma, mb);  \
        break;
        CASE(0) CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7)
#undef CASE
        default: return set_err(DQMC_ERR_INVALID, "bad tile exponent");
    }
    CK(cudaGetLastError());
    return DQMC_OK;
}

// Final stage: E (+ scan + reorder). Source: the truth table (k_small, fused
// A+E, when tt32 != null) or a merged/reduced state. Returns the prime count.
int run_final(const Plan &p, const uint32_t *tt32, const uint32_t *state, const uint32_t *kill, uint32_t ib_mask,
              int64_t rank_add, int64_t *ranks, int64_t cap, bool count_only, uint32_t *bitmap_out, int64_t *count,
              Timer &tm, cudaStream_t s, int64_t *count_dev = nullptr) {
    const uint64_t S = (uint64_t)p.nblocks * 32;
    const int64_t ntiles = p.T == 0 ? 1 : pow3l(p.T);
    const int tile_smem = (int)pow3l(p.g) * 32;
    int rc;
    if ((rc = grow(g_eng.tile_base, g_eng.tile_cap, (size_t)ntiles, 8))) return rc;
    if ((rc = grow(g_eng.tile_pos, g_eng.tile_pos_cap, (size_t)ntiles, 8))) return rc;
    if ((rc = grow(g_eng.tile_cnt, g_eng.tile_cnt_cap, (size_t)ntiles, 4))) return rc;
    if ((kill || bitmap_out) && p.T > 0 && p.pitch != pow3l(p.g))
        return set_err(DQMC_ERR_INVALID, "internal: kill/bitmap outputs need the reference layout plan");
    const bool direct = ntiles == 1;  // one tile: its ranks are already in order
    if (!count_only && !direct) {
        const size_t want = std::max<size_t>(g_eng.scratch_want, (size_t)1 << 20);
        if ((rc = grow(g_eng.scratch, g_eng.scratch_cap, want, 8))) return rc;
    }
    FinalArgs fa;
    fa.out = count_only ? nullptr : (direct ? ranks : g_eng.scratch);
    fa.cap = count_only ? 0 : (direct ? cap : (int64_t)g_eng.scratch_cap);
    fa.rank_add = rank_add;
    fa.kill = kill;
    fa.ib_mask = ib_mask;
    fa.bitmap_out = bitmap_out;
    fa.alloc = g_eng.alloc;
    fa.tile_base = g_eng.tile_base;
    fa.tile_cnt = g_eng.tile_cnt;
    fa.tile0 = 0;
    fa.pitch = p.pitch;
    fa.prefetch = 3 * g_eng.num_sms;  // one generation of resident CTAs (3 per SM): 9.23 -> 9.0 ms at n=24
    CK(cudaMemsetAsync(g_eng.alloc, 0, 8, s));
    if (tt32) {
        k_small<<<1, kTileThreads, tile_smem, s>>>(tt32, p.g, fa);
        CK(cudaGetLastError());
        tm.mark("k_small", (uint64_t)(1ull << p.H) * 4 + (bitmap_out ? S : 0));
    } else {
        CUtensorMap ma, mb;
        if ((rc = make_final_maps(p, state, &ma, &mb, fa))) return rc;
        if ((rc = launch_c0_final(p.g, ntiles, state, fa, ma, mb, s))) return rc;
        tm.mark("k_c0_final", S + (kill ? S : 0) + (bitmap_out ? S : 0));
    }
    if (ntiles <= 4096 || getenv("DQMC_NO_CUB")) {
        k_scan_tiles<<<1, 1024, 0, s>>>(g_eng.tile_cnt, g_eng.tile_pos, ntiles, g_eng.total);
        CK(cudaGetLastError());
    } else {
        // device-wide exclusive scan (CUB) of the int32 counts into int64 positions
        size_t tmp = 0;
        CK(cub::DeviceScan::ExclusiveScan(nullptr, tmp, g_eng.tile_cnt, g_eng.tile_pos, cub::Sum(), (int64_t)0,
                                          (int)ntiles, s));
        if ((rc = grow(g_eng.cub_tmp, g_eng.cub_tmp_cap, tmp, 1))) return rc;
        CK(cub::DeviceScan::ExclusiveScan(g_eng.cub_tmp, tmp, g_eng.tile_cnt, g_eng.tile_pos, cub::Sum(), (int64_t)0,
                                          (int)ntiles, s));
        k_scan_total<<<1, 32, 0, s>>>(g_eng.tile_cnt, g_eng.tile_pos, ntiles, g_eng.total);
        CK(cudaGetLastError());
    }
    tm.mark("k_scan_tiles", (uint64_t)ntiles * 12);
    if (!count_only && !direct) {
        const int grid = (int)std::min<int64_t>((ntiles + 7) / 8, (int64_t)g_eng.num_sms * 16);
        k_reorder<<<grid, 256, 0, s>>>(g_eng.scratch, g_eng.tile_base, g_eng.tile_cnt, g_eng.tile_pos, ranks, cap,
                                       ntiles, (int64_t)g_eng.scratch_cap);
        CK(cudaGetLastError());
        tm.mark("k_reorder", (uint64_t)ntiles * 16);
    }
    if (count_dev) {  // DQMC_FLAG_ASYNC: no host synchronisation
        const int64_t limit = count_only ? INT64_MAX : (direct ? cap : std::min<int64_t>(cap, (int64_t)g_eng.scratch_cap));
        k_publish_count<<<1, 1, 0, s>>>(g_eng.total, limit, count_dev);
        CK(cudaGetLastError());
        return DQMC_OK;
    }
    int64_t total = 0;
    CK(cudaMemcpyAsync(&total, g_eng.total, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    *count = total;
    return DQMC_OK;
}

// MERGE passes. full = true: every group merge-only (the complete implicant
// bitmap M is left in `state`, used by the sharded path); otherwise the last
// group is left for the fused MERGE_REDUCE pass.
int run_merge(const Plan &p, const uint32_t *tt32, uint32_t *state, bool full, Timer &tm, cudaStream_t s) {
    const uint64_t S = (uint64_t)p.nblocks * 32;
    const int tile_smem = (int)pow3l(p.g) * 32;
    const int64_t ntA = 1ll << p.T;
    const int gridA = (int)std::min<int64_t>(ntA, (int64_t)g_eng.num_sms * 8);
    k_c0_merge<<<gridA, kTileThreads, tile_smem, s>>>(tt32, state, p.g, p.T, p.pitch, p.pm ? p.r[0] : 0);
    CK(cudaGetLastError());
    tm.mark("k_c0_merge", (uint64_t)ntA * ((1ull << p.g) * 4 + (uint64_t)pow3l(p.g) * 32));
    auto frac = [&](int k) { return (double)S * std::pow(2.0 / 3.0, k); };
    const int last = full ? p.m : p.m - 1;
    for (int k = 0; k < last; k++) {
        const int64_t Q = pow3l(p.a[k] - p.g) * p.pitch;
        const int64_t ncol = (Q + kRowBlocks - 1) / kRowBlocks;
        int above = 0;
        for (int j = k + 1; j < p.m; j++) above += p.r[j];
        const int64_t nitems = ncol << above;
        launch_strided_mode<MERGE_ONLY>(p.r[k], state, Q, ncol, nitems, 0, k == 0 && p.pm, s);
        CK(cudaGetLastError());
        tm.mark("k_strided<MERGE_ONLY>", (uint64_t)frac(above));
    }
    return DQMC_OK;
}

// REDUCE passes of the strided groups. fused: the last group is merged and
// reduced in one pass (single-GPU plan); otherwise every group is reduce-only
// (sharded path, M already complete). The in-block axes of pass C go with the
// last group either way.
int run_reduce(const Plan &p, uint32_t *state, bool fused, Timer &tm, cudaStream_t s) {
    const uint64_t S = (uint64_t)p.nblocks * 32;
    int rc;
    // sparse pass D (k_reduce_sparse): piece-major group 0 behind a fused C
    // with two groups; C flags its nonzero pieces
    // Opt-in experiments, both bit-exact and both no faster than the dense TMA
    // pass at n = 24: DQMC_SPARSE_D=1 k_reduce_sparse (flagged
    // rows, cp.async), 2 k_reduce_blocks (27-row sub-blocks holding a flagged
    // row, TMA boxes). C then records its nonzero rows (+1.1 ms).
    const char *sd_env = getenv("DQMC_SPARSE_D");
    const int sparse_mode = sd_env ? atoi(sd_env) : 0;
    const bool sparse_d = fused && p.pm && p.m == 2 && p.r[0] == 6 && p.r[1] == 6 && p.ib_C && sparse_mode > 0;
    // row bits: item-major from C (ppr x 24 words), then row-major for D
    // (729 rows x PPR bits, PPR = ppr rounded up to 256, + one word of slack)
    const int64_t ppr = sparse_d ? pow3l(p.a[1] - p.g) * p.pitch / kRowBlocks : 0;
    const int64_t ppr_pad = (ppr + 255) / 256 * 256;
    uint32_t *bits_c = nullptr, *bits_d = nullptr;
    if (sparse_d) {
        const size_t wc = (size_t)ppr * 24, wd = (size_t)729 * (ppr_pad / 32) + 64;
        if ((rc = grow(g_eng.nzmap, g_eng.nzmap_cap, (wc + wd) * 4, 1))) return rc;
        bits_c = g_eng.nzmap;
        bits_d = g_eng.nzmap + wc;
    }
    {
        const int k = p.m - 1;
        const int64_t Q = pow3l(p.a[k] - p.g) * p.pitch;
        const int64_t ncol = (Q + kRowBlocks - 1) / kRowBlocks;
        if (fused) {
            if ((rc = launch_pipe_mode<MERGE_REDUCE>(p.r[k], state, Q, ncol, 1, p.ib_C, s, false, bits_c))) return rc;
            tm.mark("k_strided<MERGE_REDUCE>", (uint64_t)(S * std::pow(2.0 / 3.0, p.r[k]) + S));
            if (sparse_d) {
                k_bits_transpose<<<(unsigned)((ppr + 255) / 256), 256, 0, s>>>(bits_c, bits_d, ppr, 729, ppr_pad);
                CK(cudaGetLastError());
                tm.mark("k_bits_transpose", (uint64_t)ppr * 24 * 4 * 2);
            }
        } else {
            if ((rc = launch_pipe_mode<REDUCE_ONLY>(p.r[k], state, Q, ncol, 1, p.ib_C, s))) return rc;
            tm.mark("k_strided<REDUCE>", 2 * S);
        }
    }
    for (int k = p.m - 2; k >= 0; k--) {
        const int64_t Q = pow3l(p.a[k] - p.g) * p.pitch;
        const int64_t ncol = (Q + kRowBlocks - 1) / kRowBlocks;
        int above = 0;
        for (int j = k + 1; j < p.m; j++) above += p.r[j];
        if (k == 0 && sparse_d) {
            using SMD = PipeSmem<3, 3>;
            const int64_t nitems = (Q / kRowBlocks) * pow3l(above);
            const int grid = (int)std::min<int64_t>(nitems, g_eng.num_sms);
            if (sparse_mode == 2) {
                CUtensorMap smap;
                if ((rc = make_group_map4(&smap, state, Q, 729, pow3l(above), 27, 32, true))) return rc;
                k_reduce_blocks<3, 3><<<grid, SMD::THREADS, SMD::SMEM, s>>>(smap, bits_d, Q / kRowBlocks, nitems,
                                                                            p.ib_D[k], ppr_pad);
            } else {
                k_reduce_sparse<3, 3><<<grid, SMD::CW * 32, SMD::SMEM, s>>>(state, bits_d, nitems, p.ib_D[k],
                                                                            Q / kRowBlocks, ppr_pad);
            }
            CK(cudaGetLastError());
            tm.mark("k_reduce_sparse", 2 * S);
            if (tm.on && !tm.bytes.empty()) {  // timing mode: the bytes it moved, 2 x 128 B per flagged piece
                const int64_t nw = (int64_t)729 * (ppr_pad / 32);
                CK(cudaMemsetAsync(g_eng.alloc + 2, 0, 8, s));
                k_popc_sum<<<(unsigned)std::min<int64_t>((nw + 255) / 256, 4096), 256, 0, s>>>(bits_d, nw, g_eng.alloc + 2);
                unsigned long long nz = 0;
                CK(cudaMemcpyAsync(&nz, g_eng.alloc + 2, 8, cudaMemcpyDeviceToHost, s));
                CK(cudaStreamSynchronize(s));
                tm.bytes.back() = 2ull * 128 * nz;
            }
            continue;
        }
        if ((rc = launch_pipe_mode<REDUCE_ONLY>(p.r[k], state, Q, ncol, pow3l(above), p.ib_D[k], s, k == 0 && p.pm)))
            return rc;
        tm.mark("k_strided<REDUCE>", 2 * S);
    }
    return DQMC_OK;
}

void add_rank_bytes(Timer &tm, int64_t written) {
    if (tm.bytes.empty()) return;
    for (size_t i = 0; i < tm.names.size(); i++) {
        if (tm.names[i] == "k_c0_final" || tm.names[i] == "k_small") tm.bytes[i] += (uint64_t)written * 8;
        if (tm.names[i] == "k_reorder") tm.bytes[i] += (uint64_t)written * 16;
    }
}

// Final stage with the scratch-regrow retry (the stage does not modify the
// merged state it reads; with a bitmap output it rewrites the same P).
int run_final_retry(const Plan &p, const uint32_t *tt32, const uint32_t *state, const uint32_t *kill,
                    uint32_t ib_mask, int64_t rank_add, int64_t *ranks, int64_t cap, bool count_only,
                    uint32_t *bitmap_out, int64_t *count, Timer &tm, cudaStream_t s, int64_t *count_dev = nullptr) {
    int rc;
    if ((rc = run_final(p, tt32, state, kill, ib_mask, rank_add, ranks, cap, count_only, bitmap_out, count, tm, s,
                        count_dev)))
        return rc;
    if (count_dev) return DQMC_OK;  // async: the caller sees -(count + 1) and retries synchronously
    const bool direct = (p.T == 0);
    if (!count_only && !direct && (size_t)*count > g_eng.scratch_cap) {
        g_eng.scratch_want = (size_t)((double)*count * 1.05) + 1024;
        const bool on = tm.on;
        tm.on = false;
        rc = run_final(p, tt32, state, kill, ib_mask, rank_add, ranks, cap, count_only, bitmap_out, count, tm, s);
        tm.on = on;
        if (rc) return rc;
    }
    if (!count_only) add_rank_bytes(tm, std::min<int64_t>(*count, cap));
    return DQMC_OK;
}

// Run the whole single-GPU plan on a device-resident 32-bit truth table.
int run_plan(const Plan &p, const uint32_t *tt32, int64_t *ranks, int64_t cap, int64_t *count, uint32_t flags,
             cudaStream_t s) {
    int64_t *count_dev = (flags & DQMC_FLAG_ASYNC) ? count : nullptr;  // async: count is a device pointer
    Timer tm{(flags & DQMC_FLAG_TIMING) != 0 && !count_dev, s};
    const bool keep = (flags & DQMC_FLAG_KEEP_BITMAP) != 0;
    const bool count_only = (flags & DQMC_FLAG_COUNT_ONLY) != 0 || ranks == nullptr;
    int rc;
    const uint64_t S = (uint64_t)p.nblocks * 32;
    if (p.T > 0 || keep) {
        if ((rc = grow(g_eng.state, g_eng.state_cap, std::max<uint64_t>(S, p.sbytes), 1))) return rc;
    }
    tm.begin();
    int64_t total = 0;
    if (p.T > 0) {
        if ((rc = run_merge(p, tt32, g_eng.state, false, tm, s))) return rc;
        if ((rc = run_reduce(p, g_eng.state, true, tm, s))) return rc;
        if ((rc = run_final_retry(p, nullptr, g_eng.state, nullptr, p.ib_E, -p.rank_sub, ranks, cap, count_only,
                                  keep ? g_eng.state : nullptr, &total, tm, s, count_dev)))
            return rc;
    } else {
        if ((rc = run_final_retry(p, tt32, nullptr, nullptr, p.ib_E, -p.rank_sub, ranks, cap, count_only,
                                  keep ? g_eng.state : nullptr, &total, tm, s, count_dev)))
            return rc;
    }
    tm.finish();
    if (!count_dev) *count = total;
    note_held(p, keep);
    g_eng.state_n = keep ? p.n : -1;
    return DQMC_OK;
}

// input conversion to 32-bit truth-table words for n >= 5 (or the padded word)
int input_words(const void *in, int kind, int n, const uint32_t **tt32, cudaStream_t s) {
    int rc;
    if (n < 5) {
        if ((rc = grow(g_eng.tt_tmp, g_eng.tt_tmp_cap, 256, 1))) return rc;
        k_pad_small<<<1, 32, 0, s>>>(in, kind, n, g_eng.tt_tmp);
        CK(cudaGetLastError());
        *tt32 = g_eng.tt_tmp;
    } else if (kind == DQMC_IN_U8) {
        const int64_t nw = 1ll << (n - 5);
        if ((rc = grow(g_eng.tt_tmp, g_eng.tt_tmp_cap, (size_t)nw * 4, 1))) return rc;
        const int grid = (int)std::min<int64_t>((nw * 32 + 255) / 256, 148ll * 32);
        k_u8_to_words<<<grid, 256, 0, s>>>((const uint8_t *)in, g_eng.tt_tmp, nw);
        CK(cudaGetLastError());
        *tt32 = g_eng.tt_tmp;
    } else {
        *tt32 = (const uint32_t *)in;  // LE uint64 words viewed as uint32 words
    }
    return DQMC_OK;
}

// total device pass (input conversion + plan)
int primes_device_impl(const void *in, int kind, int n, int64_t *ranks, int64_t cap, int64_t *count,
                       uint32_t flags, cudaStream_t s) {
    const Plan p = make_plan(n, !(flags & DQMC_FLAG_KEEP_BITMAP));
    const uint32_t *tt32 = nullptr;
    int rc;
    if ((rc = input_words(in, kind, n, &tt32, s))) return rc;
    return run_plan(p, tt32, ranks, cap, count, flags, s);
}

int validate(int n, int h) {
    if (n < 1 || n > 31) return set_err(DQMC_ERR_INVALID, "variable count must be in 1..31, got " + std::to_string(n));
    if (h != 0 && (h < 1 || h > n))
        return set_err(DQMC_ERR_INVALID,
                       "split must be in 1.." + std::to_string(n) + ", got " + std::to_string(h));
    return DQMC_OK;
}

// dense.py:358-364: refuse before allocating, message names the bytes.
// Steady state (the engine already holds the buffers of a call this size, so
// nothing will be allocated) skips the free-memory query: cudaMemGetInfo is a
// driver round trip measured at p99 12 ms / max 110 ms on these boxes, which
// idled the GPU between back-to-back calls.
int check_cap(int n, int h, uint64_t mem_cap, uint64_t device_need) {
    const int hh = h == 0 ? std::min(n, 5) : h;
    const uint64_t need = state_bytes_ref(n, hh);
    const uint64_t bb = (uint64_t)state_bytes_ref(hh, hh) * 8;
    char buf[512];
    auto refuse = [&](uint64_t cap) {
        snprintf(buf, sizeof buf,
                 "dense state needs %llu bytes (%lld blocks of %llu bits), exceeding the cap of %llu bytes",
                 (unsigned long long)need, (long long)pow3l(n - hh), (unsigned long long)bb,
                 (unsigned long long)cap);
        return set_err(DQMC_ERR_RESOURCE, buf);
    };
    if (mem_cap != 0 && need > mem_cap) return refuse(mem_cap);
    if (device_need <= g_eng.held_need && need <= g_eng.state_cap) return DQMC_OK;
    size_t fr = 0, tot = 0;
    CK(cudaMemGetInfo(&fr, &tot));
    if (mem_cap == 0) {
        const uint64_t cap = (uint64_t)((double)(fr + g_eng.state_cap + g_eng.ranks_cap * 8) * 0.75);
        if (need > cap) return refuse(cap);
    }
    const uint64_t have = (uint64_t)fr + g_eng.state_cap;
    if (device_need > have) {
        snprintf(buf, sizeof buf, "device state needs %llu bytes, only %llu bytes of device memory are free",
                 (unsigned long long)device_need, (unsigned long long)have);
        return set_err(DQMC_ERR_RESOURCE, buf);
    }
    return DQMC_OK;
}

// a call of this plan finished: its buffers are held until dqmc_release
void note_held(const Plan &p, bool keep) { g_eng.held_need = std::max(g_eng.held_need, engine_device_bytes(p, keep)); }

int alloc_pinned(size_t entries, PinnedBuf &out) {
    // reuse the smallest cached buffer that fits
    int best = -1;
    for (size_t i = 0; i < g_eng.free_pinned.size(); i++)
        if (g_eng.free_pinned[i].cap >= entries && (best < 0 || g_eng.free_pinned[i].cap < g_eng.free_pinned[best].cap))
            best = (int)i;
    if (best >= 0) {
        out = g_eng.free_pinned[best];
        g_eng.free_pinned.erase(g_eng.free_pinned.begin() + best);
        return DQMC_OK;
    }
    size_t want = std::max<size_t>(entries, 1024);
    int64_t *p = nullptr;
    cudaError_t e = cudaHostAlloc((void **)&p, want * 8, cudaHostAllocDefault);
    if (e != cudaSuccess) {
        (void)cudaGetLastError();
        char buf[160];
        snprintf(buf, sizeof buf, "pinned host allocation of %llu bytes failed", (unsigned long long)(want * 8));
        return set_err(DQMC_ERR_RESOURCE, buf);
    }
    out.ptr = p;
    out.cap = want;
    return DQMC_OK;
}

// Host-API final stage, pipelined: the tiles are finished in K chunks on the
// compute stream (E, scan, running base, reorder into the device rank
// buffer); as soon as chunk c's event fires the host queues its D2H copy on
// the copy stream, so the copy engine moves chunk c while the SMs finish
// chunk c+1. Returns the total; *host_ok is false if the host buffer (sized
// from the previous call) was too small.
int run_final_pipelined(const Plan &p, const uint32_t *state, int64_t *host, int64_t host_cap, int64_t *count,
                        bool *host_ok, cudaStream_t s) {
    const int64_t ntiles = pow3l(p.T);
    const int K = (int)std::min<int64_t>(16, ntiles);
    int rc;
    if ((rc = grow(g_eng.tile_base, g_eng.tile_cap, (size_t)ntiles, 8))) return rc;
    if ((rc = grow(g_eng.tile_pos, g_eng.tile_pos_cap, (size_t)ntiles, 8))) return rc;
    if ((rc = grow(g_eng.tile_cnt, g_eng.tile_cnt_cap, (size_t)ntiles, 4))) return rc;
    if ((rc = grow(g_eng.ranks, g_eng.ranks_cap, (size_t)host_cap, 8))) return rc;
    int64_t *hbase = g_eng.hbase;  // mapped pinned mirror of the chunk bases
    for (int attempt = 0; attempt < 2; attempt++) {
        const size_t want = std::max<size_t>(g_eng.scratch_want, (size_t)1 << 20);
        if ((rc = grow(g_eng.scratch, g_eng.scratch_cap, want, 8))) return rc;
        FinalArgs fa;
        fa.out = g_eng.scratch;
        fa.cap = (int64_t)g_eng.scratch_cap;
        fa.rank_add = -p.rank_sub;
        fa.kill = nullptr;
        fa.ib_mask = p.ib_E;
        fa.bitmap_out = nullptr;
        fa.alloc = g_eng.alloc;
        fa.tile_base = g_eng.tile_base;
        fa.tile_cnt = g_eng.tile_cnt;
        fa.prefetch = 3 * g_eng.num_sms;
        fa.pitch = p.pitch;
        CUtensorMap ma, mb;
        if ((rc = make_final_maps(p, state, &ma, &mb, fa))) return rc;
        CK(cudaMemsetAsync(g_eng.alloc, 0, 8, s));
        CK(cudaMemsetAsync(g_eng.chunk_base, 0, 8, s));
        size_t tmp = 0;
        CK(cub::DeviceScan::ExclusiveScan(nullptr, tmp, g_eng.tile_cnt, g_eng.tile_pos, cub::Sum(), (int64_t)0,
                                          (int)((ntiles + K - 1) / K + 1), s));
        if ((rc = grow(g_eng.cub_tmp, g_eng.cub_tmp_cap, tmp, 1))) return rc;
        for (int c = 0; c < K; c++) {
            const int64_t t0 = ntiles * c / K, t1 = ntiles * (c + 1) / K;
            fa.tile0 = t0;
            if ((rc = launch_c0_final(p.g, t1 - t0, state, fa, ma, mb, s))) return rc;
            CK(cub::DeviceScan::ExclusiveScan(g_eng.cub_tmp, tmp, g_eng.tile_cnt + t0, g_eng.tile_pos + t0, cub::Sum(),
                                              (int64_t)0, (int)(t1 - t0), s));
            k_chunk_advance<<<1, 32, 0, s>>>(g_eng.tile_cnt + t1 - 1, g_eng.tile_pos + t1 - 1, g_eng.chunk_base + c,
                                             hbase + c);
            CK(cudaGetLastError());
            const int grid = (int)std::min<int64_t>((t1 - t0 + 7) / 8, (int64_t)g_eng.num_sms * 8);
            k_reorder<<<grid, 256, 0, s>>>(g_eng.scratch, g_eng.tile_base + t0, g_eng.tile_cnt + t0,
                                           g_eng.tile_pos + t0, g_eng.ranks, host_cap, t1 - t0,
                                           (int64_t)g_eng.scratch_cap, g_eng.chunk_base + c);
            CK(cudaGetLastError());
            CK(cudaEventRecord(g_eng.chunk_ev[c], s));
        }
        // copy-out as chunks complete (copy engine, overlapped with later chunks)
        bool fits = true;
        for (int c = 0; c < K; c++) {
            CK(cudaEventSynchronize(g_eng.chunk_ev[c]));
            const int64_t lo = hbase[c], hi = hbase[c + 1];
            if (hi > host_cap) fits = false;
            if (fits && hi > lo)
                CK(cudaMemcpyAsync(host + lo, g_eng.ranks + lo, (size_t)(hi - lo) * 8, cudaMemcpyDeviceToHost,
                                   g_eng.stream2));
        }
        int64_t used = 0;
        CK(cudaMemcpyAsync(&used, g_eng.alloc, 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        CK(cudaStreamSynchronize(g_eng.stream2));
        *count = hbase[K];
        *host_ok = fits && *count <= host_cap;
        if ((size_t)used <= g_eng.scratch_cap) break;
        g_eng.scratch_want = (size_t)((double)used * 1.05) + 1024;  // scratch overflow: once more
    }
    return DQMC_OK;
}

int primes_host_impl(const void *host_in, int kind, int n, int h, uint64_t mem_cap, uint32_t flags,
                     dqmc_result_t *out) {
    if (!out) return set_err(DQMC_ERR_INVALID, "null result pointer");
    out->count = 0;
    out->ranks = nullptr;
    out->_owner = nullptr;
    int rc;
    if ((rc = validate(n, h))) return rc;
    if (!host_in) return set_err(DQMC_ERR_INVALID, "null input pointer");
    std::lock_guard<std::mutex> lk(g_mu);
    if ((rc = ensure_device())) return rc;
    if ((rc = ensure_attrs())) return rc;
    const Plan p = make_plan(n, !(flags & DQMC_FLAG_KEEP_BITMAP));
    if ((rc = check_cap(n, h, mem_cap, engine_device_bytes(p, flags & DQMC_FLAG_KEEP_BITMAP)))) return rc;
    cudaStream_t s = g_eng.stream;
    // H2D of the input (pageable source; small relative to the state)
    const size_t in_bytes = kind == DQMC_IN_U8 ? ((size_t)1 << n) : (size_t)std::max<int64_t>(1, (1ll << n) / 64) * 8;
    if ((rc = grow(g_eng.in_tmp, g_eng.in_tmp_cap, std::max<size_t>(in_bytes, 8), 1))) return rc;
    CK(cudaMemcpyAsync(g_eng.in_tmp, host_in, in_bytes, cudaMemcpyHostToDevice, s));
    const bool count_only = (flags & DQMC_FLAG_COUNT_ONLY) != 0;
    const bool pipelined = !count_only && !(flags & (DQMC_FLAG_KEEP_BITMAP | DQMC_FLAG_TIMING)) && p.T > 0 &&
                           g_eng.hint_n == n && g_eng.hint_count > 0 && !getenv("DQMC_NO_PIPELINE");
    if (pipelined) {
        // merge/reduce passes, then the chunked final stage straight into pinned host memory
        const uint32_t *tt32 = nullptr;
        if ((rc = input_words(g_eng.in_tmp, kind, n, &tt32, s))) return rc;
        if ((rc = grow(g_eng.state, g_eng.state_cap, (size_t)p.sbytes, 1))) return rc;
        Timer tm{false, s};
        if ((rc = run_merge(p, tt32, g_eng.state, false, tm, s))) return rc;
        if ((rc = run_reduce(p, g_eng.state, true, tm, s))) return rc;
        PinnedBuf pb;
        if ((rc = alloc_pinned((size_t)((double)g_eng.hint_count * 1.02) + 4096, pb))) return rc;
        int64_t count = 0;
        bool ok = true;
        if ((rc = run_final_pipelined(p, g_eng.state, pb.ptr, (int64_t)pb.cap, &count, &ok, s))) return rc;
        if (!ok) {  // the output outgrew the hinted buffer: rerun the stage into a larger one
            g_eng.free_pinned.push_back(pb);
            if ((rc = alloc_pinned((size_t)count, pb))) return rc;
            if ((rc = run_final_pipelined(p, g_eng.state, pb.ptr, (int64_t)pb.cap, &count, &ok, s))) return rc;
        }
        g_eng.hint_count = count;
        out->count = count;
        if (count > 0) {
            out->ranks = pb.ptr;
            out->_owner = new PinnedBuf(pb);
        } else {
            g_eng.free_pinned.push_back(pb);
        }
        return DQMC_OK;
    }
    if (!count_only && g_eng.ranks_cap == 0) {
        if ((rc = grow(g_eng.ranks, g_eng.ranks_cap, (size_t)1 << 20, 8))) return rc;
    }
    int64_t count = 0;
    if ((rc = primes_device_impl(g_eng.in_tmp, kind, n, count_only ? nullptr : g_eng.ranks, (int64_t)g_eng.ranks_cap,
                                 &count, flags, s)))
        return rc;
    if (!count_only && (size_t)count > g_eng.ranks_cap) {
        // grow the output and run again (only the count was exact)
        if ((rc = grow(g_eng.ranks, g_eng.ranks_cap, (size_t)((double)count * 1.05) + 1024, 8))) return rc;
        if ((rc = primes_device_impl(g_eng.in_tmp, kind, n, g_eng.ranks, (int64_t)g_eng.ranks_cap, &count, flags, s)))
            return rc;
    }
    out->count = count;
    if (!count_only) {
        g_eng.hint_n = n;
        g_eng.hint_count = count;
    }
    if (!count_only && count > 0) {
        PinnedBuf pb;
        if ((rc = alloc_pinned((size_t)count, pb))) return rc;
        CK(cudaMemcpyAsync(pb.ptr, g_eng.ranks, (size_t)count * 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        PinnedBuf *owner = new PinnedBuf(pb);
        out->ranks = pb.ptr;
        out->_owner = owner;
    }
    return DQMC_OK;
}

// Host-API jobs, up to kJobSlots (3) in flight: submit queues the H2D of the table, every pass
// and the final stage on the engine stream and returns; collect waits for the
// job's final stage, then copies its ranks to pinned host memory on the copy
// stream while the engine stream already runs the next job. A stream of calls
// thus overlaps call i's D2H with call i+1's passes. The first job of an n (no
// count hint yet to size the outputs) runs synchronously inside submit.
int submit_impl(const void *host_in, int kind, int n, uint32_t flags, int64_t *job_out) {
    if (!job_out) return set_err(DQMC_ERR_INVALID, "null job pointer");
    int rc;
    if ((rc = validate(n, 0))) return rc;
    if (!host_in) return set_err(DQMC_ERR_INVALID, "null input pointer");
    {
        std::lock_guard<std::mutex> lk(g_mu);
        if ((rc = ensure_device())) return rc;
        if ((rc = ensure_attrs())) return rc;
        if (g_eng.jobs.size() >= (size_t)kJobSlots)
            return set_err(DQMC_ERR_INVALID, "three jobs outstanding: collect the oldest first");
        const Plan p = make_plan(n);
        const bool async = !(flags & (DQMC_FLAG_COUNT_ONLY | DQMC_FLAG_KEEP_BITMAP | DQMC_FLAG_TIMING)) && p.T > 0 &&
                           g_eng.hint_n == n && g_eng.hint_count > 0;
        if (async) {
            if ((rc = check_cap(n, 0, 0, engine_device_bytes(p, false)))) return rc;
            const int64_t id = g_eng.next_job++;
            const int slot = (int)(id % kJobSlots);
            if (!g_eng.jcount_host)
                CK(cudaHostAlloc((void **)&g_eng.jcount_host, kJobSlots * sizeof(int64_t), cudaHostAllocDefault));
            if (!g_eng.jev[slot]) CK(cudaEventCreateWithFlags(&g_eng.jev[slot], cudaEventDisableTiming));
            const size_t in_bytes =
                kind == DQMC_IN_U8 ? ((size_t)1 << n) : (size_t)std::max<int64_t>(1, (1ll << n) / 64) * 8;
            if ((rc = grow(g_eng.jin[slot], g_eng.jin_cap[slot], std::max<size_t>(in_bytes, 8), 1))) return rc;
            const size_t want = (size_t)((double)g_eng.hint_count * 1.05) + 4096;
            if ((rc = grow(g_eng.jranks[slot], g_eng.jranks_cap[slot], want, 8))) return rc;
            g_eng.scratch_want = std::max(g_eng.scratch_want, want);
            if ((rc = grow(g_eng.state, g_eng.state_cap, (size_t)p.sbytes, 1))) return rc;
            cudaStream_t s = g_eng.stream;
            CK(cudaMemcpyAsync(g_eng.jin[slot], host_in, in_bytes, cudaMemcpyHostToDevice, s));
            const uint32_t *tt32 = nullptr;
            if ((rc = input_words(g_eng.jin[slot], kind, n, &tt32, s))) return rc;
            Timer tm{false, s};
            if ((rc = run_merge(p, tt32, g_eng.state, false, tm, s))) return rc;
            if ((rc = run_reduce(p, g_eng.state, true, tm, s))) return rc;
            int64_t unused = 0;
            int64_t *cdev = g_eng.total + 8 + slot;  // device count of this slot (-(count+1): outputs too small)
            if ((rc = run_final(p, nullptr, g_eng.state, nullptr, p.ib_E, -p.rank_sub, g_eng.jranks[slot],
                                (int64_t)g_eng.jranks_cap[slot], false, nullptr, &unused, tm, s, cdev)))
                return rc;
            CK(cudaMemcpyAsync(g_eng.jcount_host + slot, cdev, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
            CK(cudaEventRecord(g_eng.jev[slot], s));
            Job j;
            j.id = id;
            j.slot = slot;
            j.in = host_in;
            j.kind = kind;
            j.n = n;
            j.flags = flags;
            g_eng.jobs.push_back(j);
            *job_out = id;
            return DQMC_OK;
        }
    }
    dqmc_result_t res{};
    if ((rc = primes_host_impl(host_in, kind, n, 0, 0, flags, &res))) return rc;
    std::lock_guard<std::mutex> lk(g_mu);
    Job j;
    j.id = g_eng.next_job++;
    j.res = res;
    g_eng.jobs.push_back(j);
    *job_out = j.id;
    return DQMC_OK;
}

int collect_impl(int64_t job, dqmc_result_t *out) {
    if (!out) return set_err(DQMC_ERR_INVALID, "null result pointer");
    out->count = 0;
    out->ranks = nullptr;
    out->_owner = nullptr;
    std::unique_lock<std::mutex> lk(g_mu);
    if (g_eng.jobs.empty() || g_eng.jobs.front().id != job)
        return set_err(DQMC_ERR_INVALID, "unknown job, or jobs collected out of submission order");
    const Job j = g_eng.jobs.front();
    g_eng.jobs.pop_front();
    if (j.slot < 0) {
        *out = j.res;
        return DQMC_OK;
    }
    CK(cudaEventSynchronize(g_eng.jev[j.slot]));
    const int64_t c = g_eng.jcount_host[j.slot];
    if (c < 0) {  // the hinted output was too small: run this job again, synchronously
        g_eng.hint_count = -c - 1;
        g_eng.scratch_want = std::max(g_eng.scratch_want, (size_t)((double)(-c - 1) * 1.05) + 4096);
        lk.unlock();
        return primes_host_impl(j.in, j.kind, j.n, 0, 0, j.flags, out);
    }
    g_eng.hint_count = c;
    if (c > 0) {
        PinnedBuf pb;
        int rc;
        if ((rc = alloc_pinned((size_t)c, pb))) return rc;
        CK(cudaMemcpyAsync(pb.ptr, g_eng.jranks[j.slot], (size_t)c * 8, cudaMemcpyDeviceToHost, g_eng.stream2));
        CK(cudaStreamSynchronize(g_eng.stream2));
        out->count = c;
        out->ranks = pb.ptr;
        out->_owner = new PinnedBuf(pb);
    }
    return DQMC_OK;
}

}  // namespace

// ---------------------------------------------------------------------------
// C ABI

// shared error channel of the state API (dqmc_state.cu); not part of the ABI
extern "C" __attribute__((visibility("hidden"))) void dqmc_internal_set_error(const char *m) { g_err = m; }

extern "C" {

int dqmc_abi_version(void) { return DQMC_ABI_VERSION; }

const char *dqmc_last_error(void) { return g_err.c_str(); }

int dqmc_device_count(void) {
    int c = 0;
    if (cudaGetDeviceCount(&c) != cudaSuccess) {
        (void)cudaGetLastError();
        return 0;
    }
    return c;
}

int dqmc_set_device(int device) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (g_eng.device == device) return DQMC_OK;
    if (g_eng.device >= 0) return set_err(DQMC_ERR_INVALID, "device already selected; call dqmc_release first");
    CK(cudaSetDevice(device));
    return DQMC_OK;
}

uint64_t dqmc_block_bits(int h) { return state_bytes_ref(h, h) * 8; }

uint64_t dqmc_state_bytes(int n, int h) { return state_bytes_ref(n, h); }

uint64_t dqmc_device_bytes(int n) {
    if (n < 1 || n > 31) return 0;
    return engine_device_bytes(make_plan(n), false);
}

int dqmc_primes_tt(const uint64_t *tt_words, int n, int h, uint64_t mem_cap, uint32_t flags, dqmc_result_t *out) {
    return primes_host_impl(tt_words, DQMC_IN_WORDS, n, h, mem_cap, flags, out);
}

int dqmc_primes_u8(const uint8_t *values, int n, int h, uint64_t mem_cap, uint32_t flags, dqmc_result_t *out) {
    return primes_host_impl(values, DQMC_IN_U8, n, h, mem_cap, flags, out);
}

void dqmc_free_result(dqmc_result_t *res) {
    if (!res) return;
    if (res->_owner) {
        std::lock_guard<std::mutex> lk(g_mu);
        PinnedBuf *pb = (PinnedBuf *)res->_owner;
        g_eng.free_pinned.push_back(*pb);
        // keep at most two cached pinned buffers
        while (g_eng.free_pinned.size() > 2) {
            auto it = std::min_element(g_eng.free_pinned.begin(), g_eng.free_pinned.end(),
                                       [](const PinnedBuf &a, const PinnedBuf &b) { return a.cap < b.cap; });
            cudaFreeHost(it->ptr);
            g_eng.free_pinned.erase(it);
        }
        delete pb;
    }
    res->_owner = nullptr;
    res->ranks = nullptr;
    res->count = 0;
}

int dqmc_primes_device(const void *input_dev, int in_kind, int n, int64_t *ranks_dev, int64_t ranks_cap,
                       int64_t *count_out, uint32_t flags, void *stream) {
    int rc;
    if ((rc = validate(n, 0))) return rc;
    if (!input_dev || !count_out) return set_err(DQMC_ERR_INVALID, "null pointer argument");
    if (in_kind != DQMC_IN_WORDS && in_kind != DQMC_IN_U8) return set_err(DQMC_ERR_INVALID, "bad input kind");
    std::lock_guard<std::mutex> lk(g_mu);
    if ((rc = ensure_device())) return rc;
    if ((rc = ensure_attrs())) return rc;
    const Plan p = make_plan(n, !(flags & DQMC_FLAG_KEEP_BITMAP));
    if ((rc = check_cap(n, 0, 0, engine_device_bytes(p, flags & DQMC_FLAG_KEEP_BITMAP)))) return rc;
    cudaStream_t s = (cudaStream_t)stream;  // 0 = the legacy default stream (CUDA convention)
    if (!ranks_dev) flags |= DQMC_FLAG_COUNT_ONLY;
    return primes_device_impl(input_dev, in_kind, n, ranks_dev, ranks_cap, count_out, flags, s);
}

int dqmc_last_timings(const char **names, float *ms, int max) {
    const int k = (int)g_eng.pass_ms.size();
    for (int i = 0; i < k && i < max; i++) {
        if (names) names[i] = g_eng.pass_names[i].c_str();
        if (ms) ms[i] = g_eng.pass_ms[i];
    }
    return k;
}

int dqmc_last_pass_bytes(uint64_t *bytes, int max) {
    const int k = (int)g_eng.pass_bytes.size();
    for (int i = 0; i < k && i < max; i++) bytes[i] = g_eng.pass_bytes[i];
    return k;
}

int dqmc_bitmap_device(void **ptr, uint64_t *bytes) {
    if (g_eng.state_n < 0) return set_err(DQMC_ERR_INVALID, "no bitmap held: run with DQMC_FLAG_KEEP_BITMAP");
    const Plan p = make_plan(g_eng.state_n, false);
    if (ptr) *ptr = g_eng.state;
    if (bytes) *bytes = (uint64_t)p.nblocks * 32;
    return DQMC_OK;
}

int dqmc_bitmap_download(void *host, uint64_t bytes) {
    if (g_eng.state_n < 0) return set_err(DQMC_ERR_INVALID, "no bitmap held: run with DQMC_FLAG_KEEP_BITMAP");
    const Plan p = make_plan(g_eng.state_n, false);
    const uint64_t need = (uint64_t)p.nblocks * 32;
    if (bytes < need) return set_err(DQMC_ERR_INVALID, "host buffer too small");
    CK(cudaMemcpy(host, g_eng.state, need, cudaMemcpyDeviceToHost));
    return DQMC_OK;
}

int dqmc_gen3_range_device(uint8_t *values_dev, int64_t x0, int64_t count, double p_on, double p_dc, uint64_t seed,
                           void *stream) {
    int rc;
    if (!values_dev || x0 < 0 || count < 0) return set_err(DQMC_ERR_INVALID, "bad generator range");
    std::lock_guard<std::mutex> lk(g_mu);
    if ((rc = ensure_device())) return rc;
    cudaStream_t s = (cudaStream_t)stream;  // 0 = the legacy default stream (CUDA convention)
    // int(p * 2^53) as Python computes it (float64 product, truncation)
    const uint64_t t_on = (uint64_t)(p_on * 9007199254740992.0);
    const uint64_t t_any = (uint64_t)((p_on + p_dc) * 9007199254740992.0);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((count + 255) / 256, 148ll * 64));
    if (count) k_gen3<<<grid, 256, 0, s>>>(values_dev, x0, count, seed, t_on, t_any);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(s));
    return DQMC_OK;
}

int dqmc_gen3_device(uint8_t *values_dev, int n, double p_on, double p_dc, uint64_t seed, void *stream) {
    int rc;
    if ((rc = validate(n, 0))) return rc;
    return dqmc_gen3_range_device(values_dev, 0, 1ll << n, p_on, p_dc, seed, stream);
}

int dqmc_submit_tt(const uint64_t *tt_words, int n, uint32_t flags, int64_t *job) {
    return submit_impl(tt_words, DQMC_IN_WORDS, n, flags, job);
}

int dqmc_submit_u8(const uint8_t *values, int n, uint32_t flags, int64_t *job) {
    return submit_impl(values, DQMC_IN_U8, n, flags, job);
}

int dqmc_collect(int64_t job, dqmc_result_t *out) { return collect_impl(job, out); }

int dqmc_ipc_get(const void *dev_ptr, void *handle_out, uint64_t *offset_out) {
    if (!dev_ptr || !handle_out || !offset_out) return set_err(DQMC_ERR_INVALID, "null pointer argument");
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
    int rc;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        if ((rc = ensure_device())) return rc;
        if (!g_eng.addr_range) {
            void *fn = nullptr;
            cudaDriverEntryPointQueryResult q;
            CK(cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q));
            if (!fn || q != cudaDriverEntryPointSuccess) return set_err(DQMC_ERR_CUDA, "cuMemGetAddressRange unavailable");
            g_eng.addr_range = (AddrRangeFn)fn;
        }
    }
    CUdeviceptr base = 0;
    size_t size = 0;
    const CUresult r = g_eng.addr_range(&base, &size, (CUdeviceptr)dev_ptr);
    if (r != CUDA_SUCCESS) return set_err(DQMC_ERR_INVALID, "not a device allocation: " + std::to_string((int)r));
    cudaIpcMemHandle_t h;
    CK(cudaIpcGetMemHandle(&h, (void *)base));
    memcpy(handle_out, &h, sizeof h);
    *offset_out = (uint64_t)((CUdeviceptr)dev_ptr - base);
    return DQMC_OK;
}

int dqmc_ipc_open(const void *handle, void **base_out) {
    if (!handle || !base_out) return set_err(DQMC_ERR_INVALID, "null pointer argument");
    int rc;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        if ((rc = ensure_device())) return rc;
    }
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof h);
    CK(cudaIpcOpenMemHandle(base_out, h, cudaIpcMemLazyEnablePeerAccess));
    return DQMC_OK;
}

int dqmc_ipc_close(void *base) {
    if (!base) return set_err(DQMC_ERR_INVALID, "null pointer argument");
    CK(cudaIpcCloseMemHandle(base));
    return DQMC_OK;
}

int dqmc_gen_sbox_device(uint8_t *values_dev, uint64_t seed, void *stream) {
    int rc;
    if (!values_dev) return set_err(DQMC_ERR_INVALID, "null output");
    std::lock_guard<std::mutex> lk(g_mu);
    if ((rc = ensure_device())) return rc;
    cudaStream_t s = (cudaStream_t)stream;
    CK(cudaMemsetAsync(values_dev, 1, (size_t)1 << 20, s));
    k_sbox<<<1, 1024, 0, s>>>(values_dev, seed);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(s));
    return DQMC_OK;
}

int dqmc_gen_sbox_host(uint8_t *values_host, uint64_t seed) {
    int rc;
    if (!values_host) return set_err(DQMC_ERR_INVALID, "null output");
    {
        std::lock_guard<std::mutex> lk(g_mu);
        if ((rc = ensure_device())) return rc;
        if ((rc = grow(g_eng.in_tmp, g_eng.in_tmp_cap, (size_t)1 << 20, 1))) return rc;
    }
    if ((rc = dqmc_gen_sbox_device((uint8_t *)g_eng.in_tmp, seed, g_eng.stream))) return rc;
    CK(cudaMemcpy(values_host, g_eng.in_tmp, (size_t)1 << 20, cudaMemcpyDeviceToHost));
    return DQMC_OK;
}

int dqmc_gen3_host(uint8_t *values_host, int n, double p_on, double p_dc, uint64_t seed) {
    int rc;
    if ((rc = validate(n, 0))) return rc;
    if (!values_host) return set_err(DQMC_ERR_INVALID, "null output");
    {
        std::lock_guard<std::mutex> lk(g_mu);
        if ((rc = ensure_device())) return rc;
        if ((rc = grow(g_eng.in_tmp, g_eng.in_tmp_cap, (size_t)1 << n, 1))) return rc;
    }
    if ((rc = dqmc_gen3_range_device((uint8_t *)g_eng.in_tmp, 0, 1ll << n, p_on, p_dc, seed, g_eng.stream))) return rc;
    CK(cudaMemcpy(values_host, g_eng.in_tmp, (size_t)1 << n, cudaMemcpyDeviceToHost));
    return DQMC_OK;
}

int dqmc_order_by_weight(const int64_t *ranks_host, int64_t count, int n, int64_t *out_host) {
    int rc;
    if ((rc = validate(n, 0))) return rc;
    if (count < 0 || (count && (!ranks_host || !out_host))) return set_err(DQMC_ERR_INVALID, "bad arguments");
    if (count == 0) return DQMC_OK;
    std::lock_guard<std::mutex> lk(g_mu);
    if ((rc = ensure_device())) return rc;
    cudaStream_t s = g_eng.stream;
    int64_t *r_in = nullptr, *r_out = nullptr;
    uint8_t *k_in = nullptr, *k_out = nullptr;
    void *tmp = nullptr;
    size_t tmpb = 0;
    CK(cudaMalloc(&r_in, (size_t)count * 8));
    CK(cudaMalloc(&r_out, (size_t)count * 8));
    CK(cudaMalloc(&k_in, (size_t)count));
    CK(cudaMalloc(&k_out, (size_t)count));
    CK(cudaMemcpyAsync(r_in, ranks_host, (size_t)count * 8, cudaMemcpyHostToDevice, s));
    const int grid = (int)std::min<int64_t>((count + 255) / 256, 148ll * 32);
    k_weight_keys<<<grid, 256, 0, s>>>(r_in, count, n, k_in);
    CK(cudaGetLastError());
    CK(cub::DeviceRadixSort::SortPairs(nullptr, tmpb, k_in, k_out, r_in, r_out, (int)count, 0, 8, s));
    CK(cudaMalloc(&tmp, tmpb));
    CK(cub::DeviceRadixSort::SortPairs(tmp, tmpb, k_in, k_out, r_in, r_out, (int)count, 0, 8, s));
    CK(cudaMemcpyAsync(out_host, r_out, (size_t)count * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    cudaFree(r_in);
    cudaFree(r_out);
    cudaFree(k_in);
    cudaFree(k_out);
    cudaFree(tmp);
    return DQMC_OK;
}

int dqmc_merge_device(const void *input_dev, int in_kind, int n, uint32_t *state_out, void *stream) {
    int rc;
    if ((rc = validate(n, 0))) return rc;
    if (n < 5) return set_err(DQMC_ERR_INVALID, "dqmc_merge_device needs n >= 5 (h=5 layout)");
    if (!input_dev || !state_out) return set_err(DQMC_ERR_INVALID, "null pointer argument");
    std::lock_guard<std::mutex> lk(g_mu);
    if ((rc = ensure_device())) return rc;
    if ((rc = ensure_attrs())) return rc;
    cudaStream_t s = (cudaStream_t)stream;  // 0 = the legacy default stream (CUDA convention)
    const Plan p = make_plan(n, false);  // caller-owned state in the reference layout
    const uint32_t *tt32 = nullptr;
    if ((rc = input_words(input_dev, in_kind, n, &tt32, s))) return rc;
    Timer tm{false, s};
    if ((rc = run_merge(p, tt32, state_out, true, tm, s))) return rc;
    CK(cudaStreamSynchronize(s));
    return DQMC_OK;
}

int dqmc_reduce_extract_device(uint32_t *state, int n, const uint32_t *kill, int64_t rank_offset, int64_t *ranks_dev,
                               int64_t ranks_cap, int64_t *count_out, uint32_t flags, void *stream) {
    int rc;
    if ((rc = validate(n, 0))) return rc;
    if (n < 5) return set_err(DQMC_ERR_INVALID, "dqmc_reduce_extract_device needs n >= 5 (h=5 layout)");
    if (!state || !count_out) return set_err(DQMC_ERR_INVALID, "null pointer argument");
    std::lock_guard<std::mutex> lk(g_mu);
    if ((rc = ensure_device())) return rc;
    if ((rc = ensure_attrs())) return rc;
    cudaStream_t s = (cudaStream_t)stream;  // 0 = the legacy default stream (CUDA convention)
    const Plan p = make_plan(n, false);  // caller-owned state in the reference layout
    const bool count_only = (flags & DQMC_FLAG_COUNT_ONLY) != 0 || ranks_dev == nullptr;
    Timer tm{(flags & DQMC_FLAG_TIMING) != 0, s};
    tm.begin();
    if (p.T > 0 && (rc = run_reduce(p, state, false, tm, s))) return rc;
    if ((rc = run_final_retry(p, nullptr, state, kill, p.ib_E, rank_offset, ranks_dev, ranks_cap, count_only,
                              (flags & DQMC_FLAG_KEEP_BITMAP) ? state : nullptr, count_out, tm, s)))
        return rc;
    tm.finish();
    return DQMC_OK;
}

int dqmc_bitop_device(uint32_t *dst, const uint32_t *a, const uint32_t *b, uint64_t nbytes, int op, void *stream) {
    int rc;
    if (!dst || !a || !b || (nbytes % 16) || (op != 0 && op != 1))
        return set_err(DQMC_ERR_INVALID, "bitop: null pointer, size not a multiple of 16, or bad op");
    std::lock_guard<std::mutex> lk(g_mu);
    if ((rc = ensure_device())) return rc;
    cudaStream_t s = (cudaStream_t)stream;  // 0 = the legacy default stream (CUDA convention)
    const int64_t n16 = (int64_t)(nbytes / 16);
    const int grid = (int)std::min<int64_t>((n16 + 255) / 256, 148ll * 16);
    if (n16) k_bitop<<<grid, 256, 0, s>>>((uint4 *)dst, (const uint4 *)a, (const uint4 *)b, n16, op);
    CK(cudaGetLastError());
    return DQMC_OK;
}

int dqmc_plan(int n, int64_t *out, int max) {
    if (n < 1 || n > 31 || !out) return 0;
    const Plan p = make_plan(n);
    int64_t v[32];
    int k = 0;
    v[k++] = p.ne;
    v[k++] = p.H;
    v[k++] = p.g;
    v[k++] = p.T;
    v[k++] = p.m;
    for (int i = 0; i < 8; i++) v[k++] = p.r[i];
    for (int i = 0; i < 8; i++) v[k++] = p.a[i];
    v[k++] = p.ib_C;
    v[k++] = p.ib_E;
    for (int i = 0; i < 8; i++) v[k++] = p.ib_D[i];
    v[k++] = p.rank_sub;
    const int w = std::min(k, max);
    for (int i = 0; i < w; i++) out[i] = v[i];
    return w;
}

void dqmc_release(void) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (g_eng.device < 0) return;
    cudaFree(g_eng.state);
    cudaFree(g_eng.nzmap);
    cudaFree(g_eng.tile_base);
    cudaFree(g_eng.tile_pos);
    cudaFree(g_eng.tile_cnt);
    cudaFree(g_eng.scratch);
    cudaFree(g_eng.alloc);
    cudaFree(g_eng.cub_tmp);
    cudaFree(g_eng.total);
    cudaFree(g_eng.tt_tmp);
    cudaFree(g_eng.in_tmp);
    cudaFree(g_eng.ranks);
    for (auto &b : g_eng.free_pinned) cudaFreeHost(b.ptr);
    if (g_eng.stream) cudaStreamDestroy(g_eng.stream);
    if (g_eng.stream2) cudaStreamDestroy(g_eng.stream2);
    for (int i = 0; i < 16; i++)
        if (g_eng.chunk_ev[i]) cudaEventDestroy(g_eng.chunk_ev[i]);
    cudaFree(g_eng.chunk_base);
    if (g_eng.hbase) cudaFreeHost(g_eng.hbase);
    for (int i = 0; i < kJobSlots; i++) {
        cudaFree(g_eng.jin[i]);
        cudaFree(g_eng.jranks[i]);
        if (g_eng.jev[i]) cudaEventDestroy(g_eng.jev[i]);
    }
    if (g_eng.jcount_host) cudaFreeHost(g_eng.jcount_host);
    g_eng = Engine();
}

}  // extern "C"
