// dqmc_final.cu — final stage E: REDUCE of the C0 axes, popcount and ordered
// compaction (extract_ranks, dense.py:376-397).
//
// Rank order is memory order in the reference layout (block a, bit b = rank
// a*243 + b), so compaction needs no sort: each tile writes its primes to a
// scratch range (its own fixed slot in the n = 24 plan, else a range reserved
// with one atomic), a scan of the per-tile counts gives every tile its
// rank-order position, and k_reorder moves the ranks there.
//
// A tile is finished one of two ways: sparse tiles reduce each
// nonzero block on its own as one parallel REDUCE step from the unmodified
// tile (tile_finish_sparse / prime_block); dense tiles go through register
// sub-cube rounds over every word (tile_reduce_c0_t) and tile_finish.
#include <cub/device/device_scan.cuh>

#include <type_traits>

#include "dqmc_internal.cuh"

namespace dqmc {
namespace {

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


// Gather finish: group-0 kills of block b of tile (u, l) read from the state.
// gb = the tile's piece 0 at row l; piece x = b / 4 is x * nr rows further;
// goff[j] = (2 - d_j) 3^j rows in words (0: digit j of l is already 2, no
// parent). Every lane reads a different 32-B sector: one 256-bit load per
// parent (the cost is the L1 tag stage, one lookup per lane and instruction).
struct Blk256 {
    uint32_t w[8];
};
__device__ __forceinline__ Blk256 ld256_nc(const uint32_t *p) {
    Blk256 r;
    // no L1 allocation: a parent sector is used once per tile (12.3 vs 12.7 ms)
    asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r.w[0]), "=r"(r.w[1]), "=r"(r.w[2]), "=r"(r.w[3]), "=r"(r.w[4]), "=r"(r.w[5]), "=r"(r.w[6]),
                   "=r"(r.w[7])
                 : "l"(p));
    return r;
}
__device__ __forceinline__ void g0_kill(const uint32_t *__restrict__ gb, int nr32, const int *goff, int b,
                                        uint32_t (&v)[8]) {
    const uint32_t *p = gb + (b >> 2) * nr32 + (b & 3) * 8;
    uint32_t k[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
#pragma unroll
    for (int j = 0; j < kGroupMax; j++) {
        const int o = goff[j];
        if (o) {
            const Blk256 a = ld256_nc(p + o);
#pragma unroll
            for (int i = 0; i < 8; i++) k[i] |= a.w[i];
        }
    }
#pragma unroll
    for (int i = 0; i < 8; i++) v[i] &= ~k[i];
}

// In-block reduce, popcount and ordered compaction of one tile
// (dense.py:376-397 extract_ranks: rank = block*243 + bit; memory order is
// rank order, so the output needs no sort). Warp w owns the contiguous block
// range [b0, b1); lane l takes blocks b0+l, b0+l+32, ... (group j = the j-th
// 32 blocks). Block counts stay in registers, two 16-bit fields per word, so
// one packed warp scan serves every group: the phases are short latency
// chains, which is what bounds this pass (3 CTAs/SM, smem-limited).
// Scratch range of a tile's primes: its own fixed slot when it fits (no
// atomic in the tile's latency chain), else a range of the overflow pool
// reserved with one atomic.
__device__ __forceinline__ int64_t tile_range(const FinalArgs &fa, int64_t tile, int64_t cnt) {
    if (!cnt) return 0;
    if (cnt <= fa.slot) return tile * fa.slot;
    return fa.ovf0 + (int64_t)atomicAdd(fa.alloc, (unsigned long long)cnt);
}

template <int NT>
__host__ __device__ constexpr int finish_iters() {  // ceil(max warp range / 32)
    return ((kC0MaxBlocks + NT / 32 - 1) / (NT / 32) + 31) / 32;
}

// shared scratch of the final stage (one instance per kernel, both paths)
// (block counts are <= 243; range-relative block indices fit a byte when a
// warp's range is at most 256 blocks: 3 CTAs of E fit the SM only so)
template <int NT>
struct FinishSmem {
    using Idx = typename std::conditional<(finish_iters<NT>() * 32 <= 256), uint8_t, uint16_t>::type;
    int64_t warp_off[NT / 32];
    int64_t tile_off;
    Idx lst[NT / 32][finish_iters<NT>() * 32];       // nonzero blocks / the emission list
    uint8_t lcnt[NT / 32][finish_iters<NT>() * 32];  // block popcounts / prime counts of the listed blocks
};

template <int NT>
__device__ __forceinline__ void tile_finish(uint32_t *sm, int nb, int64_t tile, int64_t blk0, const FinalArgs &fa,
                                            FinishSmem<NT> &fs, const uint32_t *gb = nullptr, int nr32 = 0,
                                            const int *goff = nullptr) {
    constexpr int kMaxIter = finish_iters<NT>();
    constexpr int kPk = (kMaxIter + 1) / 2;
    int64_t *s_warp_off = fs.warp_off;
    int64_t &s_tile_off = fs.tile_off;
    uint8_t(*s_cnt)[kMaxIter][32] = reinterpret_cast<uint8_t(*)[kMaxIter][32]>(&fs.lcnt[0][0]);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int nwarps = NT / 32;  // compile-time: the range split needs no runtime division
    const int b0 = nb * warp / nwarps, b1 = nb * (warp + 1) / nwarps;
    const int h = (lane >> 2) & 1;  // half-swap: conflict-free LDS.128 at 32-B lane stride
    const uint32_t ibm = fa.ib_mask | (gb ? fa.ib_gather : 0u);  // gather finish: pass D's in-block axes too

    // (1) lane = block: popcount (+ in-block axes, kills, bitmap on the slow path)
    uint32_t pk[kPk];
#pragma unroll
    for (int i = 0; i < kPk; i++) pk[i] = 0;
    // sharded path: this tile's super-block (slot), its parents and rank offset
    const int64_t slot = fa.kill_tab || fa.rank_add_tab ? tile / fa.tiles_per_slot : 0;
    const int64_t slot_blk0 = slot * fa.tiles_per_slot * nb;  // first block of the slot
    const int64_t rank_add = fa.rank_add_tab ? fa.rank_add_tab[slot] - slot_blk0 * 243 : fa.rank_add;
    const uint64_t *kills = fa.kill_tab ? fa.kill_tab + slot * kMaxKill : nullptr;
    if (!ibm && !kills && !fa.bitmap_out && !gb) {  // count only: word order does not matter
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
                if (ibm) {
                    uint32_t v[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
                    inblock_reduce(v, ibm);
                    x0 = make_uint4(v[0], v[1], v[2], v[3]);
                    x1 = make_uint4(v[4], v[5], v[6], v[7]);
                }
                if (kills && (x0.x | x0.y | x0.z | x0.w | x1.x | x1.y | x1.z | x1.w)) {
                    // top-axis parents (sharded path): OR of up to kMaxKill
                    // super-blocks read in place, local or peer memory over NVLink;
                    // only under a nonzero block (~15% at config 4: a zero block
                    // stays zero, so most parent reads are skipped)
                    uint4 k0 = make_uint4(0, 0, 0, 0), k1 = k0;
#pragma unroll
                    for (int q = 0; q < kMaxKill; q++) {  // unrolled: every parent's load in flight at once
                        const uint64_t kp = __ldg(&kills[q]);
                        if (kp) {
                            const uint4 *kq = reinterpret_cast<const uint4 *>(reinterpret_cast<const uint32_t *>(kp) +
                                                                              (blk0 + b - slot_blk0) * 8);
                            const uint4 a0 = kq[0], a1 = kq[1];
                            k0 = make_uint4(k0.x | a0.x, k0.y | a0.y, k0.z | a0.z, k0.w | a0.w);
                            k1 = make_uint4(k1.x | a1.x, k1.y | a1.y, k1.z | a1.z, k1.w | a1.w);
                        }
                    }
                    x0 = make_uint4(x0.x & ~k0.x, x0.y & ~k0.y, x0.z & ~k0.z, x0.w & ~k0.w);
                    x1 = make_uint4(x1.x & ~k1.x, x1.y & ~k1.y, x1.z & ~k1.z, x1.w & ~k1.w);
                }
                if (gb && (x0.x | x0.y | x0.z | x0.w | x1.x | x1.y | x1.z | x1.w)) {
                    uint32_t v[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
                    g0_kill(gb, nr32, goff, b, v);
                    x0 = make_uint4(v[0], v[1], v[2], v[3]);
                    x1 = make_uint4(v[4], v[5], v[6], v[7]);
                }
                if (ibm || kills || gb) {
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
            s_cnt[warp][j][lane] = (uint8_t)cj;
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
        const int64_t base = tile_range(fa, tile, acc);
        fa.tile_base[tile] = base;
        fa.tile_cnt[tile] = (int32_t)acc;
        if (fa.tile_rank0) fa.tile_rank0[tile] = blk0 * 243 + rank_add;
        s_tile_off = base;
    }
    __syncthreads();
    if (fa.out == nullptr && fa.out32 == nullptr) return;

    // (4) ordered emission. Primes are sparse (~0.2 per block at n = 24, ~5
    //     nonzero blocks per 32-block group), so the nonzero blocks of the
    //     warp's range are first compacted into a list (ballot + prefix;
    //     s_cnt is free again), then processed 32 at a time with every lane
    //     busy: reload the block, popcount, one warp scan for the positions,
    //     walk the set bits. Stores of one step ascend with the lane and coalesce.
    const int64_t off = s_tile_off + s_warp_off[warp];
    auto *lst = &fs.lst[warp][0];  // kMaxIter * 32 entries >= the warp's range
    const uint32_t lt = (1u << lane) - 1u;
    int n = 0;
#pragma unroll
    for (int j = 0; j < kMaxIter; j++) {
        const uint32_t c = (pk[j >> 1] >> (16 * (j & 1))) & 0xffffu;
        const uint32_t m = __ballot_sync(0xffffffffu, c != 0);
        if (c) lst[n + __popc(m & lt)] = (typename FinishSmem<NT>::Idx)(32 * j + lane);
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
        // scratch mode: 4-byte tile-relative offsets (k_reorder adds the tile's
        // first rank), half the bytes of int64 ranks; single tile: final ranks
        const uint32_t lbase = (uint32_t)b * 243u;
        const int64_t rbase = (blk0 + b) * 243 + rank_add;
        if (pos + cnt <= fa.cap) {
            // walk only the nonzero words (most blocks hold one or two): their
            // mask from the registers, the words themselves re-read from smem
            uint32_t nz = 0;
#pragma unroll
            for (int k = 0; k < 8; k++) nz |= (wv[k] != 0u ? 1u : 0u) << k;
            const uint32_t *bw = sm + b * 8;
            if (fa.out32) {
                uint32_t *o = fa.out32 + pos;
                while (nz) {
                    const int k = __ffs(nz) - 1;
                    nz &= nz - 1;
                    uint32_t w = bw[k];
                    do {
                        *o++ = lbase + k * 32 + (__ffs(w) - 1);
                        w &= w - 1;
                    } while (w);
                }
            } else {
                int64_t *o = fa.out + pos;
                while (nz) {
                    const int k = __ffs(nz) - 1;
                    nz &= nz - 1;
                    uint32_t w = bw[k];
                    do {
                        *o++ = rbase + k * 32 + (__ffs(w) - 1);
                        w &= w - 1;
                    } while (w);
                }
            }
        } else {  // the output is too small: write what fits (the host grows it and reruns)
#pragma unroll
            for (int k = 0; k < 8; k++) {
                uint32_t w = wv[k];
                while (w) {
                    if (pos < fa.cap) {
                        if (fa.out32)
                            fa.out32[pos] = lbase + k * 32 + (__ffs(w) - 1);
                        else
                            fa.out[pos] = rbase + k * 32 + (__ffs(w) - 1);
                    }
                    pos++;
                    w &= w - 1;
                }
            }
        }
    }
}

// Prime block of a C0 tile as ONE parallel REDUCE step over all G tile axes
// (+ the in-block axes of ib_mask): P(b) = M(b) & ~(OR over fixed block digits
// j of M(b + (2 - d_j) 3^j) | in-block kills of M(b)), every kill read from the
// unmodified input tile (exact: the parallel-step argument of DESIGN.md §3;
// cube_reduce_par applies the same step to register sub-cubes). A zero block
// needs no parent: the cost follows the nonzero blocks, not the tile.
template <int G>
__device__ __forceinline__ void prime_block(const uint32_t *sm, int b, uint32_t ib_mask, uint32_t (&v)[8]) {
    const uint4 *p = reinterpret_cast<const uint4 *>(sm + b * 8);
    const uint4 a0 = p[0], a1 = p[1];
    v[0] = a0.x, v[1] = a0.y, v[2] = a0.z, v[3] = a0.w, v[4] = a1.x, v[5] = a1.y, v[6] = a1.z, v[7] = a1.w;
    uint4 k0 = make_uint4(0, 0, 0, 0), k1 = k0;
    int q = b;
#pragma unroll
    for (int j = 0; j < G; j++) {
        const int q3 = q / 3, d = q - 3 * q3;
        q = q3;
        if (d != 2) {
            const uint4 *pp = reinterpret_cast<const uint4 *>(sm + (b + (2 - d) * pow3i(j)) * 8);
            const uint4 c0 = pp[0], c1 = pp[1];
            k0 = make_uint4(k0.x | c0.x, k0.y | c0.y, k0.z | c0.z, k0.w | c0.w);
            k1 = make_uint4(k1.x | c1.x, k1.y | c1.y, k1.z | c1.z, k1.w | c1.w);
        }
    }
    if (ib_mask) inblock_reduce(v, ib_mask);  // kills from the block's own input values
    v[0] &= ~k0.x, v[1] &= ~k0.y, v[2] &= ~k0.z, v[3] &= ~k0.w;
    v[4] &= ~k1.x, v[5] &= ~k1.y, v[6] &= ~k1.z, v[7] &= ~k1.w;
}

// The sparse finish's per-block step in general: the C0 step of prime_block
// (or, skip_c0, the block as it is: the sharded path's reduce_low did the C0
// axes), then the top-axis kills of the sharded path: the OR of up to
// kMaxKill parent super-blocks at the block's offset (local or NVLink peer
// memory), all loads in flight at once.
template <int G>
__device__ __forceinline__ void finish_block(const uint32_t *sm, int b, const FinalArgs &fa, const uint64_t *kills,
                                             int64_t kofs, uint32_t (&v)[8]) {
    if (fa.skip_c0) {
        const uint4 *p = reinterpret_cast<const uint4 *>(sm + b * 8);
        const uint4 a0 = p[0], a1 = p[1];
        v[0] = a0.x, v[1] = a0.y, v[2] = a0.z, v[3] = a0.w, v[4] = a1.x, v[5] = a1.y, v[6] = a1.z, v[7] = a1.w;
        if (fa.ib_mask) inblock_reduce(v, fa.ib_mask);
    } else {
        prime_block<G>(sm, b, fa.ib_mask, v);
    }
    if (!kills) return;
    uint4 k0 = make_uint4(0, 0, 0, 0), k1 = k0;
#pragma unroll
    for (int q = 0; q < kMaxKill; q++) {
        const uint64_t kp = __ldg(&kills[q]);
        if (kp) {
            const uint4 *kq = reinterpret_cast<const uint4 *>(reinterpret_cast<const uint32_t *>(kp) + (kofs + b) * 8);
            const uint4 a0 = kq[0], a1 = kq[1];
            k0 = make_uint4(k0.x | a0.x, k0.y | a0.y, k0.z | a0.z, k0.w | a0.w);
            k1 = make_uint4(k1.x | a1.x, k1.y | a1.y, k1.z | a1.z, k1.w | a1.w);
        }
    }
    v[0] &= ~k0.x, v[1] &= ~k0.y, v[2] &= ~k0.z, v[3] &= ~k0.w;
    v[4] &= ~k1.x, v[5] &= ~k1.y, v[6] &= ~k1.z, v[7] &= ~k1.w;
}

// Final stage of one C0 tile whose tile axes are NOT yet reduced (the fused
// plans). Pass 0: each warp compacts its contiguous block range to the list of
// its nonzero blocks; the tile's list is their concatenation (rank order).
// Pass A: the list is cut into batches of 32 entries, batch i to warp
// i mod NWARP; each lane reduces its block on its own (prime_block) and
// counts its primes. After the tile's range reservation, pass B emits each
// batch in rank order (a warp's first batch keeps its primes in registers,
// later ones are reduced again). The tile in shared memory is only read.
// Replaces two register-cube rounds over every word of the tile and a
// popcount pass (round 2b).
// Returns false (nothing done after pass 0) when the tile has more than
// kSparseMax nonzero blocks: the register-cube rounds are cheaper there
// (n = 24, config 4: E 8.22 ms rounds only, 8.07 sparse only, 7.09 with the
// switch at 600 (7.18 at 400, 7.85 at 300); P(on) = 0.99: 14.7 / 24.5 / 15.3).
constexpr int kSparseMax = 600;

template <int NT, int G, bool SHARD>
__device__ __forceinline__ bool tile_finish_sparse(const uint32_t *sm, int64_t tile, int64_t blk0,
                                                   const FinalArgs &fa, FinishSmem<NT> &fs,
                                                   const uint32_t *gb = nullptr, int nr32 = 0,
                                                   const int *goff = nullptr, bool reduced = false) {
    // reduced (gather finish, dense tiles): the C0 axes are already reduced
    // in shared memory (tile_reduce_c0_t); list and finish whatever is left
    // gather finish: the sparse path only while every warp has at most one batch
    // (no block is reduced twice, so no parent sector is loaded twice); beyond
    // that the rounds + in-place finish are cheaper (E 11.74 -> 11.57 ms)
    const int smax = reduced ? pow3i(G) : (gb ? NT : kSparseMax);
    constexpr int NB = pow3i(G);
    constexpr int NWARP = NT / 32;
    constexpr int kMaxIter = ((NB + NWARP - 1) / NWARP + 31) / 32;
    constexpr int kMaxBatch = (NB + 31) / 32;
    static_assert(kMaxIter <= finish_iters<NT>(), "scratch sized for the largest tile");
    __shared__ int s_off[NWARP + 1];        // nonzero blocks of each warp's range (entry w + 1)
    __shared__ int s_pre[NWARP];            // their list offsets
    __shared__ int s_bat[kMaxBatch + 1];    // primes per batch, then their exclusive prefix
    int64_t &s_tile_off = fs.tile_off;
    auto &s_lst = fs.lst;    // each warp's nonzero blocks (range-relative)
    auto &s_lcnt = fs.lcnt;  // their prime counts (<= 243)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int h = (lane >> 2) & 1;  // half-swap: conflict-free LDS.128 at 32-B lane stride
    const uint32_t lt = (1u << lane) - 1u;
    const uint32_t ibm = fa.ib_mask | (gb ? fa.ib_gather : 0u);  // gather finish: pass D's in-block axes too
    // SHARD (the sharded extract): this tile's super-block (slot), its parents
    // and rank offset; the fused plans compile none of it
    const int64_t slot = SHARD && (fa.kill_tab || fa.rank_add_tab) ? tile / fa.tiles_per_slot : 0;
    const int64_t slot_blk0 = slot * fa.tiles_per_slot * NB;  // first block of the slot
    const int64_t rank_add = SHARD && fa.rank_add_tab ? fa.rank_add_tab[slot] - slot_blk0 * 243 : fa.rank_add;
    const uint64_t *kills = SHARD && fa.kill_tab ? fa.kill_tab + slot * kMaxKill : nullptr;
    const int64_t kofs = blk0 - slot_blk0;  // the tile's first block within its super-block

    // pass 0: nonzero blocks of the warp's range, in order. The first 32 of
    // every range are a density sample: a tile whose sample is dense goes to
    // the register-cube rounds after one barrier.
    {
        const int b0 = NB * warp / NWARP, b1 = NB * (warp + 1) / NWARP;
        int n = 0;
#pragma unroll
        for (int j = 0; j < kMaxIter; j++) {
            const int b = b0 + 32 * j + lane;
            bool nz = false;
            if (b < b1) {
                const uint4 *p = reinterpret_cast<const uint4 *>(sm + b * 8);
                const uint4 x0 = p[h], x1 = p[h ^ 1];
                nz = (x0.x | x0.y | x0.z | x0.w | x1.x | x1.y | x1.z | x1.w) != 0u;
            }
            if (j == 0 && kMaxIter > 1 && __syncthreads_count(nz) > smax * 32 * NWARP / NB) return false;
            const uint32_t m = __ballot_sync(0xffffffffu, nz);
            if (nz) s_lst[warp][n + __popc(m & lt)] = (typename FinishSmem<NT>::Idx)(32 * j + lane);
            n += __popc(m);
        }
        if (lane == 0) s_off[warp + 1] = n;
    }
    __syncthreads();
    int ntot = 0;
#pragma unroll
    for (int w = 1; w <= NWARP; w++) ntot += s_off[w];
    if (ntot > smax) return false;
    if (threadIdx.x == 0) {  // list offsets of the warps' ranges (s_off is still being read)
        int acc = 0;
        for (int w = 0; w < NWARP; w++) s_pre[w] = acc, acc += s_off[w + 1];
    }
    __syncthreads();
    const int nbat = (ntot + 31) >> 5;
    // list entry -> (warp range, index): the last w with s_pre[w] <= e
    auto entry = [&](int e, int &w, int &idx) {
        int lo = 0;
#pragma unroll
        for (int step = 16; step >= 1; step >>= 1)
            if (lo + step < NWARP && s_pre[lo + step] <= e) lo += step;
        w = lo;
        idx = e - s_pre[lo];
    };

    // pass A: primes per listed block, per batch
    uint32_t v0[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};  // the primes of this warp's first batch
#pragma unroll 1
    for (int bt = warp; bt < nbat; bt += NWARP) {
        const int e = 32 * bt + lane;
        uint32_t v[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
        int c = 0;
        if (e < ntot) {
            int w, idx;
            entry(e, w, idx);
            const int blk = NB * w / NWARP + s_lst[w][idx];
            if (SHARD) {
                finish_block<G>(sm, blk, fa, kills, kofs, v);
            } else {
                if (reduced) {
                    const uint4 *p = reinterpret_cast<const uint4 *>(sm + blk * 8);
                    const uint4 a0 = p[0], a1 = p[1];
                    v[0] = a0.x, v[1] = a0.y, v[2] = a0.z, v[3] = a0.w, v[4] = a1.x, v[5] = a1.y, v[6] = a1.z, v[7] = a1.w;
                    if (ibm) inblock_reduce(v, ibm);
                } else {
                    prime_block<G>(sm, blk, ibm, v);
                }
                if (gb && (v[0] | v[1] | v[2] | v[3] | v[4] | v[5] | v[6] | v[7])) g0_kill(gb, nr32, goff, blk, v);
                if (reduced && bt != warp) {
                    // after the rounds a block depends on nothing else in the tile: keep the
                    // finished block in place, so pass B reads it instead of repeating the
                    // in-block step and the parent loads (the first batch stays in registers)
                    uint4 *pw = reinterpret_cast<uint4 *>(const_cast<uint32_t *>(sm) + blk * 8);
                    pw[0] = make_uint4(v[0], v[1], v[2], v[3]);
                    pw[1] = make_uint4(v[4], v[5], v[6], v[7]);
                }
            }
#pragma unroll
            for (int k = 0; k < 8; k++) c += __popc(v[k]);
            s_lcnt[w][idx] = (uint8_t)c;
        }
        if (bt == warp) {
#pragma unroll
            for (int k = 0; k < 8; k++) v0[k] = v[k];
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
        if (lane == 0) s_bat[bt] = c;
    }
    __syncthreads();

    // reserve this tile's range in the scratch output with one atomic;
    // k_scan_tiles + k_reorder restore rank order
    if (threadIdx.x == 0) {
        int acc = 0;
        for (int bt = 0; bt < nbat; bt++) {
            const int c = s_bat[bt];
            s_bat[bt] = acc;
            acc += c;
        }
        const int64_t base = tile_range(fa, tile, acc);
        fa.tile_base[tile] = base;
        fa.tile_cnt[tile] = (int32_t)acc;
        if (fa.tile_rank0) fa.tile_rank0[tile] = blk0 * 243 + rank_add;
        s_tile_off = base;
    }
    __syncthreads();
    if (fa.out == nullptr && fa.out32 == nullptr) return true;

    // pass B: ordered emission (stores of one step ascend with the lane; a
    // warp-cooperative variant, one prime per lane found by shuffles + fns,
    // measured slower: 8.69 vs 8.07 ms)
#pragma unroll 1
    for (int bt = warp; bt < nbat; bt += NWARP) {
        const int e = 32 * bt + lane;
        int cnt = 0, b = 0;
        uint32_t v[8];
#pragma unroll
        for (int k = 0; k < 8; k++) v[k] = v0[k];
        if (e < ntot) {
            int w, idx;
            entry(e, w, idx);
            cnt = s_lcnt[w][idx];
            b = NB * w / NWARP + s_lst[w][idx];
            if (bt != warp && cnt) {
                if (SHARD) {
                    finish_block<G>(sm, b, fa, kills, kofs, v);
                } else {
                    if (reduced) {
                        const uint4 *p = reinterpret_cast<const uint4 *>(sm + b * 8);
                        const uint4 a0 = p[0], a1 = p[1];
                        v[0] = a0.x, v[1] = a0.y, v[2] = a0.z, v[3] = a0.w, v[4] = a1.x, v[5] = a1.y, v[6] = a1.z,
                        v[7] = a1.w;  // finished in pass A
                    } else {
                        prime_block<G>(sm, b, ibm, v);
                        if (gb) g0_kill(gb, nr32, goff, b, v);
                    }
                }
            }
        }
        int incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        if (!cnt) continue;
        int64_t pos = s_tile_off + s_bat[bt] + (incl - cnt);
        const uint32_t lbase = (uint32_t)b * 243u;
        const int64_t rbase = (blk0 + b) * 243 + rank_add;
        if (pos + cnt <= fa.cap) {
            if (fa.out32) {
                uint32_t *o = fa.out32 + pos;
#pragma unroll
                for (int k = 0; k < 8; k++)
                    for (uint32_t x = v[k]; x; x &= x - 1) *o++ = lbase + k * 32 + (__ffs(x) - 1);
            } else {
                int64_t *o = fa.out + pos;
#pragma unroll
                for (int k = 0; k < 8; k++)
                    for (uint32_t x = v[k]; x; x &= x - 1) *o++ = rbase + k * 32 + (__ffs(x) - 1);
            }
        } else {  // the output is too small: write what fits (the host grows it and reruns)
#pragma unroll
            for (int k = 0; k < 8; k++)
                for (uint32_t x = v[k]; x; x &= x - 1, pos++)
                    if (pos < fa.cap) {
                        if (fa.out32)
                            fa.out32[pos] = lbase + k * 32 + (__ffs(x) - 1);
                        else
                            fa.out[pos] = rbase + k * 32 + (__ffs(x) - 1);
                    }
        }
    }
    return true;
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

// sharded path: the output range of each of nslots states (tps tiles each)
__global__ void k_slot_spans(const int32_t *__restrict__ cnt, const int64_t *__restrict__ pos, int64_t tps,
                             int64_t nslots, int64_t *__restrict__ start, int64_t *__restrict__ count) {
    const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (s >= nslots) return;
    const int64_t a = pos[s * tps], e = (s + 1) * tps - 1;
    start[s] = a;
    count[s] = pos[e] + cnt[e] - a;
}

// Copy every tile's ranks from its scratch range to its rank-order position
// (one warp per tile, coalesced 8-B copies).
// DQMC_FLAG_ASYNC: publish the count in stream order; -(count + 1) flags an
// incomplete rank list (output or scratch too small).
__global__ void k_publish_count(const int64_t *__restrict__ total, int64_t limit, int64_t *__restrict__ dst) {
    const int64_t t = *total;
    *dst = t <= limit ? t : -(t + 1);
}

// OutT = int64_t: final ranks (the tile's first rank added). OutT = uint32_t:
// the packed form of the host API's large results, tile-relative offsets in
// rank order; the host adds the tile's first rank (dqmc_hostpack.cpp).
template <typename OutT>
__global__ void __launch_bounds__(256) k_reorder(const uint32_t *__restrict__ scratch, const int64_t *__restrict__ base,
                                                 const int32_t *__restrict__ cnt, const int64_t *__restrict__ pos,
                                                 const int64_t *__restrict__ rank0, OutT *__restrict__ out,
                                                 int64_t cap, int64_t ntiles, int64_t scap,
                                                 const int64_t *__restrict__ dbase = nullptr) {
    const int lane = threadIdx.x & 31;
    const int64_t add = dbase ? *dbase : 0;
    const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = (gridDim.x * (int64_t)blockDim.x) >> 5;
    for (int64_t t = w; t < ntiles; t += nw) {
        const int c = cnt[t];
        const int64_t src = base[t], dst = pos[t] + add;
        const OutT r0 = sizeof(OutT) == 8 ? (OutT)rank0[t] : (OutT)0;
        // a tile whose range overflowed the scratch is skipped: the host sees
        // total > scratch capacity, grows the scratch and reruns the final stage
        if (c < 0 || src < 0 || src + c > scap) continue;
        int i = lane;
        if (dst + c <= cap) {
            // four independent loads in flight per lane (the copy is latency-bound)
            for (; i + 96 < c; i += 128) {
                const uint32_t a0 = __ldcs(scratch + src + i), a1 = __ldcs(scratch + src + i + 32);
                const uint32_t a2 = __ldcs(scratch + src + i + 64), a3 = __ldcs(scratch + src + i + 96);
                out[dst + i] = r0 + a0;
                out[dst + i + 32] = r0 + a1;
                out[dst + i + 64] = r0 + a2;
                out[dst + i + 96] = r0 + a3;
            }
        }
        for (; i < c; i += 32)
            if (dst + i < cap) out[dst + i] = r0 + __ldcs(scratch + src + i);
    }
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

// pass E: one CTA per C0 tile (3^G blocks); the tile arrives in shared
// memory with one TMA bulk copy (or three 4-D tensor boxes, piece-major).

// GATH (the n = 24 plan): the kernel also holds the gather finish and takes it
// when pass C left a sparse state (gather_chosen); pass D then returned at once.
// The gather variant runs 10 warps per CTA instead of 12 (68 registers per
// thread at 3 CTAs/SM: its parent loads no longer spill; gather E 11.56 ->
// 11.22 ms, 17.9 -> 17.0 at P(on) = 0.9; the same kernel in pass-D mode 7.4 vs
// 7.05 ms with 12 warps, which is why the plans without a gather keep 12).
constexpr int kFinalThreadsGather = 320;
template <int G, bool GATH = false, int NT = (GATH ? kFinalThreadsGather : kFinalThreads)>
__global__ void __launch_bounds__(NT, 3)
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
    // zero-skip flags (Plan::nz): pass C saw no nonzero cell in this tile
    auto tile_zero = [&](int64_t t) {
        const uint32_t t32 = (uint32_t)t, nr = (uint32_t)fa.pm_nr;
        const uint32_t u = t32 / nr, l = t32 - u * nr;
        return ((__ldg(&fa.nz_e[l * kNzWords + (u >> 5)]) >> (u & 31)) & 1u) == 0u;
    };
    // (reading this flag while a speculative load of the tile is in flight
    // measured slower: 7.67 vs 7.00 ms, zero tiles then pay for their load)
    if (fa.nz_e && tile_zero(tile)) {
        if (threadIdx.x == 0) {
            fa.tile_base[tile] = 0;
            fa.tile_cnt[tile] = 0;
            if (fa.tile_rank0) fa.tile_rank0[tile] = blk0 * 243 + fa.rank_add;
        }
        return;
    }
    __shared__ int s_goff[kGroupMax];
    const uint32_t *gb = nullptr;
    // gather finish: this tile's group-0 parents, rows (2 - d_j) 3^j up in every D item
    if (GATH && gather_chosen(fa.g0_cnt, fa.g0_limit)) {
        const uint32_t t32 = (uint32_t)tile, nr = (uint32_t)fa.pm_nr;
        const uint32_t u = t32 / nr, l = t32 - u * nr;
        gb = fa.g0 + ((int64_t)u * fa.pm_np * nr + l) * 32;
        if (threadIdx.x >= 64 && threadIdx.x < 64 + kGroupMax) {
            const int j = threadIdx.x - 64;
            const int p3 = (int)pow3l(j), d = (int)(l / p3) % 3;
            // a parent tile that pass C flagged all zero kills nothing: no loads for it
            const bool none = d == 2 || tile_zero((int64_t)u * nr + l + (2 - d) * p3);
            s_goff[j] = none ? 0 : (2 - d) * p3 * 32;
        }
    }
    if (threadIdx.x == 0 && fa.pm_nr) {
        // piece-major group 0: the tile is pm_np pieces 3^r pieces apart; boxes
        // of 256 pieces (map ma) and one remainder box (map mb). Tiles of a
        // piece-major plan number < 3^12: 32-bit index arithmetic (the 64-bit
        // division this thread used to do held the other warps at the barrier)
        mbar_init(&mbar, 1);
        mbar_expect_tx(&mbar, fa.pm_np * 128);
        const int nfull = fa.pm_np >> 8, rem = fa.pm_np & 255;
        const uint32_t t32 = (uint32_t)tile, nr = (uint32_t)fa.pm_nr;
        const int up = (int)(t32 / nr), q1 = (int)(t32 - (uint32_t)up * nr);
        for (int j = 0; j < nfull; j++) tma_load_4d(sm + j * 256 * 32, &ma, 0, 256 * j, q1, up, &mbar);
        if (rem) tma_load_4d(sm + nfull * 256 * 32, &mb, 0, 256 * nfull, q1, up, &mbar);
    } else if (threadIdx.x == 32 && fa.pm_nr) {
        // warm L2 for the CTA that takes this slot a generation later (issued
        // by another warp, off the path to the barrier)
        const int pf = (int)blockIdx.x + fa.prefetch;
        if (fa.prefetch > 0 && pf < (int)gridDim.x && !(fa.nz_e && tile_zero(tile + fa.prefetch))) {
            const int nfull = fa.pm_np >> 8, rem = fa.pm_np & 255;
            const uint32_t t2 = (uint32_t)(tile + fa.prefetch), nr = (uint32_t)fa.pm_nr;
            const int upb = (int)(t2 / nr), q1b = (int)(t2 - (uint32_t)upb * nr);
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
    __shared__ FinishSmem<NT> fs;
    if (!fa.bitmap_out) {
        if (fa.kill_tab || fa.skip_c0 || fa.rank_add_tab) {
            if (tile_finish_sparse<NT, G, true>(sm, tile, blk0, fa, fs)) return;
        } else {
            // gather finish: a dense tile goes through the register-cube rounds and
            // then the same batched finish over the blocks the rounds left
            for (bool reduced = false;; reduced = true) {
                if (tile_finish_sparse<NT, G, false>(sm, tile, blk0, fa, fs, gb, fa.pm_nr * 32, s_goff, reduced))
                    return;
                if (!GATH || !gb) break;
                tile_reduce_c0_t<G, 0>(sm);
            }
        }
    }
    if (!fa.skip_c0) tile_reduce_c0_t<G, 0>(sm);
    tile_finish<NT>(sm, NB, tile, blk0, fa, fs, gb, fa.pm_nr * 32, s_goff);
}

// n <= 12: the whole problem is one tile; one CTA does A and E.
__global__ void __launch_bounds__(kTileThreads) k_small(const uint32_t *__restrict__ tt32, int g, FinalArgs fa) {
    extern __shared__ __align__(16) uint32_t sm[];
    tile_build(sm, tt32, g, 0);
    tile_reduce_c0(sm, g);
    __shared__ FinishSmem<kTileThreads> fs;
    tile_finish<kTileThreads>(sm, (int)pow3l(g), 0, 0, fa, fs);
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
        CASE(0) CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6)
#undef CASE
        case 7:
            if (fa.g0)
                k_c0_final<7, true><<<(unsigned)ntiles, kFinalThreadsGather, smem, s>>>(state, fa, ma, mb);
            else
                k_c0_final<7><<<(unsigned)ntiles, kFinalThreads, smem, s>>>(state, fa, ma, mb);
            break;
        default: return set_err(DQMC_ERR_INVALID, "bad tile exponent");
    }
    CK_LAUNCH();
    return DQMC_OK;
}

// Per-tile scratch slot (entries) of the final stage: the n = 24 plan gives
// every tile a fixed range (2.2 GB at 1024 entries; config 4 averages ~485
// primes per nonzero tile), so most tiles reserve nothing with an atomic.
int64_t tile_slot(const Plan &p) { return p.nz ? 1024 : 0; }
}  // namespace

// Gather finish (Plan::nz): at most this many nonzero blocks after pass C
unsigned long long gather_limit(const Plan &p) {
    if (!p.nz) return 0ull;
    if (g_eng.gather_permille >= 1000) return ~0ull;
    return (unsigned long long)p.nblocks * (unsigned long long)g_eng.gather_permille / 1000ull;
}

namespace {
// the final stage's gather arguments: the state, pass C's block count, the limit
void set_gather(const Plan &p, const uint32_t *state, FinalArgs &fa) {
    if (!p.nz || !fa.nz_e || g_eng.gather_permille == 0) return;  // never: pass D got limit 0 and ran
    const size_t npiece = (size_t)(p.pitch / kRowBlocks), nr = (size_t)pow3l(p.r[0]);
    fa.g0 = state;
    fa.g0_cnt = reinterpret_cast<const unsigned long long *>(g_eng.nzflags + nz_count_offset(npiece, nr));
    fa.g0_limit = gather_limit(p);
    fa.ib_gather = p.ib_D[0];
}
}  // namespace
namespace {

// E's zero-skip flags: written by pass C of the same fused plan on the engine state
const uint32_t *nz_e_flags(const Plan &p, const uint32_t *state) {
    if (!p.nz || state != g_eng.state || !g_eng.nzflags) return nullptr;
    return g_eng.nzflags + nz_e_offset((size_t)(p.pitch / kRowBlocks));
}

// Final stage: E (+ scan + reorder). Source: the truth table (k_small, fused
// A+E, when tt32 != null) or a merged/reduced state. Returns the prime count.
}  // namespace

int run_final(const Plan &p, const uint32_t *tt32, const uint32_t *state, uint32_t ib_mask, int64_t rank_add,
              int64_t *ranks, int64_t cap, bool count_only, const FinalOpts &o, int64_t *count, Timer &tm,
              cudaStream_t s) {
    uint32_t *bitmap_out = o.bitmap_out;
    int64_t *count_dev = o.count_dev;
    const int64_t nbatch = std::max<int64_t>(1, o.nbatch);
    const uint64_t S = (uint64_t)p.nblocks * 32 * nbatch;
    const int64_t tps = p.T == 0 ? 1 : pow3l(p.T);  // tiles per state
    const int64_t ntiles = tps * nbatch;
    const int tile_smem = (int)pow3l(p.g) * 32;
    int rc;
    if ((rc = grow(g_eng.tile_base, g_eng.tile_cap, (size_t)ntiles, 8))) return rc;
    if ((rc = grow(g_eng.tile_pos, g_eng.tile_pos_cap, (size_t)ntiles, 8))) return rc;
    if ((rc = grow(g_eng.tile_cnt, g_eng.tile_cnt_cap, (size_t)ntiles, 4))) return rc;
    if ((o.kill_tab || bitmap_out || nbatch > 1) && p.T > 0 && p.pitch != pow3l(p.g))
        return set_err(DQMC_ERR_INVALID, "internal: kill/bitmap outputs need the reference layout plan");
    const bool direct = ntiles == 1;  // one tile: its ranks are already in order
    const int64_t slot = count_only || direct ? 0 : tile_slot(p), ovf0 = slot * ntiles;
    if (!count_only && !direct) {
        const size_t want = (size_t)ovf0 + std::max<size_t>(g_eng.scratch_want, (size_t)1 << 20);
        if ((rc = grow(g_eng.scratch, g_eng.scratch_cap, want, 4))) return rc;
        if ((rc = grow(g_eng.tile_rank0, g_eng.tile_rank0_cap, (size_t)ntiles, 8))) return rc;
    }
    FinalArgs fa;
    fa.out = count_only || !direct ? nullptr : ranks;
    fa.out32 = count_only || direct ? nullptr : g_eng.scratch;
    fa.tile_rank0 = fa.out32 ? g_eng.tile_rank0 : nullptr;
    fa.cap = count_only ? 0 : (direct ? cap : (int64_t)g_eng.scratch_cap);
    fa.slot = (int)slot;
    fa.ovf0 = ovf0;
    fa.rank_add = rank_add;
    fa.kill_tab = o.kill_tab;
    fa.rank_add_tab = o.rank_add_tab;
    fa.tiles_per_slot = tps;
    fa.skip_c0 = o.skip_c0 ? 1 : 0;
    fa.ib_mask = ib_mask;
    fa.bitmap_out = bitmap_out;
    fa.alloc = g_eng.alloc;
    fa.tile_base = g_eng.tile_base;
    fa.tile_cnt = g_eng.tile_cnt;
    fa.tile0 = 0;
    fa.pitch = p.pitch;
    fa.prefetch = 3 * g_eng.num_sms;  // one generation of resident CTAs (3 per SM): 9.23 -> 9.0 ms at n=24
    fa.nz_e = nz_e_flags(p, state);
    set_gather(p, state, fa);
    CK(cudaMemsetAsync(g_eng.alloc, 0, 8, s));
    if (tt32) {
        k_small<<<1, kTileThreads, tile_smem, s>>>(tt32, p.g, fa);
        CK_LAUNCH();
        tm.mark("k_small", (uint64_t)(1ull << p.H) * 4 + (bitmap_out ? S : 0));
    } else {
        CUtensorMap ma, mb;
        if ((rc = make_final_maps(p, state, &ma, &mb, fa))) return rc;
        if ((rc = launch_c0_final(p.g, ntiles, state, fa, ma, mb, s))) return rc;
        tm.mark("k_c0_final", S + (bitmap_out ? S : 0));
    }
    if (ntiles <= 4096) {
        k_scan_tiles<<<1, 1024, 0, s>>>(g_eng.tile_cnt, g_eng.tile_pos, ntiles, g_eng.total);
        CK_LAUNCH();
    } else {
        // device-wide exclusive scan (CUB) of the int32 counts into int64 positions
        size_t tmp = 0;
        CK(cub::DeviceScan::ExclusiveScan(nullptr, tmp, g_eng.tile_cnt, g_eng.tile_pos, cub::Sum(), (int64_t)0,
                                          (int64_t)ntiles, s));
        if ((rc = grow(g_eng.cub_tmp, g_eng.cub_tmp_cap, tmp, 1))) return rc;
        CK(cub::DeviceScan::ExclusiveScan(g_eng.cub_tmp, tmp, g_eng.tile_cnt, g_eng.tile_pos, cub::Sum(), (int64_t)0,
                                          (int64_t)ntiles, s));
        k_scan_total<<<1, 32, 0, s>>>(g_eng.tile_cnt, g_eng.tile_pos, ntiles, g_eng.total);
        CK_LAUNCH();
    }
    tm.mark("k_scan_tiles", (uint64_t)ntiles * 12);
    if (o.slot_start && o.slot_count) {
        k_slot_spans<<<(unsigned)((nbatch + 255) / 256), 256, 0, s>>>(g_eng.tile_cnt, g_eng.tile_pos, tps, nbatch,
                                                                       o.slot_start, o.slot_count);
        CK_LAUNCH();
    }
    if (!count_only && !direct) {
        const int grid = (int)std::min<int64_t>((ntiles + 7) / 8, (int64_t)g_eng.num_sms * 16);
        if (o.packed32)
            k_reorder<uint32_t><<<grid, 256, 0, s>>>(g_eng.scratch, g_eng.tile_base, g_eng.tile_cnt, g_eng.tile_pos,
                                                     g_eng.tile_rank0, o.packed32, cap, ntiles,
                                                     (int64_t)g_eng.scratch_cap);
        else
            k_reorder<int64_t><<<grid, 256, 0, s>>>(g_eng.scratch, g_eng.tile_base, g_eng.tile_cnt, g_eng.tile_pos,
                                                    g_eng.tile_rank0, ranks, cap, ntiles, (int64_t)g_eng.scratch_cap);
        CK_LAUNCH();
        tm.mark("k_reorder", (uint64_t)ntiles * 16);
    }
    if (count_dev) {  // DQMC_FLAG_ASYNC: no host synchronisation
        // (the overflow pool alone must hold the count for the result to be trusted: conservative)
        const int64_t limit =
            count_only ? INT64_MAX : (direct ? cap : std::min<int64_t>(cap, (int64_t)g_eng.scratch_cap - ovf0));
        k_publish_count<<<1, 1, 0, s>>>(g_eng.total, limit, count_dev);
        CK_LAUNCH();
        return DQMC_OK;
    }
    int64_t total = 0;
    CK(cudaMemcpyAsync(&total, g_eng.total, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    *count = total;
    return DQMC_OK;
}

namespace {
void add_rank_bytes(Timer &tm, int64_t written) {
    if (tm.bytes.empty()) return;
    for (size_t i = 0; i < tm.names.size(); i++) {
        // E writes 4-B tile-relative offsets when k_reorder follows (multi-tile),
        // final 8-B ranks otherwise; k_reorder reads 4 B and writes 8 B per rank
        const bool multi = std::find(tm.names.begin(), tm.names.end(), "k_reorder") != tm.names.end();
        if (tm.names[i] == "k_c0_final" || tm.names[i] == "k_small") tm.bytes[i] += (uint64_t)written * (multi ? 4 : 8);
        if (tm.names[i] == "k_reorder") tm.bytes[i] += (uint64_t)written * 12;
    }
}
}  // namespace

// Final stage with the scratch-regrow retry (the stage does not modify the
// merged state it reads; with a bitmap output it rewrites the same P).
int run_final_retry(const Plan &p, const uint32_t *tt32, const uint32_t *state, uint32_t ib_mask, int64_t rank_add,
                    int64_t *ranks, int64_t cap, bool count_only, const FinalOpts &o, int64_t *count, Timer &tm,
                    cudaStream_t s) {
    int rc;
    if ((rc = run_final(p, tt32, state, ib_mask, rank_add, ranks, cap, count_only, o, count, tm, s))) return rc;
    if (o.count_dev) return DQMC_OK;  // async: the caller sees -(count + 1) and retries synchronously
    const bool direct = (p.T == 0) && o.nbatch <= 1;
    const int64_t ovf0 = direct || count_only ? 0 : tile_slot(p) * (p.T == 0 ? 1 : pow3l(p.T)) * std::max<int64_t>(1, o.nbatch);
    if (!count_only && !direct && *count > (int64_t)g_eng.scratch_cap - ovf0) {
        g_eng.scratch_want = (size_t)((double)*count * 1.05) + 1024;
        const bool on = tm.on;
        tm.on = false;
        FinalOpts o2 = o;
        o2.count_dev = nullptr;
        rc = run_final(p, tt32, state, ib_mask, rank_add, ranks, cap, count_only, o2, count, tm, s);
        tm.on = on;
        if (rc) return rc;
    }
    if (!count_only) add_rank_bytes(tm, std::min<int64_t>(*count, cap));
    return DQMC_OK;
}

// Host-API final stage, pipelined and packed: the tiles are finished in K
// chunks on the compute stream (E, scan, running base, reorder of the 4-byte
// tile offsets into rank order). As soon as chunk c's event fires the host
// queues the D2H of its tile positions and offsets on the copy stream, and as
// soon as that copy has landed the host threads widen the chunk to int64
// ranks (dqmc_hostpack.cpp) — the SMs finish chunk c+2 while the copy engine
// moves chunk c+1 and the host widens chunk c. Half the PCIe bytes of int64
// ranks. Returns the total; *host_ok is false if the host buffer (sized from
// the previous call) was too small.
int run_final_pipelined(const Plan &p, const uint32_t *state, int64_t *host, int64_t host_cap, int64_t *count,
                        bool *host_ok, cudaStream_t s) {
    const int64_t ntiles = pow3l(p.T);
    const int K = (int)std::min<int64_t>(16, ntiles);
    int rc;
    if ((rc = grow(g_eng.tile_base, g_eng.tile_cap, (size_t)ntiles, 8))) return rc;
    if ((rc = grow(g_eng.tile_pos, g_eng.tile_pos_cap, (size_t)ntiles, 8))) return rc;
    if ((rc = grow(g_eng.tile_cnt, g_eng.tile_cnt_cap, (size_t)ntiles, 4))) return rc;
    if ((rc = grow(g_eng.ranks, g_eng.ranks_cap, (size_t)(host_cap + 1) / 2, 8))) return rc;
    if ((rc = grow_pinned((void **)&g_eng.stage32, g_eng.stage32_cap, (size_t)host_cap, 4))) return rc;
    if ((rc = grow_pinned((void **)&g_eng.stage_pos, g_eng.stage_pos_cap, (size_t)ntiles, 8))) return rc;
    uint32_t *ranks32 = (uint32_t *)g_eng.ranks;  // rank-ordered tile offsets on the device
    int64_t *hbase = g_eng.hbase;  // mapped pinned mirror of the chunk bases
    const int64_t slot = tile_slot(p), ovf0 = slot * ntiles;
    const int64_t tile_cells = pow3l(p.g) * 243;
    for (int attempt = 0; attempt < 2; attempt++) {
        const size_t want = (size_t)ovf0 + std::max<size_t>(g_eng.scratch_want, (size_t)1 << 20);
        if ((rc = grow(g_eng.scratch, g_eng.scratch_cap, want, 4))) return rc;
        if ((rc = grow(g_eng.tile_rank0, g_eng.tile_rank0_cap, (size_t)ntiles, 8))) return rc;
        FinalArgs fa;
        fa.out = nullptr;
        fa.out32 = g_eng.scratch;
        fa.tile_rank0 = g_eng.tile_rank0;
        fa.cap = (int64_t)g_eng.scratch_cap;
        fa.slot = (int)slot;
        fa.ovf0 = ovf0;
        fa.rank_add = -p.rank_sub;
        fa.ib_mask = p.ib_E;
        fa.bitmap_out = nullptr;
        fa.alloc = g_eng.alloc;
        fa.tile_base = g_eng.tile_base;
        fa.tile_cnt = g_eng.tile_cnt;
        fa.prefetch = 3 * g_eng.num_sms;
        fa.pitch = p.pitch;
        fa.nz_e = nz_e_flags(p, state);
        set_gather(p, state, fa);
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
                                              (int64_t)0, (int64_t)(t1 - t0), s));
            k_chunk_advance<<<1, 32, 0, s>>>(g_eng.tile_cnt + t1 - 1, g_eng.tile_pos + t1 - 1, g_eng.chunk_base + c,
                                             hbase + c);
            CK_LAUNCH();
            const int grid = (int)std::min<int64_t>((t1 - t0 + 7) / 8, (int64_t)g_eng.num_sms * 8);
            k_reorder<uint32_t><<<grid, 256, 0, s>>>(g_eng.scratch, g_eng.tile_base + t0, g_eng.tile_cnt + t0,
                                                     g_eng.tile_pos + t0, g_eng.tile_rank0 + t0, ranks32, host_cap,
                                                     t1 - t0, (int64_t)g_eng.scratch_cap, g_eng.chunk_base + c);
            CK_LAUNCH();
            CK(cudaEventRecord(g_eng.chunk_ev[c], s));
        }
        // copy-out and widening as chunks complete
        bool fits = true;
        int issued = 0, widened = 0;
        auto ready = [](cudaEvent_t ev) {
            if (cudaEventQuery(ev) == cudaSuccess) return true;
            (void)cudaGetLastError();  // cudaErrorNotReady
            return false;
        };
        while (widened < K) {
            while (issued < K && ready(g_eng.chunk_ev[issued])) {
                const int c = issued++;
                const int64_t t0 = ntiles * c / K, t1 = ntiles * (c + 1) / K;
                const int64_t lo = hbase[c], hi = hbase[c + 1];
                if (hi > host_cap) fits = false;
                if (fits) {
                    CK(cudaMemcpyAsync(g_eng.stage_pos + t0, g_eng.tile_pos + t0, (size_t)(t1 - t0) * 8,
                                       cudaMemcpyDeviceToHost, g_eng.stream2));
                    if (hi > lo)
                        CK(cudaMemcpyAsync(g_eng.stage32 + lo, ranks32 + lo, (size_t)(hi - lo) * 4,
                                           cudaMemcpyDeviceToHost, g_eng.stream2));
                }
                CK(cudaEventRecord(g_eng.copy_ev[c], g_eng.stream2));
            }
            if (widened < issued && (issued == K || ready(g_eng.copy_ev[widened]))) {
                const int c = widened++;
                CK(cudaEventSynchronize(g_eng.copy_ev[c]));
                if (fits) {
                    const int64_t t0 = ntiles * c / K, t1 = ntiles * (c + 1) / K;
                    host_widen(g_eng.stage32, host, g_eng.stage_pos + t0, hbase[c], hbase[c + 1], t0, t1, tile_cells,
                               -p.rank_sub);
                }
                continue;
            }
            if (issued < K) CK(cudaEventSynchronize(g_eng.chunk_ev[issued]));
        }
        int64_t used = 0;
        CK(cudaMemcpyAsync(&used, g_eng.alloc, 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        CK(cudaStreamSynchronize(g_eng.stream2));
        *count = hbase[K];
        *host_ok = fits && *count <= host_cap;
        if (ovf0 + used <= (int64_t)g_eng.scratch_cap) break;
        g_eng.scratch_want = (size_t)((double)used * 1.05) + 1024;  // scratch overflow: once more
    }
    return DQMC_OK;
}

int final_set_attrs() {
    const int tile_smem = (int)pow3l(kC0Max) * 32;
    // + one 128-B piece (the padded pitch of a piece-major tile, make_plan) + 128 B of alignment
    CK(cudaFuncSetAttribute(k_c0_final<kC0Max>, cudaFuncAttributeMaxDynamicSharedMemorySize, tile_smem + 256));
    CK(cudaFuncSetAttribute(k_c0_final<kC0Max, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, tile_smem + 256));
    CK(cudaFuncSetAttribute(k_small, cudaFuncAttributeMaxDynamicSharedMemorySize, tile_smem));
    return DQMC_OK;
}

}  // namespace dqmc
