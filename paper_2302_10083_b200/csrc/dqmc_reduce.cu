// dqmc_reduce.cu — REDUCE passes C (k_merge_reduce_pipe) and D (k_strided_pipe).
//
// Prime extraction of the reference (dense.py:174-243 with op REDUCE;
// reduce_triple dense.py:51-53). In-place REDUCE in any dimension order, and
// several axes' kills taken from one input state, equal M & ~OR_j M(parent_j)
// (SURVEY.md App. B.2), so the groups are reduced in whatever order the
// passes stream best. Both kernels are persistent (one CTA per SM) with TMA
// tensor loads and stores double-buffered against the compute warps.
#include "dqmc_internal.cuh"

namespace dqmc {
namespace {

// At n = 24 about four in five blocks of the state are zero, and reducing a
// zero cell is a no-op: the reduce rounds skip all-zero warps (warp_any).
constexpr int kSparseSkip = 1;

template <int R1, int R2>
__global__ void __launch_bounds__(PipeSmem<R1, R2>::THREADS, 1)
    k_strided_pipe(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ CUtensorMap zmap,
                   int64_t ncol, int64_t nitems, uint32_t ib_mask, int pm, int sparse,
                   const uint32_t *__restrict__ nz_b, const unsigned long long *__restrict__ g0_cnt,
                   unsigned long long g0_limit) {
    using SM = PipeSmem<R1, R2>;
    constexpr int N1 = SM::N1, N2 = SM::N2;
    constexpr int NR = SM::NR;
    constexpr int CW = SM::CW;
    constexpr int CC = pipe_cols<R1, R2>(), PITCH = SM::PITCH;
    extern __shared__ __align__(128) uint32_t smem[];
    __shared__ __align__(8) uint64_t full[2], computed[2];
    // sparse state: the final stage gathers this group's parents itself (FinalArgs::g0)
    if (gather_chosen(g0_cnt, g0_limit)) return;
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
    // zero-skip flags (piece-major, Plan::nz): box j (rows 243 j .. 243 j + 242)
    // of item (x = col, u = outer) is all zero when pass C saw no nonzero row u
    // in the items (x, l) of those rows. The producer warp lists the CTA's
    // items with a nonzero box, and their box masks, before the pipeline starts
    // (in the stage area, unused by this kernel); zero boxes are loaded from a
    // zero page (L2) and not stored back. The compute warps only need the count.
    constexpr int kListCap = 2 * SM::STAGE_WORDS;  // uint16 entries, then as many uint8 box masks
    uint16_t *s_list = reinterpret_cast<uint16_t *>(smem + 2 * SM::TILE_WORDS);
    uint8_t *s_bm = reinterpret_cast<uint8_t *>(s_list + kListCap);
    __shared__ int s_nitems;
    const bool listed = nz_b != nullptr && L <= kListCap && SM::NBOX == 3;

    if (threadIdx.x == 0) {
        for (int b = 0; b < 2; b++) {
            mbar_init(&full[b], 1);
            mbar_init(&computed[b], CW);
        }
    }
    if (warp == CW) {
        if (listed) {
            const uint32_t lt = (1u << lane) - 1u;
            int n = 0;
            for (int64_t i0 = 0; i0 < L; i0 += 8 * 32) {
                uint32_t f[8];
#pragma unroll
                for (int q = 0; q < 8; q++) {  // 24 flag loads in flight per lane
                    const int64_t i = i0 + 32 * q + lane;
                    const int64_t it = item(i < L ? i : 0);
                    const int64_t col = it % ncol, outer = it / ncol;
                    f[q] = 0u;
#pragma unroll
                    for (int j = 0; j < 3; j++)
                        f[q] |= ((__ldg(&nz_b[(col * 3 + j) * kNzWords + (outer >> 5)]) >> (outer & 31)) & 1u) << j;
                    if (i >= L) f[q] = 0u;
                }
#pragma unroll
                for (int q = 0; q < 8; q++) {
                    const uint32_t m = __ballot_sync(0xffffffffu, f[q] != 0u);
                    if (f[q]) {
                        const int e = n + __popc(m & lt);
                        s_list[e] = (uint16_t)(i0 + 32 * q + lane);
                        s_bm[e] = (uint8_t)f[q];
                    }
                    n += __popc(m);
                }
            }
            if (lane == 0) s_nitems = n;
        } else if (lane == 0) {
            s_nitems = (int)L;
        }
    }
    __syncthreads();
    const int K = s_nitems;

    if (warp == CW) {
        // ------------------------------ producer warp (one elected lane)
        if (lane == 0) {
            int64_t pend0 = -1, pend1 = -1;  // item held in buffer 0 / 1
            uint32_t bm0 = 7, bm1 = 7;       // its nonzero boxes
            auto store = [&](int64_t kk) {  // the stores of slot kk (buffer kk & 1) once computed
                const int b = (int)(kk & 1);
                const uint32_t *tile = smem + b * SM::TILE_WORDS;
                mbar_wait(&computed[b], (unsigned)((kk >> 1) & 1));
                int c0, c2, c3;
                crd(b ? pend1 : pend0, c0, c2, c3);
                const uint32_t bm = b ? bm1 : bm0;
#pragma unroll
                for (int x = 0; x < SM::NBOX; x++) {  // one bulk group per box (empty for a zero box)
                    if ((bm >> x) & 1u) tma_store_4d(&tmap, c0, x * SM::BOXR, c2, c3, tile + x * SM::BOXR * PITCH);
                    bulk_commit();
                }
            };
            for (int k = 0; k < K; k++) {
                const int64_t it = item(listed ? (int64_t)s_list[k] : (int64_t)k);
                const uint32_t bm = listed ? s_bm[k] : 7u;
                const int b = k & 1;
                uint32_t *tile = smem + b * SM::TILE_WORDS;
                const bool st = k >= 2;
                if (st) store(k - 2);
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
                    if ((bm >> x) & 1u)
                        tma_load_4d(tile + x * SM::BOXR * PITCH, &tmap, c0, x * SM::BOXR, c2, c3, &full[b]);
                    else  // all-zero box: zeros from the L2-resident zero page, no HBM read
                        tma_load_4d(tile + x * SM::BOXR * PITCH, &zmap, 0, 0, 0, 0, &full[b]);
                }
                if (st) bulk_wait_read<0>();  // buffer b is rewritten by compute only after `full`
                if (b) pend1 = it, bm1 = bm;
                else pend0 = it, bm0 = bm;
            }
            for (int kk = K >= 2 ? K - 2 : 0; kk < K; kk++) {
                store(kk);
                bulk_wait_read<0>();
            }
            bulk_wait0();
        }
        return;
    }

    // ---------------------------------- compute warps
    constexpr int NCT = CW * 32;
    for (int k = 0; k < K; k++) {
        const int b = k & 1;
        const int tb = b * SM::TILE_WORDS;
        mbar_wait(&full[b], (unsigned)((k >> 1) & 1));
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
                        int64_t ncol, int64_t nitems, uint32_t ib_mask, int sparse, uint32_t *__restrict__ nz_b,
                        uint32_t *__restrict__ nz_e, int nz_nr, unsigned long long *__restrict__ nz_cnt) {
    using SM = PipeSmem<R1, R2>;
    constexpr int N1 = SM::N1, N2 = SM::N2, B1 = 1 << R1, B2 = 1 << R2;
    constexpr int NR = SM::NR;
    constexpr int CW = SM::CW;
    constexpr int CC = pipe_cols<R1, R2>(), PITCH = SM::PITCH;
    extern __shared__ __align__(128) uint32_t smem[];
    __shared__ __align__(8) uint64_t stage_full[2], stage_free[2], tile_done[2], tile_free[2];
    __shared__ uint32_t s_blk[2][4 * kNzWords];  // nonzero blocks of the tile (zero-skip flags, CC = 1)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t L = nitems > blockIdx.x ? (nitems - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;

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
        unsigned nblk = 0;  // nonzero blocks this CTA wrote (chooses pass D or the gather finish)
        for (int64_t i = 0; i < L; i++) {
            const int b = (int)(i & 1);
            const int64_t it = blockIdx.x + i * gridDim.x;
            mbar_wait(&tile_done[b], (unsigned)((i >> 1) & 1));
            const int64_t col = it % ncol;
            if (lane == 0) {
                const uint32_t *tile = smem + b * SM::TILE_WORDS;
                const int c0 = (int)(col * 32 * CC);
#pragma unroll
                for (int x = 0; x < SM::NBOX; x++) tma_store_3d(&tmap, c0, x * SM::BOXR, 0, tile + x * SM::BOXR * PITCH);
                bulk_commit();
            }
            // the nonzero rows u (4 blocks each) of item (x, l), read before the
            // buffer is released and published after (flags do not gate it)
            uint32_t w = 0, od = ~0u, oe = ~0u;
            uint32_t *fd = nullptr, *fe = nullptr;
            if (nz_b && lane < kNzWords) {
                const int nw = (NR * kRowBlocks + 31) / 32;
#pragma unroll
                for (int q = 0; q < 4; q++)
                    if (4 * lane + q < nw) {
                        const uint32_t m = s_blk[b][4 * lane + q];
                        w |= or4_compact(m) << (8 * q);
                        nblk += __popc(m);
                    }
                // D item (x, u), E tile (u, l); dense inputs: most bits are
                // already set, so read first (in flight during the wait below)
                fd = &nz_b[((col / nz_nr) * 3 + (col % nz_nr) / (nz_nr / 3)) * kNzWords + lane];
                fe = &nz_e[(col % nz_nr) * kNzWords + lane];
                if (w) od = __ldcg(fd), oe = __ldcg(fe);
            }
            __syncwarp();
            if (lane == 0) {
                bulk_wait_read0();
                mbar_arrive(&tile_free[b]);
            }
            if ((od & w) != w) atomicOr(fd, w);
            if ((oe & w) != w) atomicOr(fe, w);
        }
        if (nz_cnt) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) nblk += __shfl_xor_sync(0xffffffffu, nblk, o);
            if (lane == 0) atomicAdd(nz_cnt, (unsigned long long)nblk);
        }
        if (lane == 0) bulk_wait0();
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
                if (sparse && !warp_any(v)) continue;
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
            inblock_round(&smem[tb], NR * kRowBlocks * CC, ib_mask, NCT, sparse, nz_b ? s_blk[b] : nullptr);
        }
        fence_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tile_done[b]);
    }
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
                uint32_t *nz, unsigned long long g0_limit) {
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
    }
    const int64_t ncolg = (ncol + CC - 1) / CC;  // column groups: one tile each per outer index
    const int64_t nitems = ncolg * nouter;
    const int grid = (int)std::min<int64_t>(nitems, g_eng.num_sms);
    if (MODE == MERGE_REDUCE)
        k_merge_reduce_pipe<R1, R2><<<grid, SM::THREADS + 32, SM::SMEM, s>>>(
            map, gmap, ncolg, nitems, ib, kSparseSkip, nz, nz ? nz + nz_e_offset(Q / kRowBlocks / pow3l(R1 + R2)) : nullptr,
            P3<R1 + R2>::v,
            nz ? reinterpret_cast<unsigned long long *>(
                     nz + nz_count_offset((size_t)(Q / kRowBlocks / pow3l(R1 + R2)), (size_t)P3<R1 + R2>::v))
               : nullptr);
    else
    {
        CUtensorMap zmap;  // zero-skip mode: the zero page, box {32, BOXR} (a fully-specified map otherwise unused)
        memset(&zmap, 0, sizeof zmap);
        if (nz) {
            if ((rc = ensure_encode())) return rc;
            const uint32_t *zp = nz + nz_zero_page((size_t)ncolg, (size_t)SM::NR);
            cuuint64_t dims[4] = {32, (cuuint64_t)SM::BOXR, 1, 1};
            cuuint64_t strides[3] = {128, (cuuint64_t)SM::BOXR * 128, (cuuint64_t)SM::BOXR * 128};
            cuuint32_t box[4] = {32, (cuuint32_t)SM::BOXR, 1, 1}, es[4] = {1, 1, 1, 1};
            CUresult r = g_eng.encode(&zmap, CU_TENSOR_MAP_DATA_TYPE_UINT32, 4, (void *)zp, dims, strides, box, es,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r != CUDA_SUCCESS) return set_err(DQMC_ERR_CUDA, "cuTensorMapEncodeTiled (zero page) failed: " + std::to_string((int)r));
        }
        k_strided_pipe<R1, R2><<<grid, SM::THREADS, SM::SMEM, s>>>(map, zmap, ncolg, nitems, ib, pm ? 1 : 0,
                                                                   kSparseSkip, nz,
                                                                   nz ? reinterpret_cast<const unsigned long long *>(
                                                                            nz + nz_count_offset((size_t)ncolg, (size_t)SM::NR))
                                                                      : nullptr,
                                                                   g0_limit);
    }
    CK_LAUNCH();
    return DQMC_OK;
}

template <int MODE>
int launch_pipe_mode(int r, uint32_t *state, int64_t Q, int64_t ncol, int64_t nouter, uint32_t ib, cudaStream_t s,
                     bool pm = false, uint32_t *nz = nullptr, unsigned long long g0_limit = 0) {
    switch (r) {
        case 1: return launch_pipe<1, 0, MODE>(state, Q, ncol, nouter, ib, pm, s, nullptr, 0);
        case 2: return launch_pipe<2, 0, MODE>(state, Q, ncol, nouter, ib, pm, s, nullptr, 0);
        case 3: return launch_pipe<3, 0, MODE>(state, Q, ncol, nouter, ib, pm, s, nullptr, 0);
        case 4: return launch_pipe<2, 2, MODE>(state, Q, ncol, nouter, ib, pm, s, nullptr, 0);
        case 5: return launch_pipe<3, 2, MODE>(state, Q, ncol, nouter, ib, pm, s, nullptr, 0);
        default: return launch_pipe<3, 3, MODE>(state, Q, ncol, nouter, ib, pm, s, nz, g0_limit);
    }
}


template <int R1, int R2>
int set_pipe_attr() {
    using SM = PipeSmem<R1, R2>;
    CK(cudaFuncSetAttribute(k_strided_pipe<R1, R2>, cudaFuncAttributeMaxDynamicSharedMemorySize, SM::SMEM));
    CK(cudaFuncSetAttribute(k_merge_reduce_pipe<R1, R2>, cudaFuncAttributeMaxDynamicSharedMemorySize, SM::SMEM));
    return DQMC_OK;
}

// Timing mode: how many D items / E tiles the zero-skip flags let through
// (out[0] += set bits of the first nd words, out[1] += of the next ne words)
__global__ void k_nz_count(const uint32_t *__restrict__ f, int nd, int ne, unsigned long long *out) {
    unsigned long long a = 0, b = 0;
    for (int i = threadIdx.x; i < nd + ne; i += blockDim.x) (i < nd ? a : b) += __popc(f[i]);
    for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        b += __shfl_xor_sync(0xffffffffu, b, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&out[0], a);
        atomicAdd(&out[1], b);
    }
}

}  // namespace

// Bytes the zero-skip passes really moved (DQMC_FLAG_TIMING): the marks of
// pass D (group 0) and pass E count only the items / tiles not skipped.
int nz_account(const Plan &p, Timer &tm, cudaStream_t s) {
    if (!tm.on || !p.nz || !g_eng.nzflags) return DQMC_OK;
    const int npiece = (int)(p.pitch / kRowBlocks), nr = (int)pow3l(p.r[0]);
    const int nd = npiece * 3 * kNzWords, ne = nr * kNzWords;
    unsigned long long *cnt = reinterpret_cast<unsigned long long *>(g_eng.total) + 4;
    CK(cudaMemsetAsync(cnt, 0, 16, s));
    k_nz_count<<<1, 1024, 0, s>>>(g_eng.nzflags, nd, ne, cnt);
    CK_LAUNCH();
    unsigned long long h[2] = {0, 0}, nblk = 0;
    CK(cudaMemcpyAsync(h, cnt, 16, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&nblk, g_eng.nzflags + nz_count_offset((size_t)npiece, (size_t)nr), 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    // gather finish: pass D returned at once; the final stage read the group-0
    // parents of its surviving blocks from L2 (no algorithmic HBM bytes)
    if (nblk <= g_eng.gather_limit_last) h[0] = 0;
    const uint64_t box_d = (uint64_t)(nr / 3) * 128, tile_e = (uint64_t)p.pitch * 32;
    int last_d = -1, e = -1;
    for (size_t i = 0; i < tm.names.size(); i++) {
        if (tm.names[i] == "k_strided<REDUCE>") last_d = (int)i;
        if (tm.names[i] == "k_c0_final") e = (int)i;
    }
    if (last_d >= 0) tm.bytes[last_d] = 2 * h[0] * box_d;  // the nonzero boxes, read and written
    if (e >= 0) tm.bytes[e] = tm.bytes[e] - (uint64_t)p.nblocks * 32 + h[1] * tile_e;  // the state part of E's bytes
    return DQMC_OK;
}

int reduce_set_attrs() {
    int rc;
    if ((rc = set_pipe_attr<1, 0>()) || (rc = set_pipe_attr<2, 0>()) || (rc = set_pipe_attr<3, 0>()) ||
        (rc = set_pipe_attr<2, 2>()) || (rc = set_pipe_attr<3, 2>()) || (rc = set_pipe_attr<3, 3>()))
        return rc;
    return DQMC_OK;
}

// REDUCE passes of the strided groups. fused: the last group is merged and
// reduced in one pass (single-GPU plan); otherwise every group is reduce-only
// (sharded path, M already complete). The in-block axes of pass C go with the
// last group either way.
int run_reduce(const Plan &p, uint32_t *state, bool fused, Timer &tm, cudaStream_t s, int64_t nbatch) {
    const uint64_t S = (uint64_t)p.nblocks * 32 * nbatch;
    if (nbatch > 1 && (fused || p.pm)) return set_err(DQMC_ERR_INVALID, "internal: batched reduce is reduce-only");
    int rc;
    // zero-skip flags (Plan::nz): pass C writes them, pass D and E read them
    uint32_t *nz = nullptr;
    size_t nz_words = 0;
    if (fused && p.nz) {
        const size_t npiece = (size_t)(p.pitch / kRowBlocks), nr = (size_t)pow3l(p.r[0]);
        nz_words = (npiece * 3 + nr) * kNzWords;  // nz_b, nz_e: zeroed per call
        const size_t zp = nz_zero_page(npiece, nr), zwords = (nr / 3) * 32;
        if ((rc = grow(g_eng.nzflags, g_eng.nzflags_cap, zp + zwords + 2, 4))) return rc;
        nz = g_eng.nzflags;
        CK(cudaMemsetAsync(nz + zp, 0, (zwords + 2) * 4, s));  // the zero page and pass C's block count
    }
    {
        const int k = p.m - 1;
        const int64_t Q = pow3l(p.a[k] - p.g) * p.pitch;
        const int64_t ncol = (Q + kRowBlocks - 1) / kRowBlocks;
        if (fused) {
            if (nz) {
                CK(cudaMemsetAsync(nz, 0, nz_words * 4, s));
                g_eng.gather_n = p.n;
                g_eng.gather_limit_last = gather_limit(p);
            }
            if ((rc = launch_pipe_mode<MERGE_REDUCE>(p.r[k], state, Q, ncol, 1, p.ib_C, s, false, nz))) return rc;
            tm.mark("k_strided<MERGE_REDUCE>", (uint64_t)(S * std::pow(2.0 / 3.0, p.r[k]) + S));
        } else {
            if ((rc = launch_pipe_mode<REDUCE_ONLY>(p.r[k], state, Q, ncol, nbatch, p.ib_C, s))) return rc;
            tm.mark("k_strided<REDUCE>", 2 * S);
        }
    }
    for (int k = p.m - 2; k >= 0; k--) {
        const int64_t Q = pow3l(p.a[k] - p.g) * p.pitch;
        const int64_t ncol = (Q + kRowBlocks - 1) / kRowBlocks;
        int above = 0;
        for (int j = k + 1; j < p.m; j++) above += p.r[j];
        if ((rc = launch_pipe_mode<REDUCE_ONLY>(p.r[k], state, Q, ncol, pow3l(above) * nbatch, p.ib_D[k], s,
                                                k == 0 && p.pm, k == 0 ? nz : nullptr,
                                                k == 0 && nz ? gather_limit(p) : 0)))
            return rc;
        tm.mark("k_strided<REDUCE>", 2 * S);
    }
    return DQMC_OK;
}

}  // namespace dqmc
