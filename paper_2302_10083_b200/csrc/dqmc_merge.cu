// dqmc_merge.cu — MERGE passes A (k_c0_merge) and B (k_strided).
//
// The ternary transform of the reference (dense.py:174-243 with op MERGE;
// merge_triple dense.py:46-48): pass A builds the in-block and C0 axes from
// the truth table in shared memory, pass B merges each further group of up to
// six block axes in one sweep (run_merge).
#include "dqmc_internal.cuh"

namespace dqmc {
namespace {

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

// ---------------------------------------------------------------------------
// Pass B, the merge of one strided group: R = R1 + R2 block axes at block
// stride Q = 3^a (the top layer of dense.py:174-212, r axes per sweep).
// Tile = 3^R rows x 4 blocks (128 B); row rho = rho1 + 3^R1 * rho2. Work item
// = (outer, column); lane = word within the 128-B row. Only rows binary on
// the group are read; only its star rows are written (SURVEY.md App. B.1:
// star cells are empty before their axis is merged).
template <int R1, int R2>
__global__ void __launch_bounds__(kStridedThreads) k_strided(uint32_t *__restrict__ state, int64_t Q, int64_t ncol,
                                                             int64_t nitems, int64_t rs, int64_t cs, int64_t os) {
    constexpr int N1 = P3<R1>::v, N2 = P3<R2>::v, B1 = 1 << R1, B2 = 1 << R2;
    extern __shared__ __align__(16) uint32_t sm[];  // 3^R rows x 32 words (rounds 1 -> 2)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nwarps = blockDim.x >> 5;
    // strides in blocks: row rs, column cs, outer os (reference layout: Q, 4,
    // 3^R Q; piece-major group 0: 4, 3^R 4, pitch 3^R)
    const int64_t Qw = rs * 8;  // row stride in words

    for (int64_t item = blockIdx.x; item < nitems; item += gridDim.x) {
        const int64_t col = item % ncol;
        const int64_t ob = bin_to_tern_rt((uint64_t)(item / ncol));  // the outer digits are binary too
        const int64_t c0 = col * kRowBlocks;
        const int valid = (int)min((int64_t)kRowBlocks, Q - c0) * 8;
        const bool act = lane < valid;
        uint32_t *g0 = state + (ob * os + col * cs) * 8 + lane;  // word of row 0

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
#pragma unroll
            for (int i = 0; i < N1; i++) {
                if (has_star(i, R1) && act) g0[(int64_t)(i + N1 * r2) * Qw] = v[i];
                if (R2 > 0) sm[(i + N1 * r2) * 32 + lane] = v[i];
            }
        }
        __syncthreads();
        if (R2 > 0) {
            // round 2: for each rho1, merge the R2 axes
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
#pragma unroll
                for (int i = 0; i < N2; i++)
                    if (has_star(i, R2) && act) g0[(int64_t)(t1 + N1 * i) * Qw] = v[i];
            }
            __syncthreads();
        }
    }
}

template <int R1, int R2>
void launch_strided(uint32_t *state, int64_t Q, int64_t ncol, int64_t nitems, bool pm, cudaStream_t s) {
    constexpr int NR = P3<R1>::v * P3<R2>::v;
    const int grid = (int)std::min<int64_t>(nitems, (int64_t)g_eng.num_sms * 16);
    k_strided<R1, R2><<<grid, kStridedThreads, NR * 32 * 4, s>>>(state, Q, ncol, nitems, pm ? kRowBlocks : Q,
                                                                 pm ? NR * kRowBlocks : kRowBlocks, pm ? Q * NR : NR * Q);
}

void launch_strided_r(int r, uint32_t *state, int64_t Q, int64_t ncol, int64_t nitems, bool pm, cudaStream_t s) {
    switch (r) {
        case 1: launch_strided<1, 0>(state, Q, ncol, nitems, pm, s); break;
        case 2: launch_strided<2, 0>(state, Q, ncol, nitems, pm, s); break;
        case 3: launch_strided<3, 0>(state, Q, ncol, nitems, pm, s); break;
        case 4: launch_strided<2, 2>(state, Q, ncol, nitems, pm, s); break;
        case 5: launch_strided<3, 2>(state, Q, ncol, nitems, pm, s); break;
        default: launch_strided<3, 3>(state, Q, ncol, nitems, pm, s); break;
    }
}

template <int R1, int R2>
int set_strided_attr() {
    constexpr int smem = P3<R1>::v * P3<R2>::v * 32 * 4;
    CK(cudaFuncSetAttribute(k_strided<R1, R2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    return DQMC_OK;
}

}  // namespace

int merge_set_attrs() {
    const int tile_smem = (int)pow3l(kC0Max) * 32;
    CK(cudaFuncSetAttribute(k_c0_merge, cudaFuncAttributeMaxDynamicSharedMemorySize, tile_smem));
    int rc;
    if ((rc = set_strided_attr<1, 0>()) || (rc = set_strided_attr<2, 0>()) || (rc = set_strided_attr<3, 0>()) ||
        (rc = set_strided_attr<2, 2>()) || (rc = set_strided_attr<3, 2>()) || (rc = set_strided_attr<3, 3>()))
        return rc;
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
    CK_LAUNCH();
    tm.mark("k_c0_merge", (uint64_t)ntA * ((1ull << p.g) * 4 + (uint64_t)pow3l(p.g) * 32));
    auto frac = [&](int k) { return (double)S * std::pow(2.0 / 3.0, k); };
    const int last = full ? p.m : p.m - 1;
    for (int k = 0; k < last; k++) {
        const int64_t Q = pow3l(p.a[k] - p.g) * p.pitch;
        const int64_t ncol = (Q + kRowBlocks - 1) / kRowBlocks;
        int above = 0;
        for (int j = k + 1; j < p.m; j++) above += p.r[j];
        const int64_t nitems = ncol << above;
        launch_strided_r(p.r[k], state, Q, ncol, nitems, k == 0 && p.pm, s);
        CK_LAUNCH();
        tm.mark("k_strided<MERGE_ONLY>", (uint64_t)frac(above));
    }
    return DQMC_OK;
}

}  // namespace dqmc
