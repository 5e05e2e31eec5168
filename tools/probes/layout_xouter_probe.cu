// Layout probe (round 2b): the x-outer layout [x][u][l][128 B] against the
// current piece-major [u][x][l][128 B]. Kernel as in layout_probe.cu:
// Layout probe: persistent TMA tensor-copy pipelines (UTMALDG/UTMASTG, 4-D
// maps, box 32 words x 243 rows) that move 729-row x 128-B items between two
// 37 GB buffers in the access patterns a re-laid-out plan would use (n = 24
// sizes), without compute. item it -> a = it % A, b = it / A; box j of the
// item sits at coordinates a*ca + b*cb + j*cj. One elected lane per CTA issues;
// two smem buffers; reads only, writes only, or copies.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
struct Side {
    int ca[4], cb[4], cj[4];
};
struct Pat {
    int64_t A, items;
    Side s, d;
    int has_src, has_dst;
};
constexpr int ROWS = 729, BOXR = 243, NBOX = 3, TILE = ROWS * 128;

__device__ __forceinline__ void coords(const Side &sd, int64_t a, int64_t b, int j, int (&c)[4]) {
    for (int k = 0; k < 4; k++) c[k] = (int)(a * sd.ca[k] + b * sd.cb[k] + j * sd.cj[k]);
}

__global__ void __launch_bounds__(32, 1) k_move(const __grid_constant__ CUtensorMap ms, const __grid_constant__ CUtensorMap md, Pat p) {
    extern __shared__ __align__(1024) char sm[];
    __shared__ __align__(8) uint64_t full[2];
    if (threadIdx.x != 0) return;
    for (int b = 0; b < 2; b++) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[b])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    int k = 0;
    int64_t prev = -1;
    for (int64_t it = blockIdx.x;; it += gridDim.x, k++) {
        const bool have = it < p.items;
        const int b = k & 1;
        if (have && p.has_src) {
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[b])), "r"((unsigned)TILE) : "memory");
            for (int j = 0; j < NBOX; j++) {
                int c[4];
                coords(p.s, it % p.A, it / p.A, j, c);
                asm volatile(
                    "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(
                        smem_u32(sm + b * TILE + j * BOXR * 128)),
                    "l"(&ms), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(smem_u32(&full[b]))
                    : "memory");
            }
        }
        if (prev >= 0) {
            const int pb = (k - 1) & 1;
            if (p.has_src) {
                const unsigned ph = (unsigned)(((k - 1) >> 1) & 1);
                asm volatile("{\n.reg .pred q;\nW: mbarrier.try_wait.parity.shared::cta.b64 q, [%0], %1;\n@!q bra W;\n}\n" ::"r"(smem_u32(&full[pb])), "r"(ph) : "memory");
            }
            if (p.has_dst) {
                if (!p.has_src) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                for (int j = 0; j < NBOX; j++) {
                    int c[4];
                    coords(p.d, prev % p.A, prev / p.A, j, c);
                    asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];" ::"l"(&md),
                                 "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(smem_u32(sm + pb * TILE + j * BOXR * 128))
                                 : "memory");
                }
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
        }
        if (!have) break;
        prev = it;
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

static PFN_cuTensorMapEncodeTiled_v12000 enc;
// 4-D map, dim0 = 32-bit words; box {32, b1, b2, b3}
static CUtensorMap mk(void *base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t d3, uint64_t s1, uint64_t s2, uint64_t s3,
                      uint32_t b1, uint32_t b2, uint32_t b3) {
    CUtensorMap m;
    cuuint64_t dims[4] = {d0, d1, d2, d3};
    cuuint64_t st[3] = {s1, s2, s3};
    cuuint32_t box[4] = {32, b1, b2, b3}, es[4] = {1, 1, 1, 1};
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 4, base, dims, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r) printf("encode failed %d\n", (int)r);
    return m;
}

static void run(const char *name, const CUtensorMap &ms, const CUtensorMap &md, Pat p) {
    const int smem = 2 * TILE;
    cudaFuncSetAttribute(k_move, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    float best = 1e9;
    for (int rep = 0; rep < 3; rep++) {
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        k_move<<<148, 32, smem>>>(ms, md, p);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms_ = 0;
        cudaEventElapsedTime(&ms_, e0, e1);
        if (ms_ < best) best = ms_;
    }
    cudaError_t e = cudaGetLastError();
    const double bytes = (double)p.items * TILE * (p.has_src + p.has_dst);
    printf("%-58s %7.2f ms  %6.0f GB/s (R+W)  %s\n", name, best, bytes / (best / 1e3) / 1e9, e ? cudaGetErrorString(e) : "");
}

int main() {
    cudaDriverEntryPointQueryResult q;
    void *fn = nullptr;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    const int X = 547, Q = 729;
    const uint64_t bytes = (uint64_t)X * Q * Q * 128 + (1 << 20);
    char *a;
    if (cudaMalloc(&a, bytes)) {
        printf("alloc failed\n");
        return 1;
    }
    cudaMemset(a, 1, bytes);
    const int64_t items = (int64_t)X * Q;
    // current piece-major layout [u][x][l][128B]: dims {32, l (128 B), x (TILE), u (X*TILE)}
    CUtensorMap pm = mk(a, 32, Q, X, Q, 128, TILE, (uint64_t)X * TILE, 243, 1, 1);
    // C now: item (x, l) over all u: box {32,1,1,243} rows along u; a = l (adjacent CTAs), b = x
    CUtensorMap pmc = mk(a, 32, Q, X, Q, 128, TILE, (uint64_t)X * TILE, 1, 1, BOXR);
    run("C now [u][x][l]: write, 128-B pieces 51 MB apart", pmc, pmc, Pat{Q, items, {}, {{0, 1, 0, 0}, {0, 0, 1, 0}, {0, 0, 0, BOXR}}, 0, 1});
    // D now: item (x, u) contiguous 93 KB
    run("D now [u][x][l]: R+W contiguous 93 KB", pm, pm, Pat{X, items, {{0, 0, 1, 0}, {0, 0, 0, 1}, {0, BOXR, 0, 0}}, {{0, 0, 1, 0}, {0, 0, 0, 1}, {0, BOXR, 0, 0}}, 1, 1});
    // E now: tile (u, l) = 547 pieces TILE apart: box {32,1,243,1}; a = l, b = u
    CUtensorMap pme = mk(a, 32, Q, X, Q, 128, TILE, (uint64_t)X * TILE, 1, BOXR, 1);
    run("E now [u][x][l]: read, 547(729) pieces 93 KB apart", pme, pme, Pat{Q, (int64_t)Q * Q, {{0, 1, 0, 0}, {0, 0, 0, 1}, {0, 0, BOXR, 0}}, {}, 1, 0});
    // x-outer layout [x][u][l][128B]: dims {32, l (128 B), u (TILE), x (Q*TILE)}
    CUtensorMap xo_c = mk(a, 32, Q, Q, X, 128, TILE, (uint64_t)Q * TILE, 1, BOXR, 1);
    run("C x-outer [x][u][l]: write, 128-B pieces 93 KB apart", xo_c, xo_c, Pat{Q, items, {}, {{0, 1, 0, 0}, {0, 0, 0, 1}, {0, 0, BOXR, 0}}, 0, 1});
    CUtensorMap xo_d = mk(a, 32, Q, Q, X, 128, TILE, (uint64_t)Q * TILE, BOXR, 1, 1);
    run("D x-outer [x][u][l]: R+W contiguous 93 KB", xo_d, xo_d, Pat{Q, items, {{0, 0, 1, 0}, {0, 0, 0, 1}, {0, BOXR, 0, 0}}, {{0, 0, 1, 0}, {0, 0, 0, 1}, {0, BOXR, 0, 0}}, 1, 1});
    CUtensorMap xo_e = mk(a, 32, Q, Q, X, 128, TILE, (uint64_t)Q * TILE, 1, 1, BOXR);
    run("E x-outer [x][u][l]: read, 547(729) pieces 68 MB apart", xo_e, xo_e, Pat{Q, (int64_t)Q * Q, {{0, 1, 0, 0}, {0, 0, 1, 0}, {0, 0, 0, BOXR}}, {}, 1, 0});
    return 0;
}
