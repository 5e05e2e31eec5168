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
    const uint64_t near = 69984, nearp = 70016, far = 51018336;  // 3^7*32, padded to 128, 3^13*32
    const int X = 547, Q = 729;
    const uint64_t bytes = (uint64_t)Q * Q * nearp + (1 << 20);
    char *a, *b;
    if (cudaMalloc(&a, bytes) || cudaMalloc(&b, bytes)) {
        printf("alloc failed\n");
        return 1;
    }
    cudaMemset(a, 1, bytes);
    cudaMemset(b, 2, bytes);
    const int64_t items = (int64_t)X * Q;
    // standard layout [q2][q1][c] with tile pitch P: dims {P/4 words, q1 rows, q2}; item (x, q2), box rows along q1
    auto stdmap = [&](char *base, uint64_t P) { return mk(base, P / 4, Q, Q, 1, P, P * Q, P * Q * Q, BOXR, 1, 1); };
    const Side std_x_q2 = {{32, 0, 0, 0}, {0, 0, 1, 0}, {0, BOXR, 0, 0}};  // a = x, b = q2
    CUtensorMap sa = stdmap(a, near), sap = stdmap(a, nearp), sbp = stdmap(b, nearp), sb_ = stdmap(b, near);
    run("D now: in place, near stride 69984", sa, sa, Pat{X, items, std_x_q2, std_x_q2, 1, 1});
    run("D now, padded pitch 70016", sap, sap, Pat{X, items, std_x_q2, std_x_q2, 1, 1});
    // C now: the far map dims {8*3^13 words, 729 rows (q2, stride far)}; item (x, q1): word q1*17496 + 32x
    CUtensorMap cf = mk(a, far / 4, Q, 1, 1, far, far * Q, far * Q, BOXR, 1, 1);
    run("C now: write only, far stride", cf, cf, Pat{X, items, {}, {{32, 0, 0, 0}, {(int)(near / 4), 0, 0, 0}, {0, BOXR, 0, 0}}, 0, 1});
    // contiguous 93 KB tiles: dims {32, 729 rows, items}
    CUtensorMap ct = mk(a, 32, Q, items, 1, 128, TILE, (uint64_t)TILE * items, BOXR, 1, 1);
    CUtensorMap ctb = mk(b, 32, Q, items, 1, 128, TILE, (uint64_t)TILE * items, BOXR, 1, 1);
    const Side cont = {{0, 0, 0, 0}, {0, 0, 1, 0}, {0, BOXR, 0, 0}};  // A = 1, b = item
    Pat pc{1, items, cont, cont, 0, 1};
    run("C new: write only, contiguous 93 KB tiles", ct, ct, pc);
    // L' = [q1][x][q2][128B]: dims {32, q2 729 (128 B), x 547 (TILE), q1 729 (X*TILE)}; item (x, q2); box rows along q1
    CUtensorMap lp = mk(a, 32, Q, X, Q, 128, TILE, (uint64_t)X * TILE, 1, 1, BOXR);
    const Side lp_x_q2 = {{0, 0, 1, 0}, {0, 1, 0, 0}, {0, 0, 0, BOXR}};
    run("D new (x fastest): far read -> near write 70016", lp, sbp, Pat{X, items, lp_x_q2, std_x_q2, 1, 1});
    run("D new (x fastest): far read -> near write 69984", lp, sb_, Pat{X, items, lp_x_q2, std_x_q2, 1, 1});
    const Side lp_q2_x = {{0, 1, 0, 0}, {0, 0, 1, 0}, {0, 0, 0, BOXR}};
    const Side std_q2_x = {{0, 0, 1, 0}, {32, 0, 0, 0}, {0, BOXR, 0, 0}};
    run("D new (q2 fastest): far read -> near write 70016", lp, sbp, Pat{Q, items, lp_q2_x, std_q2_x, 1, 1});
    run("far read only (x fastest)", lp, lp, Pat{X, items, lp_x_q2, {}, 1, 0});
    run("far read only (q2 fastest)", lp, lp, Pat{Q, items, lp_q2_x, {}, 1, 0});
    run("near read only", sap, sap, Pat{X, items, std_x_q2, {}, 1, 0});
    run("contiguous read only", ct, ct, Pat{1, items, cont, {}, 1, 0});
    run("contiguous copy", ct, ctb, Pat{1, items, cont, cont, 1, 1});
    const Side cont_x = {{0, 0, 1, 0}, {0, 0, X, 0}, {0, BOXR, 0, 0}};
    run("contiguous read -> L' far write (x fastest)", ct, lp, Pat{X, items, cont_x, lp_x_q2, 1, 1});
    run("D new2: contiguous 93 KB tiles in place", ct, ct, Pat{1, items, cont, cont, 1, 1});
    // E under layout [q2][x][q1][128B]: tile (q2, q1) = 547 pieces at stride TILE; dims {32, q1, x, q2}
    CUtensorMap ex = mk(a, 32, Q, X, Q, 128, TILE, (uint64_t)X * TILE, 1, BOXR, 1);
    const Side e_q1_q2 = {{0, 1, 0, 0}, {0, 0, 0, 1}, {0, 0, BOXR, 0}};
    run("E new2: 547 pieces at 93 KB stride (read only)", ex, ex, Pat{Q, (int64_t)Q * Q, e_q1_q2, {}, 1, 0});
    run("E now: contiguous 70 KB (read only, as 729-row box)", ct, ct, Pat{1, items, cont, {}, 1, 0});
    return 0;
}
