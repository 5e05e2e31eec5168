// Far-stride write probe: do thread-block clusters whose CTAs write adjacent
// 128-B columns, synchronised per item by a cluster barrier, behave like one
// CTA writing a wide (C x 128 B) strip? 729 rows per item, row stride ~3^13 blocks.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

template <int C>
__global__ void __launch_bounds__(1024) k_cluster_write(uint4 *s, int64_t Qv, int64_t ncolg, int64_t nitems, int rows, int sync) {
    cg::cluster_group cl = cg::this_cluster();
    const int r = (int)cl.block_rank();
    const int64_t grp = blockIdx.x / C, ngrp = gridDim.x / C;
    for (int64_t it = grp; it < nitems; it += ngrp) {
        if (sync) cl.sync();
        const int64_t colg = it % ncolg, outer = it / ncolg;
        uint4 *base = s + outer * rows * Qv + (colg * C + r) * 8;
        for (int i = threadIdx.x; i < rows * 8; i += blockDim.x) base[(i >> 3) * Qv + (i & 7)] = make_uint4(it, i, r, 0);
    }
}

template <int C>
void run(uint4 *s, int64_t total_blocks, int64_t Qb, int rows, int sync) {
    const int64_t Qv = Qb * 2, ncolg = Qb / (4 * C), nitems = ncolg * (total_blocks / (Qb * rows));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(148 / C * C);
    cfg.blockDim = dim3(1024);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C, at[0].val.clusterDim.y = 1, at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    float best = 1e9;
    for (int rep = 0; rep < 3; rep++) {
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        cudaLaunchKernelEx(&cfg, k_cluster_write<C>, s, Qv, ncolg, nitems, rows, sync);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    cudaError_t e = cudaGetLastError();
    const double bytes = (double)nitems * C * rows * 128;
    printf("cluster %d, %s: %.2f ms, %.0f GB/s %s\n", C, sync ? "barrier per item" : "no barrier      ", best,
           bytes / (best / 1e3) / 1e9, e ? cudaGetErrorString(e) : "");
}

int main() {
    const int rows = 729;
    const int64_t Qb = 1594320, total_blocks = Qb * rows;
    uint4 *s;
    if (cudaMalloc(&s, total_blocks * 32)) { printf("alloc failed\n"); return 1; }
    for (int sync = 0; sync < 2; sync++) {
        run<1>(s, total_blocks, Qb, rows, sync);
        run<2>(s, total_blocks, Qb, rows, sync);
        run<4>(s, total_blocks, Qb, rows, sync);
        run<8>(s, total_blocks, Qb, rows, sync);
    }
    return 0;
}
