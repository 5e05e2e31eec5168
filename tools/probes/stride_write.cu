// Write-pattern probe: 729-row x 128-B strips (one strip per work item) at a
// row stride of Q blocks, persistent CTAs taking items in column order, as the
// strided passes do; plus a contiguous control (each item = 93 KB in a row).
// 16-B stores (8 lanes per 128-B row, 4 rows per warp instruction).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

// wide variant: an item covers W adjacent 128-B columns of every row
__global__ void k_write_wide(uint4 *s, int64_t Qv, int64_t ncolw, int64_t nitems, int rows, int W) {
    const int t = threadIdx.x, nt = blockDim.x;
    for (int64_t it = blockIdx.x; it < nitems; it += gridDim.x) {
        const int64_t col = it % ncolw, outer = it / ncolw;
        uint4 *base = s + outer * rows * Qv + col * 8 * W;
        const int per = 8 * W;
        for (int i = t; i < rows * per; i += nt) base[(i / per) * Qv + (i % per)] = make_uint4(it, i, 0, 0);
    }
}

__global__ void k_write(uint4 *s, int64_t Qv, int64_t ncol, int64_t nitems, int rows, int contiguous) {
    const int t = threadIdx.x, nt = blockDim.x;
    for (int64_t it = blockIdx.x; it < nitems; it += gridDim.x) {
        if (contiguous) {
            uint4 *base = s + it * rows * 8;
#pragma unroll 6
            for (int i = t; i < rows * 8; i += nt) base[i] = make_uint4(it, i, 0, 0);
        } else {
            const int64_t col = it % ncol, outer = it / ncol;
            uint4 *base = s + outer * rows * Qv + col * 8;
#pragma unroll 6
            for (int i = t; i < rows * 8; i += nt) base[(i >> 3) * Qv + (i & 7)] = make_uint4(it, i, 0, 0);
        }
    }
}

int main() {
    const int rows = 729;
    const int64_t far_blocks = 1594320;  // ~3^13, multiple of 4
    const int64_t near_blocks = 2188;    // ~3^7, multiple of 4
    const int64_t total_blocks = far_blocks * rows;
    uint4 *s;
    if (cudaMalloc(&s, total_blocks * 32)) { printf("alloc failed\n"); return 1; }
    for (int W = 1; W <= 16; W *= 2) {  // far stride, W columns per item
        const int64_t Qb = far_blocks, Qv = Qb * 2, ncolw = Qb / (4 * W), nitems = ncolw * (total_blocks / (Qb * rows));
        float best = 1e9;
        for (int rep = 0; rep < 3; rep++) {
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0);
            k_write_wide<<<148, 1024>>>(s, Qv, ncolw, nitems, rows, W);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
        }
        const double bytes = (double)nitems * rows * 128 * W;
        printf("far stride, %2d columns (%4d B) per row per item: %.2f ms, %.0f GB/s\n", W, 128 * W, best, bytes / (best / 1e3) / 1e9);
    }
    for (int grid_mul = 1; grid_mul <= 4; grid_mul *= 2)
    for (int v = 0; v < 3; v++) {
        const int64_t Qb = v == 0 ? far_blocks : near_blocks;
        const int64_t Qv = Qb * 2, ncol = Qb / 4, nouter = total_blocks / (Qb * rows);
        const int64_t nitems = v == 2 ? total_blocks / (rows * 4) : ncol * nouter;
        float best = 1e9;
        for (int rep = 0; rep < 3; rep++) {
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0);
            k_write<<<148 * grid_mul, 1024 / grid_mul>>>(s, Qv, ncol, nitems, rows, v == 2);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
        }
        printf("grid %dx148 %s: %.2f ms, %.0f GB/s\n", grid_mul, v == 0 ? "far stride " : v == 1 ? "near stride" : "contiguous ",
               best, total_blocks * 32 / (best / 1e3) / 1e9);
    }
    return 0;
}
