// Read-modify-write probe in the reduce pass's pattern: items = (outer, column),
// each item reads 729 rows x 128 B at a row stride of Q blocks into smem and
// writes them back, persistent CTAs taking items strided over the grid. Q odd
// (3^7 = 2187, rows only 32-B aligned, as in the state) vs Q = 2188 (rows
// 128-B aligned), same bytes. Plain LDG/STG, 2 CTAs/SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(512) k_rmw(uint4 *s, int64_t Qv, int64_t ncol, int64_t nitems, int rows) {
    extern __shared__ uint4 t[];
    for (int64_t it = blockIdx.x; it < nitems; it += gridDim.x) {
        const int64_t col = it % ncol, outer = it / ncol;
        uint4 *base = s + outer * rows * Qv + col * 8;
        for (int i = threadIdx.x; i < rows * 8; i += blockDim.x) t[i] = base[(i >> 3) * Qv + (i & 7)];
        __syncthreads();
        for (int i = threadIdx.x; i < rows * 8; i += blockDim.x) {
            uint4 v = t[i];
            v.x ^= 1u;
            base[(i >> 3) * Qv + (i & 7)] = v;
        }
        __syncthreads();
    }
}

int main() {
    const int rows = 729;
    const int64_t outer = 729;
    for (int pass = 0; pass < 2; pass++)
    for (int v = 0; v < 2; v++) {
        const int64_t Qb = v == 0 ? 2187 : 2188;
        const int64_t total = Qb * rows * outer;  // blocks
        uint4 *s;
        if (cudaMalloc(&s, total * 32)) { printf("alloc failed\n"); return 1; }
        cudaMemset(s, 0, total * 32);
        const int64_t Qv = Qb * 2, ncol = 2187 / 4, nitems = ncol * outer;
        cudaFuncSetAttribute(k_rmw, cudaFuncAttributeMaxDynamicSharedMemorySize, rows * 128);
        float best = 1e9;
        for (int rep = 0; rep < 3; rep++) {
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0);
            k_rmw<<<148, 512, rows * 128>>>(s, Qv, ncol, nitems, rows);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
        }
        const double bytes = 2.0 * nitems * rows * 128;
        printf("Q=%lld (%s): %.2f ms, %.0f GB/s (R+W)\n", (long long)Qb, v == 0 ? "32-B aligned rows" : "128-B aligned rows",
               best, bytes / (best / 1e3) / 1e9);
        cudaFree(s);
    }
    return 0;
}
