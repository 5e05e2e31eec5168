// Far-stride write probe: a warp writes each 128-B row piece with one STG.32
// per lane (lane = word). Variant P: the warp writes the same row of P adjacent
// columns back to back (P separate 128-B stores); items are P columns wide.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int P>
__global__ void __launch_bounds__(1024) k_pair(uint32_t *s, int64_t Qw, int64_t ncolp, int64_t nitems, int rows) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int64_t it = blockIdx.x; it < nitems; it += gridDim.x) {
        const int64_t col = it % ncolp, outer = it / ncolp;
        uint32_t *base = s + outer * rows * Qw + col * 32 * P;
        for (int r = warp; r < rows; r += nw) {
#pragma unroll
            for (int p = 0; p < P; p++) base[r * Qw + p * 32 + lane] = (uint32_t)(it + r + p);
        }
    }
}

template <int P>
void run(uint32_t *s, int64_t total_blocks, int64_t Qb, int rows) {
    const int64_t Qw = Qb * 8, ncolp = Qb / (4 * P), nitems = ncolp * (total_blocks / (Qb * rows));
    float best = 1e9;
    for (int rep = 0; rep < 3; rep++) {
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        k_pair<P><<<148, 1024>>>(s, Qw, ncolp, nitems, rows);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const double bytes = (double)nitems * P * rows * 128;
    printf("P=%d (%4d B per row piece-group, %d STG.32 per row): %.2f ms, %.0f GB/s\n", P, 128 * P, P, best,
           bytes / (best / 1e3) / 1e9);
}

int main() {
    const int rows = 729;
    const int64_t Qb = 1594320, total_blocks = Qb * rows;
    uint32_t *s;
    if (cudaMalloc(&s, total_blocks * 32)) { printf("alloc failed\n"); return 1; }
    run<1>(s, total_blocks, Qb, rows);
    run<2>(s, total_blocks, Qb, rows);
    run<4>(s, total_blocks, Qb, rows);
    run<1>(s, total_blocks, Qb, rows);
    run<2>(s, total_blocks, Qb, rows);
    return 0;
}
