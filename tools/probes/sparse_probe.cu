// Sparse-piece probe (n = 24 sizes): read+write in place only the 128-B pieces
// a bitmap flags (density d, pseudo-random), tile by tile, with SM loads and
// stores (8 lanes per piece, LDG.128/STG.128). Tiles are 729 contiguous pieces
// (pass D under piece-major storage) or 547 pieces 93 KB apart (pass E's read,
// read-only). Compares with all pieces.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
    return x;
}

__global__ void k_bits(uint32_t *bits, int64_t nwords, uint32_t thresh) {
    for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < nwords; w += (int64_t)gridDim.x * blockDim.x) {
        uint32_t m = 0;
        for (int b = 0; b < 32; b++) m |= (hash32((uint32_t)(w * 32 + b)) < thresh ? 1u : 0u) << b;
        bits[w] = m;
    }
}

// D pattern: tile t = pieces [t*729, t*729+729), bits contiguous.
// rw = 1: read and write back; 0: read only (sum kept live)
__global__ void __launch_bounds__(256) k_tiles(uint4 *s, const uint32_t *bits, int64_t ntiles, int tp, int64_t stride_p,
                                               int64_t tstride_p, int rw, int dense, unsigned long long *sink) {
    __shared__ uint16_t list[1024];
    __shared__ int cnt;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    uint32_t acc = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        // tile t: pieces p = t*tstride + j*stride, j < tp; bit index = t*tp + j
        if (threadIdx.x == 0) cnt = 0;
        __syncthreads();
        for (int j0 = 0; j0 < tp; j0 += blockDim.x) {  // warp-uniform trip count (ballot)
            const int j = j0 + threadIdx.x;
            const int64_t bi = t * tp + j;
            const bool on = j < tp && (dense || ((bits[bi >> 5] >> (bi & 31)) & 1u));
            const uint32_t m = __ballot_sync(0xffffffffu, on);
            int base = 0;
            if (lane == 0 && m) base = atomicAdd(&cnt, __popc(m));
            base = __shfl_sync(0xffffffffu, base, 0);
            if (on) list[base + __popc(m & ((1u << lane) - 1u))] = (uint16_t)j;
        }
        __syncthreads();
        const int n = cnt;
        // 4 pieces per warp instruction (8 lanes x 16 B each)
        for (int e = warp * 4 + (lane >> 3); e < n; e += nw * 4) {
            const int64_t base = tstride_p ? t * tstride_p : (t / 729) * (547 * 729) + (t % 729);
            uint4 *p = s + (base + (int64_t)list[e] * stride_p) * 8 + (lane & 7);
            uint4 x = *p;
            acc += x.x;
            if (rw) *p = make_uint4(x.x ^ 1u, x.y, x.z, x.w);
        }
        __syncthreads();
    }
    if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

int main() {
    setvbuf(stdout, nullptr, _IONBF, 0);
    const int64_t X = 547, Q = 729, npieces = X * Q * Q;  // n = 24 piece-major state
    uint4 *s;
    uint32_t *bits;
    unsigned long long *sink;
    if (cudaMalloc(&s, npieces * 128) || cudaMalloc(&bits, (npieces / 32 + 64) * 4) || cudaMalloc(&sink, 8)) {
        printf("alloc failed\n");
        return 1;
    }
    cudaMemset(s, 1, npieces * 128);
    for (double d : {0.25, 0.35, 0.5, 1.0}) {
        k_bits<<<148 * 8, 256>>>(bits, npieces / 32 + 32, (uint32_t)(d * 4294967295.0));
        cudaDeviceSynchronize();
        for (int mode = 0; mode < 3; mode++) {
            for (int grid_mul : {4, 8}) {
                float best = 1e9;
                for (int rep = 0; rep < 3; rep++) {
                    cudaEvent_t e0, e1;
                    cudaEventCreate(&e0);
                    cudaEventCreate(&e1);
                    cudaEventRecord(e0);
                    if (mode == 0)  // D: contiguous 729-piece tiles, read+write
                        k_tiles<<<148 * grid_mul, 256>>>(s, bits, X * Q, 729, 1, 729, 1, d >= 1.0, sink);
                    else if (mode == 1)  // E: 547 pieces 729 apart, read only; tile (q2,q1): base q2*X*Q + q1
                        k_tiles<<<148 * grid_mul, 256>>>(s, bits, Q * Q, 547, 729, 0, 0, d >= 1.0, sink);
                    else  // D read only
                        k_tiles<<<148 * grid_mul, 256>>>(s, bits, X * Q, 729, 1, 729, 0, d >= 1.0, sink);
                    cudaEventRecord(e1);
                    cudaEventSynchronize(e1);
                    float ms = 0;
                    cudaEventElapsedTime(&ms, e0, e1);
                    if (ms < best) best = ms;
                }
                const double useful = (double)npieces * 128 * d * (mode == 0 ? 2 : 1);
                printf("density %.2f %-28s grid %dx148: %7.2f ms  %6.0f GB/s useful  %s\n", d,
                       mode == 0 ? "D tiles read+write" : mode == 1 ? "E tiles (strided) read" : "D tiles read only",
                       grid_mul, best, useful / (best / 1e3) / 1e9, cudaGetErrorString(cudaGetLastError()));
            }
        }
    }
    return 0;
}
