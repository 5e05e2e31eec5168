// dqmc_input.cu — truth-table ingestion and the synthetic input generators.
//
// DQMC_IN_U8 tables are packed to bits on the device (on ∪ dc, the only
// don't-care semantics the reference can express: TruthTable.from_bools(n,
// v != 0), ternary.py:210-218). The generators restate the reference's frozen
// counter generator (ttio.py:331-378) and the survey's config-3 S-box table
// (SURVEY.md §8(d)); k_weight_keys gives the CLI listing order (cli.py:131-138).
#include <cub/device/device_radix_sort.cuh>

#include "dqmc_internal.cuh"

namespace dqmc {
namespace {

// DQMC_IN_U8 -> 32-bit truth-table words (on ∪ dc, ternary.py:210-218), n >= 5
__global__ void k_u8_to_words(const uint8_t *__restrict__ v, uint32_t *__restrict__ out, int64_t nwords) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = (gridDim.x * (int64_t)blockDim.x) >> 5;
    for (int64_t w = warp; w < nwords; w += nwarps) {
        const unsigned bits = __ballot_sync(0xffffffffu, v[w * 32 + lane] != 0);
        if (lane == 0) out[w] = bits;
    }
}

// n < 5: pad with dummy variables n+1..5 (primes of f' = primes of f with '*'
// appended, rank shifted by 3^5 - 3^n): the 2^n-bit table is replicated.
__global__ void k_pad_small(const void *in, int kind, int n, uint32_t *out) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    uint32_t pat = 0;
    const int npts = 1 << n;
    for (int x = 0; x < npts; x++) {
        int bit;
        if (kind == DQMC_IN_U8)
            bit = ((const uint8_t *)in)[x] != 0;
        else
            bit = (int)((((const uint64_t *)in)[0] >> x) & 1ull);
        pat |= (uint32_t)bit << x;
    }
    uint32_t w = 0;
    for (int p = 0; p < 32; p++) w |= ((pat >> (p % npts)) & 1u) << p;
    out[0] = w;
}

// splitmix64 finaliser (ttio.py:331-338)
__device__ __forceinline__ uint64_t mix64(uint64_t x) {
    x ^= x >> 30;
    x *= 0xBF58476D1CE4E5B9ull;
    x ^= x >> 27;
    x *= 0x94D049BB133111EBull;
    x ^= x >> 31;
    return x;
}

// three-way generator: value of point x from the frozen
// counter generator mix(seed + (x+1)*GAMMA) >> 11 (ttio.py:341-343, 365-374)
__global__ void k_gen3(uint8_t *__restrict__ out, int64_t x0, int64_t npts, uint64_t seed, uint64_t t_on,
                       uint64_t t_any) {
    const int64_t stride = gridDim.x * (int64_t)blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < npts; i += stride) {
        const uint64_t x = (uint64_t)(x0 + i);
        const uint64_t u = mix64(seed + (x + 1) * 0x9E3779B97F4A7C15ull) >> 11;
        out[i] = u < t_on ? 1 : (u < t_any ? 2 : 0);
    }
}

// config 3 S-box table: one CTA of 1024 threads ranks the 1024 generator
// values (stable: ties by index), P[rank(i)] = i, then clears v[x | P(x) << 10]
// (the table was set to 1 beforehand).
__global__ void __launch_bounds__(1024) k_sbox(uint8_t *__restrict__ v, uint64_t seed) {
    __shared__ uint64_t val[1024];
    __shared__ uint16_t perm[1024];
    const int i = threadIdx.x;
    val[i] = mix64(seed + ((uint64_t)i + 1) * 0x9E3779B97F4A7C15ull);
    __syncthreads();
    const uint64_t me = val[i];
    int rank = 0;
    for (int j = 0; j < 1024; j++) {
        const uint64_t o = val[j];
        rank += (o < me) || (o == me && j < i);
    }
    perm[rank] = (uint16_t)i;
    __syncthreads();
    v[i | ((int)perm[i] << 10)] = 0;
}

// wildcard count of every rank (ternary.py:139-146), stored as the sort key
// n - weight so an ascending stable radix sort yields weight-descending order
// with ranks ascending inside each weight (cli.py:134-135 ordering).
__global__ void k_weight_keys(const int64_t *__restrict__ ranks, int64_t count, int n, uint8_t *__restrict__ keys) {
    const int64_t stride = gridDim.x * (int64_t)blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += stride) {
        uint64_t r = (uint64_t)ranks[i];
        int w = 0;
        for (int k = 0; k < n; k++) {
            const uint64_t q = __umul64hi(r, 0xAAAAAAAAAAAAAAABull) >> 1;  // r / 3
            w += (r - 3 * q) == 2;
            r = q;
        }
        keys[i] = (uint8_t)(n - w);
    }
}

}  // namespace

// input conversion to 32-bit truth-table words for n >= 5 (or the padded word)
int input_words(const void *in, int kind, int n, const uint32_t **tt32, cudaStream_t s) {
    int rc;
    if (n < 5) {
        if ((rc = grow(g_eng.tt_tmp, g_eng.tt_tmp_cap, 256, 1))) return rc;
        k_pad_small<<<1, 32, 0, s>>>(in, kind, n, g_eng.tt_tmp);
        CK_LAUNCH();
        *tt32 = g_eng.tt_tmp;
    } else if (kind == DQMC_IN_U8) {
        const int64_t nw = 1ll << (n - 5);
        if ((rc = grow(g_eng.tt_tmp, g_eng.tt_tmp_cap, (size_t)nw * 4, 1))) return rc;
        const int grid = (int)std::min<int64_t>((nw * 32 + 255) / 256, 148ll * 32);
        k_u8_to_words<<<grid, 256, 0, s>>>((const uint8_t *)in, g_eng.tt_tmp, nw);
        CK_LAUNCH();
        *tt32 = g_eng.tt_tmp;
    } else {
        *tt32 = (const uint32_t *)in;  // LE uint64 words viewed as uint32 words
    }
    return DQMC_OK;
}

}  // namespace dqmc

using namespace dqmc;

extern "C" {

int dqmc_gen3_range_device(uint8_t *values_dev, int64_t x0, int64_t count, double p_on, double p_dc, uint64_t seed,
                           void *stream) {
    int rc;
    if (!values_dev || x0 < 0 || count < 0) return set_err(DQMC_ERR_INVALID, "bad generator range");
    std::lock_guard<std::mutex> lk(g_mu);
    if ((rc = ensure_device())) return rc;
    cudaStream_t s = (cudaStream_t)stream;  // 0 = the legacy default stream (CUDA convention)
    // int(p * 2^53) as Python computes it (float64 product, truncation)
    const uint64_t t_on = (uint64_t)(p_on * 9007199254740992.0);
    const uint64_t t_any = (uint64_t)((p_on + p_dc) * 9007199254740992.0);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((count + 255) / 256, 148ll * 64));
    if (count) k_gen3<<<grid, 256, 0, s>>>(values_dev, x0, count, seed, t_on, t_any);
    CK_LAUNCH();
    CK(cudaStreamSynchronize(s));
    return DQMC_OK;
}

int dqmc_gen3_device(uint8_t *values_dev, int n, double p_on, double p_dc, uint64_t seed, void *stream) {
    int rc;
    if ((rc = validate(n, 0))) return rc;
    return dqmc_gen3_range_device(values_dev, 0, 1ll << n, p_on, p_dc, seed, stream);
}
int dqmc_gen_sbox_device(uint8_t *values_dev, uint64_t seed, void *stream) {
    int rc;
    if (!values_dev) return set_err(DQMC_ERR_INVALID, "null output");
    std::lock_guard<std::mutex> lk(g_mu);
    if ((rc = ensure_device())) return rc;
    cudaStream_t s = (cudaStream_t)stream;
    CK(cudaMemsetAsync(values_dev, 1, (size_t)1 << 20, s));
    k_sbox<<<1, 1024, 0, s>>>(values_dev, seed);
    CK_LAUNCH();
    CK(cudaStreamSynchronize(s));
    return DQMC_OK;
}

int dqmc_gen_sbox_host(uint8_t *values_host, uint64_t seed) {
    int rc;
    if (!values_host) return set_err(DQMC_ERR_INVALID, "null output");
    {
        std::lock_guard<std::mutex> lk(g_mu);
        if ((rc = ensure_device())) return rc;
        if ((rc = grow(g_eng.in_tmp, g_eng.in_tmp_cap, (size_t)1 << 20, 1))) return rc;
    }
    if ((rc = dqmc_gen_sbox_device((uint8_t *)g_eng.in_tmp, seed, g_eng.stream))) return rc;
    CK(cudaMemcpy(values_host, g_eng.in_tmp, (size_t)1 << 20, cudaMemcpyDeviceToHost));
    return DQMC_OK;
}

int dqmc_gen3_host(uint8_t *values_host, int n, double p_on, double p_dc, uint64_t seed) {
    int rc;
    if ((rc = validate(n, 0))) return rc;
    if (!values_host) return set_err(DQMC_ERR_INVALID, "null output");
    {
        std::lock_guard<std::mutex> lk(g_mu);
        if ((rc = ensure_device())) return rc;
        if ((rc = grow(g_eng.in_tmp, g_eng.in_tmp_cap, (size_t)1 << n, 1))) return rc;
    }
    if ((rc = dqmc_gen3_range_device((uint8_t *)g_eng.in_tmp, 0, 1ll << n, p_on, p_dc, seed, g_eng.stream))) return rc;
    CK(cudaMemcpy(values_host, g_eng.in_tmp, (size_t)1 << n, cudaMemcpyDeviceToHost));
    return DQMC_OK;
}

int dqmc_order_by_weight(const int64_t *ranks_host, int64_t count, int n, int64_t *out_host) {
    int rc;
    if ((rc = validate(n, 0))) return rc;
    if (count < 0 || (count && (!ranks_host || !out_host))) return set_err(DQMC_ERR_INVALID, "bad arguments");
    if (count == 0) return DQMC_OK;
    std::lock_guard<std::mutex> lk(g_mu);
    if ((rc = ensure_device())) return rc;
    cudaStream_t s = g_eng.stream;
    int64_t *r_in = nullptr, *r_out = nullptr;
    uint8_t *k_in = nullptr, *k_out = nullptr;
    void *tmp = nullptr;
    size_t tmpb = 0;
    CK(cudaMalloc(&r_in, (size_t)count * 8));
    CK(cudaMalloc(&r_out, (size_t)count * 8));
    CK(cudaMalloc(&k_in, (size_t)count));
    CK(cudaMalloc(&k_out, (size_t)count));
    CK(cudaMemcpyAsync(r_in, ranks_host, (size_t)count * 8, cudaMemcpyHostToDevice, s));
    const int grid = (int)std::min<int64_t>((count + 255) / 256, 148ll * 32);
    k_weight_keys<<<grid, 256, 0, s>>>(r_in, count, n, k_in);
    CK_LAUNCH();
    CK(cub::DeviceRadixSort::SortPairs(nullptr, tmpb, k_in, k_out, r_in, r_out, (int)count, 0, 8, s));
    CK(cudaMalloc(&tmp, tmpb));
    CK(cub::DeviceRadixSort::SortPairs(tmp, tmpb, k_in, k_out, r_in, r_out, (int)count, 0, 8, s));
    CK(cudaMemcpyAsync(out_host, r_out, (size_t)count * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    cudaFree(r_in);
    cudaFree(r_out);
    cudaFree(k_in);
    cudaFree(k_out);
    cudaFree(tmp);
    return DQMC_OK;
}

}  // extern "C"
