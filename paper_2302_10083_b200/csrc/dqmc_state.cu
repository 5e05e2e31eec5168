// dqmc_state.cu — device-resident DenseState for any split h.
//
// The per-dimension operations of the reference engine, on the GPU, in the
// reference's own layout for every h (dense.py:127-397): 3^(n-h) blocks of
// block_bits_for(h) bits, little-endian uint64 words, padding zero.
//   k_state_load ......... load() scatter, dense.py:340-373 / index_to_rank
//   k_state_top_dim ...... DenseState._top_dim, dense.py:174-212
//   k_state_bottom_dim ... DenseState._bottom_dim_optimized, dense.py:216-243
//                          (per block; the flat-shift leakage of the reference
//                          lands only on masked-off bits, so it is identical)
//   k_state_count/emit ... extract_ranks, dense.py:376-397 (+ padding check)
// These are one streaming pass per dimension, like the reference; the fast
// fused plan (dqmc.cu) is what dense_prime_ranks runs.
#include <cub/device/device_scan.cuh>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <string>
#include <vector>

#include "../../include/dqmc.h"

namespace {

__host__ __device__ inline int64_t p3(int k) {
    int64_t r = 1;
    for (int i = 0; i < k; i++) r *= 3;
    return r;
}

int64_t block_bits_for(int h) {
    int64_t used = p3(h), b = 1;
    while (b < used) b <<= 1;
    return b < 64 ? 64 : b;
}

__global__ void k_state_load(const uint64_t *__restrict__ tt, int n, int64_t used, int64_t bb,
                             unsigned long long *__restrict__ words) {
    const int64_t npts = 1ll << n;
    const int64_t stride = gridDim.x * (int64_t)blockDim.x;
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < npts; x += stride) {
        if (!((tt[x >> 6] >> (x & 63)) & 1ull)) continue;
        int64_t r = 0, p = 1;
        for (int i = 0; i < n; i++, p *= 3)
            if ((x >> i) & 1) r += p;
        const int64_t flat = (r / used) * bb + r % used;
        atomicOr(words + (flat >> 6), 1ull << (flat & 63));
    }
}

// op 0 MERGE: u |= s & t; op 1 REDUCE: s &= ~u, t &= ~u (merge/reduce_triple)
__global__ void k_state_top_dim(uint64_t *__restrict__ w, int64_t groups, int64_t inner, int op) {
    const int64_t total = groups * inner;
    const int64_t stride = gridDim.x * (int64_t)blockDim.x;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total; q += stride) {
        const int64_t g = q / inner, c = q % inner;
        uint64_t *s = w + g * 3 * inner + c;
        uint64_t *t = s + inner, *u = t + inner;
        if (op == 0) {
            *u |= *s & *t;
        } else {
            const uint64_t nu = ~*u;
            *s &= nu;
            *t &= nu;
        }
    }
}

__device__ inline uint64_t shr_w(const uint64_t *v, int64_t wpb, int64_t k, int64_t s) {
    const int64_t q = s >> 6, r = s & 63;
    const uint64_t lo = (k + q < wpb) ? v[k + q] : 0ull;
    const uint64_t hi = (k + q + 1 < wpb) ? v[k + q + 1] : 0ull;
    return r ? (lo >> r) | (hi << (64 - r)) : lo;
}

__device__ inline uint64_t shl_w(const uint64_t *v, int64_t k, int64_t s) {
    const int64_t q = s >> 6, r = s & 63;
    const uint64_t hi = (k - q >= 0) ? v[k - q] : 0ull;
    const uint64_t lo = (k - q - 1 >= 0) ? v[k - q - 1] : 0ull;
    return r ? (hi << r) | (lo >> (64 - r)) : hi;
}

// In-block dimension i (d = 3^(i-1)) on every block; masks = (3, wpb) digit
// masks of dim i (dense.py:70-88). Blocks of up to 4 words (h <= 5, every
// split the engine and the reference's defaults use) are copied to registers
// first (k_state_bottom_dim_reg), so shifted reads see the original block;
// wider blocks (h >= 6) work in a private scratch copy in global memory.
template <int W>
__global__ void k_state_bottom_dim_reg(uint64_t *__restrict__ w, int64_t blocks, int64_t d,
                                       const uint64_t *__restrict__ masks, int op) {
    const int64_t stride = gridDim.x * (int64_t)blockDim.x;
    for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < blocks; a += stride) {
        uint64_t *v = w + a * W;
        uint64_t o[W];
#pragma unroll
        for (int k = 0; k < W; k++) o[k] = v[k];
#pragma unroll
        for (int k = 0; k < W; k++) {
            if (op == 0) {
                v[k] = o[k] | (shl_w(o, k, 2 * d) & shl_w(o, k, d) & masks[2 * W + k]);
            } else {
                v[k] = o[k] & ~((shr_w(o, W, k, 2 * d) & masks[k]) | (shr_w(o, W, k, d) & masks[W + k]));
            }
        }
    }
}

__global__ void k_state_bottom_dim(uint64_t *__restrict__ w, uint64_t *__restrict__ tmp, int64_t blocks, int64_t wpb,
                                   int64_t d, const uint64_t *__restrict__ masks, int op) {
    const int64_t stride = gridDim.x * (int64_t)blockDim.x;
    for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < blocks; a += stride) {
        uint64_t *v = w + a * wpb;
        uint64_t *o = tmp + a * wpb;
        for (int64_t k = 0; k < wpb; k++) o[k] = v[k];
        const uint64_t *m0 = masks, *m1 = masks + wpb, *m2 = masks + 2 * wpb;
        for (int64_t k = 0; k < wpb; k++) {
            if (op == 0) {
                v[k] = o[k] | (shl_w(o, k, 2 * d) & shl_w(o, k, d) & m2[k]);
            } else {
                v[k] = o[k] & ~((shr_w(o, wpb, k, 2 * d) & m0[k]) | (shr_w(o, wpb, k, d) & m1[k]));
            }
        }
    }
}

__device__ inline uint64_t pad_mask(int64_t k, int64_t used) {
    const int64_t lo = k * 64;
    if (lo >= used) return ~0ull;
    if (lo + 64 <= used) return 0ull;
    return ~0ull << (used - lo);
}

__global__ void k_state_count(const uint64_t *__restrict__ w, int64_t nw, int64_t wpb, int64_t used,
                              int32_t *__restrict__ cnt, int *bad) {
    const int64_t stride = gridDim.x * (int64_t)blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nw; i += stride) {
        const uint64_t x = w[i];
        if (x & pad_mask(i % wpb, used)) *bad = 1;
        cnt[i] = __popcll(x);
    }
}

__global__ void k_state_emit(const uint64_t *__restrict__ w, int64_t nw, int64_t bb, int64_t used,
                             const int64_t *__restrict__ pos, int64_t *__restrict__ out) {
    const int64_t stride = gridDim.x * (int64_t)blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nw; i += stride) {
        uint64_t x = w[i];
        int64_t o = pos[i];
        while (x) {
            const int b = __ffsll((long long)x) - 1;
            x &= x - 1;
            const int64_t flat = i * 64 + b;
            out[o++] = (flat / bb) * used + flat % bb;
        }
    }
}

__global__ void k_state_cmp(const uint64_t *__restrict__ a, const uint64_t *__restrict__ b, int64_t nw, int *diff) {
    const int64_t stride = gridDim.x * (int64_t)blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nw; i += stride)
        if (a[i] != b[i]) *diff = 1;
}

}  // namespace
extern "C" void dqmc_internal_set_error(const char *m);
namespace {

int fail(int code, const std::string &m) {
    dqmc_internal_set_error(m.c_str());
    return code;
}

#define SCK(call)                                                                                          \
    do {                                                                                                   \
        cudaError_t e_ = (call);                                                                           \
        if (e_ != cudaSuccess) return fail(DQMC_ERR_CUDA, std::string(#call ": ") + cudaGetErrorString(e_)); \
    } while (0)

int grid_for(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148ll * 32)); }

}  // namespace

struct dqmc_state {
    int n, h;
    int64_t bb, wpb, used, blocks, nw;
    uint64_t *words;   // device
    uint64_t *tmp;     // device scratch for bottom dims
    uint64_t *masks;   // device (3, h, wpb)
};

extern "C" {

int dqmc_state_create(int n, int h, uint64_t mem_cap, dqmc_state_t **out) {
    if (!out) return fail(DQMC_ERR_INVALID, "null output");
    *out = nullptr;
    if (n < 1 || n > 31) return fail(DQMC_ERR_INVALID, "variable count must be in 1..31, got " + std::to_string(n));
    if (h < 1 || h > n) return fail(DQMC_ERR_INVALID, "split must be in 1.." + std::to_string(n) + ", got " + std::to_string(h));
    const int64_t bb = block_bits_for(h), blocks = p3(n - h);
    const uint64_t need = (uint64_t)blocks * bb / 8;
    if (mem_cap && need > mem_cap) {
        char buf[256];
        snprintf(buf, sizeof buf, "dense state needs %llu bytes (%lld blocks of %lld bits), exceeding the cap of %llu bytes",
                 (unsigned long long)need, (long long)blocks, (long long)bb, (unsigned long long)mem_cap);
        return fail(DQMC_ERR_RESOURCE, buf);
    }
    int cnt = 0;
    if (cudaGetDeviceCount(&cnt) != cudaSuccess || cnt == 0) {
        (void)cudaGetLastError();
        return fail(DQMC_ERR_NODEVICE, "no CUDA device visible: libdqmc has no CPU fallback");
    }
    dqmc_state_t *st = new dqmc_state_t();
    st->n = n;
    st->h = h;
    st->bb = bb;
    st->wpb = bb / 64;
    st->used = p3(h);
    st->blocks = blocks;
    st->nw = blocks * st->wpb;
    // blocks wider than 4 words (h >= 6) need a scratch copy for the in-block dims
    const bool scratch = st->wpb > 4;
    st->tmp = nullptr;
    if (cudaMalloc(&st->words, (size_t)st->nw * 8) != cudaSuccess ||
        (scratch && cudaMalloc(&st->tmp, (size_t)st->nw * 8) != cudaSuccess) ||
        cudaMalloc(&st->masks, (size_t)3 * h * st->wpb * 8) != cudaSuccess) {
        (void)cudaGetLastError();
        dqmc_state_free(st);
        return fail(DQMC_ERR_RESOURCE,
                    "device allocation of " + std::to_string(need * (scratch ? 2 : 1)) + " bytes failed");
    }
    // digit masks (dense.py:70-88): masks[(i-1)][d][k]
    std::vector<uint64_t> m((size_t)3 * h * st->wpb, 0);
    for (int i = 1; i <= h; i++)
        for (int64_t pos = 0; pos < st->used; pos++) {
            const int d = (int)((pos / p3(i - 1)) % 3);
            m[((size_t)(i - 1) * 3 + d) * st->wpb + pos / 64] |= 1ull << (pos % 64);
        }
    SCK(cudaMemcpy(st->masks, m.data(), m.size() * 8, cudaMemcpyHostToDevice));
    SCK(cudaMemset(st->words, 0, (size_t)st->nw * 8));
    *out = st;
    return DQMC_OK;
}

void dqmc_state_free(dqmc_state_t *st) {
    if (!st) return;
    cudaFree(st->words);
    cudaFree(st->tmp);
    cudaFree(st->masks);
    delete st;
}

int dqmc_state_info(const dqmc_state_t *st, int64_t *out5) {
    if (!st || !out5) return fail(DQMC_ERR_INVALID, "null pointer");
    out5[0] = st->n;
    out5[1] = st->h;
    out5[2] = st->bb;
    out5[3] = st->blocks;
    out5[4] = st->nw;
    return DQMC_OK;
}

int dqmc_state_load_tt(dqmc_state_t *st, const uint64_t *tt_words_host) {
    if (!st || !tt_words_host) return fail(DQMC_ERR_INVALID, "null pointer");
    const int64_t ntw = std::max<int64_t>(1, (1ll << st->n) / 64);
    uint64_t *d_tt = nullptr;
    SCK(cudaMalloc(&d_tt, (size_t)ntw * 8));
    SCK(cudaMemcpy(d_tt, tt_words_host, (size_t)ntw * 8, cudaMemcpyHostToDevice));
    SCK(cudaMemset(st->words, 0, (size_t)st->nw * 8));
    k_state_load<<<grid_for(1ll << st->n), 256>>>(d_tt, st->n, st->used, st->bb, (unsigned long long *)st->words);
    SCK(cudaGetLastError());
    SCK(cudaDeviceSynchronize());
    cudaFree(d_tt);
    return DQMC_OK;
}

int dqmc_state_set_words(dqmc_state_t *st, const uint64_t *words, uint64_t nwords) {
    if (!st || !words || (int64_t)nwords != st->nw) return fail(DQMC_ERR_INVALID, "state size mismatch");
    SCK(cudaMemcpy(st->words, words, nwords * 8, cudaMemcpyHostToDevice));
    return DQMC_OK;
}

int dqmc_state_get_words(const dqmc_state_t *st, uint64_t *words, uint64_t nwords) {
    if (!st || !words || (int64_t)nwords != st->nw) return fail(DQMC_ERR_INVALID, "state size mismatch");
    SCK(cudaMemcpy(words, st->words, nwords * 8, cudaMemcpyDeviceToHost));
    return DQMC_OK;
}

// dense.py:296-315. Returns block-triple counts for top dims (3^(n-h-1)), -1 for bottom dims.
int dqmc_state_run_pass(dqmc_state_t *st, int op, const int *dims, int ndims, int64_t *counts) {
    if (!st) return fail(DQMC_ERR_INVALID, "null state");
    if (op != 0 && op != 1) return fail(DQMC_ERR_INVALID, "op must be 'merge' or 'reduce'");
    for (int k = 0; k < ndims; k++)
        if (dims[k] < 1 || dims[k] > st->n)
            return fail(DQMC_ERR_INVALID, "dimension " + std::to_string(dims[k]) + " out of range 1.." + std::to_string(st->n));
    for (int k = 0; k < ndims; k++) {
        const int dim = dims[k];
        if (dim > st->h) {
            const int64_t inner = p3(dim - st->h - 1) * st->wpb;
            const int64_t groups = st->nw / (3 * inner);
            k_state_top_dim<<<grid_for(groups * inner), 256>>>(st->words, groups, inner, op);
            if (counts) counts[k] = groups * inner / st->wpb;
        } else {
            const uint64_t *mk = st->masks + (size_t)(dim - 1) * 3 * st->wpb;
            if (st->wpb == 1)
                k_state_bottom_dim_reg<1><<<grid_for(st->blocks), 256>>>(st->words, st->blocks, p3(dim - 1), mk, op);
            else if (st->wpb == 2)
                k_state_bottom_dim_reg<2><<<grid_for(st->blocks), 256>>>(st->words, st->blocks, p3(dim - 1), mk, op);
            else if (st->wpb == 4)
                k_state_bottom_dim_reg<4><<<grid_for(st->blocks), 256>>>(st->words, st->blocks, p3(dim - 1), mk, op);
            else
                k_state_bottom_dim<<<grid_for(st->blocks), 256>>>(st->words, st->tmp, st->blocks, st->wpb, p3(dim - 1),
                                                                  mk, op);
            if (counts) counts[k] = -1;
        }
        SCK(cudaGetLastError());
    }
    SCK(cudaDeviceSynchronize());
    return DQMC_OK;
}

// dense.py:317-337: top merges, bottom merges then reduces, top reduces
int dqmc_state_run_merge_reduce(dqmc_state_t *st) {
    if (!st) return fail(DQMC_ERR_INVALID, "null state");
    std::vector<int> top, bottom;
    for (int d = st->h + 1; d <= st->n; d++) top.push_back(d);
    for (int d = 1; d <= st->h; d++) bottom.push_back(d);
    int rc;
    if (!top.empty() && (rc = dqmc_state_run_pass(st, 0, top.data(), (int)top.size(), nullptr))) return rc;
    if ((rc = dqmc_state_run_pass(st, 0, bottom.data(), (int)bottom.size(), nullptr))) return rc;
    if ((rc = dqmc_state_run_pass(st, 1, bottom.data(), (int)bottom.size(), nullptr))) return rc;
    if (!top.empty() && (rc = dqmc_state_run_pass(st, 1, top.data(), (int)top.size(), nullptr))) return rc;
    return DQMC_OK;
}

// dense.py:154-160
int dqmc_state_padding_zero(const dqmc_state_t *st, int *ok) {
    if (!st || !ok) return fail(DQMC_ERR_INVALID, "null pointer");
    int32_t *cnt = nullptr;
    int *bad = nullptr;
    SCK(cudaMalloc(&cnt, (size_t)st->nw * 4));
    SCK(cudaMalloc(&bad, 4));
    SCK(cudaMemset(bad, 0, 4));
    k_state_count<<<grid_for(st->nw), 256>>>(st->words, st->nw, st->wpb, st->used, cnt, bad);
    int hb = 0;
    SCK(cudaMemcpy(&hb, bad, 4, cudaMemcpyDeviceToHost));
    cudaFree(cnt);
    cudaFree(bad);
    *ok = !hb;
    return DQMC_OK;
}

// dense.py:376-397: ranks ascending; DQMC_ERR_INVALID (AssertionError in the
// reference) if a padding bit is set. ranks_host may be NULL to query the count.
int dqmc_state_extract(const dqmc_state_t *st, int64_t *ranks_host, int64_t cap, int64_t *count) {
    if (!st || !count) return fail(DQMC_ERR_INVALID, "null pointer");
    int32_t *cnt = nullptr;
    int64_t *pos = nullptr, *out = nullptr;
    int *bad = nullptr;
    void *tmp = nullptr;
    size_t tmpb = 0;
    SCK(cudaMalloc(&cnt, (size_t)st->nw * 4));
    SCK(cudaMalloc(&pos, (size_t)(st->nw + 1) * 8));
    SCK(cudaMalloc(&bad, 4));
    SCK(cudaMemset(bad, 0, 4));
    k_state_count<<<grid_for(st->nw), 256>>>(st->words, st->nw, st->wpb, st->used, cnt, bad);
    SCK(cub::DeviceScan::ExclusiveScan(nullptr, tmpb, cnt, pos, cub::Sum(), (int64_t)0, (int64_t)st->nw));
    SCK(cudaMalloc(&tmp, tmpb));
    SCK(cub::DeviceScan::ExclusiveScan(tmp, tmpb, cnt, pos, cub::Sum(), (int64_t)0, (int64_t)st->nw));
    int hb = 0;
    int64_t lastpos = 0;
    int32_t lastcnt = 0;
    SCK(cudaMemcpy(&hb, bad, 4, cudaMemcpyDeviceToHost));
    SCK(cudaMemcpy(&lastpos, pos + st->nw - 1, 8, cudaMemcpyDeviceToHost));
    SCK(cudaMemcpy(&lastcnt, cnt + st->nw - 1, 4, cudaMemcpyDeviceToHost));
    const int64_t total = lastpos + lastcnt;
    *count = total;
    int rc = DQMC_OK;
    if (hb) {
        rc = fail(DQMC_ERR_INVALID, "padding bit set in dense state");
    } else if (ranks_host && total > 0) {
        if (total > cap) {
            rc = fail(DQMC_ERR_INVALID, "rank buffer too small");
        } else {
            SCK(cudaMalloc(&out, (size_t)total * 8));
            k_state_emit<<<grid_for(st->nw), 256>>>(st->words, st->nw, st->bb, st->used, pos, out);
            SCK(cudaMemcpy(ranks_host, out, (size_t)total * 8, cudaMemcpyDeviceToHost));
        }
    }
    cudaFree(cnt);
    cudaFree(pos);
    cudaFree(bad);
    cudaFree(tmp);
    cudaFree(out);
    return rc;
}

int dqmc_state_equal(const dqmc_state_t *a, const dqmc_state_t *b, int *eq) {
    if (!a || !b || !eq) return fail(DQMC_ERR_INVALID, "null pointer");
    if (a->n != b->n || a->h != b->h) {
        *eq = 0;
        return DQMC_OK;
    }
    int *diff = nullptr;
    SCK(cudaMalloc(&diff, 4));
    SCK(cudaMemset(diff, 0, 4));
    k_state_cmp<<<grid_for(a->nw), 256>>>(a->words, b->words, a->nw, diff);
    int hd = 0;
    SCK(cudaMemcpy(&hd, diff, 4, cudaMemcpyDeviceToHost));
    cudaFree(diff);
    *eq = !hd;
    return DQMC_OK;
}

int dqmc_state_copy(const dqmc_state_t *src, dqmc_state_t **out) {
    int rc;
    if (!src) return fail(DQMC_ERR_INVALID, "null state");
    if ((rc = dqmc_state_create(src->n, src->h, 0, out))) return rc;
    SCK(cudaMemcpy((*out)->words, src->words, (size_t)src->nw * 8, cudaMemcpyDeviceToDevice));
    return DQMC_OK;
}

}  // extern "C"
