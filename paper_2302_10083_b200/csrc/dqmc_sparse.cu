// dqmc_sparse.cu — the sparse engine on the GPU.
//
// Restates the reference's level walk (/root/reference/pkg/src/implicants/
// sparse.py:80-314) with device hash sets: cubes are packed 2 bits per
// variable (variable i in bits 2i-2..2i-1: 00 = 0, 01 = 1, 10 = *;
// ternary.py:83-103), a slot is payload | OCCUPIED (bit 62) | DELETED (bit
// 63), so an all-zero slot is empty (sparse.py:1-8). Level w holds every
// implicant with w stars:
//   k_sp_seed      level 0 = the support points (sparse.py:288-296)
//   k_sp_generate  every stored cube (tombstoned ones included) proposes
//                  the merge at position i when its digit i is 0, no star
//                  sits before i, and the digit-1 sibling is stored: each
//                  level-(w+1) implicant exactly once (sparse.py:242-266)
//   k_sp_insert    level w+1 = the candidates (distinct by construction)
//   k_sp_mark      tombstone both specialisations of every star of every
//                  candidate in level w (sparse.py:269-285)
//   k_sp_emit      the live (untombstoned) cubes of level w are prime
// then one radix sort of the ranks (the reference sorts too, sparse.py:306).
// Linear probing from splitmix64(payload) (sparse.py:37-45) with atomicCAS
// inserts; a table is a power of two >= 2 x entries (load <= 1/2) and at
// least 64 slots, refused before allocation above the memory cap with the
// reference's message (sparse.py:105-111). Work scales with the implicants,
// not 3^n: the right engine at low density.
#include <cub/device/device_radix_sort.cuh>

#include "dqmc_internal.cuh"

namespace dqmc {
namespace {

constexpr uint64_t kOccupied = 1ull << 62;
constexpr uint64_t kDeleted = 1ull << 63;
constexpr uint64_t kPayload = kOccupied - 1;
constexpr int64_t kMinTable = 64;

__device__ __forceinline__ uint64_t sp_mix(uint64_t x) {
    x ^= x >> 30;
    x *= 0xBF58476D1CE4E5B9ull;
    x ^= x >> 27;
    x *= 0x94D049BB133111EBull;
    x ^= x >> 31;
    return x;
}

// slot index of payload v, or -1 (include_deleted: tombstoned entries count)
__device__ __forceinline__ int64_t sp_find(const uint64_t *__restrict__ t, uint64_t mask, uint64_t v) {
    const uint64_t key = v | kOccupied;
    uint64_t p = sp_mix(v) & mask;
    while (true) {
        const uint64_t s = t[p];
        if ((s & ~kDeleted) == key) return (int64_t)p;
        if (s == 0) return -1;
        p = (p + 1) & mask;
    }
}

__device__ __forceinline__ void sp_insert(uint64_t *t, uint64_t mask, uint64_t v) {
    const unsigned long long key = v | kOccupied;
    uint64_t p = sp_mix(v) & mask;
    while (true) {
        const unsigned long long old = atomicCAS((unsigned long long *)(t + p), 0ull, key);
        if (old == 0 || (old & ~kDeleted) == key) return;
        p = (p + 1) & mask;
    }
}

// warp-aggregated append of `val` (lanes with `want`) at *count; writes only
// below cap (the host reruns with a larger buffer when *count > cap)
__device__ __forceinline__ void sp_append(bool want, uint64_t val, uint64_t *out, int64_t cap,
                                          unsigned long long *count) {
    const unsigned m = __ballot_sync(0xffffffffu, want);  // called by whole warps
    if (!m) return;
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(m) - 1;
    unsigned long long base = 0;
    if (lane == leader) base = atomicAdd(count, (unsigned long long)__popc(m));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (want) {
        const int64_t at = (int64_t)base + __popc(m & ((1u << lane) - 1u));
        if (at < cap) out[at] = val;
    }
}

// level 0: packed point of every set bit x (digit i = bit i of x)
__global__ void k_sp_seed(const uint64_t *__restrict__ tt, int n, uint64_t *t, uint64_t mask) {
    const int64_t npts = 1ll << n;
    const int64_t stride = gridDim.x * (int64_t)blockDim.x;
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < npts; x += stride) {
        if (!((tt[x >> 6] >> (x & 63)) & 1ull)) continue;
        uint64_t v = 0;
        for (int i = 0; i < n; i++) v |= (uint64_t)((x >> i) & 1) << (2 * i);
        sp_insert(t, mask, v);
    }
}

__global__ void k_sp_popcount(const uint64_t *__restrict__ tt, int64_t nwords, unsigned long long *count) {
    unsigned long long c = 0;
    const int64_t stride = gridDim.x * (int64_t)blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nwords; i += stride) c += __popcll(tt[i]);
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, c);
}

__global__ void k_sp_generate(const uint64_t *__restrict__ t, uint64_t mask, int64_t size, int n,
                              uint64_t *__restrict__ cand, int64_t cap, unsigned long long *count) {
    const int64_t stride = gridDim.x * (int64_t)blockDim.x;
    // warp-uniform trip counts so every append sees the whole warp
    const int64_t trips = (size + stride - 1) / stride;
    for (int64_t k = 0; k < trips; k++) {
        const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x + k * stride;
        const uint64_t slot = s < size ? t[s] : 0;
        const uint64_t v = slot & kPayload;
        bool alive = (slot & kOccupied) != 0;  // stored (tombstoned too) and no star seen yet
        for (int i = 0; i < n; i++) {
            if (!__any_sync(0xffffffffu, alive)) break;
            const uint64_t d = (v >> (2 * i)) & 3ull;
            const bool emit = alive && d == 0 && sp_find(t, mask, v | (1ull << (2 * i))) >= 0;
            sp_append(emit, v | (2ull << (2 * i)), cand, cap, count);
            alive = alive && d != 2;
        }
    }
}

__global__ void k_sp_insert(const uint64_t *__restrict__ vals, int64_t nvals, uint64_t *t, uint64_t mask) {
    const int64_t stride = gridDim.x * (int64_t)blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nvals; i += stride)
        sp_insert(t, mask, vals[i]);
}

__global__ void k_sp_mark(const uint64_t *__restrict__ cand, int64_t ncand, int n, uint64_t *t, uint64_t mask) {
    const int64_t stride = gridDim.x * (int64_t)blockDim.x;
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < ncand; c += stride) {
        const uint64_t m = cand[c];
        for (int i = 0; i < n; i++) {
            if (((m >> (2 * i)) & 3ull) != 2ull) continue;
            // star chunk 10 -> 00 (digit 0) and 01 (digit 1)
            for (uint64_t x = 2; x <= 3; x++) {
                const int64_t p = sp_find(t, mask, m ^ (x << (2 * i)));
                if (p >= 0) atomicOr((unsigned long long *)(t + p), (unsigned long long)kDeleted);
            }
        }
    }
}

// live cubes of a level -> int64 ranks (packed chunk i = digit of 3^i)
__global__ void k_sp_emit(const uint64_t *__restrict__ t, int64_t size, int n, int64_t *out, int64_t cap,
                          unsigned long long *count) {
    const int64_t stride = gridDim.x * (int64_t)blockDim.x;
    const int64_t trips = (size + stride - 1) / stride;
    for (int64_t k = 0; k < trips; k++) {
        const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x + k * stride;
        const uint64_t slot = s < size ? t[s] : 0;
        const bool live = (slot & kOccupied) && !(slot & kDeleted);
        int64_t r = 0;
        if (live) {
            int64_t p3 = 1;
            for (int i = 0; i < n; i++, p3 *= 3) r += (int64_t)((slot >> (2 * i)) & 3ull) * p3;
        }
        sp_append(live, (uint64_t)r, reinterpret_cast<uint64_t *>(out), cap, count);
    }
}

int grid_of(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)g_eng.num_sms * 16)); }

int64_t table_size(int64_t entries) {
    int64_t s = kMinTable;
    while (s < 2 * entries) s *= 2;
    return s;
}

struct DevBuf {
    void *p = nullptr;
    size_t cap = 0;  // bytes
    DevBuf() = default;
    DevBuf(const DevBuf &) = delete;
    DevBuf &operator=(const DevBuf &) = delete;
    ~DevBuf() { release(); }
    void release() {
        cudaFree(p);
        p = nullptr;
        cap = 0;
    }
    int ensure(size_t bytes) {
        if (bytes <= cap && p) return DQMC_OK;
        cudaFree(p);
        p = nullptr;
        cap = 0;
        cudaError_t e = cudaMalloc(&p, std::max<size_t>(bytes, 256));
        if (e != cudaSuccess) {
            (void)cudaGetLastError();
            return set_err(DQMC_ERR_RESOURCE, "device allocation of " + std::to_string(bytes) + " bytes failed");
        }
        cap = std::max<size_t>(bytes, 256);
        return DQMC_OK;
    }
};

struct SparseWork {
    DevBuf tt, ctr, tabA, tabB, cand, ranks, sorted, tmp;
};
SparseWork g_sp;

int refuse_table(int64_t size, uint64_t cap) {
    char buf[256];
    snprintf(buf, sizeof buf, "sparse level table needs %lld bytes (%lld slots), exceeding the cap of %llu bytes",
             (long long)(size * 8), (long long)size, (unsigned long long)cap);
    return set_err(DQMC_ERR_RESOURCE, buf);
}

int64_t read_count(unsigned long long *d, cudaStream_t s, int *rc) {
    unsigned long long h = 0;
    cudaError_t e = cudaMemcpyAsync(&h, d, 8, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) *rc = set_err(DQMC_ERR_CUDA, std::string("sparse count: ") + cudaGetErrorString(e));
    return (int64_t)h;
}

// the whole walk; ranks (ascending) into a pinned host buffer
int sparse_impl(const uint64_t *tt_host, int n, uint64_t mem_cap, dqmc_result_t *out) {
    cudaStream_t s = g_eng.stream;
    int rc = DQMC_OK;
    if (mem_cap == 0) {
        size_t fr = 0, tot = 0;
        CK(cudaMemGetInfo(&fr, &tot));
        mem_cap = (uint64_t)((double)fr * 0.75);
    }
    const int64_t nwords = std::max<int64_t>(1, (1ll << n) / 64);
    // grow-only buffers kept across calls (released by dqmc_release): no
    // cudaMalloc/cudaFree (device-wide syncs) on the steady-state path
    DevBuf &tt = g_sp.tt, &ctr = g_sp.ctr, &tabA = g_sp.tabA, &tabB = g_sp.tabB, &cand = g_sp.cand,
           &ranks = g_sp.ranks;
    if ((rc = tt.ensure((size_t)nwords * 8)) || (rc = ctr.ensure(64))) return rc;
    unsigned long long *cnt = (unsigned long long *)ctr.p;
    CK(cudaMemcpyAsync(tt.p, tt_host, (size_t)nwords * 8, cudaMemcpyHostToDevice, s));
    CK(cudaMemsetAsync(cnt, 0, 8, s));
    k_sp_popcount<<<grid_of(nwords), 256, 0, s>>>((const uint64_t *)tt.p, nwords, cnt);
    CK_LAUNCH();
    const int64_t npts = read_count(cnt, s, &rc);
    if (rc) return rc;
    int64_t size = table_size(npts);
    if ((uint64_t)size * 8 > mem_cap) return refuse_table(size, mem_cap);
    if ((rc = tabA.ensure((size_t)size * 8))) return rc;
    CK(cudaMemsetAsync(tabA.p, 0, (size_t)size * 8, s));
    k_sp_seed<<<grid_of(1ll << n), 256, 0, s>>>((const uint64_t *)tt.p, n, (uint64_t *)tabA.p, (uint64_t)(size - 1));
    CK_LAUNCH();
    DevBuf *cur = &tabA, *nxt = &tabB;
    int64_t ncap = std::max<int64_t>(npts, 1024), rcap = std::max<int64_t>(npts, 1024);
    int64_t total = 0;
    if ((rc = ranks.ensure((size_t)rcap * 8))) return rc;
    for (int level = 0; level <= n; level++) {
        const uint64_t mask = (uint64_t)(size - 1);
        // generate (rerun with a larger buffer on overflow: the table is read-only here)
        int64_t ncand = 0;
        for (int attempt = 0; attempt < 2; attempt++) {
            if ((rc = cand.ensure((size_t)ncap * 8))) return rc;
            CK(cudaMemsetAsync(cnt, 0, 8, s));
            k_sp_generate<<<grid_of(size), 256, 0, s>>>((const uint64_t *)cur->p, mask, size, n, (uint64_t *)cand.p,
                                                        ncap, cnt);
            CK_LAUNCH();
            ncand = read_count(cnt, s, &rc);
            if (rc) return rc;
            if (ncand <= ncap) break;
            ncap = ncand + ncand / 8 + 1024;
        }
        int64_t nsize = 0;
        if (ncand > 0) {
            nsize = table_size(ncand);
            if ((uint64_t)nsize * 8 > mem_cap) return refuse_table(nsize, mem_cap);
            if ((rc = nxt->ensure((size_t)nsize * 8))) return rc;
            CK(cudaMemsetAsync(nxt->p, 0, (size_t)nsize * 8, s));
            k_sp_insert<<<grid_of(ncand), 256, 0, s>>>((const uint64_t *)cand.p, ncand, (uint64_t *)nxt->p,
                                                       (uint64_t)(nsize - 1));
            CK_LAUNCH();
            k_sp_mark<<<grid_of(ncand), 256, 0, s>>>((const uint64_t *)cand.p, ncand, n, (uint64_t *)cur->p, mask);
            CK_LAUNCH();
        }
        // live cubes of this level are prime
        for (int attempt = 0; attempt < 2; attempt++) {
            CK(cudaMemsetAsync(cnt, 0, 8, s));
            k_sp_emit<<<grid_of(size), 256, 0, s>>>((const uint64_t *)cur->p, size, n, (int64_t *)ranks.p + total,
                                                    rcap - total, cnt);
            CK_LAUNCH();
            const int64_t got = read_count(cnt, s, &rc);
            if (rc) return rc;
            if (total + got <= rcap) {
                total += got;
                break;
            }
            // grow the rank buffer, keeping what is there
            DevBuf bigger;
            const int64_t ncap2 = (total + got) * 2 + 1024;
            if ((rc = bigger.ensure((size_t)ncap2 * 8))) return rc;
            if (total) CK(cudaMemcpyAsync(bigger.p, ranks.p, (size_t)total * 8, cudaMemcpyDeviceToDevice, s));
            std::swap(ranks.p, bigger.p);
            std::swap(ranks.cap, bigger.cap);
            rcap = ncap2;
        }
        if (ncand == 0) break;
        std::swap(cur, nxt);
        size = nsize;
    }
    // ascending ranks (one radix sort; the reference sorts too)
    out->count = total;
    out->ranks = nullptr;
    out->_owner = nullptr;
    if (total == 0) return DQMC_OK;
    DevBuf &sorted = g_sp.sorted, &tmp = g_sp.tmp;
    size_t tmpb = 0;
    if ((rc = sorted.ensure((size_t)total * 8))) return rc;
    int bits = 1;
    while (bits < 64 && (pow3l(std::min(n, 39)) >> bits) > 0) bits++;
    CK(cub::DeviceRadixSort::SortKeys(nullptr, tmpb, (const int64_t *)ranks.p, (int64_t *)sorted.p, total, 0, bits, s));
    if ((rc = tmp.ensure(tmpb))) return rc;
    CK(cub::DeviceRadixSort::SortKeys(tmp.p, tmpb, (const int64_t *)ranks.p, (int64_t *)sorted.p, total, 0, bits, s));
    PinnedBuf pb;  // from the engine's pinned pool (dqmc_free_result returns it)
    if ((rc = alloc_pinned((size_t)total, pb))) return rc;
    CK(cudaMemcpyAsync(pb.ptr, sorted.p, (size_t)total * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    out->ranks = pb.ptr;
    out->_owner = new PinnedBuf(pb);
    return DQMC_OK;
}

}  // namespace

void sparse_release() {
    for (DevBuf *b : {&g_sp.tt, &g_sp.ctr, &g_sp.tabA, &g_sp.tabB, &g_sp.cand, &g_sp.ranks, &g_sp.sorted, &g_sp.tmp})
        b->release();
}

}  // namespace dqmc

using namespace dqmc;

extern "C" {

int dqmc_sparse_primes_tt(const uint64_t *tt_words, int n, uint64_t mem_cap, dqmc_result_t *out) {
    if (!out) return set_err(DQMC_ERR_INVALID, "null result pointer");
    out->count = 0;
    out->ranks = nullptr;
    out->_owner = nullptr;
    int rc;
    if ((rc = validate(n, 0))) return rc;
    if (!tt_words) return set_err(DQMC_ERR_INVALID, "null input pointer");
    std::lock_guard<std::mutex> lk(g_mu);
    if ((rc = ensure_device())) return rc;
    if ((rc = ensure_attrs())) return rc;
    if ((rc = engine_begin(g_eng.stream))) return rc;
    if ((rc = sparse_impl(tt_words, n, mem_cap, out))) return rc;
    return engine_done(g_eng.stream);
}

}  // extern "C"
