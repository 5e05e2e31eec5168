// Host half of the packed rank transfer (plain C++, no CUDA).
//
// The final stage leaves every prime as a 4-byte cell offset inside its C0
// tile, in rank order (k_reorder<uint32_t>, dqmc_final.cu). Large results
// cross PCIe in that form — half the bytes of the int64 ranks the reference
// returns (dense.py:376-397, np.int64) — and the host widens them while the
// next chunk is still on the wire:
//     rank(i) = tile_first_rank(t) + off32[i],   start[t] <= i < start[t+1]
// A small persistent pool of host threads does the widening with non-temporal
// 64-byte stores (the 8-byte output is written once and not read here, so it
// should not be read for ownership first): AVX-512 or AVX2 when the CPU has
// them, plain stores otherwise. Measured on this pool's hosts by
// tools/probes/host_expand_nt.cpp.
#include <immintrin.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace dqmc {

namespace {

typedef void (*WidenFn)(const uint32_t *, int64_t *, int64_t, int64_t, int64_t);

void widen_plain(const uint32_t *off, int64_t *out, int64_t a, int64_t b, int64_t base) {
    for (int64_t i = a; i < b; i++) out[i] = base + off[i];
}

__attribute__((target("avx2"))) void widen_avx2(const uint32_t *off, int64_t *out, int64_t a, int64_t b,
                                                int64_t base) {
    int64_t i = a;
    for (; i < b && ((uintptr_t)(out + i) & 31); i++) out[i] = base + off[i];
    const __m256i vb = _mm256_set1_epi64x(base);
    for (; i + 4 <= b; i += 4) {
        const __m128i x = _mm_loadu_si128((const __m128i *)(off + i));
        _mm256_stream_si256((__m256i *)(out + i), _mm256_add_epi64(_mm256_cvtepu32_epi64(x), vb));
    }
    for (; i < b; i++) out[i] = base + off[i];
}

__attribute__((target("avx512f"))) void widen_avx512(const uint32_t *off, int64_t *out, int64_t a, int64_t b,
                                                     int64_t base) {
    int64_t i = a;
    for (; i < b && ((uintptr_t)(out + i) & 63); i++) out[i] = base + off[i];
    const __m512i vb = _mm512_set1_epi64(base);
    for (; i + 8 <= b; i += 8) {
        const __m256i x = _mm256_loadu_si256((const __m256i *)(off + i));
        _mm512_stream_si512((__m512i *)(out + i), _mm512_add_epi64(_mm512_cvtepu32_epi64(x), vb));
    }
    for (; i < b; i++) out[i] = base + off[i];
}

WidenFn pick_widen() {
    __builtin_cpu_init();
    if (__builtin_cpu_supports("avx512f")) return widen_avx512;
    if (__builtin_cpu_supports("avx2")) return widen_avx2;
    return widen_plain;
}

// Persistent workers: run(fn) calls fn(k) for k in [0, size) on the workers
// and the calling thread (which takes k = 0), and returns when all are done.
class Pool {
  public:
    explicit Pool(int n) : n_(std::max(1, n)) {
        for (int k = 1; k < n_; k++) th_.emplace_back([this, k] { loop(k); });
    }
    ~Pool() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
            gen_++;
        }
        cv_.notify_all();
        for (auto &t : th_) t.join();
    }
    int size() const { return n_; }
    void run(const std::function<void(int)> &fn) {
        if (n_ == 1) {
            fn(0);
            return;
        }
        {
            std::lock_guard<std::mutex> lk(mu_);
            fn_ = &fn;
            left_ = n_ - 1;
            gen_++;
        }
        cv_.notify_all();
        fn(0);
        std::unique_lock<std::mutex> lk(mu_);
        done_.wait(lk, [this] { return left_ == 0; });
        fn_ = nullptr;
    }

  private:
    void loop(int k) {
        uint64_t seen = 0;
        for (;;) {
            const std::function<void(int)> *fn;
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return gen_ != seen; });
                seen = gen_;
                if (stop_) return;
                fn = fn_;
            }
            (*fn)(k);
            {
                std::lock_guard<std::mutex> lk(mu_);
                if (--left_ == 0) done_.notify_one();
            }
        }
    }
    const int n_;
    std::vector<std::thread> th_;
    std::mutex mu_;
    std::condition_variable cv_, done_;
    const std::function<void(int)> *fn_ = nullptr;
    uint64_t gen_ = 0;
    int left_ = 0;
    bool stop_ = false;
};

std::mutex g_pool_mu;
Pool *g_pool = nullptr;
int g_threads = 0;  // 0: min(hardware threads, 16)

Pool &pool() {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    const unsigned hw = std::thread::hardware_concurrency();
    const int want = g_threads > 0 ? g_threads : (int)std::min(16u, std::max(1u, hw));
    if (!g_pool || g_pool->size() != want) {
        delete g_pool;
        g_pool = new Pool(want);
    }
    return *g_pool;
}

}  // namespace

// host threads of the widening pool (0 = default: min(hardware threads, 16)); returns the previous setting
int host_widen_threads(int n) {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    const int prev = g_threads;
    g_threads = std::max(0, std::min(n, 256));
    return prev;
}

// Widen tiles [t0, t1): out[i] = (t * tile_cells + rank_add) + off32[i] for
// start(t) <= i < start(t + 1), where start(t) = add + pos[t - t0] for t < t1
// and start(t1) = end. `pos` are the tiles' exclusive positions relative to
// `add` (the chunk's device scan); out and off32 are indexed by the absolute
// position i. The output range is cut into 64-byte-aligned pieces, one per
// thread (no output cache line is shared by two threads).
void host_widen(const uint32_t *off32, int64_t *out, const int64_t *pos, int64_t add, int64_t end, int64_t t0,
                int64_t t1, int64_t tile_cells, int64_t rank_add) {
    static const WidenFn widen = pick_widen();
    if (t1 <= t0) return;
    const int64_t lo = add + pos[0], hi = end;
    if (hi <= lo) return;
    const int64_t nt = t1 - t0;
    auto piece = [&](int64_t a, int64_t b) {
        if (b <= a) return;
        // first tile whose range reaches past a: the last t with start(t) <= a
        int64_t t = std::upper_bound(pos, pos + nt, a - add) - pos - 1;
        for (; t < nt; t++) {
            const int64_t s = add + pos[t], e = t + 1 < nt ? add + pos[t + 1] : hi;
            if (s >= b) break;
            const int64_t x = std::max(a, s), y = std::min(b, e);
            if (y > x) widen(off32, out, x, y, (t0 + t) * tile_cells + rank_add);
        }
        _mm_sfence();
    };
    Pool &pl = pool();
    const int W = (hi - lo) < (1 << 16) ? 1 : pl.size();
    if (W == 1) {
        piece(lo, hi);
        return;
    }
    pl.run([&](int k) {
        // cut points on 8-entry (64-byte) boundaries of the output array
        auto cut = [&](int j) {
            if (j <= 0) return lo;
            if (j >= W) return hi;
            const int64_t c = lo + (hi - lo) * j / W;
            const int64_t al = c - (int64_t)(((uintptr_t)(out + c) & 63) / 8);
            return std::max(lo, std::min(hi, al));
        };
        piece(cut(k), cut(k + 1));
    });
}

}  // namespace dqmc
