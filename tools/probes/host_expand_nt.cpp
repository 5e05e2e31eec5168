// Host probe: the host half of a packed rank transfer. Expands rank-ordered
// uint32 tile offsets + per-tile first ranks into int64 ranks with T threads,
// three ways: plain stores, AVX2 and AVX-512 non-temporal stores (no
// read-for-ownership of the 8-byte output). Also the raw NT memset rate.
// g++ -O3 -pthread -o host_expand_nt host_expand_nt.cpp && ./host_expand_nt 16
#include <immintrin.h>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

static void expand_plain(const uint32_t *off, int64_t *out, int64_t a, int64_t b, int64_t base) {
    for (int64_t i = a; i < b; i++) out[i] = base + off[i];
}
__attribute__((target("avx2"))) static void expand_avx2(const uint32_t *off, int64_t *out, int64_t a, int64_t b,
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
__attribute__((target("avx512f"))) static void expand_avx512(const uint32_t *off, int64_t *out, int64_t a, int64_t b,
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

int main(int argc, char **argv) {
    const int64_t n = 210000000, ntiles = 531441;
    const int T = argc > 1 ? atoi(argv[1]) : 16;
    printf("hw threads %u, avx2 %d, avx512f %d\n", std::thread::hardware_concurrency(), __builtin_cpu_supports("avx2"),
           __builtin_cpu_supports("avx512f"));
    uint32_t *off = (uint32_t *)aligned_alloc(4096, n * 4);
    std::vector<int64_t> pos(ntiles + 1);
    for (int64_t t = 0; t <= ntiles; t++) pos[t] = n * t / ntiles;
    for (int64_t i = 0; i < n; i++) off[i] = (uint32_t)(i % 531441);
    int64_t *out = (int64_t *)aligned_alloc(4096, n * 8);
    memset(out, 0, n * 8);
    for (int mode = 0; mode < 3; mode++) {
        if (mode == 1 && !__builtin_cpu_supports("avx2")) continue;
        if (mode == 2 && !__builtin_cpu_supports("avx512f")) continue;
        for (int rep = 0; rep < 3; rep++) {
            auto t0 = std::chrono::steady_clock::now();
            std::vector<std::thread> th;
            for (int k = 0; k < T; k++)
                th.emplace_back([&, k] {
                    const int64_t a = ntiles * k / T, b = ntiles * (k + 1) / T;
                    for (int64_t t = a; t < b; t++) {
                        const int64_t base = t * 531441;
                        if (mode == 0) expand_plain(off, out, pos[t], pos[t + 1], base);
                        if (mode == 1) expand_avx2(off, out, pos[t], pos[t + 1], base);
                        if (mode == 2) expand_avx512(off, out, pos[t], pos[t + 1], base);
                    }
                    _mm_sfence();
                });
            for (auto &x : th) x.join();
            double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            printf("expand mode %d (0 plain, 1 avx2 nt, 2 avx512 nt) T=%d: %.1f ms (%.1f GB/s written)\n", mode, T,
                   s * 1e3, n * 8 / s / 1e9);
        }
        int64_t bad = 0;
        for (int64_t t = 0; t < ntiles; t += 997)
            for (int64_t i = pos[t]; i < pos[t + 1]; i++) bad += out[i] != t * 531441 + off[i];
        printf("  check: %lld mismatches\n", (long long)bad);
    }
    return 0;
}
