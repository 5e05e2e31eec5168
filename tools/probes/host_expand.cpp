// Host probe: expand rank-ordered uint32 tile offsets + per-tile first ranks
// into int64 ranks with T threads (the host half of a compressed D2H), and
// the plain memcpy / memset rates of this host for comparison.
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

int main(int argc, char **argv) {
    const int64_t n = 210000000, ntiles = 531441;
    const int T = argc > 1 ? atoi(argv[1]) : 16;
    std::vector<uint32_t> off(n);
    std::vector<int64_t> pos(ntiles + 1), r0(ntiles);
    for (int64_t t = 0; t <= ntiles; t++) pos[t] = n * t / ntiles;
    for (int64_t t = 0; t < ntiles; t++) r0[t] = t * 531441;
    for (int64_t i = 0; i < n; i++) off[i] = (uint32_t)(i % 531441);
    int64_t *out = (int64_t *)aligned_alloc(4096, n * 8);
    memset(out, 0, n * 8);
    for (int rep = 0; rep < 3; rep++) {
        auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> th;
        for (int k = 0; k < T; k++)
            th.emplace_back([&, k] {
                const int64_t a = ntiles * k / T, b = ntiles * (k + 1) / T;
                for (int64_t t = a; t < b; t++) {
                    const int64_t base = r0[t];
                    for (int64_t i = pos[t]; i < pos[t + 1]; i++) out[i] = base + off[i];
                }
            });
        for (auto &x : th) x.join();
        auto t1 = std::chrono::steady_clock::now();
        double s = std::chrono::duration<double>(t1 - t0).count();
        printf("expand T=%d: %.1f ms (%.1f GB/s written)\n", T, s * 1e3, n * 8 / s / 1e9);
    }
    int64_t *dst = (int64_t *)aligned_alloc(4096, n * 8);
    memset(dst, 0, n * 8);
    for (int rep = 0; rep < 2; rep++) {
        auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> th;
        for (int k = 0; k < T; k++)
            th.emplace_back([&, k] { memcpy(dst + n * k / T, out + n * k / T, (n * (k + 1) / T - n * k / T) * 8); });
        for (auto &x : th) x.join();
        double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        printf("memcpy T=%d: %.1f ms (%.1f GB/s)\n", T, s * 1e3, n * 8 / s / 1e9);
    }
    printf("check %lld\n", (long long)(out[n - 1] + dst[n / 2]));
    return 0;
}
