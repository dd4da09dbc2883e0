// Host-side cost of producing result std::vectors on this machine: value-initialised allocation
// (4 KB page faults), the same with MADV_HUGEPAGE before the first touch, and the copy into them.
// Build: g++ -std=c++20 -O2 -pthread tools/alloc_probe.cpp -o tools/alloc_probe
#include <sys/mman.h>

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

static double now_ms() {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

static std::vector<double> make(size_t n, bool huge) {
    std::vector<double> v;
    v.reserve(n);
    if (huge) {
        const uintptr_t a = (reinterpret_cast<uintptr_t>(v.data()) + (2u << 20) - 1) & ~uintptr_t((2u << 20) - 1);
        const uintptr_t e = (reinterpret_cast<uintptr_t>(v.data() + n)) & ~uintptr_t((2u << 20) - 1);
        if (e > a) madvise(reinterpret_cast<void*>(a), e - a, MADV_HUGEPAGE);
    }
    v.resize(n);
    return v;
}

int main() {
    const size_t n = size_t(1) << 21;  // 16.8 MB, one config-2 column
    std::vector<double> src(n, 1.0);
    for (int huge = 0; huge < 2; ++huge)
        for (int threads : {1, 4}) {
            double best = 1e30, best_cp = 1e30;
            for (int rep = 0; rep < 6; ++rep) {
                std::vector<std::vector<double>> cols(4);
                const double t0 = now_ms();
                std::vector<std::thread> team;
                for (int w = 0; w < threads; ++w)
                    team.emplace_back([&, w] {
                        for (int k = w; k < 4; k += threads) cols[k] = make(n, huge);
                    });
                for (auto& t : team) t.join();
                const double t1 = now_ms();
                for (int k = 0; k < 4; ++k) std::memcpy(cols[k].data(), src.data(), n * 8);
                const double t2 = now_ms();
                best = std::min(best, t1 - t0);
                best_cp = std::min(best_cp, t2 - t1);
            }
            std::printf("{\"huge\": %d, \"threads\": %d, \"alloc_4x16.8MB_ms\": %.2f, \"copy_1thread_ms\": %.2f}\n", huge,
                        threads, best, best_cp);
        }
    FILE* f = std::fopen("/sys/kernel/mm/transparent_hugepage/enabled", "r");
    char buf[256] = {0};
    if (f) {
        if (!std::fgets(buf, sizeof buf, f)) buf[0] = 0;
        std::fclose(f);
    }
    std::printf("{\"thp\": \"%s\"}\n", std::strtok(buf, "\n"));
}
