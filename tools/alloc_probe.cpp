// Host allocation probe for the drop-in: cost of FrameBuffers-sized std::vector
// allocation (serial assign), parallel first touch, and memset of touched memory.
#include <chrono>
#include <cstdio>
#include <cstring>
#include <sys/mman.h>
#include <thread>
#include <vector>
int main() {
    using clk = std::chrono::steady_clock;
    auto ms = [](clk::time_point a) { return std::chrono::duration<double, std::milli>(clk::now() - a).count(); };
    const size_t n = 300ull << 20;
    for (int rep = 0; rep < 3; ++rep) {
        auto t = clk::now();
        { std::vector<double> v(n / 8, 0.0); }
        std::printf("vector assign 300MB: %.1f ms\n", ms(t));
        t = clk::now();
        char* p = static_cast<char*>(mmap(nullptr, n, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0));
        const int T = 16;
        std::vector<std::thread> th;
        for (int i = 0; i < T; ++i)
            th.emplace_back([=] { for (size_t o = n / T * i; o < n / T * (i + 1); o += 4096) p[o] = 0; });
        for (auto& x : th) x.join();
        std::printf("parallel first touch (16 thr): %.1f ms\n", ms(t));
        t = clk::now();
        std::memset(p, 1, n);
        std::printf("memset touched: %.1f ms\n", ms(t));
        munmap(p, n);
        t = clk::now();
        p = static_cast<char*>(mmap(nullptr, n, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0));
        madvise(p, n, MADV_HUGEPAGE);
        std::memset(p, 1, n);
        std::printf("madvise hugepage + memset: %.1f ms\n", ms(t));
        munmap(p, n);
    }
}
