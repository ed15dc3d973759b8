// Probe: the pooled closed-form partition (hoare_rewrite_par) against the
// single-thread one (hoare_rewrite_avx512) on random segments, bit for bit,
// and a whole-row replay timing at n_s = 1e7 with and without the pool.
// Build: g++ -O2 -std=c++17 -I.. replay_par_check.cpp -lpthread
#include "../../paper_2406_10938_b200/csrc/host_core.cpp"
#include <chrono>
#include <cstdio>
#include <cstring>
using namespace detlsh_b200;
int main(int argc, char** argv) {
    std::mt19937_64 g(11);
    std::normal_distribution<float> nd(0.f, 300.f);
    int bad = 0, tried = 0, done = 0;
    for (int trial = 0; trial < 60; ++trial) {
        const size_t len = (size_t{1} << 18) + g() % 3000000;
        std::vector<float> a(len + 8), b;
        for (auto& v : a) v = nd(g);
        const size_t lo = 3, hi = lo + len - 5;
        // the caller's median-of-three prologue, on a copy of the same data
        const size_t mid = lo + (hi - lo) / 2;
        std::swap(a[mid], a[lo + g() % (hi - lo)]);
        if (a[mid] < a[lo]) std::swap(a[lo], a[mid]);
        if (a[hi - 1] < a[lo]) std::swap(a[lo], a[hi - 1]);
        if (a[hi - 1] < a[mid]) std::swap(a[mid], a[hi - 1]);
        std::swap(a[mid], a[lo + 1]);
        const float pv = a[lo + 1];
        b = a;
        std::vector<float> buf1(2 * a.size() + 64), buf2(2 * a.size() + 64);
        size_t p1 = 0, p2 = 0;
        const bool ok1 = hoare_rewrite_avx512(a.data(), lo, hi, pv, buf1.data(), &p1);
        const bool ok2 = hoare_rewrite_par(b.data(), lo, hi, pv, buf2.data(), &p2);
        ++tried;
        if (ok1 != ok2 || (ok1 && (p1 != p2 || std::memcmp(a.data(), b.data(), a.size() * 4) != 0))) ++bad;
        done += ok1;
    }
    printf("segments %d (closed form taken %d): mismatches %d\n", tried, done, bad);
    // whole rows
    const size_t ns = argc > 1 ? static_cast<size_t>(atol(argv[1])) : 10000000;
    const int lo_shift = argc > 2 ? atoi(argv[2]) : 15;
    std::vector<float> base(ns), work(ns), row(257);
    for (auto& v : base) v = nd(g);
    for (int mode = 0; mode < 4; ++mode) {
        kParMin = mode ? (size_t{1} << (lo_shift + mode)) : ~size_t{0};
        Rng rng(5);
        uint64_t draws = 0;
        double t = 0;
        std::vector<float> out(257 * 48);
        for (int r = 0; r < (ns < 1000000 ? 48 : 4); ++r) {
            work = base;
            const auto t0 = std::chrono::steady_clock::now();
            select_row_breakpoints(work.data(), ns, 256, rng, out.data() + r * 257, &draws);
            t += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        }
        printf("%s (par from 2^%d): %.1f ms/row, draws %llu, row0[128] %.6f\n", mode ? "pool" : "single", lo_shift + mode, t / (ns < 1000000 ? 48 : 4),
               (unsigned long long)draws, out[128]);
    }
    return bad != 0;
}
