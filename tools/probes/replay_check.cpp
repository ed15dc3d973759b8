// Probe: the closed-form rewrite partition (host_core.cpp: hoare_rewrite_avx512)
// against the sentinel loop on random segments (with and without ties), and the
// per-row replay time at n_s = 100 000 vs the rewrite threshold.
#include "../../paper_2406_10938_b200/csrc/host_core.cpp"
#include <chrono>
#include <cstdio>
#include <cstring>
using namespace detlsh_b200;
int main(int argc, char** argv) {
    std::mt19937_64 g(11);
    std::vector<float> buf(1 << 22);
    long bad = 0, fast = 0;
    for (int it = 0; it < 200000; ++it) {
        size_t len = 3 + g() % (it < 150000 ? 300 : 20000);
        std::vector<float> a(len + 4);
        int mode = g() % 3;
        for (auto& v : a) v = mode == 0 ? (float)(g() % 1000000) : mode == 1 ? (float)(g() % 50) : std::ldexp((float)(g() % 100000) - 50000.f, -10);
        std::vector<float> b = a;
        size_t lo = 2, hi = 2 + len;
        // same prologue for both (pv = a[lo+1]), as hoare_partition arranges it
        uint64_t r = g() % len;
        for (auto* x : {&a, &b}) {
            auto& y = *x;
            size_t mid = lo + len / 2;
            std::swap(y[mid], y[lo + r]);
            if (y[mid] < y[lo]) std::swap(y[lo], y[mid]);
            if (y[hi - 1] < y[lo]) std::swap(y[lo], y[hi - 1]);
            if (y[hi - 1] < y[mid]) std::swap(y[mid], y[hi - 1]);
            std::swap(y[mid], y[lo + 1]);
        }
        if (len < 3) continue;
        float pv = a[lo + 1];
        size_t j = hoare_scan_simple(a.data(), lo, hi, pv);
        std::swap(a[lo + 1], a[j]);
        size_t p;
        if (hoare_rewrite_avx512(b.data(), lo, hi, pv, buf.data(), &p)) {
            ++fast;
            if (p != j || memcmp(a.data(), b.data(), a.size() * 4)) ++bad;
        }
    }
    printf("rewrite checked on %ld segments, %ld mismatches\n", fast, bad);
    const size_t ns = 100000;
    const int rows = 48;
    std::normal_distribution<float> nd(0.f, 300.f);
    std::vector<float> base(ns * rows);
    for (auto& v : base) v = nd(g);
    std::vector<float> row(257), row2(257);
    for (size_t thr : {(size_t)1 << 40, (size_t)48, (size_t)64, (size_t)128, (size_t)256, (size_t)1024}) {
        kRewriteMin = thr;
        double best = 1e30;
        uint64_t draws = 0, nxt = 0;
        for (int rep = 0; rep < 5; ++rep) {
            std::vector<float> w = base;
            Rng rng(5);
            draws = 0;
            auto T = std::chrono::steady_clock::now();
            for (int r = 0; r < rows; ++r) select_row_breakpoints(w.data() + r * ns, ns, 256, rng, row.data(), &draws);
            best = std::min(best, std::chrono::duration<double>(std::chrono::steady_clock::now() - T).count() * 1e3 / rows);
            nxt = rng.next_u64();
        }
        printf("thr %-14zu %.3f ms/row (min of 5) draws %lu next %016lx\n", thr, best, (unsigned long)draws, (unsigned long)nxt);
    }
}
