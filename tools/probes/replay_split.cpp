// Probe: where does one reference-sample replay row (encoder.cpp:57-103,
// n_s = 100 000, 255 targets) spend its time?  Times each partition and bins
// it by segment length.  Build: g++ -O2 -std=c++17 -I.. replay_split.cpp
#include "../../paper_2406_10938_b200/csrc/host_core.cpp"
#include <chrono>
#include <cstdio>
using namespace detlsh_b200;
int main(int argc, char** argv) {
    const size_t ns = argc > 1 ? atol(argv[1]) : 100000;
    const int rows = 48;
    std::mt19937_64 g(7);
    std::normal_distribution<float> nd(0.f, 300.f);
    std::vector<float> base(ns * rows);
    for (auto& v : base) v = nd(g);
    Rng rng(123);
    double tb[8] = {0};
    uint64_t cb[8] = {0}, eb[8] = {0};
    const size_t edges[7] = {16, 64, 256, 1024, 4096, 16384, 65536};
    std::vector<float> row(257), sbuf(2 * ns);
    auto T0 = std::chrono::steady_clock::now();
    double t_other = 0;
    for (int r = 0; r < rows; ++r) {
        float* a = base.data() + r * ns;
        const size_t span = ns / 256, nt = 255;
        struct Item { size_t lo, hi, tlo, thi; };
        std::vector<Item> st{{0, ns, 0, nt}};
        while (!st.empty()) {
            Item it = st.back(); st.pop_back();
            if (it.tlo >= it.thi) continue;
            if (it.hi - it.lo <= 8) { small_sort(a, it.lo, it.hi); continue; }
            const size_t len = it.hi - it.lo;
            int b = 0; while (b < 7 && len > edges[b]) ++b;
            auto t0 = std::chrono::steady_clock::now();
            const size_t p = hoare_partition(a, it.lo, it.hi, rng, sbuf.data());
            auto t1 = std::chrono::steady_clock::now();
            tb[b] += std::chrono::duration<double>(t1 - t0).count();
            cb[b]++; eb[b] += len;
            const size_t below = std::min(std::max(p / span, it.tlo), it.thi);
            const size_t above = std::min(std::max((p + 1) / span, it.tlo), it.thi);
            st.push_back({it.lo, p, it.tlo, below});
            st.push_back({p + 1, it.hi, above, it.thi});
        }
    }
    double tot = std::chrono::duration<double>(std::chrono::steady_clock::now() - T0).count();
    // plain timing through the shipped entry point
    std::vector<float> base2(ns * rows);
    for (auto& v : base2) v = nd(g);
    auto T1 = std::chrono::steady_clock::now();
    for (int r = 0; r < rows; ++r) select_row_breakpoints(base2.data() + r * ns, ns, 256, rng, row.data(), nullptr);
    double tot2 = std::chrono::duration<double>(std::chrono::steady_clock::now() - T1).count();
    printf("ns=%zu rows=%d instrumented %.3f ms/row, shipped %.3f ms/row\n", ns, rows, tot / rows * 1e3, tot2 / rows * 1e3);
    const char* nm[8] = {"<=16", "<=64", "<=256", "<=1K", "<=4K", "<=16K", "<=64K", ">64K"};
    for (int b = 0; b < 8; ++b)
        printf("%6s: %7.1f parts/row %9.0f elems/row %8.4f ms/row  %.2f ns/elem\n", nm[b], cb[b] / (double)rows,
               eb[b] / (double)rows, tb[b] / rows * 1e3, eb[b] ? tb[b] / eb[b] * 1e9 : 0.);
}
