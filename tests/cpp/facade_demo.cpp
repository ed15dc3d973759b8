// Drives the C++ facade (include/detlsh_b200.hpp) the way a caller of the
// reference's detlsh::build_index / detlsh::ck_ann would.  Data comes from a
// tiny LCG so tests/test_facade.py can regenerate the same bytes in Python.
// Prints: r_min, then per query "q rank id dist" lines.
#include <cstdio>
#include <cstdint>
#include <memory>
#include <vector>

#include "detlsh_b200.hpp"

static float lcg(uint64_t& s) {
    s = s * 6364136223846793005ULL + 1442695040888963407ULL;
    return static_cast<float>((s >> 40) % 256);  // 8-bit values
}

int main(int argc, char** argv) {
    const std::size_t n = 5000, nq = 5;
    const int d = 24, k = 7;
    uint64_t s = 12345;
    std::vector<float> data(n * d), q(nq * d);
    for (auto& v : data) v = lcg(s);
    for (auto& v : q) v = lcg(s);
    detlsh_b200::LshParams p;
    p.beta = 0.1;
    p.k = k;
    p.leaf_capacity = 32;
    try {
        auto idx = detlsh_b200::build_index(data, n, d, p, 77);
        std::printf("r_min %.17g\n", idx.params.r_min);
        for (std::size_t i = 0; i < nq; ++i) {
            auto r = detlsh_b200::ck_ann(idx, std::span<const float>(q.data() + i * d, d), k);
            for (std::size_t t = 0; t < r.hits.size(); ++t)
                std::printf("%zu %zu %u %.17g\n", i, t, r.hits[t].first, r.hits[t].second);
        }
        // the reference's own signature: shared_ptr<const Dataset>
        auto ds = std::make_shared<detlsh_b200::Dataset>();
        ds->n = n;
        ds->d = d;
        ds->values = data;
        auto idx2 = detlsh_b200::build_index(std::shared_ptr<const detlsh_b200::Dataset>(ds), p, 77);
        std::printf("dataset_build %d %zu %zu %zu\n", idx2.params.r_min == idx.params.r_min ? 1 : 0,
                    idx2.family.coeffs.size(), idx2.table.boundaries.size(), idx2.trees().size());
        std::vector<std::vector<float>> probes;
        for (std::size_t i = 0; i < 3; ++i) probes.emplace_back(q.begin() + i * d, q.begin() + (i + 1) * d);
        std::printf("estimate_rmin %.17g\n", detlsh_b200::estimate_rmin(idx2, probes, k));
        const auto qp = idx2.project_query(std::span<const float>(q.data(), d), 1);
        const double rad = idx2.params.epsilon * idx2.params.r_min;
        std::vector<std::uint32_t> drained;
        detlsh_b200::range_query_optimized(idx2, 1, qp, rad, [&](std::uint32_t pos) {
            drained.push_back(pos);
            return drained.size() < 40;
        });
        const auto exact = detlsh_b200::range_query_exact(idx2, 1, qp, rad);
        std::printf("range %zu %zu", drained.size(), exact.size());
        for (std::size_t i = 0; i < drained.size() && i < 5; ++i) std::printf(" %u", drained[i]);
        std::printf("\n");
        // save_index: DETL v1 bytes (the reference's persist format)
        const auto blob = detlsh_b200::save_index(idx);
        std::printf("detl %zu %c%c%c%c\n", blob.size(), blob[0], blob[1], blob[2], blob[3]);
        // the reference's precondition errors surface as std::invalid_argument
        try {
            detlsh_b200::ck_ann(idx, std::span<const float>(q.data(), d - 1), k);
            return 3;
        } catch (const std::invalid_argument&) {
        }
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 2;
    }
    return 0;
}
