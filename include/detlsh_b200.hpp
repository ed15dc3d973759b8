// detlsh_b200.hpp — header-only C++ facade over the C ABI (detlsh_b200.h) that
// restores the reference's own C++ API for the hot path, so a caller of
// /root/reference/proj/include/detlsh/index.hpp switches by changing the
// namespace and the include:
//
//     detlsh::build_index(data, params, seed)   ->  detlsh_b200::build_index(...)  (index.hpp:39)
//     detlsh::build_index_with_family(...)      ->  detlsh_b200::build_index_with_family(...) (:42-43)
//     detlsh::build_det_only_index(...)         ->  detlsh_b200::build_det_only_index(...) (:46-47)
//     detlsh::ck_ann(index, q, k)               ->  detlsh_b200::ck_ann(...)       (index.hpp:87)
//     detlsh::rc_ann(index, q, r, c)            ->  detlsh_b200::rc_ann(...)
//     detlsh::estimate_rmin(index, probes, k)   ->  detlsh_b200::estimate_rmin(...) (index.hpp:91)
//     detlsh::candidate_budget(beta, n, k)      ->  detlsh_b200::candidate_budget  (index.hpp:50)
//     detlsh::derive_params(K, c, L)            ->  detlsh_b200::derive_params     (projection.hpp:75)
//     detlsh::range_query_optimized / _exact    ->  detlsh_b200::range_query_*     (de_tree.hpp:85-100)
//     detlsh::save_index(index)                 ->  detlsh_b200::save_index        (persist.hpp:17)
//
// `data` is a std::shared_ptr<const Dataset> exactly as in the reference
// (detlsh::Dataset, dataset.hpp:12-21: n, d, row-major values); the returned
// DetIndex carries params, family, table and the data handle like
// detlsh::DetIndex (index.hpp:24-37), with the trees exported on demand
// (trees(): the flattened node arrays in the reference's node order) and
// project_query.  Plus ck_ann_batch (the batched GPU entry point).  Errors
// follow the reference: std::invalid_argument for precondition failures,
// FormatError for format problems, std::runtime_error for device failures.
#pragma once

#include <cstdint>
#include <functional>
#include <memory>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "detlsh_b200.h"

namespace detlsh_b200 {

// detlsh::LshParams (projection.hpp:79-92), same defaults.
struct LshParams {
    int K = 16;
    int L = 4;
    double c = 1.5;
    double beta = 0.0;
    double epsilon = 0.0;
    double alpha1 = 0.0;
    double alpha2 = 0.0;
    int n_regions = 256;
    double sample_fraction = 0.1;
    int leaf_capacity = 128;
    double r_min = 0.0;
    int k = 50;
};

struct DerivedParams {
    double alpha1 = 0.0, alpha2 = 0.0, epsilon = 0.0, beta = 0.0;
};

// detlsh::QueryResult (index.hpp:79-83).
struct QueryResult {
    std::vector<std::pair<std::uint32_t, double>> hits;
    double radius_used = 0.0;
    std::size_t candidates_seen = 0;
};

class FormatError : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};

// detlsh::Dataset (dataset.hpp:12-21): row-major n x d.
struct Dataset {
    std::size_t n = 0;
    int d = 0;
    std::vector<float> values;  // n * d
    std::span<const float> row(std::size_t i) const {
        return {values.data() + i * static_cast<std::size_t>(d), static_cast<std::size_t>(d)};
    }
};

// detlsh::HashFamily (projection.hpp:14-28).
struct HashFamily {
    int d = 0, K = 0, L = 0;
    std::uint64_t seed = 0;
    std::vector<float> coeffs;  // vector (i, j) at offset (i*K + j) * d
    std::span<const float> vec(int space, int dim) const {
        return {coeffs.data() + (static_cast<std::size_t>(space) * K + dim) * static_cast<std::size_t>(d),
                static_cast<std::size_t>(d)};
    }
    bool empty() const { return coeffs.empty(); }
};

// detlsh::BreakpointTable (encoder.hpp:15-31).
struct BreakpointTable {
    int L = 0, K = 0, n_regions = 0;
    std::size_t sample_size = 0;
    std::vector<float> boundaries;  // [L][K][n_regions + 1]
    std::span<const float> row(int space, int dim) const {
        return {boundaries.data() + (static_cast<std::size_t>(space) * K + dim) * (n_regions + 1),
                static_cast<std::size_t>(n_regions) + 1};
    }
};

// A DE-Tree (de_tree.hpp:44-58) flattened: nodes in the reference's node
// order; leaf entries concatenated (ebegin/ecount index `positions`).
struct DeTreeExport {
    std::vector<std::int32_t> root_children;  // [2^K]
    std::vector<std::uint8_t> is_leaf, split_dim;
    std::vector<std::int32_t> left, right;
    std::vector<std::uint8_t> bits, value;  // [nodes][K]
    std::vector<std::uint64_t> ebegin;
    std::vector<std::uint32_t> ecount;
    std::vector<std::uint32_t> positions;
};

using CandidateSink = std::function<bool(std::uint32_t)>;

namespace detail {
inline void check(int rc) {
    if (rc == DETLSH_OK) return;
    const std::string msg = detlsh_gpu_last_error();
    if (rc == DETLSH_E_INVALID) throw std::invalid_argument(msg);
    if (rc == DETLSH_E_FORMAT) throw FormatError(msg);
    throw std::runtime_error(msg);
}
inline detlsh_params to_c(const LshParams& p) {
    return detlsh_params{p.K, p.L, p.c, p.beta, p.epsilon, p.alpha1, p.alpha2, p.n_regions,
                         p.sample_fraction, p.leaf_capacity, p.r_min, p.k};
}
inline LshParams from_c(const detlsh_params& c) {
    return LshParams{c.K, c.L, c.c, c.beta, c.epsilon, c.alpha1, c.alpha2, c.n_regions,
                     c.sample_fraction, c.leaf_capacity, c.r_min, c.k};
}
struct Free {
    void operator()(detlsh_gpu_index* p) const { detlsh_gpu_free(p); }
};
}  // namespace detail

// The assembled index (detlsh::DetIndex, index.hpp:24-37): immutable after
// build; queries from several host threads are safe.
class DetIndex {
public:
    LshParams params;  // derived fields (alpha1, alpha2, epsilon, beta, r_min) populated
    HashFamily family;  // empty for the DET-ONLY (PAA) variant
    BreakpointTable table;
    std::shared_ptr<const Dataset> data;  // the caller's dataset handle (null for span builds)

    std::size_t n() const { return detlsh_gpu_n(h_.get()); }
    int d() const { return detlsh_gpu_d(h_.get()); }
    const detlsh_gpu_index* handle() const { return h_.get(); }

    // DetIndex::project_query (index.cpp:181-188)
    std::vector<float> project_query(std::span<const float> q, int space) const {
        if (q.size() != static_cast<std::size_t>(d())) throw std::invalid_argument("project_query: dimension mismatch");
        if (space < 0 || space >= params.L) throw std::invalid_argument("project_query: space out of range");
        std::vector<float> all(static_cast<std::size_t>(params.L) * params.K);
        detail::check(detlsh_gpu_project_query(h_.get(), q.data(), 1, all.data(), 0));
        return {all.begin() + static_cast<std::ptrdiff_t>(space) * params.K,
                all.begin() + static_cast<std::ptrdiff_t>(space + 1) * params.K};
    }

    // The L trees, exported from the device (one D2H per call).
    std::vector<DeTreeExport> trees() const {
        std::vector<DeTreeExport> out(static_cast<std::size_t>(params.L));
        for (int i = 0; i < params.L; ++i) {
            std::uint64_t nn = 0;
            detail::check(detlsh_gpu_tree_num_nodes(h_.get(), i, &nn));
            DeTreeExport& t = out[static_cast<std::size_t>(i)];
            const std::size_t K = static_cast<std::size_t>(params.K);
            t.root_children.resize(std::size_t{1} << params.K);
            t.is_leaf.resize(nn);
            t.split_dim.resize(nn);
            t.left.resize(nn);
            t.right.resize(nn);
            t.bits.resize(nn * K);
            t.value.resize(nn * K);
            t.ebegin.resize(nn);
            t.ecount.resize(nn);
            t.positions.resize(n());
            detail::check(detlsh_gpu_export_tree(h_.get(), i, t.root_children.data(), t.is_leaf.data(),
                                                 t.split_dim.data(), t.left.data(), t.right.data(), t.bits.data(),
                                                 t.value.data(), t.ebegin.data(), t.ecount.data(), t.positions.data()));
        }
        return out;
    }

private:
    friend DetIndex detail_wrap(detlsh_gpu_index*, const detlsh_params&, std::shared_ptr<const Dataset>);
    std::shared_ptr<detlsh_gpu_index> h_;
};

inline DetIndex detail_wrap(detlsh_gpu_index* h, const detlsh_params& c, std::shared_ptr<const Dataset> data) {
    DetIndex idx;
    idx.h_ = std::shared_ptr<detlsh_gpu_index>(h, detail::Free{});
    idx.params = detail::from_c(c);
    idx.data = std::move(data);
    const int d = detlsh_gpu_d(h);
    if (idx.params.L >= 1) {
        idx.table.L = idx.params.L;
        idx.table.K = idx.params.K;
        idx.table.n_regions = idx.params.n_regions;
        idx.table.sample_size = detlsh_gpu_sample_size(h);
        idx.table.boundaries.resize(static_cast<std::size_t>(idx.params.L) * idx.params.K * (idx.params.n_regions + 1));
        detail::check(detlsh_gpu_export_table(h, idx.table.boundaries.data()));
    }
    const std::uint64_t fs = detlsh_gpu_family_seed(h);
    if (detlsh_gpu_has_family(h)) {
        idx.family.d = d;
        idx.family.K = idx.params.K;
        idx.family.L = idx.params.L;
        idx.family.seed = fs;
        idx.family.coeffs.resize(static_cast<std::size_t>(idx.params.L) * idx.params.K * d);
        detail::check(detlsh_gpu_export_family(h, idx.family.coeffs.data()));
    }
    return idx;
}

inline std::size_t candidate_budget(double beta, std::size_t n, int k) {
    return detlsh_candidate_budget(beta, n, k);
}

inline DerivedParams derive_params(int K, double c, int L) {
    double o[4];
    detail::check(detlsh_derive_params(K, c, L, o));
    return DerivedParams{o[0], o[1], o[2], o[3]};
}

// build_index (index.hpp:39): `values` is the row-major n x d dataset (the
// reference's Dataset::values); the index keeps its own device copy.
inline DetIndex build_index(std::span<const float> values, std::size_t n, int d, LshParams params,
                            std::uint64_t seed, int device = 0, std::uint32_t flags = 0) {
    if (values.size() != n * static_cast<std::size_t>(d))
        throw std::invalid_argument("build_index: values.size() != n * d");
    detlsh_params c = detail::to_c(params);
    detlsh_gpu_index* h = nullptr;
    detail::check(detlsh_gpu_build(values.data(), n, d, &c, seed, device, flags, &h));
    return detail_wrap(h, c, nullptr);
}

// build_index (index.hpp:39) with the reference's own signature.
inline DetIndex build_index(std::shared_ptr<const Dataset> data, LshParams params, std::uint64_t seed,
                            int device = 0, std::uint32_t flags = 0) {
    if (!data) throw std::invalid_argument("build_index: data is null");
    DetIndex idx = build_index(data->values, data->n, data->d, params, seed, device, flags);
    idx.data = std::move(data);
    return idx;
}

// build_index_with_family (index.hpp:42-43): coefficients [L][K][d].
inline DetIndex build_index_with_family(std::span<const float> values, std::size_t n, int d,
                                        LshParams params, std::span<const float> coeffs, int K,
                                        int L, std::uint64_t family_seed, std::uint64_t seed,
                                        int device = 0) {
    if (coeffs.size() != static_cast<std::size_t>(K) * L * d)
        throw std::invalid_argument("build_index: family size does not match K * L * d");
    detlsh_params c = detail::to_c(params);
    detlsh_gpu_index* h = nullptr;
    detail::check(detlsh_gpu_build_with_family(values.data(), n, d, &c, coeffs.data(), K, L,
                                               family_seed, seed, device, 0, &h));
    return detail_wrap(h, c, nullptr);
}

inline DetIndex build_index_with_family(std::shared_ptr<const Dataset> data, LshParams params, HashFamily family,
                                        std::uint64_t seed, int device = 0) {
    if (!data) throw std::invalid_argument("build_index: data is null");
    if (family.d != data->d) throw std::invalid_argument("build_index: family dimension does not match the dataset");
    DetIndex idx = build_index_with_family(data->values, data->n, data->d, params, family.coeffs, family.K, family.L,
                                           family.seed, seed, device);
    idx.data = std::move(data);
    return idx;
}

// Batched ck_ann: queries [nq][d] row-major, one QueryResult per query.
inline std::vector<QueryResult> ck_ann_batch(const DetIndex& index, std::span<const float> queries,
                                             int k) {
    const std::size_t d = static_cast<std::size_t>(index.d());
    if (d == 0 || queries.size() % d != 0)
        throw std::invalid_argument("ck_ann: query dimension mismatch");
    const std::size_t nq = queries.size() / d;
    std::vector<std::uint32_t> ids(nq * static_cast<std::size_t>(k));
    std::vector<double> dists(ids.size()), radius(nq);
    std::vector<std::int32_t> hits(nq);
    std::vector<std::uint64_t> cands(nq);
    detail::check(detlsh_gpu_query(index.handle(), queries.data(), nq, k, 0, ids.data(),
                                   dists.data(), hits.data(), radius.data(), cands.data(), nullptr));
    std::vector<QueryResult> out(nq);
    for (std::size_t q = 0; q < nq; ++q) {
        for (int t = 0; t < hits[q]; ++t)
            out[q].hits.emplace_back(ids[q * k + t], dists[q * k + t]);
        out[q].radius_used = radius[q];
        out[q].candidates_seen = cands[q];
    }
    return out;
}

// ck_ann (index.hpp:87, index.cpp:292-331).
inline QueryResult ck_ann(const DetIndex& index, std::span<const float> q, int k) {
    if (q.size() != static_cast<std::size_t>(index.d()))
        throw std::invalid_argument("ck_ann: query dimension mismatch");
    return std::move(ck_ann_batch(index, q, k).front());
}

// build_det_only_index (index.cpp:220-232): PAA projection, L = 1.
inline DetIndex build_det_only_index(std::span<const float> values, std::size_t n, int d, LshParams params,
                                     std::uint64_t seed, int device = 0) {
    return build_index(values, n, d, params, seed, device, DETLSH_F_PAA);
}
inline DetIndex build_det_only_index(std::shared_ptr<const Dataset> data, LshParams params, std::uint64_t seed,
                                     int device = 0) {
    return build_index(std::move(data), params, seed, device, DETLSH_F_PAA);
}

// estimate_rmin (index.hpp:91, index.cpp:333-374).
inline double estimate_rmin(const DetIndex& index, std::span<const std::vector<float>> probes, int k) {
    const std::size_t d = static_cast<std::size_t>(index.d());
    std::vector<float> flat;
    flat.reserve(probes.size() * d);
    for (const auto& p : probes) {
        if (p.size() != d) throw std::invalid_argument("estimate_rmin: probe dimension mismatch");
        flat.insert(flat.end(), p.begin(), p.end());
    }
    double r = 0.0;
    detail::check(detlsh_gpu_estimate_rmin(index.handle(), flat.data(), probes.size(), k, 0, &r));
    return r;
}

// range_query_optimized (de_tree.hpp:93-100) on tree `tree` of the index: the
// leaves with mindist <= radius drained in (mindist, node index) order into
// `sink` until it returns false.
inline void range_query_optimized(const DetIndex& index, int tree, std::span<const float> q_proj, double radius,
                                  const CandidateSink& sink) {
    if (q_proj.size() != static_cast<std::size_t>(index.params.K))
        throw std::invalid_argument("range_query: projected query must have K coordinates");
    std::uint64_t count = 0;
    detail::check(detlsh_gpu_range_query(index.handle(), tree, q_proj.data(), 1, &radius, ~0ULL, 0, nullptr, 0, &count));
    std::vector<std::uint32_t> pos(count);
    if (count)
        detail::check(detlsh_gpu_range_query(index.handle(), tree, q_proj.data(), 1, &radius, ~0ULL, 0, pos.data(),
                                             count, &count));
    for (const std::uint32_t p : pos)
        if (!sink(p)) return;
}

// range_query_exact (de_tree.hpp:85-91): {pos : ||q', o'_pos|| <= radius} in DFS order.
inline std::vector<std::uint32_t> range_query_exact(const DetIndex& index, int tree, std::span<const float> q_proj,
                                                    double radius) {
    if (q_proj.size() != static_cast<std::size_t>(index.params.K))
        throw std::invalid_argument("range_query: projected query must have K coordinates");
    std::uint64_t count = 0;
    detail::check(detlsh_gpu_range_query(index.handle(), tree, q_proj.data(), 1, &radius, ~0ULL, DETLSH_RANGE_EXACT,
                                         nullptr, 0, &count));
    std::vector<std::uint32_t> pos(count);
    if (count)
        detail::check(detlsh_gpu_range_query(index.handle(), tree, q_proj.data(), 1, &radius, ~0ULL,
                                             DETLSH_RANGE_EXACT, pos.data(), count, &count));
    return pos;
}

// rc_ann (index.cpp:267-290): the closest candidate, or nullopt.
inline std::optional<std::pair<std::uint32_t, double>> rc_ann(const DetIndex& index, std::span<const float> q,
                                                              double r, double c) {
    if (q.size() != static_cast<std::size_t>(index.d()))
        throw std::invalid_argument("rc_ann: query dimension mismatch");
    std::uint32_t id = 0;
    double dist = 0.0;
    std::int32_t found = 0;
    detail::check(detlsh_gpu_rc_ann(index.handle(), q.data(), 1, r, c, 0, &id, &dist, &found, nullptr, nullptr));
    if (!found) return std::nullopt;
    return std::make_pair(id, dist);
}

// save_index (persist.hpp:17): the DETL v1 bytes detlsh::save_index writes for
// the same build; detlsh::load_index reads them back.
inline std::vector<std::uint8_t> save_index(const DetIndex& index) {
    auto* h = const_cast<detlsh_gpu_index*>(index.handle());
    std::uint64_t size = 0;
    detail::check(detlsh_gpu_save_detl(h, nullptr, 0, &size));
    std::vector<std::uint8_t> bytes(size);
    detail::check(detlsh_gpu_save_detl(h, bytes.data(), bytes.size(), &size));
    return bytes;
}

}  // namespace detlsh_b200
