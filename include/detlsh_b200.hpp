// detlsh_b200.hpp — header-only C++ facade over the C ABI (detlsh_b200.h) that
// restores the reference's own C++ API for the hot path, so a caller of
// /root/reference/proj/include/detlsh/index.hpp switches by changing the
// namespace and the include:
//
//     detlsh::build_index(data, params, seed)   ->  detlsh_b200::build_index(...)  (index.hpp:39)
//     detlsh::build_index_with_family(...)      ->  detlsh_b200::build_index_with_family(...) (:42-43)
//     detlsh::ck_ann(index, q, k)               ->  detlsh_b200::ck_ann(...)       (index.hpp:87)
//     detlsh::candidate_budget(beta, n, k)      ->  detlsh_b200::candidate_budget  (index.hpp:50)
//     detlsh::derive_params(K, c, L)            ->  detlsh_b200::derive_params     (projection.hpp:75)
//
// plus ck_ann_batch (the batched GPU entry point).  Errors follow the
// reference: std::invalid_argument for precondition failures, FormatError for
// format problems, std::runtime_error for device failures.
#pragma once

#include <cstdint>
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
    LshParams params;
    std::size_t n() const { return detlsh_gpu_n(h_.get()); }
    int d() const { return detlsh_gpu_d(h_.get()); }
    const detlsh_gpu_index* handle() const { return h_.get(); }
    std::vector<float> table() const {
        std::vector<float> t(static_cast<std::size_t>(params.L) * params.K * (params.n_regions + 1));
        detail::check(detlsh_gpu_export_table(h_.get(), t.data()));
        return t;
    }

private:
    friend DetIndex build_index(std::span<const float>, std::size_t, int, LshParams, std::uint64_t,
                                int, std::uint32_t);
    friend DetIndex build_index_with_family(std::span<const float>, std::size_t, int, LshParams,
                                            std::span<const float>, int, int, std::uint64_t,
                                            std::uint64_t, int);
    std::shared_ptr<detlsh_gpu_index> h_;
};

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
    DetIndex idx;
    idx.h_ = std::shared_ptr<detlsh_gpu_index>(h, detail::Free{});
    idx.params = detail::from_c(c);
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
    DetIndex idx;
    idx.h_ = std::shared_ptr<detlsh_gpu_index>(h, detail::Free{});
    idx.params = detail::from_c(c);
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
