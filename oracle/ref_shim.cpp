// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" shim over the UNMODIFIED reference library (compiled from the
// sources under /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libdetlsh_ref.so).  It lets the pytest parity suite and the
// bench's `--impl reference` arm call the reference's own C++ API
// (include/detlsh/index.hpp:39-91, encoder.hpp:41-63, de_tree.hpp:61-100)
// through ctypes.  Nothing here re-implements reference behaviour; every
// function forwards to the reference.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include <cmath>

#include "detlsh/chi2.hpp"
#include "detlsh/de_tree.hpp"
#include "detlsh/encoder.hpp"
#include "detlsh/index.hpp"
#include "detlsh/metrics.hpp"
#include "detlsh/persist.hpp"
#include "detlsh/projection.hpp"
#include "detlsh/rng.hpp"

using namespace detlsh;

extern "C" {

// Same field order as detlsh::LshParams (projection.hpp:79-92).
struct ref_params {
    int32_t K, L;
    double c, beta, epsilon, alpha1, alpha2;
    int32_t n_regions;
    double sample_fraction;
    int32_t leaf_capacity;
    double r_min;
    int32_t k;
};

static thread_local std::string g_err;
const char* ref_last_error() { return g_err.c_str(); }

static LshParams to_lsh(const ref_params* p) {
    LshParams q;
    q.K = p->K;
    q.L = p->L;
    q.c = p->c;
    q.beta = p->beta;
    q.n_regions = p->n_regions;
    q.sample_fraction = p->sample_fraction;
    q.leaf_capacity = p->leaf_capacity;
    q.r_min = p->r_min;
    q.k = p->k;
    return q;
}
static void from_lsh(const LshParams& q, ref_params* p) {
    p->K = q.K;
    p->L = q.L;
    p->c = q.c;
    p->beta = q.beta;
    p->epsilon = q.epsilon;
    p->alpha1 = q.alpha1;
    p->alpha2 = q.alpha2;
    p->n_regions = q.n_regions;
    p->sample_fraction = q.sample_fraction;
    p->leaf_capacity = q.leaf_capacity;
    p->r_min = q.r_min;
    p->k = q.k;
}

static std::shared_ptr<const Dataset> make_dataset(const float* data, uint64_t n, int32_t d) {
    auto ds = std::make_shared<Dataset>();
    ds->n = n;
    ds->d = d;
    ds->values.assign(data, data + n * static_cast<uint64_t>(d));
    return ds;
}

// ---- scalar numerics --------------------------------------------------------
double ref_chi2_cdf(double x, int k) { return chi2_cdf(x, k); }
double ref_chi2_quantile(double a, int k) { return chi2_quantile(a, k); }
double ref_regularized_gamma_p(double a, double x) { return regularized_gamma_p(a, x); }
int ref_derive_params(int K, double c, int L, double* out4) {
    try {
        DerivedParams d = derive_params(K, c, L);
        out4[0] = d.alpha1;
        out4[1] = d.alpha2;
        out4[2] = d.epsilon;
        out4[3] = d.beta;
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}
uint64_t ref_candidate_budget(double beta, uint64_t n, int k) { return candidate_budget(beta, n, k); }
uint64_t ref_mix_seed(uint64_t seed, uint64_t stream) { return mix_seed(seed, stream); }
void ref_rng_stream(uint64_t seed, uint64_t count, uint64_t* out_u64, double* out_normal) {
    Rng a(seed), b(seed);
    for (uint64_t i = 0; i < count; ++i) {
        if (out_u64) out_u64[i] = a.next_u64();
        if (out_normal) out_normal[i] = b.normal();
    }
}

// ---- stage functions ----------------------------------------------------------
int ref_sample_hash_family(int d, int K, int L, uint64_t seed, float* out) {
    try {
        HashFamily f = sample_hash_family(d, K, L, seed);
        std::copy(f.coeffs.begin(), f.coeffs.end(), out);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

static HashFamily family_from(const float* coeffs, int d, int K, int L, uint64_t seed) {
    HashFamily f;
    f.d = d;
    f.K = K;
    f.L = L;
    f.seed = seed;
    f.coeffs.assign(coeffs, coeffs + static_cast<size_t>(L) * K * d);
    return f;
}

// out: [L][n][K]
int ref_project_dataset(const float* coeffs, int K, int L, const float* data, uint64_t n, int d,
                        float* out) {
    try {
        HashFamily f = family_from(coeffs, d, K, L, 0);
        Dataset ds;
        ds.n = n;
        ds.d = d;
        ds.values.assign(data, data + n * static_cast<uint64_t>(d));
        ProjectedDataset p = project_dataset(f, ds);
        std::copy(p.values.begin(), p.values.end(), out);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

static ProjectedDataset projected_from(const float* proj, uint64_t n, int K, int L) {
    ProjectedDataset p;
    p.L = L;
    p.K = K;
    p.n = n;
    p.values.assign(proj, proj + static_cast<size_t>(L) * n * K);
    return p;
}

// out: [L][K][n_regions+1]
int ref_select_breakpoints(const float* proj, uint64_t n, int K, int L, int n_regions,
                           double sample_fraction, uint64_t seed, float* out,
                           uint64_t* sample_size) {
    try {
        ProjectedDataset p = projected_from(proj, n, K, L);
        BreakpointTable t = select_breakpoints(p, n_regions, sample_fraction, seed);
        std::copy(t.boundaries.begin(), t.boundaries.end(), out);
        if (sample_size) *sample_size = t.sample_size;
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

int ref_select_row_breakpoints(float* sample, uint64_t n_s, int n_regions, uint64_t rng_seed,
                               float* out_row) {
    try {
        Rng rng(rng_seed);
        auto row = select_row_breakpoints(std::span<float>(sample, n_s), n_regions, rng);
        std::copy(row.begin(), row.end(), out_row);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

int ref_locate_region(float v, const float* row, int n_regions) {
    return locate_region(v, std::span<const float>(row, static_cast<size_t>(n_regions) + 1),
                         n_regions);
}

static BreakpointTable table_from(const float* table, int K, int L, int n_regions) {
    BreakpointTable t;
    t.L = L;
    t.K = K;
    t.n_regions = n_regions;
    t.boundaries.assign(table, table + static_cast<size_t>(L) * K * (n_regions + 1));
    return t;
}

int ref_encode_dataset(const float* proj, uint64_t n, int K, int L, const float* table,
                       int n_regions, uint8_t* out) {
    try {
        ProjectedDataset p = projected_from(proj, n, K, L);
        BreakpointTable t = table_from(table, K, L, n_regions);
        EncodedDataset e = encode_dataset(p, t);
        std::copy(e.symbols.begin(), e.symbols.end(), out);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// ---- tree handles ---------------------------------------------------------------
struct RefTree {
    DeTree tree;
};

void* ref_build_tree(const uint8_t* codes, uint64_t n, int K, int L, int n_regions, int space,
                     int max_size) {
    try {
        EncodedDataset e;
        e.L = L;
        e.K = K;
        e.n = n;
        e.n_regions = n_regions;
        e.symbols.assign(codes, codes + static_cast<size_t>(L) * n * K);
        auto* t = new RefTree{build_tree(e, space, max_size)};
        return t;
    } catch (const std::exception& ex) {
        g_err = ex.what();
        return nullptr;
    }
}

void ref_tree_free(void* h) { delete static_cast<RefTree*>(h); }

static const DeTree& tree_of(void* h) { return static_cast<RefTree*>(h)->tree; }

uint64_t ref_tree_num_nodes(void* h) { return tree_of(h).nodes.size(); }
uint64_t ref_tree_total_entries(void* h) { return tree_of(h).total_entries(); }

// Flattens the tree in the reference's own node order (build order).
static void export_tree(const DeTree& t, int32_t* root_children, uint8_t* is_leaf,
                        uint8_t* split_dim, int32_t* left, int32_t* right, uint8_t* bits,
                        uint8_t* value, uint64_t* ebegin, uint32_t* ecount, uint32_t* positions) {
    if (root_children) std::copy(t.root_children.begin(), t.root_children.end(), root_children);
    uint64_t off = 0;
    const size_t K = static_cast<size_t>(t.K);
    for (size_t i = 0; i < t.nodes.size(); ++i) {
        const DeTreeNode& nd = t.nodes[i];
        if (is_leaf) is_leaf[i] = nd.is_leaf ? 1 : 0;
        if (split_dim) split_dim[i] = nd.split_dim;
        if (left) left[i] = nd.left;
        if (right) right[i] = nd.right;
        if (bits) std::copy(nd.prefix.bits.begin(), nd.prefix.bits.end(), bits + i * K);
        if (value) std::copy(nd.prefix.value.begin(), nd.prefix.value.end(), value + i * K);
        if (ebegin) ebegin[i] = off;
        if (ecount) ecount[i] = static_cast<uint32_t>(nd.entries.size());
        if (positions)
            std::copy(nd.entries.positions.begin(), nd.entries.positions.end(), positions + off);
        off += nd.entries.size();
    }
}

void ref_tree_export(void* h, int32_t* root_children, uint8_t* is_leaf, uint8_t* split_dim,
                     int32_t* left, int32_t* right, uint8_t* bits, uint8_t* value,
                     uint64_t* ebegin, uint32_t* ecount, uint32_t* positions) {
    export_tree(tree_of(h), root_children, is_leaf, split_dim, left, right, bits, value, ebegin,
                ecount, positions);
}

// range_query_optimized (de_tree.cpp:229-258) with a sink that stops after
// `limit` positions; returns the number written.
uint64_t ref_range_query_optimized(void* h, const float* table, int n_regions, const float* q_proj,
                                   double radius, uint64_t limit, uint32_t* out) {
    const DeTree& t = tree_of(h);
    BreakpointTable tb;
    tb.L = t.space + 1;
    tb.K = t.K;
    tb.n_regions = n_regions;
    // table passed as the full [L][K][N_r+1] array; only row (space, *) is read.
    tb.boundaries.assign(table, table + static_cast<size_t>(tb.L) * t.K * (n_regions + 1));
    uint64_t count = 0;
    range_query_optimized(t, tb, std::span<const float>(q_proj, static_cast<size_t>(t.K)), radius,
                          [&](uint32_t pos) {
                              out[count++] = pos;
                              return count < limit;
                          });
    return count;
}

double ref_mindist(void* h, int node, const float* table, int n_regions, const float* q_proj) {
    const DeTree& t = tree_of(h);
    BreakpointTable tb;
    tb.L = t.space + 1;
    tb.K = t.K;
    tb.n_regions = n_regions;
    tb.boundaries.assign(table, table + static_cast<size_t>(tb.L) * t.K * (n_regions + 1));
    return mindist(std::span<const float>(q_proj, static_cast<size_t>(t.K)), t,
                   t.nodes[static_cast<size_t>(node)], tb);
}

// ---- full index ------------------------------------------------------------------
struct RefIndex {
    DetIndex index;
};

void* ref_build_index(const float* data, uint64_t n, int32_t d, ref_params* params, uint64_t seed,
                      double* seconds) {
    try {
        auto ds = make_dataset(data, n, d);
        auto t0 = std::chrono::steady_clock::now();
        auto* h = new RefIndex{build_index(ds, to_lsh(params), seed)};
        auto t1 = std::chrono::steady_clock::now();
        if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
        from_lsh(h->index.params, params);
        return h;
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

// Hybrid oracle: the reference's own stage functions, but with a caller-
// supplied breakpoint table (used to pin the GPU-native sample mode).  Mirrors
// assemble (index.cpp:138-177) using only the public API: r_min comes from
// estimate_rmin (index.cpp:333-374) over the same probe rows assemble draws.
void* ref_build_index_with_table(const float* data, uint64_t n, int32_t d, ref_params* params,
                                 uint64_t seed, const float* table, uint64_t sample_size) {
    try {
        auto ds = make_dataset(data, n, d);
        LshParams p = to_lsh(params);
        HashFamily fam = sample_hash_family(d, p.K, p.L, mix_seed(seed, 0));
        DerivedParams der = derive_params(p.K, p.c, p.L);
        p.alpha1 = der.alpha1;
        p.alpha2 = der.alpha2;
        p.epsilon = der.epsilon;
        if (p.beta <= 0.0) p.beta = der.beta;
        auto* h = new RefIndex{};
        DetIndex& idx = h->index;
        idx.params = p;
        idx.family = fam;
        idx.table = table_from(table, p.K, p.L, p.n_regions);
        idx.table.sample_size = sample_size;
        ProjectedDataset proj = project_dataset(fam, *ds);
        EncodedDataset enc = encode_dataset(proj, idx.table);
        for (int i = 0; i < p.L; ++i) idx.trees.push_back(build_tree(enc, i, p.leaf_capacity));
        idx.data = ds;
        idx.fingerprint = dataset_fingerprint(*ds);
        if (idx.params.r_min <= 0.0) {
            Rng rng(mix_seed(seed, 2));
            const size_t n_probes = std::min<size_t>(10, n);
            std::vector<std::vector<float>> probes;
            for (size_t t = 0; t < n_probes; ++t) {
                const auto pos = rng.bounded(n);
                auto r = ds->row(pos);
                probes.emplace_back(r.begin(), r.end());
            }
            idx.params.r_min = estimate_rmin(idx, probes, idx.params.k);
        }
        from_lsh(idx.params, params);
        return h;
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

void ref_index_free(void* h) { delete static_cast<RefIndex*>(h); }

static const DetIndex& idx_of(void* h) { return static_cast<RefIndex*>(h)->index; }

void ref_index_params(void* h, ref_params* out) { from_lsh(idx_of(h).params, out); }
void ref_index_table(void* h, float* out) {
    const auto& b = idx_of(h).table.boundaries;
    std::copy(b.begin(), b.end(), out);
}
uint64_t ref_index_sample_size(void* h) { return idx_of(h).table.sample_size; }
void ref_index_family(void* h, float* out) {
    const auto& c = idx_of(h).family.coeffs;
    std::copy(c.begin(), c.end(), out);
}
uint64_t ref_index_fingerprint(void* h) { return idx_of(h).fingerprint; }
uint64_t ref_index_tree_nodes(void* h, int tree) {
    return idx_of(h).trees[static_cast<size_t>(tree)].nodes.size();
}
void ref_index_tree_export(void* h, int tree, int32_t* root_children, uint8_t* is_leaf,
                           uint8_t* split_dim, int32_t* left, int32_t* right, uint8_t* bits,
                           uint8_t* value, uint64_t* ebegin, uint32_t* ecount,
                           uint32_t* positions) {
    export_tree(idx_of(h).trees[static_cast<size_t>(tree)], root_children, is_leaf, split_dim,
                left, right, bits, value, ebegin, ecount, positions);
}

// estimate_rmin (index.cpp:333-374) for caller probes [np][d]; NaN on error.
double ref_index_estimate_rmin(void* h, const float* probes, uint64_t np, int k) {
    try {
        const DetIndex& idx = idx_of(h);
        std::vector<std::vector<float>> pr;
        for (uint64_t p = 0; p < np; ++p)
            pr.emplace_back(probes + p * idx.d(), probes + (p + 1) * idx.d());
        return estimate_rmin(idx, pr, k);
    } catch (const std::exception& e) {
        g_err = e.what();
        return std::nan("");
    }
}

// DetIndex::project_query (index.cpp:181-188): out [K]
void ref_index_project_query(void* h, const float* q, int space, float* out) {
    const DetIndex& idx = idx_of(h);
    const auto v = idx.project_query(std::span<const float>(q, static_cast<size_t>(idx.d())), space);
    std::copy(v.begin(), v.end(), out);
}

// range_query_optimized / range_query_exact (de_tree.cpp:199-258) on tree
// `tree` of a built index; exact mode looks projected coordinates up by
// projecting the dataset row (the reference's ProjectedLookup).  Returns the
// list length; the first `cap` positions go to out.
uint64_t ref_index_range_query(void* h, int tree, const float* q_proj, double radius, uint64_t limit, int exact,
                               uint32_t* out, uint64_t cap) {
    const DetIndex& idx = idx_of(h);
    const DeTree& t = idx.trees[static_cast<size_t>(tree)];
    const std::span<const float> q(q_proj, static_cast<size_t>(t.K));
    std::vector<uint32_t> got;
    if (exact) {
        std::vector<float> buf(static_cast<size_t>(t.K));
        const ProjectedLookup lookup = [&](uint32_t pos) -> const float* {
            project_point_into(idx.family, idx.data->row(pos), tree, buf.data());
            return buf.data();
        };
        got = range_query_exact(t, idx.table, q, radius, lookup);
    } else {
        range_query_optimized(t, idx.table, q, radius, [&](uint32_t pos) {
            got.push_back(pos);
            return got.size() < limit;
        });
    }
    for (uint64_t i = 0; i < got.size() && i < cap; ++i) out[i] = got[i];
    return got.size();
}

// ck_ann (index.cpp:292-331) for one query; hits written ascending.
int ref_ck_ann(void* h, const float* q, int k, uint32_t* ids, double* dists, int* n_hits,
               double* radius_used, uint64_t* cands_seen) {
    try {
        const DetIndex& idx = idx_of(h);
        QueryResult r = ck_ann(idx, std::span<const float>(q, static_cast<size_t>(idx.d())), k);
        for (size_t i = 0; i < r.hits.size(); ++i) {
            ids[i] = r.hits[i].first;
            dists[i] = r.hits[i].second;
        }
        *n_hits = static_cast<int>(r.hits.size());
        *radius_used = r.radius_used;
        *cands_seen = r.candidates_seen;
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// Batched ck_ann over `threads` std::threads (the index is immutable and
// concurrent ck_ann is safe, README.md:138-139).  Row-major outputs [nq][k].
int ref_ck_ann_batch(void* h, const float* Q, uint64_t nq, int k, int threads, uint32_t* ids,
                     double* dists, int32_t* n_hits, double* radius_used, uint64_t* cands_seen,
                     double* seconds) {
    const DetIndex& idx = idx_of(h);
    const size_t d = static_cast<size_t>(idx.d());
    std::atomic<uint64_t> next{0};
    std::atomic<int> failed{0};
    auto worker = [&]() {
        for (;;) {
            const uint64_t qi = next.fetch_add(1);
            if (qi >= nq) return;
            try {
                QueryResult r = ck_ann(idx, std::span<const float>(Q + qi * d, d), k);
                for (size_t i = 0; i < r.hits.size(); ++i) {
                    ids[qi * k + i] = r.hits[i].first;
                    dists[qi * k + i] = r.hits[i].second;
                }
                n_hits[qi] = static_cast<int32_t>(r.hits.size());
                radius_used[qi] = r.radius_used;
                cands_seen[qi] = r.candidates_seen;
            } catch (...) {
                failed = 1;
            }
        }
    };
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int t = 0; t < std::max(1, threads); ++t) pool.emplace_back(worker);
    for (auto& th : pool) th.join();
    auto t1 = std::chrono::steady_clock::now();
    if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
    return failed.load();
}

// metrics.cpp:8-33 brute force kNN (positions/dists row-major [nq][k]).
int ref_brute_force_knn(const float* data, uint64_t n, int32_t d, const float* Q, uint64_t nq,
                        int k, uint32_t* ids, double* dists) {
    try {
        Dataset ds;
        ds.n = n;
        ds.d = d;
        ds.values.assign(data, data + n * static_cast<uint64_t>(d));
        Dataset qs;
        qs.n = nq;
        qs.d = d;
        qs.values.assign(Q, Q + nq * static_cast<uint64_t>(d));
        GroundTruth gt = brute_force_knn(ds, qs, k);
        std::copy(gt.positions.begin(), gt.positions.end(), ids);
        std::copy(gt.distances.begin(), gt.distances.end(), dists);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// DETL v1 serialization of an index (persist.cpp:99-149) into a caller buffer.
uint64_t ref_index_save(void* h, uint8_t* out, uint64_t cap) {
    std::ostringstream s;
    save_index(idx_of(h), s);
    const std::string b = s.str();
    if (out && cap >= b.size()) std::memcpy(out, b.data(), b.size());
    return b.size();
}

// detlsh::build_det_only_index (index.cpp:220-232): PAA projection, L = 1.
void* ref_build_det_only_index(const float* data, uint64_t n, int32_t d, ref_params* params, uint64_t seed) {
    try {
        auto* h = new RefIndex{build_det_only_index(make_dataset(data, n, d), to_lsh(params), seed)};
        from_lsh(h->index.params, params);
        return h;
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

// detlsh::rc_ann (index.cpp:267-290): 1 found / 0 none / -1 error.
int ref_rc_ann(void* h, const float* q, double r, double c, uint32_t* pos, double* dist) {
    try {
        const auto& idx = static_cast<RefIndex*>(h)->index;
        const auto best = rc_ann(idx, std::span<const float>(q, static_cast<size_t>(idx.d())), r, c);
        if (!best) return 0;
        *pos = best->first;
        *dist = best->second;
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// detlsh::load_index (persist.cpp:157-246) of a DETL v1 byte stream against a
// dataset; nullptr with the message in ref_last_error on FormatError.
void* ref_index_load(const uint8_t* bytes, uint64_t size, const float* data, uint64_t n, int32_t d) {
    try {
        std::istringstream in(std::string(reinterpret_cast<const char*>(bytes), size), std::ios::binary);
        return new RefIndex{load_index(in, make_dataset(data, n, d))};
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

}  // extern "C"
