// Index orchestration (build_index / ck_ann) and the extern "C" boundary
// declared in include/detlsh_b200.h.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/detlsh_b200.h"
#include "common.cuh"
#include "host_core.hpp"
#include "index.cuh"
#include "vecio.cuh"
#include "gt.cuh"
#include "query.cuh"
#include "sharded.cuh"
#include "stages.cuh"
#include "tree.cuh"

namespace detlsh_b200 {

void synth_generate(int kind, uint64_t seed, uint64_t row0, uint64_t n, int d, float* out, cudaStream_t s);

int sm_count(int device) {
    static int cached[64] = {0};
    if (device >= 0 && device < 64 && cached[device]) return cached[device];
    int v = 0;
    DETLSH_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device));
    if (device >= 0 && device < 64) cached[device] = v;
    return v;
}

namespace {

thread_local std::string g_last_error;

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return DETLSH_OK;
    } catch (const InvalidArgument& e) {
        g_last_error = e.what();
        return DETLSH_E_INVALID;
    } catch (const std::invalid_argument& e) {
        g_last_error = e.what();
        return DETLSH_E_INVALID;
    } catch (const CudaError& e) {
        g_last_error = e.what();
        return DETLSH_E_CUDA;
    } catch (const FormatError& e) {
        g_last_error = e.what();
        return DETLSH_E_FORMAT;
    } catch (const std::bad_alloc& e) {
        g_last_error = std::string("out of host memory: ") + e.what();
        return DETLSH_E_CUDA;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return DETLSH_E_CUDA;
    }
}

// Copies between caller buffers (host or device per flags) and device memory.
void to_device(void* dst, const void* src, size_t bytes, bool src_dev, cudaStream_t s) {
    DETLSH_CUDA(cudaMemcpyAsync(dst, src, bytes, src_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s));
}
void from_device(void* dst, const void* src, size_t bytes, bool dst_dev, cudaStream_t s) {
    DETLSH_CUDA(cudaMemcpyAsync(dst, src, bytes, dst_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, s));
}

}  // namespace
}  // namespace detlsh_b200

using namespace detlsh_b200;

struct detlsh_gpu_index {
    std::unique_ptr<GpuIndex> impl;
};
struct detlsh_gpu_sharded_index {
    std::unique_ptr<ShardedIndex> impl;
    // borrowed per-shard handles (own nothing: release() before destruction)
    std::vector<std::unique_ptr<detlsh_gpu_index>> views;
    ~detlsh_gpu_sharded_index() {
        for (auto& v : views) (void)v->impl.release();
    }
};
struct detlsh_gpu_tree {
    std::unique_ptr<DevTree> impl;
    int device = 0;
};

extern "C" {

const char* detlsh_gpu_last_error(void) { return g_last_error.c_str(); }
const char* detlsh_version(void) { return "detlsh_b200 0.1 (sm_100a)"; }

uint64_t detlsh_candidate_budget(double beta, uint64_t n, int32_t k) {
    return candidate_budget(beta, n, k);
}

int detlsh_derive_params(int32_t K, double c, int32_t L, double* out4) {
    return guarded([&] {
        const Derived d = derive_params(K, c, L);
        out4[0] = d.alpha1;
        out4[1] = d.alpha2;
        out4[2] = d.epsilon;
        out4[3] = d.beta;
    });
}

int detlsh_sample_hash_family(int32_t d, int32_t K, int32_t L, uint64_t seed, float* out) {
    return guarded([&] { sample_hash_family(d, K, L, seed, out); });
}

double detlsh_chi2_cdf(double x, int32_t k) {
    try {
        return chi2_cdf(x, k);
    } catch (...) {
        return NAN;
    }
}
double detlsh_chi2_quantile(double a, int32_t k) {
    try {
        return chi2_quantile(a, k);
    } catch (...) {
        return NAN;
    }
}

int detlsh_select_row_breakpoints(float* sample, uint64_t n_s, int32_t n_regions,
                                  uint64_t rng_seed, float* row, uint64_t* draws) {
    return guarded([&] {
        if (!is_pow2(n_regions) || n_regions < 2)
            throw InvalidArgument("select_row_breakpoints: n_regions must be a power of two >= 2");
        if (n_s < static_cast<uint64_t>(n_regions))
            throw InvalidArgument("select_row_breakpoints: sample smaller than region count");
        Rng rng(rng_seed);
        uint64_t nd = 0;
        select_row_breakpoints(sample, n_s, n_regions, rng, row, &nd);
        if (draws) *draws = nd;
    });
}

uint64_t detlsh_launch_count(void) { return launch_count(); }
void detlsh_query_phase_cycles(double* out6) { last_query_phases(out6); }
int detlsh_test_tc_gemm_u8(const uint8_t* A, const uint8_t* B, int32_t N, int32_t K, int32_t* C) {
    return guarded([&] { tc_gemm_u8_test(A, B, N, K, C); });
}
void detlsh_profile_enable(int32_t on) { profile_enable(on != 0); }
int detlsh_profile_collect(char* names, int32_t names_cap, double* ms, uint64_t* launches,
                           int32_t cap) {
    return profile_collect(names, names_cap, ms, launches, cap);
}

int detlsh_device_count(void) {
    int c = 0;
    if (cudaGetDeviceCount(&c) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return c;
}

int detlsh_gpu_build(const float* points, uint64_t n, int32_t d, detlsh_params* params,
                     uint64_t seed, int32_t device, uint32_t flags, detlsh_gpu_index** out) {
    return guarded([&] {
        if (!out) throw InvalidArgument("build_index: out is null");
        *out = nullptr;
        auto X = build_index_impl(points, n, d, params, nullptr, 0, seed, device, flags);
        *out = new detlsh_gpu_index{std::move(X)};
    });
}

int detlsh_gpu_build_with_family(const float* points, uint64_t n, int32_t d,
                                 detlsh_params* params, const float* coeffs, int32_t K,
                                 int32_t L, uint64_t family_seed, uint64_t seed, int32_t device,
                                 uint32_t flags, detlsh_gpu_index** out) {
    return guarded([&] {
        if (!out || !params || !coeffs) throw InvalidArgument("build_index: null argument");
        *out = nullptr;
        params->K = K;  // the family's K / L win (index.cpp:199-200)
        params->L = L;
        auto X = build_index_impl(points, n, d, params, coeffs, family_seed, seed, device, flags);
        *out = new detlsh_gpu_index{std::move(X)};
    });
}

void detlsh_gpu_free(detlsh_gpu_index* index) {
    if (!index) return;
    try {
        DeviceGuard dg(index->impl->device);
        delete index;
    } catch (...) {
        delete index;
    }
}

int detlsh_gpu_query(const detlsh_gpu_index* index, const float* queries, uint64_t nq,
                     int32_t k, uint32_t flags, uint32_t* ids, double* dists, int32_t* n_hits,
                     double* radius_used, uint64_t* cands_seen, void* stream) {
    return guarded([&] {
        if (!index) throw InvalidArgument("ck_ann: index is null");
        query_impl(*index->impl, queries, nq, k, flags, ids, dists, n_hits, radius_used,
                   cands_seen, static_cast<cudaStream_t>(stream));
    });
}

int detlsh_gpu_query_check(const detlsh_gpu_index* index, void* stream) {
    return guarded([&] {
        if (!index) throw InvalidArgument("ck_ann: index is null");
        GpuIndex& X = *index->impl;
        DeviceGuard dg(X.device);
        std::lock_guard<std::mutex> lock(X.qmu);
        cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : X.main.s;
        if (query_invariant_failed(X.scratch, s))
            throw CudaError("ck_ann: internal invariant violated (budget cut emitted != budget rows)");
    });
}

int detlsh_gpu_synth(int32_t kind, uint64_t seed, uint64_t row0, uint64_t n, int32_t d, float* out, int32_t device,
                     void* stream) {
    return guarded([&] {
        if (!out && n) throw InvalidArgument("synth: out is null");
        DeviceGuard dg(device);
        synth_generate(kind, seed, row0, n, d, out, static_cast<cudaStream_t>(stream));
        if (!stream) DETLSH_CUDA(cudaStreamSynchronize(nullptr));
    });
}

int detlsh_gpu_estimate_rmin(const detlsh_gpu_index* index, const float* probes, uint64_t n_probes, int32_t k,
                             uint32_t flags, double* r_min) {
    return guarded([&] {
        if (!index) throw InvalidArgument("estimate_rmin: index is null");
        if (!r_min) throw InvalidArgument("estimate_rmin: r_min is null");
        *r_min = estimate_rmin_impl(*index->impl, probes, n_probes, k, flags);
    });
}

int detlsh_gpu_project_query(const detlsh_gpu_index* index, const float* queries, uint64_t nq, float* out,
                             uint32_t flags) {
    return guarded([&] {
        if (!index) throw InvalidArgument("project_query: index is null");
        project_queries_impl(*index->impl, queries, nq, out, flags);
    });
}

int detlsh_gpu_range_query(const detlsh_gpu_index* index, int32_t tree, const float* q_proj, uint64_t nq,
                           const double* radius, uint64_t limit, uint32_t flags, uint32_t* positions, uint64_t cap,
                           uint64_t* counts) {
    return guarded([&] {
        if (!index) throw InvalidArgument("range_query: index is null");
        if (flags & DETLSH_F_DEVICE_PTRS) throw InvalidArgument("range_query: host pointers only");
        range_query_impl(*index->impl, tree, q_proj, nq, radius, limit, (flags & DETLSH_RANGE_EXACT) != 0, positions,
                         cap, counts);
    });
}

int detlsh_gpu_sharded_build(const float* points, uint64_t n, int32_t d, detlsh_params* params, uint64_t seed,
                             const int32_t* devices, int32_t shards, uint32_t flags,
                             detlsh_gpu_sharded_index** out) {
    return guarded([&] {
        if (!out) throw InvalidArgument("build_index: out is null");
        *out = nullptr;
        auto h = std::make_unique<detlsh_gpu_sharded_index>();
        h->impl = sharded_build(points, n, d, params, seed, devices, shards, flags);
        for (auto& sh : h->impl->shards) {
            h->views.push_back(std::make_unique<detlsh_gpu_index>());
            h->views.back()->impl.reset(sh.get());
        }
        *out = h.release();
    });
}

int detlsh_gpu_sharded_query(detlsh_gpu_sharded_index* index, const float* queries, uint64_t nq, int32_t k,
                             uint32_t flags, uint64_t* ids, double* dists, int32_t* n_hits, void* stream) {
    return guarded([&] {
        if (!index) throw InvalidArgument("ck_ann: index is null");
        sharded_query(*index->impl, queries, nq, k, flags, ids, dists, n_hits, static_cast<cudaStream_t>(stream));
    });
}

int32_t detlsh_gpu_sharded_count(const detlsh_gpu_sharded_index* index) {
    return index ? static_cast<int32_t>(index->views.size()) : 0;
}

const detlsh_gpu_index* detlsh_gpu_sharded_shard(const detlsh_gpu_sharded_index* index, int32_t s,
                                                 uint64_t* row_begin, uint64_t* row_end) {
    if (!index || s < 0 || s >= static_cast<int32_t>(index->views.size())) return nullptr;
    if (row_begin) *row_begin = index->impl->offsets[s];
    if (row_end) *row_end = index->impl->offsets[s + 1];
    return index->views[s].get();
}

void detlsh_gpu_sharded_free(detlsh_gpu_sharded_index* index) { delete index; }

int detlsh_gpu_rc_ann(const detlsh_gpu_index* index, const float* queries, uint64_t nq, double r,
                      double c, uint32_t flags, uint32_t* ids, double* dists, int32_t* found,
                      uint64_t* cands_seen, void* stream) {
    return guarded([&] {
        if (!index) throw InvalidArgument("rc_ann: index is null");
        const RcArgs rc{r, c};
        query_impl(*index->impl, queries, nq, 1, flags, ids, dists, found, nullptr, cands_seen,
                   static_cast<cudaStream_t>(stream), &rc);
    });
}

int detlsh_gpu_brute_force_knn(const float* data, uint64_t n, int32_t d, const float* queries, uint64_t nq,
                               int32_t k, const double* dist2_bound, uint32_t flags, uint32_t* ids,
                               double* dists, int32_t device, void* stream) {
    return guarded([&] {
        if (!data || !queries || !ids || !dists) throw InvalidArgument("brute_force_knn: null pointer");
        if (d < 1 || n == 0) throw InvalidArgument("brute_force_knn: empty dataset");
        DeviceGuard dg(device);
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        StreamScope scope(s);
        if (flags & DETLSH_F_DEVICE_PTRS) {
            brute_force_knn_gpu(data, n, d, queries, nq, k, dist2_bound, ids, dists, device, s);
            return;
        }
        DevBuf<float> X(n * static_cast<size_t>(d)), Q(nq * static_cast<size_t>(d));
        DevBuf<uint32_t> oi(nq * static_cast<size_t>(k));
        DevBuf<double> od(nq * static_cast<size_t>(k));
        DETLSH_CUDA(cudaMemcpyAsync(X.get(), data, X.bytes(), cudaMemcpyHostToDevice, s));
        DETLSH_CUDA(cudaMemcpyAsync(Q.get(), queries, Q.bytes(), cudaMemcpyHostToDevice, s));
        brute_force_knn_gpu(X.get(), n, d, Q.get(), nq, k, dist2_bound, oi.get(), od.get(), device, s);
        DETLSH_CUDA(cudaMemcpyAsync(ids, oi.get(), oi.bytes(), cudaMemcpyDeviceToHost, s));
        DETLSH_CUDA(cudaMemcpyAsync(dists, od.get(), od.bytes(), cudaMemcpyDeviceToHost, s));
        DETLSH_CUDA(cudaStreamSynchronize(s));
    });
}

int detlsh_vectors_shape(const char* path, uint64_t* n, int32_t* d, int32_t* kind) {
    return guarded([&] {
        const int k = vec_kind_from_path(path);
        int dd = 0;
        vectors_shape(path, k, n, &dd);
        *d = dd;
        if (kind) *kind = k;
    });
}

int detlsh_gpu_read_vectors(const char* path, float* values, uint64_t n, int32_t d, int32_t device,
                            void* stream) {
    return guarded([&] {
        DeviceGuard dg(device);
        read_vectors_into(path, vec_kind_from_path(path), values, n, d, static_cast<cudaStream_t>(stream));
    });
}

int detlsh_gpu_merge_topk(const double* shard_dists, const uint64_t* shard_ids,
                          const int32_t* shard_hits, int32_t shards, uint64_t nq, int32_t k,
                          double* out_dists, uint64_t* out_ids, int32_t* out_hits, void* stream) {
    return guarded([&] {
        launch_merge_topk(shard_dists, shard_ids, shard_hits, shards, nq, k, out_dists, out_ids,
                          out_hits, static_cast<cudaStream_t>(stream));
    });
}

int detlsh_gpu_get_params(const detlsh_gpu_index* index, detlsh_params* out) {
    return guarded([&] { *out = index->impl->params; });
}
uint64_t detlsh_gpu_n(const detlsh_gpu_index* index) { return index ? index->impl->n : 0; }
int32_t detlsh_gpu_d(const detlsh_gpu_index* index) { return index ? index->impl->d : 0; }
uint64_t detlsh_gpu_family_seed(const detlsh_gpu_index* index) { return index ? index->impl->family_seed : 0; }
int32_t detlsh_gpu_has_family(const detlsh_gpu_index* index) { return index && !index->impl->paa ? 1 : 0; }
int32_t detlsh_gpu_row_u8(const detlsh_gpu_index* index) {
    return index ? index->impl->row_u8 : 0;
}
uint64_t detlsh_gpu_sample_size(const detlsh_gpu_index* index) {
    return index ? index->impl->sample_size : 0;
}

int detlsh_gpu_export_family(const detlsh_gpu_index* index, float* out) {
    return guarded([&] {
        const auto& c = index->impl->h_coeffs;
        std::copy(c.begin(), c.end(), out);
    });
}

int detlsh_gpu_export_table(const detlsh_gpu_index* index, float* out) {
    return guarded([&] {
        const auto& t = index->impl->h_table;
        std::copy(t.begin(), t.end(), out);
    });
}

int detlsh_gpu_export_codes(const detlsh_gpu_index* index, uint8_t* out) {
    return guarded([&] {
        const GpuIndex& X = *index->impl;
        if (!X.codes.get()) throw InvalidArgument("export_codes: codes were dropped (DETLSH_F_NO_CODES)");
        DeviceGuard dg(X.device);
        DETLSH_CUDA(cudaMemcpy(out, X.codes.get(), X.codes.size(), cudaMemcpyDeviceToHost));
    });
}

int detlsh_gpu_tree_num_nodes(const detlsh_gpu_index* index, int32_t tree, uint64_t* out) {
    return guarded([&] {
        if (tree < 0 || tree >= index->impl->params.L) throw InvalidArgument("tree index out of range");
        *out = index->impl->trees[tree]->num_nodes;
    });
}

static void copy_export(const HostTreeExport& e, int32_t* root_children, uint8_t* is_leaf,
                        uint8_t* split_dim, int32_t* left, int32_t* right, uint8_t* bits,
                        uint8_t* value, uint64_t* ebegin, uint32_t* ecount, uint32_t* positions) {
    auto cp = [](auto& v, auto* dst) {
        if (dst) std::copy(v.begin(), v.end(), dst);
    };
    cp(e.root_children, root_children);
    cp(e.is_leaf, is_leaf);
    cp(e.split_dim, split_dim);
    cp(e.left, left);
    cp(e.right, right);
    cp(e.bits, bits);
    cp(e.value, value);
    cp(e.ebegin, ebegin);
    cp(e.ecount, ecount);
    cp(e.positions, positions);
}

int detlsh_gpu_export_tree(const detlsh_gpu_index* index, int32_t tree, int32_t* root_children,
                           uint8_t* is_leaf, uint8_t* split_dim, int32_t* left, int32_t* right,
                           uint8_t* bits, uint8_t* value, uint64_t* ebegin, uint32_t* ecount,
                           uint32_t* positions) {
    return guarded([&] {
        const GpuIndex& X = *index->impl;
        if (tree < 0 || tree >= X.params.L) throw InvalidArgument("tree index out of range");
        DeviceGuard dg(X.device);
        HostTreeExport e;
        export_tree(*X.trees[tree], e);
        copy_export(e, root_children, is_leaf, split_dim, left, right, bits, value, ebegin, ecount,
                    positions);
    });
}

int detlsh_gpu_save_detl(detlsh_gpu_index* index, uint8_t* out, uint64_t cap, uint64_t* size) {
    return guarded([&] {
        GpuIndex& X = *index->impl;
        std::lock_guard<std::mutex> lock(X.qmu);
        const std::vector<uint8_t> b = save_detl(X);
        if (size) *size = b.size();
        if (out) {
            if (cap < b.size()) throw InvalidArgument("save_index: output buffer too small");
            std::memcpy(out, b.data(), b.size());
        }
    });
}

int detlsh_gpu_build_timings(const detlsh_gpu_index* index, double* ms, int32_t cap, char* names,
                             int32_t names_cap) {
    const auto& t = index->impl->timings;
    std::string all;
    const int m = std::min<int>(cap, static_cast<int>(t.size()));
    for (int i = 0; i < m; ++i) {
        ms[i] = t[i].second;
        all += t[i].first;
        if (i + 1 < m) all += ";";
    }
    if (names && names_cap > 0) {
        std::strncpy(names, all.c_str(), static_cast<size_t>(names_cap) - 1);
        names[names_cap - 1] = 0;
    }
    return m;
}

int detlsh_gpu_project(const float* coeffs, int32_t K, int32_t L, const float* points,
                       uint64_t n, int32_t d, float* out, int32_t device, uint32_t flags) {
    return guarded([&] {
        if (K < 1 || L < 1 || d < 1 || n == 0) throw InvalidArgument("project_dataset: bad shape");
        DeviceGuard dg(device);
        const bool dev = flags & DETLSH_F_DEVICE_PTRS;
        cudaStream_t s = nullptr;
        const size_t LK = static_cast<size_t>(K) * L;
        DevBuf<float> c(LK * d), pts, o;
        to_device(c.get(), coeffs, LK * d * 4, dev, s);
        const float* P = points;
        if (!dev) {
            pts.alloc(n * d);
            to_device(pts.get(), points, n * d * 4, false, s);
            P = pts.get();
        }
        float* O = out;
        if (!dev) {
            o.alloc(LK * n);
            O = o.get();
        }
        DevBuf<double> ct(static_cast<size_t>(lk_padded(static_cast<int>(LK))) * d);
        prepare_coeffs_t(c.get(), static_cast<int>(LK), d, ct.get(), s);
        ProjTc tc;
        prepare_proj_tc(c.get(), static_cast<int>(LK), d, tc, s);
        launch_project_exact(P, n, d, ct.get(), K, L, O, s, "project_exact", &tc);
        if (!dev) from_device(out, O, LK * n * 4, false, s);
        DETLSH_CUDA(cudaStreamSynchronize(s));
    });
}

int detlsh_gpu_select_breakpoints(const float* projected, uint64_t n, int32_t K, int32_t L,
                                  int32_t n_regions, double sample_fraction, uint64_t seed,
                                  float* table, uint64_t* sample_size, int32_t device,
                                  uint32_t flags) {
    return guarded([&] {
        if (!is_pow2(n_regions) || n_regions < 2 || n_regions > 256)
            throw InvalidArgument("select_breakpoints: n_regions must be a power of two in [2, 256]");
        if (!(sample_fraction > 0.0) || sample_fraction > 1.0)
            throw InvalidArgument("select_breakpoints: sample_fraction must lie in (0, 1]");
        if (K < 1 || L < 1 || n == 0) throw InvalidArgument("select_breakpoints: bad shape");
        DeviceGuard dg(device);
        ensure_mempool(device);
        const bool dev = flags & DETLSH_F_DEVICE_PTRS;
        const uint64_t n_s = sample_size_for(sample_fraction, n, n_regions);
        OwnedStream os;  // declared before the buffers freed on it
        os.create();
        cudaStream_t st = os.s;
        StreamScope sc(st);
        DevBuf<float> pr;
        const float* P = projected;
        const size_t total = static_cast<size_t>(L) * n * K;
        if (!dev) {
            pr.alloc(total);
            to_device(pr.get(), projected, total * 4, false, st);
            P = pr.get();
        }
        const size_t W = static_cast<size_t>(n_regions) + 1;
        DevBuf<float> d_table(static_cast<size_t>(L) * K * W);
        // `seed` is select_breakpoints' own seed argument (index.cpp passes
        // mix_seed(seed, 1)); the GPU-native mode derives one key per space.
        if (flags & DETLSH_F_SAMPLE_GPU) {
            DevBuf<uint32_t> d_idx(n_s);
            DevBuf<float> rows(static_cast<size_t>(L) * K * n_s);
            for (int i = 0; i < L; ++i) {
                launch_feistel_sample(n, n_s, mix_seed(seed, static_cast<uint64_t>(i)), d_idx.get(), st);
                launch_gather_sample(P + static_cast<size_t>(i) * n * K, d_idx.get(), n_s, K,
                                     rows.get() + static_cast<size_t>(i) * K * n_s, st);
            }
            gpu_order_stat_table(rows.get(), L * K, n_s, n_regions, d_table.get(), st);
        } else {
            RefSampler sampler(n, n_s, n_regions, seed);
            DevBuf<uint32_t> d_idx(n_s);
            DevBuf<float> d_sample(static_cast<size_t>(K) * n_s);
            std::vector<float> h_sample(static_cast<size_t>(K) * n_s);
            std::vector<float> h_table(static_cast<size_t>(L) * K * W, 0.0f);
            for (int i = 0; i < L; ++i) {
                const auto& idx = sampler.next_space_indices();
                DETLSH_CUDA(cudaMemcpyAsync(d_idx.get(), idx.data(), n_s * 4, cudaMemcpyHostToDevice, st));
                launch_gather_sample(P + static_cast<size_t>(i) * n * K, d_idx.get(), n_s, K,
                                     d_sample.get(), st);
                DETLSH_CUDA(cudaMemcpyAsync(h_sample.data(), d_sample.get(), h_sample.size() * 4,
                                            cudaMemcpyDeviceToHost, st));
                DETLSH_CUDA(cudaStreamSynchronize(st));
                for (int j = 0; j < K; ++j)
                    sampler.select_row(h_sample.data() + static_cast<size_t>(j) * n_s,
                                       h_table.data() + (static_cast<size_t>(i) * K + j) * W);
            }
            DETLSH_CUDA(cudaMemcpyAsync(d_table.get(), h_table.data(), h_table.size() * 4,
                                        cudaMemcpyHostToDevice, st));
            DETLSH_CUDA(cudaStreamSynchronize(st));
        }
        from_device(table, d_table.get(), d_table.bytes(), dev, st);
        DETLSH_CUDA(cudaStreamSynchronize(st));
        if (sample_size) *sample_size = n_s;
    });
}

int detlsh_gpu_encode(const float* projected, uint64_t n, int32_t K, int32_t L,
                      const float* table, int32_t n_regions, uint8_t* out, int32_t device,
                      uint32_t flags) {
    return guarded([&] {
        if (K < 1 || L < 1 || n == 0 || !is_pow2(n_regions) || n_regions > 256)
            throw InvalidArgument("encode_dataset: bad shape");
        DeviceGuard dg(device);
        const bool dev = flags & DETLSH_F_DEVICE_PTRS;
        cudaStream_t s = nullptr;
        const size_t total = static_cast<size_t>(L) * n * K;
        const size_t tsz = static_cast<size_t>(L) * K * (n_regions + 1);
        DevBuf<float> pr, tb;
        DevBuf<uint8_t> o;
        const float* P = projected;
        const float* T = table;
        uint8_t* O = out;
        if (!dev) {
            pr.alloc(total);
            tb.alloc(tsz);
            o.alloc(total);
            to_device(pr.get(), projected, total * 4, false, s);
            to_device(tb.get(), table, tsz * 4, false, s);
            P = pr.get();
            T = tb.get();
            O = o.get();
        }
        launch_encode(P, n, K, L, T, n_regions, O, s);
        if (!dev) from_device(out, O, total, false, s);
        DETLSH_CUDA(cudaStreamSynchronize(s));
    });
}

int detlsh_gpu_build_tree(const uint8_t* codes, uint64_t n, int32_t K, int32_t L,
                          int32_t n_regions, int32_t space, int32_t max_size, int32_t device,
                          uint32_t flags, detlsh_gpu_tree** out) {
    return guarded([&] {
        if (!out) throw InvalidArgument("build_tree: out is null");
        *out = nullptr;
        if (space < 0 || space >= L) throw InvalidArgument("build_tree: space index out of range");
        DeviceGuard dg(device);
        const bool dev = flags & DETLSH_F_DEVICE_PTRS;
        cudaStream_t s = nullptr;
        DevBuf<uint8_t> c;
        const uint8_t* C = codes + static_cast<size_t>(space) * n * K;
        if (!dev) {
            c.alloc(n * static_cast<size_t>(K));
            to_device(c.get(), C, n * static_cast<size_t>(K), false, s);
            C = c.get();
        }
        auto T = std::make_unique<DevTree>();
        build_tree_gpu(C, n, K, n_regions, space, max_size, *T, s);
        DETLSH_CUDA(cudaStreamSynchronize(s));
        *out = new detlsh_gpu_tree{std::move(T), device};
    });
}

int detlsh_gpu_tree_nodes(const detlsh_gpu_tree* tree, uint64_t* out) {
    return guarded([&] { *out = tree->impl->num_nodes; });
}

int detlsh_gpu_tree_export(const detlsh_gpu_tree* tree, int32_t* root_children, uint8_t* is_leaf,
                           uint8_t* split_dim, int32_t* left, int32_t* right, uint8_t* bits,
                           uint8_t* value, uint64_t* ebegin, uint32_t* ecount,
                           uint32_t* positions) {
    return guarded([&] {
        DeviceGuard dg(tree->device);
        HostTreeExport e;
        export_tree(*tree->impl, e);
        copy_export(e, root_children, is_leaf, split_dim, left, right, bits, value, ebegin, ecount,
                    positions);
    });
}

void detlsh_gpu_tree_free(detlsh_gpu_tree* tree) { delete tree; }

}  // extern "C"
