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
#include "query.cuh"
#include "stages.cuh"
#include "tree.cuh"

namespace detlsh_b200 {

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

using Clock = std::chrono::steady_clock;
double ms_since(Clock::time_point t0) {
    return std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
}

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        DETLSH_CUDA(cudaGetDevice(&prev));
        if (prev != dev) DETLSH_CUDA(cudaSetDevice(dev));
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

bool is_pow2(int v) { return v > 0 && (v & (v - 1)) == 0; }

void validate(const detlsh_params& p, uint64_t n, int d) {
    // validate_params (index.cpp:16-24) + stage preconditions
    if (n == 0) throw InvalidArgument("build_index: empty dataset");
    if (d < 1) throw InvalidArgument("build_index: d must be positive");
    if (n > 0xffffffffULL) throw InvalidArgument("build_index: n must be < 2^32 (u32 positions)");
    if (p.K < 1 || p.K > 24) throw InvalidArgument("build_index: K must lie in [1, 24]");
    if (p.L < 1) throw InvalidArgument("build_index: L must be positive");
    if (!(p.c > 1.0)) throw InvalidArgument("build_index: c must exceed 1");
    if (p.leaf_capacity < 1) throw InvalidArgument("build_index: leaf_capacity must be positive");
    if (!is_pow2(p.n_regions) || p.n_regions < 2 || p.n_regions > 256)
        throw InvalidArgument("select_breakpoints: n_regions must be a power of two in [2, 256]");
    if (!(p.sample_fraction > 0.0) || p.sample_fraction > 1.0)
        throw InvalidArgument("select_breakpoints: sample_fraction must lie in (0, 1]");
    uint64_t n_s = static_cast<uint64_t>(std::ceil(p.sample_fraction * static_cast<double>(n)));
    n_s = std::max<uint64_t>(n_s, static_cast<uint64_t>(p.n_regions));
    if (n_s > n) throw InvalidArgument("select_breakpoints: sample too small for region count");
}

uint64_t sample_size_for(double frac, uint64_t n, int NR) {
    uint64_t n_s = static_cast<uint64_t>(std::ceil(frac * static_cast<double>(n)));
    n_s = std::max<uint64_t>(n_s, static_cast<uint64_t>(NR));
    if (n_s > n) throw InvalidArgument("select_breakpoints: sample too small for region count");
    return n_s;
}

}  // namespace

struct GpuIndex {
    int device = 0;
    cudaStream_t stream = nullptr;
    detlsh_params params{};
    uint64_t n = 0;
    int d = 0;
    uint64_t family_seed = 0, sample_size = 0;
    bool sample_gpu = false;
    const float* data = nullptr;  // device
    DevBuf<float> data_buf;
    std::vector<float> h_coeffs;  // [L][K][d]
    DevBuf<float> coeffs;
    DevBuf<double> coeffs_t;
    DevBuf<float> table;
    std::vector<float> h_table;
    DevBuf<uint8_t> codes;
    std::vector<std::unique_ptr<DevTree>> trees;
    DevBuf<QTree> qtrees;
    uint32_t max_leaves = 0;
    QueryScratch scratch;
    std::mutex qmu;
    std::vector<std::pair<std::string, double>> timings;

    ~GpuIndex() {
        if (stream) cudaStreamDestroy(stream);
    }
};

namespace {

// Breakpoints in the reference-compatible mode: the host replays the shared
// RNG stream (encoder.cpp:105-143) on exact sample values gathered on device.
void breakpoints_ref(GpuIndex& X, const float* d_proj, uint64_t seed) {
    const int K = X.params.K, L = X.params.L, NR = X.params.n_regions;
    const uint64_t n = X.n, n_s = X.sample_size;
    const size_t W = static_cast<size_t>(NR) + 1;
    RefSampler sampler(n, n_s, NR, mix_seed(seed, kStreamBreakpoints));
    DevBuf<uint32_t> d_idx(n_s);
    DevBuf<float> d_sample(static_cast<size_t>(K) * n_s);
    float* h_sample = nullptr;
    DETLSH_CUDA(cudaMallocHost(&h_sample, static_cast<size_t>(K) * n_s * sizeof(float)));
    std::unique_ptr<float, decltype(&cudaFreeHost)> guard(h_sample, &cudaFreeHost);
    X.h_table.assign(static_cast<size_t>(L) * K * W, 0.0f);
    for (int i = 0; i < L; ++i) {
        const auto& idx = sampler.next_space_indices();
        DETLSH_CUDA(cudaMemcpyAsync(d_idx.get(), idx.data(), n_s * 4, cudaMemcpyHostToDevice, X.stream));
        launch_gather_sample(d_proj + static_cast<size_t>(i) * n * K, d_idx.get(), n_s, K,
                             d_sample.get(), X.stream);
        DETLSH_CUDA(cudaMemcpyAsync(h_sample, d_sample.get(), static_cast<size_t>(K) * n_s * 4,
                                    cudaMemcpyDeviceToHost, X.stream));
        DETLSH_CUDA(cudaStreamSynchronize(X.stream));
        for (int j = 0; j < K; ++j)
            sampler.select_row(h_sample + static_cast<size_t>(j) * n_s,
                               X.h_table.data() + (static_cast<size_t>(i) * K + j) * W);
    }
    DETLSH_CUDA(cudaMemcpyAsync(X.table.get(), X.h_table.data(), X.h_table.size() * 4,
                                cudaMemcpyHostToDevice, X.stream));
}

// GPU-native sample: per-space Feistel sample + exact order statistics.
void breakpoints_gpu(GpuIndex& X, const float* d_proj, uint64_t seed) {
    const int K = X.params.K, L = X.params.L, NR = X.params.n_regions;
    const uint64_t n = X.n, n_s = X.sample_size;
    DevBuf<uint32_t> d_idx(n_s);
    DevBuf<float> rows(static_cast<size_t>(L) * K * n_s);
    const uint64_t bseed = mix_seed(seed, kStreamBreakpoints);
    for (int i = 0; i < L; ++i) {
        launch_feistel_sample(n, n_s, mix_seed(bseed, static_cast<uint64_t>(i)), d_idx.get(), X.stream);
        launch_gather_sample(d_proj + static_cast<size_t>(i) * n * K, d_idx.get(), n_s, K,
                             rows.get() + static_cast<size_t>(i) * K * n_s, X.stream);
    }
    gpu_order_stat_table(rows.get(), L * K, n_s, NR, X.table.get(), X.stream);
    X.h_table.resize(static_cast<size_t>(L) * K * (NR + 1));
    DETLSH_CUDA(cudaMemcpyAsync(X.h_table.data(), X.table.get(), X.h_table.size() * 4,
                                cudaMemcpyDeviceToHost, X.stream));
}

// r_min (index.cpp:75-136, 153-175) via per-probe order statistics.
double estimate_rmin_gpu(GpuIndex& X, const float* d_proj, uint64_t seed) {
    const int K = X.params.K, L = X.params.L;
    const uint64_t n = X.n;
    Rng rng(mix_seed(seed, kStreamProbes));
    const int np = static_cast<int>(std::min<uint64_t>(10, n));
    std::vector<uint64_t> pos(np);
    for (int p = 0; p < np; ++p) pos[p] = rng.bounded(n);
    DevBuf<float> probe(static_cast<size_t>(np) * L * K);
    for (int p = 0; p < np; ++p)
        for (int i = 0; i < L; ++i)
            DETLSH_CUDA(cudaMemcpyAsync(probe.get() + (static_cast<size_t>(p) * L + i) * K,
                                        d_proj + (static_cast<size_t>(i) * n + pos[p]) * K,
                                        K * sizeof(float), cudaMemcpyDeviceToDevice, X.stream));
    // initial guess: median pairwise distance of 32 strided points (space 0)
    const uint64_t m = std::min<uint64_t>(32, n);
    std::vector<float> sc(m * K);
    for (uint64_t t = 0; t < m; ++t)
        DETLSH_CUDA(cudaMemcpyAsync(sc.data() + t * K, d_proj + (t * n / m) * K, K * sizeof(float),
                                    cudaMemcpyDeviceToHost, X.stream));
    const uint64_t budget = candidate_budget(X.params.beta, n, X.params.k);
    DevBuf<double> D(static_cast<size_t>(np) * n);
    DevBuf<uint32_t> hist(static_cast<size_t>(np) * 65536);
    std::vector<uint64_t> Tbits(np);
    rmin_order_stats(d_proj, n, K, L, probe.get(), np, budget, D.get(), hist.get(), Tbits.data(),
                     X.stream);
    std::vector<double> pd;
    pd.reserve(m * (m - 1) / 2);
    for (uint64_t a = 0; a < m; ++a)
        for (uint64_t b = a + 1; b < m; ++b) {
            double acc = 0.0;
            for (int j = 0; j < K; ++j) {
                const double diff = static_cast<double>(sc[a * K + j]) - static_cast<double>(sc[b * K + j]);
                acc += diff * diff;
            }
            pd.push_back(std::sqrt(acc));
        }
    double guess = 1.0;
    if (!pd.empty()) {
        std::nth_element(pd.begin(), pd.begin() + pd.size() / 2, pd.end());
        const double med = pd[pd.size() / 2];
        if (med > 0.0) guess = med / X.params.epsilon;
    }
    std::vector<double> T(np);
    for (int p = 0; p < np; ++p) std::memcpy(&T[p], &Tbits[p], 8);
    return rmin_from_order_stats(T, guess, X.params.epsilon, X.params.c);
}

std::unique_ptr<GpuIndex> build_index_impl(const float* points, uint64_t n, int d,
                                           detlsh_params* params, const float* coeffs_host,
                                           uint64_t family_seed, uint64_t seed, int device,
                                           uint32_t flags) {
    if (!params) throw InvalidArgument("build_index: params is null");
    if (!points) throw InvalidArgument("build_index: points is null");
    validate(*params, n, d);
    DeviceGuard dg(device);
    auto X = std::make_unique<GpuIndex>();
    X->device = device;
    X->n = n;
    X->d = d;
    X->sample_gpu = (flags & DETLSH_F_SAMPLE_GPU) != 0;
    DETLSH_CUDA(cudaStreamCreateWithFlags(&X->stream, cudaStreamNonBlocking));
    cudaStream_t s = X->stream;
    detlsh_params p = *params;
    const auto t_all = Clock::now();
    auto t0 = Clock::now();
    // derived parameters (index.cpp:202-206)
    const Derived der = derive_params(p.K, p.c, p.L);
    p.alpha1 = der.alpha1;
    p.alpha2 = der.alpha2;
    p.epsilon = der.epsilon;
    if (p.beta <= 0.0) p.beta = der.beta;
    X->params = p;
    const int K = p.K, L = p.L, NR = p.n_regions;
    const int LK = K * L;
    // hash family (projection.cpp:11-23), host, seeded stream 0
    X->h_coeffs.resize(static_cast<size_t>(LK) * d);
    if (coeffs_host) {
        std::memcpy(X->h_coeffs.data(), coeffs_host, X->h_coeffs.size() * sizeof(float));
        X->family_seed = family_seed;
    } else {
        X->family_seed = mix_seed(seed, kStreamFamily);
        sample_hash_family(d, K, L, X->family_seed, X->h_coeffs.data());
    }
    X->timings.emplace_back("host_params_family", ms_since(t0));
    t0 = Clock::now();
    // dataset
    if (flags & DETLSH_F_DEVICE_PTRS) {
        if (flags & DETLSH_F_BORROW_DATA) {
            X->data = points;
        } else {
            X->data_buf.alloc(n * static_cast<size_t>(d));
            DETLSH_CUDA(cudaMemcpyAsync(X->data_buf.get(), points, n * static_cast<size_t>(d) * 4,
                                        cudaMemcpyDeviceToDevice, s));
            X->data = X->data_buf.get();
        }
    } else {
        X->data_buf.alloc(n * static_cast<size_t>(d));
        DETLSH_CUDA(cudaMemcpyAsync(X->data_buf.get(), points, n * static_cast<size_t>(d) * 4,
                                    cudaMemcpyHostToDevice, s));
        X->data = X->data_buf.get();
    }
    X->coeffs.alloc(X->h_coeffs.size());
    DETLSH_CUDA(cudaMemcpyAsync(X->coeffs.get(), X->h_coeffs.data(), X->h_coeffs.size() * 4,
                                cudaMemcpyHostToDevice, s));
    X->coeffs_t.alloc(static_cast<size_t>(lk_padded(LK)) * d);
    prepare_coeffs_t(X->coeffs.get(), LK, d, X->coeffs_t.get(), s);
    DETLSH_CUDA(cudaStreamSynchronize(s));
    X->timings.emplace_back("upload", ms_since(t0));
    // projection (exact)
    t0 = Clock::now();
    DevBuf<float> proj(static_cast<size_t>(L) * n * K);
    launch_project_exact(X->data, n, d, X->coeffs_t.get(), K, L, proj.get(), s);
    DETLSH_CUDA(cudaStreamSynchronize(s));
    X->timings.emplace_back("project", ms_since(t0));
    // breakpoints
    t0 = Clock::now();
    X->sample_size = sample_size_for(p.sample_fraction, n, NR);
    X->table.alloc(static_cast<size_t>(L) * K * (NR + 1));
    if (X->sample_gpu) breakpoints_gpu(*X, proj.get(), seed);
    else breakpoints_ref(*X, proj.get(), seed);
    DETLSH_CUDA(cudaStreamSynchronize(s));
    X->timings.emplace_back("breakpoints", ms_since(t0));
    // encode
    t0 = Clock::now();
    X->codes.alloc(static_cast<size_t>(L) * n * K);
    launch_encode(proj.get(), n, K, L, X->table.get(), NR, X->codes.get(), s);
    DETLSH_CUDA(cudaStreamSynchronize(s));
    X->timings.emplace_back("encode", ms_since(t0));
    // trees
    t0 = Clock::now();
    std::vector<QTree> qt(L);
    for (int i = 0; i < L; ++i) {
        auto T = std::make_unique<DevTree>();
        build_tree_gpu(X->codes.get() + static_cast<size_t>(i) * n * K, n, K, NR, i,
                       p.leaf_capacity, *T, s);
        qt[i] = QTree{T->leaf_node.get(), T->leaf_begin.get(), T->leaf_count.get(),
                      T->leaf_box.get(), T->perm.get(), static_cast<uint32_t>(T->num_leaves)};
        X->max_leaves = std::max<uint32_t>(X->max_leaves, static_cast<uint32_t>(T->num_leaves));
        X->trees.push_back(std::move(T));
    }
    X->qtrees.alloc(L);
    DETLSH_CUDA(cudaMemcpyAsync(X->qtrees.get(), qt.data(), L * sizeof(QTree), cudaMemcpyHostToDevice, s));
    DETLSH_CUDA(cudaStreamSynchronize(s));
    X->timings.emplace_back("trees", ms_since(t0));
    // r_min
    t0 = Clock::now();
    if (X->params.r_min <= 0.0) X->params.r_min = estimate_rmin_gpu(*X, proj.get(), seed);
    X->timings.emplace_back("rmin", ms_since(t0));
    if (flags & DETLSH_F_NO_CODES) X->codes.release();
    X->timings.emplace_back("total", ms_since(t_all));
    *params = X->params;
    return X;
}

void query_impl(GpuIndex& X, const float* queries, uint64_t nq, int k, uint32_t flags,
                uint32_t* ids, double* dists, int32_t* n_hits, double* radius, uint64_t* cands,
                cudaStream_t user_stream) {
    if (k < 1 || static_cast<uint64_t>(k) > X.n) throw InvalidArgument("ck_ann: k must lie in [1, n]");
    if (!(X.params.r_min > 0.0)) throw InvalidArgument("ck_ann: index has no initial radius");
    if (nq == 0) return;
    if (!queries) throw InvalidArgument("ck_ann: queries is null");
    DeviceGuard dg(X.device);
    std::lock_guard<std::mutex> lock(X.qmu);
    cudaStream_t s = user_stream ? user_stream : X.stream;
    const bool dev = (flags & DETLSH_F_DEVICE_PTRS) != 0;
    const int K = X.params.K, L = X.params.L, d = X.d;
    DevBuf<float> dq;
    const float* q = queries;
    if (!dev) {
        dq.alloc(nq * static_cast<size_t>(d));
        DETLSH_CUDA(cudaMemcpyAsync(dq.get(), queries, nq * static_cast<size_t>(d) * 4, cudaMemcpyHostToDevice, s));
        q = dq.get();
    }
    DevBuf<float> qproj(static_cast<size_t>(L) * nq * K);
    launch_project_exact(q, nq, d, X.coeffs_t.get(), K, L, qproj.get(), s);
    DevBuf<uint32_t> o_ids;
    DevBuf<double> o_d, o_r;
    DevBuf<int32_t> o_h;
    DevBuf<uint64_t> o_c;
    QueryPlan P{};
    P.data = X.data;
    P.n = X.n;
    P.d = d;
    P.K = K;
    P.L = L;
    P.NR = X.params.n_regions;
    P.table = X.table.get();
    P.trees = X.qtrees.get();
    P.eps = X.params.epsilon;
    P.c = X.params.c;
    P.r_min = X.params.r_min;
    P.budget = candidate_budget(X.params.beta, X.n, k);
    P.k = k;
    P.max_leaves = X.max_leaves;
    P.q = q;
    P.qproj = qproj.get();
    P.nq = nq;
    if (dev) {
        P.ids = ids;
        P.dists = dists;
        P.n_hits = n_hits;
        P.radius = radius;
        P.cands = cands;
    } else {
        if (ids) { o_ids.alloc(nq * k); P.ids = o_ids.get(); }
        if (dists) { o_d.alloc(nq * k); P.dists = o_d.get(); }
        if (n_hits) { o_h.alloc(nq); P.n_hits = o_h.get(); }
        if (radius) { o_r.alloc(nq); P.radius = o_r.get(); }
        if (cands) { o_c.alloc(nq); P.cands = o_c.get(); }
    }
    run_query_batch(P, X.scratch, X.device, s);
    if (!dev) {
        if (ids) DETLSH_CUDA(cudaMemcpyAsync(ids, P.ids, nq * k * 4, cudaMemcpyDeviceToHost, s));
        if (dists) DETLSH_CUDA(cudaMemcpyAsync(dists, P.dists, nq * k * 8, cudaMemcpyDeviceToHost, s));
        if (n_hits) DETLSH_CUDA(cudaMemcpyAsync(n_hits, P.n_hits, nq * 4, cudaMemcpyDeviceToHost, s));
        if (radius) DETLSH_CUDA(cudaMemcpyAsync(radius, P.radius, nq * 8, cudaMemcpyDeviceToHost, s));
        if (cands) DETLSH_CUDA(cudaMemcpyAsync(cands, P.cands, nq * 8, cudaMemcpyDeviceToHost, s));
    }
    // temporaries (query copy, projections, outputs) are freed on return
    DETLSH_CUDA(cudaStreamSynchronize(s));
}

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

uint64_t detlsh_launch_count(void) { return launch_count(); }
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
        launch_project_exact(P, n, d, ct.get(), K, L, O, s);
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
        const bool dev = flags & DETLSH_F_DEVICE_PTRS;
        GpuIndex X;
        X.device = device;
        X.n = n;
        X.params.K = K;
        X.params.L = L;
        X.params.n_regions = n_regions;
        X.sample_gpu = flags & DETLSH_F_SAMPLE_GPU;
        X.sample_size = sample_size_for(sample_fraction, n, n_regions);
        DETLSH_CUDA(cudaStreamCreateWithFlags(&X.stream, cudaStreamNonBlocking));
        DevBuf<float> pr;
        const float* P = projected;
        const size_t total = static_cast<size_t>(L) * n * K;
        if (!dev) {
            pr.alloc(total);
            to_device(pr.get(), projected, total * 4, false, X.stream);
            P = pr.get();
        }
        X.table.alloc(static_cast<size_t>(L) * K * (n_regions + 1));
        // `seed` is select_breakpoints' own seed argument (index.cpp passes
        // mix_seed(seed, 1)); the GPU-native mode derives one key per space.
        if (X.sample_gpu) {
            DevBuf<uint32_t> d_idx(X.sample_size);
            DevBuf<float> rows(static_cast<size_t>(L) * K * X.sample_size);
            for (int i = 0; i < L; ++i) {
                launch_feistel_sample(n, X.sample_size, mix_seed(seed, static_cast<uint64_t>(i)),
                                      d_idx.get(), X.stream);
                launch_gather_sample(P + static_cast<size_t>(i) * n * K, d_idx.get(), X.sample_size,
                                     K, rows.get() + static_cast<size_t>(i) * K * X.sample_size, X.stream);
            }
            gpu_order_stat_table(rows.get(), L * K, X.sample_size, n_regions, X.table.get(), X.stream);
        } else {
            const size_t W = static_cast<size_t>(n_regions) + 1;
            RefSampler sampler(n, X.sample_size, n_regions, seed);
            DevBuf<uint32_t> d_idx(X.sample_size);
            DevBuf<float> d_sample(static_cast<size_t>(K) * X.sample_size);
            std::vector<float> h_sample(static_cast<size_t>(K) * X.sample_size);
            X.h_table.assign(static_cast<size_t>(L) * K * W, 0.0f);
            for (int i = 0; i < L; ++i) {
                const auto& idx = sampler.next_space_indices();
                DETLSH_CUDA(cudaMemcpyAsync(d_idx.get(), idx.data(), X.sample_size * 4, cudaMemcpyHostToDevice, X.stream));
                launch_gather_sample(P + static_cast<size_t>(i) * n * K, d_idx.get(), X.sample_size, K,
                                     d_sample.get(), X.stream);
                DETLSH_CUDA(cudaMemcpyAsync(h_sample.data(), d_sample.get(), h_sample.size() * 4,
                                            cudaMemcpyDeviceToHost, X.stream));
                DETLSH_CUDA(cudaStreamSynchronize(X.stream));
                for (int j = 0; j < K; ++j)
                    sampler.select_row(h_sample.data() + static_cast<size_t>(j) * X.sample_size,
                                       X.h_table.data() + (static_cast<size_t>(i) * K + j) * W);
            }
            DETLSH_CUDA(cudaMemcpyAsync(X.table.get(), X.h_table.data(), X.h_table.size() * 4,
                                        cudaMemcpyHostToDevice, X.stream));
        }
        from_device(table, X.table.get(), X.table.bytes(), dev, X.stream);
        DETLSH_CUDA(cudaStreamSynchronize(X.stream));
        if (sample_size) *sample_size = X.sample_size;
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
