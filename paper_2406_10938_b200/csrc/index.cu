// build_index (index.cpp:138-218) and batched ck_ann orchestration.
//
// Build pipeline (one index, one device):
//   main stream : upload -> exact projection -> per space i: gather the sample,
//                 GPU sort -> that space's boundary rows, record event e_i
//   host        : replay of the reference quickselects of spaces 0..L-2
//                 (RefSampler): their RNG draws pick the next space's sample
//   side[i]     : wait e_i -> encode space i -> DE-Tree i      (own host thread)
//   side[L]     : r_min order statistics (needs projections only; own thread)
// so the trees and r_min overlap the sequential host replay of later spaces.
#include <algorithm>
#include <cstdio>
#include <chrono>
#include <cmath>
#include <cstring>
#include <exception>
#include <memory>
#include <numeric>
#include <stdexcept>
#include <thread>

#include "host_core.hpp"
#include "index.cuh"
#include "stages.cuh"

namespace detlsh_b200 {

namespace {

using Clock = std::chrono::steady_clock;
double ms_since(Clock::time_point t0) {
    return std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
}

// Runs fn on a host thread bound to `device`; the first exception is kept.
class Worker {
public:
    template <typename F>
    void run(int device, F fn) {
        threads_.emplace_back([this, device, fn]() {
            try {
                DETLSH_CUDA(cudaSetDevice(device));
                fn();
            } catch (...) {
                std::lock_guard<std::mutex> lk(mu_);
                if (!err_) err_ = std::current_exception();
            }
        });
    }
    void join() {
        for (auto& t : threads_) t.join();
        threads_.clear();
        if (err_) std::rethrow_exception(err_);
    }
    ~Worker() {
        for (auto& t : threads_)
            if (t.joinable()) t.join();
    }

private:
    std::vector<std::thread> threads_;
    std::mutex mu_;
    std::exception_ptr err_;
};

// Per-thread pinned staging buffer, grown on demand and kept across builds
// (cudaMallocHost costs milliseconds per call).
struct PinnedBuf {
    void* p = nullptr;
    size_t bytes = 0;
    ~PinnedBuf() {
        if (p) cudaFreeHost(p);
    }
};

float* pinned_scratch(size_t bytes, int slot = 0) {
    // 0: build samples, 1: sample rows, 2: query results, 3: query upload,
    // 4: sample indices, 5: space-0 sample indices
    thread_local PinnedBuf bufs[6];
    PinnedBuf& buf = bufs[slot];
    if (buf.bytes < bytes) {
        if (buf.p) cudaFreeHost(buf.p);
        buf.p = nullptr;
        buf.bytes = 0;
        DETLSH_CUDA(cudaMallocHost(&buf.p, bytes));
        buf.bytes = bytes;
    }
    return static_cast<float*>(buf.p);
}

// GPU-native sample: per-space Feistel sample + exact order statistics.
void breakpoints_gpu(GpuIndex& X, const float* d_proj, uint64_t seed, cudaStream_t s) {
    const int K = X.params.K, L = X.params.L, NR = X.params.n_regions;
    const uint64_t n = X.n, n_s = X.sample_size;
    DevBuf<uint32_t> d_idx(n_s);
    DevBuf<float> rows(static_cast<size_t>(L) * K * n_s);
    const uint64_t bseed = mix_seed(seed, kStreamBreakpoints);
    for (int i = 0; i < L; ++i) {
        launch_feistel_sample(n, n_s, mix_seed(bseed, static_cast<uint64_t>(i)), d_idx.get(), s);
        launch_gather_sample(d_proj + static_cast<size_t>(i) * n * K, d_idx.get(), n_s, K,
                             rows.get() + static_cast<size_t>(i) * K * n_s, s);
    }
    gpu_order_stat_table(rows.get(), L * K, n_s, NR, X.table.get(), s);
    X.h_table.resize(static_cast<size_t>(L) * K * (NR + 1));
    DETLSH_CUDA(cudaMemcpyAsync(X.h_table.data(), X.table.get(), X.h_table.size() * 4,
                                cudaMemcpyDeviceToHost, s));
    DETLSH_CUDA(cudaStreamSynchronize(s));
}

// r_min (index.cpp:75-136, 153-175) via per-probe order statistics.
double estimate_rmin_gpu(GpuIndex& X, const float* d_proj, uint64_t seed, cudaStream_t s) {
    StreamScope sc(s);
    const int K = X.params.K, L = X.params.L;
    const uint64_t n = X.n;
    Rng rng(mix_seed(seed, kStreamProbes));
    const int np = static_cast<int>(std::min<uint64_t>(10, n));
    std::vector<uint64_t> pos(np);
    for (int p = 0; p < np; ++p) pos[p] = rng.bounded(n);
    DevBuf<float> probe(static_cast<size_t>(np) * L * K);
    // initial guess: median pairwise distance of 32 strided points (space 0);
    // the probes' and those points' projected rows come over in two gathers
    const uint64_t m = std::min<uint64_t>(32, n);
    std::vector<uint64_t> gpos(pos.begin(), pos.end());
    for (uint64_t t = 0; t < m; ++t) gpos.push_back(t * n / m);
    DevBuf<uint64_t> d_gpos(gpos.size());
    DevBuf<float> d_sc(m * K);
    DETLSH_CUDA(cudaMemcpyAsync(d_gpos.get(), gpos.data(), gpos.size() * 8, cudaMemcpyHostToDevice, s));
    launch_gather_proj_rows(d_proj, n, K, L, d_gpos.get(), np, probe.get(), s);
    launch_gather_proj_rows(d_proj, n, K, 1, d_gpos.get() + np, static_cast<int>(m), d_sc.get(), s);
    std::vector<float> sc_rows(m * K);
    DETLSH_CUDA(cudaMemcpyAsync(sc_rows.data(), d_sc.get(), m * K * 4, cudaMemcpyDeviceToHost, s));
    const uint64_t budget = candidate_budget(X.params.beta, n, X.params.k);
    DevBuf<double> D(static_cast<size_t>(np) * n);
    DevBuf<uint32_t> hist(static_cast<size_t>(np) * 65536);
    std::vector<uint64_t> Tbits(np);
    rmin_order_stats(d_proj, n, K, L, probe.get(), np, budget, D.get(), hist.get(), Tbits.data(), s);
    std::vector<double> pd;
    pd.reserve(m * (m - 1) / 2);
    for (uint64_t a = 0; a < m; ++a)
        for (uint64_t b = a + 1; b < m; ++b) {
            double acc = 0.0;
            for (int j = 0; j < K; ++j) {
                const double diff =
                    static_cast<double>(sc_rows[a * K + j]) - static_cast<double>(sc_rows[b * K + j]);
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

}  // namespace

DeviceGuard::DeviceGuard(int dev) {
    DETLSH_CUDA(cudaGetDevice(&prev));
    if (prev != dev) DETLSH_CUDA(cudaSetDevice(dev));
}
DeviceGuard::~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
}

bool is_pow2(int v) { return v > 0 && (v & (v - 1)) == 0; }

uint64_t sample_size_for(double frac, uint64_t n, int NR) {
    uint64_t n_s = static_cast<uint64_t>(std::ceil(frac * static_cast<double>(n)));
    n_s = std::max<uint64_t>(n_s, static_cast<uint64_t>(NR));
    if (n_s > n) throw InvalidArgument("select_breakpoints: sample too small for region count");
    return n_s;
}

void validate_params(const detlsh_params& p, uint64_t n, int d) {
    // validate_params (index.cpp:16-24) + the stage preconditions build_index reaches
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
    sample_size_for(p.sample_fraction, n, p.n_regions);
}

// Device-side alias of a page-locked host pointer (UVA), or null for pageable memory.
static const float* mapped_host_ptr(const float* p) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    if (at.type != cudaMemoryTypeHost || at.devicePointer == nullptr) return nullptr;
    return static_cast<const float*>(at.devicePointer);
}

std::unique_ptr<GpuIndex> build_index_impl(const float* points, uint64_t n, int d,
                                           detlsh_params* params, const float* coeffs_host,
                                           uint64_t family_seed, uint64_t seed, int device,
                                           uint32_t flags) {
    if (!params) throw InvalidArgument("build_index: params is null");
    if (!points) throw InvalidArgument("build_index: points is null");
    const bool paa = (flags & DETLSH_F_PAA) != 0;
    if (paa) {  // build_det_only_index (index.cpp:220-232)
        if (coeffs_host) throw InvalidArgument("build_index: a hash family does not apply to PAA");
        params->L = 1;
        if (params->K > d) throw InvalidArgument("build_index: PAA requires K <= d");
    }
    validate_params(*params, n, d);
    DeviceGuard dg(device);
    ensure_mempool(device);
    auto X = std::make_unique<GpuIndex>();
    X->device = device;
    X->n = n;
    X->d = d;
    X->sample_gpu = (flags & DETLSH_F_SAMPLE_GPU) != 0;
    X->paa = paa;
    X->main.create();
    cudaStream_t s = X->main.s;
    StreamScope scope(s);
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
    const size_t W = static_cast<size_t>(NR) + 1;
    // reference-compatible sample (encoder.cpp:105-143): one RNG stream picks
    // every space's sample and pivots, so the host replay is sequential.  Space
    // 0's indices depend on the seed alone: drawn on a helper thread while the
    // hash family and the device set-up proceed.
    X->sample_size = sample_size_for(p.sample_fraction, n, NR);
    std::unique_ptr<RefSampler> sampler_ptr;
    const std::vector<uint32_t>* idx0_early = nullptr;
    std::exception_ptr fy_err;
    std::thread fy_thread;
    if (!X->sample_gpu) {
        const uint64_t ns0 = X->sample_size;
        fy_thread = std::thread([&sampler_ptr, &idx0_early, &fy_err, n, ns0, NR, seed]() {
            try {
                sampler_ptr = std::make_unique<RefSampler>(n, ns0, NR, mix_seed(seed, kStreamBreakpoints));
                idx0_early = &sampler_ptr->next_space_indices();
            } catch (...) {
                fy_err = std::current_exception();
            }
        });
    }
    struct FyJoin {
        std::thread& t;
        ~FyJoin() {
            if (t.joinable()) t.join();
        }
    } fy_join{fy_thread};
    auto join_fy = [&]() {
        if (fy_thread.joinable()) fy_thread.join();
        if (fy_err) std::rethrow_exception(fy_err);
    };
    for (int i = 0; i <= L; ++i) {
        X->side.push_back(std::make_unique<OwnedStream>());
        X->side.back()->create();
    }
    // hash family (projection.cpp:11-23): host, seeded sub-stream 0 (none for PAA)
    X->h_coeffs.resize(paa ? 0 : static_cast<size_t>(LK) * d);
    if (paa) {
        X->family_seed = 0;
    } else if (coeffs_host) {
        std::memcpy(X->h_coeffs.data(), coeffs_host, X->h_coeffs.size() * sizeof(float));
        X->family_seed = family_seed;
    } else {
        X->family_seed = mix_seed(seed, kStreamFamily);
        sample_hash_family(d, K, L, X->family_seed, X->h_coeffs.data());
    }
    X->timings.emplace_back("host_params_family", ms_since(t0));
    t0 = Clock::now();
    {  // peak device footprint of the build (projections, codes, trees and their
       // sort temporaries, verification rows, r_min distances)
        const size_t per_pt = static_cast<size_t>(LK) * 5 + 2 * (static_cast<size_t>(d) + 32) +
                              4 * static_cast<size_t>(d) + static_cast<size_t>(L) * 64 + 96;
        reserve_mempool(device, n * per_pt, s);
    }
    if (!paa) {
        X->coeffs.alloc(X->h_coeffs.size());
        DETLSH_CUDA(cudaMemcpyAsync(X->coeffs.get(), X->h_coeffs.data(), X->h_coeffs.size() * 4,
                                    cudaMemcpyHostToDevice, s));
        X->coeffs_t.alloc(static_cast<size_t>(lk_padded(LK)) * d);
        prepare_coeffs_t(X->coeffs.get(), LK, d, X->coeffs_t.get(), s);
        prepare_proj_tc(X->coeffs.get(), LK, d, X->proj_tc, s);
    }
    DevBuf<float> proj(static_cast<size_t>(L) * n * K);
    const uint64_t n_s = X->sample_size;
    X->table.alloc(static_cast<size_t>(L) * K * W);
    X->codes.alloc(static_cast<size_t>(L) * n * K);
    X->trees.resize(L);
    for (auto& t : X->trees) t = std::make_unique<DevTree>();
    // the tensor-core projection checks every value for [0, 255] integrality on
    // its way through: its verdict replaces a separate pass (0xffffffff: not run)
    DevBuf<uint32_t> nonint(1);
    bool probe_nonint = false;
    DETLSH_CUDA(cudaMemsetAsync(nonint.get(), 0xff, 4, s));
    auto project_all = [&]() {
        if (paa) {
            launch_project_paa(X->data, n, d, K, proj.get(), s);
            return;
        }
        // a glance at the first rows (a few KB) keeps float datasets off the
        // tensor-core attempt, whose full pass would only end in the FP64 rerun
        const bool try_tc = X->proj_tc.ok && data_is_u8(X->data, std::min<uint64_t>(n, 4096) * d, s);
        if (X->proj_tc.ok && !try_tc) probe_nonint = true;  // a non-integral value seen: no u8 rows
        launch_project_exact(X->data, n, d, X->coeffs_t.get(), K, L, proj.get(), s, "project_exact",
                             try_tc ? &X->proj_tc : nullptr, nonint.get());
    };
    std::vector<float> h_rows;  // replayed boundary rows [L][K][W]
    if (!X->sample_gpu) h_rows.assign(static_cast<size_t>(L) * K * W, 0.0f);
    // Host input in reference mode: space 0's sample positions depend on the
    // seed alone, so its rows are gathered on the host, uploaded and projected
    // on their own (a row's projection does not depend on the other rows), and
    // space 0's replay runs while the full dataset is still being uploaded and
    // projected by a helper thread.
    const bool dev_in = (flags & DETLSH_F_DEVICE_PTRS) != 0;
    const bool early0 = !X->sample_gpu;
    DevBuf<float> d_sample0;
    cudaEvent_t table0 = nullptr;
    struct EvOne0 {
        cudaEvent_t& e;
        ~EvOne0() {
            if (e) cudaEventDestroy(e);
        }
    } table0_guard{table0};
    if (!early0 && dev_in && (flags & DETLSH_F_BORROW_DATA)) {
        X->data = points;
        project_all();
    } else if (!early0) {
        X->data_buf.alloc(n * static_cast<size_t>(d));
        DETLSH_CUDA(cudaMemcpyAsync(X->data_buf.get(), points, n * static_cast<size_t>(d) * 4,
                                    (flags & DETLSH_F_DEVICE_PTRS) ? cudaMemcpyDeviceToDevice
                                                                   : cudaMemcpyHostToDevice,
                                    s));
        X->data = X->data_buf.get();
        project_all();
    } else {
        // device input: the dataset is (copied) on the device and projected on s
        // at once; space 0's sample rows are gathered by a kernel on s2
        if (dev_in && (flags & DETLSH_F_BORROW_DATA)) {
            X->data = points;
        } else {
            X->data_buf.alloc(n * static_cast<size_t>(d));
            X->data = X->data_buf.get();
            if (dev_in)
                DETLSH_CUDA(cudaMemcpyAsync(X->data_buf.get(), points, n * static_cast<size_t>(d) * 4,
                                            cudaMemcpyDeviceToDevice, s));
        }
        cudaEvent_t coeffs_ready;
        DETLSH_CUDA(cudaEventCreateWithFlags(&coeffs_ready, cudaEventDisableTiming));
        DETLSH_CUDA(cudaEventRecord(coeffs_ready, s));  // (device input: the dataset copy too)
        if (dev_in) project_all();
        cudaStream_t s2 = X->side[L]->s;  // free until the r_min worker starts
        {
            StreamScope sc(s2);
            const bool zero_copy_sample = !dev_in && mapped_host_ptr(points) != nullptr;
            join_fy();
            const auto& idx0 = *idx0_early;
            const bool dbg = std::getenv("DETLSH_DEBUG_BUILD") != nullptr;
            if (dbg) fprintf(stderr, "[build] fy %.2f ms mapped=%d\n", ms_since(t0), zero_copy_sample ? 1 : 0);
            DevBuf<float> dG(n_s * static_cast<size_t>(d)), dGp(static_cast<size_t>(L) * n_s * K);
            DevBuf<uint32_t> iota(n_s);
            // host arrays go over through page-locked staging (a pageable copy
            // is staged by the driver and could wait behind other threads' copies)
            auto staged_idx0 = [&]() {
                uint32_t* h = reinterpret_cast<uint32_t*>(pinned_scratch(n_s * 4, 5));
                std::memcpy(h, idx0.data(), n_s * 4);
                return h;
            };
            if (dev_in) {
                DevBuf<uint32_t> d_idx0(n_s);
                DETLSH_CUDA(cudaMemcpyAsync(d_idx0.get(), staged_idx0(), n_s * 4, cudaMemcpyHostToDevice, s2));
                DETLSH_CUDA(cudaStreamWaitEvent(s2, coeffs_ready, 0));
                launch_pack_f32(X->data, d_idx0.get(), n_s, d, dG.get(), s2);  // rows idx0[t]
            } else if (const float* mapped = zero_copy_sample ? mapped_host_ptr(points) : nullptr) {
                // page-locked host input: the GPU gathers the sample rows over the
                // bus itself (zero-copy), no host-side gather on the critical path
                DevBuf<uint32_t> d_idx0(n_s);
                DETLSH_CUDA(cudaMemcpyAsync(d_idx0.get(), staged_idx0(), n_s * 4, cudaMemcpyHostToDevice, s2));
                launch_pack_f32(mapped, d_idx0.get(), n_s, d, dG.get(), s2);
            } else {
                float* G = pinned_scratch(n_s * static_cast<size_t>(d) * sizeof(float), 1);
                const int nt = 8;
                std::vector<std::thread> gth;
                for (int w = 0; w < nt; ++w)
                    gth.emplace_back([&, w]() {
                        for (uint64_t t = w; t < n_s; t += nt)
                            std::memcpy(G + t * d, points + static_cast<uint64_t>(idx0[t]) * d, d * sizeof(float));
                    });
                for (auto& th : gth) th.join();
                DETLSH_CUDA(cudaMemcpyAsync(dG.get(), G, n_s * static_cast<size_t>(d) * 4, cudaMemcpyHostToDevice, s2));
            }
            launch_iota_u32(iota.get(), n_s, s2);
            DETLSH_CUDA(cudaStreamWaitEvent(s2, coeffs_ready, 0));
            if (paa) launch_project_paa(dG.get(), n_s, d, K, dGp.get(), s2, "project_sample");
            else launch_project_exact(dG.get(), n_s, d, X->coeffs_t.get(), K, L, dGp.get(), s2, "project_sample", &X->proj_tc);
            d_sample0.alloc(static_cast<size_t>(K) * n_s);
            launch_gather_sample(dGp.get(), iota.get(), n_s, K, d_sample0.get(), s2);
            float* h_sample = pinned_scratch(static_cast<size_t>(K) * n_s * sizeof(float));
            DETLSH_CUDA(cudaMemcpyAsync(h_sample, d_sample0.get(), static_cast<size_t>(K) * n_s * 4,
                                        cudaMemcpyDeviceToHost, s2));
            cudaEvent_t copied0;
            DETLSH_CUDA(cudaEventCreateWithFlags(&copied0, cudaEventDisableTiming));
            DETLSH_CUDA(cudaEventRecord(copied0, s2));
            if (dbg) fprintf(stderr, "[build] enqueued %.2f ms\n", ms_since(t0));
            gpu_order_stat_table(d_sample0.get(), K, n_s, NR, X->table.get(), s2, /*sync=*/false);
            DETLSH_CUDA(cudaEventCreateWithFlags(&table0, cudaEventDisableTiming));
            DETLSH_CUDA(cudaEventRecord(table0, s2));
            // helper: full upload (blocks for pageable sources) + full projection on s,
            // issued after the sample rows so their copy is not queued behind it
            std::exception_ptr up_err;
            std::thread uploader([&]() {
                if (dev_in) return;  // already projecting on s
                try {
                    DETLSH_CUDA(cudaSetDevice(device));
                    StreamScope sc(s);
                    // the sample rows first: with page-locked input the GPU gathers
                    // them over the bus, which the bulk upload would otherwise share
                    if (zero_copy_sample) DETLSH_CUDA(cudaStreamWaitEvent(s, copied0, 0));
                    DETLSH_CUDA(cudaMemcpyAsync(X->data_buf.get(), points, n * static_cast<size_t>(d) * 4,
                                                cudaMemcpyHostToDevice, s));
                    project_all();
                } catch (...) {
                    up_err = std::current_exception();
                }
            });
            struct Joiner {
                std::thread& t;
                ~Joiner() {
                    if (t.joinable()) t.join();
                }
            } joiner{uploader};
            DETLSH_CUDA(cudaEventSynchronize(copied0));
            if (dbg) fprintf(stderr, "[build] sample on host %.2f ms\n", ms_since(t0));
            X->timings.emplace_back("bp_space0_sample", ms_since(t0));
            const auto tr = Clock::now();
            if (L > 1)
                for (int j = 0; j < K; ++j)
                    sampler_ptr->select_row(h_sample + static_cast<size_t>(j) * n_s, h_rows.data() + j * W);
            X->timings.emplace_back("bp_space0_replay", ms_since(tr));
            if (dbg) fprintf(stderr, "[build] space-0 replay done %.2f ms\n", ms_since(t0));
            uploader.join();
            cudaEventDestroy(copied0);  // (after the uploader's wait on it)
            if (up_err) std::rethrow_exception(up_err);
        }
        cudaEventDestroy(coeffs_ready);
        DETLSH_CUDA(cudaStreamWaitEvent(s, table0, 0));  // space 0's boundaries before its encode
    }
    DETLSH_CUDA(cudaStreamSynchronize(s));
    X->timings.emplace_back("upload_project", ms_since(t0));

    // exact u8 verification rows (integral datasets): decided now, packed in
    // tree-0 leaf order by the space-0 worker right after tree 0 (query.cu)
    t0 = Clock::now();
    uint32_t h_nonint = 0xffffffffu;
    if (!(flags & DETLSH_F_NO_U8)) {
        DETLSH_CUDA(cudaMemcpyAsync(&h_nonint, nonint.get(), 4, cudaMemcpyDeviceToHost, s));
        DETLSH_CUDA(cudaStreamSynchronize(s));
    }
    const bool want_u8 = !(flags & DETLSH_F_NO_U8) && !probe_nonint &&
                         (h_nonint == 0xffffffffu ? data_is_u8(X->data, n * static_cast<uint64_t>(d), s) : h_nonint == 0);
    if (want_u8) {
        X->row_u8 = (d + 31) / 32 * 32;  // whole 32-byte MMA K steps
        const int chunks = X->row_u8 / 16;
        int lpr = 1;
        while (lpr < chunks && lpr < 32) lpr <<= 1;
        X->u8_lpr = lpr;
    } else {
        // float rows in tree-0 leaf order and their bf16-triple tiles: the pool
        // grows for them here, on this thread, before the tree workers start
        // (grown from the tree-0 worker during the replay, the mappings held the
        // replay's stream for up to 0.3 s at C4)
        const size_t Rf = (6 * static_cast<size_t>(d) + 31) / 32 * 32;
        reserve_mempool(device, n * (4 * static_cast<size_t>(d) + Rf + 4), s);
    }
    X->timings.emplace_back("u8_check", ms_since(t0));

    Worker workers;
    double rmin_ms = 0.0;
    double r_min = X->params.r_min;
    GpuIndex* Xp = X.get();
    const float* d_proj = proj.get();
    if (!(r_min > 0.0)) {
        workers.run(device, [Xp, d_proj, seed, &r_min, &rmin_ms, L]() {
            const auto ta = Clock::now();
            r_min = estimate_rmin_gpu(*Xp, d_proj, seed, Xp->side[L]->s);
            rmin_ms = ms_since(ta);
        });
    }
    std::vector<cudaEvent_t> ready(L);
    for (auto& e : ready) DETLSH_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    struct EvGuard {
        std::vector<cudaEvent_t>& v;
        ~EvGuard() {
            for (auto e : v) cudaEventDestroy(e);
        }
    } evg{ready};
    const int cap = p.leaf_capacity;
    auto launch_space = [&](int i) {
        DETLSH_CUDA(cudaEventRecord(ready[i], s));
        cudaEvent_t ev = ready[i];
        workers.run(device, [Xp, d_proj, ev, i, n, K, NR, W, cap, want_u8]() {
            cudaStream_t ts = Xp->side[i]->s;
            StreamScope sc(ts);
            DETLSH_CUDA(cudaStreamWaitEvent(ts, ev, 0));
            launch_encode(d_proj + static_cast<size_t>(i) * n * K, n, K, 1,
                          Xp->table.get() + static_cast<size_t>(i) * K * W, NR,
                          Xp->codes.get() + static_cast<size_t>(i) * n * K, ts);
            build_tree_gpu(Xp->codes.get() + static_cast<size_t>(i) * n * K, n, K, NR, i, cap,
                           *Xp->trees[i], ts);
            if (i == 0 && want_u8) {  // overlaps the other trees
                const int d = Xp->d, R = Xp->row_u8;
                Xp->data_u8.alloc(n * static_cast<size_t>(R));
                launch_pack_u8(Xp->data, Xp->trees[0]->perm.get(), n, d, R, Xp->data_u8.get(), ts);
                Xp->xn_u8.alloc(n);
                launch_row_norms_u8(Xp->data_u8.get(), n, R, Xp->xn_u8.get(), ts);
                if (tc_score_fits(R)) {  // tensor-core verification operand tiles
                    Xp->data_tc.alloc((n + 127) / 128 * 128 * static_cast<uint64_t>(R));
                    launch_pack_tc_tiles(Xp->data_u8.get(), n, R, Xp->data_tc.get(), ts);
                }
                DETLSH_CUDA(cudaStreamSynchronize(ts));
            } else if (i == 0) {  // fp32 rows in leaf order: contiguous per-leaf candidate reads
                Xp->data_leaf.alloc(n * static_cast<size_t>(Xp->d));
                launch_pack_f32(Xp->data, Xp->trees[0]->perm.get(), n, Xp->d, Xp->data_leaf.get(), ts);
                const int Rf = (6 * Xp->d + 31) / 32 * 32;  // [hi, lo, hi] bf16 along K
                if (Rf > 256 && tc_score_fits(Rf)) {  // bf16x3 verification operand tiles
                    Xp->row_f = Rf;
                    Xp->data_tcf.alloc((n + 127) / 128 * 128 * static_cast<uint64_t>(Rf));
                    Xp->xnf.alloc(n);
                    launch_pack_tcf_tiles(Xp->data_leaf.get(), n, Xp->d, Rf, Xp->data_tcf.get(), Xp->xnf.get(), ts);
                }
                DETLSH_CUDA(cudaStreamSynchronize(ts));
            }
        });
    };
    // breakpoints
    t0 = Clock::now();
    if (X->sample_gpu) {
        breakpoints_gpu(*X, d_proj, seed, s);
        for (int i = 0; i < L; ++i) launch_space(i);
    } else {
        // reference-compatible sample (encoder.cpp:105-143).  A boundary is an
        // order statistic of the space's sample, whatever pivots the
        // reference's quickselect draws, so the table rows come from a GPU
        // sort of the gathered sample and space i's trees start at once.  The
        // host replays the quickselects only because their draws advance the
        // RNG that picks the NEXT space's sample: spaces 0..L-2 are replayed
        // while the GPU encodes and builds, space L-1 not at all.  The one
        // value an order statistic leaves open is the sign of a zero
        // boundary (-0 == +0); those rows take the replayed value.
        // (host input: space 0 was sampled, sorted and replayed during the upload)
        RefSampler& sampler = *sampler_ptr;
        DevBuf<uint32_t> d_idx(n_s);
        DevBuf<float> d_sample(static_cast<size_t>(K) * n_s);
        // the per-space order statistics' temporaries, reserved before the tree
        // workers start (their GB-sized allocations would hold this thread --
        // the replay's -- in the allocator for up to hundreds of ms at C4)
        OrderStatWork os_work;
        os_work.reserve(K, n_s, s);
        float* h_sample = pinned_scratch(static_cast<size_t>(K) * n_s * sizeof(float));
        cudaEvent_t copied;
        DETLSH_CUDA(cudaEventCreateWithFlags(&copied, cudaEventDisableTiming));
        struct EvOne {
            cudaEvent_t e;
            ~EvOne() { cudaEventDestroy(e); }
        } copied_guard{copied};
        auto replay_space = [&](int i, int rows_needed) {
            float* rows = h_rows.data() + static_cast<size_t>(i) * K * W;
            for (int j = 0; j < rows_needed; ++j)
                sampler.select_row(h_sample + static_cast<size_t>(j) * n_s, rows + j * W);
        };
        double t_idx = 0.0, t_wait = 0.0, t_replay = 0.0, t_enq = 0.0;
        const bool dbg_loop = std::getenv("DETLSH_DEBUG_BUILD") != nullptr;
        const auto t_loop = Clock::now();
        for (int i = 0; i < L; ++i) {
            if (i == 0 && early0) {
                launch_space(0);  // s already waits for space 0's table
                continue;
            }
            auto tq = Clock::now();
            const auto& idx = sampler.next_space_indices();
            t_idx += ms_since(tq);
            const auto te = Clock::now();
            // (through page-locked staging: a pageable copy is staged by the
            // driver and could wait behind the tree workers' transfers)
            uint32_t* h_idx = reinterpret_cast<uint32_t*>(pinned_scratch(n_s * 4, 4));
            std::memcpy(h_idx, idx.data(), n_s * 4);
            const double e0 = ms_since(te);
            DETLSH_CUDA(cudaMemcpyAsync(d_idx.get(), h_idx, n_s * 4, cudaMemcpyHostToDevice, s));
            launch_gather_sample(d_proj + static_cast<size_t>(i) * n * K, d_idx.get(), n_s, K,
                                 d_sample.get(), s);
            const double e1 = ms_since(te);
            const bool replay = i + 1 < L;
            if (replay) {
                DETLSH_CUDA(cudaMemcpyAsync(h_sample, d_sample.get(), static_cast<size_t>(K) * n_s * 4,
                                            cudaMemcpyDeviceToHost, s));
                DETLSH_CUDA(cudaEventRecord(copied, s));
            }
            const double e2 = ms_since(te);
            gpu_order_stat_table(d_sample.get(), K, n_s, NR, X->table.get() + static_cast<size_t>(i) * K * W,
                                 s, /*sync=*/false, &os_work);
            const double e3 = ms_since(te);
            launch_space(i);
            t_enq += ms_since(te);
            if (dbg_loop)
                fprintf(stderr, "[build] space %d enqueue: staged %.2f copy+gather %.2f d2h %.2f os %.2f launch %.2f ms\n",
                        i, e0, e1 - e0, e2 - e1, e3 - e2, ms_since(te) - e3);
            if (dbg_loop) fprintf(stderr, "[build] space %d enqueued %.2f ms into the loop\n", i, ms_since(t_loop));
            if (replay) {
                tq = Clock::now();
                DETLSH_CUDA(cudaEventSynchronize(copied));
                t_wait += ms_since(tq);
                tq = Clock::now();
                replay_space(i, K);
                t_replay += ms_since(tq);
            }
        }
        X->timings.emplace_back("bp_sample_indices", t_idx);
        X->timings.emplace_back("bp_sample_wait", t_wait);
        X->timings.emplace_back("bp_replay", t_replay);
        X->timings.emplace_back("bp_enqueue", t_enq);
        X->timings.emplace_back("bp_loop", ms_since(t_loop));
        X->h_table.assign(static_cast<size_t>(L) * K * W, 0.0f);
        {  // (page-locked staging, like the index copies above)
            float* h_tab = pinned_scratch(X->h_table.size() * 4, 4);
            DETLSH_CUDA(cudaMemcpyAsync(h_tab, X->table.get(), X->h_table.size() * 4, cudaMemcpyDeviceToHost, s));
            DETLSH_CUDA(cudaStreamSynchronize(s));
            std::memcpy(X->h_table.data(), h_tab, X->h_table.size() * 4);
        }
        // last space: replay only up to its last row holding a zero boundary
        int last_zero = -1;
        const size_t base = static_cast<size_t>(L - 1) * K * W;
        for (int j = 0; j < K; ++j)
            for (int b = 0; b < W; ++b)
                if (X->h_table[base + static_cast<size_t>(j) * W + b] == 0.0f) last_zero = j;
        if (last_zero >= 0) {
            const float* last_sample = (early0 && L == 1) ? d_sample0.get() : d_sample.get();
            DETLSH_CUDA(cudaMemcpyAsync(h_sample, last_sample, static_cast<size_t>(K) * n_s * 4,
                                        cudaMemcpyDeviceToHost, s));
            DETLSH_CUDA(cudaStreamSynchronize(s));
            replay_space(L - 1, last_zero + 1);
        }
        bool patched = false;
        for (int i = 0; i < L; ++i) {
            const int rows_known = i + 1 < L ? K : last_zero + 1;
            for (int j = 0; j < rows_known; ++j)
                for (int b = 0; b < W; ++b) {
                    const size_t at = (static_cast<size_t>(i) * K + j) * W + b;
                    const float g = X->h_table[at], h = h_rows[at];
                    if (std::memcmp(&g, &h, 4) == 0) continue;
                    if (!(g == 0.0f && h == 0.0f))
                        throw std::runtime_error("breakpoints: GPU order statistic differs from the replay");
                    X->h_table[at] = h;  // zero sign: the codes are unaffected (-0 == +0)
                    patched = true;
                }
        }
        if (patched) {
            workers.join();  // encode read the table; patch only after it
            DETLSH_CUDA(cudaMemcpyAsync(X->table.get(), X->h_table.data(), X->h_table.size() * 4,
                                        cudaMemcpyHostToDevice, s));
            DETLSH_CUDA(cudaStreamSynchronize(s));
        }
    }
    X->timings.emplace_back("breakpoints", ms_since(t0));
    t0 = Clock::now();
    workers.join();
    X->timings.emplace_back("trees_rmin_tail", ms_since(t0));
    double tree_ms = 0.0;
    std::vector<QTree> qt(L);
    for (int i = 0; i < L; ++i) {
        const DevTree& T = *X->trees[i];
        qt[i] = QTree{T.leaf_node.get(), T.leaf_begin.get(), T.leaf_count.get(), T.leaf_box.get(),
                      T.leaf_cr.get(), T.perm.get(), static_cast<uint32_t>(T.num_leaves)};
        X->max_leaves = std::max<uint32_t>(X->max_leaves, static_cast<uint32_t>(T.num_leaves));
        tree_ms += T.build_ms;
    }
    X->qtrees.alloc(L);
    DETLSH_CUDA(cudaMemcpyAsync(X->qtrees.get(), qt.data(), L * sizeof(QTree), cudaMemcpyHostToDevice, s));
    X->params.r_min = r_min;
    if (flags & DETLSH_F_NO_CODES) X->codes.release();
    proj.release();
    DETLSH_CUDA(cudaStreamSynchronize(s));
    X->timings.emplace_back("trees_sum", tree_ms);
    X->timings.emplace_back("rmin", rmin_ms);
    X->timings.emplace_back("total", ms_since(t_all));
    if (std::getenv("DETLSH_DEBUG_BUILD")) {
        fprintf(stderr, "[build] stages");
        for (const auto& t : X->timings) fprintf(stderr, " %s=%.2f", t.first.c_str(), t.second);
        fprintf(stderr, "\n");
    }
    *params = X->params;
    return X;
}

// estimate_rmin (index.hpp:91, index.cpp:333-374) for caller-supplied probe
// queries: the same order-statistic form as the build's r_min,
// with the probes projected by the index's own projection kernel
// (project_query, index.cpp:181-188) and the dataset re-projected chunk by
// chunk (the index keeps no projections, like the reference's DetIndex).
double estimate_rmin_impl(GpuIndex& X, const float* probes, uint64_t np, int k, uint32_t flags) {
    if (np == 0) throw InvalidArgument("estimate_rmin: no probe queries");
    if (!probes) throw InvalidArgument("estimate_rmin: probes is null");
    DeviceGuard dg(X.device);
    std::lock_guard<std::mutex> lock(X.qmu);
    cudaStream_t s = X.main.s;
    StreamScope scope(s);
    const int K = X.params.K, L = X.params.L, d = X.d;
    const uint64_t n = X.n;
    const bool dev = (flags & DETLSH_F_DEVICE_PTRS) != 0;
    auto project = [&](const float* pts, uint64_t m, float* out) {
        if (X.paa) launch_project_paa(pts, m, d, K, out, s, "project_probe");
        else launch_project_exact(pts, m, d, X.coeffs_t.get(), K, L, out, s, "project_probe", &X.proj_tc);
    };
    // probe projections [L][np][K] -> [np][L][K] (the order-statistic kernel's layout)
    DevBuf<float> dprobe(np * static_cast<size_t>(d)), pp(static_cast<size_t>(L) * np * K),
        ppt(static_cast<size_t>(L) * np * K);
    DETLSH_CUDA(cudaMemcpyAsync(dprobe.get(), probes, np * static_cast<size_t>(d) * 4,
                                dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s));
    project(dprobe.get(), np, pp.get());
    std::vector<float> h_pp(static_cast<size_t>(L) * np * K), h_ppt(h_pp.size());
    DETLSH_CUDA(cudaMemcpyAsync(h_pp.data(), pp.get(), h_pp.size() * 4, cudaMemcpyDeviceToHost, s));
    DETLSH_CUDA(cudaStreamSynchronize(s));
    for (uint64_t p = 0; p < np; ++p)
        for (int i = 0; i < L; ++i)
            std::memcpy(&h_ppt[(p * L + i) * K], &h_pp[(static_cast<size_t>(i) * np + p) * K], K * 4);
    DETLSH_CUDA(cudaMemcpyAsync(ppt.get(), h_ppt.data(), h_ppt.size() * 4, cudaMemcpyHostToDevice, s));
    // initial guess: median pairwise projected distance of 32 strided points, space 0 (index.cpp:84-109)
    const uint64_t m = std::min<uint64_t>(32, n);
    std::vector<uint32_t> h_pos(m);
    for (uint64_t t = 0; t < m; ++t) h_pos[t] = static_cast<uint32_t>(t * n / m);
    DevBuf<uint32_t> d_pos(m);
    DevBuf<float> rows(m * static_cast<size_t>(d)), rp(static_cast<size_t>(L) * m * K);
    DETLSH_CUDA(cudaMemcpyAsync(d_pos.get(), h_pos.data(), m * 4, cudaMemcpyHostToDevice, s));
    launch_pack_f32(X.data, d_pos.get(), m, d, rows.get(), s);
    project(rows.get(), m, rp.get());
    std::vector<float> sc(m * K);
    DETLSH_CUDA(cudaMemcpyAsync(sc.data(), rp.get(), sc.size() * 4, cudaMemcpyDeviceToHost, s));
    DETLSH_CUDA(cudaStreamSynchronize(s));
    std::vector<double> pd;
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
    // reaches(r) <=> the budget-th smallest D <= eps r; a budget of 0 stops at
    // the first point found, like budget 1 (count_range_reaches, index.cpp:48)
    const uint64_t rank = std::max<uint64_t>(1, candidate_budget(X.params.beta, n, k));
    constexpr int kGroup = 10;
    const uint64_t chunk = std::min<uint64_t>(n, 1ULL << 22);
    DevBuf<double> D(std::min<uint64_t>(np, kGroup) * n);
    DevBuf<float> pc(static_cast<size_t>(L) * chunk * K);
    std::vector<uint64_t> Tbits(np);
    for (uint64_t g0 = 0; g0 < np; g0 += kGroup) {
        const int gn = static_cast<int>(std::min<uint64_t>(kGroup, np - g0));
        RminSelect sel(gn);
        rmin_begin(sel, s);
        for (uint64_t z0 = 0; z0 < n; z0 += chunk) {
            const uint64_t mz = std::min(chunk, n - z0);
            project(X.data + z0 * static_cast<uint64_t>(d), mz, pc.get());
            launch_rmin_dist(pc.get(), mz, z0, n, K, L, ppt.get() + g0 * L * K, sel, D.get(), s);
        }
        rmin_select(sel, D.get(), n, rank, Tbits.data() + g0, s);
    }
    std::vector<double> T(np);
    for (uint64_t p = 0; p < np; ++p) std::memcpy(&T[p], &Tbits[p], 8);
    return rmin_from_order_stats(T, guess, X.params.epsilon, X.params.c);
}

void project_queries_impl(GpuIndex& X, const float* q, uint64_t nq, float* out, uint32_t flags) {
    if (nq == 0) return;
    if (!q || !out) throw InvalidArgument("project_query: null argument");
    DeviceGuard dg(X.device);
    std::lock_guard<std::mutex> lock(X.qmu);
    cudaStream_t s = X.main.s;
    StreamScope scope(s);
    const bool dev = (flags & DETLSH_F_DEVICE_PTRS) != 0;
    const int K = X.params.K, L = X.params.L, d = X.d;
    DevBuf<float> dq, dout;
    const float* src = q;
    float* dst = out;
    if (!dev) {
        dq.alloc(nq * static_cast<size_t>(d));
        DETLSH_CUDA(cudaMemcpyAsync(dq.get(), q, nq * static_cast<size_t>(d) * 4, cudaMemcpyHostToDevice, s));
        src = dq.get();
        dout.alloc(static_cast<size_t>(L) * nq * K);
        dst = dout.get();
    }
    if (X.paa) launch_project_paa(src, nq, d, K, dst, s, "project_query");
    else launch_project_exact(src, nq, d, X.coeffs_t.get(), K, L, dst, s, "project_query", &X.proj_tc);
    if (!dev)
        DETLSH_CUDA(cudaMemcpyAsync(out, dst, static_cast<size_t>(L) * nq * K * 4, cudaMemcpyDeviceToHost, s));
    DETLSH_CUDA(cudaStreamSynchronize(s));
}

void query_impl(GpuIndex& X, const float* queries, uint64_t nq, int k, uint32_t flags,
                uint32_t* ids, double* dists, int32_t* n_hits, double* radius, uint64_t* cands,
                cudaStream_t user_stream, const RcArgs* rc) {
    if (rc) {  // rc_ann (index.cpp:271-274)
        if (!(rc->r > 0.0)) throw InvalidArgument("rc_ann: radius must be positive");
        if (!(rc->c > 1.0)) throw InvalidArgument("rc_ann: c must exceed 1");
        k = 1;
    } else {
        if (k < 1 || static_cast<uint64_t>(k) > X.n) throw InvalidArgument("ck_ann: k must lie in [1, n]");
        if (!(X.params.r_min > 0.0)) throw InvalidArgument("ck_ann: index has no initial radius");
    }
    if (nq == 0) return;
    if (!queries) throw InvalidArgument("ck_ann: queries is null");
    DeviceGuard dg(X.device);
    std::lock_guard<std::mutex> lock(X.qmu);
    cudaStream_t s = user_stream ? user_stream : X.main.s;
    StreamScope scope(s);
    const bool dev = (flags & DETLSH_F_DEVICE_PTRS) != 0;
    const int K = X.params.K, L = X.params.L, d = X.d;
    DevBuf<float> dq;
    const float* q = queries;
    if (!dev) {
        const size_t qbytes = nq * static_cast<size_t>(d) * 4;
        dq.alloc(nq * static_cast<size_t>(d));
        cudaPointerAttributes at{};
        const bool pageable = cudaPointerGetAttributes(&at, queries) != cudaSuccess ||
                              at.type == cudaMemoryTypeUnregistered;
        cudaGetLastError();
        const void* src = queries;
        if (pageable) {  // staged through pinned memory (see the result copies below)
            float* stage = pinned_scratch(qbytes, 3);
            std::memcpy(stage, queries, qbytes);
            src = stage;
        }
        DETLSH_CUDA(cudaMemcpyAsync(dq.get(), src, qbytes, cudaMemcpyHostToDevice, s));
        q = dq.get();
    }
    DevBuf<float> qproj(static_cast<size_t>(L) * nq * K);
    if (X.paa) launch_project_paa(q, nq, d, K, qproj.get(), s);  // DetIndex::project_query (index.cpp:181-188)
    else launch_project_exact(q, nq, d, X.coeffs_t.get(), K, L, qproj.get(), s, "project_exact", &X.proj_tc);
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
    P.perm0 = X.trees[0]->perm.get();
    P.data_u8 = X.data_u8.get();
    P.xn_u8 = X.xn_u8.get();
    P.data_tc = X.data_tc.get();
    P.data_leaf = X.data_leaf.get();
    P.data_tcf = X.data_tcf.get();
    P.xnf = X.xnf.get();
    P.row_f = X.row_f;
    P.trees_num_leaves0 = static_cast<uint32_t>(X.trees[0]->num_leaves);
    P.trees_leaf_begin0 = X.trees[0]->leaf_begin.get();
    P.trees_leaf_count0 = X.trees[0]->leaf_count.get();
    P.q_begin = 0;
    P.q_end = nq;
    P.tc_allowed = (flags & DETLSH_F_NO_TC) ? 0 : 1;
    P.row_u8 = X.row_u8;
    P.u8_lpr = X.u8_lpr;
    P.eps = X.params.epsilon;
    P.c = rc ? rc->c : X.params.c;
    P.r_min = rc ? rc->r : X.params.r_min;
    P.rc_mode = rc ? 1 : 0;
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
    run_query_batch(P, X.scratch, X.device, s, X.main.s);
    if (!dev) {
        // results to host: pageable destinations go through one pinned staging
        // buffer (a pageable D2H is staged by the driver at a fraction of the
        // link rate), then a host copy; pinned destinations are copied directly
        struct Out {
            void* dst;
            const void* src;
            size_t bytes;
        };
        const Out outs[5] = {{ids, P.ids, nq * k * 4}, {dists, P.dists, nq * k * 8}, {n_hits, P.n_hits, nq * 4},
                             {radius, P.radius, nq * 8}, {cands, P.cands, nq * 8}};
        auto pageable = [](const void* ptr) {
            cudaPointerAttributes at{};
            if (cudaPointerGetAttributes(&at, ptr) != cudaSuccess) {
                cudaGetLastError();
                return true;
            }
            return at.type == cudaMemoryTypeUnregistered;
        };
        size_t staged = 0;
        for (const Out& o : outs)
            if (o.dst && pageable(o.dst)) staged += (o.bytes + 255) / 256 * 256;
        uint8_t* stage = staged ? reinterpret_cast<uint8_t*>(pinned_scratch(staged, 2)) : nullptr;
        size_t off = 0;
        std::vector<std::pair<const Out*, size_t>> copies;
        for (const Out& o : outs) {
            if (!o.dst) continue;
            if (pageable(o.dst)) {
                DETLSH_CUDA(cudaMemcpyAsync(stage + off, o.src, o.bytes, cudaMemcpyDeviceToHost, s));
                copies.emplace_back(&o, off);
                off += (o.bytes + 255) / 256 * 256;
            } else {
                DETLSH_CUDA(cudaMemcpyAsync(o.dst, o.src, o.bytes, cudaMemcpyDeviceToHost, s));
            }
        }
        DETLSH_CUDA(cudaStreamSynchronize(s));
        for (const auto& c : copies) std::memcpy(c.first->dst, stage + c.second, c.first->bytes);
        // host mode returns results, so it also reports a failed internal
        // check (device mode: detlsh_gpu_query_check)
        if (query_invariant_failed(X.scratch, s))
            throw CudaError("ck_ann: internal invariant violated (budget cut emitted != budget rows)");
    }
    // device mode: stream-ordered, returns once enqueued
}

}  // namespace detlsh_b200
