// The assembled GPU index (detlsh::DetIndex, index.hpp:24-37) and its
// build / query orchestration.
#pragma once

#include <cuda_runtime.h>

#include <memory>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "../../include/detlsh_b200.h"
#include "common.cuh"
#include "query.cuh"
#include "stages.cuh"
#include "tree.cuh"

namespace detlsh_b200 {

struct GpuIndex {
    // streams first: members are destroyed in reverse order, so every buffer
    // below is released (stream-ordered) before its stream goes away
    OwnedStream main;
    std::vector<std::unique_ptr<OwnedStream>> side;  // [0, L): trees, [L]: r_min
    int device = 0;
    detlsh_params params{};
    uint64_t n = 0;
    int d = 0;
    uint64_t family_seed = 0, sample_size = 0;
    bool sample_gpu = false;
    bool paa = false;  // DET-ONLY variant: PAA projection (projection.cpp:62-90), L = 1
    const float* data = nullptr;  // device, [n][d]
    DevBuf<float> data_buf;
    std::vector<float> h_coeffs;  // [L][K][d]
    DevBuf<float> coeffs;
    DevBuf<double> coeffs_t;
    ProjTc proj_tc;  // tensor-core projection operand (8-bit-integer data)
    DevBuf<float> table;
    std::vector<float> h_table;
    DevBuf<uint8_t> codes;
    DevBuf<uint8_t> data_u8;  // exact u8 rows in tree-0 leaf order (integral datasets)
    DevBuf<int32_t> xn_u8;    // |x|^2 of those rows (tensor-core verification)
    DevBuf<uint8_t> data_tc;  // those rows as 128-row MMA operand tiles
    DevBuf<float> data_leaf;  // non-integral datasets: fp32 rows in tree-0 leaf order
    DevBuf<uint8_t> data_tcf; // those rows as bf16-triple MMA tiles (bf16x3 verification)
    DevBuf<float> xnf;        // (1 - kappa)|x|^2 of those rows, rounded down
    int row_f = 0;            // bytes per bf16-triple row
    int row_u8 = 0, u8_lpr = 0;
    std::vector<std::unique_ptr<DevTree>> trees;
    // per tree: leaf indices in the reference's DFS order (range_query_exact), built on first use
    std::vector<std::unique_ptr<DevBuf<uint32_t>>> dfs_leaves;
    DevBuf<QTree> qtrees;
    uint32_t max_leaves = 0;
    QueryScratch scratch;
    std::mutex qmu;
    std::vector<std::pair<std::string, double>> timings;
};

std::unique_ptr<GpuIndex> build_index_impl(const float* points, uint64_t n, int d,
                                           detlsh_params* params, const float* coeffs_host,
                                           uint64_t family_seed, uint64_t seed, int device,
                                           uint32_t flags);

// rc_ann (index.cpp:267-290) instead of ck_ann: one pass over the trees at
// radius eps * r with budget B(k = 1), then the closest candidate (n_hits 1) if
// the budget was reached or it lies within c * r, else none (n_hits 0).
struct RcArgs {
    double r, c;
};

void query_impl(GpuIndex& X, const float* queries, uint64_t nq, int k, uint32_t flags,
                uint32_t* ids, double* dists, int32_t* n_hits, double* radius, uint64_t* cands,
                cudaStream_t user_stream, const RcArgs* rc = nullptr);

void validate_params(const detlsh_params& p, uint64_t n, int d);
// estimate_rmin (index.hpp:91) for caller probes [np][d] (host or device per flags)
double estimate_rmin_impl(GpuIndex& X, const float* probes, uint64_t np, int k, uint32_t flags);
// range_query_optimized / range_query_exact (de_tree.cpp:199-258) on tree `tree`
// for projected queries [nq][K] (host); positions [nq][cap], counts [nq]
void range_query_impl(GpuIndex& X, int tree, const float* q_proj, uint64_t nq, const double* radius, uint64_t limit,
                      bool exact, uint32_t* out, uint64_t cap, uint64_t* counts);
// DetIndex::project_query (index.cpp:181-188) for a batch: out [L][nq][K]
void project_queries_impl(GpuIndex& X, const float* q, uint64_t nq, float* out, uint32_t flags);
// DETL v1 byte stream of the index (persist.cu), identical to detlsh::save_index
std::vector<uint8_t> save_detl(GpuIndex& X);
uint64_t sample_size_for(double frac, uint64_t n, int NR);
bool is_pow2(int v);

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev);
    ~DeviceGuard();
};

}  // namespace detlsh_b200
