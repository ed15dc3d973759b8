// Batched c^2-k-ANN query (ck_ann, index.cpp:292-331) on the GPU.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"

namespace detlsh_b200 {

struct QTree {
    const uint32_t* leaf_node;
    const uint32_t* leaf_begin;
    const uint32_t* leaf_count;
    const uint8_t* leaf_box;
    const uint32_t* perm;
    uint32_t num_leaves;
};

struct QueryPlan {
    // index
    const float* data;  // [n][d]
    uint64_t n;
    int d, K, L, NR;
    const float* table;   // [L][K][NR+1]
    const QTree* trees;   // device array [L]
    const uint32_t* perm0;   // tree 0 permutation (row index -> dataset position)
    const uint8_t* data_u8;  // exact u8 rows in tree-0 order, or null
    int row_u8;              // bytes per u8 row (d rounded up to 16)
    int u8_lpr;              // lanes per u8 row (power of two <= 32)
    double eps, c, r_min;
    uint64_t budget;
    int k;
    uint32_t max_leaves;  // max num_leaves over trees
    // batch
    const float* q;      // [nq][d]
    const float* qproj;  // [L][nq][K]
    uint64_t nq;
    // outputs ([nq][k] / [nq])
    uint32_t* ids;
    double* dists;
    int32_t* n_hits;
    double* radius;
    uint64_t* cands;
    // optional: per-phase SM cycles of the fast path (setup, leaf scan, cut,
    // emission, verification+top-k, output), summed over CTAs
    unsigned long long* phase_cycles;
    // optional processing order (locality): processing slot i handles query order[i]
    const uint32_t* order;
};

constexpr int kQueryThreads = 256;
constexpr int kFastMaxK = 1024;  // k handled by the fast path (larger k: general path)

// Launch the batched query: fast path for every query (budget fills in tree 0,
// round 0, no dedup needed), then the general path for the rest.  Scratch is
// owned by the caller-provided QueryScratch (grown on demand).
struct QueryScratch {
    DevBuf<uint8_t> fast;  // per-CTA leaf item lists + candidate positions
    DevBuf<uint8_t> slow;  // per-slot bitmap + members
    DevBuf<uint32_t> slow_list;
    DevBuf<uint32_t> counters;
    DevBuf<unsigned long long> phases;  // [6] fast-path phase cycles (profiling only)
    size_t fast_slots = 0, slow_slots = 0;
};

// tcgen05 kind::i8 self-test (tc_score.cu): C[128][N] = A[128][K] . B[N][K]^T.
void tc_gemm_u8_test(const uint8_t* hA, const uint8_t* hB, int N, int K, int32_t* hC);

// Phase cycles of the last profiled fast-path launch (setup, leaf scan, cut,
// emission, verification+top-k, output), summed over CTAs.
void last_query_phases(double* out6);

void run_query_batch(const QueryPlan& plan, QueryScratch& scratch, int device, cudaStream_t s,
                     cudaStream_t alloc_s);

// k-way merge of per-shard top-k lists: [shards][nq][k] -> [nq][k].
void launch_merge_topk(const double* sd, const uint64_t* sid, const int32_t* sh, int shards,
                       uint64_t nq, int k, double* od, uint64_t* oid, int32_t* oh,
                       cudaStream_t s);

}  // namespace detlsh_b200
