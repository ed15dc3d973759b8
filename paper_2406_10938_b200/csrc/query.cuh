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
    const uint2* leaf_cr;  // {half code | refined dims << 16, count} per leaf (tree.cuh)
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
    const int32_t* xn_u8;    // |x|^2 of those rows
    const uint8_t* data_tc;  // the same rows in MMA tiles (launch_pack_tc_tiles)
    const float* data_leaf;  // fp32 rows in tree-0 leaf order (non-integral datasets), or null
    const uint8_t* data_tcf; // those rows as bf16-triple MMA tiles (launch_pack_tcf_tiles), or null
    const float* xnf;        // (1 - kTcF32Kappa)|x|^2 of those rows, rounded down
    int row_f;               // bytes per bf16-triple row (round32(6 d))
    int tc_f32;              // this batch hands float queries to the bf16x3 scorer
    int row_u8;              // bytes per u8 row (d rounded up to 16)
    int u8_lpr;              // lanes per u8 row (power of two <= 32)
    double eps, c, r_min;
    uint64_t budget;
    int k;
    uint32_t max_leaves;  // max num_leaves over trees
    uint32_t trees_num_leaves0;  // tree 0's leaf count
    const uint32_t* trees_leaf_begin0;  // tree 0's leaf row ranges (host-visible copy of trees[0])
    const uint32_t* trees_leaf_count0;
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
    // processed range of processing slots [q_begin, q_end); with q_count set
    // the range ends at min(q_end, *q_count) (a count produced on the device)
    uint64_t q_begin, q_end;
    const uint32_t* q_count;
    // tensor-core verification hand-off (null: score every candidate here).
    // Indexed by slot - q_begin: the candidate set as a bitmap over tree-0
    // rows ([tc_W] words per slot: whole leaves + the cut leaf's taken
    // prefix), written by the plan kernel itself, and tau^2.
    uint32_t* tc_bm;
    uint64_t tc_W;
    int32_t* tc_tau2;
    int tc_allowed;  // host-side switch (DETLSH_F_NO_TC clears it)
    int force_exact;  // test hook: skip the approximate leaf scan
    int rc_mode;      // rc_ann: one pass at radius eps * r_min (= r), k = 1, c * r acceptance
    uint32_t tc_tau_rows;  // rows of the nearest leaves scored exactly for tau^2
    // tensor-core launches of the plan kernel compiled without the gather
    // verification: a query that cannot hand off is listed here instead and
    // verified by the gather re-run
    uint32_t* tc_over_list;
    uint32_t* tc_over_n;
};

constexpr int kQueryThreads = 256;
constexpr int kFastMaxK = 1024;  // k handled by the fast path (larger k: general path)

// Launch the batched query: fast path for every query (budget fills in tree 0,
// round 0, no dedup needed), then the general path for the rest.  Scratch is
// owned by the caller-provided QueryScratch (grown on demand).
struct QueryScratch {
    DevBuf<uint8_t> fast;  // per-CTA leaf item lists + candidate positions
    DevBuf<uint8_t> slow;  // per-slot leaf items + members
    DevBuf<uint32_t> slow_bm;  // per-slot n-bit member bitmaps (zero between queries)
    DevBuf<uint32_t> slow_list;
    DevBuf<uint64_t> slow_rec;  // [slots] deferred general-path queries (SlowRec)
    DevBuf<uint32_t> counters;
    DevBuf<unsigned long long> phases;  // [6] fast-path phase cycles (profiling only)
    size_t fast_slots = 0, slow_slots = 0;
    // the memory figure the scratch was sized against, per batch shape
    uint64_t avail_nq = 0, avail_budget = 0;
    size_t avail_bytes = 0;
    // tensor-core hand-off staging (per chunk of queries), kept across calls:
    // several of these are GB-sized and re-allocating them from the pool per
    // batch costs fresh mappings whenever the pool is fragmented.  Nothing reads
    // them after run_query_batch's last host sync, so the next call may reuse them.
    DevBuf<uint32_t> tc_bm, tc_surv_cnt;
    DevBuf<int32_t> tc_tau2, tc_qn;
    DevBuf<uint8_t> tc_q8;
    DevBuf<uint64_t> tc_surv;
    DevBuf<uint4> tc_rec;
    DevBuf<unsigned long long> tc_rec_cnt;
    DevBuf<uint32_t> over_list;
    DevBuf<uint32_t> tc_big;  // [chunk] slots whose survivors need the wide tc_finish
    // completion of the last batch that used this scratch: a batch on another
    // stream waits for it (the enqueue is serialised by the index mutex)
    cudaEvent_t done = nullptr;
    ~QueryScratch() {
        if (done) cudaEventDestroy(done);
    }
};

// ---- tensor-core exact verification (tc_score.cu) ----
constexpr uint32_t kTcFinishCap = 4096;  // survivors staged per query
constexpr uint32_t kTcFinishCapF32 = 16384;  // the same for float rows (tc_finish_f32 sorts in dynamic smem)
// pass-record slots one tc_score CTA may hold reserved ahead of use
// (epilogue warps x the run each reserves; checked in tc_score.cu)
constexpr uint64_t kTcRecReserve = 16 * 1024;

struct TcScoreArgs {
    const uint8_t* rows;   // u8 rows, tree-0 order, packed by launch_pack_tc_tiles
    const int32_t* xn;     // [n] |x|^2
    const uint8_t* q8;     // [nq][R] u8 queries
    const int32_t* qn;     // [nq] |q|^2
    const int32_t* tau2;   // [nq] inclusive dist^2 threshold; < 0: not a TC query
    const uint32_t* bm;    // [nq][W] candidate bits over tree-0 rows
    uint64_t W;            // words per query bitmap
    uint64_t n, nq;
    int R;
    uint32_t* surv_cnt;    // [nq]
    uint64_t* surv;        // [nq][cap] (dist^2 << 32 | row)
    uint32_t cap;
    // slot s of this batch is query order[slot0 + s] (or slot0 + s)
    const uint32_t* order;
    uint64_t slot0;
    uint32_t* work;        // unit counter (zeroed by the caller)
    uint4* rec;            // threshold passes {row, slot, dist^2, 0}; row ~0u: padding
    unsigned long long* rec_cnt;  // reserved records (zeroed by the caller)
    uint64_t rec_cap;
    // float datasets (f32 = 1): rows / queries are bf16 triples [hi, lo, hi] /
    // [hi, hi, lo] of R bytes, xn / qn are the float bits of (1 - kTcF32Kappa)
    // |x|^2 / |q|^2 rounded down, tau2 the float bits of an upper bound on the
    // k-th smallest exact dist^2; survivors are rescored exactly in fp64
    int f32;
};
constexpr float kTcF32Kappa = 1.0f / 4096.0f;  // relative slack of the bf16x3 dot product

size_t tc_score_smem(int R);
// rows of R bytes fit the scorer (R % 32 == 0; R > 256 takes the 128-query, K-chunked shape)
bool tc_score_fits(int R);
// float rows -> bf16-triple MMA tiles (R = round32(6 d) bytes) + (1 - kappa)|x|^2 (float, rounded down)
void launch_pack_tcf_tiles(const float* rows_leaf, uint64_t n, int d, int R, uint8_t* tiles, float* xnf,
                           cudaStream_t s);
void launch_tc_pack_queries_f32(const float* q, const uint32_t* order, uint64_t slot0, uint64_t m, int d,
                                int R, uint8_t* q16, float* qnf, cudaStream_t s);
void launch_tc_finish_f32(const TcScoreArgs& a, const uint32_t* perm0, const float* rows_leaf, const float* q,
                          int d, int k, double r_min, uint64_t budget, uint32_t* ids, double* dists,
                          int32_t* n_hits, double* radius, uint64_t* cands, uint32_t* overflow_list,
                          uint32_t* overflow_n, cudaStream_t s);
void launch_tc_pack_queries(const float* q, const uint32_t* order, uint64_t slot0, uint64_t m, int d,
                            int R, uint8_t* q8, int32_t* qn, cudaStream_t s);
void launch_row_norms_u8(const uint8_t* rows, uint64_t n, int R, int32_t* xn, cudaStream_t s);
// u8 rows -> 128-row tiles in the MMA operand layout ([ceil(n/128)][R/16][128][16] bytes)
void launch_pack_tc_tiles(const uint8_t* rows, uint64_t n, int R, uint8_t* tiles, cudaStream_t s);
void launch_tc_score(const TcScoreArgs& a, int device, cudaStream_t s);
// big_list [a.nq] / big_n (zeroed by the caller): the queries with more
// survivors than the first launch's sort width, finished by a second launch
void launch_tc_finish(const TcScoreArgs& a, const uint32_t* perm0, int k, double r_min,
                      uint64_t budget, uint32_t* ids, double* dists, int32_t* n_hits, double* radius,
                      uint64_t* cands, uint32_t* overflow_list, uint32_t* overflow_n, uint32_t* big_list,
                      uint32_t* big_n, cudaStream_t s);
// counters[] of QueryScratch: [0] slow-path queries, [1] sticky internal-invariant
// flag, [2] tensor-core overflow queries, [3] tc_score work counter
constexpr int kCntSlow = 0, kCntInvariant = 1, kCntOver = 2, kCntWork = 3, kCntTaken = 4, kCntBig = 6;

// tcgen05 kind::i8 self-test (tc_score.cu): C[128][N] = A[128][K] . B[N][K]^T.
void tc_gemm_u8_test(const uint8_t* hA, const uint8_t* hB, int N, int K, int32_t* hC);

// Phase cycles of the last profiled fast-path launch (setup, leaf scan, cut,
// emission, verification+top-k, output), summed over CTAs.
void last_query_phases(double* out6);

// Stream-ordered: every decision (tensor-core overflow, slow-path queries) is
// taken on the device; the host never waits, except to grow the scratch on the
// first call with a larger shape, and when profiling is enabled.
void run_query_batch(const QueryPlan& plan, QueryScratch& scratch, int device, cudaStream_t s,
                     cudaStream_t alloc_s);
// Reads the sticky internal-invariant flag (synchronises s).
bool query_invariant_failed(QueryScratch& scratch, cudaStream_t s);

// k-way merge of per-shard top-k lists: [shards][nq][k] -> [nq][k].
void launch_merge_topk(const double* sd, const uint64_t* sid, const int32_t* sh, int shards,
                       uint64_t nq, int k, double* od, uint64_t* oid, int32_t* oh,
                       cudaStream_t s);

}  // namespace detlsh_b200
