/* detlsh_b200 — B200-native (sm_100a) DET-LSH index build and c^2-k-ANN query.
 *
 * This is the drop-in boundary: a C ABI (plain pointers and sizes, no torch or
 * C++ types) over the CUDA implementation in paper_2406_10938_b200/csrc.  Each
 * entry point names the reference interface it replaces (paths relative to
 * /root/reference/proj).  The C++ facade in include/detlsh_b200.hpp restores
 * the reference's own C++ signatures on top of it.
 *
 * Errors: every int-returning call returns DETLSH_OK (0) or a status code;
 * the message is in detlsh_gpu_last_error() (thread-local).  Status codes map
 * onto the reference's exception taxonomy:
 *     DETLSH_E_INVALID  -> std::invalid_argument (index.cpp:17-23, 293-298)
 *     DETLSH_E_CUDA     -> std::runtime_error (device failure / out of memory)
 *     DETLSH_E_FORMAT   -> detlsh::FormatError (errors.hpp:19-28)
 * No C++ exception ever crosses this boundary.
 *
 * Ownership: a detlsh_gpu_index owns its device buffers (dataset copy unless
 * DETLSH_F_BORROW_DATA, hash family, breakpoint table, codes, trees).  Callers
 * own every host buffer they pass.  An index is immutable after build; queries
 * against one index may run concurrently from several host threads.
 */
#ifndef DETLSH_B200_H
#define DETLSH_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DETLSH_OK 0
#define DETLSH_E_INVALID 1
#define DETLSH_E_CUDA 2
#define DETLSH_E_FORMAT 3

/* flags */
#define DETLSH_F_DEVICE_PTRS 0x1u  /* point / query / output pointers are device pointers */
#define DETLSH_F_SAMPLE_GPU 0x2u   /* GPU-native breakpoint sample;
                                      default is the reference-compatible sample */
#define DETLSH_F_BORROW_DATA 0x4u  /* with DEVICE_PTRS: keep the caller's device dataset */
#define DETLSH_F_NO_CODES 0x8u     /* drop the [L][n][K] code array after build */
#define DETLSH_F_NO_U8 0x10u       /* never use the exact u8 verification rows (fp64 path only) */
#define DETLSH_F_PAA 0x40u         /* build: the DET-ONLY variant (build_det_only_index,
                                      index.cpp:220-232): PAA segment means, L = 1 */
#define DETLSH_F_NO_TC 0x20u       /* query: verify on the per-query gather path only (no
                                      tcgen05 dataset-major scoring); results are identical */

/* detlsh::LshParams (projection.hpp:79-92), same field order and meaning:
 * beta <= 0 -> derived; r_min <= 0 -> estimated at build; epsilon/alpha1/
 * alpha2 are outputs (filled by build). */
typedef struct detlsh_params {
    int32_t K, L;
    double c, beta, epsilon, alpha1, alpha2;
    int32_t n_regions;
    double sample_fraction;
    int32_t leaf_capacity;
    double r_min;
    int32_t k;
} detlsh_params;

typedef struct detlsh_gpu_index detlsh_gpu_index;
typedef struct detlsh_gpu_tree detlsh_gpu_tree;

/* ---- host-only numerics (no GPU needed) ---------------------------------- */

/* candidate_budget (index.hpp:50, index.cpp:190-194). */
uint64_t detlsh_candidate_budget(double beta, uint64_t n, int32_t k);
/* derive_params (projection.hpp:75-77, projection.cpp:92-102); out4 =
 * {alpha1, alpha2, epsilon, beta}. */
int detlsh_derive_params(int32_t K, double c, int32_t L, double* out4);
/* sample_hash_family (projection.hpp:30, projection.cpp:11-23); out [L][K][d]. */
int detlsh_sample_hash_family(int32_t d, int32_t K, int32_t L, uint64_t seed, float* out);
/* chi2_cdf / chi2_quantile (chi2.hpp:10-17). */
double detlsh_chi2_cdf(double x, int32_t k);
double detlsh_chi2_quantile(double alpha, int32_t k);
/* select_row_breakpoints (encoder.hpp:36, encoder.cpp:57-103) as replayed by
 * the host for the reference-compatible sample: reorders `sample` in place
 * exactly as the reference does, writes n_regions+1 boundaries, and reports
 * how many RNG draws (partition calls) it consumed from Rng(rng_seed). */
int detlsh_select_row_breakpoints(float* sample, uint64_t n_s, int32_t n_regions,
                                  uint64_t rng_seed, float* row, uint64_t* draws);

int detlsh_device_count(void);
const char* detlsh_gpu_last_error(void);
const char* detlsh_version(void);

/* ---- instrumentation -------------------------------------------------------- */
/* Kernels this library has launched in this process (every launch site). */
uint64_t detlsh_launch_count(void);
/* Per-kernel CUDA-event timing on the launching stream (off by default). */
void detlsh_profile_enable(int32_t on);
/* Drains recorded events: up to cap entries of (total ms, launches); names
 * ';'-separated into `names`.  Returns the number of entries. */
int detlsh_profile_collect(char* names, int32_t names_cap, double* ms, uint64_t* launches,
                           int32_t cap);
/* Self-test of the tensor-core path: C[128][N] = A[128][K] . B[N][K]^T on one
 * tcgen05 (kind::i8, u8 x u8 -> s32) tile; host pointers. */
int detlsh_test_tc_gemm_u8(const uint8_t* A, const uint8_t* B, int32_t N, int32_t K, int32_t* C);
/* SM cycles per phase of the last profiled query batch, summed over CTAs:
 * setup, leaf scan, budget cut, candidate emission, verification+top-k, output. */
void detlsh_query_phase_cycles(double* out6);

/* ---- index build ----------------------------------------------------------- */

/* build_index (index.hpp:39, index.cpp:212-218): points [n][d] fp32 row-major.
 * params->epsilon/alpha1/alpha2/beta/r_min are written back as build derives
 * them (the reference's DetIndex::params). */
int detlsh_gpu_build(const float* points, uint64_t n, int32_t d, detlsh_params* params,
                     uint64_t seed, int32_t device, uint32_t flags, detlsh_gpu_index** out);

/* build_index_with_family (index.hpp:42-43, index.cpp:196-210): caller-supplied
 * coefficients [L][K][d] (host memory); K and L come from the family. */
int detlsh_gpu_build_with_family(const float* points, uint64_t n, int32_t d,
                                 detlsh_params* params, const float* coeffs, int32_t K,
                                 int32_t L, uint64_t family_seed, uint64_t seed, int32_t device,
                                 uint32_t flags, detlsh_gpu_index** out);

void detlsh_gpu_free(detlsh_gpu_index* index);

/* ---- queries ------------------------------------------------------------------ */

/* ck_ann (index.hpp:87, index.cpp:292-331), batched: nq queries [nq][d].
 * Outputs row-major [nq][k]: ids (dataset positions) and exact distances,
 * ascending by (distance, position); n_hits[q] <= k (the reference returns
 * min(k, |S|) hits); radius_used[q] = r_min * c^t; cands_seen[q] = |S|.
 * Any output pointer may be NULL.  stream: cudaStream_t or NULL (the index's
 * own stream).  With DETLSH_F_DEVICE_PTRS all pointers are device pointers and
 * the call is stream-ordered: it returns once enqueued, every decision (the
 * tensor-core overflow re-runs, the general-path queries) is taken on the
 * device, and batches on different streams are ordered through the index's
 * scratch.  The host waits only when a batch needs more scratch than every
 * earlier batch of the index (the first call of a shape), and when the
 * per-kernel profile is enabled; after that first call the enqueue can be
 * captured into a CUDA graph.  Host pointers: the call returns with the
 * results and reports an internal failure as DETLSH_E_CUDA. */
int detlsh_gpu_query(const detlsh_gpu_index* index, const float* queries, uint64_t nq,
                     int32_t k, uint32_t flags, uint32_t* ids, double* dists, int32_t* n_hits,
                     double* radius_used, uint64_t* cands_seen, void* stream);

/* Synchronises `stream` (NULL: the index's own) and reports, as DETLSH_E_CUDA,
 * a failed internal check of any earlier device-pointer batch (the check is
 * sticky: host-pointer calls report it on return). */
int detlsh_gpu_query_check(const detlsh_gpu_index* index, void* stream);

/* rc_ann (index.hpp, index.cpp:267-290), batched: for each query the closest
 * candidate of one pass over the trees at radius epsilon * r (budget
 * candidate_budget(beta, n, 1)); found[q] = 1 with (ids[q], dists[q]) when the
 * budget was reached or that candidate lies within c * r, else found[q] = 0
 * (the reference's std::nullopt).  r > 0 and c > 1, else DETLSH_E_INVALID.
 * cands_seen may be NULL.  Pointer/stream conventions as detlsh_gpu_query. */
int detlsh_gpu_rc_ann(const detlsh_gpu_index* index, const float* queries, uint64_t nq, double r,
                      double c, uint32_t flags, uint32_t* ids, double* dists, int32_t* found,
                      uint64_t* cands_seen, void* stream);

/* estimate_rmin (index.hpp:91, index.cpp:333-374): the smallest radius on the
 * geometric grid (anchored at the median pairwise projected distance of 32
 * strided points / epsilon) whose candidate count reaches
 * candidate_budget(beta, n, k) while radius / c falls short, median over the
 * n_probes probe queries [n_probes][d] (host, or device with
 * DETLSH_F_DEVICE_PTRS).  n_probes == 0 -> DETLSH_E_INVALID ("no probe queries"). */
int detlsh_gpu_estimate_rmin(const detlsh_gpu_index* index, const float* probes, uint64_t n_probes, int32_t k,
                             uint32_t flags, double* r_min);

/* DetIndex::project_query (index.cpp:181-188) for a batch: out [L][nq][K], the
 * same bits as the reference's project_point (host, or device pointers). */
int detlsh_gpu_project_query(const detlsh_gpu_index* index, const float* queries, uint64_t nq, float* out,
                             uint32_t flags);

/* Range queries on one DE-Tree (de_tree.hpp:85-100), host pointers: q_proj
 * [nq][K] projected queries of that tree's space, radius [nq].
 *   default: range_query_optimized -- the entries of every leaf with
 *     mindist <= radius in ascending (mindist, node index) order, leaf by leaf,
 *     stopping after `limit` positions (the CandidateSink returning false);
 *   DETLSH_RANGE_EXACT: range_query_exact -- exactly the positions whose
 *     projected distance is <= radius, in the reference's DFS order.
 * positions [nq][cap] (the first cap of each list), counts[q] = the list's
 * full length. */
#define DETLSH_RANGE_EXACT 0x100u
int detlsh_gpu_range_query(const detlsh_gpu_index* index, int32_t tree, const float* q_proj, uint64_t nq,
                           const double* radius, uint64_t limit, uint32_t flags, uint32_t* positions, uint64_t cap,
                           uint64_t* counts);

/* ---- exact ground truth ------------------------------------------------------- */
/* brute_force_knn (metrics.hpp, metrics.cpp:8-33) on the GPU: for each query
 * the k smallest l2_distance_sq (sequential fp64, dataset.hpp:23-30) over all
 * n points, ordered by (dist^2, position); dists = sqrt(dist^2).  dist2_bound
 * (optional, [nq], host or device) is an upper bound per query on the k-th
 * smallest dist^2 (e.g. the squared k-th distance ck_ann returned); without
 * it a strided sample sets the threshold.  Same answers either way.  k <= 1024.
 * Pointers are device pointers with DETLSH_F_DEVICE_PTRS, else host. */
int detlsh_gpu_brute_force_knn(const float* data, uint64_t n, int32_t d, const float* queries, uint64_t nq,
                               int32_t k, const double* dist2_bound, uint32_t flags, uint32_t* ids,
                               double* dists, int32_t device, void* stream);

/* ---- vector files (io.hpp, io.cpp:28-85) ------------------------------------ */
/* Shape of a .fvecs / .bvecs / .ivecs file (kind: 0 f32, 1 u8, 2 i32, from the
 * extension as vec_element_from_path): every record header is validated.
 * Errors: unknown extension -> DETLSH_E_INVALID; unreadable, truncated,
 * non-positive or inconsistent dimension -> DETLSH_E_FORMAT (FormatError). */
int detlsh_vectors_shape(const char* path, uint64_t* n, int32_t* d, int32_t* kind);
/* read_vectors straight to device memory: `values` is a caller-owned device
 * buffer [n][d] fp32 (n, d from detlsh_vectors_shape); the file streams through
 * pinned chunks and u8 / i32 elements are widened to fp32 on the GPU. */
int detlsh_gpu_read_vectors(const char* path, float* values, uint64_t n, int32_t d, int32_t device,
                            void* stream);

/* Multi-GPU merge: per-shard top-k lists gathered from `shards`
 * ranks, layout [shards][nq][k] (dist, global id); writes the global top-k
 * ascending by (dist, id).  Device pointers, stream-ordered. */
int detlsh_gpu_merge_topk(const double* shard_dists, const uint64_t* shard_ids,
                          const int32_t* shard_hits, int32_t shards, uint64_t nq, int32_t k,
                          double* out_dists, uint64_t* out_ids, int32_t* out_hits,
                          void* stream);

/* ---- point-sharded index, one process --------------------------
 * The dataset splits into `shards` contiguous row ranges [s*n/S, (s+1)*n/S);
 * shard s is an independent DET-LSH index (own sample, breakpoints, trees and
 * r_min; budget ceil(beta * n_s + k)) built on devices[s] with the same seed,
 * all shards concurrently (a device may hold several).  A query batch runs on
 * every shard at once; each shard's top-k goes to devices[0] (peer copies over
 * NVLink) and is merged by (distance, global position) -- the same answer as
 * the reference's build_index + ck_ann on each shard followed by that merge.
 * params: the template in, the derived fields (shared by all shards) out;
 * per-shard r_min through detlsh_gpu_sharded_shard + detlsh_gpu_get_params. */
typedef struct detlsh_gpu_sharded_index detlsh_gpu_sharded_index;
int detlsh_gpu_sharded_build(const float* points, uint64_t n, int32_t d, detlsh_params* params, uint64_t seed,
                             const int32_t* devices, int32_t shards, uint32_t flags,
                             detlsh_gpu_sharded_index** out);
/* ids are global u64 positions, [nq][k] ascending by (distance, position).
 * Device pointers (DETLSH_F_DEVICE_PTRS) live on devices[0] and the call is
 * stream-ordered on `stream` (a stream of devices[0], or NULL). */
int detlsh_gpu_sharded_query(detlsh_gpu_sharded_index* index, const float* queries, uint64_t nq, int32_t k,
                             uint32_t flags, uint64_t* ids, double* dists, int32_t* n_hits, void* stream);
int32_t detlsh_gpu_sharded_count(const detlsh_gpu_sharded_index* index);
/* Borrowed handle of shard s (valid while the sharded index lives; never freed
 * by the caller): every export / query entry point above accepts it. */
const detlsh_gpu_index* detlsh_gpu_sharded_shard(const detlsh_gpu_sharded_index* index, int32_t s,
                                                 uint64_t* row_begin, uint64_t* row_end);
void detlsh_gpu_sharded_free(detlsh_gpu_sharded_index* index);

/* ---- synthetic data (bench / test utility) ----------------------------------
 * Rows [row0, row0 + n) of a seeded synthetic dataset, written as fp32
 * [n][d] into device memory `out` (generated on the GPU: config 5's 51 GB does
 * not go through host memory).  kind 0: 0 with probability 1/2, else
 * min(255, geometric(p = 0.05)) -- BASELINE.json configs 2 / 5.  Element
 * (r, t) depends on (seed, r * d + t) only.  stream NULL: synchronous. */
int detlsh_gpu_synth(int32_t kind, uint64_t seed, uint64_t row0, uint64_t n, int32_t d, float* out, int32_t device,
                     void* stream);

/* ---- export (DetIndex fields, index.hpp:24-37) ------------------------------ */
int detlsh_gpu_get_params(const detlsh_gpu_index* index, detlsh_params* out);
uint64_t detlsh_gpu_n(const detlsh_gpu_index* index);
int32_t detlsh_gpu_d(const detlsh_gpu_index* index);
uint64_t detlsh_gpu_sample_size(const detlsh_gpu_index* index);
/* HashFamily::seed (projection.hpp:18): mix_seed(seed, 0) for build_index, the
 * caller's for build_index_with_family; has_family is 0 for DET-ONLY (PAA). */
uint64_t detlsh_gpu_family_seed(const detlsh_gpu_index* index);
int32_t detlsh_gpu_has_family(const detlsh_gpu_index* index);
/* Bytes per exact-u8 verification row (0 when the dataset is not integral in [0,255]). */
int32_t detlsh_gpu_row_u8(const detlsh_gpu_index* index);
int detlsh_gpu_export_family(const detlsh_gpu_index* index, float* out /* [L][K][d] */);
int detlsh_gpu_export_table(const detlsh_gpu_index* index, float* out /* [L][K][N_r+1] */);
int detlsh_gpu_export_codes(const detlsh_gpu_index* index, uint8_t* out /* [L][n][K] */);
/* DeTree (de_tree.hpp:44-58) of tree `tree`, nodes in the reference's build
 * order; positions concatenated leaf by leaf (ebegin/ecount index them). */
int detlsh_gpu_tree_num_nodes(const detlsh_gpu_index* index, int32_t tree, uint64_t* out);
int detlsh_gpu_export_tree(const detlsh_gpu_index* index, int32_t tree, int32_t* root_children,
                           uint8_t* is_leaf, uint8_t* split_dim, int32_t* left, int32_t* right,
                           uint8_t* bits, uint8_t* value, uint64_t* ebegin, uint32_t* ecount,
                           uint32_t* positions);
/* detlsh::save_index (persist.hpp:17, persist.cpp:99-149): the DETL v1 byte
 * stream of the index -- the same bytes the reference writes for the same
 * build, so detlsh::load_index + ck_ann serve a GPU-built index.  *size gets
 * the stream length; out (may be NULL) must hold cap >= *size bytes.  Entry
 * symbols are recomputed on the GPU if the build dropped the codes; the
 * dataset fingerprint (FNV-1a, dataset.cpp:22-30) is computed on the host. */
int detlsh_gpu_save_detl(detlsh_gpu_index* index, uint8_t* out, uint64_t cap, uint64_t* size);

/* Per-stage device/host milliseconds of the last build (diagnostics):
 * names written as a ';'-separated list into `names` (cap bytes). */
int detlsh_gpu_build_timings(const detlsh_gpu_index* index, double* ms, int32_t cap,
                             char* names, int32_t names_cap);

/* ---- stage functions (reference stage API on the device) ------------------- */

/* project_dataset (projection.hpp:58, projection.cpp:47-60): out [L][n][K]. */
int detlsh_gpu_project(const float* coeffs, int32_t K, int32_t L, const float* points,
                       uint64_t n, int32_t d, float* out, int32_t device, uint32_t flags);
/* select_breakpoints (encoder.hpp:41-42, encoder.cpp:105-143): projected
 * [L][n][K] -> table [L][K][N_r+1]. */
int detlsh_gpu_select_breakpoints(const float* projected, uint64_t n, int32_t K, int32_t L,
                                  int32_t n_regions, double sample_fraction, uint64_t seed,
                                  float* table, uint64_t* sample_size, int32_t device,
                                  uint32_t flags);
/* encode_dataset (encoder.hpp:63, encoder.cpp:155-176): out [L][n][K] u8. */
int detlsh_gpu_encode(const float* projected, uint64_t n, int32_t K, int32_t L,
                      const float* table, int32_t n_regions, uint8_t* out, int32_t device,
                      uint32_t flags);
/* build_tree (de_tree.hpp:61, de_tree.cpp:133-152) from codes [L][n][K]. */
int detlsh_gpu_build_tree(const uint8_t* codes, uint64_t n, int32_t K, int32_t L,
                          int32_t n_regions, int32_t space, int32_t max_size, int32_t device,
                          uint32_t flags, detlsh_gpu_tree** out);
int detlsh_gpu_tree_nodes(const detlsh_gpu_tree* tree, uint64_t* out);
int detlsh_gpu_tree_export(const detlsh_gpu_tree* tree, int32_t* root_children,
                           uint8_t* is_leaf, uint8_t* split_dim, int32_t* left, int32_t* right,
                           uint8_t* bits, uint8_t* value, uint64_t* ebegin, uint32_t* ecount,
                           uint32_t* positions);
void detlsh_gpu_tree_free(detlsh_gpu_tree* tree);

#ifdef __cplusplus
}
#endif
#endif /* DETLSH_B200_H */
