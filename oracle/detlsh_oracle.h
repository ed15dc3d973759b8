/* TEST INFRASTRUCTURE ONLY — the CPU oracle for the DET-LSH hot path.
 *
 * A plain-C restatement of the reference algorithm (arxiv 2406.10938,
 * /root/reference/proj).  Each function cites the reference file:line it
 * follows.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
 * leg may load it, and only as the checker.  The product never links it.
 *
 * Parity of this oracle is pinned two ways (tests/test_oracle.py):
 *   - golden values from the reference's own tests (test_cli.cpp:60-61,
 *     test_projection.cpp:14-16, test_query.cpp:36-41, ...);
 *   - bit-exact agreement with the reference library itself, compiled from the
 *     reference sources into oracle/_ref/libdetlsh_ref.so (oracle/Makefile).
 */
#ifndef DETLSH_ORACLE_H
#define DETLSH_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Same field order as detlsh::LshParams (projection.hpp:79-92). */
typedef struct orc_params {
    int32_t K, L;
    double c, beta, epsilon, alpha1, alpha2;
    int32_t n_regions;
    double sample_fraction;
    int32_t leaf_capacity;
    double r_min;
    int32_t k;
} orc_params;

typedef struct orc_rng {
    uint64_t mt[312];
    int mti;
    double spare;
    int have_spare;
} orc_rng;

void orc_rng_seed(orc_rng* r, uint64_t seed);
uint64_t orc_rng_next(orc_rng* r);
uint64_t orc_rng_bounded(orc_rng* r, uint64_t bound);
double orc_rng_normal(orc_rng* r);
uint64_t orc_mix_seed(uint64_t seed, uint64_t stream);
void orc_rng_stream(uint64_t seed, uint64_t count, uint64_t* out_u64, double* out_normal);

double orc_regularized_gamma_p(double a, double x);
double orc_chi2_cdf(double x, int k);
double orc_chi2_pdf(double x, int k);
double orc_chi2_quantile(double alpha, int k);
int orc_derive_params(int K, double c, int L, double* out4 /* alpha1 alpha2 epsilon beta */);
uint64_t orc_candidate_budget(double beta, uint64_t n, int k);

void orc_sample_hash_family(int d, int K, int L, uint64_t seed, float* out);
void orc_project_dataset(const float* coeffs, int K, int L, const float* data, uint64_t n, int d,
                         float* out /* [L][n][K] */);
int orc_select_row_breakpoints(float* sample, uint64_t n_s, int n_regions, orc_rng* rng,
                               float* out_row);
int orc_select_breakpoints(const float* proj, uint64_t n, int K, int L, int n_regions,
                           double sample_fraction, uint64_t seed, float* out_table,
                           uint64_t* sample_size, uint64_t* sample_idx /* [L][n_s] or NULL */,
                           uint64_t* draws_per_row /* [L*K] or NULL */);
int orc_locate_region(float v, const float* row, int n_regions);
void orc_encode_dataset(const float* proj, uint64_t n, int K, int L, const float* table,
                        int n_regions, uint8_t* out);

typedef struct orc_tree orc_tree;
orc_tree* orc_build_tree(const uint8_t* codes, uint64_t n, int K, int L, int n_regions, int space,
                         int max_size);
void orc_tree_free(orc_tree* t);
uint64_t orc_tree_num_nodes(const orc_tree* t);
void orc_tree_export(const orc_tree* t, int32_t* root_children, uint8_t* is_leaf,
                     uint8_t* split_dim, int32_t* left, int32_t* right, uint8_t* bits,
                     uint8_t* value, uint64_t* ebegin, uint32_t* ecount, uint32_t* positions);
double orc_mindist(const orc_tree* t, int node, const float* table, const float* q_proj);
uint64_t orc_range_query_optimized(const orc_tree* t, const float* table, const float* q_proj,
                                   double radius, uint64_t limit, uint32_t* out);

typedef struct orc_index orc_index;
orc_index* orc_build_index(const float* data, uint64_t n, int d, orc_params* params,
                           uint64_t seed);
/* Same pipeline with a caller-supplied breakpoint table (hybrid oracle). */
orc_index* orc_build_index_with_table(const float* data, uint64_t n, int d, orc_params* params,
                                      uint64_t seed, const float* table);
void orc_index_free(orc_index* x);
void orc_index_params(const orc_index* x, orc_params* out);
void orc_index_table(const orc_index* x, float* out);
const orc_tree* orc_index_tree(const orc_index* x, int i);
int orc_ck_ann(const orc_index* x, const float* q, int k, uint32_t* ids, double* dists,
               int* n_hits, double* radius_used, uint64_t* cands_seen);
void orc_brute_force_knn(const float* data, uint64_t n, int d, const float* Q, uint64_t nq, int k,
                         uint32_t* ids, double* dists);

#ifdef __cplusplus
}
#endif
#endif
