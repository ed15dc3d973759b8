// Launchers for the build-stage kernels (stages.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"

namespace detlsh_b200 {

// coeffs [L][K][d] fp32 -> transposed double [d][LKp] (LKp = LK rounded up to 64)
int lk_padded(int LK);
void prepare_coeffs_t(const float* d_coeffs, int LK, int d, double* d_coeffs_t, cudaStream_t s);

// project_dataset (projection.cpp:47-60), exact: fp64 FMA chain in t order
// (float x float is exact in double, so fma == mul+add), rounded once.
// out [L][n][K] fp32.
// `prof` names the profile scope (the early sample-row projection is reported apart)
//
// With `tc` (prepared by prepare_proj_tc for the same coefficients) the exact
// projection of 8-bit-integer data runs on the tensor cores (project_tc.cu:
// tcgen05 kind::i8 over base-256 coefficient digits, each output certified
// against the reference's fp64 rounding, undecided ones recomputed); non-
// integral data falls back to the FP64 DMMA kernel on the device.  With
// `d_nonint`, the word receives 0 iff every value was an integer in [0, 255]
// (the tensor-core pass only; the DMMA path leaves it untouched).
struct ProjTc;
void launch_project_exact(const float* d_points, uint64_t n, int d, const double* d_coeffs_t,
                          int K, int L, float* d_out, cudaStream_t s, const char* prof = "project_exact",
                          const ProjTc* tc = nullptr, uint32_t* d_nonint = nullptr);

// Operand image for the tensor-core projection: coefficient digits
// [N = 5 LKp columns][R bytes] in the UMMA K-major layout (pieces of P
// columns), fp32 2^sc per output.  ok = false when the shape is not covered
// (LK > 96, d > 256, d % 4 != 0) or DETLSH_PROJ_TC=0; a launch also declines
// (-> DMMA) when four 32-row staging chunks do not fit beside the operands (d > ~200).
struct ProjTc {
    bool ok = false;
    int LK = 0, LKp = 0, d = 0, R = 0, N = 0, P = 0;
    const float* coeffs = nullptr;  // [LK][d] fp32, caller-owned (the fixup reads it)
    DevBuf<uint8_t> bimg;
    DevBuf<int> scale;  // [0, LKp): grid exponent sc_o, [LKp, 2 LKp): truncated coefficients
};
void prepare_proj_tc(const float* d_coeffs, int LK, int d, ProjTc& tc, cudaStream_t s);
bool launch_project_tc(const float* d_points, uint64_t n, int d, const ProjTc& tc, const double* d_ct,
                       int K, int L, float* d_out, cudaStream_t s, const char* prof, uint32_t* d_nonint);
void launch_project_dmma_guarded(const float* d_points, uint64_t n, int d, const double* d_ct, int K,
                                 int L, float* d_out, const uint32_t* d_guard, uint32_t cap, cudaStream_t s);

// paa_project_dataset (projection.cpp:62-90): out [1][n][K] fp32, segment j =
// [j*(d/K), (j+1)*(d/K)) (the last takes the remainder), mean = sequential
// double sum / length, rounded once to float.
void launch_project_paa(const float* d_points, uint64_t n, int d, int K, float* d_out, cudaStream_t s,
                        const char* prof = "project_paa");

// sample values: out[j][t] = proj[space][idx[t]][j]  (j < K, t < n_s)
// out[(r Lg + i) K + j] = proj[(i n + pos[r]) K + j] for r < m, i < Lg (device positions)
void launch_gather_proj_rows(const float* d_proj, uint64_t n, int K, int Lg, const uint64_t* d_pos, int m,
                             float* d_out, cudaStream_t s);
// v[i] = i for i < n
void launch_iota_u32(uint32_t* v, uint64_t n, cudaStream_t s);
void launch_gather_sample(const float* d_proj_space, const uint32_t* d_idx, uint64_t n_s, int K,
                          float* d_out, cudaStream_t s);

// GPU-native sample indices for one space: first n_s values of a keyed
// Feistel permutation of [0, n).
void launch_feistel_sample(uint64_t n, uint64_t n_s, uint64_t key, uint32_t* d_idx,
                           cudaStream_t s);

// Exact order statistics per row (GPU sample mode): rows [R][n_s] (fp32),
// writes table rows [R][NR+1]: row[0]=min, row[t]=sorted[span*t-1], row[NR]=max.
// `sync` = false leaves the work queued on s (temporaries are stream-ordered).
// `work` (optional): temporaries kept by the caller across calls -- the
// build's breakpoint loop reserves them before its tree workers start, whose
// GB-sized allocations would otherwise hold this thread in the allocator.
struct OrderStatWork {
    DevBuf<uint32_t> kmin, kmax, hist, tcount, count, v0, v1, tmp;
    DevBuf<uint8_t> flags;
    DevBuf<uint64_t> k0, k1;
    void reserve(int R, uint64_t n_s, cudaStream_t s);
};
void gpu_order_stat_table(const float* d_rows, int R, uint64_t n_s, int n_regions,
                          float* d_table, cudaStream_t s, bool sync = true, OrderStatWork* work = nullptr);

// encode_dataset (encoder.cpp:155-176): branchless lower_bound over the
// N_r+1 boundaries staged in shared memory; out [L][n][K] u8.
void launch_encode(const float* d_proj, uint64_t n, int K, int L, const float* d_table,
                   int n_regions, uint8_t* d_codes, cudaStream_t s);

// r_min support (index.cpp:33-136 restated as an order statistic):
// D[p][z] = min_i l2_double(probe_proj[p][i], proj[i][z]); returns via d_T
// the bits of the `rank`-th smallest (1-based) D per probe.
void rmin_order_stats(const float* d_proj, uint64_t n, int K, int L, const float* d_probe_proj,
                      int n_probes, uint64_t rank, double* d_D, uint32_t* d_hist,
                      uint64_t* h_T_bits, cudaStream_t s);

// The same in pieces, for projections produced chunk by chunk: rmin_begin,
// then launch_rmin_dist per chunk of m points starting at z0 (projections
// [L][m][K]; D is [np][n_total]), then rmin_select.  At most 10 probes.
struct RminSelect {
    int np;
    DevBuf<unsigned long long> lo, hi;
    DevBuf<uint64_t> need;
    DevBuf<int> shift;
    DevBuf<uint32_t> hist;
    explicit RminSelect(int np);
};
void rmin_begin(RminSelect& sel, cudaStream_t s);
void launch_rmin_dist(const float* d_proj_chunk, uint64_t m, uint64_t z0, uint64_t n_total, int K, int L,
                      const float* d_probe_proj, RminSelect& sel, double* d_D, cudaStream_t s);
void rmin_select(RminSelect& sel, const double* d_D, uint64_t n, uint64_t rank, uint64_t* h_T_bits,
                 cudaStream_t s);

}  // namespace detlsh_b200

namespace detlsh_b200 {
// True when every value is an integer in [0, 255] (exact u8 verification path).
bool data_is_u8(const float* d_x, uint64_t total, cudaStream_t s);
// rows [perm[r]] -> out[r] (fp32, tree-0 leaf order)
void launch_pack_f32(const float* d_x, const uint32_t* d_perm, uint64_t n, int d, float* d_out, cudaStream_t s);
// Rows of d_x re-ordered by d_perm and narrowed to u8, row_bytes per row.
void launch_pack_u8(const float* d_x, const uint32_t* d_perm, uint64_t n, int d, int row_bytes,
                    uint8_t* d_out, cudaStream_t s);
}  // namespace detlsh_b200
