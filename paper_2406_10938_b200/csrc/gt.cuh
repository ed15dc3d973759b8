// Exact kNN ground truth on the GPU (gt.cu; metrics.cpp:8-33 semantics).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace detlsh_b200 {

// X [n][d], Q [nq][d] fp32 device; outputs ids/dists [nq][k] device.
// thr_hint (optional, host or device): per query an upper bound on the k-th
// smallest dist^2 (at least k points lie within it).
void brute_force_knn_gpu(const float* X, uint64_t n, int d, const float* Q, uint64_t nq, int k,
                         const double* thr_hint, uint32_t* ids, double* dists, int device, cudaStream_t s);

}  // namespace detlsh_b200
