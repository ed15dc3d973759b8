// Vector file ingestion (io.hpp: read_vectors, vec_element_from_path) into
// caller-owned device memory; see vecio.cu.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace detlsh_b200 {

constexpr int kVecF32 = 0, kVecU8 = 1, kVecI32 = 2;  // .fvecs / .bvecs / .ivecs

int vec_kind_from_path(const char* path);
// n records of dimension d (validates every record header and the tail).
void vectors_shape(const char* path, int kind, uint64_t* n, int* d);
// Fills out [n][d] fp32 (device) from the file, widening u8 / i32 on the GPU.
void read_vectors_into(const char* path, int kind, float* d_out, uint64_t n, int d, cudaStream_t s);

}  // namespace detlsh_b200
