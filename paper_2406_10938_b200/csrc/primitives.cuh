// Device-wide primitives written for this library: exclusive scan and a
// stable LSD radix sort of (key, u32 value) pairs.  They back the DE-Tree
// build (root-slot sort, node-id assignment) — the "radix sort on interleaved
// codes" the north star asks for.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"

namespace detlsh_b200 {

// Exclusive prefix sum of n u32 values (in may alias out).  Returns the total.
// `tmp` must hold scan_temp_elems(n) u32.
size_t scan_temp_elems(size_t n);
void exclusive_scan_u32(const uint32_t* in, uint32_t* out, size_t n, uint32_t* tmp,
                        uint32_t* d_total, cudaStream_t s);

// Stable LSD radix sort on bits [begin_bit, end_bit) of the keys.  Pairs are
// ping-ponged between (k0,v0) and (k1,v1); returns true if the result ended in
// (k1,v1).  `tmp` must hold radix_temp_elems(n) u32.
size_t radix_temp_elems(size_t n);
// d_n (optional): the pair count on the device (<= n, the capacity the tiles
// are laid out for), so a count produced by an earlier kernel needs no host read.
template <typename KeyT>
bool radix_sort_pairs(KeyT* k0, uint32_t* v0, KeyT* k1, uint32_t* v1, size_t n, int begin_bit,
                      int end_bit, uint32_t* tmp, cudaStream_t s, const uint32_t* d_n = nullptr);

}  // namespace detlsh_b200
