// DE-Tree build on the GPU (tree.cu) and its flattened device layout.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "common.cuh"

namespace detlsh_b200 {

constexpr int kBoxStride = 32;  // padded dims per leaf box row (K <= 24)

// One DE-Tree, flattened.  Node ids follow the reference's build order
// (de_tree.cpp:49-131: a node's index is its creation time), so every
// (mindist, node index) tie-break of range_query_optimized matches.
struct DevTree {
    int space = 0, K = 0, n_regions = 0, sbits = 0, max_size = 0;
    uint64_t n = 0;
    uint64_t num_nodes = 0, num_leaves = 0;
    DevBuf<int32_t> root_children;  // [2^K]
    DevBuf<uint8_t> is_leaf, split_dim;
    DevBuf<int32_t> left, right;
    DevBuf<uint8_t> bits, value;  // [num_nodes][K]
    DevBuf<uint32_t> node_begin, node_count;  // into perm (leaves; 0 count for internal)
    DevBuf<uint32_t> perm;  // positions in leaf order; each leaf contiguous, ascending
    // query-side leaf arrays, leaves in node-id order
    DevBuf<uint32_t> leaf_node, leaf_begin, leaf_count;
    DevBuf<uint8_t> leaf_box;  // [num_leaves][kBoxStride][2] (lo region, hi region)
    // [num_leaves] {code | refined << 16, count} (K <= 16): bit j of code = the
    // half (top region bit) dim j's box lies in; bit j of refined = the box is
    // narrower than that half.  0xffffffff: no half form (the root leaf, or
    // K > 16) -- the scan then takes the general per-dimension path.
    DevBuf<uint2> leaf_cr;
    uint32_t max_leaf_count = 0;
    double build_ms = 0.0;
};

// build_tree (de_tree.cpp:133-152) from device codes of one space ([n][K] u8).
void build_tree_gpu(const uint8_t* d_codes_space, uint64_t n, int K, int n_regions, int space,
                    int max_size, DevTree& out, cudaStream_t s);

// Host export in the reference layout (nodes in build order).
struct HostTreeExport {
    std::vector<int32_t> root_children;
    std::vector<uint8_t> is_leaf, split_dim;
    std::vector<int32_t> left, right;
    std::vector<uint8_t> bits, value;
    std::vector<uint64_t> ebegin;
    std::vector<uint32_t> ecount;
    std::vector<uint32_t> positions;
};
void export_tree(const DevTree& t, HostTreeExport& out);

}  // namespace detlsh_b200
