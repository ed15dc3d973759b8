// Point-sharded index in one process (sharded.cu): shard s holds rows
// [offsets[s], offsets[s+1]) on devices[s]; queries merge on devices[0].
#pragma once

#include <cuda_runtime.h>

#include <memory>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "index.cuh"

namespace detlsh_b200 {

struct ShardedIndex {
    std::vector<std::unique_ptr<GpuIndex>> shards;
    std::vector<uint64_t> offsets;  // [S + 1]
    std::vector<int> devices;       // [S]
    int merge_device = 0;
    struct ShardQuery {  // per-shard query staging on the shard's device (stream first)
        OwnedStream stream;
        DevBuf<float> q;          // the batch, when the shard is not on the merge device
        DevBuf<uint32_t> ids;     // shard-local top-k positions
        DevBuf<uint64_t> ids64;   // the same as global positions
        DevBuf<double> dists;
        DevBuf<int32_t> hits;
        cudaEvent_t done = nullptr;
    };
    std::vector<std::unique_ptr<ShardQuery>> q;
    OwnedStream main;  // merge device
    DevBuf<float> q_stage;
    DevBuf<double> g_dists;  // [S][nq][k] gathered lists
    DevBuf<uint64_t> g_ids;
    DevBuf<int32_t> g_hits;
    DevBuf<double> o_dists;  // merged (host-pointer calls)
    DevBuf<uint64_t> o_ids;
    DevBuf<int32_t> o_hits;
    cudaEvent_t inputs_ready = nullptr;
    cudaEvent_t merge_done = nullptr;
    bool merged_once = false;
    std::mutex mu;
    ShardedIndex() = default;
    ShardedIndex(const ShardedIndex&) = delete;
    ShardedIndex& operator=(const ShardedIndex&) = delete;
    ~ShardedIndex();
};

std::unique_ptr<ShardedIndex> sharded_build(const float* points, uint64_t n, int d, detlsh_params* params,
                                            uint64_t seed, const int32_t* devices, int shards,
                                            uint32_t flags);

// ck_ann over every shard + merge by (distance, global position).  ids are
// global u64 positions.  Device pointers (on the merge device): stream-ordered.
void sharded_query(ShardedIndex& X, const float* queries, uint64_t nq, int k, uint32_t flags, uint64_t* ids,
                   double* dists, int32_t* n_hits, cudaStream_t user_stream);

}  // namespace detlsh_b200
