// Seeded synthetic datasets generated on the device (bench / test utility).
// BASELINE.json config 5 (n = 1e8, d = 128, ~51 GB fp32) is too large to
// build on the host with numpy in a bench run, so its stand-in is generated
// here, straight into HBM, from a counter-based hash (element (r, t) depends on
// (seed, r * d + t) only, so any row range can be produced independently and
// shards match the full dataset byte for byte):
//
//   kind 0 "sparse geometric" (configs 2 / 5): 0 with probability 1/2, else
//   min(255, G) with G ~ geometric(p = 0.05) on {1, 2, ...}, as fp32.
#include <algorithm>
#include <cmath>

#include "../../include/detlsh_b200.h"
#include "common.cuh"

namespace detlsh_b200 {

namespace {

__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
    z += 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

__global__ void synth_sparse_geometric_kernel(uint64_t seed, uint64_t e0, uint64_t total, double inv_log_q,
                                              float* __restrict__ out) {
    const uint64_t key = splitmix64(seed);
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t h = splitmix64(key ^ splitmix64(e0 + i));
        float v = 0.0f;
        if (h >> 63) {  // non-zero with probability 1/2
            // u in (0, 1] from 53 bits; inverse CDF of the geometric law on {1, 2, ...}
            const double u = (static_cast<double>((h << 1) >> 11) + 1.0) * 0x1p-53;
            const double g = floor(log(u) * inv_log_q) + 1.0;
            v = static_cast<float>(g < 255.0 ? g : 255.0);
        }
        out[i] = v;
    }
}

}  // namespace

void synth_generate(int kind, uint64_t seed, uint64_t row0, uint64_t n, int d, float* out, cudaStream_t s) {
    if (kind != 0) throw InvalidArgument("synth: unknown dataset kind");
    if (d < 1) throw InvalidArgument("synth: d must be positive");
    const uint64_t total = n * static_cast<uint64_t>(d);
    if (total == 0) return;
    int dev = 0;
    cudaGetDevice(&dev);
    const unsigned grid = static_cast<unsigned>(
        std::min<uint64_t>((total + 255) / 256, static_cast<uint64_t>(sm_count(dev)) * 16));
    synth_sparse_geometric_kernel<<<grid, 256, 0, s>>>(seed, row0 * static_cast<uint64_t>(d), total,
                                                       1.0 / std::log(1.0 - 0.05), out);
    DETLSH_LAUNCH_CHECK();
}

}  // namespace detlsh_b200
