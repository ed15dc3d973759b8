// Scan + stable radix sort (see primitives.cuh).
#include "primitives.cuh"

#include <algorithm>

namespace detlsh_b200 {

namespace {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;  // 2048

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
    }
    return v;
}

// Block-wide exclusive scan of one value per thread; returns the block total.
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t& excl) {
    __shared__ uint32_t warp_tot[32];
    __shared__ uint32_t total_s;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nwarps = (blockDim.x + 31) >> 5;
    const uint32_t inc = warp_incl_scan(v);
    if (lane == 31) warp_tot[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        uint32_t t = lane < nwarps ? warp_tot[lane] : 0;
        const uint32_t ti = warp_incl_scan(t);
        if (lane < nwarps) warp_tot[lane] = ti - t;
        if (lane == nwarps - 1) total_s = ti;
    }
    __syncthreads();
    excl = warp_tot[warp] + inc - v;
    const uint32_t total = total_s;
    __syncthreads();
    return total;
}

__global__ void scan_reduce_kernel(const uint32_t* __restrict__ in, size_t n,
                                   uint32_t* __restrict__ block_sums) {
    const size_t base = static_cast<size_t>(blockIdx.x) * kScanTile;
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        const size_t idx = base + static_cast<size_t>(i) * kScanThreads + threadIdx.x;
        if (idx < n) s += in[idx];
    }
    uint32_t ex;
    const uint32_t tot = block_excl_scan(s, ex);
    if (threadIdx.x == 0) block_sums[blockIdx.x] = tot;
}

__global__ void scan_down_kernel(const uint32_t* in, uint32_t* out, size_t n,
                                 const uint32_t* __restrict__ block_offsets) {
    const size_t base = static_cast<size_t>(blockIdx.x) * kScanTile;
    uint32_t v[kScanItems];
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        const size_t idx = base + static_cast<size_t>(threadIdx.x) * kScanItems + i;
        v[i] = idx < n ? in[idx] : 0;
        s += v[i];
    }
    uint32_t ex;
    block_excl_scan(s, ex);
    uint32_t run = block_offsets[blockIdx.x] + ex;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        const size_t idx = base + static_cast<size_t>(threadIdx.x) * kScanItems + i;
        if (idx < n) out[idx] = run;
        run += v[i];
    }
}

// Single-block scan for small arrays (n <= 1024*kScanItems...), writes total.
__global__ void scan_single_kernel(const uint32_t* in, uint32_t* out, size_t n, uint32_t* total) {
    // processes n in chunks of blockDim*kScanItems sequentially
    __shared__ uint32_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const size_t chunk = static_cast<size_t>(blockDim.x) * kScanItems;
    for (size_t base = 0; base < n; base += chunk) {
        uint32_t v[kScanItems];
        uint32_t s = 0;
#pragma unroll
        for (int i = 0; i < kScanItems; ++i) {
            const size_t idx = base + static_cast<size_t>(threadIdx.x) * kScanItems + i;
            v[i] = idx < n ? in[idx] : 0;
            s += v[i];
        }
        uint32_t ex;
        const uint32_t tot = block_excl_scan(s, ex);
        uint32_t run = carry + ex;
#pragma unroll
        for (int i = 0; i < kScanItems; ++i) {
            const size_t idx = base + static_cast<size_t>(threadIdx.x) * kScanItems + i;
            if (idx < n) out[idx] = run;
            run += v[i];
        }
        __syncthreads();
        if (threadIdx.x == 0) carry += tot;
        __syncthreads();
    }
    if (threadIdx.x == 0 && total) *total = carry;
}

}  // namespace

size_t scan_temp_elems(size_t n) {
    size_t blocks = (n + kScanTile - 1) / kScanTile;
    return 2 * blocks + 64;
}

void exclusive_scan_u32(const uint32_t* in, uint32_t* out, size_t n, uint32_t* tmp,
                        uint32_t* d_total, cudaStream_t s) {
    if (n == 0) {
        if (d_total) DETLSH_CUDA(cudaMemsetAsync(d_total, 0, sizeof(uint32_t), s));
        return;
    }
    const size_t blocks = (n + kScanTile - 1) / kScanTile;
    if (blocks == 1) {
        scan_single_kernel<<<1, 1024, 0, s>>>(in, out, n, d_total);
        DETLSH_LAUNCH_CHECK();
        return;
    }
    uint32_t* sums = tmp;
    uint32_t* offs = tmp + blocks;
    scan_reduce_kernel<<<static_cast<unsigned>(blocks), kScanThreads, 0, s>>>(in, n, sums);
    DETLSH_LAUNCH_CHECK();
    scan_single_kernel<<<1, 1024, 0, s>>>(sums, offs, blocks, d_total);
    DETLSH_LAUNCH_CHECK();
    scan_down_kernel<<<static_cast<unsigned>(blocks), kScanThreads, 0, s>>>(in, out, n, offs);
    DETLSH_LAUNCH_CHECK();
}

// ---------------------------------------------------------------------------
// Radix sort: 8-bit digits, tiles of 4096 pairs; upsweep histogram per tile
// (digit-major so one global scan yields every (digit, tile) offset), stable
// downsweep ranking with warp match + per-warp digit counts.
// ---------------------------------------------------------------------------
namespace {

constexpr int kRadixThreads = 256;
constexpr int kRadixMaxRounds = 16;

// Rounds of 256 keys per tile: enough tiles to give every SM several CTAs
// (small sorts such as the node-id sort would otherwise run a handful of
// CTAs through 16 serial rounds each), at most 16 (tiles of 4096).
int radix_rounds(size_t n) {
    const size_t want_tiles = 148 * 4;
    size_t r = (n + 256 * want_tiles - 1) / (256 * want_tiles);
    return static_cast<int>(std::max<size_t>(1, std::min<size_t>(kRadixMaxRounds, r)));
}

template <typename KeyT>
__global__ void radix_upsweep(const KeyT* __restrict__ keys, size_t n, int shift,
                              uint32_t* __restrict__ hist, uint32_t num_tiles, int rounds, const uint32_t* d_n) {
    __shared__ uint32_t h[256];
    if (d_n && *d_n < n) n = *d_n;
    h[threadIdx.x] = 0;
    __syncthreads();
    const size_t base = static_cast<size_t>(blockIdx.x) * kRadixThreads * rounds;
#pragma unroll 4
    for (int r = 0; r < rounds; ++r) {
        const size_t idx = base + static_cast<size_t>(r) * kRadixThreads + threadIdx.x;
        if (idx < n) atomicAdd(&h[(keys[idx] >> shift) & 0xff], 1u);
    }
    __syncthreads();
    hist[static_cast<size_t>(threadIdx.x) * num_tiles + blockIdx.x] = h[threadIdx.x];
}

// Stable downsweep: each 256-key round is ranked (warp match + per-warp digit
// counts) into a shared-memory copy of the tile ordered by digit; the tile is
// then written out in that order, so consecutive threads store consecutive
// positions of a digit's run (coalesced) instead of one scattered key each.
template <typename KeyT>
__global__ void radix_downsweep(const KeyT* __restrict__ kin, const uint32_t* __restrict__ vin,
                                KeyT* __restrict__ kout, uint32_t* __restrict__ vout, size_t n,
                                int shift, const uint32_t* __restrict__ offsets,
                                const uint32_t* __restrict__ hist, uint32_t num_tiles, int rounds,
                                const uint32_t* d_n) {
    extern __shared__ __align__(16) uint8_t radix_smem[];
    if (d_n && *d_n < n) n = *d_n;
    KeyT* sk = reinterpret_cast<KeyT*>(radix_smem);
    uint32_t* sv = reinterpret_cast<uint32_t*>(sk + static_cast<size_t>(rounds) * kRadixThreads);
    __shared__ uint32_t wh[kRadixThreads / 32][256];
    __shared__ uint32_t gbase[256];
    __shared__ uint32_t toff[256];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    {
        uint32_t ex;
        block_excl_scan(hist[static_cast<size_t>(tid) * num_tiles + blockIdx.x], ex);
        toff[tid] = ex;  // this digit's first slot in the tile
    }
    gbase[tid] = offsets[static_cast<size_t>(tid) * num_tiles + blockIdx.x];
    uint32_t running = 0;  // keys of digit `tid` in the earlier rounds
    const size_t base = static_cast<size_t>(blockIdx.x) * kRadixThreads * rounds;
    if (base >= n) return;  // (a tile past a device-side count; uniform)
    const size_t tile_cap = static_cast<size_t>(kRadixThreads) * rounds;
    const uint32_t tile_n = static_cast<uint32_t>(n - base < tile_cap ? n - base : tile_cap);
    const uint32_t lt_mask = (1u << lane) - 1u;
    for (int r = 0; r < rounds; ++r) {
        const size_t idx = base + static_cast<size_t>(r) * kRadixThreads + tid;
        if (base + static_cast<size_t>(r) * kRadixThreads >= n) break;  // uniform
#pragma unroll
        for (int w = 0; w < kRadixThreads / 32; ++w) wh[w][tid] = 0;
        const bool valid = idx < n;
        KeyT key{};
        uint32_t val = 0;
        uint32_t d = 256;
        if (valid) {
            key = kin[idx];
            val = vin[idx];
            d = static_cast<uint32_t>((key >> shift) & 0xff);
        }
        __syncthreads();
        const uint32_t peers = __match_any_sync(0xffffffffu, d);
        const uint32_t rank = __popc(peers & lt_mask);
        if (valid && rank == 0) wh[warp][d] = __popc(peers);
        __syncthreads();
        {
            uint32_t run = toff[tid] + running;
#pragma unroll
            for (int w = 0; w < kRadixThreads / 32; ++w) {
                const uint32_t c = wh[w][tid];
                wh[w][tid] = run;
                run += c;
            }
            running = run - toff[tid];
        }
        __syncthreads();
        if (valid) {
            const uint32_t at = wh[warp][d] + rank;
            sk[at] = key;
            sv[at] = val;
        }
        __syncthreads();  // wh is reset by the next round
    }
    __syncthreads();
    for (uint32_t i = tid; i < tile_n; i += kRadixThreads) {
        const KeyT key = sk[i];
        const uint32_t d = static_cast<uint32_t>((key >> shift) & 0xff);
        const size_t pos = static_cast<size_t>(gbase[d]) + (i - toff[d]);
        kout[pos] = key;
        vout[pos] = sv[i];
    }
}

}  // namespace

size_t radix_temp_elems(size_t n) {
    const size_t tile = static_cast<size_t>(kRadixThreads) * radix_rounds(n);
    const size_t tiles = (n + tile - 1) / tile;
    return 256 * tiles * 2 + scan_temp_elems(256 * tiles) + 8;
}

template <typename KeyT>
bool radix_sort_pairs(KeyT* k0, uint32_t* v0, KeyT* k1, uint32_t* v1, size_t n, int begin_bit,
                      int end_bit, uint32_t* tmp, cudaStream_t s, const uint32_t* d_n) {
    if (n <= 1) return false;
    const int rounds = radix_rounds(n);
    const size_t tile = static_cast<size_t>(kRadixThreads) * rounds;
    const uint32_t tiles = static_cast<uint32_t>((n + tile - 1) / tile);
    uint32_t* hist = tmp;
    uint32_t* offs = tmp + 256 * static_cast<size_t>(tiles);
    uint32_t* stmp = offs + 256 * static_cast<size_t>(tiles);
    const size_t smem = tile * (sizeof(KeyT) + sizeof(uint32_t));  // the tile, digit-ordered
    // (per device: set on every call, a host-side attribute write)
    DETLSH_CUDA(cudaFuncSetAttribute(radix_downsweep<KeyT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(kRadixThreads * kRadixMaxRounds * (sizeof(KeyT) + 4))));
    bool flipped = false;
    for (int bit = begin_bit; bit < end_bit; bit += 8) {
        KeyT* ki = flipped ? k1 : k0;
        uint32_t* vi = flipped ? v1 : v0;
        KeyT* ko = flipped ? k0 : k1;
        uint32_t* vo = flipped ? v0 : v1;
        radix_upsweep<KeyT><<<tiles, kRadixThreads, 0, s>>>(ki, n, bit, hist, tiles, rounds, d_n);
        DETLSH_LAUNCH_CHECK();
        exclusive_scan_u32(hist, offs, 256 * static_cast<size_t>(tiles), stmp, nullptr, s);
        radix_downsweep<KeyT><<<tiles, kRadixThreads, smem, s>>>(ki, vi, ko, vo, n, bit, offs, hist, tiles, rounds, d_n);
        DETLSH_LAUNCH_CHECK();
        flipped = !flipped;
    }
    return flipped;
}

template bool radix_sort_pairs<uint32_t>(uint32_t*, uint32_t*, uint32_t*, uint32_t*, size_t, int,
                                         int, uint32_t*, cudaStream_t, const uint32_t*);
template bool radix_sort_pairs<uint64_t>(uint64_t*, uint32_t*, uint64_t*, uint32_t*, size_t, int,
                                         int, uint32_t*, cudaStream_t, const uint32_t*);

}  // namespace detlsh_b200
