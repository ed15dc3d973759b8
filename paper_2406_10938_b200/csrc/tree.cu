// DE-Tree construction on the GPU.
//
// The reference inserts points one at a time (de_tree.cpp:49-75) and splits a
// full leaf before inserting into it, on the dimension whose next bit best
// balances the leaf's CURRENT entries (de_tree.cpp:77-131).  Those entries are
// exactly the first `max_size` members, in position order, of the node's
// prefix region, so the same tree is produced top-down:
//
//   node N splits  <=>  |S(N)| > max_size and some dimension is unsaturated;
//   split dim       =  argmin |zeros - ones| over the first max_size of S(N)
//                      (ties to the lowest dim);
//   children        =  STABLE partition of S(N) by that bit (left = 0).
//
// and every node's reference index is its creation time: a root is created
// when its first member arrives (z_first), children when the parent's
// (max_size+1)-th member arrives (z_split), cascades ordered by depth, left
// before right.  Sorting nodes by (z, depth, side) reproduces the indices.
//
// GPU form: root-slot keys -> stable radix sort -> level-synchronous segmented
// splitting (one CTA per splitting node) -> node-id radix sort -> flatten.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <optional>

#include "primitives.cuh"
#include "tree.cuh"

namespace detlsh_b200 {

namespace {

constexpr uint32_t kDepthShift = 9;  // key = z << 9 | depth << 1 | side

struct BuildNodes {
    DevBuf<uint64_t> key;
    DevBuf<uint32_t> begin, count;
    DevBuf<uint8_t> depth;
    DevBuf<int8_t> split;  // -1 leaf, -2 invalid (unused child slot), >=0 split dim
    DevBuf<int32_t> left, right;
    DevBuf<uint8_t> bits, value;  // [cap][K]
    size_t cap = 0;

    void grow(size_t want, size_t keep, int K, cudaStream_t s) {
        if (want <= cap) return;
        size_t nc = std::max<size_t>(want, cap * 2);
        key.grow(nc, keep, s);
        begin.grow(nc, keep, s);
        count.grow(nc, keep, s);
        depth.grow(nc, keep, s);
        split.grow(nc, keep, s);
        left.grow(nc, keep, s);
        right.grow(nc, keep, s);
        bits.grow(nc * K, keep * K, s);
        value.grow(nc * K, keep * K, s);
        cap = nc;
    }
};

__global__ void slot_key_kernel(const uint8_t* __restrict__ codes, uint64_t n, int K, int sbits,
                                uint32_t* __restrict__ keys, uint32_t* __restrict__ vals) {
    for (uint64_t z = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; z < n;
         z += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint8_t* c = codes + z * K;
        uint32_t slot = 0;
        for (int j = 0; j < K; ++j) slot |= static_cast<uint32_t>((c[j] >> (sbits - 1)) & 1) << j;
        keys[z] = slot;
        vals[z] = static_cast<uint32_t>(z);
    }
}

__global__ void head_flag_kernel(const uint32_t* __restrict__ keys, uint64_t n,
                                 uint32_t* __restrict__ flags) {
    for (uint64_t z = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; z < n;
         z += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        flags[z] = (z == 0 || keys[z] != keys[z - 1]) ? 1u : 0u;
}

__global__ void root_init_kernel(const uint32_t* __restrict__ keys, const uint32_t* __restrict__ perm,
                                 const uint32_t* __restrict__ flags, const uint32_t* __restrict__ ridx,
                                 uint64_t n, int K, uint64_t* nkey, uint32_t* nbegin, uint8_t* ndepth,
                                 int8_t* nsplit, uint8_t* nbits, uint8_t* nvalue,
                                 uint32_t* rslot) {
    for (uint64_t z = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; z < n;
         z += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        if (!flags[z]) continue;
        const uint32_t r = ridx[z];
        const uint32_t slot = keys[z];
        nbegin[r] = static_cast<uint32_t>(z);
        rslot[r] = slot;
        nkey[r] = static_cast<uint64_t>(perm[z]) << kDepthShift;
        ndepth[r] = 0;
        nsplit[r] = -1;
        for (int j = 0; j < K; ++j) {
            nbits[static_cast<size_t>(r) * K + j] = 1;
            nvalue[static_cast<size_t>(r) * K + j] = static_cast<uint8_t>((slot >> j) & 1);
        }
    }
}

__global__ void root_count_kernel(const uint32_t* __restrict__ nbegin, uint32_t R, uint64_t n,
                                  uint32_t* __restrict__ ncount, uint32_t cap,
                                  uint32_t* __restrict__ act, uint32_t* __restrict__ act_n) {
    for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < R; r += gridDim.x * blockDim.x) {
        const uint32_t end = r + 1 < R ? nbegin[r + 1] : static_cast<uint32_t>(n);
        const uint32_t c = end - nbegin[r];
        ncount[r] = c;
        if (c > cap) act[atomicAdd(act_n, 1u)] = r;
    }
}

// One CTA per splitting node (de_tree.cpp:77-131 restated top-down).
constexpr int kLevelThreads = 256;

__global__ void __launch_bounds__(kLevelThreads) level_split_kernel(
    const uint8_t* __restrict__ codes, int K, int sbits, uint32_t cap,
    const uint32_t* __restrict__ act, uint32_t base_bn, uint32_t* __restrict__ perm,
    uint32_t* __restrict__ tmp, uint64_t* nkey, uint32_t* nbegin, uint32_t* ncount,
    uint8_t* ndepth, int8_t* nsplit, int32_t* nleft, int32_t* nright, uint8_t* nbits,
    uint8_t* nvalue, uint32_t* __restrict__ next_act, uint32_t* __restrict__ next_n,
    uint32_t* __restrict__ invalid_n) {
    __shared__ int used[kMaxK];
    __shared__ uint32_t ones[kMaxK];
    __shared__ int best_s;
    __shared__ uint32_t wsum[kLevelThreads / 32];
    __shared__ uint32_t n1_s;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t bn = act[blockIdx.x];
    const uint32_t begin = nbegin[bn], cnt = ncount[bn];
    if (tid < K) {
        used[tid] = nbits[static_cast<size_t>(bn) * K + tid];
        ones[tid] = 0;
    }
    if (tid == 0) n1_s = 0;
    __syncthreads();
    // popcount of the next bit per unsaturated dim over the first `cap` entries
    uint32_t loc[kMaxK];
#pragma unroll
    for (int j = 0; j < kMaxK; ++j) loc[j] = 0;
    for (uint32_t e = tid; e < cap; e += kLevelThreads) {
        const uint8_t* c = codes + static_cast<size_t>(perm[begin + e]) * K;
#pragma unroll
        for (int j = 0; j < kMaxK; ++j)
            if (j < K && used[j] < sbits) loc[j] += (c[j] >> (sbits - 1 - used[j])) & 1;
    }
#pragma unroll
    for (int j = 0; j < kMaxK; ++j) {
        if (j >= K) break;
        uint32_t v = loc[j];
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0 && v) atomicAdd(&ones[j], v);
    }
    __syncthreads();
    if (tid == 0) {
        int best = -1;
        uint32_t best_imb = 0;
        for (int j = 0; j < K; ++j) {
            if (used[j] >= sbits) continue;
            const uint32_t o = ones[j], z = cap - o;
            const uint32_t imb = z > o ? z - o : o - z;
            if (best < 0 || imb < best_imb) {
                best = j;
                best_imb = imb;
            }
        }
        best_s = best;
    }
    __syncthreads();
    const int best = best_s;
    const uint32_t c0 = base_bn + 2 * blockIdx.x, c1 = c0 + 1;
    if (best < 0) {  // every dimension at full depth: the leaf overflows
        if (tid == 0) {
            nsplit[c0] = nsplit[c1] = -2;
            nkey[c0] = nkey[c1] = ~0ULL;
            atomicAdd(invalid_n, 2u);
        }
        return;
    }
    const int shift = sbits - 1 - used[best];
    const uint32_t z_split = perm[begin + cap];  // the (max_size+1)-th member
    // pass 1: ones count
    uint32_t my1 = 0;
    for (uint32_t e = tid; e < cnt; e += kLevelThreads)
        my1 += (codes[static_cast<size_t>(perm[begin + e]) * K + best] >> shift) & 1;
    for (int o = 16; o; o >>= 1) my1 += __shfl_xor_sync(0xffffffffu, my1, o);
    if (lane == 0) atomicAdd(&n1_s, my1);
    __syncthreads();
    const uint32_t n1 = n1_s, n0 = cnt - n1;
    // pass 2: stable scatter into tmp, chunk by chunk
    uint32_t run0 = 0, run1 = 0;
    for (uint32_t base = 0; base < cnt; base += kLevelThreads) {
        const uint32_t e = base + tid;
        uint32_t pos = 0, b = 0;
        if (e < cnt) {
            pos = perm[begin + e];
            b = (codes[static_cast<size_t>(pos) * K + best] >> shift) & 1;
        }
        const uint32_t bal = __ballot_sync(0xffffffffu, b);
        const uint32_t in_warp_ones = __popc(bal & ((1u << lane) - 1u));
        if (lane == 0) wsum[warp] = __popc(bal);
        __syncthreads();
        uint32_t ones_before = in_warp_ones, chunk_ones = 0;
#pragma unroll
        for (int w = 0; w < kLevelThreads / 32; ++w) {
            if (w < warp) ones_before += wsum[w];
            chunk_ones += wsum[w];
        }
        const uint32_t chunk_n = min(static_cast<uint32_t>(kLevelThreads), cnt - base);
        if (e < cnt) {
            const uint32_t zeros_before = tid - ones_before;
            const uint32_t dst = b ? (n0 + run1 + ones_before) : (run0 + zeros_before);
            tmp[begin + dst] = pos;
        }
        run1 += chunk_ones;
        run0 += chunk_n - chunk_ones;
        __syncthreads();
    }
    for (uint32_t e = tid; e < cnt; e += kLevelThreads) perm[begin + e] = tmp[begin + e];
    // children records
    const uint8_t dep = static_cast<uint8_t>(ndepth[bn] + 1);
    if (tid < K) {
        const uint8_t bv = nbits[static_cast<size_t>(bn) * K + tid];
        const uint8_t vv = nvalue[static_cast<size_t>(bn) * K + tid];
        const bool at = tid == best;
        nbits[static_cast<size_t>(c0) * K + tid] = at ? bv + 1 : bv;
        nbits[static_cast<size_t>(c1) * K + tid] = at ? bv + 1 : bv;
        nvalue[static_cast<size_t>(c0) * K + tid] = at ? static_cast<uint8_t>(vv << 1) : vv;
        nvalue[static_cast<size_t>(c1) * K + tid] = at ? static_cast<uint8_t>((vv << 1) | 1) : vv;
    }
    if (tid == 0) {
        const uint64_t kb = (static_cast<uint64_t>(z_split) << kDepthShift) | (static_cast<uint64_t>(dep) << 1);
        nkey[c0] = kb;
        nkey[c1] = kb | 1;
        nbegin[c0] = begin;
        ncount[c0] = n0;
        nbegin[c1] = begin + n0;
        ncount[c1] = n1;
        ndepth[c0] = ndepth[c1] = dep;
        nsplit[c0] = nsplit[c1] = -1;
        nleft[c0] = nright[c0] = nleft[c1] = nright[c1] = -1;
        nsplit[bn] = static_cast<int8_t>(best);
        nleft[bn] = static_cast<int32_t>(c0);
        nright[bn] = static_cast<int32_t>(c1);
        if (n0 > cap) next_act[atomicAdd(next_n, 1u)] = c0;
        if (n1 > cap) next_act[atomicAdd(next_n, 1u)] = c1;
    }
}

__global__ void iota_kernel(uint32_t* v, uint64_t n) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        v[i] = static_cast<uint32_t>(i);
}

__global__ void clamp_invalid_keys(uint64_t* key, uint64_t total, uint64_t invalid_key) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        if (key[i] == ~0ULL) key[i] = invalid_key;
}

__global__ void scatter_ids(const uint32_t* __restrict__ sorted_bn, uint64_t valid,
                            uint32_t* __restrict__ id_of_bn) {
    for (uint64_t r = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; r < valid;
         r += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        id_of_bn[sorted_bn[r]] = static_cast<uint32_t>(r);
}

__global__ void finalize_nodes(const uint32_t* __restrict__ sorted_bn, uint64_t valid, int K,
                               const uint32_t* __restrict__ id_of_bn, const uint32_t* nbegin,
                               const uint32_t* ncount, const int8_t* nsplit, const int32_t* nleft,
                               const int32_t* nright, const uint8_t* nbits, const uint8_t* nvalue,
                               uint8_t* is_leaf, uint8_t* split_dim, int32_t* left, int32_t* right,
                               uint8_t* bits, uint8_t* value, uint32_t* node_begin,
                               uint32_t* node_count, uint32_t* leaf_flag) {
    for (uint64_t id = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; id < valid;
         id += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint32_t bn = sorted_bn[id];
        const int8_t sp = nsplit[bn];
        const bool leaf = sp < 0;
        is_leaf[id] = leaf ? 1 : 0;
        split_dim[id] = leaf ? 0 : static_cast<uint8_t>(sp);
        left[id] = leaf ? -1 : static_cast<int32_t>(id_of_bn[nleft[bn]]);
        right[id] = leaf ? -1 : static_cast<int32_t>(id_of_bn[nright[bn]]);
        for (int j = 0; j < K; ++j) {
            bits[id * K + j] = nbits[static_cast<size_t>(bn) * K + j];
            value[id * K + j] = nvalue[static_cast<size_t>(bn) * K + j];
        }
        node_begin[id] = nbegin[bn];
        node_count[id] = leaf ? ncount[bn] : 0;
        leaf_flag[id] = leaf ? 1u : 0u;
    }
}

__global__ void root_children_kernel(const uint32_t* __restrict__ rslot, uint32_t R,
                                     const uint32_t* __restrict__ id_of_bn, int32_t* rc) {
    for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < R; r += gridDim.x * blockDim.x)
        rc[rslot[r]] = static_cast<int32_t>(id_of_bn[r]);
}

__global__ void leaves_kernel(uint64_t num_nodes, int K, int sbits,
                              const uint32_t* __restrict__ leaf_flag,
                              const uint32_t* __restrict__ leaf_idx, const uint8_t* __restrict__ bits,
                              const uint8_t* __restrict__ value, const uint32_t* __restrict__ node_begin,
                              const uint32_t* __restrict__ node_count, uint32_t* leaf_node,
                              uint32_t* leaf_begin, uint32_t* leaf_count, uint8_t* leaf_box,
                              uint2* leaf_cr, uint32_t* max_count) {
    for (uint64_t id = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; id < num_nodes;
         id += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        if (!leaf_flag[id]) continue;
        const uint32_t li = leaf_idx[id];
        leaf_node[li] = static_cast<uint32_t>(id);
        leaf_begin[li] = node_begin[id];
        leaf_count[li] = node_count[id];
        atomicMax(max_count, node_count[id]);
        uint8_t* box = leaf_box + static_cast<size_t>(li) * kBoxStride * 2;
        uint32_t code = 0, refined = 0;
        bool half_form = K <= 16;
        for (int j = 0; j < K; ++j) {
            const int b = bits[id * K + j], v = value[id * K + j];
            if (b == 0) half_form = false;
            else code |= static_cast<uint32_t>((v >> (b - 1)) & 1) << j;
            if (b != 1) refined |= 1u << j;
        }
        leaf_cr[li] = make_uint2(half_form ? (code | refined << 16) : 0xffffffffu, node_count[id]);
        for (int j = 0; j < kBoxStride; ++j) {
            if (j < K) {
                const int b = bits[id * K + j], v = value[id * K + j];
                const int w = sbits - b;
                box[2 * j] = static_cast<uint8_t>(v << w);
                box[2 * j + 1] = static_cast<uint8_t>(((v + 1) << w) - 1);
            } else {
                box[2 * j] = 0;
                box[2 * j + 1] = 0;
            }
        }
    }
}

unsigned grid_for(uint64_t n, int threads = 256) {
    return static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>((n + threads - 1) / threads, 65535)));
}

}  // namespace

// Counter reads through page-locked words: a pageable device-to-host copy is
// staged by the driver, and the trees are built on several threads at once
// next to the breakpoint loop's own transfers.  One process-wide block of
// slots handed out round-robin (the tree threads live for one build, so a
// per-thread buffer would be a cudaMallocHost/cudaFreeHost pair per build,
// and cudaFreeHost synchronises the device).
uint32_t read_word(const uint32_t* d, cudaStream_t s) {
    constexpr uint32_t kSlots = 1024, kStride = 16;  // one 64-B line per slot
    static uint32_t* block = []() {
        uint32_t* p = nullptr;
        DETLSH_CUDA(cudaMallocHost(&p, kSlots * kStride * sizeof(uint32_t)));
        return p;  // process lifetime
    }();
    static std::atomic<uint32_t> next{0};
    uint32_t* w = block + (next.fetch_add(1, std::memory_order_relaxed) % kSlots) * kStride;
    DETLSH_CUDA(cudaMemcpyAsync(w, d, 4, cudaMemcpyDeviceToHost, s));
    DETLSH_CUDA(cudaStreamSynchronize(s));
    return *w;
}

void build_tree_gpu(const uint8_t* d_codes, uint64_t n, int K, int n_regions, int space,
                    int max_size, DevTree& T, cudaStream_t s) {
    const auto t0 = std::chrono::steady_clock::now();
    StreamScope scope(s);
    if (max_size < 1) throw InvalidArgument("build_tree: max_size must be positive");
    if (K < 1 || K > kMaxK) throw InvalidArgument("build_tree: K must lie in [1, 24]");
    if (n_regions < 2 || (n_regions & (n_regions - 1)) || n_regions > kMaxRegions)
        throw InvalidArgument("build_tree: n_regions must be a power of two >= 2");
    if (n == 0 || n > 0xffffffffULL) throw InvalidArgument("build_tree: n must lie in [1, 2^32)");
    int sbits = 0;
    while ((1 << sbits) < n_regions) ++sbits;
    T.space = space;
    T.K = K;
    T.n_regions = n_regions;
    T.sbits = sbits;
    T.max_size = max_size;
    T.n = n;
    const uint32_t cap = static_cast<uint32_t>(max_size);

    // 1-2. root-slot keys, stable sort -> perm
    DevBuf<uint32_t> k0(n), k1(n), v1(n), flags(n), ridx(n);
    T.perm.alloc(n);
    DevBuf<uint32_t> rtmp(std::max(radix_temp_elems(n), scan_temp_elems(n)));
    // profile scopes cover device work only (the host reads between phases
    // are outside them), so each is a kernel-time figure
    bool flip = false;
    {
        ProfScope ps("tree_sort", s);
        slot_key_kernel<<<grid_for(n), 256, 0, s>>>(d_codes, n, K, sbits, k0.get(), T.perm.get());
        DETLSH_LAUNCH_CHECK();
        flip = radix_sort_pairs<uint32_t>(k0.get(), T.perm.get(), k1.get(), v1.get(), n, 0, ((K + 7) / 8) * 8,
                                          rtmp.get(), s);
        if (flip) DETLSH_CUDA(cudaMemcpyAsync(T.perm.get(), v1.get(), n * 4, cudaMemcpyDeviceToDevice, s));
    }
    uint32_t* skeys = flip ? k1.get() : k0.get();

    // 3-4. root nodes
    DevBuf<uint32_t> counters(4);
    {
        ProfScope ps("tree_roots", s);
        head_flag_kernel<<<grid_for(n), 256, 0, s>>>(skeys, n, flags.get());
        DETLSH_LAUNCH_CHECK();
        DETLSH_CUDA(cudaMemsetAsync(counters.get(), 0, 4 * sizeof(uint32_t), s));
        exclusive_scan_u32(flags.get(), ridx.get(), n, rtmp.get(), counters.get(), s);
    }
    const uint32_t R = read_word(counters.get(), s);

    BuildNodes B;
    B.grow(std::max<size_t>(R + 2 * (n / (cap + 1)) + 64, 1024), 0, K, s);
    DevBuf<uint32_t> rslot(R);
    DevBuf<uint32_t> actA(std::max<size_t>(R, 1)), actB;
    uint32_t* d_act_n = counters.get() + 1;
    uint32_t* d_next_n = counters.get() + 2;
    uint32_t* d_invalid = counters.get() + 3;
    {
        ProfScope ps("tree_roots", s);
        root_init_kernel<<<grid_for(n), 256, 0, s>>>(skeys, T.perm.get(), flags.get(), ridx.get(), n, K,
                                                     B.key.get(), B.begin.get(), B.depth.get(),
                                                     B.split.get(), B.bits.get(), B.value.get(),
                                                     rslot.get());
        DETLSH_LAUNCH_CHECK();
        DETLSH_CUDA(cudaMemsetAsync(counters.get() + 1, 0, 3 * sizeof(uint32_t), s));
        root_count_kernel<<<grid_for(R), 256, 0, s>>>(B.begin.get(), R, n, B.count.get(), cap,
                                                      actA.get(), d_act_n);
        DETLSH_LAUNCH_CHECK();
    }
    uint32_t A = read_word(d_act_n, s);

    // 5. level-synchronous splitting
    uint64_t total = R;
    DevBuf<uint32_t> ptmp(n);
    int levels = 0;
    while (A > 0) {
        B.grow(total + 2 * static_cast<size_t>(A), total, K, s);
        actB.grow(2 * static_cast<size_t>(A), 0, s);
        DETLSH_CUDA(cudaMemsetAsync(d_next_n, 0, 4, s));
        {
            ProfScope ps("tree_level_split", s);
            level_split_kernel<<<A, kLevelThreads, 0, s>>>(
                d_codes, K, sbits, cap, actA.get(), static_cast<uint32_t>(total), T.perm.get(),
                ptmp.get(), B.key.get(), B.begin.get(), B.count.get(), B.depth.get(), B.split.get(),
                B.left.get(), B.right.get(), B.bits.get(), B.value.get(), actB.get(), d_next_n,
                d_invalid);
            DETLSH_LAUNCH_CHECK();
        }
        total += 2 * static_cast<uint64_t>(A);
        A = read_word(d_next_n, s);
        std::swap(actA, actB);
        ++levels;
    }
    const uint32_t invalid = read_word(d_invalid, s);
    const uint64_t valid = total - invalid;

    // 6. node ids = rank of (z, depth, side)
    int zbits = 0;
    while ((1ULL << zbits) < n + 1) ++zbits;
    const int kbits = zbits + static_cast<int>(kDepthShift);
    const uint64_t invalid_key = (kbits >= 64) ? ~0ULL : ((1ULL << kbits) - 1);
    DevBuf<uint64_t> ka(total), kb(total);
    DevBuf<uint32_t> va(total), vb(total), id_of_bn(total);
    DevBuf<uint32_t> stmp(radix_temp_elems(total) + scan_temp_elems(total));
    std::optional<ProfScope> ps_ids;
    ps_ids.emplace("tree_ids", s);
    DETLSH_CUDA(cudaMemcpyAsync(ka.get(), B.key.get(), total * 8, cudaMemcpyDeviceToDevice, s));
    clamp_invalid_keys<<<grid_for(total), 256, 0, s>>>(ka.get(), total, invalid_key);
    DETLSH_LAUNCH_CHECK();
    iota_kernel<<<grid_for(total), 256, 0, s>>>(va.get(), total);
    DETLSH_LAUNCH_CHECK();
    const bool f2 = radix_sort_pairs<uint64_t>(ka.get(), va.get(), kb.get(), vb.get(), total, 0,
                                               ((kbits + 7) / 8) * 8, stmp.get(), s);
    const uint32_t* sorted_bn = f2 ? vb.get() : va.get();
    scatter_ids<<<grid_for(valid), 256, 0, s>>>(sorted_bn, valid, id_of_bn.get());
    DETLSH_LAUNCH_CHECK();

    // 7. flatten in id order
    T.num_nodes = valid;
    T.is_leaf.alloc(valid);
    T.split_dim.alloc(valid);
    T.left.alloc(valid);
    T.right.alloc(valid);
    T.bits.alloc(valid * K);
    T.value.alloc(valid * K);
    T.node_begin.alloc(valid);
    T.node_count.alloc(valid);
    DevBuf<uint32_t> leaf_flag(valid), leaf_idx(valid);
    finalize_nodes<<<grid_for(valid), 256, 0, s>>>(
        sorted_bn, valid, K, id_of_bn.get(), B.begin.get(), B.count.get(), B.split.get(),
        B.left.get(), B.right.get(), B.bits.get(), B.value.get(), T.is_leaf.get(),
        T.split_dim.get(), T.left.get(), T.right.get(), T.bits.get(), T.value.get(),
        T.node_begin.get(), T.node_count.get(), leaf_flag.get());
    DETLSH_LAUNCH_CHECK();
    T.root_children.alloc(static_cast<size_t>(1) << K);
    DETLSH_CUDA(cudaMemsetAsync(T.root_children.get(), 0xff, (static_cast<size_t>(1) << K) * 4, s));
    root_children_kernel<<<grid_for(R), 256, 0, s>>>(rslot.get(), R, id_of_bn.get(),
                                                     T.root_children.get());
    DETLSH_LAUNCH_CHECK();
    DETLSH_CUDA(cudaMemsetAsync(counters.get(), 0, 8, s));
    exclusive_scan_u32(leaf_flag.get(), leaf_idx.get(), valid, stmp.get(), counters.get(), s);
    ps_ids.reset();
    const uint32_t nl = read_word(counters.get(), s);
    T.num_leaves = nl;
    T.leaf_node.alloc(nl);
    T.leaf_begin.alloc(nl);
    T.leaf_count.alloc(nl);
    T.leaf_box.alloc(static_cast<size_t>(nl) * kBoxStride * 2);
    T.leaf_cr.alloc(nl);
    {
        ProfScope ps("tree_leaves", s);
        leaves_kernel<<<grid_for(valid), 256, 0, s>>>(valid, K, sbits, leaf_flag.get(), leaf_idx.get(),
                                                      T.bits.get(), T.value.get(), T.node_begin.get(),
                                                      T.node_count.get(), T.leaf_node.get(),
                                                      T.leaf_begin.get(), T.leaf_count.get(),
                                                      T.leaf_box.get(), T.leaf_cr.get(), counters.get() + 1);
        DETLSH_LAUNCH_CHECK();
    }
    const uint32_t mx = read_word(counters.get() + 1, s);
    T.max_leaf_count = mx;
    T.build_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    (void)levels;
}

void export_tree(const DevTree& t, HostTreeExport& o) {
    const uint64_t nn = t.num_nodes;
    const int K = t.K;
    o.root_children.resize(static_cast<size_t>(1) << K);
    o.is_leaf.resize(nn);
    o.split_dim.resize(nn);
    o.left.resize(nn);
    o.right.resize(nn);
    o.bits.resize(nn * K);
    o.value.resize(nn * K);
    o.ebegin.resize(nn);
    o.ecount.resize(nn);
    std::vector<uint32_t> nb(nn), perm(t.n);
    DETLSH_CUDA(cudaMemcpy(o.root_children.data(), t.root_children.get(), o.root_children.size() * 4, cudaMemcpyDeviceToHost));
    DETLSH_CUDA(cudaMemcpy(o.is_leaf.data(), t.is_leaf.get(), nn, cudaMemcpyDeviceToHost));
    DETLSH_CUDA(cudaMemcpy(o.split_dim.data(), t.split_dim.get(), nn, cudaMemcpyDeviceToHost));
    DETLSH_CUDA(cudaMemcpy(o.left.data(), t.left.get(), nn * 4, cudaMemcpyDeviceToHost));
    DETLSH_CUDA(cudaMemcpy(o.right.data(), t.right.get(), nn * 4, cudaMemcpyDeviceToHost));
    DETLSH_CUDA(cudaMemcpy(o.bits.data(), t.bits.get(), nn * K, cudaMemcpyDeviceToHost));
    DETLSH_CUDA(cudaMemcpy(o.value.data(), t.value.get(), nn * K, cudaMemcpyDeviceToHost));
    DETLSH_CUDA(cudaMemcpy(nb.data(), t.node_begin.get(), nn * 4, cudaMemcpyDeviceToHost));
    DETLSH_CUDA(cudaMemcpy(o.ecount.data(), t.node_count.get(), nn * 4, cudaMemcpyDeviceToHost));
    DETLSH_CUDA(cudaMemcpy(perm.data(), t.perm.get(), t.n * 4, cudaMemcpyDeviceToHost));
    o.positions.resize(t.n);
    uint64_t off = 0;
    for (uint64_t i = 0; i < nn; ++i) {
        o.ebegin[i] = off;
        const uint32_t c = o.ecount[i];
        std::copy(perm.begin() + nb[i], perm.begin() + nb[i] + c, o.positions.begin() + off);
        off += c;
    }
}

}  // namespace detlsh_b200
