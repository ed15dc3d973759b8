// Stage functions of the DE-Tree range queries (de_tree.hpp:85-100) on the
// device, for one tree and a batch of projected queries:
//
//   range_query_optimized (de_tree.cpp:229-258): every leaf with
//     mindist <= radius, drained in ascending (mindist, node index) order, each
//     leaf's entries in order, stopping after `limit` positions (the sink).
//   range_query_exact (de_tree.cpp:199-227): exactly the positions whose
//     projected distance is <= radius, in the reference's DFS order (root
//     children ascending, left subtree first, entries in leaf order).
//
// mindist follows de_tree.cpp:154-184 operation for operation (float
// boundaries widened to double, pen = lo - v or v - hi, acc += pen * pen, sqrt;
// infinite outer edges).  For the exact form the mindist prune and maxdist
// accept are exact, so the result set is {pos : l2 <= radius}
// over the exact fp32 projections (projection kernel), ordered by DFS leaf.
#include <algorithm>
#include <vector>

#include "index.cuh"
#include "primitives.cuh"
#include "stages.cuh"
#include "tree.cuh"

namespace detlsh_b200 {

namespace {

__global__ void leaf_mindist_kernel(const uint8_t* __restrict__ box, uint64_t num_leaves, int K, int NR,
                                    const float* __restrict__ row0, const float* __restrict__ qp,
                                    double radius, uint64_t* __restrict__ key, uint32_t* __restrict__ flag) {
    for (uint64_t li = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; li < num_leaves;
         li += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint8_t* b = box + li * (kBoxStride * 2);
        double acc = 0.0;
        for (int j = 0; j < K; ++j) {
            const int lo = b[2 * j], hi = b[2 * j + 1];
            const float* row = row0 + static_cast<size_t>(j) * (NR + 1);
            const double v = static_cast<double>(qp[j]);
            double pen = 0.0;
            if (lo > 0 && v < static_cast<double>(row[lo])) pen = __dsub_rn(static_cast<double>(row[lo]), v);
            else if (hi < NR - 1 && v > static_cast<double>(row[hi + 1]))
                pen = __dsub_rn(v, static_cast<double>(row[hi + 1]));
            acc = __dadd_rn(acc, __dmul_rn(pen, pen));
        }
        const double md = __dsqrt_rn(acc);
        key[li] = static_cast<uint64_t>(__double_as_longlong(md));  // md >= 0: bits order like values
        flag[li] = md <= radius ? 1u : 0u;
    }
}

// stable compaction of the flagged leaves (offsets = exclusive scan of flags)
__global__ void compact_leaves_kernel(const uint64_t* __restrict__ key, const uint32_t* __restrict__ flag,
                                      const uint32_t* __restrict__ off, uint64_t num_leaves,
                                      uint64_t* __restrict__ okey, uint32_t* __restrict__ oleaf) {
    for (uint64_t li = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; li < num_leaves;
         li += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        if (!flag[li]) continue;
        okey[off[li]] = key[li];
        oleaf[off[li]] = static_cast<uint32_t>(li);
    }
}

__global__ void leaf_counts_kernel(const uint32_t* __restrict__ leaves, uint64_t m,
                                   const uint32_t* __restrict__ leaf_count, uint32_t* __restrict__ cnt) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < m;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        cnt[i] = leaf_count[leaves[i]];
}

// drain: the entries of leaves[i] at output offsets off[i].., up to `limit`
__global__ void drain_kernel(const uint32_t* __restrict__ leaves, uint64_t m, const uint32_t* __restrict__ off,
                             const uint32_t* __restrict__ leaf_begin, const uint32_t* __restrict__ leaf_count,
                             const uint32_t* __restrict__ perm, uint64_t limit, uint32_t* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const uint64_t warps = static_cast<uint64_t>(gridDim.x) * (blockDim.x / 32);
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x / 32) + (threadIdx.x >> 5); i < m; i += warps) {
        const uint32_t li = leaves[i], b0 = leaf_begin[li], c = leaf_count[li];
        for (uint32_t e = lane; e < c; e += 32) {
            const uint64_t o = static_cast<uint64_t>(off[i]) + e;
            if (o < limit) out[o] = perm[b0 + e];
        }
    }
}

// exact: pass[pos] = l2(q', p'_pos) <= radius over the fp32 projections of the space
__global__ void exact_pass_kernel(const float* __restrict__ proj, uint64_t n, int K, const float* __restrict__ qp,
                                  double radius, uint8_t* __restrict__ pass) {
    for (uint64_t z = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; z < n;
         z += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        double acc = 0.0;
        for (int j = 0; j < K; ++j) {
            const double diff = __dsub_rn(static_cast<double>(qp[j]), static_cast<double>(proj[z * K + j]));
            acc = __dadd_rn(acc, __dmul_rn(diff, diff));
        }
        pass[z] = __dsqrt_rn(acc) <= radius ? 1 : 0;
    }
}

// per DFS leaf slot: entries that pass (counted, then written in entry order)
__global__ void exact_emit_kernel(const uint32_t* __restrict__ dfs, uint64_t m, const uint32_t* __restrict__ leaf_begin,
                                  const uint32_t* __restrict__ leaf_count, const uint32_t* __restrict__ perm,
                                  const uint8_t* __restrict__ pass, const uint32_t* __restrict__ off,
                                  uint32_t* __restrict__ cnt, uint32_t* __restrict__ out, uint64_t cap) {
    const int lane = threadIdx.x & 31;
    const uint64_t warps = static_cast<uint64_t>(gridDim.x) * (blockDim.x / 32);
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x / 32) + (threadIdx.x >> 5); i < m; i += warps) {
        const uint32_t li = dfs[i], b0 = leaf_begin[li], c = leaf_count[li];
        uint32_t taken = 0;
        for (uint32_t base = 0; base < c; base += 32) {
            const uint32_t e = base + lane;
            const uint32_t pos = e < c ? perm[b0 + e] : 0;
            const bool ok = e < c && pass[pos];
            const uint32_t bal = __ballot_sync(0xffffffffu, ok);
            if (off && ok) {
                const uint64_t o = static_cast<uint64_t>(off[i]) + taken + __popc(bal & ((1u << lane) - 1u));
                if (o < cap) out[o] = pos;
            }
            taken += __popc(bal);
        }
        if (!off && lane == 0) cnt[i] = taken;
    }
}

unsigned grid_for(uint64_t m) {
    return static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>((m + 255) / 256, 8192)));
}

// leaf indices of tree T in the reference's DFS order (root children ascending,
// left before right), cached on the index
const DevBuf<uint32_t>& dfs_leaf_order(GpuIndex& X, int tree, cudaStream_t s) {
    if (X.dfs_leaves.size() < X.trees.size()) X.dfs_leaves.resize(X.trees.size());
    auto& slot = X.dfs_leaves[tree];
    if (slot) return *slot;
    const DevTree& T = *X.trees[tree];
    HostTreeExport e;
    export_tree(T, e);
    std::vector<uint32_t> leaf_node(T.num_leaves);
    DETLSH_CUDA(cudaMemcpy(leaf_node.data(), T.leaf_node.get(), T.num_leaves * 4, cudaMemcpyDeviceToHost));
    std::vector<int32_t> leaf_of(e.is_leaf.size(), -1);
    for (uint32_t li = 0; li < T.num_leaves; ++li) leaf_of[leaf_node[li]] = static_cast<int32_t>(li);
    std::vector<uint32_t> order;
    order.reserve(T.num_leaves);
    std::vector<int32_t> stack;
    for (const int32_t root : e.root_children) {
        if (root < 0) continue;
        stack.push_back(root);
        while (!stack.empty()) {
            const int32_t v = stack.back();
            stack.pop_back();
            if (e.is_leaf[v]) {
                order.push_back(static_cast<uint32_t>(leaf_of[v]));
            } else {
                stack.push_back(e.right[v]);  // left is visited first
                stack.push_back(e.left[v]);
            }
        }
    }
    slot = std::make_unique<DevBuf<uint32_t>>();
    {
        StreamScope sc(X.main.s);
        slot->alloc(order.size());
    }
    DETLSH_CUDA(cudaMemcpyAsync(slot->get(), order.data(), order.size() * 4, cudaMemcpyHostToDevice, s));
    DETLSH_CUDA(cudaStreamSynchronize(s));
    return *slot;
}

}  // namespace

void range_query_impl(GpuIndex& X, int tree, const float* q_proj, uint64_t nq, const double* radius, uint64_t limit,
                      bool exact, uint32_t* out, uint64_t cap, uint64_t* counts) {
    if (tree < 0 || tree >= X.params.L) throw InvalidArgument("range_query: tree index out of range");
    if (nq == 0) return;
    if (!q_proj || !radius || !counts) throw InvalidArgument("range_query: null argument");
    if (cap && !out) throw InvalidArgument("range_query: out is null");
    DeviceGuard dg(X.device);
    std::lock_guard<std::mutex> lock(X.qmu);
    cudaStream_t s = X.main.s;
    StreamScope scope(s);
    const DevTree& T = *X.trees[tree];
    const int K = X.params.K, NR = X.params.n_regions;
    const uint64_t nl = T.num_leaves, n = X.n;
    const float* row0 = X.table.get() + static_cast<size_t>(tree) * K * (NR + 1);
    DevBuf<float> qd(static_cast<size_t>(nq) * K);
    DETLSH_CUDA(cudaMemcpyAsync(qd.get(), q_proj, nq * K * 4, cudaMemcpyHostToDevice, s));
    DevBuf<uint32_t> res(std::max<uint64_t>(cap, 1)), total(1);
    DevBuf<uint32_t> tmp(scan_temp_elems(std::max(nl, n)));
    if (!exact) {
        DevBuf<uint64_t> key(nl), k0(nl), k1(nl);
        DevBuf<uint32_t> flag(nl), off(nl), v0(nl), v1(nl), cnt(nl), coff(nl), rtmp(radix_temp_elems(nl));
        for (uint64_t q = 0; q < nq; ++q) {
            leaf_mindist_kernel<<<grid_for(nl), 256, 0, s>>>(T.leaf_box.get(), nl, K, NR, row0, qd.get() + q * K,
                                                             radius[q], key.get(), flag.get());
            DETLSH_LAUNCH_CHECK();
            exclusive_scan_u32(flag.get(), off.get(), nl, tmp.get(), total.get(), s);
            uint32_t m = 0;
            DETLSH_CUDA(cudaMemcpyAsync(&m, total.get(), 4, cudaMemcpyDeviceToHost, s));
            DETLSH_CUDA(cudaStreamSynchronize(s));
            uint64_t emitted = 0;
            if (m) {
                compact_leaves_kernel<<<grid_for(nl), 256, 0, s>>>(key.get(), flag.get(), off.get(), nl, k0.get(),
                                                                   v0.get());
                DETLSH_LAUNCH_CHECK();
                // stable sort by mindist: ties stay in node-id order (leaves are in node-id order)
                const bool flip = radix_sort_pairs<uint64_t>(k0.get(), v0.get(), k1.get(), v1.get(), m, 0, 64,
                                                             rtmp.get(), s);
                const uint32_t* leaves = flip ? v1.get() : v0.get();
                leaf_counts_kernel<<<grid_for(m), 256, 0, s>>>(leaves, m, T.leaf_count.get(), cnt.get());
                DETLSH_LAUNCH_CHECK();
                exclusive_scan_u32(cnt.get(), coff.get(), m, tmp.get(), total.get(), s);
                uint32_t all = 0;
                DETLSH_CUDA(cudaMemcpyAsync(&all, total.get(), 4, cudaMemcpyDeviceToHost, s));
                DETLSH_CUDA(cudaStreamSynchronize(s));
                emitted = std::min<uint64_t>(all, limit);
                drain_kernel<<<grid_for(m * 32), 256, 0, s>>>(leaves, m, coff.get(), T.leaf_begin.get(),
                                                              T.leaf_count.get(), T.perm.get(),
                                                              std::min<uint64_t>(emitted, cap), res.get());
                DETLSH_LAUNCH_CHECK();
            }
            counts[q] = emitted;
            if (cap && emitted)
                DETLSH_CUDA(cudaMemcpyAsync(out + q * cap, res.get(), std::min(emitted, cap) * 4,
                                            cudaMemcpyDeviceToHost, s));
            DETLSH_CUDA(cudaStreamSynchronize(s));
        }
        return;
    }
    // exact: the space's fp32 projections (the reference's ProjectedLookup), DFS leaf order
    const DevBuf<uint32_t>& dfs = dfs_leaf_order(X, tree, s);
    const int L = X.params.L;
    DevBuf<float> proj(static_cast<size_t>(L) * n * K);
    if (X.paa) launch_project_paa(X.data, n, X.d, K, proj.get(), s);
    else launch_project_exact(X.data, n, X.d, X.coeffs_t.get(), K, L, proj.get(), s, "project_exact", &X.proj_tc);
    const float* pspace = proj.get() + static_cast<size_t>(tree) * n * K;
    DevBuf<uint8_t> pass(n);
    DevBuf<uint32_t> cnt(nl), off(nl);
    for (uint64_t q = 0; q < nq; ++q) {
        exact_pass_kernel<<<grid_for(n), 256, 0, s>>>(pspace, n, K, qd.get() + q * K, radius[q], pass.get());
        DETLSH_LAUNCH_CHECK();
        exact_emit_kernel<<<grid_for(nl * 32), 256, 0, s>>>(dfs.get(), nl, T.leaf_begin.get(), T.leaf_count.get(),
                                                            T.perm.get(), pass.get(), nullptr, cnt.get(), nullptr, 0);
        DETLSH_LAUNCH_CHECK();
        exclusive_scan_u32(cnt.get(), off.get(), nl, tmp.get(), total.get(), s);
        uint32_t all = 0;
        DETLSH_CUDA(cudaMemcpyAsync(&all, total.get(), 4, cudaMemcpyDeviceToHost, s));
        DETLSH_CUDA(cudaStreamSynchronize(s));
        if (cap && all) {
            exact_emit_kernel<<<grid_for(nl * 32), 256, 0, s>>>(dfs.get(), nl, T.leaf_begin.get(), T.leaf_count.get(),
                                                                T.perm.get(), pass.get(), off.get(), nullptr, res.get(),
                                                                cap);
            DETLSH_LAUNCH_CHECK();
            DETLSH_CUDA(cudaMemcpyAsync(out + q * cap, res.get(), std::min<uint64_t>(all, cap) * 4,
                                        cudaMemcpyDeviceToHost, s));
        }
        counts[q] = all;
        DETLSH_CUDA(cudaStreamSynchronize(s));
    }
}

}  // namespace detlsh_b200
