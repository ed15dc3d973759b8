// Point-sharded DET-LSH in one process: the dataset
// splits into contiguous row ranges, each an independent index (own sample,
// breakpoints, trees, r_min, budget ceil(beta * n_s + k)) on its device; a
// query batch runs on every shard's stream at once (device-side decisions, no
// host waits), each shard's top-k ids are widened to global positions on its
// device, copied to the merge device (peer copies over NVLink; a plain copy
// when a device holds several shards) and merged by (distance, global id).
// The multi-process form of the same exchange is the NCCL all-gather in
// bench.py / shard.py (one rank per GPU).
#include <algorithm>
#include <exception>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include "index.cuh"
#include "query.cuh"
#include "sharded.cuh"

namespace detlsh_b200 {

namespace {

__global__ void widen_ids_kernel(const uint32_t* __restrict__ ids, uint64_t m, uint64_t offset,
                                 uint64_t* __restrict__ out) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < m;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        out[i] = static_cast<uint64_t>(ids[i]) + offset;
}

void enable_peer(int a, int b) {
    if (a == b) return;
    int can = 0;
    DETLSH_CUDA(cudaDeviceCanAccessPeer(&can, a, b));
    if (!can) return;
    DeviceGuard dg(a);
    const cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
    if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) DETLSH_CUDA(e);
    cudaGetLastError();
}

}  // namespace

ShardedIndex::~ShardedIndex() {
    for (auto& sh : q)
        if (sh && sh->done) cudaEventDestroy(sh->done);
    if (inputs_ready) cudaEventDestroy(inputs_ready);
    if (merge_done) cudaEventDestroy(merge_done);
}

std::unique_ptr<ShardedIndex> sharded_build(const float* points, uint64_t n, int d, detlsh_params* params,
                                            uint64_t seed, const int32_t* devices, int shards,
                                            uint32_t flags) {
    if (!params) throw InvalidArgument("build_index: params is null");
    if (!points) throw InvalidArgument("build_index: points is null");
    if (!devices || shards < 1) throw InvalidArgument("sharded build: need at least one shard");
    if (static_cast<uint64_t>(shards) > n) throw InvalidArgument("sharded build: more shards than points");
    if (flags & DETLSH_F_BORROW_DATA) throw InvalidArgument("sharded build: shards own their rows");
    int ndev = 0;
    DETLSH_CUDA(cudaGetDeviceCount(&ndev));
    for (int s = 0; s < shards; ++s)
        if (devices[s] < 0 || devices[s] >= ndev) throw InvalidArgument("sharded build: no such device");
    auto X = std::make_unique<ShardedIndex>();
    X->devices.assign(devices, devices + shards);
    X->offsets.resize(shards + 1);
    for (int s = 0; s <= shards; ++s) X->offsets[s] = static_cast<uint64_t>(s) * n / shards;  // shard.py shard_bounds
    X->shards.resize(shards);
    std::vector<detlsh_params> ps(shards, *params);
    std::vector<std::exception_ptr> errs(shards);
    std::vector<std::thread> th;
    for (int s = 0; s < shards; ++s)
        th.emplace_back([&, s]() {
            try {
                DETLSH_CUDA(cudaSetDevice(devices[s]));
                const uint64_t r0 = X->offsets[s], r1 = X->offsets[s + 1];
                X->shards[s] = build_index_impl(points + r0 * static_cast<uint64_t>(d), r1 - r0, d, &ps[s],
                                                nullptr, 0, seed, devices[s], flags);
            } catch (...) {
                errs[s] = std::current_exception();
            }
        });
    for (auto& t : th) t.join();
    for (auto& e : errs)
        if (e) std::rethrow_exception(e);
    X->merge_device = devices[0];
    for (int s = 1; s < shards; ++s) {
        enable_peer(X->merge_device, devices[s]);
        enable_peer(devices[s], X->merge_device);
    }
    for (int s = 0; s < shards; ++s) {
        DeviceGuard dg(devices[s]);
        X->q.push_back(std::make_unique<ShardedIndex::ShardQuery>());
        X->q[s]->stream.create();
        DETLSH_CUDA(cudaEventCreateWithFlags(&X->q[s]->done, cudaEventDisableTiming));
    }
    {
        DeviceGuard dg(X->merge_device);
        X->main.create();
        DETLSH_CUDA(cudaEventCreateWithFlags(&X->inputs_ready, cudaEventDisableTiming));
        DETLSH_CUDA(cudaEventCreateWithFlags(&X->merge_done, cudaEventDisableTiming));
    }
    *params = ps[0];  // the derived fields are shared; r_min is per shard
    return X;
}

void sharded_query(ShardedIndex& X, const float* queries, uint64_t nq, int k, uint32_t flags, uint64_t* ids,
                   double* dists, int32_t* n_hits, cudaStream_t user_stream) {
    const int S = static_cast<int>(X.shards.size());
    for (const auto& sh : X.shards)
        if (k < 1 || static_cast<uint64_t>(k) > sh->n) throw InvalidArgument("ck_ann: k must lie in [1, n] of every shard");
    if (nq == 0) return;
    if (!queries) throw InvalidArgument("ck_ann: queries is null");
    std::lock_guard<std::mutex> lock(X.mu);
    DeviceGuard dg(X.merge_device);
    cudaStream_t ms = user_stream ? user_stream : X.main.s;
    const bool dev = (flags & DETLSH_F_DEVICE_PTRS) != 0;
    const int d = X.shards[0]->d;
    const size_t qbytes = nq * static_cast<size_t>(d) * 4;
    const size_t lists = static_cast<size_t>(S) * nq * k;
    // merge-device staging: queries (host input), gathered per-shard lists, outputs
    auto grow = [&](auto& buf, size_t count, int device, cudaStream_t s) {
        if (buf.size() >= count) return;
        if (X.merged_once) DETLSH_CUDA(cudaEventSynchronize(X.merge_done));  // last batch done reading
        DeviceGuard g(device);
        DETLSH_CUDA(cudaStreamSynchronize(s));
        StreamScope sc(s);
        buf.alloc(count);
        DETLSH_CUDA(cudaStreamSynchronize(s));
    };
    grow(X.g_dists, lists, X.merge_device, X.main.s);
    grow(X.g_ids, lists, X.merge_device, X.main.s);
    grow(X.g_hits, static_cast<size_t>(S) * nq, X.merge_device, X.main.s);
    // the previous batch (possibly on another stream) is done with the staging
    if (X.merged_once) DETLSH_CUDA(cudaStreamWaitEvent(ms, X.merge_done, 0));
    const float* q_merge = queries;
    if (!dev) {
        grow(X.q_stage, nq * static_cast<size_t>(d), X.merge_device, X.main.s);
        DETLSH_CUDA(cudaMemcpyAsync(X.q_stage.get(), queries, qbytes, cudaMemcpyHostToDevice, ms));
        q_merge = X.q_stage.get();
    }
    DETLSH_CUDA(cudaEventRecord(X.inputs_ready, ms));
    for (int s = 0; s < S; ++s) {
        ShardedIndex::ShardQuery& Q = *X.q[s];
        GpuIndex& G = *X.shards[s];
        DeviceGuard gs(G.device);
        cudaStream_t ss = Q.stream.s;
        grow(Q.ids, nq * static_cast<size_t>(k), G.device, ss);
        grow(Q.ids64, nq * static_cast<size_t>(k), G.device, ss);
        grow(Q.dists, nq * static_cast<size_t>(k), G.device, ss);
        grow(Q.hits, nq, G.device, ss);
        const float* qs = q_merge;
        if (G.device != X.merge_device) grow(Q.q, nq * static_cast<size_t>(d), G.device, ss);
        DETLSH_CUDA(cudaStreamWaitEvent(ss, X.inputs_ready, 0));
        if (G.device != X.merge_device) {
            DETLSH_CUDA(cudaMemcpyPeerAsync(Q.q.get(), G.device, q_merge, X.merge_device, qbytes, ss));
            qs = Q.q.get();
        }
        query_impl(G, qs, nq, k, DETLSH_F_DEVICE_PTRS | (flags & DETLSH_F_NO_TC), Q.ids.get(), Q.dists.get(),
                   Q.hits.get(), nullptr, nullptr, ss);
        const uint64_t m = nq * static_cast<uint64_t>(k);
        const unsigned grid = static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>((m + 255) / 256, 4096)));
        widen_ids_kernel<<<grid, 256, 0, ss>>>(Q.ids.get(), m, X.offsets[s], Q.ids64.get());
        DETLSH_LAUNCH_CHECK();
        // this shard's lists into slot s of the merge device's [S][nq][k] arrays
        const size_t at = static_cast<size_t>(s) * nq * k;
        DETLSH_CUDA(cudaMemcpyPeerAsync(X.g_dists.get() + at, X.merge_device, Q.dists.get(), G.device, m * 8, ss));
        DETLSH_CUDA(cudaMemcpyPeerAsync(X.g_ids.get() + at, X.merge_device, Q.ids64.get(), G.device, m * 8, ss));
        DETLSH_CUDA(cudaMemcpyPeerAsync(X.g_hits.get() + static_cast<size_t>(s) * nq, X.merge_device, Q.hits.get(),
                                        G.device, nq * 4, ss));
        DETLSH_CUDA(cudaEventRecord(Q.done, ss));
    }
    for (int s = 0; s < S; ++s) DETLSH_CUDA(cudaStreamWaitEvent(ms, X.q[s]->done, 0));
    if (dev) {
        launch_merge_topk(X.g_dists.get(), X.g_ids.get(), X.g_hits.get(), S, nq, k, dists, ids, n_hits, ms);
        DETLSH_CUDA(cudaEventRecord(X.merge_done, ms));
        X.merged_once = true;
        return;  // stream-ordered
    }
    grow(X.o_dists, nq * static_cast<size_t>(k), X.merge_device, X.main.s);
    grow(X.o_ids, nq * static_cast<size_t>(k), X.merge_device, X.main.s);
    grow(X.o_hits, nq, X.merge_device, X.main.s);
    launch_merge_topk(X.g_dists.get(), X.g_ids.get(), X.g_hits.get(), S, nq, k, X.o_dists.get(), X.o_ids.get(),
                      X.o_hits.get(), ms);
    if (ids) DETLSH_CUDA(cudaMemcpyAsync(ids, X.o_ids.get(), nq * k * 8, cudaMemcpyDeviceToHost, ms));
    if (dists) DETLSH_CUDA(cudaMemcpyAsync(dists, X.o_dists.get(), nq * k * 8, cudaMemcpyDeviceToHost, ms));
    if (n_hits) DETLSH_CUDA(cudaMemcpyAsync(n_hits, X.o_hits.get(), nq * 4, cudaMemcpyDeviceToHost, ms));
    DETLSH_CUDA(cudaEventRecord(X.merge_done, ms));
    X.merged_once = true;
    DETLSH_CUDA(cudaStreamSynchronize(ms));
    for (auto& sh : X.shards)
        if (query_invariant_failed(sh->scratch, sh->main.s))
            throw CudaError("ck_ann: internal invariant violated (budget cut emitted != budget rows)");
}

}  // namespace detlsh_b200
