// DETL v1 export of a GPU-built index (persist.cpp:99-149): the byte stream the
// reference's save_index writes for the same index, so the reference's
// load_index + ck_ann can serve a GPU-built index (and the bytes themselves
// are a parity anchor: trees, table, params and fingerprint in one blob).
//
// Layout (little-endian): "DETL", u32 version 1; params (i32 K, L; f64 c, beta,
// epsilon, alpha1, alpha2; i32 n_regions; f64 sample_fraction; i32
// leaf_capacity; f64 r_min; i32 k; u8 projection kind = lsh); u64 family seed,
// i32 d, K, L; table (i32 L, K, n_regions; u64 sample_size; f32 boundaries);
// u64 n, i32 d; u32 tree count, per tree: i32 space, i32 max_size, u32 filled
// root slots, per slot (ascending) u32 slot + preorder subtree (u8 is_leaf;
// leaf: u32 count, count*K u8 symbols, count u32 positions; inner: u8
// split_dim, left, right); u64 dataset fingerprint (FNV-1a 64 over n, d and the
// float bytes, dataset.cpp:22-30).
#include <cstring>
#include <vector>

#include "index.cuh"
#include "stages.cuh"
#include "tree.cuh"

namespace detlsh_b200 {

namespace {

struct Out {
    std::vector<uint8_t> b;
    void put(const void* p, size_t len) {
        const auto* c = static_cast<const uint8_t*>(p);
        b.insert(b.end(), c, c + len);
    }
    template <typename T>
    void scalar(T v) {
        put(&v, sizeof(T));
    }
};

constexpr uint64_t kFnvOffset = 0xcbf29ce484222325ULL;
constexpr uint64_t kFnvPrime = 0x100000001b3ULL;

void fnv_mix(uint64_t& h, const void* bytes, size_t len) {
    const auto* p = static_cast<const unsigned char*>(bytes);
    for (size_t i = 0; i < len; ++i) {
        h ^= p[i];
        h *= kFnvPrime;
    }
}

// Preorder subtree of node `id` (reference ids), leaf entries in leaf order
// (ascending position = the reference's insertion order).
void write_subtree(Out& o, const HostTreeExport& t, int32_t id, const uint8_t* codes, int K) {
    // explicit stack: (node) in preorder, right pushed before left
    std::vector<int32_t> st{id};
    while (!st.empty()) {
        const int32_t v = st.back();
        st.pop_back();
        if (t.is_leaf[v]) {
            o.scalar<uint8_t>(1);
            const uint32_t cnt = t.ecount[v];
            const uint64_t b0 = t.ebegin[v];
            o.scalar<uint32_t>(cnt);
            for (uint32_t e = 0; e < cnt; ++e) o.put(codes + static_cast<size_t>(t.positions[b0 + e]) * K, K);
            o.put(t.positions.data() + b0, static_cast<size_t>(cnt) * 4);
        } else {
            o.scalar<uint8_t>(0);
            o.scalar<uint8_t>(t.split_dim[v]);
            st.push_back(t.right[v]);
            st.push_back(t.left[v]);
        }
    }
}

}  // namespace

std::vector<uint8_t> save_detl(GpuIndex& X) {
    DeviceGuard dg(X.device);
    cudaStream_t s = X.main.s;
    StreamScope scope(s);
    const detlsh_params& p = X.params;
    const int K = p.K, L = p.L, d = X.d;
    const uint64_t n = X.n;
    Out o;
    o.put("DETL", 4);
    o.scalar<uint32_t>(1);
    o.scalar<int32_t>(p.K);
    o.scalar<int32_t>(p.L);
    o.scalar<double>(p.c);
    o.scalar<double>(p.beta);
    o.scalar<double>(p.epsilon);
    o.scalar<double>(p.alpha1);
    o.scalar<double>(p.alpha2);
    o.scalar<int32_t>(p.n_regions);
    o.scalar<double>(p.sample_fraction);
    o.scalar<int32_t>(p.leaf_capacity);
    o.scalar<double>(p.r_min);
    o.scalar<int32_t>(p.k);
    o.scalar<uint8_t>(X.paa ? 1 : 0);  // ProjectionKind lsh / paa (index.hpp:16-19)
    o.scalar<uint64_t>(X.family_seed);  // PAA: an empty HashFamily (all zero)
    o.scalar<int32_t>(X.paa ? 0 : d);
    o.scalar<int32_t>(X.paa ? 0 : K);
    o.scalar<int32_t>(X.paa ? 0 : L);
    o.scalar<int32_t>(L);
    o.scalar<int32_t>(K);
    o.scalar<int32_t>(p.n_regions);
    o.scalar<uint64_t>(X.sample_size);
    o.put(X.h_table.data(), X.h_table.size() * sizeof(float));
    o.scalar<uint64_t>(n);
    o.scalar<int32_t>(d);
    // entry symbols = the codes of every point in each space: kept from the
    // build, or recomputed (projection + encode) when the build dropped them
    std::vector<uint8_t> codes(n * static_cast<size_t>(K));
    DevBuf<float> proj;
    DevBuf<uint8_t> dcodes;
    if (!X.codes.get()) {
        proj.alloc(static_cast<size_t>(L) * n * K);
        if (X.paa) launch_project_paa(X.data, n, d, K, proj.get(), s);
        else launch_project_exact(X.data, n, d, X.coeffs_t.get(), K, L, proj.get(), s, "project_exact", &X.proj_tc);
        dcodes.alloc(static_cast<size_t>(L) * n * K);
        launch_encode(proj.get(), n, K, L, X.table.get(), p.n_regions, dcodes.get(), s);
    }
    const uint8_t* all_codes = X.codes.get() ? X.codes.get() : dcodes.get();
    o.scalar<uint32_t>(static_cast<uint32_t>(L));
    for (int i = 0; i < L; ++i) {
        DETLSH_CUDA(cudaMemcpyAsync(codes.data(), all_codes + static_cast<size_t>(i) * n * K, codes.size(),
                                    cudaMemcpyDeviceToHost, s));
        DETLSH_CUDA(cudaStreamSynchronize(s));
        HostTreeExport t;
        export_tree(*X.trees[i], t);
        o.scalar<int32_t>(i);
        o.scalar<int32_t>(p.leaf_capacity);
        uint32_t filled = 0;
        for (const int32_t c : t.root_children) filled += c >= 0;
        o.scalar<uint32_t>(filled);
        for (size_t slot = 0; slot < t.root_children.size(); ++slot) {
            if (t.root_children[slot] < 0) continue;
            o.scalar<uint32_t>(static_cast<uint32_t>(slot));
            write_subtree(o, t, t.root_children[slot], codes.data(), K);
        }
    }
    // dataset fingerprint, on the host (FNV is a sequential byte chain)
    {
        std::vector<float> h(n * static_cast<size_t>(d));
        DETLSH_CUDA(cudaMemcpyAsync(h.data(), X.data, h.size() * 4, cudaMemcpyDeviceToHost, s));
        DETLSH_CUDA(cudaStreamSynchronize(s));
        uint64_t fp = kFnvOffset;
        const uint32_t d32 = static_cast<uint32_t>(d);
        fnv_mix(fp, &n, sizeof(n));
        fnv_mix(fp, &d32, sizeof(d32));
        fnv_mix(fp, h.data(), h.size() * sizeof(float));
        o.scalar<uint64_t>(fp);
    }
    return std::move(o.b);
}

}  // namespace detlsh_b200
