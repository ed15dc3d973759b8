// Batched ck_ann (index.cpp:292-331) on the GPU.
//
// Semantics reproduced exactly:
//   * radius schedule r = r_min * c^t (repeated multiply), range radius eps*r;
//   * range_query_optimized (de_tree.cpp:229-258): the leaves with
//     mindist <= radius (DFS pruning is monotone, so that is exactly the set
//     the DFS reaches), drained in ascending (mindist, node index) order;
//     mindist = sqrt of the sequential fp64 sum of per-dim squared penalties
//     from the float breakpoint edges, +-inf at regions 0 / N_r-1;
//   * CandidateSet dedup; the sink stops after the budget-th NEW position
//     (mid-leaf); count_within(c*r) >= k ends a round; top-k by (dist, pos).
//
// Instead of a heap drain, a weighted radix select over the 96-bit key
// (mindist bits, node id) finds the leaf where the budget trips and how many
// of its entries are taken: the emitted SET is identical, which is all the
// top-k depends on.  Fast path (one CTA per query): tree 0, round 0, no dedup.
// General path: bitmap dedup across trees and rounds, exact count_within.
#include <algorithm>

#include "query.cuh"

namespace detlsh_b200 {

namespace {

struct LeafItem {
    uint64_t mdb;  // mindist bits (non-negative double: bit order == value order)
    uint32_t id;   // node id (reference build order)
    uint32_t w;    // weight: entries this leaf would contribute
    uint32_t li;   // leaf index into QTree arrays
    uint32_t pad;
};

__device__ __forceinline__ bool key_less(uint64_t am, uint32_t ai, uint64_t bm, uint32_t bi) {
    return am < bm || (am == bm && ai < bi);
}

struct Smem {
    double* sq;       // [K][NR+1]
    int* lbv;         // [K]  #{b : row[b] <  v}
    int* ubv;         // [K]  #{b : row[b] <= v}
    float* qv;        // [d]
    float* qp;        // [K]
    double* td;       // [kTopCap]
    uint32_t* tp;     // [kTopCap]
    unsigned long long* hist;  // [256]
    unsigned long long* u64s;  // scratch scalars
    uint32_t* u32s;
};

__device__ __forceinline__ Smem carve(uint8_t* base, int K, int NR, int d) {
    Smem s;
    size_t off = 0;
    auto take = [&](size_t bytes, size_t align) {
        off = (off + align - 1) / align * align;
        uint8_t* p = base + off;
        off += bytes;
        return p;
    };
    s.sq = reinterpret_cast<double*>(take(sizeof(double) * K * (NR + 1), 16));
    s.td = reinterpret_cast<double*>(take(sizeof(double) * kTopCap, 16));
    s.hist = reinterpret_cast<unsigned long long*>(take(8 * 256, 16));
    s.u64s = reinterpret_cast<unsigned long long*>(take(8 * 16, 16));
    s.tp = reinterpret_cast<uint32_t*>(take(4 * kTopCap, 16));
    s.lbv = reinterpret_cast<int*>(take(4 * kMaxK, 16));
    s.ubv = reinterpret_cast<int*>(take(4 * kMaxK, 16));
    s.u32s = reinterpret_cast<uint32_t*>(take(4 * 16, 16));
    s.qp = reinterpret_cast<float*>(take(4 * kMaxK, 16));
    s.qv = reinterpret_cast<float*>(take(4 * static_cast<size_t>(d), 16));
    return s;
}

size_t smem_bytes(int K, int NR, int d) {
    size_t off = 0;
    auto take = [&](size_t bytes, size_t align) {
        off = (off + align - 1) / align * align;
        off += bytes;
    };
    take(sizeof(double) * K * (NR + 1), 16);
    take(sizeof(double) * kTopCap, 16);
    take(8 * 256, 16);
    take(8 * 16, 16);
    take(4 * kTopCap, 16);
    take(4 * kMaxK, 16);
    take(4 * kMaxK, 16);
    take(4 * 16, 16);
    take(4 * kMaxK, 16);
    take(4 * static_cast<size_t>(d), 16);
    return off + 16;
}

// Per (query, tree): squared edge penalties in fp64, exactly as mindist
// (de_tree.cpp:169-184) forms them: pen = double(edge) - double(v), pen*pen.
__device__ void build_sq(const QueryPlan& P, int tree, const Smem& S) {
    const int W = P.NR + 1;
    const float* tb = P.table + static_cast<size_t>(tree) * P.K * W;
    for (int j = threadIdx.x; j < P.K; j += blockDim.x) {
        S.lbv[j] = 0;
        S.ubv[j] = 0;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < P.K * W; i += blockDim.x) {
        const int j = i / W;
        const float row = tb[i];
        const float v = S.qp[j];
        const double D = __dsub_rn(static_cast<double>(row), static_cast<double>(v));
        S.sq[i] = __dmul_rn(D, D);
        if (row < v) atomicAdd(&S.lbv[j], 1);
        if (row <= v) atomicAdd(&S.ubv[j], 1);
    }
    __syncthreads();
}

__device__ __forceinline__ double leaf_mindist(const QueryPlan& P, const QTree& T, uint32_t li,
                                               const Smem& S) {
    const uint8_t* box = T.leaf_box + static_cast<size_t>(li) * 64;
    uint4 raw[3];
    raw[0] = reinterpret_cast<const uint4*>(box)[0];
    raw[1] = reinterpret_cast<const uint4*>(box)[1];
    if (P.K > 16) raw[2] = reinterpret_cast<const uint4*>(box)[2];
    const uint8_t* b = reinterpret_cast<const uint8_t*>(raw);
    const int W = P.NR + 1;
    double acc = 0.0;
#pragma unroll 4
    for (int j = 0; j < P.K; ++j) {
        const int lo = b[2 * j], hi = b[2 * j + 1];
        double pen_sq = 0.0;
        if (lo > 0 && lo >= S.ubv[j]) pen_sq = S.sq[j * W + lo];
        else if (hi < P.NR - 1 && hi + 1 < S.lbv[j]) pen_sq = S.sq[j * W + hi + 1];
        acc = __dadd_rn(acc, pen_sq);
    }
    return __dsqrt_rn(acc);
}

// Exact original-space distance (dataset.hpp:23-34): sequential fp64 sum.
__device__ __forceinline__ double l2_exact(const float* __restrict__ q, const float* __restrict__ x,
                                           int d) {
    double acc = 0.0;
    if ((d & 3) == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0) {
        const float4* x4 = reinterpret_cast<const float4*>(x);
        for (int t = 0; t < d / 4; ++t) {
            const float4 xv = __ldg(x4 + t);
            const float* qq = q + 4 * t;
            double df;
            df = __dsub_rn(static_cast<double>(qq[0]), static_cast<double>(xv.x));
            acc = __dadd_rn(acc, __dmul_rn(df, df));
            df = __dsub_rn(static_cast<double>(qq[1]), static_cast<double>(xv.y));
            acc = __dadd_rn(acc, __dmul_rn(df, df));
            df = __dsub_rn(static_cast<double>(qq[2]), static_cast<double>(xv.z));
            acc = __dadd_rn(acc, __dmul_rn(df, df));
            df = __dsub_rn(static_cast<double>(qq[3]), static_cast<double>(xv.w));
            acc = __dadd_rn(acc, __dmul_rn(df, df));
        }
    } else {
        for (int t = 0; t < d; ++t) {
            const double df = __dsub_rn(static_cast<double>(q[t]), static_cast<double>(__ldg(x + t)));
            acc = __dadd_rn(acc, __dmul_rn(df, df));
        }
    }
    return __dsqrt_rn(acc);
}

// Warp-aggregated append of `item` to list (counter in smem).
__device__ __forceinline__ void warp_append(bool ok, const LeafItem& it, LeafItem* list,
                                            uint32_t* counter) {
    const uint32_t m = __ballot_sync(0xffffffffu, ok);
    if (!m) return;
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(m) - 1;
    uint32_t base = 0;
    if (lane == leader) base = atomicAdd(counter, static_cast<uint32_t>(__popc(m)));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (ok) list[base + __popc(m & ((1u << lane) - 1u))] = it;
}

// Scan every leaf of tree `tree`, appending those with mindist <= radius.
// weight: leaf size, or (bitmap != null) the entries not yet in S.
__device__ void scan_leaves(const QueryPlan& P, int tree, double radius, const Smem& S,
                            LeafItem* A, const uint32_t* bitmap, uint32_t& nA, uint64_t& W) {
    const QTree T = P.trees[tree];
    if (threadIdx.x == 0) {
        S.u32s[0] = 0;
        S.u64s[0] = 0;
    }
    __syncthreads();
    unsigned long long wsum = 0;
    const uint32_t nl = T.num_leaves;
    for (uint32_t base = 0; base < nl; base += blockDim.x) {
        const uint32_t li = base + threadIdx.x;
        bool ok = false;
        LeafItem it;
        if (li < nl) {
            const double md = leaf_mindist(P, T, li, S);
            if (md <= radius) {
                uint32_t w = T.leaf_count[li];
                if (bitmap) {
                    const uint32_t b0 = T.leaf_begin[li];
                    uint32_t nw = 0;
                    for (uint32_t e = 0; e < w; ++e) {
                        const uint32_t pos = T.perm[b0 + e];
                        nw += ((bitmap[pos >> 5] >> (pos & 31)) & 1u) ? 0u : 1u;
                    }
                    w = nw;
                }
                if (w > 0) {
                    ok = true;
                    it.mdb = static_cast<uint64_t>(__double_as_longlong(md));
                    it.id = T.leaf_node[li];
                    it.w = w;
                    it.li = li;
                    it.pad = 0;
                    wsum += w;
                }
            }
        }
        warp_append(ok, it, A, &S.u32s[0]);
    }
    for (int o = 16; o; o >>= 1) wsum += __shfl_xor_sync(0xffffffffu, wsum, o);
    if ((threadIdx.x & 31) == 0 && wsum) atomicAdd(&S.u64s[0], wsum);
    __syncthreads();
    nA = S.u32s[0];
    W = S.u64s[0];
    __syncthreads();
}

__device__ __forceinline__ uint32_t key_digit(const LeafItem& it, int k) {
    return k < 8 ? static_cast<uint32_t>((it.mdb >> (56 - 8 * k)) & 0xff)
                 : static_cast<uint32_t>((it.id >> (24 - 8 * (k - 8))) & 0xff);
}

// Weighted radix select: the smallest key whose inclusive weight prefix
// reaches `need` (>= 1, <= total).  Leaves A untouched.
__device__ void weighted_select(LeafItem* A, uint32_t nA, uint64_t need, LeafItem* Bf,
                                LeafItem* Cf, const Smem& S, uint64_t& kmdb, uint32_t& kid,
                                uint64_t& take_cut) {
    LeafItem* src = A;
    uint32_t nsrc = nA;
    LeafItem* dst = Bf;
    const int lane = threadIdx.x & 31;
    for (int dg = 0; dg < 12 && nsrc > 1; ++dg) {
        for (int i = threadIdx.x; i < 256; i += blockDim.x) S.hist[i] = 0;
        if (threadIdx.x == 0) S.u32s[1] = 0;
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < nsrc; i += blockDim.x)
            atomicAdd(&S.hist[key_digit(src[i], dg)], static_cast<unsigned long long>(src[i].w));
        __syncthreads();
        if (threadIdx.x < 32) {
            unsigned long long part = 0;
            for (int b = 0; b < 8; ++b) part += S.hist[lane * 8 + b];
            unsigned long long incl = part;
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned long long t = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += t;
            }
            const unsigned long long excl = incl - part;
            const bool here = excl < need && need <= incl;
            if (here) {
                unsigned long long cum = excl;
                int bin = lane * 8;
                for (int b = 0; b < 8; ++b, ++bin) {
                    const unsigned long long c = S.hist[bin];
                    if (cum + c >= need) break;
                    cum += c;
                }
                S.u32s[2] = static_cast<uint32_t>(bin);
                S.u64s[1] = need - cum;
            }
        }
        __syncthreads();
        const uint32_t dsel = S.u32s[2];
        need = S.u64s[1];
        for (uint32_t base = 0; base < nsrc; base += blockDim.x) {
            const uint32_t i = base + threadIdx.x;
            bool ok = false;
            LeafItem it;
            if (i < nsrc) {
                it = src[i];
                ok = key_digit(it, dg) == dsel;
            }
            warp_append(ok, it, dst, &S.u32s[1]);
        }
        __syncthreads();
        nsrc = S.u32s[1];
        src = dst;
        dst = (dst == Bf) ? Cf : Bf;
        __syncthreads();
    }
    kmdb = src[0].mdb;
    kid = src[0].id;
    take_cut = need;
    __syncthreads();
}

// ---- block top-k over (dist, pos), ascending ---------------------------------
__device__ __forceinline__ bool dp_less(double a, uint32_t ap, double b, uint32_t bp) {
    return a < b || (a == b && ap < bp);
}

__device__ void topk_sort(const Smem& S) {
    const uint32_t cnt = S.u32s[4];
    for (uint32_t i = threadIdx.x + cnt; i < kTopCap; i += blockDim.x) {
        S.td[i] = __longlong_as_double(0x7ff0000000000000LL);
        S.tp[i] = 0xffffffffu;
    }
    __syncthreads();
    for (int size = 2; size <= kTopCap; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = threadIdx.x; i < kTopCap / 2; i += blockDim.x) {
                const int lo = 2 * i - (i & (stride - 1));
                const int hi = lo + stride;
                const bool asc = (lo & size) == 0;
                const double a = S.td[lo], b = S.td[hi];
                const uint32_t ap = S.tp[lo], bp = S.tp[hi];
                if (dp_less(b, bp, a, ap) == asc) {
                    S.td[lo] = b;
                    S.td[hi] = a;
                    S.tp[lo] = bp;
                    S.tp[hi] = ap;
                }
            }
            __syncthreads();
        }
    }
}

__device__ __forceinline__ void topk_init(const Smem& S) {
    if (threadIdx.x == 0) {
        S.u32s[4] = 0;  // count
        S.u32s[5] = 0;  // full
        S.u32s[6] = 0;  // tau pos
        S.u64s[2] = 0;  // tau dist bits
    }
    __syncthreads();
}

// Called by all threads; (valid, d, p) one candidate each.  Optional strict
// lower bound (lbd, lbp) for chunked extraction of large k.
__device__ void topk_push(const Smem& S, bool valid, double d, uint32_t p, int k) {
    bool take = valid;
    if (take && S.u32s[5]) {
        const double td = __longlong_as_double(static_cast<long long>(S.u64s[2]));
        take = dp_less(d, p, td, S.u32s[6]);
    }
    const uint32_t m = __ballot_sync(0xffffffffu, take);
    if (m) {
        const int lane = threadIdx.x & 31;
        const int leader = __ffs(m) - 1;
        uint32_t base = 0;
        if (lane == leader) base = atomicAdd(&S.u32s[4], static_cast<uint32_t>(__popc(m)));
        base = __shfl_sync(0xffffffffu, base, leader);
        if (take) {
            const uint32_t slot = base + __popc(m & ((1u << lane) - 1u));
            S.td[slot] = d;
            S.tp[slot] = p;
        }
    }
    __syncthreads();
    if (S.u32s[4] > static_cast<uint32_t>(kTopCap - blockDim.x)) {
        topk_sort(S);
        if (threadIdx.x == 0) {
            const uint32_t c = min(S.u32s[4], static_cast<uint32_t>(k));
            S.u32s[4] = c;
            if (c >= static_cast<uint32_t>(k)) {
                S.u32s[5] = 1;
                S.u64s[2] = static_cast<unsigned long long>(__double_as_longlong(S.td[k - 1]));
                S.u32s[6] = S.tp[k - 1];
            }
        }
        __syncthreads();
    }
}

// Sort and return count (<= k) of the staged entries.
__device__ uint32_t topk_finish(const Smem& S, int k) {
    topk_sort(S);
    const uint32_t c = min(S.u32s[4], static_cast<uint32_t>(k));
    __syncthreads();
    return c;
}

// ---------------------------------------------------------------------------
// Fast path: tree 0, round 0 fills the budget.
// ---------------------------------------------------------------------------
struct FastSlot {
    LeafItem *A, *B, *C;
    uint32_t* pre;
    uint32_t* cand;
};

__device__ __forceinline__ FastSlot fast_slot(uint8_t* base, size_t slot_bytes, uint32_t maxl,
                                              uint64_t budget) {
    uint8_t* p = base + static_cast<size_t>(blockIdx.x) * slot_bytes;
    FastSlot f;
    f.A = reinterpret_cast<LeafItem*>(p);
    f.B = f.A + maxl;
    f.C = f.B + maxl;
    f.pre = reinterpret_cast<uint32_t*>(f.C + maxl);
    f.cand = f.pre + maxl;
    (void)budget;
    return f;
}

__device__ void load_query(const QueryPlan& P, uint64_t q, int tree, const Smem& S, bool vec) {
    if (vec)
        for (int t = threadIdx.x; t < P.d; t += blockDim.x) S.qv[t] = P.q[q * P.d + t];
    for (int j = threadIdx.x; j < P.K; j += blockDim.x)
        S.qp[j] = P.qproj[(static_cast<uint64_t>(tree) * P.nq + q) * P.K + j];
    __syncthreads();
}

__global__ void __launch_bounds__(kQueryThreads) query_fast_kernel(
    QueryPlan P, uint8_t* scratch, size_t slot_bytes, uint32_t* slow_list, uint32_t* slow_n) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    const Smem S = carve(smem_raw, P.K, P.NR, P.d);
    const FastSlot F = fast_slot(scratch, slot_bytes, P.max_leaves, P.budget);
    const double radius = __dmul_rn(P.eps, P.r_min);
    const uint32_t B32 = static_cast<uint32_t>(P.budget);
    for (uint64_t q = blockIdx.x; q < P.nq; q += gridDim.x) {
        load_query(P, q, 0, S, true);
        build_sq(P, 0, S);
        uint32_t nA;
        uint64_t W;
        scan_leaves(P, 0, radius, S, F.A, nullptr, nA, W);
        if (W < P.budget) {  // budget does not fill in tree 0 round 0
            if (threadIdx.x == 0) slow_list[atomicAdd(slow_n, 1u)] = static_cast<uint32_t>(q);
            __syncthreads();
            continue;
        }
        uint64_t kmdb, take_cut;
        uint32_t kid;
        weighted_select(F.A, nA, P.budget, F.B, F.C, S, kmdb, kid, take_cut);
        // exclusive prefix of the taken counts, in A order
        if (threadIdx.x == 0) S.u32s[3] = 0;
        __syncthreads();
        for (uint32_t base = 0; base < nA; base += blockDim.x) {
            const uint32_t i = base + threadIdx.x;
            uint32_t take = 0;
            if (i < nA) {
                const LeafItem it = F.A[i];
                if (key_less(it.mdb, it.id, kmdb, kid)) take = it.w;
                else if (it.mdb == kmdb && it.id == kid) take = static_cast<uint32_t>(take_cut);
            }
            // block exclusive scan
            uint32_t incl = take;
            const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += t;
            }
            uint32_t* wt = reinterpret_cast<uint32_t*>(S.hist);
            if (lane == 31) wt[warp] = incl;
            __syncthreads();
            uint32_t wpre = 0, tot = 0;
            for (int w = 0; w < kQueryThreads / 32; ++w) {
                if (w < warp) wpre += wt[w];
                tot += wt[w];
            }
            if (i < nA) F.pre[i] = S.u32s[3] + wpre + incl - take;
            __syncthreads();
            if (threadIdx.x == 0) S.u32s[3] += tot;
            __syncthreads();
        }
        // candidate positions, one warp per leaf (coalesced along the leaf)
        {
            const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
            const QTree T = P.trees[0];
            for (uint32_t i = warp; i < nA; i += kQueryThreads / 32) {
                const LeafItem it = F.A[i];
                uint32_t take = 0;
                if (key_less(it.mdb, it.id, kmdb, kid)) take = it.w;
                else if (it.mdb == kmdb && it.id == kid) take = static_cast<uint32_t>(take_cut);
                const uint32_t dst = F.pre[i], src = T.leaf_begin[it.li];
                for (uint32_t e = lane; e < take; e += 32) F.cand[dst + e] = T.perm[src + e];
            }
        }
        __syncthreads();
        // exact verification + top-k
        topk_init(S);
        for (uint32_t c0 = 0; c0 < B32; c0 += blockDim.x) {
            const uint32_t c = c0 + threadIdx.x;
            double dist = 0.0;
            uint32_t pos = 0;
            const bool valid = c < B32;
            if (valid) {
                pos = F.cand[c];
                dist = l2_exact(S.qv, P.data + static_cast<uint64_t>(pos) * P.d, P.d);
            }
            topk_push(S, valid, dist, pos, P.k);
        }
        const uint32_t nh = topk_finish(S, P.k);
        for (uint32_t t = threadIdx.x; t < nh; t += blockDim.x) {
            if (P.ids) P.ids[q * P.k + t] = S.tp[t];
            if (P.dists) P.dists[q * P.k + t] = S.td[t];
        }
        if (threadIdx.x == 0) {
            if (P.n_hits) P.n_hits[q] = static_cast<int32_t>(nh);
            if (P.radius) P.radius[q] = P.r_min;
            if (P.cands) P.cands[q] = P.budget;
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// General path: every tree, every round, bitmap dedup (CandidateSet).
// ---------------------------------------------------------------------------
struct SlowSlot {
    LeafItem *A, *B, *C;
    uint32_t* bitmap;  // n bits
    uint32_t* mpos;    // members
    double* mdist;
};

__device__ __forceinline__ SlowSlot slow_slot(uint8_t* base, size_t slot_bytes, uint32_t maxl,
                                              uint64_t n, uint64_t budget) {
    uint8_t* p = base + static_cast<size_t>(blockIdx.x) * slot_bytes;
    SlowSlot s;
    s.A = reinterpret_cast<LeafItem*>(p);
    s.B = s.A + maxl;
    s.C = s.B + maxl;
    s.mdist = reinterpret_cast<double*>(s.C + maxl);
    s.mpos = reinterpret_cast<uint32_t*>(s.mdist + budget);
    s.bitmap = s.mpos + budget;
    (void)n;
    return s;
}

// Emit the NEW entries of the selected leaves (all, or the first `take_cut`
// new ones of the cut leaf) into the member list.
__device__ void emit_members(const QueryPlan& P, int tree, const LeafItem* A, uint32_t nA,
                             bool select, uint64_t kmdb, uint32_t kid, uint64_t take_cut,
                             const SlowSlot& L, const Smem& S) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const QTree T = P.trees[tree];
    for (uint32_t i = warp; i < nA; i += blockDim.x / 32) {
        const LeafItem it = A[i];
        uint64_t limit = 0xffffffffffffffffULL;
        if (select) {
            if (key_less(it.mdb, it.id, kmdb, kid)) limit = it.w;
            else if (it.mdb == kmdb && it.id == kid) limit = take_cut;
            else continue;
        }
        const uint32_t b0 = T.leaf_begin[it.li], cnt = T.leaf_count[it.li];
        uint64_t emitted = 0;
        for (uint32_t base = 0; base < cnt && emitted < limit; base += 32) {
            const uint32_t e = base + lane;
            uint32_t pos = 0;
            bool isnew = false;
            if (e < cnt) {
                pos = T.perm[b0 + e];
                isnew = !((L.bitmap[pos >> 5] >> (pos & 31)) & 1u);
            }
            const uint32_t m = __ballot_sync(0xffffffffu, isnew);
            const uint32_t rank = __popc(m & ((1u << lane) - 1u));
            const bool take = isnew && emitted + rank < limit;
            const uint32_t tm = __ballot_sync(0xffffffffu, take);
            if (tm) {
                const int leader = __ffs(tm) - 1;
                uint32_t slot0 = 0;
                if (lane == leader) slot0 = atomicAdd(&S.u32s[7], static_cast<uint32_t>(__popc(tm)));
                slot0 = __shfl_sync(0xffffffffu, slot0, leader);
                if (take) {
                    atomicOr(&L.bitmap[pos >> 5], 1u << (pos & 31));
                    const uint32_t slot = slot0 + __popc(tm & ((1u << lane) - 1u));
                    L.mpos[slot] = pos;
                    L.mdist[slot] = l2_exact(S.qv, P.data + static_cast<uint64_t>(pos) * P.d, P.d);
                }
            }
            emitted += __popc(tm);
        }
    }
    __syncthreads();
}

__global__ void __launch_bounds__(kQueryThreads) query_slow_kernel(
    QueryPlan P, const uint32_t* list, uint32_t count, uint8_t* scratch, size_t slot_bytes) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    const Smem S = carve(smem_raw, P.K, P.NR, P.d);
    const SlowSlot L = slow_slot(scratch, slot_bytes, P.max_leaves, P.n, P.budget);
    for (uint32_t qi = blockIdx.x; qi < count; qi += gridDim.x) {
        const uint64_t q = list ? list[qi] : qi;
        if (threadIdx.x == 0) S.u32s[7] = 0;  // |S|
        __syncthreads();
        for (int t = threadIdx.x; t < P.d; t += blockDim.x) S.qv[t] = P.q[q * P.d + t];
        double r = P.r_min;
        bool done = false;
        for (;;) {
            for (int tree = 0; tree < P.L && !done; ++tree) {
                load_query(P, q, tree, S, false);
                build_sq(P, tree, S);
                const double radius = __dmul_rn(P.eps, r);
                const uint32_t have = S.u32s[7];
                uint32_t nA;
                uint64_t W;
                scan_leaves(P, tree, radius, S, L.A, have ? L.bitmap : nullptr, nA, W);
                const uint64_t need = P.budget - have;
                if (W >= need) {
                    uint64_t kmdb, take_cut;
                    uint32_t kid;
                    weighted_select(L.A, nA, need, L.B, L.C, S, kmdb, kid, take_cut);
                    emit_members(P, tree, L.A, nA, true, kmdb, kid, take_cut, L, S);
                    done = true;
                } else {
                    emit_members(P, tree, L.A, nA, false, 0, 0, 0, L, S);
                }
            }
            if (done) break;
            // count_within(c * r) (index.cpp:244-249, 328)
            const double lim = __dmul_rn(P.c, r);
            const uint32_t msz = S.u32s[7];
            uint32_t mine = 0;
            for (uint32_t i = threadIdx.x; i < msz; i += blockDim.x) mine += L.mdist[i] <= lim ? 1u : 0u;
            for (int o = 16; o; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
            if (threadIdx.x == 0) S.u32s[8] = 0;
            __syncthreads();
            if ((threadIdx.x & 31) == 0 && mine) atomicAdd(&S.u32s[8], mine);
            __syncthreads();
            const bool enough = S.u32s[8] >= static_cast<uint32_t>(P.k);
            __syncthreads();
            if (enough) break;
            r = __dmul_rn(r, P.c);
        }
        // top-k of the members, extracted in chunks (any k)
        const uint32_t msz = S.u32s[7];
        const uint32_t want = min(msz, static_cast<uint32_t>(P.k));
        uint32_t out = 0;
        double lbd = -1.0;
        uint32_t lbp = 0;
        while (out < want) {
            const int kk = static_cast<int>(min(want - out, static_cast<uint32_t>(kFastMaxK)));
            topk_init(S);
            for (uint32_t c0 = 0; c0 < msz; c0 += blockDim.x) {
                const uint32_t c = c0 + threadIdx.x;
                bool valid = c < msz;
                double dist = 0.0;
                uint32_t pos = 0;
                if (valid) {
                    dist = L.mdist[c];
                    pos = L.mpos[c];
                    valid = dp_less(lbd, lbp, dist, pos);
                }
                topk_push(S, valid, dist, pos, kk);
            }
            const uint32_t got = topk_finish(S, kk);
            for (uint32_t t = threadIdx.x; t < got; t += blockDim.x) {
                if (P.ids) P.ids[q * P.k + out + t] = S.tp[t];
                if (P.dists) P.dists[q * P.k + out + t] = S.td[t];
            }
            lbd = S.td[got - 1];
            lbp = S.tp[got - 1];
            out += got;
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            if (P.n_hits) P.n_hits[q] = static_cast<int32_t>(want);
            if (P.radius) P.radius[q] = r;
            if (P.cands) P.cands[q] = msz;
        }
        // clear the bitmap words we touched
        for (uint32_t i = threadIdx.x; i < msz; i += blockDim.x) L.bitmap[L.mpos[i] >> 5] = 0;
        __syncthreads();
    }
}

__global__ void merge_topk_kernel(const double* __restrict__ sd, const uint64_t* __restrict__ sid,
                                  const int32_t* __restrict__ sh, int shards, uint64_t nq, int k,
                                  double* od, uint64_t* oid, int32_t* oh) {
    for (uint64_t q = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; q < nq;
         q += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        int head[16];
        for (int s = 0; s < shards; ++s) head[s] = 0;
        int out = 0;
        for (; out < k; ++out) {
            int best = -1;
            double bd = 0;
            uint64_t bi = 0;
            for (int s = 0; s < shards; ++s) {
                const uint64_t row = static_cast<uint64_t>(s) * nq + q;
                if (head[s] >= sh[row]) continue;
                const double d = sd[row * k + head[s]];
                const uint64_t id = sid[row * k + head[s]];
                if (best < 0 || d < bd || (d == bd && id < bi)) {
                    best = s;
                    bd = d;
                    bi = id;
                }
            }
            if (best < 0) break;
            od[q * k + out] = bd;
            oid[q * k + out] = bi;
            head[best]++;
        }
        oh[q] = out;
    }
}

}  // namespace

void run_query_batch(const QueryPlan& P, QueryScratch& X, int device, cudaStream_t s,
                     cudaStream_t alloc_s) {
    const int sms = sm_count(device);
    const size_t smem = smem_bytes(P.K, P.NR, P.d);
    if (smem > 220 * 1024) throw InvalidArgument("ck_ann: query dimension too large for the staging buffer");
    DETLSH_CUDA(cudaFuncSetAttribute(query_fast_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    DETLSH_CUDA(cudaFuncSetAttribute(query_slow_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    // persistent scratch lives on the index's own stream (it outlives any
    // caller stream); make it visible to `s` before use
    auto grow_scratch = [&](auto& buf, size_t count) {
        if (buf.size() >= count) return;
        {
            StreamScope sc(alloc_s);
            buf.alloc(count);
        }
        DETLSH_CUDA(cudaStreamSynchronize(alloc_s));
    };
    grow_scratch(X.counters, 4);
    grow_scratch(X.slow_list, P.nq);
    DETLSH_CUDA(cudaMemsetAsync(X.counters.get(), 0, 16, s));
    const size_t items = 3 * static_cast<size_t>(P.max_leaves) * sizeof(LeafItem);
    uint32_t slow_count = 0;
    const uint32_t* slow_list = X.slow_list.get();
    if (P.k <= kFastMaxK) {
        const size_t fast_bytes = (items + 4 * static_cast<size_t>(P.max_leaves) + 4 * P.budget + 255) / 256 * 256;
        const size_t slots = std::min<size_t>(P.nq, static_cast<size_t>(sms) * 2);
        grow_scratch(X.fast, slots * fast_bytes);
        ProfScope ps("query_fast", s);
        query_fast_kernel<<<static_cast<unsigned>(slots), kQueryThreads, smem, s>>>(
            P, X.fast.get(), fast_bytes, X.slow_list.get(), X.counters.get());
        DETLSH_LAUNCH_CHECK();
        DETLSH_CUDA(cudaMemcpyAsync(&slow_count, X.counters.get(), 4, cudaMemcpyDeviceToHost, s));
        DETLSH_CUDA(cudaStreamSynchronize(s));
    } else {
        slow_count = static_cast<uint32_t>(P.nq);
        slow_list = nullptr;  // every query takes the general path
    }
    if (slow_count == 0) return;
    const size_t slow_bytes = (items + 12 * P.budget + ((P.n + 31) / 32) * 4 + 255) / 256 * 256;
    const size_t slots = std::min<size_t>(slow_count, static_cast<size_t>(sms));
    if (X.slow_slots < slots || X.slow.size() < slots * slow_bytes) {
        X.slow.release();
        grow_scratch(X.slow, slots * slow_bytes);
        DETLSH_CUDA(cudaMemsetAsync(X.slow.get(), 0, slots * slow_bytes, s));
        X.slow_slots = slots;
    }
    ProfScope ps("query_slow", s);
    query_slow_kernel<<<static_cast<unsigned>(slots), kQueryThreads, smem, s>>>(
        P, slow_list, slow_count, X.slow.get(), slow_bytes);
    DETLSH_LAUNCH_CHECK();
}

void launch_merge_topk(const double* sd, const uint64_t* sid, const int32_t* sh, int shards,
                       uint64_t nq, int k, double* od, uint64_t* oid, int32_t* oh, cudaStream_t s) {
    if (shards > 16) throw InvalidArgument("merge_topk: at most 16 shards");
    const unsigned grid = static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>((nq + 127) / 128, 65535)));
    merge_topk_kernel<<<grid, 128, 0, s>>>(sd, sid, sh, shards, nq, k, od, oid, oh);
    DETLSH_LAUNCH_CHECK();
}

}  // namespace detlsh_b200
