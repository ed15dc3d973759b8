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
//
// Exact verification, two data paths:
//   * fp32 rows: sequential fp64 sum of (q_t - x_t)^2, one thread per row;
//   * u8 rows (dataset and query integral in [0,255], detected at build /
//     per query): int32 sum of squared byte differences (vabsdiffu4 + dp4a),
//     rows stored in tree-0 leaf order so a leaf's candidates are contiguous.
//     Every partial sum of the reference's double accumulation is then an
//     exact integer < 2^53, so sqrt(double(int sum)) is bit-identical.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "primitives.cuh"
#include "query.cuh"

namespace detlsh_b200 {

namespace {

constexpr int kBatch = 1024;                    // candidates scored per block step
constexpr int kTopCap = 2048;                   // staged (key, pos) entries
constexpr int kBins = 1024;                     // mindist histogram bins (fast-path cut)
constexpr int kFine = kBins * 32;               // approximate round: fine bins kept per leaf
constexpr uint32_t kTcMinBudget = 8192;         // tensor-core hand-off from this budget on
constexpr int kMergeMaxShards = 1024;           // merge_topk: shards per call
constexpr uint32_t kTauRows = 512;              // min rows scored exactly to set tau^2
// max rows scored for tau^2: the nearest leaves beat a uniform sample by far
// at large budgets (C5, budget 1e7: 131072 rows leave 857 survivors at the
// median and 2574 at most against the 4096 staged; the uniform estimate asks
// for 488 K rows, 4x the plan time).  Overflowing queries take the gather path.
constexpr uint64_t kTauRowsMax = 1u << 17;
static_assert(kFastMaxK == kTopCap - kBatch, "fast-path k bound");

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

// Shared memory: phase A (leaf scan) needs the penalty table, phase C (top-k)
// the staging buffers; they share one region.
struct Smem {
    double* sq;                // [K][NR+1]                       (phase A)
    float* tlo;                // [K][NR] fast path: fp32 penalty if the box starts at region r
    float* thi;                // [K][NR] fast path: fp32 penalty if the box ends at region r
    uint64_t* th;              // [kTopCap] top-k key hi           (phase C)
    uint32_t* tl;              // [kTopCap] top-k key lo (position)
    uint64_t* bh;              // [kBatch] batch key hi
    uint32_t* bl;              // [kBatch] batch key lo
    unsigned long long* hist;  // [256]
    uint32_t* bins;            // [kBins] leaf-weight histogram over mindist / radius
    unsigned long long* u64s;  // scalars
    uint32_t* u32s;
    int* lbv;                  // [K]  #{b : row[b] <  v}
    int* ubv;                  // [K]  #{b : row[b] <= v}
    float* qp;                 // [K]
    float* qv;                 // [d]
    uint8_t* q8;               // [row_u8]
};

struct Carver {
    uint8_t* base;
    size_t off = 0;
    __device__ uint8_t* take(size_t bytes, size_t align = 16) {
        off = (off + align - 1) / align * align;
        uint8_t* p = base + off;
        off += bytes;
        return p;
    }
};

__host__ __device__ inline size_t union_bytes(int K, int NR) {
    const size_t a = sizeof(double) * K * (NR + 1);
    const size_t c = (8 + 4) * static_cast<size_t>(kTopCap) + (8 + 4) * static_cast<size_t>(kBatch) + 64;
    return (a > c ? a : c + 0) + 64;
}

__device__ __forceinline__ Smem carve(uint8_t* base, int K, int NR, int d, int row_u8) {
    Carver c{base};
    Smem s;
    uint8_t* u = c.take(union_bytes(K, NR));
    s.sq = reinterpret_cast<double*>(u);
    s.tlo = reinterpret_cast<float*>(u);
    s.thi = s.tlo + static_cast<size_t>(K) * NR;
    s.th = reinterpret_cast<uint64_t*>(u);
    s.bh = s.th + kTopCap;
    s.tl = reinterpret_cast<uint32_t*>(s.bh + kBatch);
    s.bl = s.tl + kTopCap;
    s.hist = reinterpret_cast<unsigned long long*>(c.take(8 * 256));
    s.bins = reinterpret_cast<uint32_t*>(c.take(4 * kBins));
    s.u64s = reinterpret_cast<unsigned long long*>(c.take(8 * 16));
    s.u32s = reinterpret_cast<uint32_t*>(c.take(4 * 16));
    s.lbv = reinterpret_cast<int*>(c.take(4 * kMaxK));
    s.ubv = reinterpret_cast<int*>(c.take(4 * kMaxK));
    s.qp = reinterpret_cast<float*>(c.take(4 * kMaxK));
    s.qv = reinterpret_cast<float*>(c.take(4 * static_cast<size_t>(d)));
    s.q8 = c.take(static_cast<size_t>(row_u8) + 16);
    return s;
}

size_t smem_bytes(int K, int NR, int d, int row_u8) {
    size_t off = 0;
    auto take = [&](size_t bytes) {
        off = (off + 15) / 16 * 16;
        off += bytes;
    };
    take(union_bytes(K, NR));
    take(8 * 256);
    take(4 * kBins);
    take(8 * 16);
    take(4 * 16);
    take(4 * kMaxK);
    take(4 * kMaxK);
    take(4 * kMaxK);
    take(4 * static_cast<size_t>(d));
    take(static_cast<size_t>(row_u8) + 16);
    return off + 16;
}

// lbv[j] = #{b : row_j[b] < v_j}, ubv[j] = #{b : row_j[b] <= v_j}: one warp per
// dimension, lane-strided counts and a warp reduction (no contended atomics).
__device__ void count_below(const float* tb, int K, int W, const Smem& S) {
    const int lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    for (int j = threadIdx.x >> 5; j < K; j += nw) {
        const float v = S.qp[j];
        uint32_t lb = 0, ub = 0;
        for (int b = lane; b < W; b += 32) {
            const float row = tb[j * W + b];
            lb += row < v;
            ub += row <= v;
        }
        lb = __reduce_add_sync(0xffffffffu, lb);
        ub = __reduce_add_sync(0xffffffffu, ub);
        if (lane == 0) {
            S.lbv[j] = static_cast<int>(lb);
            S.ubv[j] = static_cast<int>(ub);
        }
    }
    __syncthreads();
}

// Per (query, tree): squared edge penalties in fp64, exactly as mindist
// (de_tree.cpp:169-184) forms them: pen = double(edge) - double(v), pen*pen.
__device__ void build_sq(const QueryPlan& P, int tree, const Smem& S) {
    const int W = P.NR + 1;
    const float* tb = P.table + static_cast<size_t>(tree) * P.K * W;
    count_below(tb, P.K, W, S);
    for (int i = threadIdx.x; i < P.K * W; i += blockDim.x) {
        const int j = i / W;
        const double D = __dsub_rn(static_cast<double>(tb[i]), static_cast<double>(S.qp[j]));
        S.sq[i] = __dmul_rn(D, D);
    }
    __syncthreads();
}

// Fast path, per (query, tree 0): the penalty of a box edge split by side, so
// the scan needs no per-dimension branches: for a box [lo, hi] in dim j the
// reference's penalty (de_tree.cpp:169-184) is tlo[j][lo] + thi[j][hi], at
// most one of them non-zero:
//   tlo[j][r] = pen(j, r)     if r > 0      and r >= ubv_j  (query below the box)
//   thi[j][r] = pen(j, r + 1) if r < NR - 1 and r + 1 < lbv_j (query above it)
// with pen(j, e) = (double(row_j[e]) - double(v_j))^2 rounded to fp32.
__device__ void build_pen_tables(const QueryPlan& P, const Smem& S) {
    const int W = P.NR + 1, NR = P.NR;
    const float* tb = P.table;
    count_below(tb, P.K, W, S);
    for (int i = threadIdx.x; i < P.K * NR; i += blockDim.x) {
        const int j = i / NR, r = i % NR;
        const double v = static_cast<double>(S.qp[j]);
        float lo = 0.0f, hi = 0.0f;
        if (r > 0 && r >= S.ubv[j]) {
            const double D = __dsub_rn(static_cast<double>(tb[j * W + r]), v);
            lo = __double2float_rn(__dmul_rn(D, D));
        }
        if (r < NR - 1 && r + 1 < S.lbv[j]) {
            const double D = __dsub_rn(static_cast<double>(tb[j * W + r + 1]), v);
            hi = __double2float_rn(__dmul_rn(D, D));
        }
        S.tlo[i] = lo;
        S.thi[i] = hi;
    }
    __syncthreads();
}

// Per query, after build_pen_tables: the penalty of each half of each dim
// (hp[j][b] for the box covering regions [b NR/2, (b+1) NR/2 - 1], the root
// split) and their fp32 sums over dims 8c..8c+7 for every 8-bit half pattern
// (tcd[c][x]); they live in the union right after tlo/thi (K <= 16).
__device__ void build_half_tables(const QueryPlan& P, const Smem& S) {
    const int NR = P.NR, H = NR / 2;
    float* hp = S.tlo + 2 * P.K * NR;
    float* tcd = hp + 2 * kMaxK;
    for (int i = threadIdx.x; i < 2 * P.K; i += blockDim.x) {
        const int j = i >> 1, b = i & 1;
        hp[i] = __fadd_rn(S.tlo[j * NR + b * H], S.thi[j * NR + b * H + H - 1]);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 512; i += blockDim.x) {
        const int c = i >> 8, x = i & 255;
        float sum = 0.0f;
        for (int t = 0; t < 8; ++t) {
            const int j = 8 * c + t;
            if (j < P.K) sum = __fadd_rn(sum, hp[2 * j + ((x >> t) & 1)]);
        }
        tcd[i] = sum;
    }
    __syncthreads();
}

__device__ __forceinline__ double leaf_mindist(const QueryPlan& P, const QTree& T, uint32_t li,
                                               const Smem& S) {
    // box: per dim j, bytes (lo region, hi region) at 2j, 2j+1; kept in
    // registers (byte extraction by shifts, fully unrolled)
    const uint4* box = reinterpret_cast<const uint4*>(T.leaf_box + static_cast<size_t>(li) * 64);
    uint32_t w[12];
    {
        const uint4 a = __ldg(box), b = __ldg(box + 1);
        w[0] = a.x; w[1] = a.y; w[2] = a.z; w[3] = a.w;
        w[4] = b.x; w[5] = b.y; w[6] = b.z; w[7] = b.w;
        if (P.K > 16) {
            const uint4 c = __ldg(box + 2);
            w[8] = c.x; w[9] = c.y; w[10] = c.z; w[11] = c.w;
        } else {
            w[8] = w[9] = w[10] = w[11] = 0;
        }
    }
    const int W = P.NR + 1;
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < kMaxK; ++j) {
        if (j < P.K) {
            const uint32_t half = w[j >> 1] >> ((j & 1) * 16);
            const int lo = half & 0xff, hi = (half >> 8) & 0xff;
            double pen_sq = 0.0;
            if (lo > 0 && lo >= S.ubv[j]) pen_sq = S.sq[j * W + lo];
            else if (hi < P.NR - 1 && hi + 1 < S.lbv[j]) pen_sq = S.sq[j * W + hi + 1];
            acc = __dadd_rn(acc, pen_sq);
        }
    }
    return __dsqrt_rn(acc);
}

// A leaf's 64-byte (lo, hi) region box as eight words.
__device__ __forceinline__ void box_words(const QTree& T, uint32_t li, uint32_t (&w)[8]) {
    const uint4* box = reinterpret_cast<const uint4*>(T.leaf_box + static_cast<size_t>(li) * 64);
    const uint4 a = __ldg(box), b = __ldg(box + 1);
    w[0] = a.x; w[1] = a.y; w[2] = a.z; w[3] = a.w;
    w[4] = b.x; w[5] = b.y; w[6] = b.z; w[7] = b.w;
}

// Exact round: histogram bin of an exact mindist (0xffff: outside the radius).
__device__ __forceinline__ uint32_t exact_bin(double md, double radius, double scale) {
    if (!(md <= radius)) return 0xffffu;
    const double fb = __dmul_rn(md, scale);
    return fb >= static_cast<double>(kBins - 1) ? kBins - 1 : static_cast<uint32_t>(fb);
}

// Approximate round: the reference's penalties rounded to fp32 (tlo/thi, at
// most one non-zero per dimension, so tlo + thi is exact), summed in fp32 in
// dimension order, no square root.  |result - exact squared mindist| <=
// (2K + 1) * 2^-24 * exact (+ denormal rounding), which the caller's bound
// rel = (K + 2) * 2^-22 covers.
__device__ __forceinline__ void leaf_a2_k16_f32(const QueryPlan& P, const QTree& T, uint32_t li0, uint32_t li1,
                                                const Smem& S, float& a0, float& a1) {
    uint32_t w0[8], w1[8];
    box_words(T, li0, w0);
    box_words(T, li1, w1);
    const int NR = P.NR;
    float s0 = 0.0f, s1 = 0.0f;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        if (j < P.K) {
            // byte offsets of lo / hi entries: one shift + one mask each
            const char* tl = reinterpret_cast<const char*>(S.tlo + j * NR);
            const char* th = reinterpret_cast<const char*>(S.thi + j * NR);
            const int sl = (j & 1) * 16;
            const uint32_t l0 = (w0[j >> 1] >> sl << 2) & 0x3fcu, u0 = (w0[j >> 1] >> (sl + 6)) & 0x3fcu;
            const uint32_t l1 = (w1[j >> 1] >> sl << 2) & 0x3fcu, u1 = (w1[j >> 1] >> (sl + 6)) & 0x3fcu;
            s0 = __fadd_rn(s0, __fadd_rn(*reinterpret_cast<const float*>(tl + l0), *reinterpret_cast<const float*>(th + u0)));
            s1 = __fadd_rn(s1, __fadd_rn(*reinterpret_cast<const float*>(tl + l1), *reinterpret_cast<const float*>(th + u1)));
        }
    }
    a0 = s0;
    a1 = s1;
}

// Exact original-space squared distance (dataset.hpp:23-30): sequential fp64.
__device__ __forceinline__ double l2sq_exact(const float* __restrict__ q, const float* __restrict__ x,
                                             int d) {
    double acc = 0.0;
    if ((d & 3) == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0) {
        const float4* x4 = reinterpret_cast<const float4*>(x);
#pragma unroll 4
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
    return acc;
}

__device__ __forceinline__ double l2_exact(const float* q, const float* x, int d) {
    return __dsqrt_rn(l2sq_exact(q, x, d));
}

// The same distance when the row and the query hold integers in [0, 255]
// (a u8 index and a u8-exact query): every partial sum of l2sq_exact is then
// an integer below 2^53, so integer arithmetic in any order gives the same
// double.  No dependent fp64 chain: ~10x the rows per SM.
__device__ __forceinline__ double l2_exact_u8(const float* __restrict__ q, const float* __restrict__ x, int d) {
    unsigned long long acc = 0;
    if ((d & 3) == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0) {
        const float4* x4 = reinterpret_cast<const float4*>(x);
#pragma unroll 8
        for (int t = 0; t < d / 4; ++t) {
            const float4 xv = __ldg(x4 + t);
            const float* qq = q + 4 * t;
            const int a = static_cast<int>(qq[0]) - static_cast<int>(xv.x);
            const int b = static_cast<int>(qq[1]) - static_cast<int>(xv.y);
            const int c = static_cast<int>(qq[2]) - static_cast<int>(xv.z);
            const int e = static_cast<int>(qq[3]) - static_cast<int>(xv.w);
            acc += static_cast<unsigned>(a * a + b * b + c * c + e * e);
        }
    } else {
        for (int t = 0; t < d; ++t) {
            const int a = static_cast<int>(q[t]) - static_cast<int>(__ldg(x + t));
            acc += static_cast<unsigned>(a * a);
        }
    }
    return __dsqrt_rn(static_cast<double>(acc));
}

// Warp-aggregated append of `item` to list (counter in smem).
__device__ __forceinline__ void warp_append(bool ok, const LeafItem& it, LeafItem* list,
                                            uint32_t* counter, uint32_t cap = 0xffffffffu) {
    const uint32_t m = __ballot_sync(0xffffffffu, ok);
    if (!m) return;
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(m) - 1;
    uint32_t base = 0;
    if (lane == leader) base = atomicAdd(counter, static_cast<uint32_t>(__popc(m)));
    base = __shfl_sync(0xffffffffu, base, leader);
    const uint32_t at = base + __popc(m & ((1u << lane) - 1u));
    if (ok && at < cap) list[at] = it;
}

// Scan every leaf of tree `tree`, appending those with mindist <= radius.
// weight: leaf size, or (bitmap != null) the entries not yet in S.
// Each appended item also records its histogram bin floor(md * kBins / radius)
// (monotone in md) in `pad`, and its weight is added to S.bins.
__device__ void scan_leaves(const QueryPlan& P, int tree, double radius, const Smem& S,
                            LeafItem* A, const uint32_t* bitmap, uint32_t& nA, uint64_t& W, LeafItem* tmp) {
    const QTree T = P.trees[tree];
    if (threadIdx.x == 0) {
        S.u32s[0] = 0;
        S.u64s[0] = 0;
    }
    for (int i = threadIdx.x; i < kBins; i += blockDim.x) S.bins[i] = 0;
    const double scale = radius > 0.0 ? static_cast<double>(kBins) / radius : 0.0;
    __syncthreads();
    unsigned long long wsum = 0;
    const uint32_t nl = T.num_leaves;
    auto add_weight = [&](const LeafItem& it) {
        wsum += it.w;
        atomicAdd(&S.bins[it.pad], it.w);
    };
    // pass A: every leaf's exact mindist; leaves within the radius are listed
    // (weight = leaf size; with a bitmap, corrected in pass B)
    for (uint32_t base = 0; base < nl; base += blockDim.x) {
        const uint32_t li = base + threadIdx.x;
        bool ok = false;
        LeafItem it;
        if (li < nl) {
            const double md = leaf_mindist(P, T, li, S);
            if (md <= radius) {
                const uint32_t w = T.leaf_count[li];
                if (w > 0) {
                    ok = true;
                    it.mdb = static_cast<uint64_t>(__double_as_longlong(md));
                    it.id = T.leaf_node[li];
                    it.w = w;
                    it.li = li;
                    const double fb = __dmul_rn(md, scale);
                    it.pad = fb >= static_cast<double>(kBins - 1) ? kBins - 1 : static_cast<uint32_t>(fb);
                    if (!bitmap) add_weight(it);
                }
            }
        }
        warp_append(ok, it, bitmap ? tmp : A, &S.u32s[0]);
    }
    if (bitmap) {
        // pass B: each listed leaf's entries not yet in S, one leaf per thread
        // with every lane busy and eight rows' loads in flight.  (C5: ~4x10^7
        // random bitmap reads per query and tree, bound by one SM's L1 request
        // rate: ~75% of the general path's scan time.)
        __syncthreads();
        const uint32_t n0 = S.u32s[0];
        __syncthreads();
        if (threadIdx.x == 0) S.u32s[0] = 0;
        __syncthreads();
        for (uint32_t base = 0; base < n0; base += blockDim.x) {
            const uint32_t i = base + threadIdx.x;
            bool ok = false;
            LeafItem it;
            if (i < n0) {
                it = tmp[i];
                const uint32_t b0 = T.leaf_begin[it.li], w = it.w;
                uint32_t nw = 0;
                for (uint32_t e0 = 0; e0 < w; e0 += 8) {
                    uint32_t pos[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) pos[u] = e0 + u < w ? __ldg(T.perm + b0 + e0 + u) : 0xffffffffu;
#pragma unroll
                    for (int u = 0; u < 8; ++u)
                        if (pos[u] != 0xffffffffu) nw += ((bitmap[pos[u] >> 5] >> (pos[u] & 31)) & 1u) ? 0u : 1u;
                }
                it.w = nw;
                ok = nw > 0;
                if (ok) add_weight(it);
            }
            warp_append(ok, it, A, &S.u32s[0]);
        }
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
            if (excl < need && need <= incl) {
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

// weighted_select for n <= blockDim.x items: every thread ranks its item by
// summing the weights of the smaller keys (n^2 / blockDim compares, no radix
// passes).  The item list is read through L1 (every thread reads the same
// entries in the same order).
__device__ void small_weighted_select(const LeafItem* A, uint32_t n, uint64_t need, const Smem& S,
                                      uint64_t& kmdb, uint32_t& kid, uint64_t& take_cut) {
    const uint32_t i = threadIdx.x;
    if (i < n) {
        const LeafItem me = A[i];
        uint64_t before = 0;
        for (uint32_t j = 0; j < n; ++j) {
            const uint64_t mj = __ldg(&A[j].mdb);
            const uint32_t ij = __ldg(&A[j].id), wj = __ldg(&A[j].w);
            if (key_less(mj, ij, me.mdb, me.id)) before += wj;
        }
        if (before < need && need <= before + me.w) {
            S.u64s[4] = me.mdb;
            S.u32s[13] = me.id;
            S.u64s[5] = need - before;
        }
    }
    __syncthreads();
    kmdb = S.u64s[4];
    kid = S.u32s[13];
    take_cut = S.u64s[5];
    __syncthreads();
}

// ---- block top-k over (hi, lo) keys, ascending --------------------------------
// hi = distance bits (non-negative double) or exact integer squared distance,
// lo = dataset position: lexicographic order == the reference's (dist, pos).
__device__ void topk_sort(const Smem& S) {
    const uint32_t cnt = S.u32s[4];
    for (uint32_t i = threadIdx.x + cnt; i < kTopCap; i += blockDim.x) {
        S.th[i] = ~0ULL;
        S.tl[i] = 0xffffffffu;
    }
    __syncthreads();
    for (int size = 2; size <= kTopCap; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = threadIdx.x; i < kTopCap / 2; i += blockDim.x) {
                const int lo = 2 * i - (i & (stride - 1));
                const int hi = lo + stride;
                const bool asc = (lo & size) == 0;
                const uint64_t a = S.th[lo], b = S.th[hi];
                const uint32_t al = S.tl[lo], bl = S.tl[hi];
                if (key_less(b, bl, a, al) == asc) {
                    S.th[lo] = b;
                    S.th[hi] = a;
                    S.tl[lo] = bl;
                    S.tl[hi] = al;
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
        S.u32s[6] = 0;  // tau lo
        S.u64s[2] = 0;  // tau hi
    }
    __syncthreads();
}

// Stage the batch keys [0, nb) that beat the current k-th key; compact when
// the staging area would overflow.  Called by all threads after the batch is
// written (and synchronised).
// `row_to_pos` non-null: bl holds row indices that map to dataset positions
// through it; the lookup is only done for keys that can still enter.
__device__ void topk_absorb(const Smem& S, uint32_t nb, int k, const uint32_t* row_to_pos) {
    const bool full = S.u32s[5] != 0;
    const uint64_t th = S.u64s[2];
    const uint32_t tl = S.u32s[6];
    const int lane = threadIdx.x & 31;
    for (uint32_t base = 0; base < nb; base += blockDim.x) {
        const uint32_t i = base + threadIdx.x;
        bool take = false;
        uint64_t h = 0;
        uint32_t l = 0;
        if (i < nb) {
            h = S.bh[i];
            l = S.bl[i];
            if (row_to_pos) {
                if (!full || h <= th) {
                    l = __ldg(row_to_pos + l);
                    take = !full || key_less(h, l, th, tl);
                }
            } else {
                take = !full || key_less(h, l, th, tl);
            }
        }
        const uint32_t m = __ballot_sync(0xffffffffu, take);
        if (m) {
            const int leader = __ffs(m) - 1;
            uint32_t slot0 = 0;
            if (lane == leader) slot0 = atomicAdd(&S.u32s[4], static_cast<uint32_t>(__popc(m)));
            slot0 = __shfl_sync(0xffffffffu, slot0, leader);
            if (take) {
                const uint32_t slot = slot0 + __popc(m & ((1u << lane) - 1u));
                S.th[slot] = h;
                S.tl[slot] = l;
            }
        }
    }
    __syncthreads();
    if (S.u32s[4] > static_cast<uint32_t>(kTopCap - kBatch)) {
        topk_sort(S);
        if (threadIdx.x == 0) {
            const uint32_t c = min(S.u32s[4], static_cast<uint32_t>(k));
            S.u32s[4] = c;
            if (c >= static_cast<uint32_t>(k)) {
                S.u32s[5] = 1;
                S.u64s[2] = S.th[k - 1];
                S.u32s[6] = S.tl[k - 1];
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

// OR rows [a0, a1) into a row bitmap (global atomics: neighbouring leaves share words)
__device__ __forceinline__ void or_row_range(uint32_t* bm, uint32_t a0, uint32_t a1) {
    for (uint32_t w = a0 >> 5; a0 < a1 && w <= (a1 - 1) >> 5; ++w) {
        const uint32_t lo = max(a0, w << 5), hi = min(a1, (w << 5) + 32);
        const uint32_t nbits = hi - lo;
        atomicOr(bm + w, (nbits == 32 ? 0xffffffffu : ((1u << nbits) - 1u)) << (lo & 31));
    }
}

__device__ __forceinline__ uint32_t sqdiff4(uint32_t a, uint32_t b, uint32_t acc) {
    const uint32_t d = __vabsdiffu4(a, b);
    return __dp4a(d, d, acc);
}

// ---------------------------------------------------------------------------
// Fast path: tree 0, round 0 fills the budget.
// ---------------------------------------------------------------------------
struct FastSlot {
    LeafItem *A, *B, *C;  // bin-b* items and the select's ping-pong buffers
    uint32_t* full;       // leaves taken whole (leaf indices)
    uint32_t* tau;        // whole leaves of the bins <= b_tau (tensor-core hand-off)
    uint16_t* bin16;      // per-leaf histogram bin (0xffff: outside the radius), 16-B aligned
    uint32_t* cand;       // candidate rows as tree-0 permutation indices
};

// The per-CTA leaf lists are capped (bin-b* items and the select's ping-pong
// buffers: a few hundred per query; whole leaves; tau leaves) so the slots of a
// 1e8-point index (6.7 M leaves per tree) stay small enough for many CTAs.  A
// query that overflows one takes the general path.
constexpr uint32_t kItemCap = 1u << 20;   // bin-b* items (C5: up to ~10^5 in the crossing bins)
constexpr uint32_t kFullCap = 0xffffffffu; // whole leaves: not capped (up to budget leaves at C5)
constexpr uint32_t kTauCap = 1u << 20;    // tau leaves (<= tau rows: C5 ~33 K per query)
__host__ __device__ __forceinline__ uint32_t item_cap(uint32_t maxl) { return maxl < kItemCap ? maxl : kItemCap; }
__host__ __device__ __forceinline__ uint32_t full_cap(uint32_t maxl) { return maxl < kFullCap ? maxl : kFullCap; }
__host__ __device__ __forceinline__ uint32_t tau_cap(uint32_t maxl) { return maxl < kTauCap ? maxl : kTauCap; }

__device__ __forceinline__ FastSlot fast_slot(uint8_t* base, size_t slot_bytes, uint32_t maxl,
                                              uint64_t budget) {
    uint8_t* p = base + static_cast<size_t>(blockIdx.x) * slot_bytes;
    const uint32_t ic = item_cap(maxl);
    FastSlot f;
    f.A = reinterpret_cast<LeafItem*>(p);
    f.B = f.A + ic;
    f.C = f.B + ic;
    f.full = reinterpret_cast<uint32_t*>(f.C + ic);
    f.tau = f.full + full_cap(maxl);
    f.cand = f.tau + tau_cap(maxl);
    f.bin16 = reinterpret_cast<uint16_t*>((reinterpret_cast<uintptr_t>(f.cand + budget) + 15) & ~uintptr_t(15));
    return f;
}

// Device-memory ceilings of the per-CTA query scratch (the fast path's slots
// hold 4 B per budget candidate; the general path's an n-bit bitmap plus 12 B
// per candidate); DETLSH_FAST_SCRATCH_MB / DETLSH_SLOW_SCRATCH_MB override.
size_t scratch_limit_env(const char* name, size_t dflt_mb) {
    const char* e = std::getenv(name);
    const size_t mb = e ? static_cast<size_t>(std::max(1L, std::atol(e))) : dflt_mb;
    return mb << 20;
}
// Memory the query scratch may take: the free device memory plus what the
// stream-ordered pool holds but does not use (freed build temporaries).
size_t device_memory_available(int device) {
    size_t fr = 0, tot = 0;
    if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t reserved = 0, used = 0;
        if (cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved) == cudaSuccess &&
            cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used) == cudaSuccess && reserved > used)
            fr += static_cast<size_t>(reserved - used);
    }
    cudaGetLastError();
    return fr;
}
// `avail`: the available memory plus the query scratch already held (it is
// reused).  Fast path: 8 GB, or up to a third of it for large indexes (C5's
// slots are ~150 MB each: more of them keep more SMs busy).
size_t fast_scratch_limit(size_t avail) {
    if (std::getenv("DETLSH_FAST_SCRATCH_MB")) return scratch_limit_env("DETLSH_FAST_SCRATCH_MB", 8192);
    return std::max<size_t>(size_t(8192) << 20, std::min<size_t>(size_t(32768) << 20, avail / 3));
}
// general path: 2 GB, or up to a fifth for large indexes (C5: ~210 MB per
// slot; 2 GB kept it to 9 CTAs)
size_t slow_scratch_limit(size_t avail) {
    if (std::getenv("DETLSH_SLOW_SCRATCH_MB")) return scratch_limit_env("DETLSH_SLOW_SCRATCH_MB", 2048);
    return std::max<size_t>(size_t(2048) << 20, std::min<size_t>(size_t(24576) << 20, avail / 5));
}

size_t fast_slot_bytes(uint32_t maxl, uint64_t budget) {
    const size_t b = 3 * static_cast<size_t>(item_cap(maxl)) * sizeof(LeafItem) +
                     4 * (static_cast<size_t>(full_cap(maxl)) + tau_cap(maxl)) + 4 * budget +
                     2 * (static_cast<size_t>(maxl) + 8) + 16;
    return (b + 255) / 256 * 256;
}

__device__ void load_query_proj(const QueryPlan& P, uint64_t q, int tree, const Smem& S) {
    for (int j = threadIdx.x; j < P.K; j += blockDim.x)
        S.qp[j] = P.qproj[(static_cast<uint64_t>(tree) * P.nq + q) * P.K + j];
    __syncthreads();
}

// Loads the query vector (fp32, and u8 when the index has u8 rows); returns
// whether the u8 path is exact for this query (all values integral in [0,255]).
__device__ bool load_query_vec(const QueryPlan& P, uint64_t q, const Smem& S) {
    if (threadIdx.x == 0) S.u32s[9] = 1;
    __syncthreads();
    bool ok = true;
    for (int t = threadIdx.x; t < P.d; t += blockDim.x) {
        const float v = P.q[q * P.d + t];
        S.qv[t] = v;
        if (P.data_u8) {
            const bool integral = v >= 0.0f && v <= 255.0f && v == floorf(v);
            ok = ok && integral;
            S.q8[t] = integral ? static_cast<uint8_t>(v) : 0;
        }
    }
    if (P.data_u8)
        for (int t = P.d + threadIdx.x; t < P.row_u8; t += blockDim.x) S.q8[t] = 0;
    if (!ok) S.u32s[9] = 0;
    __syncthreads();
    const bool u8 = P.data_u8 != nullptr && S.u32s[9] != 0;
    __syncthreads();
    return u8;
}

// Scores candidates [base, base+nb) into the batch keys.
__device__ void score_batch(const QueryPlan& P, const FastSlot& F, const Smem& S, uint32_t base,
                            uint32_t nb, bool u8) {
    if (u8) {
        // LPR lanes per row, 16 B per lane-chunk; int32 exact squared distance.
        // Candidate rows are staged in smem first, then every lane keeps kU
        // row loads in flight.  bl holds the ROW index (tree-0 permutation
        // index); topk_absorb maps it to the dataset position only for the
        // rare keys that can enter the top-k.
        constexpr int kU = 8;
        for (uint32_t i = threadIdx.x; i < nb; i += blockDim.x) S.bl[i] = F.cand[base + i];
        __syncthreads();
        const int lpr = P.u8_lpr;
        const int rpw = 32 / lpr;
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        const int sub = lane & (lpr - 1), rsub = lane / lpr;
        const int chunks = P.row_u8 / 16;
        const uint4* q4 = reinterpret_cast<const uint4*>(S.q8);
        const uint32_t step = (blockDim.x / 32) * rpw * kU;
        for (uint32_t r0 = warp * rpw * kU; r0 < nb; r0 += step) {
            uint32_t acc[kU];
#pragma unroll
            for (int u = 0; u < kU; ++u) acc[u] = 0;
            for (int ch0 = 0; ch0 < chunks; ch0 += lpr) {
                const int ch = ch0 + sub;
                uint4 x[kU];
#pragma unroll
                for (int u = 0; u < kU; ++u) {
                    const uint32_t r = r0 + u * rpw + rsub;
                    x[u] = make_uint4(0, 0, 0, 0);
                    if (r < nb && ch < chunks)
                        x[u] = __ldg(reinterpret_cast<const uint4*>(P.data_u8 + static_cast<uint64_t>(S.bl[r]) * P.row_u8) + ch);
                }
                if (ch < chunks) {
                    const uint4 qq = q4[ch];
#pragma unroll
                    for (int u = 0; u < kU; ++u) {
                        acc[u] = sqdiff4(qq.x, x[u].x, acc[u]);
                        acc[u] = sqdiff4(qq.y, x[u].y, acc[u]);
                        acc[u] = sqdiff4(qq.z, x[u].z, acc[u]);
                        acc[u] = sqdiff4(qq.w, x[u].w, acc[u]);
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                for (int o = lpr >> 1; o; o >>= 1) acc[u] += __shfl_xor_sync(0xffffffffu, acc[u], o);
                const uint32_t r = r0 + u * rpw + rsub;
                if (sub == 0 && r < nb) S.bh[r] = acc[u];
            }
        }
    } else {
        // one thread per row, two rows in flight per thread (independent fp64 chains)
        for (uint32_t r = threadIdx.x; r < nb; r += 2 * blockDim.x) {
            const uint32_t r2 = r + blockDim.x;
            // leaf-ordered rows when the index keeps them (contiguous per leaf;
            // bl then holds the row and topk_absorb maps survivors to positions)
            const bool leaf = P.data_leaf != nullptr;
            const uint32_t c1 = F.cand[base + r];
            const bool two = r2 < nb;
            const uint32_t c2 = two ? F.cand[base + r2] : c1;
            const uint32_t p1 = leaf ? c1 : __ldg(P.perm0 + c1);
            const uint32_t p2 = leaf ? c2 : __ldg(P.perm0 + c2);
            const float* x1 = (leaf ? P.data_leaf : P.data) + static_cast<uint64_t>(p1) * P.d;
            const float* x2 = (leaf ? P.data_leaf : P.data) + static_cast<uint64_t>(p2) * P.d;
            double a1 = 0.0, a2 = 0.0;
            int t = 0;
            if ((P.d & 3) == 0) {
                // 32 floats of each row in flight (8 x 16-byte loads per row) before
                // the chain consumes them: one L1 miss per 128-byte line instead of
                // one per element (thread-private rows would otherwise thrash L1)
                for (; t + 32 <= P.d; t += 32) {
                    float4 v1[8], v2[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        v1[u] = __ldg(reinterpret_cast<const float4*>(x1 + t) + u);
                        v2[u] = __ldg(reinterpret_cast<const float4*>(x2 + t) + u);
                    }
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const float e1[4] = {v1[u].x, v1[u].y, v1[u].z, v1[u].w};
                        const float e2[4] = {v2[u].x, v2[u].y, v2[u].z, v2[u].w};
#pragma unroll
                        for (int w = 0; w < 4; ++w) {
                            const double qv = static_cast<double>(S.qv[t + 4 * u + w]);
                            const double d1 = __dsub_rn(qv, static_cast<double>(e1[w]));
                            const double d2 = __dsub_rn(qv, static_cast<double>(e2[w]));
                            a1 = __dadd_rn(a1, __dmul_rn(d1, d1));
                            a2 = __dadd_rn(a2, __dmul_rn(d2, d2));
                        }
                    }
                }
            }
            for (; t < P.d; ++t) {
                const double qv = static_cast<double>(S.qv[t]);
                const double d1 = __dsub_rn(qv, static_cast<double>(__ldg(x1 + t)));
                const double d2 = __dsub_rn(qv, static_cast<double>(__ldg(x2 + t)));
                a1 = __dadd_rn(a1, __dmul_rn(d1, d1));
                a2 = __dadd_rn(a2, __dmul_rn(d2, d2));
            }
            S.bh[r] = static_cast<uint64_t>(__double_as_longlong(__dsqrt_rn(a1)));
            S.bl[r] = p1;
            if (two) {
                S.bh[r2] = static_cast<uint64_t>(__double_as_longlong(__dsqrt_rn(a2)));
                S.bl[r2] = p2;
            }
        }
    }
}

// Writes the rows of whole leaves `list[0..n)` (tree-0 permutation indices,
// contiguous per leaf) to cand[0..): a block prefix over leaf sizes, then one
// warp per leaf.  Returns the number of rows (writes beyond `cap` dropped).
__device__ uint32_t emit_rows(const uint32_t* list, uint32_t n, const QTree& T0, uint32_t* cand,
                              uint32_t cap, const Smem& S) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) S.u32s[3] = 0;
    __syncthreads();
    uint32_t* st_dst = S.tl;  // the top-k staging area is free outside verification
    uint32_t* st_src = S.tl + blockDim.x;  // (3 x blockDim.x <= kTopCap)
    uint32_t* st_take = S.tl + 2 * blockDim.x;
    for (uint32_t base = 0; base < n; base += blockDim.x) {
        const uint32_t i = base + threadIdx.x;
        uint32_t take = 0, src = 0;
        if (i < n) {
            const uint32_t li = list[i];
            take = __ldg(T0.leaf_count + li);
            src = __ldg(T0.leaf_begin + li);
        }
        uint32_t incl = take;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        uint32_t* wt = reinterpret_cast<uint32_t*>(S.hist);
        if (lane == 31) wt[warp] = incl;
        __syncthreads();
        uint32_t wpre = 0, tot = 0;
        for (int w = 0; w < static_cast<int>(blockDim.x / 32); ++w) {
            if (w < warp) wpre += wt[w];
            tot += wt[w];
        }
        st_dst[threadIdx.x] = S.u32s[3] + wpre + incl - take;
        st_src[threadIdx.x] = src;
        st_take[threadIdx.x] = take;
        __syncthreads();
        for (int t = warp * 32; t < warp * 32 + 32; ++t) {
            const uint32_t d0 = st_dst[t], s0 = st_src[t], tk = st_take[t];
            for (uint32_t e = lane; e < tk && d0 + e < cap; e += 32) cand[d0 + e] = s0 + e;
        }
        __syncthreads();
        if (threadIdx.x == 0) S.u32s[3] += tot;
        __syncthreads();
    }
    const uint32_t total = S.u32s[3];
    __syncthreads();
    return total;
}

// Block-wide: the bin of hist[0..nbins) (nbins a multiple of blockDim.x) where
// the running count reaches `need` (>= 1, <= total); *before = count below it.
__device__ void select_count_bin(const uint32_t* hist, int nbins, uint32_t need, const Smem& S, uint32_t& bin,
                                 uint32_t& before) {
    const int per = nbins / blockDim.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t part = 0;
    for (int b = 0; b < per; ++b) part += hist[threadIdx.x * per + b];
    uint32_t incl = part;
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    uint32_t* wt = reinterpret_cast<uint32_t*>(S.hist);
    if (lane == 31) wt[warp] = incl;
    __syncthreads();
    uint32_t wpre = 0;
    for (int w = 0; w < warp; ++w) wpre += wt[w];
    incl += wpre;
    const uint32_t excl = incl - part;
    if (excl < need && need <= incl) {
        uint32_t cum = excl;
        int b = threadIdx.x * per;
        for (int e = 0; e < per; ++e, ++b) {
            const uint32_t c = hist[b];
            if (cum + c >= need) break;
            cum += c;
        }
        S.u32s[13] = static_cast<uint32_t>(b);
        S.u32s[14] = cum;
    }
    __syncthreads();
    bin = S.u32s[13];
    before = S.u32s[14];
    __syncthreads();
}

// Exact k-th smallest integer dist^2 over the u8 rows F.cand[0..nt) (tree-0
// row indices; overwritten with their dist^2): two counting passes over
// dist^2 >> s and its low s bits.  INT_MAX when nt < k.
__device__ int32_t kth_dist2(const QueryPlan& P, const FastSlot& F, const Smem& S, uint32_t nt, int k) {
    if (nt < static_cast<uint32_t>(k)) return 0x7fffffff;
    uint32_t* hist = reinterpret_cast<uint32_t*>(S.th);  // 4096 bins: top-k staging is idle here
    int sh = 0;
    while (((65025u * static_cast<uint32_t>(P.d)) >> sh) >= 4096u) ++sh;
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    for (uint32_t c0 = 0; c0 < nt; c0 += kBatch) {
        const uint32_t nb = min(static_cast<uint32_t>(kBatch), nt - c0);
        score_batch(P, F, S, c0, nb, true);
        __syncthreads();
        for (uint32_t r = threadIdx.x; r < nb; r += blockDim.x) {
            const uint32_t d2 = static_cast<uint32_t>(S.bh[r]);
            F.cand[c0 + r] = d2;
            atomicAdd(&hist[d2 >> sh], 1u);
        }
        __syncthreads();
    }
    // 12-bit digits from the top: the coarse level above, then as many finer
    // levels as the dist^2 range needs (d > 256 spans more than 24 bits)
    uint32_t cb, before;
    select_count_bin(hist, 4096, static_cast<uint32_t>(k), S, cb, before);
    uint32_t prefix = cb, need = static_cast<uint32_t>(k) - before;
    while (sh > 0) {
        const int nsh = sh > 12 ? sh - 12 : 0;   // the next digit: bits [nsh, sh)
        const int nb = 1 << (sh - nsh);
        for (int i = threadIdx.x; i < 4096; i += blockDim.x) hist[i] = 0;
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < nt; i += blockDim.x) {
            const uint32_t d2 = F.cand[i];
            if ((d2 >> sh) == prefix) atomicAdd(&hist[(d2 >> nsh) & (nb - 1)], 1u);
        }
        __syncthreads();
        uint32_t fb, before2;
        select_count_bin(hist, nb >= static_cast<int>(blockDim.x) ? nb : static_cast<int>(blockDim.x), need, S, fb,
                         before2);
        prefix = (prefix << (sh - nsh)) | fb;
        need -= before2;
        sh = nsh;
    }
    return static_cast<int32_t>(prefix);
}

// Float data: the k-th smallest exact distance among the nt rows (fp64, the
// reference's l2), each rounded UP to fp32 so the order statistic of the rounded
// keys bounds the exact one from above; returns the float bits of tau^2, rounded up.
__device__ int32_t kth_dist2_f32up(const QueryPlan& P, const FastSlot& F, const Smem& S, uint32_t nt, int k) {
    if (nt < static_cast<uint32_t>(k)) return __float_as_int(3.0e38f);
    uint32_t* hist = reinterpret_cast<uint32_t*>(S.th);  // 4096 bins: top-k staging is idle here
    int sh = 20;                                         // 12-bit digits of the 32-bit keys: 20, 8, 0
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    for (uint32_t c0 = 0; c0 < nt; c0 += kBatch) {
        const uint32_t nb = min(static_cast<uint32_t>(kBatch), nt - c0);
        score_batch(P, F, S, c0, nb, false);
        __syncthreads();
        for (uint32_t r = threadIdx.x; r < nb; r += blockDim.x) {
            const double dist = __longlong_as_double(static_cast<long long>(S.bh[r]));
            const uint32_t key = __float_as_uint(__double2float_ru(dist));  // positive: bits are monotone
            F.cand[c0 + r] = key;
            atomicAdd(&hist[key >> sh], 1u);
        }
        __syncthreads();
    }
    uint32_t cb, before;
    select_count_bin(hist, 4096, static_cast<uint32_t>(k), S, cb, before);
    uint32_t prefix = cb, need = static_cast<uint32_t>(k) - before;
    while (sh > 0) {
        const int nsh = sh > 12 ? sh - 12 : 0;
        const int nb = 1 << (sh - nsh);
        for (int i = threadIdx.x; i < 4096; i += blockDim.x) hist[i] = 0;
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < nt; i += blockDim.x) {
            const uint32_t key = F.cand[i];
            if ((key >> sh) == prefix) atomicAdd(&hist[(key >> nsh) & (nb - 1)], 1u);
        }
        __syncthreads();
        uint32_t fb, before2;
        select_count_bin(hist, nb >= static_cast<int>(blockDim.x) ? nb : static_cast<int>(blockDim.x), need, S, fb,
                         before2);
        prefix = (prefix << (sh - nsh)) | fb;
        need -= before2;
        sh = nsh;
    }
    const float tau = __uint_as_float(prefix);
    return __float_as_int(__fmul_ru(tau, tau));
}


// MINB CTAs per SM: 5 for u8 rows (the plan / u8 scoring is load-latency bound
// and gains from more CTAs), 3 for fp32 rows (the 32-float row chunks in
// flight need the registers; at 48 registers they spill)
// F32TC: the float bf16x3 hand-off is compiled only into its own instance, so
// the u8 instance keeps its register budget.  NT: threads per CTA (512 for
// indexes with ~10^6 leaves per tree, whose slots are few: memory-bound)
template <int MINB, bool F32TC, int NT = kQueryThreads, bool TCO = false>
__global__ void __launch_bounds__(NT, MINB) query_fast_kernel(
    QueryPlan P, uint8_t* scratch, size_t slot_bytes, uint32_t* slow_list, uint32_t* slow_n) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    const Smem S = carve(smem_raw, P.K, P.NR, P.d, P.row_u8);
    const FastSlot F = fast_slot(scratch, slot_bytes, P.max_leaves, P.budget);
    const double radius = __dmul_rn(P.eps, P.r_min);
    const uint32_t B32 = static_cast<uint32_t>(P.budget);
    const QTree T0 = P.trees[0];
    long long t_prev = clock64();
    auto phase = [&](int i) {  // per-phase cycle accounting (thread 0, optional)
        if (P.phase_cycles && threadIdx.x == 0) {
            const long long t = clock64();
            atomicAdd(P.phase_cycles + i, static_cast<unsigned long long>(t - t_prev));
            t_prev = t;
        }
    };
    const uint64_t q_end = P.q_count ? min(P.q_end, P.q_begin + static_cast<uint64_t>(*P.q_count)) : P.q_end;
    for (uint64_t qs = P.q_begin + blockIdx.x; qs < q_end; qs += gridDim.x) {
        const uint64_t q = P.order ? P.order[qs] : qs;
        const bool u8 = load_query_vec(P, q, S);
        load_query_proj(P, q, 0, S);
        phase(0);
        // Leaf scan + budget cut.  Approximate round (K <= 16): fp32 squared
        // mindists with a rigorous relative error bound `rel` bin the leaves;
        // only leaves whose position against the crossing bin is ambiguous get
        // exact fp64 mindists, and the exact cut is then checked to lie
        // strictly between the leaves taken whole and the ones dropped.  Any
        // doubt (crossing bin in the radius band, a check failing) re-runs the
        // query in the exact round: exact mindist for every leaf.
        const uint32_t nl = T0.num_leaves;
        const double r2 = __dmul_rn(radius, radius);
        const double rel = static_cast<double>(P.K + 2) * 0x1p-22;  // >= 2K ulp(fp32) of the sum
        const double aabs = 1e-36;                                   // fp32 denormal rounding
        const double r2_in = r2 * (1.0 - 1e-12), r2_out = r2 * (1.0 + 1e-12);
        bool approx = P.K <= 16 && r2 > 1e-30 && r2 < 1e30 && !P.force_exact;
        // tensor-core hand-off for this query (u8 rows, large budget)
        const bool tc_eligible = P.tc_bm != nullptr && (F32TC || u8) && B32 >= kTcMinBudget;
        if (approx) build_pen_tables(P, S);
        else build_sq(P, 0, S);
        if (approx) build_half_tables(P, S);
        const int lane = threadIdx.x & 31;
        uint32_t n_full = 0, cut_li = 0, bstar = 0;
        uint64_t take_cut = 0;
        bool to_slow = false;
        double scale = 0.0;
        // approximate round: fine bin (kFine = 32 per histogram bin) of a leaf
        // from its fp32 squared mindist; kFine-1: the radius band, 0xffff:
        // certainly outside.  A fine bin is wider than the error margin
        // (rel * kFine < 1), so only leaves in the fine bins next to the
        // crossing bin's edges can be on the wrong side of them.
        // All in fp32: a < t_in  =>  a (1 + rel) + aabs < r2_in (threshold rounded
        // down), a > t_out  =>  a (1 - rel) - aabs > r2_out (rounded up); the
        // fine bin floor(a * scale_f) is within 2^-23 relative of a * scale,
        // which the margin analysis absorbs ((rel + 2^-22) * kFine < 1).
        const float t_in = __double2float_rd((r2_in - aabs) / (1.0 + rel));
        const float t_out = __double2float_ru((r2_out + aabs) / (1.0 - rel));
        float scale_f = 0.0f;
        auto approx_bin = [&](float a) -> uint32_t {
            if (a < t_in) {
                const float fb = a * scale_f;
                return fb >= static_cast<float>(kFine - 33) ? kFine - 33 : static_cast<uint32_t>(fb);
            }
            return a > t_out ? 0xffffu : kFine - 1;
        };
        for (;;) {
            for (int i = threadIdx.x; i < kBins; i += blockDim.x) S.bins[i] = 0;
            if (threadIdx.x == 0) {
                S.u64s[0] = 0;
                S.u64s[2] = 0;  // W_D: weight taken whole (approximate round)
                S.u64s[3] = 0;  // W_M: in-radius weight of the ambiguous leaves
            }
            scale = approx ? static_cast<double>(kFine) / r2
                           : (radius > 0.0 ? static_cast<double>(kBins) / radius : 0.0);
            scale_f = __double2float_rn(scale);
            __syncthreads();
            // pass 1: every leaf of tree 0 -> weight histogram over bins
            // monotone in mindist; the per-leaf key is kept for pass 2
            {
                unsigned long long wsum = 0;
                uint32_t nin = 0;  // (profiling) leaves not certainly outside
                auto record = [&](uint32_t li, uint32_t b, uint32_t cnt) {
                    if (b != 0xffffu) {
                        ++nin;
                        wsum += cnt;
                        atomicAdd(&S.bins[approx ? b >> 5 : b], cnt);
                    }
                    F.bin16[li] = static_cast<uint16_t>(b);
                };
                if (approx) {
                    // a leaf's box lies in one half of every dimension (the root
                    // split), refined in a few: sum the half penalties by two
                    // 8-dimension table lookups, then add the refinements
                    const float* hp = S.tlo + 2 * P.K * P.NR;  // [K][2] half penalties
                    const float* tcd = hp + 2 * kMaxK;          // [2][256] sums over 8 dims
                    // four leaf records per thread in flight per step (the scan is
                    // load-latency bound otherwise)
                    constexpr int kU = 4;
                    for (uint32_t l0 = threadIdx.x; l0 < nl; l0 += kU * blockDim.x) {
                      uint2 crs[kU];
#pragma unroll
                      for (int u = 0; u < kU; ++u) {
                          const uint32_t lu = l0 + u * blockDim.x;
                          crs[u] = lu < nl ? __ldg(T0.leaf_cr + lu) : make_uint2(0u, 0u);
                      }
#pragma unroll
                      for (int u = 0; u < kU; ++u) {
                        const uint32_t li = l0 + u * blockDim.x;
                        if (li >= nl) break;
                        const uint2 cr = crs[u];
                        float a;
                        if (cr.x == 0xffffffffu) {  // no half form: every dimension from the box
                            float a1;
                            leaf_a2_k16_f32(P, T0, li, li, S, a, a1);
                        } else {
                            a = __fadd_rn(tcd[cr.x & 0xffu], tcd[256 + ((cr.x >> 8) & 0xffu)]);
                            for (uint32_t m = cr.x >> 16; m; m &= m - 1) {  // refined dims: + (box penalty - half penalty) >= 0
                                const int j = __ffs(m) - 1;
                                const uint32_t h = __ldg(reinterpret_cast<const uint16_t*>(T0.leaf_box + static_cast<size_t>(li) * 64) + j);
                                const float pen = __fadd_rn(S.tlo[j * P.NR + (h & 0xffu)], S.thi[j * P.NR + (h >> 8)]);
                                a = __fadd_rn(a, __fsub_rn(pen, hp[2 * j + ((cr.x >> j) & 1u)]));
                            }
                        }
                        record(li, approx_bin(a), cr.y);
                      }
                    }
                } else {  // exact round (rare): exact mindists (fp64 table built below)
                    for (uint32_t li = threadIdx.x; li < nl; li += blockDim.x)
                        record(li, exact_bin(leaf_mindist(P, T0, li, S), radius, scale), __ldg(T0.leaf_count + li));
                }
                for (int o = 16; o; o >>= 1) wsum += __shfl_xor_sync(0xffffffffu, wsum, o);
                if (lane == 0 && wsum) atomicAdd(&S.u64s[0], wsum);
                if (P.phase_cycles) {
                    for (int o = 16; o; o >>= 1) nin += __shfl_xor_sync(0xffffffffu, nin, o);
                    if (lane == 0) atomicAdd(P.phase_cycles + 16, static_cast<unsigned long long>(nin));
                    if (threadIdx.x == 0) atomicAdd(P.phase_cycles + 17, static_cast<unsigned long long>(nl));
                }
            }
            __syncthreads();
            const uint64_t W = S.u64s[0];  // approximate round: an upper bound
            __syncthreads();
            // the fp32 side tables are dead now: the fp64 penalty table takes
            // their place for the exact mindists of the ambiguous leaves
            if (approx) build_sq(P, 0, S);
            phase(1);
            if (W < P.budget) {  // budget does not fill in tree 0 round 0
                to_slow = true;
                break;
            }
            // the budget trips inside bin b*: leaves of lower bins are taken whole,
            // only b*'s leaves need the exact (mindist, node id) order
            if (threadIdx.x < 32) {
                constexpr int per = kBins / 32;
                unsigned long long part = 0;
                for (int b = 0; b < per; ++b) part += S.bins[lane * per + b];
                unsigned long long incl = part;
                for (int o = 1; o < 32; o <<= 1) {
                    const unsigned long long t = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += t;
                }
                const unsigned long long excl = incl - part;
                if (excl < P.budget && P.budget <= incl) {
                    unsigned long long cum = excl;
                    int bin = lane * per;
                    for (int b = 0; b < per; ++b, ++bin) {
                        const unsigned long long c = S.bins[bin];
                        if (cum + c >= P.budget) break;
                        cum += c;
                    }
                    S.u32s[2] = static_cast<uint32_t>(bin);
                    S.u64s[1] = P.budget - cum;
                }
                if (lane == 0) {
                    S.u32s[0] = 0;   // whole-leaf list
                    S.u32s[1] = 0;   // ambiguous / bin-b* items
                    S.u32s[15] = 0;  // ambiguous leaf indices
                    S.u32s[11] = 0xffffffffu;  // b_tau
                    S.u32s[12] = 0;  // tau leaf list
                }
                if (tc_eligible) {  // b_tau: first bin whose cumulative rows reach tc_tau_rows
                    const unsigned long long want = P.tc_tau_rows;
                    if (excl < want && want <= incl) {
                        unsigned long long cum = excl;
                        int bin = lane * per;
                        for (int b = 0; b < per; ++b, ++bin) {
                            cum += S.bins[bin];
                            if (cum >= want) break;
                        }
                        S.u32s[11] = static_cast<uint32_t>(bin);
                    }
                }
            }
            __syncthreads();
            bstar = S.u32s[2];
            const bool do_tau = S.u32s[11] < bstar;  // tau leaves must be whole leaves
            const uint32_t b_tau = S.u32s[11];
            if (approx && bstar == kBins - 1) {  // crossing in the radius band
                if (P.phase_cycles && threadIdx.x == 0) atomicAdd(P.phase_cycles + 6, 1ULL);
                approx = false;
                __syncthreads();
                continue;
            }
            const double lo_edge = approx ? static_cast<double>(bstar * 32) / scale : 0.0;
            const double hi_edge = approx ? static_cast<double>((bstar + 1) * 32) / scale : 0.0;
            const uint32_t lo_f = bstar * 32, hi_f = bstar * 32 + 31;  // b*'s fine bins
            // pass 2: leaves taken whole -> F.full; ambiguous leaves (exact round:
            // bin b*; approximate round: b*'s fine bins and the fine bin on
            // either side) -> exact items in F.B.  Eight leaf bins per thread
            // per step (one 16-byte load).
            {
                unsigned long long w_margin = 0, wm = 0;
                uint32_t* amb_list = reinterpret_cast<uint32_t*>(F.C);  // free until the select
                const uint32_t amb_cap = item_cap(P.max_leaves) * static_cast<uint32_t>(sizeof(LeafItem) / 4);
                // 32 leaf bins per thread per step: four 16-byte loads in flight
                const uint32_t nv = (nl + 7) / 8, nv4 = (nv + 3) / 4;
                for (uint32_t vb = 0; vb < nv4; vb += blockDim.x) {
                    const uint32_t v4 = vb + threadIdx.x;
                    uint4 pk[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        pk[u] = make_uint4(0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu);
                        if (v4 * 4 + u < nv) pk[u] = reinterpret_cast<const uint4*>(F.bin16)[v4 * 4 + u];
                    }
                    const uint32_t v = v4 * 4;  // first 8-leaf vector of this thread
                    uint32_t wmask = 0, amask = 0, tmask = 0;
#pragma unroll
                    for (int e = 0; e < 32; ++e) {
                        const uint4& q4 = pk[e >> 3];
                        const uint32_t wd = ((e >> 1) & 3) == 0 ? q4.x : ((e >> 1) & 3) == 1 ? q4.y : ((e >> 1) & 3) == 2 ? q4.z : q4.w;
                        uint32_t b = (wd >> (16 * (e & 1))) & 0xffffu;
                        if (v * 8 + e >= nl) b = 0xffffu;
                        if (b == 0xffffu) continue;
                        if (approx) {  // fine bins: certainly before / ambiguous / after
                            if (b + 1 < lo_f) wmask |= 1u << e;
                            else if (b <= hi_f + 1) amask |= 1u << e;
                            if (do_tau && b + 1 < lo_f && (b >> 5) <= b_tau) tmask |= 1u << e;
                        } else {
                            if (b < bstar) wmask |= 1u << e;
                            else if (b == bstar) amask |= 1u << e;
                            if (do_tau && b < bstar && b <= b_tau) tmask |= 1u << e;
                        }
                    }
                    // whole leaves: warp-aggregated append
                    const uint32_t cnt = __popc(wmask);
                    uint32_t incl = cnt;
                    for (int o = 1; o < 32; o <<= 1) {
                        const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
                        if (lane >= o) incl += t;
                    }
                    const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
                    uint32_t b0 = 0;
                    if (lane == 31 && tot) b0 = atomicAdd(&S.u32s[0], tot);
                    b0 = __shfl_sync(0xffffffffu, b0, 31) + incl - cnt;
                    for (uint32_t m = wmask; m; m &= m - 1, ++b0)
                        if (b0 < full_cap(P.max_leaves)) F.full[b0] = v * 8 + __ffs(m) - 1;
                    if (__any_sync(0xffffffffu, tmask != 0)) {  // tau leaves (nearest bins)
                        const uint32_t tcnt = __popc(tmask);
                        uint32_t tinc = tcnt;
                        for (int o = 1; o < 32; o <<= 1) {
                            const uint32_t t = __shfl_up_sync(0xffffffffu, tinc, o);
                            if (lane >= o) tinc += t;
                        }
                        const uint32_t ttot = __shfl_sync(0xffffffffu, tinc, 31);
                        uint32_t t0 = 0;
                        if (lane == 31) t0 = atomicAdd(&S.u32s[12], ttot);
                        t0 = __shfl_sync(0xffffffffu, t0, 31) + tinc - tcnt;
                        for (uint32_t m = tmask; m; m &= m - 1, ++t0)
                            if (t0 < tau_cap(P.max_leaves)) F.tau[t0] = v * 8 + __ffs(m) - 1;
                    }
                    // ambiguous leaves (a few hundred per query): listed, then
                    // scored exactly below, one per thread
                    const uint32_t acnt = __popc(amask);
                    uint32_t ainc = acnt;
                    for (int o = 1; o < 32; o <<= 1) {
                        const uint32_t t = __shfl_up_sync(0xffffffffu, ainc, o);
                        if (lane >= o) ainc += t;
                    }
                    const uint32_t atot = __shfl_sync(0xffffffffu, ainc, 31);
                    uint32_t a0 = 0;
                    if (lane == 31 && atot) a0 = atomicAdd(&S.u32s[15], atot);
                    a0 = __shfl_sync(0xffffffffu, a0, 31) + ainc - acnt;
                    for (uint32_t m = amask; m; m &= m - 1, ++a0)
                        if (a0 < amb_cap) amb_list[a0] = v * 8 + __ffs(m) - 1;
                }
                __syncthreads();
                const uint32_t n_amb = S.u32s[15];
                if (n_amb > amb_cap) {  // (uniform) far more ambiguous leaves than the lists hold
                    to_slow = true;
                    break;
                }
                for (uint32_t base = 0; base < n_amb; base += blockDim.x) {
                    const uint32_t i = base + threadIdx.x;
                    bool ok = false;
                    LeafItem it;
                    if (i < n_amb) {
                        const uint32_t li = amb_list[i];
                        const uint32_t w = __ldg(T0.leaf_count + li);
                        if (approx && F.bin16[li] < lo_f) w_margin += w;  // counted below b* by the histogram
                        const double md = leaf_mindist(P, T0, li, S);
                        ok = md <= radius;
                        it.mdb = static_cast<uint64_t>(__double_as_longlong(md));
                        it.id = __ldg(T0.leaf_node + li);
                        it.w = w;
                        it.li = li;
                        it.pad = 0;
                        if (ok) wm += w;
                    }
                    warp_append(ok, it, F.B, &S.u32s[1], item_cap(P.max_leaves));
                }
                for (int o = 16; o; o >>= 1) {
                    w_margin += __shfl_xor_sync(0xffffffffu, w_margin, o);
                    wm += __shfl_xor_sync(0xffffffffu, wm, o);
                }
                if (lane == 0 && w_margin) atomicAdd(&S.u64s[2], w_margin);
                if (lane == 0 && wm) atomicAdd(&S.u64s[3], wm);
            }
            __syncthreads();
            const uint32_t n_bin = S.u32s[1];  // weighted_select reuses this counter
            if (n_bin > item_cap(P.max_leaves)) {  // (uniform) list overflow: the general path
                to_slow = true;
                break;
            }
            // approximate round: weight taken whole = histogram weight below b*
            // minus the margin leaves of bin b*-1 that turned out ambiguous
            const uint64_t need = approx ? S.u64s[1] + S.u64s[2] : S.u64s[1];
            const uint64_t w_whole = P.budget - need, w_amb = S.u64s[3];
            __syncthreads();
            if (approx && (need == 0 || need > w_amb)) {
                if (P.phase_cycles && threadIdx.x == 0) atomicAdd(P.phase_cycles + 6, 1ULL);
                approx = false;
                continue;
            }
            uint64_t kmdb;
            uint32_t kid;
            if (n_bin <= static_cast<uint32_t>(blockDim.x))
                small_weighted_select(F.B, n_bin, need, S, kmdb, kid, take_cut);
            else
                weighted_select(F.B, n_bin, need, F.C, F.A, S, kmdb, kid, take_cut);
            if (P.phase_cycles && threadIdx.x == 0) atomicAdd(P.phase_cycles + 7, static_cast<unsigned long long>(n_bin));
            if (approx) {  // the cut must lie strictly between whole and dropped leaves
                const double mdc = __longlong_as_double(static_cast<long long>(kmdb));
                const bool lo_ok = w_whole == 0 || mdc > __dsqrt_rn(lo_edge);
                const bool hi_ok = mdc < __dsqrt_rn(hi_edge);
                if (!(lo_ok && hi_ok)) {
                    if (P.phase_cycles && threadIdx.x == 0) atomicAdd(P.phase_cycles + 6, 1ULL);
                    approx = false;
                    continue;
                }
            }
            // ambiguous leaves ordered before the cut leaf are whole too; find the cut leaf
            for (uint32_t base = 0; base < n_bin; base += blockDim.x) {
                const uint32_t i = base + threadIdx.x;
                bool before = false;
                uint32_t li = 0;
                if (i < n_bin) {
                    const LeafItem it = F.B[i];
                    li = it.li;
                    before = key_less(it.mdb, it.id, kmdb, kid);
                    if (it.mdb == kmdb && it.id == kid) S.u32s[10] = it.li;
                }
                const uint32_t m = __ballot_sync(0xffffffffu, before);
                if (m) {
                    const int leader = __ffs(m) - 1;
                    uint32_t b0 = 0;
                    if (lane == leader) b0 = atomicAdd(&S.u32s[0], static_cast<uint32_t>(__popc(m)));
                    b0 = __shfl_sync(0xffffffffu, b0, leader);
                    const uint32_t at = b0 + __popc(m & ((1u << lane) - 1u));
                    if (before && at < full_cap(P.max_leaves)) F.full[at] = li;
                }
            }
            __syncthreads();
            n_full = S.u32s[0];
            if (n_full > full_cap(P.max_leaves) || S.u32s[12] > tau_cap(P.max_leaves)) {  // (uniform) lists full
                to_slow = true;
                break;
            }
            cut_li = S.u32s[10];

            break;
        }
        if (to_slow) {
            if (threadIdx.x == 0) slow_list[atomicAdd(slow_n, 1u)] = static_cast<uint32_t>(q);
            __syncthreads();
            continue;
        }
        phase(2);
        // ---- tensor-core hand-off (u8 rows): exact tau^2 from the nearest
        // leaves, the candidate SET as leaf flags; tc_score_kernel verifies it
        const bool tc = tc_eligible && S.u32s[11] < bstar;  // b_tau found below the crossing bin
        if (tc) {
            const uint32_t n_tau = S.u32s[12];
            __syncthreads();
            const uint32_t nt = min(emit_rows(F.tau, n_tau, T0, F.cand, B32, S), B32);
            // exact k-th smallest dist^2 among those rows (float data: an fp32
            // upper bound of it, from the exact fp64 distances)
            int32_t tau2;
            if constexpr (F32TC) tau2 = kth_dist2_f32up(P, F, S, nt, P.k);
            else tau2 = kth_dist2(P, F, S, nt, P.k);
            phase(4);  // (profiling: tau rows + tau^2 apart from the bitmap)
            // candidate set: this query's row bitmap over tree-0 rows, written
            // here (zeroed, then each whole leaf's row range and the cut leaf's
            // taken prefix OR-ed in); tc_score_kernel reads it
            const uint64_t slot = qs - P.q_begin;
            uint32_t* row = P.tc_bm + slot * P.tc_W;
            for (uint64_t w = threadIdx.x; w < P.tc_W / 4; w += blockDim.x)
                reinterpret_cast<uint4*>(row)[w] = make_uint4(0u, 0u, 0u, 0u);
            __syncthreads();  // (the zeros are visible to the whole block)
            for (uint32_t i = threadIdx.x; i < n_full; i += blockDim.x) {
                const uint32_t li = F.full[i];
                const uint32_t a0 = __ldg(T0.leaf_begin + li);
                or_row_range(row, a0, a0 + __ldg(T0.leaf_count + li));
            }
            if (threadIdx.x == 0) {
                const uint32_t a0 = __ldg(T0.leaf_begin + cut_li);
                or_row_range(row, a0, a0 + static_cast<uint32_t>(take_cut));
            }
            if (threadIdx.x == 0) P.tc_tau2[qs - P.q_begin] = tau2;
            __syncthreads();
            phase(3);
            continue;
        }
        if constexpr (TCO) {  // (tensor-core-only instance: the gather re-run verifies it)
            if (threadIdx.x == 0) P.tc_over_list[atomicAdd(P.tc_over_n, 1u)] = static_cast<uint32_t>(q);
            __syncthreads();
            continue;
        }
        // emission: whole leaves (block prefix of their sizes, then one warp per
        // leaf writes its contiguous row range), then the cut leaf's prefix
        const uint32_t n_whole_rows = emit_rows(F.full, n_full, T0, F.cand, B32, S);
        {
            const uint32_t d0 = n_whole_rows;
            const uint32_t s0 = __ldg(T0.leaf_begin + cut_li);
            for (uint32_t e = threadIdx.x; e < take_cut && d0 + e < B32; e += blockDim.x)
                F.cand[d0 + e] = s0 + e;
        }
        if (n_whole_rows + take_cut != B32) {  // invariant: exactly `budget` rows emitted
            if (threadIdx.x == 0) atomicOr(slow_n + 1, 1u);
            __syncthreads();
            continue;
        }
        __syncthreads();
        phase(3);
        // exact verification + top-k (the penalty table region is reused)
        topk_init(S);
        for (uint32_t c0 = 0; c0 < B32; c0 += kBatch) {
            const uint32_t nb = min(static_cast<uint32_t>(kBatch), B32 - c0);
            score_batch(P, F, S, c0, nb, u8);
            __syncthreads();
            topk_absorb(S, nb, P.k, (u8 || P.data_leaf) ? P.perm0 : nullptr);
        }
        const uint32_t nh = topk_finish(S, P.k);
        phase(4);
        for (uint32_t t = threadIdx.x; t < nh; t += blockDim.x) {
            const uint64_t h = S.th[t];
            const double dist = u8 ? __dsqrt_rn(static_cast<double>(h)) : __longlong_as_double(static_cast<long long>(h));
            if (P.ids) P.ids[q * P.k + t] = S.tl[t];
            if (P.dists) P.dists[q * P.k + t] = dist;
        }
        if (threadIdx.x == 0) {
            if (P.n_hits) P.n_hits[q] = static_cast<int32_t>(nh);
            if (P.radius) P.radius[q] = P.r_min;
            if (P.cands) P.cands[q] = P.budget;
        }
        __syncthreads();
        phase(5);
    }
}

// ---------------------------------------------------------------------------
// General path: every tree, every round, bitmap dedup (CandidateSet).
// ---------------------------------------------------------------------------
// A deferred general-path query (query_slow_kernel -> slow_score_kernel ->
// slow_topk_kernel), one per slot.
struct SlowRec {
    uint32_t q, msz, scored, done;
    double r;
};
constexpr uint32_t kNoQuery = 0xffffffffu;
// budget from which the general path defers member distances (C5: 10^7)
constexpr uint64_t kSlowDeferMinBudget = 1u << 18;

struct SlowSlot {
    LeafItem *A, *B, *C;
    uint32_t* bitmap;  // n bits
    uint32_t* mpos;    // members
    double* mdist;
};

// The slot's bitmap lives apart (`bitmaps`, bm_words per slot, zeroed once
// and cleared by each query): the rest of a slot is laid out by the budget,
// which changes with k from one batch to the next.
__device__ __forceinline__ SlowSlot slow_slot(uint8_t* base, size_t slot_bytes, uint32_t maxl,
                                              uint64_t budget, uint32_t slot, uint32_t* bitmaps = nullptr,
                                              uint64_t bm_words = 0) {
    uint8_t* p = base + static_cast<size_t>(slot) * slot_bytes;
    SlowSlot s;
    s.A = reinterpret_cast<LeafItem*>(p);
    s.B = s.A + maxl;
    s.C = s.B + maxl;
    s.mdist = reinterpret_cast<double*>(s.C + maxl);
    s.mpos = reinterpret_cast<uint32_t*>(s.mdist + budget);
    s.bitmap = bitmaps ? bitmaps + static_cast<uint64_t>(slot) * bm_words : nullptr;
    return s;
}

// Emit the NEW entries of the selected leaves (all, or the first `take_cut`
// new ones of the cut leaf) into the member list.
__device__ void emit_members(const QueryPlan& P, int tree, const LeafItem* A, uint32_t nA,
                             bool select, uint64_t kmdb, uint32_t kid, uint64_t take_cut,
                             const SlowSlot& L, const Smem& S, bool score, bool u8q) {
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
                    if (score) {
                        const float* x = P.data + static_cast<uint64_t>(pos) * P.d;
                        L.mdist[slot] = u8q ? l2_exact_u8(S.qv, x, P.d) : l2_exact(S.qv, x, P.d);
                    }
                }
            }
            emitted += __popc(tm);
        }
    }
    __syncthreads();
}

// Top-k of a general-path query's members (extracted kFastMaxK at a time,
// any k) and its outputs.
__device__ void slow_finish(const QueryPlan& P, const Smem& S, const SlowSlot& L, uint64_t q, uint32_t msz,
                            double r, bool done) {
    uint32_t want = min(msz, static_cast<uint32_t>(P.k));
    uint32_t out = 0;
    uint64_t lbh = 0;
    uint32_t lbl = 0;
    bool have_lb = false;
    while (out < want) {
        const int kk = static_cast<int>(min(want - out, static_cast<uint32_t>(kFastMaxK)));
        topk_init(S);
        for (uint32_t c0 = 0; c0 < msz; c0 += kBatch) {
            const uint32_t nb = min(static_cast<uint32_t>(kBatch), msz - c0);
            for (uint32_t i = threadIdx.x; i < nb; i += blockDim.x) {
                const uint64_t h = static_cast<uint64_t>(__double_as_longlong(L.mdist[c0 + i]));
                const uint32_t l = L.mpos[c0 + i];
                const bool above = !have_lb || key_less(lbh, lbl, h, l);
                S.bh[i] = above ? h : ~0ULL;  // sentinels never beat a real key
                S.bl[i] = above ? l : 0xffffffffu;
            }
            __syncthreads();
            topk_absorb(S, nb, kk, nullptr);
        }
        uint32_t got = topk_finish(S, kk);
        // drop sentinel entries (only possible when fewer than kk remain)
        while (got > 0 && S.th[got - 1] == ~0ULL && S.tl[got - 1] == 0xffffffffu) --got;
        for (uint32_t t = threadIdx.x; t < got; t += blockDim.x) {
            if (P.ids) P.ids[q * P.k + out + t] = S.tl[t];
            if (P.dists) P.dists[q * P.k + out + t] = __longlong_as_double(static_cast<long long>(S.th[t]));
        }
        lbh = S.th[got - 1];
        lbl = S.tl[got - 1];
        have_lb = true;
        out += got;
        __syncthreads();
    }
    // rc_ann: without the budget reached, the closest counts only within c * r
    if (P.rc_mode && !done && want > 0 && !(__longlong_as_double(static_cast<long long>(lbh)) <= __dmul_rn(P.c, r)))
        want = 0;
    if (threadIdx.x == 0) {
        if (P.n_hits) P.n_hits[q] = static_cast<int32_t>(want);
        if (P.radius) P.radius[q] = r;
        if (P.cands) P.cands[q] = msz;
    }
}

// Exact distances of members [from, msz) by the whole block.
__device__ void score_members(const QueryPlan& P, const float* qv, const SlowSlot& L, uint32_t from, uint32_t msz,
                              bool u8q) {
    for (uint32_t i = from + threadIdx.x; i < msz; i += blockDim.x) {
        const float* x = P.data + static_cast<uint64_t>(L.mpos[i]) * P.d;
        L.mdist[i] = u8q ? l2_exact_u8(qv, x, P.d) : l2_exact(qv, x, P.d);
    }
    __syncthreads();
}

// The listed queries are claimed one at a time through `taken` (never past
// `count`): a slot that finishes early takes the next one.
//
// Deferred mode (recs != null and no more listed queries than slots): a
// query with a large budget is ~10^7 members, and one CTA computing their
// distances and top-k leaves the GPU idle (C5: ~0.5 s per query).  Each CTA
// then takes at most one query and records its member list (rec); the
// distances are computed grid-wide (slow_score_kernel) and the top-k by
// slow_topk_kernel.  Distances a round's count_within needs are computed
// here as before.
template <int NT>
__global__ void __launch_bounds__(NT) query_slow_kernel(
    QueryPlan P, const uint32_t* list, uint32_t count, const uint32_t* count_dev, uint32_t* taken,
    uint8_t* scratch, size_t slot_bytes, uint32_t* bitmaps, uint64_t bm_words, SlowRec* recs) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    __shared__ uint32_t s_qi;
    const Smem S = carve(smem_raw, P.K, P.NR, P.d, P.row_u8);
    const SlowSlot L = slow_slot(scratch, slot_bytes, P.max_leaves, P.budget, blockIdx.x, bitmaps, bm_words);
    if (count_dev) count = min(count, *count_dev);
    const bool defer = recs != nullptr && count <= gridDim.x;
    if (recs && threadIdx.x == 0) recs[blockIdx.x].q = kNoQuery;
    long long t_prev = clock64();
    auto phase = [&](int i, unsigned long long add = 0) {  // profiling: slots 8.. of the phase array
        if (P.phase_cycles && threadIdx.x == 0) {
            const long long t = clock64();
            atomicAdd(P.phase_cycles + 8 + i, add ? add : static_cast<unsigned long long>(t - t_prev));
            t_prev = t;
        }
    };
    for (;;) {
        if (threadIdx.x == 0) {
            uint32_t cur = *static_cast<volatile uint32_t*>(taken), got = count;
            while (cur < count) {
                const uint32_t prev = atomicCAS(taken, cur, cur + 1);
                if (prev == cur) {
                    got = cur;
                    break;
                }
                cur = prev;
            }
            s_qi = got;
        }
        __syncthreads();
        const uint32_t qi = s_qi;
        __syncthreads();
        if (qi >= count) break;
        const uint64_t q = list ? list[qi] : qi;
        if (threadIdx.x == 0) S.u32s[7] = 0;  // |S|
        __syncthreads();
        const bool u8q = load_query_vec(P, q, S);  // u8 index and u8-exact query: integer distances
        double r = P.r_min;
        bool done = false;
        uint32_t scored = 0;  // members [0, scored) have distances
        for (;;) {
            for (int tree = 0; tree < P.L && !done; ++tree) {
                load_query_proj(P, q, tree, S);
                build_sq(P, tree, S);
                const double radius = __dmul_rn(P.eps, r);
                const uint32_t have = S.u32s[7];
                uint32_t nA;
                uint64_t W;
                scan_leaves(P, tree, radius, S, L.A, have ? L.bitmap : nullptr, nA, W, L.C);
                phase(0);
                const uint64_t need = P.budget - have;
                if (W >= need) {
                    uint64_t kmdb, take_cut;
                    uint32_t kid;
                    weighted_select(L.A, nA, need, L.B, L.C, S, kmdb, kid, take_cut);
                    phase(1);
                    emit_members(P, tree, L.A, nA, true, kmdb, kid, take_cut, L, S, !defer, u8q);
                    done = true;
                } else {
                    emit_members(P, tree, L.A, nA, false, 0, 0, 0, L, S, !defer, u8q);
                }
                if (!defer) scored = S.u32s[7];
                phase(2);
                phase(5, nA);
            }
            if (done || P.rc_mode) break;  // rc_ann: a single pass (index.cpp:278-289)
            // count_within(c * r) (index.cpp:244-249, 328)
            const double lim = __dmul_rn(P.c, r);
            const uint32_t msz = S.u32s[7];
            if (scored < msz) score_members(P, S.qv, L, scored, msz, u8q);
            scored = msz;
            uint32_t mine = 0;
            for (uint32_t i = threadIdx.x; i < msz; i += blockDim.x) mine += L.mdist[i] <= lim ? 1u : 0u;
            for (int o = 16; o; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
            if (threadIdx.x == 0) S.u32s[8] = 0;
            __syncthreads();
            if ((threadIdx.x & 31) == 0 && mine) atomicAdd(&S.u32s[8], mine);
            __syncthreads();
            const bool enough = S.u32s[8] >= static_cast<uint32_t>(P.k);
            __syncthreads();
            phase(3);
            phase(6, 1);
            if (enough) break;
            r = __dmul_rn(r, P.c);
        }
        const uint32_t msz = S.u32s[7];
        if (!defer) slow_finish(P, S, L, q, msz, r, done);
        // clear the bitmap words we touched
        for (uint32_t i = threadIdx.x; i < msz; i += blockDim.x) L.bitmap[L.mpos[i] >> 5] = 0;
        __syncthreads();
        phase(4);
        phase(7, msz + 1);
        if (defer) {
            if (threadIdx.x == 0) {
                SlowRec rc;
                rc.q = static_cast<uint32_t>(q);
                rc.msz = msz;
                rc.scored = scored;
                rc.done = done ? 1u : 0u;
                rc.r = r;
                recs[blockIdx.x] = rc;
            }
            break;  // the slot's members wait for slow_score_kernel
        }
    }
}

// Deferred members' exact distances: blockIdx.y = slot, blockIdx.x strides
// over its members (one thread per member, the same fp64 chain as above).
__global__ void __launch_bounds__(256) slow_score_kernel(QueryPlan P, const SlowRec* recs, uint8_t* scratch,
                                                        size_t slot_bytes) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    const SlowRec rc = recs[blockIdx.y];
    if (rc.q == kNoQuery || rc.scored >= rc.msz) return;
    float* qv = reinterpret_cast<float*>(smem_raw);
    __shared__ int s_nonint;
    if (threadIdx.x == 0) s_nonint = 0;
    __syncthreads();
    for (int t = threadIdx.x; t < P.d; t += blockDim.x) {
        const float v = P.q[static_cast<uint64_t>(rc.q) * P.d + t];
        qv[t] = v;
        if (!(v >= 0.0f && v <= 255.0f && v == floorf(v))) s_nonint = 1;
    }
    __syncthreads();
    const SlowSlot L = slow_slot(scratch, slot_bytes, P.max_leaves, P.budget, blockIdx.y);
    const uint32_t stride = gridDim.x * blockDim.x;
    uint32_t i = rc.scored + blockIdx.x * blockDim.x + threadIdx.x;
    if (P.data_u8 && !s_nonint) {
        // u8 index, u8-exact query: integer sums (the same doubles), so a warp
        // reads a member's row as whole 128-byte lines and reduces across
        // lanes; four rows in flight per warp
        const int lane = threadIdx.x & 31;
        const uint32_t wstride = gridDim.x * (blockDim.x / 32);
        const int d4 = (P.d & 3) == 0 ? P.d / 4 : 0;
        for (uint32_t j = rc.scored + (blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5)) * 4; j < rc.msz;
             j += wstride * 4) {
            unsigned acc[4] = {0, 0, 0, 0};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if (j + u >= rc.msz) break;
                const float* x = P.data + static_cast<uint64_t>(L.mpos[j + u]) * P.d;
                if (d4) {
                    for (int t = lane; t < d4; t += 32) {
                        const float4 xv = __ldg(reinterpret_cast<const float4*>(x) + t);
                        const int a = static_cast<int>(qv[4 * t]) - static_cast<int>(xv.x);
                        const int b = static_cast<int>(qv[4 * t + 1]) - static_cast<int>(xv.y);
                        const int c = static_cast<int>(qv[4 * t + 2]) - static_cast<int>(xv.z);
                        const int e = static_cast<int>(qv[4 * t + 3]) - static_cast<int>(xv.w);
                        acc[u] += static_cast<unsigned>(a * a + b * b + c * c + e * e);
                    }
                } else {
                    for (int t = lane; t < P.d; t += 32) {
                        const int a = static_cast<int>(qv[t]) - static_cast<int>(__ldg(x + t));
                        acc[u] += static_cast<unsigned>(a * a);
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                unsigned long long v = acc[u];
                for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                if (lane == u && j + u < rc.msz) L.mdist[j + u] = __dsqrt_rn(static_cast<double>(v));
            }
        }
        return;
    }
    // two members in flight per thread (independent fp64 chains)
    for (; i + stride < rc.msz; i += 2 * stride) {
        const double a = l2_exact(qv, P.data + static_cast<uint64_t>(L.mpos[i]) * P.d, P.d);
        const double b = l2_exact(qv, P.data + static_cast<uint64_t>(L.mpos[i + stride]) * P.d, P.d);
        L.mdist[i] = a;
        L.mdist[i + stride] = b;
    }
    if (i < rc.msz) L.mdist[i] = l2_exact(qv, P.data + static_cast<uint64_t>(L.mpos[i]) * P.d, P.d);
}

// Deferred queries' top-k and outputs: one CTA per slot.
template <int NT>
__global__ void __launch_bounds__(NT) slow_topk_kernel(QueryPlan P, const SlowRec* recs, uint8_t* scratch,
                                                                 size_t slot_bytes) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    const SlowRec rc = recs[blockIdx.x];
    if (rc.q == kNoQuery) return;
    const Smem S = carve(smem_raw, P.K, P.NR, P.d, P.row_u8);
    const SlowSlot L = slow_slot(scratch, slot_bytes, P.max_leaves, P.budget, blockIdx.x);
    slow_finish(P, S, L, rc.q, rc.msz, rc.r, rc.done != 0);
}

// One warp per query: lane l owns shards l, l+32, ...; every step the warp
// takes the smallest (distance, id) head over all shards (two-key shuffle
// argmin) and the owning lane advances that shard's head.  Any shard count.
__global__ void merge_topk_kernel(const double* __restrict__ sd, const uint64_t* __restrict__ sid,
                                  const int32_t* __restrict__ sh, int shards, uint64_t nq, int k,
                                  double* od, uint64_t* oid, int32_t* oh) {
    const int lane = threadIdx.x & 31;
    const uint64_t warps = static_cast<uint64_t>(gridDim.x) * (blockDim.x / 32);
    for (uint64_t q = blockIdx.x * static_cast<uint64_t>(blockDim.x / 32) + (threadIdx.x >> 5); q < nq;
         q += warps) {
        // this lane's best head over its shards (sentinel: +inf, max id)
        auto lane_best = [&](double& bd, uint64_t& bi, int& bs, const int* head) {
            bd = __longlong_as_double(0x7ff0000000000000LL);
            bi = ~0ULL;
            bs = -1;
            for (int j = 0, s = lane; s < shards; ++j, s += 32) {
                const uint64_t row = static_cast<uint64_t>(s) * nq + q;
                if (head[j] >= sh[row]) continue;
                const double d = sd[row * k + head[j]];
                const uint64_t id = sid[row * k + head[j]];
                if (bs < 0 || d < bd || (d == bd && id < bi)) {
                    bd = d;
                    bi = id;
                    bs = s;
                }
            }
        };
        int head[kMergeMaxShards / 32];
        for (int j = 0; j < kMergeMaxShards / 32; ++j) head[j] = 0;
        double bd;
        uint64_t bi;
        int bs;
        lane_best(bd, bi, bs, head);
        int out = 0;
        for (; out < k; ++out) {
            double wd = bd;
            uint64_t wi = bi;
            int ws = bs;
            for (int off = 16; off > 0; off >>= 1) {
                const double od2 = __shfl_xor_sync(0xffffffffu, wd, off);
                const uint64_t oi2 = __shfl_xor_sync(0xffffffffu, wi, off);
                const int os2 = __shfl_xor_sync(0xffffffffu, ws, off);
                if (os2 >= 0 && (ws < 0 || od2 < wd || (od2 == wd && (oi2 < wi || (oi2 == wi && os2 < ws))))) {
                    wd = od2;
                    wi = oi2;
                    ws = os2;
                }
            }
            if (ws < 0) break;
            if (lane == 0) {
                od[q * k + out] = wd;
                oid[q * k + out] = wi;
            }
            if (lane == (ws & 31)) {
                head[ws >> 5]++;
                lane_best(bd, bi, bs, head);
            }
        }
        if (lane == 0) oh[q] = out;
    }
}

// Locality key of a query: the tree-0 path bits of its space-0 codes -- the
// top bit of every dim (the root slot) above the second bit of every dim.
// Sorting by it lets concurrently running CTAs share candidate rows in L2.
__global__ void query_order_keys(const float* __restrict__ qproj0, uint64_t nq, int K,
                                 const float* __restrict__ table0, int NR, int sbits,
                                 uint32_t* __restrict__ keys, uint32_t* __restrict__ idx) {
    for (uint64_t q = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; q < nq;
         q += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        uint32_t top = 0, second = 0;
        const int W = NR + 1;
        for (int j = 0; j < K && j < 16; ++j) {
            const float v = qproj0[q * K + j];
            const float* row = table0 + static_cast<size_t>(j) * W;
            int lo = 0, hi = W;  // lower_bound
            while (lo < hi) {
                const int m = (lo + hi) >> 1;
                if (row[m] < v) lo = m + 1; else hi = m;
            }
            int reg = lo - 1;
            reg = reg < 0 ? 0 : (reg > NR - 1 ? NR - 1 : reg);
            top |= static_cast<uint32_t>((reg >> (sbits - 1)) & 1) << j;
            if (sbits > 1) second |= static_cast<uint32_t>((reg >> (sbits - 2)) & 1) << j;
        }
        keys[q] = (top << 16) | second;
        idx[q] = static_cast<uint32_t>(q);
    }
}

std::mutex g_phase_mu;
double g_phase[8] = {0, 0, 0, 0, 0, 0, 0, 0};

}  // namespace

void last_query_phases(double* out6) {
    std::lock_guard<std::mutex> lk(g_phase_mu);
    for (int i = 0; i < 8; ++i) out6[i] = g_phase[i];
}

void run_query_batch(const QueryPlan& P, QueryScratch& X, int device, cudaStream_t s,
                     cudaStream_t alloc_s) {
    const int sms = sm_count(device);
    const size_t smem = smem_bytes(P.K, P.NR, P.d, P.row_u8);
    if (smem > 220 * 1024) throw InvalidArgument("ck_ann: query dimension too large for the staging buffer");
    // tau^2 = k-th smallest dist^2 over the rows of the nearest leaves.  If
    // those rows were a uniform sample of the candidates, about
    // k * budget / tau_rows candidates would pass it; size the sample so
    // that is a quarter of the survivor staging buffer (nearest-leaf rows
    // do better than uniform; measured on C2, 2x this sample trades 1 ms
    // of plan for 2.5 ms of scoring), and keep the tensor-core path only
    // where the sample is a small part of the budget.
    // 8-bit rows: exact int8 scores; float rows: bf16x3 scores filtered with a
    // rigorous slack, survivors rescored exactly in fp64 (tc_finish_f32).  The
    // float path stages 4x more survivors per query (kTcFinishCapF32): its tau
    // rows are fp64 chains, so 4x fewer of them is the better trade.  So do
    // 8-bit rows wider than 256 B (C3, d = 784): there the tau rows are read
    // from HBM (the rows exceed L2) and were ~2/3 of the plan kernel's time.
    const bool f32_rows = !P.data_u8 && P.data_leaf && P.data_tcf && P.xnf && P.row_f > 256 && tc_score_fits(P.row_f);
    // Likewise for budgets of 10^6+ (C5: 4x fewer tau rows, 32 K instead of
    // 131 K, which were ~half the plan kernel's HBM reads; the survivors,
    // 3.3 K at the median and 11 K at most, fit the wider staging).
    const bool wide_u8 = P.data_u8 && (P.row_u8 > 256 || P.budget >= (1u << 20) || std::getenv("DETLSH_TEST_WIDE_FIN_CAP")) &&
                         !std::getenv("DETLSH_TEST_NARROW_FIN_CAP");
    const uint32_t fin_cap = (f32_rows || wide_u8) ? kTcFinishCapF32 : kTcFinishCap;
    const uint64_t tau_max = kTauRowsMax * kTcFinishCap / fin_cap;  // the same survivor margin
    uint64_t tau_rows = std::max<uint64_t>(
        std::max<uint64_t>(kTauRows, 2ULL * P.k),
        std::min<uint64_t>(tau_max, (4ULL * P.k * P.budget + fin_cap - 1) / fin_cap));
    if (const char* e = std::getenv("DETLSH_TAU_ROWS"))  // measurement hook
        tau_rows = std::max<uint64_t>(2ULL * P.k, std::strtoull(e, nullptr, 10));
    const bool tc_any = P.tc_allowed && P.budget >= kTcMinBudget && P.budget <= 0xffffffffULL &&
                        2ULL * P.k <= fin_cap && 8 * tau_rows <= P.budget && P.k <= kFastMaxK && !P.rc_mode;
    const bool tc_u8 = tc_any && P.data_u8 && P.xn_u8 && P.data_tc && tc_score_fits(P.row_u8);
    const bool tc_f32 = tc_any && f32_rows;
    const bool tc_ok = tc_u8 || tc_f32;
    // plan-kernel occupancy: 5 CTAs/SM when it hands verification to the
    // tensor cores (load-latency bound plan), 3 when it verifies candidates
    // itself (the row chunks in flight need the registers); measured on C1-C4.
    // DETLSH_FAST_MINB=3|5 overrides (measurement hook).
    const char* minb_env = std::getenv("DETLSH_FAST_MINB");
    const bool five = minb_env ? std::atoi(minb_env) == 5 : tc_u8;  // (float tau rows: fp64 chains, 3/SM)
    // Indexes with ~10^6 leaves per tree (C5): a slot's scratch is ~100 MB,
    // so memory, not occupancy, bounds the CTAs in flight; 512 threads per CTA
    // halve each query's scan.  DETLSH_FAST_THREADS=256|512 overrides.
    const char* nt_env = std::getenv("DETLSH_FAST_THREADS");
    const bool wide = nt_env ? std::atoi(nt_env) == 512 : (tc_u8 && P.max_leaves >= (1u << 19));
    const int fast_nt = wide && !tc_f32 ? 512 : kQueryThreads;
    auto* const fast_kernel = tc_f32 ? &query_fast_kernel<3, true>
                              : fast_nt == 512 ? &query_fast_kernel<2, false, 512>
                              : five ? &query_fast_kernel<5, false> : &query_fast_kernel<3, false>;
    // the same plan kernel without the gather verification, for the
    // tensor-core launches (smaller code and register footprint)
    auto* const tco_kernel = tc_f32 ? &query_fast_kernel<3, true, kQueryThreads, true>
                             : fast_nt == 512 ? &query_fast_kernel<2, false, 512, true>
                             : five ? &query_fast_kernel<5, false, kQueryThreads, true>
                                    : &query_fast_kernel<3, false, kQueryThreads, true>;
    DETLSH_CUDA(cudaFuncSetAttribute(fast_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    DETLSH_CUDA(cudaFuncSetAttribute(tco_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    // general path: 1024 threads per query for large budgets (few slots, each
    // query's scans and member lists ~10^6-10^7 long), 256 otherwise
    const char* snt_env = std::getenv("DETLSH_SLOW_THREADS");  // 256|1024 (test hook)
    const bool slow_wide = snt_env ? std::atoi(snt_env) == 1024 : P.budget >= kSlowDeferMinBudget;
    const int slow_nt = slow_wide ? 1024 : kQueryThreads;
    auto* const slow_kernel = slow_wide ? &query_slow_kernel<1024> : &query_slow_kernel<kQueryThreads>;
    auto* const slow_topk = slow_wide ? &slow_topk_kernel<1024> : &slow_topk_kernel<kQueryThreads>;
    DETLSH_CUDA(cudaFuncSetAttribute(slow_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    DETLSH_CUDA(cudaFuncSetAttribute(slow_topk, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    // Persistent scratch lives on the index's own stream (it outlives any
    // caller stream).  Growing it is the one host wait of a batch, and only
    // happens when a batch needs more scratch than every earlier one.
    // under stream capture the graph's own dependencies order its replays;
    // otherwise the batch waits for the previous one (any stream) to release
    // the scratch
    cudaStreamCaptureStatus cap_st = cudaStreamCaptureStatusNone;
    DETLSH_CUDA(cudaStreamIsCapturing(s, &cap_st));
    const bool capturing = cap_st != cudaStreamCaptureStatusNone;
    bool grew = false;
    auto grow_scratch = [&](auto& buf, size_t count) {
        if (buf.size() >= count) return;
        if (capturing) throw InvalidArgument("ck_ann: the first batch of a shape cannot be captured (scratch grows)");
        if (!grew && X.done) DETLSH_CUDA(cudaEventSynchronize(X.done));  // earlier batches still read it
        grew = true;
        if (std::getenv("DETLSH_DEBUG_GROW"))
            std::fprintf(stderr, "[query] scratch grows %zu -> %zu elements\n", buf.size(), count);
        {
            StreamScope sc(alloc_s);
            buf.alloc(count);
        }
        DETLSH_CUDA(cudaStreamSynchronize(alloc_s));
    };
    if (!X.done) DETLSH_CUDA(cudaEventCreateWithFlags(&X.done, cudaEventDisableTiming));
    else if (!capturing) DETLSH_CUDA(cudaStreamWaitEvent(s, X.done, 0));
    if (X.counters.size() < 8) {
        grow_scratch(X.counters, 8);
        DETLSH_CUDA(cudaMemsetAsync(X.counters.get(), 0, 32, s));  // incl. the sticky invariant flag
    }
    grow_scratch(X.slow_list, P.nq);
    // counters: slow-path and overflow counts reset per batch; the invariant flag is sticky
    DETLSH_CUDA(cudaMemsetAsync(X.counters.get() + kCntSlow, 0, 4, s));
    DETLSH_CUDA(cudaMemsetAsync(X.counters.get() + kCntOver, 0, 4, s));
    DETLSH_CUDA(cudaMemsetAsync(X.counters.get() + kCntTaken, 0, 8, s));  // general-path claims + published count
    QueryPlan Pp = P;
    Pp.q_count = nullptr;
    if (profiling_enabled()) {
        grow_scratch(X.phases, 24);
        DETLSH_CUDA(cudaMemsetAsync(X.phases.get(), 0, 24 * sizeof(unsigned long long), s));
        Pp.phase_cycles = X.phases.get();
    }
    // locality-aware processing order for large batches (results are written
    // to each query's own slot, so the order is invisible to the caller)
    DevBuf<uint32_t> ok0, ok1, ov0, ov1, otmp;  // freed stream-ordered after the kernels
    if (P.nq >= 4096) {
        const uint64_t nq = P.nq;
        ok0.alloc(nq);
        ok1.alloc(nq);
        ov0.alloc(nq);
        ov1.alloc(nq);
        otmp.alloc(radix_temp_elems(nq));
        int sbits = 0;
        while ((1 << sbits) < P.NR) ++sbits;
        const unsigned g = static_cast<unsigned>(std::min<uint64_t>((nq + 255) / 256, 4096));
        query_order_keys<<<g, 256, 0, s>>>(P.qproj, nq, P.K, P.table, P.NR, sbits, ok0.get(), ov0.get());
        DETLSH_LAUNCH_CHECK();
        const bool flip = radix_sort_pairs<uint32_t>(ok0.get(), ov0.get(), ok1.get(), ov1.get(), nq, 0,
                                                     32, otmp.get(), s);
        Pp.order = flip ? ov1.get() : ov0.get();
    }
    const size_t items = 3 * static_cast<size_t>(P.max_leaves) * sizeof(LeafItem);
    // memory the scratch may be sized against (no query under capture).  Asked
    // of the driver once per batch shape: cudaMemGetInfo on every batch was a
    // host stall of up to ~100 ms whenever another thread was in the driver
    // (an NVML clock sampler), leaving the GPU idle between device-mode batches.
    size_t avail = 0;
    if (!capturing) {
        if (X.avail_nq != P.nq || X.avail_budget != P.budget) {
            X.avail_bytes = device_memory_available(device) + X.fast.size() + X.slow.size() +
                            (X.slow_bm.size() + X.tc_bm.size()) * sizeof(uint32_t);
            X.avail_nq = P.nq;
            X.avail_budget = P.budget;
        }
        avail = X.avail_bytes;
    }
    const bool fast_path = P.k <= kFastMaxK && !P.rc_mode;
    // general path: the queries the fast path listed (count on the device), or
    // every query (k beyond the fast path, rc_ann).  A fixed number of slots,
    // each looping over the list; a slot's bitmap is cleared by the kernel.
    const uint64_t n_list = P.nq;
    const size_t slow_bytes = (items + 12 * P.budget + 255) / 256 * 256;
    const uint64_t bm_words = ((P.n + 31) / 32 + 3) / 4 * 4;  // per-slot bitmap (n bits), kept zero
    size_t gslots = std::min<size_t>(n_list, static_cast<size_t>(sms));
    const size_t slow_lim = capturing ? std::max<size_t>(X.slow.size(), slow_bytes) : slow_scratch_limit(avail);
    gslots = std::max<size_t>(1, std::min<size_t>(gslots, slow_lim / (slow_bytes + 4 * bm_words)));
    if (std::getenv("DETLSH_DEBUG_QUERY"))
        std::fprintf(stderr, "[query] general path: slots=%zu bytes/slot=%zu\n", gslots, slow_bytes);
    grow_scratch(X.slow, gslots * slow_bytes);
    if (X.slow_slots < gslots || X.slow_bm.size() < gslots * bm_words) {
        if (capturing) throw InvalidArgument("ck_ann: the first batch of a shape cannot be captured (scratch grows)");
        if (X.done) DETLSH_CUDA(cudaEventSynchronize(X.done));
        X.slow_bm.release();
        grow_scratch(X.slow_bm, gslots * bm_words);
        DETLSH_CUDA(cudaMemsetAsync(X.slow_bm.get(), 0, gslots * bm_words * 4, s));
        X.slow_slots = gslots;
    }
    if (fast_path) {
        int per_sm = 0;
        DETLSH_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fast_kernel, fast_nt, smem));
        per_sm = std::max(1, std::min(per_sm, 6));
        const size_t fast_bytes = fast_slot_bytes(P.max_leaves, P.budget);
        // processing slots: a CTA each, bounded by the scratch they need
        // (fast_bytes grows with the budget: 4 B per candidate)
        size_t slots = std::min<size_t>(P.nq, static_cast<size_t>(sms) * per_sm);
        // (under stream capture no memory query: the scratch an earlier,
        // uncaptured batch of this shape sized is what the slots get)
        const size_t lim = capturing ? std::max<size_t>(X.fast.size(), fast_bytes) : fast_scratch_limit(avail);
        slots = std::max<size_t>(1, std::min<size_t>(slots, lim / fast_bytes));
        grow_scratch(X.fast, slots * fast_bytes);
        auto launch_fast = [&](const QueryPlan& Pc, bool tco = false) {
            const uint64_t m = Pc.q_end - Pc.q_begin;
            if (m == 0) return;
            ProfScope ps("query_fast", s);
            (tco ? tco_kernel : fast_kernel)<<<static_cast<unsigned>(std::min<uint64_t>(slots, m)), fast_nt, smem, s>>>(
                Pc, X.fast.get(), fast_bytes, X.slow_list.get(), X.counters.get());
            DETLSH_LAUNCH_CHECK();
        };
        // test hook: exact fp64 mindists for every leaf (no approximate round)
        if (std::getenv("DETLSH_TEST_EXACT_SCAN")) Pp.force_exact = 1;
        Pp.tc_tau_rows = static_cast<uint32_t>(std::min<uint64_t>(tau_rows, 0xffffffffULL));
        if (!tc_ok) {
            launch_fast(Pp);
        } else {
            // u8 rows with a large budget: the plan kernel hands each query's
            // candidate set to the tcgen05 dataset-major scorer (tc_score.cu)
            const int R = tc_f32 ? P.row_f : P.row_u8;
            Pp.tc_f32 = tc_f32 ? 1 : 0;
            const uint64_t W = ((P.n + 31) / 32 + 3) / 4 * 4;  // bitmap words per query, rows 16-B aligned
            // test hook: a smaller staging buffer forces the overflow re-run
            uint32_t tc_cap = fin_cap;
            if (const char* e = std::getenv("DETLSH_TEST_TC_CAP"))
                tc_cap = static_cast<uint32_t>(std::max(1L, std::min<long>(std::atol(e), fin_cap)));
            // per processing slot: row bitmap (n/8 bytes), survivors (8 B each),
            // pass records (128 KB); a chunk stays under ~3 GB
            // pass records (128 KB); a chunk stays under ~3 GB, or up to an
            // eighth of the memory (16 GB) when the bitmaps are large.  Whole
            // 256-query tiles of tc_score (C5: 1024 queries per chunk, 3.8
            // rounds of the plan kernel's 271 CTAs; 813 = 3 whole rounds left
            // a 45-query tile per chunk)
            const uint64_t per_q = W * 4 + 8ULL * fin_cap + 2ULL * fin_cap * sizeof(uint4);
            const uint64_t chunk_bytes =
                capturing ? (3ULL << 30)
                          : std::max<uint64_t>(3ULL << 30, std::min<uint64_t>(16ULL << 30, avail / 8));
            uint64_t chunk = chunk_bytes / per_q;
            chunk = chunk >= P.nq ? (P.nq + 255) / 256 * 256 : std::max<uint64_t>(256, chunk / 256 * 256);
            // pass records staged per chunk: ~8192 per query, plus the runs of
            // kTcRecChunk slots the scorer's warps reserve ahead of use
            uint64_t rec_cap = chunk * 2ULL * fin_cap + static_cast<uint64_t>(sms) * kTcRecReserve;
            if (const char* e = std::getenv("DETLSH_TEST_REC_CAP"))  // test hook: force the overflow path
                rec_cap = std::max<uint64_t>(1, std::min<uint64_t>(std::strtoull(e, nullptr, 10), rec_cap));
            grow_scratch(X.tc_bm, chunk * W);
            grow_scratch(X.tc_tau2, chunk);
            grow_scratch(X.tc_qn, chunk);
            grow_scratch(X.tc_surv_cnt, chunk);
            grow_scratch(X.tc_q8, chunk * R);
            grow_scratch(X.tc_surv, chunk * fin_cap);
            grow_scratch(X.tc_rec, rec_cap);
            grow_scratch(X.tc_rec_cnt, 1);
            grow_scratch(X.over_list, P.nq);
            grow_scratch(X.tc_big, chunk);
            for (uint64_t c0 = 0; c0 < P.nq; c0 += chunk) {
                const uint64_t m = std::min<uint64_t>(chunk, P.nq - c0);
                DETLSH_CUDA(cudaMemsetAsync(X.tc_tau2.get(), 0xff, m * 4, s));
                DETLSH_CUDA(cudaMemsetAsync(X.tc_surv_cnt.get(), 0, m * 4, s));
                DETLSH_CUDA(cudaMemsetAsync(X.counters.get() + kCntWork, 0, 4, s));
                DETLSH_CUDA(cudaMemsetAsync(X.counters.get() + kCntBig, 0, 4, s));
                QueryPlan Pc = Pp;
                Pc.q_begin = c0;
                Pc.q_end = c0 + m;
                Pc.tc_bm = X.tc_bm.get();
                Pc.tc_W = W;
                Pc.tc_tau2 = X.tc_tau2.get();
                Pc.tc_over_list = X.over_list.get();
                Pc.tc_over_n = X.counters.get() + kCntOver;
                launch_fast(Pc, !std::getenv("DETLSH_TEST_NO_TCO"));
                if (tc_f32)
                    launch_tc_pack_queries_f32(P.q, Pp.order, c0, m, P.d, R, X.tc_q8.get(),
                                               reinterpret_cast<float*>(X.tc_qn.get()), s);
                else
                    launch_tc_pack_queries(P.q, Pp.order, c0, m, P.d, R, X.tc_q8.get(), X.tc_qn.get(), s);
                TcScoreArgs a{};
                a.f32 = tc_f32 ? 1 : 0;
                a.rows = tc_f32 ? P.data_tcf : P.data_tc;
                a.xn = tc_f32 ? reinterpret_cast<const int32_t*>(P.xnf) : P.xn_u8;
                a.q8 = X.tc_q8.get();
                a.qn = X.tc_qn.get();
                a.tau2 = X.tc_tau2.get();
                a.bm = X.tc_bm.get();
                a.W = W;
                a.n = P.n;
                a.nq = m;
                a.R = R;
                a.surv_cnt = X.tc_surv_cnt.get();
                a.surv = X.tc_surv.get();
                a.cap = tc_cap;
                a.order = Pp.order;
                a.slot0 = c0;
                a.work = X.counters.get() + kCntWork;
                a.rec = X.tc_rec.get();
                a.rec_cnt = X.tc_rec_cnt.get();
                a.rec_cap = rec_cap;
                DETLSH_CUDA(cudaMemsetAsync(X.tc_rec_cnt.get(), 0, 8, s));
                launch_tc_score(a, device, s);
                // queries whose survivors overflowed (or whose chunk's pass
                // records did) are listed for the gather path below
                if (tc_f32)
                    launch_tc_finish_f32(a, P.perm0, P.data_leaf, P.q, P.d, P.k, P.r_min, P.budget, P.ids, P.dists,
                                         P.n_hits, P.radius, P.cands, X.over_list.get(), X.counters.get() + kCntOver,
                                         s);
                else
                    launch_tc_finish(a, P.perm0, P.k, P.r_min, P.budget, P.ids, P.dists, P.n_hits, P.radius,
                                     P.cands, X.over_list.get(), X.counters.get() + kCntOver, X.tc_big.get(),
                                     X.counters.get() + kCntBig, s);
                if (std::getenv("DETLSH_DEBUG_QUERY")) {  // survivor-count spread per chunk (syncs)
                    std::vector<uint32_t> sc(m);
                    uint32_t over = 0, slow = 0;
                    DETLSH_CUDA(cudaMemcpyAsync(sc.data(), X.tc_surv_cnt.get(), m * 4, cudaMemcpyDeviceToHost, s));
                    DETLSH_CUDA(cudaMemcpyAsync(&over, X.counters.get() + kCntOver, 4, cudaMemcpyDeviceToHost, s));
                    DETLSH_CUDA(cudaMemcpyAsync(&slow, X.counters.get() + kCntSlow, 4, cudaMemcpyDeviceToHost, s));
                    DETLSH_CUDA(cudaStreamSynchronize(s));
                    std::sort(sc.begin(), sc.end());
                    std::fprintf(stderr,
                                 "[query] chunk %llu+%llu slots=%zu chunk=%llu tau_rows=%llu cap=%u surv p50=%u p90=%u "
                                 "max=%u over_total=%u slow_total=%u\n",
                                 (unsigned long long)c0, (unsigned long long)m, slots, (unsigned long long)chunk,
                                 (unsigned long long)tau_rows, tc_cap, sc[m / 2], sc[m * 9 / 10], sc[m - 1], over, slow);
                }
            }
            // gather path for the listed queries: the count stays on the device
            QueryPlan Pc = Pp;
            Pc.order = X.over_list.get();
            Pc.q_begin = 0;
            Pc.q_end = P.nq;
            Pc.q_count = X.counters.get() + kCntOver;
            launch_fast(Pc);
        }
        if (Pp.phase_cycles && !capturing) {  // profiling only: the phase split is read back here
            unsigned long long ph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            DETLSH_CUDA(cudaMemcpyAsync(ph, Pp.phase_cycles, sizeof(ph), cudaMemcpyDeviceToHost, s));
            DETLSH_CUDA(cudaStreamSynchronize(s));
            std::lock_guard<std::mutex> lk(g_phase_mu);
            for (int i = 0; i < 8; ++i) g_phase[i] = static_cast<double>(ph[i]);
        }
    }
    {
        // deferred mode for large budgets (the member distances grid-wide);
        // DETLSH_SLOW_DEFER_MIN sets the budget threshold (test hook)
        uint64_t defer_min = kSlowDeferMinBudget;
        if (const char* e = std::getenv("DETLSH_SLOW_DEFER_MIN")) defer_min = std::strtoull(e, nullptr, 10);
        const bool defer = P.budget >= defer_min;
        static_assert(sizeof(SlowRec) == 3 * sizeof(uint64_t), "SlowRec layout");
        if (defer) grow_scratch(X.slow_rec, 3 * X.slow_slots);
        SlowRec* recs = defer ? reinterpret_cast<SlowRec*>(X.slow_rec.get()) : nullptr;
        QueryPlan Ps = P;
        Ps.phase_cycles = profiling_enabled() ? X.phases.get() : nullptr;
        {
            ProfScope ps("query_slow", s);
            slow_kernel<<<static_cast<unsigned>(gslots), slow_nt, smem, s>>>(
                Ps, fast_path ? X.slow_list.get() : nullptr, static_cast<uint32_t>(n_list),
                fast_path ? X.counters.get() + kCntSlow : nullptr, X.counters.get() + kCntTaken, X.slow.get(),
                slow_bytes, X.slow_bm.get(), bm_words, recs);
            DETLSH_LAUNCH_CHECK();
        }
        if (defer) {
            {
                ProfScope ps("query_slow_score", s);
                const unsigned gx = static_cast<unsigned>(std::max<int>(1, 4 * sms));
                slow_score_kernel<<<dim3(gx, static_cast<unsigned>(gslots)), 256, static_cast<size_t>(P.d) * 4, s>>>(
                    P, recs, X.slow.get(), slow_bytes);
                DETLSH_LAUNCH_CHECK();
            }
            ProfScope ps("query_slow_topk", s);
            slow_topk<<<static_cast<unsigned>(gslots), slow_nt, smem, s>>>(P, recs, X.slow.get(),
                                                                                    slow_bytes);
            DETLSH_LAUNCH_CHECK();
        }
    }
    if (profiling_enabled() && !capturing && std::getenv("DETLSH_DEBUG_QUERY")) {  // general-path phase split
        unsigned long long ph[10];
        DETLSH_CUDA(cudaMemcpyAsync(ph, X.phases.get() + 8, sizeof(ph), cudaMemcpyDeviceToHost, s));
        DETLSH_CUDA(cudaStreamSynchronize(s));
        std::fprintf(stderr, "[query] fast-path leaf scan: %llu of %llu leaves not certainly outside\n", ph[8], ph[9]);
        std::fprintf(stderr,
                     "[query] general path cycles: scan %llu select %llu emit %llu count %llu topk %llu | "
                     "leaf items %llu rounds %llu members+queries %llu\n",
                     ph[0], ph[1], ph[2], ph[3], ph[4], ph[5], ph[6], ph[7]);
    }
    if (!capturing) DETLSH_CUDA(cudaEventRecord(X.done, s));
}

bool query_invariant_failed(QueryScratch& X, cudaStream_t s) {
    if (!X.counters.get()) return false;
    uint32_t flag = 0;
    DETLSH_CUDA(cudaMemcpyAsync(&flag, X.counters.get() + kCntInvariant, 4, cudaMemcpyDeviceToHost, s));
    DETLSH_CUDA(cudaStreamSynchronize(s));
    return flag != 0;
}

void launch_merge_topk(const double* sd, const uint64_t* sid, const int32_t* sh, int shards,
                       uint64_t nq, int k, double* od, uint64_t* oid, int32_t* oh, cudaStream_t s) {
    if (shards < 1 || shards > kMergeMaxShards) throw InvalidArgument("merge_topk: 1 to 1024 shards");
    const unsigned grid = static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>((nq + 3) / 4, 65535)));
    merge_topk_kernel<<<grid, 128, 0, s>>>(sd, sid, sh, shards, nq, k, od, oid, oh);
    DETLSH_LAUNCH_CHECK();
}

}  // namespace detlsh_b200
