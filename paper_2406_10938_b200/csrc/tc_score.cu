// Tensor-core (tcgen05, kind::i8) building blocks for exact u8 verification.
// tc_gemm_u8_test: one 128 x N x K tile, C = A . B^T, used by the tests to pin
// the descriptor / TMEM plumbing before it is used in the query path.
#include <algorithm>

#include <cuda_bf16.h>

#include "common.cuh"
#include "query.cuh"
#include "umma.cuh"

namespace detlsh_b200 {

namespace {

__global__ void __launch_bounds__(128) tc_gemm_u8_test_kernel(const uint8_t* __restrict__ A,
                                                              const uint8_t* __restrict__ B, int N,
                                                              int K, int32_t* __restrict__ C) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tslot;
    uint8_t* sA = sm;
    uint8_t* sB = sm + 128 * K;
    const int tid = threadIdx.x;
    const int kch = K / 16;
    for (int i = tid; i < 128 * kch; i += blockDim.x) {
        const int r = i / kch, kc = i % kch;
        *reinterpret_cast<uint4*>(sA + umma::tile_off(r, kc, 128)) =
            reinterpret_cast<const uint4*>(A + static_cast<size_t>(r) * K)[kc];
    }
    for (int i = tid; i < N * kch; i += blockDim.x) {
        const int r = i / kch, kc = i % kch;
        *reinterpret_cast<uint4*>(sB + umma::tile_off(r, kc, N)) =
            reinterpret_cast<const uint4*>(B + static_cast<size_t>(r) * K)[kc];
    }
    if (tid == 0) {
        umma::mbar_init(&bar, 1);
        umma::fence_mbar_init();
    }
    umma::fence_async_smem();
    __syncthreads();
    if (tid < 32) umma::tmem_alloc(&tslot, 256);
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
    const uint32_t tmem = tslot;
    if (tid == 0) {
        const uint32_t idesc = umma::idesc_u8_s32(128, N);
        for (int s = 0; s < K / 32; ++s) {
            const uint64_t da = umma::smem_desc(umma::smem_u32(sA) + 2 * s * 128 * 16, 128 * 16, 128);
            const uint64_t db = umma::smem_desc(umma::smem_u32(sB) + 2 * s * N * 16, N * 16, 128);
            umma::mma_u8(tmem, da, db, idesc, s > 0 ? 1u : 0u);
        }
        umma::commit(&bar);
    }
    umma::mbar_wait(&bar, 0);
    umma::fence_after_sync();
    const int w = tid >> 5, lane = tid & 31;
    for (int c0 = 0; c0 < N; c0 += 32) {
        uint32_t v[32];
        umma::tmem_ld32(tmem + (static_cast<uint32_t>(32 * w) << 16) + c0, v);
#pragma unroll
        for (int i = 0; i < 32; ++i)
            if (c0 + i < N) C[(32 * w + lane) * N + c0 + i] = static_cast<int32_t>(v[i]);
    }
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
    if (tid < 32) umma::tmem_free(tmem, 256);
}

// ---------------------------------------------------------------------------
// Dataset-major exact verification for u8 data.
//
// For a batch of queries, the candidate SET of each query is a bitmap over the
// rows in tree-0 order (written by the plan kernel).  This kernel streams row
// tiles (128 rows) against query tiles (256 queries): one tcgen05 kind::i8
// MMA chain per tile computes every dot product q.x exactly in s32 (TMEM),
// then the epilogue keeps, for each (row, query) whose candidate bit is set,
// dist^2 = |q|^2 + |x|^2 - 2 q.x (exact integers) if it is <= the query's
// threshold tau^2 (the k-th smallest dist^2 of a subset of its candidates, so
// every true top-k member survives).  tc_finish ranks the survivors by
// (dist^2, position) exactly.
// ---------------------------------------------------------------------------
constexpr int kTcRows = 128;     // rows per tile (MMA M, TMEM lanes)
constexpr int kTcQueries = 256;  // queries per tile (MMA N, TMEM columns)

// Slot s of the batch <- query order[slot0 + s]: u8 row (non-integral values
// become 0; such queries never take the tensor-core path) and |q|^2.
__global__ void tc_pack_queries_kernel(const float* __restrict__ q, const uint32_t* __restrict__ order,
                                       uint64_t slot0, uint64_t m, int d, int R,
                                       uint8_t* __restrict__ q8, int32_t* __restrict__ qn) {
    const int lane = threadIdx.x & 31;  // one warp per slot
    for (uint64_t i = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5; i < m;
         i += (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5) {
        const uint64_t qi = order ? order[slot0 + i] : slot0 + i;
        int32_t s = 0;
        for (int t = lane; t < R; t += 32) {
            uint8_t b = 0;
            if (t < d) {
                const float v = q[qi * d + t];
                const bool integral = v >= 0.0f && v <= 255.0f && v == floorf(v);
                b = integral ? static_cast<uint8_t>(v) : 0;
            }
            q8[i * R + t] = b;
            s += static_cast<int32_t>(b) * b;
        }
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) qn[i] = s;
    }
}

__global__ void row_norms_u8_kernel(const uint8_t* __restrict__ rows, uint64_t n, int R,
                                    int32_t* __restrict__ xn) {
    for (uint64_t r = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; r < n;
         r += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint4* p = reinterpret_cast<const uint4*>(rows + r * R);
        uint32_t acc = 0;
        for (int c = 0; c < R / 16; ++c) {
            const uint4 v = __ldg(p + c);
            acc = __dp4a(v.x, v.x, acc);
            acc = __dp4a(v.y, v.y, acc);
            acc = __dp4a(v.z, v.z, acc);
            acc = __dp4a(v.w, v.w, acc);
        }
        xn[r] = static_cast<int32_t>(acc);
    }
}

// ---- float datasets: bf16-triple operands ------------------------------------
// x = x_hi + x_lo + r with x_hi = bf16(x), x_lo = bf16(x - x_hi), |r| <= 2^-16 |x|.
// Rows hold [x_hi, x_lo, x_hi] and queries [q_hi, q_hi, q_lo] along K, so one
// kind::f16 accumulation gives q_hi.x_hi + q_hi.x_lo + q_lo.x_hi: within
// ~2^-13.6 |q||x| of q.x (dropped lo.lo and residual terms, fp32 accumulation
// of 3 d exact bf16 products), inside kTcF32Kappa = 2^-12.
__device__ __forceinline__ uint16_t bf16_bits(float v) {
    return __bfloat16_as_ushort(__float2bfloat16_rn(v));
}
__device__ __forceinline__ float bf16_hi(float v) { return __bfloat162float(__float2bfloat16_rn(v)); }

// element e of a float row in the triple layout (K-major, zero past 3 d)
__device__ __forceinline__ uint16_t row_elem(const float* x, int d, int e) {
    if (e < d) return bf16_bits(x[e]);
    if (e < 2 * d) {
        const float v = x[e - d];
        return bf16_bits(__fsub_rn(v, bf16_hi(v)));  // exact: |v - hi| has fewer bits than v
    }
    if (e < 3 * d) return bf16_bits(x[e - 2 * d]);
    return 0;
}
__device__ __forceinline__ uint16_t query_elem(const float* q, int d, int e) {
    if (e < 2 * d) return bf16_bits(q[e < d ? e : e - d]);
    if (e < 3 * d) {
        const float v = q[e - 2 * d];
        return bf16_bits(__fsub_rn(v, bf16_hi(v)));
    }
    return 0;
}

// rows (tree-0 leaf order) -> 128-row tiles, chunk kc (8 elements) of row r at
// tile + kc * 2048 + r * 16; xnf[r] = (1 - kappa) |x_r|^2 rounded down
__global__ void pack_tcf_tiles_kernel(const float* __restrict__ rows, uint64_t n, int d, int R,
                                      uint8_t* __restrict__ tiles, float* __restrict__ xnf) {
    const int kch = R / 16;
    const uint64_t total = (n + kTcRows - 1) / kTcRows * kTcRows * kch;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t t = i / (static_cast<uint64_t>(kch) * kTcRows);
        const uint32_t rem = static_cast<uint32_t>(i % (static_cast<uint64_t>(kch) * kTcRows));
        const uint32_t kc = rem / kTcRows, r = rem % kTcRows;
        const uint64_t row = t * kTcRows + r;
        uint32_t w[4] = {0, 0, 0, 0};
        if (row < n) {
            const float* x = rows + row * d;
#pragma unroll
            for (int h = 0; h < 4; ++h)
                w[h] = row_elem(x, d, 8 * kc + 2 * h) | static_cast<uint32_t>(row_elem(x, d, 8 * kc + 2 * h + 1)) << 16;
        }
        reinterpret_cast<uint4*>(tiles)[i] = make_uint4(w[0], w[1], w[2], w[3]);
    }
    for (uint64_t row = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; row < n;
         row += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const float* x = rows + row * d;
        double s2 = 0.0;
        for (int t = 0; t < d; ++t) s2 = __fma_rn(static_cast<double>(x[t]), static_cast<double>(x[t]), s2);
        xnf[row] = __double2float_rd(s2 * (1.0 - static_cast<double>(kTcF32Kappa)) * (1.0 - 0x1p-40));
    }
}

// Slot s <- query order[slot0 + s]: [q_hi, q_hi, q_lo] bf16 (R bytes) and
// (1 - kappa)|q|^2 rounded down.
__global__ void tc_pack_queries_f32_kernel(const float* __restrict__ q, const uint32_t* __restrict__ order,
                                           uint64_t slot0, uint64_t m, int d, int R, uint8_t* __restrict__ q16,
                                           float* __restrict__ qnf) {
    const int lane = threadIdx.x & 31;  // one warp per slot
    for (uint64_t i = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5; i < m;
         i += (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5) {
        const uint64_t qi = order ? order[slot0 + i] : slot0 + i;
        const float* qv = q + qi * d;
        uint16_t* out = reinterpret_cast<uint16_t*>(q16 + i * R);
        for (int e = lane; e < R / 2; e += 32) out[e] = query_elem(qv, d, e);
        if (lane == 0) {
            double s2 = 0.0;
            for (int t = 0; t < d; ++t) s2 = __fma_rn(static_cast<double>(qv[t]), static_cast<double>(qv[t]), s2);
            qnf[i] = __double2float_rd(s2 * (1.0 - static_cast<double>(kTcF32Kappa)) * (1.0 - 0x1p-40));
        }
    }
}

// Exact top-k of each float query's survivors: the reference's fp64 distance
// (dataset.hpp:23-34: sequential (q - x)^2 sums, sqrt) per survivor row, then a
// bitonic sort by (distance, dataset position).
__global__ void __launch_bounds__(256) tc_finish_f32_kernel(TcScoreArgs a, const uint32_t* __restrict__ perm0,
                                                            const float* __restrict__ rows, const float* __restrict__ qs,
                                                            int d, int k, double r_min, uint64_t budget,
                                                            uint32_t* ids, double* dists, int32_t* n_hits,
                                                            double* radius, uint64_t* cands, uint32_t* overflow_list,
                                                            uint32_t* overflow_n) {
    extern __shared__ uint64_t fkey[];  // [cap2] distance bits, then [cap2] u32 positions
    uint32_t cap2 = 64;                 // the widest sort: a power of two >= cap
    while (cap2 < a.cap) cap2 <<= 1;
    uint32_t* fpos = reinterpret_cast<uint32_t*>(fkey + cap2);
    const bool rec_over = *a.rec_cnt > a.rec_cap;
    for (uint64_t slot = blockIdx.x; slot < a.nq; slot += gridDim.x) {
        if (a.tau2[slot] < 0) continue;
        const uint64_t q = a.order ? a.order[a.slot0 + slot] : a.slot0 + slot;
        const uint32_t cnt = a.surv_cnt[slot];
        if (rec_over || cnt > a.cap) {
            if (threadIdx.x == 0) overflow_list[atomicAdd(overflow_n, 1u)] = static_cast<uint32_t>(q);
            continue;
        }
        uint32_t n2 = 64;
        while (n2 < cnt) n2 <<= 1;
        const float* qv = qs + q * d;
        for (uint32_t i = threadIdx.x; i < n2; i += blockDim.x) {
            uint64_t kd = ~0ULL;
            uint32_t kp = 0xffffffffu;
            if (i < cnt) {
                const uint32_t row = static_cast<uint32_t>(a.surv[slot * a.cap + i]);
                const float* x = rows + static_cast<uint64_t>(row) * d;
                double acc = 0.0;
                for (int t = 0; t < d; ++t) {
                    const double df = __dsub_rn(static_cast<double>(__ldg(qv + t)), static_cast<double>(__ldg(x + t)));
                    acc = __dadd_rn(acc, __dmul_rn(df, df));
                }
                kd = static_cast<uint64_t>(__double_as_longlong(__dsqrt_rn(acc)));
                kp = __ldg(perm0 + row);
            }
            fkey[i] = kd;
            fpos[i] = kp;
        }
        __syncthreads();
        for (uint32_t size = 2; size <= n2; size <<= 1) {
            for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
                for (uint32_t i = threadIdx.x; i < n2 / 2; i += blockDim.x) {
                    const int lo = 2 * i - (i & (stride - 1));
                    const int hi = lo + stride;
                    const bool asc = (lo & size) == 0;
                    const uint64_t x = fkey[lo], y = fkey[hi];
                    const uint32_t px = fpos[lo], py = fpos[hi];
                    const bool y_less = y < x || (y == x && py < px);
                    if (y_less == asc) {
                        fkey[lo] = y;
                        fkey[hi] = x;
                        fpos[lo] = py;
                        fpos[hi] = px;
                    }
                }
                __syncthreads();
            }
        }
        const uint32_t nh = min(cnt, static_cast<uint32_t>(k));
        for (uint32_t t = threadIdx.x; t < nh; t += blockDim.x) {
            if (ids) ids[q * k + t] = fpos[t];
            if (dists) dists[q * k + t] = __longlong_as_double(static_cast<long long>(fkey[t]));
        }
        if (threadIdx.x == 0) {
            if (n_hits) n_hits[q] = static_cast<int32_t>(nh);
            if (radius) radius[q] = r_min;
            if (cands) cands[q] = budget;
        }
        __syncthreads();
    }
}

// Rows -> HBM tiles of 128 rows in the canonical no-swizzle K-major layout
// (chunk kc of row r at kc * 2048 + r * 16), zero rows past n: one tile is one
// contiguous 128 * R byte block, moved by a single bulk copy.
__global__ void pack_tc_tiles_kernel(const uint8_t* __restrict__ rows, uint64_t n, int R,
                                     uint8_t* __restrict__ tiles) {
    const int kch = R / 16;
    const uint64_t total = (n + kTcRows - 1) / kTcRows * kTcRows * kch;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        // i enumerates destination chunks in order: tile, kc, row
        const uint64_t t = i / (static_cast<uint64_t>(kch) * kTcRows);
        const uint32_t rem = static_cast<uint32_t>(i % (static_cast<uint64_t>(kch) * kTcRows));
        const uint32_t kc = rem / kTcRows, r = rem % kTcRows;
        const uint64_t row = t * kTcRows + r;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (row < n) v = __ldg(reinterpret_cast<const uint4*>(rows + row * R) + kc);
        reinterpret_cast<uint4*>(tiles)[i] = v;
    }
}

// Warp-specialised, persistent: warp EW (the producer) streams row tiles
// (pre-tiled in HBM in the canonical no-swizzle K-major layout, one 1-D bulk
// copy per tile, or per 256-byte K chunk) into a staging ring; warp EW + 1
// issues the tcgen05 MMAs into one of two TMEM accumulators (2 x 256 columns,
// one MMA per query half); warps 0 .. EW-1 drain the other one.  Work units
// (query tile, row-tile range) are handed out dynamically; every row tile of
// a unit is scored (the candidate sets of a locality-ordered 256-query tile
// reach almost every tile).  The epilogue is branch-free: 2 q.x + (tau^2 -
// |q|^2) - |x|^2 >= 0 per element (IMAD, IMAD, funnel shift of the sign into
// a fail mask); only columns where some lane passes and whose query has a
// candidate in these 32 rows are revisited, from a shared-memory stash of the
// loaded values, to write pass records.
// Two shapes of the same kernel: QT queries per tile, EW epilogue warps (4 per
// TMEM lane quarter per 4-warp group).  Rows of R <= 256 bytes: 256-query
// tiles, 16 epilogue warps, whole row tiles per stage.  Wider rows (C3,
// d = 784): the 256-query operand would not fit beside the row stages, so
// 128-query tiles, 8 epilogue warps, and row tiles streamed in 256-byte K
// chunks (32 KB per stage, accumulated in TMEM across the chunks).
constexpr int kEpiWarps = 16;                      // the wide-tile shape's epilogue warps (scratch sizing)
constexpr uint32_t kTcRecChunk = 1024;  // records reserved per warp at a time
static_assert(kTcRecReserve >= static_cast<uint64_t>(kEpiWarps) * kTcRecChunk, "rec_cap slack");
constexpr uint32_t kTcChunkBytes = kTcRows * 256;  // one 256-byte K chunk of a 128-row tile
constexpr int kTcStash = 36;             // words per lane of the rare-path stash (bank spread)
constexpr uint32_t kWaitHintNs = 20000;  // mbarrier try_wait suspend hint (woken on completion)
#ifndef DETLSH_TC_QSPLIT
#define DETLSH_TC_QSPLIT 2
#endif
constexpr int kQSplitMax = 2;            // MMAs (and accumulator barriers) per tile, one per query part (4: slower)

__host__ __device__ __forceinline__ uint32_t tc_stages(int R) { return R <= 128 ? 3u : 2u; }
// the K-chunked shape (R > 256, 128-query tiles, 8 epilogue warps): three
// 32 KB row-chunk stages when they fit beside the query tile, else two
__host__ __device__ __forceinline__ uint32_t tc_chunk_stages(int R) {
    const uint32_t fixed = 128u * static_cast<uint32_t>(R) + 2u * 128u * 4u + 8u * 32u * static_cast<uint32_t>(kTcStash) * 4u +
                           1024u + 2048u;  // (+ static smem, alignment)
    return fixed + 3u * kTcChunkBytes <= 227u * 1024u ? 3u : 2u;
}

// A warp's next run of kTcRecChunk record slots; the unused tail of the old
// run becomes padding.  (Called warp-uniformly.)
__device__ __noinline__ void tc_reserve(uint4* rec, unsigned long long* rec_cnt, uint64_t rec_cap, uint64_t& next,
                                        uint64_t& end, int lane) {
    for (uint64_t x = next + lane; x < end && x < rec_cap; x += 32) rec[x] = make_uint4(0xffffffffu, 0, 0, 0);
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(rec_cnt, static_cast<unsigned long long>(kTcRecChunk));
    base = __shfl_sync(0xffffffffu, base, 0);
    next = base;
    end = base + kTcRecChunk;
}

template <int QT, int EW, bool F32>
__global__ void __launch_bounds__(32 * (EW + 2), 1) tc_score_kernel(TcScoreArgs a, uint32_t n_rt, uint32_t n_qt,
                                                                   uint32_t G) {
    constexpr int kTcQueries = QT, kEpiWarps = EW;
    // one MMA per query part: two 128-query parts for 256-query tiles (each
    // part's epilogue warps wait only for their own MMA); one 128-wide MMA for
    // 128-query tiles (N = 64 halves measured ~2x slower on the bf16 path)
    constexpr int kQSplit = QT >= 256 ? DETLSH_TC_QSPLIT : 1;
    constexpr int kEpiCols = kTcQueries / (kEpiWarps / 4);  // query columns per epilogue warp
    constexpr int kEpiWords = kEpiCols / 32;                // candidate words per lane (columns per lane)
    constexpr int kProducerWarp = kEpiWarps, kMmaWarp = kEpiWarps + 1;
    extern __shared__ __align__(1024) uint8_t sm[];
    // tfull/tempty per (accumulator, query part): the kQSplit query parts of a
    // tile are separate MMAs, so the epilogue warps of one part never wait for
    // another part's stragglers
    __shared__ __align__(8) uint64_t full[6], empty[6], tfull[2][kQSplitMax], tempty[2][kQSplitMax];
    __shared__ uint32_t tslot, unit_s;
    const int R = a.R, kch = R / 16;
    const bool chunked = R > 256;  // rows streamed in 256-byte K chunks
    const uint32_t stages = chunked ? tc_chunk_stages(R) : tc_stages(R);
    const uint32_t tile_bytes = static_cast<uint32_t>(kTcRows * R);
    const uint32_t nkc = chunked ? static_cast<uint32_t>((kch + 15) / 16) : 1u;  // K chunks per row tile
    const uint32_t stage_bytes = chunked ? kTcChunkBytes : tile_bytes;
    uint8_t* sB = sm;                                    // [QT][R] core layout
    uint8_t* sA = sB + kTcQueries * R;                   // [stages][128][R or 256] core layout
    int32_t* snh = reinterpret_cast<int32_t*>(sA + stages * stage_bytes);  // tau^2 - |q|^2
    int32_t* sqn = snh + kTcQueries;
    uint32_t* sstash = reinterpret_cast<uint32_t*>(sqn + kTcQueries);  // [kEpiWarps][32 lanes][kTcStash]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) {
        for (uint32_t s = 0; s < stages; ++s) {
            umma::mbar_init(&full[s], 1);
            umma::mbar_init(&empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            for (int h = 0; h < kQSplit; ++h) {
                umma::mbar_init(&tfull[s][h], 1);
                umma::mbar_init(&tempty[s][h], kEpiWarps / kQSplit);
            }
        }
        umma::fence_mbar_init();
    }
    if (warp == kMmaWarp) umma::tmem_alloc(&tslot, 512);
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
    const uint32_t tmem = tslot;
    const uint32_t idesc = F32 ? umma::idesc_bf16_f32(kTcRows, kTcQueries / kQSplit)  // one query part per MMA
                               : umma::idesc_u8_s32(kTcRows, kTcQueries / kQSplit);
    const uint32_t units = n_qt * G;
    uint32_t it = 0;  // tiles processed by this CTA so far (accumulator phases)
    uint32_t ic = 0;  // row-tile K chunks loaded so far (stage phases; == it unless chunked)
    uint32_t loaded_qt = 0xffffffffu;
    uint64_t res_next = 0, res_end = 0;  // this warp's reservation in a.rec
    for (;;) {
        if (tid == 0) unit_s = atomicAdd(a.work, 1u);
        __syncthreads();
        const uint32_t u = unit_s;
        __syncthreads();  // unit_s is rewritten next iteration
        if (u >= units) break;
        // query-tile-minor: CTAs running at the same time stream the same row
        // range for different query tiles, so each row tile comes from HBM once
        const uint32_t qt = u % n_qt, g = u / n_qt;
        const uint32_t rt0 = static_cast<uint32_t>(static_cast<uint64_t>(n_rt) * g / G);
        const uint32_t rt1 = static_cast<uint32_t>(static_cast<uint64_t>(n_rt) * (g + 1) / G);
        const uint64_t q0 = static_cast<uint64_t>(qt) * kTcQueries;
        // dense: each query tile's candidates reach nearly every row tile, so
        // every tile of the range is scored (no per-tile occupancy lookups)
        const uint32_t ntiles = rt1 - rt0;
        if (ntiles == 0) continue;  // uniform
        if (qt != loaded_qt) {  // every MMA of the previous unit has completed (epilogue drained it)
            for (int i = tid; i < kTcQueries * kch; i += blockDim.x) {
                const int kc = i / kTcQueries, r = i % kTcQueries;
                const uint64_t qq = q0 + r;
                uint4 v = make_uint4(0, 0, 0, 0);
                if (qq < a.nq) v = __ldg(reinterpret_cast<const uint4*>(a.q8 + qq * R) + kc);
                *reinterpret_cast<uint4*>(sB + umma::tile_off(r, kc, kTcQueries)) = v;
            }
            for (int r = tid; r < kTcQueries; r += blockDim.x) {
                const uint64_t qq = q0 + r;
                const int32_t t = qq < a.nq ? a.tau2[qq] : -1;
                const int32_t qn = qq < a.nq ? a.qn[qq] : 0;
                sqn[r] = qn;
                if (F32)  // tau^2 - (1 - kappa)|q|^2, rounded up (the filter only ever widens)
                    snh[r] = __float_as_int(t < 0 ? -3.0e38f : __fsub_ru(__int_as_float(t), __int_as_float(qn)));
                else
                    snh[r] = t < 0 ? -0x20000000 : t - qn;  // -2^29: no row can pass
            }
            umma::fence_async_smem();
            umma::fence_before_sync();
            __syncthreads();
            umma::fence_after_sync();
            loaded_qt = qt;
        }
        if (warp == kProducerWarp) {
            if (lane == 0) {
                for (uint32_t t = rt0, j = 0; t < rt1; ++t) {
                    for (uint32_t c = 0; c < nkc; ++c, ++j) {
                        const uint32_t i = ic + j, s = i % stages, ph = (i / stages) & 1;
                        // chunk c: 16-byte K columns [16 c, 16 c + 16) of the tile, contiguous
                        const uint32_t bytes = chunked ? min(16u, static_cast<uint32_t>(kch) - 16u * c) * kTcRows * 16u
                                                       : tile_bytes;
                        umma::mbar_wait_hint(&empty[s], ph ^ 1, kWaitHintNs);
                        umma::mbar_arrive_expect_tx(&full[s], bytes);
                        umma::bulk_g2s(sA + s * stage_bytes,
                                       a.rows + static_cast<uint64_t>(t) * tile_bytes + c * kTcChunkBytes, bytes,
                                       &full[s]);
                    }
                }
            }
        } else if (warp == kMmaWarp) {
            if (lane == 0) {
                for (uint32_t t = rt0, j = 0, jc = 0; t < rt1; ++t, ++j) {
                    const uint32_t i = it + j;
                    const uint32_t acc = i & 1, aph = (i >> 1) & 1;
                    for (uint32_t c = 0; c < nkc; ++c, ++jc) {
                        const uint32_t ii = ic + jc, s = ii % stages, ph = (ii / stages) & 1;
                        const int ksteps = chunked ? static_cast<int>(min(16u, static_cast<uint32_t>(kch) - 16u * c)) / 2
                                                   : R / 32;
                        umma::mbar_wait_hint(&full[s], ph, kWaitHintNs);
                        const uint32_t a0 = umma::smem_u32(sA + s * stage_bytes), b0 = umma::smem_u32(sB);
                        for (int h = 0; h < kQSplit; ++h) {
                            if (c == 0) umma::mbar_wait_hint(&tempty[acc][h], aph ^ 1, kWaitHintNs);
                            umma::fence_after_sync();
                            // part h's queries start (QT / kQSplit) / 8 eight-row groups in (K-major core layout)
                            constexpr int kQP = kTcQueries / kQSplit;
                            for (int k = 0; k < ksteps; ++k) {
                                const int kg = static_cast<int>(8 * c) + k;  // K step within the whole row
                                const uint64_t da = umma::smem_desc(a0 + 2 * k * kTcRows * 16, kTcRows * 16, 128);
                                const uint64_t db = umma::smem_desc(b0 + 2 * kg * kTcQueries * 16 + h * kQP * 16,
                                                                    kTcQueries * 16, 128);
                                if (F32)
                                    umma::mma_f16(tmem + acc * kTcQueries + h * kQP, da, db, idesc,
                                                  (c > 0 || k > 0) ? 1u : 0u);
                                else
                                    umma::mma_u8(tmem + acc * kTcQueries + h * kQP, da, db, idesc,
                                                 (c > 0 || k > 0) ? 1u : 0u);
                            }
                            if (c + 1 == nkc) umma::commit(&tfull[acc][h]);
                        }
                        umma::commit(&empty[s]);
                    }
                }
            }
        } else {
            const int sub = warp & 3, part = warp >> 2;
            const int half = part * kQSplit / (kEpiWarps / 4);  // this warp's MMA query part
            const int row = sub * 32 + lane;
            const int cbeg = part * kEpiCols;  // this warp's query columns [cbeg, cbeg + kEpiCols)
            // candidate words of this warp's 32 rows for its query columns (lane l
            // holds column cbeg + 32 e + l in slot e: chunk e's words sit in one
            // register across the warp), prefetched one tile ahead
            // (per-lane row pointers hoisted out of the tile loop; a query
            // past the batch reads nothing)
            const uint32_t* wrow[kEpiWords];
#pragma unroll
            for (int e = 0; e < kEpiWords; ++e) {
                const uint64_t qq = q0 + cbeg + 32 * e + lane;
                wrow[e] = qq < a.nq ? a.bm + qq * a.W + sub : nullptr;
            }
            auto load_words = [&](uint32_t t, uint32_t (&w)[kEpiWords]) {
                const bool in = static_cast<uint64_t>(t) * 4 + sub < a.W;
#pragma unroll
                for (int e = 0; e < kEpiWords; ++e) w[e] = (in && wrow[e]) ? __ldg(wrow[e] + 4ull * t) : 0u;
            };
            const int32_t one = 1 + static_cast<int32_t>(a.n >> 62), two = one + one;  // 1, 2 at run time
            uint32_t pw[kEpiWords], nw[kEpiWords];
#pragma unroll
            for (int e = 0; e < kEpiWords; ++e) nw[e] = 0;
            load_words(rt0, pw);
            const uint32_t lt_mask = (1u << lane) - 1u;
            for (uint32_t t = rt0, j = 0; t < rt1; ++t, ++j) {
                const uint32_t i = it + j, acc = i & 1, aph = (i >> 1) & 1;
                const uint64_t r = static_cast<uint64_t>(t) * kTcRows + row;
                // padded rows never pass (integers: 2^30; floats: +3e38)
                const int32_t xn = r < a.n ? __ldg(a.xn + r) : (F32 ? __float_as_int(3.0e38f) : 0x40000000);
                const int32_t nxn = F32 ? (xn ^ static_cast<int32_t>(0x80000000u)) : -xn;  // float: flip the sign
                const uint32_t tn = t + 1;
                if (tn < rt1) load_words(tn, nw);  // next tile's words, in flight during this one
                umma::mbar_wait_hint(&tfull[acc][half], aph, kWaitHintNs);
                umma::fence_after_sync();
                const uint32_t tbase = tmem + (static_cast<uint32_t>(sub * 32) << 16) + acc * kTcQueries;
#pragma unroll
                for (int k = 0; k < kEpiWords; ++k) {
                    const int c0 = cbeg + 32 * k;
                    uint32_t v[32];
                    umma::tmem_ld32(tbase + c0, v);
                    if (k == kEpiWords - 1) {  // this warp's last TMEM read of the tile: release the
                        umma::fence_before_sync();  // accumulator before testing (the MMA two tiles
                        __syncwarp();               // ahead can start while the values are in registers)
                        if (lane == 0) umma::mbar_arrive(&tempty[acc][half]);
                    }
                    // threshold mask: bit e <=> 2 q.x + tau^2 - |q|^2 - |x|^2 >= 0.
                    // t = (2 v + h) - |x|^2 as two IMADs (FMA pipe: `two`/`one`
                    // are opaque to the compiler, which would otherwise pick
                    // ALU adds), its sign bit funnel-shifted into a fail mask
                    // (one ALU op per element; |t| < 2^31 by the bounds above)
                    // (four independent 8-column chains keep the shifts off
                    // each other's latency)
                    uint32_t fail[4] = {0, 0, 0, 0};
                    const int4* nh4 = reinterpret_cast<const int4*>(snh + c0);
                    auto step = [&](uint32_t& f, uint32_t vv, int32_t h) {
                        if (F32) {  // 2 acc + h - (1 - kappa)|x|^2 < 0: sign bit
                            const float t = __fadd_rn(__fmaf_rn(__uint_as_float(vv), 2.0f, __int_as_float(h)),
                                                      __int_as_float(nxn));
                            f = __funnelshift_l(__float_as_uint(t), f, 1);
                        } else {
                            const int32_t t = static_cast<int32_t>(vv) * two + h;
                            f = __funnelshift_l(static_cast<uint32_t>(t * one + nxn), f, 1);
                        }
                    };
#pragma unroll
                    for (int e4 = 1; e4 >= 0; --e4) {
#pragma unroll
                        for (int g = 0; g < 4; ++g) {  // chain g: columns 8g .. 8g+7
                            const int4 h = nh4[2 * g + e4];
                            step(fail[g], v[8 * g + 4 * e4 + 3], h.w);
                            step(fail[g], v[8 * g + 4 * e4 + 2], h.z);
                            step(fail[g], v[8 * g + 4 * e4 + 1], h.y);
                            step(fail[g], v[8 * g + 4 * e4 + 0], h.x);
                        }
                    }
                    const uint32_t mask = ~(fail[0] | fail[1] << 8 | fail[2] << 16 | fail[3] << 24);
                    // rare: columns where some lane passed.  The chunk's values are
                    // stashed in shared memory so this loop stays small and indexes
                    // them dynamically; candidate (row, query, dist^2) records go to
                    // a global list through a per-warp reservation (no round trip on
                    // the critical path)
                    // (only columns whose 32-row block holds a candidate: ~16% on C2)
                    uint32_t cols = __reduce_or_sync(0xffffffffu, mask) & __ballot_sync(0xffffffffu, pw[k] != 0u);
                    if (cols) {
                        uint32_t* sv = sstash + (warp * 32 + lane) * kTcStash;
#pragma unroll
                        for (int e4 = 0; e4 < 8; ++e4)
                            *reinterpret_cast<uint4*>(sv + 4 * e4) =
                                make_uint4(v[4 * e4], v[4 * e4 + 1], v[4 * e4 + 2], v[4 * e4 + 3]);
                        while (cols) {
                            const int e = __ffs(cols) - 1;
                            cols &= cols - 1;
                            const uint32_t b = __ballot_sync(0xffffffffu, (mask >> e) & 1u) &
                                               __shfl_sync(0xffffffffu, pw[k], e);  // lane e holds column c0 + e
                            if (!b) continue;
                            const uint32_t cnt = __popc(b);
                            if (res_next + cnt > res_end) tc_reserve(a.rec, a.rec_cnt, a.rec_cap, res_next, res_end, lane);
                            const uint64_t slot = res_next + __popc(b & lt_mask);
                            res_next += cnt;
                            if (((b >> lane) & 1u) && slot < a.rec_cap) {
                                const int c = c0 + e;
                                a.rec[slot] = make_uint4(static_cast<uint32_t>(r), static_cast<uint32_t>(q0 + c),
                                                         F32 ? 0u : static_cast<uint32_t>(sqn[c] + xn - 2 * static_cast<int32_t>(sv[e])),
                                                         0);
                            }
                        }
                        __syncwarp();
                    }
                }
#pragma unroll
                for (int e = 0; e < kEpiWords; ++e) pw[e] = nw[e];
            }
        }
        it += ntiles;
        ic += ntiles * nkc;
        umma::fence_before_sync();
        __syncthreads();
        umma::fence_after_sync();
    }
    for (uint64_t x = res_next + lane; x < res_end && x < a.rec_cap; x += 32) a.rec[x] = make_uint4(0xffffffffu, 0, 0, 0);
    if (warp == kMmaWarp) umma::tmem_free(tmem, 512);
}

// Candidate threshold passes -> per-query survivor lists.
__global__ void tc_collect_kernel(TcScoreArgs a) {
    const uint64_t total = min(static_cast<uint64_t>(*a.rec_cnt), a.rec_cap);
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint4 e = a.rec[i];
        if (e.x == 0xffffffffu) continue;
        const uint32_t slot = atomicAdd(a.surv_cnt + e.y, 1u);
        if (slot < a.cap) a.surv[static_cast<uint64_t>(e.y) * a.cap + slot] = (static_cast<uint64_t>(e.z) << 32) | e.x;
    }
}

// Exact top-k of each TC query's survivors by (dist^2, dataset position).
// Two launches: the first sorts up to `width` survivors per query (small
// shared memory, many CTAs per SM) and lists the queries with more in
// big_list; the second (width = the staging cap) takes only those.
__global__ void __launch_bounds__(256) tc_finish_kernel(TcScoreArgs a, const uint32_t* __restrict__ perm0,
                                                        int k, double r_min, uint64_t budget,
                                                        uint32_t* ids, double* dists, int32_t* n_hits,
                                                        double* radius, uint64_t* cands,
                                                        uint32_t* overflow_list, uint32_t* overflow_n,
                                                        uint32_t width, uint32_t* big_list, uint32_t* big_n,
                                                        const uint32_t* only_list, const uint32_t* only_n) {
    extern __shared__ uint64_t key[];  // [width] (d2 << 32) | position, sorted ascending
    // the pass-record list overflowed: no survivor list of this chunk is
    // complete, so every tensor-core query of the chunk takes the gather path
    const bool rec_over = *a.rec_cnt > a.rec_cap;
    const uint64_t nslots = only_list ? *only_n : a.nq;
    for (uint64_t it = blockIdx.x; it < nslots; it += gridDim.x) {
        const uint64_t slot = only_list ? only_list[it] : it;
        if (a.tau2[slot] < 0) continue;
        const uint64_t q = a.order ? a.order[a.slot0 + slot] : a.slot0 + slot;
        const uint32_t cnt = a.surv_cnt[slot];
        if (rec_over || cnt > a.cap) {  // threshold too loose for the staging: rerun on the gather path
            if (threadIdx.x == 0) overflow_list[atomicAdd(overflow_n, 1u)] = static_cast<uint32_t>(q);
            continue;
        }
        if (cnt > width) {  // (first launch only: width < cap)
            if (threadIdx.x == 0) big_list[atomicAdd(big_n, 1u)] = static_cast<uint32_t>(slot);
            continue;
        }
        uint32_t n2 = 64;  // sort width: power of two >= cnt
        while (n2 < cnt) n2 <<= 1;
        for (uint32_t i = threadIdx.x; i < n2; i += blockDim.x) {
            uint64_t kk = ~0ULL;
            if (i < cnt) {
                const uint64_t s = a.surv[slot * a.cap + i];
                kk = (s & 0xffffffff00000000ULL) | __ldg(perm0 + static_cast<uint32_t>(s));
            }
            key[i] = kk;
        }
        __syncthreads();
        for (uint32_t size = 2; size <= n2; size <<= 1) {
            for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
                for (uint32_t i = threadIdx.x; i < n2 / 2; i += blockDim.x) {
                    const int lo = 2 * i - (i & (stride - 1));
                    const int hi = lo + stride;
                    const bool asc = (lo & size) == 0;
                    const uint64_t x = key[lo], y = key[hi];
                    if ((y < x) == asc) {
                        key[lo] = y;
                        key[hi] = x;
                    }
                }
                __syncthreads();
            }
        }
        const uint32_t nh = min(cnt, static_cast<uint32_t>(k));
        for (uint32_t t = threadIdx.x; t < nh; t += blockDim.x) {
            const uint64_t kk = key[t];
            if (ids) ids[q * k + t] = static_cast<uint32_t>(kk);
            if (dists) dists[q * k + t] = __dsqrt_rn(static_cast<double>(kk >> 32));
        }
        if (threadIdx.x == 0) {
            if (n_hits) n_hits[q] = static_cast<int32_t>(nh);
            if (radius) radius[q] = r_min;
            if (cands) cands[q] = budget;
        }
        __syncthreads();
    }
}

}  // namespace

size_t tc_score_smem(int R) {
    const bool chunked = R > 256;
    const size_t qt = chunked ? 128 : kTcQueries, ew = chunked ? 8 : 16;
    const size_t rows = chunked ? static_cast<size_t>(tc_chunk_stages(R)) * kTcChunkBytes
                                : static_cast<size_t>(tc_stages(R)) * kTcRows * R;
    const size_t need = qt * R + rows + 2 * qt * 4 + ew * 32 * kTcStash * 4 + 1024;
    return std::max<size_t>(need, 120 * 1024);  // one CTA per SM: it owns all 512 TMEM columns
}

bool tc_score_fits(int R) { return R % 32 == 0 && tc_score_smem(R) <= 227 * 1024; }

void launch_tc_pack_queries(const float* q, const uint32_t* order, uint64_t slot0, uint64_t m, int d,
                            int R, uint8_t* q8, int32_t* qn, cudaStream_t s) {
    const unsigned grid = static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>((m * 32 + 255) / 256, 8192)));
    tc_pack_queries_kernel<<<grid, 256, 0, s>>>(q, order, slot0, m, d, R, q8, qn);
    DETLSH_LAUNCH_CHECK();
}

void launch_row_norms_u8(const uint8_t* rows, uint64_t n, int R, int32_t* xn, cudaStream_t s) {
    const unsigned grid = static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, 8192)));
    row_norms_u8_kernel<<<grid, 256, 0, s>>>(rows, n, R, xn);
    DETLSH_LAUNCH_CHECK();
}

void launch_tc_score(const TcScoreArgs& a, int device, cudaStream_t s) {
    const uint32_t n_rt = static_cast<uint32_t>((a.n + kTcRows - 1) / kTcRows);
    const bool chunked = a.R > 256;
    const uint32_t qt = chunked ? 128u : static_cast<uint32_t>(kTcQueries);
    const uint32_t n_qt = static_cast<uint32_t>((a.nq + qt - 1) / qt);
    const size_t smem = tc_score_smem(a.R);
    auto* const kern = a.f32 ? &tc_score_kernel<128, 8, true>
                             : chunked ? &tc_score_kernel<128, 8, false> : &tc_score_kernel<kTcQueries, 16, false>;
    if (a.f32 && !chunked) throw InvalidArgument("tc_score: float rows are bf16 triples of more than 256 bytes");
    const int threads = chunked ? 32 * (8 + 2) : 32 * (16 + 2);
    DETLSH_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    // persistent: one CTA per SM; work units = (query tile, row-tile range),
    // about 8 per CTA, handed out by an atomic counter
    const uint32_t sms = static_cast<uint32_t>(sm_count(device));
    // row ranges of at most ~8 MB: the CTAs working on one range at the same
    // time (one per query tile) then read it from L2, not each from HBM
    // (C4's 5.8 GB of bf16 rows; C2's 128 MB of u8 rows fit L2 whole)
    const uint64_t row_bytes_all = static_cast<uint64_t>(n_rt) * kTcRows * a.R;
    const uint32_t g_l2 = static_cast<uint32_t>(std::min<uint64_t>(n_rt, (row_bytes_all + (8u << 20) - 1) >> 23));
    const uint32_t G = std::max<uint32_t>(
        std::max<uint32_t>(1, std::min<uint32_t>((n_rt + 7) / 8, (8 * sms + n_qt - 1) / n_qt)), g_l2);
    const uint32_t grid = std::min<uint32_t>(sms, n_qt * G);
    {
        ProfScope ps("tc_score", s);
        kern<<<grid, threads, smem, s>>>(a, n_rt, n_qt, G);
        DETLSH_LAUNCH_CHECK();
    }
    ProfScope ps("tc_collect", s);
    tc_collect_kernel<<<sms * 8, 256, 0, s>>>(a);
    DETLSH_LAUNCH_CHECK();
}

void launch_pack_tcf_tiles(const float* rows_leaf, uint64_t n, int d, int R, uint8_t* tiles, float* xnf,
                           cudaStream_t s) {
    const uint64_t chunks = (n + kTcRows - 1) / kTcRows * kTcRows * (R / 16);
    const unsigned grid = static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>((chunks + 255) / 256, 16384)));
    pack_tcf_tiles_kernel<<<grid, 256, 0, s>>>(rows_leaf, n, d, R, tiles, xnf);
    DETLSH_LAUNCH_CHECK();
}

void launch_tc_pack_queries_f32(const float* q, const uint32_t* order, uint64_t slot0, uint64_t m, int d, int R,
                                uint8_t* q16, float* qnf, cudaStream_t s) {
    const unsigned grid = static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>((m * 32 + 255) / 256, 8192)));
    tc_pack_queries_f32_kernel<<<grid, 256, 0, s>>>(q, order, slot0, m, d, R, q16, qnf);
    DETLSH_LAUNCH_CHECK();
}

void launch_tc_finish_f32(const TcScoreArgs& a, const uint32_t* perm0, const float* rows_leaf, const float* q,
                          int d, int k, double r_min, uint64_t budget, uint32_t* ids, double* dists,
                          int32_t* n_hits, double* radius, uint64_t* cands, uint32_t* overflow_list,
                          uint32_t* overflow_n, cudaStream_t s) {
    const unsigned grid = static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>(a.nq, 4096)));
    uint32_t cap2 = 64;
    while (cap2 < a.cap) cap2 <<= 1;
    const size_t smem = static_cast<size_t>(cap2) * 12;
    static bool attr = false;
    if (!attr) {
        DETLSH_CUDA(cudaFuncSetAttribute(tc_finish_f32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(kTcFinishCapF32 * 12)));
        attr = true;
    }
    ProfScope ps("tc_finish", s);
    tc_finish_f32_kernel<<<grid, 256, smem, s>>>(a, perm0, rows_leaf, q, d, k, r_min, budget, ids, dists, n_hits,
                                                 radius, cands, overflow_list, overflow_n);
    DETLSH_LAUNCH_CHECK();
}

void launch_pack_tc_tiles(const uint8_t* rows, uint64_t n, int R, uint8_t* tiles, cudaStream_t s) {
    const uint64_t chunks = (n + kTcRows - 1) / kTcRows * kTcRows * (R / 16);
    const unsigned grid = static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>((chunks + 255) / 256, 16384)));
    pack_tc_tiles_kernel<<<grid, 256, 0, s>>>(rows, n, R, tiles);
    DETLSH_LAUNCH_CHECK();
}

void launch_tc_finish(const TcScoreArgs& a, const uint32_t* perm0, int k, double r_min,
                      uint64_t budget, uint32_t* ids, double* dists, int32_t* n_hits, double* radius,
                      uint64_t* cands, uint32_t* overflow_list, uint32_t* overflow_n, uint32_t* big_list,
                      uint32_t* big_n, cudaStream_t s) {
    const unsigned grid = static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>(a.nq, 4096)));
    uint32_t cap2 = 64;  // the sort width for a full staging list
    while (cap2 < a.cap) cap2 <<= 1;
    const uint32_t w1 = std::min<uint32_t>(cap2, kTcFinishCap);  // 32 KB: several CTAs per SM
    DETLSH_CUDA(cudaFuncSetAttribute(tc_finish_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(cap2 * sizeof(uint64_t))));
    ProfScope ps("tc_finish", s);
    tc_finish_kernel<<<grid, 256, w1 * sizeof(uint64_t), s>>>(a, perm0, k, r_min, budget, ids, dists, n_hits,
                                                              radius, cands, overflow_list, overflow_n, w1, big_list,
                                                              big_n, nullptr, nullptr);
    DETLSH_LAUNCH_CHECK();
    if (cap2 > w1) {
        int sms = 148;
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        tc_finish_kernel<<<static_cast<unsigned>(sms), 256, cap2 * sizeof(uint64_t), s>>>(
            a, perm0, k, r_min, budget, ids, dists, n_hits, radius, cands, overflow_list, overflow_n, cap2, nullptr,
            nullptr, big_list, big_n);
        DETLSH_LAUNCH_CHECK();
    }
    DETLSH_LAUNCH_CHECK();
}

void tc_gemm_u8_test(const uint8_t* hA, const uint8_t* hB, int N, int K, int32_t* hC) {
    if (N < 32 || N > 256 || N % 32 || K < 32 || K > 256 || K % 32)
        throw InvalidArgument("tc_gemm_u8_test: N in {32..256 step 32}, K in {32..256 step 32}");
    DevBuf<uint8_t> A(128 * static_cast<size_t>(K)), B(static_cast<size_t>(N) * K);
    DevBuf<int32_t> Cd(128 * static_cast<size_t>(N));
    DETLSH_CUDA(cudaMemcpy(A.get(), hA, A.bytes(), cudaMemcpyHostToDevice));
    DETLSH_CUDA(cudaMemcpy(B.get(), hB, B.bytes(), cudaMemcpyHostToDevice));
    const size_t smem = static_cast<size_t>(128 + N) * K;
    DETLSH_CUDA(cudaFuncSetAttribute(tc_gemm_u8_test_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(smem)));
    tc_gemm_u8_test_kernel<<<1, 128, smem>>>(A.get(), B.get(), N, K, Cd.get());
    DETLSH_LAUNCH_CHECK();
    DETLSH_CUDA(cudaMemcpy(hC, Cd.get(), Cd.bytes(), cudaMemcpyDeviceToHost));
}

}  // namespace detlsh_b200
