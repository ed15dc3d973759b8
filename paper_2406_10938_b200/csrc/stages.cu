// Build-stage kernels: exact projection, sample gather, GPU-native sample,
// order-statistic breakpoints, encoding and the r_min order statistics.
#include <algorithm>
#include <cstring>
#include <vector>

#include "primitives.cuh"
#include "stages.cuh"

#include <cstdlib>

namespace detlsh_b200 {

int lk_padded(int LK) { return (LK + 63) / 64 * 64; }

namespace {

__global__ void coeffs_t_kernel(const float* __restrict__ c, int LK, int d, int LKp,
                                double* __restrict__ out) {
    const int64_t total = static_cast<int64_t>(d) * LKp;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int t = static_cast<int>(i / LKp), j = static_cast<int>(i % LKp);
        out[i] = j < LK ? static_cast<double>(c[static_cast<int64_t>(j) * d + t]) : 0.0;
    }
}

constexpr int kPT = 128;  // points per tile
constexpr int kDC = 32;   // dims per chunk

// Exact projection (projection.cpp:31-37) on the FP64 tensor cores: mma.sync m8n8k4 f64 chains
// accumulate exactly as the sequential fma chain in k order (pinned on B200 by
// tools/probes/dmma_order.cu, 0 mismatches in 128 000 dot products, and by the
// projection parity tests), so k-steps issued in t order reproduce the
// reference's double sum bit for bit.  Warp tile: 16 points x 64 outputs
// (2 x 8 m8n8 tiles, 32 fp64 accumulators per lane); CTA tile 128 points.
constexpr int kPS = 36;  // padded point row (floats): A-fragment loads hit 32 distinct banks
constexpr int kAS = 72;  // padded coefficient row (doubles): B-fragment loads in 2 clean wavefronts

__global__ void __launch_bounds__(256) project_dmma_kernel(
    const float* __restrict__ pts, uint64_t n, int d, const double* __restrict__ ct, int LK,
    int LKp, int K, float* __restrict__ out, const uint32_t* __restrict__ guard = nullptr,
    uint32_t guard_cap = 0) {
    // guarded mode (project_tc.cu): run only when the tensor-core pass saw a
    // non-integral value or queued more undecided outputs than it could hold
    if (guard && guard[0] == 0 && guard[1] <= guard_cap) return;
    __shared__ __align__(16) float sx[kPT][kPS];
    __shared__ __align__(16) double sa[kDC][kAS];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int ar = lane >> 2, ac = lane & 3;  // fragment row / k-column
    const uint64_t tiles = (n + kPT - 1) / kPT;
    for (uint64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
        const uint64_t z0 = tile * kPT;
        for (int jp = 0; jp < LKp; jp += 64) {
            double acc[2][8][2];
#pragma unroll
            for (int m = 0; m < 2; ++m)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[m][j][0] = acc[m][j][1] = 0.0;
            for (int t0 = 0; t0 < d; t0 += kDC) {
                __syncthreads();
                for (int i = tid; i < kPT * kDC; i += 256) {
                    const int pp = i / kDC, c = i % kDC;
                    const uint64_t z = z0 + pp;
                    const int t = t0 + c;
                    sx[pp][c] = (z < n && t < d) ? pts[z * d + t] : 0.0f;
                }
                for (int i = tid; i < kDC * 64; i += 256) {
                    const int c = i / 64, j = i % 64;
                    const int t = t0 + c;
                    sa[c][j] = t < d ? ct[static_cast<int64_t>(t) * LKp + jp + j] : 0.0;
                }
                __syncthreads();
                // past t = d - 1 the chunk is zero-padded: fma(0, 0, acc) == acc for every
                // reachable acc (a chain started at +0 never holds -0 under round-to-nearest)
                const int kmax = min(kDC, d - t0);
                for (int c0 = 0; c0 < kmax; c0 += 4) {
                    double a[2], b[8];
#pragma unroll
                    for (int m = 0; m < 2; ++m) a[m] = static_cast<double>(sx[warp * 16 + m * 8 + ar][c0 + ac]);
#pragma unroll
                    for (int j = 0; j < 8; ++j) b[j] = sa[c0 + ac][8 * j + ar];
#pragma unroll
                    for (int m = 0; m < 2; ++m)
#pragma unroll
                        for (int j = 0; j < 8; ++j)
                            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                                         : "+d"(acc[m][j][0]), "+d"(acc[m][j][1])
                                         : "d"(a[m]), "d"(b[j]));
                }
            }
            // D fragment: point warp*16 + m*8 + ar, outputs jp + 8j + 2ac + {0,1}
#pragma unroll
            for (int m = 0; m < 2; ++m) {
                const uint64_t z = z0 + warp * 16 + m * 8 + ar;
                if (z >= n) continue;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const int jj = jp + 8 * j + 2 * ac;
                    if (K % 2 == 0 && jj + 1 < LK && (jj % K) + 1 < K) {
                        const int sp = jj / K, dim = jj % K;
                        *reinterpret_cast<float2*>(out + (static_cast<uint64_t>(sp) * n + z) * K + dim) =
                            make_float2(static_cast<float>(acc[m][j][0]), static_cast<float>(acc[m][j][1]));
                    } else {
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const int jh = jj + h;
                            if (jh < LK) {
                                const int sp = jh / K, dim = jh % K;
                                out[(static_cast<uint64_t>(sp) * n + z) * K + dim] = static_cast<float>(acc[m][j][h]);
                            }
                        }
                    }
                }
            }
        }
    }
}

__global__ void project_paa_kernel(const float* __restrict__ pts, uint64_t n, int d, int K,
                                   float* __restrict__ out) {
    const int seg = d / K;
    const uint64_t total = n * static_cast<uint64_t>(K);
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t z = i / K;
        const int j = static_cast<int>(i % K);
        const int begin = j * seg, end = (j == K - 1) ? d : begin + seg;
        const float* x = pts + z * d;
        double sum = 0.0;
        for (int t = begin; t < end; ++t) sum = __dadd_rn(sum, static_cast<double>(__ldg(x + t)));
        out[i] = static_cast<float>(__ddiv_rn(sum, static_cast<double>(end - begin)));
    }
}

// out[(r * Lg + i) * K + j] = proj[(i * n + pos[r]) * K + j]: whole projected
// rows of a few points (r_min probes, the initial-guess points), one launch.
__global__ void gather_proj_rows_kernel(const float* __restrict__ proj, uint64_t n, int K, int Lg,
                                        const uint64_t* __restrict__ pos, int m, float* __restrict__ out) {
    const int total = m * Lg * K;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
        const int r = t / (Lg * K), i = (t / K) % Lg, j = t % K;
        out[t] = proj[(static_cast<uint64_t>(i) * n + pos[r]) * K + j];
    }
}

__global__ void gather_sample_kernel(const float* __restrict__ proj, const uint32_t* __restrict__ idx,
                                     uint64_t n_s, int K, float* __restrict__ out) {
    for (uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; t < n_s;
         t += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const float* row = proj + static_cast<uint64_t>(idx[t]) * K;
        for (int j = 0; j < K; ++j) out[static_cast<uint64_t>(j) * n_s + t] = row[j];
    }
}

// Keyed Feistel bijection on [0, 2^(2h)) with cycle walking into [0, n).
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

__global__ void feistel_sample_kernel(uint64_t n, uint64_t n_s, uint64_t key, int half_bits,
                                      uint32_t* __restrict__ idx) {
    const uint64_t mask = (1ULL << half_bits) - 1;
    for (uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; t < n_s;
         t += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        uint64_t v = t;
        do {
            uint64_t l = v >> half_bits, r = v & mask;
#pragma unroll
            for (int round = 0; round < 4; ++round) {
                const uint64_t f = mix64(key + 0x9e3779b97f4a7c15ULL * (round + 1) + r) & mask;
                const uint64_t nl = r;
                r = l ^ f;
                l = nl;
            }
            v = (l << half_bits) | r;
        } while (v >= n);
        idx[t] = static_cast<uint32_t>(v);
    }
}

// float -> order-preserving u32
__device__ __forceinline__ uint32_t fkey(float f) {
    const uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float fval(uint32_t k) {
    const uint32_t u = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
    return __uint_as_float(u);
}

__global__ void order_keys_kernel(const float* __restrict__ rows, uint64_t total, uint64_t n_s,
                                  uint64_t* __restrict__ keys, uint32_t* __restrict__ vals) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t r = i / n_s;
        keys[i] = (r << 32) | fkey(rows[i]);
        vals[i] = 0;
    }
}

__global__ void order_pick_kernel(const uint64_t* __restrict__ sorted, int R, uint64_t n_s,
                                  int NR, float* __restrict__ table) {
    const int r = blockIdx.x;
    const uint64_t span = n_s / NR;
    for (int b = threadIdx.x; b <= NR; b += blockDim.x) {
        uint64_t rank;
        if (b == 0) rank = 0;
        else if (b == NR) rank = n_s - 1;
        else rank = span * b - 1;
        table[static_cast<uint64_t>(r) * (NR + 1) + b] =
            fval(static_cast<uint32_t>(sorted[static_cast<uint64_t>(r) * n_s + rank]));
    }
}

// ---- order statistics by binning (gpu_order_stat_table, large samples) ----
constexpr int kOsBins = 16384;

__global__ void os_minmax_kernel(const float* __restrict__ rows, uint64_t n_s, uint32_t* kmin, uint32_t* kmax) {
    const float* row = rows + static_cast<uint64_t>(blockIdx.y) * n_s;
    uint32_t lo = 0xffffffffu, hi = 0;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n_s;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint32_t k = fkey(row[i]);
        lo = min(lo, k);
        hi = max(hi, k);
    }
    for (int o = 16; o; o >>= 1) {
        lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(kmin + blockIdx.y, lo);
        atomicMax(kmax + blockIdx.y, hi);
    }
}

// Monotone bin of a key: linear in the value between the row's min and max
// (exact double difference, rounded product: non-decreasing in the value;
// -0 and +0 share a bin).  Non-finite extremes: one bin.
struct OsGrid {
    double vmin, scale;
    __device__ OsGrid(uint32_t kmin, uint32_t kmax) {
        const float a = fval(kmin), b = fval(kmax);
        vmin = a;
        scale = (isfinite(a) && isfinite(b) && b > a) ? static_cast<double>(kOsBins - 1) / (static_cast<double>(b) - a) : 0.0;
    }
    __device__ uint32_t bin(uint32_t k) const {
        if (scale == 0.0) return 0;
        const double x = (static_cast<double>(fval(k)) - vmin) * scale;
        return x <= 0.0 ? 0u : (x >= kOsBins - 1 ? kOsBins - 1 : static_cast<uint32_t>(x));
    }
};

__global__ void os_hist_kernel(const float* __restrict__ rows, uint64_t n_s, const uint32_t* kmin,
                               const uint32_t* kmax, uint32_t* __restrict__ hist) {
    extern __shared__ uint32_t h[];
    for (int b = threadIdx.x; b < kOsBins; b += blockDim.x) h[b] = 0;
    __syncthreads();
    const OsGrid G(kmin[blockIdx.y], kmax[blockIdx.y]);
    const float* row = rows + static_cast<uint64_t>(blockIdx.y) * n_s;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n_s;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        atomicAdd(&h[G.bin(fkey(row[i]))], 1u);
    __syncthreads();
    uint32_t* g = hist + static_cast<uint64_t>(blockIdx.y) * kOsBins;
    if (gridDim.x == 1) {
        for (int b = threadIdx.x; b < kOsBins; b += blockDim.x) g[b] = h[b];
    } else {
        for (int b = threadIdx.x; b < kOsBins; b += blockDim.x)
            if (h[b]) atomicAdd(g + b, h[b]);
    }
}

// Exclusive scan of kOsBins counts in shared memory by a 1024-thread block
// (16 consecutive bins per thread); returns the total.
__device__ uint32_t os_block_scan(const uint32_t* in, uint32_t* out) {
    __shared__ uint32_t wsum[32];
    constexpr int per = kOsBins / 1024;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    uint32_t loc = 0;
    for (int j = 0; j < per; ++j) loc += in[t * per + j];
    uint32_t inc = loc;
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += v;
    }
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        const uint32_t w = wsum[lane];
        uint32_t wi = w;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += v;
        }
        wsum[lane] = wi - w;
    }
    __syncthreads();
    uint32_t run = wsum[warp] + inc - loc;
    for (int j = 0; j < per; ++j) {
        const uint32_t c = in[t * per + j];
        out[t * per + j] = run;
        run += c;
    }
    __syncthreads();
    const uint32_t total = out[kOsBins - 1] + in[kOsBins - 1];
    __syncthreads();
    return total;
}

// rank b of a table row (order_pick_kernel's ranks)
__device__ __forceinline__ uint64_t os_rank(int b, uint64_t n_s, int NR) {
    return b == 0 ? 0 : (b == NR ? n_s - 1 : (n_s / NR) * b - 1);
}

// the bin holding rank rho: the last bin with pre[bin] <= rho (non-empty)
__device__ __forceinline__ uint32_t os_find(const uint32_t* pre, const uint32_t* h, uint64_t rho) {
    uint32_t lo = 0, hi = kOsBins - 1;
    while (lo < hi) {
        const uint32_t mid = (lo + hi + 1) >> 1;
        if (pre[mid] <= rho) lo = mid;
        else hi = mid - 1;
    }
    while (h[lo] == 0) --lo;  // (empty bins share the next bin's prefix)
    return lo;
}

__global__ void __launch_bounds__(1024) os_mark_kernel(const uint32_t* __restrict__ hist, uint64_t n_s, int NR,
                                                       uint8_t* __restrict__ flags, uint32_t* __restrict__ tcount) {
    extern __shared__ __align__(16) uint8_t os_smem[];
    uint32_t* pre = reinterpret_cast<uint32_t*>(os_smem);
    uint8_t* fl = os_smem + kOsBins * 4;
    const uint32_t* hr = hist + static_cast<uint64_t>(blockIdx.x) * kOsBins;
    for (int b = threadIdx.x; b < kOsBins; b += blockDim.x) fl[b] = 0;
    os_block_scan(hr, pre);
    for (int b = threadIdx.x; b <= NR; b += blockDim.x) fl[os_find(pre, hr, os_rank(b, n_s, NR))] = 1;
    __syncthreads();
    uint32_t t = 0;
    uint8_t* fo = flags + static_cast<uint64_t>(blockIdx.x) * kOsBins;
    for (int b = threadIdx.x; b < kOsBins; b += blockDim.x) {
        fo[b] = fl[b];
        if (fl[b]) t += hr[b];
    }
    for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if ((threadIdx.x & 31) == 0 && t) atomicAdd(tcount + blockIdx.x, t);
}

__global__ void os_compact_kernel(const float* __restrict__ rows, uint64_t n_s, const uint32_t* kmin,
                                  const uint32_t* kmax, const uint8_t* __restrict__ flags, uint64_t* __restrict__ keys,
                                  uint32_t* __restrict__ vals, uint32_t* count) {
    // one counter reservation per block step (warp counts -> block prefix)
    __shared__ uint32_t wcnt[32];
    __shared__ uint32_t bbase;
    const OsGrid G(kmin[blockIdx.y], kmax[blockIdx.y]);
    const float* row = rows + static_cast<uint64_t>(blockIdx.y) * n_s;
    const uint8_t* fr = flags + static_cast<uint64_t>(blockIdx.y) * kOsBins;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t base = blockIdx.x * static_cast<uint64_t>(blockDim.x); base < n_s; base += stride) {
        const uint64_t i = base + threadIdx.x;
        uint32_t k = 0;
        bool keep = false;
        if (i < n_s) {
            k = fkey(row[i]);
            keep = fr[G.bin(k)] != 0;
        }
        const uint32_t m = __ballot_sync(0xffffffffu, keep);
        if (lane == 0) wcnt[warp] = __popc(m);
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t t = 0;
            for (int w = 0; w < nw; ++w) {
                const uint32_t c = wcnt[w];
                wcnt[w] = t;
                t += c;
            }
            bbase = t ? atomicAdd(count, t) : 0u;
        }
        __syncthreads();
        if (keep) {
            const uint32_t at = bbase + wcnt[warp] + __popc(m & ((1u << lane) - 1u));
            keys[at] = (static_cast<uint64_t>(blockIdx.y) << 32) | k;
            vals[at] = 0;
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(1024) os_pick_kernel(const uint32_t* __restrict__ hist, const uint8_t* __restrict__ flags,
                                                       const uint32_t* __restrict__ tcount,
                                                       const uint64_t* __restrict__ sorted, uint64_t n_s, int NR,
                                                       float* __restrict__ table) {
    extern __shared__ __align__(16) uint8_t os_smem[];
    uint32_t* pre = reinterpret_cast<uint32_t*>(os_smem);
    uint32_t* tpre = pre + kOsBins;
    const int r = blockIdx.x;
    const uint32_t* hr = hist + static_cast<uint64_t>(r) * kOsBins;
    const uint8_t* fr = flags + static_cast<uint64_t>(r) * kOsBins;
    __shared__ uint64_t rowstart;
    if (threadIdx.x == 0) {
        uint64_t a = 0;
        for (int q = 0; q < r; ++q) a += tcount[q];
        rowstart = a;
    }
    os_block_scan(hr, pre);
    // flagged-only prefix: scan of (flag ? count : 0), staged in tpre first
    for (int b = threadIdx.x; b < kOsBins; b += blockDim.x) tpre[b] = fr[b] ? hr[b] : 0u;
    __syncthreads();
    {
        constexpr int per = kOsBins / 1024;
        uint32_t v[per];
        for (int j = 0; j < per; ++j) v[j] = tpre[threadIdx.x * per + j];
        __syncthreads();
        uint32_t loc = 0;
        for (int j = 0; j < per; ++j) loc += v[j];
        __shared__ uint32_t wsum[32];
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        uint32_t inc = loc;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t x = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += x;
        }
        if (lane == 31) wsum[warp] = inc;
        __syncthreads();
        if (warp == 0) {
            const uint32_t w = wsum[lane];
            uint32_t wi = w;
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t x = __shfl_up_sync(0xffffffffu, wi, o);
                if (lane >= o) wi += x;
            }
            wsum[lane] = wi - w;
        }
        __syncthreads();
        uint32_t run = wsum[warp] + inc - loc;
        for (int j = 0; j < per; ++j) {
            tpre[threadIdx.x * per + j] = run;
            run += v[j];
        }
    }
    __syncthreads();
    for (int b = threadIdx.x; b <= NR; b += blockDim.x) {
        const uint64_t rho = os_rank(b, n_s, NR);
        const uint32_t b1 = os_find(pre, hr, rho);
        const uint64_t pos = rho - pre[b1] + tpre[b1];
        table[static_cast<uint64_t>(r) * (NR + 1) + b] = fval(static_cast<uint32_t>(sorted[rowstart + pos]));
    }
}

// Encode: one thread per (space, point); the space's K boundary rows sit in
// shared memory in Eytzinger (BFS) order, padded with +inf to a complete tree
// of 2^H - 1 nodes, so lower_bound = #{b : row[b] < v} is H branch-free steps
// i = 2i + (e[i] < v) ending at i = 2^H + count.  Level l touches 2^l
// consecutive words, so the first six levels are bank-conflict free (the
// sorted-array search strides by multiples of 32 words and serialises).
__global__ void encode_kernel(const float* __restrict__ proj, uint64_t n, int K,
                              const float* __restrict__ table, int NR, int H,
                              uint8_t* __restrict__ codes) {
    extern __shared__ float se[];  // [K][2^H], node i of dim j at se[j * 2^H + i]
    const int sp = blockIdx.y;
    const int W = NR + 1;
    const int T = 1 << H;
    for (int x = threadIdx.x; x < K * T; x += blockDim.x) {
        const int j = x >> H, i = x & (T - 1);
        float val = __int_as_float(0x7f800000);  // +inf padding (and unused slot 0)
        if (i > 0) {
            const int dpt = 31 - __clz(i);
            const int sidx = ((2 * (i - (1 << dpt)) + 1) << (H - 1 - dpt)) - 1;
            if (sidx < W) val = table[static_cast<uint64_t>(sp) * K * W + static_cast<uint64_t>(j) * W + sidx];
        }
        se[x] = val;
    }
    __syncthreads();
    const float* P = proj + static_cast<uint64_t>(sp) * n * K;
    uint8_t* C = codes + static_cast<uint64_t>(sp) * n * K;
    auto region = [&](const float* e, float v) {
        uint32_t i = 1;
        for (int s = 0; s < H; ++s) i = 2 * i + (e[i] < v ? 1u : 0u);
        int reg = static_cast<int>(i - static_cast<uint32_t>(T)) - 1;  // lower_bound - 1
        return reg < 0 ? 0 : (reg > NR - 1 ? NR - 1 : reg);
    };
    for (uint64_t z = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; z < n;
         z += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        if (K == 16) {
            const float4* src = reinterpret_cast<const float4*>(P + z * 16);
            float v[16];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const float4 f = src[q];
                v[4 * q] = f.x; v[4 * q + 1] = f.y; v[4 * q + 2] = f.z; v[4 * q + 3] = f.w;
            }
            // the 16 searches advance level by level together (16 independent loads in flight)
            uint32_t idx[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) idx[j] = 1;
            for (int st = 0; st < H; ++st) {
#pragma unroll
                for (int j = 0; j < 16; ++j) idx[j] = 2 * idx[j] + (se[j * T + idx[j]] < v[j] ? 1u : 0u);
            }
            uint32_t packed[4] = {0, 0, 0, 0};
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                int reg = static_cast<int>(idx[j] - static_cast<uint32_t>(T)) - 1;  // lower_bound - 1
                reg = reg < 0 ? 0 : (reg > NR - 1 ? NR - 1 : reg);
                packed[j >> 2] |= static_cast<uint32_t>(reg) << (8 * (j & 3));
            }
            reinterpret_cast<uint4*>(C + z * 16)[0] = make_uint4(packed[0], packed[1], packed[2], packed[3]);
        } else {
            for (int j = 0; j < K; ++j)
                C[z * K + j] = static_cast<uint8_t>(region(se + j * T, P[z * K + j]));
        }
    }
}

// D[p][z] = min over spaces of the exact projected l2 (dataset.hpp:23-34 over K floats).
// D[p][z] = min over spaces of the exact projected l2 distance; since sqrt is
// monotone, min_i sqrt(acc_i) == sqrt(min_i acc_i) bit for bit, so one sqrt
// per probe.  Also tracks each probe's min / max bit pattern (doubles >= 0
// order like their bits) to seed the range-narrowing select.
constexpr int kMaxProbes = 10;

template <int KT>
__global__ void __launch_bounds__(256) rmin_dist_kernel(
    const float* __restrict__ proj, uint64_t n, int K, int L, const float* __restrict__ probe_proj,
    int np, double* __restrict__ D, unsigned long long* __restrict__ lo_bits,
    unsigned long long* __restrict__ hi_bits, uint64_t z0, uint64_t d_stride) {
    extern __shared__ float spp[];  // [np][L][K]
    for (int i = threadIdx.x; i < np * L * K; i += blockDim.x) spp[i] = probe_proj[i];
    __syncthreads();
    unsigned long long mn[kMaxProbes], mx[kMaxProbes];
#pragma unroll
    for (int p = 0; p < kMaxProbes; ++p) {
        mn[p] = ~0ULL;
        mx[p] = 0;
    }
    for (uint64_t z = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; z < n;
         z += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        double best[kMaxProbes];
#pragma unroll
        for (int p = 0; p < kMaxProbes; ++p) best[p] = __longlong_as_double(0x7ff0000000000000LL);
        for (int i = 0; i < L; ++i) {
            float x[KT];
            const float* row = proj + (static_cast<uint64_t>(i) * n + z) * K;
            if (KT == 16 && K == 16) {
#pragma unroll
                for (int q4 = 0; q4 < 4; ++q4) {
                    const float4 v = __ldg(reinterpret_cast<const float4*>(row) + q4);
                    x[4 * q4] = v.x; x[4 * q4 + 1] = v.y; x[4 * q4 + 2] = v.z; x[4 * q4 + 3] = v.w;
                }
            } else {
#pragma unroll
                for (int j = 0; j < KT; ++j) x[j] = j < K ? __ldg(row + j) : 0.0f;
            }
#pragma unroll
            for (int p = 0; p < kMaxProbes; ++p) {
                if (p < np) {
                    const float* q = spp + (p * L + i) * K;
                    double acc = 0.0;
#pragma unroll
                    for (int j = 0; j < KT; ++j) {
                        if (j < K) {
                            const double diff = __dsub_rn(static_cast<double>(q[j]), static_cast<double>(x[j]));
                            acc = __dadd_rn(acc, __dmul_rn(diff, diff));
                        }
                    }
                    best[p] = acc < best[p] ? acc : best[p];
                }
            }
        }
#pragma unroll
        for (int p = 0; p < kMaxProbes; ++p) {
            if (p < np) {
                const double dist = __dsqrt_rn(best[p]);
                D[static_cast<uint64_t>(p) * d_stride + z0 + z] = dist;
                const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(dist));
                mn[p] = b < mn[p] ? b : mn[p];
                mx[p] = b > mx[p] ? b : mx[p];
            }
        }
    }
#pragma unroll
    for (int p = 0; p < kMaxProbes; ++p) {
        if (p < np) {
            unsigned long long a = mn[p], b = mx[p];
            for (int o = 16; o; o >>= 1) {
                const unsigned long long ta = __shfl_xor_sync(0xffffffffu, a, o);
                const unsigned long long tb = __shfl_xor_sync(0xffffffffu, b, o);
                a = ta < a ? ta : a;
                b = tb > b ? tb : b;
            }
            if ((threadIdx.x & 31) == 0) {
                atomicMin(lo_bits + p, a);
                atomicMax(hi_bits + p, b);
            }
        }
    }
}

// Exact rank selection by range narrowing: each pass histograms the bit
// patterns in [lo, hi] into 2048 bins of width 2^shift (block-private smem
// histograms), keeps the bin holding the wanted rank.  shift reaches 0 after
// at most 6 passes, leaving lo == the exact order statistic.
constexpr int kSelBins = 2048;

__global__ void rmin_sel_init(const unsigned long long* lo, const unsigned long long* hi, int np,
                              int* shift) {
    const int p = threadIdx.x;
    if (p < np) {
        const unsigned long long span = hi[p] - lo[p];
        const int bits = span ? 64 - __clzll(static_cast<long long>(span)) : 0;
        shift[p] = bits > 11 ? bits - 11 : 0;
    }
}

__global__ void rmin_sel_hist(const double* __restrict__ D, uint64_t n,
                              const unsigned long long* __restrict__ lo, const int* __restrict__ shift,
                              uint32_t* __restrict__ ghist) {
    __shared__ uint32_t h[kSelBins];
    for (int i = threadIdx.x; i < kSelBins; i += blockDim.x) h[i] = 0;
    __syncthreads();
    const int p = blockIdx.y;
    const unsigned long long L0 = lo[p];
    const int sh = shift[p];
    const double* Dp = D + static_cast<uint64_t>(p) * n;
    for (uint64_t z = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; z < n;
         z += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(Dp[z]));
        if (b >= L0) {
            const unsigned long long off = (b - L0) >> sh;
            if (off < kSelBins) atomicAdd(&h[off], 1u);
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kSelBins; i += blockDim.x)
        if (h[i]) atomicAdd(&ghist[static_cast<size_t>(p) * kSelBins + i], h[i]);
}

// The bin holding the wanted rank: block-wide exclusive scan over the 2048 bin
// counts (8 per thread), then the owning thread walks its 8 bins.
__global__ void __launch_bounds__(256) rmin_sel_pick(uint32_t* __restrict__ ghist, unsigned long long* lo,
                                                     unsigned long long* hi, int* shift, uint64_t* need) {
    const int p = blockIdx.x, t = threadIdx.x, lane = t & 31, w = t >> 5;
    uint32_t* h = ghist + static_cast<size_t>(p) * kSelBins;
    __shared__ unsigned long long wsum[8];
    constexpr int kPer = kSelBins / 256;
    uint32_t c[kPer];
    unsigned long long mine = 0;
#pragma unroll
    for (int e = 0; e < kPer; ++e) {
        c[e] = h[t * kPer + e];
        mine += c[e];
    }
    unsigned long long incl = mine;
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    if (lane == 31) wsum[w] = incl;
    __syncthreads();
    unsigned long long base = 0;
    for (int i = 0; i < w; ++i) base += wsum[i];
    const unsigned long long excl = base + incl - mine;
    const uint64_t want = need[p];
    __syncthreads();  // every thread has read need[p] and the bins
    if (excl < want && want <= excl + mine) {
        unsigned long long cum = excl;
        int bin = t * kPer;
        for (int e = 0; e < kPer; ++e, ++bin) {
            if (cum + c[e] >= want) break;
            cum += c[e];
        }
        const int sh = shift[p];
        const unsigned long long nlo = lo[p] + (static_cast<unsigned long long>(bin) << sh);
        unsigned long long nhi = nlo + ((1ULL << sh) - 1);
        if (nhi > hi[p] || nhi < nlo) nhi = hi[p];
        need[p] = want - cum;
        lo[p] = nlo;
        hi[p] = nhi;
        const unsigned long long span = nhi - nlo;
        const int bits = span ? 64 - __clzll(static_cast<long long>(span)) : 0;
        shift[p] = bits > 11 ? bits - 11 : 0;
    }
#pragma unroll
    for (int e = 0; e < kPer; ++e) h[t * kPer + e] = 0;
}

}  // namespace

void prepare_coeffs_t(const float* d_coeffs, int LK, int d, double* d_ct, cudaStream_t s) {
    const int LKp = lk_padded(LK);
    const int64_t total = static_cast<int64_t>(d) * LKp;
    coeffs_t_kernel<<<static_cast<unsigned>(std::min<int64_t>((total + 255) / 256, 4096)), 256, 0, s>>>(
        d_coeffs, LK, d, LKp, d_ct);
    DETLSH_LAUNCH_CHECK();
}

void launch_project_dmma_guarded(const float* d_points, uint64_t n, int d, const double* d_ct, int K,
                                 int L, float* d_out, const uint32_t* d_guard, uint32_t cap, cudaStream_t s) {
    const int LK = K * L;
    const uint64_t tiles = (n + kPT - 1) / kPT;
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t grid = std::min<uint64_t>(tiles, static_cast<uint64_t>(sm_count(dev)) * 2);
    project_dmma_kernel<<<static_cast<unsigned>(grid), 256, 0, s>>>(d_points, n, d, d_ct, LK, lk_padded(LK),
                                                                     K, d_out, d_guard, cap);
    DETLSH_LAUNCH_CHECK();
}

void launch_project_exact(const float* d_points, uint64_t n, int d, const double* d_ct, int K,
                          int L, float* d_out, cudaStream_t s, const char* prof, const ProjTc* tc,
                          uint32_t* d_nonint) {
    if (n == 0) return;
    if (tc && launch_project_tc(d_points, n, d, *tc, d_ct, K, L, d_out, s,
                                std::strcmp(prof, "project_exact") == 0 ? "project_tc" : prof, d_nonint))
        return;
    const int LK = K * L;
    const uint64_t tiles = (n + kPT - 1) / kPT;
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t grid = std::min<uint64_t>(tiles, static_cast<uint64_t>(sm_count(dev)) * 8);
    ProfScope ps(prof, s);
    project_dmma_kernel<<<static_cast<unsigned>(grid), 256, 0, s>>>(d_points, n, d, d_ct, LK,
                                                                     lk_padded(LK), K, d_out);
    DETLSH_LAUNCH_CHECK();
}

void launch_project_paa(const float* d_points, uint64_t n, int d, int K, float* d_out, cudaStream_t s,
                        const char* prof) {
    const unsigned grid = static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>((n * K + 255) / 256, 65535)));
    ProfScope ps(prof, s);
    project_paa_kernel<<<grid, 256, 0, s>>>(d_points, n, d, K, d_out);
    DETLSH_LAUNCH_CHECK();
}

void launch_gather_proj_rows(const float* d_proj, uint64_t n, int K, int Lg, const uint64_t* d_pos, int m,
                             float* d_out, cudaStream_t s) {
    if (m <= 0) return;
    gather_proj_rows_kernel<<<(m * Lg * K + 255) / 256, 256, 0, s>>>(d_proj, n, K, Lg, d_pos, m, d_out);
    DETLSH_LAUNCH_CHECK();
}

__global__ void iota_u32_kernel(uint32_t* v, uint64_t n) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        v[i] = static_cast<uint32_t>(i);
}
void launch_iota_u32(uint32_t* v, uint64_t n, cudaStream_t s) {
    const unsigned grid = static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, 4096)));
    iota_u32_kernel<<<grid, 256, 0, s>>>(v, n);
    DETLSH_LAUNCH_CHECK();
}

void launch_gather_sample(const float* d_proj_space, const uint32_t* d_idx, uint64_t n_s, int K,
                          float* d_out, cudaStream_t s) {
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((n_s + 255) / 256, 65535));
    ProfScope ps("gather_sample", s);
    gather_sample_kernel<<<grid, 256, 0, s>>>(d_proj_space, d_idx, n_s, K, d_out);
    DETLSH_LAUNCH_CHECK();
}

void launch_feistel_sample(uint64_t n, uint64_t n_s, uint64_t key, uint32_t* d_idx,
                           cudaStream_t s) {
    int bits = 1;
    while ((1ULL << bits) < n) ++bits;
    const int half = (bits + 1) / 2;
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((n_s + 255) / 256, 65535));
    feistel_sample_kernel<<<grid, 256, 0, s>>>(n, n_s, key, half, d_idx);
    DETLSH_LAUNCH_CHECK();
}

void OrderStatWork::reserve(int R, uint64_t n_s, cudaStream_t s) {
    const uint64_t total = static_cast<uint64_t>(R) * n_s;
    kmin.grow(R, 0, s);
    kmax.grow(R, 0, s);
    tcount.grow(R, 0, s);
    count.grow(1, 0, s);
    hist.grow(static_cast<size_t>(R) * kOsBins, 0, s);
    flags.grow(static_cast<size_t>(R) * kOsBins, 0, s);
    k0.grow(total, 0, s);
    k1.grow(total, 0, s);
    v0.grow(total, 0, s);
    v1.grow(total, 0, s);
    tmp.grow(radix_temp_elems(total), 0, s);
}

void gpu_order_stat_table(const float* d_rows, int R, uint64_t n_s, int n_regions,
                          float* d_table, cudaStream_t s, bool sync, OrderStatWork* work) {
    StreamScope scope(s);
    const uint64_t total = static_cast<uint64_t>(R) * n_s;
    int rbits = 0;
    while ((1 << rbits) < R) ++rbits;
    const int end_bit = 32 + ((rbits + 7) / 8) * 8;
    OrderStatWork local;
    OrderStatWork& w = work ? *work : local;
    w.reserve(R, n_s, s);  // (no-op when the caller reserved enough)
    if (n_s < 4 * static_cast<uint64_t>(kOsBins) || std::getenv("DETLSH_TEST_FULL_ORDER_SORT")) {
        // small samples: sort everything
        const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((total + 255) / 256, 65535));
        order_keys_kernel<<<grid, 256, 0, s>>>(d_rows, total, n_s, w.k0.get(), w.v0.get());
        DETLSH_LAUNCH_CHECK();
        const bool flip = radix_sort_pairs<uint64_t>(w.k0.get(), w.v0.get(), w.k1.get(), w.v1.get(), total, 0,
                                                     end_bit, w.tmp.get(), s);
        order_pick_kernel<<<R, 256, 0, s>>>(flip ? w.k1.get() : w.k0.get(), R, n_s, n_regions, d_table);
        DETLSH_LAUNCH_CHECK();
    } else {
        // Only the N_r + 1 ranks are needed: bin each row's values on a
        // monotone (linear in value, between the row's min and max) 16 K-bin
        // grid, keep just the values of the bins that hold a wanted rank, sort
        // those, and read the ranks off with the bins' prefix counts.  Same
        // order (the order-preserving key), so the same values as a full sort.
        DETLSH_CUDA(cudaMemsetAsync(w.kmin.get(), 0xff, R * 4, s));
        DETLSH_CUDA(cudaMemsetAsync(w.kmax.get(), 0, R * 4, s));
        DETLSH_CUDA(cudaMemsetAsync(w.hist.get(), 0, static_cast<size_t>(R) * kOsBins * 4, s));
        DETLSH_CUDA(cudaMemsetAsync(w.count.get(), 0, 4, s));
        DETLSH_CUDA(cudaMemsetAsync(w.tcount.get(), 0, R * 4, s));
        const unsigned gx = static_cast<unsigned>(std::min<uint64_t>((n_s + 16383) / 16384, 1024));
        os_minmax_kernel<<<dim3(gx, R), 256, 0, s>>>(d_rows, n_s, w.kmin.get(), w.kmax.get());
        DETLSH_LAUNCH_CHECK();
        DETLSH_CUDA(cudaFuncSetAttribute(os_hist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kOsBins * 4));
        // (a few blocks per row: each flushes its whole histogram)
        const unsigned gh = static_cast<unsigned>(std::min<uint64_t>((n_s + 262143) / 262144, 256));
        os_hist_kernel<<<dim3(gh, R), 1024, kOsBins * 4, s>>>(d_rows, n_s, w.kmin.get(), w.kmax.get(), w.hist.get());
        DETLSH_LAUNCH_CHECK();
        DETLSH_CUDA(cudaFuncSetAttribute(os_mark_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         kOsBins * 4 + kOsBins));
        os_mark_kernel<<<R, 1024, kOsBins * 4 + kOsBins, s>>>(w.hist.get(), n_s, n_regions, w.flags.get(),
                                                              w.tcount.get());
        DETLSH_LAUNCH_CHECK();
        os_compact_kernel<<<dim3(gx, R), 256, 0, s>>>(d_rows, n_s, w.kmin.get(), w.kmax.get(), w.flags.get(),
                                                     w.k0.get(), w.v0.get(), w.count.get());
        DETLSH_LAUNCH_CHECK();
        const bool flip = radix_sort_pairs<uint64_t>(w.k0.get(), w.v0.get(), w.k1.get(), w.v1.get(), total, 0,
                                                     end_bit, w.tmp.get(), s, w.count.get());
        DETLSH_CUDA(cudaFuncSetAttribute(os_pick_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         kOsBins * 4 * 2));
        os_pick_kernel<<<R, 1024, kOsBins * 4 * 2, s>>>(w.hist.get(), w.flags.get(), w.tcount.get(),
                                                        flip ? w.k1.get() : w.k0.get(), n_s, n_regions, d_table);
        DETLSH_LAUNCH_CHECK();
    }
    if (sync) DETLSH_CUDA(cudaStreamSynchronize(s));
}

void launch_encode(const float* d_proj, uint64_t n, int K, int L, const float* d_table,
                   int n_regions, uint8_t* d_codes, cudaStream_t s) {
    if (n == 0) return;
    int H = 1;  // complete tree of 2^H - 1 >= N_r + 1 nodes
    while ((1 << H) - 1 < n_regions + 1) ++H;
    const size_t smem = static_cast<size_t>(K) * (static_cast<size_t>(1) << H) * sizeof(float);
    DETLSH_CUDA(cudaFuncSetAttribute(encode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(smem)));
    int dev = 0;
    cudaGetDevice(&dev);
    const unsigned gx = static_cast<unsigned>(
        std::min<uint64_t>((n + 255) / 256, static_cast<uint64_t>(sm_count(dev)) * 8));
    ProfScope ps("encode", s);
    encode_kernel<<<dim3(gx, L), 256, smem, s>>>(d_proj, n, K, d_table, n_regions, H, d_codes);
    DETLSH_LAUNCH_CHECK();
}

RminSelect::RminSelect(int np_) : np(np_), lo(np_), hi(np_), need(np_), shift(np_), hist(static_cast<size_t>(np_) * kSelBins) {}

void rmin_order_stats(const float* d_proj, uint64_t n, int K, int L, const float* d_probe_proj,
                      int np, uint64_t rank, double* d_D, uint32_t* d_hist, uint64_t* h_T_bits,
                      cudaStream_t s) {
    (void)d_hist;
    StreamScope scope(s);
    RminSelect sel(np);
    rmin_begin(sel, s);
    launch_rmin_dist(d_proj, n, 0, n, K, L, d_probe_proj, sel, d_D, s);
    rmin_select(sel, d_D, n, rank, h_T_bits, s);
}

void rmin_begin(RminSelect& sel, cudaStream_t s) {
    if (sel.np > kMaxProbes || sel.np < 1) throw InvalidArgument("estimate_rmin: 1 to 10 probes per group");
    DETLSH_CUDA(cudaMemsetAsync(sel.lo.get(), 0xff, sel.np * sizeof(unsigned long long), s));
    DETLSH_CUDA(cudaMemsetAsync(sel.hi.get(), 0, sel.np * sizeof(unsigned long long), s));
}

void launch_rmin_dist(const float* d_proj_chunk, uint64_t m, uint64_t z0, uint64_t n_total, int K, int L,
                      const float* d_probe_proj, RminSelect& sel, double* d_D, cudaStream_t s) {
    if (m == 0) return;
    int dev = 0;
    cudaGetDevice(&dev);
    const unsigned gx = static_cast<unsigned>(
        std::max<uint64_t>(1, std::min<uint64_t>((m + 255) / 256, static_cast<uint64_t>(sm_count(dev)) * 8)));
    ProfScope ps("rmin_dist", s);
    const int np = sel.np;
    const size_t smem = static_cast<size_t>(np) * L * K * sizeof(float);
    if (K == 16)
        rmin_dist_kernel<16><<<gx, 256, smem, s>>>(d_proj_chunk, m, K, L, d_probe_proj, np, d_D, sel.lo.get(),
                                                   sel.hi.get(), z0, n_total);
    else
        rmin_dist_kernel<kMaxK><<<gx, 256, smem, s>>>(d_proj_chunk, m, K, L, d_probe_proj, np, d_D, sel.lo.get(),
                                                      sel.hi.get(), z0, n_total);
    DETLSH_LAUNCH_CHECK();
}

void rmin_select(RminSelect& sel, const double* d_D, uint64_t n, uint64_t rank, uint64_t* h_T_bits,
                 cudaStream_t s) {
    int dev = 0;
    cudaGetDevice(&dev);
    const int np = sel.np;
    // two CTAs per SM over all probes: each CTA clears and flushes a 2048-bin
    // histogram, so more CTAs than that cost more than they hide
    const unsigned gx = static_cast<unsigned>(std::max<uint64_t>(
        1, std::min<uint64_t>((n + 255) / 256, (static_cast<uint64_t>(sm_count(dev)) * 2 + np - 1) / np)));
    std::vector<uint64_t> h(np, rank);
    DETLSH_CUDA(cudaMemcpyAsync(sel.need.get(), h.data(), np * sizeof(uint64_t), cudaMemcpyHostToDevice, s));
    DETLSH_CUDA(cudaMemsetAsync(sel.hist.get(), 0, static_cast<size_t>(np) * kSelBins * sizeof(uint32_t), s));
    unsigned long long* const lo_p = sel.lo.get();
    unsigned long long* const hi_p = sel.hi.get();
    uint64_t* const need_p = sel.need.get();
    int* const shift_p = sel.shift.get();
    uint32_t* const d_hist = sel.hist.get();
    ProfScope ps("rmin_select", s);
    rmin_sel_init<<<1, 32, 0, s>>>(lo_p, hi_p, np, shift_p);
    DETLSH_LAUNCH_CHECK();
    for (int pass = 0; pass < 6; ++pass) {  // 53-bit spans need at most 5 passes of 11 bits
        rmin_sel_hist<<<dim3(gx, np), 256, 0, s>>>(d_D, n, lo_p, shift_p, d_hist);
        DETLSH_LAUNCH_CHECK();
        rmin_sel_pick<<<np, 256, 0, s>>>(d_hist, lo_p, hi_p, shift_p, need_p);
        DETLSH_LAUNCH_CHECK();
    }
    DETLSH_CUDA(cudaMemcpyAsync(h_T_bits, lo_p, np * sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
    DETLSH_CUDA(cudaStreamSynchronize(s));
}

}  // namespace detlsh_b200

namespace detlsh_b200 {
namespace {

__global__ void integral_u8_kernel(const float* __restrict__ x, uint64_t total,
                                   unsigned int* __restrict__ bad) {
    bool ok = true;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const float v = x[i];
        ok = ok && v >= 0.0f && v <= 255.0f && v == floorf(v);
    }
    if (__any_sync(0xffffffffu, !ok) && (threadIdx.x & 31) == 0) atomicOr(bad, 1u);
}

// out[p'] = u8(rows[perm[p']]), zero-padded to row_bytes (multiple of 16).
// One thread per 16-byte output chunk: four float4 reads of the gathered row
// (d % 4 == 0; scalar reads otherwise), one 16-byte store.
__global__ void pack_u8_kernel(const float* __restrict__ x, const uint32_t* __restrict__ perm,
                               uint64_t n, int d, int row_bytes, uint8_t* __restrict__ out) {
    const uint32_t cpr = static_cast<uint32_t>(row_bytes) / 16;  // chunks per row
    const uint64_t total = n * cpr;
    const bool vec = (d & 3) == 0;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t r = i / cpr;
        const int t0 = static_cast<int>(i - r * cpr) * 16;
        const float* src = x + static_cast<uint64_t>(__ldg(perm + r)) * d;
        uint32_t w[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            float f[4];
            const int t = t0 + 4 * q;
            if (vec && t + 4 <= d) {
                const float4 v = __ldg(reinterpret_cast<const float4*>(src + t));
                f[0] = v.x, f[1] = v.y, f[2] = v.z, f[3] = v.w;
            } else {
#pragma unroll
                for (int e = 0; e < 4; ++e) f[e] = t + e < d ? __ldg(src + t + e) : 0.0f;
            }
            w[q] = static_cast<uint32_t>(f[0]) | static_cast<uint32_t>(f[1]) << 8 | static_cast<uint32_t>(f[2]) << 16 |
                   static_cast<uint32_t>(f[3]) << 24;
        }
        reinterpret_cast<uint4*>(out)[i] = make_uint4(w[0], w[1], w[2], w[3]);
    }
}

// fp32 rows gathered into tree-0 leaf order (or a sample's rows): one warp per
// row, 16-byte moves when d % 4 == 0 (no per-element index division).
__global__ void pack_f32_kernel(const float* __restrict__ x, const uint32_t* __restrict__ perm, uint64_t n,
                                int d, float* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const uint64_t warps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
    for (uint64_t r = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5; r < n; r += warps) {
        const uint64_t src = static_cast<uint64_t>(__ldg(perm + r)) * d;
        if ((d & 3) == 0) {
            const float4* s4 = reinterpret_cast<const float4*>(x + src);
            float4* d4 = reinterpret_cast<float4*>(out + r * d);
            for (int q = lane; q < d / 4; q += 32) d4[q] = __ldg(s4 + q);
        } else {
            for (int t = lane; t < d; t += 32) out[r * d + t] = __ldg(x + src + t);
        }
    }
}

}  // namespace

void launch_pack_f32(const float* d_x, const uint32_t* d_perm, uint64_t n, int d, float* d_out, cudaStream_t s) {
    const unsigned grid = static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>((n + 7) / 8, 65535)));
    ProfScope ps("pack_f32", s);
    pack_f32_kernel<<<grid, 256, 0, s>>>(d_x, d_perm, n, d, d_out);
    DETLSH_LAUNCH_CHECK();
}

bool data_is_u8(const float* d_x, uint64_t total, cudaStream_t s) {
    StreamScope scope(s);
    DevBuf<unsigned int> bad(1);
    DETLSH_CUDA(cudaMemsetAsync(bad.get(), 0, 4, s));
    int dev = 0;
    cudaGetDevice(&dev);
    const unsigned grid = static_cast<unsigned>(
        std::max<uint64_t>(1, std::min<uint64_t>((total + 255) / 256, static_cast<uint64_t>(sm_count(dev)) * 8)));
    integral_u8_kernel<<<grid, 256, 0, s>>>(d_x, total, bad.get());
    DETLSH_LAUNCH_CHECK();
    unsigned int h = 1;
    DETLSH_CUDA(cudaMemcpyAsync(&h, bad.get(), 4, cudaMemcpyDeviceToHost, s));
    DETLSH_CUDA(cudaStreamSynchronize(s));
    return h == 0;
}

void launch_pack_u8(const float* d_x, const uint32_t* d_perm, uint64_t n, int d, int row_bytes,
                    uint8_t* d_out, cudaStream_t s) {
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t total = n * static_cast<uint64_t>(row_bytes / 16);
    const unsigned grid = static_cast<unsigned>(
        std::max<uint64_t>(1, std::min<uint64_t>((total + 255) / 256, static_cast<uint64_t>(sm_count(dev)) * 16)));
    ProfScope ps("pack_u8", s);
    pack_u8_kernel<<<grid, 256, 0, s>>>(d_x, d_perm, n, d, row_bytes, d_out);
    DETLSH_LAUNCH_CHECK();
}

}  // namespace detlsh_b200
