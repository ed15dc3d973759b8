// Exact k-nearest-neighbour ground truth (brute_force_knn, metrics.cpp:8-33):
// for every query, all n points scored with l2_distance_sq (dataset.hpp:23-30:
// sequential fp64, diff = q - x, acc += diff * diff, no contraction) and the k
// smallest by (dist^2, position); distances returned as sqrt(dist^2).
//
// Three steps per batch of queries: (1) a threshold per query -- the k-th
// smallest dist^2 over a strided sample of rows, or a caller's upper bound
// (e.g. the squared k-th distance an ANN query returned: k real points lie
// within it); (2) every (query, point) pair exactly, keeping those within the
// threshold as (dist^2, position) records; (3) per query, the records sorted
// by (dist^2, position).  A query whose records overflow the staging buffer
// is redone alone with every point sorted (radix sort, stable in position).
#include <algorithm>
#include <vector>

#include "common.cuh"
#include "gt.cuh"
#include "primitives.cuh"

namespace detlsh_b200 {

namespace {

constexpr int kGtQ = 32;     // queries per CTA tile
constexpr int kGtR = 64;     // rows per CTA tile
constexpr int kGtT = 64;     // dims per smem chunk
constexpr uint32_t kGtCap = 4096;  // records staged per query

__device__ __forceinline__ double sq_step(double acc, float a, float b) {
    const double diff = __dsub_rn(static_cast<double>(a), static_cast<double>(b));
    return __dadd_rn(acc, __dmul_rn(diff, diff));
}

// Exact dist^2 of query tile x row tile, 8 pairs per thread (q = tid % 32,
// rows tid / 32 + 8 j).  Rows [r0, r1) of this CTA's split, strided rows when
// `stride` > 1 (the threshold sample).  Pairs within thr[q] are appended.
__global__ void __launch_bounds__(256) gt_pairs_kernel(const float* __restrict__ X, uint64_t n, int d,
                                                       const float* __restrict__ Q, uint64_t nq,
                                                       const double* __restrict__ thr, uint64_t stride,
                                                       uint64_t rows_total, uint32_t splits,
                                                       uint32_t* __restrict__ cnt, uint64_t* __restrict__ key,
                                                       uint32_t* __restrict__ pos, uint32_t cap,
                                                       double* __restrict__ all_d2) {
    __shared__ float qs[kGtQ][kGtT + 1];
    __shared__ float xs[kGtR][kGtT + 1];
    const int tid = threadIdx.x, q = tid % kGtQ, rb = tid / kGtQ;
    const uint64_t qtiles = (nq + kGtQ - 1) / kGtQ;
    const uint64_t qt = blockIdx.x % qtiles, split = blockIdx.x / qtiles;
    const uint64_t q0 = qt * kGtQ;
    const uint64_t rtiles = (rows_total + kGtR - 1) / kGtR;
    const uint64_t t0 = rtiles * split / splits, t1 = rtiles * (split + 1) / splits;
    const uint64_t qg = q0 + q;
    const double th = qg < nq && thr ? thr[qg] : 0.0;
    for (uint64_t rt = t0; rt < t1; ++rt) {
        double acc[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] = 0.0;
        for (int c0 = 0; c0 < d; c0 += kGtT) {
            const int w = min(kGtT, d - c0);
            __syncthreads();
            for (int i = tid; i < kGtQ * kGtT; i += blockDim.x) {
                const int qq = i / kGtT, t = i % kGtT;
                qs[qq][t] = (q0 + qq < nq && t < w) ? Q[(q0 + qq) * d + c0 + t] : 0.0f;
            }
            for (int i = tid; i < kGtR * kGtT; i += blockDim.x) {
                const int r = i / kGtT, t = i % kGtT;
                const uint64_t rr = rt * kGtR + r;
                xs[r][t] = (rr < rows_total && t < w) ? X[(rr * stride) * d + c0 + t] : 0.0f;
            }
            __syncthreads();
            for (int t = 0; t < w; ++t) {
                const float a = qs[q][t];
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[j] = sq_step(acc[j], a, xs[rb + 8 * j][t]);
            }
        }
        if (qg >= nq) continue;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const uint64_t rr = rt * kGtR + rb + 8 * j;
            if (rr >= rows_total) continue;
            if (all_d2) {  // sample pass: keep every distance
                all_d2[qg * rows_total + rr] = acc[j];
            } else if (acc[j] <= th) {
                const uint32_t slot = atomicAdd(cnt + qg, 1u);
                if (slot < cap) {
                    key[qg * cap + slot] = static_cast<uint64_t>(__double_as_longlong(acc[j]));
                    pos[qg * cap + slot] = static_cast<uint32_t>(rr * stride);
                }
            }
        }
    }
}

// k-th smallest of each query's S sample distances (non-negative doubles
// order as their bit patterns): an 8-pass byte-wise radix select per query.
__global__ void gt_sample_kth_kernel(const double* __restrict__ all_d2, uint64_t S, uint64_t nq, int k,
                                     double* __restrict__ thr) {
    __shared__ uint32_t hist[256];
    __shared__ uint32_t sel_byte, sel_before;
    for (uint64_t q = blockIdx.x; q < nq; q += gridDim.x) {
        const unsigned long long* v = reinterpret_cast<const unsigned long long*>(all_d2) + q * S;
        uint64_t prefix = 0, mask = 0;
        uint32_t need = static_cast<uint32_t>(k);
        for (int p = 7; p >= 0; --p) {
            for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
            __syncthreads();
            for (uint64_t i = threadIdx.x; i < S; i += blockDim.x) {
                const uint64_t key = v[i];
                if ((key & mask) == prefix) atomicAdd(&hist[(key >> (8 * p)) & 255u], 1u);
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                uint32_t cum = 0;
                int b = 0;
                for (; b < 256; ++b) {
                    if (cum + hist[b] >= need) break;
                    cum += hist[b];
                }
                sel_byte = static_cast<uint32_t>(b);
                sel_before = cum;
            }
            __syncthreads();
            prefix |= static_cast<uint64_t>(sel_byte) << (8 * p);
            mask |= 255ULL << (8 * p);
            need -= sel_before;
            __syncthreads();
        }
        if (threadIdx.x == 0) thr[q] = __longlong_as_double(static_cast<long long>(prefix));
        __syncthreads();
    }
}

// Per query: records sorted by (dist^2, position) -> top k.  Overflowing
// queries are listed for the exhaustive redo.
__global__ void gt_finish_kernel(const uint32_t* __restrict__ cnt, const uint64_t* __restrict__ key,
                                 const uint32_t* __restrict__ pos, uint32_t cap, uint64_t nq, int k,
                                 uint32_t* __restrict__ ids, double* __restrict__ dists,
                                 uint32_t* __restrict__ over, uint32_t* __restrict__ n_over) {
    __shared__ uint64_t sk[kGtCap];
    __shared__ uint32_t sp[kGtCap];
    for (uint64_t q = blockIdx.x; q < nq; q += gridDim.x) {
        const uint32_t c = cnt[q];
        if (c > cap || c < static_cast<uint32_t>(k)) {  // overflow (or an invalid bound): exhaustive
            if (threadIdx.x == 0) over[atomicAdd(n_over, 1u)] = static_cast<uint32_t>(q);
            continue;
        }
        uint32_t n2 = 64;
        while (n2 < c) n2 <<= 1;
        for (uint32_t i = threadIdx.x; i < n2; i += blockDim.x) {
            sk[i] = i < c ? key[q * cap + i] : ~0ULL;
            sp[i] = i < c ? pos[q * cap + i] : 0xffffffffu;
        }
        __syncthreads();
        for (uint32_t size = 2; size <= n2; size <<= 1)
            for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
                for (uint32_t i = threadIdx.x; i < n2 / 2; i += blockDim.x) {
                    const uint32_t lo = 2 * i - (i & (stride - 1)), hi = lo + stride;
                    const bool asc = (lo & size) == 0;
                    const uint64_t a = sk[lo], b = sk[hi];
                    const uint32_t pa = sp[lo], pb = sp[hi];
                    const bool less = b < a || (b == a && pb < pa);
                    if (less == asc) {
                        sk[lo] = b;
                        sk[hi] = a;
                        sp[lo] = pb;
                        sp[hi] = pa;
                    }
                }
                __syncthreads();
            }
        for (int t = threadIdx.x; t < k; t += blockDim.x) {
            ids[q * k + t] = sp[t];
            dists[q * k + t] = __dsqrt_rn(__longlong_as_double(static_cast<long long>(sk[t])));
        }
        __syncthreads();
    }
}

__global__ void gt_one_query_kernel(const float* __restrict__ X, uint64_t n, int d, const float* __restrict__ q,
                                    uint64_t* __restrict__ key, uint32_t* __restrict__ val) {
    for (uint64_t z = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; z < n;
         z += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        double acc = 0.0;
        for (int t = 0; t < d; ++t) acc = sq_step(acc, __ldg(q + t), __ldg(X + z * d + t));
        key[z] = static_cast<uint64_t>(__double_as_longlong(acc));
        val[z] = static_cast<uint32_t>(z);
    }
}

__global__ void gt_one_out_kernel(const uint64_t* __restrict__ key, const uint32_t* __restrict__ val, int k,
                                  uint32_t* __restrict__ ids, double* __restrict__ dists) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < k; t += gridDim.x * blockDim.x) {
        ids[t] = val[t];
        dists[t] = __dsqrt_rn(__longlong_as_double(static_cast<long long>(key[t])));
    }
}

}  // namespace

namespace {

void brute_force_chunk(const float* X, uint64_t n, int d, const float* Q, uint64_t nq, int k,
                       const double* thr_hint, uint32_t* ids, double* dists, int device, cudaStream_t s) {
    const uint32_t sms = static_cast<uint32_t>(sm_count(device));
    const uint64_t qtiles = (nq + kGtQ - 1) / kGtQ;
    DevBuf<double> thr(nq);
    if (thr_hint) {
        DETLSH_CUDA(cudaMemcpyAsync(thr.get(), thr_hint, nq * 8, cudaMemcpyDefault, s));
    } else {  // threshold: k-th smallest over a strided sample sized so that about
              // cap / 4 points per query fall within it
        const uint64_t S = std::min<uint64_t>(n, std::max<uint64_t>(2048, 4ULL * k * n / kGtCap)), stride = n / S;
        DevBuf<double> all(nq * S);
        const uint32_t splits = std::max<uint32_t>(1, std::min<uint32_t>(static_cast<uint32_t>((S + kGtR - 1) / kGtR),
                                                                         (4 * sms + qtiles - 1) / qtiles));
        gt_pairs_kernel<<<static_cast<unsigned>(qtiles * splits), 256, 0, s>>>(
            X, n, d, Q, nq, nullptr, stride, S, splits, nullptr, nullptr, nullptr, 0, all.get());
        DETLSH_LAUNCH_CHECK();
        gt_sample_kth_kernel<<<static_cast<unsigned>(std::min<uint64_t>(nq, 8192)), 256, 0, s>>>(all.get(), S, nq, k,
                                                                                            thr.get());
        DETLSH_LAUNCH_CHECK();
    }
    DevBuf<uint32_t> cnt(nq), over(nq), n_over(1);
    DevBuf<uint64_t> key(nq * kGtCap);
    DevBuf<uint32_t> pos(nq * kGtCap);
    DETLSH_CUDA(cudaMemsetAsync(cnt.get(), 0, nq * 4, s));
    DETLSH_CUDA(cudaMemsetAsync(n_over.get(), 0, 4, s));
    const uint64_t rtiles = (n + kGtR - 1) / kGtR;
    const uint32_t splits = static_cast<uint32_t>(std::max<uint64_t>(1, std::min<uint64_t>(rtiles, (8 * sms + qtiles - 1) / qtiles)));
    {
        ProfScope ps("gt_pairs", s);
        gt_pairs_kernel<<<static_cast<unsigned>(qtiles * splits), 256, 0, s>>>(
            X, n, d, Q, nq, thr.get(), 1, n, splits, cnt.get(), key.get(), pos.get(), kGtCap, nullptr);
        DETLSH_LAUNCH_CHECK();
    }
    gt_finish_kernel<<<static_cast<unsigned>(std::min<uint64_t>(nq, 8192)), 256, 0, s>>>(
        cnt.get(), key.get(), pos.get(), kGtCap, nq, k, ids, dists, over.get(), n_over.get());
    DETLSH_LAUNCH_CHECK();
    uint32_t h_over = 0;
    DETLSH_CUDA(cudaMemcpyAsync(&h_over, n_over.get(), 4, cudaMemcpyDeviceToHost, s));
    DETLSH_CUDA(cudaStreamSynchronize(s));
    if (!h_over) return;
    // exhaustive redo: every point of the query, radix-sorted by dist^2 bits
    // (stable, positions ascending within equal keys)
    std::vector<uint32_t> list(h_over);
    DETLSH_CUDA(cudaMemcpyAsync(list.data(), over.get(), h_over * 4, cudaMemcpyDeviceToHost, s));
    DETLSH_CUDA(cudaStreamSynchronize(s));
    DevBuf<uint64_t> k0(n), k1(n);
    DevBuf<uint32_t> v0(n), v1(n), tmp(radix_temp_elems(n));
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((n + 255) / 256, 65535));
    for (const uint32_t q : list) {
        gt_one_query_kernel<<<grid, 256, 0, s>>>(X, n, d, Q + static_cast<uint64_t>(q) * d, k0.get(), v0.get());
        DETLSH_LAUNCH_CHECK();
        const bool flip = radix_sort_pairs<uint64_t>(k0.get(), v0.get(), k1.get(), v1.get(), n, 0, 64, tmp.get(), s);
        gt_one_out_kernel<<<1, 256, 0, s>>>(flip ? k1.get() : k0.get(), flip ? v1.get() : v0.get(), k,
                                            ids + static_cast<uint64_t>(q) * k, dists + static_cast<uint64_t>(q) * k);
        DETLSH_LAUNCH_CHECK();
    }
    DETLSH_CUDA(cudaStreamSynchronize(s));
}

}  // namespace

void brute_force_knn_gpu(const float* X, uint64_t n, int d, const float* Q, uint64_t nq, int k,
                         const double* thr_hint, uint32_t* ids, double* dists, int device, cudaStream_t s) {
    if (k < 1 || static_cast<uint64_t>(k) > n) throw InvalidArgument("brute_force_knn: k must lie in [1, n]");
    if (k > 1024) throw InvalidArgument("brute_force_knn: k above 1024 is not supported");
    if (nq == 0) return;
    StreamScope scope(s);
    // query chunks keep the sample distances (nq x S doubles) and the staged
    // records (nq x 4096) within a few hundred MB
    const uint64_t S = std::min<uint64_t>(n, std::max<uint64_t>(2048, 4ULL * k * n / kGtCap));
    const uint64_t per_q = (thr_hint ? 0 : S * 8) + kGtCap * 12 + 64;
    const uint64_t qc = std::max<uint64_t>(32, (512ULL << 20) / per_q / 32 * 32);
    for (uint64_t q0 = 0; q0 < nq; q0 += qc) {
        const uint64_t m = std::min(qc, nq - q0);
        brute_force_chunk(X, n, d, Q + q0 * d, m, k, thr_hint ? thr_hint + q0 : nullptr, ids + q0 * k,
                          dists + q0 * k, device, s);
    }
}

}  // namespace detlsh_b200
