// TMEM -> register load throughput on one SM: W warps (W/4 per lane quarter)
// each issue `iters` tcgen05.ld.32x32b.x32 (4 KB per warp-load) over a
// 512-column allocation and fold the values (XOR) so nothing is dead.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2406_10938_b200/csrc tmem_ld_bw.cu
#include <cstdio>
#include <cstdint>
#include "umma.cuh"
using namespace detlsh_b200;

template <int W, bool WAIT_EACH>
__global__ void __launch_bounds__(W * 32, 1) ld_kernel(int iters, uint32_t* out, long long* cyc) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) umma::tmem_alloc(&slot, 512);
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
    const uint32_t t = slot;
    const uint32_t lanebase = static_cast<uint32_t>((warp & 3) * 32) << 16;
    uint32_t acc = 0;
    __syncthreads();
    const long long c0 = clock64();
    for (int i = 0; i < iters; ++i) {
        const uint32_t col = ((i * (W / 4) + (warp >> 2)) * 32) & 511;
        uint32_t v[32];
        umma::tmem_ld32_nowait(t + lanebase + col, v);
        if (WAIT_EACH) {
            umma::tmem_wait_ld32(v);
#pragma unroll
            for (int e = 0; e < 32; ++e) acc ^= v[e];
        } else {
            uint32_t w[32];
            umma::tmem_ld32_nowait(t + lanebase + ((col + 256) & 511), w);
            umma::tmem_wait_ld32(v);
            umma::tmem_wait_ld32(w);
#pragma unroll
            for (int e = 0; e < 32; ++e) acc ^= v[e] + w[e];
            ++i;
        }
    }
    __syncthreads();
    const long long c1 = clock64();
    if (threadIdx.x == 0) *cyc = c1 - c0;
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    umma::fence_before_sync();
    __syncthreads();
    if (warp == 0) umma::tmem_free(t, 512);
}

template <int W, bool WAIT_EACH>
void run(uint32_t* out, long long* cyc) {
    const int iters = 4096;
    ld_kernel<W, WAIT_EACH><<<148, W * 32>>>(iters, out, cyc);
    cudaDeviceSynchronize();
    ld_kernel<W, WAIT_EACH><<<148, W * 32>>>(iters, out, cyc);
    long long c = 0;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    const double bytes = static_cast<double>(iters) * W * 4096.0;
    printf("W=%2d %s: %.1f B/cycle/SM (%lld cycles)  err=%s\n", W, WAIT_EACH ? "wait-each " : "2-in-flight", bytes / c, c,
           cudaGetErrorString(cudaGetLastError()));
}

int main() {
    uint32_t* out;
    long long* cyc;
    cudaMalloc(&out, 148 * 1024 * 4);
    cudaMalloc(&cyc, 8);
    run<4, true>(out, cyc);
    run<8, true>(out, cyc);
    run<16, true>(out, cyc);
    run<4, false>(out, cyc);
    run<8, false>(out, cyc);
    run<16, false>(out, cyc);
    return 0;
}
