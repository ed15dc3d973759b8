// Measured compute peaks on this B200 for the two tensor pipes the DET-LSH
// kernels use, so bench.py's rooflines divide by measured numbers, not
// datasheet ones:
//   * FP64 tensor (mma.sync.m8n8k4.f64, DMMA): the exact-projection fallback
//     for non-integral data (stages.cu project_dmma_kernel);
//   * tcgen05.mma kind::i8 (128 x 256 x 32, s32 in TMEM): project_tc and
//     tc_score.
// Every SM runs a persistent CTA issuing independent MMA chains from registers
// (DMMA) or from a resident shared-memory operand (tcgen05; one elected thread,
// mbarrier commit every 64 MMAs).  Timed with CUDA events, clocks unlocked.
// Prints one JSON line.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2406_10938_b200/csrc peaks.cu -o peaks
#include <cstdio>
#include <cstdint>

#include "umma.cuh"
using namespace detlsh_b200;

__global__ void __launch_bounds__(256) dmma_kernel(int iters, double* out) {
    double acc[8][2];
    double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[c][0] = acc[c][1] = 0.0;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < 8; ++c)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(acc[c][0]), "+d"(acc[c][1])
                         : "d"(a), "d"(b));
    }
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < 8; ++c) s += acc[c][0] + acc[c][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

constexpr int kN = 256, kK = 32;  // one MMA: 128 x 256 x 32 int8

__global__ void __launch_bounds__(128, 1) i8_kernel(int iters, uint32_t* out) {
    __shared__ __align__(1024) uint8_t sA[128 * kK];
    __shared__ __align__(1024) uint8_t sB[kN * kK];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t slot;
    for (int i = threadIdx.x; i < 128 * kK; i += blockDim.x) sA[i] = static_cast<uint8_t>(i * 7);
    for (int i = threadIdx.x; i < kN * kK; i += blockDim.x) sB[i] = static_cast<uint8_t>(i * 13);
    if (threadIdx.x == 0) {
        umma::mbar_init(&bar, 1);
        umma::fence_mbar_init();
    }
    umma::fence_async_smem();
    if (threadIdx.x < 32) umma::tmem_alloc(&slot, 512);
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
    const uint32_t tmem = slot;
    if (threadIdx.x == 0) {
        const uint32_t idesc = umma::idesc_u8_s32(128, kN);
        const uint64_t da = umma::smem_desc(umma::smem_u32(sA), 128 * 16, 128);
        const uint64_t db = umma::smem_desc(umma::smem_u32(sB), kN * 16, 128);
        uint32_t ph = 0;
        for (int i = 0; i < iters; ++i) {
            umma::mma_u8(tmem + (i & 1) * kN, da, db, idesc, 1u);
            if ((i & 63) == 63) {
                umma::commit(&bar);
                umma::mbar_wait(&bar, ph);
                ph ^= 1;
            }
        }
        umma::commit(&bar);
        umma::mbar_wait(&bar, ph);
    }
    __syncthreads();
    umma::fence_after_sync();
    uint32_t v[32];
    umma::tmem_ld32(tmem + (static_cast<uint32_t>(threadIdx.x & 96) << 16), v);
    out[blockIdx.x * blockDim.x + threadIdx.x] = v[0] ^ v[31];
    umma::fence_before_sync();
    __syncthreads();
    if (threadIdx.x < 32) umma::tmem_free(tmem, 512);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* dout;
    uint32_t* iout;
    cudaMalloc(&dout, sizeof(double) * sms * 8 * 256);
    cudaMalloc(&iout, sizeof(uint32_t) * sms * 128);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms = 0.f;
    // FP64 DMMA: 8 CTAs x 8 warps per SM, 8 independent chains per warp
    const int diters = 20000;
    dmma_kernel<<<sms * 8, 256>>>(100, dout);
    cudaEventRecord(e0);
    dmma_kernel<<<sms * 8, 256>>>(diters, dout);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double dflops = 2.0 * 8 * 8 * 4 * 8.0 * diters * (sms * 8 * 8);  // m8n8k4 = 256 FMA per warp-MMA
    const double dmma_tf = dflops / (ms * 1e-3) / 1e12;
    // tcgen05 kind::i8
    const int iiters = 200000;
    i8_kernel<<<sms, 128>>>(1000, iout);
    cudaEventRecord(e0);
    i8_kernel<<<sms, 128>>>(iiters, iout);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double iops = 2.0 * 128 * kN * kK * static_cast<double>(iiters) * sms;
    const double i8_tops = iops / (ms * 1e-3) / 1e12;
    printf("{\"fp64_dmma_tflops\": %.2f, \"int8_tcgen05_tops\": %.1f, \"sms\": %d, \"err\": \"%s\"}\n", dmma_tf,
           i8_tops, sms, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
