// Tensor-core (tcgen05, kind::i8) building blocks for exact u8 verification.
// tc_gemm_u8_test: one 128 x N x K tile, C = A . B^T, used by the tests to pin
// the descriptor / TMEM plumbing before it is used in the query path.
#include "common.cuh"
#include "umma.cuh"

namespace detlsh_b200 {

namespace {

__global__ void __launch_bounds__(128) tc_gemm_u8_test_kernel(const uint8_t* __restrict__ A,
                                                              const uint8_t* __restrict__ B, int N,
                                                              int K, int32_t* __restrict__ C) {
    extern __shared__ __align__(128) uint8_t sm[];
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

}  // namespace

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
