// Probe: does mma.sync m8n8k4 f64 accumulate as a sequential fma chain over k
// (bit-identical to acc = fma(a_t, b_t, acc) for t = 0..3)?  Prints mismatches.
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cmath>
#include <random>
#include <vector>

__global__ void k_dmma(const double* A, const double* B, const double* C, double* D, int steps) {
    // one warp: A [8][4*steps] row-major (row = output row), B [4*steps][8] col-major-ish per step
    const int lane = threadIdx.x;
    // fragment layout m8n8k4 f64: A: each thread holds 1 element: row = lane / 4, col = lane % 4
    // B: each thread holds 1 element: row(k) = lane % 4, col = lane / 4
    // C/D: each thread holds 2 elements: row = lane / 4, cols = (lane % 4) * 2 + {0,1}
    double c0 = C[(lane / 4) * 8 + (lane % 4) * 2], c1 = C[(lane / 4) * 8 + (lane % 4) * 2 + 1];
    for (int s = 0; s < steps; ++s) {
        const double a = A[(lane / 4) * (4 * steps) + 4 * s + (lane % 4)];
        const double b = B[(4 * s + (lane % 4)) * 8 + lane / 4];
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
    }
    D[(lane / 4) * 8 + (lane % 4) * 2] = c0;
    D[(lane / 4) * 8 + (lane % 4) * 2 + 1] = c1;
}

int main() {
    const int steps = 32, K = 4 * steps;
    std::mt19937_64 g(7);
    std::uniform_real_distribution<float> u(-1.f, 1.f);
    std::uniform_int_distribution<int> e(-20, 20);
    long mism = 0, total = 0;
    double *dA, *dB, *dC, *dD;
    cudaMalloc(&dA, 8 * K * 8); cudaMalloc(&dB, K * 8 * 8); cudaMalloc(&dC, 64 * 8); cudaMalloc(&dD, 64 * 8);
    for (int trial = 0; trial < 2000; ++trial) {
        std::vector<double> A(8 * K), B(K * 8), C(64, 0.0), D(64);
        for (auto& x : A) x = (double)std::ldexp(u(g), e(g));   // float values, exact in double
        for (auto& x : B) x = (double)std::ldexp(u(g), e(g));
        cudaMemcpy(dA, A.data(), A.size() * 8, cudaMemcpyHostToDevice);
        cudaMemcpy(dB, B.data(), B.size() * 8, cudaMemcpyHostToDevice);
        cudaMemcpy(dC, C.data(), 64 * 8, cudaMemcpyHostToDevice);
        k_dmma<<<1, 32>>>(dA, dB, dC, dD, steps);
        cudaMemcpy(D.data(), dD, 64 * 8, cudaMemcpyDeviceToHost);
        for (int r = 0; r < 8; ++r)
            for (int c = 0; c < 8; ++c) {
                double acc = 0.0;
                for (int t = 0; t < K; ++t) acc = std::fma(A[r * K + t], B[t * 8 + c], acc);
                ++total;
                if (std::memcmp(&acc, &D[r * 8 + c], 8)) ++mism;
            }
    }
    printf("dmma vs sequential fma chain: %ld mismatches of %ld\n", mism, total);
    return 0;
}
