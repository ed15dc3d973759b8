// Shared helpers for the sm_100a kernels and their host launchers.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>

#include "prof.cuh"

namespace detlsh_b200 {

// Maps onto DETLSH_E_INVALID (std::invalid_argument in the reference).
struct InvalidArgument : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
// Maps onto DETLSH_E_CUDA.
struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

#define DETLSH_CUDA(expr)                                                                     \
    do {                                                                                      \
        cudaError_t _e = (expr);                                                              \
        if (_e != cudaSuccess)                                                                \
            throw ::detlsh_b200::CudaError(std::string(#expr) + ": " + cudaGetErrorString(_e) + \
                                           " (" + __FILE__ + ":" + std::to_string(__LINE__) + ")"); \
    } while (0)

#define DETLSH_LAUNCH_CHECK()             \
    do {                                    \
        ::detlsh_b200::count_launch();      \
        DETLSH_CUDA(cudaGetLastError());    \
    } while (0)

constexpr int kMaxK = 24;      // validate_params: K in [1, 24] (index.cpp:17)
constexpr int kMaxRegions = 256;

// Owning device buffer (cudaMalloc / cudaFree), movable.
template <typename T>
class DevBuf {
public:
    DevBuf() = default;
    explicit DevBuf(size_t count) { alloc(count); }
    ~DevBuf() { release(); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p_(o.p_), n_(o.n_) {
        o.p_ = nullptr;
        o.n_ = 0;
    }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) {
            release();
            p_ = o.p_;
            n_ = o.n_;
            o.p_ = nullptr;
            o.n_ = 0;
        }
        return *this;
    }
    void alloc(size_t count) {
        release();
        if (count) DETLSH_CUDA(cudaMalloc(&p_, count * sizeof(T)));
        n_ = count;
    }
    // grow-only reallocation that keeps the first `keep` elements
    void grow(size_t count, size_t keep, cudaStream_t s) {
        if (count <= n_) return;
        T* np = nullptr;
        DETLSH_CUDA(cudaMalloc(&np, count * sizeof(T)));
        if (keep && p_) DETLSH_CUDA(cudaMemcpyAsync(np, p_, keep * sizeof(T), cudaMemcpyDeviceToDevice, s));
        DETLSH_CUDA(cudaStreamSynchronize(s));
        release();
        p_ = np;
        n_ = count;
    }
    void release() {
        if (p_) cudaFree(p_);
        p_ = nullptr;
        n_ = 0;
    }
    T* get() const { return p_; }
    size_t size() const { return n_; }
    size_t bytes() const { return n_ * sizeof(T); }

private:
    T* p_ = nullptr;
    size_t n_ = 0;
};

inline int ceil_div(int64_t a, int64_t b) { return static_cast<int>((a + b - 1) / b); }

int sm_count(int device);

}  // namespace detlsh_b200
