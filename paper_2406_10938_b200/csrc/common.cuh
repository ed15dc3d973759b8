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
// Maps onto DETLSH_E_FORMAT (detlsh::FormatError, errors.hpp:19-28).
struct FormatError : std::runtime_error {
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

// Stream-ordered allocation.  Every DevBuf is allocated (cudaMallocAsync) and
// freed (cudaFreeAsync) on the stream that is current for its thread when it
// is allocated — set with StreamScope by every host function that launches
// work — so buffers never need a device-wide cudaFree sync and concurrent
// builds on several streams do not serialise.  The device's default memory
// pool keeps freed blocks cached (release threshold raised at first use).
cudaStream_t& alloc_stream();
void ensure_mempool(int device);
// Grows the pool in one mapping to hold `bytes` beyond what is in use, so a
// build's many stream-ordered temporaries (several streams at once) do not
// each map fresh memory the first times round.
void reserve_mempool(int device, size_t bytes, cudaStream_t s);

struct StreamScope {
    cudaStream_t prev;
    explicit StreamScope(cudaStream_t s) : prev(alloc_stream()) { alloc_stream() = s; }
    ~StreamScope() { alloc_stream() = prev; }
};

// Owning device buffer, movable.
template <typename T>
class DevBuf {
public:
    DevBuf() = default;
    explicit DevBuf(size_t count) { alloc(count); }
    ~DevBuf() { release(); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p_(o.p_), n_(o.n_), s_(o.s_) {
        o.p_ = nullptr;
        o.n_ = 0;
    }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) {
            release();
            p_ = o.p_;
            n_ = o.n_;
            s_ = o.s_;
            o.p_ = nullptr;
            o.n_ = 0;
        }
        return *this;
    }
    void alloc(size_t count) {
        release();
        s_ = alloc_stream();
        if (count) DETLSH_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p_), count * sizeof(T), s_));
        n_ = count;
    }
    // grow-only reallocation that keeps the first `keep` elements (stream-ordered)
    void grow(size_t count, size_t keep, cudaStream_t s) {
        if (count <= n_) return;
        T* np = nullptr;
        DETLSH_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&np), count * sizeof(T), s));
        if (keep && p_) DETLSH_CUDA(cudaMemcpyAsync(np, p_, keep * sizeof(T), cudaMemcpyDeviceToDevice, s));
        if (p_) cudaFreeAsync(p_, s);
        p_ = np;
        n_ = count;
        s_ = s;
    }
    void release() {
        if (p_) cudaFreeAsync(p_, s_);
        p_ = nullptr;
        n_ = 0;
    }
    T* get() const { return p_; }
    size_t size() const { return n_; }
    size_t bytes() const { return n_ * sizeof(T); }

private:
    T* p_ = nullptr;
    size_t n_ = 0;
    cudaStream_t s_ = nullptr;
};

// Owned stream, synchronised and destroyed last (declare before the buffers
// that are freed on it).
struct OwnedStream {
    cudaStream_t s = nullptr;
    OwnedStream() = default;
    OwnedStream(const OwnedStream&) = delete;
    OwnedStream& operator=(const OwnedStream&) = delete;
    void create() {
        if (!s) DETLSH_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    }
    ~OwnedStream() {
        if (s) {
            cudaStreamSynchronize(s);
            cudaStreamDestroy(s);
        }
    }
};

inline int ceil_div(int64_t a, int64_t b) { return static_cast<int>((a + b - 1) / b); }

int sm_count(int device);

}  // namespace detlsh_b200
