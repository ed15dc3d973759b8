// Launch accounting and optional per-kernel CUDA-event timing.
//   * every kernel launch bumps a process-wide counter (detlsh_launch_count)
//   * with profiling enabled (detlsh_profile_enable), ProfScope records an
//     event pair on the launching stream around the kernel; collect() sums
//     elapsed milliseconds per kernel name.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace detlsh_b200 {

void count_launch();
uint64_t launch_count();
bool profiling_enabled();
void profile_enable(bool on);

class ProfScope {
public:
    ProfScope(const char* name, cudaStream_t s);
    ~ProfScope();

private:
    int slot_ = -1;
    cudaStream_t s_;
};

// Writes up to cap (name, total ms, launches) entries; returns count.
int profile_collect(char* names, int names_cap, double* ms, uint64_t* counts, int cap);

}  // namespace detlsh_b200
