#include <cstdlib>
#include <atomic>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"
#include "prof.cuh"

namespace detlsh_b200 {

namespace {
std::atomic<uint64_t> g_launches{0};
std::atomic<bool> g_prof{false};
struct Rec {
    const char* name;
    cudaEvent_t a, b;
};
std::mutex g_mu;
std::vector<Rec> g_recs;
std::vector<std::pair<cudaEvent_t, cudaEvent_t>> g_pool;
}  // namespace

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
uint64_t launch_count() { return g_launches.load(); }
bool profiling_enabled() { return g_prof.load(); }
void profile_enable(bool on) { g_prof.store(on); }

ProfScope::ProfScope(const char* name, cudaStream_t s) : s_(s) {
    if (!g_prof.load()) return;
    std::lock_guard<std::mutex> lk(g_mu);
    Rec r{name, nullptr, nullptr};
    if (!g_pool.empty()) {
        r.a = g_pool.back().first;
        r.b = g_pool.back().second;
        g_pool.pop_back();
    } else {
        cudaEventCreate(&r.a);
        cudaEventCreate(&r.b);
    }
    cudaEventRecord(r.a, s);
    slot_ = static_cast<int>(g_recs.size());
    g_recs.push_back(r);
}

ProfScope::~ProfScope() {
    if (slot_ < 0) return;
    std::lock_guard<std::mutex> lk(g_mu);
    cudaEventRecord(g_recs[slot_].b, s_);
}

int profile_collect(char* names, int names_cap, double* ms, uint64_t* counts, int cap) {
    std::lock_guard<std::mutex> lk(g_mu);
    std::map<std::string, std::pair<double, uint64_t>> acc;
    for (auto& r : g_recs) {
        float t = 0.f;
        cudaEventSynchronize(r.b);
        cudaEventElapsedTime(&t, r.a, r.b);
        auto& e = acc[r.name];
        e.first += t;
        e.second += 1;
        g_pool.emplace_back(r.a, r.b);
    }
    g_recs.clear();
    std::string all;
    int m = 0;
    for (auto& kv : acc) {
        if (m >= cap) break;
        ms[m] = kv.second.first;
        counts[m] = kv.second.second;
        if (!all.empty()) all += ";";
        all += kv.first;
        ++m;
    }
    if (names && names_cap > 0) {
        const size_t c = std::min<size_t>(all.size(), static_cast<size_t>(names_cap - 1));
        all.copy(names, c);
        names[c] = 0;
    }
    return m;
}

}  // namespace detlsh_b200

namespace detlsh_b200 {

cudaStream_t& alloc_stream() {
    thread_local cudaStream_t s = nullptr;
    return s;
}

void ensure_mempool(int device) {
    static std::mutex mu;
    static bool done[64] = {false};
    std::lock_guard<std::mutex> lk(mu);
    if (device < 0 || device >= 64 || done[device]) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t thr = ~0ULL;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        if (const char* e = std::getenv("DETLSH_POOL_RESERVE_GB")) {  // measurement hook: pre-grow the pool
            void* p = nullptr;
            const size_t bytes = static_cast<size_t>(std::atof(e) * 1073741824.0);
            if (bytes && cudaMallocAsync(&p, bytes, 0) == cudaSuccess) cudaFreeAsync(p, 0);
            cudaGetLastError();
            cudaDeviceSynchronize();
        }
    }
    done[device] = true;
}

void reserve_mempool(int device, size_t bytes, cudaStream_t s) {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) != cudaSuccess) return;
    uint64_t reserved = 0, used = 0;
    cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved);
    cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used);
    if (reserved >= used + bytes) return;
    void* p = nullptr;
    if (cudaMallocAsync(&p, bytes, s) != cudaSuccess) {
        cudaGetLastError();  // best effort: the build allocates what it needs anyway
        return;
    }
    cudaFreeAsync(p, s);
}

}  // namespace detlsh_b200
