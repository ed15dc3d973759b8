// fvecs / bvecs / ivecs ingestion straight to device memory (io.cpp:37-85
// semantics): records are (i32 dim, dim elements), every record must carry the
// first record's dimension, the file must end on a record boundary.  The file
// is streamed through two pinned chunk buffers; each chunk's raw bytes (dim
// headers included) go to the device as they are and a kernel strips the
// headers and widens the elements to fp32 in place in the caller's [n][d]
// buffer -- a bvecs file moves 1 byte per element over PCIe, not 4.
#include <cstdio>
#include <cstring>
#include <string>

#include "common.cuh"
#include "vecio.cuh"

namespace detlsh_b200 {

namespace {

int element_width(int kind) { return kind == kVecU8 ? 1 : 4; }

struct File {
    FILE* f = nullptr;
    explicit File(const char* path) : f(std::fopen(path, "rb")) {}
    ~File() {
        if (f) std::fclose(f);
    }
};

std::string str(const char* p) { return p ? std::string(p) : std::string(); }

// rows [row0, row0 + m) of the file, raw (with headers) in `raw`; out [n][d]
__global__ void widen_kernel(const uint8_t* __restrict__ raw, uint64_t m, int d, int kind, uint64_t row0,
                             float* __restrict__ out) {
    const int w = kind == kVecU8 ? 1 : 4;
    const uint64_t rec = 4 + static_cast<uint64_t>(d) * w;
    const uint64_t total = m * static_cast<uint64_t>(d);
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t r = i / d;
        const int t = static_cast<int>(i % d);
        const uint8_t* p = raw + r * rec + 4 + static_cast<uint64_t>(t) * w;
        float v;
        if (kind == kVecU8) {
            v = static_cast<float>(*p);
        } else if (kind == kVecI32) {
            int32_t x;
            memcpy(&x, p, 4);
            v = static_cast<float>(x);
        } else {
            memcpy(&v, p, 4);
        }
        out[(row0 + r) * d + t] = v;
    }
}

}  // namespace

int vec_kind_from_path(const char* path) {
    const std::string p = str(path);
    const auto dot = p.find_last_of('.');
    const std::string ext = dot == std::string::npos ? "" : p.substr(dot);
    if (ext == ".fvecs") return kVecF32;
    if (ext == ".bvecs") return kVecU8;
    if (ext == ".ivecs") return kVecI32;
    throw InvalidArgument("unrecognized vector file extension: " + p);
}

void vectors_shape(const char* path, int kind, uint64_t* n, int* d) {
    File in(path);
    if (!in.f) throw FormatError("cannot open " + str(path));
    const int w = element_width(kind);
    uint64_t rows = 0;
    int dim0 = 0;
    for (;;) {
        int32_t dim = 0;
        const size_t got = std::fread(&dim, 1, 4, in.f);
        if (got == 0) break;  // clean end of file
        if (got != 4) throw FormatError(str(path) + ": truncated dimension field");
        if (dim <= 0) throw FormatError(str(path) + ": non-positive record dimension");
        if (rows == 0) dim0 = dim;
        else if (dim != dim0) throw FormatError(str(path) + ": records disagree on dimension");
        const long body = static_cast<long>(dim) * w;
        const long here = std::ftell(in.f);
        if (std::fseek(in.f, 0, SEEK_END) != 0) throw FormatError("seek failed: " + str(path));
        const long end = std::ftell(in.f);
        if (end - here < body) throw FormatError(str(path) + ": truncated record body");
        std::fseek(in.f, here + body, SEEK_SET);
        ++rows;
    }
    *n = rows;
    *d = dim0;
}

void read_vectors_into(const char* path, int kind, float* d_out, uint64_t n, int d, cudaStream_t s) {
    File in(path);
    if (!in.f) throw FormatError("cannot open " + str(path));
    const int w = element_width(kind);
    const uint64_t rec = 4 + static_cast<uint64_t>(d) * w;
    const uint64_t chunk_rows = std::max<uint64_t>(1, (16ULL << 20) / rec);
    const size_t chunk_bytes = chunk_rows * rec;
    uint8_t* pinned[2] = {nullptr, nullptr};
    cudaEvent_t done[2] = {nullptr, nullptr};
    DevBuf<uint8_t> raw[2];
    struct Cleanup {
        uint8_t** p;
        cudaEvent_t* e;
        ~Cleanup() {
            for (int i = 0; i < 2; ++i) {
                if (e[i]) cudaEventSynchronize(e[i]), cudaEventDestroy(e[i]);
                if (p[i]) cudaFreeHost(p[i]);
            }
        }
    } cleanup{pinned, done};
    StreamScope scope(s);
    for (int i = 0; i < 2; ++i) {
        DETLSH_CUDA(cudaMallocHost(&pinned[i], chunk_bytes));
        DETLSH_CUDA(cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming));
        raw[i].alloc(chunk_bytes);
    }
    uint64_t row = 0;
    for (int b = 0; row < n; b ^= 1) {
        const uint64_t m = std::min<uint64_t>(chunk_rows, n - row);
        DETLSH_CUDA(cudaEventSynchronize(done[b]));  // buffer b's previous copy has drained
        if (std::fread(pinned[b], 1, m * rec, in.f) != m * rec)
            throw FormatError(str(path) + ": truncated record body");
        for (uint64_t r = 0; r < m; ++r) {  // every record carries the same dimension
            int32_t dim;
            std::memcpy(&dim, pinned[b] + r * rec, 4);
            if (dim != d) throw FormatError(str(path) + ": records disagree on dimension");
        }
        DETLSH_CUDA(cudaMemcpyAsync(raw[b].get(), pinned[b], m * rec, cudaMemcpyHostToDevice, s));
        DETLSH_CUDA(cudaEventRecord(done[b], s));
        const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((m * d + 255) / 256, 8192));
        widen_kernel<<<grid, 256, 0, s>>>(raw[b].get(), m, d, kind, row, d_out);
        DETLSH_LAUNCH_CHECK();
        row += m;
    }
    DETLSH_CUDA(cudaStreamSynchronize(s));
}

}  // namespace detlsh_b200
