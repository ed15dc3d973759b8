// Host-side determinism core of the B200 DET-LSH path.
//
// Everything that must be bit-identical to the reference and is inherently
// scalar/sequential lives here, in host C++: the mt19937_64 stream and its
// transforms (rng.hpp:13-61), chi^2 numerics (chi2.cpp), derived parameters
// (projection.cpp:92-102), the hash family (projection.cpp:11-23), the
// reference-compatible breakpoint sample replay (encoder.cpp:29-143) and the
// r_min grid walk (index.cpp:60-136).  The data-parallel work is in the .cu
// files.
#pragma once

#include <cstdint>
#include <memory>
#include <random>
#include <vector>

namespace detlsh_b200 {

class Rng {
public:
    explicit Rng(uint64_t seed) : gen_(seed) {}
    uint64_t next_u64() { return gen_(); }
    // rng.hpp:20-26
    uint64_t bounded(uint64_t bound) {
        // threshold = 2^64 mod bound < bound, so r >= bound accepts without it
        for (;;) {
            const uint64_t r = gen_();
            if (r >= bound || r >= (0 - bound) % bound) return r % bound;
        }
    }
    double real01() { return static_cast<double>(gen_() >> 11) * 0x1.0p-53; }
    double normal();  // rng.hpp:32-47

private:
    std::mt19937_64 gen_;
    double spare_ = 0.0;
    bool have_spare_ = false;
};

uint64_t mix_seed(uint64_t seed, uint64_t stream);  // rng.hpp:56-61

enum : uint64_t { kStreamFamily = 0, kStreamBreakpoints = 1, kStreamProbes = 2 };  // index.cpp:14

double regularized_gamma_p(double a, double x);
double chi2_cdf(double x, int k);
double chi2_pdf(double x, int k);
double chi2_quantile(double alpha, int k);

struct Derived {
    double alpha1, alpha2, epsilon, beta;
};
Derived derive_params(int K, double c, int L);
uint64_t candidate_budget(double beta, uint64_t n, int k);

void sample_hash_family(int d, int K, int L, uint64_t seed, float* out);

// Reference-compatible breakpoint sample (encoder.cpp:105-143) driven by the
// host: the partial Fisher-Yates over a persistent index array and every
// quickselect pivot share ONE stream, so space i's sample depends on how many
// draws space i-1's quickselects consumed.  The replay therefore re-runs the
// multi-target quickselect (encoder.cpp:57-103) on the exact sample values.
class RefSampler {
public:
    RefSampler(uint64_t n, uint64_t n_s, int n_regions, uint64_t seed);
    // Draws space i's sample positions (call once per space, in order).
    const std::vector<uint32_t>& next_space_indices();
    // Replays one (space, dim) row: `sample` is reordered in place, the
    // n_regions+1 boundaries go to `row_out`.  Rows must be fed in order.
    void select_row(float* sample, float* row_out);
    uint64_t draws() const { return draws_; }

private:
    uint64_t n_, n_s_;
    int n_regions_;
    Rng rng_;
    std::unique_ptr<uint32_t[]> idx_;  // [n] (filled in parallel: no serial first touch)
    std::vector<uint32_t> sample_idx_;
    std::vector<uint32_t> targets_;
    std::vector<uint64_t> raw_;  // one space's raw draws
    uint64_t draws_ = 0;
};

// Stateless multi-target quickselect replay on one sample (encoder.cpp:57-103).
void select_row_breakpoints(float* a, uint64_t n_s, int n_regions, Rng& rng, float* row_out,
                            uint64_t* draws);

// r_min grid walk (index.cpp:60-73, 126-135) given, per probe, the budget-th
// smallest exact projected distance T_p: reaches(r) <=> T_p <= eps * r.
double rmin_from_order_stats(const std::vector<double>& T, double guess, double epsilon,
                             double c);

}  // namespace detlsh_b200
