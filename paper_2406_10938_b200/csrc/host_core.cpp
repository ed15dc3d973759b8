// Host determinism core — see host_core.hpp.
#include "host_core.hpp"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <numeric>
#include <mutex>
#include <functional>
#include <condition_variable>
#include <stdexcept>
#include <thread>

#include <immintrin.h>

namespace detlsh_b200 {

double Rng::normal() {
    if (have_spare_) {
        have_spare_ = false;
        return spare_;
    }
    double u1;
    do {
        u1 = real01();
    } while (u1 <= 0.0);
    const double u2 = real01();
    const double mag = std::sqrt(-2.0 * std::log(u1));
    const double ang = 2.0 * 3.141592653589793 * u2;
    spare_ = mag * std::sin(ang);
    have_spare_ = true;
    return mag * std::cos(ang);
}

uint64_t mix_seed(uint64_t seed, uint64_t stream) {
    uint64_t z = seed + 0x9e3779b97f4a7c15ULL * (stream + 1);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

// ---- chi^2 (chi2.cpp:12-107) ------------------------------------------------
namespace {
double series_p(double a, double x) {
    double ap = a, sum = 1.0 / a, del = sum;
    for (int i = 0; i < 1000; ++i) {
        ap += 1.0;
        del *= x / ap;
        sum += del;
        if (std::fabs(del) < std::fabs(sum) * 1e-16) break;
    }
    return sum * std::exp(-x + a * std::log(x) - std::lgamma(a));
}
double contfrac_q(double a, double x) {
    constexpr double tiny = 1e-300;
    double b = x + 1.0 - a, c = 1.0 / tiny, d = 1.0 / b, h = d;
    for (int i = 1; i <= 1000; ++i) {
        const double an = -static_cast<double>(i) * (static_cast<double>(i) - a);
        b += 2.0;
        d = an * d + b;
        if (std::fabs(d) < tiny) d = tiny;
        c = b + an / c;
        if (std::fabs(c) < tiny) c = tiny;
        d = 1.0 / d;
        const double del = d * c;
        h *= del;
        if (std::fabs(del - 1.0) < 1e-16) break;
    }
    return std::exp(-x + a * std::log(x) - std::lgamma(a)) * h;
}
}  // namespace

double regularized_gamma_p(double a, double x) {
    if (a <= 0.0) throw std::invalid_argument("regularized_gamma_p: a must be positive");
    if (x < 0.0) throw std::invalid_argument("regularized_gamma_p: x must be non-negative");
    if (x == 0.0) return 0.0;
    return x < a + 1.0 ? series_p(a, x) : 1.0 - contfrac_q(a, x);
}

double chi2_cdf(double x, int k) {
    if (k < 1) throw std::invalid_argument("chi2_cdf: k must be positive");
    return x <= 0.0 ? 0.0 : regularized_gamma_p(0.5 * k, 0.5 * x);
}

double chi2_pdf(double x, int k) {
    if (k < 1) throw std::invalid_argument("chi2_pdf: k must be positive");
    if (x <= 0.0) return 0.0;
    const double hk = 0.5 * k;
    return std::exp((hk - 1.0) * std::log(x) - 0.5 * x - hk * 0.6931471805599453 -
                    std::lgamma(hk));
}

double chi2_quantile(double alpha, int k) {
    if (k < 1) throw std::invalid_argument("chi2_quantile: k must be positive");
    if (!(alpha > 0.0) || alpha > 1.0)
        throw std::invalid_argument("chi2_quantile: alpha must lie in (0, 1]");
    if (alpha == 1.0) return 0.0;
    const double target = 1.0 - alpha;
    double lo = 0.0;
    double hi = static_cast<double>(k) + 10.0 * std::sqrt(2.0 * k) + 10.0;
    for (int i = 0; i < 200 && chi2_cdf(hi, k) < target; ++i) hi *= 2.0;
    for (int i = 0; i < 200; ++i) {
        const double mid = 0.5 * (lo + hi);
        if (mid == lo || mid == hi) break;
        (chi2_cdf(mid, k) < target ? lo : hi) = mid;
    }
    double x = 0.5 * (lo + hi);
    for (int i = 0; i < 32; ++i) {
        const double f = chi2_cdf(x, k) - target;
        if (std::fabs(f) < 1e-12) break;
        const double df = chi2_pdf(x, k);
        if (df <= 0.0) break;
        const double nx = x - f / df;
        if (nx <= lo || nx >= hi) break;
        x = nx;
    }
    return x;
}

Derived derive_params(int K, double c, int L) {
    if (K < 1 || L < 1) throw std::invalid_argument("derive_params: K, L must be positive");
    if (!(c > 1.0)) throw std::invalid_argument("derive_params: c must exceed 1");
    Derived p;
    p.alpha1 = std::exp(-1.0 / static_cast<double>(L));
    const double eps_sq = chi2_quantile(p.alpha1, K);
    p.epsilon = std::sqrt(eps_sq);
    p.alpha2 = 1.0 - chi2_cdf(eps_sq / (c * c), K);
    p.beta = 2.0 * (1.0 - std::pow(p.alpha2, static_cast<double>(L)));
    return p;
}

uint64_t candidate_budget(double beta, uint64_t n, int k) {
    const double raw = std::max(0.0, beta) * static_cast<double>(n) + static_cast<double>(k);
    const auto b = static_cast<uint64_t>(std::ceil(raw));
    return std::min<uint64_t>(b, n);
}

void sample_hash_family(int d, int K, int L, uint64_t seed, float* out) {
    if (d < 1 || K < 1 || L < 1)
        throw std::invalid_argument("sample_hash_family: d, K, L must be positive");
    Rng rng(seed);
    const size_t total = static_cast<size_t>(L) * K * d;
    for (size_t i = 0; i < total; ++i) out[i] = static_cast<float>(rng.normal());
}

// ---- breakpoint replay (encoder.cpp:14-103) ---------------------------------
namespace {

// The sentinel scan-and-swap loop of partition_around (encoder.cpp:41-52):
// a[lo+1] == pivot bounds the right scan, a[hi-1] >= pivot the left scan.
size_t hoare_scan_simple(float* a, size_t lo, size_t hi, float pv) {
    size_t i = lo + 1, j = hi - 1;
    for (;;) {
        while (a[++i] < pv) {
        }
        while (a[--j] > pv) {
        }
        if (i >= j) break;
        std::swap(a[i], a[j]);
    }
    return j;
}

// The same loop, branch-light.  Hoare swaps the k-th left stopper (a >= pv,
// ascending) with the k-th right stopper (a <= pv, descending) while they are
// ordered; every position strictly between the current i and j still holds
// its original value, so stoppers can be collected ahead of time in blocks
// (cmov-style appends, no data-dependent branch per element).  Crossing rule,
// derived from the sentinel loop: i' = next left stopper below j, else j;
// j' = next right stopper at or above i', else i' - 1; stop when i' >= j'.
// Buffered stoppers that fell outside (i, j) by the time they are consumed
// are exactly the positions the sentinel loop would have crossed.
size_t hoare_scan_blocked(float* a, size_t lo, size_t hi, float pv) {
    constexpr int64_t B = 64;
    int64_t lb[B], rb[B];
    int ln = 0, lh = 0, rn = 0, rh = 0;
    int64_t i = static_cast<int64_t>(lo) + 1, j = static_cast<int64_t>(hi) - 1;
    int64_t lgen = i + 1, rgen = j - 1;
    for (;;) {
        int64_t in;
        for (;;) {  // next left stopper in (i, j)
            if (lh < ln) {
                in = lb[lh++];
                if (in >= j) in = j;
                break;
            }
            if (lgen >= j) {
                in = j;
                break;
            }
            const int64_t end = std::min(lgen + B, j);
            ln = 0;
            lh = 0;
            for (int64_t x = lgen; x < end; ++x) {
                lb[ln] = x;
                ln += a[x] >= pv;
            }
            lgen = end;
        }
        int64_t jn;
        for (;;) {  // next right stopper in [in, j)
            if (rh < rn) {
                jn = rb[rh++];
                if (jn < in) jn = in - 1;
                break;
            }
            if (rgen < in) {
                jn = in - 1;
                break;
            }
            const int64_t end = std::max(rgen - B, in - 1);
            rn = 0;
            rh = 0;
            for (int64_t y = rgen; y > end; --y) {
                rb[rn] = y;
                rn += a[y] <= pv;
            }
            rgen = end;
        }
        if (in >= jn) return static_cast<size_t>(jn);
        std::swap(a[in], a[jn]);
        i = in;
        j = jn;
    }
}

// AVX2 flavour of hoare_scan_blocked: the stopper lists are filled 8 floats at
// a time (compare + movemask + a compress LUT); the pairing loop is unchanged,
// so the swaps and the returned position are the same.
struct CompressLut {
    alignas(32) int32_t asc[256][8];
    alignas(32) int32_t desc[256][8];
    CompressLut() {
        for (int m = 0; m < 256; ++m) {
            int k = 0;
            for (int b = 0; b < 8; ++b)
                if ((m >> b) & 1) asc[m][k++] = b;
            for (; k < 8; ++k) asc[m][k] = 0;
            k = 0;
            for (int b = 7; b >= 0; --b)
                if ((m >> b) & 1) desc[m][k++] = b;
            for (; k < 8; ++k) desc[m][k] = 0;
        }
    }
};
const CompressLut kLut;

__attribute__((target("avx2,popcnt"))) size_t hoare_scan_avx2(float* a, size_t lo, size_t hi,
                                                              float pv) {
    constexpr int64_t B = 64;
    alignas(32) int32_t lb[B + 8], rb[B + 8];
    int ln = 0, lh = 0, rn = 0, rh = 0;
    int64_t i = static_cast<int64_t>(lo) + 1, j = static_cast<int64_t>(hi) - 1;
    int64_t lgen = i + 1, rgen = j - 1;
    const __m256 vp = _mm256_set1_ps(pv);
    for (;;) {
        // batch of ordered pairs straight from both buffers: L ascending, R
        // descending, so L_t < R_t already implies L_t < j and R_t > i
        {
            const int avail = std::min(ln - lh, rn - rh);
            int t = 0;
            while (t < avail && lb[lh + t] < rb[rh + t]) {
                std::swap(a[lb[lh + t]], a[rb[rh + t]]);
                ++t;
            }
            if (t) {
                i = lb[lh + t - 1];
                j = rb[rh + t - 1];
                lh += t;
                rh += t;
            }
        }
        int64_t in;
        for (;;) {  // next left stopper in (i, j)
            if (lh < ln) {
                in = lb[lh++];
                if (in >= j) in = j;
                break;
            }
            if (lgen >= j) {
                in = j;
                break;
            }
            const int64_t end = std::min(lgen + B, j);
            ln = 0;
            lh = 0;
            int64_t x = lgen;
            for (; x + 8 <= end; x += 8) {
                const int m = _mm256_movemask_ps(_mm256_cmp_ps(_mm256_loadu_ps(a + x), vp, _CMP_GE_OQ));
                const __m256i pos = _mm256_add_epi32(
                    _mm256_load_si256(reinterpret_cast<const __m256i*>(kLut.asc[m])),
                    _mm256_set1_epi32(static_cast<int32_t>(x)));
                _mm256_storeu_si256(reinterpret_cast<__m256i*>(lb + ln), pos);
                ln += __builtin_popcount(static_cast<unsigned>(m));
            }
            for (; x < end; ++x) {
                lb[ln] = static_cast<int32_t>(x);
                ln += a[x] >= pv;
            }
            lgen = end;
        }
        int64_t jn;
        for (;;) {  // next right stopper in [in, j)
            if (rh < rn) {
                jn = rb[rh++];
                if (jn < in) jn = in - 1;
                break;
            }
            if (rgen < in) {
                jn = in - 1;
                break;
            }
            const int64_t end = std::max(rgen - B, in - 1);
            rn = 0;
            rh = 0;
            int64_t y = rgen;
            for (; y - 8 >= end; y -= 8) {
                const int64_t b0 = y - 7;
                const int m = _mm256_movemask_ps(_mm256_cmp_ps(_mm256_loadu_ps(a + b0), vp, _CMP_LE_OQ));
                const __m256i pos = _mm256_add_epi32(
                    _mm256_load_si256(reinterpret_cast<const __m256i*>(kLut.desc[m])),
                    _mm256_set1_epi32(static_cast<int32_t>(b0)));
                _mm256_storeu_si256(reinterpret_cast<__m256i*>(rb + rn), pos);
                rn += __builtin_popcount(static_cast<unsigned>(m));
            }
            for (; y > end; --y) {
                rb[rn] = static_cast<int32_t>(y);
                rn += a[y] <= pv;
            }
            rgen = end;
        }
        if (in >= jn) return static_cast<size_t>(jn);
        std::swap(a[in], a[jn]);
        i = in;
        j = jn;
    }
}

// AVX-512 flavour: 16-wide compares with compressed stopper stores, and the
// ordered pairs swapped 16 at a time by gather/scatter (within a batch the left
// positions ascend, the right ones descend and every left < its right, so no
// position repeats).  Same swaps, same result as hoare_scan_simple.
__attribute__((target("avx512f,avx512vl,avx512bw,avx512dq,popcnt,bmi,bmi2")))
size_t hoare_scan_avx512(float* a, size_t lo, size_t hi, float pv) {
    constexpr int64_t B = 128;
    alignas(64) int32_t lb[B + 16], rb[B + 16];
    int ln = 0, lh = 0, rn = 0, rh = 0;
    int64_t i = static_cast<int64_t>(lo) + 1, j = static_cast<int64_t>(hi) - 1;
    int64_t lgen = i + 1, rgen = j - 1;
    const __m512 vp = _mm512_set1_ps(pv);
    const __m512i iota = _mm512_setr_epi32(0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15);
    const __m512i rev = _mm512_setr_epi32(15, 14, 13, 12, 11, 10, 9, 8, 7, 6, 5, 4, 3, 2, 1, 0);
    for (;;) {
        {  // ordered pairs straight from both buffers, 16 per gather/scatter
            const int avail = std::min(ln - lh, rn - rh);
            int t = 0;
            while (t < avail) {
                const int w = std::min(16, avail - t);
                const __mmask16 live = static_cast<__mmask16>((1u << w) - 1u);
                const __m512i L = _mm512_maskz_loadu_epi32(live, lb + lh + t);
                const __m512i R = _mm512_maskz_loadu_epi32(live, rb + rh + t);
                const __mmask16 ok = _mm512_mask_cmplt_epi32_mask(live, L, R);
                const int nv = static_cast<int>(_tzcnt_u32(~static_cast<uint32_t>(ok)));
                const __mmask16 km = static_cast<__mmask16>((1u << nv) - 1u);
                if (nv) {
                    const __m512 vl = _mm512_mask_i32gather_ps(_mm512_setzero_ps(), km, L, a, 4);
                    const __m512 vr = _mm512_mask_i32gather_ps(_mm512_setzero_ps(), km, R, a, 4);
                    _mm512_mask_i32scatter_ps(a, km, L, vr, 4);
                    _mm512_mask_i32scatter_ps(a, km, R, vl, 4);
                }
                t += nv;
                if (nv < w) break;
            }
            if (t) {
                i = lb[lh + t - 1];
                j = rb[rh + t - 1];
                lh += t;
                rh += t;
            }
        }
        int64_t in;
        for (;;) {  // next left stopper in (i, j)
            if (lh < ln) {
                in = lb[lh++];
                if (in >= j) in = j;
                break;
            }
            if (lgen >= j) {
                in = j;
                break;
            }
            const int64_t end = std::min(lgen + B, j);
            ln = 0;
            lh = 0;
            int64_t x = lgen;
            for (; x + 16 <= end; x += 16) {
                const __mmask16 m = _mm512_cmp_ps_mask(_mm512_loadu_ps(a + x), vp, _CMP_GE_OQ);
                _mm512_mask_compressstoreu_epi32(lb + ln, m, _mm512_add_epi32(iota, _mm512_set1_epi32(static_cast<int32_t>(x))));
                ln += _mm_popcnt_u32(m);
            }
            for (; x < end; ++x) {
                lb[ln] = static_cast<int32_t>(x);
                ln += a[x] >= pv;
            }
            lgen = end;
        }
        int64_t jn;
        for (;;) {  // next right stopper in [in, j)
            if (rh < rn) {
                jn = rb[rh++];
                if (jn < in) jn = in - 1;
                break;
            }
            if (rgen < in) {
                jn = in - 1;
                break;
            }
            const int64_t end = std::max(rgen - B, in - 1);
            rn = 0;
            rh = 0;
            int64_t y = rgen;
            for (; y - 16 >= end; y -= 16) {  // a[y], a[y-1], ..., a[y-15]
                const __m512 v = _mm512_permutexvar_ps(rev, _mm512_loadu_ps(a + y - 15));
                const __mmask16 m = _mm512_cmp_ps_mask(v, vp, _CMP_LE_OQ);
                _mm512_mask_compressstoreu_epi32(rb + rn, m, _mm512_sub_epi32(_mm512_set1_epi32(static_cast<int32_t>(y)), iota));
                rn += _mm_popcnt_u32(m);
            }
            for (; y > end; --y) {
                rb[rn] = static_cast<int32_t>(y);
                rn += a[y] <= pv;
            }
            rgen = end;
        }
        if (in >= jn) return static_cast<size_t>(jn);
        std::swap(a[in], a[jn]);
        i = in;
        j = jn;
    }
}

bool have_avx512() {
    static const bool v = __builtin_cpu_supports("avx512f") && __builtin_cpu_supports("avx512vl") &&
                          __builtin_cpu_supports("avx512bw") && __builtin_cpu_supports("avx512dq") &&
                          __builtin_cpu_supports("bmi2");
    return v;
}

// Closed form of the sentinel loop when the pivot value is unique in the
// segment (no other element compares equal to pv, a[lo] < pv < a[hi-1]).  Then
// the segment holds `lt` smaller elements in the scan region [lo+2, hi-2], the
// pivot ends at p = lo + 1 + lt, and the loop swaps the k-th element > pv of
// the left region [lo+2, p] (ascending) with the k-th element < pv of the right
// region [p+1, hi-2] (descending) for every k <= m, m being the count of either
// (equal by the rank balance) — the crossing test fails exactly after the m-th
// pair.  So the partition is three streaming passes instead of a data-dependent
// two-pointer walk: count (gives p), compress the right region's small values
// top-down, then rewrite the left region (compress its large values, expand the
// small ones into their slots) and the right region (expand the large ones,
// bottom-up).  Returns false, touching nothing, when pv is not unique; the
// caller then runs the loop itself.  `buf` holds >= 2 * (hi - lo) + 32 floats
// (full-width stores past the live entries).
__attribute__((target("avx512f,avx512vl,avx512bw,avx512dq,popcnt,bmi,bmi2")))
bool hoare_rewrite_avx512(float* a, size_t lo, size_t hi, float pv, float* buf, size_t* p_out) {
    if (!(a[lo] < pv) || !(a[hi - 1] > pv)) return false;
    const __m512 vp = _mm512_set1_ps(pv);
    const __m512i rev = _mm512_setr_epi32(15, 14, 13, 12, 11, 10, 9, 8, 7, 6, 5, 4, 3, 2, 1, 0);
    const int64_t s0 = static_cast<int64_t>(lo) + 2, s1 = static_cast<int64_t>(hi) - 1;  // scan region [s0, s1)
    // pass 1: ranks
    uint64_t lt = 0, eq = 0;
    int64_t x = s0;
    for (; x + 16 <= s1; x += 16) {
        const __m512 v = _mm512_loadu_ps(a + x);
        lt += _mm_popcnt_u32(_mm512_cmp_ps_mask(v, vp, _CMP_LT_OQ));
        eq += _mm_popcnt_u32(_mm512_cmp_ps_mask(v, vp, _CMP_EQ_OQ));
    }
    if (x < s1) {
        const __mmask16 k = static_cast<__mmask16>((1u << (s1 - x)) - 1u);
        const __m512 v = _mm512_maskz_loadu_ps(k, a + x);
        lt += _mm_popcnt_u32(_mm512_mask_cmp_ps_mask(k, v, vp, _CMP_LT_OQ));
        eq += _mm_popcnt_u32(_mm512_mask_cmp_ps_mask(k, v, vp, _CMP_EQ_OQ));
    }
    if (eq) return false;
    const int64_t p = static_cast<int64_t>(lo) + 1 + static_cast<int64_t>(lt);
    float* bl = buf;              // left region's large values, ascending
    float* br = buf + (hi - lo) + 16;  // right region's small values, descending position
    // pass 2: right region [p+1, s1), top-down
    int64_t nr = 0;
    int64_t y = s1;  // exclusive top
    for (; y - 16 >= p + 1; y -= 16) {
        const __m512 v = _mm512_permutexvar_ps(rev, _mm512_loadu_ps(a + y - 16));
        const __mmask16 m = _mm512_cmp_ps_mask(v, vp, _CMP_LT_OQ);
        _mm512_storeu_ps(br + nr, _mm512_maskz_compress_ps(m, v));  // register compress: no
        nr += _mm_popcnt_u32(m);                                     // microcoded memory form
    }
    const int64_t rtail = y - (p + 1);  // positions [p+1, y)
    if (rtail > 0) {
        for (int64_t t = y - 1; t >= p + 1; --t) {
            br[nr] = a[t];
            nr += a[t] < pv;
        }
    }
    // pass 3: left region [s0, p] ascending — collect its large values, drop
    // the right region's small ones into their slots
    int64_t nl = 0, used = 0;
    x = s0;
    const int64_t lend = p + 1;
    for (; x + 16 <= lend; x += 16) {
        const __m512 v = _mm512_loadu_ps(a + x);
        const __mmask16 m = _mm512_cmp_ps_mask(v, vp, _CMP_GT_OQ);
        if (m) {
            _mm512_storeu_ps(bl + nl, _mm512_maskz_compress_ps(m, v));
            _mm512_storeu_ps(a + x, _mm512_mask_expand_ps(v, m, _mm512_loadu_ps(br + used)));
            const int c = _mm_popcnt_u32(m);
            nl += c;
            used += c;
        }
    }
    if (x < lend) {
        const __mmask16 k = static_cast<__mmask16>((1u << (lend - x)) - 1u);
        const __m512 v = _mm512_maskz_loadu_ps(k, a + x);
        const __mmask16 m = _mm512_mask_cmp_ps_mask(k, v, vp, _CMP_GT_OQ);
        if (m) {
            _mm512_storeu_ps(bl + nl, _mm512_maskz_compress_ps(m, v));
            _mm512_mask_storeu_ps(a + x, k, _mm512_mask_expand_ps(v, m, _mm512_loadu_ps(br + used)));
            const int c = _mm_popcnt_u32(m);
            nl += c;
            used += c;
        }
    }
    if (nl != nr) throw std::logic_error("hoare_rewrite: stopper counts differ");  // rank balance
    // pass 4: right region top-down, the k-th small slot from the top takes bl[k]
    used = 0;
    y = s1;
    for (; y - 16 >= p + 1; y -= 16) {
        const __m512 v = _mm512_permutexvar_ps(rev, _mm512_loadu_ps(a + y - 16));
        const __mmask16 m = _mm512_cmp_ps_mask(v, vp, _CMP_LT_OQ);
        if (m) {
            _mm512_storeu_ps(a + y - 16,
                             _mm512_permutexvar_ps(rev, _mm512_mask_expand_ps(v, m, _mm512_loadu_ps(bl + used))));
            used += _mm_popcnt_u32(m);
        }
    }
    for (int64_t t = y - 1; t >= p + 1; --t)
        if (a[t] < pv) a[t] = bl[used++];
    std::swap(a[lo + 1], a[p]);
    *p_out = static_cast<size_t>(p);
    return true;
}

bool have_avx2() {
    static const bool v = __builtin_cpu_supports("avx2") && __builtin_cpu_supports("popcnt");
    return v;
}

// ---- the closed form on several threads (segments of kParMin+ values) ----
// A small persistent pool: workers spin briefly, then sleep on a condition
// variable; run(n, f) executes f(0..n-1) across the workers and the caller.
class ParPool {
public:
    static ParPool& get() {
        static ParPool pool;
        return pool;
    }
    int threads() const { return static_cast<int>(workers_.size()) + 1; }
    template <typename F>
    void run(int n, F&& f) {
        if (workers_.empty() || n <= 1) {
            for (int i = 0; i < n; ++i) f(i);
            return;
        }
        std::lock_guard<std::mutex> one_caller(call_mu_);  // (builds on several threads share the pool)
        std::function<void(int)> job(std::forward<F>(f));
        {
            std::lock_guard<std::mutex> lk(mu_);
            job_ = &job;
            ntasks_ = n;
            done_.store(0, std::memory_order_relaxed);
            gen_.fetch_add(1, std::memory_order_release);
        }
        cv_.notify_all();
        work(0);
        while (done_.load(std::memory_order_acquire) < n) _mm_pause();
        std::lock_guard<std::mutex> lk(mu_);
        job_ = nullptr;
    }

private:
    ParPool() {
        const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
        const unsigned nw = std::min(7u, hw > 1 ? hw - 1 : 0u);  // (16 on the 16-core box: no faster, bandwidth-bound)
        for (unsigned w = 0; w < nw; ++w) workers_.emplace_back([this, w]() { loop(static_cast<int>(w) + 1); });
    }
    ~ParPool() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
            gen_.fetch_add(1);
        }
        cv_.notify_all();
        for (auto& t : workers_) t.join();
    }
    // static assignment: participant `me` (0 = the caller) runs tasks me,
    // me + P, ... (a chunk index stays on one core from pass to pass)
    void work(int me) {
        const int P = threads();
        for (int t = me; t < ntasks_; t += P) {
            (*job_)(t);
            done_.fetch_add(1, std::memory_order_acq_rel);
        }
    }
    void loop(int me) {
        uint64_t seen = 0;  // (a worker starting late still takes a job posted before it ran)
        for (;;) {
            for (int spin = 0; gen_.load(std::memory_order_acquire) == seen; ++spin) {
                if (spin < 200000) {  // (~5 ms: the next partition of the replay usually comes sooner)
                    _mm_pause();
                    continue;
                }
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&]() { return gen_.load() != seen; });
            }
            seen = gen_.load(std::memory_order_acquire);
            {
                std::lock_guard<std::mutex> lk(mu_);
                if (stop_) return;
                if (!job_) continue;
            }
            work(me);
        }
    }
    std::vector<std::thread> workers_;
    std::mutex mu_, call_mu_;
    std::condition_variable cv_;
    std::atomic<uint64_t> gen_{0};
    std::atomic<int> done_{0};
    int ntasks_ = 0;
    std::function<void(int)>* job_ = nullptr;
    bool stop_ = false;
};

// Chunk kernels of the closed form (AVX-512, masked tails).
__attribute__((target("avx512f,avx512vl,avx512bw,avx512dq,popcnt,bmi,bmi2")))
void par_count(const float* a, int64_t x0, int64_t x1, float pv, uint64_t* lt, uint64_t* eq, uint64_t* gt) {
    const __m512 vp = _mm512_set1_ps(pv);
    uint64_t l = 0, e = 0, g = 0;
    int64_t x = x0;
    for (; x + 16 <= x1; x += 16) {
        const __m512 v = _mm512_loadu_ps(a + x);
        l += _mm_popcnt_u32(_mm512_cmp_ps_mask(v, vp, _CMP_LT_OQ));
        e += _mm_popcnt_u32(_mm512_cmp_ps_mask(v, vp, _CMP_EQ_OQ));
        g += _mm_popcnt_u32(_mm512_cmp_ps_mask(v, vp, _CMP_GT_OQ));
    }
    for (; x < x1; ++x) {
        l += a[x] < pv;
        e += a[x] == pv;
        g += a[x] > pv;
    }
    *lt = l;
    *eq = e;
    *gt = g;
}

// values > pv of [x0, x1), ascending position, into out
__attribute__((target("avx512f,avx512vl,avx512bw,avx512dq,popcnt,bmi,bmi2")))
void par_collect_gt(const float* a, int64_t x0, int64_t x1, float pv, float* out) {
    const __m512 vp = _mm512_set1_ps(pv);
    int64_t n = 0, x = x0;
    for (; x + 16 <= x1; x += 16) {
        const __m512 v = _mm512_loadu_ps(a + x);
        const __mmask16 m = _mm512_cmp_ps_mask(v, vp, _CMP_GT_OQ);
        _mm512_mask_compressstoreu_ps(out + n, m, v);
        n += _mm_popcnt_u32(m);
    }
    for (; x < x1; ++x)
        if (a[x] > pv) out[n++] = a[x];
}

// values < pv of [x0, x1), descending position, into out
__attribute__((target("avx512f,avx512vl,avx512bw,avx512dq,popcnt,bmi,bmi2")))
void par_collect_lt_desc(const float* a, int64_t x0, int64_t x1, float pv, float* out) {
    const __m512 vp = _mm512_set1_ps(pv);
    const __m512i rev = _mm512_setr_epi32(15, 14, 13, 12, 11, 10, 9, 8, 7, 6, 5, 4, 3, 2, 1, 0);
    int64_t n = 0, y = x1;
    for (; y - 16 >= x0; y -= 16) {
        const __m512 v = _mm512_permutexvar_ps(rev, _mm512_loadu_ps(a + y - 16));
        const __mmask16 m = _mm512_cmp_ps_mask(v, vp, _CMP_LT_OQ);
        _mm512_mask_compressstoreu_ps(out + n, m, v);
        n += _mm_popcnt_u32(m);
    }
    for (int64_t t = y - 1; t >= x0; --t)
        if (a[t] < pv) out[n++] = a[t];
}

// the i-th position of [x0, x1) holding a value > pv (ascending) takes src[i]
__attribute__((target("avx512f,avx512vl,avx512bw,avx512dq,popcnt,bmi,bmi2")))
void par_fill_gt(float* a, int64_t x0, int64_t x1, float pv, const float* src) {
    const __m512 vp = _mm512_set1_ps(pv);
    int64_t u = 0, x = x0;
    for (; x + 16 <= x1; x += 16) {
        const __m512 v = _mm512_loadu_ps(a + x);
        const __mmask16 m = _mm512_cmp_ps_mask(v, vp, _CMP_GT_OQ);
        if (m) {
            _mm512_storeu_ps(a + x, _mm512_mask_expandloadu_ps(v, m, src + u));
            u += _mm_popcnt_u32(m);
        }
    }
    for (; x < x1; ++x)
        if (a[x] > pv) a[x] = src[u++];
}

// the i-th position of [x0, x1) holding a value < pv (descending) takes src[i]
__attribute__((target("avx512f,avx512vl,avx512bw,avx512dq,popcnt,bmi,bmi2")))
void par_fill_lt_desc(float* a, int64_t x0, int64_t x1, float pv, const float* src) {
    const __m512 vp = _mm512_set1_ps(pv);
    const __m512i rev = _mm512_setr_epi32(15, 14, 13, 12, 11, 10, 9, 8, 7, 6, 5, 4, 3, 2, 1, 0);
    int64_t u = 0, y = x1;
    for (; y - 16 >= x0; y -= 16) {
        const __m512 v = _mm512_permutexvar_ps(rev, _mm512_loadu_ps(a + y - 16));
        const __mmask16 m = _mm512_cmp_ps_mask(v, vp, _CMP_LT_OQ);
        if (m) {
            _mm512_storeu_ps(a + y - 16, _mm512_permutexvar_ps(rev, _mm512_mask_expandloadu_ps(v, m, src + u)));
            u += _mm_popcnt_u32(m);
        }
    }
    for (int64_t t = y - 1; t >= x0; --t)
        if (a[t] < pv) a[t] = src[u++];
}

size_t kParMin = size_t{1} << 18;  // segment length from which the closed form runs on the pool

// hoare_rewrite_avx512's closed form with every pass split over the pool:
// counts (p), per-chunk stopper counts and their prefix sums, the stoppers
// gathered into buf (left region's large values ascending, right region's
// small values descending), then written back crosswise.  Same result.
bool hoare_rewrite_par(float* a, size_t lo, size_t hi, float pv, float* buf, size_t* p_out) {
    if (!(a[lo] < pv) || !(a[hi - 1] > pv)) return false;
    ParPool& pool = ParPool::get();
    const int T = pool.threads();
    const int64_t s0 = static_cast<int64_t>(lo) + 2, s1 = static_cast<int64_t>(hi) - 1;  // scan region
    // one chunking of the scan region for every pass (chunk t stays on one core)
    std::vector<int64_t> cb(T + 1);
    for (int t = 0; t <= T; ++t) cb[t] = s0 + (s1 - s0) * t / T;
    std::vector<uint64_t> lt(T), eq(T), gt(T);
    pool.run(T, [&](int t) { par_count(a, cb[t], cb[t + 1], pv, &lt[t], &eq[t], &gt[t]); });
    uint64_t nlt = 0, neq = 0;
    for (int t = 0; t < T; ++t) {
        nlt += lt[t];
        neq += eq[t];
    }
    if (neq) return false;
    const int64_t p = static_cast<int64_t>(lo) + 1 + static_cast<int64_t>(nlt);
    // left region [s0, p], right region [p+1, s1): chunk t's part of each
    auto lpart = [&](int t, int64_t& x0, int64_t& x1) {
        x0 = cb[t];
        x1 = std::min(cb[t + 1], p + 1);
    };
    auto rpart = [&](int t, int64_t& x0, int64_t& x1) {
        x0 = std::max(cb[t], p + 1);
        x1 = cb[t + 1];
    };
    // stopper counts per chunk: large values in its left part, small in its
    // right part; only the chunk holding p needs a recount
    std::vector<uint64_t> cl(T), cr(T);
    int tb = -1;
    for (int t = 0; t < T; ++t) {
        if (cb[t + 1] <= p + 1) {
            cl[t] = gt[t];
            cr[t] = 0;
        } else if (cb[t] >= p + 1) {
            cl[t] = 0;
            cr[t] = lt[t];
        } else {
            tb = t;
        }
    }
    if (tb >= 0) {
        uint64_t a1, a2, a3, b1, b2, b3;
        par_count(a, cb[tb], p + 1, pv, &a1, &a2, &a3);
        par_count(a, p + 1, cb[tb + 1], pv, &b1, &b2, &b3);
        cl[tb] = a3;
        cr[tb] = b1;
    }
    std::vector<uint64_t> offl(T), offr(T);
    uint64_t m = 0, mr = 0;
    for (int t = 0; t < T; ++t) {
        offl[t] = m;
        m += cl[t];
    }
    for (int t = T - 1; t >= 0; --t) {  // the right region is taken top-down
        offr[t] = mr;
        mr += cr[t];
    }
    if (m != mr) throw std::logic_error("hoare_rewrite: stopper counts differ");  // rank balance
    float* bl = buf;                   // left region's large values, ascending
    float* br = buf + (hi - lo) + 16;  // right region's small values, descending position
    pool.run(T, [&](int t) {
        int64_t x0, x1;
        lpart(t, x0, x1);
        if (x0 < x1) par_collect_gt(a, x0, x1, pv, bl + offl[t]);
        rpart(t, x0, x1);
        if (x0 < x1) par_collect_lt_desc(a, x0, x1, pv, br + offr[t]);
    });
    pool.run(T, [&](int t) {
        int64_t x0, x1;
        lpart(t, x0, x1);
        if (x0 < x1) par_fill_gt(a, x0, x1, pv, br + offl[t]);
        rpart(t, x0, x1);
        if (x0 < x1) par_fill_lt_desc(a, x0, x1, pv, bl + offr[t]);
    });
    std::swap(a[lo + 1], a[p]);
    *p_out = static_cast<size_t>(p);
    return true;
}

size_t kRewriteMin = 64;  // >= 32 (buffer layout);  // segment length from which the closed-form rewrite pays (measured)

// Median-of-three around a seeded pick, sentinel Hoare scan; one bounded()
// draw per call.  Returns the pivot's sorted position.
size_t hoare_partition(float* a, size_t lo, size_t hi, Rng& rng, float* buf = nullptr) {
    const size_t len = hi - lo;
    const size_t mid = lo + len / 2;
    std::swap(a[mid], a[lo + rng.bounded(len)]);
    if (a[mid] < a[lo]) std::swap(a[lo], a[mid]);
    if (a[hi - 1] < a[lo]) std::swap(a[lo], a[hi - 1]);
    if (a[hi - 1] < a[mid]) std::swap(a[mid], a[hi - 1]);
    std::swap(a[mid], a[lo + 1]);
    const float pv = a[lo + 1];
    size_t pr;
    if (buf && len >= kParMin && have_avx512() && ParPool::get().threads() > 1 &&
        hoare_rewrite_par(a, lo, hi, pv, buf, &pr))
        return pr;
    if (buf && len >= kRewriteMin && have_avx512() && hoare_rewrite_avx512(a, lo, hi, pv, buf, &pr)) return pr;
    const size_t j = len < 12        ? hoare_scan_simple(a, lo, hi, pv)  // (measured crossover)
                     : have_avx512() ? hoare_scan_avx512(a, lo, hi, pv)
                     : have_avx2()   ? hoare_scan_avx2(a, lo, hi, pv)
                                     : hoare_scan_blocked(a, lo, hi, pv);
    std::swap(a[lo + 1], a[j]);
    return j;
}

void small_sort(float* a, size_t lo, size_t hi) {
    for (size_t i = lo + 1; i < hi; ++i) {
        const float v = a[i];
        size_t j = i;
        for (; j > lo && a[j - 1] > v; --j) a[j] = a[j - 1];
        a[j] = v;
    }
}

}  // namespace

void select_row_breakpoints(float* a, uint64_t n_s, int n_regions, Rng& rng, float* row_out,
                            uint64_t* draws) {
    const size_t span = n_s / static_cast<size_t>(n_regions);
    const size_t nt = static_cast<size_t>(n_regions) - 1;
    // target t sits at rank span*(t+1)-1; work items are (lo, hi, tlo, thi)
    struct Item {
        size_t lo, hi, tlo, thi;
    };
    std::vector<Item> stack;
    stack.reserve(256);
    stack.push_back({0, n_s, 0, nt});
    auto target = [span](size_t t) { return span * (t + 1) - 1; };
    // exact floor(x / span) for x, span < 2^32: x * ceil(2^64 / span) >> 64
    const unsigned __int128 recip = span > 1 ? (~static_cast<unsigned __int128>(0) >> 64) / span + 1 : 0;
    auto div_span = [span, recip](size_t x) -> size_t {
        if (span == 1) return x;
        if ((x | span) >> 32) return x / span;
        return static_cast<size_t>((static_cast<unsigned __int128>(x) * recip) >> 64);
    };
    thread_local std::vector<float> scratch;
    if (scratch.size() < 2 * n_s + 64) scratch.resize(2 * n_s + 64);
    float* buf = scratch.data();
    uint64_t nd = 0;
    while (!stack.empty()) {
        const Item it = stack.back();
        stack.pop_back();
        if (it.tlo >= it.thi) continue;
        if (it.hi - it.lo <= 8) {
            small_sort(a, it.lo, it.hi);
            continue;
        }
        const size_t p = hoare_partition(a, it.lo, it.hi, rng, buf);
        ++nd;
        // targets are an arithmetic progression: #{t : span(t+1)-1 < p} =
        // floor(p / span), #{t : span(t+1)-1 <= p} = floor((p+1) / span),
        // clamped to the item's target range (lower_bound / upper_bound)
        const size_t below = std::min(std::max(div_span(p), it.tlo), it.thi);
        const size_t above = std::min(std::max(div_span(p + 1), it.tlo), it.thi);
        stack.push_back({it.lo, p, it.tlo, below});
        stack.push_back({p + 1, it.hi, above, it.thi});
    }
    for (size_t t = 0; t < nt; ++t) row_out[t + 1] = a[target(t)];
    row_out[0] = *std::min_element(a, a + target(0) + 1);
    row_out[n_regions] = *std::max_element(a + target(nt - 1), a + n_s);
    if (draws) *draws += nd;
}

namespace {
// Runs f(begin, end) over [0, n) on up to 8 threads (one when n is small).
template <typename F>
void parallel_ranges(uint64_t n, uint64_t min_per_thread, F&& f) {
    const uint64_t want = std::min<uint64_t>(8, std::max<uint64_t>(1, n / min_per_thread));
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const uint64_t nt = std::min<uint64_t>(want, hw);
    if (nt <= 1) {
        f(uint64_t{0}, n);
        return;
    }
    std::vector<std::thread> th;
    for (uint64_t w = 0; w < nt; ++w)
        th.emplace_back([&, w]() { f(n * w / nt, n * (w + 1) / nt); });
    for (auto& t : th) t.join();
}
}  // namespace

RefSampler::RefSampler(uint64_t n, uint64_t n_s, int n_regions, uint64_t seed)
    : n_(n), n_s_(n_s), n_regions_(n_regions), rng_(seed), idx_(new uint32_t[n]), sample_idx_(n_s) {
    uint32_t* idx = idx_.get();
    parallel_ranges(n, uint64_t{1} << 22, [idx](uint64_t a, uint64_t b) {
        for (uint64_t t = a; t < b; ++t) idx[t] = static_cast<uint32_t>(t);
    });
}

const std::vector<uint32_t>& RefSampler::next_space_indices() {
    // Partial Fisher-Yates (encoder.cpp:133-134).  The swap targets depend only
    // on the RNG stream, so they are drawn first (same draws, same order) and
    // the random-access swaps then run with the targets prefetched ahead.
    // bounded() takes one raw draw unless r < bound and r < 2^64 mod bound
    // (probability < n / 2^64): the raw draws are taken in order, the 64-bit
    // remainders (the costly part) computed on several threads, and in the
    // rejection case the space is redrawn exactly from the saved state.
    constexpr uint64_t kAhead = 16;
    std::vector<uint32_t>& tgt = targets_;
    tgt.resize(n_s_);
    if (n_s_ >= (uint64_t{1} << 20)) {  // (below: thread start-up outweighs the remainders)
        const Rng saved = rng_;
        raw_.resize(n_s_);
        for (uint64_t t = 0; t < n_s_; ++t) raw_[t] = rng_.next_u64();
        std::atomic<bool> rejected{false};
        const uint64_t n = n_;
        const uint64_t* raw = raw_.data();
        uint32_t* tg = tgt.data();
        parallel_ranges(n_s_, uint64_t{1} << 15, [&rejected, n, raw, tg](uint64_t a, uint64_t b) {
            bool rej = false;
            for (uint64_t t = a; t < b; ++t) {
                const uint64_t bound = n - t, r = raw[t];
                if (r < bound && r < (0 - bound) % bound) rej = true;
                tg[t] = static_cast<uint32_t>(t + r % bound);
            }
            if (rej) rejected = true;
        });
        if (rejected) {
            rng_ = saved;
            for (uint64_t t = 0; t < n_s_; ++t) tgt[t] = static_cast<uint32_t>(t + rng_.bounded(n_ - t));
        }
    } else {
        for (uint64_t t = 0; t < n_s_; ++t) tgt[t] = static_cast<uint32_t>(t + rng_.bounded(n_ - t));
    }
    uint32_t* idx = idx_.get();
    for (uint64_t t = 0; t < n_s_; ++t) {
        if (t + kAhead < n_s_) __builtin_prefetch(idx + tgt[t + kAhead], 1);
        std::swap(idx[t], idx[tgt[t]]);
    }
    std::copy(idx, idx + n_s_, sample_idx_.begin());
    return sample_idx_;
}

void RefSampler::select_row(float* sample, float* row_out) {
    select_row_breakpoints(sample, n_s_, n_regions_, rng_, row_out, &draws_);
}

double rmin_from_order_stats(const std::vector<double>& T, double guess, double epsilon,
                             double c) {
    std::vector<double> results;
    results.reserve(T.size());
    double start = guess;
    for (const double tp : T) {
        const auto reaches = [&](double r) { return tp <= epsilon * r; };
        double r = start;
        if (reaches(r)) {
            for (int i = 0; i < 200 && r / c > 0.0 && reaches(r / c); ++i) r /= c;
        } else {
            for (int i = 0; i < 200; ++i) {
                r *= c;
                if (reaches(r)) break;
            }
        }
        results.push_back(r);
        start = r;
    }
    std::sort(results.begin(), results.end());
    return results[(results.size() - 1) / 2];
}

}  // namespace detlsh_b200
