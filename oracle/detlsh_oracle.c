/* TEST INFRASTRUCTURE ONLY — see detlsh_oracle.h.
 *
 * Plain-C restatement of the DET-LSH reference (/root/reference/proj).  It is
 * deliberately written in a different language and shape from the reference
 * (flat arrays, explicit heaps, no std::function), but reproduces its
 * arithmetic operation for operation so results are bit-identical.
 */
#define _GNU_SOURCE
#include "detlsh_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------------------
 * RNG: std::mt19937_64 + the explicit transforms of rng.hpp:13-61.
 * ------------------------------------------------------------------------- */
#define MT_N 312
#define MT_M 156

void orc_rng_seed(orc_rng* r, uint64_t seed) {
    r->mt[0] = seed;
    for (int i = 1; i < MT_N; ++i)
        r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    r->mti = MT_N;
    r->spare = 0.0;
    r->have_spare = 0;
}

static void mt_twist(orc_rng* r) {
    const uint64_t upper = 0xFFFFFFFF80000000ULL, lower = 0x7FFFFFFFULL;
    for (int i = 0; i < MT_N; ++i) {
        uint64_t x = (r->mt[i] & upper) | (r->mt[(i + 1) % MT_N] & lower);
        uint64_t xa = x >> 1;
        if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
        r->mt[i] = r->mt[(i + MT_M) % MT_N] ^ xa;
    }
    r->mti = 0;
}

uint64_t orc_rng_next(orc_rng* r) {
    if (r->mti >= MT_N) mt_twist(r);
    uint64_t y = r->mt[r->mti++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= (y >> 43);
    return y;
}

/* rng.hpp:20-26 — rejection sampling against (2^64 - bound) mod bound. */
uint64_t orc_rng_bounded(orc_rng* r, uint64_t bound) {
    const uint64_t threshold = (0 - bound) % bound;
    for (;;) {
        uint64_t v = orc_rng_next(r);
        if (v >= threshold) return v % bound;
    }
}

/* rng.hpp:29 */
static double rng_real01(orc_rng* r) { return (double)(orc_rng_next(r) >> 11) * 0x1.0p-53; }

/* rng.hpp:32-47 — Box-Muller, cos value first, sin value cached. */
double orc_rng_normal(orc_rng* r) {
    if (r->have_spare) {
        r->have_spare = 0;
        return r->spare;
    }
    double u1;
    do {
        u1 = rng_real01(r);
    } while (u1 <= 0.0);
    const double u2 = rng_real01(r);
    const double mag = sqrt(-2.0 * log(u1));
    const double ang = 2.0 * 3.141592653589793 * u2;
    r->spare = mag * sin(ang);
    r->have_spare = 1;
    return mag * cos(ang);
}

/* rng.hpp:56-61 — splitmix64 sub-stream derivation. */
uint64_t orc_mix_seed(uint64_t seed, uint64_t stream) {
    uint64_t z = seed + 0x9e3779b97f4a7c15ULL * (stream + 1);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

void orc_rng_stream(uint64_t seed, uint64_t count, uint64_t* out_u64, double* out_normal) {
    orc_rng* a = malloc(sizeof(orc_rng));
    orc_rng* b = malloc(sizeof(orc_rng));
    orc_rng_seed(a, seed);
    orc_rng_seed(b, seed);
    for (uint64_t i = 0; i < count; ++i) {
        if (out_u64) out_u64[i] = orc_rng_next(a);
        if (out_normal) out_normal[i] = orc_rng_normal(b);
    }
    free(a);
    free(b);
}

/* ---------------------------------------------------------------------------
 * chi^2 numerics (chi2.cpp:12-107).
 * ------------------------------------------------------------------------- */
static double gamma_series(double a, double x) { /* chi2.cpp:12-22 */
    double ap = a, sum = 1.0 / a, del = sum;
    for (int i = 0; i < 1000; ++i) {
        ap += 1.0;
        del *= x / ap;
        sum += del;
        if (fabs(del) < fabs(sum) * 1e-16) break;
    }
    return sum * exp(-x + a * log(x) - lgamma(a));
}

static double gamma_cf(double a, double x) { /* chi2.cpp:25-44, modified Lentz */
    const double tiny = 1e-300;
    double b = x + 1.0 - a, c = 1.0 / tiny, d = 1.0 / b, h = d;
    for (int i = 1; i <= 1000; ++i) {
        const double an = -(double)i * ((double)i - a);
        b += 2.0;
        d = an * d + b;
        if (fabs(d) < tiny) d = tiny;
        c = b + an / c;
        if (fabs(c) < tiny) c = tiny;
        d = 1.0 / d;
        const double del = d * c;
        h *= del;
        if (fabs(del - 1.0) < 1e-16) break;
    }
    return exp(-x + a * log(x) - lgamma(a)) * h;
}

double orc_regularized_gamma_p(double a, double x) { /* chi2.cpp:49-55 */
    if (x == 0.0) return 0.0;
    if (x < a + 1.0) return gamma_series(a, x);
    return 1.0 - gamma_cf(a, x);
}

double orc_chi2_cdf(double x, int k) { /* chi2.cpp:57-61 */
    if (x <= 0.0) return 0.0;
    return orc_regularized_gamma_p(0.5 * k, 0.5 * x);
}

double orc_chi2_pdf(double x, int k) { /* chi2.cpp:63-69 */
    if (x <= 0.0) return 0.0;
    const double hk = 0.5 * k;
    return exp((hk - 1.0) * log(x) - 0.5 * x - hk * 0.6931471805599453 - lgamma(hk));
}

double orc_chi2_quantile(double alpha, int k) { /* chi2.cpp:71-107 */
    if (alpha == 1.0) return 0.0;
    const double target = 1.0 - alpha;
    double lo = 0.0;
    double hi = (double)k + 10.0 * sqrt(2.0 * k) + 10.0;
    for (int i = 0; i < 200 && orc_chi2_cdf(hi, k) < target; ++i) hi *= 2.0;
    for (int i = 0; i < 200; ++i) {
        const double mid = 0.5 * (lo + hi);
        if (mid == lo || mid == hi) break;
        if (orc_chi2_cdf(mid, k) < target)
            lo = mid;
        else
            hi = mid;
    }
    double x = 0.5 * (lo + hi);
    for (int i = 0; i < 32; ++i) {
        const double f = orc_chi2_cdf(x, k) - target;
        if (fabs(f) < 1e-12) break;
        const double df = orc_chi2_pdf(x, k);
        if (df <= 0.0) break;
        const double next = x - f / df;
        if (next <= lo || next >= hi) break;
        x = next;
    }
    return x;
}

int orc_derive_params(int K, double c, int L, double* out4) { /* projection.cpp:92-102 */
    if (K < 1 || L < 1 || !(c > 1.0)) return 1;
    const double a1 = exp(-1.0 / (double)L);
    const double eps_sq = orc_chi2_quantile(a1, K);
    const double eps = sqrt(eps_sq);
    const double a2 = 1.0 - orc_chi2_cdf(eps_sq / (c * c), K);
    out4[0] = a1;
    out4[1] = a2;
    out4[2] = eps;
    out4[3] = 2.0 * (1.0 - pow(a2, (double)L));
    return 0;
}

uint64_t orc_candidate_budget(double beta, uint64_t n, int k) { /* index.cpp:190-194 */
    const double raw = (beta > 0.0 ? beta : 0.0) * (double)n + (double)k;
    const uint64_t b = (uint64_t)ceil(raw);
    return b < n ? b : n;
}

/* ---------------------------------------------------------------------------
 * Projection (projection.cpp:11-60).
 * ------------------------------------------------------------------------- */
void orc_sample_hash_family(int d, int K, int L, uint64_t seed, float* out) {
    orc_rng* r = malloc(sizeof(orc_rng));
    orc_rng_seed(r, seed);
    const size_t total = (size_t)L * K * d;
    for (size_t i = 0; i < total; ++i) out[i] = (float)orc_rng_normal(r);
    free(r);
}

/* projection.cpp:25-38: float x float widened to double (exact), summed
 * sequentially in t, rounded once to float. */
static void project_row(const float* coeffs, int K, int d, int space, const float* x, float* out) {
    for (int j = 0; j < K; ++j) {
        const float* a = coeffs + ((size_t)space * K + j) * d;
        double dot = 0.0;
        for (int t = 0; t < d; ++t) {
            const double p = (double)a[t] * (double)x[t];
            dot = dot + p;
        }
        out[j] = (float)dot;
    }
}

void orc_project_dataset(const float* coeffs, int K, int L, const float* data, uint64_t n, int d,
                         float* out) {
    for (int i = 0; i < L; ++i)
        for (uint64_t z = 0; z < n; ++z)
            project_row(coeffs, K, d, i, data + z * (size_t)d, out + ((size_t)i * n + z) * K);
}

/* ---------------------------------------------------------------------------
 * Breakpoints (encoder.cpp:14-143).
 * ------------------------------------------------------------------------- */
static void fswap(float* a, size_t i, size_t j) {
    float t = a[i];
    a[i] = a[j];
    a[j] = t;
}

static void isort(float* a, size_t lo, size_t hi) { /* encoder.cpp:14-24 */
    for (size_t i = lo + 1; i < hi; ++i) {
        const float v = a[i];
        size_t j = i;
        while (j > lo && a[j - 1] > v) {
            a[j] = a[j - 1];
            --j;
        }
        a[j] = v;
    }
}

/* encoder.cpp:29-53: one bounded() draw, median-of-three, sentinel Hoare scan. */
static size_t hoare(float* a, size_t lo, size_t hi, orc_rng* rng) {
    const size_t len = hi - lo, mid = lo + len / 2;
    fswap(a, mid, lo + orc_rng_bounded(rng, len));
    if (a[mid] < a[lo]) fswap(a, lo, mid);
    if (a[hi - 1] < a[lo]) fswap(a, lo, hi - 1);
    if (a[hi - 1] < a[mid]) fswap(a, mid, hi - 1);
    fswap(a, mid, lo + 1);
    const float pivot = a[lo + 1];
    size_t i = lo + 1, j = hi - 1;
    for (;;) {
        do ++i; while (a[i] < pivot);
        do --j; while (a[j] > pivot);
        if (i >= j) break;
        fswap(a, i, j);
    }
    fswap(a, lo + 1, j);
    return j;
}

/* first index in [lo,hi) of targets with targets[idx] >= p / > p */
static size_t lbound(const size_t* t, size_t lo, size_t hi, size_t p) {
    while (lo < hi) {
        size_t m = lo + (hi - lo) / 2;
        if (t[m] < p) lo = m + 1; else hi = m;
    }
    return lo;
}
static size_t ubound(const size_t* t, size_t lo, size_t hi, size_t p) {
    while (lo < hi) {
        size_t m = lo + (hi - lo) / 2;
        if (t[m] <= p) lo = m + 1; else hi = m;
    }
    return lo;
}

static uint64_t g_draw_counter; /* draws consumed by the last row (diagnostic) */

/* encoder.cpp:57-103: LIFO work list of (data range, target range) items. */
int orc_select_row_breakpoints(float* a, uint64_t n_s, int n_regions, orc_rng* rng,
                               float* out_row) {
    if (n_regions < 2 || (n_regions & (n_regions - 1))) return 1;
    if (n_s < (uint64_t)n_regions) return 1;
    const size_t region = n_s / (size_t)n_regions, nt = (size_t)n_regions - 1;
    size_t* targets = malloc(nt * sizeof(size_t));
    for (size_t t = 0; t < nt; ++t) targets[t] = region * (t + 1) - 1;
    size_t cap = 64, top = 0;
    size_t(*stack)[4] = malloc(cap * sizeof *stack);
    stack[top][0] = 0;
    stack[top][1] = n_s;
    stack[top][2] = 0;
    stack[top][3] = nt;
    ++top;
    g_draw_counter = 0;
    while (top) {
        --top;
        const size_t lo = stack[top][0], hi = stack[top][1], tlo = stack[top][2],
                     thi = stack[top][3];
        if (tlo >= thi) continue;
        if (hi - lo <= 8) {
            isort(a, lo, hi);
            continue;
        }
        const size_t p = hoare(a, lo, hi, rng);
        ++g_draw_counter;
        const size_t below = lbound(targets, tlo, thi, p);
        const size_t above = ubound(targets, tlo, thi, p);
        if (top + 2 > cap) {
            cap *= 2;
            stack = realloc(stack, cap * sizeof *stack);
        }
        stack[top][0] = lo; stack[top][1] = p; stack[top][2] = tlo; stack[top][3] = below;
        ++top;
        stack[top][0] = p + 1; stack[top][1] = hi; stack[top][2] = above; stack[top][3] = thi;
        ++top;
    }
    for (size_t t = 0; t < nt; ++t) out_row[t + 1] = a[targets[t]];
    float mn = a[0];
    for (size_t i = 1; i <= targets[0]; ++i)
        if (a[i] < mn) mn = a[i];
    float mx = a[targets[nt - 1]];
    for (size_t i = targets[nt - 1] + 1; i < n_s; ++i)
        if (mx < a[i]) mx = a[i];
    out_row[0] = mn;
    out_row[n_regions] = mx;
    free(targets);
    free(stack);
    return 0;
}

/* encoder.cpp:105-143: ONE rng for the per-space partial Fisher-Yates AND for
 * every quickselect pivot; idx persists across spaces. */
int orc_select_breakpoints(const float* proj, uint64_t n, int K, int L, int n_regions,
                           double sample_fraction, uint64_t seed, float* out_table,
                           uint64_t* sample_size, uint64_t* sample_idx, uint64_t* draws) {
    if (n_regions < 2 || n_regions > 256 || (n_regions & (n_regions - 1))) return 1;
    if (!(sample_fraction > 0.0) || sample_fraction > 1.0) return 1;
    uint64_t n_s = (uint64_t)ceil(sample_fraction * (double)n);
    if (n_s < (uint64_t)n_regions) n_s = (uint64_t)n_regions;
    if (n_s > n) return 1;
    if (sample_size) *sample_size = n_s;
    orc_rng* rng = malloc(sizeof(orc_rng));
    orc_rng_seed(rng, seed);
    uint64_t* idx = malloc(n * sizeof(uint64_t));
    for (uint64_t i = 0; i < n; ++i) idx[i] = i;
    float* sample = malloc(n_s * sizeof(float));
    const size_t w = (size_t)n_regions + 1;
    for (int i = 0; i < L; ++i) {
        for (uint64_t t = 0; t < n_s; ++t) {
            const uint64_t s = t + orc_rng_bounded(rng, n - t);
            uint64_t tmp = idx[t];
            idx[t] = idx[s];
            idx[s] = tmp;
        }
        if (sample_idx) memcpy(sample_idx + (size_t)i * n_s, idx, n_s * sizeof(uint64_t));
        for (int j = 0; j < K; ++j) {
            for (uint64_t t = 0; t < n_s; ++t) sample[t] = proj[((size_t)i * n + idx[t]) * K + j];
            orc_select_row_breakpoints(sample, n_s, n_regions, rng,
                                       out_table + ((size_t)i * K + j) * w);
            if (draws) draws[i * K + j] = g_draw_counter;
        }
    }
    free(rng);
    free(idx);
    free(sample);
    return 0;
}

/* encoder.cpp:145-153: lower_bound over n_regions+1 boundaries, clamp. */
int orc_locate_region(float v, const float* row, int n_regions) {
    size_t lo = 0, hi = (size_t)n_regions + 1;
    while (lo < hi) {
        size_t m = lo + (hi - lo) / 2;
        if (row[m] < v) lo = m + 1; else hi = m;
    }
    int region = (int)lo - 1;
    if (region < 0) return 0;
    if (region > n_regions - 1) return n_regions - 1;
    return region;
}

void orc_encode_dataset(const float* proj, uint64_t n, int K, int L, const float* table,
                        int n_regions, uint8_t* out) { /* encoder.cpp:155-176 */
    const size_t w = (size_t)n_regions + 1;
    for (int i = 0; i < L; ++i)
        for (uint64_t z = 0; z < n; ++z)
            for (int j = 0; j < K; ++j) {
                const size_t o = ((size_t)i * n + z) * K + j;
                out[o] = (uint8_t)orc_locate_region(proj[o], table + ((size_t)i * K + j) * w,
                                                    n_regions);
            }
}

/* ---------------------------------------------------------------------------
 * DE-Tree (de_tree.cpp).  Leaves hold positions; symbols are read from the
 * encoded dataset (the reference copies them into the leaf; same values).
 * ------------------------------------------------------------------------- */
typedef struct {
    uint8_t is_leaf, split_dim;
    int32_t left, right;
    uint32_t* pos;
    uint32_t count, cap;
} onode;

struct orc_tree {
    int space, K, n_regions, sbits, max_size;
    int32_t* root;   /* 2^K */
    onode* nodes;
    uint8_t* bits;   /* [node][K] */
    uint8_t* value;  /* [node][K] */
    size_t nn, ncap;
    const uint8_t* codes; /* [n][K] of this space (borrowed during build) */
};

static int next_bit(uint8_t sym, int used, int sbits) { return (sym >> (sbits - 1 - used)) & 1; }

static int32_t new_node(orc_tree* t) {
    if (t->nn == t->ncap) {
        t->ncap = t->ncap ? t->ncap * 2 : 64;
        t->nodes = realloc(t->nodes, t->ncap * sizeof(onode));
        t->bits = realloc(t->bits, t->ncap * (size_t)t->K);
        t->value = realloc(t->value, t->ncap * (size_t)t->K);
    }
    onode* nd = &t->nodes[t->nn];
    memset(nd, 0, sizeof *nd);
    nd->is_leaf = 1;
    nd->left = nd->right = -1;
    return (int32_t)t->nn++;
}

static void push_pos(onode* nd, uint32_t p) {
    if (nd->count == nd->cap) {
        nd->cap = nd->cap ? nd->cap * 2 : 8;
        nd->pos = realloc(nd->pos, nd->cap * sizeof(uint32_t));
    }
    nd->pos[nd->count++] = p;
}

/* de_tree.cpp:77-131: most balanced next bit among unsaturated dims, ties to
 * the lowest dim; children appended left (bit 0) then right (bit 1). */
static int split(orc_tree* t, int32_t ni) {
    const int K = t->K;
    const uint8_t* b = t->bits + (size_t)ni * K;
    int best = -1;
    uint32_t best_imb = 0;
    for (int dim = 0; dim < K; ++dim) {
        if (b[dim] >= t->sbits) continue;
        uint32_t ones = 0;
        for (uint32_t e = 0; e < t->nodes[ni].count; ++e)
            ones += (uint32_t)next_bit(t->codes[(size_t)t->nodes[ni].pos[e] * K + dim], b[dim],
                                       t->sbits);
        const uint32_t zeros = t->nodes[ni].count - ones;
        const uint32_t imb = zeros > ones ? zeros - ones : ones - zeros;
        if (best < 0 || imb < best_imb) {
            best = dim;
            best_imb = imb;
        }
    }
    if (best < 0) return 0;
    const int32_t l = new_node(t);
    const int32_t r = new_node(t);
    memcpy(t->bits + (size_t)l * K, t->bits + (size_t)ni * K, K);
    memcpy(t->bits + (size_t)r * K, t->bits + (size_t)ni * K, K);
    memcpy(t->value + (size_t)l * K, t->value + (size_t)ni * K, K);
    memcpy(t->value + (size_t)r * K, t->value + (size_t)ni * K, K);
    const int used = t->bits[(size_t)ni * K + best];
    t->bits[(size_t)l * K + best] += 1;
    t->bits[(size_t)r * K + best] += 1;
    t->value[(size_t)l * K + best] = (uint8_t)(t->value[(size_t)l * K + best] << 1);
    t->value[(size_t)r * K + best] = (uint8_t)((t->value[(size_t)r * K + best] << 1) | 1);
    onode* p = &t->nodes[ni];
    for (uint32_t e = 0; e < p->count; ++e) {
        const uint32_t pos = p->pos[e];
        const int bit = next_bit(t->codes[(size_t)pos * K + best], used, t->sbits);
        push_pos(&t->nodes[bit ? r : l], pos);
    }
    p = &t->nodes[ni];
    free(p->pos);
    p->pos = NULL;
    p->count = p->cap = 0;
    p->is_leaf = 0;
    p->split_dim = (uint8_t)best;
    p->left = l;
    p->right = r;
    return 1;
}

/* de_tree.cpp:40-75: root slot from top bits; descend; split-before-insert. */
static void tree_insert(orc_tree* t, uint32_t pos) {
    const int K = t->K;
    const uint8_t* sym = t->codes + (size_t)pos * K;
    uint32_t slot = 0;
    for (int j = 0; j < K; ++j) slot |= (uint32_t)next_bit(sym[j], 0, t->sbits) << j;
    if (t->root[slot] < 0) {
        const int32_t nd = new_node(t);
        for (int j = 0; j < K; ++j) {
            t->bits[(size_t)nd * K + j] = 1;
            t->value[(size_t)nd * K + j] = (uint8_t)((slot >> j) & 1);
        }
        t->root[slot] = nd;
    }
    int32_t cur = t->root[slot];
    for (;;) {
        while (!t->nodes[cur].is_leaf) {
            const onode* nd = &t->nodes[cur];
            const int dim = nd->split_dim;
            const int bit = next_bit(sym[dim], t->bits[(size_t)cur * K + dim], t->sbits);
            cur = bit ? nd->right : nd->left;
        }
        if (t->nodes[cur].count < (uint32_t)t->max_size) break;
        if (!split(t, cur)) break;
    }
    push_pos(&t->nodes[cur], pos);
}

orc_tree* orc_build_tree(const uint8_t* codes, uint64_t n, int K, int L, int n_regions, int space,
                         int max_size) { /* de_tree.cpp:133-152 */
    if (max_size < 1 || K < 1 || K > 24 || space < 0 || space >= L) return NULL;
    orc_tree* t = calloc(1, sizeof(orc_tree));
    t->space = space;
    t->K = K;
    t->n_regions = n_regions;
    int sb = 0;
    while ((1 << sb) < n_regions) ++sb;
    t->sbits = sb;
    t->max_size = max_size;
    t->root = malloc(((size_t)1 << K) * sizeof(int32_t));
    for (size_t s = 0; s < ((size_t)1 << K); ++s) t->root[s] = -1;
    t->codes = codes + (size_t)space * n * K;
    for (uint64_t z = 0; z < n; ++z) tree_insert(t, (uint32_t)z);
    t->codes = NULL;
    return t;
}

void orc_tree_free(orc_tree* t) {
    if (!t) return;
    for (size_t i = 0; i < t->nn; ++i) free(t->nodes[i].pos);
    free(t->nodes);
    free(t->bits);
    free(t->value);
    free(t->root);
    free(t);
}

uint64_t orc_tree_num_nodes(const orc_tree* t) { return t->nn; }

void orc_tree_export(const orc_tree* t, int32_t* root_children, uint8_t* is_leaf,
                     uint8_t* split_dim, int32_t* left, int32_t* right, uint8_t* bits,
                     uint8_t* value, uint64_t* ebegin, uint32_t* ecount, uint32_t* positions) {
    if (root_children) memcpy(root_children, t->root, ((size_t)1 << t->K) * sizeof(int32_t));
    uint64_t off = 0;
    for (size_t i = 0; i < t->nn; ++i) {
        const onode* nd = &t->nodes[i];
        if (is_leaf) is_leaf[i] = nd->is_leaf;
        if (split_dim) split_dim[i] = nd->split_dim;
        if (left) left[i] = nd->left;
        if (right) right[i] = nd->right;
        if (bits) memcpy(bits + i * t->K, t->bits + i * t->K, t->K);
        if (value) memcpy(value + i * t->K, t->value + i * t->K, t->K);
        if (ebegin) ebegin[i] = off;
        if (ecount) ecount[i] = nd->count;
        if (positions && nd->count) memcpy(positions + off, nd->pos, nd->count * sizeof(uint32_t));
        off += nd->count;
    }
}

/* de_tree.cpp:154-167 — box edge along dim; +-inf when touching region 0 /
 * region n_regions-1. Returns lo/hi via pointers, flags for infinities. */
static void node_iv(const orc_tree* t, int ni, int dim, const float* table, double* lo,
                    double* hi) {
    const int bits = t->bits[(size_t)ni * t->K + dim];
    *lo = -INFINITY;
    *hi = INFINITY;
    if (bits == 0) return;
    const int value = t->value[(size_t)ni * t->K + dim];
    const int width = t->sbits - bits;
    const int lo_r = value << width;
    const int hi_r = ((value + 1) << width) - 1;
    const float* row = table + ((size_t)t->space * t->K + dim) * ((size_t)t->n_regions + 1);
    if (lo_r > 0) *lo = row[lo_r];
    if (hi_r < t->n_regions - 1) *hi = row[hi_r + 1];
}

/* de_tree.cpp:169-184 */
double orc_mindist(const orc_tree* t, int ni, const float* table, const float* q) {
    double acc = 0.0;
    for (int dim = 0; dim < t->K; ++dim) {
        double lo, hi;
        node_iv(t, ni, dim, table, &lo, &hi);
        const double v = q[dim];
        double pen = 0.0;
        if (v < lo)
            pen = lo - v;
        else if (v > hi)
            pen = v - hi;
        const double sq = pen * pen;
        acc = acc + sq;
    }
    return sqrt(acc);
}

/* de_tree.cpp:186-197 */
static double maxdist(const orc_tree* t, int ni, const float* table, const float* q) {
    double acc = 0.0;
    for (int dim = 0; dim < t->K; ++dim) {
        double lo, hi;
        node_iv(t, ni, dim, table, &lo, &hi);
        if (!isfinite(lo) || !isfinite(hi)) return INFINITY;
        const double v = q[dim];
        const double a = fabs(v - lo), b = fabs(v - hi);
        const double far = a > b ? a : b;
        const double sq = far * far;
        acc = acc + sq;
    }
    return sqrt(acc);
}

/* l2 over K projected floats, sequential double (dataset.hpp:23-34) */
static double l2f(const float* a, const float* b, int K) {
    double acc = 0.0;
    for (int t = 0; t < K; ++t) {
        const double diff = (double)a[t] - (double)b[t];
        const double sq = diff * diff;
        acc = acc + sq;
    }
    return sqrt(acc);
}

/* Min-heap over (mindist, node) pairs, lexicographic like std::pair. */
typedef struct {
    double key;
    int32_t node;
} hitem;

static int hless(hitem a, hitem b) { return a.key < b.key || (a.key == b.key && a.node < b.node); }

typedef struct {
    hitem* v;
    size_t n, cap;
} heap;

static void hpush(heap* h, hitem x) {
    if (h->n == h->cap) {
        h->cap = h->cap ? 2 * h->cap : 64;
        h->v = realloc(h->v, h->cap * sizeof(hitem));
    }
    size_t i = h->n++;
    h->v[i] = x;
    while (i > 0) {
        size_t p = (i - 1) / 2;
        if (!hless(h->v[i], h->v[p])) break;
        hitem tmp = h->v[i];
        h->v[i] = h->v[p];
        h->v[p] = tmp;
        i = p;
    }
}

static hitem hpop(heap* h) {
    hitem top = h->v[0];
    h->v[0] = h->v[--h->n];
    size_t i = 0;
    for (;;) {
        size_t l = 2 * i + 1, r = l + 1, m = i;
        if (l < h->n && hless(h->v[l], h->v[m])) m = l;
        if (r < h->n && hless(h->v[r], h->v[m])) m = r;
        if (m == i) break;
        hitem tmp = h->v[i];
        h->v[i] = h->v[m];
        h->v[m] = tmp;
        i = m;
    }
    return top;
}

typedef int (*sink_fn)(void* ctx, uint32_t pos); /* returns 0 to stop */

/* de_tree.cpp:229-258: DFS collects leaves with mindist <= radius into a
 * min-heap, then drains whole leaves in (mindist, node) order. */
static void range_opt(const orc_tree* t, const float* table, const float* q, double radius,
                      sink_fn sink, void* ctx) {
    heap h = {0};
    int32_t* stack = malloc(64 * sizeof(int32_t));
    size_t sn = 0, scap = 64;
    const size_t slots = (size_t)1 << t->K;
    for (size_t s = 0; s < slots; ++s)
        if (t->root[s] >= 0) {
            if (sn == scap) stack = realloc(stack, (scap *= 2) * sizeof(int32_t));
            stack[sn++] = t->root[s];
        }
    while (sn) {
        const int32_t ni = stack[--sn];
        const double lower = orc_mindist(t, ni, table, q);
        if (lower > radius) continue;
        if (t->nodes[ni].is_leaf) {
            hitem it = {lower, ni};
            hpush(&h, it);
        } else {
            if (sn + 2 > scap) stack = realloc(stack, (scap *= 2) * sizeof(int32_t));
            stack[sn++] = t->nodes[ni].left;
            stack[sn++] = t->nodes[ni].right;
        }
    }
    free(stack);
    int go = 1;
    while (go && h.n) {
        const hitem it = hpop(&h);
        const onode* nd = &t->nodes[it.node];
        for (uint32_t e = 0; e < nd->count; ++e)
            if (!sink(ctx, nd->pos[e])) {
                go = 0;
                break;
            }
    }
    free(h.v);
}

typedef struct {
    uint32_t* out;
    uint64_t count, limit;
} collect_ctx;

static int collect_sink(void* c, uint32_t pos) {
    collect_ctx* x = c;
    x->out[x->count++] = pos;
    return x->count < x->limit;
}

uint64_t orc_range_query_optimized(const orc_tree* t, const float* table, const float* q_proj,
                                   double radius, uint64_t limit, uint32_t* out) {
    collect_ctx c = {out, 0, limit};
    range_opt(t, table, q_proj, radius, collect_sink, &c);
    return c.count;
}

/* ---------------------------------------------------------------------------
 * Index assembly and queries (index.cpp).
 * ------------------------------------------------------------------------- */
struct orc_index {
    orc_params p;
    uint64_t n;
    int d;
    float* data;    /* copy of the dataset */
    float* coeffs;  /* [L][K][d] */
    float* table;   /* [L][K][N_r+1] */
    float* proj;    /* [L][n][K] (kept: the oracle's r_min lookup) */
    orc_tree** trees;
};

/* index.cpp:33-54: exact-membership DFS count with dedup, abort at budget. */
typedef struct {
    const orc_tree* t;
    const float* table;
    const float* q;
    const float* proj_space; /* [n][K] */
    double radius;
    uint8_t* seen;
    uint64_t count, budget;
} reach_ctx;

static int reach_visit(reach_ctx* c, int32_t ni) {
    const orc_tree* t = c->t;
    if (orc_mindist(t, ni, c->table, c->q) > c->radius) return 0;
    if (!t->nodes[ni].is_leaf) return reach_visit(c, t->nodes[ni].left) || reach_visit(c, t->nodes[ni].right);
    const int whole = maxdist(t, ni, c->table, c->q) <= c->radius;
    const onode* nd = &t->nodes[ni];
    for (uint32_t e = 0; e < nd->count; ++e) {
        const uint32_t pos = nd->pos[e];
        if (c->seen[pos]) continue;
        if (!whole && l2f(c->q, c->proj_space + (size_t)pos * t->K, t->K) > c->radius) continue;
        c->seen[pos] = 1;
        if (++c->count >= c->budget) return 1;
    }
    return 0;
}

static int reaches(const orc_index* x, const float* probe_proj /* [L][K] */, double r,
                   uint8_t* seen, uint64_t budget) {
    memset(seen, 0, x->n);
    reach_ctx c = {0};
    c.table = x->table;
    c.seen = seen;
    c.budget = budget;
    c.count = 0;
    for (int i = 0; i < x->p.L; ++i) {
        c.t = x->trees[i];
        c.q = probe_proj + (size_t)i * x->p.K;
        c.proj_space = x->proj + (size_t)i * x->n * x->p.K;
        c.radius = x->p.epsilon * r;
        const size_t slots = (size_t)1 << x->p.K;
        for (size_t s = 0; s < slots; ++s)
            if (c.t->root[s] >= 0 && reach_visit(&c, c.t->root[s])) return 1;
    }
    return 0;
}

/* index.cpp:60-73 */
static double grid_walk(const orc_index* x, const float* pp, double start, uint8_t* seen,
                        uint64_t budget) {
    const double c = x->p.c;
    double r = start;
    if (reaches(x, pp, r, seen, budget)) {
        for (int i = 0; i < 200 && r / c > 0.0 && reaches(x, pp, r / c, seen, budget); ++i) r /= c;
    } else {
        for (int i = 0; i < 200; ++i) {
            r *= c;
            if (reaches(x, pp, r, seen, budget)) break;
        }
    }
    return r;
}

static int cmp_double(const void* a, const void* b) {
    const double x = *(const double*)a, y = *(const double*)b;
    return (x > y) - (x < y);
}

/* index.cpp:75-136 + 153-175 */
static double estimate_rmin(const orc_index* x, uint64_t seed) {
    const uint64_t n = x->n;
    const int K = x->p.K, L = x->p.L;
    const uint64_t budget = orc_candidate_budget(x->p.beta, n, x->p.k);
    /* probes first: assemble draws them before estimate_rmin_core runs */
    orc_rng* rng = malloc(sizeof(orc_rng));
    orc_rng_seed(rng, orc_mix_seed(seed, 2));
    const uint64_t np = n < 10 ? n : 10;
    float* pp = malloc(np * (size_t)L * K * sizeof(float));
    for (uint64_t p = 0; p < np; ++p) {
        const uint64_t pos = orc_rng_bounded(rng, n);
        for (int i = 0; i < L; ++i)
            memcpy(pp + (p * L + i) * K, x->proj + ((size_t)i * n + pos) * K, K * sizeof(float));
    }
    free(rng);
    const uint64_t m = n < 32 ? n : 32;
    size_t npairs = (size_t)(m * (m - 1) / 2), q = 0;
    double* pd = malloc((npairs ? npairs : 1) * sizeof(double));
    for (uint64_t a = 0; a < m; ++a)
        for (uint64_t b = a + 1; b < m; ++b) {
            const uint64_t pa = a * n / m, pb = b * n / m;
            pd[q++] = l2f(x->proj + pa * K, x->proj + pb * K, K);
        }
    double guess = 1.0;
    if (npairs) {
        qsort(pd, npairs, sizeof(double), cmp_double);
        const double med = pd[npairs / 2];
        if (med > 0.0) guess = med / x->p.epsilon;
    }
    free(pd);
    uint8_t* seen = malloc(n);
    double* res = malloc(np * sizeof(double));
    double start = guess;
    for (uint64_t p = 0; p < np; ++p) {
        res[p] = grid_walk(x, pp + p * (size_t)L * K, start, seen, budget);
        start = res[p];
    }
    qsort(res, np, sizeof(double), cmp_double);
    const double out = res[(np - 1) / 2];
    free(seen);
    free(res);
    free(pp);
    return out;
}

static orc_index* assemble(const float* data, uint64_t n, int d, orc_params* params,
                           uint64_t seed, const float* table_in) {
    if (!data || n == 0) return NULL;
    orc_params p = *params;
    if (p.K < 1 || p.K > 24 || p.L < 1 || !(p.c > 1.0) || p.leaf_capacity < 1) return NULL;
    double der[4];
    orc_derive_params(p.K, p.c, p.L, der);
    p.alpha1 = der[0];
    p.alpha2 = der[1];
    p.epsilon = der[2];
    if (p.beta <= 0.0) p.beta = der[3];
    orc_index* x = calloc(1, sizeof(orc_index));
    x->n = n;
    x->d = d;
    x->data = malloc(n * (size_t)d * sizeof(float));
    memcpy(x->data, data, n * (size_t)d * sizeof(float));
    const size_t LK = (size_t)p.L * p.K, w = (size_t)p.n_regions + 1;
    x->coeffs = malloc(LK * d * sizeof(float));
    orc_sample_hash_family(d, p.K, p.L, orc_mix_seed(seed, 0), x->coeffs);
    x->proj = malloc(LK * n * sizeof(float));
    orc_project_dataset(x->coeffs, p.K, p.L, data, n, d, x->proj);
    x->table = malloc(LK * w * sizeof(float));
    if (table_in) {
        memcpy(x->table, table_in, LK * w * sizeof(float));
    } else if (orc_select_breakpoints(x->proj, n, p.K, p.L, p.n_regions, p.sample_fraction,
                                      orc_mix_seed(seed, 1), x->table, NULL, NULL, NULL)) {
        orc_index_free(x);
        return NULL;
    }
    uint8_t* codes = malloc(LK * n);
    orc_encode_dataset(x->proj, n, p.K, p.L, x->table, p.n_regions, codes);
    x->trees = calloc((size_t)p.L, sizeof(orc_tree*));
    for (int i = 0; i < p.L; ++i)
        x->trees[i] = orc_build_tree(codes, n, p.K, p.L, p.n_regions, i, p.leaf_capacity);
    free(codes);
    x->p = p;
    if (x->p.r_min <= 0.0) x->p.r_min = estimate_rmin(x, seed);
    *params = x->p;
    return x;
}

orc_index* orc_build_index(const float* data, uint64_t n, int d, orc_params* params,
                           uint64_t seed) {
    return assemble(data, n, d, params, seed, NULL);
}

orc_index* orc_build_index_with_table(const float* data, uint64_t n, int d, orc_params* params,
                                      uint64_t seed, const float* table) {
    return assemble(data, n, d, params, seed, table);
}

void orc_index_free(orc_index* x) {
    if (!x) return;
    if (x->trees)
        for (int i = 0; i < x->p.L; ++i) orc_tree_free(x->trees[i]);
    free(x->trees);
    free(x->data);
    free(x->coeffs);
    free(x->table);
    free(x->proj);
    free(x);
}

void orc_index_params(const orc_index* x, orc_params* out) { *out = x->p; }
void orc_index_table(const orc_index* x, float* out) {
    memcpy(out, x->table, (size_t)x->p.L * x->p.K * (x->p.n_regions + 1) * sizeof(float));
}
const orc_tree* orc_index_tree(const orc_index* x, int i) { return x->trees[i]; }

/* CandidateSet (index.cpp:234-265). */
typedef struct {
    const float* data;
    const float* q;
    int d;
    uint8_t* seen;
    double* dist;
    uint32_t* pos;
    uint64_t size, budget;
} cset;

static double l2_row(const float* a, const float* b, int d) {
    double acc = 0.0;
    for (int t = 0; t < d; ++t) {
        const double diff = (double)a[t] - (double)b[t];
        const double sq = diff * diff;
        acc = acc + sq;
    }
    return sqrt(acc);
}

static int cset_sink(void* c, uint32_t p) { /* index.cpp:322-325 */
    cset* s = c;
    if (!s->seen[p]) {
        s->seen[p] = 1;
        s->dist[s->size] = l2_row(s->q, s->data + (size_t)p * s->d, s->d);
        s->pos[s->size] = p;
        s->size++;
    }
    return s->size < s->budget;
}

typedef struct {
    double dist;
    uint32_t pos;
} dp;

static int cmp_dp(const void* a, const void* b) {
    const dp* x = a;
    const dp* y = b;
    if (x->dist < y->dist) return -1;
    if (x->dist > y->dist) return 1;
    return (x->pos > y->pos) - (x->pos < y->pos);
}

/* index.cpp:292-331 */
int orc_ck_ann(const orc_index* x, const float* q, int k, uint32_t* ids, double* dists,
               int* n_hits, double* radius_used, uint64_t* cands_seen) {
    if (k < 1 || (uint64_t)k > x->n || !(x->p.r_min > 0.0)) return 1;
    const int K = x->p.K, L = x->p.L;
    const uint64_t budget = orc_candidate_budget(x->p.beta, x->n, k);
    float* qp = malloc((size_t)L * K * sizeof(float));
    for (int i = 0; i < L; ++i) project_row(x->coeffs, K, x->d, i, q, qp + (size_t)i * K);
    cset s = {x->data, q, x->d, calloc(x->n, 1), malloc(x->n * sizeof(double)),
              malloc(x->n * sizeof(uint32_t)), 0, budget};
    double r = x->p.r_min;
    for (;;) {
        int done = 0;
        for (int i = 0; i < L; ++i) {
            range_opt(x->trees[i], x->table, qp + (size_t)i * K, x->p.epsilon * r, cset_sink, &s);
            if (s.size >= budget) {
                done = 1;
                break;
            }
        }
        if (!done) {
            uint64_t within = 0;
            const double lim = x->p.c * r;
            for (uint64_t m = 0; m < s.size; ++m)
                if (s.dist[m] <= lim) ++within;
            if (within >= (uint64_t)k) done = 1;
        }
        if (done) break;
        r *= x->p.c;
    }
    dp* all = malloc((s.size ? s.size : 1) * sizeof(dp));
    for (uint64_t m = 0; m < s.size; ++m) {
        all[m].dist = s.dist[m];
        all[m].pos = s.pos[m];
    }
    qsort(all, s.size, sizeof(dp), cmp_dp);
    const uint64_t take = s.size < (uint64_t)k ? s.size : (uint64_t)k;
    for (uint64_t m = 0; m < take; ++m) {
        ids[m] = all[m].pos;
        dists[m] = all[m].dist;
    }
    *n_hits = (int)take;
    *radius_used = r;
    *cands_seen = s.size;
    free(all);
    free(s.seen);
    free(s.dist);
    free(s.pos);
    free(qp);
    return 0;
}

/* metrics.cpp:8-33: exact kNN ordered by (dist, pos). */
void orc_brute_force_knn(const float* data, uint64_t n, int d, const float* Q, uint64_t nq, int k,
                         uint32_t* ids, double* dists) {
    dp* all = malloc(n * sizeof(dp));
    for (uint64_t qi = 0; qi < nq; ++qi) {
        for (uint64_t z = 0; z < n; ++z) {
            double acc = 0.0; /* squared distance; ordered by (dist^2, pos) */
            for (int t = 0; t < d; ++t) {
                const double diff = (double)Q[qi * d + t] - (double)data[z * d + t];
                const double sq = diff * diff;
                acc = acc + sq;
            }
            all[z].dist = acc;
            all[z].pos = (uint32_t)z;
        }
        qsort(all, n, sizeof(dp), cmp_dp);
        for (int t = 0; t < k; ++t) {
            ids[qi * k + t] = all[t].pos;
            dists[qi * k + t] = sqrt(all[t].dist);
        }
    }
    free(all);
}
