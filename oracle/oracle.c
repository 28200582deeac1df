/*
 * oracle.c — CPU restatement of the reference DoRA hot path (TEST INFRASTRUCTURE).
 *
 * Build: oracle/Makefile, `gcc -O2 -ffp-contract=off` — the reference's own
 * no-contraction discipline (proj/CMakeLists.txt:13).  On x86-64 float
 * arithmetic is SSE single precision, so every `float` expression below
 * rounds exactly once per operation, as in the reference.
 *
 * File:line citations refer to /root/reference/proj/src/.
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- numerics */

/* round_to_limits (dtype.cpp:25-40): scale so one target ulp is 1.0, round to
 * integer under the ambient RNE mode, scale back; subnormal spacing pinned. */
static double round_to_limits(double x, int sig_bits, int min_normal_exp, double max_finite) {
    if (x == 0.0 || !isfinite(x)) return x;
    int bexp = 0;
    (void)frexp(x, &bexp);
    int shift = sig_bits - bexp;
    const int sub_shift = sig_bits - 1 - min_normal_exp;
    if (shift > sub_shift) shift = sub_shift;
    const double rounded = ldexp(nearbyint(ldexp(x, shift)), -shift);
    if (fabs(rounded) > max_finite) return copysign(HUGE_VAL, x);
    return rounded;
}

/* round_to_dtype (dtype.cpp:77-85) with the limits of dtype.cpp:22-23. */
double orc_round_to_dtype(double x, int dtype) {
    switch (dtype) {
        case ORC_F64: return x;
        case ORC_F32: return (double)(float)x;
        case ORC_BF16: return round_to_limits(x, 8, -126, 0x1.FEp127);
        case ORC_F16: return round_to_limits(x, 11, -14, 65504.0);
    }
    return x;
}

/* DTypeSpec::norm_eps (dtype.cpp:10-13). */
double orc_norm_eps(int dtype) { return (dtype == ORC_BF16 || dtype == ORC_F16) ? 1e-6 : 1e-12; }

static inline float rnd_f(float x, int dtype) { return (float)orc_round_to_dtype((double)x, dtype); }

/* ---------------------------------------------------------------- planning */

/* plan_chunks (matrix.cpp:28-51). */
int orc_plan_chunks(size_t d_out, size_t d_in, uint64_t budget, size_t* chunk_size,
                    size_t* num_chunks) {
    const size_t align = 64;
    if (d_out < 1 || d_in < 1 || budget < 256) return -1;
    const uint64_t fit = budget / ((uint64_t)d_out * 4u);
    if (d_in >= align && fit < align) return -1;
    size_t cs = d_in < fit ? d_in : (size_t)fit;
    cs = (cs / align) * align;
    const size_t floor_cs = d_in < align ? d_in : align;
    if (cs < floor_cs) cs = floor_cs;
    *chunk_size = cs;
    *num_chunks = (d_in + cs - 1) / cs;
    return 0;
}

/* ------------------------------------------------------------ factored norm */

/* factored_norm_terms (factored_norm.cpp:27-120).  Chunk loop ascending; per
 * chunk: serial fp32 base_sq partial (:52-61), Gram partial per (p,q) (:65-76),
 * U_c with serial-k fp32 accumulation (:78-89), cross partial (:91-100); then
 * ba_sq = rowsum((B G) .* B) (:103-117).  s == 0 skips the adapter terms (:37). */
int orc_norm_terms(const float* w, const float* a, const float* b, size_t d_out, size_t d_in,
                   size_t r, double s, size_t chunk_size, float* base_sq, float* cross,
                   float* ba_sq) {
    if (r < 1 || chunk_size < 1) return -1;
    const int skip = (s == 0.0);
    for (size_t i = 0; i < d_out; ++i) base_sq[i] = cross[i] = ba_sq[i] = 0.0f;
    float* gram = skip ? NULL : (float*)calloc(r * r, sizeof(float));
    float* u = skip ? NULL : (float*)malloc(r * sizeof(float));
    for (size_t c0 = 0; c0 < d_in; c0 += chunk_size) {
        const size_t c1 = c0 + chunk_size < d_in ? c0 + chunk_size : d_in;
        for (size_t i = 0; i < d_out; ++i) {
            float partial = 0.0f;
            const float* wr = w + i * d_in;
            for (size_t k = c0; k < c1; ++k) partial += wr[k] * wr[k];
            base_sq[i] += partial;
        }
        if (skip) continue;
        for (size_t p = 0; p < r; ++p) {
            const float* ap = a + p * d_in;
            for (size_t q = 0; q < r; ++q) {
                const float* aq = a + q * d_in;
                float partial = 0.0f;
                for (size_t k = c0; k < c1; ++k) partial += ap[k] * aq[k];
                gram[p * r + q] += partial;
            }
        }
        /* U_c row by row; the reference materialises the chunk's U (:47, :87) but
         * consumes it strictly row-wise in :91-100, so a row buffer is equivalent. */
        for (size_t i = 0; i < d_out; ++i) {
            const float* wr = w + i * d_in;
            for (size_t l = 0; l < r; ++l) {
                const float* al = a + l * d_in;
                float acc = 0.0f;
                for (size_t k = c0; k < c1; ++k) acc += wr[k] * al[k];
                u[l] = acc;
            }
            float partial = 0.0f;
            const float* br = b + i * r;
            for (size_t l = 0; l < r; ++l) partial += br[l] * u[l];
            cross[i] += partial;
        }
    }
    if (!skip) {
        for (size_t i = 0; i < d_out; ++i) {
            const float* br = b + i * r;
            float rowsum = 0.0f;
            for (size_t l = 0; l < r; ++l) {
                float bg = 0.0f;
                for (size_t q = 0; q < r; ++q) bg += br[q] * gram[q * r + l];
                rowsum += bg * br[l];
            }
            ba_sq[i] = rowsum;
        }
    }
    free(gram);
    free(u);
    return 0;
}

/* assemble_norm (factored_norm.cpp:122-136): fp64 scale products rounded to
 * fp32, fp32 adds, NaN-preserving clamp at 0 (dtype.cpp:91-94), IEEE sqrt. */
void orc_assemble(const float* base_sq, const float* cross, const float* ba_sq, double two_s,
                  double s2, size_t n, float* out) {
    for (size_t j = 0; j < n; ++j) {
        const float c1 = (float)(two_s * (double)cross[j]);
        const float t1 = base_sq[j] + c1;
        const float c2 = (float)(s2 * (double)ba_sq[j]);
        float t2 = t1 + c2;
        if (!isnan(t2) && t2 < 0.0f) t2 = 0.0f;
        out[j] = sqrtf(t2);
    }
}

/* factored_row_norm (factored_norm.cpp:204-217), non-fp64 weights. */
int orc_row_norm(int dtype, const float* w, const float* a, const float* b, size_t d_out,
                 size_t d_in, size_t r, double s, size_t chunk_size, float* out) {
    if (dtype == ORC_F64) return -1;
    float* t = (float*)malloc(3 * d_out * sizeof(float) + 1);
    const int rc = orc_norm_terms(w, a, b, d_out, d_in, r, s, chunk_size, t, t + d_out,
                                  t + 2 * d_out);
    if (rc == 0) {
        orc_assemble(t, t + d_out, t + 2 * d_out, 2.0 * s, s * s, d_out, out);
        for (size_t j = 0; j < d_out; ++j) out[j] = rnd_f(out[j], dtype);
    }
    free(t);
    return rc;
}

/* magnitude_scale (factored_norm.cpp:232-239): fp32 divide by the eps-floored
 * norm (`wn < eps ? eps : wn`, so NaN passes through), result rounded to dtype. */
void orc_magnitude_scale(int dtype, const double* m, const float* w_norm, size_t n, float* g) {
    const float eps = (float)orc_norm_eps(dtype);
    for (size_t j = 0; j < n; ++j) {
        const float wn = w_norm[j];
        const float denom = wn < eps ? eps : wn;
        const float q = (float)m[j] / denom;
        g[j] = rnd_f(q, dtype);
    }
}

/* ------------------------------------------------------------------ compose */

/* stable_element (compose.cpp:19-24) + the store rounding of :34-41; the dual
 * variant's inner = round(t + base) (compose.cpp:131-137). */
void orc_compose_fwd(int dtype, const float* base, const float* lora, const float* g, double s,
                     size_t rows, size_t d_out, float* delta, float* inner) {
    const float sf = (float)s;
    for (size_t i = 0; i < rows; ++i) {
        for (size_t j = 0; j < d_out; ++j) {
            const size_t e = i * d_out + j;
            const float gf = g[j];
            const float t = sf * lora[e];
            const float u = gf * t;
            const float v = (gf - 1.0f) * base[e];
            delta[e] = rnd_f(v + u, dtype);
            if (inner) inner[e] = rnd_f(t + base[e], dtype);
        }
    }
}

/* working_matmul (layer.cpp:15-17 over matrix.cpp:53-78): C = A . B^T with A [m, k] and
 * Bt [n, k] row-major, fp32 accumulation ascending in k, result rounded to dtype. */
void orc_working_matmul_nt(int dtype, const float* a, const float* bt, size_t m, size_t n,
                           size_t k, float* out) {
    for (size_t i = 0; i < m; ++i) {
        for (size_t j = 0; j < n; ++j) {
            float acc = 0.0f;
            for (size_t kk = 0; kk < k; ++kk) acc += a[i * k + kk] * bt[j * k + kk];
            out[i * n + j] = rnd_f(acc, dtype);
        }
    }
}

/* Residual and bias after the compose (layer.cpp:108-120): y = round(base + delta), then
 * y = round(y + bias[j]) when bias is given; all adds in fp32. */
void orc_residual(int dtype, const float* base, const float* delta, const float* bias,
                  size_t rows, size_t d_out, float* y) {
    for (size_t i = 0; i < rows; ++i) {
        for (size_t j = 0; j < d_out; ++j) {
            const size_t e = i * d_out + j;
            float v = rnd_f(base[e] + delta[e], dtype);
            if (bias) v = rnd_f(v + bias[j], dtype);
            y[e] = v;
        }
    }
}

/* naive_compose (compose.cpp:47-68): every intermediate re-rounded to dtype. */
void orc_naive_compose(int dtype, const float* base, const float* lora, const float* g, double s,
                       size_t rows, size_t d_out, float* delta) {
    const float sf = (float)s;
    for (size_t i = 0; i < rows; ++i) {
        for (size_t j = 0; j < d_out; ++j) {
            const size_t e = i * d_out + j;
            const float t1 = rnd_f(sf * lora[e], dtype);
            const float t2 = rnd_f(t1 + base[e], dtype);
            const float t3 = rnd_f(g[j] * t2, dtype);
            delta[e] = rnd_f(t3 - base[e], dtype);
        }
    }
}

/* compose_backward (compose.cpp:154-201): elementwise d_lora = round(g*(s*dy)),
 * d_base = round((g-1)*dy) (:177-185); d_mag[j] = serial-over-rows fp32 sum of
 * dy*inner, divided once by fl32(w_norm[j]) (:187-199), not dtype-rounded. */
int orc_compose_bwd(int dtype, const float* dy, const float* g, double s, const float* inner,
                    const float* w_norm, size_t rows, size_t d_out, int mag_grad, float* d_lora,
                    float* d_base, float* d_mag) {
    if (mag_grad && (inner == NULL || w_norm == NULL || d_mag == NULL)) return -1;
    const float sf = (float)s;
    for (size_t i = 0; i < rows; ++i) {
        for (size_t j = 0; j < d_out; ++j) {
            const size_t e = i * d_out + j;
            const float gf = g[j];
            const float t = sf * dy[e];
            d_lora[e] = rnd_f(gf * t, dtype);
            d_base[e] = rnd_f((gf - 1.0f) * dy[e], dtype);
        }
    }
    if (mag_grad) {
        for (size_t j = 0; j < d_out; ++j) {
            float acc = 0.0f;
            for (size_t i = 0; i < rows; ++i) acc += dy[i * d_out + j] * inner[i * d_out + j];
            d_mag[j] = acc / w_norm[j];
        }
    }
    return 0;
}

/* dense_row_norm_f64 (reference.cpp:19-50): materialise BA in fp64 (matmul_f64,
 * :33-44) and take the per-row L2 norm of W + s*BA. */
void orc_dense_row_norm_f64(const float* w, const float* a, const float* b, size_t d_out,
                            size_t d_in, size_t r, double s, double* out) {
    double* row = (double*)malloc((d_in ? d_in : 1) * sizeof(double));
    for (size_t i = 0; i < d_out; ++i) {
        for (size_t k = 0; k < d_in; ++k) {
            double acc = 0.0;
            for (size_t l = 0; l < r; ++l) acc += (double)b[i * r + l] * (double)a[l * d_in + k];
            row[k] = acc;
        }
        double acc = 0.0;
        for (size_t k = 0; k < d_in; ++k) {
            const double v = (double)w[i * d_in + k] + s * row[k];
            acc += v * v;
        }
        out[i] = sqrt(acc);
    }
    free(row);
}

/* ----------------------------------------------------------------- fixtures */

/* mt19937_64 (the std::mt19937_64 the reference seeds directly, matrix.cpp:84). */
typedef struct {
    uint64_t mt[312];
    int idx;
    int have_spare;
    double spare;
} orc_rng;

static void rng_seed(orc_rng* g, uint64_t seed) {
    g->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
    g->idx = 312;
    g->have_spare = 0;
    g->spare = 0.0;
}

static uint64_t rng_next(orc_rng* g) {
    static const uint64_t mag[2] = {0ULL, 0xB5026F5AA96619E9ULL};
    if (g->idx >= 312) {
        int i;
        for (i = 0; i < 312 - 156; ++i) {
            const uint64_t y = (g->mt[i] & 0xFFFFFFFF80000000ULL) | (g->mt[i + 1] & 0x7FFFFFFFULL);
            g->mt[i] = g->mt[i + 156] ^ (y >> 1) ^ mag[y & 1];
        }
        for (; i < 311; ++i) {
            const uint64_t y = (g->mt[i] & 0xFFFFFFFF80000000ULL) | (g->mt[i + 1] & 0x7FFFFFFFULL);
            g->mt[i] = g->mt[i - 156] ^ (y >> 1) ^ mag[y & 1];
        }
        const uint64_t y = (g->mt[311] & 0xFFFFFFFF80000000ULL) | (g->mt[0] & 0x7FFFFFFFULL);
        g->mt[311] = g->mt[155] ^ (y >> 1) ^ mag[y & 1];
        g->idx = 0;
    }
    uint64_t x = g->mt[g->idx++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= x >> 43;
    return x;
}

/* FixtureRng::uniform / gaussian (matrix.cpp:86-107). */
static double rng_uniform(orc_rng* g) { return (double)(rng_next(g) >> 11) * 0x1p-53; }

static double rng_gaussian(orc_rng* g) {
    if (g->have_spare) {
        g->have_spare = 0;
        return g->spare;
    }
    double u1 = rng_uniform(g);
    if (u1 <= 0.0) u1 = 0x1p-53;
    const double u2 = rng_uniform(g);
    const double radius = sqrt(-2.0 * log(u1));
    const double theta = 2.0 * 3.14159265358979323846 * u2;
    g->spare = radius * sin(theta);
    g->have_spare = 1;
    return radius * cos(theta);
}

/* derive_seed (matrix.cpp:142-148): splitmix64 finaliser. */
uint64_t orc_derive_seed(uint64_t base, uint64_t index) {
    uint64_t z = base + 0x9e3779b97f4a7c15ULL * (index + 1);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

/* seeded_fixture(Gaussian) (matrix.cpp:114-123). */
void orc_seeded_gaussian(size_t n, uint64_t seed, int dtype, float* out) {
    orc_rng g;
    rng_seed(&g, seed);
    for (size_t i = 0; i < n; ++i) out[i] = (float)orc_round_to_dtype(rng_gaussian(&g), dtype);
}

/* gaussian_fixture (matrix.cpp:125-133). */
void orc_gaussian_fixture(size_t n, double mean, double stddev, uint64_t seed, int dtype,
                          float* out) {
    orc_rng g;
    rng_seed(&g, seed);
    for (size_t i = 0; i < n; ++i)
        out[i] = (float)orc_round_to_dtype(mean + stddev * rng_gaussian(&g), dtype);
}

/* gaussian_vector (matrix.cpp:135-140): fp64, not rounded. */
void orc_gaussian_vector(size_t n, double mean, double stddev, uint64_t seed, double* out) {
    orc_rng g;
    rng_seed(&g, seed);
    for (size_t i = 0; i < n; ++i) out[i] = mean + stddev * rng_gaussian(&g);
}
