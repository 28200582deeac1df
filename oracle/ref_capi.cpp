// ref_capi.cpp — a C shim over the UNMODIFIED reference sources (TEST INFRASTRUCTURE).
//
// oracle/Makefile compiles this file together with /root/reference/proj/src/
// {dtype,matrix,factored_norm,compose,reference}.cpp, with `-Ddorafactor=dorafactor_ref`
// so the archive exports no `dorafactor::` symbols, into oracle/_ref/libdfx_ref.so.
// The shim only converts packed fp32 buffers to/from RealMatrix and calls the
// reference entry points; it adds no arithmetic of its own.  It is used to pin
// oracle/oracle.c (tests/test_oracle.py), to generate tests/golden/, and as the
// `--impl reference` CPU arm of bench.py.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <optional>
#include <vector>

#include "dorafactor/compose.hpp"
#include "dorafactor/factored_norm.hpp"
#include "dorafactor/layer.hpp"
#include "dorafactor/reference.hpp"

namespace R = dorafactor;  // renamed to dorafactor_ref by the -D flag

namespace {

// wall time of the last reference call made by this thread, packing excluded
thread_local std::int64_t g_last_ns = 0;

struct CallTimer {
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    ~CallTimer() {
        g_last_ns = std::chrono::duration_cast<std::chrono::nanoseconds>(
                        std::chrono::steady_clock::now() - t0)
                        .count();
    }
};

const R::DTypeSpec& spec(int dtype) {
    switch (dtype) {
        case 0: return R::DTypeSpec::fp32();
        case 1: return R::DTypeSpec::bf16e();
        case 2: return R::DTypeSpec::fp16e();
        default: return R::DTypeSpec::fp64();
    }
}

R::RealMatrix pack(const float* p, std::size_t rows, std::size_t cols, int dtype) {
    R::RealMatrix m(rows, cols, spec(dtype));
    auto& d = m.mutable_data();
    for (std::size_t i = 0; i < rows * cols; ++i) d[i] = static_cast<double>(p[i]);
    return m;
}

void unpack(const R::RealMatrix& m, float* out) {
    const auto& d = m.data();
    for (std::size_t i = 0; i < d.size(); ++i) out[i] = static_cast<float>(d[i]);
}

}  // namespace

extern "C" {

std::int64_t ref_last_call_ns() { return g_last_ns; }

int ref_plan_chunks(std::size_t d_out, std::size_t d_in, std::uint64_t budget,
                    std::size_t* chunk_size, std::size_t* num_chunks) {
    try {
        const R::ChunkPlan p = R::plan_chunks(d_out, d_in, budget);
        *chunk_size = p.chunk_size;
        *num_chunks = p.num_chunks;
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}

double ref_round_to_dtype(double x, int dtype) { return R::round_to_dtype(x, spec(dtype)); }

// W/A/B are packed with the given dtype tag; chunk_size builds a plan whose
// num_chunks matches d_in (the reference validates the pair).
int ref_norm_terms(int dtype, const float* w, const float* a, const float* b, std::size_t d_out,
                   std::size_t d_in, std::size_t r, double s, std::size_t chunk_size,
                   float* base_sq, float* cross, float* ba_sq) {
    try {
        const R::RealMatrix W = pack(w, d_out, d_in, dtype);
        const R::AdapterPair ad{pack(a, r, d_in, dtype), pack(b, d_out, r, dtype), s};
        R::ChunkPlan plan;
        plan.chunk_size = chunk_size;
        plan.num_chunks = (d_in + chunk_size - 1) / chunk_size;
        const R::NormTerms t = R::factored_norm_terms(W, ad, plan);
        std::memcpy(base_sq, t.base_sq.data(), d_out * sizeof(float));
        std::memcpy(cross, t.cross.data(), d_out * sizeof(float));
        std::memcpy(ba_sq, t.ba_sq.data(), d_out * sizeof(float));
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}

int ref_row_norm(int dtype, const float* w, const float* a, const float* b, std::size_t d_out,
                 std::size_t d_in, std::size_t r, double s, std::size_t chunk_size, double* out) {
    try {
        const R::RealMatrix W = pack(w, d_out, d_in, dtype);
        const R::AdapterPair ad{pack(a, r, d_in, dtype), pack(b, d_out, r, dtype), s};
        R::ChunkPlan plan;
        plan.chunk_size = chunk_size;
        plan.num_chunks = (d_in + chunk_size - 1) / chunk_size;
        std::vector<double> n;
        {
            CallTimer t;
            n = R::factored_row_norm(W, ad, plan);
        }
        std::memcpy(out, n.data(), d_out * sizeof(double));
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}

int ref_assemble(const float* base_sq, const float* cross, const float* ba_sq, double two_s,
                 double s2, std::size_t n, float* out) {
    R::NormTerms t;
    t.base_sq.assign(base_sq, base_sq + n);
    t.cross.assign(cross, cross + n);
    t.ba_sq.assign(ba_sq, ba_sq + n);
    t.two_s = two_s;
    t.s2 = s2;
    const std::vector<float> o = R::assemble_norm(t);
    std::memcpy(out, o.data(), n * sizeof(float));
    return 0;
}

int ref_magnitude_scale(int dtype, const double* m, const double* w_norm, std::size_t n,
                        double* g) {
    try {
        R::Magnitude mag{std::vector<double>(m, m + n), spec(dtype)};
        const std::vector<double> out =
            R::magnitude_scale(mag, std::vector<double>(w_norm, w_norm + n), spec(dtype));
        std::memcpy(g, out.data(), n * sizeof(double));
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}

// variant: 0 stable_compose, 1 fused_compose, 2 dual_output_compose, 3 naive_compose
int ref_compose(int variant, int dtype, const float* base, const float* lora, const double* g,
                double s, std::size_t rows, std::size_t d_out, float* delta, float* inner) {
    try {
        const R::RealMatrix Bm = pack(base, rows, d_out, dtype);
        const R::RealMatrix Lm = pack(lora, rows, d_out, dtype);
        const std::vector<double> gv(g, g + d_out);
        const R::ComposeInputs in{Bm, Lm, gv, s, spec(dtype)};
        R::RealMatrix d;
        std::optional<R::RealMatrix> inn;
        {
            CallTimer t;
            switch (variant) {
                case 0: d = R::stable_compose(in); break;
                case 1: d = R::fused_compose(in).delta; break;
                case 2: {
                    R::DualResult r = R::dual_output_compose(in, inner != nullptr);
                    d = std::move(r.delta);
                    inn = std::move(r.inner);
                    break;
                }
                default: d = R::naive_compose(in); break;
            }
        }
        unpack(d, delta);
        if (inner && inn) unpack(*inn, inner);
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}

int ref_compose_bwd(int dtype, const float* dy, const double* g, double s, const float* inner,
                    const double* w_norm, std::size_t rows, std::size_t d_out, int mag_grad,
                    float* d_lora, float* d_base, double* d_mag) {
    try {
        const R::RealMatrix D = pack(dy, rows, d_out, dtype);
        R::RealMatrix I;
        if (inner) I = pack(inner, rows, d_out, dtype);
        const std::vector<double> gv(g, g + d_out);
        const std::vector<double> wn =
            w_norm ? std::vector<double>(w_norm, w_norm + d_out) : std::vector<double>();
        R::GradBundle gb{R::RealMatrix(), R::RealMatrix(), std::nullopt};
        {
            CallTimer t;
            gb = R::compose_backward(D, gv, s, inner ? &I : nullptr, wn, mag_grad != 0);
        }
        unpack(gb.d_lora, d_lora);
        unpack(gb.d_base, d_base);
        if (mag_grad && d_mag) std::memcpy(d_mag, gb.d_mag->data(), d_out * sizeof(double));
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}

int ref_dense_row_norm_f64(const float* w, const float* a, const float* b, std::size_t d_out,
                           std::size_t d_in, std::size_t r, double s, double* out) {
    try {
        const R::RealMatrix W = pack(w, d_out, d_in, 0);
        const R::AdapterPair ad{pack(a, r, d_in, 0), pack(b, d_out, r, 0), s};
        const std::vector<double> n = R::dense_row_norm_f64(W, ad);
        std::memcpy(out, n.data(), d_out * sizeof(double));
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}

void ref_seeded_gaussian(std::size_t rows, std::size_t cols, std::uint64_t seed, int dtype,
                         float* out) {
    unpack(R::seeded_fixture(R::FixtureKind::Gaussian, rows, cols, seed, spec(dtype)), out);
}

void ref_gaussian_fixture(std::size_t rows, std::size_t cols, double mean, double stddev,
                          std::uint64_t seed, int dtype, float* out) {
    unpack(R::gaussian_fixture(rows, cols, mean, stddev, seed, spec(dtype)), out);
}

void ref_gaussian_vector(std::size_t n, double mean, double stddev, std::uint64_t seed,
                         double* out) {
    const std::vector<double> v = R::gaussian_vector(n, mean, stddev, seed);
    std::memcpy(out, v.data(), n * sizeof(double));
}

std::uint64_t ref_derive_seed(std::uint64_t base, std::uint64_t index) {
    return R::derive_seed(base, index);
}

// layer_forward (layer.cpp:51-127) on packed inputs: X [rows, d_in], W [d_out, d_in],
// A [r, d_in], B [d_out, r]; m / bias (nullable) [d_out].  Writes y, lora_mid, base_out,
// lora_out, inner (when the magnitude trains), g and w_norm.
int ref_layer_forward(int dtype, const float* x, const float* w, const float* a, const float* b,
                      double s, const double* m, const double* bias, std::size_t rows,
                      std::size_t d_in, std::size_t d_out, std::size_t r, float* y, float* lora_mid,
                      float* base_out, float* lora_out, float* inner, double* g, double* w_norm) {
    try {
        R::AdapterPair ad{pack(a, r, d_in, dtype), pack(b, d_out, r, dtype), s};
        R::Magnitude mag{std::vector<double>(m, m + d_out), spec(dtype)};
        std::optional<std::vector<double>> bv;
        if (bias) bv = std::vector<double>(bias, bias + d_out);
        const R::DoraLinearState st =
            R::make_layer_state(pack(w, d_out, d_in, dtype), ad, mag, bv, spec(dtype));
        const R::RealMatrix X = pack(x, rows, d_in, dtype);
        R::LayerForwardResult res{R::RealMatrix(), {}};
        {
            CallTimer t;
            res = R::layer_forward(st, X);
        }
        unpack(res.y, y);
        if (lora_mid) unpack(res.saved.lora_mid, lora_mid);
        if (base_out) unpack(res.saved.base_out, base_out);
        if (lora_out) unpack(res.saved.lora_out, lora_out);
        if (inner && res.saved.inner) unpack(*res.saved.inner, inner);
        if (g) std::memcpy(g, res.saved.g.data(), d_out * sizeof(double));
        if (w_norm) std::memcpy(w_norm, res.saved.w_norm.data(), d_out * sizeof(double));
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}

}  // extern "C"
