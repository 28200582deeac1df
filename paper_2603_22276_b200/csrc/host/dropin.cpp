// dropin.cpp — the reference C++ API (namespace dorafactor) implemented over the C ABI.
//
// This is the host-side mirror of proj/include/dorafactor/{dtype,matrix,factored_norm,
// compose}.hpp.  It validates exactly where the reference throws (same conditions,
// std::invalid_argument), packs RealMatrix fp64 storage into the dtype's bits, runs the
// sm_100a kernels through include/dfx.h, and unpacks.  There is no CPU fallback for the
// hot path: without a usable B200 every call throws std::runtime_error.
//
// Performance is measured at the C ABI on device-resident buffers; this layer is the
// drop-in convenience surface (its cost is the fp64 packing and the PCIe copies).
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <random>
#include <stdexcept>
#include <string>

#include "dfx.h"
#include "dorafactor/compose.hpp"
#include "dorafactor/dispatch.hpp"
#include "dorafactor/factored_norm.hpp"
#include "dorafactor/layer.hpp"

namespace dorafactor {

// ===================================================================== numerics
namespace {

constexpr DTypeSpec kSpecF64{DTypeKind::FP64, 52, 1e-12, 0x1p-52, 0x1p-53, 8};
constexpr DTypeSpec kSpecF32{DTypeKind::FP32, 23, 1e-12, 0x1p-23, 0x1p-24, 4};
constexpr DTypeSpec kSpecBF16{DTypeKind::BF16E, 7, 1e-6, 0x1p-7, 0x1p-8, 2};
constexpr DTypeSpec kSpecF16{DTypeKind::FP16E, 10, 1e-6, 0x1p-10, 0x1p-11, 2};

// RNE onto a binary grid with `prec` significand bits, minimum normal exponent
// `emin` (subnormal spacing 2^(emin-prec+1)) and largest finite value `vmax`.
double round_to_grid(double x, int prec, int emin, double vmax) {
    if (!std::isfinite(x) || x == 0.0) return x;
    const int e = std::max(std::ilogb(x), emin);       // exponent of the binade
    const int q = e - prec + 1;                          // exponent of one ulp there
    const double r = std::scalbn(std::nearbyint(std::scalbn(x, -q)), q);
    return std::fabs(r) > vmax ? std::copysign(INFINITY, x) : r;
}

}  // namespace

const DTypeSpec& DTypeSpec::fp64() { return kSpecF64; }
const DTypeSpec& DTypeSpec::fp32() { return kSpecF32; }
const DTypeSpec& DTypeSpec::bf16e() { return kSpecBF16; }
const DTypeSpec& DTypeSpec::fp16e() { return kSpecF16; }

const DTypeSpec& DTypeSpec::from_kind(DTypeKind kind) {
    switch (kind) {
        case DTypeKind::FP64: return kSpecF64;
        case DTypeKind::FP32: return kSpecF32;
        case DTypeKind::BF16E: return kSpecBF16;
        case DTypeKind::FP16E: return kSpecF16;
    }
    throw std::invalid_argument("unknown dtype kind");
}

const DTypeSpec& DTypeSpec::from_name(const std::string& name) {
    if (name == "fp64" || name == "f64") return kSpecF64;
    if (name == "fp32" || name == "f32") return kSpecF32;
    if (name == "bf16" || name == "bf16e") return kSpecBF16;
    if (name == "fp16" || name == "fp16e") return kSpecF16;
    throw std::invalid_argument("unknown dtype name: " + name);
}

const char* DTypeSpec::name() const {
    switch (kind) {
        case DTypeKind::FP64: return "fp64";
        case DTypeKind::FP32: return "fp32";
        case DTypeKind::BF16E: return "bf16";
        case DTypeKind::FP16E: return "fp16";
    }
    return "?";
}

double round_to_dtype(double x, const DTypeSpec& spec) {
    switch (spec.kind) {
        case DTypeKind::FP64: return x;
        case DTypeKind::FP32: return static_cast<double>(static_cast<float>(x));
        case DTypeKind::BF16E: return round_to_grid(x, 8, -126, 0x1.FEp127);
        case DTypeKind::FP16E: return round_to_grid(x, 11, -14, 65504.0);
    }
    return x;
}

float correctly_rounded_sqrt_f32(float x) { return std::sqrt(x); }

float nan_preserving_clamp_min(float x, float floor) {
    return std::isnan(x) ? x : (x < floor ? floor : x);
}

// ======================================================================= matrix
RealMatrix RealMatrix::to_dtype(const DTypeSpec& target) const {
    RealMatrix out(rows_, cols_, target);
    auto& d = out.mutable_data();
    for (index_t i = 0; i < data_.size(); ++i) d[i] = round_to_dtype(data_[i], target);
    return out;
}

RealMatrix transpose(const RealMatrix& m) {
    RealMatrix out(m.cols(), m.rows(), m.dtype());
    auto& d = out.mutable_data();
    for (index_t i = 0; i < m.rows(); ++i)
        for (index_t j = 0; j < m.cols(); ++j) d[j * m.rows() + i] = m(i, j);
    return out;
}

ChunkPlan plan_chunks(index_t d_out, index_t d_in, std::uint64_t budget_bytes) {
    std::uint64_t cs = 0, nc = 0;
    if (dfx_plan_chunks(d_out, d_in, budget_bytes, &cs, &nc) != DFX_OK)
        throw std::invalid_argument(dfx_last_error());
    ChunkPlan p;
    p.budget_bytes = budget_bytes;
    p.chunk_size = static_cast<index_t>(cs);
    p.alignment = 64;
    p.num_chunks = static_cast<index_t>(nc);
    return p;
}

namespace {

// mt19937_64 stream with Box-Muller pairs (the fixture contract of matrix.hpp).
class Draws {
public:
    explicit Draws(std::uint64_t seed) : gen_(seed) {}
    double uniform() { return static_cast<double>(gen_() >> 11) * 0x1p-53; }
    double normal() {
        if (cached_) {
            cached_ = false;
            return cache_;
        }
        const double u1 = std::max(uniform(), 0x1p-53);
        const double u2 = uniform();
        const double rad = std::sqrt(-2.0 * std::log(u1));
        const double ang = 2.0 * 3.14159265358979323846 * u2;
        cache_ = rad * std::sin(ang);
        cached_ = true;
        return rad * std::cos(ang);
    }

private:
    std::mt19937_64 gen_;
    bool cached_ = false;
    double cache_ = 0.0;
};

}  // namespace

RealMatrix seeded_fixture(FixtureKind kind, index_t rows, index_t cols, std::uint64_t seed,
                          const DTypeSpec& dtype) {
    RealMatrix out(rows, cols, dtype);
    Draws d(seed);
    for (double& v : out.mutable_data())
        v = round_to_dtype(kind == FixtureKind::Gaussian ? d.normal() : d.uniform(), dtype);
    return out;
}

RealMatrix gaussian_fixture(index_t rows, index_t cols, double mean, double stddev,
                            std::uint64_t seed, const DTypeSpec& dtype) {
    RealMatrix out(rows, cols, dtype);
    Draws d(seed);
    for (double& v : out.mutable_data()) v = round_to_dtype(mean + stddev * d.normal(), dtype);
    return out;
}

std::vector<double> gaussian_vector(index_t n, double mean, double stddev, std::uint64_t seed) {
    std::vector<double> out(n);
    Draws d(seed);
    for (double& v : out) v = mean + stddev * d.normal();
    return out;
}

std::uint64_t derive_seed(std::uint64_t base, std::uint64_t index) {
    std::uint64_t z = base + 0x9e3779b97f4a7c15ULL * (index + 1);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

// ================================================================ device plumbing
namespace {

dfx_ctx* device_ctx() {
    static std::once_flag once;
    static dfx_ctx* ctx = nullptr;
    static std::string why;
    std::call_once(once, [] {
        int dev = 0;
        if (const char* e = std::getenv("DFX_DEVICE")) dev = std::atoi(e);
        if (dfx_ctx_create(dev, &ctx) != DFX_OK) {
            why = dfx_last_error();
            ctx = nullptr;
        }
    });
    if (!ctx) throw std::runtime_error("dorafactor (B200 build): no usable sm_100 device: " + why);
    return ctx;
}

void check(int rc) {
    if (rc == DFX_OK) return;
    if (rc == DFX_EINVAL) throw std::invalid_argument(dfx_last_error());
    throw std::runtime_error(std::string("dorafactor (B200 build): ") + dfx_last_error());
}

void check_cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// Owned device allocation.
struct DevBuf {
    void* p = nullptr;
    explicit DevBuf(size_t bytes) { check_cuda(cudaMalloc(&p, bytes ? bytes : 16), "cudaMalloc"); }
    ~DevBuf() { if (p) cudaFree(p); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p) { o.p = nullptr; }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) {
            if (p) cudaFree(p);
            p = o.p;
            o.p = nullptr;
        }
        return *this;
    }
    template <typename T> T* as() const { return static_cast<T*>(p); }
};

dfx_dtype to_dfx(const DTypeSpec& s) {
    switch (s.kind) {
        case DTypeKind::FP32: return DFX_F32;
        case DTypeKind::BF16E: return DFX_BF16;
        case DTypeKind::FP16E: return DFX_F16;
        default: return DFX_F32;
    }
}

size_t elem_size(dfx_dtype dt) { return dt == DFX_F32 ? 4 : 2; }

// fp64 storage -> dtype bits.  Values are representable in the tag, so the fp32
// conversion is exact and the 16-bit conversions are exact RNE no-ops.
std::vector<unsigned char> pack(const std::vector<double>& v, dfx_dtype dt) {
    std::vector<unsigned char> out(v.size() * elem_size(dt));
    if (dt == DFX_F32) {
        float* o = reinterpret_cast<float*>(out.data());
        for (size_t i = 0; i < v.size(); ++i) o[i] = static_cast<float>(v[i]);
    } else if (dt == DFX_BF16) {
        __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(out.data());
        for (size_t i = 0; i < v.size(); ++i) o[i] = __float2bfloat16_rn(static_cast<float>(v[i]));
    } else {
        __half* o = reinterpret_cast<__half*>(out.data());
        for (size_t i = 0; i < v.size(); ++i) o[i] = __float2half_rn(static_cast<float>(v[i]));
    }
    return out;
}

void unpack(const std::vector<unsigned char>& raw, dfx_dtype dt, std::vector<double>& out) {
    if (dt == DFX_F32) {
        const float* p = reinterpret_cast<const float*>(raw.data());
        for (size_t i = 0; i < out.size(); ++i) out[i] = static_cast<double>(p[i]);
    } else if (dt == DFX_BF16) {
        const __nv_bfloat16* p = reinterpret_cast<const __nv_bfloat16*>(raw.data());
        for (size_t i = 0; i < out.size(); ++i) out[i] = static_cast<double>(__bfloat162float(p[i]));
    } else {
        const __half* p = reinterpret_cast<const __half*>(raw.data());
        for (size_t i = 0; i < out.size(); ++i) out[i] = static_cast<double>(__half2float(p[i]));
    }
}

DevBuf upload(const std::vector<double>& v, dfx_dtype dt) {
    const std::vector<unsigned char> h = pack(v, dt);
    DevBuf d(h.size());
    check_cuda(cudaMemcpy(d.p, h.data(), h.size(), cudaMemcpyHostToDevice), "H2D");
    return d;
}

DevBuf upload_f32(const std::vector<float>& v) {
    DevBuf d(v.size() * 4);
    check_cuda(cudaMemcpy(d.p, v.data(), v.size() * 4, cudaMemcpyHostToDevice), "H2D");
    return d;
}

std::vector<float> download_f32(const DevBuf& d, size_t n) {
    std::vector<float> out(n);
    if (n) check_cuda(cudaMemcpy(out.data(), d.p, n * 4, cudaMemcpyDeviceToHost), "D2H");
    return out;
}

void download(const DevBuf& d, dfx_dtype dt, RealMatrix& m) {
    std::vector<unsigned char> raw(m.data().size() * elem_size(dt));
    if (!raw.empty())
        check_cuda(cudaMemcpy(raw.data(), d.p, raw.size(), cudaMemcpyDeviceToHost), "D2H");
    unpack(raw, dt, m.mutable_data());
}

// One dtype shared by the operands (the C ABI takes one).  When the tags differ
// the operands are widened to fp32 exactly, which is what the reference computes
// with anyway (static_cast<float> of every element).
dfx_dtype common_dtype(std::initializer_list<const RealMatrix*> ms) {
    const DTypeKind k = (*ms.begin())->dtype().kind;
    for (const RealMatrix* m : ms)
        if (m->dtype().kind != k) return DFX_F32;
    return to_dfx((*ms.begin())->dtype());
}

void check_norm_shapes(const RealMatrix& w, const AdapterPair& ad, const ChunkPlan& plan) {
    // factored_norm.cpp:11-23
    const index_t d_out = w.rows(), d_in = w.cols(), r = ad.A.rows();
    if (ad.A.cols() != d_in) throw std::invalid_argument("factored_norm: A.cols != W.cols");
    if (ad.B.rows() != d_out || ad.B.cols() != r)
        throw std::invalid_argument("factored_norm: B shape inconsistent with W/A");
    if (r < 1) throw std::invalid_argument("factored_norm: rank must be >= 1");
    if (plan.chunk_size < 1 || plan.num_chunks != (d_in + plan.chunk_size - 1) / plan.chunk_size)
        throw std::invalid_argument("factored_norm: chunk plan does not match W.cols");
}

}  // namespace

// ================================================================ factored norm
NormTerms factored_norm_terms(const RealMatrix& w, const AdapterPair& adapter,
                              const ChunkPlan& plan) {
    if (w.dtype().kind == DTypeKind::FP64)
        throw std::invalid_argument(
            "factored_norm_terms: fp32 term accumulation requires non-FP64 weights");
    check_norm_shapes(w, adapter, plan);
    dfx_ctx* ctx = device_ctx();
    const index_t d_out = w.rows(), d_in = w.cols(), r = adapter.A.rows();
    const dfx_dtype dt = common_dtype({&w, &adapter.A, &adapter.B});
    const DevBuf dW = upload(w.data(), dt), dA = upload(adapter.A.data(), dt),
                 dB = upload(adapter.B.data(), dt);
    DevBuf terms(3 * d_out * sizeof(float));
    float* t = terms.as<float>();
    check(dfx_norm_terms(ctx, dt, dW.p, dA.p, dB.p, d_out, d_in, r, adapter.s, plan.chunk_size,
                         t, t + d_out, t + 2 * d_out, nullptr));
    const std::vector<float> all = download_f32(terms, 3 * d_out);
    NormTerms out;
    out.base_sq.assign(all.begin(), all.begin() + d_out);
    out.cross.assign(all.begin() + d_out, all.begin() + 2 * d_out);
    out.ba_sq.assign(all.begin() + 2 * d_out, all.end());
    out.two_s = 2.0 * adapter.s;
    out.s2 = adapter.s * adapter.s;
    return out;
}

std::vector<float> assemble_norm(const NormTerms& terms) {
    const index_t n = terms.base_sq.size();
    if (terms.cross.size() != n || terms.ba_sq.size() != n)
        throw std::invalid_argument("assemble_norm: term vectors differ in length");
    dfx_ctx* ctx = device_ctx();
    const DevBuf b = upload_f32(terms.base_sq), c = upload_f32(terms.cross),
                 q = upload_f32(terms.ba_sq);
    DevBuf out(n * sizeof(float));
    check(dfx_assemble_norm(ctx, b.as<float>(), c.as<float>(), q.as<float>(), terms.two_s,
                            terms.s2, n, DFX_F32, out.as<float>(), nullptr));
    return download_f32(out, n);
}

std::vector<double> factored_row_norm(const RealMatrix& w, const AdapterPair& adapter,
                                      const ChunkPlan& plan) {
    if (w.dtype().kind == DTypeKind::FP64) {
        check_norm_shapes(w, adapter, plan);
        throw std::invalid_argument(
            "factored_row_norm: FP64 weights are the reference's oracle-only mode; the B200 "
            "path computes fp32/bf16/fp16 weights");
    }
    check_norm_shapes(w, adapter, plan);
    dfx_ctx* ctx = device_ctx();
    const index_t d_out = w.rows(), d_in = w.cols(), r = adapter.A.rows();
    const dfx_dtype dt = common_dtype({&w, &adapter.A, &adapter.B});
    const DevBuf dW = upload(w.data(), dt), dA = upload(adapter.A.data(), dt),
                 dB = upload(adapter.B.data(), dt);
    DevBuf norm(d_out * sizeof(float));
    // round to W's own dtype (factored_norm.cpp:213-215), even when operands widened
    if (dt == to_dfx(w.dtype())) {
        check(dfx_row_norm(ctx, dt, dW.p, dA.p, dB.p, d_out, d_in, r, adapter.s, plan.chunk_size,
                           nullptr, dt, norm.as<float>(), nullptr, nullptr, nullptr));
    } else {
        DevBuf terms(3 * d_out * sizeof(float));
        float* t = terms.as<float>();
        check(dfx_norm_terms(ctx, dt, dW.p, dA.p, dB.p, d_out, d_in, r, adapter.s,
                             plan.chunk_size, t, t + d_out, t + 2 * d_out, nullptr));
        check(dfx_assemble_norm(ctx, t, t + d_out, t + 2 * d_out, 2.0 * adapter.s,
                                adapter.s * adapter.s, d_out, to_dfx(w.dtype()), norm.as<float>(),
                                nullptr));
    }
    const std::vector<float> n32 = download_f32(norm, d_out);
    return std::vector<double>(n32.begin(), n32.end());
}

std::vector<double> magnitude_scale(const Magnitude& m, const std::vector<double>& w_norm,
                                    const DTypeSpec& dtype) {
    if (m.values.size() != w_norm.size())
        throw std::invalid_argument("magnitude_scale: length mismatch");
    if (dtype.kind == DTypeKind::FP64)
        throw std::invalid_argument(
            "magnitude_scale: FP64 working dtype is the reference's oracle-only mode");
    dfx_ctx* ctx = device_ctx();
    const index_t n = w_norm.size();
    std::vector<float> mf(n), wf(n);
    for (index_t j = 0; j < n; ++j) {
        mf[j] = static_cast<float>(m.values[j]);
        wf[j] = static_cast<float>(w_norm[j]);
    }
    const DevBuf dm = upload_f32(mf), dw = upload_f32(wf);
    DevBuf dg(n * sizeof(float));
    check(dfx_magnitude_scale(ctx, to_dfx(dtype), dm.as<float>(), dw.as<float>(), n,
                              dg.as<float>(), nullptr));
    const std::vector<float> g = download_f32(dg, n);
    return std::vector<double>(g.begin(), g.end());
}

// ====================================================================== compose
namespace {

void check_compose(const ComposeInputs& in) {
    // compose.cpp:9-16
    if (in.base.rows() != in.lora.rows() || in.base.cols() != in.lora.cols())
        throw std::invalid_argument("compose: base/lora shapes differ");
    if (in.g.size() != in.base.cols()) throw std::invalid_argument("compose: g length != d_out");
}

// Runs the forward kernel; returns delta (and inner when requested) in in.dtype.
void run_compose(const ComposeInputs& in, RealMatrix& delta, RealMatrix* inner) {
    if (in.dtype.kind == DTypeKind::FP64)
        throw std::invalid_argument("compose: FP64 working dtype is not a B200 storage format");
    dfx_ctx* ctx = device_ctx();
    const index_t rows = in.base.rows(), d_out = in.base.cols();
    const dfx_dtype out_dt = to_dfx(in.dtype);
    // inputs stored in a different format than the working dtype: compute the same
    // fp32 expression with fp32 storage, then apply the single store rounding here
    const bool same = in.base.dtype() == in.dtype && in.lora.dtype() == in.dtype;
    const dfx_dtype dt = same ? out_dt : DFX_F32;
    const DevBuf db = upload(in.base.data(), dt), dl = upload(in.lora.data(), dt);
    std::vector<float> gf(d_out);
    for (index_t j = 0; j < d_out; ++j) gf[j] = static_cast<float>(in.g[j]);
    const DevBuf dg = upload_f32(gf);
    DevBuf dd(rows * d_out * elem_size(dt));
    std::unique_ptr<DevBuf> di(inner ? new DevBuf(rows * d_out * elem_size(dt)) : nullptr);
    check(dfx_compose_fwd(ctx, dt, db.p, dl.p, dg.as<float>(), in.s, rows, d_out, dd.p,
                          di ? di->p : nullptr, nullptr));
    download(dd, dt, delta);
    if (inner) download(*di, dt, *inner);
    if (!same) {
        for (double& v : delta.mutable_data()) v = round_to_dtype(v, in.dtype);
        if (inner)
            for (double& v : inner->mutable_data()) v = round_to_dtype(v, in.dtype);
    }
}

TrafficReport fused_report(index_t rows, index_t d_out, index_t tile_rows, int writes,
                           const DTypeSpec& dt) {
    // compose.cpp:99-105 / :143-149
    if (tile_rows < 1) tile_rows = 1;
    const std::uint64_t tiles = rows == 0 ? 0 : (rows + tile_rows - 1) / tile_rows;
    const std::uint64_t act = static_cast<std::uint64_t>(rows) * d_out;
    const std::uint64_t eb = static_cast<std::uint64_t>(dt.storage_bytes);
    TrafficReport t;
    t.activation_reads = 2;
    t.activation_writes = static_cast<std::uint64_t>(writes);
    t.vector_reads = tiles;
    t.bytes_total = (2 + t.activation_writes) * act * eb + tiles * d_out * eb;
    t.pass_count = 1;
    return t;
}

}  // namespace

RealMatrix stable_compose(const ComposeInputs& in) {
    check_compose(in);
    RealMatrix delta(in.base.rows(), in.base.cols(), in.dtype);
    run_compose(in, delta, nullptr);
    return delta;
}

RealMatrix naive_compose(const ComposeInputs& in) {
    // compose.cpp:47-68 — host only: the stability lab's deliberately unstable form.
    check_compose(in);
    const index_t rows = in.base.rows(), d_out = in.base.cols();
    RealMatrix delta(rows, d_out, in.dtype);
    const float sf = static_cast<float>(in.s);
    auto rnd = [&](float x) { return static_cast<float>(round_to_dtype(x, in.dtype)); };
    auto& d = delta.mutable_data();
    for (index_t i = 0; i < rows; ++i)
        for (index_t j = 0; j < d_out; ++j) {
            const float b = static_cast<float>(in.base(i, j));
            const float t1 = rnd(sf * static_cast<float>(in.lora(i, j)));
            const float t2 = rnd(t1 + b);
            const float t3 = rnd(static_cast<float>(in.g[j]) * t2);
            d[i * d_out + j] = round_to_dtype(static_cast<double>(t3 - b), in.dtype);
        }
    return delta;
}

FusedResult fused_compose(const ComposeInputs& in, index_t tile_rows) {
    check_compose(in);
    if (!in.base.contiguous() || !in.lora.contiguous())
        throw std::invalid_argument(
            "fused_compose: inputs must be contiguous (dispatch routes non-contiguous tensors "
            "to the eager path)");
    FusedResult out{RealMatrix(in.base.rows(), in.base.cols(), in.dtype), {}};
    run_compose(in, out.delta, nullptr);
    out.traffic = fused_report(in.base.rows(), in.base.cols(), tile_rows, 1, in.dtype);
    return out;
}

DualResult dual_output_compose(const ComposeInputs& in, bool need_inner, index_t tile_rows) {
    check_compose(in);
    if (!in.base.contiguous() || !in.lora.contiguous())
        throw std::invalid_argument("dual_output_compose: inputs must be contiguous");
    const index_t rows = in.base.rows(), d_out = in.base.cols();
    DualResult out{RealMatrix(rows, d_out, in.dtype), std::nullopt, {}};
    if (need_inner) out.inner.emplace(rows, d_out, in.dtype);
    run_compose(in, out.delta, need_inner ? &*out.inner : nullptr);
    out.traffic = fused_report(rows, d_out, tile_rows, need_inner ? 2 : 1, in.dtype);
    return out;
}

GradBundle compose_backward(const RealMatrix& d_y, const std::vector<double>& g, double s,
                            const RealMatrix* inner, const std::vector<double>& w_norm,
                            bool mag_grad) {
    // compose.cpp:158-169
    const index_t rows = d_y.rows(), d_out = d_y.cols();
    if (g.size() != d_out) throw std::invalid_argument("compose_backward: g length != d_out");
    if (mag_grad) {
        if (inner == nullptr)
            throw std::invalid_argument("compose_backward: magnitude gradient requires inner");
        if (inner->rows() != rows || inner->cols() != d_out)
            throw std::invalid_argument("compose_backward: inner shape mismatch");
        if (w_norm.size() != d_out)
            throw std::invalid_argument("compose_backward: w_norm length != d_out");
    }
    if (d_y.dtype().kind == DTypeKind::FP64)
        throw std::invalid_argument("compose_backward: FP64 is not a B200 storage format");
    dfx_ctx* ctx = device_ctx();
    const dfx_dtype out_dt = to_dfx(d_y.dtype());
    const bool same = !mag_grad || inner->dtype() == d_y.dtype();
    const dfx_dtype dt = same ? out_dt : DFX_F32;
    const DevBuf dy = upload(d_y.data(), dt);
    std::unique_ptr<DevBuf> din;
    if (mag_grad) din = std::make_unique<DevBuf>(upload(inner->data(), dt));
    std::vector<float> gf(d_out), wf(mag_grad ? d_out : 0);
    for (index_t j = 0; j < d_out; ++j) gf[j] = static_cast<float>(g[j]);
    for (index_t j = 0; j < wf.size(); ++j) wf[j] = static_cast<float>(w_norm[j]);
    const DevBuf dg = upload_f32(gf), dw = upload_f32(wf);
    DevBuf dl(rows * d_out * elem_size(dt)), dbb(rows * d_out * elem_size(dt));
    DevBuf dm(d_out * sizeof(float));
    check(dfx_compose_bwd(ctx, dt, dy.p, dg.as<float>(), s, mag_grad ? din->p : nullptr,
                          mag_grad ? dw.as<float>() : nullptr, rows, d_out, dl.p, dbb.p,
                          mag_grad ? dm.as<float>() : nullptr, nullptr));
    GradBundle out{RealMatrix(rows, d_out, d_y.dtype()), RealMatrix(rows, d_out, d_y.dtype()),
                   std::nullopt};
    download(dl, dt, out.d_lora);
    download(dbb, dt, out.d_base);
    if (!same) {
        for (double& v : out.d_lora.mutable_data()) v = round_to_dtype(v, d_y.dtype());
        for (double& v : out.d_base.mutable_data()) v = round_to_dtype(v, d_y.dtype());
    }
    if (mag_grad) {
        const std::vector<float> m = download_f32(dm, d_out);
        out.d_mag = std::vector<double>(m.begin(), m.end());
    }
    return out;
}

TrafficReport eager_traffic_model(index_t rows, index_t d_out, const DTypeSpec& dtype) {
    // compose.cpp:203-217: t1 = s*lora; t2 = g*t1; t3 = (g-1)*base; delta = t3 + t2
    TrafficReport t;
    t.activation_reads = 5;
    t.activation_writes = 4;
    t.vector_reads = 2;
    t.pass_count = static_cast<int>(t.activation_reads + t.activation_writes + t.vector_reads);
    const std::uint64_t act = static_cast<std::uint64_t>(rows) * d_out;
    const std::uint64_t eb = static_cast<std::uint64_t>(dtype.storage_bytes);
    t.bytes_total = (t.activation_reads + t.activation_writes) * act * eb +
                    t.vector_reads * static_cast<std::uint64_t>(d_out) * eb;
    return t;
}

// ================================================================== layer (8f row 2)
// The hot path's production caller on the device: the plain GEMMs run dfx_working_matmul
// (the reference's serial-k fp32 order, bitwise) on device-resident operands addressed
// with strides (no transposed copies), the norm / compose / backward kernels follow, and
// only the results come back.  Operands whose dtype tag differs from the working dtype
// take the same steps through fp32 storage with the working-dtype rounding applied on the
// host, which is where the reference applies it (rounded_to after matmul_f32).
namespace {

// C = a' . b' on the device; strides in elements (see dfx_working_matmul)
DevBuf gemm(dfx_dtype dt, const DevBuf& a, int64_t sa_i, int64_t sa_k, const DevBuf& b,
            int64_t sb_k, int64_t sb_j, index_t M, index_t N, index_t K) {
    DevBuf c(M * N * elem_size(dt));
    check(dfx_working_matmul(device_ctx(), dt, a.p, sa_i, sa_k, b.p, sb_k, sb_j, M, N, K, c.p,
                             nullptr));
    return c;
}

RealMatrix fetch(const DevBuf& d, dfx_dtype dt, index_t rows, index_t cols, const DTypeSpec& tag) {
    RealMatrix m(rows, cols, tag);
    download(d, dt, m);
    return m;
}

void round_all(RealMatrix& m, const DTypeSpec& dt) {
    for (double& v : m.mutable_data()) v = round_to_dtype(v, dt);
}

}  // namespace

ForceMode force_mode_from_name(const std::string& name) {
    if (name == "auto") return ForceMode::Auto;
    if (name == "on" || name == "1") return ForceMode::On;
    if (name == "off" || name == "0") return ForceMode::Off;
    throw std::invalid_argument("unknown force mode: " + name);
}

const char* force_mode_name(ForceMode mode) {
    static const char* const names[] = {"auto", "on", "off"};
    const int i = static_cast<int>(mode);
    return i >= 0 && i < 3 ? names[i] : "?";
}

const char* dispatch_reason_name(DispatchReason r) {
    static const char* const names[] = {"NO_ACCELERATOR", "NO_KERNELS", "FORCED",
                                        "NON_CONTIGUOUS", "SHAPE_GUARD", "BELOW_CROSSOVER",
                                        "ABOVE_CROSSOVER", "INFERENCE", "GRAD_OUTSIDE_TRAINING"};
    const int i = static_cast<int>(r);
    return i >= 0 && i < 9 ? names[i] : "?";
}

bool TierDecision::has_reason(DispatchReason r) const {
    return std::find(reasons.begin(), reasons.end(), r) != reasons.end();
}

TierDecision select_tier(const DispatchContext& c) {
    TierDecision d;
    using R = DispatchReason;
    // hard guards, all recorded (dispatch.cpp:46-57)
    const std::pair<bool, R> guards[] = {
        {!c.accelerator_available, R::NO_ACCELERATOR}, {!c.kernels_available, R::NO_KERNELS},
        {c.force_fused == ForceMode::Off, R::FORCED},  {!c.contiguous, R::NON_CONTIGUOUS},
        {!c.mag_broadcast_last_dim, R::SHAPE_GUARD},   {!c.d_out_divisible_128, R::SHAPE_GUARD}};
    for (const auto& gr : guards)
        if (gr.first) d.reasons.push_back(gr.second);
    if (!d.reasons.empty()) return d;                                   // Eager
    if (!c.requires_grad) {
        d.tier = Tier::FusedForward;
        d.reasons.push_back(R::INFERENCE);
    } else if (!c.training) {
        d.reasons.push_back(R::GRAD_OUTSIDE_TRAINING);                  // Eager
    } else if (c.force_fused_backward != ForceMode::Auto) {
        d.tier = c.force_fused_backward == ForceMode::On ? Tier::FusedBackward : Tier::Eager;
        d.reasons.push_back(R::FORCED);
    } else {
        const bool above = c.d_out >= c.crossover_min_d_out &&
                           std::uint64_t(c.rows) * c.d_out >= c.crossover_min_elems;
        d.tier = above ? Tier::FusedBackward : Tier::Eager;
        d.reasons.push_back(above ? R::ABOVE_CROSSOVER : R::BELOW_CROSSOVER);
    }
    return d;
}

bool shape_guard(index_t activation_last_dim, index_t magnitude_len,
                 const std::vector<index_t>& broadcast_dims) {
    if (magnitude_len != activation_last_dim) return false;
    if (broadcast_dims.empty()) return true;
    if (broadcast_dims.back() != magnitude_len) return false;
    return std::all_of(broadcast_dims.begin(), broadcast_dims.end() - 1,
                       [](index_t v) { return v == 1; });
}

RealMatrix matmul_f32(const RealMatrix& a, const RealMatrix& b) {
    if (a.cols() != b.rows())
        throw std::invalid_argument("matmul_f32: inner dimensions disagree (" +
                                    std::to_string(a.cols()) + " vs " + std::to_string(b.rows()) + ")");
    const index_t m = a.rows(), k = a.cols(), n = b.cols();
    const DevBuf da = upload(a.data(), DFX_F32), db = upload(b.data(), DFX_F32);
    const DevBuf dc = gemm(DFX_F32, da, int64_t(k), 1, db, int64_t(n), 1, m, n, k);
    return fetch(dc, DFX_F32, m, n, DTypeSpec::fp32());
}

DoraLinearState make_layer_state(RealMatrix w, AdapterPair adapter, Magnitude magnitude,
                                 std::optional<std::vector<double>> bias,
                                 const DTypeSpec& working_dtype) {
    const index_t d_out = w.rows(), d_in = w.cols();
    if (adapter.A.cols() != d_in || adapter.B.rows() != d_out ||
        adapter.A.rows() != adapter.B.cols())
        throw std::invalid_argument("layer: adapter shapes inconsistent with W");
    if (magnitude.values.size() != d_out)
        throw std::invalid_argument("layer: magnitude length != d_out");
    if (bias && bias->size() != d_out) throw std::invalid_argument("layer: bias length != d_out");
    DoraLinearState st;
    st.working_dtype = working_dtype;
    magnitude.dtype = working_dtype;
    for (double& v : magnitude.values) v = round_to_dtype(v, working_dtype);
    if (bias)
        for (double& v : *bias) v = round_to_dtype(v, working_dtype);
    st.w = std::move(w);
    st.adapter = std::move(adapter);
    st.magnitude = std::move(magnitude);
    st.bias = std::move(bias);
    st.chunk_plan = plan_chunks(d_out, d_in);
    st.dispatch_cfg.training = true;
    st.dispatch_cfg.requires_grad = true;
    return st;
}

LayerForwardResult layer_forward(const DoraLinearState& st, const RealMatrix& x) {
    if (x.cols() != st.d_in()) throw std::invalid_argument("layer_forward: X.cols != d_in");
    const DTypeSpec& wd = st.working_dtype;
    if (wd.kind == DTypeKind::FP64)
        throw std::invalid_argument("layer_forward: FP64 working dtype is not a B200 storage format");
    const index_t rows = x.rows(), d_in = st.d_in(), d_out = st.d_out(), r = st.adapter.A.rows();
    const AdapterPair& ad = st.adapter;
    dfx_ctx* ctx = device_ctx();
    // native: every operand already carries the working dtype, so the GEMMs store their
    // rounded results directly; otherwise fp32 storage and host-side rounding
    const bool native = x.dtype() == wd && st.w.dtype() == wd && ad.A.dtype() == wd &&
                        ad.B.dtype() == wd;
    const dfx_dtype gt = native ? to_dfx(wd) : DFX_F32;
    const DevBuf dX = upload(x.data(), gt), dW = upload(st.w.data(), gt),
                 dA = upload(ad.A.data(), gt), dB = upload(ad.B.data(), gt);
    const int64_t Ri = int64_t(r), Di = int64_t(d_in);
    DevBuf base = gemm(gt, dX, Di, 1, dW, 1, Di, rows, d_out, d_in);     // X W^T
    DevBuf mid = gemm(gt, dX, Di, 1, dA, 1, Di, rows, r, d_in);          // X A^T
    if (!native) {                      // round the fp32 products to wd, back to wd storage
        RealMatrix m = fetch(mid, gt, rows, r, wd);
        round_all(m, wd);
        mid = upload(m.data(), gt);
    }
    DevBuf lora = gemm(gt, mid, Ri, 1, dB, 1, Ri, rows, d_out, r);       // mid B^T

    LayerSaved sv;
    sv.x = x;
    sv.lora_mid = fetch(mid, gt, rows, r, wd);
    sv.base_out = fetch(base, gt, rows, d_out, wd);
    sv.lora_out = fetch(lora, gt, rows, d_out, wd);
    if (!native) {
        round_all(sv.base_out, wd);
        round_all(sv.lora_out, wd);
    }
    // detached norm, recomputed every call, and g (factored_row_norm + magnitude_scale)
    sv.w_norm = factored_row_norm(st.w, ad, st.chunk_plan);
    sv.g = magnitude_scale(st.magnitude, sv.w_norm, wd);

    DispatchContext dc = st.dispatch_cfg;
    dc.rows = rows;
    dc.d_out = d_out;
    dc.contiguous = true;
    dc.mag_broadcast_last_dim = true;
    dc.d_out_divisible_128 = d_out % 128 == 0;
    sv.decision = select_tier(dc);
    const bool want_inner = dc.training && dc.requires_grad && st.mag_trainable;

    // every tier computes the same canonical compose; the dual kernel provides inner
    const dfx_dtype ct = to_dfx(wd);
    const DevBuf cb = upload(sv.base_out.data(), ct), cl = upload(sv.lora_out.data(), ct);
    std::vector<float> gf(d_out);
    for (index_t j = 0; j < d_out; ++j) gf[j] = static_cast<float>(sv.g[j]);
    const DevBuf dg = upload_f32(gf);
    DevBuf delta(rows * d_out * elem_size(ct));
    std::unique_ptr<DevBuf> inner(want_inner ? new DevBuf(rows * d_out * elem_size(ct)) : nullptr);
    check(dfx_compose_fwd(ctx, ct, cb.p, cl.p, dg.as<float>(), ad.s, rows, d_out, delta.p,
                          inner ? inner->p : nullptr, nullptr));
    const RealMatrix dm = fetch(delta, ct, rows, d_out, wd);
    if (inner) sv.inner = fetch(*inner, ct, rows, d_out, wd);

    // residual, then bias, each an fp32 add stored in the working dtype
    RealMatrix y(rows, d_out, wd);
    std::vector<double>& yv = y.mutable_data();
    const std::vector<double>& bv = sv.base_out.data();
    const std::vector<double>& dv = dm.data();
    for (index_t e = 0; e < rows * d_out; ++e) {
        double v = round_to_dtype(static_cast<double>(static_cast<float>(bv[e]) +
                                                      static_cast<float>(dv[e])), wd);
        if (st.bias)
            v = round_to_dtype(static_cast<double>(static_cast<float>(v) +
                                                   static_cast<float>((*st.bias)[e % d_out])), wd);
        yv[e] = v;
    }
    return LayerForwardResult{std::move(y), std::move(sv)};
}

LayerGrads layer_backward(const DoraLinearState& st, const LayerSaved& sv, const RealMatrix& d_y) {
    const index_t rows = sv.x.rows(), d_out = st.d_out(), d_in = st.d_in(), r = st.adapter.A.rows();
    if (d_y.rows() != rows || d_y.cols() != d_out)
        throw std::invalid_argument("layer_backward: dY shape mismatch");
    const bool mag_grad = st.mag_trainable;
    if (mag_grad && !sv.inner)
        throw std::invalid_argument("layer_backward: saved bundle lacks inner for magnitude grad");
    const DTypeSpec& wd = st.working_dtype;
    GradBundle gb = compose_backward(d_y, sv.g, st.adapter.s, sv.inner ? &*sv.inner : nullptr,
                                     sv.w_norm, mag_grad);
    // dB = d_lora^T mid, d_mid = d_lora B, dA = d_mid^T X: strided operands, no transposes
    const bool native = gb.d_lora.dtype() == wd && sv.lora_mid.dtype() == wd &&
                        st.adapter.B.dtype() == wd && sv.x.dtype() == wd;
    const dfx_dtype gt = native ? to_dfx(wd) : DFX_F32;
    const DevBuf dl = upload(gb.d_lora.data(), gt), mid = upload(sv.lora_mid.data(), gt),
                 dB = upload(st.adapter.B.data(), gt), dX = upload(sv.x.data(), gt);
    const int64_t Ri = int64_t(r), Oi = int64_t(d_out), Di = int64_t(d_in);
    const DevBuf db = gemm(gt, dl, 1, Oi, mid, Ri, 1, d_out, r, rows);
    DevBuf dmid = gemm(gt, dl, Oi, 1, dB, Ri, 1, rows, r, d_out);
    if (!native) {
        RealMatrix m = fetch(dmid, gt, rows, r, wd);
        round_all(m, wd);
        dmid = upload(m.data(), gt);
    }
    const DevBuf da = gemm(gt, dmid, 1, Ri, dX, Di, 1, r, d_in, rows);
    LayerGrads out{fetch(da, gt, r, d_in, wd), fetch(db, gt, d_out, r, wd), std::move(gb.d_mag)};
    if (!native) {
        round_all(out.d_a, wd);
        round_all(out.d_b, wd);
    }
    return out;
}

}  // namespace dorafactor
