// dfx_capi.cu — the C ABI (include/dfx.h): context, validation, orchestration.
//
// Validation mirrors the reference's throw sites so the C++ drop-in can map
// DFX_EINVAL back to std::invalid_argument one-for-one:
//   factored_norm.cpp:11-23 (shapes, rank, plan), :28-30 (FP64 weights)
//   factored_norm.cpp:124-126 (assemble length), :221-223 (magnitude length)
//   compose.cpp:9-16 (base/lora/g shapes), :72-75 (contiguity, host side),
//   compose.cpp:158-169 (backward: g length, inner required/shape, w_norm length)
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>
#include <algorithm>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/dfx.h"
#include "kernels/launch.h"

namespace dfx {

struct Workspace {
    int device = 0;
    int sms = 0;
    int sm_budget = 0;      // dfx_ctx_set_sm_budget: cap on the SMs the norm's GEMMs plan for
    cudaStream_t cur = nullptr;     // the calling entry point's stream (capture check)
    bool grow_in_capture = false;   // a call needed to grow the workspace during capture
    std::vector<void*> ptr;
    std::vector<size_t> cap;
    std::vector<void*> retired;     // outgrown buffers: freed at dfx_ctx_destroy only
    cudaStream_t side = nullptr;
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
    Workspace() : ptr(16, nullptr), cap(16, 0) {}
    ~Workspace() {
        for (void* p : ptr)
            if (p) cudaFree(p);
        for (void* p : retired) cudaFree(p);
        for (cudaEvent_t e : ev)
            if (e) cudaEventDestroy(e);
        if (side) cudaStreamDestroy(side);
    }
};

cudaStream_t ws_side_stream(Workspace* ws, cudaError_t* err) {
    *err = cudaSuccess;
    if (!ws->side) *err = cudaStreamCreateWithFlags(&ws->side, cudaStreamNonBlocking);
    return ws->side;
}

cudaEvent_t ws_event(Workspace* ws, int idx, cudaError_t* err) {
    if (!ws->ev[idx]) {
        const cudaError_t e = cudaEventCreateWithFlags(&ws->ev[idx], cudaEventDisableTiming);
        if (e != cudaSuccess) *err = e;
    }
    return ws->ev[idx];
}

int device_sm_count() {
    static int cache[64] = {0};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
    if (!cache[dev]) {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        cache[dev] = v > 0 ? v : 148;
    }
    return cache[dev];
}

int device_smem_optin() {
    static int cache[64] = {0};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 227 * 1024;
    if (!cache[dev]) {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        cache[dev] = v > 0 ? v : 227 * 1024;
    }
    return cache[dev];
}

int ws_sm_count(Workspace* ws) {
    if (!ws->sms) cudaDeviceGetAttribute(&ws->sms, cudaDevAttrMultiProcessorCount, ws->device);
    const int n = ws->sms > 0 ? ws->sms : 148;
    return ws->sm_budget > 0 ? std::min(n, std::max(ws->sm_budget, 4)) : n;
}

// Grow-only workspace slots.  Growth never synchronises and never frees: the outgrown buffer
// may still be read by queued work on any stream or be baked into a CUDA graph captured
// earlier, so it is retired and freed only by dfx_ctx_destroy.  Growth is refused (the call
// fails with DFX_EUNSUPPORTED) while the calling stream is capturing a graph: run the call
// once eagerly at the largest shape first.
void* ws_get(Workspace* ws, int slot, size_t bytes, cudaError_t* err) {
    *err = cudaSuccess;
    if (bytes == 0) bytes = 16;
    if (ws->cap[slot] >= bytes) return ws->ptr[slot];
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(ws->cur, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
        cudaGetLastError();
        ws->grow_in_capture = true;
        *err = cudaErrorStreamCaptureUnsupported;
        return nullptr;
    }
    const size_t want = bytes + bytes / 4;
    void* p = nullptr;
    *err = cudaMalloc(&p, want);
    if (*err != cudaSuccess) return nullptr;
    if (ws->ptr[slot]) ws->retired.push_back(ws->ptr[slot]);
    ws->ptr[slot] = p;
    ws->cap[slot] = want;
    return p;
}

void* ws_get_zeroed(Workspace* ws, int slot, size_t bytes, cudaError_t* err) {
    const bool fresh = ws->cap[slot] < (bytes ? bytes : 16);
    void* p = ws_get(ws, slot, bytes, err);
    if (*err == cudaSuccess && fresh) *err = cudaMemsetAsync(p, 0, ws->cap[slot], ws->cur);
    return p;
}

namespace {
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeFn encode_fn() {
    static EncodeFn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return static_cast<EncodeFn>(nullptr);
        return reinterpret_cast<EncodeFn>(p);
    }();
    return fn;
}
}  // namespace

cudaError_t ensure_max_dyn_smem(const void* func, int bytes) {
    static std::mutex mu;
    static std::vector<std::pair<std::pair<const void*, int>, int>> done;   // (func, dev) -> bytes
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lk(mu);
    for (auto& d : done)
        if (d.first.first == func && d.first.second == dev && d.second >= bytes) return cudaSuccess;
    e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) done.push_back({{func, dev}, bytes});
    return e;
}

cudaError_t make_tmap_2d(CUtensorMap* out, int dt, const void* base, uint64_t rows, uint64_t cols,
                         uint64_t row_pitch_bytes, uint32_t box_cols, uint32_t box_rows,
                         bool swizzle128) {
    return make_tmap_2d_sw(out, dt, base, rows, cols, row_pitch_bytes, box_cols, box_rows,
                           swizzle128 ? 128 : 0);
}

cudaError_t make_tmap_2d_sw(CUtensorMap* out, int dt, const void* base, uint64_t rows,
                            uint64_t cols, uint64_t row_pitch_bytes, uint32_t box_cols,
                            uint32_t box_rows, int swizzle_bytes) {
    EncodeFn fn = encode_fn();
    if (!fn) return cudaErrorNotSupported;
    const CUtensorMapDataType t = dt == kF32    ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                  : dt == kBF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                                : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
    const cuuint64_t dims[2] = {cols, rows};
    const cuuint64_t strides[1] = {row_pitch_bytes};
    const cuuint32_t box[2] = {box_cols, box_rows};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = fn(out, t, 2, const_cast<void*>(base), dims, strides, box, estr,
                          CU_TENSOR_MAP_INTERLEAVE_NONE,
                          swizzle_bytes == 128  ? CU_TENSOR_MAP_SWIZZLE_128B
                          : swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                          : swizzle_bytes == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                                : CU_TENSOR_MAP_SWIZZLE_NONE,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

// A row-major [rows x cols] matrix viewed as [cols/64 atoms][rows][64]: box {64, box_rows, atoms}
// lands `atoms` consecutive 64-wide K blocks as separate 128B-swizzled [box_rows][64] tiles
// (the UMMA K-major layout of each atom), in one TMA instruction.  cols % 64 == 0.
cudaError_t make_tmap_3d_katoms(CUtensorMap* out, int dt, const void* base, uint64_t rows,
                                uint64_t cols, uint64_t row_pitch_bytes, uint32_t box_rows,
                                uint32_t atoms) {
    EncodeFn fn = encode_fn();
    if (!fn) return cudaErrorNotSupported;
    if (cols % 64 != 0 || dt == kF32) return cudaErrorInvalidValue;
    const CUtensorMapDataType t = dt == kBF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                              : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
    const cuuint64_t dims[3] = {64, rows, cols / 64};
    const cuuint64_t strides[2] = {row_pitch_bytes, 128};
    const cuuint32_t box[3] = {64, box_rows, atoms};
    const cuuint32_t estr[3] = {1, 1, 1};
    const CUresult r = fn(out, t, 3, const_cast<void*>(base), dims, strides, box, estr,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

// ----------------------------------------------------------------- profiling
struct Profiler {
    struct Rec {
        const char* name;
        cudaEvent_t a, b;
    };
    std::vector<Rec> recs;
    std::vector<cudaEvent_t> pool;
    const char* open_name = nullptr;
    cudaEvent_t open_ev = nullptr;
    cudaEvent_t take() {
        cudaEvent_t e;
        if (!pool.empty()) {
            e = pool.back();
            pool.pop_back();
        } else {
            cudaEventCreate(&e);
        }
        return e;
    }
    ~Profiler() {
        for (auto& r : recs) {
            cudaEventDestroy(r.a);
            cudaEventDestroy(r.b);
        }
        for (auto e : pool) cudaEventDestroy(e);
    }
};

thread_local Profiler* g_prof = nullptr;

void prof_begin(const char* name, cudaStream_t st) {
    if (!g_prof) return;
    g_prof->open_name = name;
    g_prof->open_ev = g_prof->take();
    cudaEventRecord(g_prof->open_ev, st);
}

void prof_end(cudaStream_t st) {
    if (!g_prof || !g_prof->open_ev) return;
    cudaEvent_t b = g_prof->take();
    cudaEventRecord(b, st);
    g_prof->recs.push_back({g_prof->open_name, g_prof->open_ev, b});
    g_prof->open_ev = nullptr;
}

}  // namespace dfx

struct dfx_ctx {
    int device = 0;
    dfx::Workspace ws;
    int64_t launches = 0;
    bool profiling = false;
    dfx::Profiler prof;
    // module_fwd_host staging
    cudaStream_t st_h2d = nullptr, st_comp = nullptr, st_d2h = nullptr;
    std::vector<void*> stage;
    std::vector<size_t> stage_cap;
    std::vector<void*> stage_retired;
};

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    std::vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

int cuda_fail(cudaError_t e, const char* where) {
    return fail(DFX_ECUDA, "%s: %s", where, cudaGetErrorString(e));
}

bool valid_dtype(int dt) { return dt == DFX_F32 || dt == DFX_BF16 || dt == DFX_F16; }

// Restores the caller's current device when an entry point returns (the host framework's
// device state is not ours to change).
struct DeviceGuard {
    int prev = -1;
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

// Binds the calling thread to the context's device (restored by `dg` on return), records the
// call's stream for the workspace's capture check, checks that the stream belongs to the
// context's device, and attaches the context's profiler if enabled.
int enter(dfx_ctx* ctx, DeviceGuard& dg, cudaStream_t st = nullptr) {
    if (!ctx) return fail(DFX_EINVAL, "null context");
    int cur = -1;
    cudaError_t e = cudaGetDevice(&cur);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    if (cur != ctx->device) {
        e = cudaSetDevice(ctx->device);
        if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
        dg.prev = cur;
    }
#if CUDART_VERSION >= 12080
    // (outside graph capture only: the query is not a capturable call)
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (st && cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs == cudaStreamCaptureStatusNone) {
        int sdev = -1;
        if (cudaStreamGetDevice(st, &sdev) == cudaSuccess && sdev != ctx->device)
            return fail(DFX_EINVAL, "stream belongs to device %d, context to device %d", sdev,
                        ctx->device);
        cudaGetLastError();
    }
#endif
    ctx->ws.cur = st;
    ctx->ws.grow_in_capture = false;
    dfx::g_prof = ctx->profiling ? &ctx->prof : nullptr;
    return DFX_OK;
}

int finish_call(dfx_ctx* ctx, cudaError_t e, const char* where) {
    if (e != cudaSuccess && ctx && ctx->ws.grow_in_capture) {
        cudaGetLastError();
        return fail(DFX_EUNSUPPORTED,
                    "%s: the workspace must grow for this shape/plan but the stream is capturing "
                    "a graph; call once eagerly first", where);
    }
    if (e != cudaSuccess) return cuda_fail(e, where);
    g_err.clear();
    return DFX_OK;
}

}  // namespace

extern "C" {

int dfx_abi_version(void) { return DFX_ABI_VERSION; }

const char* dfx_last_error(void) { return g_err.c_str(); }

int dfx_ctx_create(int device, dfx_ctx** out) {
    if (!out) return fail(DFX_EINVAL, "dfx_ctx_create: null out");
    *out = nullptr;
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0)
        return fail(DFX_ENODEV, "dfx_ctx_create: no CUDA device (%s)",
                    e == cudaSuccess ? "count 0" : cudaGetErrorString(e));
    if (device < 0 || device >= n) return fail(DFX_EINVAL, "dfx_ctx_create: bad device %d", device);
    cudaDeviceProp prop;
    e = cudaGetDeviceProperties(&prop, device);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceProperties");
    if (prop.major != 10 || prop.minor != 0)
        return fail(DFX_ENODEV, "dfx: built for sm_100a, device %d is sm_%d%d", device, prop.major,
                    prop.minor);
    dfx_ctx* c = new dfx_ctx();
    c->device = device;
    c->ws.device = device;
    c->stage.assign(16, nullptr);
    c->stage_cap.assign(16, 0);
    *out = c;
    g_err.clear();
    return DFX_OK;
}

void dfx_ctx_destroy(dfx_ctx* ctx) {
    if (!ctx) return;
    DeviceGuard dg;
    int cur = -1;
    if (cudaGetDevice(&cur) == cudaSuccess && cur != ctx->device) {
        cudaSetDevice(ctx->device);
        dg.prev = cur;
    }
    cudaDeviceSynchronize();
    for (void* p : ctx->stage)
        if (p) cudaFree(p);
    for (void* p : ctx->stage_retired) cudaFree(p);
    if (ctx->st_h2d) cudaStreamDestroy(ctx->st_h2d);
    if (ctx->st_comp) cudaStreamDestroy(ctx->st_comp);
    if (ctx->st_d2h) cudaStreamDestroy(ctx->st_d2h);
    delete ctx;
}

int64_t dfx_ctx_launches(const dfx_ctx* ctx) { return ctx ? ctx->launches : 0; }

int dfx_profile_enable(dfx_ctx* ctx, int on) {
    if (!ctx) return fail(DFX_EINVAL, "null context");
    ctx->profiling = on != 0;
    if (!ctx->profiling) dfx::g_prof = nullptr;
    g_err.clear();
    return DFX_OK;
}

int dfx_profile_report(dfx_ctx* ctx, char* buf, size_t len) {
    DeviceGuard dg;
    int rc = enter(ctx, dg);
    if (rc) return rc;
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return cuda_fail(e, "dfx_profile_report");
    struct Agg {
        std::string name;
        long n = 0;
        double tot = 0, mn = 1e30, mx = 0;
    };
    std::vector<Agg> agg;
    dfx::Profiler& P = ctx->prof;
    for (auto& r : P.recs) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, r.a, r.b);
        Agg* a = nullptr;
        for (auto& x : agg)
            if (x.name == r.name) a = &x;
        if (!a) {
            agg.push_back(Agg{r.name});
            a = &agg.back();
        }
        ++a->n;
        a->tot += ms;
        a->mn = std::min<double>(a->mn, ms);
        a->mx = std::max<double>(a->mx, ms);
        P.pool.push_back(r.a);
        P.pool.push_back(r.b);
    }
    P.recs.clear();
    std::string out;
    for (auto& a : agg) {
        char line[256];
        std::snprintf(line, sizeof(line), "%s %ld %.6f %.6f %.6f\n", a.name.c_str(), a.n, a.tot,
                      a.mn, a.mx);
        out += line;
    }
    if (buf && len) {
        std::snprintf(buf, len, "%s", out.c_str());
        if (out.size() + 1 > len) return fail(DFX_EINVAL, "dfx_profile_report: buffer too small");
    }
    g_err.clear();
    return DFX_OK;
}

int dfx_plan_chunks(uint64_t d_out, uint64_t d_in, uint64_t budget, uint64_t* chunk_size,
                    uint64_t* num_chunks) {
    // matrix.cpp:28-51
    if (d_out < 1 || d_in < 1) return fail(DFX_EINVAL, "plan_chunks: dims must be >= 1");
    if (budget < 256) return fail(DFX_EINVAL, "plan_chunks: budget below 256 bytes");
    const uint64_t align = 64;
    const uint64_t fit = budget / (d_out * 4);
    if (d_in >= align && fit < align)
        return fail(DFX_EINVAL,
                    "plan_chunks: budget of %llu bytes cannot hold one 64-wide fp32 chunk at "
                    "d_out=%llu",
                    (unsigned long long)budget, (unsigned long long)d_out);
    uint64_t cs = d_in < fit ? d_in : fit;
    cs = (cs / align) * align;
    const uint64_t floor_cs = d_in < align ? d_in : align;
    if (cs < floor_cs) cs = floor_cs;
    if (chunk_size) *chunk_size = cs;
    if (num_chunks) *num_chunks = (d_in + cs - 1) / cs;
    g_err.clear();
    return DFX_OK;
}

int dfx_norm_plan(dfx_ctx* ctx, dfx_dtype dtype, int64_t d_out, int64_t d_in, int64_t r,
                  int64_t chunk_size, int* u_sms, int* side_sms, int* strategy) {
    DeviceGuard dg;
    int rc = enter(ctx, dg);
    if (rc) return rc;
    if ((dtype != DFX_BF16 && dtype != DFX_F16) || chunk_size <= 0 || chunk_size % 64 != 0 ||
        !dfx::norm_uses_tensor_cores(dtype, d_out, d_in, r))
        return fail(DFX_EUNSUPPORTED, "dfx_norm_plan: not the bf16 / fp16 tensor-core path");
    dfx::norm_plan_info(d_out, d_in, r, chunk_size, dfx::ws_sm_count(&ctx->ws), u_sms, side_sms,
                        strategy);
    return DFX_OK;
}

int dfx_norm_uses_tensor_cores(dfx_dtype dtype, int64_t d_out, int64_t d_in, int64_t r) {
    return dfx::norm_uses_tensor_cores(dtype, d_out, d_in, r);
}

static int check_norm_args(dfx_dtype dtype, const void* W, const void* A, const void* B,
                           int64_t d_out, int64_t d_in, int64_t r, int64_t chunk_size) {
    if (!valid_dtype(dtype))
        return fail(DFX_EINVAL,
                    "factored_norm_terms: fp32 term accumulation requires non-FP64 weights");
    if (d_out < 0 || d_in < 0) return fail(DFX_EINVAL, "factored_norm: negative dims");
    if (r < 1) return fail(DFX_EINVAL, "factored_norm: rank must be >= 1");
    if (chunk_size < 1) return fail(DFX_EINVAL, "factored_norm: chunk plan does not match W.cols");
    if (d_out > 0 && d_in > 0 && (!W || !A || !B))
        return fail(DFX_EINVAL, "factored_norm: null operand");
    return DFX_OK;
}

static int run_norm(dfx_ctx* ctx, dfx_dtype dtype, const void* W, const void* A, const void* B,
                    int64_t d_out, int64_t d_in, int64_t r, double s, int64_t chunk_size,
                    float* base_sq, float* cross, float* ba_sq, const float* m,
                    dfx_dtype mag_dtype, float* w_norm, float* g, int round_dt,
                    cudaStream_t st, const char* where) {
    dfx::NormArgs a{};
    a.dt = dtype; a.w = W; a.a = A; a.b = B;
    a.d_out = d_out; a.d_in = d_in; a.r = r; a.s = s; a.chunk_size = chunk_size;
    a.base_sq = base_sq; a.cross = cross; a.ba_sq = ba_sq;
    a.m = m; a.w_norm = w_norm; a.g = g;
    a.round_dt = round_dt; a.mag_dt = mag_dtype;
    int launches = 0;
    const cudaError_t e = dfx::launch_norm(a, &ctx->ws, st, &launches);
    ctx->launches += launches;
    return finish_call(ctx, e, where);
}

int dfx_norm_terms(dfx_ctx* ctx, dfx_dtype dtype, const void* W, const void* A, const void* B,
                   int64_t d_out, int64_t d_in, int64_t r, double s, int64_t chunk_size,
                   float* base_sq, float* cross, float* ba_sq, dfx_stream_t stream) {
    DeviceGuard dg;
    int rc = enter(ctx, dg, stream);
    if (rc) return rc;
    rc = check_norm_args(dtype, W, A, B, d_out, d_in, r, chunk_size);
    if (rc) return rc;
    return run_norm(ctx, dtype, W, A, B, d_out, d_in, r, s, chunk_size, base_sq, cross, ba_sq,
                    nullptr, DFX_F32, nullptr, nullptr, dfx::kF32, stream, "dfx_norm_terms");
}

int dfx_row_norm(dfx_ctx* ctx, dfx_dtype dtype, const void* W, const void* A, const void* B,
                 int64_t d_out, int64_t d_in, int64_t r, double s, int64_t chunk_size,
                 const float* m, dfx_dtype mag_dtype, float* w_norm, float* g, float* terms,
                 dfx_stream_t stream) {
    DeviceGuard dg;
    int rc = enter(ctx, dg, stream);
    if (rc) return rc;
    rc = check_norm_args(dtype, W, A, B, d_out, d_in, r, chunk_size);
    if (rc) return rc;
    if (m && !valid_dtype(mag_dtype)) return fail(DFX_EUNSUPPORTED, "dfx_row_norm: mag dtype");
    if (m && !g) return fail(DFX_EINVAL, "dfx_row_norm: m given without g output");
    float* bs = terms ? terms : nullptr;
    float* cr = terms ? terms + d_out : nullptr;
    float* bq = terms ? terms + 2 * d_out : nullptr;
    return run_norm(ctx, dtype, W, A, B, d_out, d_in, r, s, chunk_size, bs, cr, bq, m, mag_dtype,
                    w_norm, g, dtype, stream, "dfx_row_norm");
}

int dfx_row_norm_cached(dfx_ctx* ctx, dfx_dtype dtype, const void* W, const void* A,
                        const void* B, int64_t d_out, int64_t d_in, int64_t r, double s,
                        int64_t chunk_size, float* base_sq_cache, int refresh, const float* m,
                        dfx_dtype mag_dtype, float* w_norm, float* g, dfx_stream_t stream) {
    DeviceGuard dg;
    int rc = enter(ctx, dg, stream);
    if (rc) return rc;
    rc = check_norm_args(dtype, W, A, B, d_out, d_in, r, chunk_size);
    if (rc) return rc;
    if (!base_sq_cache && d_out > 0) return fail(DFX_EINVAL, "dfx_row_norm_cached: null cache");
    if (m && !valid_dtype(mag_dtype)) return fail(DFX_EUNSUPPORTED, "dfx_row_norm_cached: mag dtype");
    if (m && !g) return fail(DFX_EINVAL, "dfx_row_norm_cached: m given without g output");
    if (dtype == DFX_F32 || s == 0.0 || chunk_size % 64 != 0 ||
        !dfx::norm_uses_tensor_cores(dtype, d_out, d_in, r))
        return fail(DFX_EUNSUPPORTED, "dfx_row_norm_cached: needs the bf16 tensor-core path");
    if (refresh)
        return run_norm(ctx, dtype, W, A, B, d_out, d_in, r, s, chunk_size, base_sq_cache, nullptr,
                        nullptr, m, mag_dtype, w_norm, g, dtype, stream, "dfx_row_norm_cached");
    dfx::NormArgs a{};
    a.dt = dtype; a.w = W; a.a = A; a.b = B;
    a.d_out = d_out; a.d_in = d_in; a.r = r; a.s = s; a.chunk_size = chunk_size;
    a.m = m; a.w_norm = w_norm; a.g = g;
    a.round_dt = dtype; a.mag_dt = mag_dtype;
    a.base_cached = base_sq_cache;
    int launches = 0;
    const cudaError_t e = dfx::launch_norm(a, &ctx->ws, stream, &launches);
    ctx->launches += launches;
    return finish_call(ctx, e, "dfx_row_norm_cached");
}

int dfx_norm_adapter(dfx_ctx* ctx, dfx_dtype dtype, const void* A, const void* B,
                     int64_t d_out, int64_t d_in, int64_t r, int sms, float* ba_sq,
                     dfx_stream_t stream) {
    DeviceGuard dg;
    int rc = enter(ctx, dg, stream);
    if (rc) return rc;
    if (d_out < 0 || d_in < 0 || r < 1) return fail(DFX_EINVAL, "dfx_norm_adapter: bad dims");
    if (!A || !B || (!ba_sq && d_out > 0)) return fail(DFX_EINVAL, "dfx_norm_adapter: null operand");
    if ((dtype != DFX_BF16 && dtype != DFX_F16) || !dfx::norm_uses_tensor_cores(dtype, d_out, d_in, r))
        return fail(DFX_EUNSUPPORTED, "dfx_norm_adapter: needs the bf16 / fp16 tensor-core path");
    dfx::NormArgs a{};
    a.dt = dtype; a.a = A; a.b = B;
    a.d_out = d_out; a.d_in = d_in; a.r = r; a.s = 1.0; a.chunk_size = 64;
    a.ba_sq = ba_sq; a.mode = dfx::kNormAdapter;
    if (sms < 0) return fail(DFX_EINVAL, "dfx_norm_adapter: negative SM cap");
    // plan the Gram and V for at most `sms` SMs (the call runs beside other work)
    const int saved = ctx->ws.sm_budget;
    if (sms > 0) ctx->ws.sm_budget = saved > 0 ? std::min(saved, sms) : sms;
    int launches = 0;
    const cudaError_t e = dfx::launch_norm(a, &ctx->ws, stream, &launches);
    ctx->ws.sm_budget = saved;
    ctx->launches += launches;
    return finish_call(ctx, e, "dfx_norm_adapter");
}

int dfx_row_norm_ba(dfx_ctx* ctx, dfx_dtype dtype, const void* W, const void* A, const void* B,
                    int64_t d_out, int64_t d_in, int64_t r, double s, int64_t chunk_size,
                    const float* ba_sq, const float* m, dfx_dtype mag_dtype, float* w_norm,
                    float* g, float* terms, dfx_stream_t stream) {
    DeviceGuard dg;
    int rc = enter(ctx, dg, stream);
    if (rc) return rc;
    rc = check_norm_args(dtype, W, A, B, d_out, d_in, r, chunk_size);
    if (rc) return rc;
    if (!ba_sq && d_out > 0) return fail(DFX_EINVAL, "dfx_row_norm_ba: null ba_sq");
    if (m && !valid_dtype(mag_dtype)) return fail(DFX_EUNSUPPORTED, "dfx_row_norm_ba: mag dtype");
    if (m && !g) return fail(DFX_EINVAL, "dfx_row_norm_ba: m given without g output");
    if ((dtype != DFX_BF16 && dtype != DFX_F16) || s == 0.0 || chunk_size % 64 != 0 ||
        !dfx::norm_uses_tensor_cores(dtype, d_out, d_in, r))
        return fail(DFX_EUNSUPPORTED, "dfx_row_norm_ba: needs the bf16 / fp16 tensor-core path");
    dfx::NormArgs a{};
    a.dt = dtype; a.w = W; a.a = A; a.b = B;
    a.d_out = d_out; a.d_in = d_in; a.r = r; a.s = s; a.chunk_size = chunk_size;
    if (terms) { a.base_sq = terms; a.cross = terms + d_out; a.ba_sq = terms + 2 * d_out; }
    a.m = m; a.w_norm = w_norm; a.g = g;
    a.round_dt = dtype; a.mag_dt = mag_dtype;
    a.ba_given = ba_sq;
    int launches = 0;
    const cudaError_t e = dfx::launch_norm(a, &ctx->ws, stream, &launches);
    ctx->launches += launches;
    return finish_call(ctx, e, "dfx_row_norm_ba");
}

int dfx_norm_partial(dfx_ctx* ctx, dfx_dtype dtype, const void* W_k, const void* A_k,
                     const void* B, int64_t d_out, int64_t d_in_k, int64_t r, int64_t chunk_size,
                     float* gram, float* base_sq, float* cross, dfx_stream_t stream) {
    DeviceGuard dg;
    int rc = enter(ctx, dg, stream);
    if (rc) return rc;
    rc = check_norm_args(dtype, W_k, A_k, B, d_out, d_in_k, r, chunk_size);
    if (rc) return rc;
    if (!gram || (d_out > 0 && (!base_sq || !cross)))
        return fail(DFX_EINVAL, "dfx_norm_partial: null output");
    dfx::NormArgs a{};
    a.dt = dtype; a.w = W_k; a.a = A_k; a.b = B;
    a.d_out = d_out; a.d_in = d_in_k; a.r = r; a.s = 1.0; a.chunk_size = chunk_size;
    a.base_sq = base_sq; a.cross = cross;
    a.round_dt = dtype; a.mag_dt = dtype;
    a.mode = dfx::kNormPartial; a.gram_out = gram;
    int launches = 0;
    const cudaError_t e = dfx::launch_norm(a, &ctx->ws, stream, &launches);
    ctx->launches += launches;
    return finish_call(ctx, e, "dfx_norm_partial");
}

int dfx_norm_finish(dfx_ctx* ctx, dfx_dtype dtype, const void* B, const float* gram,
                    const float* base_sq, const float* cross, int64_t d_out, int64_t r, double s,
                    const float* m, dfx_dtype mag_dtype, float* w_norm, float* g, float* terms,
                    dfx_stream_t stream) {
    DeviceGuard dg;
    int rc = enter(ctx, dg, stream);
    if (rc) return rc;
    if (!valid_dtype(dtype)) return fail(DFX_EINVAL, "dfx_norm_finish: dtype");
    if (d_out < 0 || r < 1) return fail(DFX_EINVAL, "factored_norm: rank must be >= 1");
    if (d_out > 0 && (!B || !gram || !base_sq || !cross))
        return fail(DFX_EINVAL, "dfx_norm_finish: null operand");
    if (m && (!g || !valid_dtype(mag_dtype))) return fail(DFX_EINVAL, "dfx_norm_finish: m without g");
    dfx::NormArgs a{};
    a.dt = dtype; a.b = B; a.d_out = d_out; a.d_in = 0; a.r = r; a.s = s; a.chunk_size = 64;
    a.base_sq = terms ? terms : nullptr;
    a.cross = terms ? terms + d_out : nullptr;
    a.ba_sq = terms ? terms + 2 * d_out : nullptr;
    a.m = m; a.w_norm = w_norm; a.g = g;
    a.round_dt = dtype; a.mag_dt = mag_dtype;
    a.mode = dfx::kNormFinish; a.gram_in = gram; a.base_in = base_sq; a.cross_in = cross;
    int launches = 0;
    const cudaError_t e = dfx::launch_norm(a, &ctx->ws, stream, &launches);
    ctx->launches += launches;
    return finish_call(ctx, e, "dfx_norm_finish");
}

int dfx_assemble_norm(dfx_ctx* ctx, const float* base_sq, const float* cross,
                      const float* ba_sq, double two_s, double s2, int64_t n,
                      dfx_dtype round_to, float* w_norm, dfx_stream_t stream) {
    DeviceGuard dg;
    int rc = enter(ctx, dg, stream);
    if (rc) return rc;
    if (n < 0) return fail(DFX_EINVAL, "assemble_norm: term vectors differ in length");
    if (!valid_dtype(round_to)) return fail(DFX_EUNSUPPORTED, "assemble_norm: dtype");
    if (n > 0 && (!base_sq || !cross || !ba_sq || !w_norm))
        return fail(DFX_EINVAL, "assemble_norm: null vector");
    int launches = 0;
    const cudaError_t e = dfx::launch_assemble(base_sq, cross, ba_sq, two_s, s2, n, round_to,
                                               w_norm, stream, &launches);
    ctx->launches += launches;
    return finish_call(ctx, e, "dfx_assemble_norm");
}

int dfx_magnitude_scale(dfx_ctx* ctx, dfx_dtype dtype, const float* m, const float* w_norm,
                        int64_t n, float* g, dfx_stream_t stream) {
    DeviceGuard dg;
    int rc = enter(ctx, dg, stream);
    if (rc) return rc;
    if (!valid_dtype(dtype)) return fail(DFX_EUNSUPPORTED, "magnitude_scale: fp64 is host-only");
    if (n < 0) return fail(DFX_EINVAL, "magnitude_scale: length mismatch");
    if (n > 0 && (!m || !w_norm || !g)) return fail(DFX_EINVAL, "magnitude_scale: null vector");
    int launches = 0;
    const cudaError_t e = dfx::launch_magnitude_scale(dtype, m, w_norm, n, g, stream, &launches);
    ctx->launches += launches;
    return finish_call(ctx, e, "dfx_magnitude_scale");
}

int dfx_compose_fwd(dfx_ctx* ctx, dfx_dtype dtype, const void* base, const void* lora,
                    const float* g, double s, int64_t rows, int64_t d_out, void* delta,
                    void* inner, dfx_stream_t stream) {
    DeviceGuard dg;
    int rc = enter(ctx, dg, stream);
    if (rc) return rc;
    if (!valid_dtype(dtype)) return fail(DFX_EUNSUPPORTED, "compose: dtype");
    if (rows < 0 || d_out < 0) return fail(DFX_EINVAL, "compose: base/lora shapes differ");
    if (rows > 0 && d_out > 0 && (!base || !lora || !g || !delta))
        return fail(DFX_EINVAL, "compose: null operand");
    int launches = 0;
    const cudaError_t e =
        dfx::launch_compose_fwd(dtype, base, lora, g, static_cast<float>(s), rows, d_out, delta,
                                inner, stream, &launches);
    ctx->launches += launches;
    return finish_call(ctx, e, "dfx_compose_fwd");
}

int dfx_compose_bwd(dfx_ctx* ctx, dfx_dtype dtype, const void* dy, const float* g, double s,
                    const void* inner, const float* w_norm, int64_t rows, int64_t d_out,
                    void* d_lora, void* d_base, float* d_mag, dfx_stream_t stream) {
    DeviceGuard dg;
    int rc = enter(ctx, dg, stream);
    if (rc) return rc;
    if (!valid_dtype(dtype)) return fail(DFX_EUNSUPPORTED, "compose_backward: dtype");
    if (rows < 0 || d_out < 0) return fail(DFX_EINVAL, "compose_backward: g length != d_out");
    // an empty inner (rows == 0) may legitimately have a null data pointer
    if (d_mag && !inner && rows > 0)
        return fail(DFX_EINVAL, "compose_backward: magnitude gradient requires inner");
    if (d_mag && !w_norm) return fail(DFX_EINVAL, "compose_backward: w_norm length != d_out");
    // d_lora and d_base may both be null when d_mag is requested: magnitude gradient only
    const bool mag_only = d_mag && !d_lora && !d_base;
    if (rows > 0 && d_out > 0 && (!dy || !g || (!mag_only && (!d_lora || !d_base))))
        return fail(DFX_EINVAL, "compose_backward: null operand");
    int launches = 0;
    const cudaError_t e =
        dfx::launch_compose_bwd(dtype, dy, g, static_cast<float>(s), inner, w_norm, rows, d_out,
                                d_lora, d_base, d_mag, stream, &launches, ctx->ws.sm_budget > 0);
    ctx->launches += launches;
    return finish_call(ctx, e, "dfx_compose_bwd");
}

// Host-entry staging buffers (grow-only).  An outgrown buffer is retired, not freed: freeing
// would synchronise the device; the retired ones are released by dfx_ctx_destroy.
static void* stage_buf(dfx_ctx* ctx, int slot, size_t bytes, cudaError_t* e) {
    *e = cudaSuccess;
    if (bytes == 0) bytes = 16;
    if (ctx->stage_cap[slot] >= bytes) return ctx->stage[slot];
    void* p = nullptr;
    *e = cudaMalloc(&p, bytes);
    if (*e != cudaSuccess) return nullptr;
    if (ctx->stage[slot]) ctx->stage_retired.push_back(ctx->stage[slot]);
    ctx->stage[slot] = p;
    ctx->stage_cap[slot] = bytes;
    return p;
}

// One blocking host-buffer call: records the first failing CUDA call and, however the call
// ends (success or any error path), waits for all three staging streams before returning, so
// no DMA into or out of the caller's host buffers is in flight afterwards, then releases the
// call's events.
struct HostCall {
    dfx_ctx* c;
    std::vector<cudaEvent_t> evs;
    cudaError_t first = cudaSuccess;
    const char* where = "";
    explicit HostCall(dfx_ctx* ctx) : c(ctx) {}
    bool ok(cudaError_t e, const char* w) {
        if (e != cudaSuccess && first == cudaSuccess) {
            first = e;
            where = w;
        }
        return first == cudaSuccess;
    }
    cudaEvent_t event() {
        cudaEvent_t ev = nullptr;
        if (ok(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "cudaEventCreate"))
            evs.push_back(ev);
        return ev;
    }
    // stream `to` waits for the work queued so far on `from`
    bool link(cudaStream_t from, cudaStream_t to) {
        cudaEvent_t ev = event();
        return ok(ev ? cudaEventRecord(ev, from) : first, "cudaEventRecord") &&
               ok(cudaStreamWaitEvent(to, ev, 0), "cudaStreamWaitEvent");
    }
    bool copy(void* dst, const void* src, size_t bytes, cudaMemcpyKind kind, cudaStream_t st) {
        return ok(cudaMemcpyAsync(dst, src, bytes, kind, st), "cudaMemcpyAsync");
    }
    cudaError_t drain() {
        const cudaError_t a = cudaStreamSynchronize(c->st_h2d);
        const cudaError_t b = cudaStreamSynchronize(c->st_comp);
        const cudaError_t d = cudaStreamSynchronize(c->st_d2h);
        return a != cudaSuccess ? a : b != cudaSuccess ? b : d;
    }
    ~HostCall() {
        if (c->st_h2d) drain();
        for (cudaEvent_t ev : evs) cudaEventDestroy(ev);
    }
};

static int host_streams(dfx_ctx* ctx) {
    cudaError_t e = cudaSuccess;
    if (!ctx->st_h2d) {
        if ((e = cudaStreamCreateWithFlags(&ctx->st_h2d, cudaStreamNonBlocking)) != cudaSuccess ||
            (e = cudaStreamCreateWithFlags(&ctx->st_comp, cudaStreamNonBlocking)) != cudaSuccess ||
            (e = cudaStreamCreateWithFlags(&ctx->st_d2h, cudaStreamNonBlocking)) != cudaSuccess)
            return cuda_fail(e, "stream create");
    }
    ctx->ws.cur = ctx->st_comp;
    return DFX_OK;
}

int dfx_ctx_set_sm_budget(dfx_ctx* ctx, int sms) {
    if (!ctx) return fail(DFX_EINVAL, "dfx_ctx_set_sm_budget: null context");
    if (sms < 0) return fail(DFX_EINVAL, "dfx_ctx_set_sm_budget: negative budget");
    ctx->ws.sm_budget = sms;
    return DFX_OK;
}

int dfx_working_matmul(dfx_ctx* ctx, dfx_dtype dtype, const void* A, int64_t sa_i, int64_t sa_k,
                       const void* B, int64_t sb_k, int64_t sb_j, int64_t M, int64_t N, int64_t K,
                       void* C, dfx_stream_t stream) {
    DeviceGuard dg;
    int rc = enter(ctx, dg, stream);
    if (rc) return rc;
    if (!valid_dtype(dtype)) return fail(DFX_EUNSUPPORTED, "working_matmul: dtype");
    if (M < 0 || N < 0 || K < 0) return fail(DFX_EINVAL, "working_matmul: negative dimension");
    if (M > 0 && N > 0 && (!C || (K > 0 && (!A || !B))))
        return fail(DFX_EINVAL, "working_matmul: null operand");
    int launches = 0;
    const cudaError_t e = dfx::launch_working_matmul(dtype, A, sa_i, sa_k, B, sb_k, sb_j, M, N, K, C,
                                                     stream, &launches);
    ctx->launches += launches;
    return finish_call(ctx, e, "dfx_working_matmul");
}

int dfx_lora_compose(dfx_ctx* ctx, dfx_dtype dtype, const void* mid, const void* B,
                     const void* base, const float* g, double s, const float* bias, int64_t rows,
                     int64_t d_out, int64_t r, void* y, void* delta, void* inner, void* lora,
                     dfx_stream_t stream) {
    DeviceGuard dg;
    int rc = enter(ctx, dg, stream);
    if (rc) return rc;
    if (dtype != DFX_BF16 && dtype != DFX_F16)
        return fail(DFX_EUNSUPPORTED, "lora_compose: bf16 / fp16 only (tcgen05 kind::f16)");
    if (rows < 0 || d_out < 0 || r <= 0) return fail(DFX_EINVAL, "lora_compose: shape");
    if (d_out % 8 != 0 || r % 8 != 0)
        return fail(DFX_EINVAL, "lora_compose: d_out and r must be multiples of 8 (16-byte rows)");
    const int n_out = (y != nullptr) + (delta != nullptr) + (inner != nullptr) + (lora != nullptr);
    if (n_out > 3) return fail(DFX_EINVAL, "lora_compose: at most three outputs per call");
    if (rows > 0 && d_out > 0 && (!mid || !B || !base || !g || n_out == 0))
        return fail(DFX_EINVAL, "lora_compose: null operand");
    if ((reinterpret_cast<uintptr_t>(g) | reinterpret_cast<uintptr_t>(bias)) & 15u)
        return fail(DFX_EINVAL, "lora_compose: g and bias must be 16-byte aligned");
    const uintptr_t tiles = reinterpret_cast<uintptr_t>(mid) | reinterpret_cast<uintptr_t>(B) |
                            reinterpret_cast<uintptr_t>(base) | reinterpret_cast<uintptr_t>(y) |
                            reinterpret_cast<uintptr_t>(delta) | reinterpret_cast<uintptr_t>(inner) |
                            reinterpret_cast<uintptr_t>(lora);
    if (tiles & 15u)
        return fail(DFX_EINVAL, "lora_compose: matrices must be 16-byte aligned (TMA / 128-bit access)");
    int launches = 0;
    const cudaError_t e = dfx::launch_lora_compose(dtype, mid, B, base, g, static_cast<float>(s),
                                                   bias, rows, d_out, r, y, delta, inner, lora,
                                                   stream, &launches);
    ctx->launches += launches;
    return finish_call(ctx, e, "dfx_lora_compose");
}

// ------------------------------------------------------- symmetric-memory all-reduce
}  // extern "C"

struct dfx_comm {
    dfx_ctx* ctx = nullptr;
    int rank = 0, world = 1;
    int64_t count = 0;
    char* base = nullptr;
    size_t bytes = 0;
    dfx::CommArgs args{};
    std::vector<void*> opened;   // peer bases mapped through CUDA IPC (closed at destroy)
    bool ready = false;
};

extern "C" {

int dfx_comm_create(dfx_ctx* ctx, int rank, int world, int64_t count, dfx_comm** out) {
    DeviceGuard dg;
    int rc = enter(ctx, dg);
    if (rc) return rc;
    if (!out) return fail(DFX_EINVAL, "dfx_comm_create: null out");
    *out = nullptr;
    if (world < 1 || world > dfx::kCommMaxRanks || rank < 0 || rank >= world)
        return fail(DFX_EINVAL, "dfx_comm_create: rank %d of world %d (max %d ranks)", rank, world,
                    dfx::kCommMaxRanks);
    if (count < 0) return fail(DFX_EINVAL, "dfx_comm_create: negative count");
    const size_t data = (size_t(count) * 4 + 255) / 256 * 256;
    const size_t flags = size_t(dfx::kCommMaxBlocks) * dfx::kCommMaxRanks * 4;
    dfx_comm* c = new dfx_comm();
    c->ctx = ctx;
    c->rank = rank;
    c->world = world;
    c->count = count;
    c->args.rank = rank;
    c->args.world = world;
    c->args.start_off = data;
    c->args.end_off = data + flags;
    c->args.epoch_off = data + 2 * flags;
    c->args.err_off = c->args.epoch_off + dfx::kCommMaxBlocks * 4;
    c->bytes = c->args.err_off + 256;
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, c->bytes);
    if (e == cudaSuccess) e = cudaMemset(p, 0, c->bytes);   // flags, epochs, error word = 0
    if (e != cudaSuccess) {
        if (p) cudaFree(p);
        delete c;
        return cuda_fail(e, "dfx_comm_create");
    }
    c->base = static_cast<char*>(p);
    c->args.peers[rank] = c->base;
    c->ready = world == 1;
    *out = c;
    g_err.clear();
    return DFX_OK;
}

void dfx_comm_destroy(dfx_comm* comm) {
    if (!comm) return;
    DeviceGuard dg;
    if (enter(comm->ctx, dg) == DFX_OK) {
        cudaDeviceSynchronize();
        for (void* p : comm->opened) cudaIpcCloseMemHandle(p);
        if (comm->base) cudaFree(comm->base);
    }
    delete comm;
}

float* dfx_comm_buffer(dfx_comm* comm) {
    return comm ? reinterpret_cast<float*>(comm->base) : nullptr;
}

void* dfx_comm_base(dfx_comm* comm) { return comm ? comm->base : nullptr; }

int dfx_comm_ipc_handle(dfx_comm* comm, void* out) {
    if (!comm || !out) return fail(DFX_EINVAL, "dfx_comm_ipc_handle: null argument");
    DeviceGuard dg;
    int rc = enter(comm->ctx, dg);
    if (rc) return rc;
    static_assert(sizeof(cudaIpcMemHandle_t) == DFX_IPC_HANDLE_BYTES, "IPC handle size");
    cudaIpcMemHandle_t h;
    const cudaError_t e = cudaIpcGetMemHandle(&h, comm->base);
    if (e != cudaSuccess) return cuda_fail(e, "cudaIpcGetMemHandle");
    std::memcpy(out, &h, sizeof(h));
    g_err.clear();
    return DFX_OK;
}

int dfx_comm_open(dfx_comm* comm, const void* handles) {
    if (!comm || !handles) return fail(DFX_EINVAL, "dfx_comm_open: null argument");
    DeviceGuard dg;
    int rc = enter(comm->ctx, dg);
    if (rc) return rc;
    if (comm->ready && comm->world > 1) return fail(DFX_EINVAL, "dfx_comm_open: peers already set");
    for (int k = 0; k < comm->world; ++k) {
        if (k == comm->rank) continue;
        cudaIpcMemHandle_t h;
        std::memcpy(&h, static_cast<const char*>(handles) + size_t(k) * sizeof(h), sizeof(h));
        void* p = nullptr;
        const cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) return cuda_fail(e, "cudaIpcOpenMemHandle");
        comm->opened.push_back(p);
        comm->args.peers[k] = static_cast<char*>(p);
    }
    comm->ready = true;
    g_err.clear();
    return DFX_OK;
}

int dfx_comm_set_peers(dfx_comm* comm, void* const* bases) {
    if (!comm || !bases) return fail(DFX_EINVAL, "dfx_comm_set_peers: null argument");
    for (int k = 0; k < comm->world; ++k) {
        if (k == comm->rank) continue;
        if (!bases[k]) return fail(DFX_EINVAL, "dfx_comm_set_peers: null base for rank %d", k);
        comm->args.peers[k] = static_cast<char*>(bases[k]);
    }
    comm->ready = true;
    g_err.clear();
    return DFX_OK;
}

int dfx_norm_allreduce(dfx_comm* comm, float* out, int64_t count, dfx_stream_t stream) {
    if (!comm) return fail(DFX_EINVAL, "dfx_norm_allreduce: null comm");
    dfx_ctx* ctx = comm->ctx;
    DeviceGuard dg;
    int rc = enter(ctx, dg, stream);
    if (rc) return rc;
    if (!comm->ready) return fail(DFX_EINVAL, "dfx_norm_allreduce: peers not opened");
    if (count < 0 || count > comm->count)
        return fail(DFX_EINVAL, "dfx_norm_allreduce: count %lld outside the symmetric buffer (%lld)",
                    (long long)count, (long long)comm->count);
    if (count > 0 && !out) return fail(DFX_EINVAL, "dfx_norm_allreduce: null out");
    dfx::CommArgs a = comm->args;
    if (a.world == 1) {
        // one rank: the sum is this rank's own data — a stream-ordered device copy (the
        // barrier kernel's system-scope fences cost ~25 us for nothing to exchange)
        const float* mine = reinterpret_cast<const float*>(a.peers[0]);
        cudaError_t e = cudaSuccess;
        if (count > 0 && out != mine)
            e = cudaMemcpyAsync(out, mine, size_t(count) * sizeof(float), cudaMemcpyDeviceToDevice,
                                stream);
        return finish_call(ctx, e, "dfx_norm_allreduce");
    }
    a.count = count;
    a.out = out;
    const int64_t n4 = (count + 3) / 4;
    a.max_blocks = static_cast<int>(std::min<int64_t>(
        dfx::kCommMaxBlocks, std::max<int64_t>(1, (n4 + dfx::kCommThreads - 1) / dfx::kCommThreads)));
    int launches = 0;
    const cudaError_t e = dfx::launch_allreduce(a, stream, &launches);
    ctx->launches += launches;
    return finish_call(ctx, e, "dfx_norm_allreduce");
}

int dfx_comm_status(dfx_comm* comm, int* timed_out) {
    if (!comm || !timed_out) return fail(DFX_EINVAL, "dfx_comm_status: null argument");
    DeviceGuard dg;
    int rc = enter(comm->ctx, dg);
    if (rc) return rc;
    uint32_t err = 0;
    const cudaError_t e = cudaMemcpy(&err, comm->base + comm->args.err_off, 4, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_fail(e, "dfx_comm_status");
    *timed_out = err ? 1 : 0;
    g_err.clear();
    return DFX_OK;
}

int dfx_module_fwd_host(dfx_ctx* ctx, dfx_dtype dtype, const void* W, const void* A,
                        const void* B, const float* m, const void* base, const void* lora,
                        double s, int64_t d_out, int64_t d_in, int64_t r, int64_t rows,
                        int64_t chunk_size, void* delta, float* g) {
    DeviceGuard dg;
    int rc = enter(ctx, dg);
    if (rc) return rc;
    rc = check_norm_args(dtype, W, A, B, d_out, d_in, r, chunk_size);
    if (rc) return rc;
    if (rows < 0 || !m || !g || (rows > 0 && (!base || !lora || !delta)))
        return fail(DFX_EINVAL, "dfx_module_fwd_host: null operand");
    if ((rc = host_streams(ctx))) return rc;
    const size_t eb = dtype == DFX_F32 ? 4 : 2;
    const size_t nW = size_t(d_out) * d_in, nA = size_t(r) * d_in, nB = size_t(d_out) * r;
    const size_t nact = size_t(rows) * d_out;
    const size_t sizes[9] = {nW * eb, nA * eb, nB * eb, size_t(d_out) * 4, size_t(d_out) * 4,
                             size_t(d_out) * 4, nact * eb, nact * eb, nact * eb};
    void* buf[9];
    cudaError_t e = cudaSuccess;
    for (int i = 0; i < 9; ++i) {
        buf[i] = stage_buf(ctx, i, sizes[i], &e);
        if (e) return cuda_fail(e, "stage alloc");
    }
    void *dW = buf[0], *dA = buf[1], *dB = buf[2];
    float *dm = static_cast<float*>(buf[3]), *dg_ = static_cast<float*>(buf[4]);
    float* dwn = static_cast<float*>(buf[5]);
    void *dbase = buf[6], *dlora = buf[7], *ddelta = buf[8];

    HostCall hc(ctx);
    // weights first: the norm overlaps the activation upload
    hc.copy(dA, A, nA * eb, cudaMemcpyHostToDevice, ctx->st_h2d);
    hc.copy(dB, B, nB * eb, cudaMemcpyHostToDevice, ctx->st_h2d);
    hc.copy(dm, m, d_out * 4, cudaMemcpyHostToDevice, ctx->st_h2d);
    hc.copy(dW, W, nW * eb, cudaMemcpyHostToDevice, ctx->st_h2d);
    if (!hc.link(ctx->st_h2d, ctx->st_comp)) return cuda_fail(hc.first, hc.where);
    rc = run_norm(ctx, dtype, dW, dA, dB, d_out, d_in, r, s, chunk_size, nullptr, nullptr,
                  nullptr, dm, dtype, dwn, dg_, dtype, ctx->st_comp, "dfx_module_fwd_host/norm");
    if (rc) return rc;
    if (!hc.link(ctx->st_comp, ctx->st_d2h) ||
        !hc.copy(g, dg_, d_out * 4, cudaMemcpyDeviceToHost, ctx->st_d2h))
        return cuda_fail(hc.first, hc.where);

    // activations in row chunks: upload chunk c+1 while composing c and downloading c-1
    const int64_t nchunk = rows >= 1024 ? 8 : 1;
    const int64_t crow = rows > 0 ? (rows + nchunk - 1) / nchunk : 1;
    for (int64_t r0 = 0; r0 < rows; r0 += crow) {
        const int64_t nr = std::min(crow, rows - r0);
        const size_t off = size_t(r0) * d_out * eb, bytes = size_t(nr) * d_out * eb;
        auto at = [&](void* p) { return static_cast<char*>(p) + off; };
        auto atc = [&](const void* p) { return static_cast<const char*>(p) + off; };
        hc.copy(at(dbase), atc(base), bytes, cudaMemcpyHostToDevice, ctx->st_h2d);
        hc.copy(at(dlora), atc(lora), bytes, cudaMemcpyHostToDevice, ctx->st_h2d);
        if (!hc.link(ctx->st_h2d, ctx->st_comp)) return cuda_fail(hc.first, hc.where);
        int launches = 0;
        e = dfx::launch_compose_fwd(dtype, at(dbase), at(dlora), dg_, static_cast<float>(s), nr,
                                    d_out, at(ddelta), nullptr, ctx->st_comp, &launches);
        ctx->launches += launches;
        if (e != cudaSuccess) return cuda_fail(e, "dfx_module_fwd_host/compose");
        if (!hc.link(ctx->st_comp, ctx->st_d2h) ||
            !hc.copy(static_cast<char*>(delta) + off, at(ddelta), bytes, cudaMemcpyDeviceToHost,
                     ctx->st_d2h))
            return cuda_fail(hc.first, hc.where);
    }
    e = hc.drain();
    if (e == cudaSuccess) e = cudaGetLastError();
    return finish_call(ctx, e, "dfx_module_fwd_host");
}

int dfx_module_train_host(dfx_ctx* ctx, dfx_dtype dtype, const void* W, const void* A,
                          const void* B, const float* m, const void* base, const void* lora,
                          const void* dy, double s, int64_t d_out, int64_t d_in, int64_t r,
                          int64_t rows, int64_t chunk_size, void* delta, void* d_lora,
                          void* d_base, float* d_mag, float* g) {
    DeviceGuard dg;
    int rc = enter(ctx, dg);
    if (rc) return rc;
    rc = check_norm_args(dtype, W, A, B, d_out, d_in, r, chunk_size);
    if (rc) return rc;
    if (rows < 0 || !m || !g || !d_mag ||
        (rows > 0 && (!base || !lora || !dy || !delta || !d_lora || !d_base)))
        return fail(DFX_EINVAL, "dfx_module_train_host: null operand");
    if ((rc = host_streams(ctx))) return rc;
    const size_t eb = dtype == DFX_F32 ? 4 : 2;
    const size_t nW = size_t(d_out) * d_in, nA = size_t(r) * d_in, nB = size_t(d_out) * r;
    const size_t nact = size_t(rows) * d_out;
    const size_t sizes[14] = {nW * eb, nA * eb, nB * eb, size_t(d_out) * 4, size_t(d_out) * 4,
                              size_t(d_out) * 4, nact * eb, nact * eb, nact * eb, nact * eb,
                              nact * eb, nact * eb, nact * eb, size_t(d_out) * 4};
    void* buf[14];
    cudaError_t e = cudaSuccess;
    for (int i = 0; i < 14; ++i) {
        buf[i] = stage_buf(ctx, i, sizes[i], &e);
        if (e) return cuda_fail(e, "stage alloc");
    }
    void *dW = buf[0], *dA = buf[1], *dB = buf[2];
    float *dm = static_cast<float*>(buf[3]), *dg_ = static_cast<float*>(buf[4]);
    float* dwn = static_cast<float*>(buf[5]);
    void *dbase = buf[6], *dlora = buf[7], *ddelta = buf[8], *dinner = buf[9], *ddy = buf[10];
    void *ddl = buf[11], *ddb = buf[12];
    float* ddm = static_cast<float*>(buf[13]);

    HostCall hc(ctx);
    // weights first: the norm overlaps the activation upload
    hc.copy(dA, A, nA * eb, cudaMemcpyHostToDevice, ctx->st_h2d);
    hc.copy(dB, B, nB * eb, cudaMemcpyHostToDevice, ctx->st_h2d);
    hc.copy(dm, m, d_out * 4, cudaMemcpyHostToDevice, ctx->st_h2d);
    hc.copy(dW, W, nW * eb, cudaMemcpyHostToDevice, ctx->st_h2d);
    if (!hc.link(ctx->st_h2d, ctx->st_comp)) return cuda_fail(hc.first, hc.where);
    rc = run_norm(ctx, dtype, dW, dA, dB, d_out, d_in, r, s, chunk_size, nullptr, nullptr,
                  nullptr, dm, dtype, dwn, dg_, dtype, ctx->st_comp, "dfx_module_train_host/norm");
    if (rc) return rc;
    if (!hc.link(ctx->st_comp, ctx->st_d2h) ||
        !hc.copy(g, dg_, d_out * 4, cudaMemcpyDeviceToHost, ctx->st_d2h))
        return cuda_fail(hc.first, hc.where);

    // Row chunks: upload base / lora / dY of chunk c+1 while chunk c runs the dual compose and
    // the elementwise backward (d_lora, d_base) and chunk c-1 downloads delta / d_lora /
    // d_base; the serial d_mag chain needs every row, so it runs last over the resident dY
    // and inner (magnitude-gradient-only backward) — PCIe stays busy in both directions.
    const int64_t nchunk = rows >= 1024 ? 8 : 1;
    const int64_t crow = rows > 0 ? (rows + nchunk - 1) / nchunk : 1;
    for (int64_t r0 = 0; r0 < rows; r0 += crow) {
        const int64_t nr = std::min(crow, rows - r0);
        const size_t off = size_t(r0) * d_out * eb, bytes = size_t(nr) * d_out * eb;
        auto at = [&](void* p) { return static_cast<char*>(p) + off; };
        auto atc = [&](const void* p) { return static_cast<const char*>(p) + off; };
        hc.copy(at(dbase), atc(base), bytes, cudaMemcpyHostToDevice, ctx->st_h2d);
        hc.copy(at(dlora), atc(lora), bytes, cudaMemcpyHostToDevice, ctx->st_h2d);
        hc.copy(at(ddy), atc(dy), bytes, cudaMemcpyHostToDevice, ctx->st_h2d);
        if (!hc.link(ctx->st_h2d, ctx->st_comp)) return cuda_fail(hc.first, hc.where);
        int launches = 0;
        e = dfx::launch_compose_fwd(dtype, at(dbase), at(dlora), dg_, static_cast<float>(s), nr,
                                    d_out, at(ddelta), at(dinner), ctx->st_comp, &launches);
        if (e == cudaSuccess)
            e = dfx::launch_compose_bwd(dtype, at(ddy), dg_, static_cast<float>(s), nullptr,
                                        nullptr, nr, d_out, at(ddl), at(ddb), nullptr,
                                        ctx->st_comp, &launches);
        ctx->launches += launches;
        if (e != cudaSuccess) return cuda_fail(e, "dfx_module_train_host/compose");
        if (!hc.link(ctx->st_comp, ctx->st_d2h) ||
            !hc.copy(static_cast<char*>(delta) + off, at(ddelta), bytes, cudaMemcpyDeviceToHost,
                     ctx->st_d2h) ||
            !hc.copy(static_cast<char*>(d_lora) + off, at(ddl), bytes, cudaMemcpyDeviceToHost,
                     ctx->st_d2h) ||
            !hc.copy(static_cast<char*>(d_base) + off, at(ddb), bytes, cudaMemcpyDeviceToHost,
                     ctx->st_d2h))
            return cuda_fail(hc.first, hc.where);
    }
    int launches = 0;
    e = dfx::launch_compose_bwd(dtype, ddy, dg_, static_cast<float>(s), dinner, dwn, rows, d_out,
                                nullptr, nullptr, ddm, ctx->st_comp, &launches);
    ctx->launches += launches;
    if (e != cudaSuccess) return cuda_fail(e, "dfx_module_train_host/d_mag");
    if (!hc.link(ctx->st_comp, ctx->st_d2h) ||
        !hc.copy(d_mag, ddm, d_out * 4, cudaMemcpyDeviceToHost, ctx->st_d2h))
        return cuda_fail(hc.first, hc.where);
    e = hc.drain();
    if (e == cudaSuccess) e = cudaGetLastError();
    return finish_call(ctx, e, "dfx_module_train_host");
}

}  // extern "C"
