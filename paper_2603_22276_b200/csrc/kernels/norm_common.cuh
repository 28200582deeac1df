// norm_common.cuh — shared pieces of the factored row-norm kernels.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "launch.h"
#include "ptx.cuh"

namespace dfx {

// Workspace slots owned by the context.
enum WsSlot : int {
    kWsGramPart = 0,   // gram partial tiles   [k_split][tiles][128*128] fp32
    kWsGram2 = 1,      // [G_hi | G_lo] bf16   [r][2*r_pad]
    kWsCross = 2,      // cross partials       [k_split*n_split][d_out] fp32
    kWsBa = 3,         // ba_sq partials       [n_split][d_out] fp32
    kWsBase = 4,       // base_sq partials     [k_split][d_out] fp32
    kWsGram = 5,       // G fp32               [r][r]          (SIMT path)
    kWsTerms = 6,      // base_sq/cross/ba_sq  [3][d_out]      (when caller wants none)
    kWsGramCount = 7,  // per-128-row-block tile counters of the fused finisher (zeroed)
    kWsScale = 8,      // fp16 V operand: 2^-e of the scaled Gram split (one float)
    kWsAdaptCount = 9, // per-128-row-block counters of the adapter-only call (kNormAdapter)
    kWsCount = 10
};

struct FinishArgs {
    const float* base_part;  int base_parts;   // [base_parts][d_out]
    const float* cross_part; int cross_parts;  // [cross_parts][d_out]
    const float* ba_part;    int ba_parts;     // [ba_parts][d_out]
    int64_t d_out;
    double two_s, s2;
    float* base_sq; float* cross; float* ba_sq;   // optional term outputs
    int round_dt;                                  // kF32 = no extra rounding
    float* w_norm;                                 // optional
    const float* m; int mag_dt; float* g;          // optional magnitude division
};

cudaError_t launch_finish(const FinishArgs& f, cudaStream_t st);

// The stored value of round_to_dtype(x) for x already fp32 (dtype.cpp:77-85):
// RNE to the target grid, result kept in fp32 storage.
__device__ __forceinline__ float round_store(float x, int dt) {
    if (dt == kBF16) return __bfloat162float(__float2bfloat16_rn(x));
    if (dt == kF16) return __half2float(__float2half_rn(x));
    return x;
}

// Row j of the finisher: the partials summed in fixed (ascending) order, then assemble_norm
// (factored_norm.cpp:128-134) -> round to the W dtype (:213-216) -> magnitude_scale
// (:232-239).  Partials are read through L2 (ld.global.cg): in the fused form (the last
// GEMM tile of a row block finishes it, norm_tc.cu) other CTAs wrote them in this launch.
__device__ __forceinline__ void finish_row(const FinishArgs& f, int64_t j) {
    float b = 0.0f, c = 0.0f, q = 0.0f;
    if (f.base_part) {
        b = __ldcg(f.base_part + j);
        for (int p = 1; p < f.base_parts; ++p) b = __fadd_rn(b, __ldcg(f.base_part + p * f.d_out + j));
    }
    if (f.cross_part) {
        c = __ldcg(f.cross_part + j);
        for (int p = 1; p < f.cross_parts; ++p) c = __fadd_rn(c, __ldcg(f.cross_part + p * f.d_out + j));
    }
    if (f.ba_part) {
        q = __ldcg(f.ba_part + j);
        for (int p = 1; p < f.ba_parts; ++p) q = __fadd_rn(q, __ldcg(f.ba_part + p * f.d_out + j));
    }
    if (f.base_sq) f.base_sq[j] = b;
    if (f.cross) f.cross[j] = c;
    if (f.ba_sq) f.ba_sq[j] = q;
    if (!f.w_norm && !f.g) return;
    const float c1 = __double2float_rn(__dmul_rn(f.two_s, static_cast<double>(c)));
    const float t1 = __fadd_rn(b, c1);
    const float c2 = __double2float_rn(__dmul_rn(f.s2, static_cast<double>(q)));
    float t2 = __fadd_rn(t1, c2);
    t2 = (t2 < 0.0f) ? 0.0f : t2;  // NaN compares false and passes through
    const float nrm = round_store(__fsqrt_rn(t2), f.round_dt);
    if (f.w_norm) f.w_norm[j] = nrm;
    if (f.g) {
        const float eps = (f.mag_dt == kF32) ? static_cast<float>(1e-12) : static_cast<float>(1e-6);
        const float denom = nrm < eps ? eps : nrm;
        f.g[j] = round_store(__fdiv_rn(f.m[j], denom), f.mag_dt);
    }
}

// bf16 tensor-core pipeline (norm_tc.cu); returns cudaErrorNotSupported when the
// shape/dtype is outside the TMA/UMMA envelope so the caller can use the SIMT path.
cudaError_t launch_norm_tc(const NormArgs& a, Workspace* ws, cudaStream_t st, int* launches);
bool norm_tc_supported(int dt, int64_t d_out, int64_t d_in, int64_t r);
// fp32 weights on the tensor cores (3xTF32); DFX_NORM_TF32=0 keeps them on the SIMT path.
bool norm_tc_f32_supported(int64_t d_out, int64_t d_in, int64_t r, int64_t chunk);
bool norm_tf32_enabled();
cudaError_t launch_norm_tc_f32(const NormArgs& a, Workspace* ws, cudaStream_t st, int* launches);

}  // namespace dfx
