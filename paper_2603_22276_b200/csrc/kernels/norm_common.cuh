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
    kWsGramCount = 7,  // per-tile split counters for the fused Gram reduction (zeroed)
    kWsScale = 8,      // fp16 V operand: 2^-e of the scaled Gram split (one float)
    kWsCount = 9
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

// bf16 tensor-core pipeline (norm_tc.cu); returns cudaErrorNotSupported when the
// shape/dtype is outside the TMA/UMMA envelope so the caller can use the SIMT path.
cudaError_t launch_norm_tc(const NormArgs& a, Workspace* ws, cudaStream_t st, int* launches);
bool norm_tc_supported(int dt, int64_t d_out, int64_t d_in, int64_t r);
// fp32 weights on the tensor cores (3xTF32); DFX_NORM_TF32=0 keeps them on the SIMT path.
bool norm_tc_f32_supported(int64_t d_out, int64_t d_in, int64_t r, int64_t chunk);
bool norm_tf32_enabled();
cudaError_t launch_norm_tc_f32(const NormArgs& a, Workspace* ws, cudaStream_t st, int* launches);

// The stored value of round_to_dtype(x) for x already fp32 (dtype.cpp:77-85):
// RNE to the target grid, result kept in fp32 storage.
__device__ __forceinline__ float round_store(float x, int dt) {
    if (dt == kBF16) return __bfloat162float(__float2bfloat16_rn(x));
    if (dt == kF16) return __half2float(__float2half_rn(x));
    return x;
}

}  // namespace dfx
