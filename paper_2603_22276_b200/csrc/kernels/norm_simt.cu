// norm_simt.cu — CUDA-core (FFMA) factored row norm, the finishing epilogue, and the
// stand-alone assemble / magnitude kernels.
//
// The SIMT path serves fp32 weights (the accuracy configuration), fp16, and every
// shape outside the bf16 TMA/UMMA envelope (ragged d_in / r, tiny matrices).  It
// follows factored_norm.cpp:27-120 term by term:
//   base_sq  per-row serial fp32 chain of w*w, partial reset at every ChunkPlan
//            boundary and added in ascending chunk order (:49-61)  -> bitwise equal
//   G        = A A^T, fp32 accumulate                              (:65-76)
//   cross    = rowsum(B .* (W A^T)), fp32                          (:78-100)
//   ba_sq    = rowsum((B G) .* B), fp32                            (:103-117)
// The assemble / magnitude epilogue is bitwise equal to factored_norm.cpp:122-136 and
// :219-240 (fp64 scale products, separately rounded fp32 adds, NaN-preserving clamp,
// IEEE sqrt, RNE to the storage dtype).
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <algorithm>

#include "norm_common.cuh"

namespace dfx {
namespace {

template <typename T>
__device__ __forceinline__ float ldf(const T* p) { return Elem<T>::to_f(*p); }

constexpr int kBM = 64, kBN = 64, kBK = 16;

enum Mode { kRowdot = 0, kStore = 1 };

// D = X * Y^T over a 64x64 tile (X: [M x K] ld=ldx, Y: [N x K] ld=ldy).
//   kRowdot: part[blockIdx.y][m] = sum_n D[m,n] * Z[m,n]  (Z: [M x N] ld=ldz)
//   kStore : out[m*N + n] = D[m,n]
//   chain  : blockIdx.y == 0 CTAs also run the base_sq chain over their X rows.
template <typename TX, typename TY, int kMode, bool kChain>
__global__ void __launch_bounds__(256) simt_gemm(const TX* __restrict__ X, int64_t ldx,
                                                 const TY* __restrict__ Y, int64_t ldy,
                                                 const TX* __restrict__ Z, int64_t ldz,
                                                 int64_t M, int64_t N, int64_t K,
                                                 int64_t chunk, float* __restrict__ out,
                                                 float* __restrict__ base_out) {
    __shared__ __align__(16) float sX[kBK][kBM + 4];
    __shared__ __align__(16) float sY[kBK][kBN + 4];
    const int t = threadIdx.x;
    const int tx = t % 16, ty = t / 16;
    const int64_t m0 = static_cast<int64_t>(blockIdx.x) * kBM;
    const int64_t n0 = static_cast<int64_t>(blockIdx.y) * kBN;
    const bool chain = kChain && blockIdx.y == 0;

    float acc[4][4] = {};
    float partial = 0.0f, base = 0.0f;

    for (int64_t k0 = 0; k0 < K; k0 += kBK) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int idx = t + 256 * q;
            const int rr = idx / kBK, kk = idx % kBK;
            const int64_t gm = m0 + rr, gn = n0 + rr, gk = k0 + kk;
            sX[kk][rr] = (gm < M && gk < K) ? ldf(X + gm * ldx + gk) : 0.0f;
            sY[kk][rr] = (gn < N && gk < K) ? ldf(Y + gn * ldy + gk) : 0.0f;
        }
        __syncthreads();
        if (chain && t < kBM) {
            for (int kk = 0; kk < kBK && k0 + kk < K; ++kk) {
                const int64_t gk = k0 + kk;
                if (gk > 0 && gk % chunk == 0) {
                    base = __fadd_rn(base, partial);
                    partial = 0.0f;
                }
                const float v = sX[kk][t];
                partial = __fadd_rn(partial, __fmul_rn(v, v));
            }
        }
#pragma unroll
        for (int kk = 0; kk < kBK; ++kk) {
            const float4 xa = *reinterpret_cast<const float4*>(&sX[kk][ty * 4]);
            const float4 yb = *reinterpret_cast<const float4*>(&sY[kk][tx * 4]);
            const float xv[4] = {xa.x, xa.y, xa.z, xa.w};
            const float yv[4] = {yb.x, yb.y, yb.z, yb.w};
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(xv[i], yv[j], acc[i][j]);
        }
        __syncthreads();
    }
    if (chain && t < kBM && m0 + t < M) base_out[m0 + t] = __fadd_rn(base, partial);

    if (kMode == kStore) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int64_t gm = m0 + ty * 4 + i;
            if (gm >= M) continue;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int64_t gn = n0 + tx * 4 + j;
                if (gn < N) out[gm * N + gn] = acc[i][j];
            }
        }
    } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int64_t gm = m0 + ty * 4 + i;
            float rp = 0.0f;
            if (gm < M) {
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int64_t gn = n0 + tx * 4 + j;
                    if (gn < N) rp = fmaf(acc[i][j], ldf(Z + gm * ldz + gn), rp);
                }
            }
            // reduce over the 16 tx lanes that share this row (fixed xor tree)
            rp += __shfl_xor_sync(0xffffffffu, rp, 8);
            rp += __shfl_xor_sync(0xffffffffu, rp, 4);
            rp += __shfl_xor_sync(0xffffffffu, rp, 2);
            rp += __shfl_xor_sync(0xffffffffu, rp, 1);
            if (tx == 0 && gm < M) out[static_cast<int64_t>(blockIdx.y) * M + gm] = rp;
        }
    }
}

// base_sq only (s == 0 fast path, factored_norm.cpp:37,63): 32 rows per CTA,
// coalesced 32x256 tiles staged in smem, one serial chain per row.
template <typename T>
__global__ void __launch_bounds__(256) base_chain(const T* __restrict__ W, int64_t d_out,
                                                  int64_t d_in, int64_t chunk,
                                                  float* __restrict__ base_out) {
    __shared__ float tile[32][257];
    const int t = threadIdx.x;
    const int64_t r0 = static_cast<int64_t>(blockIdx.x) * 32;
    float partial = 0.0f, base = 0.0f;
    for (int64_t k0 = 0; k0 < d_in; k0 += 256) {
        for (int idx = t; idx < 32 * 256; idx += 256) {
            const int rr = idx / 256, kk = idx % 256;
            const int64_t gr = r0 + rr, gk = k0 + kk;
            tile[rr][kk] = (gr < d_out && gk < d_in) ? ldf(W + gr * d_in + gk) : 0.0f;
        }
        __syncthreads();
        if (t < 32) {
            for (int kk = 0; kk < 256 && k0 + kk < d_in; ++kk) {
                const int64_t gk = k0 + kk;
                if (gk > 0 && gk % chunk == 0) {
                    base = __fadd_rn(base, partial);
                    partial = 0.0f;
                }
                const float v = tile[t][kk];
                partial = __fadd_rn(partial, __fmul_rn(v, v));
            }
        }
        __syncthreads();
    }
    if (t < 32 && r0 + t < d_out) base_out[r0 + t] = __fadd_rn(base, partial);
}

// Sum partials in fixed (ascending) order, then assemble_norm -> round -> magnitude.
__global__ void __launch_bounds__(256) finish_kernel(FinishArgs f) {
    const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j < f.d_out) finish_row(f, j);
}

__global__ void __launch_bounds__(256) magnitude_kernel(const float* __restrict__ m,
                                                        const float* __restrict__ w_norm,
                                                        int64_t n, int dt, float* __restrict__ g) {
    const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= n) return;
    const float eps = (dt == kF32) ? static_cast<float>(1e-12) : static_cast<float>(1e-6);
    const float wn = w_norm[j];
    const float denom = wn < eps ? eps : wn;
    g[j] = round_store(__fdiv_rn(m[j], denom), dt);
}

inline unsigned blocks_for(int64_t n, int bs) { return static_cast<unsigned>((n + bs - 1) / bs); }

template <typename T>
cudaError_t norm_simt_impl(const NormArgs& a, Workspace* ws, cudaStream_t st, int* launches) {
    const T* W = static_cast<const T*>(a.w);
    const T* A = static_cast<const T*>(a.a);
    const T* B = static_cast<const T*>(a.b);
    cudaError_t err = cudaSuccess;
    FinishArgs f{};
    f.d_out = a.d_out;
    f.two_s = 2.0 * a.s;
    f.s2 = a.s * a.s;
    f.base_sq = a.base_sq; f.cross = a.cross; f.ba_sq = a.ba_sq;
    f.round_dt = a.round_dt; f.w_norm = a.w_norm;
    f.m = a.m; f.mag_dt = a.mag_dt; f.g = a.m ? a.g : nullptr;

    if (a.mode == kNormFinish) {
        // d_in split, step 2: ba_sq from the reduced Gram, then assemble / round / g
        f.base_part = a.base_in; f.base_parts = 1;
        if (a.s != 0.0) {  // s == 0: the reference skips cross / ba_sq (factored_norm.cpp:37)
            const int64_t nt = (a.r + kBN - 1) / kBN;
            float* ba = static_cast<float*>(ws_get(ws, kWsBa, nt * a.d_out * sizeof(float), &err));
            if (err != cudaSuccess) return err;
            prof_begin("simt_ba_rowdot", st);
            simt_gemm<T, float, kRowdot, false>
                <<<dim3(blocks_for(a.d_out, kBM), static_cast<unsigned>(nt)), 256, 0, st>>>(
                    B, a.r, a.gram_in, a.r, B, a.r, a.d_out, a.r, a.r, a.chunk_size, ba, nullptr);
            prof_end(st);
            if (launches) ++*launches;
            f.cross_part = a.cross_in; f.cross_parts = 1;
            f.ba_part = ba; f.ba_parts = static_cast<int>(nt);
        }
        err = cudaGetLastError();
        if (err != cudaSuccess) return err;
        if (launches) ++*launches;
        return launch_finish(f, st);
    }

    float* base = static_cast<float*>(ws_get(ws, kWsBase, a.d_out * sizeof(float), &err));
    if (err != cudaSuccess) return err;
    f.base_part = base; f.base_parts = 1;

    if (a.s == 0.0 && a.mode == kNormFull) {
        prof_begin("base_chain", st);
        base_chain<T><<<blocks_for(a.d_out, 32), 256, 0, st>>>(W, a.d_out, a.d_in, a.chunk_size, base);
        prof_end(st);
        if (launches) ++*launches;
    } else {
        const int64_t nt = (a.r + kBN - 1) / kBN;
        float* G = a.mode == kNormPartial
                       ? a.gram_out
                       : static_cast<float*>(ws_get(ws, kWsGram, a.r * a.r * sizeof(float), &err));
        if (err != cudaSuccess) return err;
        float* cross = static_cast<float*>(ws_get(ws, kWsCross, nt * a.d_out * sizeof(float), &err));
        if (err != cudaSuccess) return err;
        float* ba = static_cast<float*>(ws_get(ws, kWsBa, nt * a.d_out * sizeof(float), &err));
        if (err != cudaSuccess) return err;
        // G = A A^T
        prof_begin("simt_gram", st);
        simt_gemm<T, T, kStore, false>
            <<<dim3(blocks_for(a.r, kBM), static_cast<unsigned>(nt)), 256, 0, st>>>(
                A, a.d_in, A, a.d_in, nullptr, 0, a.r, a.r, a.d_in, a.chunk_size, G, nullptr);
        prof_end(st);
        // ba_sq partials: rowdot(B G, B); G is exactly symmetric (p,q and q,p use the
        // same products in the same order), so Y = G serves as (G^T)
        if (a.mode == kNormFull) {
            prof_begin("simt_ba_rowdot", st);
            simt_gemm<T, float, kRowdot, false>
                <<<dim3(blocks_for(a.d_out, kBM), static_cast<unsigned>(nt)), 256, 0, st>>>(
                    B, a.r, G, a.r, B, a.r, a.d_out, a.r, a.r, a.chunk_size, ba, nullptr);
            prof_end(st);
        }
        // cross partials + base_sq chain: rowdot(W A^T, B)
        prof_begin("simt_u_rowdot", st);
        simt_gemm<T, T, kRowdot, true>
            <<<dim3(blocks_for(a.d_out, kBM), static_cast<unsigned>(nt)), 256, 0, st>>>(
                W, a.d_in, A, a.d_in, B, a.r, a.d_out, a.r, a.d_in, a.chunk_size, cross, base);
        prof_end(st);
        if (launches) *launches += 3;
        f.cross_part = cross; f.cross_parts = static_cast<int>(nt);
        if (a.mode == kNormFull) { f.ba_part = ba; f.ba_parts = static_cast<int>(nt); }
    }
    if (a.mode == kNormPartial) { f.w_norm = nullptr; f.g = nullptr; f.ba_sq = nullptr; }
    err = cudaGetLastError();
    if (err != cudaSuccess) return err;
    if (launches) ++*launches;
    return launch_finish(f, st);
}

}  // namespace

cudaError_t launch_finish(const FinishArgs& f, cudaStream_t st) {
    if (f.d_out <= 0) return cudaSuccess;
    prof_begin("finish", st);
    finish_kernel<<<blocks_for(f.d_out, 256), 256, 0, st>>>(f);
    prof_end(st);
    return cudaGetLastError();
}

cudaError_t launch_assemble(const float* base_sq, const float* cross, const float* ba_sq,
                            double two_s, double s2, int64_t n, int round_dt, float* out,
                            cudaStream_t st, int* launches) {
    FinishArgs f{};
    f.base_part = base_sq; f.base_parts = 1;
    f.cross_part = cross; f.cross_parts = 1;
    f.ba_part = ba_sq; f.ba_parts = 1;
    f.d_out = n; f.two_s = two_s; f.s2 = s2;
    f.round_dt = round_dt; f.w_norm = out;
    if (launches && n > 0) ++*launches;
    return launch_finish(f, st);
}

cudaError_t launch_magnitude_scale(int dt, const float* m, const float* w_norm, int64_t n,
                                   float* g, cudaStream_t st, int* launches) {
    if (n <= 0) return cudaSuccess;
    prof_begin("magnitude", st);
    magnitude_kernel<<<blocks_for(n, 256), 256, 0, st>>>(m, w_norm, n, dt, g);
    prof_end(st);
    if (launches) ++*launches;
    return cudaGetLastError();
}

int norm_uses_tensor_cores(int dt, int64_t d_out, int64_t d_in, int64_t r) {
    if (dt == kF32) return norm_tf32_enabled() && norm_tc_f32_supported(d_out, d_in, r, 32) ? 1 : 0;
    return norm_tc_supported(dt, d_out, d_in, r) ? 1 : 0;
}

cudaError_t launch_norm(const NormArgs& a, Workspace* ws, cudaStream_t st, int* launches) {
    if (a.d_out == 0) return cudaSuccess;
    // the tensor-core chain walks 64-wide K blocks: chunk boundaries must align to them
    const int64_t tc_din = a.mode == kNormFinish ? 64 : a.d_in;  // finish reads no W
    const bool tc = a.chunk_size % 64 == 0 && norm_tc_supported(a.dt, a.d_out, tc_din, a.r);
    if (a.mode == kNormAdapter || a.ba_given) {   // split form: tensor-core path only
        if ((a.mode != kNormAdapter && a.mode != kNormFull) || !tc || a.s == 0.0)
            return cudaErrorNotSupported;
        return launch_norm_tc(a, ws, st, launches);
    }
    if (a.base_cached) {   // only the tensor-core U kernel can drop its chain
        if (a.mode != kNormFull || !tc || a.s == 0.0) return cudaErrorNotSupported;
        return launch_norm_tc(a, ws, st, launches);
    }
    if ((a.s != 0.0 || a.mode == kNormPartial) && tc) return launch_norm_tc(a, ws, st, launches);
    if (a.dt == kF32 && a.s != 0.0 && a.mode == kNormFull && norm_tf32_enabled() &&
        norm_tc_f32_supported(a.d_out, a.d_in, a.r, a.chunk_size))
        return launch_norm_tc_f32(a, ws, st, launches);
    switch (a.dt) {
        case kF32: return norm_simt_impl<float>(a, ws, st, launches);
        case kBF16: return norm_simt_impl<__nv_bfloat16>(a, ws, st, launches);
        default: return norm_simt_impl<__half>(a, ws, st, launches);
    }
}

}  // namespace dfx
