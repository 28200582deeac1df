// layer_gemm.cu — the layer's plain GEMMs with the reference's working_matmul semantics
// (layer.cpp:15-17 over matrix.cpp:53-78): C[i, j] = round_dtype(serial-k fp32 sum of
// fl32(a[i, k]) * fl32(b[k, j])), products and adds individually rounded (no FMA), k
// ascending — bitwise the reference's, for the C++ layer drop-in.
// A CUDA-core kernel: the serial order per output is the contract, so the tensor cores
// (whose accumulation order differs) are deliberately not used here; the fused
// tensor-core path for frameworks is lora_compose.cu.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "launch.h"
#include "ptx.cuh"

namespace dfx {
namespace {

// 128 x 128 outputs per CTA, 8 x 8 per thread (register tiling: each operand value read from
// shared memory feeds eight products); K staged through shared memory 16 at a time.  Every
// output still runs its own serial chain over k ascending.
constexpr int kBM = 128, kBN = 128, kBK = 16, kTM = 8, kTN = 8;

template <typename T>
__global__ void __launch_bounds__(256) working_matmul_kernel(
    const T* __restrict__ a, int64_t sa_i, int64_t sa_k, const T* __restrict__ b, int64_t sb_k,
    int64_t sb_j, int64_t M, int64_t N, int64_t K, T* __restrict__ c) {
    __shared__ __align__(16) float sa[kBK][kBM + 4];
    __shared__ __align__(16) float sb[kBK][kBN + 4];
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    const int64_t i0 = static_cast<int64_t>(blockIdx.y) * kBM, j0 = static_cast<int64_t>(blockIdx.x) * kBN;
    float acc[kTM][kTN];
#pragma unroll
    for (int m = 0; m < kTM; ++m)
#pragma unroll
        for (int n = 0; n < kTN; ++n) acc[m][n] = 0.0f;
    for (int64_t k0 = 0; k0 < K; k0 += kBK) {
#pragma unroll
        for (int q = 0; q < kBM * kBK / 256; ++q) {
            const int e = q * 256 + threadIdx.x;
            const int r = e / kBK, kk = e % kBK;          // consecutive threads: consecutive k
            const int64_t gi = i0 + r, gk = k0 + kk;
            sa[kk][r] = (gi < M && gk < K) ? Elem<T>::to_f(a[gi * sa_i + gk * sa_k]) : 0.0f;
        }
#pragma unroll
        for (int q = 0; q < kBK * kBN / 256; ++q) {
            const int e = q * 256 + threadIdx.x;
            const int kk = e / kBN, cc = e % kBN;         // consecutive threads: consecutive j
            const int64_t gk = k0 + kk, gj = j0 + cc;
            sb[kk][cc] = (gk < K && gj < N) ? Elem<T>::to_f(b[gk * sb_k + gj * sb_j]) : 0.0f;
        }
        __syncthreads();
        const int kn = static_cast<int>(K - k0 < kBK ? K - k0 : kBK);
        for (int kk = 0; kk < kn; ++kk) {
            float av[kTM], bv[kTN];
#pragma unroll
            for (int m = 0; m < kTM; m += 4) {
                const float4 v = *reinterpret_cast<const float4*>(&sa[kk][ty * kTM + m]);
                av[m] = v.x; av[m + 1] = v.y; av[m + 2] = v.z; av[m + 3] = v.w;
            }
#pragma unroll
            for (int n = 0; n < kTN; n += 4) {
                const float4 v = *reinterpret_cast<const float4*>(&sb[kk][tx * kTN + n]);
                bv[n] = v.x; bv[n + 1] = v.y; bv[n + 2] = v.z; bv[n + 3] = v.w;
            }
#pragma unroll
            for (int m = 0; m < kTM; ++m)
#pragma unroll
                for (int n = 0; n < kTN; ++n) acc[m][n] = __fadd_rn(acc[m][n], __fmul_rn(av[m], bv[n]));
        }
        __syncthreads();
    }
#pragma unroll
    for (int m = 0; m < kTM; ++m) {
        const int64_t i = i0 + ty * kTM + m;
        if (i >= M) continue;
#pragma unroll
        for (int n = 0; n < kTN; ++n) {
            const int64_t j = j0 + tx * kTN + n;
            if (j < N) c[i * N + j] = Elem<T>::from_f(acc[m][n]);
        }
    }
}

template <typename T>
cudaError_t launch_t(const void* a, int64_t sa_i, int64_t sa_k, const void* b, int64_t sb_k,
                     int64_t sb_j, int64_t M, int64_t N, int64_t K, void* c, cudaStream_t st) {
    const dim3 grid(static_cast<unsigned>((N + kBN - 1) / kBN), static_cast<unsigned>((M + kBM - 1) / kBM));
    prof_begin("working_matmul", st);
    working_matmul_kernel<T><<<grid, 256, 0, st>>>(static_cast<const T*>(a), sa_i, sa_k,
                                                   static_cast<const T*>(b), sb_k, sb_j, M, N, K,
                                                   static_cast<T*>(c));
    prof_end(st);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_working_matmul(int dt, const void* a, int64_t sa_i, int64_t sa_k, const void* b,
                                  int64_t sb_k, int64_t sb_j, int64_t M, int64_t N, int64_t K,
                                  void* c, cudaStream_t st, int* launches) {
    if (M == 0 || N == 0) return cudaSuccess;
    if (M > 65535LL * kBM) return cudaErrorInvalidValue;
    if (launches) ++*launches;
    switch (dt) {
        case kF32: return launch_t<float>(a, sa_i, sa_k, b, sb_k, sb_j, M, N, K, c, st);
        case kBF16: return launch_t<__nv_bfloat16>(a, sa_i, sa_k, b, sb_k, sb_j, M, N, K, c, st);
        default: return launch_t<__half>(a, sa_i, sa_k, b, sb_k, sb_j, M, N, K, c, st);
    }
}

}  // namespace dfx
