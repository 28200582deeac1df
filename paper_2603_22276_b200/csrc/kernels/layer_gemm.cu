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

constexpr int kT = 16;    // 16 x 16 outputs per CTA, one per thread
constexpr int kKT = 32;   // K staged through shared memory in 32-wide slices

template <typename T>
__global__ void __launch_bounds__(256) working_matmul_kernel(
    const T* __restrict__ a, int64_t sa_i, int64_t sa_k, const T* __restrict__ b, int64_t sb_k,
    int64_t sb_j, int64_t M, int64_t N, int64_t K, T* __restrict__ c) {
    __shared__ float sa[kT][kKT + 1];
    __shared__ float sb[kKT][kT + 1];
    const int tx = threadIdx.x % kT, ty = threadIdx.x / kT;
    const int64_t i0 = static_cast<int64_t>(blockIdx.y) * kT, j0 = static_cast<int64_t>(blockIdx.x) * kT;
    float acc = 0.0f;
    for (int64_t k0 = 0; k0 < K; k0 += kKT) {
        for (int e = threadIdx.x; e < kT * kKT; e += 256) {
            const int r = e / kKT, kk = e % kKT;
            const int64_t gi = i0 + r, gk = k0 + kk;
            sa[r][kk] = (gi < M && gk < K) ? Elem<T>::to_f(a[gi * sa_i + gk * sa_k]) : 0.0f;
        }
        for (int e = threadIdx.x; e < kKT * kT; e += 256) {
            const int kk = e / kT, cc = e % kT;
            const int64_t gk = k0 + kk, gj = j0 + cc;
            sb[kk][cc] = (gk < K && gj < N) ? Elem<T>::to_f(b[gk * sb_k + gj * sb_j]) : 0.0f;
        }
        __syncthreads();
        const int kn = static_cast<int>(K - k0 < kKT ? K - k0 : kKT);
        for (int kk = 0; kk < kn; ++kk) acc = __fadd_rn(acc, __fmul_rn(sa[ty][kk], sb[kk][tx]));
        __syncthreads();
    }
    const int64_t i = i0 + ty, j = j0 + tx;
    if (i < M && j < N) c[i * N + j] = Elem<T>::from_f(acc);
}

template <typename T>
cudaError_t launch_t(const void* a, int64_t sa_i, int64_t sa_k, const void* b, int64_t sb_k,
                     int64_t sb_j, int64_t M, int64_t N, int64_t K, void* c, cudaStream_t st) {
    const dim3 grid(static_cast<unsigned>((N + kT - 1) / kT), static_cast<unsigned>((M + kT - 1) / kT));
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
    if (M > 65535LL * kT) return cudaErrorInvalidValue;
    if (launches) ++*launches;
    switch (dt) {
        case kF32: return launch_t<float>(a, sa_i, sa_k, b, sb_k, sb_j, M, N, K, c, st);
        case kBF16: return launch_t<__nv_bfloat16>(a, sa_i, sa_k, b, sb_k, sb_j, M, N, K, c, st);
        default: return launch_t<__half>(a, sa_i, sa_k, b, sb_k, sb_j, M, N, K, c, st);
    }
}

}  // namespace dfx
