// mma_ts_micro.cu — tcgen05.mma issue cost vs N with the M-side operand in shared memory
// (SS) or in tensor memory (TS), 1-SM (M=128) and 2-SM (M=256).  Development tool, not
// product: decides whether staging the W tile in TMEM lifts the N=192 UMMA rate.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I../paper_2603_22276_b200/csrc/kernels mma_ts_micro.cu -o mma_ts_micro
#include <cstdio>
#include <cuda_runtime.h>
#include "ptx.cuh"
using namespace dfx;

__device__ __forceinline__ void umma_ts(uint32_t d, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                        uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
        "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_ts_pair(uint32_t d, uint32_t a_tmem, uint64_t bdesc,
                                             uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
        "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc));
}

template <int kPair, int kTs>
__global__ void __launch_bounds__(128, 1) mma_loop(int n, int iters, long long* cycles, int per_commit, int variant) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sa = smem;              // 128 rows x 128 B
    uint8_t* sb = smem + 16384;      // up to 256 rows x 128 B
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 16384 + 32768);
    uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 10);
    for (int i = threadIdx.x; i < (16384 + 32768) / 4; i += blockDim.x) {
        uint32_t v = 0x3c003c00u;
        if (variant >= 3) {   // random bf16 pairs (exponent kept sane)
            uint32_t h = (uint32_t(i) * 2654435761u) ^ (blockIdx.x * 97u);
            h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
            v = (h & 0x80ff80ffu) | 0x3f003f00u;
        }
        reinterpret_cast<uint32_t*>(smem)[i] = v;
    }
    if (threadIdx.x == 0) { for (int i = 0; i < 10; ++i) mbar_init(&bar[i], 1); slot[4] = 0; fence_mbar_init(); }
    if (threadIdx.x / 32 == 0) { if (kPair) tmem_alloc_pair<512>(slot); else tmem_alloc<512>(slot); }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before(); __syncthreads(); if (kPair) cluster_sync(); tc_fence_after();
    const uint32_t tmem = *slot;
    const bool issuer = threadIdx.x == 0 && (!kPair || cluster_ctarank() == 0);
    long long t0 = clock64();
    if (variant == 4 && threadIdx.x >= 32) {
        // three warps stream 16-byte stores into a 64 KB scratch region until the issuer is done
        uint8_t* scratch = smem + 16384 + 32768 + 2048;
        volatile uint32_t* flag = reinterpret_cast<volatile uint32_t*>(slot + 4);
        uint32_t x = threadIdx.x;
        while (*flag == 0) {
            for (int r = 0; r < 64; ++r) {
                const int off = ((threadIdx.x - 32) * 16 + r * 96 * 16) & (65536 - 16);
                asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(smem_u32(scratch + off)), "r"(x));
            }
            ++x;
        }
    }
    if (issuer) {
        const uint32_t idesc = umma_idesc_f16(1u, kPair ? 256 : 128, n);
        const uint32_t a = smem_u32(sa), b = smem_u32(sb);
        uint32_t ph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        const int groups = iters * 4 / per_commit;
        for (int it = 0; it < groups; ++it) {
            const int s = it & 7;
            if (it >= 8 && variant != 2) { mbar_wait(&bar[s], ph[s]); ph[s] ^= 1; }
            for (int k = 0; k < per_commit; ++k) {
                const int kk = k & 3;
                const uint64_t bd = umma_desc_k_sw128(b + kk * 32);
                if (kTs) {
                    const uint32_t at = tmem + 256u + uint32_t(kk) * 8u;   // A: 8 columns per K=16
                    if (kPair) umma_ts_pair(tmem, at, bd, idesc, 1); else umma_ts(tmem, at, bd, idesc, 1);
                } else {
                    const uint64_t ad = umma_desc_k_sw128(a + kk * 32);
                    if (kPair) umma_f16_pair(tmem, ad, bd, idesc, 1); else umma_f16(tmem, ad, bd, idesc, 1);
                }
            }
            if (kPair) umma_commit_pair_mc(&bar[s], 0x1); else umma_commit(&bar[s]);
            if (variant == 1) { if (kPair) umma_commit_pair_mc(&bar[s ^ 1], 0x1); else umma_commit(&bar[s ^ 1]); }
        }
        if (variant == 2) {
            if (kPair) umma_commit_pair_mc(&bar[9], 0x1); else umma_commit(&bar[9]);
            mbar_wait(&bar[9], 0);
            cycles[blockIdx.x] = clock64() - t0;
        }
        if (variant == 2) {} else
        for (int j = 0; j < 8; ++j) {
            const int it = groups + j; const int s = it & 7;
            if (it >= 8) { mbar_wait(&bar[s], ph[s]); ph[s] ^= 1; }
        }
        cycles[blockIdx.x] = clock64() - t0;
        *reinterpret_cast<volatile uint32_t*>(slot + 4) = 1;
    }
    tc_fence_before(); __syncthreads(); if (kPair) cluster_sync();
    if (threadIdx.x / 32 == 0) { tc_fence_after(); if (kPair) tmem_dealloc_pair<512>(tmem); else tmem_dealloc<512>(tmem); }
}

template <int kPair, int kTs>
void run(int n, int per_commit, int sms, long long* d, int variant = 0) {
    const int iters = 4000, smem = 16384 + 32768 + 2048 + 65536 + 1024;
    auto kern = mma_loop<kPair, kTs>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int grid = kPair ? (sms / 2) * 2 : sms;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid); cfg.blockDim = dim3(128); cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = kPair ? 2 : 1; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float ms = 0;
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        cudaError_t err = cudaLaunchKernelEx(&cfg, kern, n, iters, d, per_commit, variant);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        if (err != cudaSuccess || cudaGetLastError() != cudaSuccess) { printf("launch failed\n"); return; }
    }
    cudaEventElapsedTime(&ms, e0, e1);
    long long h[512]; cudaMemcpy(h, d, sizeof(long long) * 512, cudaMemcpyDeviceToHost);
    const double instr = double(iters) * 4;
    printf("v%d %s %s M=%d N=%3d commit/%d: %.1f us, %.1f cycles/UMMA -> %.0f MAC/clk/SM, %.0f TFLOP/s chip\n",
           variant, kTs ? "TS" : "SS", kPair ? "2-SM" : "1-SM", kPair ? 256 : 128, n, per_commit, ms * 1e3,
           double(h[0]) / instr, instr * 128 * n * 16 / double(h[0]),
           2.0 * instr * 128.0 * n * 16 * grid / (ms * 1e-3) / 1e12);
}

int main() {
    setvbuf(stdout, nullptr, _IONBF, 0);
    int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    long long* d; cudaMalloc(&d, sizeof(long long) * 512);
    for (int v : {0, 3, 4}) for (int pc : {8, 16, 32}) {
        run<1, 0>(192, pc, sms, d, v);
    }
    for (int v : {0, 3}) run<1, 0>(256, 16, sms, d, v);
    return 0;
}
