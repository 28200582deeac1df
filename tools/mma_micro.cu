// mma_micro.cu — tcgen05.mma throughput microbenchmark (development tool, not product).
// Each CTA (one per SM) issues `iters` x 4 UMMAs (K=16 each) from resident smem tiles
// into TMEM, committing to an mbarrier every 4 instructions and keeping `depth` commit
// groups in flight.  Reports MAC/cycle/SM for 1-SM (M=128) and 2-SM (M=256) shapes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2603_22276_b200/csrc/kernels mma_micro.cu -o mma_micro
#include <cstdio>
#include <cuda_runtime.h>
#include "ptx.cuh"
using namespace dfx;

template <int kPair>
__global__ void __launch_bounds__(128, 1) mma_loop(int n, int iters, long long* cycles, int inter) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sa = smem;              // 128 rows x 128 B (one K=64 block of A)
    uint8_t* sb = smem + 16384;      // up to 256 rows x 128 B
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 16384 + 32768);
    uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 8);
    for (int i = threadIdx.x; i < (16384 + 32768) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
    if (threadIdx.x == 0) { for (int i = 0; i < 8; ++i) mbar_init(&bar[i], 1); fence_mbar_init(); }
    if (threadIdx.x / 32 == 0) { if (kPair) tmem_alloc_pair<512>(slot); else tmem_alloc<512>(slot); }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before(); __syncthreads(); if (kPair) cluster_sync(); tc_fence_after();
    const uint32_t tmem = *slot;
    const bool issuer = threadIdx.x == 0 && (!kPair || cluster_ctarank() == 0);
    long long t0 = clock64();
    if (issuer) {
        const uint32_t idesc = umma_idesc_f16(1u, kPair ? 256 : 128, n);
        const uint32_t a = smem_u32(sa), b = smem_u32(sb);
        uint32_t ph[8] = {0,0,0,0,0,0,0,0};
        for (int it = 0; it < iters; ++it) {
            const int s = it & 7;
            if (it >= 8) { mbar_wait(&bar[s], ph[s]); ph[s] ^= 1; }
            for (int k = 0; k < 4; ++k) {
                const uint32_t acc = tmem + (inter ? uint32_t(k & 1) * uint32_t(n) : 0u);
                if (kPair) umma_f16_pair(acc, umma_desc_k_sw128(a + k * 32), umma_desc_k_sw128(b + k * 32), idesc, 1);
                else umma_f16(acc, umma_desc_k_sw128(a + k * 32), umma_desc_k_sw128(b + k * 32), idesc, 1);
            }
            if (kPair) umma_commit_pair_mc(&bar[s], 0x1); else umma_commit(&bar[s]);
        }
        for (int j = 0; j < 8; ++j) { const int it = iters + j; const int s = it & 7; if (it >= 8) { mbar_wait(&bar[s], ph[s]); ph[s] ^= 1; } }
        cycles[blockIdx.x] = clock64() - t0;
    }
    tc_fence_before(); __syncthreads(); if (kPair) cluster_sync();
    if (threadIdx.x / 32 == 0) { tc_fence_after(); if (kPair) tmem_dealloc_pair<512>(tmem); else tmem_dealloc<512>(tmem); }
}

int main() {
    int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    long long* d; cudaMalloc(&d, sizeof(long long) * 512);
    const int iters = 4000, smem = 16384 + 32768 + 2048;
    cudaFuncSetAttribute(mma_loop<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(mma_loop<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int inter = 0; inter < 2; ++inter) for (int pair = 0; pair < 2; ++pair) for (int n : {64, 128, 192, 256}) {
        const int grid = pair ? (sms / 2) * 2 : sms;
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(grid); cfg.blockDim = dim3(128); cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = pair ? 2 : 1; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        cfg.attrs = at; cfg.numAttrs = 1;
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            cudaError_t err = pair ? cudaLaunchKernelEx(&cfg, mma_loop<1>, n, iters, d, inter) : cudaLaunchKernelEx(&cfg, mma_loop<0>, n, iters, d, inter);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            if (err != cudaSuccess || cudaGetLastError() != cudaSuccess) { printf("launch failed %s\n", cudaGetErrorString(err)); return 1; }
        }
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        long long h[512]; cudaMemcpy(h, d, sizeof(long long) * 512, cudaMemcpyDeviceToHost);
        const double macs_per_sm = double(iters) * 4 * 128 * n * 16;   // per SM (M=128 rows each)
        const long long cyc = h[0];
        printf("%s%s M=%d N=%3d: %.1f us, %lld cycles on CTA0 -> %.0f MAC/cycle/SM, %.0f TFLOP/s chip\n",
               inter ? "2acc " : "", pair ? "2-SM" : "1-SM", pair ? 256 : 128, n, ms * 1e3, cyc, macs_per_sm / cyc,
               2.0 * macs_per_sm * (pair ? grid : grid) / (ms * 1e-3) / 1e12);
    }
    return 0;
}
