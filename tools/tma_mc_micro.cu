// tma_mc_micro.cu — does TMA multicast raise the per-SM operand ingest of the W.A^T kernel?
// Each CTA streams, per K block, a private 16 KB "W" slab (HBM, read once) and a shared
// "A" slab of kA bytes (L2-resident, the same for every CTA).  Unicast: every CTA fetches all
// of A.  Multicast (cluster of C): CTA q fetches A's q-th 1/C and multicasts it to the cluster.
// Reports delivered bytes per SM per cycle.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I paper_2603_22276_b200/csrc/kernels tools/tma_mc_micro.cu -o tools/tma_mc_micro
#include <cstdio>
#include <cuda_runtime.h>

#include "ptx.cuh"

using namespace dfx;

constexpr int kStages = 4;
constexpr uint32_t kW = 16384;

__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void bulk_load_mc(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                             uint16_t mask) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
        " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "h"(mask)
        : "memory");
}

template <int C>
__global__ void __launch_bounds__(64) stream_kernel(const char* __restrict__ w, const char* __restrict__ a,
                                                    uint32_t kA, int iters, long long* cycles, size_t wrap) {
    extern __shared__ __align__(1024) char smem[];
    __shared__ uint64_t full[kStages], empty[kStages];
    const uint32_t stage_bytes = kW + kA;
    const uint32_t rank = C > 1 ? cluster_ctarank() : 0;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], C);
        }
        fence_mbar_init();
    }
    __syncthreads();
    if (C > 1) cluster_sync();
    const long long t0 = clock64();
    if (threadIdx.x == 0) {                      // producer
        for (int it = 0; it < iters; ++it) {
            const int s = it % kStages;
            if (it >= kStages) mbar_wait(&empty[s], ((it / kStages) - 1) & 1);
            char* dst = smem + s * stage_bytes;
            mbar_arrive_expect_tx(&full[s], stage_bytes);
            bulk_load(dst, w + ((static_cast<size_t>(blockIdx.x) * iters + it) % wrap) * kW, kW, &full[s]);
            const char* asrc = a + static_cast<size_t>(it % 64) * kA;
            if (C == 1) {
                bulk_load(dst + kW, asrc, kA, &full[s]);
            } else {
                const uint32_t part = kA / C;
                bulk_load_mc(dst + kW + rank * part, asrc + rank * part, part, &full[s],
                             static_cast<uint16_t>((1u << C) - 1));
            }
        }
    } else if (threadIdx.x == 32) {              // consumer: release the stage cluster-wide
        for (int it = 0; it < iters; ++it) {
            const int s = it % kStages;
            mbar_wait(&full[s], (it / kStages) & 1);
            if (C == 1) {
                mbar_arrive(&empty[s]);
            } else {
                for (uint32_t q = 0; q < static_cast<uint32_t>(C); ++q)
                    mbar_arrive_remote(mapa_shared(smem_u32(&empty[s]), q), 1);
            }
        }
    }
    __syncthreads();
    if (C > 1) cluster_sync();
    if (threadIdx.x == 0) cycles[blockIdx.x] = clock64() - t0;
}

template <int C>
void run(const char* w, const char* a, uint32_t kA, int iters, long long* cyc, int sms, size_t wrap) {
    const int grid = (sms / C) * C;
    const size_t smem = kStages * (kW + kA);
    cudaFuncSetAttribute(stream_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(64);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        cudaError_t err = cudaLaunchKernelEx(&cfg, stream_kernel<C>, w, a, kA, iters, cyc, wrap);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        if (err != cudaSuccess || cudaGetLastError() != cudaSuccess) {
            std::printf("C=%d launch failed: %s\n", C, cudaGetErrorString(err));
            return;
        }
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        long long h[1];
        cudaMemcpy(h, cyc, sizeof(long long), cudaMemcpyDeviceToHost);
        const double per_sm = double(kW + kA) * iters / double(h[0]);
        if (rep == 2)
            std::printf("wrap=%zu C=%d grid=%d kA=%u: %.1f us, %.1f B/clk/SM delivered (W+A), chip %.2f TB/s delivered\n",
                        wrap, C, grid, kA, ms * 1e3, per_sm, double(kW + kA) * iters * grid / (ms * 1e-3) / 1e12);
    }
}

int main() {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int iters = 128;
    char *w, *a;
    long long* cyc;
    cudaMalloc(&w, size_t(sms) * iters * kW);
    cudaMalloc(&a, size_t(64) * 32768);
    cudaMalloc(&cyc, sizeof(long long) * sms);
    cudaMemset(w, 1, size_t(sms) * iters * kW);
    cudaMemset(a, 2, size_t(64) * 32768);
    for (size_t wrap : {size_t(sms) * iters, size_t(2048)}) {   // W from HBM / W L2-resident
        for (uint32_t kA : {12288u, 24576u}) {
            run<1>(w, a, kA, iters, cyc, sms, wrap);
            run<2>(w, a, kA, iters, cyc, sms, wrap);
            run<4>(w, a, kA, iters, cyc, sms, wrap);
            run<8>(w, a, kA, iters, cyc, sms, wrap);
        }
        run<1>(w, a, 12288u, iters, cyc, 64, wrap);
        run<4>(w, a, 12288u, iters, cyc, 64, wrap);
        run<8>(w, a, 12288u, iters, cyc, 64, wrap);
    }
    return 0;
}
