// tma_tensor_micro.cu — per-SM ingest of the W.A^T operand stream with TENSOR TMA boxes.
// Each CTA streams the K blocks of one 128-row W tile (box {64, 128}, SW128) plus a 96-row A
// slab (box {64, 96}) per K block, exactly the U kernel's per-SM operand traffic, with no MMA.
// Variants: 2-D boxes (one K block per request) vs 3-D boxes {64, rows, kk} that fetch kk
// consecutive K blocks per request (rows then carry kk*128 contiguous bytes in global memory),
// and the L2 promotion setting.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lcuda \
//        -I paper_2603_22276_b200/csrc/kernels tools/tma_tensor_micro.cu -o tools/tma_tensor_micro
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdio>

#include "ptx.cuh"

using namespace dfx;

constexpr int kStages = 6;
constexpr int kStages8 = 8;
constexpr int kRowsW = 128, kRowsA = 96;
constexpr uint32_t kBlockBytes = (kRowsW + kRowsA) * 128;   // one K block of W + A: 28 KB

__device__ __forceinline__ void tma_load_3d(const void* desc, uint64_t* bar, void* dst, int32_t c0,
                                            int32_t c1, int32_t c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(desc)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}

template <int KK>   // K blocks per request (1 = 2-D boxes)
__global__ void __launch_bounds__(64) ingest_kernel(const __grid_constant__ CUtensorMap tw,
                                                    const __grid_constant__ CUtensorMap ta, int kblocks,
                                                    int wtiles, long long* cycles) {
    extern __shared__ __align__(1024) char smem_raw[];
    char* smem = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t full[kStages], empty[kStages];
    const uint32_t stage_bytes = kBlockBytes * KK;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        fence_mbar_init();
    }
    __syncthreads();
    const int row0 = (blockIdx.x % wtiles) * kRowsW;
    const int arow0 = ((blockIdx.x / wtiles) % 4) * kRowsA;
    const int iters = kblocks / KK;
    const long long t0 = clock64();
    if (threadIdx.x == 0) {
        const uint64_t pol = policy_evict_first();
        for (int it = 0; it < iters; ++it) {
            const int s = it % kStages;
            if (it >= kStages) mbar_wait(&empty[s], ((it / kStages) - 1) & 1);
            char* dst = smem + s * stage_bytes;
            mbar_arrive_expect_tx(&full[s], stage_bytes);
            if (KK == 1) {
                tma_load_2d(&tw, &full[s], dst, it * 64, row0, pol);
                tma_load_2d(&ta, &full[s], dst + kRowsW * 128, it * 64, arow0, pol);
            } else {
                tma_load_3d(&tw, &full[s], dst, 0, row0, it * KK);
                tma_load_3d(&ta, &full[s], dst + KK * kRowsW * 128, 0, arow0, it * KK);
            }
        }
    } else if (threadIdx.x == 32) {
        for (int it = 0; it < iters; ++it) {
            const int s = it % kStages;
            mbar_wait(&full[s], (it / kStages) & 1);
            mbar_arrive(&empty[s]);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) cycles[blockIdx.x] = clock64() - t0;
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode() {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    return reinterpret_cast<EncodeFn>(fn);
}

// kk = 1: 2-D map {cols, rows}, box {64, box_rows}; kk > 1: 3-D view {64, rows, cols/64}
CUtensorMap make_map(void* base, uint64_t rows, uint64_t cols, uint32_t box_rows, int kk,
                     CUtensorMapL2promotion promo) {
    CUtensorMap m;
    const cuuint32_t estr[3] = {1, 1, 1};
    CUresult r;
    if (kk == 1) {
        const cuuint64_t dims[2] = {cols, rows};
        const cuuint64_t str[1] = {cols * 2};
        const cuuint32_t box[2] = {64, box_rows};
        r = encode()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, str, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, promo,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    } else {
        const cuuint64_t dims[3] = {64, rows, cols / 64};
        const cuuint64_t str[2] = {cols * 2, 128};
        const cuuint32_t box[3] = {64, box_rows, static_cast<cuuint32_t>(kk)};
        r = encode()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, base, dims, str, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, promo,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    if (r != CUDA_SUCCESS) std::printf("encode failed %d\n", int(r));
    return m;
}

template <int KK>
void run(void* w, void* a, uint64_t d_out, uint64_t d_in, int grid, CUtensorMapL2promotion promo,
         long long* cyc, const char* tag) {
    const CUtensorMap tw = make_map(w, d_out, d_in, kRowsW, KK, promo);
    const CUtensorMap ta = make_map(a, 384, d_in, kRowsA, KK, promo);
    const size_t smem = kStages * kBlockBytes * KK + 1024;
    if (smem > 227 * 1024) return;
    cudaFuncSetAttribute(ingest_kernel<KK>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int kblocks = static_cast<int>(d_in / 64), wtiles = static_cast<int>(d_out / kRowsW);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        ingest_kernel<KK><<<grid, 64, smem>>>(tw, ta, kblocks, wtiles, cyc);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        if (cudaGetLastError() != cudaSuccess) {
            std::printf("%s: launch failed\n", tag);
            return;
        }
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        long long h;
        cudaMemcpy(&h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
        if (rep == 2)
            std::printf("%-28s kk=%d grid=%3d d_out=%5lu: %6.1f us, %5.1f B/clk/SM, chip %.2f TB/s\n", tag, KK, grid,
                        (unsigned long)d_out, ms * 1e3, double(kBlockBytes) * kblocks / double(h),
                        double(kBlockBytes) * kblocks * grid / (ms * 1e-3) / 1e12);
    }
}

// Pair modes, cluster of 2 (the U kernel's cta_group::2 layout): every CTA loads its own W
// tile and A half.  kMode 1: loads complete on the LEADER's full barrier (cta_group::2 form,
// what u_rowdot_tc does); kMode 2: loads complete locally and the peer forwards "landed" to
// the leader with a remote arrive.  The leader's consumer releases both CTAs' stages.
template <int kMode>
__global__ void __launch_bounds__(256) pair_kernel(const __grid_constant__ CUtensorMap tw,
                                                  const __grid_constant__ CUtensorMap ta, int kblocks,
                                                  int wtiles, long long* cycles) {
    extern __shared__ __align__(1024) char smem_raw[];
    char* smem = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t full[8], empty[8], done;
    const int stages = kStages8;
    const uint32_t rank = cluster_ctarank();
    if (threadIdx.x == 0) mbar_init(&done, 1);
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            mbar_init(&full[s], kMode == 2 && rank == 0 ? 2 : 1);
            mbar_init(&empty[s], 1);
        }
        fence_mbar_init();
    }
    __syncthreads();
    cluster_sync();
    const int pair = blockIdx.x / 2;
    const int row0 = ((pair / 2) % wtiles) * 2 * kRowsW + rank * kRowsW;
    const int arow0 = (pair % 2) * 2 * kRowsA + rank * kRowsA;
    const long long t0 = clock64();
    if (threadIdx.x == 0) {
        const uint64_t pol = policy_evict_last();
        for (int it = 0; it < kblocks; ++it) {
            const int s = it % stages;
            if (it >= stages) mbar_wait(&empty[s], ((it / stages) - 1) & 1);
            char* dst = smem + s * kBlockBytes;
            if (kMode == 1) {
                if (rank == 0) mbar_arrive_expect_tx(&full[s], 2 * kBlockBytes);
                const uint32_t lbar = mapa_shared(smem_u32(&full[s]), 0);
                tma_load_2d_pair(&tw, lbar, dst, it * 64, row0, pol);
                tma_load_2d_pair(&ta, lbar, dst + kRowsW * 128, it * 64, arow0, pol);
            } else {
                mbar_arrive_expect_tx(&full[s], kBlockBytes);
                tma_load_2d(&tw, &full[s], dst, it * 64, row0, pol);
                tma_load_2d(&ta, &full[s], dst + kRowsW * 128, it * 64, arow0, pol);
            }
        }
    } else if (blockDim.x > 64 && threadIdx.x >= 64 && threadIdx.x < 192 && kMode == 1) {
        mbar_wait(&done, 0);          // 4 warps idle-spinning for the whole stream (like the
                                      // norm kernel's epilogue warps waiting for the accumulator)
    } else if (threadIdx.x == 32) {
        for (int it = 0; it < kblocks; ++it) {
            const int s = it % stages;
            if (rank == 0) {
                mbar_wait(&full[s], (it / stages) & 1);
                mbar_arrive(&empty[s]);
                mbar_arrive_remote(mapa_shared(smem_u32(&empty[s]), 1), 1);
            } else if (kMode == 2) {
                mbar_wait(&full[s], (it / stages) & 1);
                mbar_arrive_remote(mapa_shared(smem_u32(&full[s]), 0), 1);
            }
        }
    }
    if (threadIdx.x == 32) mbar_arrive(&done);
    __syncthreads();
    cluster_sync();
    if (threadIdx.x == 0) cycles[blockIdx.x] = clock64() - t0;
}

template <int kMode>
void run_pair(void* w, void* a, uint64_t d_out, uint64_t d_in, int grid, long long* cyc, const char* tag,
              int threads = 64) {
    const CUtensorMap tw = make_map(w, d_out, d_in, kRowsW, 1, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
    const CUtensorMap ta = make_map(a, 384, d_in, kRowsA, 1, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
    const size_t smem = kStages8 * kBlockBytes + 1024;
    cudaFuncSetAttribute(pair_kernel<kMode>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int kblocks = static_cast<int>(d_in / 64), wtiles = static_cast<int>(d_out / (2 * kRowsW));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        cudaError_t err = cudaLaunchKernelEx(&cfg, pair_kernel<kMode>, tw, ta, kblocks, wtiles, cyc);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        if (err != cudaSuccess || cudaGetLastError() != cudaSuccess) {
            std::printf("%s: launch failed\n", tag);
            return;
        }
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        long long h;
        cudaMemcpy(&h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
        if (rep == 2)
            std::printf("%-28s grid=%3d d_out=%5lu: %6.1f us, %5.1f B/clk/SM, chip %.2f TB/s\n", tag, grid,
                        (unsigned long)d_out, ms * 1e3, double(kBlockBytes) * kblocks / double(h),
                        double(kBlockBytes) * kblocks * grid / (ms * 1e-3) / 1e12);
    }
}

__global__ void fill_hash(uint32_t* p, size_t n) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
        uint32_t x = static_cast<uint32_t>(i) * 2654435761u;
        x ^= x >> 15;
        p[i] = x * 2246822519u;
    }
}

int main(int argc, char** argv) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const uint64_t d_in = 8192;
    void *w, *a;
    long long* cyc;
    cudaMalloc(&w, 8192ull * d_in * 2);
    cudaMalloc(&a, 384ull * d_in * 2);
    cudaMalloc(&cyc, sizeof(long long) * sms);
    const bool zeros = argc > 1;
    cudaMemset(w, 0, 8192ull * d_in * 2);
    cudaMemset(a, 0, 384ull * d_in * 2);
    if (!zeros) {
        fill_hash<<<1024, 256>>>(static_cast<uint32_t*>(w), 8192ull * d_in / 2);
        fill_hash<<<64, 256>>>(static_cast<uint32_t*>(a), 384ull * d_in / 2);
    }
    std::printf("data: %s\n", zeros ? "zeros" : "hashed");
    for (uint64_t d_out : {8192ull, 1024ull}) {   // W from HBM (128 MB) / W L2-resident (16 MB)
        run<1>(w, a, d_out, d_in, sms, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, cyc, "single, 148 CTAs");
        run<1>(w, a, d_out, d_in, 128, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, cyc, "single, 128 CTAs");
        run_pair<1>(w, a, d_out, d_in, 128, cyc, "pair, leader-barrier loads");
        run_pair<1>(w, a, d_out, d_in, 128, cyc, "pair, leader-barrier, 256 thr + 4 spinning warps", 256);
        run_pair<2>(w, a, d_out, d_in, 128, cyc, "pair, local + forward");
        run_pair<1>(w, a, d_out, d_in, 64, cyc, "pair, leader-barrier, 64");
        run_pair<2>(w, a, d_out, d_in, 64, cyc, "pair, local + forward, 64");
    }
    return 0;
}
