// comm.cu — symmetric-memory all-reduce of the d_in-split norm's exchange (SURVEY 8(e)/8(f)
// row 3; the paper's FSDP2 gap).
//
// Every rank owns one symmetric allocation (same layout on every rank):
//   [data: count fp32, 256-byte padded][start flags][end flags][epochs][error word]
// and maps every peer's allocation into its address space (CUDA IPC across processes, plain
// pointers for ranks that share a process).  dfx_norm_partial writes the rank's
// {G, base_sq, cross} straight into its data region; one kernel then
//   1. entry barrier: block b of every rank tells block b of every peer that it started (its
//      data, written by the stream's earlier kernels, is complete) and waits for all of them;
//   2. reduce: out[i] = ((d_0[i] + d_1[i]) + d_2[i]) + ... in RANK ORDER, reading every peer's
//      data over NVLink (peer loads, 16 bytes per access, L1 bypassed) — every rank computes
//      the identical bits, independent of timing;
//   3. exit barrier: block b waits until block b of every rank finished reading slice b, so
//      when the kernel completes on a rank, no peer still reads its data region and the next
//      call's partial kernel may overwrite it.
// The message is small (r*r + 2*d_out fp32 = 0.66 MB at C2): a one-shot kernel, one launch,
// no host synchronisation, capturable in CUDA graphs (the per-block epochs live in device
// memory).  Spins are bounded (~5 s of %globaltimer): a missing peer sets the error word
// (dfx_comm_status) instead of hanging the GPU.
#include <cstdint>

#include "launch.h"

namespace dfx {

namespace {

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ uint64_t globaltimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ float4 ld_peer(const float4* p) {
    float4 v;
    asm volatile("ld.global.relaxed.sys.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p));
    return v;
}

__device__ __forceinline__ float ld_peer1(const float* p) {
    float v;
    asm volatile("ld.global.relaxed.sys.f32 %0, [%1];" : "=f"(v) : "l"(p));
    return v;
}

constexpr uint64_t kSpinNs = 5ull * 1000 * 1000 * 1000;

// Thread k < world of the block signals peer k's flag slot [block][my rank] and waits for its
// own slot [block][k]; the CTA barrier then publishes the acquired state to the whole block.
__device__ __forceinline__ void block_barrier(const CommArgs& a, size_t flags_off, uint32_t e) {
    const int k = threadIdx.x;
    if (k < a.world) {
        __threadfence_system();
        uint32_t* remote = reinterpret_cast<uint32_t*>(a.peers[k] + flags_off) +
                           blockIdx.x * kCommMaxRanks + a.rank;
        st_release_sys(remote, e);
        const uint32_t* mine = reinterpret_cast<const uint32_t*>(a.peers[a.rank] + flags_off) +
                               blockIdx.x * kCommMaxRanks + k;
        const uint64_t t0 = globaltimer();
        while (ld_acquire_sys(mine) < e) {
            if (globaltimer() - t0 > kSpinNs) {
                atomicExch(reinterpret_cast<uint32_t*>(a.peers[a.rank] + a.err_off), 1u);
                break;
            }
        }
        __threadfence_system();
    }
    __syncthreads();
}

__global__ void __launch_bounds__(kCommThreads) allreduce_oneshot(const CommArgs a) {
    uint32_t* epoch = reinterpret_cast<uint32_t*>(a.peers[a.rank] + a.epoch_off) + blockIdx.x;
    __shared__ uint32_t e_sh;
    if (threadIdx.x == 0) e_sh = *epoch + 1;
    __syncthreads();
    const uint32_t e = e_sh;
    block_barrier(a, a.start_off, e);

    const int64_t n4 = a.count / 4;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += stride) {
        float4 acc = ld_peer(reinterpret_cast<const float4*>(a.peers[0]) + i);
        for (int k = 1; k < a.world; ++k) {
            const float4 v = ld_peer(reinterpret_cast<const float4*>(a.peers[k]) + i);
            acc.x = __fadd_rn(acc.x, v.x);
            acc.y = __fadd_rn(acc.y, v.y);
            acc.z = __fadd_rn(acc.z, v.z);
            acc.w = __fadd_rn(acc.w, v.w);
        }
        reinterpret_cast<float4*>(a.out)[i] = acc;
    }
    for (int64_t i = 4 * n4 + int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < a.count;
         i += stride) {
        float acc = ld_peer1(reinterpret_cast<const float*>(a.peers[0]) + i);
        for (int k = 1; k < a.world; ++k)
            acc = __fadd_rn(acc, ld_peer1(reinterpret_cast<const float*>(a.peers[k]) + i));
        a.out[i] = acc;
    }
    __syncthreads();
    block_barrier(a, a.end_off, e);
    if (threadIdx.x == 0) *epoch = e;
}

}  // namespace

cudaError_t launch_allreduce(const CommArgs& a, cudaStream_t st, int* launches) {
    if (a.count <= 0) return cudaSuccess;
    const int64_t n4 = (a.count + 3) / 4;
    int blocks = static_cast<int>((n4 + kCommThreads - 1) / kCommThreads);
    if (blocks > a.max_blocks) blocks = a.max_blocks;
    if (blocks < 1) blocks = 1;
    prof_begin("norm_allreduce", st);
    allreduce_oneshot<<<blocks, kCommThreads, 0, st>>>(a);
    prof_end(st);
    if (launches) ++*launches;
    return cudaGetLastError();
}

}  // namespace dfx
