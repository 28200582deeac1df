// lora_compose.cu — layer_forward's LoRA-up GEMM fused with the compose and the residual
// (reference layer.cpp:57-58, 73-120).
//
// The reference materialises lora = round(mid . B^T) (layer.cpp:58) and then composes
// it with base (compose.cpp:19-24) and adds the residual (layer.cpp:108-120).  Here the
// [rows x d_out] lora never reaches HBM: a persistent warp-specialised tcgen05 kernel
// computes 128 x 256 tiles of mid . B^T into a double-buffered TMEM accumulator (K = r,
// both operands K-major, TMA with the 128-byte swizzle), and the epilogue rounds each
// accumulator to the working dtype (exactly the reference's working_matmul store), then
// applies the canonical compose, the inner of the dual output and the residual
//     lora  = round(acc)
//     delta = round((g-1)*base + g*(s*lora))            compose.cpp:19-24
//     inner = round(s*lora + base)                      compose.cpp:131-137
//     y     = round(base + delta) [then round(y + bias)] layer.cpp:108-120
// with every op an explicit RN fp32 op, so each output is bitwise the reference's given
// the same lora; lora itself is an fp32-accumulated GEMM (its summation order is the
// tensor core's, not the reference's serial k loop).
//
// Epilogue: each thread owns one token row; base arrives through L1 in 64-byte row pieces,
// every dtype rounding is a packed two-value F2FP conversion, and results are written to a
// double-buffered 64-byte-swizzled smem slice (32 columns) that leaves by a
// cp.async.bulk.tensor store (clipped at the tensor edges) while the next slice computes.
//
// Warp roles (320 threads): 0-7 epilogue (warp w owns TMEM lane quadrant w % 4, warps
// 0-3 take column slices 0-1 of a tile, warps 4-7 slices 2-3), 8 operand producer,
// 9 MMA issuer.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <algorithm>

#include "launch.h"
#include "ptx.cuh"

namespace dfx {
namespace {

constexpr int kLM = 128;                      // token rows per tile
constexpr int kLN = 256;                      // d_out columns per tile
constexpr int kLK = 64;                       // K block: one 128-byte swizzle atom
constexpr int kLSlice = 32;                   // epilogue column slice (64-byte swizzle)
constexpr int kLThreads = 320;
#ifndef DFX_LC_AHEAD
#define DFX_LC_AHEAD 1
#endif
// base slices in flight ahead of the arithmetic (1 or 2; 2 measured no faster: 63.2 vs 62.9 us
// at C2, the epilogue is issue-bound — ncu: 160 MB of DRAM traffic in 68 us)
constexpr int kLBaseAhead = DFX_LC_AHEAD;
constexpr int kWProd = 8, kWMma = 9;
constexpr int kAStage = kLM * kLK * 2;        // 16 KiB of mid
constexpr int kBStage = kLN * kLK * 2;        // 32 KiB of B
constexpr int kSlice = kLM * kLSlice * 2;     // 8 KiB
constexpr int kMaxOut = 4;                    // y, delta, inner, lora

struct LcMaps {
    CUtensorMap mid, b;
    CUtensorMap out[kMaxOut];
};

struct LcParams {
    int64_t rows, d_out;
    int kb;                 // K blocks (ceil(r / 64))
    int m_tiles, tiles;
    int stages;
    int n_out;              // enabled outputs, compacted in out[] / the smem buffers
    int slot[kMaxOut];      // kind (0 y, 1 delta, 2 inner, 3 lora) -> buffer index, -1 = off
    float s;
    const float* g;
    const float* bias;      // nullable (values representable in the working dtype)
    const void* base;       // [rows, d_out], read by the epilogue through L1
    int fp16;
};

__device__ __forceinline__ void tma_store_2d(const void* desc, const void* smem_src, int32_t c0,
                                             int32_t c1) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(desc)),
                 "r"(smem_u32(smem_src)), "r"(c0), "r"(c1)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read1() {
    asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ uint4 ldg_nc_v4(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

__device__ __forceinline__ void sts_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c,
                                       uint32_t d) {
    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c),
                 "r"(d)
                 : "memory");
}

template <typename T> struct LcT;
template <> struct LcT<__nv_bfloat16> {
    static __device__ __forceinline__ float rnd(float x) {
        return __bfloat162float(__float2bfloat16_rn(x));
    }
    static __device__ __forceinline__ float lo(uint32_t w) { return __uint_as_float(w << 16); }
    static __device__ __forceinline__ float hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }
    static __device__ __forceinline__ uint32_t pack(float a, float b) {
        __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
        return *reinterpret_cast<uint32_t*>(&h);
    }
};
template <> struct LcT<__half> {
    static __device__ __forceinline__ float rnd(float x) { return __half2float(__float2half_rn(x)); }
    static __device__ __forceinline__ float lo(uint32_t w) {
        return __half2float(__ushort_as_half(static_cast<unsigned short>(w & 0xFFFFu)));
    }
    static __device__ __forceinline__ float hi(uint32_t w) {
        return __half2float(__ushort_as_half(static_cast<unsigned short>(w >> 16)));
    }
    static __device__ __forceinline__ uint32_t pack(float a, float b) {
        __half2 h = __floats2half2_rn(a, b);
        return *reinterpret_cast<uint32_t*>(&h);
    }
};

template <typename T>
__global__ void __launch_bounds__(kLThreads, 1)
    lora_compose_kernel(const __grid_constant__ LcMaps maps, const LcParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    constexpr int kStage = kAStage + kBStage;
    uint8_t* s_out = smem + p.stages * kStage;           // [2 groups][2 buffers][n_out][8 KiB]
    uint64_t* full = reinterpret_cast<uint64_t*>(s_out + 4 * p.n_out * kSlice);
    uint64_t* empty = full + p.stages;
    uint64_t* tmem_full = empty + p.stages;      // [2]
    uint64_t* tmem_empty = tmem_full + 2;        // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);

    __shared__ __align__(16) float s_gw[8][3][kLN / 2];   // epilogue warp: g, g - 1, bias
    const int warp = warp_id(), lane = lane_id();
    if (threadIdx.x == 0) {
        for (int i = 0; i < p.stages; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tmem_full[i], 1);
            mbar_init(&tmem_empty[i], 8);
        }
        fence_mbar_init();
    }
    if (warp == kWMma) tmem_alloc<512>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == kWProd) {
        // ================= mid / B operand producer =================
        if (lane == 0) {
            tma_prefetch_desc(&maps.mid);
            tma_prefetch_desc(&maps.b);
            const uint64_t pol = policy_evict_last();   // mid and B are re-read across tiles
            int s = 0;
            uint32_t ph = 0;
            for (int t = blockIdx.x; t < p.tiles; t += gridDim.x) {
                const int32_t m0 = (t % p.m_tiles) * kLM, n0 = (t / p.m_tiles) * kLN;
                for (int kb = 0; kb < p.kb; ++kb) {
                    mbar_wait(&empty[s], ph ^ 1);
                    mbar_arrive_expect_tx(&full[s], kStage);
                    uint8_t* sa = smem + s * kStage;
                    tma_load_2d(&maps.mid, &full[s], sa, kb * kLK, m0, pol);
                    tma_load_2d(&maps.b, &full[s], sa + kAStage, kb * kLK, n0, pol);
                    if (++s == p.stages) { s = 0; ph ^= 1; }
                }
            }
        }
    } else if (warp == kWMma) {
        // ================= MMA issuer (single thread) =================
        if (lane == 0) {
            const uint32_t idesc = umma_idesc_f16(p.fp16 ? 0u : 1u, kLM, kLN);
            int s = 0;
            uint32_t ph = 0;
            int local = 0;
            for (int t = blockIdx.x; t < p.tiles; t += gridDim.x, ++local) {
                const int slot = local & 1;
                const uint32_t tacc = tmem_base + static_cast<uint32_t>(slot * kLN);
                mbar_wait(&tmem_empty[slot], ((local >> 1) & 1) ^ 1);
                tc_fence_after();
                for (int kb = 0; kb < p.kb; ++kb) {
                    mbar_wait(&full[s], ph);
                    tc_fence_after();
                    const uint32_t sa = smem_u32(smem + s * kStage);
                    const uint32_t sb = sa + kAStage;
#pragma unroll
                    for (int k = 0; k < kLK / 16; ++k)
                        umma_f16(tacc, umma_desc_k_sw128(sa + k * 32), umma_desc_k_sw128(sb + k * 32),
                                 idesc, (kb > 0 || k > 0) ? 1u : 0u);
                    umma_commit(&empty[s]);
                    if (++s == p.stages) { s = 0; ph ^= 1; }
                }
                umma_commit(&tmem_full[slot]);
            }
        }
    } else if (warp < 8) {
        // ================= epilogue: one token row per thread =================
        // Warp w (TMEM lane quadrant q = w % 4) owns the 32 rows 32q.. of each tile and the
        // column half grp = w / 4, in four 32-column slices.  Each slice's outputs go to the
        // warp's part of a double-buffered 64-byte-swizzled smem slice and leave by the
        // warp's own TMA store (32 x 32 box) while the next slice computes: no cross-warp
        // synchronisation in the epilogue.
        const int grp = warp >> 2, q = warp & 3;
        const int row = q * 32 + lane;
        const int sw = (row >> 1) & 3;                          // SWIZZLE_64B chunk XOR
        uint8_t* obase = s_out + grp * 2 * p.n_out * kSlice;    // [2 buffers][n_out][slice]
        float (*gw)[kLN / 2] = s_gw[warp];                      // [g | g - 1 | bias][column]
        const float sf = p.s;
        // this thread's 64-byte base piece of a slice (row clamped in the token tail, columns
        // in the d_out tail; those outputs are clipped by the TMA store), read through L1
        // one slice ahead so the DRAM latency hides behind the current slice's arithmetic
        auto load_base = [&](int tt, int cs, uint4 (&v)[4]) {
            if (tt >= p.tiles) return;
            const int64_t r0 = min(int64_t((tt % p.m_tiles) * kLM + row), p.rows - 1);
            const int64_t c0 = int64_t(tt / p.m_tiles) * kLN + 128 * grp + kLSlice * cs;
            const T* src = static_cast<const T*>(p.base) + r0 * p.d_out;
#pragma unroll
            for (int k = 0; k < 4; ++k)
                v[k] = ldg_nc_v4(src + min(c0 + 8 * k, p.d_out - 8));
        };
        // base runs kLBaseAhead slices ahead of the arithmetic (the epilogue's HBM stream is
        // latency-bound: each thread keeps its next slices' 64-byte pieces in flight)
        uint4 bnext[4], bnext2[4];
        load_base(blockIdx.x, 0, bnext);
        if (kLBaseAhead > 1) load_base(blockIdx.x, 1, bnext2);
        int local = 0, nslice = 0;
        for (int t = blockIdx.x; t < p.tiles; t += gridDim.x, ++local) {
            const int32_t m0 = (t % p.m_tiles) * kLM, n0 = (t / p.m_tiles) * kLN;
            // g, g - 1 and bias for the warp's 128 columns (a missing bias is -0.0, an exact
            // no-op in the fp32 add; columns past d_out are clamped, their outputs clipped)
            {
                const int64_t j = min(int64_t(n0 + 128 * grp + 4 * lane), p.d_out - 4);
                const float4 gv4 = __ldg(reinterpret_cast<const float4*>(p.g + j));
                const float4 bv4 = p.bias ? __ldg(reinterpret_cast<const float4*>(p.bias + j))
                                          : make_float4(-0.0f, -0.0f, -0.0f, -0.0f);
                reinterpret_cast<float4*>(gw[0])[lane] = gv4;
                reinterpret_cast<float4*>(gw[1])[lane] =
                    make_float4(__fsub_rn(gv4.x, 1.0f), __fsub_rn(gv4.y, 1.0f),
                                __fsub_rn(gv4.z, 1.0f), __fsub_rn(gv4.w, 1.0f));
                reinterpret_cast<float4*>(gw[2])[lane] = bv4;
            }
            __syncwarp();
            const int slot = local & 1;
            mbar_wait(&tmem_full[slot], (local >> 1) & 1);
            tc_fence_after();
            for (int cs = 0; cs < 4; ++cs, ++nslice) {
                const int cl = 128 * grp + kLSlice * cs;        // slice's first column in the tile
                const int col0 = n0 + cl;
                uint4 bv[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) bv[k] = bnext[k];
                if (kLBaseAhead > 1) {
#pragma unroll
                    for (int k = 0; k < 4; ++k) bnext[k] = bnext2[k];
                    if (cs < 2) load_base(t, cs + 2, bnext2);
                    else load_base(t + gridDim.x, cs - 2, bnext2);
                } else {
                    if (cs < 3) load_base(t, cs + 1, bnext);
                    else load_base(t + gridDim.x, 0, bnext);
                }
                uint32_t acc[32];
                tmem_ld_32x32b_x32(tmem_base + static_cast<uint32_t>(slot * kLN + cl) +
                                       (static_cast<uint32_t>(q * 32) << 16),
                                   acc);
                tmem_ld_wait();
                if (cs == 3) {                                   // accumulator slot consumed
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&tmem_empty[slot]);
                }
                uint8_t* obuf = obase + (nslice & 1) * p.n_out * kSlice;
                const uint32_t orow = smem_u32(obuf) + static_cast<uint32_t>(row * (kLSlice * 2));
#pragma unroll
                for (int k = 0; k < 4; ++k) {                 // 8 columns per 16-byte chunk
                    const int c8 = kLSlice * cs + 8 * k;        // column within the warp's half
                    const float4 g0 = *reinterpret_cast<const float4*>(&gw[0][c8]);
                    const float4 g1 = *reinterpret_cast<const float4*>(&gw[0][c8 + 4]);
                    const float4 h0 = *reinterpret_cast<const float4*>(&gw[1][c8]);
                    const float4 h1 = *reinterpret_cast<const float4*>(&gw[1][c8 + 4]);
                    const float4 b0 = *reinterpret_cast<const float4*>(&gw[2][c8]);
                    const float4 b1 = *reinterpret_cast<const float4*>(&gw[2][c8 + 4]);
                    const float gv[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
                    const float gm[8] = {h0.x, h0.y, h0.z, h0.w, h1.x, h1.y, h1.z, h1.w};
                    const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
                    const uint32_t bw[4] = {bv[k].x, bv[k].y, bv[k].z, bv[k].w};
                    // element pairs: every dtype rounding is one packed F2FP conversion of
                    // two values (RNE, identical to two scalar roundings), unpacked by shifts
                    uint32_t o[kMaxOut][4];                  // packed y, delta, inner, lora
#pragma unroll
                    for (int e2 = 0; e2 < 4; ++e2) {
                        const int e = 2 * e2;
                        const float b0f = LcT<T>::lo(bw[e2]), b1f = LcT<T>::hi(bw[e2]);
                        const uint32_t lw = LcT<T>::pack(__uint_as_float(acc[8 * k + e]),
                                                         __uint_as_float(acc[8 * k + e + 1]));
                        const float l0 = LcT<T>::lo(lw), l1 = LcT<T>::hi(lw);
                        const float t0 = __fmul_rn(sf, l0), t1 = __fmul_rn(sf, l1);
                        const float u0 = __fmul_rn(gv[e], t0), u1 = __fmul_rn(gv[e + 1], t1);
                        const float v0 = __fmul_rn(gm[e], b0f), v1 = __fmul_rn(gm[e + 1], b1f);
                        const uint32_t dw = LcT<T>::pack(__fadd_rn(v0, u0), __fadd_rn(v1, u1));
                        const uint32_t y0w = LcT<T>::pack(__fadd_rn(b0f, LcT<T>::lo(dw)),
                                                          __fadd_rn(b1f, LcT<T>::hi(dw)));
                        o[0][e2] = p.bias ? LcT<T>::pack(__fadd_rn(LcT<T>::lo(y0w), bb[e]),
                                                         __fadd_rn(LcT<T>::hi(y0w), bb[e + 1]))
                                          : y0w;
                        o[1][e2] = dw;
                        o[2][e2] = LcT<T>::pack(__fadd_rn(t0, b0f), __fadd_rn(t1, b1f));
                        o[3][e2] = lw;
                    }
#pragma unroll
                    for (int kind = 0; kind < kMaxOut; ++kind) {
                        if (p.slot[kind] < 0) continue;      // output not requested (uniform)
                        sts_v4(orow + static_cast<uint32_t>(p.slot[kind] * kSlice + ((k ^ sw) << 4)),
                               o[kind][0], o[kind][1], o[kind][2], o[kind][3]);
                    }
                }
                // the warp's 32 rows of the slice go out by its own TMA store; before the
                // next slice reuses the other buffer, the store issued from it two slices
                // ago must have read its smem
                fence_async_smem();
                __syncwarp();
                if (lane == 0) {
                    for (int oi = 0; oi < p.n_out; ++oi)
                        tma_store_2d(&maps.out[oi], obuf + oi * kSlice + q * 32 * (kLSlice * 2),
                                     col0, m0 + 32 * q);
                    bulk_commit();
                    bulk_wait_read1();
                }
                __syncwarp();
            }
        }
        if (lane == 0) bulk_wait0();
    }
    tc_fence_before();
    __syncthreads();
    if (warp == kWMma) {
        tc_fence_after();
        tmem_dealloc<512>(tmem_base);
    }
}

size_t lc_smem(int stages, int n_out) {
    return size_t(stages) * (kAStage + kBStage) + size_t(4) * n_out * kSlice + 1024 + 256;
}

}  // namespace

cudaError_t launch_lora_compose(int dt, const void* mid, const void* b, const void* base,
                                const float* g, float s, const float* bias, int64_t rows,
                                int64_t d_out, int64_t r, void* y, void* delta, void* inner,
                                void* lora, cudaStream_t st, int* launches) {
    if (rows == 0 || d_out == 0) return cudaSuccess;
    if (dt != kBF16 && dt != kF16) return cudaErrorNotSupported;
    LcMaps maps;
    LcParams p{};
    void* outs[kMaxOut] = {y, delta, inner, lora};
    for (int k = 0; k < kMaxOut; ++k) {
        p.slot[k] = -1;
        if (!outs[k]) continue;
        cudaError_t e = make_tmap_2d_sw(&maps.out[p.n_out], dt, outs[k], rows, d_out, d_out * 2,
                                        kLSlice, 32, 64);      // one warp's 32 rows
        if (e != cudaSuccess) return e;
        p.slot[k] = p.n_out++;
    }
    if (p.n_out == 0) return cudaSuccess;
    cudaError_t e = make_tmap_2d(&maps.mid, dt, mid, rows, r, r * 2, kLK, kLM, true);
    if (e != cudaSuccess) return e;
    e = make_tmap_2d(&maps.b, dt, b, d_out, r, r * 2, kLK, kLN, true);
    if (e != cudaSuccess) return e;
    p.rows = rows;
    p.d_out = d_out;
    p.kb = static_cast<int>((r + kLK - 1) / kLK);
    p.m_tiles = static_cast<int>((rows + kLM - 1) / kLM);
    p.tiles = static_cast<int>(p.m_tiles * ((d_out + kLN - 1) / kLN));
    const int sms = device_sm_count(), optin = device_smem_optin();
    auto kern = dt == kBF16 ? lora_compose_kernel<__nv_bfloat16> : lora_compose_kernel<__half>;
    cudaFuncAttributes fa{};
    e = cudaFuncGetAttributes(&fa, kern);
    if (e != cudaSuccess) return e;
    const size_t budget = size_t(optin) - fa.sharedSizeBytes;   // dynamic shared memory
    p.stages = 4;
    while (p.stages > 1 && lc_smem(p.stages, p.n_out) > budget) --p.stages;
    if (p.stages < 2) return cudaErrorNotSupported;   // > 3 outputs at once
    p.s = s;
    p.g = g;
    p.bias = bias;
    p.base = base;
    p.fp16 = dt == kF16;
    const size_t smem = lc_smem(p.stages, p.n_out);
    e = ensure_max_dyn_smem(reinterpret_cast<const void*>(kern), static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    const int grid = std::min(p.tiles, sms);
    prof_begin("lora_compose_tc", st);
    kern<<<grid, kLThreads, smem, st>>>(maps, p);
    prof_end(st);
    if (launches) ++*launches;
    return cudaGetLastError();
}

}  // namespace dfx
