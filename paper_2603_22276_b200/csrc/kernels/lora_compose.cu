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
//
// Default build (profiles/r02_lora_epilogue_sweep.txt): CTA pairs (DFX_LC_PAIR: M = 256, each
// CTA stages half of B) and, when d_out % 16 == 0 and the outputs are 32-byte aligned, outputs
// stored straight from registers as 256-bit no-allocate stores (DFX_LC_DIRECT); otherwise the
// smem-staged TMA stores below.  Measured slower and kept as switches, all parity-green:
// DFX_LC_EPI_WARPS=16 (+ DFX_LC_TMEM_X16), DFX_LC_GSTORE=1, DFX_LC_FMUL2.  Knock-out switches
// DFX_LC_KO_{BASE,STORE,MMA,EPI} split the kernel's time.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <cstdlib>

#include "launch.h"
#include "ptx.cuh"

namespace dfx {
namespace {

constexpr int kLM = 128;                      // token rows per tile
constexpr int kLN = 256;                      // d_out columns per tile
constexpr int kLK = 64;                       // K block: one 128-byte swizzle atom
constexpr int kLSlice = 32;                   // epilogue column slice (64-byte swizzle)
#ifndef DFX_LC_EPI_WARPS
#define DFX_LC_EPI_WARPS 8
#endif
constexpr int kEpiWarps = DFX_LC_EPI_WARPS;           // 8 or 16 epilogue warps
constexpr int kGroups = kEpiWarps / 4;                // column groups (4 TMEM lane quadrants each)
constexpr int kLThreads = (kEpiWarps + 2) * 32;
#ifndef DFX_LC_SLEEP
#define DFX_LC_SLEEP 128
#endif
// back-off of the producer / MMA warps' barrier waits (ns; 0 = spin): the kernel is bounded by
// the epilogue's instruction issue, and a spinning try_wait loop takes issue slots on the
// schedulers it shares with epilogue warps
constexpr uint32_t kLSleepNs = DFX_LC_SLEEP;
__device__ __forceinline__ void lc_wait(uint64_t* bar, uint32_t phase) {
    if (kLSleepNs) mbar_wait_sleep(bar, phase, kLSleepNs);
    else mbar_wait(bar, phase);
}
constexpr int kWProd = kEpiWarps, kWMma = kEpiWarps + 1;
constexpr int kAStage = kLM * kLK * 2;        // 16 KiB of mid
#ifndef DFX_LC_PAIR
#define DFX_LC_PAIR 1
#endif
#ifndef DFX_LC_GSTORE
#define DFX_LC_GSTORE 0
#endif
// group stores: the four warps of a column group stage one 128-row slice together and one
// thread issues a single 128 x 32 TMA store per output (instead of one 32 x 32 store per
// warp): the TMA engine's per-instruction cost, not bytes, paced the epilogue's stores
constexpr bool kGStore = DFX_LC_GSTORE != 0;
// CTA pairs (cta_group::2): a cluster of two CTAs owns a 256-token x 256-column tile, each CTA
// staging its own 128 mid rows and HALF of the tile's B rows; the leader issues M = 256 UMMAs
// that read both CTAs' shared memory and accumulate into both CTAs' TMEM (each its own 128
// rows).  Per SM, B traffic through shared memory halves (the kernel is bound by its shared-
// memory traffic: operand TMA writes + tensor-core reads + output staging).
constexpr bool kPair = DFX_LC_PAIR != 0;
constexpr int kBRows = kPair ? kLN / 2 : kLN;      // B rows per CTA per stage
constexpr int kBStage = kBRows * kLK * 2;          // 16 KiB (pair) / 32 KiB of B
constexpr int kTileM = kPair ? 2 * kLM : kLM;      // token rows per (pair) tile
constexpr int kMaxStages = kPair ? 6 : 4;
constexpr int kSlice = kLM * kLSlice * 2;     // 8 KiB
constexpr int kWCols = kLN / kGroups;         // columns of a tile per epilogue warp
constexpr int kWSlices = kWCols / kLSlice;    // 32-column slices per warp and tile
#ifdef DFX_LC_TMEM_X16
constexpr int kAccCols = 16;                   // accumulator columns per tcgen05.ld
#else
constexpr int kAccCols = 32;
#endif
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
    int nbuf;               // output staging buffers per group (2: double-buffered)
    int n_out;              // enabled outputs, compacted in out[] / the smem buffers
    int slot[kMaxOut];      // kind (0 y, 1 delta, 2 inner, 3 lora) -> buffer index, -1 = off
    float s;
    const float* g;
    const float* bias;      // nullable (values representable in the working dtype)
    const void* base;       // [rows, d_out], read by the epilogue through L1
    int fp16;
    int v8;                 // base rows 32-byte aligned (d_out % 16 == 0): 256-bit loads
    int direct;             // outputs stored from registers (256-bit, no smem staging)
    void* outp[kMaxOut];    // enabled outputs' base pointers, compacted like the maps
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
__device__ __forceinline__ void bulk_wait_read0() {
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
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

// 256-bit load (sm_100: LDG.256): two 16-byte pieces of one 32-byte sector pair per thread
__device__ __forceinline__ void ldg_nc_v8(const void* p, uint4& a, uint4& b) {
#ifndef DFX_LC_V8_ALLOC   // no L1 allocation: the pieces use whole sectors, never re-read
    asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
#else
    asm volatile("ld.global.nc.v8.u32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
#endif
                 : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z),
                   "=r"(b.w)
                 : "l"(p));
}

// Two RN fp32 products in one packed FMUL2 (mul.rn.f32x2): bitwise two __fmul_rn.  Only the
// products use it; every add stays a scalar add.rn (a packed add after a packed mul is
// contracted into FFMA2 by ptxas, see compose.cu).
#ifdef DFX_LC_FMUL2
__device__ __forceinline__ void lc_fmul2(float a0, float a1, float b0, float b1, float& d0, float& d1) {
    const uint64_t a = (uint64_t(__float_as_uint(a1)) << 32) | __float_as_uint(a0);
    const uint64_t b = (uint64_t(__float_as_uint(b1)) << 32) | __float_as_uint(b0);
    uint64_t d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    d0 = __uint_as_float(static_cast<uint32_t>(d));
    d1 = __uint_as_float(static_cast<uint32_t>(d >> 32));
}
#endif

// 256-bit store without L1 allocation: 32 bytes of one row per thread
__device__ __forceinline__ void stg_na_v8(void* p, const uint32_t (&a)[4], const uint32_t (&b)[4]) {
    asm volatile("st.global.L1::no_allocate.v8.u32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p),
                 "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]), "r"(b[2]), "r"(b[3])
                 : "memory");
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

template <typename T, bool kBias>
__global__ void __launch_bounds__(kLThreads, 1)
    lora_compose_kernel(const __grid_constant__ LcMaps maps, const LcParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    constexpr int kStage = kAStage + kBStage;
    uint8_t* s_out = smem + p.stages * kStage;   // [kGroups][nbuf buffers][n_out][8 KiB]
    uint64_t* full = reinterpret_cast<uint64_t*>(s_out + kGroups * p.nbuf * p.n_out * kSlice);
    uint64_t* empty = full + p.stages;
    uint64_t* tmem_full = empty + p.stages;      // [2]
    uint64_t* tmem_empty = tmem_full + 2;        // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);

    __shared__ __align__(16) float s_gw[kEpiWarps][3][kWCols];   // epilogue warp: g, g - 1, bias
    const int warp = warp_id(), lane = lane_id();
    const uint32_t rank = kPair ? cluster_ctarank() : 0;
    const bool leader = rank == 0;
    const int unit = kPair ? static_cast<int>(blockIdx.x >> 1) : static_cast<int>(blockIdx.x);
    const int nunits = kPair ? static_cast<int>(gridDim.x >> 1) : static_cast<int>(gridDim.x);
    // this CTA's first token row of tile t (its half of a pair tile)
    auto tile_m0 = [&](int t) { return (t % p.m_tiles) * kTileM + static_cast<int>(rank) * kLM; };
    if (threadIdx.x == 0) {
        for (int i = 0; i < p.stages; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tmem_full[i], 1);
            mbar_init(&tmem_empty[i], kPair ? 2 * kEpiWarps : kEpiWarps);   // leader's counts both
        }
        fence_mbar_init();
    }
    if (warp == kWMma) {
        if (kPair) tmem_alloc_pair<512>(tmem_slot);
        else tmem_alloc<512>(tmem_slot);
    }
    tc_fence_before();
    __syncthreads();
    if (kPair) cluster_sync();      // the peer's barriers exist before any cross-CTA arrive
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
            for (int t = unit; t < p.tiles; t += nunits) {
                const int32_t m0 = tile_m0(t);
                const int32_t n0 = (t / p.m_tiles) * kLN + static_cast<int>(rank) * kBRows;
                for (int kb = 0; kb < p.kb; ++kb) {
                    lc_wait(&empty[s], ph ^ 1);
                    uint8_t* sa = smem + s * kStage;
                    if (kPair) {
                        // both CTAs' loads complete on the leader's barrier
                        if (leader) mbar_arrive_expect_tx(&full[s], 2 * kStage);
                        const uint32_t lbar = mapa_shared(smem_u32(&full[s]), 0);
                        tma_load_2d_pair(&maps.mid, lbar, sa, kb * kLK, m0, pol);
                        tma_load_2d_pair(&maps.b, lbar, sa + kAStage, kb * kLK, n0, pol);
                    } else {
                        mbar_arrive_expect_tx(&full[s], kStage);
                        tma_load_2d(&maps.mid, &full[s], sa, kb * kLK, m0, pol);
                        tma_load_2d(&maps.b, &full[s], sa + kAStage, kb * kLK, n0, pol);
                    }
                    if (++s == p.stages) { s = 0; ph ^= 1; }
                }
            }
        }
    } else if (warp == kWMma) {
        // ================= MMA issuer (single thread) =================
        if (lane == 0 && leader) {
            const uint32_t idesc = umma_idesc_f16(p.fp16 ? 0u : 1u, kTileM, kLN);
            int s = 0;
            uint32_t ph = 0;
            int local = 0;
            for (int t = unit; t < p.tiles; t += nunits, ++local) {
                const int slot = local & 1;
                const uint32_t tacc = tmem_base + static_cast<uint32_t>(slot * kLN);
                lc_wait(&tmem_empty[slot], ((local >> 1) & 1) ^ 1);
                tc_fence_after();
                for (int kb = 0; kb < p.kb; ++kb) {
                    lc_wait(&full[s], ph);
                    tc_fence_after();
                    const uint32_t sa = smem_u32(smem + s * kStage);
                    const uint32_t sb = sa + kAStage;
#ifndef DFX_LC_KO_MMA
#pragma unroll
                    for (int k = 0; k < kLK / 16; ++k) {
                        const uint64_t ad = umma_desc_k_sw128(sa + k * 32);
                        const uint64_t bd = umma_desc_k_sw128(sb + k * 32);
                        if (kPair) umma_f16_pair(tacc, ad, bd, idesc, (kb > 0 || k > 0) ? 1u : 0u);
                        else umma_f16(tacc, ad, bd, idesc, (kb > 0 || k > 0) ? 1u : 0u);
                    }
#else
                    (void)sb; (void)tacc;
#endif
                    if (kPair) umma_commit_pair_mc(&empty[s], 0x3);
                    else umma_commit(&empty[s]);
                    if (++s == p.stages) { s = 0; ph ^= 1; }
                }
                if (kPair) umma_commit_pair_mc(&tmem_full[slot], 0x3);
                else umma_commit(&tmem_full[slot]);
            }
        }
    } else if (warp < kEpiWarps) {
        // ================= epilogue: one token row per thread =================
        // Warp w (TMEM lane quadrant q = w % 4) owns the 32 rows 32q.. of each tile and the
        // kWCols columns of group grp = w / 4, in 32-column slices.  Each slice's outputs go
        // to the warp's part of a (double-buffered where shared memory allows) 64-byte-
        // swizzled smem slice and leave by the warp's own TMA store (32 x 32 box) while the
        // next slice computes: no cross-warp synchronisation in the epilogue.
        const int grp = warp >> 2, q = warp & 3;
        const int row = q * 32 + lane;
        const int sw = (row >> 1) & 3;                          // SWIZZLE_64B chunk XOR
        uint8_t* obase = s_out + grp * p.nbuf * p.n_out * kSlice;  // [nbuf][n_out][slice]
        float (*gw)[kWCols] = s_gw[warp];                       // [g | g - 1 | bias][column]
        const float sf = p.s;
        // this thread's 64-byte base piece of a slice (row clamped in the token tail, columns
        // in the d_out tail; those outputs are clipped by the TMA store), read through L1
        // one slice ahead so the DRAM latency hides behind the current slice's arithmetic
        // (two slices or a whole tile ahead measured no faster)
        auto load_base = [&](int tt, int cs, uint4 (&v)[4]) {
            if (tt >= p.tiles) return;
            const int64_t r0 = min(int64_t(tile_m0(tt) + row), p.rows - 1);
            const int64_t c0 = int64_t(tt / p.m_tiles) * kLN + kWCols * grp + kLSlice * cs;
            const T* src = static_cast<const T*>(p.base) + r0 * p.d_out;
#ifdef DFX_LC_KO_BASE
            v[0] = v[1] = v[2] = v[3] = make_uint4(0, 0, 0, 0);   // knock-out: no base stream
            (void)src; (void)c0;
#else
            if (p.v8) {      // rows 32-byte aligned: 32-byte pieces, whole or past d_out
#pragma unroll
                for (int k = 0; k < 4; k += 2)
                    ldg_nc_v8(src + min(c0 + 8 * k, p.d_out - 16), v[k], v[k + 1]);
            } else {
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    v[k] = ldg_nc_v4(src + min(c0 + 8 * k, p.d_out - 8));
            }
#endif
        };
        uint4 bnext[4];
        load_base(unit, 0, bnext);
        int local = 0, nslice = 0;
        for (int t = unit; t < p.tiles; t += nunits, ++local) {
            const int32_t m0 = tile_m0(t), n0 = (t / p.m_tiles) * kLN;
            // g, g - 1 and bias for the warp's columns (a missing bias is -0.0, an exact
            // no-op in the fp32 add; columns past d_out are clamped, their outputs clipped)
            {
                constexpr int kPer = kWCols / 32;                // 4 (8 warps) or 2 (16 warps)
                const int64_t j = min(int64_t(n0 + kWCols * grp + kPer * lane), p.d_out - kPer);
#pragma unroll
                for (int i = 0; i < kPer; ++i) {
                    const float gv = __ldg(p.g + j + i);
                    gw[0][kPer * lane + i] = gv;
                    gw[1][kPer * lane + i] = __fsub_rn(gv, 1.0f);
                    gw[2][kPer * lane + i] = kBias ? __ldg(p.bias + j + i) : -0.0f;
                }
            }
            __syncwarp();
            const int slot = local & 1;
            mbar_wait(&tmem_full[slot], (local >> 1) & 1);
            tc_fence_after();
#pragma unroll
            for (int cs = 0; cs < kWSlices; ++cs, ++nslice) {
                const int cl = kWCols * grp + kLSlice * cs;     // slice's first column in the tile
                const int col0 = n0 + cl;
                uint4 bv[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) bv[k] = bnext[k];
                if (cs < kWSlices - 1) load_base(t, cs + 1, bnext);
                else load_base(t + nunits, 0, bnext);
                // the slice's accumulator columns, all 32 at once or in two 16-column halves
                // (DFX_LC_TMEM_X16: 16 fewer registers per thread)
                uint32_t acc[kAccCols];
                uint32_t oprev[kMaxOut][4];                 // direct stores: the even chunk
                auto load_acc = [&](int c) {
                    const uint32_t ta = tmem_base + static_cast<uint32_t>(slot * kLN + cl + c) +
                                        (static_cast<uint32_t>(q * 32) << 16);
                    if constexpr (kAccCols == 32)
                        tmem_ld_32x32b_x32(ta, *reinterpret_cast<uint32_t(*)[32]>(acc));
                    else
                        tmem_ld_32x32b_x16(ta, *reinterpret_cast<uint32_t(*)[16]>(acc));
                    tmem_ld_wait();
                    if (cs == kWSlices - 1 && c + kAccCols == kLSlice) {   // slot consumed
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) {
                            if (kPair) mbar_arrive_remote(mapa_shared(smem_u32(&tmem_empty[slot]), 0), 1);
                            else mbar_arrive(&tmem_empty[slot]);
                        }
                    }
                };
                uint8_t* obuf = obase + (p.nbuf == 2 ? (nslice & 1) : 0) * p.n_out * kSlice;
                const uint32_t orow = smem_u32(obuf) + static_cast<uint32_t>(row * (kLSlice * 2));
                if (kGStore) {
                    // the group's store thread has waited for the store that last read obuf
                    named_bar_sync(1 + grp, 128);
                } else {
                    if (p.nbuf == 1 && !p.direct && lane == 0) bulk_wait_read0();   // single buffer: last store read it
                    __syncwarp();
                }
#pragma unroll
                for (int k = 0; k < 4; ++k) {                 // 8 columns per 16-byte chunk
                    if ((8 * k) % kAccCols == 0) load_acc(8 * k);
#ifndef DFX_LC_KO_EPI   // knock-out: no epilogue arithmetic / staging stores
                    const int c8 = kLSlice * cs + 8 * k;        // column within the warp's group
                    const float4 g0 = *reinterpret_cast<const float4*>(&gw[0][c8]);
                    const float4 g1 = *reinterpret_cast<const float4*>(&gw[0][c8 + 4]);
                    const float4 h0 = *reinterpret_cast<const float4*>(&gw[1][c8]);
                    const float4 h1 = *reinterpret_cast<const float4*>(&gw[1][c8 + 4]);
                    float bb[8] = {};
                    if (kBias) {
                        const float4 b0 = *reinterpret_cast<const float4*>(&gw[2][c8]);
                        const float4 b1 = *reinterpret_cast<const float4*>(&gw[2][c8 + 4]);
                        bb[0] = b0.x; bb[1] = b0.y; bb[2] = b0.z; bb[3] = b0.w;
                        bb[4] = b1.x; bb[5] = b1.y; bb[6] = b1.z; bb[7] = b1.w;
                    }
                    const float gv[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
                    const float gm[8] = {h0.x, h0.y, h0.z, h0.w, h1.x, h1.y, h1.z, h1.w};
                    const uint32_t bw[4] = {bv[k].x, bv[k].y, bv[k].z, bv[k].w};
                    // element pairs: every dtype rounding is one packed F2FP conversion of
                    // two values (RNE, identical to two scalar roundings), unpacked by shifts
                    uint32_t o[kMaxOut][4];                  // packed y, delta, inner, lora
#pragma unroll
                    for (int e2 = 0; e2 < 4; ++e2) {
                        const int e = 2 * e2;
                        const float b0f = LcT<T>::lo(bw[e2]), b1f = LcT<T>::hi(bw[e2]);
                        const int ai = (8 * k) % kAccCols + e;
                        const uint32_t lw = LcT<T>::pack(__uint_as_float(acc[ai]),
                                                         __uint_as_float(acc[ai + 1]));
                        const float l0 = LcT<T>::lo(lw), l1 = LcT<T>::hi(lw);
#ifdef DFX_LC_FMUL2
                        float t0, t1, u0, u1, v0, v1;
                        lc_fmul2(sf, sf, l0, l1, t0, t1);
                        lc_fmul2(gv[e], gv[e + 1], t0, t1, u0, u1);
                        lc_fmul2(gm[e], gm[e + 1], b0f, b1f, v0, v1);
#else
                        const float t0 = __fmul_rn(sf, l0), t1 = __fmul_rn(sf, l1);
                        const float u0 = __fmul_rn(gv[e], t0), u1 = __fmul_rn(gv[e + 1], t1);
                        const float v0 = __fmul_rn(gm[e], b0f), v1 = __fmul_rn(gm[e + 1], b1f);
#endif
                        const uint32_t dw = LcT<T>::pack(__fadd_rn(v0, u0), __fadd_rn(v1, u1));
                        const uint32_t y0w = LcT<T>::pack(__fadd_rn(b0f, LcT<T>::lo(dw)),
                                                          __fadd_rn(b1f, LcT<T>::hi(dw)));
                        o[0][e2] = kBias ? LcT<T>::pack(__fadd_rn(LcT<T>::lo(y0w), bb[e]),
                                                         __fadd_rn(LcT<T>::hi(y0w), bb[e + 1]))
                                          : y0w;
                        o[1][e2] = dw;
                        o[2][e2] = LcT<T>::pack(__fadd_rn(t0, b0f), __fadd_rn(t1, b1f));
                        o[3][e2] = lw;
                    }
                    if (p.direct) {
                        // two chunks (16 columns, 32 bytes) per 256-bit store of this row; rows
                        // past the token tail and 16-column pieces past d_out are not written
                        if (k & 1) {
                            const int64_t gr = int64_t(m0) + row;
                            const int64_t gc = int64_t(col0) + 8 * (k - 1);
                            if (gr < p.rows && gc < p.d_out) {
#pragma unroll
                                for (int kind = 0; kind < kMaxOut; ++kind) {
                                    if (p.slot[kind] < 0) continue;
                                    T* dst = static_cast<T*>(p.outp[p.slot[kind]]) + gr * p.d_out + gc;
                                    stg_na_v8(dst, oprev[kind], o[kind]);
                                }
                            }
                        } else {
#pragma unroll
                            for (int kind = 0; kind < kMaxOut; ++kind)
#pragma unroll
                                for (int i = 0; i < 4; ++i) oprev[kind][i] = o[kind][i];
                        }
                    } else {
#pragma unroll
                    for (int kind = 0; kind < kMaxOut; ++kind) {
                        if (p.slot[kind] < 0) continue;      // output not requested (uniform)
                        sts_v4(orow + static_cast<uint32_t>(p.slot[kind] * kSlice + ((k ^ sw) << 4)),
                               o[kind][0], o[kind][1], o[kind][2], o[kind][3]);
                    }
                    }
#endif
                }
                // the warp's 32 rows of the slice go out by its own TMA store; with two
                // buffers, before the next slice reuses the other buffer, the store issued
                // from it two slices ago must have read its smem
                if (!p.direct) fence_async_smem();
#ifndef DFX_LC_KO_STORE
                if (kGStore && !p.direct) {
                    named_bar_sync(1 + grp, 128);                // the group's 128 rows staged
                    if (q == 0 && lane == 0) {
                        for (int oi = 0; oi < p.n_out; ++oi)
                            tma_store_2d(&maps.out[oi], obuf + oi * kSlice, col0, m0);
                        bulk_commit();
                        if (p.nbuf == 2) bulk_wait_read1();
                        else bulk_wait_read0();
                    }
                }
#endif
                __syncwarp();
#ifndef DFX_LC_KO_STORE
                if (!kGStore && !p.direct && lane == 0) {
                    for (int oi = 0; oi < p.n_out; ++oi)
                        tma_store_2d(&maps.out[oi], obuf + oi * kSlice + q * 32 * (kLSlice * 2),
                                     col0, m0 + 32 * q);
                    bulk_commit();
                    if (p.nbuf == 2) bulk_wait_read1();
                }
#endif
                __syncwarp();
            }
        }
        if (lane == 0) bulk_wait0();
    }
    tc_fence_before();
    __syncthreads();
    if (kPair) cluster_sync();      // the leader's MMAs wrote this CTA's TMEM
    if (warp == kWMma) {
        tc_fence_after();
        if (kPair) tmem_dealloc_pair<512>(tmem_base);
        else tmem_dealloc<512>(tmem_base);
    }
}

size_t lc_smem(int stages, int n_out, int nbuf) {
    return size_t(stages) * (kAStage + kBStage) + size_t(kGroups) * nbuf * n_out * kSlice + 1024 +
           256;
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
                                        kLSlice, kGStore ? kLM : 32, 64);   // a group's / warp's rows
        if (e != cudaSuccess) return e;
        p.outp[p.n_out] = outs[k];
        p.slot[k] = p.n_out++;
    }
    if (p.n_out == 0) return cudaSuccess;
    cudaError_t e = make_tmap_2d(&maps.mid, dt, mid, rows, r, r * 2, kLK, kLM, true);
    if (e != cudaSuccess) return e;
    e = make_tmap_2d(&maps.b, dt, b, d_out, r, r * 2, kLK, kBRows, true);
    if (e != cudaSuccess) return e;
    p.rows = rows;
    p.d_out = d_out;
    p.kb = static_cast<int>((r + kLK - 1) / kLK);
    p.m_tiles = static_cast<int>((rows + kTileM - 1) / kTileM);
    p.tiles = static_cast<int>(p.m_tiles * ((d_out + kLN - 1) / kLN));
    const int sms = device_sm_count(), optin = device_smem_optin();
    // the bias add is a template switch: a per-element select would issue its FADD / F2FP /
    // unpack whether or not a bias was passed
    auto kern = dt == kBF16 ? (bias ? lora_compose_kernel<__nv_bfloat16, true>
                                    : lora_compose_kernel<__nv_bfloat16, false>)
                            : (bias ? lora_compose_kernel<__half, true> : lora_compose_kernel<__half, false>);
    cudaFuncAttributes fa{};
    e = cudaFuncGetAttributes(&fa, kern);
    if (e != cudaSuccess) return e;
    const size_t budget = size_t(optin) - fa.sharedSizeBytes;   // dynamic shared memory
    // double-buffered output staging while at least min_st operand stages fit beside it,
    // else one staging buffer (each slice waits for its previous store to read it)
    static const int min_st = [] {
        const char* e = std::getenv("DFX_LC_MIN_STAGES");
        return e ? std::atoi(e) : 3;
    }();
#ifndef DFX_LC_DIRECT
#define DFX_LC_DIRECT 1
#endif
    // outputs straight from registers (256-bit stores, no staging) when every output row is
    // 32-byte aligned
    p.direct = 0;
    if (DFX_LC_DIRECT && d_out % 16 == 0) {
        p.direct = 1;
        for (int k = 0; k < p.n_out; ++k)
            if (reinterpret_cast<uintptr_t>(p.outp[k]) % 32 != 0) p.direct = 0;
    }
    p.nbuf = p.direct ? 0 : 2;
    p.stages = kMaxStages;
    while (p.stages > min_st && lc_smem(p.stages, p.n_out, p.nbuf) > budget) --p.stages;
    if (!p.direct && lc_smem(p.stages, p.n_out, 2) > budget) {
        p.nbuf = 1;
        p.stages = kMaxStages;
        while (p.stages > 2 && lc_smem(p.stages, p.n_out, 1) > budget) --p.stages;
        if (lc_smem(p.stages, p.n_out, 1) > budget) return cudaErrorNotSupported;  // > 3 outputs
    }
    p.s = s;
    p.g = g;
    p.bias = bias;
    p.base = base;
    p.fp16 = dt == kF16;
#ifndef DFX_LC_NO_V8
    p.v8 = d_out % 16 == 0 && reinterpret_cast<uintptr_t>(base) % 32 == 0;
#endif
    const size_t smem = lc_smem(p.stages, p.n_out, p.nbuf);
    e = ensure_max_dyn_smem(reinterpret_cast<const void*>(kern), static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    prof_begin("lora_compose_tc", st);
    if (kPair) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(2 * std::min(p.tiles, sms / 2), 1, 1);
        cfg.blockDim = dim3(kLThreads, 1, 1);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        e = cudaLaunchKernelEx(&cfg, kern, maps, p);
    } else {
        kern<<<std::min(p.tiles, sms), kLThreads, smem, st>>>(maps, p);
        e = cudaGetLastError();
    }
    prof_end(st);
    if (e != cudaSuccess) return e;
    if (launches) ++*launches;
    return cudaGetLastError();
}

}  // namespace dfx
