// compose.cu — the fused DoRA compose, forward (plain / dual-output) and backward.
//
// Arithmetic contract (bitwise): per element, fp32 with every op individually
// rounded (no FMA contraction — explicit __fmul_rn/__fadd_rn), in the canonical
// order of the reference's stable_element (compose.cpp:19-24):
//     t = s*lora;  u = g*t;  v = (g-1)*base;  delta = round_dtype(v + u)
//     inner = round_dtype(t + base)                          (compose.cpp:131-137)
// backward (compose.cpp:177-185):
//     d_lora = round_dtype(g*(s*dy));  d_base = round_dtype((g-1)*dy)
//     d_mag[j] = (serial-over-rows fp32 sum of dy*inner) / w_norm[j]   (:187-199)
// round_dtype is IEEE RNE (__float2bfloat16_rn / __float2half_rn), which the survey
// measured equal to the reference's round_to_limits on 24.4M inputs.
//
// Kernels
//   compose_fwd_vec        128-bit LDG/STG, g held in registers per column vector,
//                          R rows in flight per thread (HBM-bound: 3 or 4 streams)
//   compose_fwd_generic    scalar, any d_out / alignment (ragged shapes)
//   compose_bwd_vec        elementwise backward without d_mag (1 read, 2 writes)
//   compose_bwd_serial     TMA-fed column slabs: one thread per column runs the
//                          reference's serial fp32 d_mag chain over ALL rows (bitwise
//                          equal to compose.cpp:189-197) while other warps stream the
//                          elementwise d_lora/d_base out of the same smem stages
//   compose_bwd_generic    scalar fallback (ragged shapes), same serial chain
#include <cuda_bf16.h>

#include <cstdlib>
#include <string>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "launch.h"
#include "ptx.cuh"

namespace dfx {
namespace {

// ------------------------------------------------------------- vector helpers
// Two independent RN fp32 products in one packed FMUL2 (sm_100 mul.rn.f32x2): bitwise two
// __fmul_rn.  Used only where no add follows that ptxas could fuse with it.
__device__ __forceinline__ void fmul2_rn(float a0, float a1, float b0, float b1, float& d0, float& d1) {
    uint64_t a = (uint64_t(__float_as_uint(a1)) << 32) | __float_as_uint(a0);
    uint64_t b = (uint64_t(__float_as_uint(b1)) << 32) | __float_as_uint(b0);
    uint64_t d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    d0 = __uint_as_float(static_cast<uint32_t>(d));
    d1 = __uint_as_float(static_cast<uint32_t>(d >> 32));
}

template <typename T> struct Vec;  // 16-byte packs
template <> struct Vec<float> {
    static constexpr int N = 4;
    static __device__ __forceinline__ void unpack(const uint4& v, float (&f)[4]) {
        f[0] = __uint_as_float(v.x); f[1] = __uint_as_float(v.y);
        f[2] = __uint_as_float(v.z); f[3] = __uint_as_float(v.w);
    }
    static __device__ __forceinline__ uint4 pack(const float (&f)[4]) {
        return make_uint4(__float_as_uint(f[0]), __float_as_uint(f[1]), __float_as_uint(f[2]),
                          __float_as_uint(f[3]));
    }
};
template <> struct Vec<__nv_bfloat16> {
    static constexpr int N = 8;
    static __device__ __forceinline__ void unpack(const uint4& v, float (&f)[8]) {
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            f[2 * i] = __uint_as_float(w[i] << 16);
            f[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
        }
    }
    static __device__ __forceinline__ uint32_t pk(float lo, float hi) {
        __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
        return *reinterpret_cast<uint32_t*>(&h);
    }
    static __device__ __forceinline__ uint4 pack(const float (&f)[8]) {
        return make_uint4(pk(f[0], f[1]), pk(f[2], f[3]), pk(f[4], f[5]), pk(f[6], f[7]));
    }
};
template <> struct Vec<__half> {
    static constexpr int N = 8;
    static __device__ __forceinline__ void unpack(const uint4& v, float (&f)[8]) {
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const __half2 h = *reinterpret_cast<const __half2*>(&w[i]);
            const float2 p = __half22float2(h);
            f[2 * i] = p.x;
            f[2 * i + 1] = p.y;
        }
    }
    static __device__ __forceinline__ uint32_t pk(float lo, float hi) {
        __half2 h = __floats2half2_rn(lo, hi);
        return *reinterpret_cast<uint32_t*>(&h);
    }
    static __device__ __forceinline__ uint4 pack(const float (&f)[8]) {
        return make_uint4(pk(f[0], f[1]), pk(f[2], f[3]), pk(f[4], f[5]), pk(f[6], f[7]));
    }
};

// one 32-bit shared-memory word -> its 1 (fp32) or 2 (16-bit) values
template <typename T> struct Word;
template <> struct Word<float> {
    static __device__ __forceinline__ void unpack(uint32_t w, float (&f)[1]) { f[0] = __uint_as_float(w); }
};
template <> struct Word<__nv_bfloat16> {
    static __device__ __forceinline__ void unpack(uint32_t w, float (&f)[2]) {
        f[0] = __uint_as_float(w << 16);
        f[1] = __uint_as_float(w & 0xFFFF0000u);
    }
};
template <> struct Word<__half> {
    static __device__ __forceinline__ void unpack(uint32_t w, float (&f)[2]) {
        const float2 v = __half22float2(*reinterpret_cast<const __half2*>(&w));
        f[0] = v.x;
        f[1] = v.y;
    }
};

__device__ __forceinline__ uint32_t lds_u32(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}

__device__ __forceinline__ uint4 ld_stream(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}
__device__ __forceinline__ void st_stream(void* p, const uint4& v) {
    asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x),
                 "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}

// ------------------------------------------------------------------ forward
// blockDim = (BX, BY); thread (x, y) owns column vector c and R consecutive rows per
// grid step.  g and g-1 for its V columns stay in registers.
template <typename T, bool kInner, int R>
// 96 registers (256-thread CTAs; the compiler would take 97): one such CTA (24,576 registers)
// then fits beside a W.A^T CTA (160 x 256 = 40,960) in an SM's 65,536, so the forward compose
// can use the GEMM's SMs too when the two run concurrently (pipelined layer stack).  A/B:
// inference variant 10.5-11.3k -> 11.5k modules/s on one box, no difference on another;
// training unchanged; no spills.
__global__ void __maxnreg__(96) compose_fwd_vec(const T* __restrict__ base,
                                                       const T* __restrict__ lora,
                                                       const float* __restrict__ g, float sf,
                                                       int64_t rows, int64_t d_out,
                                                       T* __restrict__ delta,
                                                       T* __restrict__ inner, int pf_rows) {
    constexpr int V = Vec<T>::N;
    const int64_t cv = d_out / V;
    // L2 prefetch of the block `pf_rows` rows ahead (about one wave of resident CTAs), so
    // the loads of the CTAs that follow this one hit L2: bytes in flight per SM are capped
    // by the registers of the ~2 resident CTAs, L2 latency is far below HBM's
    if (pf_rows > 0 && threadIdx.x == 0 && threadIdx.y == 0) {
        const int64_t c0 = static_cast<int64_t>(blockIdx.x) * blockDim.x;
        const int64_t nvec = min(int64_t(blockDim.x), cv - c0);
        const uint32_t bytes = static_cast<uint32_t>(nvec * 16);
        const int64_t rp0 = static_cast<int64_t>(blockIdx.y) * blockDim.y * R + pf_rows;
        for (int i = 0; i < blockDim.y * R; ++i) {
            const int64_t rr = rp0 + i;
            if (rr >= rows) break;
            const int64_t off = rr * d_out + c0 * V;
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(base + off), "r"(bytes) : "memory");
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(lora + off), "r"(bytes) : "memory");
        }
    }
    const int64_t c = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (c >= cv) return;
    float gv[V], gm1[V];
#pragma unroll
    for (int k = 0; k < V; ++k) {
        gv[k] = __ldg(g + c * V + k);
        gm1[k] = __fsub_rn(gv[k], 1.0f);
    }
    const int64_t row_step = static_cast<int64_t>(gridDim.y) * blockDim.y * R;
    for (int64_t r0 = (static_cast<int64_t>(blockIdx.y) * blockDim.y + threadIdx.y) * R;
         r0 < rows; r0 += row_step) {
        uint4 bv[R], lv[R];
#pragma unroll
        for (int i = 0; i < R; ++i) {
            if (r0 + i < rows) {
                const int64_t off = (r0 + i) * d_out + c * V;
                bv[i] = ld_stream(base + off);
                lv[i] = ld_stream(lora + off);
            }
        }
#pragma unroll
        for (int i = 0; i < R; ++i) {
            if (r0 + i < rows) {
                float fb[V], fl[V], fd[V], fi[V];
                Vec<T>::unpack(bv[i], fb);
                Vec<T>::unpack(lv[i], fl);
#pragma unroll
                for (int k = 0; k < V; ++k) {
                    const float t = __fmul_rn(sf, fl[k]);
                    const float u = __fmul_rn(gv[k], t);
                    const float v = __fmul_rn(gm1[k], fb[k]);
                    fd[k] = __fadd_rn(v, u);
                    if (kInner) fi[k] = __fadd_rn(t, fb[k]);
                }
                const int64_t off = (r0 + i) * d_out + c * V;
                st_stream(delta + off, Vec<T>::pack(fd));
                if (kInner) st_stream(inner + off, Vec<T>::pack(fi));
            }
        }
    }
}

template <typename T, bool kInner>
__global__ void __launch_bounds__(256) compose_fwd_generic(const T* __restrict__ base,
                                                           const T* __restrict__ lora,
                                                           const float* __restrict__ g, float sf,
                                                           int64_t rows, int64_t d_out,
                                                           T* __restrict__ delta,
                                                           T* __restrict__ inner) {
    const int64_t n = rows * d_out;
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const float gf = __ldg(g + e % d_out);
        const float b = Elem<T>::to_f(base[e]);
        const float t = __fmul_rn(sf, Elem<T>::to_f(lora[e]));
        const float u = __fmul_rn(gf, t);
        const float v = __fmul_rn(__fsub_rn(gf, 1.0f), b);
        delta[e] = Elem<T>::from_f(__fadd_rn(v, u));
        if (kInner) inner[e] = Elem<T>::from_f(__fadd_rn(t, b));
    }
}

// ----------------------------------------------------------------- backward
template <typename T, int R>
__global__ void __launch_bounds__(256) compose_bwd_vec(const T* __restrict__ dy,
                                                       const float* __restrict__ g, float sf,
                                                       int64_t rows, int64_t d_out,
                                                       T* __restrict__ d_lora,
                                                       T* __restrict__ d_base) {
    constexpr int V = Vec<T>::N;
    const int64_t cv = d_out / V;
    const int64_t c = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (c >= cv) return;
    float gv[V], gm1[V];
#pragma unroll
    for (int k = 0; k < V; ++k) {
        gv[k] = __ldg(g + c * V + k);
        gm1[k] = __fsub_rn(gv[k], 1.0f);
    }
    const int64_t row_step = static_cast<int64_t>(gridDim.y) * blockDim.y * R;
    for (int64_t r0 = (static_cast<int64_t>(blockIdx.y) * blockDim.y + threadIdx.y) * R;
         r0 < rows; r0 += row_step) {
        uint4 dv[R];
#pragma unroll
        for (int i = 0; i < R; ++i)
            if (r0 + i < rows) dv[i] = ld_stream(dy + (r0 + i) * d_out + c * V);
#pragma unroll
        for (int i = 0; i < R; ++i) {
            if (r0 + i < rows) {
                float fy[V], fl[V], fb[V];
                Vec<T>::unpack(dv[i], fy);
#pragma unroll
                for (int k = 0; k < V; ++k) {
                    fl[k] = __fmul_rn(gv[k], __fmul_rn(sf, fy[k]));
                    fb[k] = __fmul_rn(gm1[k], fy[k]);
                }
                const int64_t off = (r0 + i) * d_out + c * V;
                st_stream(d_lora + off, Vec<T>::pack(fl));
                st_stream(d_base + off, Vec<T>::pack(fb));
            }
        }
    }
}

// Serial d_mag with TMA-staged column slabs.
//   slab      = kSC columns (128 bytes of a row), one CTA per slab, ALL rows
//   stage     = kRB rows x slab, for dy and inner (2 x kRB x 128 B)
//   warp 0    = TMA producer
//   warps 1.. = chain warps, one thread per column, serial over rows (bitwise ref order)
//   last 4    = elementwise warps: d_lora / d_base from the same stage, 16 B stores
template <typename T, int S = 6, int Wd = 1>
struct SerialCfg {
    static constexpr int kRowBytes = 128 * Wd;              // slab width: Wd x 128 bytes
    static constexpr int kSC = kRowBytes / sizeof(T);       // slab columns
    static constexpr int kRB = 64;                          // rows per stage
    static constexpr int kStages = S;
    static constexpr int kStageBytes = kRB * kRowBytes;     // per tensor
    static constexpr int kCPT = 4 / sizeof(T);              // chain columns per thread
    static constexpr int kChainWarps = Wd;                  // 32 threads x kCPT columns each
    static constexpr int kEltWarps = 4 * Wd;
    static constexpr int kThreads = 32 * (1 + kChainWarps + kEltWarps);
    static constexpr int kSmem = 2 * kStages * kStageBytes + 2 * kStages * 8 + 1024;
};

template <typename T, int S, int Wd = 1>
__global__ void __launch_bounds__(SerialCfg<T, S, Wd>::kThreads, 1)
    compose_bwd_serial(const __grid_constant__ CUtensorMap tm_dy,
                       const __grid_constant__ CUtensorMap tm_inner, const float* __restrict__ g,
                       float sf, const float* __restrict__ w_norm, int64_t rows, int64_t d_out,
                       T* __restrict__ d_lora, T* __restrict__ d_base, float* __restrict__ d_mag) {
    using C = SerialCfg<T, S, Wd>;
    constexpr int V = Vec<T>::N;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    uint8_t* s_dy = smem;
    uint8_t* s_in = smem + C::kStages * C::kStageBytes;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + 2 * C::kStages * C::kStageBytes);
    uint64_t* empty = full + C::kStages;

    const int warp = warp_id(), lane = lane_id();
    const int64_t col0 = static_cast<int64_t>(blockIdx.x) * C::kSC;
    const int n_iter = static_cast<int>((rows + C::kRB - 1) / C::kRB);

    if (threadIdx.x == 0) {
        tma_prefetch_desc(&tm_dy);
        tma_prefetch_desc(&tm_inner);
        for (int s = 0; s < C::kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], C::kChainWarps + C::kEltWarps);
        }
        fence_mbar_init();
    }
    __syncthreads();

    if (warp == 0) {
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();
            for (int it = 0; it < n_iter; ++it) {
                const int s = it % C::kStages;
                mbar_wait(&empty[s], ((it / C::kStages) & 1) ^ 1);
                mbar_arrive_expect_tx(&full[s], 2 * C::kStageBytes);
                tma_load_2d(&tm_dy, &full[s], s_dy + s * C::kStageBytes,
                            static_cast<int32_t>(col0), it * C::kRB, pol);
                tma_load_2d(&tm_inner, &full[s], s_in + s * C::kStageBytes,
                            static_cast<int32_t>(col0), it * C::kRB, pol);
            }
        }
    } else if (warp <= C::kChainWarps) {
        // chain thread: kCPT adjacent columns (one 32-bit shared-memory word per row), one
        // serial fp32 accumulator per column over rows ascending (independent chains)
        constexpr int P = C::kCPT;
        const int jc = (warp - 1) * (128 / int(sizeof(T))) + lane * P;
        float acc[P];
#pragma unroll
        for (int c = 0; c < P; ++c) acc[c] = 0.0f;
        for (int it = 0; it < n_iter; ++it) {
            const int s = it % C::kStages;
            mbar_wait(&full[s], (it / C::kStages) & 1);
            const uint32_t py = smem_u32(s_dy + s * C::kStageBytes) + jc * sizeof(T);
            const uint32_t pi = smem_u32(s_in + s * C::kStageBytes) + jc * sizeof(T);
            const int64_t rem = rows - int64_t(it) * C::kRB;
            const int nr = rem < C::kRB ? static_cast<int>(rem) : C::kRB;
            if (nr == C::kRB) {
                // Full stage: a batch of 16 rows is loaded first, the (independent)
                // products formed, then the dependent adds run in row order, so the
                // shared-memory latency is paid once per batch, not once per row.
#pragma unroll
                for (int i0 = 0; i0 < C::kRB; i0 += 16) {
                    float p[16][P];
#pragma unroll
                    for (int u = 0; u < 16; ++u) {
                        float fy[P], fi[P];
                        Word<T>::unpack(lds_u32(py + (i0 + u) * C::kRowBytes), fy);
                        Word<T>::unpack(lds_u32(pi + (i0 + u) * C::kRowBytes), fi);
#pragma unroll
                        for (int c = 0; c < P; ++c) p[u][c] = __fmul_rn(fy[c], fi[c]);
                    }
#pragma unroll
                    for (int u = 0; u < 16; ++u)
#pragma unroll
                        for (int c = 0; c < P; ++c) acc[c] = __fadd_rn(acc[c], p[u][c]);
                }
            } else {
                for (int i = 0; i < nr; ++i) {
                    float fy[P], fi[P];
                    Word<T>::unpack(lds_u32(py + i * C::kRowBytes), fy);
                    Word<T>::unpack(lds_u32(pi + i * C::kRowBytes), fi);
#pragma unroll
                    for (int c = 0; c < P; ++c) acc[c] = __fadd_rn(acc[c], __fmul_rn(fy[c], fi[c]));
                }
            }
            // every word read from the slot fed the chain above before this release, so the
            // reads are complete when the TMA may refill it (no proxy fence needed)
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
        }
#pragma unroll
        for (int c = 0; c < P; ++c) {
            const int64_t j = col0 + jc + c;
            if (j < d_out) d_mag[j] = __fdiv_rn(acc[c], __ldg(w_norm + j));
        }
    } else {
        // elementwise warps: 128 threads per 128 bytes of slab, each a fixed 16-byte vector
        const int t = threadIdx.x - 32 * (1 + C::kChainWarps);
        constexpr int kVecPerRow = C::kRowBytes / 16;
        constexpr int kEltThreads = 32 * C::kEltWarps;
        const int cvec = t % kVecPerRow;
        const int64_t j0 = col0 + cvec * V;
        // d_lora == d_base == null: magnitude gradient only (the warps still pace the ring)
        const bool col_ok = j0 < d_out && d_lora != nullptr;     // d_out % V == 0 here
        float gv[V], gm1[V];
#pragma unroll
        for (int k = 0; k < V; ++k) {
            gv[k] = col_ok ? __ldg(g + j0 + k) : 0.0f;
            gm1[k] = __fsub_rn(gv[k], 1.0f);
        }
        for (int it = 0; it < n_iter; ++it) {
            const int s = it % C::kStages;
            mbar_wait(&full[s], (it / C::kStages) & 1);
            const uint4* sy = reinterpret_cast<const uint4*>(s_dy + s * C::kStageBytes);
#pragma unroll
            for (int q = 0; q < C::kRB * kVecPerRow / kEltThreads; ++q) {
                const int idx = q * kEltThreads + t;
                const int rr = idx / kVecPerRow;
                const int64_t row = int64_t(it) * C::kRB + rr;
                const uint4 v = sy[idx];
                if (col_ok && row < rows) {
                    float fy[V], fl[V], fb[V];
                    Vec<T>::unpack(v, fy);
#ifndef DFX_NO_FMUL2
#pragma unroll
                    for (int k = 0; k < V; k += 2) {   // packed: t = s*dy, d_lora = g*t, d_base = (g-1)*dy
                        float t0, t1;
                        fmul2_rn(sf, sf, fy[k], fy[k + 1], t0, t1);
                        fmul2_rn(gv[k], gv[k + 1], t0, t1, fl[k], fl[k + 1]);
                        fmul2_rn(gm1[k], gm1[k + 1], fy[k], fy[k + 1], fb[k], fb[k + 1]);
                    }
#else
#pragma unroll
                    for (int k = 0; k < V; ++k) {
                        fl[k] = __fmul_rn(gv[k], __fmul_rn(sf, fy[k]));
                        fb[k] = __fmul_rn(gm1[k], fy[k]);
                    }
#endif
                    st_stream(d_lora + row * d_out + j0, Vec<T>::pack(fl));
                    st_stream(d_base + row * d_out + j0, Vec<T>::pack(fb));
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
        }
    }
}

// Scalar fallback: thread per column, rows ascending (bitwise serial chain).
template <typename T, bool kMag>
__global__ void __launch_bounds__(128) compose_bwd_generic(const T* __restrict__ dy,
                                                           const float* __restrict__ g, float sf,
                                                           const T* __restrict__ inner,
                                                           const float* __restrict__ w_norm,
                                                           int64_t rows, int64_t d_out,
                                                           T* __restrict__ d_lora,
                                                           T* __restrict__ d_base,
                                                           float* __restrict__ d_mag) {
    const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= d_out) return;
    const float gf = __ldg(g + j);
    const float gm1 = __fsub_rn(gf, 1.0f);
    float acc = 0.0f;
    for (int64_t i = 0; i < rows; ++i) {
        const int64_t e = i * d_out + j;
        const float y = Elem<T>::to_f(dy[e]);
        if (d_lora) {                       // null with kMag: magnitude gradient only
            d_lora[e] = Elem<T>::from_f(__fmul_rn(gf, __fmul_rn(sf, y)));
            d_base[e] = Elem<T>::from_f(__fmul_rn(gm1, y));
        }
        if (kMag) acc = __fadd_rn(acc, __fmul_rn(y, Elem<T>::to_f(inner[e])));
    }
    if (kMag) d_mag[j] = __fdiv_rn(acc, __ldg(w_norm + j));
}

// ------------------------------------------------------------------ launchers
inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

template <typename T, bool kInner>
cudaError_t fwd_impl(const void* base, const void* lora, const float* g, float sf, int64_t rows,
                     int64_t d_out, void* delta, void* inner, cudaStream_t st) {
    constexpr int V = Vec<T>::N;
    const T* b = static_cast<const T*>(base);
    const T* l = static_cast<const T*>(lora);
    T* d = static_cast<T*>(delta);
    T* in = static_cast<T*>(inner);
    const bool vec = d_out % V == 0 && aligned16(base) && aligned16(lora) && aligned16(delta) &&
                     (!kInner || aligned16(inner));
    if (vec) {
        constexpr int R = 4;
        const int64_t cv = d_out / V;
        int bx = 32;
        while (bx < 256 && bx < cv) bx *= 2;
        const int by = 256 / bx;
        const int64_t gx = (cv + bx - 1) / bx;
        const int64_t gy = std::min<int64_t>((rows + by * R - 1) / (by * R), 65535);
        // prefetch distance: one wave of resident CTAs (2 per SM at this register count);
        // measured at C2: dual 45.8 -> 43.3 us, 71 -> 61 us on a 76-SM partition
        const int sms = device_sm_count();
        const int pf_rows = static_cast<int>(2 * sms / gx) * by * R;
        prof_begin(kInner ? "compose_fwd_dual" : "compose_fwd", st);
        compose_fwd_vec<T, kInner, R>
            <<<dim3(static_cast<unsigned>(gx), static_cast<unsigned>(gy)), dim3(bx, by), 0, st>>>(
                b, l, g, sf, rows, d_out, d, in, pf_rows);
        prof_end(st);
    } else {
        const int64_t n = rows * d_out;
        const int64_t blocks = std::min<int64_t>((n + 255) / 256, 148 * 16);
        prof_begin("compose_fwd_generic", st);
        compose_fwd_generic<T, kInner><<<static_cast<unsigned>(blocks), 256, 0, st>>>(
            b, l, g, sf, rows, d_out, d, in);
        prof_end(st);
    }
    return cudaGetLastError();
}

template <typename T, int S, int Wd = 1>
cudaError_t bwd_serial_launch(int dt, const void* dy, const float* g, float sf, const void* inner,
                              const float* w_norm, int64_t rows, int64_t d_out, T* dl, T* db,
                              float* d_mag, cudaStream_t st) {
    using C = SerialCfg<T, S, Wd>;
    CUtensorMap tm_dy, tm_in;
    const uint64_t pitch = static_cast<uint64_t>(d_out) * sizeof(T);
    cudaError_t e = make_tmap_2d(&tm_dy, dt, dy, rows, d_out, pitch, C::kSC, C::kRB, false);
    if (e != cudaSuccess) return e;
    e = make_tmap_2d(&tm_in, dt, inner, rows, d_out, pitch, C::kSC, C::kRB, false);
    if (e != cudaSuccess) return e;
    e = ensure_max_dyn_smem(reinterpret_cast<const void*>(compose_bwd_serial<T, S, Wd>), C::kSmem);
    if (e != cudaSuccess) return e;
    const unsigned grid = static_cast<unsigned>((d_out + C::kSC - 1) / C::kSC);
    prof_begin("compose_bwd_dmag", st);
    compose_bwd_serial<T, S, Wd><<<grid, C::kThreads, C::kSmem, st>>>(tm_dy, tm_in, g, sf, w_norm, rows,
                                                                   d_out, dl, db, d_mag);
    prof_end(st);
    return cudaGetLastError();
}

template <typename T>
cudaError_t bwd_impl(int dt, const void* dy, const float* g, float sf, const void* inner,
                     const float* w_norm, int64_t rows, int64_t d_out, void* d_lora, void* d_base,
                     float* d_mag, cudaStream_t st, bool partitioned) {
    constexpr int V = Vec<T>::N;
    const T* y = static_cast<const T*>(dy);
    T* dl = static_cast<T*>(d_lora);
    T* db = static_cast<T*>(d_base);
    const bool vec = d_out % V == 0 && aligned16(dy) && aligned16(d_lora) && aligned16(d_base) &&
                     (d_mag == nullptr || aligned16(inner));
    if (d_mag == nullptr) {
        if (vec) {
            constexpr int R = 4;
            const int64_t cv = d_out / V;
            int bx = 32;
            while (bx < 256 && bx < cv) bx *= 2;
            const int by = 256 / bx;
            const int64_t gx = (cv + bx - 1) / bx;
            const int64_t gy = std::min<int64_t>((rows + by * R - 1) / (by * R), 65535);
            prof_begin("compose_bwd", st);
            compose_bwd_vec<T, R><<<dim3(static_cast<unsigned>(gx), static_cast<unsigned>(gy)),
                                    dim3(bx, by), 0, st>>>(y, g, sf, rows, d_out, dl, db);
            prof_end(st);
        } else {
            prof_begin("compose_bwd_generic", st);
            compose_bwd_generic<T, false>
                <<<static_cast<unsigned>((d_out + 127) / 128), 128, 0, st>>>(
                    y, g, sf, nullptr, nullptr, rows, d_out, dl, db, nullptr);
            prof_end(st);
        }
        return cudaGetLastError();
    }
    const T* in = static_cast<const T*>(inner);
    if (vec && rows > 0) {
        // one CTA per 128-byte column slab runs the whole column height; when the slabs
        // outnumber two per SM, a shallower ring (3 stages, ~49 KB) lets four share an SM so
        // the grid stays one wave (C3: 448 slabs)
        const int sms = device_sm_count();
        const int64_t slabs = (d_out + SerialCfg<T>::kSC - 1) / SerialCfg<T>::kSC;
        // beside the norm GEMMs (an SM budget is set): 256-byte slabs, half as many CTAs, each
        // filling an SM — measured +1.5-2.7 % on the pipelined C2 training step (A/B on one
        // box); alone they are slower (57 vs 47 us), so the full-GPU launch keeps 128-byte slabs
        // DFX_BWD_CFG=<stages>x<slab width / 128 B> overrides the choice (measurements)
        static const char* cfg = std::getenv("DFX_BWD_CFG");
        if (cfg) {
            const std::string c(cfg);
            if (c == "6x2") return bwd_serial_launch<T, 6, 2>(dt, dy, g, sf, inner, w_norm, rows, d_out, dl, db, d_mag, st);
            if (c == "4x2") return bwd_serial_launch<T, 4, 2>(dt, dy, g, sf, inner, w_norm, rows, d_out, dl, db, d_mag, st);
            if (c == "3x2") return bwd_serial_launch<T, 3, 2>(dt, dy, g, sf, inner, w_norm, rows, d_out, dl, db, d_mag, st);
            if (c == "6x1") return bwd_serial_launch<T, 6>(dt, dy, g, sf, inner, w_norm, rows, d_out, dl, db, d_mag, st);
            if (c == "12x1") return bwd_serial_launch<T, 12>(dt, dy, g, sf, inner, w_norm, rows, d_out, dl, db, d_mag, st);
            if (c == "4x1") return bwd_serial_launch<T, 4>(dt, dy, g, sf, inner, w_norm, rows, d_out, dl, db, d_mag, st);
        }
        if (partitioned && slabs <= 2 * int64_t(sms))
            return bwd_serial_launch<T, 6, 2>(dt, dy, g, sf, inner, w_norm, rows, d_out, dl, db, d_mag, st);
        return slabs > 2 * int64_t(sms)
                   ? bwd_serial_launch<T, 3>(dt, dy, g, sf, inner, w_norm, rows, d_out, dl, db, d_mag, st)
                   : bwd_serial_launch<T, 6>(dt, dy, g, sf, inner, w_norm, rows, d_out, dl, db, d_mag, st);
    } else {
        prof_begin("compose_bwd_dmag_generic", st);
        compose_bwd_generic<T, true><<<static_cast<unsigned>((d_out + 127) / 128), 128, 0, st>>>(
            y, g, sf, in, w_norm, rows, d_out, dl, db, d_mag);
        prof_end(st);
    }
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_compose_fwd(int dt, const void* base, const void* lora, const float* g, float sf,
                               int64_t rows, int64_t d_out, void* delta, void* inner,
                               cudaStream_t st, int* launches) {
    if (rows == 0 || d_out == 0) return cudaSuccess;
    if (launches) ++*launches;
    const bool wi = inner != nullptr;
    switch (dt) {
        case kF32:
            return wi ? fwd_impl<float, true>(base, lora, g, sf, rows, d_out, delta, inner, st)
                      : fwd_impl<float, false>(base, lora, g, sf, rows, d_out, delta, inner, st);
        case kBF16:
            return wi ? fwd_impl<__nv_bfloat16, true>(base, lora, g, sf, rows, d_out, delta, inner, st)
                      : fwd_impl<__nv_bfloat16, false>(base, lora, g, sf, rows, d_out, delta, inner,
                                                       st);
        default:
            return wi ? fwd_impl<__half, true>(base, lora, g, sf, rows, d_out, delta, inner, st)
                      : fwd_impl<__half, false>(base, lora, g, sf, rows, d_out, delta, inner, st);
    }
}

cudaError_t launch_compose_bwd(int dt, const void* dy, const float* g, float sf, const void* inner,
                               const float* w_norm, int64_t rows, int64_t d_out, void* d_lora,
                               void* d_base, float* d_mag, cudaStream_t st, int* launches,
                               bool partitioned) {
    if (d_out == 0) return cudaSuccess;
    // rows == 0 with d_mag: the reference yields 0 / w_norm per column; the
    // generic kernel's empty row loop reproduces that.
    if (rows == 0 && d_mag == nullptr) return cudaSuccess;
    if (launches) ++*launches;
    switch (dt) {
        case kF32:
            return bwd_impl<float>(dt, dy, g, sf, inner, w_norm, rows, d_out, d_lora, d_base, d_mag, st,
                                   partitioned);
        case kBF16:
            return bwd_impl<__nv_bfloat16>(dt, dy, g, sf, inner, w_norm, rows, d_out, d_lora, d_base,
                                           d_mag, st, partitioned);
        default:
            return bwd_impl<__half>(dt, dy, g, sf, inner, w_norm, rows, d_out, d_lora, d_base, d_mag,
                                    st, partitioned);
    }
}

}  // namespace dfx
