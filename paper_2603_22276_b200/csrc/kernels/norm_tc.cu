// norm_tc.cu — bf16 factored row norm on the 5th-generation tensor cores.
//
// One warp-specialised kernel template, tc_rowdot, serves all three contractions of
// factored_norm.cpp:27-120 with fused epilogues (nothing [d_out x r]-sized ever
// reaches HBM):
//   U = W A^T   (M=d_out, N=r, K=d_in)  epilogue: cross partial = rowdot(U, B)
//               + the base_sq chain: the same W tiles the UMMA consumes are read from
//                 shared memory by the epilogue warps, which run the reference's
//                 serial fp32 sum of w*w per row (reset at ChunkPlan boundaries)
//   G = A A^T   (M=N=r, upper-triangle tiles, split-K)  epilogue: store fp32 partials
//   V = B G     (M=d_out, N=r, K=2r: G split into bf16 hi+lo)  epilogue: ba_sq = rowdot(V, B)
//
// Per CTA: a 128-row tile of X, BN columns of Y (BN <= 256, multiple of 16), the
// whole K range of its split.  Operands arrive by TMA (128-byte swizzle, 64-wide
// K blocks) into a STAGES-deep mbarrier ring; one elected thread of warp 1 issues
// tcgen05.mma (M=128, N=BN, K=16) into a TMEM accumulator of BN fp32 columns;
// warps 4..7 own TMEM lane quadrants 0..3 (one row per thread) for the chain and
// the epilogue (tcgen05.ld 32x32b.x32).
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdio>

#include "norm_common.cuh"

namespace dfx {
namespace {

constexpr int kBM = 128;
constexpr int kBK = 64;                          // one 128-byte swizzle atom of bf16
constexpr int kXStage = kBM * kBK * 2;           // 16 KiB
constexpr int kThreads = 256;
constexpr int kMaxSmem = 227 * 1024;

enum TcMode { kTcRowdot = 0, kTcStore = 1 };

struct TcParams {
    int64_t M, N;           // logical rows of X / rows of Y
    int64_t k_total;        // K extent (elements) iterated by the whole grid
    int kb_per_split;       // 64-wide K blocks per K split
    int n_split;            // CTAs along N per M tile
    int bn;                 // N per CTA (multiple of 16, <= 256)
    int stages;
    int x_kwrap;            // X k coordinate wraps modulo this (ba_sq: r_pad); 0 = none
    int64_t chunk;          // ChunkPlan chunk size (chain), multiple of 64
    // rowdot
    const __nv_bfloat16* Z; int64_t ldz;
    float* out;             // rowdot: [k_split*n_split][M]; store: tiles
    float* base_out;        // chain: [num_chunks][M], one serial partial per chunk
    int do_chain;
    // store (gram): tile index mapping
    int gram_nt;            // tiles per side
};

__device__ __forceinline__ void unpack_bf16x8(const uint4& v, float (&f)[8]) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        f[2 * i] = __uint_as_float(w[i] << 16);
        f[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
    }
}

template <int kMode>
__global__ void __launch_bounds__(kThreads, 1)
    tc_rowdot(const __grid_constant__ CUtensorMap tmx, const __grid_constant__ CUtensorMap tmy,
              const TcParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    const int y_stage = p.bn * kBK * 2;
    const int stage_bytes = kXStage + y_stage;  // both multiples of 1024
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + p.stages * stage_bytes);
    uint64_t* empty = full + p.stages;
    uint64_t* tmem_full = empty + p.stages;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

    const int warp = warp_id(), lane = lane_id();

    // ---- tile coordinates
    int64_t m0, n0;
    int ks;
    if (kMode == kTcStore) {
        // blockIdx.x enumerates upper-triangle tiles (pi <= qi), blockIdx.y the K split
        int t = blockIdx.x, pi = 0;
        while (t >= p.gram_nt - pi) { t -= p.gram_nt - pi; ++pi; }
        const int qi = pi + t;
        m0 = int64_t(pi) * kBM;
        n0 = int64_t(qi) * p.bn;
        ks = blockIdx.y;
    } else {
        const int ns = blockIdx.x % p.n_split;
        m0 = int64_t(blockIdx.x / p.n_split) * kBM;
        n0 = int64_t(ns) * p.bn;
        ks = blockIdx.y;
    }
    const bool chain = (kMode == kTcRowdot) && p.do_chain && (n0 == 0);
    const int kb0 = ks * p.kb_per_split;
    const int64_t total_kb = (p.k_total + kBK - 1) / kBK;
    const int64_t kb_left = total_kb - kb0;
    const int nkb = static_cast<int>(kb_left < p.kb_per_split ? kb_left : p.kb_per_split);

    uint32_t tmem_cols = 32;
    while (tmem_cols < static_cast<uint32_t>(p.bn)) tmem_cols <<= 1;

    if (threadIdx.x == 0) {
        tma_prefetch_desc(&tmx);
        tma_prefetch_desc(&tmy);
        for (int s = 0; s < p.stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1 + (chain ? 4 : 0));
        }
        mbar_init(tmem_full, 1);
        fence_mbar_init();
    }
    if (warp == 1) {
        switch (tmem_cols) {
            case 32: tmem_alloc<32>(tmem_slot); break;
            case 64: tmem_alloc<64>(tmem_slot); break;
            case 128: tmem_alloc<128>(tmem_slot); break;
            case 256: tmem_alloc<256>(tmem_slot); break;
            default: tmem_alloc<512>(tmem_slot); break;
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        // ================= TMA producer =================
        if (lane == 0 && nkb > 0) {
            const uint64_t pol_x = (kMode == kTcRowdot && !p.x_kwrap) ? policy_evict_first()
                                                                       : policy_evict_last();
            const uint64_t pol_y = policy_evict_last();
            for (int it = 0; it < nkb; ++it) {
                const int s = it % p.stages;
                mbar_wait(&empty[s], ((it / p.stages) & 1) ^ 1);
                mbar_arrive_expect_tx(&full[s], stage_bytes);
                uint8_t* sx = smem + s * stage_bytes;
                uint8_t* sy = sx + kXStage;
                const int kc = (kb0 + it) * kBK;
                const int kx = p.x_kwrap ? kc % p.x_kwrap : kc;
                tma_load_2d(&tmx, &full[s], sx, kx, static_cast<int32_t>(m0), pol_x);
                tma_load_2d(&tmy, &full[s], sy, kc, static_cast<int32_t>(n0), pol_y);
            }
        }
    } else if (warp == 1) {
        // ================= MMA issuer (single thread) =================
        if (lane == 0 && nkb > 0) {
            const uint32_t idesc = umma_idesc_f16(1u, kBM, static_cast<uint32_t>(p.bn));
            for (int it = 0; it < nkb; ++it) {
                const int s = it % p.stages;
                mbar_wait(&full[s], (it / p.stages) & 1);
                tc_fence_after();
                const uint32_t sx = smem_u32(smem + s * stage_bytes);
                const uint32_t sy = sx + kXStage;
#pragma unroll
                for (int k = 0; k < kBK / 16; ++k) {
                    const uint64_t ad = umma_desc_k_sw128(sx + k * 32);
                    const uint64_t bd = umma_desc_k_sw128(sy + k * 32);
                    umma_f16(tmem_base, ad, bd, idesc, (it > 0 || k > 0) ? 1u : 0u);
                }
                umma_commit(&empty[s]);
            }
            umma_commit(tmem_full);
        }
    } else if (warp >= 4) {
        // ================= chain + epilogue (one row per thread) =================
        const int q = warp - 4;               // TMEM lane quadrant
        const int row = q * 32 + lane;        // row inside the tile
        const int64_t gm = m0 + row;
        if (chain) {
            // one serial fp32 partial per ChunkPlan chunk (factored_norm.cpp:52-60); the
            // finisher adds the chunk partials in ascending order (:60), so K splits on
            // chunk boundaries keep base_sq bitwise equal to the reference
            float partial = 0.0f;
            int64_t cur = -1;
            for (int it = 0; it < nkb; ++it) {
                const int s = it % p.stages;
                mbar_wait(&full[s], (it / p.stages) & 1);
                const int64_t chunk_idx = (int64_t(kb0 + it) * kBK) / p.chunk;
                if (chunk_idx != cur) {
                    if (cur >= 0 && gm < p.M) p.base_out[cur * p.M + gm] = partial;
                    partial = 0.0f;
                    cur = chunk_idx;
                }
                const uint8_t* rowp = smem + s * stage_bytes + row * 128;
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    const uint4 v = *reinterpret_cast<const uint4*>(rowp + ((c ^ (row & 7)) << 4));
                    float f[8];
                    unpack_bf16x8(v, f);
#pragma unroll
                    for (int e = 0; e < 8; ++e) partial = __fadd_rn(partial, __fmul_rn(f[e], f[e]));
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[s]);
            }
            if (cur >= 0 && gm < p.M) p.base_out[cur * p.M + gm] = partial;
        }
        // wait for the accumulator
        if (nkb > 0) {
            mbar_wait(tmem_full, 0);
            tc_fence_after();
        }
        const uint32_t trow = tmem_base + (static_cast<uint32_t>(q * 32) << 16);
        if (kMode == kTcRowdot) {
            float acc = 0.0f;
            for (int c0 = 0; c0 < p.bn; c0 += 32) {
                uint32_t u[32];
                tmem_ld_32x32b_x32(trow + c0, u);
                tmem_ld_wait();
                if (gm < p.M && nkb > 0) {
                    const __nv_bfloat16* zr = p.Z + gm * p.ldz + n0 + c0;
#pragma unroll
                    for (int v = 0; v < 4; ++v) {
                        if (n0 + c0 + 8 * v < p.N) {
                            float z[8];
                            unpack_bf16x8(*reinterpret_cast<const uint4*>(zr + 8 * v), z);
#pragma unroll
                            for (int e = 0; e < 8; ++e)
                                acc = fmaf(__uint_as_float(u[8 * v + e]), z[e], acc);
                        }
                    }
                }
            }
            if (gm < p.M)
                p.out[(int64_t(ks) * p.n_split + (n0 / p.bn)) * p.M + gm] = acc;
        } else {
            // gram tile store: out[(ks * tiles + tile) * 128*bn + row*bn + col]
            float* dst = p.out + (int64_t(ks) * gridDim.x + blockIdx.x) * (int64_t(kBM) * p.bn) +
                         int64_t(row) * p.bn;
            for (int c0 = 0; c0 < p.bn; c0 += 32) {
                uint32_t u[32];
                tmem_ld_32x32b_x32(trow + c0, u);
                tmem_ld_wait();
#pragma unroll
                for (int e = 0; e < 32; e += 4) {
                    float4 v = make_float4(__uint_as_float(u[e]), __uint_as_float(u[e + 1]),
                                           __uint_as_float(u[e + 2]), __uint_as_float(u[e + 3]));
                    if (nkb == 0) v = make_float4(0.f, 0.f, 0.f, 0.f);
                    *reinterpret_cast<float4*>(dst + c0 + e) = v;
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        switch (tmem_cols) {
            case 32: tmem_dealloc<32>(tmem_base); break;
            case 64: tmem_dealloc<64>(tmem_base); break;
            case 128: tmem_dealloc<128>(tmem_base); break;
            case 256: tmem_dealloc<256>(tmem_base); break;
            default: tmem_dealloc<512>(tmem_base); break;
        }
    }
}

// Reduce gram partial tiles in fixed split order and emit [G_hi | G_lo] (bf16) with
// G mirrored from the upper triangle, so the hi/lo operand is exactly symmetric.
__global__ void __launch_bounds__(256) gram_reduce(const float* __restrict__ part, int k_split,
                                                   int nt, int64_t r, int64_t r_pad,
                                                   __nv_bfloat16* __restrict__ g2) {
    const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= r * r_pad) return;
    const int64_t i = idx / r_pad, j = idx % r_pad;
    float gsum = 0.0f;
    if (j < r) {
        const int64_t pi0 = i < j ? i : j, qi0 = i < j ? j : i;  // upper-triangle element
        const int pt = static_cast<int>(pi0 / kBM), qt = static_cast<int>(qi0 / kBM);
        // tile index of (pt, qt) in row-major upper-triangle enumeration
        const int tile = pt * nt - pt * (pt - 1) / 2 + (qt - pt);
        const int64_t off = (pi0 % kBM) * kBM + (qi0 % kBM);
        const int tiles = nt * (nt + 1) / 2;
        gsum = part[int64_t(tile) * kBM * kBM + off];
        for (int s = 1; s < k_split; ++s)
            gsum = __fadd_rn(gsum, part[(int64_t(s) * tiles + tile) * kBM * kBM + off]);
    }
    const __nv_bfloat16 hi = __float2bfloat16_rn(gsum);
    const __nv_bfloat16 lo = __float2bfloat16_rn(__fsub_rn(gsum, __bfloat162float(hi)));
    g2[i * 2 * r_pad + j] = hi;
    g2[i * 2 * r_pad + r_pad + j] = lo;
}

int stages_for(int bn) {
    const int stage = kXStage + bn * kBK * 2;
    const int avail = kMaxSmem - 1024 - 256;
    return std::min(8, avail / stage);
}

size_t smem_for(int bn, int stages) {
    return size_t(stages) * (kXStage + bn * kBK * 2) + 1024 + 256;
}

cudaError_t launch_tc(int mode, const CUtensorMap& tx, const CUtensorMap& ty, TcParams p,
                      dim3 grid, cudaStream_t st) {
    static bool attr[2] = {false, false};
    const size_t smem = smem_for(p.bn, p.stages);
    cudaError_t e;
    if (mode == kTcRowdot) {
        if (!attr[0]) {
            e = cudaFuncSetAttribute(tc_rowdot<kTcRowdot>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     kMaxSmem);
            if (e != cudaSuccess) return e;
            attr[0] = true;
        }
        tc_rowdot<kTcRowdot><<<grid, kThreads, smem, st>>>(tx, ty, p);
    } else {
        if (!attr[1]) {
            e = cudaFuncSetAttribute(tc_rowdot<kTcStore>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     kMaxSmem);
            if (e != cudaSuccess) return e;
            attr[1] = true;
        }
        tc_rowdot<kTcStore><<<grid, kThreads, smem, st>>>(tx, ty, p);
    }
    return cudaGetLastError();
}

// (n_split, k_split) for a rowdot GEMM with m_tiles 128-row tiles: fill the 148 SMs in
// as few waves as possible; BN <= 256.  Prefers N splits (keeps the base_sq chain of a
// row in one CTA, bitwise) and uses K splits only when N splitting cannot fill.
struct Split { int ns, ks, bn; };

Split choose_split(int64_t m_tiles, int64_t r, int64_t kb_total, int max_ks) {
    const int kSMs = 148;
    Split best{1, 1, 0};
    double best_score = -1.0;
    const int ns_min = static_cast<int>((r + 255) / 256);
    for (int ns = ns_min; ns <= 8; ++ns) {
        const int bn = static_cast<int>(((r + ns - 1) / ns + 15) / 16 * 16);
        if (bn > 256 || bn < 16) continue;
        if (ns > ns_min && bn < 64) break;
        for (int ks = 1; ks <= max_ks && ks <= 8; ks *= 2) {
            if (ks > 1 && kb_total / ks < 4) break;
            const int64_t ctas = m_tiles * ns * ks;
            const int64_t waves = (ctas + kSMs - 1) / kSMs;
            const double eff = double(ctas) / double(waves * kSMs);
            // penalise redundant operand traffic from splitting
            const double score = eff - 0.02 * (ns - ns_min) - 0.03 * (ks > 1 ? ks : 0);
            if (score > best_score + 1e-9) {
                best_score = score;
                best = {ns, ks, bn};
            }
        }
    }
    return best;
}

}  // namespace

bool norm_tc_supported(int dt, int64_t d_out, int64_t d_in, int64_t r) {
    return dt == kBF16 && d_in >= 64 && d_in % 8 == 0 && r % 8 == 0 && r >= 16 && r <= 2048 &&
           d_out >= 1 && d_in < (int64_t(1) << 31) && d_out < (int64_t(1) << 31);
}

cudaError_t launch_norm_tc(const NormArgs& a, Workspace* ws, cudaStream_t st, int* launches) {
    if (!norm_tc_supported(a.dt, a.d_out, a.d_in, a.r)) return cudaErrorNotSupported;
    cudaError_t err = cudaSuccess;
    const int64_t r = a.r, d_out = a.d_out, d_in = a.d_in;
    const int64_t r_pad = (r + kBK - 1) / kBK * kBK;

    // ---------------- G = A A^T (upper-triangle tiles, split-K) ----------------
    const int nt = static_cast<int>((r + kBM - 1) / kBM);
    const int tiles = nt * (nt + 1) / 2;
    const int64_t kb_in = (d_in + kBK - 1) / kBK;
    int g_ks = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(148 / tiles, kb_in / 4)));
    const int g_kbps = static_cast<int>((kb_in + g_ks - 1) / g_ks);
    g_ks = static_cast<int>((kb_in + g_kbps - 1) / g_kbps);
    float* gpart = static_cast<float*>(
        ws_get(ws, kWsGramPart, size_t(g_ks) * tiles * kBM * kBM * sizeof(float), &err));
    if (err != cudaSuccess) return err;
    __nv_bfloat16* g2 = static_cast<__nv_bfloat16*>(
        ws_get(ws, kWsGram2, size_t(r) * 2 * r_pad * sizeof(__nv_bfloat16), &err));
    if (err != cudaSuccess) return err;
    {
        CUtensorMap ta;
        err = make_tmap_2d(&ta, kBF16, a.a, r, d_in, d_in * 2, kBK, kBM, true);
        if (err != cudaSuccess) return err;
        TcParams p{};
        p.M = r; p.N = r; p.k_total = d_in; p.kb_per_split = g_kbps; p.n_split = 1;
        p.bn = kBM; p.stages = stages_for(kBM); p.chunk = a.chunk_size;
        p.out = gpart; p.gram_nt = nt;
        err = launch_tc(kTcStore, ta, ta, p, dim3(tiles, g_ks), st);
        if (err != cudaSuccess) return err;
        const int64_t n = r * r_pad;
        gram_reduce<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(gpart, g_ks, nt, r,
                                                                             r_pad, g2);
        err = cudaGetLastError();
        if (err != cudaSuccess) return err;
        if (launches) *launches += 2;
    }

    const int64_t m_tiles = (d_out + kBM - 1) / kBM;
    // ---------------- ba_sq partials: rowdot(B [G_hi|G_lo], B) ----------------
    const Split sb = choose_split(m_tiles, r, 2 * r_pad / kBK, 1);
    float* ba = static_cast<float*>(ws_get(ws, kWsBa, size_t(sb.ns) * d_out * sizeof(float), &err));
    if (err != cudaSuccess) return err;
    {
        CUtensorMap tb, tg;
        err = make_tmap_2d(&tb, kBF16, a.b, d_out, r, r * 2, kBK, kBM, true);
        if (err != cudaSuccess) return err;
        err = make_tmap_2d(&tg, kBF16, g2, r, 2 * r_pad, 2 * r_pad * 2, kBK, sb.bn, true);
        if (err != cudaSuccess) return err;
        TcParams p{};
        p.M = d_out; p.N = r; p.k_total = 2 * r_pad;
        p.kb_per_split = static_cast<int>(2 * r_pad / kBK);
        p.n_split = sb.ns; p.bn = sb.bn; p.stages = stages_for(sb.bn);
        p.x_kwrap = static_cast<int>(r_pad); p.chunk = a.chunk_size;
        p.Z = static_cast<const __nv_bfloat16*>(a.b); p.ldz = r;
        p.out = ba; p.do_chain = 0;
        err = launch_tc(kTcRowdot, tb, tg, p, dim3(static_cast<unsigned>(m_tiles * sb.ns), 1), st);
        if (err != cudaSuccess) return err;
        if (launches) ++*launches;
    }

    // ---------------- cross partials + base_sq chain: rowdot(W A^T, B) ----------------
    // K splits only on ChunkPlan boundaries (each split = whole chunks)
    const int64_t chunk_blocks = a.chunk_size / kBK;
    const int64_t n_chunks = (d_in + a.chunk_size - 1) / a.chunk_size;
    const Split su = choose_split(m_tiles, r, kb_in, static_cast<int>(std::min<int64_t>(n_chunks, 8)));
    const int64_t chunks_per_split = (n_chunks + su.ks - 1) / su.ks;
    const int kbps = static_cast<int>(chunks_per_split * chunk_blocks);
    const int ks = static_cast<int>((kb_in + kbps - 1) / kbps);
    float* cross = static_cast<float*>(
        ws_get(ws, kWsCross, size_t(ks) * su.ns * d_out * sizeof(float), &err));
    if (err != cudaSuccess) return err;
    float* base = static_cast<float*>(
        ws_get(ws, kWsBase, size_t(n_chunks) * d_out * sizeof(float), &err));
    if (err != cudaSuccess) return err;
    {
        CUtensorMap tw, ta;
        err = make_tmap_2d(&tw, kBF16, a.w, d_out, d_in, d_in * 2, kBK, kBM, true);
        if (err != cudaSuccess) return err;
        err = make_tmap_2d(&ta, kBF16, a.a, r, d_in, d_in * 2, kBK, su.bn, true);
        if (err != cudaSuccess) return err;
        TcParams p{};
        p.M = d_out; p.N = r; p.k_total = d_in; p.kb_per_split = kbps;
        p.n_split = su.ns; p.bn = su.bn; p.stages = stages_for(su.bn);
        p.x_kwrap = 0; p.chunk = a.chunk_size;
        p.Z = static_cast<const __nv_bfloat16*>(a.b); p.ldz = r;
        p.out = cross; p.base_out = base; p.do_chain = 1;
        err = launch_tc(kTcRowdot, tw, ta, p,
                        dim3(static_cast<unsigned>(m_tiles * su.ns), static_cast<unsigned>(ks)), st);
        if (err != cudaSuccess) return err;
        if (launches) ++*launches;
    }

    FinishArgs f{};
    f.base_part = base; f.base_parts = static_cast<int>(n_chunks);
    f.cross_part = cross; f.cross_parts = ks * su.ns;
    f.ba_part = ba; f.ba_parts = sb.ns;
    f.d_out = d_out; f.two_s = 2.0 * a.s; f.s2 = a.s * a.s;
    f.base_sq = a.base_sq; f.cross = a.cross; f.ba_sq = a.ba_sq;
    f.round_dt = a.round_dt; f.w_norm = a.w_norm;
    f.m = a.m; f.mag_dt = a.mag_dt; f.g = a.m ? a.g : nullptr;
    if (launches) ++*launches;
    return launch_finish(f, st);
}

}  // namespace dfx
