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
// warps 0..3 own TMEM lane quadrants 0..3 (one row per thread) for the chain and
// the epilogue (tcgen05.ld 32x32b.x32); warp 4 produces, warp 5 issues MMAs.
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "norm_common.cuh"

namespace dfx {
namespace {

constexpr int kBM = 128;
constexpr int kBK = 64;                          // one 128-byte swizzle atom of bf16
constexpr int kXStage = kBM * kBK * 2;           // 16 KiB
constexpr int kThreads = 256;
// Warp roles (SMSP = wid % 4).  Epilogue warps are 0..3 so that warp w owns TMEM lane
// quadrant w; the producer (4) and MMA issuer (5) share SMSPs 0 and 1 with epilogue warps
// that are idle during the main loop, and the base_sq chain runs on warps 2 and 3, whose
// SMSPs carry no pipeline role (see chain_units).
constexpr int kWarpProducer = 4;
constexpr int kWarpMma = 5;
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
    const void* Z; int64_t ldz;   // bf16, or fp32 in the 3xTF32 kernel
    float* out;             // rowdot: [k_split*n_split][M]; store: tiles
    float* base_out;        // chain: [num_chunks][M], one serial partial per chunk
    int do_chain;
    // store (gram): tile index mapping
    int gram_nt;            // tiles per side
    int tiles;              // tiles per K split (the persistent loop's extent)
    int w_prefetch;         // K blocks of X (W) prefetched into L2 ahead of the loads
    int nh;                 // pair kernel: UMMAs per K step (N per CTA pair = nh * bn)
    int ka;                 // pair kernel: 64-wide K blocks ("atoms") per ring stage (1 or 2)
    int tma3d;              // pair kernel: tmx / tmy are K-atom 3-D maps, one TMA per operand per stage
    int zsmem;              // pair kernel, one tile per CTA: the epilogue's B rows arrive by TMA
                            // into a ring slot freed after the last K stage (tmz, 128B swizzle)
    const float* out_scale; // rowdot: multiply each row's sum by *out_scale (fp16 V: 2^-e)
    // Fused finisher (rowdot): every tile of a 128-row block counts itself in
    // fin_count[block]; the tile completing the block (fin_total tiles over U and V) runs
    // finish_row for its rows, so no separate finish launch sits on the critical path.
    // Blocks past M (the phantom half of a 256-row pair tile) never count: only real blocks
    // have counters, and every kernel contributes to each real block exactly once per tile.
    FinishArgs fin;
    unsigned* fin_count;
    int fin_total;
};

// Epilogue warps 0..3 (128 threads) after a tile's outputs are stored: count the tile in
// its group; true in all 128 threads of the CTA whose tile completed the group.  The last
// arrival resets the counter, so the next launch (stream-ordered) starts from zero.
// `flag` is a word of the CTA's barrier area (no static shared memory: the kernels use the
// whole 227 KiB opt-in dynamically).  Ordering: the named barrier orders the 128 threads'
// stores before thread 0's acq_rel atomic at GPU scope (cumulative release: the same
// pattern as a CTA-wide semaphore), and the winner's acquire is ordered before the other
// threads' loads by the second barrier; -DDFX_FENCE_ALL keeps a fence in every thread.
__device__ __forceinline__ bool last_arrival(unsigned* count, int total, volatile uint32_t* flag) {
#ifdef DFX_FENCE_ALL
    __threadfence();
#endif
    named_bar_sync(1, 128);
    if (threadIdx.x == 0) {
        unsigned old;
        asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(count) : "memory");
        const bool last = old + 1u == static_cast<unsigned>(total);
        if (last) atomicExch(count, 0u);
        *flag = last ? 1u : 0u;
    }
    named_bar_sync(1, 128);
    const bool last = *flag != 0;
#ifdef DFX_FENCE_ALL
    if (last) __threadfence();
#endif
    return last;
}

// -DDFX_TRACE (experiment builds only): the pair kernel stamps %globaltimer at pipeline events
// of its first kTrN stages into g_trace[cta][ev][i]; the launcher appends the array to the file
// named by $DFX_TRACE after the launch (events: 0 producer issues stage j, 1 MMA sees stage i
// full, 2 MMA released stage i, 3 producer sees stage j empty).
#ifdef DFX_TRACE
constexpr int kTrN = 128, kTrEv = 4, kTrCta = 148;
__device__ unsigned long long g_trace[kTrCta][kTrEv][kTrN];
// V (tc_pair_gstat) timeline per CTA: 0 entry, 1 after the cluster sync, 2 producer issued the
// G slice, 3 MMA saw the G slice, 4 MMA saw the first B stage, 5 MMA issued the tile's last
// commit, 6 epilogue had its B slice in registers, 7 epilogue saw the accumulator, 8 epilogue
// stored ba_sq, 9 epilogue done (finisher included)
constexpr int kVtrEv = 10;
__device__ unsigned long long g_vtrace[kTrCta][kVtrEv];
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define DFX_TR(ev, i) do { if ((i) < kTrN && blockIdx.x < kTrCta) g_trace[blockIdx.x][ev][i] = gtimer(); } while (0)
#define VTR(ev) do { if (blockIdx.x < kTrCta) g_vtrace[blockIdx.x][ev] = gtimer(); } while (0)
#else
#define DFX_TR(ev, i) do { } while (0)
#define VTR(ev) do { } while (0)
#endif

__device__ __forceinline__ void unpack_bf16x8(const uint4& v, float (&f)[8]) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        f[2 * i] = __uint_as_float(w[i] << 16);
        f[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
    }
}

// Eight 16-bit elements of the operand dtype (kEl = kBF16 or kF16) widened to fp32 (exact).
template <int kEl>
__device__ __forceinline__ void unpack8(const uint4& v, float (&f)[8]) {
    if (kEl == kBF16) {
        unpack_bf16x8(v, f);
    } else {
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float2 t = __half22float2(*reinterpret_cast<const __half2*>(&w[i]));
            f[2 * i] = t.x;
            f[2 * i + 1] = t.y;
        }
    }
}

// kind::f16 instruction-descriptor operand format: 1 = bf16, 0 = fp16.
__host__ __device__ constexpr uint32_t ab_fmt(int el) { return el == kBF16 ? 1u : 0u; }

// The base_sq chain of a row tile (4 units of 32 rows) is spread over the CTAs that
// share the tile (its N splits): unit u belongs to the CTA whose N index is u*n_split/4.
// Inside a CTA only warps 2 and 3 chain (up to two units = two interleaved rows per
// thread): they share SMSPs with no single-thread pipeline role, so the chain's
// dependent FADD stream neither starves nor is starved by the producer / MMA issuer.
struct ChainUnits {
    int n;
    int u[2];
};

__device__ __forceinline__ ChainUnits chain_units(int warp, int n_idx, int n_split) {
    ChainUnits cu{0, {0, 0}};
    if (warp != 2 && warp != 3) return cu;
    int pos = 0;
    for (int u = 0; u < 4; ++u) {
        if ((u * n_split / 4) != n_idx) continue;
        if ((pos & 1) == warp - 2 && cu.n < 2) cu.u[cu.n++] = u;
        ++pos;
    }
    return cu;
}

__device__ __forceinline__ int chain_active_warps(int n_idx, int n_split) {
    return (chain_units(2, n_idx, n_split).n > 0) + (chain_units(3, n_idx, n_split).n > 0);
}

// Serial fp32 sum of w*w for kRows rows of the tile (rows 32*u + lane), one partial per
// ChainPlan chunk (factored_norm.cpp:52-60); partials go to base_out[chunk][row] and the
// finisher adds them in ascending order (:60), so base_sq is bitwise the reference's.
// The stage is released only after the chain consumed its registers.
template <int kRows, int kEl = kBF16>
__device__ __forceinline__ void chain_tile(const ChainUnits& cu, const uint8_t* smem,
                                           int stage_bytes, uint64_t* ready, uint64_t* empty,
                                           int stages, int start, int nkb, int kb0, int64_t chunk,
                                           int64_t m0, int64_t M, float* base_out, int lane,
                                           int ka = 1) {
    constexpr bool kIsF32 = kEl == kF32;
    int s = start % stages;
    uint32_t ph = static_cast<uint32_t>((start / stages) & 1);
    float part[kRows];
    int row[kRows];
#pragma unroll
    for (int j = 0; j < kRows; ++j) {
        part[j] = 0.0f;
        row[j] = 32 * cu.u[j] + lane;
    }
    int64_t kpos = int64_t(kb0) * (kIsF32 ? 32 : 64);
    int64_t cur = kpos / chunk;
    int64_t boundary = (cur + 1) * chunk;
    for (int it = 0; it < nkb; ++it) {
        mbar_wait(&ready[s], ph);
        for (int a = 0; a < ka; ++a) {   // K atoms of the stage, ascending K (X atoms first)
        uint4 v[kRows][8];
#pragma unroll
        for (int j = 0; j < kRows; ++j) {
            const uint8_t* rowp = smem + s * stage_bytes + a * kXStage + row[j] * 128;
#pragma unroll
            for (int c = 0; c < 8; ++c)
                v[j][c] = *reinterpret_cast<const uint4*>(rowp + ((c ^ (row[j] & 7)) << 4));
        }
        if (kpos >= boundary) {
#pragma unroll
            for (int j = 0; j < kRows; ++j) {
                if (m0 + row[j] < M) base_out[cur * M + m0 + row[j]] = part[j];
                part[j] = 0.0f;
            }
            ++cur;
            boundary += chunk;
        }
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            constexpr int kE = kIsF32 ? 4 : 8;             // elements per 16-byte chunk
            float f[kRows][8];
#pragma unroll
            for (int j = 0; j < kRows; ++j) {
                if (kIsF32) {
                    f[j][0] = __uint_as_float(v[j][c].x); f[j][1] = __uint_as_float(v[j][c].y);
                    f[j][2] = __uint_as_float(v[j][c].z); f[j][3] = __uint_as_float(v[j][c].w);
                } else {
                    unpack8<kEl>(v[j][c], f[j]);
                }
            }
#pragma unroll
            for (int e = 0; e < kE; ++e)
#pragma unroll
                for (int j = 0; j < kRows; ++j)
                    part[j] = __fadd_rn(part[j], __fmul_rn(f[j][e], f[j][e]));
        }
        kpos += kIsF32 ? 32 : 64;
        }
        // The release lets the TMA (async proxy) refill the slot.  Every loaded word fed the
        // FADD chain above, and in-order issue puts the arrive after those FADDs, which wait
        // for the loads' data: the generic reads are complete before the release, so no
        // fence.proxy.async is needed here (a ring whose reads are NOT consumed before the
        // release needs one: profiles/r02_lora_tma_base.txt).
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        if (++s == stages) { s = 0; ph ^= 1; }
    }
#pragma unroll
    for (int j = 0; j < kRows; ++j)
        if (m0 + row[j] < M) base_out[cur * M + m0 + row[j]] = part[j];
}

// Tile t of split z (blockIdx.y): rowdot -> (m, n) = (t / n_split, t % n_split), adjacent
// tiles share the X (W) rows; store (Gram) -> the t-th upper-triangle tile (pi <= qi).
__device__ __forceinline__ void tile_coords(int kMode, const TcParams& p, int t, int64_t& m0,
                                            int64_t& n0) {
    if (kMode == kTcStore) {
        int pi = 0;
        while (t >= p.gram_nt - pi) { t -= p.gram_nt - pi; ++pi; }
        m0 = int64_t(pi) * kBM;
        n0 = int64_t(pi + t) * p.bn;
    } else {
        m0 = int64_t(t / p.n_split) * kBM;
        n0 = int64_t(t % p.n_split) * p.bn;
    }
}

// Persistent: CTA b walks tiles b, b + gridDim.x, ...; the smem stage ring and its
// phases run on across tiles, and the TMEM accumulator is double-buffered (2 x BN
// columns) so the MMA of tile i+1 overlaps the epilogue of tile i.
// kF32: the 3xTF32 variant for fp32 operands.  A K block is 32 fp32 (the same 128-byte
// swizzle row); two split warps write each stage's low parts x - tf32(x) next to the raw
// tiles, and every K=8 step issues three kind::tf32 UMMAs, X.Y + X.Y_lo + X_lo.Y (the raw
// fp32 operand is read as its TF32 truncation), which carries ~2^-21 relative error —
// fp32-class accumulation on the tensor cores.
constexpr int kSplitWarps = 4;                   // 3xTF32: warps 6 .. 6 + kSplitWarps - 1

template <int kMode, int kEl = kBF16>
__global__ void __launch_bounds__(kEl == kF32 ? kThreads + 32 * (kSplitWarps - 2) : kThreads, 1)
    tc_rowdot(const __grid_constant__ CUtensorMap tmx, const __grid_constant__ CUtensorMap tmy,
              const TcParams p) {
    constexpr bool kIsF32 = kEl == dfx::kF32;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    const int y_stage = p.bn * kBK * 2;
    const int raw_bytes = kXStage + y_stage;    // both multiples of 1024
    const int stage_bytes = kIsF32 ? 2 * raw_bytes : raw_bytes;   // [raw X | raw Y | lo X | lo Y]
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + p.stages * stage_bytes);
    uint64_t* empty = full + p.stages;
    uint64_t* tmem_full = empty + p.stages;     // [2]
    uint64_t* tmem_empty = tmem_full + 2;       // [2]
    uint64_t* split = tmem_empty + 2;           // [stages] (kIsF32: low parts written)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(split + p.stages);

    const int warp = warp_id(), lane = lane_id();
    const int ks = blockIdx.y;
    const int kb0 = ks * p.kb_per_split;
    constexpr int kBKe = kIsF32 ? 32 : kBK;       // K elements per 128-byte block
    const int64_t total_kb = (p.k_total + kBKe - 1) / kBKe;
    const int64_t kb_left = total_kb - kb0;
    const int nkb = static_cast<int>(kb_left < p.kb_per_split ? kb_left : p.kb_per_split);
    const bool do_chain = (kMode == kTcRowdot) && p.do_chain;

    // two accumulator slots, each starting on a 32-column boundary
    const uint32_t slot_cols = static_cast<uint32_t>((p.bn + 31) / 32 * 32);
    uint32_t tmem_cols = 32;
    while (tmem_cols < 2 * slot_cols) tmem_cols <<= 1;

    if (threadIdx.x == 0) {
        tma_prefetch_desc(&tmx);
        tma_prefetch_desc(&tmy);
        for (int s = 0; s < p.stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1 + (do_chain ? 2 : 0));
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tmem_full[a], 1);
            mbar_init(&tmem_empty[a], 4);
        }
        for (int s = 0; s < p.stages; ++s) mbar_init(&split[s], kSplitWarps);
        fence_mbar_init();
    }
    if (warp == kWarpMma) {
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

    if (nkb > 0 && warp == kWarpProducer) {
        // ================= TMA producer =================
        if (lane == 0) {
            const uint64_t pol_x = (kMode == kTcRowdot && !p.x_kwrap && p.n_split == 1)
                                       ? policy_evict_first()
                                       : policy_evict_last();
            const uint64_t pol_y = policy_evict_last();
            int s = 0;
            uint32_t ph = 0;
            const int pf = p.w_prefetch;
            for (int t = blockIdx.x; t < p.tiles; t += gridDim.x) {
                int64_t m0, n0;
                tile_coords(kMode, p, t, m0, n0);
                for (int it = 0; it < pf && it < nkb; ++it)
                    tma_prefetch_2d(&tmx, (kb0 + it) * kBK, static_cast<int32_t>(m0));
                for (int it = 0; it < nkb; ++it) {
                    if (pf > 0 && it + pf < nkb)   // (pf = 0: no prefetch — not of the block being loaded)
                        tma_prefetch_2d(&tmx, (kb0 + it + pf) * kBK, static_cast<int32_t>(m0));
                    mbar_wait(&empty[s], ph ^ 1);
                    mbar_arrive_expect_tx(&full[s], raw_bytes);
                    uint8_t* sx = smem + s * stage_bytes;
                    uint8_t* sy = sx + kXStage;
                    const int kc = (kb0 + it) * (kIsF32 ? 32 : kBK);
                    const int kx = (p.x_kwrap && kc >= p.x_kwrap) ? kc - p.x_kwrap : kc;
                    tma_load_2d(&tmx, &full[s], sx, kx, static_cast<int32_t>(m0), pol_x);
                    tma_load_2d(&tmy, &full[s], sy, kc, static_cast<int32_t>(n0), pol_y);
                    if (++s == p.stages) { s = 0; ph ^= 1; }
                }
            }
        }
    } else if (nkb > 0 && warp == kWarpMma) {
        // ================= MMA issuer (single thread) =================
        if (lane == 0) {
            const uint32_t idesc = kIsF32 ? umma_idesc_tf32(kBM, static_cast<uint32_t>(p.bn))
                                        : umma_idesc_f16(ab_fmt(kEl), kBM, static_cast<uint32_t>(p.bn));
            int s = 0;
            uint32_t ph = 0;
            int local = 0;
            for (int t = blockIdx.x; t < p.tiles; t += gridDim.x, ++local) {
                int64_t m0, n0;
                tile_coords(kMode, p, t, m0, n0);
                const int stand_in = do_chain ? 2 - chain_active_warps(t % p.n_split, p.n_split) : 0;
                const int slot = local & 1;
                const uint32_t tacc = tmem_base + static_cast<uint32_t>(slot) * slot_cols;
                mbar_wait(&tmem_empty[slot], ((local >> 1) & 1) ^ 1);
                tc_fence_after();
                for (int it = 0; it < nkb; ++it) {
                    mbar_wait(kIsF32 ? &split[s] : &full[s], ph);
                    tc_fence_after();
                    const uint32_t sx = smem_u32(smem + s * stage_bytes);
                    const uint32_t sy = sx + kXStage;
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const uint64_t ad = umma_desc_k_sw128(sx + k * 32);
                        const uint64_t bd = umma_desc_k_sw128(sy + k * 32);
                        if (kIsF32) {
                            const uint64_t adl = umma_desc_k_sw128(sx + raw_bytes + k * 32);
                            const uint64_t bdl = umma_desc_k_sw128(sy + raw_bytes + k * 32);
                            umma_tf32(tacc, ad, bd, idesc, (it > 0 || k > 0) ? 1u : 0u);
                            umma_tf32(tacc, ad, bdl, idesc, 1u);
                            umma_tf32(tacc, adl, bd, idesc, 1u);
                        } else {
                            umma_f16(tacc, ad, bd, idesc, (it > 0 || k > 0) ? 1u : 0u);
                        }
                    }
                    umma_commit(&empty[s]);
                    // stand in for the epilogue warps that do not chain in this tile
                    if (stand_in) mbar_arrive_cnt(&empty[s], stand_in);
                    if (++s == p.stages) { s = 0; ph ^= 1; }
                }
                umma_commit(&tmem_full[slot]);
            }
        }
    } else if (kIsF32 && nkb > 0 && warp >= 6) {
        // ================= 3xTF32 split: low parts x - tf32(x) of both tiles ==========
        const int st = (warp - 6) * 32 + lane;                  // 0 .. 32 * kSplitWarps - 1
        constexpr int kST = 32 * kSplitWarps;
        int s = 0;
        uint32_t ph = 0;
        for (int t = blockIdx.x; t < p.tiles; t += gridDim.x) {
            for (int it = 0; it < nkb; ++it) {
                mbar_wait(&full[s], ph);
                const uint32_t src = smem_u32(smem + s * stage_bytes);
                const uint32_t dst = src + static_cast<uint32_t>(raw_bytes);
                // batches of 8 16-byte words per thread: all loads first, then the stores
                const int n16 = raw_bytes / 16;
                for (int i0 = st; i0 < n16; i0 += kST * 8) {
                    uint32_t w[8][4];
#pragma unroll
                    for (int b = 0; b < 8; ++b) {
                        const int i = i0 + kST * b;
                        if (i < n16)
                            asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                                         : "=r"(w[b][0]), "=r"(w[b][1]), "=r"(w[b][2]), "=r"(w[b][3])
                                         : "r"(src + i * 16));
                    }
#pragma unroll
                    for (int b = 0; b < 8; ++b) {
                        const int i = i0 + kST * b;
                        if (i >= n16) break;
                        uint32_t l[4];
#pragma unroll
                        for (int e = 0; e < 4; ++e)
                            l[e] = __float_as_uint(__fsub_rn(__uint_as_float(w[b][e]),
                                                             __uint_as_float(w[b][e] & 0xFFFFE000u)));
                        asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(dst + i * 16),
                                     "r"(l[0]), "r"(l[1]), "r"(l[2]), "r"(l[3])
                                     : "memory");
                    }
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive(&split[s]);
                if (++s == p.stages) { s = 0; ph ^= 1; }
            }
        }
    } else if (nkb > 0 && warp < 4) {
        // ================= chain + epilogue (one row per thread) =================
        const int q = warp;               // TMEM lane quadrant
        const int row = q * 32 + lane;        // row inside the tile
        int local = 0;
        for (int t = blockIdx.x; t < p.tiles; t += gridDim.x, ++local) {
            int64_t m0, n0;
            tile_coords(kMode, p, t, m0, n0);
            const int64_t gm = m0 + row;
            if (do_chain) {
                const ChainUnits cu = chain_units(warp, static_cast<int>(t % p.n_split), p.n_split);
                if (cu.n == 2)
                    chain_tile<2, kEl>(cu, smem, stage_bytes, full, empty, p.stages, local * nkb, nkb,
                                        kb0, p.chunk, m0, p.M, p.base_out, lane);
                else if (cu.n == 1)
                    chain_tile<1, kEl>(cu, smem, stage_bytes, full, empty, p.stages, local * nkb, nkb,
                                        kb0, p.chunk, m0, p.M, p.base_out, lane);
            }
            // ---- epilogue: TMEM accumulator -> rowdot / tile store
            const int slot = local & 1;
            mbar_wait(&tmem_full[slot], (local >> 1) & 1);
            tc_fence_after();
            const uint32_t trow = tmem_base + static_cast<uint32_t>(slot) * slot_cols +
                                  (static_cast<uint32_t>(q * 32) << 16);
            if (kMode == kTcRowdot) {
                float acc = 0.0f;
                for (int c0 = 0; c0 < p.bn; c0 += 32) {
                    uint32_t u[32];
                    tmem_ld_32x32b_x32(trow + c0, u);
                    tmem_ld_wait();
                    if (gm < p.M) {
#pragma unroll
                        for (int v = 0; v < 4; ++v) {
                            // columns past the tile (bn % 32 != 0) belong to the other slot
                            if (c0 + 8 * v < p.bn && n0 + c0 + 8 * v < p.N) {
                                float z[8];
                                if (kIsF32) {
                                    const float* zr = static_cast<const float*>(p.Z) + gm * p.ldz + n0 + c0;
                                    const float4 z0 = *reinterpret_cast<const float4*>(zr + 8 * v);
                                    const float4 z1 = *reinterpret_cast<const float4*>(zr + 8 * v + 4);
                                    z[0] = z0.x; z[1] = z0.y; z[2] = z0.z; z[3] = z0.w;
                                    z[4] = z1.x; z[5] = z1.y; z[6] = z1.z; z[7] = z1.w;
                                } else {
                                    const uint16_t* zr =
                                        static_cast<const uint16_t*>(p.Z) + gm * p.ldz + n0 + c0;
                                    unpack8<kEl>(*reinterpret_cast<const uint4*>(zr + 8 * v), z);
                                }
#pragma unroll
                                for (int e = 0; e < 8; ++e)
                                    acc = fmaf(__uint_as_float(u[8 * v + e]), z[e], acc);
                            }
                        }
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&tmem_empty[slot]);
                if (p.out_scale) acc = __fmul_rn(acc, *p.out_scale);   // exact power of two
                if (gm < p.M) p.out[(int64_t(ks) * p.n_split + (n0 / p.bn)) * p.M + gm] = acc;
                if (p.fin_count && m0 < p.M && last_arrival(p.fin_count + m0 / kBM, p.fin_total, tmem_slot + 1) && gm < p.M)
                    finish_row(p.fin, gm);
            } else {
                // gram tile store: out[(ks * tiles + t) * 128*bn + row*bn + col]
                float* dst = p.out + (int64_t(ks) * p.tiles + t) * (int64_t(kBM) * p.bn) +
                             int64_t(row) * p.bn;
                for (int c0 = 0; c0 < p.bn; c0 += 32) {
                    uint32_t u[32];
                    tmem_ld_32x32b_x32(trow + c0, u);
                    tmem_ld_wait();
#pragma unroll
                    for (int e = 0; e < 32; e += 4)
                        *reinterpret_cast<float4*>(dst + c0 + e) =
                            make_float4(__uint_as_float(u[e]), __uint_as_float(u[e + 1]),
                                        __uint_as_float(u[e + 2]), __uint_as_float(u[e + 3]));
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&tmem_empty[slot]);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == kWarpMma) {
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

// 2-SM (cta_group::2) variant of the W.A^T rowdot, used for the dominant GEMM.
//
// A cluster of two CTAs owns a 256-row pair tile: each CTA stages its own 128 W rows and
// HALF of the BN A rows, so per-SM operand ingest per K block drops from
// 16 KiB + BN*128 B to 16 KiB + BN*64 B for the same MMA work; the leader (rank 0)
// issues tcgen05.mma.cta_group::2 (M = 256) reading both CTAs' shared memory and
// accumulating into both CTAs' TMEM (each its own 128 rows).  Both CTAs' TMA loads
// complete on the leader's full barrier; the leader forwards "stage full" to the peer
// (whose chain warps read their own W rows) and multicasts its commits to both CTAs'
// empty / tmem_full barriers; both CTAs' epilogue warps release the accumulator slot on
// the leader's tmem_empty barrier.
template <int kEl>
__global__ void __launch_bounds__(kThreads, 1)
    tc_pair_rowdot(const __grid_constant__ CUtensorMap tmx, const __grid_constant__ CUtensorMap tmy,
                   const __grid_constant__ CUtensorMap tmz, const TcParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    const int half_n = p.bn / 2;                          // A rows per CTA per UMMA
    const int nh = p.nh > 0 ? p.nh : 1;
    const int ka = p.ka > 0 ? p.ka : 1;                   // K atoms per stage
    const int y_bytes = half_n * kBK * 2;
    // this CTA's share of a stage: [X atom 0 .. ka-1 | Y (h, atom) h-major]
    const int stage_bytes = ka * (kXStage + nh * y_bytes);
    const int bn_pair = nh * p.bn;                        // N of the pair's tile
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + p.stages * stage_bytes);
    uint64_t* pfull = full + p.stages;
    uint64_t* empty = pfull + p.stages;
    uint64_t* tmem_full = empty + p.stages;     // [2]
    uint64_t* tmem_empty = tmem_full + 2;       // [2]
    uint64_t* zfull = tmem_empty + 2;           // the epilogue's B tile landed (p.zsmem)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(zfull + 1);

    const int warp = warp_id(), lane = lane_id();
    const uint32_t rank = cluster_ctarank();
    const bool leader = rank == 0;
    const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
    const int ks = blockIdx.y;
    const int kb0 = ks * p.kb_per_split;
    const int64_t total_kb = (p.k_total + kBK - 1) / kBK;
    const int64_t kb_left = total_kb - kb0;
    const int nkb_blocks = static_cast<int>(kb_left < p.kb_per_split ? kb_left : p.kb_per_split);
    const int nkb = nkb_blocks / ka;             // ring stages per tile (the planner keeps ka | nkb)
    const bool do_chain = p.do_chain != 0;

    // accumulator slots: double-buffered when two fit in the 512 TMEM columns
    const uint32_t slot_cols = static_cast<uint32_t>((bn_pair + 31) / 32 * 32);
    const int nslots = slot_cols * 2 <= 512 ? 2 : 1;
    uint32_t tmem_cols = 32;
    while (tmem_cols < nslots * slot_cols) tmem_cols <<= 1;

    if (threadIdx.x == 0) {
        tma_prefetch_desc(&tmx);
        tma_prefetch_desc(&tmy);
        for (int s = 0; s < p.stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&pfull[s], 1);
            mbar_init(&empty[s], 1 + (do_chain ? 2 : 0));
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tmem_full[a], 1);
            mbar_init(&tmem_empty[a], 8);
        }
        mbar_init(zfull, 1);
        fence_mbar_init();
    }
#ifdef DFX_KO_TMEM
    if (threadIdx.x == 0) *tmem_slot = 0;
    if (false) {
#else
    if (warp == kWarpMma) {
#endif
        switch (tmem_cols) {
            case 32: tmem_alloc_pair<32>(tmem_slot); break;
            case 64: tmem_alloc_pair<64>(tmem_slot); break;
            case 128: tmem_alloc_pair<128>(tmem_slot); break;
            case 256: tmem_alloc_pair<256>(tmem_slot); break;
            default: tmem_alloc_pair<512>(tmem_slot); break;
        }
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (nkb > 0 && warp == kWarpProducer) {
        // ================= TMA producer (both CTAs) =================
        if (lane == 0) {
            const uint64_t pol_x = p.n_split == 1 ? policy_evict_first() : policy_evict_last();
            const uint64_t pol_y = policy_evict_last();
            int s = 0;
            uint32_t ph = 0;
            const int pf = p.w_prefetch;
            for (int t = pair; t < p.tiles; t += npairs) {
                const int64_t m0 = int64_t(t / p.n_split) * (2 * kBM) + int64_t(rank) * kBM;
                const int64_t n0 = int64_t(t % p.n_split) * bn_pair + int64_t(rank) * half_n;
                // W streams from HBM in 128-byte row pieces: warm L2 `pf` K blocks ahead
                // (W's map is the 3-D K-atom view when p.tma3d: prefetch with its coordinates;
                // a 2-D prefetch on a 3-D map is an illegal instruction)
                auto prefetch_w = [&](int64_t kb) {
                    if (p.tma3d) tma_prefetch_3d(&tmx, 0, static_cast<int32_t>(m0), static_cast<int32_t>(kb));
                    else tma_prefetch_2d(&tmx, static_cast<int32_t>(kb * kBK), static_cast<int32_t>(m0));
                };
                for (int it = 0; it < pf && it < nkb_blocks; ++it) prefetch_w(kb0 + it);
                for (int it = 0; it < nkb; ++it) {
                    for (int a = 0; a < ka; ++a)
                        if (pf > 0 && it * ka + a + pf < nkb_blocks) prefetch_w(kb0 + it * ka + a + pf);
                    mbar_wait(&empty[s], ph ^ 1);
                    DFX_TR(3, it);
                    if (leader) mbar_arrive_expect_tx(&full[s], 2 * stage_bytes);
                    const uint32_t lbar = mapa_shared(smem_u32(&full[s]), 0);
                    uint8_t* sx = smem + s * stage_bytes;
                    uint8_t* sy = sx + ka * kXStage;
                    if (p.tma3d) {
                        // all ka atoms of an operand in one instruction ([atom][rows][64] tiles):
                        // half the TMA instructions of the 2-D form, whose per-instruction cost
                        // paced the bare ring (profiles/r02_u_knockouts.txt)
                        const int kb = kb0 + it * ka;
                        tma_load_3d_pair(&tmx, lbar, sx, 0, static_cast<int32_t>(m0), kb, pol_x);
                        for (int h = 0; h < nh; ++h)
                            tma_load_3d_pair(&tmy, lbar, sy + h * ka * y_bytes, 0,
                                             static_cast<int32_t>(n0 + int64_t(h) * p.bn), kb, pol_y);
                    } else {
                        for (int a = 0; a < ka; ++a) {
                            const int kc = (kb0 + it * ka + a) * kBK;
                            tma_load_2d_pair(&tmx, lbar, sx + a * kXStage, kc, static_cast<int32_t>(m0), pol_x);
                            for (int h = 0; h < nh; ++h)
                                tma_load_2d_pair(&tmy, lbar, sy + (h * ka + a) * y_bytes, kc,
                                                 static_cast<int32_t>(n0 + int64_t(h) * p.bn), pol_y);
                        }
                    }
                    DFX_TR(0, it);
                    if (++s == p.stages) { s = 0; ph ^= 1; }
                }
                if (p.zsmem) {
                    // this CTA's B rows of the tile (bn_pair columns, 64-column SW128 boxes)
                    // into the next ring slot once the tensor cores have released it
                    mbar_wait(&empty[s], ph ^ 1);
                    const int nbox = (bn_pair + kBK - 1) / kBK;
                    mbar_arrive_expect_tx(zfull, static_cast<uint32_t>(nbox * kXStage));
                    const int64_t zc = int64_t(t % p.n_split) * bn_pair;
                    uint8_t* sz = smem + s * stage_bytes;
                    for (int bx = 0; bx < nbox; ++bx)
                        tma_load_2d(&tmz, zfull, sz + bx * kXStage, static_cast<int32_t>(zc + bx * kBK),
                                    static_cast<int32_t>(m0), pol_y);
                }
            }
        }
    } else if (nkb > 0 && warp == kWarpMma) {
        // ================= MMA issuer (leader CTA, single thread) =================
        if (leader && lane == 0) {
            const uint32_t idesc = umma_idesc_f16(ab_fmt(kEl), 2 * kBM, static_cast<uint32_t>(p.bn));
            int s = 0;
            uint32_t ph = 0;
            int local = 0;
            for (int t = pair; t < p.tiles; t += npairs, ++local) {
                const int slot = nslots == 2 ? (local & 1) : 0;
                const int use = nslots == 2 ? (local >> 1) : local;
                const uint32_t tacc = tmem_base + static_cast<uint32_t>(slot) * slot_cols;
                mbar_wait(&tmem_empty[slot], (use & 1) ^ 1);
                tc_fence_after();
                for (int it = 0; it < nkb; ++it) {
                    mbar_wait(&full[s], ph);
                    DFX_TR(1, it);
#ifndef DFX_KO_FENCE
                    tc_fence_after();
#endif
                    const uint32_t sx0 = smem_u32(smem + s * stage_bytes);
                    for (int h = 0; h < nh; ++h) {
                        for (int a = 0; a < ka; ++a) {
                            const uint32_t sx = sx0 + a * kXStage;
                            const uint32_t sy = sx0 + ka * kXStage + (h * ka + a) * y_bytes;
#pragma unroll
                            for (int k = 0; k < kBK / 16; ++k) {
                                const uint64_t ad = umma_desc_k_sw128(sx + k * 32);
                                const uint64_t bd = umma_desc_k_sw128(sy + k * 32);
#ifndef DFX_KO_MMA
                                umma_f16_pair(tacc + static_cast<uint32_t>(h * p.bn), ad, bd, idesc,
                                              (it > 0 || a > 0 || k > 0) ? 1u : 0u);
#else
                                (void)ad; (void)bd;
#endif
                            }
                        }
                    }
                    DFX_TR(2, it);
#ifndef DFX_KO_COMMIT
                    umma_commit_pair_mc(&empty[s], 0x3);
#else
                    mbar_arrive(&empty[s]);
                    mbar_arrive_remote(mapa_shared(smem_u32(&empty[s]), 1), 1);
#endif
                    if (++s == p.stages) { s = 0; ph ^= 1; }
                }
#ifndef DFX_KO_TMEM
                umma_commit_pair_mc(&tmem_full[slot], 0x3);
#else
                mbar_arrive(&tmem_full[slot]);
                mbar_arrive_remote(mapa_shared(smem_u32(&tmem_full[slot]), 1), 1);
#endif
            }
        }
    } else if (nkb > 0 && warp < 4) {
        // ================= forwarder + chain + epilogue (own 128 rows) =================
        const int q = warp;
        const int row = q * 32 + lane;
        uint64_t* ready = leader ? full : pfull;   // "stage s landed" as seen by this CTA
        // Leader warp 0 (idle until the epilogue) forwards "stage landed" to the peer's
        // chain warps (the peer's TMA completes on the leader's barrier) and stands in for
        // the chain warps that do not chain this tile, in both CTAs.
        int fs = 0;
        uint32_t fph = 0;
        auto forward_tile = [&](int t) {
            if (lane == 0) {
                const int stand_in = do_chain ? 2 - chain_active_warps(t % p.n_split, p.n_split) : 0;
                for (int it = 0; it < nkb; ++it) {
                    mbar_wait(&full[fs], fph);
                    mbar_arrive_remote(mapa_shared(smem_u32(&pfull[fs]), 1), 1);
                    if (stand_in) {
                        mbar_arrive_cnt(&empty[fs], stand_in);
                        mbar_arrive_remote(mapa_shared(smem_u32(&empty[fs]), 1), stand_in);
                    }
                    if (++fs == p.stages) { fs = 0; fph ^= 1; }
                }
            }
            __syncwarp();
        };
        int local = 0;
        for (int t = pair; t < p.tiles; t += npairs, ++local) {
            const int64_t m0 = int64_t(t / p.n_split) * (2 * kBM) + int64_t(rank) * kBM;
            const int64_t n0 = int64_t(t % p.n_split) * bn_pair;
            const int64_t gm = m0 + row;
#ifndef DFX_KO_FWD
            if (leader && warp == 0) forward_tile(t);
#endif
            if (do_chain) {
                const ChainUnits cu = chain_units(warp, static_cast<int>(t % p.n_split), p.n_split);
                if (cu.n == 2)
                    chain_tile<2, kEl>(cu, smem, stage_bytes, ready, empty, p.stages, local * nkb, nkb, kb0,
                                  p.chunk, m0, p.M, p.base_out, lane, ka);
                else if (cu.n == 1)
                    chain_tile<1, kEl>(cu, smem, stage_bytes, ready, empty, p.stages, local * nkb, nkb, kb0,
                                  p.chunk, m0, p.M, p.base_out, lane, ka);
            }
            const int slot = nslots == 2 ? (local & 1) : 0;
            const int use = nslots == 2 ? (local >> 1) : local;
#ifdef DFX_SLEEPWAIT
            mbar_wait_sleep(&tmem_full[slot], use & 1, DFX_SLEEPWAIT);
#else
            mbar_wait(&tmem_full[slot], use & 1);
#endif
            tc_fence_after();
            const uint32_t trow = tmem_base + static_cast<uint32_t>(slot) * slot_cols +
                                  (static_cast<uint32_t>(q * 32) << 16);
            float acc = 0.0f;
            if (p.zsmem) {
                // B from the staged tile: row `row` of 64-column boxes, 16-byte chunk c of a
                // box row at (c ^ (row & 7)) (the 128-byte swizzle), conflict-free like the chain
                mbar_wait(zfull, 0);
                const uint8_t* zslot = smem + (((local + 1) * nkb) % p.stages) * stage_bytes;  // slot after the tile
                for (int c0 = 0; c0 < bn_pair; c0 += 32) {
                    uint32_t u[32];
                    tmem_ld_32x32b_x32(trow + c0, u);
                    tmem_ld_wait();
                    if (gm < p.M) {
                        const uint8_t* zrow = zslot + (c0 / kBK) * kXStage + row * 128;
#pragma unroll
                        for (int v = 0; v < 4; ++v) {
                            if (c0 + 8 * v < bn_pair && n0 + c0 + 8 * v < p.N) {
                                const int ch = ((c0 % kBK) / 8 + v) ^ (row & 7);
                                float z[8];
                                unpack8<kEl>(*reinterpret_cast<const uint4*>(zrow + (ch << 4)), z);
#pragma unroll
                                for (int e = 0; e < 8; ++e)
                                    acc = fmaf(__uint_as_float(u[8 * v + e]), z[e], acc);
                            }
                        }
                    }
                }
            } else
#ifdef DFX_KO_EPI
            if (bn_pair < 0)
#endif
            for (int c0 = 0; c0 < bn_pair; c0 += 32) {
                uint32_t u[32];
                tmem_ld_32x32b_x32(trow + c0, u);
                tmem_ld_wait();
                if (gm < p.M) {
                    const uint16_t* zr = static_cast<const uint16_t*>(p.Z) + gm * p.ldz + n0 + c0;
#pragma unroll
                    for (int v = 0; v < 4; ++v) {
                        if (c0 + 8 * v < bn_pair && n0 + c0 + 8 * v < p.N) {
                            float z[8];
                            unpack8<kEl>(*reinterpret_cast<const uint4*>(zr + 8 * v), z);
#pragma unroll
                            for (int e = 0; e < 8; ++e)
                                acc = fmaf(__uint_as_float(u[8 * v + e]), z[e], acc);
                        }
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if (leader) mbar_arrive(&tmem_empty[slot]);
                else mbar_arrive_remote(mapa_shared(smem_u32(&tmem_empty[slot]), 0), 1);
            }
            if (gm < p.M) p.out[(int64_t(ks) * p.n_split + (n0 / bn_pair)) * p.M + gm] = acc;
            if (p.fin_count && m0 < p.M && last_arrival(p.fin_count + m0 / kBM, p.fin_total, tmem_slot + 1) && gm < p.M)
                finish_row(p.fin, gm);
        }
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync();
#ifdef DFX_KO_TMEM
    if (false) {
#else
    if (warp == kWarpMma) {
#endif
        tc_fence_after();
        switch (tmem_cols) {
            case 32: tmem_dealloc_pair<32>(tmem_base); break;
            case 64: tmem_dealloc_pair<64>(tmem_base); break;
            case 128: tmem_dealloc_pair<128>(tmem_base); break;
            case 256: tmem_dealloc_pair<256>(tmem_base); break;
            default: tmem_dealloc_pair<512>(tmem_base); break;
        }
    }
}

// V = B [G_hi | G_lo] with ba_sq = rowdot(V, B), G-stationary on CTA pairs.
//
// G is small (r x r) and every row tile of B multiplies the same G, so each CTA pair keeps
// its N slice of [G_hi | G_lo] resident in shared memory (loaded once: this CTA's half_n = bn/2
// G rows x 2 r_pad K, 2 * kx swizzle atoms) and streams only B: per 256-row pair tile, kx atoms
// of the CTA's own 128 B rows, each consumed by two UMMA groups (against the G_hi atom and the
// G_lo atom of the same K range: B G_hi + B G_lo = B (G_hi + G_lo)).  Pair p owns N slice
// p % n_split and walks the row tiles p / n_split, + pairs per slice, ...; the accumulator is
// double-buffered in TMEM so a tile's epilogue (rowdot with B from L2, the fused finisher)
// overlaps the next tile's UMMAs.  Operand traffic per pair tile: 2 x 16 KiB x kx of B, instead
// of re-streaming the G slice (96 rows x 2 r_pad) with every tile as the generic V kernel does.
constexpr int kGstatBars = 16;   // G-slice barrier groups (K atoms share one beyond 16)

template <int kEl>
__global__ void __launch_bounds__(kThreads, 1)
    tc_pair_gstat(const __grid_constant__ CUtensorMap tmb, const __grid_constant__ CUtensorMap tmg,
                  const TcParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    const int half_n = p.bn / 2;
    const int kx = p.ka;                                  // K atoms of B (r_pad / 64)
    const int g_atom = half_n * kBK * 2;                  // one G atom of this CTA's rows
    uint8_t* sg = smem;                                   // [2 kx] G atoms (hi 0..kx-1, lo kx..)
    uint8_t* sb = smem + 2 * kx * g_atom;                 // [stages] B atoms
    uint64_t* full = reinterpret_cast<uint64_t*>(sb + p.stages * kXStage);
    uint64_t* empty = full + p.stages;
    uint64_t* tmem_full = empty + p.stages;     // [2]
    uint64_t* tmem_empty = tmem_full + 2;       // [2]
    uint64_t* gfull = tmem_empty + 2;           // [ngb] G slice atoms landed
    const int gsz = (kx + kGstatBars - 1) / kGstatBars;    // K atoms per G barrier
    const int ngb = (kx + gsz - 1) / gsz;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(gfull + ngb);

    const int warp = warp_id(), lane = lane_id();
    const uint32_t rank = cluster_ctarank();
    const bool leader = rank == 0;
    const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
    const int nsl = p.n_split;
    const int slice = pair % nsl;
    const int pps = (npairs - slice + nsl - 1) / nsl;     // pairs serving this slice
    const int first = pair / nsl;
    const int64_t n0 = int64_t(slice) * p.bn;             // the slice's first G row / V column
    const uint32_t slot_cols = static_cast<uint32_t>((p.bn + 31) / 32 * 32);

    if (threadIdx.x == 0) {
        VTR(0);
        tma_prefetch_desc(&tmb);
        tma_prefetch_desc(&tmg);
        for (int s = 0; s < p.stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tmem_full[a], 1);
            mbar_init(&tmem_empty[a], 8);
        }
        for (int g = 0; g < ngb; ++g) mbar_init(&gfull[g], 1);
        fence_mbar_init();
    }
    if (warp == kWarpMma) tmem_alloc_pair<512>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    if (threadIdx.x == 0) VTR(1);

    if (warp == kWarpProducer) {
        if (lane == 0) {
            const uint64_t pol = policy_evict_last();
            // The resident G slice (this CTA's half_n rows; hi atoms 0..kx-1, lo atoms kx..):
            // atom a of G_hi and G_lo ahead of the first tile's B atom a, each group of atoms
            // on its own barrier, so the first UMMAs start when their operands land instead
            // of after the whole slice.
            int s = 0;
            uint32_t ph = 0;
            int g_next = 0;                       // next G barrier group to issue
            auto issue_g = [&](int upto) {        // G atoms of the groups covering K atoms < upto
                for (; g_next < ngb && g_next * gsz < upto; ++g_next) {
                    const int a0 = g_next * gsz, a1 = a0 + gsz < kx ? a0 + gsz : kx;
                    if (leader) mbar_arrive_expect_tx(&gfull[g_next], 2u * 2u * (a1 - a0) * g_atom);
                    const uint32_t gbar = mapa_shared(smem_u32(&gfull[g_next]), 0);
                    for (int a = a0; a < a1; ++a)
                        for (int hl = 0; hl < 2; ++hl)
                            tma_load_2d_pair(&tmg, gbar, sg + (hl * kx + a) * g_atom, (hl * kx + a) * kBK,
                                             static_cast<int32_t>(n0 + int64_t(rank) * half_n), pol);
                }
            };
            bool first_tile = true;
            for (int t = first; t < p.tiles; t += pps) {
                const int64_t m0 = int64_t(t) * (2 * kBM) + int64_t(rank) * kBM;
                for (int a = 0; a < kx; ++a) {
                    if (first_tile) issue_g(a + 1);
                    if (first_tile && a == 0) VTR(2);
                    mbar_wait(&empty[s], ph ^ 1);
                    if (leader) mbar_arrive_expect_tx(&full[s], 2 * kXStage);
                    tma_load_2d_pair(&tmb, mapa_shared(smem_u32(&full[s]), 0), sb + s * kXStage,
                                     a * kBK, static_cast<int32_t>(m0), pol);
                    if (++s == p.stages) { s = 0; ph ^= 1; }
                }
                first_tile = false;               // (a pair with no tile loads no G)
            }
        }
    } else if (warp == kWarpMma) {
        if (leader && lane == 0) {
            const uint32_t idesc = umma_idesc_f16(ab_fmt(kEl), 2 * kBM, static_cast<uint32_t>(p.bn));
            int s = 0;
            uint32_t ph = 0;
            int local = 0;
            for (int t = first; t < p.tiles; t += pps, ++local) {
                const int slot = local & 1;
                const uint32_t tacc = tmem_base + static_cast<uint32_t>(slot) * slot_cols;
                mbar_wait(&tmem_empty[slot], ((local >> 1) & 1) ^ 1);
                tc_fence_after();
                for (int a = 0; a < kx; ++a) {
                    if (local == 0) {
                        mbar_wait(&gfull[a / gsz], 0);   // G atoms of this K range (first tile)
                        if (a == 0) VTR(3);
                    }
                    mbar_wait(&full[s], ph);
                    if (local == 0 && a == 0) VTR(4);
                    tc_fence_after();
                    const uint32_t bx = smem_u32(sb + s * kXStage);
                    for (int hl = 0; hl < 2; ++hl) {
                        const uint32_t gy = smem_u32(sg + (hl * kx + a) * g_atom);
#pragma unroll
                        for (int k = 0; k < kBK / 16; ++k)
                            umma_f16_pair(tacc, umma_desc_k_sw128(bx + k * 32), umma_desc_k_sw128(gy + k * 32),
                                          idesc, (a > 0 || hl > 0 || k > 0) ? 1u : 0u);
                    }
                    umma_commit_pair_mc(&empty[s], 0x3);
                    if (++s == p.stages) { s = 0; ph ^= 1; }
                }
                umma_commit_pair_mc(&tmem_full[slot], 0x3);
                VTR(5);
            }
        }
    } else if (warp < 4) {
        const int q = warp;
        const int row = q * 32 + lane;
        int local = 0;
        for (int t = first; t < p.tiles; t += pps, ++local) {
            const int64_t m0 = int64_t(t) * (2 * kBM) + int64_t(rank) * kBM;
            const int64_t gm = m0 + row;
            const int slot = local & 1;
            // this row's B slice (<= 256 values) into registers while the tile's UMMAs run, so
            // the epilogue is TMEM loads + FMAs only (an L2 round trip per 32 columns otherwise
            // made the epilogue, not the MMA, the per-tile critical path)
            uint4 zb[32];
            {
                const uint16_t* zr = static_cast<const uint16_t*>(p.Z) + gm * p.ldz + n0;
#pragma unroll
                for (int v = 0; v < 32; ++v)
                    zb[v] = (gm < p.M && 8 * v < p.bn && n0 + 8 * v < p.N)
                                ? *reinterpret_cast<const uint4*>(zr + 8 * v) : make_uint4(0, 0, 0, 0);
            }
#ifdef DFX_TRACE
            if (threadIdx.x == 0) { uint32_t x = 0; for (int v = 0; v < 32; ++v) x ^= zb[v].x; if (x == 0x9e3779b9u) g_vtrace[0][0] = 0; VTR(6); }
#endif
            mbar_wait(&tmem_full[slot], (local >> 1) & 1);
            if (threadIdx.x == 0) VTR(7);
            tc_fence_after();
            const uint32_t trow = tmem_base + static_cast<uint32_t>(slot) * slot_cols +
                                  (static_cast<uint32_t>(q * 32) << 16);
            float acc = 0.0f;
#pragma unroll
            for (int c0 = 0; c0 < 256; c0 += 32) {
                if (c0 >= p.bn) break;
                uint32_t u[32];
                tmem_ld_32x32b_x32(trow + c0, u);
                tmem_ld_wait();
#pragma unroll
                for (int v = 0; v < 4; ++v) {
                    if (c0 + 8 * v < p.bn && n0 + c0 + 8 * v < p.N) {
                        float z[8];
                        unpack8<kEl>(zb[c0 / 8 + v], z);
#pragma unroll
                        for (int e = 0; e < 8; ++e)
                            acc = fmaf(__uint_as_float(u[8 * v + e]), z[e], acc);
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if (leader) mbar_arrive(&tmem_empty[slot]);
                else mbar_arrive_remote(mapa_shared(smem_u32(&tmem_empty[slot]), 0), 1);
            }
            if (p.out_scale) acc = __fmul_rn(acc, *p.out_scale);   // exact power of two
            if (gm < p.M) p.out[int64_t(slice) * p.M + gm] = acc;
            if (threadIdx.x == 0) VTR(8);
            if (p.fin_count && m0 < p.M && last_arrival(p.fin_count + m0 / kBM, p.fin_total, tmem_slot + 1) && gm < p.M)
                finish_row(p.fin, gm);
            if (threadIdx.x == 0) VTR(9);
        }
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    if (warp == kWarpMma) {
        tc_fence_after();
        tmem_dealloc_pair<512>(tmem_base);
    }
}

// Reduce gram partial tiles in fixed split order and emit [G_hi | G_lo] (bf16) with
// G mirrored from the upper triangle, so the hi/lo operand is exactly symmetric.
__global__ void __launch_bounds__(256) gram_reduce(const float* __restrict__ part, int k_split,
                                                   int nt, int64_t r, int64_t r_pad,
                                                   __nv_bfloat16* __restrict__ g2,
                                                   float* __restrict__ gout) {
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
    if (gout && j < r) gout[i * r + j] = gsum;       // d_in-split partial: fp32 Gram out
    if (!g2) return;
    const __nv_bfloat16 hi = __float2bfloat16_rn(gsum);
    const __nv_bfloat16 lo = __float2bfloat16_rn(__fsub_rn(gsum, __bfloat162float(hi)));
    g2[i * 2 * r_pad + j] = hi;
    g2[i * 2 * r_pad + r_pad + j] = lo;
}

// fp32 Gram -> [G_hi | G_lo] (K padded with 0) as the V GEMM's operand.
// bf16: hi = bf16(G), lo = bf16(G - hi), unscaled (bf16 has fp32's range).
// fp16: fp16's range (|x| <= 65504, normal >= 2^-14) cannot hold a Gram of arbitrary scale,
//   so G is scaled by 2^e first, e = 14 - ilogb(max diag G) (|G_lq| <= max diag, G is PSD), so
//   the largest entry lands in [2^14, 2^15); the V epilogue multiplies each row's sum by 2^-e
//   (exact).  Every block finds the max diagonal itself (r <= 2048 reads), so no extra pass.
//   Non-finite diagonals (NaN / inf in A) leave e = 0 and propagate.
template <typename T>
__global__ void __launch_bounds__(256) gram_split(const float* __restrict__ g, int64_t r,
                                                  int64_t r_pad, T* __restrict__ g2,
                                                  float* __restrict__ inv_scale) {
    constexpr bool kHalf = std::is_same<T, __half>::value;
    float scale = 1.0f;
    if (kHalf) {
        __shared__ float red[8];
        float mx = 0.0f;
        bool bad = false;
        for (int64_t i = threadIdx.x; i < r; i += blockDim.x) {
            const float d = g[i * r + i];
            bad |= !isfinite(d);
            mx = fmaxf(mx, fabsf(d));
        }
        bad = __syncthreads_or(bad);
        for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
        __syncthreads();
        mx = red[0];
        for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) mx = fmaxf(mx, red[w]);
        int e = 0;
        if (!bad && mx > 0.0f) e = max(-120, min(120, 14 - ilogbf(mx)));
        scale = ldexpf(1.0f, e);
        if (blockIdx.x == 0 && threadIdx.x == 0) *inv_scale = ldexpf(1.0f, -e);
    }
    const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= r * r_pad) return;
    const int64_t i = idx / r_pad, j = idx % r_pad;
    const float v = j < r ? __fmul_rn(g[i * r + j], scale) : 0.0f;
    const T hi = Elem<T>::from_f(v);
    g2[i * 2 * r_pad + j] = hi;
    g2[i * 2 * r_pad + r_pad + j] = Elem<T>::from_f(__fsub_rn(v, Elem<T>::to_f(hi)));
}

int stages_for(int bn, bool f32 = false) {
    const int stage = (kXStage + bn * kBK * 2) * (f32 ? 2 : 1);
    const int avail = kMaxSmem - 1024 - 256;
    return std::min(8, avail / stage);
}

size_t smem_for(int bn, int stages, bool f32 = false) {
    return size_t(stages) * (kXStage + bn * kBK * 2) * (f32 ? 2 : 1) + 1024 + 256;
}

// tpc_pairs: launch as clusters of 2 so the kernel occupies whole TPCs (used for the
// side-stream GEMMs that run beside the 2-SM W.A^T kernel, whose CTA pairs each need
// a whole TPC; a lone side CTA per TPC would strand its sibling SM).
cudaError_t launch_tc(int mode, const CUtensorMap& tx, const CUtensorMap& ty, TcParams p,
                      dim3 grid, cudaStream_t st, const char* name, bool tpc_pairs = false,
                      int el = kBF16) {
    const bool f32 = el == kF32;
    const size_t smem = smem_for(p.bn, p.stages, f32);
    cudaError_t e;
    auto kern = el == kF32   ? (mode == kTcRowdot ? tc_rowdot<kTcRowdot, kF32> : tc_rowdot<kTcStore, kF32>)
                : el == kF16 ? (mode == kTcRowdot ? tc_rowdot<kTcRowdot, kF16> : tc_rowdot<kTcStore, kF16>)
                             : (mode == kTcRowdot ? tc_rowdot<kTcRowdot, kBF16> : tc_rowdot<kTcStore, kBF16>);
    if ((e = ensure_max_dyn_smem(reinterpret_cast<const void*>(kern), kMaxSmem)) != cudaSuccess) return e;
    if (tpc_pairs) grid.x = (grid.x + 1) / 2 * 2;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(f32 ? kThreads + 32 * (kSplitWarps - 2) : kThreads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = tpc_pairs ? 2 : 1;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    prof_begin(name, st);
    e = cudaLaunchKernelEx(&cfg, kern, tx, ty, p);
    prof_end(st);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

size_t smem_for_pair(int bn, int stages, int nh = 1, int ka = 1) {
    return size_t(stages) * ka * (kXStage + nh * (bn / 2) * kBK * 2) + 1024 + 256;
}

int stages_for_pair(int bn, int nh = 1, int ka = 1) {
    const int stage = ka * (kXStage + nh * (bn / 2) * kBK * 2);
    return std::min(8, (kMaxSmem - 1024 - 256) / stage);
}

int env_int(const char* name, int dflt) {
    const char* e = std::getenv(name);
    return e ? std::atoi(e) : dflt;
}

// K atoms per ring stage of the pair kernel.  A stage's UMMAs are released by one
// tcgen05.commit, and a commit costs the tensor pipe ~400 cycles (tools/mma_ts_micro.cu:
// a 2-SM N=192 UMMA takes 196 cycles at one commit per 4 UMMAs, 124 per 8, 96 at 32), so
// two 64-wide K blocks per stage (8 UMMAs per commit) when N per UMMA is one r half;
// DFX_PAIR_KA overrides for measurements.
int pair_atoms(int nh, int64_t kb_per_split, int64_t total_kb) {
    static const int env = env_int("DFX_PAIR_KA", 0);
    int ka = env > 0 ? env : (nh == 1 ? 2 : 1);
    if (ka > 1 && (kb_per_split % ka != 0 || total_kb % ka != 0)) ka = 1;
    return ka;
}

cudaError_t launch_tc_pair(const CUtensorMap& tx, const CUtensorMap& ty, const CUtensorMap& tz,
                           TcParams p, int pairs, int ks, cudaStream_t st, const char* name, int el) {
    cudaError_t e;
    auto kern = el == kF16 ? tc_pair_rowdot<kF16> : tc_pair_rowdot<kBF16>;
    if ((e = ensure_max_dyn_smem(reinterpret_cast<const void*>(kern), kMaxSmem)) != cudaSuccess)
        return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * pairs, ks, 1);
    cfg.blockDim = dim3(kThreads, 1, 1);
    cfg.dynamicSmemBytes = smem_for_pair(p.bn, p.stages, p.nh > 0 ? p.nh : 1, p.ka > 0 ? p.ka : 1);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    prof_begin(name, st);
#ifdef DFX_TRACE
    const char* trace_file = std::getenv("DFX_TRACE");
    if (trace_file) {
        void* tp = nullptr;
        cudaGetSymbolAddress(&tp, g_trace);
        cudaMemsetAsync(tp, 0, sizeof(g_trace), st);
    }
#endif
    e = cudaLaunchKernelEx(&cfg, kern, tx, ty, tz, p);
    prof_end(st);
    if (e != cudaSuccess) return e;
#ifdef DFX_TRACE
    if (trace_file) {
        static unsigned long long host[kTrCta][kTrEv][kTrN];
        cudaStreamSynchronize(st);
        cudaMemcpyFromSymbol(host, g_trace, sizeof(host));
        if (FILE* f = std::fopen(trace_file, "ab")) {
            const int hdr[8] = {2 * pairs, p.stages, p.kb_per_split, p.nh, p.bn, p.ka, p.tiles, ks};
            std::fwrite(hdr, sizeof(hdr), 1, f);
            std::fwrite(host, sizeof(host), 1, f);
            std::fclose(f);
        }
    }
#endif
    return cudaGetLastError();
}

// (n_split, k_split) for a rowdot GEMM with m_tiles 128-row tiles on a budget of `ctas`
// persistent CTAs.  Cost model (measured with tools/mma_micro.cu): one tcgen05.mma
// K=16 step costs ~120 cycles for any N <= 192 and ~128 at N = 256, so a tile costs
// kb * 4 * max(120, N/2) cycles and the kernel costs rounds * tile cost (+ a per-tile
// epilogue/prologue term).  N splits keep a row's base_sq chain in whole chunks; K splits
// only on ChunkPlan boundaries (max_ks).
struct Split { int ns, ks, bn; };

Split choose_split(int64_t m_tiles, int64_t r, int64_t kb_total, int max_ks, int ctas,
                   int bn_align = 16) {
    Split best{1, 1, 0};
    double best_cost = 1e300;
    const int ns_min = static_cast<int>((r + 255) / 256);
    for (int ns = ns_min; ns <= 8; ++ns) {
        const int bn = static_cast<int>(((r + ns - 1) / ns + bn_align - 1) / bn_align * bn_align);
        if (bn > 256 || bn < 16) continue;
        for (int ks = 1; ks <= max_ks && ks <= 8; ks *= 2) {
            if (ks > 1 && kb_total / ks < 4) break;
            const int64_t work = m_tiles * ns * ks;                 // tile-splits
            const int64_t rounds = (work + ctas - 1) / ctas;
            const double kb = double((kb_total + ks - 1) / ks);
            const double per_tile = kb * 4.0 * std::max(120.0, 0.5 * bn) + 2500.0;
            const double cost = double(rounds) * per_tile * (1.0 + 0.02 * (ns - ns_min));
            if (cost < best_cost * (1.0 - 1e-9)) {
                best_cost = cost;
                best = {ns, ks, bn};
            }
        }
    }
    if (best.bn == 0)
        best = {ns_min, 1,
                static_cast<int>(((r + ns_min - 1) / ns_min + bn_align - 1) / bn_align * bn_align)};
    return best;
}

}  // namespace

// DFX_NORM_PAIR=0 selects the 1-SM kernel for the W.A^T GEMM (A/B measurements; the
// two are within ~1% at module level on C2, the 2-SM one is the faster GEMM).
bool pair_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("DFX_NORM_PAIR");
        return !(e && e[0] == '0');
    }();
    return on;
}

// DFX_NORM_FUSE=0: a separate finish launch (A/B measurements).
bool norm_fuse_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("DFX_NORM_FUSE");
        return !(e && e[0] == '0');
    }();
    return on;
}

bool norm_tc_supported(int dt, int64_t d_out, int64_t d_in, int64_t r) {
    return (dt == kBF16 || dt == kF16) && d_in >= 64 && d_in % 8 == 0 && r % 8 == 0 && r >= 16 && r <= 2048 &&
           d_out >= 1 && d_in < (int64_t(1) << 31) && d_out < (int64_t(1) << 31);
}

cudaError_t launch_norm_finish_tc(const NormArgs& a, Workspace* ws, cudaStream_t st,
                                  int* launches);

// ------------------------------------------------------------------- planning
// Cycle model of one persistent GEMM launch (tools/mma_micro.cu: a K=16 UMMA step costs
// ~120 cycles for N <= 192, ~N/2 above; + a per-tile prologue/epilogue term).
double gemm_cycles(int64_t work, int ctas, int64_t kb, int bn) {
    if (work <= 0) return 0.0;
    const int64_t rounds = (work + ctas - 1) / ctas;
    return double(rounds) * (double(kb) * 4.0 * std::max(120.0, 0.5 * bn) + 2500.0);
}

// The norm's three GEMMs: U = W A^T (+ base_sq chain), G = A A^T (+ fixed-order split
// reduction to [G_hi | G_lo]) and V = B [G_hi | G_lo].  Only U reads W; G and V depend on
// the adapter alone.  Strategies (chosen per shape by the cycle model):
//   kSideAll   G, reduce, V on a side stream on `side` SMs, concurrent with U
//   kSideGram  G, reduce on the side SMs concurrent with U; V after U on all SMs
//   kSerial    G (all SMs), reduce, U (all SMs), V (all SMs)
enum Strategy { kSideAll = 0, kSideGram = 1, kSerial = 2 };

struct UPlan {
    bool pair;
    int nh;         // pair kernel: UMMAs per K step (2 = full r per CTA pair, W ingested once)
    Split sp;
    int ks, kbps;
    int64_t work;   // CTAs per K split
    int ctas;       // CTAs launched
    double cycles;
};

struct NormPlan {
    Strategy strategy;
    int side;       // side-stream SM budget (kSideAll / kSideGram)
    UPlan u;
    int g_ks, g_kbps, g_ctas;
    Split sb;
    int b_ctas;
    bool v_gstat;   // V on tc_pair_gstat (b_ctas = 2 x pairs, sb.ns = N slices, sb.bn = N slice)
    double cycles;
};

// G-stationary V (tc_pair_gstat): the N slice (bn, n slices) whose resident [G_hi | G_lo] rows
// (bn / 2 per CTA x 2 r_pad) leave at least 3 B stages; {0, 0} when none fits.
struct GstatShape { int bn, nsl, stages; };

size_t smem_for_gstat(int bn, int64_t r_pad, int stages) {
    return size_t(2 * (r_pad / kBK)) * (bn / 2) * kBK * 2 + size_t(stages) * kXStage + 1024 + 512;
}

GstatShape gstat_shape(int64_t r) {
    const int64_t r_pad = (r + kBK - 1) / kBK * kBK;
    for (int nsl = 1; nsl <= 64; ++nsl) {
        const int bn = static_cast<int>(((r + nsl - 1) / nsl + 31) / 32 * 32);
        if (bn > 256) continue;
        for (int st = 6; st >= 3; --st)
            if (smem_for_gstat(bn, r_pad, st) <= size_t(kMaxSmem)) return {bn, static_cast<int>((r + bn - 1) / bn), st};
    }
    return {0, 0, 0};
}

// DFX_V_GSTAT: -1 (default) the cycle model picks the V kernel, 0 generic tc_rowdot, 1 G-stationary.
int v_gstat_mode() {
    static const int m = env_int("DFX_V_GSTAT", -1);
    return m;
}

cudaError_t launch_gstat(const CUtensorMap& tb, const CUtensorMap& tg, const TcParams& p, int pairs,
                         cudaStream_t st, int el) {
    cudaError_t e;
    auto kern = el == kF16 ? tc_pair_gstat<kF16> : tc_pair_gstat<kBF16>;
    if ((e = ensure_max_dyn_smem(reinterpret_cast<const void*>(kern), kMaxSmem)) != cudaSuccess)
        return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * pairs, 1, 1);
    cfg.blockDim = dim3(kThreads, 1, 1);
    cfg.dynamicSmemBytes = smem_for_gstat(p.bn, int64_t(p.ka) * kBK, p.stages);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    prof_begin("ba_rowdot_tc", st);
#ifdef DFX_TRACE
    const char* trace_file = std::getenv("DFX_VTRACE");
    if (trace_file) {
        void* tp = nullptr;
        cudaGetSymbolAddress(&tp, g_vtrace);
        cudaMemsetAsync(tp, 0, sizeof(g_vtrace), st);
    }
#endif
    e = cudaLaunchKernelEx(&cfg, kern, tb, tg, p);
    prof_end(st);
    if (e != cudaSuccess) return e;
#ifdef DFX_TRACE
    if (trace_file) {
        static unsigned long long host[kTrCta][kVtrEv];
        cudaStreamSynchronize(st);
        cudaMemcpyFromSymbol(host, g_vtrace, sizeof(host));
        if (FILE* f = std::fopen(trace_file, "ab")) {
            const int hdr[8] = {2 * pairs, p.stages, p.ka, p.bn, p.n_split, p.tiles, 0, 0};
            std::fwrite(hdr, sizeof(hdr), 1, f);
            std::fwrite(host, sizeof(host), 1, f);
            std::fclose(f);
        }
    }
#endif
    return cudaGetLastError();
}


UPlan plan_u(int64_t d_out, int64_t r, int64_t kb_in, int64_t chunk_blocks, int64_t n_chunks,
             int budget) {
    UPlan u{};
    const int64_t m_tiles = (d_out + kBM - 1) / kBM;
    const int64_t pm_tiles = (d_out + 2 * kBM - 1) / (2 * kBM);
    u.pair = m_tiles >= 2 && pair_enabled() && budget >= 2;
    const int max_ks = static_cast<int>(std::min<int64_t>(n_chunks, 8));
    u.sp = u.pair ? choose_split(pm_tiles, r, kb_in, max_ks, budget / 2, 32)
                  : choose_split(m_tiles, r, kb_in, max_ks, budget);
    const int64_t chunks_per_split = (n_chunks + u.sp.ks - 1) / u.sp.ks;
    u.kbps = static_cast<int>(chunks_per_split * chunk_blocks);
    u.ks = static_cast<int>((kb_in + u.kbps - 1) / u.kbps);
    u.work = (u.pair ? 2 * pm_tiles : m_tiles) * u.sp.ns;
    u.ctas = static_cast<int>(std::min<int64_t>(u.work * u.ks, budget));
    u.cycles = u.pair ? gemm_cycles(pm_tiles * u.sp.ns * u.ks, std::max(1, u.ctas / 2), u.kbps, u.sp.bn)
                      : gemm_cycles(u.work * u.ks, std::max(1, u.ctas), u.kbps, u.sp.bn);
    u.nh = 1;
    // Full r per CTA pair (two UMMAs of N = r/2 per K step): W is ingested by one pair
    // instead of one per N split, at twice the MMA work per SM.  On a full GPU the N-split
    // tiling is faster; under an SM budget (dfx_ctx_set_sm_budget, compose kernels running
    // beside the norm) the one-pass tiling wins once the N splits would need a second round.
    const int64_t bnh = ((r + 1) / 2 + 31) / 32 * 32;
    if (u.pair && r > 256 && 2 * bnh <= 512 && u.sp.ns > 1) {
        const int pairs = std::max(1, budget / 2);
        const int64_t kbps1 = int64_t(chunks_per_split) * chunk_blocks;
        const double c1 = gemm_cycles(pm_tiles * u.ks, pairs, kbps1, static_cast<int>(bnh)) +
                          double((pm_tiles * u.ks + pairs - 1) / pairs) * double(kbps1) * 4.0 *
                              std::max(120.0, 0.5 * double(bnh));
        // Decide with the ingest-aware model (a K block costs max(129 cycles per UMMA, TMA
        // ingest bytes / 42 B per cycle per SM), tools/mma_micro.cu + scripts/exp_sweep.sh):
        // W once per row pair vs once per N split.  Measured: C3 norm 219 -> 176 us with the
        // full-r tiling, C2 / C4 r=512 faster with N splits (enough row pairs to fill the SMs).
        const int64_t pt1 = pm_tiles * u.sp.ns * u.ks, pt2 = pm_tiles * u.ks;
        const double kb1 = std::max(4.0 * 129.0, (16384.0 + u.sp.bn / 2 * 128.0) / 42.0);
        const double kb2 = std::max(8.0 * 129.0, (16384.0 + double(bnh) * 128.0) / 42.0);
        const double i1 = double((pt1 + pairs - 1) / pairs) * kb1;
        const double i2 = double((pt2 + pairs - 1) / pairs) * kb2;
        if (i2 < i1 || c1 <= u.cycles) {
            u.nh = 2;
            u.sp = {1, u.sp.ks, static_cast<int>(bnh)};
            u.work = 2 * pm_tiles;
            u.ctas = static_cast<int>(std::min<int64_t>(u.work * u.ks, budget));
            u.cycles = c1;
        }
    }
    // DFX_U_KS / DFX_U_NH: measurement overrides of the K-split count and the UMMAs per K step
    static const int force_ks = env_int("DFX_U_KS", 0), force_nh = env_int("DFX_U_NH", 0);
    if (u.pair && (force_ks > 0 || force_nh > 0)) {
        const int nh = force_nh > 0 ? force_nh : u.nh;
        int ks = force_ks > 0 ? force_ks : u.ks;
        ks = static_cast<int>(std::min<int64_t>(ks, n_chunks));
        const int64_t chunks_per_split = (n_chunks + ks - 1) / ks;
        u.kbps = static_cast<int>(chunks_per_split * chunk_blocks);
        u.ks = static_cast<int>((kb_in + u.kbps - 1) / u.kbps);
        if (nh == 2 && r > 256 && 2 * bnh <= 512) {
            u.nh = 2;
            u.sp = {1, u.ks, static_cast<int>(bnh)};
            u.work = 2 * pm_tiles;
        } else if (nh == 1) {
            const int ns = static_cast<int>((r + 255) / 256) < 2 && r > 128 ? 2 : static_cast<int>((r + 255) / 256);
            const int bn = static_cast<int>(((r + ns - 1) / ns + 31) / 32 * 32);
            u.nh = 1;
            u.sp = {ns, u.ks, bn};
            u.work = 2 * pm_tiles * ns;
        }
        u.ctas = static_cast<int>(std::min<int64_t>(u.work * u.ks, budget));
    }
    return u;
}

NormPlan plan_norm(int64_t d_out, int64_t d_in, int64_t r, int64_t chunk_size, int sms,
                   bool need_v, bool force_serial = false) {
    const int64_t r_pad = (r + kBK - 1) / kBK * kBK;
    const int64_t m_tiles = (d_out + kBM - 1) / kBM;
    const int64_t kb_in = (d_in + kBK - 1) / kBK;
    const int64_t chunk_blocks = chunk_size / kBK;
    const int64_t n_chunks = (d_in + chunk_size - 1) / chunk_size;
    const int nt = static_cast<int>((r + kBM - 1) / kBM);
    const int gtiles = nt * (nt + 1) / 2;
    const int64_t pm_tiles_n = (d_out + 2 * kBM - 1) / (2 * kBM);
    const double kReduce = 12000.0;  // fixed-order split reduction kernel

    auto gram = [&](int budget, int& ks, int& kbps, int& ctas) {
        ks = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(budget / gtiles, kb_in / 8)));
        kbps = static_cast<int>((kb_in + ks - 1) / ks);
        ks = static_cast<int>((kb_in + kbps - 1) / kbps);
        ctas = std::min(gtiles, std::max(1, budget / ks)) * ks;
        return gemm_cycles(int64_t(gtiles) * ks, ctas, kbps, kBM) + kReduce;
    };
    // V cycle model with an operand-ingest term (~42 B per cycle per SM, DESIGN 5.1): the generic
    // kernel re-streams its G slice with every 128-row tile, the G-stationary pair kernel streams
    // only B (twice per pair tile: two CTAs) after loading its G slice once.
    auto vgemm = [&](int budget, Split& sb, int& ctas, bool& gs) {
        gs = false;
        if (!need_v) { sb = {1, 1, 16}; ctas = 0; return 0.0; }
        const int64_t kb = 2 * r_pad / kBK;
        sb = choose_split(m_tiles, r, kb, 1, budget);
        ctas = static_cast<int>(std::min<int64_t>(m_tiles * sb.ns, budget));
        // calibrated on the B200 (round 2): the model's per-tile figures x 1.4-1.5 ~ the measured
        // steady-state tile times (generic ~19.5k cycles, G-stationary ~13-14.5k per pair tile
        // at r = 384), plus the G-stationary kernel's G-slice prologue; at C2 on all SMs the
        // G-stationary kernel measures 15.6 vs 16.7 us (ncu) and is the one chosen
        const double tile_g = 1.4 * (std::max(double(kb) * 4.0 * std::max(120.0, 0.5 * sb.bn),
                                              double(kb) * (16384.0 + sb.bn * 128.0) / 42.0) + 2500.0);
        const double generic = double((m_tiles * sb.ns + ctas - 1) / ctas) * tile_g;
        const GstatShape gsh = gstat_shape(r);
        const int mode = v_gstat_mode();
        if (mode == 0 || gsh.bn == 0 || budget < 2 * gsh.nsl) return generic;
        const int pairs = std::min<int>(static_cast<int>(pm_tiles_n * gsh.nsl), budget / 2) / gsh.nsl * gsh.nsl;
        const int64_t kx = r_pad / kBK;
        const double tile_s = 1.5 * (std::max(double(kx) * 8.0 * 130.0, double(kx) * 16384.0 / 42.0) + 2500.0);
        const double gstat = double((pm_tiles_n + pairs / gsh.nsl - 1) / (pairs / gsh.nsl)) * tile_s +
                             1000.0 * double(kx);
        if (mode == 1 || gstat < generic) {
            gs = true;
            sb = {gsh.nsl, 1, gsh.bn};
            ctas = 2 * pairs;
            return gstat;
        }
        return generic;
    };

    // DFX_NORM_STRATEGY (0 side-all, 1 side-gram, 2 serial) / DFX_NORM_SIDE (side-stream SMs):
    // measurement overrides of the cycle model's choice
    static const int force_st = env_int("DFX_NORM_STRATEGY", -1);
    static const int force_side = env_int("DFX_NORM_SIDE", 0);
    NormPlan best{};
    best.cycles = 1e300;
    // serial on all SMs
    {
        NormPlan p{};
        p.strategy = kSerial;
        p.side = 0;
        p.u = plan_u(d_out, r, kb_in, chunk_blocks, n_chunks, sms);
        const double g = gram(sms, p.g_ks, p.g_kbps, p.g_ctas);
        const double v = vgemm(sms, p.sb, p.b_ctas, p.v_gstat);
        p.cycles = g + p.u.cycles + v;
        best = p;
        if (force_st == kSerial || force_serial) return best;
    }
    for (int side : {8, 12, 20, 28, 36, 52, 74}) {
        if (side >= sms) break;
        if (force_side > 0 && side != force_side) continue;
        UPlan u = plan_u(d_out, r, kb_in, chunk_blocks, n_chunks, sms - side);
        // leave exactly the SMs U does not use to the side stream
        const int side_eff = std::max(side, sms - u.ctas) & ~1;
        int gks, gkbps, gctas;
        const double g = gram(side_eff, gks, gkbps, gctas);
        for (Strategy st : {kSideAll, kSideGram}) {
            NormPlan p{};
            p.strategy = st;
            p.side = side_eff;
            p.u = u;
            p.g_ks = gks; p.g_kbps = gkbps; p.g_ctas = gctas;
            if (st == kSideAll) {
                // DFX_V_WIDE=1: V on the side stream but with an all-SM grid (its first CTAs run
                // on the side SMs, the rest as U's CTAs retire) — measurement switch
                static const bool wide = env_int("DFX_V_WIDE", 0) != 0;
                const double v = vgemm(wide ? sms : side_eff, p.sb, p.b_ctas, p.v_gstat);
                p.cycles = std::max(u.cycles, g + v);
            } else {
                const double v = vgemm(sms, p.sb, p.b_ctas, p.v_gstat);
                p.cycles = std::max(u.cycles, g) + v;
            }
            if (force_st >= 0 && st != force_st) continue;
            if (p.cycles < best.cycles * 0.999 || (force_st >= 0 && best.strategy == kSerial)) best = p;
        }
    }
    return best;
}

// The planner's decision for (shape, SM budget), for callers sizing what runs beside the norm
// and for the bench's roofline context: SMs the W.A^T kernel occupies, SMs of the side
// stream (Gram / V beside it; 0 when serial), the strategy (0 side-all, 1 side-gram, 2 serial).
void norm_plan_info(int64_t d_out, int64_t d_in, int64_t r, int64_t chunk_size, int sms,
                    int* u_ctas, int* side_ctas, int* strategy) {
    const NormPlan plan = plan_norm(d_out, d_in, r, chunk_size, sms, true);
    const UPlan& u = plan.u;
    const int64_t pm_tiles = (d_out + 2 * kBM - 1) / (2 * kBM);
    const int64_t m_tiles = (d_out + kBM - 1) / kBM;
    int ctas;
    if (u.pair) {
        const int pairs = static_cast<int>(std::min<int64_t>(pm_tiles * u.sp.ns, std::max(1, u.ctas / (2 * u.ks))));
        ctas = 2 * pairs * u.ks;
    } else {
        ctas = static_cast<int>(std::min<int64_t>(m_tiles * u.sp.ns, std::max(1, u.ctas / u.ks))) * u.ks;
    }
    if (u_ctas) *u_ctas = std::min(ctas, sms);
    if (side_ctas) *side_ctas = plan.strategy == kSerial ? 0 : plan.side;
    if (strategy) *strategy = static_cast<int>(plan.strategy);
}

cudaError_t launch_norm_tc(const NormArgs& a, Workspace* ws, cudaStream_t st, int* launches) {
    if (a.mode == kNormFinish) return launch_norm_finish_tc(a, ws, st, launches);
    if (!norm_tc_supported(a.dt, a.d_out, a.d_in, a.r)) return cudaErrorNotSupported;
    cudaError_t err = cudaSuccess;
    const bool partial = a.mode == kNormPartial;
    const int64_t r = a.r, d_out = a.d_out, d_in = a.d_in;
    const int64_t r_pad = (r + kBK - 1) / kBK * kBK;
    const int64_t m_tiles = (d_out + kBM - 1) / kBM;
    const int64_t pm_tiles = (d_out + 2 * kBM - 1) / (2 * kBM);
    const int64_t n_chunks = (d_in + a.chunk_size - 1) / a.chunk_size;
    const int sms = ws_sm_count(ws);

    // split form: the adapter-only call (Gram + V on all of the budget's SMs, one stream) and
    // the W call given ba_sq (W.A^T only) both plan serially
    const bool adapter = a.mode == kNormAdapter;
    const bool given = a.ba_given != nullptr;
    const NormPlan plan = plan_norm(d_out, d_in, r, a.chunk_size, sms, !partial && !given,
                                    adapter || given);
    const UPlan& u = plan.u;
    const bool forked = plan.strategy != kSerial;
    // side kernels occupy whole TPCs beside the 2-SM U pairs
    const bool tpc = forked && u.pair;

    float* cross = static_cast<float*>(
        ws_get(ws, kWsCross, size_t(u.ks) * u.sp.ns * d_out * sizeof(float), &err));
    if (err != cudaSuccess) return err;
    float* base = static_cast<float*>(
        ws_get(ws, kWsBase, size_t(n_chunks) * d_out * sizeof(float), &err));
    if (err != cudaSuccess) return err;
    const int nt = static_cast<int>((r + kBM - 1) / kBM);
    const int gtiles = nt * (nt + 1) / 2;
    float* gpart = static_cast<float*>(
        ws_get(ws, kWsGramPart, size_t(plan.g_ks) * gtiles * kBM * kBM * sizeof(float), &err));
    if (err != cudaSuccess) return err;
    __nv_bfloat16* g2 = static_cast<__nv_bfloat16*>(
        ws_get(ws, kWsGram2, size_t(r) * 2 * r_pad * sizeof(__nv_bfloat16), &err));
    if (err != cudaSuccess) return err;
    float* ba = static_cast<float*>(
        ws_get(ws, kWsBa, size_t(plan.sb.ns) * d_out * sizeof(float), &err));
    if (err != cudaSuccess) return err;
    // fp16 operands: the Gram goes through fp32 and a scaled fp16 hi/lo split (gram_split)
    const int el = a.dt;
    const bool half = el == kF16;
    float* gf32 = nullptr;
    float* inv_scale = nullptr;
    if (half && !partial) {
        gf32 = static_cast<float*>(ws_get(ws, kWsGram, size_t(r) * r * sizeof(float), &err));
        if (err != cudaSuccess) return err;
        inv_scale = static_cast<float*>(ws_get(ws, kWsScale, 256, &err));
        if (err != cudaSuccess) return err;
    }

    // Fused finisher (DFX_NORM_FUSE=0 restores the separate finish launch): the last U / V
    // tile of each 128-row block runs the finisher for its rows; one counter per block.
    const bool fuse = norm_fuse_enabled();
    unsigned* counters = nullptr;
    if (fuse || adapter) {
        counters = static_cast<unsigned*>(
            ws_get_zeroed(ws, adapter ? kWsAdaptCount : kWsGramCount, size_t(m_tiles) * sizeof(unsigned),
                          &err));
        if (err != cudaSuccess) return err;
    }
    FinishArgs f{};
    f.base_part = base; f.base_parts = static_cast<int>(n_chunks);
    if (a.base_cached) { f.base_part = a.base_cached; f.base_parts = 1; }
    f.cross_part = cross; f.cross_parts = u.ks * u.sp.ns;
    if (!partial) { f.ba_part = ba; f.ba_parts = plan.sb.ns; }
    if (given) { f.ba_part = a.ba_given; f.ba_parts = 1; }
    f.d_out = d_out; f.two_s = 2.0 * a.s; f.s2 = a.s * a.s;
    f.base_sq = a.base_sq; f.cross = a.cross; f.ba_sq = a.ba_sq;
    f.round_dt = a.round_dt; f.w_norm = a.w_norm;
    f.m = a.m; f.mag_dt = a.mag_dt; f.g = a.m ? a.g : nullptr;
    if (partial) { f.w_norm = nullptr; f.g = nullptr; f.ba_sq = nullptr; }
    if (adapter) {
        // the V tiles of each block sum its slices into ba_sq (fixed order, as the finisher)
        FinishArgs fa{};
        fa.ba_part = ba; fa.ba_parts = plan.sb.ns; fa.d_out = d_out; fa.ba_sq = a.ba_sq;
        f = fa;
    }
    const int fin_total = adapter ? plan.sb.ns
                                  : u.ks * u.sp.ns + ((partial || given) ? 0 : plan.sb.ns);
    auto set_fin = [&](TcParams& p) {
        if (!fuse && !adapter) return;
        p.fin = f;
        p.fin_count = counters;
        p.fin_total = fin_total;
    };

    // DFX_FIN_RESET=1: zero the counters at the start of every call — a guard against callers
    // that overlap two calls of one context (outside the contract, dfx.h).  Measured: the
    // memset node costs the pipelined C2 step 2.4 % (training) and 14 % (inference), so off.
    static const bool fin_reset = env_int("DFX_FIN_RESET", 0) != 0;
    if (fuse && fin_reset &&
        (err = cudaMemsetAsync(counters, 0, size_t(m_tiles) * sizeof(unsigned), st)) != cudaSuccess)
        return err;
    cudaStream_t side = st;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    if (forked) {
        side = ws_side_stream(ws, &err);
        if (err != cudaSuccess) return err;
        ev_fork = ws_event(ws, 0, &err);
        ev_join = ws_event(ws, 1, &err);
        if (err != cudaSuccess) return err;
        if ((err = cudaEventRecord(ev_fork, st)) != cudaSuccess) return err;
        if ((err = cudaStreamWaitEvent(side, ev_fork, 0)) != cudaSuccess) return err;
    }

    auto launch_u = [&]() -> cudaError_t {
        CUtensorMap tw, ta;
        cudaError_t e = make_tmap_2d(&tw, el, a.w, d_out, d_in, d_in * 2, kBK, kBM, true);
        if (e != cudaSuccess) return e;
        TcParams p{};
        p.M = d_out; p.N = r; p.k_total = d_in; p.kb_per_split = u.kbps;
        p.n_split = u.sp.ns; p.bn = u.sp.bn;
        p.x_kwrap = 0; p.chunk = a.chunk_size;
        p.Z = a.b; p.ldz = r;
        p.out = cross; p.base_out = base; p.do_chain = 1;
        if (a.base_cached) p.do_chain = 0;     // frozen W: base_sq comes from the cache
        set_fin(p);
#ifdef DFX_KO_CHAIN
        p.do_chain = 0;
#endif
        if (u.pair) {
            // A box = half of the pair's BN rows (each CTA of the pair loads its half)
            e = make_tmap_2d(&ta, el, a.a, r, d_in, d_in * 2, kBK, u.sp.bn / 2, true);
            if (e != cudaSuccess) return e;
            p.nh = u.nh;
            p.ka = pair_atoms(u.nh, u.kbps, (d_in + kBK - 1) / kBK);
            // one 3-D TMA per operand per stage when the stage holds several atoms
            static const int t3 = env_int("DFX_PAIR_TMA3D", 1);
            if (t3 && p.ka > 1 && d_in % kBK == 0 &&
                make_tmap_3d_katoms(&tw, el, a.w, d_out, d_in, d_in * 2, kBM, p.ka) == cudaSuccess &&
                make_tmap_3d_katoms(&ta, el, a.a, r, d_in, d_in * 2, u.sp.bn / 2, p.ka) == cudaSuccess)
                p.tma3d = 1;
            static const int wpf = env_int("DFX_W_PREFETCH", 0);   // K blocks of W warmed into L2 ahead
            p.w_prefetch = wpf;
            p.stages = stages_for_pair(u.sp.bn, u.nh, p.ka);
            // DFX_PAIR_STAGES caps the ring (measurement: leaves shared memory for a co-resident CTA)
            static const int cap_st = env_int("DFX_PAIR_STAGES", 0);
            if (cap_st >= 2) p.stages = std::min(p.stages, cap_st);
            p.tiles = static_cast<int>(pm_tiles * u.sp.ns);
            const int pairs = std::min<int>(p.tiles, std::max(1, u.ctas / (2 * u.ks)));
            if (std::getenv("DFX_PLAN_PRINT"))
                std::fprintf(stderr, "u plan: pairs %d ks %d kbps %d tiles %d n_split %d bn %d nh %d stages %d"
                             " strategy %d side %d sms %d\n", pairs, u.ks, u.kbps, p.tiles, p.n_split, p.bn,
                             p.nh, p.stages, int(plan.strategy), plan.side, sms);
            // one tile per CTA and a ring slot that holds the tile's B rows: stage them by TMA
            // for the epilogue (DFX_PAIR_ZSMEM=0 keeps per-thread loads from L2)
            CUtensorMap tz = tw;
            static const int zs = env_int("DFX_PAIR_ZSMEM", 1);
            const int bn_pair = p.nh * p.bn;
            const int stage_b = p.ka * (kXStage + p.nh * (p.bn / 2) * kBK * 2);
            if (zs && p.tiles <= pairs && (bn_pair + kBK - 1) / kBK * kXStage <= stage_b &&
                make_tmap_2d(&tz, el, a.b, d_out, r, r * 2, kBK, kBM, true) == cudaSuccess)
                p.zsmem = 1;
            e = launch_tc_pair(tw, ta, tz, p, pairs, u.ks, st, "u_rowdot_tc", el);
        } else {
            e = make_tmap_2d(&ta, el, a.a, r, d_in, d_in * 2, kBK, u.sp.bn, true);
            if (e != cudaSuccess) return e;
            p.stages = stages_for(u.sp.bn);
            p.tiles = static_cast<int>(m_tiles * u.sp.ns);
            const int gx = std::min<int>(p.tiles, std::max(1, u.ctas / u.ks));
            e = launch_tc(kTcRowdot, tw, ta, p, dim3(gx, u.ks), st, "u_rowdot_tc", false, el);
        }
        if (e == cudaSuccess && launches) ++*launches;
        return e;
    };
    auto launch_gram = [&](cudaStream_t gs) -> cudaError_t {
        CUtensorMap ta;
        cudaError_t e = make_tmap_2d(&ta, el, a.a, r, d_in, d_in * 2, kBK, kBM, true);
        if (e != cudaSuccess) return e;
        TcParams p{};
        p.M = r; p.N = r; p.k_total = d_in; p.kb_per_split = plan.g_kbps; p.n_split = 1;
        p.bn = kBM; p.stages = stages_for(kBM); p.chunk = a.chunk_size;
        p.out = gpart; p.gram_nt = nt; p.tiles = gtiles;
        const int gx = std::min(gtiles, std::max(1, plan.g_ctas / plan.g_ks));
        e = launch_tc(kTcStore, ta, ta, p, dim3(gx, plan.g_ks), gs, "gram_tc", tpc && gs != st, el);
        if (e != cudaSuccess) return e;
        const int64_t n = r * r_pad;
        prof_begin("gram_reduce", gs);
        gram_reduce<<<static_cast<unsigned>((n + 255) / 256), 256, 0, gs>>>(
            gpart, plan.g_ks, nt, r, r_pad, (partial || half) ? nullptr : g2,
            partial ? a.gram_out : gf32);
        prof_end(gs);
        if (launches) *launches += 2;
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        if (!half || partial) return cudaSuccess;
        prof_begin("gram_split", gs);
        gram_split<__half><<<static_cast<unsigned>((n + 255) / 256), 256, 0, gs>>>(
            gf32, r, r_pad, reinterpret_cast<__half*>(g2), inv_scale);
        prof_end(gs);
        if (launches) *launches += 1;
        return cudaGetLastError();
    };
    auto launch_v = [&](cudaStream_t vs) -> cudaError_t {
        CUtensorMap tb, tg;
        cudaError_t e = make_tmap_2d(&tb, el, a.b, d_out, r, r * 2, kBK, kBM, true);
        if (e != cudaSuccess) return e;
        if (plan.v_gstat) {
            e = make_tmap_2d(&tg, el, g2, r, 2 * r_pad, 2 * r_pad * 2, kBK, plan.sb.bn / 2, true);
            if (e != cudaSuccess) return e;
            TcParams p{};
            p.M = d_out; p.N = r; p.bn = plan.sb.bn; p.n_split = plan.sb.ns;
            p.ka = static_cast<int>(r_pad / kBK);
            p.stages = gstat_shape(r).stages;
            p.Z = a.b; p.ldz = r; p.out = ba; p.out_scale = inv_scale;
            p.tiles = static_cast<int>(pm_tiles);
            set_fin(p);
            // Measurement switches: DFX_V_HALF=1 runs V on half the planned pairs under an SM
            // budget (two tiles each, G slice resident, the other SMs left to the compose
            // stream), DFX_V_PAIRS=n caps the pairs.  C2 training +0.3-1 %, but C3 -2.5 / -8 %
            // and the C5 stack -18 % (profiles/r02_v_pairs_sweep.txt): off.
            static const int v_cap = env_int("DFX_V_PAIRS", 0);
            static const int v_half = env_int("DFX_V_HALF", 0);
            const int nsl = std::max(1, gstat_shape(r).nsl);
            int v_pairs = plan.b_ctas / 2;
            if (v_cap > 0) v_pairs = std::min(v_cap, v_pairs);
            else if (v_half && sms < device_sm_count())
                v_pairs = std::max(nsl, v_pairs / 2 / nsl * nsl);
            e = launch_gstat(tb, tg, p, v_pairs, vs, el);
            if (e == cudaSuccess && launches) ++*launches;
            return e;
        }
        e = make_tmap_2d(&tg, el, g2, r, 2 * r_pad, 2 * r_pad * 2, kBK, plan.sb.bn, true);
        if (e != cudaSuccess) return e;
        TcParams p{};
        p.M = d_out; p.N = r; p.k_total = 2 * r_pad;
        p.kb_per_split = static_cast<int>(2 * r_pad / kBK);
        p.n_split = plan.sb.ns; p.bn = plan.sb.bn; p.stages = stages_for(plan.sb.bn);
        p.x_kwrap = static_cast<int>(r_pad); p.chunk = a.chunk_size;
        p.Z = a.b; p.ldz = r;
        p.out = ba; p.do_chain = 0;
        p.out_scale = inv_scale;
        p.tiles = static_cast<int>(m_tiles * plan.sb.ns);
        set_fin(p);
        e = launch_tc(kTcRowdot, tb, tg, p, dim3(std::max(1, plan.b_ctas), 1), vs, "ba_rowdot_tc",
                      tpc && vs != st, el);
        if (e == cudaSuccess && launches) ++*launches;
        return e;
    };

    auto run = [&]() -> cudaError_t {
        cudaError_t e;
        if (adapter) {
            if ((e = launch_gram(st)) != cudaSuccess) return e;
            return launch_v(st);
        }
        if (given) return launch_u();
        if (plan.strategy == kSerial) {
            if ((e = launch_gram(st)) != cudaSuccess) return e;
            if ((e = launch_u()) != cudaSuccess) return e;
            if (!partial && (e = launch_v(st)) != cudaSuccess) return e;
        } else {
            // U first on the caller's stream (it claims its SMs), the adapter chain beside it
            if ((e = launch_u()) != cudaSuccess) return e;
            if ((e = launch_gram(side)) != cudaSuccess) return e;
            if (plan.strategy == kSideAll && !partial && (e = launch_v(side)) != cudaSuccess)
                return e;
            if ((e = cudaEventRecord(ev_join, side)) != cudaSuccess) return e;
            if ((e = cudaStreamWaitEvent(st, ev_join, 0)) != cudaSuccess) return e;
            if (plan.strategy == kSideGram && !partial && (e = launch_v(st)) != cudaSuccess)
                return e;
        }
        return cudaSuccess;
    };
    if ((err = run()) != cudaSuccess) {
        // a launch failed after others were queued: the fused finisher's counters would keep
        // the queued tiles' arrivals; clear them behind everything queued on both streams
        if (counters) {
            if (forked && cudaEventRecord(ev_join, side) == cudaSuccess)
                cudaStreamWaitEvent(st, ev_join, 0);
            cudaMemsetAsync(counters, 0, size_t(m_tiles) * sizeof(unsigned), st);
        }
        return err;
    }

    if (fuse || adapter) return cudaSuccess;
    if (launches) ++*launches;
    return launch_finish(f, st);
}

// fp32 weights (the accuracy configuration, BASELINE configs[0]): the same three GEMMs on
// the tensor cores with 3xTF32 operands (tc_rowdot<., true>), serially on all SMs:
// G = A A^T (split-K partial tiles, fixed-order reduction to fp32 G), U = W A^T with the
// bitwise fp32 base_sq chain, V = B G (K = r), then the finisher.
bool norm_tf32_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("DFX_NORM_TF32");
        return !(e && e[0] == '0');
    }();
    return on;
}

bool norm_tc_f32_supported(int64_t d_out, int64_t d_in, int64_t r, int64_t chunk) {
    return d_in >= 32 && d_in % 4 == 0 && r % 8 == 0 && r >= 16 && r <= 2048 && chunk % 32 == 0 &&
           d_out >= 1 && d_in < (int64_t(1) << 31) && d_out < (int64_t(1) << 31);
}

cudaError_t launch_norm_tc_f32(const NormArgs& a, Workspace* ws, cudaStream_t st, int* launches) {
    cudaError_t err = cudaSuccess;
    constexpr int64_t kKB = 32;                       // fp32 elements per K block (128 bytes)
    const int64_t r = a.r, d_out = a.d_out, d_in = a.d_in;
    const int64_t m_tiles = (d_out + kBM - 1) / kBM;
    const int64_t kb_in = (d_in + kKB - 1) / kKB;
    const int64_t chunk_blocks = a.chunk_size / kKB;
    const int64_t n_chunks = (d_in + a.chunk_size - 1) / a.chunk_size;
    const int sms = ws_sm_count(ws);
    const int nt = static_cast<int>((r + kBM - 1) / kBM);
    const int gtiles = nt * (nt + 1) / 2;

    // U: N / K splits as for bf16 (K splits only on ChunkPlan boundaries)
    Split sp = choose_split(m_tiles, r, kb_in, static_cast<int>(std::min<int64_t>(n_chunks, 8)), sms);
    {
        // 3xTF32 issues the same 12 UMMAs per K block whatever N is, and its stage holds the
        // low parts too: use as many N splits as fill the SMs (smaller stages, more of them;
        // measured at C1: N = 96 x 4 splits 230 us vs N = 192 x 2 313 us)
        const int ns_min = static_cast<int>((r + 255) / 256);
        const int ns = static_cast<int>(std::max<int64_t>(
            ns_min, std::min<int64_t>(std::max<int64_t>(1, sms / std::max<int64_t>(1, m_tiles * sp.ks)),
                                      std::max<int64_t>(1, r / 32))));
        sp = {ns, sp.ks, static_cast<int>(((r + ns - 1) / ns + 15) / 16 * 16)};
    }
    const int64_t kbps = (n_chunks + sp.ks - 1) / sp.ks * chunk_blocks;
    const int uks = static_cast<int>((kb_in + kbps - 1) / kbps);
    // G: split-K over the SMs
    int gks = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(sms / gtiles, kb_in / 8)));
    const int64_t gkbps = (kb_in + gks - 1) / gks;
    gks = static_cast<int>((kb_in + gkbps - 1) / gkbps);
    // V = B G: K = r
    const int64_t kb_r = (r + kKB - 1) / kKB;
    const Split sb = choose_split(m_tiles, r, kb_r, 1, sms);

    float* cross = static_cast<float*>(ws_get(ws, kWsCross, size_t(uks) * sp.ns * d_out * 4, &err));
    if (err != cudaSuccess) return err;
    float* base = static_cast<float*>(ws_get(ws, kWsBase, size_t(n_chunks) * d_out * 4, &err));
    if (err != cudaSuccess) return err;
    float* gpart = static_cast<float*>(ws_get(ws, kWsGramPart, size_t(gks) * gtiles * kBM * kBM * 4, &err));
    if (err != cudaSuccess) return err;
    float* G = static_cast<float*>(ws_get(ws, kWsGram, size_t(r) * r * 4, &err));
    if (err != cudaSuccess) return err;
    float* ba = static_cast<float*>(ws_get(ws, kWsBa, size_t(sb.ns) * d_out * 4, &err));
    if (err != cudaSuccess) return err;

    // G = A A^T -> fixed-order split sum, mirrored, fp32
    {
        CUtensorMap ta;
        if ((err = make_tmap_2d(&ta, kF32, a.a, r, d_in, d_in * 4, kKB, kBM, true)) != cudaSuccess) return err;
        TcParams p{};
        p.M = r; p.N = r; p.k_total = d_in; p.kb_per_split = static_cast<int>(gkbps); p.n_split = 1;
        p.bn = kBM; p.stages = stages_for(kBM, true); p.chunk = a.chunk_size;
        p.out = gpart; p.gram_nt = nt; p.tiles = gtiles;
        const int gx = std::min(gtiles, std::max(1, sms / gks));
        if ((err = launch_tc(kTcStore, ta, ta, p, dim3(gx, gks), st, "gram_tf32x3", false, kF32)) != cudaSuccess)
            return err;
        prof_begin("gram_reduce", st);
        gram_reduce<<<static_cast<unsigned>((r * r + 255) / 256), 256, 0, st>>>(gpart, gks, nt, r, r,
                                                                                 nullptr, G);
        prof_end(st);
        if ((err = cudaGetLastError()) != cudaSuccess) return err;
    }
    // U = W A^T, cross = rowdot(U, B), base_sq chain
    {
        CUtensorMap tw, ta;
        if ((err = make_tmap_2d(&tw, kF32, a.w, d_out, d_in, d_in * 4, kKB, kBM, true)) != cudaSuccess) return err;
        if ((err = make_tmap_2d(&ta, kF32, a.a, r, d_in, d_in * 4, kKB, sp.bn, true)) != cudaSuccess) return err;
        TcParams p{};
        p.M = d_out; p.N = r; p.k_total = d_in; p.kb_per_split = static_cast<int>(kbps);
        p.n_split = sp.ns; p.bn = sp.bn; p.stages = stages_for(sp.bn, true); p.chunk = a.chunk_size;
        p.Z = a.b; p.ldz = r; p.out = cross; p.base_out = base; p.do_chain = 1;
        p.tiles = static_cast<int>(m_tiles * sp.ns);
        const int gx = std::min<int>(p.tiles, std::max(1, sms / uks));
        if ((err = launch_tc(kTcRowdot, tw, ta, p, dim3(gx, uks), st, "u_rowdot_tf32x3", false, kF32)) != cudaSuccess)
            return err;
    }
    // V = B G, ba_sq = rowdot(V, B)
    {
        CUtensorMap tb, tg;
        if ((err = make_tmap_2d(&tb, kF32, a.b, d_out, r, r * 4, kKB, kBM, true)) != cudaSuccess) return err;
        if ((err = make_tmap_2d(&tg, kF32, G, r, r, r * 4, kKB, sb.bn, true)) != cudaSuccess) return err;
        TcParams p{};
        p.M = d_out; p.N = r; p.k_total = r; p.kb_per_split = static_cast<int>(kb_r);
        p.n_split = sb.ns; p.bn = sb.bn; p.stages = stages_for(sb.bn, true); p.chunk = a.chunk_size;
        p.Z = a.b; p.ldz = r; p.out = ba; p.do_chain = 0;
        p.tiles = static_cast<int>(m_tiles * sb.ns);
        if ((err = launch_tc(kTcRowdot, tb, tg, p, dim3(std::min(p.tiles, sms), 1), st, "ba_rowdot_tf32x3",
                             false, kF32)) != cudaSuccess)
            return err;
    }
    if (launches) *launches += 5;
    FinishArgs f{};
    f.base_part = base; f.base_parts = static_cast<int>(n_chunks);
    f.cross_part = cross; f.cross_parts = uks * sp.ns;
    f.ba_part = ba; f.ba_parts = sb.ns;
    f.d_out = d_out; f.two_s = 2.0 * a.s; f.s2 = a.s * a.s;
    f.base_sq = a.base_sq; f.cross = a.cross; f.ba_sq = a.ba_sq;
    f.round_dt = a.round_dt; f.w_norm = a.w_norm;
    f.m = a.m; f.mag_dt = a.mag_dt; f.g = a.m ? a.g : nullptr;
    return launch_finish(f, st);
}

// d_in split, step 2 (after the caller's all-reduce of {G, base_sq, cross}): B [G_hi|G_lo]
// on all SMs, then assemble / round / magnitude.  Reads no W.
cudaError_t launch_norm_finish_tc(const NormArgs& a, Workspace* ws, cudaStream_t st,
                                  int* launches) {
    cudaError_t err = cudaSuccess;
    const int64_t r = a.r, d_out = a.d_out;
    const int64_t r_pad = (r + kBK - 1) / kBK * kBK;
    const int64_t m_tiles = (d_out + kBM - 1) / kBM;
    const int sms = ws_sm_count(ws);
    FinishArgs f{};
    f.base_part = a.base_in; f.base_parts = 1;
    f.d_out = d_out; f.two_s = 2.0 * a.s; f.s2 = a.s * a.s;
    f.base_sq = a.base_sq; f.cross = a.cross; f.ba_sq = a.ba_sq;
    f.round_dt = a.round_dt; f.w_norm = a.w_norm;
    f.m = a.m; f.mag_dt = a.mag_dt; f.g = a.m ? a.g : nullptr;
    if (a.s != 0.0) {  // s == 0: the reference skips cross / ba_sq (factored_norm.cpp:37)
        __nv_bfloat16* g2 = static_cast<__nv_bfloat16*>(
            ws_get(ws, kWsGram2, size_t(r) * 2 * r_pad * sizeof(__nv_bfloat16), &err));
        if (err != cudaSuccess) return err;
        const Split sb = choose_split(m_tiles, r, 2 * r_pad / kBK, 1, sms);
        float* ba = static_cast<float*>(ws_get(ws, kWsBa, size_t(sb.ns) * d_out * sizeof(float), &err));
        if (err != cudaSuccess) return err;
        const int64_t n = r * r_pad;
        const bool half = a.dt == kF16;
        float* inv_scale = nullptr;
        if (half) {
            inv_scale = static_cast<float*>(ws_get(ws, kWsScale, 256, &err));
            if (err != cudaSuccess) return err;
        }
        prof_begin("gram_split", st);
        if (half)
            gram_split<__half><<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(
                a.gram_in, r, r_pad, reinterpret_cast<__half*>(g2), inv_scale);
        else
            gram_split<__nv_bfloat16><<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(
                a.gram_in, r, r_pad, g2, nullptr);
        prof_end(st);
        if ((err = cudaGetLastError()) != cudaSuccess) return err;
        CUtensorMap tb, tg;
        err = make_tmap_2d(&tb, a.dt, a.b, d_out, r, r * 2, kBK, kBM, true);
        if (err != cudaSuccess) return err;
        err = make_tmap_2d(&tg, a.dt, g2, r, 2 * r_pad, 2 * r_pad * 2, kBK, sb.bn, true);
        if (err != cudaSuccess) return err;
        TcParams p{};
        p.M = d_out; p.N = r; p.k_total = 2 * r_pad;
        p.kb_per_split = static_cast<int>(2 * r_pad / kBK);
        p.n_split = sb.ns; p.bn = sb.bn; p.stages = stages_for(sb.bn);
        p.x_kwrap = static_cast<int>(r_pad); p.chunk = 64;
        p.Z = a.b; p.ldz = r;
        p.out = ba; p.do_chain = 0;
        p.out_scale = inv_scale;
        p.tiles = static_cast<int>(m_tiles * sb.ns);
        err = launch_tc(kTcRowdot, tb, tg, p, dim3(std::min(p.tiles, sms), 1), st, "ba_rowdot_tc",
                        false, a.dt);
        if (err != cudaSuccess) return err;
        if (launches) *launches += 2;
        f.cross_part = a.cross_in; f.cross_parts = 1;
        f.ba_part = ba; f.ba_parts = sb.ns;
    }
    if (launches) ++*launches;
    return launch_finish(f, st);
}

}  // namespace dfx
