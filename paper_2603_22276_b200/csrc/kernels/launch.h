// launch.h — internal launcher interface between the C-ABI layer (dfx_capi.cu) and the
// kernel translation units.  Not installed; the public boundary is include/dfx.h.
#pragma once

#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace dfx {

enum DType : int { kF32 = 0, kBF16 = 1, kF16 = 2 };

inline int elem_bytes(int dt) { return dt == kF32 ? 4 : 2; }

// Encodes a 2-D row-major tensor map (rows x cols elements, row pitch in bytes)
// with the given box; swizzle128 selects CU_TENSOR_MAP_SWIZZLE_128B.
// Returns cudaSuccess or an error (driver entry point missing / encode failure).
cudaError_t make_tmap_2d(CUtensorMap* out, int dt, const void* base, uint64_t rows, uint64_t cols,
                         uint64_t row_pitch_bytes, uint32_t box_cols, uint32_t box_rows,
                         bool swizzle128);
// Same with an explicit swizzle span in bytes (0, 32, 64 or 128).
cudaError_t make_tmap_2d_sw(CUtensorMap* out, int dt, const void* base, uint64_t rows,
                            uint64_t cols, uint64_t row_pitch_bytes, uint32_t box_cols,
                            uint32_t box_rows, int swizzle_bytes);

// [rows x cols] viewed as [cols/64][rows][64], box {64, box_rows, atoms}: `atoms` consecutive
// 64-wide K blocks per TMA instruction (cols % 64 == 0, 16-bit types).
cudaError_t make_tmap_3d_katoms(CUtensorMap* out, int dt, const void* base, uint64_t rows,
                                uint64_t cols, uint64_t row_pitch_bytes, uint32_t box_rows,
                                uint32_t atoms);

// Attributes of the current device, queried once per device and cached (launch paths call
// these on every launch).
int device_sm_count();
int device_smem_optin();

// cudaFuncAttributeMaxDynamicSharedMemorySize for `func` on the current device, set once per
// (function, device) pair (thread-safe; a process may drive several devices).
cudaError_t ensure_max_dyn_smem(const void* func, int bytes);

// ---------------------------------------------------------------- compose
cudaError_t launch_compose_fwd(int dt, const void* base, const void* lora, const float* g, float sf,
                               int64_t rows, int64_t d_out, void* delta, void* inner,
                               cudaStream_t st, int* launches);

// partitioned: the caller runs this beside the norm GEMMs on an SM budget
// (dfx_ctx_set_sm_budget): the d_mag backward then uses 256-byte column slabs (half the CTAs,
// each a whole SM), which co-schedules better with the GEMM's CTA pairs (DESIGN 5.3)
cudaError_t launch_compose_bwd(int dt, const void* dy, const float* g, float sf, const void* inner,
                               const float* w_norm, int64_t rows, int64_t d_out, void* d_lora,
                               void* d_base, float* d_mag, cudaStream_t st, int* launches,
                               bool partitioned = false);

// LoRA-up GEMM (mid . B^T on tcgen05) fused with compose + residual (lora_compose.cu).
// Outputs y / delta / inner / lora are each optional (at most three at once).
cudaError_t launch_lora_compose(int dt, const void* mid, const void* b, const void* base,
                                const float* g, float s, const float* bias, int64_t rows,
                                int64_t d_out, int64_t r, void* y, void* delta, void* inner,
                                void* lora, cudaStream_t st, int* launches);

// The layer's plain GEMMs with the reference's working_matmul semantics (layer_gemm.cu):
// C [M x N] row-major = round_dtype(serial-k fp32 sum of a(i, k) * b(k, j)), with
// a(i, k) = a[i * sa_i + k * sa_k] and b(k, j) = b[k * sb_k + j * sb_j] (element strides).
cudaError_t launch_working_matmul(int dt, const void* a, int64_t sa_i, int64_t sa_k, const void* b,
                                  int64_t sb_k, int64_t sb_j, int64_t M, int64_t N, int64_t K,
                                  void* c, cudaStream_t st, int* launches);

// ------------------------------------------------------------------- norm
struct NormArgs {
    int dt;
    const void* w;
    const void* a;
    const void* b;
    int64_t d_out, d_in, r;
    double s;
    int64_t chunk_size;
    // outputs (device): any of these may be null except where noted
    float* base_sq;
    float* cross;
    float* ba_sq;
    const float* m;   // magnitude (fp32), null => no g
    float* w_norm;    // dtype-rounded norm (fp32 storage)
    float* g;         // dtype-rounded scale (fp32 storage)
    int round_dt;     // dtype the norm is rounded to (kF32 => plain fp32 assemble)
    int mag_dt;       // working dtype of the magnitude division
    // d_in split (FSDP2-style): kNormPartial computes this rank's K-slice terms
    // (gram_out, base_sq, cross); kNormFinish completes from reduced inputs.
    int mode;
    float* gram_out;        // partial: fp32 [r x r]
    const float* gram_in;   // finish: reduced fp32 Gram [r x r]
    const float* base_in;   // finish: reduced base_sq [d_out]
    const float* cross_in;  // finish: reduced cross [d_out]
    // full mode with a cached base_sq [d_out] of a frozen W (from an
    // earlier call's base_sq output): the U kernel runs without its base_sq chain and the
    // finisher takes the cached value.  bf16 tensor-core path only.
    const float* base_cached;
    // Split form for pipelined stacks (bf16 / fp16 tensor-core path): kNormAdapter computes
    // only the adapter term ba_sq (Gram + V, no W) into `ba_sq`; a kNormFull call with
    // ba_given runs only W.A^T (+ chain) and finishes with that ba_sq.  The two use disjoint
    // workspace, so an adapter call may overlap a ba_given call of the same context.
    const float* ba_given;
};

enum NormMode : int { kNormFull = 0, kNormPartial = 1, kNormFinish = 2, kNormAdapter = 3 };

// Per-launch device timing (dfx_profile_enable): launch sites bracket each kernel
// with these; they are no-ops unless the calling thread is inside a call on a
// profiling context.
void prof_begin(const char* name, cudaStream_t st);
void prof_end(cudaStream_t st);

// ------------------------------------------------------------ symmetric all-reduce (comm.cu)
constexpr int kCommMaxRanks = 16;
constexpr int kCommMaxBlocks = 64;
constexpr int kCommThreads = 512;
struct CommArgs {
    char* peers[kCommMaxRanks];   // every rank's symmetric allocation, mapped here (rank order)
    int rank, world;
    int64_t count;                // fp32 elements reduced
    float* out;                   // local result [count]
    size_t start_off, end_off, epoch_off, err_off;   // byte offsets inside an allocation
    int max_blocks;               // identical on every rank (block b pairs with block b)
};
cudaError_t launch_allreduce(const CommArgs& a, cudaStream_t st, int* launches);

struct Workspace;  // owned by the context (dfx_capi.cu)
void* ws_get(Workspace* ws, int slot, size_t bytes, cudaError_t* err);
// Same, zero-filled when (re)allocated (kernels keep it zero between calls).
void* ws_get_zeroed(Workspace* ws, int slot, size_t bytes, cudaError_t* err);
// Context-owned side stream (non-blocking) and fork/join events for intra-call concurrency.
cudaStream_t ws_side_stream(Workspace* ws, cudaError_t* err);
cudaEvent_t ws_event(Workspace* ws, int idx, cudaError_t* err);
int ws_sm_count(Workspace* ws);

cudaError_t launch_norm(const NormArgs& a, Workspace* ws, cudaStream_t st, int* launches);

cudaError_t launch_assemble(const float* base_sq, const float* cross, const float* ba_sq,
                            double two_s, double s2, int64_t n, int round_dt, float* out,
                            cudaStream_t st, int* launches);

cudaError_t launch_magnitude_scale(int dt, const float* m, const float* w_norm, int64_t n,
                                   float* g, cudaStream_t st, int* launches);

// Chooses the tensor-core path for (dt, shape); exposed for tests/bench reporting.
int norm_uses_tensor_cores(int dt, int64_t d_out, int64_t d_in, int64_t r);
void norm_plan_info(int64_t d_out, int64_t d_in, int64_t r, int64_t chunk_size, int sms,
                    int* u_ctas, int* side_ctas, int* strategy);

}  // namespace dfx
