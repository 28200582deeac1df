/*
 * dfx.h — C ABI of the B200-native DoRA hot path (libdfx.so).
 *
 * This is the drop-in boundary.  Every entry point replaces one function of the
 * reference C++ API (/root/reference/proj/include/dorafactor/, cited per entry)
 * with a device-pointer, caller-owned-buffer, stream-ordered equivalent.  The C++
 * drop-in (include/dorafactor/ headers, libdorafactor_b200.so) implements the
 * reference signatures on top of these calls; other hosts bind them directly
 * (ctypes / cgo / JNI stubs in INTEGRATION.md).
 *
 * Conventions
 *   - Matrices are dense row-major device arrays of the call's dtype (fp32, bf16 or
 *     fp16 bits).  Per-row vectors (g, w_norm, m, terms, d_mag) are fp32 device
 *     arrays; where the reference rounds a vector to the working dtype the fp32
 *     array holds the rounded (exactly representable) value.
 *   - Calls are asynchronous on `stream` (a cudaStream_t; NULL = legacy default).
 *     They never allocate on the hot path except to grow the context workspace on
 *     first use of a larger shape, and never synchronise the device.
 *   - Return value: DFX_OK, or an error code with a message in dfx_last_error()
 *     (thread-local).  DFX_EINVAL is raised exactly where the reference throws
 *     std::invalid_argument.  Non-finite values propagate (IEEE), never error.
 *   - A context is bound to one device; concurrent calls on one context must be
 *     serialised by the caller (its workspace is shared).  Use one context per
 *     concurrently used stream.  Two calls of one context that overlap in time (e.g.
 *     issued on two streams without an event between them) produce undefined results,
 *     and leave the fused finisher's per-block arrival counters inconsistent for the
 *     context's later norm calls: recreate the context after such a misuse.
 *   - There is no CPU fallback: every call runs sm_100a kernels and fails with
 *     DFX_ENODEV when no usable device is present.
 */
#ifndef DFX_H
#define DFX_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* dfx_stream_t; /* == cudaStream_t */
typedef struct dfx_ctx dfx_ctx;

typedef enum dfx_dtype {
    DFX_F32 = 0,  /* DTypeKind::FP32  (dtype.hpp:12) */
    DFX_BF16 = 1, /* DTypeKind::BF16E */
    DFX_F16 = 2   /* DTypeKind::FP16E */
} dfx_dtype;

enum {
    DFX_OK = 0,
    DFX_EINVAL = 1,      /* reference would throw std::invalid_argument */
    DFX_ECUDA = 2,       /* CUDA runtime / driver error */
    DFX_ENOMEM = 3,      /* workspace allocation failed */
    DFX_ENODEV = 4,      /* no sm_100 device / context for another device */
    DFX_EUNSUPPORTED = 5 /* dtype not handled by this entry point */
};

#define DFX_ABI_VERSION 1

int dfx_abi_version(void);
const char* dfx_last_error(void);

/* Context: device binding + grow-only workspace (Gram partials, bf16 hi/lo Gram,
 * per-split row partials). */
int dfx_ctx_create(int device, dfx_ctx** out);
void dfx_ctx_destroy(dfx_ctx* ctx);
/* Number of kernels launched by this context since creation (evidence counter). */
int64_t dfx_ctx_launches(const dfx_ctx* ctx);

/* Cap the SMs the row-norm GEMMs plan for (0 = all).  A caller that streams compose kernels
 * concurrently with the next module's norm (a pipelined layer stack) leaves the remaining SMs
 * to them; the planner then prefers the 2-SM W.A^T tiling that ingests W once (full r per CTA
 * pair), which needs fewer SMs.  Results are identical for every budget. */
int dfx_ctx_set_sm_budget(dfx_ctx* ctx, int sms);

/* Per-kernel device timing.  While enabled, every kernel the context launches is
 * bracketed by CUDA events on its stream.  dfx_profile_report synchronises the device,
 * writes one line per kernel ("name launches total_ms min_ms max_ms\n") into buf and
 * resets the records. */
int dfx_profile_enable(dfx_ctx* ctx, int on);
int dfx_profile_report(dfx_ctx* ctx, char* buf, size_t len);

/* plan_chunks (matrix.hpp:68, matrix.cpp:28-51): host-only, no device needed.
 * DFX_EINVAL where the reference throws. */
int dfx_plan_chunks(uint64_t d_out, uint64_t d_in, uint64_t budget_bytes,
                    uint64_t* chunk_size, uint64_t* num_chunks);

/* factored_norm_terms (factored_norm.hpp:44): base_sq / cross / ba_sq for
 * ||W + sBA||^2_row.  W [d_out x d_in], A [r x d_in], B [d_out x r] (dtype).
 * chunk_size is ChunkPlan::chunk_size (base_sq chunk-partial semantics).
 * Outputs are fp32 [d_out]; any of them may be NULL. */
int dfx_norm_terms(dfx_ctx* ctx, dfx_dtype dtype, const void* W, const void* A, const void* B,
                   int64_t d_out, int64_t d_in, int64_t r, double s, int64_t chunk_size,
                   float* base_sq, float* cross, float* ba_sq, dfx_stream_t stream);

/* assemble_norm (factored_norm.hpp:51) when round_to == DFX_F32; with round_to =
 * BF16/F16 additionally the round_to_dtype of factored_row_norm (:213-215). */
int dfx_assemble_norm(dfx_ctx* ctx, const float* base_sq, const float* cross,
                      const float* ba_sq, double two_s, double s2, int64_t n,
                      dfx_dtype round_to, float* w_norm, dfx_stream_t stream);

/* magnitude_scale (factored_norm.hpp:63-64), non-fp64 working dtype:
 * g = round_dtype(fl32(m) / max(fl32(w_norm), fl32(eps_dtype))). */
int dfx_magnitude_scale(dfx_ctx* ctx, dfx_dtype dtype, const float* m, const float* w_norm,
                        int64_t n, float* g, dfx_stream_t stream);

/* factored_row_norm (factored_norm.hpp:57-58) fused with magnitude_scale: one launch
 * sequence producing w_norm (rounded to `dtype`) and, when m != NULL, g (rounded to
 * `mag_dtype`).  terms (3 x d_out fp32: base_sq, cross, ba_sq) may be NULL. */
int dfx_row_norm(dfx_ctx* ctx, dfx_dtype dtype, const void* W, const void* A, const void* B,
                 int64_t d_out, int64_t d_in, int64_t r, double s, int64_t chunk_size,
                 const float* m, dfx_dtype mag_dtype, float* w_norm, float* g, float* terms,
                 dfx_stream_t stream);

/* SURVEY 8(f) row 4, opt-in: the factored norm with a cached ||W||^2_row for a FROZEN W.
 * refresh != 0: the full dfx_row_norm, which also writes base_sq [d_out] (fp32, the serial
 * chain's value) into base_sq_cache.  refresh == 0: the W.A^T kernel runs without its
 * base_sq chain and the finisher reads base_sq_cache instead; the result is bitwise the
 * full call's as long as W is unchanged since the refresh.  This departs from the
 * reference's contract, which recomputes the norm from W on every call
 * (factored_norm.cpp:52-61) — the caller owns the cache's validity.  W is still read (the
 * cross term needs W.A^T).  bf16 tensor-core shapes only (DFX_EUNSUPPORTED otherwise). */
int dfx_row_norm_cached(dfx_ctx* ctx, dfx_dtype dtype, const void* W, const void* A,
                        const void* B, int64_t d_out, int64_t d_in, int64_t r, double s,
                        int64_t chunk_size, float* base_sq_cache, int refresh, const float* m,
                        dfx_dtype mag_dtype, float* w_norm, float* g, dfx_stream_t stream);

/* d_in-split (FSDP2-style) factored norm — the exchange the paper leaves open
 * (PAPER.md:1073-1078).  Step 1 on every rank: the terms of this rank's K slice,
 * W_k [d_out x d_in_k], A_k [r x d_in_k], full B [d_out x r]:
 *   gram [r x r] = A_k A_k^T, base_sq [d_out] = serial chain over the slice (chunked by
 *   chunk_size), cross [d_out] = rowdot(W_k A_k^T, B)   (all fp32)
 * The caller sums {gram, base_sq, cross} over ranks (one all-reduce of r*r + 2*d_out
 * floats) and then calls dfx_norm_finish, which needs no W. */
int dfx_norm_partial(dfx_ctx* ctx, dfx_dtype dtype, const void* W_k, const void* A_k,
                     const void* B, int64_t d_out, int64_t d_in_k, int64_t r, int64_t chunk_size,
                     float* gram, float* base_sq, float* cross, dfx_stream_t stream);

/* Step 2: ba_sq = rowquad(B, G) from the reduced Gram, assemble_norm, round to `dtype`,
 * magnitude (when m != NULL).  terms (3 x d_out) optional, like dfx_row_norm. */
int dfx_norm_finish(dfx_ctx* ctx, dfx_dtype dtype, const void* B, const float* gram,
                    const float* base_sq, const float* cross, int64_t d_out, int64_t r, double s,
                    const float* m, dfx_dtype mag_dtype, float* w_norm, float* g, float* terms,
                    dfx_stream_t stream);

/* Split form of dfx_row_norm for pipelined layer stacks (bf16 / fp16 tensor-core path).
 * factored_norm_terms (factored_norm.cpp:27-120) splits into a part that reads only the
 * adapter — ba_sq = rowquad(B, A A^T) (:65-77, :104-117), the Gram and B.G GEMMs — and a part
 * that reads W: base_sq, cross = rowdot(W A^T, B), assemble, round, magnitude (:204-240).
 *   dfx_norm_adapter  writes ba_sq [d_out] (fp32);
 *   dfx_row_norm_ba   runs the W part and finishes with that ba_sq (terms, if non-null, as
 *                     dfx_row_norm's).  Same arithmetic as dfx_row_norm; the Gram's split-K
 *                     partition follows the SM budget the adapter call plans for, so ba_sq (and
 *                     through it w_norm, g) can differ from a dfx_row_norm call in the last bits,
 *                     as dfx_row_norm's own results do between SM budgets.
 * The two use disjoint context workspace, so an adapter call may run concurrently with a
 * dfx_row_norm_ba call of the same context (e.g. module i+1's adapter beside module i's W
 * part); two adapter calls, or two W calls, still must not overlap. */
/* sms > 0 caps the SMs the adapter's GEMMs plan for (it is meant to run beside other work);
 * 0 = the context's SM budget. */
int dfx_norm_adapter(dfx_ctx* ctx, dfx_dtype dtype, const void* A, const void* B,
                     int64_t d_out, int64_t d_in, int64_t r, int sms, float* ba_sq,
                     dfx_stream_t stream);
int dfx_row_norm_ba(dfx_ctx* ctx, dfx_dtype dtype, const void* W, const void* A, const void* B,
                    int64_t d_out, int64_t d_in, int64_t r, double s, int64_t chunk_size,
                    const float* ba_sq, const float* m, dfx_dtype mag_dtype, float* w_norm,
                    float* g, float* terms, dfx_stream_t stream);

/* stable_compose / fused_compose / dual_output_compose (compose.hpp:43,53-57,62-68):
 * delta = (g-1)*base + g*(s*lora) in the canonical rounding order, bitwise equal to
 * the reference; inner = s*lora + base when inner != NULL (dual output). */
int dfx_compose_fwd(dfx_ctx* ctx, dfx_dtype dtype, const void* base, const void* lora,
                    const float* g, double s, int64_t rows, int64_t d_out, void* delta,
                    void* inner, dfx_stream_t stream);

/* compose_backward (compose.hpp:73-75): d_lora = g*s*dY, d_base = (g-1)*dY; when
 * d_mag != NULL (mag_grad) also d_mag = serial-per-column sum(dY*inner) / w_norm,
 * bitwise equal to the reference's fixed serial order.  inner/w_norm required then.
 * With d_mag != NULL, d_lora and d_base may both be NULL: magnitude gradient only (a caller
 * that produced d_lora / d_base per row chunk with d_mag == NULL). */
int dfx_compose_bwd(dfx_ctx* ctx, dfx_dtype dtype, const void* dy, const float* g, double s,
                    const void* inner, const float* w_norm, int64_t rows, int64_t d_out,
                    void* d_lora, void* d_base, float* d_mag, dfx_stream_t stream);

/* The layer's plain GEMMs with the reference's working_matmul semantics (layer.cpp:15-17 over
 * matrix.cpp:53-78), bitwise: C [M x N] row-major (dtype) = round(serial-k fp32 sum of
 * a(i,k) * b(k,j)), a(i,k) = A[i*sa_i + k*sa_k], b(k,j) = B[k*sb_k + j*sb_j] (element strides,
 * so transposed operands need no copy).  CUDA cores: the serial order is the contract. */
int dfx_working_matmul(dfx_ctx* ctx, dfx_dtype dtype, const void* A, int64_t sa_i, int64_t sa_k,
                       const void* B, int64_t sb_k, int64_t sb_j, int64_t M, int64_t N, int64_t K,
                       void* C, dfx_stream_t stream);

/* layer_forward's LoRA-up GEMM fused with the compose and the residual (layer.cpp:57-58,
 * 73-120): lora = round(mid . B^T) is formed on the tensor cores and
 * never reaches HBM; per element delta = round((g-1)*base + g*(s*lora)) (compose.cpp:19-24),
 * inner = round(s*lora + base), y = round(base + delta) then round(y + bias) when bias != NULL.
 * mid [rows, r], B [d_out, r], base / outputs [rows, d_out] row-major (bf16 or fp16);
 * g, bias fp32 [d_out] holding working-dtype values.  Outputs y, delta, inner, lora are each
 * optional (NULL = not written), at most three per call.  Given the same lora, every output
 * is bitwise the reference's; lora is an fp32-accumulated tensor-core GEMM. */
int dfx_lora_compose(dfx_ctx* ctx, dfx_dtype dtype, const void* mid, const void* B,
                     const void* base, const float* g, double s, const float* bias, int64_t rows,
                     int64_t d_out, int64_t r, void* y, void* delta, void* inner, void* lora,
                     dfx_stream_t stream);

/* One whole DoRA module forward from HOST buffers (the end-to-end call a host
 * framework makes): H2D of W, A, B, m, base, lora; row norm + g; compose; D2H of
 * delta and g.  Host buffers should be pinned for full PCIe bandwidth.  Blocks
 * until the results are in host memory. */
int dfx_module_fwd_host(dfx_ctx* ctx, dfx_dtype dtype, const void* W, const void* A,
                        const void* B, const float* m, const void* base, const void* lora,
                        double s, int64_t d_out, int64_t d_in, int64_t r, int64_t rows,
                        int64_t chunk_size, void* delta, float* g);

/* One whole DoRA module TRAINING step from HOST buffers (layer_forward's hot path with a
 * trainable magnitude, then layer_backward's compose_backward, layer.cpp:61-89,139):
 * H2D of W, A, B, m, base, lora, dY; row norm + g; dual-output compose (inner stays on
 * the device); compose backward with the magnitude gradient; D2H of delta, d_lora,
 * d_base, d_mag and g.  Host buffers should be pinned.  Blocks until done. */
int dfx_module_train_host(dfx_ctx* ctx, dfx_dtype dtype, const void* W, const void* A,
                          const void* B, const float* m, const void* base, const void* lora,
                          const void* dy, double s, int64_t d_out, int64_t d_in, int64_t r,
                          int64_t rows, int64_t chunk_size, void* delta, void* d_lora,
                          void* d_base, float* d_mag, float* g);

/* ---- Symmetric-memory all-reduce for the d_in-split norm ----
 * The exchange between dfx_norm_partial and dfx_norm_finish as one kernel
 * over peer memory instead of a library collective.  Each rank creates a comm whose symmetric
 * allocation holds `count` fp32 (count >= r*r + 2*d_out); the ranks exchange their IPC handles
 * out of band (e.g. torch.distributed all_gather_object) and open them (ranks that share a
 * process pass each other's bases with dfx_comm_set_peers instead).  The rank writes its
 * partial terms into dfx_comm_buffer(); dfx_norm_allreduce then writes
 *     out[i] = ((buf_0[i] + buf_1[i]) + buf_2[i]) + ...      (rank order, fp32, RN)
 * on every rank — identical bits on every rank — with an entry and an exit barrier over
 * device flags (no host synchronisation; capturable in a CUDA graph).  Every rank must issue
 * the same sequence of dfx_norm_allreduce calls.  Spins are bounded (~5 s): a missing peer
 * raises the comm's error word (dfx_comm_status) rather than hanging the device. */
typedef struct dfx_comm dfx_comm;
#define DFX_IPC_HANDLE_BYTES 64
int dfx_comm_create(dfx_ctx* ctx, int rank, int world, int64_t count, dfx_comm** out);
void dfx_comm_destroy(dfx_comm* comm);
/* This rank's symmetric data region [count fp32] (device pointer). */
float* dfx_comm_buffer(dfx_comm* comm);
/* Base of this rank's symmetric allocation (what peers in the same process map). */
void* dfx_comm_base(dfx_comm* comm);
/* cudaIpcMemHandle_t of this rank's allocation (DFX_IPC_HANDLE_BYTES bytes into `out`). */
int dfx_comm_ipc_handle(dfx_comm* comm, void* out);
/* Open the peers' allocations: `handles` = world * DFX_IPC_HANDLE_BYTES bytes in rank order
 * (this rank's own entry is ignored). */
int dfx_comm_open(dfx_comm* comm, const void* handles);
/* Same-process peers: bases[k] = dfx_comm_base of rank k's comm (bases[rank] ignored). */
int dfx_comm_set_peers(dfx_comm* comm, void* const* bases);
/* out [count] = rank-order sum of every rank's dfx_comm_buffer (stream-ordered). */
int dfx_norm_allreduce(dfx_comm* comm, float* out, int64_t count, dfx_stream_t stream);
/* *timed_out = 0 when every barrier so far completed, 1 when a spin timed out (a peer never
 * arrived; the results of that call are invalid).  Synchronises with the comm's device. */
int dfx_comm_status(dfx_comm* comm, int* timed_out);

/* The bf16 tensor-core norm's plan for this shape under the context's SM budget
 * (dfx_ctx_set_sm_budget): SMs the W.A^T kernel occupies, SMs given to the Gram / V
 * kernels on the side stream (0 when they run after it), strategy (0 Gram and V beside
 * W.A^T, 1 Gram beside and V after, 2 serial).  DFX_EUNSUPPORTED off the tensor-core path. */
int dfx_norm_plan(dfx_ctx* ctx, dfx_dtype dtype, int64_t d_out, int64_t d_in, int64_t r,
                  int64_t chunk_size, int* u_sms, int* side_sms, int* strategy);

/* 1 when dfx_row_norm takes the tcgen05/TMA path for this (dtype, shape). */
int dfx_norm_uses_tensor_cores(dfx_dtype dtype, int64_t d_out, int64_t d_in, int64_t r);

#ifdef __cplusplus
}
#endif
#endif /* DFX_H */
