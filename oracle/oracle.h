/*
 * oracle.h — CPU restatement of the reference DoRA hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_2603_22276_b200/,
 * include/dfx.h, the C++ drop-in) links or calls this code.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load it, and only as the checker or the timed CPU baseline.
 *
 * Every function restates the arithmetic of the reference C++ implementation
 * in /root/reference/proj (cited per function in oracle.c) on packed fp32
 * buffers.  Element values are always exactly representable in the tagged
 * dtype, exactly like the reference's RealMatrix (matrix.hpp:13-16), so the
 * widening `static_cast<float>(double)` of the reference is the identity here.
 *
 * Parity pin: tests/test_oracle.py checks every function against the
 * reference itself (oracle/_ref, compiled from the reference sources by
 * oracle/Makefile) and against the committed golden vectors in tests/golden/.
 */
#ifndef DFX_ORACLE_H
#define DFX_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* dtype codes shared with include/dfx.h: 0 fp32, 1 bf16, 2 fp16, 3 fp64 */
enum { ORC_F32 = 0, ORC_BF16 = 1, ORC_F16 = 2, ORC_F64 = 3 };

double orc_round_to_dtype(double x, int dtype);
double orc_norm_eps(int dtype);

/* plan_chunks (matrix.cpp:28-51). Returns 0, or -1 when the reference throws. */
int orc_plan_chunks(size_t d_out, size_t d_in, uint64_t budget, size_t* chunk_size,
                    size_t* num_chunks);

/* factored_norm_terms (factored_norm.cpp:27-120). Returns 0, or -1 on invalid args. */
int orc_norm_terms(const float* w, const float* a, const float* b, size_t d_out, size_t d_in,
                   size_t r, double s, size_t chunk_size, float* base_sq, float* cross,
                   float* ba_sq);

/* assemble_norm (factored_norm.cpp:122-136). */
void orc_assemble(const float* base_sq, const float* cross, const float* ba_sq, double two_s,
                  double s2, size_t n, float* out);

/* factored_row_norm (factored_norm.cpp:204-217) for fp32/bf16/fp16 weights;
 * out[j] is the dtype-rounded norm (exact in float). */
int orc_row_norm(int dtype, const float* w, const float* a, const float* b, size_t d_out,
                 size_t d_in, size_t r, double s, size_t chunk_size, float* out);

/* magnitude_scale (factored_norm.cpp:219-240), non-fp64 branch. m is fp64 like
 * Magnitude::values; w_norm holds dtype-representable values. */
void orc_magnitude_scale(int dtype, const double* m, const float* w_norm, size_t n, float* g);

/* stable_compose / fused_compose / dual_output_compose (compose.cpp:19-45, 70-152).
 * inner may be NULL. */
void orc_compose_fwd(int dtype, const float* base, const float* lora, const float* g, double s,
                     size_t rows, size_t d_out, float* delta, float* inner);

/* naive_compose (compose.cpp:47-68) — the stability lab's counterexample. */
void orc_working_matmul_nt(int dtype, const float* a, const float* bt, size_t m, size_t n,
                           size_t k, float* out);
void orc_residual(int dtype, const float* base, const float* delta, const float* bias,
                  size_t rows, size_t d_out, float* y);
void orc_naive_compose(int dtype, const float* base, const float* lora, const float* g, double s,
                       size_t rows, size_t d_out, float* delta);

/* compose_backward (compose.cpp:154-201). inner / w_norm / d_mag may be NULL
 * when mag_grad is 0. */
int orc_compose_bwd(int dtype, const float* dy, const float* g, double s, const float* inner,
                    const float* w_norm, size_t rows, size_t d_out, int mag_grad, float* d_lora,
                    float* d_base, float* d_mag);

/* dense_row_norm_f64 (reference.cpp:46-50): fp64 ground truth. */
void orc_dense_row_norm_f64(const float* w, const float* a, const float* b, size_t d_out,
                            size_t d_in, size_t r, double s, double* out);

/* Fixtures (matrix.cpp:82-148): mt19937_64 + Box-Muller, values rounded to dtype. */
uint64_t orc_derive_seed(uint64_t base, uint64_t index);
void orc_seeded_gaussian(size_t n, uint64_t seed, int dtype, float* out);
void orc_gaussian_fixture(size_t n, double mean, double stddev, uint64_t seed, int dtype,
                          float* out);
void orc_gaussian_vector(size_t n, double mean, double stddev, uint64_t seed, double* out);

#ifdef __cplusplus
}
#endif
#endif
