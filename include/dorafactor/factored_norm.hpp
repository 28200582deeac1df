// dorafactor/factored_norm.hpp — factored row norm + magnitude scale, B200 drop-in.
//
// Same declarations as the reference proj/include/dorafactor/factored_norm.hpp
// (:11-64).  Every call runs on the GPU through include/dfx.h: inputs are packed
// to their dtype's bits, copied to the device, and the results copied back.
#pragma once

#include <vector>

#include "dorafactor/matrix.hpp"

namespace dorafactor {

struct AdapterPair {
    RealMatrix A;  // [r x d_in]
    RealMatrix B;  // [d_out x r]
    double s = 1.0;
    index_t rank() const { return A.rows(); }
};

// ||W + sBA||^2_row = base_sq + 2s*cross + s^2*ba_sq, fp32 terms, fp64 scales.
struct NormTerms {
    std::vector<float> base_sq;
    std::vector<float> cross;
    std::vector<float> ba_sq;
    double two_s = 0.0;
    double s2 = 0.0;
};

struct Magnitude {
    std::vector<double> values;
    DTypeSpec dtype = DTypeSpec::fp32();
};

NormTerms factored_norm_terms(const RealMatrix& w, const AdapterPair& adapter,
                              const ChunkPlan& plan);
std::vector<float> assemble_norm(const NormTerms& terms);
std::vector<double> factored_row_norm(const RealMatrix& w, const AdapterPair& adapter,
                                      const ChunkPlan& plan);
std::vector<double> magnitude_scale(const Magnitude& m, const std::vector<double>& w_norm,
                                    const DTypeSpec& dtype);

}  // namespace dorafactor
