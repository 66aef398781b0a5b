// spgemm_b200/baseline.hpp — the drop-in for the reference's column SpGEMM
// baselines (proj/include/spgemm/baseline.hpp:21-24): same names and
// signatures, computed on the B200 by the column hash kernels of
// pbg_hash.cuh (C-ABI pbg_hash_multiply_begin). Both return C = A·B in CSC
// with sorted columns and duplicates summed; they differ only in summation
// order, so heap_multiply runs the same GPU path. nthreads is ignored.
// Errors: parameter_error (dimension mismatch, flop overflow);
// std::runtime_error on CUDA failure or no GPU.
#pragma once

#include "spgemm_b200/types.hpp"

namespace spgemm {

CscMatrix hash_multiply(const CscMatrix& a, const CscMatrix& b, int nthreads = 0);
CscMatrix heap_multiply(const CscMatrix& a, const CscMatrix& b, int nthreads = 0);

}  // namespace spgemm
