#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cuda.h>
#include "mk_plan.h"

#define MK_COMBINE_MAX 8

namespace mk {
cudaError_t launch_combine(double* dst, int64_t ldd, const double* const* src, const int64_t* lds,
                           const double* sign, int nsrc, int64_t rows, int64_t cols, cudaStream_t stream);
cudaError_t launch_i64_to_f64(const int64_t* src, int64_t lds, double* dst, int64_t ldd, int64_t rows,
                              int64_t cols, cudaStream_t stream);
cudaError_t launch_f64_to_i64(const double* src, int64_t lds, int64_t* dst, int64_t ldd, int64_t rows,
                              int64_t cols, cudaStream_t stream);
cudaError_t launch_absmax_f64(const double* src, int64_t lds, int64_t rows, int64_t cols,
                              unsigned long long* out, cudaStream_t stream);
cudaError_t launch_absmax_i64(const int64_t* src, int64_t lds, int64_t rows, int64_t cols,
                              unsigned long long* out, cudaStream_t stream);
cudaError_t measure_dmma_peak(double* tflops_out, cudaStream_t st);
cudaError_t launch_fused_product(const CUtensorMap& tmA, const CUtensorMap& tmB, const CUtensorMap& tmC,
                                 const MkGemmArgs& args, const MkProduct& prod, cudaStream_t stream);
int consumer_layout();
}  // namespace mk
