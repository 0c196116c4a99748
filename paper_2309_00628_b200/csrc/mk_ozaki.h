// FP64 leaf product on the INT8 tensor cores (Ozaki scheme I), sm_100a.
//
//   P = X * Y  (FP64, row-major, X: m x k, Y: k x n)
//
// Each row i of X is scaled by 2^-e_i (e_i: exponent of the row's largest |x|) and written as
// S signed 7-bit digits, x = 2^e_i * sum_s 2^(-7(s+1)) a_s  (|a_s| <= 127, exact truncation
// digits); each column j of Y likewise with 2^f_j and digits b_t. Then
//
//   P_ij = 2^(e_i + f_j) * sum_{s+t <= S-1} 2^(-7(s+t+2)) * (a_s . b_t)_ij
//
// where every a_s . b_t is an exact int8 x int8 -> int32 tensor-core product (tcgen05.mma
// kind::i8, accumulators in TMEM), pairs on the same anti-diagonal d = s + t share one
// accumulator (still exact: <= S pairs * K * 127^2 < 2^31 for K < 2^31 / (S * 16129)), and the
// S diagonal sums are combined in FP64 in the epilogue (Horner in 2^-7, one rounding per step).
// Dropped digit pairs (s + t >= S) and the truncated remainders bound the error per product term
// by (S + 2) * 2^(-7S) * 2^(e_i + f_j); integer-valued data with <= 7S significant bits relative
// to its row/column maximum is reproduced exactly.
#pragma once
#include <cstddef>
#include <cstdint>
#include <string>

#include <cuda_runtime.h>

namespace mk {

constexpr int kOzMinSlices = 4;
constexpr int kOzMaxSlices = 8;

// Largest K one call accumulates exactly in int32 (per anti-diagonal).
int64_t ozaki_max_k(int slices);

// Device workspace for one product (digit planes of both operands, exponents, status word).
size_t ozaki_workspace_bytes(int64_t m, int64_t n, int64_t k, int slices);

// C (+)= sign * X * Y on `st`. accumulate = 0 overwrites C. Returns 0 or an MK_ERR_* code with
// *err set. Non-finite operand entries make the result NaN in the affected rows/columns
// (they cannot be written as digits); the caller may check `nonfinite_flag` (device int, may be
// null) which is set to 1 when that happens.
int ozaki_product(const double* X, int64_t ldx, const double* Y, int64_t ldy, double* C, int64_t ldc, int64_t m,
                  int64_t n, int64_t k, int slices, int accumulate, double sign, void* ws, size_t ws_bytes,
                  cudaStream_t st, std::string* err);

}  // namespace mk
