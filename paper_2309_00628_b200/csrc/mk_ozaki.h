// FP64 leaf product on the INT8 tensor cores (Ozaki scheme I), sm_100a.
//
//   P = X * Y  (FP64, row-major, X: m x k, Y: k x n)
//
// Each row i of X is scaled by 2^-e_i (e_i: exponent of the row's largest |x|, so |x| < 2^e_i)
// and written as S digit planes, x = 2^(e_i - 7) * sum_s a_s 2^(-8s) with a_0 = floor(128 x 2^-e_i)
// signed in [-128, 127] and a_1.. unsigned in [0, 255] (floor digits of the remainder): 7 + 8(S-1)
// bits, every step exact. Each column j of Y likewise with 2^f_j and digits b_t. Then
//
//   P_ij = 2^(e_i + f_j - 14) * sum_{s+t <= S-1} 2^(-8(s+t)) * (a_s . b_t)_ij
//
// where every a_s . b_t is an exact 8-bit x 8-bit -> int32 tensor-core product (tcgen05.mma
// kind::i8, accumulators in TMEM; Y's signed plane is stored with a +128 offset so every Y plane
// is unsigned, and 128 * rowsum(a_d) is subtracted per diagonal), pairs on the same
// anti-diagonal d = s + t share one accumulator (still exact for K <= ozaki_max_k(S): 4402 at
// S = 8; longer K runs in chunks), and the S diagonal sums are recombined exactly in int64
// (hi / lo) and rounded once to FP64 in the epilogue. Floor truncation and the dropped pairs
// (s + t >= S) bound the error per product term by
// about (S + 2) * 2^(2 - 8S) * 2^(e_i + f_j) -- far below FP64 rounding at S = 8 (63 digit bits);
// integer-valued data is reproduced exactly while it fits the digits (|x| < 2^56 at S = 8).
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

// One destination block of a leaf product (the Kronecker post-addition list of the engine):
// C[row.., col..] (+)= sign * P.
struct OzDest {
  int64_t row, col;
  double sign;
  int32_t accumulate, pad_;
};
constexpr int kOzMaxDests = 16;

// An operand as the signed sum of up to 4 equally shaped blocks of one base (leading dimension
// ld): the pre-additions are formed by the digit-splitting kernels as they load.
constexpr int kOzMaxTerms = 4;
struct OzOperand {
  const double* p[kOzMaxTerms];
  double s[kOzMaxTerms];
  int n;
  int64_t ld;
};

// Row-slab output (fused multi-GPU reduce-scatter): C row R (relative to C's base) lives at
// p[R / rows] + (R % rows) * ldc; every contribution is an atomic add (other ranks add too).
constexpr int kOzMaxSlabs = 8;
struct OzSlabs {
  int n;
  int64_t rows;
  double* p[kOzMaxSlabs];
};

// P = X * Y written to every destination of `d` (stream-ordered workspace from the CUDA pool;
// K beyond ozaki_max_k is processed in chunks). slabs: optional row-slab routing of C.
int ozaki_product_multi(const OzOperand& X, const OzOperand& Y, double* C, int64_t ldc, int64_t m, int64_t n,
                        int64_t k, int slices, const OzDest* d, int nd, cudaStream_t st, std::string* err,
                        const OzSlabs* slabs = nullptr);

// Several leaf products in stream order on `st`; the digit splitting of the next K chunk / item
// runs on a side stream while the current product kernel runs (two pooled workspaces).
struct OzItem {
  OzOperand X, Y;
  double* C;
  int64_t ldc, m, n, k;
  int nd;
  int group;  // items of one group have disjoint destinations and may share one launch
  OzDest d[kOzMaxDests];
};
int ozaki_product_batch(const OzItem* items, int count, int slices, cudaStream_t st, std::string* err);

// C (+)= sign * X * Y on `st` with a caller-owned workspace (ozaki_workspace_bytes).
// accumulate = 0 overwrites C. Returns 0 or an MK_ERR_* code with *err set. A non-finite operand
// entry cannot be written as digits: every result entry in its row (X) or column (Y) is NaN.
int ozaki_product(const double* X, int64_t ldx, const double* Y, int64_t ldy, double* C, int64_t ldc, int64_t m,
                  int64_t n, int64_t k, int slices, int accumulate, double sign, void* ws, size_t ws_bytes,
                  cudaStream_t st, std::string* err);

}  // namespace mk
