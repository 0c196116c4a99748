#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cuda.h>
#include "mk_plan.h"

#define MK_COMBINE_MAX 8
#define MK_XFORM_MAX 8

// One job of a batched "quadrant transform": dst_j = sum_i coef[j][i] * src_i (all blocks
// rows x cols). Used for a node's operand sums (4 quadrant sources -> up to 8 children, one
// pass) and for hierarchical post-additions (7-8 child products -> 4 parent quadrants).
struct MkXformJob {
  const double* src[MK_XFORM_MAX];
  double* dst[MK_XFORM_MAX];
  int64_t lds[MK_XFORM_MAX];
  int64_t ldd[MK_XFORM_MAX];
  int32_t nsrc, ndst;
  int8_t coef[MK_XFORM_MAX][MK_XFORM_MAX];  // [dst][src] in {-1, 0, 1}
  // destination j written only for rows < clip_rows[j] and columns < clip_cols[j] (0: whole
  // block; a clipped column count is a multiple of the access width) -- the pipelined plan's
  // epilogue writing the caller's unpadded C
  int32_t clip_rows[MK_XFORM_MAX], clip_cols[MK_XFORM_MAX];
};

// One job of the two-level operand transform: a node's operand block (4 x 4 sub-blocks of
// rows x cols, base src, leading dimension lds) -> its grandchildren's operands, grandchild
// (p, p2) into dst[p * np + p2] (leading dimension ldd); nullptr = not written (a view of src,
// or not part of this pass).
#define MK_XFORM2_MAX 64
struct MkXform2Job {
  const double* src;
  int64_t lds;
  double* dst[MK_XFORM2_MAX];
  int64_t ldd;
};

// One job of the two-level post-addition: a node's grandchildren's outputs (src[p * np + p2],
// common leading dimension lds, rows x cols each) -> the node's output block (dst, 4 x 4
// sub-blocks of rows x cols, leading dimension ldd).
// src entries may be nullptr (products outside a grouped pass: contribute nothing); bit
// 4 * q1 + q2 of acc_mask adds the sub-block's previous contents after the sum (a grouped pass
// accumulating onto the earlier passes' partial C).
struct MkXpost2Job {
  const double* src[MK_XFORM2_MAX];
  int64_t lds;
  double* dst;
  int64_t ldd;
  uint32_t acc_mask;
  uint32_t pad_;
};

// One product of a batched leaf launch (device table, 64-byte aligned entries).
struct alignas(64) MkBatchEntry {
  CUtensorMap tmA, tmB, tmC;
  MkProduct prod;
  double* C;
  int64_t ldc;
};

namespace mk {

// Programmatic dependent launch for the one-at-a-time launch chains of the literal schedules
// (MK_OPT_PDL; env MK_PDL=0 disables): sub-wave leaf launches and small two-source additions carry
// cudaLaunchAttributeProgrammaticStreamSerialization (`dep`), so the next kernel of the stream
// is resident, past its shared-memory prologue and parked in pdl_wait() when the previous one
// ends. Larger launches stay plain: a parked grid would hold the SMs that fall idle in a big
// launch's tail, which the side streams' additions use (measured +0.2-0.4 ms on the n = 16384
// literal plans with every launch dependent). Only kernels that call pdl_wait() before their
// first global access may be launched through launch_dep.
bool pdl_enabled();
void set_pdl(bool on);  // mk_set_option(MK_OPT_PDL, ...)
template <typename... KArgs, typename... Args>
inline cudaError_t launch_dep(bool dep, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t stream, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = (dep && pdl_enabled()) ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}
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
// jobs_dev: device array of njobs jobs (identical rows x cols).
cudaError_t launch_xform_batch(const MkXformJob* jobs_dev, int njobs, int64_t rows, int64_t cols, int width,
                               cudaStream_t stream);
cudaError_t measure_dmma_peak(double* tflops_out, cudaStream_t st);
// table: 0 Strassen, 1 Winograd block, 2 Winograd Knuth, 3 Knuth 8-call; side: 0 A, 1 B.
cudaError_t launch_xform2_batch(const MkXform2Job* jobs_dev, int njobs, int table, int side, int64_t rows,
                                int64_t cols, int width, cudaStream_t stream);
int xform2_table_coef(int table, int side, int p, int q);
cudaError_t launch_xpost2_batch(const MkXpost2Job* jobs_dev, int njobs, int table, int64_t rows, int64_t cols,
                                int width, cudaStream_t stream);
int xpost2_table_coef(int table, int q, int p);
// One-level operand transform: a node's quadrants -> its children's operands (MkXform2Job, dst[0..np-1]).
cudaError_t launch_xform1_batch(const MkXform2Job* jobs_dev, int njobs, int table, int side, int64_t rows,
                                int64_t cols, int width, cudaStream_t stream);
// One-level post-addition: a node's quadrants from its children's outputs (MkXpost2Job, src[0..np-1]).
cudaError_t launch_xpost1_batch(const MkXpost2Job* jobs_dev, int njobs, int table, int64_t rows, int64_t cols,
                                int width, cudaStream_t stream);
// dst (rows_d x cols_d) = src (rows_s x cols_s) zero-padded to the right and below, one pass.
cudaError_t launch_pad_copy(double* dst, int64_t ldd, int64_t rows_d, int64_t cols_d, const double* src, int64_t lds,
                            int64_t rows_s, int64_t cols_s, cudaStream_t stream);
// One side-work task (mk_plan.h) as a stand-alone launch (a leaf launch that cannot carry it).
cudaError_t launch_side_task(const MkSideTask& task, cudaStream_t stream);
cudaError_t launch_fused_product(const CUtensorMap& tmA, const CUtensorMap& tmB, const CUtensorMap& tmC,
                                 const MkGemmArgs& args, const MkProduct& prod, cudaStream_t stream);
int consumer_layout();
bool persistent_enabled();  // the persistent leaf kernel (env MK_PERSISTENT=0 disables it)
// Tile width (64 or 128) the persistent kernel will use for a launch, and the row height of the
// TMA epilogue's C boxes that launch needs (32 for narrow tiles and the 16-warp layout, else 64).
int persistent_tile_n(int64_t tiles_m, int64_t N, int nprod);
int epilogue_box_rows(int64_t M, int64_t N, int nprod, bool single_terms);

// Launch `nprod` single-term products of identical M x N x K (entries already in device memory).
cudaError_t launch_product_batch(const MkBatchEntry* entries_dev, int nprod, const MkGemmArgs& args,
                                 cudaStream_t stream);
}  // namespace mk
