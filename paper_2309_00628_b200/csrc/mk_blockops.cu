// K4: HBM-bound block kernels used around the fused products.
//
//   combine   dst = sum_t s_t * src_t over an h x w block (up to 8 strided sources);
//             dst may alias a source exactly (reference core.py:153-169 block_add allows it).
//             Used for materialised outer-level operand sums, literal two-temp / in-place
//             schedule steps (schedules.py:62-112), post-adds, and pad/unpad copies.
//   i64->f64 / f64->i64 conversions for integer operands (reference tests use int64,
//             conftest.py:29-30), and an |x|max reduction for the exactness guard.
// Roofline: every kernel here is bandwidth-bound (FP64: 8 B per element per stream).
#include <cuda_runtime.h>
#include <atomic>
#include <cstdint>
#include <cstdlib>
#include "mk_blockops.h"
#include "mk_device.cuh"
#include "mk_xform.cuh"

namespace mk {

static std::atomic<int> g_pdl{-1};
bool pdl_enabled() {
  if (g_pdl < 0) {
    const char* e = getenv("MK_PDL");
    g_pdl = (e && e[0] == '0') ? 0 : 1;
  }
  return g_pdl == 1;
}
void set_pdl(bool on) { g_pdl = on ? 1 : 0; }

static int64_t pdl_max_elems() {
  const char* e = getenv("MK_PDL_MAX_LOG2");  // study knob: largest addition launched as a dependent
  const int v = e ? atoi(e) : 22;
  return (int64_t)1 << (v < 0 ? 0 : v > 40 ? 40 : v);
}
static const int64_t kPdlMaxElems = pdl_max_elems();

struct CombineArgs {
  double* dst;
  int64_t ldd;
  const double* src[MK_COMBINE_MAX];
  int64_t lds[MK_COMBINE_MAX];
  double sign[MK_COMBINE_MAX];
  int nsrc;
  int64_t rows, cols;
};

// Each thread handles 2 consecutive columns (16 B) when vectorisable.
template <bool VEC>
__global__ void combine_kernel(const __grid_constant__ CombineArgs a) {
  pdl_trigger();
  pdl_wait();
  const int64_t cols_v = VEC ? (a.cols >> 1) : a.cols;
  const int64_t total = a.rows * cols_v;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx / cols_v;
    const int64_t c = (idx - r * cols_v) * (VEC ? 2 : 1);
    if (VEC) {
      double2 acc = make_double2(0.0, 0.0);
      for (int t = 0; t < a.nsrc; ++t) {
        const double2 v = *reinterpret_cast<const double2*>(a.src[t] + r * a.lds[t] + c);  // dst may be a source
        acc.x = fma(a.sign[t], v.x, acc.x);
        acc.y = fma(a.sign[t], v.y, acc.y);
      }
      *reinterpret_cast<double2*>(a.dst + r * a.ldd + c) = acc;
    } else {
      double acc = 0.0;
      for (int t = 0; t < a.nsrc; ++t) acc = fma(a.sign[t], a.src[t][r * a.lds[t] + c], acc);
      a.dst[r * a.ldd + c] = acc;
    }
  }
}

// Two-source sums (every step of the literal schedules is X = Y +- Z, schedules.py:62-112). The
// generic kernel keeps two 16-byte loads per thread in flight, which holds a lone SM to ~57 GB/s
// -- and a handful of SMs is what an addition gets when it runs beside a one-at-a-time leaf launch
// (128 tiles on 148 SMs). Here a thread issues 2 x U loads before its first use. Same arithmetic
// as combine_kernel (fma from zero in source order): bit-identical. dst may alias a source
// exactly: a thread reads its elements before it writes them.
template <int U>
__global__ void __launch_bounds__(256) combine2_kernel(const __grid_constant__ CombineArgs a) {
  pdl_trigger();  // short kernel: the next launch's CTAs may queue up behind this one's at once
  pdl_wait();
  const uint32_t cv = (uint32_t)(a.cols >> 1);
  const uint32_t total = (uint32_t)a.rows * cv;  // < 2^31 (checked by the launcher)
  const double s0 = a.sign[0], s1 = a.sign[1];
  for (uint32_t base = blockIdx.x * (256u * U) + threadIdx.x; base < total; base += gridDim.x * (256u * U)) {
    double2 x[U], y[U];
    int64_t off[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const uint32_t idx = base + (uint32_t)k * 256u;
      if (idx < total) {
        const uint32_t r = idx / cv;
        const int64_t c = (int64_t)(idx - r * cv) * 2;
        // plain loads, not ld.global.nc: dst may be one of the sources (Table 3 stores S1 over A21)
        x[k] = *reinterpret_cast<const double2*>(a.src[0] + (int64_t)r * a.lds[0] + c);
        y[k] = *reinterpret_cast<const double2*>(a.src[1] + (int64_t)r * a.lds[1] + c);
        off[k] = (int64_t)r * a.ldd + c;
      }
    }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const uint32_t idx = base + (uint32_t)k * 256u;
      if (idx < total) {
        double2 acc;
        acc.x = fma(s1, y[k].x, fma(s0, x[k].x, 0.0));
        acc.y = fma(s1, y[k].y, fma(s0, x[k].y, 0.0));
        *reinterpret_cast<double2*>(a.dst + off[k]) = acc;
      }
    }
  }
}

static int grid_for(int64_t work, int threads) {
  int64_t blocks = (work + threads - 1) / threads;
  const int64_t cap = 148 * 16;  // 16 resident 256-thread CTAs per SM
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  return (int)blocks;
}

cudaError_t launch_combine(double* dst, int64_t ldd, const double* const* src, const int64_t* lds,
                           const double* sign, int nsrc, int64_t rows, int64_t cols, cudaStream_t stream) {
  if (rows <= 0 || cols <= 0) return cudaSuccess;
  if (nsrc < 0 || nsrc > MK_COMBINE_MAX) return cudaErrorInvalidValue;
  CombineArgs a{};
  a.dst = dst;
  a.ldd = ldd;
  a.nsrc = nsrc;
  a.rows = rows;
  a.cols = cols;
  bool vec = (cols % 2 == 0) && (ldd % 2 == 0) && ((uintptr_t)dst % 16 == 0);
  for (int t = 0; t < nsrc; ++t) {
    a.src[t] = src[t];
    a.lds[t] = lds[t];
    a.sign[t] = sign[t];
    vec = vec && (lds[t] % 2 == 0) && ((uintptr_t)src[t] % 16 == 0);
  }
  const int threads = 256;
  const bool dep = rows * cols <= kPdlMaxElems;  // see launch_dep
  if (vec && nsrc == 2 && rows * (cols / 2) < ((int64_t)1 << 31)) {
    constexpr int U = 4;
    const int64_t work = rows * (cols / 2);
    int64_t blocks = (work + threads * U - 1) / (threads * U);
    if (blocks > 148 * 8) blocks = 148 * 8;
    return launch_dep(dep, combine2_kernel<U>, dim3((unsigned)blocks), dim3(threads), 0, stream, a);
  } else if (vec)
    return launch_dep(dep, combine_kernel<true>, dim3(grid_for(rows * (cols / 2), threads)), dim3(threads), 0, stream, a);
  return launch_dep(dep, combine_kernel<false>, dim3(grid_for(rows * cols, threads)), dim3(threads), 0, stream, a);
}

// Batched quadrant transform: blockIdx.y = job, grid-stride over the job's elements. Each
// thread reads every source once (W consecutive doubles: 8, 16 or 32-byte accesses) and
// writes every destination.
template <int W>
__global__ void __launch_bounds__(256) xform_kernel(const MkXformJob* __restrict__ jobs, int64_t rows, int64_t cols) {
  const MkXformJob& jb = jobs[blockIdx.y];
  const int64_t cv = cols / W;
  // rows x cv < 2^32 for every block the planner forms (checked by the launcher)
  const uint32_t total = (uint32_t)(rows * cv), ucv = (uint32_t)cv;
  for (uint32_t idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += gridDim.x * blockDim.x) {
    const uint32_t r = idx / ucv;
    xform_elem<W>(jb, r, (int64_t)(idx - r * ucv) * W);
  }
}

cudaError_t launch_xform_batch(const MkXformJob* jobs_dev, int njobs, int64_t rows, int64_t cols, int width,
                               cudaStream_t stream) {
  if (njobs <= 0 || rows <= 0 || cols <= 0) return cudaSuccess;
  if (width != 4 && width != 2) width = 1;
  const int64_t work = rows * (cols / width);
  if (work >= (int64_t)1 << 32) return cudaErrorInvalidValue;
  int64_t bx = (work + 255) / 256;
#ifndef MK_XFORM_CTAS_PER_SM
#define MK_XFORM_CTAS_PER_SM 32
#endif
  const int64_t cap = (148 * MK_XFORM_CTAS_PER_SM + njobs - 1) / njobs;  // resident CTAs per SM, all jobs
  if (bx > cap) bx = cap;
  if (bx < 1) bx = 1;
  for (int j0 = 0; j0 < njobs; j0 += 65535) {
    const int nj = njobs - j0 < 65535 ? njobs - j0 : 65535;
    dim3 grid((unsigned)bx, (unsigned)nj);
    if (width == 4)
      xform_kernel<4><<<grid, 256, 0, stream>>>(jobs_dev + j0, rows, cols);
    else if (width == 2)
      xform_kernel<2><<<grid, 256, 0, stream>>>(jobs_dev + j0, rows, cols);
    else
      xform_kernel<1><<<grid, 256, 0, stream>>>(jobs_dev + j0, rows, cols);
  }
  return cudaGetLastError();
}

// ---- two-level operand transform (breadth-first plan, K2'') ---------------------------------
// One job = one recursion node's operand block X (4 x 4 sub-blocks of rows x cols: sub-block
// (q1, q2) is sub-quadrant q2 of quadrant q1) -> all its grandchildren's operands
//     G(p, p2) = sum_q2 c[p2][q2] * ( sum_q1 c[p][q1] * X(q1, q2) )
// in one pass: the children's sums T(p, .) stay in registers, so two depths of the recursion
// cost one read of X and one write of the grandchildren instead of writing and re-reading the
// children. The coefficient tables are compile-time constants (every zero term is skipped at
// compile time, so the kernel stays memory-bound; the round-1 runtime-table version was
// instruction-bound); sums run in quadrant order from zero, exactly as two one-level passes
// would compute them (bit-identical results). Tables: reference kernels.py:66-160.
int xform2_table_coef(int tab, int side, int p, int q) {
  switch (tab * 2 + side) {
    case 0: return X2Tab<0, 0>::cf(p, q);
    case 1: return X2Tab<0, 1>::cf(p, q);
    case 2: return X2Tab<1, 0>::cf(p, q);
    case 3: return X2Tab<1, 1>::cf(p, q);
    case 4: return X2Tab<2, 0>::cf(p, q);
    case 5: return X2Tab<2, 1>::cf(p, q);
    case 6: return X2Tab<3, 0>::cf(p, q);
    default: return X2Tab<3, 1>::cf(p, q);
  }
}

template <int TAB, int SIDE, int W>
__global__ void __launch_bounds__(256) xform2_kernel(const MkXform2Job* __restrict__ jobs, int64_t rows,
                                                     int64_t cols) {
  constexpr int NP = X2Tab<TAB, SIDE>::np;
  __shared__ double* dst_sh[MK_XFORM2_MAX];
  const MkXform2Job& jb = jobs[blockIdx.y];
  if (threadIdx.x < NP * NP) dst_sh[threadIdx.x] = jb.dst[threadIdx.x];
  __syncthreads();
  const int64_t cv = cols / W;
  const uint32_t total = (uint32_t)(rows * cv), ucv = (uint32_t)cv;
  for (uint32_t idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += gridDim.x * blockDim.x) {
    const uint32_t r = idx / ucv;
    xform2_elem<TAB, SIDE, W>(jb.src, jb.lds, static_cast<double* const*>(dst_sh), jb.ldd, rows, cols, r,
                              (int64_t)(idx - r * ucv) * W);
  }
}

int xpost2_table_coef(int tab, int q, int p) {
  switch (tab) {
    case 0: return XCTab<0>::cf(q, p);
    case 1: return XCTab<1>::cf(q, p);
    case 2: return XCTab<2>::cf(q, p);
    default: return XCTab<3>::cf(q, p);
  }
}

template <int TAB, int W>
__global__ void __launch_bounds__(256) xpost2_kernel(const MkXpost2Job* __restrict__ jobs, int64_t rows,
                                                     int64_t cols) {
  constexpr int NP = XCTab<TAB>::np;
  __shared__ const double* src_sh[MK_XFORM2_MAX];
  const MkXpost2Job& jb = jobs[blockIdx.y];
  if (threadIdx.x < NP * NP) src_sh[threadIdx.x] = jb.src[threadIdx.x];
  __syncthreads();
  const int64_t cv = cols / W;
  const uint32_t total = (uint32_t)(rows * cv), ucv = (uint32_t)cv;
  for (uint32_t idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += gridDim.x * blockDim.x) {
    const uint32_t r = idx / ucv;
    xpost2_elem<TAB, W>(static_cast<const double* const*>(src_sh), jb.lds, jb.dst, jb.ldd, jb.acc_mask, rows, cols, r,
                        (int64_t)(idx - r * ucv) * W);
  }
}

template <int TAB, int SIDE, int W>
__global__ void __launch_bounds__(256) xform1_kernel(const MkXform2Job* __restrict__ jobs, int64_t rows,
                                                     int64_t cols) {
  constexpr int NP = X2Tab<TAB, SIDE>::np;
  __shared__ double* dst_sh[MK_XFORM2_MAX];
  const MkXform2Job& jb = jobs[blockIdx.y];
  if (threadIdx.x < NP) dst_sh[threadIdx.x] = jb.dst[threadIdx.x];
  __syncthreads();
  const int64_t cv = cols / W;
  const uint32_t total = (uint32_t)(rows * cv), ucv = (uint32_t)cv;
  for (uint32_t idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += gridDim.x * blockDim.x) {
    const uint32_t r = idx / ucv;
    xform1_elem<TAB, SIDE, W>(jb.src, jb.lds, static_cast<double* const*>(dst_sh), jb.ldd, rows, cols, r,
                              (int64_t)(idx - r * ucv) * W);
  }
}

cudaError_t launch_xform1_batch(const MkXform2Job* jobs_dev, int njobs, int table, int side, int64_t rows,
                                int64_t cols, int width, cudaStream_t stream) {
  if (njobs <= 0 || rows <= 0 || cols <= 0) return cudaSuccess;
  if (table < 0 || table > 3 || side < 0 || side > 1) return cudaErrorInvalidValue;
  if (width != 2) width = 1;
  const int64_t work = rows * (cols / width);
  if (work >= (int64_t)1 << 32) return cudaErrorInvalidValue;
  int64_t bx = (work + 255) / 256;
  const int64_t cap = (148 * 16 + njobs - 1) / njobs;
  if (bx > cap) bx = cap;
  if (bx < 1) bx = 1;
  for (int j0 = 0; j0 < njobs; j0 += 65535) {
    const int nj = njobs - j0 < 65535 ? njobs - j0 : 65535;
    dim3 grid((unsigned)bx, (unsigned)nj);
    const MkXform2Job* jb = jobs_dev + j0;
#define MK_XF1(T, S)                                                         \
  if (width == 2)                                                            \
    xform1_kernel<T, S, 2><<<grid, 256, 0, stream>>>(jb, rows, cols);       \
  else                                                                       \
    xform1_kernel<T, S, 1><<<grid, 256, 0, stream>>>(jb, rows, cols);
    switch (table * 2 + side) {
      case 0: MK_XF1(0, 0) break;
      case 1: MK_XF1(0, 1) break;
      case 2: MK_XF1(1, 0) break;
      case 3: MK_XF1(1, 1) break;
      case 4: MK_XF1(2, 0) break;
      case 5: MK_XF1(2, 1) break;
      case 6: MK_XF1(3, 0) break;
      default: MK_XF1(3, 1) break;
    }
#undef MK_XF1
  }
  return cudaGetLastError();
}

template <int TAB, int W>
__global__ void __launch_bounds__(256) xpost1_kernel(const MkXpost2Job* __restrict__ jobs, int64_t rows,
                                                     int64_t cols) {
  constexpr int NP = XCTab<TAB>::np;
  __shared__ const double* src_sh[MK_XFORM2_MAX];
  const MkXpost2Job& jb = jobs[blockIdx.y];
  if (threadIdx.x < NP) src_sh[threadIdx.x] = jb.src[threadIdx.x];
  __syncthreads();
  const int64_t cv = cols / W;
  const uint32_t total = (uint32_t)(rows * cv), ucv = (uint32_t)cv;
  for (uint32_t idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += gridDim.x * blockDim.x) {
    const uint32_t r = idx / ucv;
    xpost1_elem<TAB, W>(static_cast<const double* const*>(src_sh), jb.lds, jb.dst, jb.ldd, jb.acc_mask, rows, cols, r,
                        (int64_t)(idx - r * ucv) * W);
  }
}

cudaError_t launch_xpost1_batch(const MkXpost2Job* jobs_dev, int njobs, int table, int64_t rows, int64_t cols,
                                int width, cudaStream_t stream) {
  if (njobs <= 0 || rows <= 0 || cols <= 0) return cudaSuccess;
  if (table < 0 || table > 3) return cudaErrorInvalidValue;
  if (width != 2) width = 1;
  const int64_t work = rows * (cols / width);
  if (work >= (int64_t)1 << 32) return cudaErrorInvalidValue;
  int64_t bx = (work + 255) / 256;
  const int64_t cap = (148 * 16 + njobs - 1) / njobs;
  if (bx > cap) bx = cap;
  if (bx < 1) bx = 1;
  for (int j0 = 0; j0 < njobs; j0 += 65535) {
    const int nj = njobs - j0 < 65535 ? njobs - j0 : 65535;
    dim3 grid((unsigned)bx, (unsigned)nj);
    const MkXpost2Job* jb = jobs_dev + j0;
#define MK_XP1(T)                                                            \
  if (width == 2)                                                            \
    xpost1_kernel<T, 2><<<grid, 256, 0, stream>>>(jb, rows, cols);          \
  else                                                                       \
    xpost1_kernel<T, 1><<<grid, 256, 0, stream>>>(jb, rows, cols);
    switch (table) {
      case 0: MK_XP1(0) break;
      case 1: MK_XP1(1) break;
      case 2: MK_XP1(2) break;
      default: MK_XP1(3) break;
    }
#undef MK_XP1
  }
  return cudaGetLastError();
}

template <int TAB>
static void launch_xpost2_t(dim3 grid, const MkXpost2Job* jobs, int64_t rows, int64_t cols, int width,
                            cudaStream_t stream) {
  if (width == 2)
    xpost2_kernel<TAB, 2><<<grid, 256, 0, stream>>>(jobs, rows, cols);
  else
    xpost2_kernel<TAB, 1><<<grid, 256, 0, stream>>>(jobs, rows, cols);
}

cudaError_t launch_xpost2_batch(const MkXpost2Job* jobs_dev, int njobs, int table, int64_t rows, int64_t cols,
                                int width, cudaStream_t stream) {
  if (njobs <= 0 || rows <= 0 || cols <= 0) return cudaSuccess;
  if (table < 0 || table > 3) return cudaErrorInvalidValue;
  if (width != 2) width = 1;
  const int64_t work = rows * (cols / width);
  if (work >= (int64_t)1 << 32) return cudaErrorInvalidValue;
  int64_t bx = (work + 255) / 256;
  const int64_t cap = (148 * 16 + njobs - 1) / njobs;
  if (bx > cap) bx = cap;
  if (bx < 1) bx = 1;
  for (int j0 = 0; j0 < njobs; j0 += 65535) {
    const int nj = njobs - j0 < 65535 ? njobs - j0 : 65535;
    dim3 grid((unsigned)bx, (unsigned)nj);
    const MkXpost2Job* jb = jobs_dev + j0;
    switch (table) {
      case 0: launch_xpost2_t<0>(grid, jb, rows, cols, width, stream); break;
      case 1: launch_xpost2_t<1>(grid, jb, rows, cols, width, stream); break;
      case 2: launch_xpost2_t<2>(grid, jb, rows, cols, width, stream); break;
      default: launch_xpost2_t<3>(grid, jb, rows, cols, width, stream); break;
    }
  }
  return cudaGetLastError();
}

template <int TAB, int SIDE>
static void launch_xform2_t(dim3 grid, const MkXform2Job* jobs, int64_t rows, int64_t cols, int width,
                            cudaStream_t stream) {
  if (width == 4)
    xform2_kernel<TAB, SIDE, 4><<<grid, 256, 0, stream>>>(jobs, rows, cols);
  else if (width == 2)
    xform2_kernel<TAB, SIDE, 2><<<grid, 256, 0, stream>>>(jobs, rows, cols);
  else
    xform2_kernel<TAB, SIDE, 1><<<grid, 256, 0, stream>>>(jobs, rows, cols);
}

cudaError_t launch_xform2_batch(const MkXform2Job* jobs_dev, int njobs, int table, int side, int64_t rows,
                                int64_t cols, int width, cudaStream_t stream) {
  if (njobs <= 0 || rows <= 0 || cols <= 0) return cudaSuccess;
  if (table < 0 || table > 3 || side < 0 || side > 1) return cudaErrorInvalidValue;
  if (width != 4 && width != 2) width = 1;
  const int64_t work = rows * (cols / width);
  if (work >= (int64_t)1 << 32) return cudaErrorInvalidValue;
  int64_t bx = (work + 255) / 256;
  const int64_t cap = (148 * 16 + njobs - 1) / njobs;
  if (bx > cap) bx = cap;
  if (bx < 1) bx = 1;
  for (int j0 = 0; j0 < njobs; j0 += 65535) {
    const int nj = njobs - j0 < 65535 ? njobs - j0 : 65535;
    dim3 grid((unsigned)bx, (unsigned)nj);
    const MkXform2Job* jb = jobs_dev + j0;
    switch (table * 2 + side) {
      case 0: launch_xform2_t<0, 0>(grid, jb, rows, cols, width, stream); break;
      case 1: launch_xform2_t<0, 1>(grid, jb, rows, cols, width, stream); break;
      case 2: launch_xform2_t<1, 0>(grid, jb, rows, cols, width, stream); break;
      case 3: launch_xform2_t<1, 1>(grid, jb, rows, cols, width, stream); break;
      case 4: launch_xform2_t<2, 0>(grid, jb, rows, cols, width, stream); break;
      case 5: launch_xform2_t<2, 1>(grid, jb, rows, cols, width, stream); break;
      case 6: launch_xform2_t<3, 0>(grid, jb, rows, cols, width, stream); break;
      default: launch_xform2_t<3, 1>(grid, jb, rows, cols, width, stream); break;
    }
  }
  return cudaGetLastError();
}

// Padded copy: dst (rows_d x cols_d) = src (rows_s x cols_s) with zeros to the right and below
// -- one pass over dst instead of a memset followed by a copy (rectangular driver, hybrid.py:130-146).
template <bool VEC>
__global__ void pad_copy_kernel(double* __restrict__ dst, int64_t ldd, int64_t rows_d, int64_t cols_d,
                                const double* __restrict__ src, int64_t lds, int64_t rows_s, int64_t cols_s) {
  const int64_t cv = VEC ? cols_d / 2 : cols_d;
  const int64_t total = rows_d * cv;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx / cv;
    const int64_t c = (idx - r * cv) * (VEC ? 2 : 1);
    if (VEC) {
      double2 v = make_double2(0.0, 0.0);
      if (r < rows_s) {
        if (c + 1 < cols_s)
          v = __ldg(reinterpret_cast<const double2*>(src + r * lds + c));
        else if (c < cols_s)
          v.x = __ldg(src + r * lds + c);
      }
      *reinterpret_cast<double2*>(dst + r * ldd + c) = v;
    } else {
      dst[r * ldd + c] = (r < rows_s && c < cols_s) ? __ldg(src + r * lds + c) : 0.0;
    }
  }
}

cudaError_t launch_pad_copy(double* dst, int64_t ldd, int64_t rows_d, int64_t cols_d, const double* src, int64_t lds,
                            int64_t rows_s, int64_t cols_s, cudaStream_t stream) {
  if (rows_d <= 0 || cols_d <= 0) return cudaSuccess;
  const bool vec = cols_d % 2 == 0 && ldd % 2 == 0 && lds % 2 == 0 && (uintptr_t)dst % 16 == 0 &&
                   (uintptr_t)src % 16 == 0;
  if (vec)
    pad_copy_kernel<true><<<grid_for(rows_d * (cols_d / 2), 256), 256, 0, stream>>>(dst, ldd, rows_d, cols_d, src, lds,
                                                                                   rows_s, cols_s);
  else
    pad_copy_kernel<false><<<grid_for(rows_d * cols_d, 256), 256, 0, stream>>>(dst, ldd, rows_d, cols_d, src, lds,
                                                                              rows_s, cols_s);
  return cudaGetLastError();
}

cudaError_t launch_side_task(const MkSideTask& t, cudaStream_t stream) {
  switch (t.kind) {
    case 1: return launch_xform_batch(static_cast<const MkXformJob*>(t.jobs), t.njobs, t.rows, t.cols, t.width, stream);
    case 2:
      return launch_xform2_batch(static_cast<const MkXform2Job*>(t.jobs), t.njobs, t.table, t.side, t.rows, t.cols,
                                 t.width, stream);
    case 3:
      return launch_xpost2_batch(static_cast<const MkXpost2Job*>(t.jobs), t.njobs, t.table, t.rows, t.cols, t.width,
                                 stream);
    case 5:
      return launch_xform1_batch(static_cast<const MkXform2Job*>(t.jobs), t.njobs, t.table, t.side, t.rows, t.cols,
                                 t.width, stream);
    case 4:
      return launch_xpost1_batch(static_cast<const MkXpost2Job*>(t.jobs), t.njobs, t.table, t.rows, t.cols, t.width,
                                 stream);
    default: return cudaErrorInvalidValue;
  }
}

__global__ void i64_to_f64_kernel(const int64_t* src, int64_t lds, double* dst, int64_t ldd, int64_t rows,
                                  int64_t cols) {
  const int64_t total = rows * cols;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx / cols, c = idx - r * cols;
    dst[r * ldd + c] = (double)src[r * lds + c];
  }
}

__global__ void f64_to_i64_kernel(const double* src, int64_t lds, int64_t* dst, int64_t ldd, int64_t rows,
                                  int64_t cols) {
  const int64_t total = rows * cols;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx / cols, c = idx - r * cols;
    dst[r * ldd + c] = __double2ll_rn(src[r * lds + c]);
  }
}

cudaError_t launch_i64_to_f64(const int64_t* src, int64_t lds, double* dst, int64_t ldd, int64_t rows,
                              int64_t cols, cudaStream_t stream) {
  if (rows <= 0 || cols <= 0) return cudaSuccess;
  i64_to_f64_kernel<<<grid_for(rows * cols, 256), 256, 0, stream>>>(src, lds, dst, ldd, rows, cols);
  return cudaGetLastError();
}

cudaError_t launch_f64_to_i64(const double* src, int64_t lds, int64_t* dst, int64_t ldd, int64_t rows,
                              int64_t cols, cudaStream_t stream) {
  if (rows <= 0 || cols <= 0) return cudaSuccess;
  f64_to_i64_kernel<<<grid_for(rows * cols, 256), 256, 0, stream>>>(src, lds, dst, ldd, rows, cols);
  return cudaGetLastError();
}

// max |x| over a strided block; result (as the bit pattern of a non-negative double,
// which orders like an unsigned integer) is atomically max-ed into *out.
template <typename T>
__global__ void absmax_kernel(const T* src, int64_t lds, int64_t rows, int64_t cols,
                              unsigned long long* out) {
  double m = 0.0;
  const int64_t total = rows * cols;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx / cols, c = idx - r * cols;
    const double v = fabs((double)src[r * lds + c]);
    m = (v > m || v != v) ? v : m;  // NaN propagates
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double x = __shfl_xor_sync(0xffffffffu, m, o);
    m = (x > m || x != x) ? x : m;
  }
  if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(m));
}

cudaError_t launch_absmax_f64(const double* src, int64_t lds, int64_t rows, int64_t cols,
                              unsigned long long* out, cudaStream_t stream) {
  if (rows <= 0 || cols <= 0) return cudaSuccess;
  absmax_kernel<double><<<grid_for(rows * cols, 256), 256, 0, stream>>>(src, lds, rows, cols, out);
  return cudaGetLastError();
}

cudaError_t launch_absmax_i64(const int64_t* src, int64_t lds, int64_t rows, int64_t cols,
                              unsigned long long* out, cudaStream_t stream) {
  if (rows <= 0 || cols <= 0) return cudaSuccess;
  absmax_kernel<int64_t><<<grid_for(rows * cols, 256), 256, 0, stream>>>(src, lds, rows, cols, out);
  return cudaGetLastError();
}

}  // namespace mk
