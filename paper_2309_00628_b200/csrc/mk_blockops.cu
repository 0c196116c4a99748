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
#include <cstdint>
#include "mk_blockops.h"

namespace mk {

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
  const int64_t cols_v = VEC ? (a.cols >> 1) : a.cols;
  const int64_t total = a.rows * cols_v;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx / cols_v;
    const int64_t c = (idx - r * cols_v) * (VEC ? 2 : 1);
    if (VEC) {
      double2 acc = make_double2(0.0, 0.0);
      for (int t = 0; t < a.nsrc; ++t) {
        const double2 v = __ldg(reinterpret_cast<const double2*>(a.src[t] + r * a.lds[t] + c));
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
  if (vec)
    combine_kernel<true><<<grid_for(rows * (cols / 2), threads), threads, 0, stream>>>(a);
  else
    combine_kernel<false><<<grid_for(rows * cols, threads), threads, 0, stream>>>(a);
  return cudaGetLastError();
}

// Batched quadrant transform: blockIdx.y = job, grid-stride over the job's elements. Each
// thread reads every source once (W consecutive doubles: 8, 16 or 32-byte accesses) and
// writes every destination.
template <int W>
struct Vec {
  double v[W];
};
template <int W>
__device__ __forceinline__ Vec<W> ld_vec(const double* p) {
  Vec<W> r;
  if constexpr (W == 4) {
    asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(r.v[0]), "=d"(r.v[1]), "=d"(r.v[2]), "=d"(r.v[3])
                 : "l"(p));
  } else if constexpr (W == 2) {
    const double2 t = __ldg(reinterpret_cast<const double2*>(p));
    r.v[0] = t.x;
    r.v[1] = t.y;
  } else {
    r.v[0] = __ldg(p);
  }
  return r;
}
template <int W>
__device__ __forceinline__ void st_vec(double* p, const Vec<W>& r) {
  if constexpr (W == 4) {
    asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(r.v[0]), "d"(r.v[1]), "d"(r.v[2]),
                 "d"(r.v[3])
                 : "memory");
  } else if constexpr (W == 2) {
    *reinterpret_cast<double2*>(p) = make_double2(r.v[0], r.v[1]);
  } else {
    *p = r.v[0];
  }
}

template <int W>
__global__ void __launch_bounds__(256) xform_kernel(const MkXformJob* __restrict__ jobs, int64_t rows, int64_t cols) {
  const MkXformJob& jb = jobs[blockIdx.y];
  const int ns = jb.nsrc, nd = jb.ndst;
  const int64_t cv = cols / W;
  // rows x cv < 2^32 for every block the planner forms (checked by the launcher)
  const uint32_t total = (uint32_t)(rows * cv), ucv = (uint32_t)cv;
  for (uint32_t idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += gridDim.x * blockDim.x) {
    const uint32_t r = idx / ucv;
    const int64_t c = (int64_t)(idx - r * ucv) * W;
    Vec<W> v[MK_XFORM_MAX];
#pragma unroll
    for (int i = 0; i < MK_XFORM_MAX; ++i)
      if (i < ns) v[i] = ld_vec<W>(jb.src[i] + r * jb.lds[i] + c);
#pragma unroll
    for (int j = 0; j < MK_XFORM_MAX; ++j) {
      if (j < nd) {
        Vec<W> acc;
#pragma unroll
        for (int u = 0; u < W; ++u) acc.v[u] = 0.0;
#pragma unroll
        for (int i = 0; i < MK_XFORM_MAX; ++i) {
          const int cf = i < ns ? jb.coef[j][i] : 0;  // job-uniform: zero terms are skipped,
          if (cf > 0) {                               // so an inf elsewhere cannot become NaN
#pragma unroll
            for (int u = 0; u < W; ++u) acc.v[u] += v[i].v[u];
          } else if (cf < 0) {
#pragma unroll
            for (int u = 0; u < W; ++u) acc.v[u] -= v[i].v[u];
          }
        }
        st_vec<W>(jb.dst[j] + r * jb.ldd[j] + c, acc);
      }
    }
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
