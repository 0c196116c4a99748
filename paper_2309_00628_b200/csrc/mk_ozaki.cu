// FP64 products on the INT8 tensor cores (Ozaki scheme I) for sm_100a: digit splitting kernels
// and the tcgen05 kind::i8 product kernel with TMEM anti-diagonal accumulators. See mk_ozaki.h
// for the arithmetic; DESIGN.md §3 (K5) for the roofline.
#include <cuda.h>
#include <cuda_runtime.h>

#include <climits>
#include <cmath>
#include <mutex>

#include "../../include/mk_strassen.h"
#include "mk_device.cuh"
#include "mk_ozaki.h"

namespace mk {
namespace oz {

constexpr int BM = 128;      // tile rows = TMEM lanes
constexpr int BN = 64;       // tile columns = TMEM columns per anti-diagonal accumulator
constexpr int BK = 32;       // int8 k per stage = one UMMA K step (32 bytes = the 32B swizzle span)
constexpr int STAGES = 4;
constexpr int NTHREADS = 192;  // warp 0 TMA, warp 1 MMA issuer + TMEM owner, warps 2-5 epilogue
constexpr int KPAD = 16;       // digit-plane row pitch granularity (TMA stride alignment)
constexpr int EXP_NONFINITE = INT_MIN;

struct Args {
  const int32_t* ex;  // row exponents of X (m)
  const int32_t* fy;  // column exponents of Y (n)
  double* C;
  int64_t ldc;
  int32_t M, N, K, tiles_n;
  int32_t accumulate;
  double sign;
};

// ---------------------------------------------------------------------------------------------
// tcgen05 helpers (kind::i8, cta_group::1)
// ---------------------------------------------------------------------------------------------
// Shared-memory matrix descriptor, K-major operand, 32-byte swizzle: rows of 32 bytes, 8-row
// core groups 256 bytes apart (SBO); LBO unused (the K extent of one MMA is one swizzle span).
__device__ __forceinline__ uint64_t smem_desc_sw32(const void* p) {
  const uint64_t addr = smem_u32(p);
  uint64_t d = 0;
  d |= (addr >> 4) & 0x3FFFull;          // start address
  d |= (uint64_t)1 << 16;                // LBO (ignored)
  d |= (uint64_t)(256 >> 4) << 32;       // SBO
  d |= (uint64_t)1 << 46;                // descriptor version (sm_100)
  d |= (uint64_t)6 << 61;                // SWIZZLE_32B
  return d;
}

// Instruction descriptor: s8 x s8 -> s32, both K-major, M = BM, N = BN.
__host__ __device__ constexpr uint32_t idesc_i8() {
  return (2u << 4)                  // D format S32
         | (1u << 7) | (1u << 10)   // A, B signed 8-bit
         | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* m, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

// ---------------------------------------------------------------------------------------------
// Product kernel: one CTA per 128 x 64 output tile; S anti-diagonal int32 accumulators of 64
// TMEM columns each (S * 64 <= 512). Per 32-k stage the TMA brings all S digit planes of the
// X rows and the Y columns (S * 6 KiB) and the issuer runs the S(S+1)/2 digit-pair MMAs, so each
// staged byte feeds (S+1)/2 MMAs.
// ---------------------------------------------------------------------------------------------
template <int S>
__global__ void __launch_bounds__(NTHREADS, 1)
    ozaki_product_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmY, Args a) {
  constexpr int A_TILE = BM * BK;
  constexpr int B_TILE = BN * BK;
  constexpr int STAGE_BYTES = S * (A_TILE + B_TILE);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tmem_full = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tm = blockIdx.x / a.tiles_n, tn = blockIdx.x % a.tiles_n;
  const int nkb = (a.K + BK - 1) / BK;

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmX);
    tma_prefetch_desc(&tmY);
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(tmem_full, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      for (int kb = 0; kb < nkb; ++kb) {
        const int st = kb % STAGES;
        if (kb >= STAGES) mbar_wait(&empty[st], ((kb / STAGES) - 1) & 1);
        uint8_t* sa = smem + st * STAGE_BYTES;
        mbar_arrive_expect_tx(&full[st], STAGE_BYTES);
        tma_load_3d(sa, &tmX, kb * BK, tm * BM, 0, &full[st]);
        tma_load_3d(sa + S * A_TILE, &tmY, kb * BK, tn * BN, 0, &full[st]);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_i8();
      for (int kb = 0; kb < nkb; ++kb) {
        const int st = kb % STAGES;
        mbar_wait(&full[st], (kb / STAGES) & 1);
        tmem_fence_after();
        const uint8_t* sa = smem + st * STAGE_BYTES;
        const uint8_t* sb = sa + S * A_TILE;
#pragma unroll
        for (int s = 0; s < S; ++s) {
          const uint64_t da = smem_desc_sw32(sa + s * A_TILE);
#pragma unroll
          for (int t = 0; t < S - s; ++t)
            mma_i8(tmem + (uint32_t)((s + t) * BN), da, smem_desc_sw32(sb + t * B_TILE), idesc,
                   (kb > 0 || s > 0) ? 1u : 0u);
        }
        mma_commit(&empty[st]);  // frees the stage once these MMAs have read it
      }
      mma_commit(tmem_full);
    }
  } else {
    // epilogue: warp w reads TMEM lanes 32*(w%4)..+31 (one output row per thread)
    const int q = warp & 3;
    const int row = tm * BM + q * 32 + lane;
    mbar_wait(tmem_full, 0);
    tmem_fence_after();
    const uint32_t tl = tmem + ((uint32_t)(q * 32) << 16);
    const bool row_ok = row < a.M;
    const int e = row_ok ? a.ex[row] : 0;
    double* crow = a.C + (int64_t)row * a.ldc;
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 16) {
      uint32_t r[S][16];
#pragma unroll
      for (int d = 0; d < S; ++d) tmem_ld16(tl + (uint32_t)(d * BN + c0), r[d]);
      tmem_wait_ld();
      if (!row_ok) continue;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int col = tn * BN + c0 + j;
        if (col >= a.N) break;
        double v = (double)(int32_t)r[S - 1][j];
#pragma unroll
        for (int d = S - 2; d >= 0; --d) v = fma(v, 0.0078125, (double)(int32_t)r[d][j]);
        const int f = a.fy[col];
        double p;
        if (e == EXP_NONFINITE || f == EXP_NONFINITE)
          p = __longlong_as_double(0x7ff8000000000000ll);
        else
          p = a.sign * ldexp(v, e + f - 14);
        double* dst = crow + col;
        *dst = a.accumulate ? *dst + p : p;
      }
    }
  }
  tmem_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

// ---------------------------------------------------------------------------------------------
// Digit splitting (HBM bound): X rows -> exponents + S int8 planes [S][rows][kp].
// One warp per row; lane handles 4 consecutive k per iteration (one 32-bit store per plane).
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ int row_exponent(double mx) {
  if (!(mx <= 1.7976931348623157e308)) return EXP_NONFINITE;  // inf / nan
  if (mx == 0.0) return 0;
  int e;
  frexp(mx, &e);  // mx = f * 2^e, f in [0.5, 1): every |x| < 2^e
  return e;
}

template <int S>
__device__ __forceinline__ void digits4(const double x[4], double scale, uint32_t out[S]) {
  double y[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) y[i] = x[i] * scale;  // |y| < 1, exact (power-of-two scaling)
#pragma unroll
  for (int s = 0; s < S; ++s) {
    uint32_t w = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const double z = y[i] * 128.0;  // exact
      const double dg = trunc(z);     // |dg| <= 127
      y[i] = z - dg;                  // exact remainder, |y| < 1
      w |= ((uint32_t)(uint8_t)(int8_t)(int)dg) << (8 * i);
    }
    out[s] = w;
  }
}

template <int S>
__global__ void split_rows_kernel(const double* __restrict__ X, int64_t ldx, int rows, int K, int kp,
                                  int32_t* __restrict__ ex, uint8_t* __restrict__ planes) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= rows) return;
  const double* xr = X + (int64_t)warp * ldx;
  double mx = 0.0;
  bool bad = false;  // inf / nan (fmax alone would drop a NaN)
  for (int k = lane; k < K; k += 32) {
    const double v = fabs(xr[k]);
    bad |= !(v <= 1.7976931348623157e308);
    mx = fmax(mx, v);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  bad = __any_sync(0xffffffffu, bad);
  const int e = bad ? EXP_NONFINITE : row_exponent(mx);
  if (lane == 0) ex[warp] = e;
  const double scale = (e == EXP_NONFINITE) ? 0.0 : ldexp(1.0, -e);
  const int64_t plane = (int64_t)rows * kp;
  uint8_t* pr = planes + (int64_t)warp * kp;
  for (int k0 = 4 * lane; k0 < kp; k0 += 128) {
    double x[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) x[i] = (k0 + i < K && e != EXP_NONFINITE) ? xr[k0 + i] : 0.0;
    uint32_t w[S];
    digits4<S>(x, scale, w);
#pragma unroll
    for (int s = 0; s < S; ++s) *reinterpret_cast<uint32_t*>(pr + s * plane + k0) = w[s];
  }
}

// Column maxima of Y (k x n) as IEEE bit patterns (monotone for |y|): grid (n/256, k/256).
__global__ void colmax_kernel(const double* __restrict__ Y, int64_t ldy, int K, int N,
                              unsigned long long* __restrict__ cmax) {
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= N) return;
  const int k0 = blockIdx.y * 256, k1 = min(K, k0 + 256);
  double mx = 0.0;
  bool bad = false;
  for (int k = k0; k < k1; ++k) {
    const double y = Y[(int64_t)k * ldy + col];
    bad |= !(fabs(y) <= 1.7976931348623157e308);
    mx = fmax(mx, fabs(y));
  }
  const unsigned long long bits = bad ? 0x7ff0000000000000ull : (unsigned long long)__double_as_longlong(mx);
  atomicMax(&cmax[col], bits);
}

__global__ void colexp_kernel(const unsigned long long* __restrict__ cmax, int N, int32_t* __restrict__ fy) {
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= N) return;
  fy[col] = row_exponent(__longlong_as_double((long long)cmax[col]));
}

// Y (k x n, row-major) -> S planes of Y^T [S][n][kp] (K-major for the B operand), 32 x 32 tiles
// through shared memory. Block (32, 8).
template <int S>
__global__ void split_cols_kernel(const double* __restrict__ Y, int64_t ldy, int K, int N, int kp,
                                  const int32_t* __restrict__ fy, uint8_t* __restrict__ planes) {
  __shared__ uint32_t sm[S][32][9];  // [plane][col][k/4] (+1 pad)
  const int n0 = blockIdx.x * 32, k0 = blockIdx.y * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int col = n0 + tx;
  const int f = col < N ? fy[col] : 0;
  const double scale = (col < N && f != EXP_NONFINITE) ? ldexp(1.0, -f) : 0.0;
  // thread (tx, ty) converts k = k0 + 4*ty .. +3 of column col
  double x[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int k = k0 + 4 * ty + i;
    x[i] = (col < N && k < K && scale != 0.0) ? Y[(int64_t)k * ldy + col] : 0.0;
  }
  uint32_t w[S];
  digits4<S>(x, scale, w);
#pragma unroll
  for (int s = 0; s < S; ++s) sm[s][tx][ty] = w[s];
  __syncthreads();
  // write: plane s, rows n0..n0+31, bytes k0..k0+31 -> 32 rows x 8 words; 256 threads, one word each
  const int t = ty * 32 + tx;
  const int r = t >> 3, wi = t & 7;
  const int n = n0 + r, k = k0 + 4 * wi;
  if (n < N && k < kp) {
    const int64_t plane = (int64_t)N * kp;
#pragma unroll
    for (int s = 0; s < S; ++s) *reinterpret_cast<uint32_t*>(planes + s * plane + (int64_t)n * kp + k) = sm[s][r][wi];
  }
}

// ---------------------------------------------------------------------------------------------
// Host side
// ---------------------------------------------------------------------------------------------
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static PFN_encodeTiled get_encode() {
  static PFN_encodeTiled fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled>(p);
  });
  return fn;
}

static int64_t kpad(int64_t k) { return (k + KPAD - 1) / KPAD * KPAD; }
static size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

struct Layout {
  size_t planes_x, planes_y, ex, fy, cmax, total;
};
static Layout layout(int64_t m, int64_t n, int64_t k, int S) {
  Layout L;
  const int64_t kp = kpad(k);
  L.planes_x = 0;
  L.planes_y = align256(L.planes_x + (size_t)S * m * kp);
  L.ex = align256(L.planes_y + (size_t)S * n * kp);
  L.fy = align256(L.ex + 4 * (size_t)m);
  L.cmax = align256(L.fy + 4 * (size_t)n);
  L.total = align256(L.cmax + 8 * (size_t)n);
  return L;
}

template <int S>
static size_t smem_bytes() {
  return STAGES * S * (BM + BN) * BK + 1024 /*align*/ + 256 /*barriers*/;
}

template <int S>
static int run(const double* X, int64_t ldx, const double* Y, int64_t ldy, double* C, int64_t ldc, int64_t m,
               int64_t n, int64_t k, int accumulate, double sign, uint8_t* ws, cudaStream_t st, std::string* err) {
  const Layout L = layout(m, n, k, S);
  const int64_t kp = kpad(k);
  uint8_t* px = ws + L.planes_x;
  uint8_t* py = ws + L.planes_y;
  int32_t* ex = reinterpret_cast<int32_t*>(ws + L.ex);
  int32_t* fy = reinterpret_cast<int32_t*>(ws + L.fy);
  auto* cmax = reinterpret_cast<unsigned long long*>(ws + L.cmax);

  split_rows_kernel<S><<<(unsigned)((m * 32 + 255) / 256), 256, 0, st>>>(X, ldx, (int)m, (int)k, (int)kp, ex, px);
  cudaMemsetAsync(cmax, 0, 8 * (size_t)n, st);
  colmax_kernel<<<dim3((unsigned)((n + 255) / 256), (unsigned)((k + 255) / 256)), 256, 0, st>>>(Y, ldy, (int)k,
                                                                                                (int)n, cmax);
  colexp_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(cmax, (int)n, fy);
  split_cols_kernel<S><<<dim3((unsigned)((n + 31) / 32), (unsigned)((kp + 31) / 32)), dim3(32, 8), 0, st>>>(
      Y, ldy, (int)k, (int)n, (int)kp, fy, py);

  PFN_encodeTiled enc = get_encode();
  if (!enc) {
    *err = "cuTensorMapEncodeTiled unavailable";
    return MK_ERR_CUDA;
  }
  CUtensorMap tmX, tmY;
  {
    cuuint64_t dims[3] = {(cuuint64_t)kp, (cuuint64_t)m, (cuuint64_t)S};
    cuuint64_t strides[2] = {(cuuint64_t)kp, (cuuint64_t)(m * kp)};
    cuuint32_t box[3] = {BK, BM, S};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc(&tmX, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, px, dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      *err = "cuTensorMapEncodeTiled (X digits) failed: " + std::to_string((int)r);
      return MK_ERR_CUDA;
    }
  }
  {
    cuuint64_t dims[3] = {(cuuint64_t)kp, (cuuint64_t)n, (cuuint64_t)S};
    cuuint64_t strides[2] = {(cuuint64_t)kp, (cuuint64_t)(n * kp)};
    cuuint32_t box[3] = {BK, BN, S};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc(&tmY, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, py, dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      *err = "cuTensorMapEncodeTiled (Y digits) failed: " + std::to_string((int)r);
      return MK_ERR_CUDA;
    }
  }
  Args a;
  a.ex = ex;
  a.fy = fy;
  a.C = C;
  a.ldc = ldc;
  a.M = (int)m;
  a.N = (int)n;
  a.K = (int)k;
  a.tiles_n = (int)((n + BN - 1) / BN);
  a.accumulate = accumulate;
  a.sign = sign;
  const int tiles = (int)((m + BM - 1) / BM) * a.tiles_n;
  const size_t smem = smem_bytes<S>();
  static std::once_flag attr_once;
  std::call_once(attr_once, [&] {
    cudaFuncSetAttribute(ozaki_product_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  });
  ozaki_product_kernel<S><<<tiles, NTHREADS, smem, st>>>(tmX, tmY, a);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    *err = std::string("ozaki_product_kernel launch: ") + cudaGetErrorString(e);
    return MK_ERR_CUDA;
  }
  return MK_OK;
}

}  // namespace oz

int64_t ozaki_max_k(int slices) {
  // <= slices digit pairs per anti-diagonal, each |a*b| <= 127^2, summed over K in int32
  return (int64_t)(2147483647ll / ((int64_t)slices * 16129));
}

size_t ozaki_workspace_bytes(int64_t m, int64_t n, int64_t k, int slices) {
  return oz::layout(m, n, k, slices).total;
}

int ozaki_product(const double* X, int64_t ldx, const double* Y, int64_t ldy, double* C, int64_t ldc, int64_t m,
                  int64_t n, int64_t k, int slices, int accumulate, double sign, void* ws, size_t ws_bytes,
                  cudaStream_t st, std::string* err) {
  if (slices < kOzMinSlices || slices > kOzMaxSlices) {
    *err = "slices must be in [4, 8]";
    return MK_ERR_ARG;
  }
  if (k > ozaki_max_k(slices)) {
    *err = "k too large for exact int32 accumulation";
    return MK_ERR_ARG;
  }
  if (m > INT_MAX / 2 || n > INT_MAX / 2) {
    *err = "extent too large";
    return MK_ERR_DIMENSION;
  }
  if (ws_bytes < ozaki_workspace_bytes(m, n, k, slices) || (reinterpret_cast<uintptr_t>(ws) & 255)) {
    *err = "workspace too small or not 256-byte aligned";
    return MK_ERR_WORKSPACE;
  }
  auto* w = static_cast<uint8_t*>(ws);
  switch (slices) {
    case 4: return oz::run<4>(X, ldx, Y, ldy, C, ldc, m, n, k, accumulate, sign, w, st, err);
    case 5: return oz::run<5>(X, ldx, Y, ldy, C, ldc, m, n, k, accumulate, sign, w, st, err);
    case 6: return oz::run<6>(X, ldx, Y, ldy, C, ldc, m, n, k, accumulate, sign, w, st, err);
    case 7: return oz::run<7>(X, ldx, Y, ldy, C, ldc, m, n, k, accumulate, sign, w, st, err);
    default: return oz::run<8>(X, ldx, Y, ldy, C, ldc, m, n, k, accumulate, sign, w, st, err);
  }
}

}  // namespace mk
