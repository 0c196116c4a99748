// FP64 products on the INT8 tensor cores (Ozaki scheme I) for sm_100a: digit splitting kernels
// and the tcgen05 kind::i8 product kernel with TMEM anti-diagonal accumulators. See mk_ozaki.h
// for the arithmetic; DESIGN.md §3 (K5) for the roofline.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
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
  int32_t nd, pad_;
  OzDest d[kOzMaxDests];  // destinations: C[d.row + i][d.col + j] (+)= d.sign * P_ij
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

// Instruction descriptor: 8-bit x 8-bit -> s32, both K-major, M = BM, N = n; sa / sb: operand
// signed (the leading digit plane) or unsigned (every later plane).
__host__ __device__ constexpr uint32_t idesc_i8(int n, bool sa, bool sb) {
  return (2u << 4)                                 // D format S32
         | ((sa ? 1u : 0u) << 7) | ((sb ? 1u : 0u) << 10)  // A, B: 1 signed / 0 unsigned 8-bit
         | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
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
      for (int kb = 0; kb < nkb; ++kb) {
        const int st = kb % STAGES;
        mbar_wait(&full[st], (kb / STAGES) & 1);
        tmem_fence_after();
        const uint8_t* sa = smem + st * STAGE_BYTES;
        const uint8_t* sb = sa + S * A_TILE;
        // X digit plane s meets Y planes t = 0..S-1-s. The Y planes are consecutive 64-row
        // blocks of one K-major operand and their accumulators (anti-diagonals s+t) are
        // consecutive 64-column TMEM blocks, so one MMA with N = 64 * #planes (<= 256) covers
        // several pairs of one signedness: plane 0 (signed) alone, planes 1.. (unsigned) in
        // groups of 4 -- S(S+1)/2 pairs in sum_s (1 + ceil((S-1-s)/4)) MMAs.
#pragma unroll
        for (int s = 0; s < S; ++s) {
          const uint64_t da = smem_desc_sw32(sa + s * A_TILE);
          const uint32_t acc = (kb > 0 || s > 0) ? 1u : 0u;
          mma_i8(tmem + (uint32_t)(s * BN), da, smem_desc_sw32(sb), idesc_i8(BN, s == 0, true), acc);
#pragma unroll
          for (int t0 = 1; t0 < S - s; t0 += 4) {
            const int cnt = (S - s - t0) < 4 ? (S - s - t0) : 4;
            mma_i8(tmem + (uint32_t)((s + t0) * BN), da, smem_desc_sw32(sb + t0 * B_TILE),
                   idesc_i8(cnt * BN, s == 0, false), acc);
          }
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
        for (int d = S - 2; d >= 0; --d) v = fma(v, 0.00390625, (double)(int32_t)r[d][j]);
        const int f = a.fy[col];
        double p;
        if (e == EXP_NONFINITE || f == EXP_NONFINITE)
          p = __longlong_as_double(0x7ff8000000000000ll);
        else
          p = ldexp(v, e + f - 14);
        for (int t = 0; t < a.nd; ++t) {
          double* dst = crow + a.d[t].row * a.ldc + a.d[t].col + col;
          *dst = a.d[t].accumulate ? fma(a.d[t].sign, p, *dst) : a.d[t].sign * p;
        }
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

// x * scale = y in (-1, 1) is written as 2^-7 * sum_s d_s 2^(-8s): d_0 = floor(128 y) in
// [-128, 127] (signed plane), then d_s = floor(256 r) in [0, 255] of the remainder r in [0, 1)
// (unsigned planes, 8 bits each): 7 + 8 (S - 1) bits. Every step is exact in FP64.
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
      const double z = y[i] * (s == 0 ? 128.0 : 256.0);  // exact
      const double dg = floor(z);
      y[i] = z - dg;  // exact remainder in [0, 1)
      w |= ((uint32_t)(s == 0 ? (uint8_t)(int8_t)(int)dg : (uint8_t)(int)dg)) << (8 * i);
    }
    out[s] = w;
  }
}

// Operand value at (r, c): the signed sum of up to 4 blocks of one base (the Strassen / Winograd
// pre-addition, formed on load instead of materialised), in table order.
__device__ __forceinline__ double term_sum(const OzOperand& o, int64_t r, int64_t c) {
  const int64_t off = r * o.ld + c;
  double v = o.s[0] * o.p[0][off];
  for (int i = 1; i < o.n; ++i) v = fma(o.s[i], o.p[i][off], v);
  return v;
}

// X rows -> exponents + S digit planes [S][rows][kp]: one warp per row, each lane 4 consecutive
// k per iteration (one 32-bit store per plane).
template <int S>
__global__ void split_rows_kernel(const OzOperand X, int rows, int K, int kp, int32_t* __restrict__ ex,
                                  uint8_t* __restrict__ planes) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= rows) return;
  double mx = 0.0;
  bool bad = false;  // inf / nan (fmax alone would drop a NaN)
  for (int k = lane; k < K; k += 32) {
    const double v = fabs(term_sum(X, warp, k));
    bad |= !(v <= 1.7976931348623157e308);
    mx = fmax(mx, v);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  bad = __any_sync(0xffffffffu, bad);
  const int e = bad ? EXP_NONFINITE : row_exponent(mx);
  if (lane == 0) ex[warp] = e;
  const double scale = (e == EXP_NONFINITE) ? 0.0 : ldexp(1.0, -e);
  const int64_t plane = (int64_t)rows * kp;
  uint8_t* pr = planes + (int64_t)warp * kp;
  for (int k0 = 4 * lane; k0 < kp; k0 += 128) {
    double x[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) x[i] = (k0 + i < K && e != EXP_NONFINITE) ? term_sum(X, warp, k0 + i) : 0.0;
    uint32_t w[S];
    digits4<S>(x, scale, w);
#pragma unroll
    for (int s = 0; s < S; ++s) *reinterpret_cast<uint32_t*>(pr + s * plane + k0) = w[s];
  }
}

// Column maxima of Y (k x n) as IEEE bit patterns (monotone for |y|): grid (n/256, k/256).
__global__ void colmax_kernel(const OzOperand Y, int K, int N, unsigned long long* __restrict__ cmax) {
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= N) return;
  const int k0 = blockIdx.y * 256, k1 = min(K, k0 + 256);
  double mx = 0.0;
  bool bad = false;
  for (int k = k0; k < k1; ++k) {
    const double y = fabs(term_sum(Y, k, col));
    bad |= !(y <= 1.7976931348623157e308);
    mx = fmax(mx, y);
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
__global__ void split_cols_kernel(const OzOperand Y, int K, int N, int kp, const int32_t* __restrict__ fy,
                                  uint8_t* __restrict__ planes) {
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
    x[i] = (col < N && k < K && scale != 0.0) ? term_sum(Y, k, col) : 0.0;
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

// K per call: the whole K when it fits the exact int32 accumulation, else equal chunks
static int64_t chunk_k(int64_t k, int S) {
  const int64_t mx = ozaki_max_k(S) / KPAD * KPAD;
  const int64_t nc = (k + mx - 1) / mx;
  return std::min(mx, kpad((k + nc - 1) / nc));
}

static int encode_planes(CUtensorMap* tm, uint8_t* planes, int64_t rows, int64_t kp, int S, uint32_t box_rows,
                         std::string* err) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) {
    *err = "cuTensorMapEncodeTiled unavailable";
    return MK_ERR_CUDA;
  }
  cuuint64_t dims[3] = {(cuuint64_t)kp, (cuuint64_t)rows, (cuuint64_t)S};
  cuuint64_t strides[2] = {(cuuint64_t)kp, (cuuint64_t)(rows * kp)};
  cuuint32_t box[3] = {BK, box_rows, (cuuint32_t)S};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, planes, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    *err = "cuTensorMapEncodeTiled (digit planes) failed: " + std::to_string((int)r);
    return MK_ERR_CUDA;
  }
  return MK_OK;
}

template <int S>
static size_t smem_bytes() {
  return STAGES * S * (BM + BN) * BK + 1024 /*align*/ + 256 /*barriers*/;
}

// One K chunk: split both operands, then the product kernel into every destination.
template <int S>
static int run(const OzOperand& X, const OzOperand& Y, double* C, int64_t ldc, int64_t m, int64_t n, int64_t k,
               const OzDest* d, int nd, uint8_t* ws, cudaStream_t st, std::string* err) {
  const Layout L = layout(m, n, k, S);
  const int64_t kp = kpad(k);
  uint8_t* px = ws + L.planes_x;
  uint8_t* py = ws + L.planes_y;
  int32_t* ex = reinterpret_cast<int32_t*>(ws + L.ex);
  int32_t* fy = reinterpret_cast<int32_t*>(ws + L.fy);
  auto* cmax = reinterpret_cast<unsigned long long*>(ws + L.cmax);

  split_rows_kernel<S><<<(unsigned)((m * 32 + 255) / 256), 256, 0, st>>>(X, (int)m, (int)k, (int)kp, ex, px);
  cudaMemsetAsync(cmax, 0, 8 * (size_t)n, st);
  colmax_kernel<<<dim3((unsigned)((n + 255) / 256), (unsigned)((k + 255) / 256)), 256, 0, st>>>(Y, (int)k, (int)n,
                                                                                                cmax);
  colexp_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(cmax, (int)n, fy);
  split_cols_kernel<S><<<dim3((unsigned)((n + 31) / 32), (unsigned)((kp + 31) / 32)), dim3(32, 8), 0, st>>>(
      Y, (int)k, (int)n, (int)kp, fy, py);

  CUtensorMap tmX, tmY;
  if (int rc = encode_planes(&tmX, px, m, kp, S, BM, err)) return rc;
  if (int rc = encode_planes(&tmY, py, n, kp, S, BN, err)) return rc;
  Args a;
  a.ex = ex;
  a.fy = fy;
  a.C = C;
  a.ldc = ldc;
  a.M = (int)m;
  a.N = (int)n;
  a.K = (int)k;
  a.tiles_n = (int)((n + BN - 1) / BN);
  a.nd = nd;
  a.pad_ = 0;
  for (int i = 0; i < nd; ++i) a.d[i] = d[i];
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

// Whole product: K in chunks of chunk_k (later chunks accumulate into every destination).
static int product_chunks(const OzOperand& X, const OzOperand& Y, double* C, int64_t ldc, int64_t m, int64_t n,
                          int64_t k, int S, const OzDest* d, int nd, uint8_t* ws, cudaStream_t st, std::string* err) {
  const int64_t kc = chunk_k(k, S);
  OzDest dd[kOzMaxDests];
  for (int i = 0; i < nd; ++i) dd[i] = d[i];
  for (int64_t k0 = 0; k0 < k; k0 += kc) {
    const int64_t kk = std::min(kc, k - k0);
    OzOperand Xc = X, Yc = Y;
    for (int i = 0; i < X.n; ++i) Xc.p[i] = X.p[i] + k0;
    for (int i = 0; i < Y.n; ++i) Yc.p[i] = Y.p[i] + k0 * Y.ld;
    int rc;
    switch (S) {
      case 4: rc = run<4>(Xc, Yc, C, ldc, m, n, kk, dd, nd, ws, st, err); break;
      case 5: rc = run<5>(Xc, Yc, C, ldc, m, n, kk, dd, nd, ws, st, err); break;
      case 6: rc = run<6>(Xc, Yc, C, ldc, m, n, kk, dd, nd, ws, st, err); break;
      case 7: rc = run<7>(Xc, Yc, C, ldc, m, n, kk, dd, nd, ws, st, err); break;
      default: rc = run<8>(Xc, Yc, C, ldc, m, n, kk, dd, nd, ws, st, err); break;
    }
    if (rc != MK_OK) return rc;
    for (int i = 0; i < nd; ++i) dd[i].accumulate = 1;
  }
  return MK_OK;
}

}  // namespace oz

int64_t ozaki_max_k(int slices) {
  // anti-diagonal d = S-1 sums 2 signed x unsigned pairs (|.| <= 128 * 255) and S-2 unsigned
  // pairs (<= 255^2) per k; the int32 accumulator must hold K of them
  const int64_t worst = 2 * 128 * 255 + (int64_t)(slices - 2) * 255 * 255;
  return 2147483647ll / worst;
}

size_t ozaki_workspace_bytes(int64_t m, int64_t n, int64_t k, int slices) {
  return oz::layout(m, n, oz::chunk_k(k, slices), slices).total;
}

static int check_args(int64_t m, int64_t n, int slices, int nd, std::string* err) {
  if (slices < kOzMinSlices || slices > kOzMaxSlices) {
    *err = "slices must be in [4, 8]";
    return MK_ERR_ARG;
  }
  if (nd < 1 || nd > kOzMaxDests) {
    *err = "internal: destination count out of range";
    return MK_ERR_ARG;
  }
  if (m > INT_MAX / 2 || n > INT_MAX / 2) {
    *err = "extent too large";
    return MK_ERR_DIMENSION;
  }
  return MK_OK;
}

int ozaki_product(const double* X, int64_t ldx, const double* Y, int64_t ldy, double* C, int64_t ldc, int64_t m,
                  int64_t n, int64_t k, int slices, int accumulate, double sign, void* ws, size_t ws_bytes,
                  cudaStream_t st, std::string* err) {
  if (int rc = check_args(m, n, slices, 1, err)) return rc;
  if (ws_bytes < ozaki_workspace_bytes(m, n, k, slices) || (reinterpret_cast<uintptr_t>(ws) & 255)) {
    *err = "workspace too small or not 256-byte aligned";
    return MK_ERR_WORKSPACE;
  }
  const OzOperand ox{{X}, {1.0}, 1, ldx}, oy{{Y}, {1.0}, 1, ldy};
  const OzDest dst{0, 0, sign, accumulate, 0};
  return oz::product_chunks(ox, oy, C, ldc, m, n, k, slices, &dst, 1, static_cast<uint8_t*>(ws), st, err);
}

int ozaki_product_multi(const OzOperand& X, const OzOperand& Y, double* C, int64_t ldc, int64_t m, int64_t n,
                        int64_t k, int slices, const OzDest* d, int nd, cudaStream_t st, std::string* err) {
  if (int rc = check_args(m, n, slices, nd, err)) return rc;
  if (X.n < 1 || X.n > kOzMaxTerms || Y.n < 1 || Y.n > kOzMaxTerms) {
    *err = "internal: operand term count out of range";
    return MK_ERR_ARG;
  }
  const size_t wsb = ozaki_workspace_bytes(m, n, k, slices);
  void* ws = nullptr;
  cudaError_t e = cudaMallocAsync(&ws, wsb, st);
  if (e != cudaSuccess) {
    cudaGetLastError();
    *err = std::string("Ozaki leaf workspace: ") + cudaGetErrorString(e);
    return e == cudaErrorMemoryAllocation ? MK_ERR_WORKSPACE : MK_ERR_CUDA;
  }
  int rc = oz::product_chunks(X, Y, C, ldc, m, n, k, slices, d, nd, static_cast<uint8_t*>(ws), st, err);
  e = cudaFreeAsync(ws, st);
  if (rc == MK_OK && e != cudaSuccess) {
    *err = std::string("Ozaki leaf workspace free: ") + cudaGetErrorString(e);
    rc = MK_ERR_CUDA;
  }
  return rc;
}

}  // namespace mk
