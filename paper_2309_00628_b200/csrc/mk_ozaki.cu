// FP64 products on the INT8 tensor cores (Ozaki scheme I) for sm_100a: digit splitting kernels
// and the tcgen05 kind::i8 product kernel with TMEM anti-diagonal accumulators. See mk_ozaki.h
// for the arithmetic; DESIGN.md §3 (K5) for the roofline.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <map>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <type_traits>
#include <vector>

#include "../../include/mk_strassen.h"
#include "mk_device.cuh"
#include "mk_ozaki.h"

namespace mk {
namespace oz {

constexpr int BM = 128;      // tile rows = TMEM lanes
constexpr int BN = 64;       // tile columns = TMEM columns per anti-diagonal accumulator
constexpr int BK = 32;       // int8 k per stage = one UMMA K step (32 bytes = the 32B swizzle span)
constexpr int STAGES = 4;
constexpr int NTHREADS = 256;  // warp 0 TMA, warp 1 MMA issuer + TMEM owner; then all 8 warps run the epilogue
                               // (2 per TMEM lane quarter; 8 warps = 2 per SM sub-partition: up to 255 registers)
constexpr int KPAD = BK;       // K padding: whole 32-byte k-blocks
constexpr int EXP_NONFINITE = INT_MIN;
#ifndef MK_OZ_GROUP
#define MK_OZ_GROUP 8  // tile rows per rasterisation group (16: +1.3% bench step, 4: +1.2%)
#endif

struct Args {
  const uint8_t* px;  // X digit tiles [tiles_m][nkb][S][128 rows x 32 B] (smem images, 32B swizzle)
  const uint8_t* py;  // Y digit tiles [tiles_n][nkb][S][64 rows x 32 B]
  const int32_t* ex;  // row exponents of X (m)
  const int32_t* fy;  // column exponents of Y (n)
  const int32_t* rs;  // [S][m] row sums of the X digit planes (offset correction of Y's plane 0)
  double* C;
  int64_t ldc;
  int32_t M, N, K, tiles_n;
  int32_t nd, pad_;
  unsigned long long* trace;  // debug (MK_OZ_TRACE=1): 7 %globaltimer stamps per tile
  OzSlabs slabs;              // slabs.n > 0: C rows routed to owner slabs, atomic adds (persistent kernel)
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
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  for (;;) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (ok) return;
    __nanosleep(256);
  }
}
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
// Contiguous global -> shared bulk copy (one large request stream instead of one 32-byte
// request per tile row), completes on `bar`.
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Byte offset of (row r, byte c) in a K-major tile of 32-byte rows under the 32B swizzle
// (CuTe Swizzle<1,4,3>: address bit 7 flips bit 4 -- the 16-byte halves of rows 4..7 of each
// 8-row group swap), i.e. the image the UMMA descriptor's SWIZZLE_32B layout reads.
__host__ __device__ __forceinline__ uint32_t swz32(uint32_t r, uint32_t c) {
  const uint32_t o = r * 32 + c;
  return o ^ ((o >> 3) & 0x10);
}

// ---------------------------------------------------------------------------------------------
// Product kernel: one CTA per 128 x 64 output tile; S anti-diagonal int32 accumulators of 64
// TMEM columns each (S * 64 <= 512). Per 32-k stage the TMA brings all S digit planes of the
// X rows and the Y columns (S * 6 KiB) and the issuer runs the S(S+1)/2 digit-pair MMAs, so each
// staged byte feeds (S+1)/2 MMAs.
// ---------------------------------------------------------------------------------------------
template <int S>
__global__ void __launch_bounds__(NTHREADS, 1)
    ozaki_product_kernel(const __grid_constant__ Args a) {
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
  // grouped rasterisation: 16 tile rows at a time, column-major inside the group, so the digit
  // planes a wave of CTAs reads (16 X panels + a few Y panels) stay in L2
  int tm, tn;
  {
    const int tiles_m = (a.M + BM - 1) / BM, g = MK_OZ_GROUP;
    const int per_group = g * a.tiles_n, grp = blockIdx.x / per_group, first = grp * g;
    const int rows = min(g, tiles_m - first), local = blockIdx.x - grp * per_group;
    tm = first + local % rows;
    tn = local / rows;
  }
  const int nkb = (a.K + BK - 1) / BK;
  unsigned long long* tr = a.trace ? a.trace + 10 * (size_t)blockIdx.x : nullptr;
  if (tr && threadIdx.x == 0) tr[0] = gtimer();

  if (threadIdx.x == 0) {
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
  if (tr && threadIdx.x == 0) tr[1] = gtimer();

  if (warp == 0) {
    if (lane == 0) {
      for (int kb = 0; kb < nkb; ++kb) {
        const int st = kb % STAGES;
        if (kb >= STAGES) mbar_wait(&empty[st], ((kb / STAGES) - 1) & 1);
        uint8_t* sa = smem + st * STAGE_BYTES;
        mbar_arrive_expect_tx(&full[st], STAGE_BYTES);
        bulk_load(sa, a.px + ((int64_t)tm * nkb + kb) * (S * A_TILE), S * A_TILE, &full[st]);
        bulk_load(sa + S * A_TILE, a.py + ((int64_t)tn * nkb + kb) * (S * B_TILE), S * B_TILE, &full[st]);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      for (int kb = 0; kb < nkb; ++kb) {
        const int st = kb % STAGES;
        mbar_wait(&full[st], (kb / STAGES) & 1);
        tmem_fence_after();
        if (tr && kb == 0) tr[2] = gtimer();
        const uint8_t* sa = smem + st * STAGE_BYTES;
        const uint8_t* sb = sa + S * A_TILE;
        // X digit plane s meets Y planes t = 0..S-1-s. The Y planes are consecutive 64-row
        // blocks of one K-major operand (all unsigned: plane 0 carries a +128 offset) and their
        // accumulators (anti-diagonals s+t) are consecutive 64-column TMEM blocks, so one MMA
        // with N = 64 * #planes (<= 256) covers up to 4 pairs: S(S+1)/2 pairs in
        // sum_s ceil((S-s)/4) MMAs, each reading its X plane once.
#pragma unroll
        for (int s = 0; s < S; ++s) {
          const uint64_t da = smem_desc_sw32(sa + s * A_TILE);
          const uint32_t acc = (kb > 0 || s > 0) ? 1u : 0u;
#pragma unroll
          for (int t0 = 0; t0 < S - s; t0 += 4) {
            const int cnt = (S - s - t0) < 4 ? (S - s - t0) : 4;
            mma_i8(tmem + (uint32_t)((s + t0) * BN), da, smem_desc_sw32(sb + t0 * B_TILE),
                   idesc_i8(cnt * BN, s == 0, false), acc);
          }
        }
        mma_commit(&empty[st]);  // frees the stage once these MMAs have read it
      }
      mma_commit(tmem_full);
      if (tr) tr[3] = gtimer();
    }
  }
  __syncwarp();
  {
    // epilogue (all 8 warps): warp w reads TMEM lanes 32*(w%4)..+31 (one output row per thread)
    // and column half w/4, forms 16 columns at a time, stages them in shared memory (the
    // operand ring is idle once every MMA has completed) and writes them back
    // row-contiguously: 4 rows of 128 bytes per warp instruction.
    const int q = warp & 3, half = warp >> 2;
    const int row = tm * BM + q * 32 + lane;
    mbar_wait_sleep(tmem_full, 0);  // the whole main loop: back off, leave issue slots to the MMA / TMA warps
    tmem_fence_after();
    if (tr && warp == 2 && lane == 0) tr[4] = gtimer();
    const uint32_t tl = tmem + ((uint32_t)(q * 32) << 16);
    const bool row_ok = row < a.M;
    const int e = row_ok ? a.ex[row] : 0;
    // Exact integer recombination: with acc'_d = acc_d - 128 * rowsum(a_d) (the +128 offset of
    // Y's plane 0 taken back out), v = sum_d acc'_d 2^(-8d) = 2^-24 (hi + 2^-32 lo) where
    // hi = sum_{d<4} acc'_d 2^(8(3-d)) and lo = sum_{d>=4} acc'_d 2^(8(7-d)) are exact int64
    // (|acc'| < 2^32: < 2^57); two int64 -> FP64 conversions and one FMA instead of a serial
    // S-step FP64 Horner chain per element.
    long long chi = 0, clo = 0;
#pragma unroll
    for (int d = 0; d < S; ++d) {
      const long long c = row_ok ? 128ll * a.rs[(int64_t)d * a.M + row] : 0ll;
      if (d < 4) chi += c << (8 * (3 - d));
      else clo += c << (8 * (7 - d));
    }
    // P = 2^-24 (hi + 2^-32 lo) * 2^(e - 7) * 2^(f - 7): exact power-of-two scaling while normal
    const bool e_fast = e > -900 && e < 900;
    const double escale = e_fast ? __longlong_as_double((long long)(e - 7 - 24 + 1023) << 52) : 0.0;
    double* stage = reinterpret_cast<double*>(smem) + warp * (32 * 18);  // [32 rows][18] doubles per warp
    // column exponents of this warp's 32 columns: one coalesced load, shuffled out per element
    const int mycol = tn * BN + half * (BN / 2) + lane;
    const int fl = mycol < a.N ? a.fy[mycol] : 0;
#pragma unroll 1
    for (int c0 = half * (BN / 2); c0 < (half + 1) * (BN / 2); c0 += 16) {
      // diagonals two at a time (bounded registers): hi/lo accumulate in int64
      long long hi[16], lo[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) hi[j] = lo[j] = 0;
#pragma unroll
      for (int d0 = 0; d0 < S; d0 += 2) {
        uint32_t r[2][16];
        tmem_ld16(tl + (uint32_t)(d0 * BN + c0), r[0]);
        if (d0 + 1 < S) tmem_ld16(tl + (uint32_t)((d0 + 1) * BN + c0), r[1]);
        tmem_wait_ld();
#pragma unroll
        for (int dd = 0; dd < 2; ++dd) {
          const int d = d0 + dd;
          if (d >= S) break;
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const long long x = (long long)(int32_t)r[dd][j];
            if (d < 4) hi[j] += x << (8 * (3 - d));
            else lo[j] += x << (8 * (7 - d));
          }
        }
      }
      if (tr && warp == 2 && lane == 0 && c0 == 0) tr[7] = gtimer();
      double p[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const double v = fma((double)(lo[j] - clo), 2.3283064365386963e-10 /* 2^-32 */, (double)(hi[j] - chi));
        const int f = __shfl_sync(0xffffffffu, fl, (c0 & 16) + j);
        const bool fast = e_fast && f > -900 && f < 900;
        p[j] = (v * escale) * __longlong_as_double((long long)((fast ? f : 0) - 7 + 1023) << 52);
        if (!fast)  // rare: extreme exponents (exact ldexp) or non-finite operands (NaN)
          p[j] = (e == EXP_NONFINITE || f == EXP_NONFINITE) ? __longlong_as_double(0x7ff8000000000000ll)
                                                              : ldexp(v, e + f - 38);
      }
      // stage: lane = row, 16 doubles as 8 x 16-byte stores (row pitch 144 B: conflict-free)
#pragma unroll
      for (int j = 0; j < 16; j += 2)
        *reinterpret_cast<double2*>(stage + lane * 18 + j) = make_double2(p[j], p[j + 1]);
      __syncwarp();
      if (tr && warp == 2 && lane == 0 && c0 == 0) tr[8] = gtimer();
      // write back: lanes 8*i + c -> row rr + i, columns c0 + 2c, c0 + 2c + 1
      const int cc = 2 * (lane & 7), col = tn * BN + c0 + cc;
      double2 v[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = *reinterpret_cast<const double2*>(stage + (4 * i + (lane >> 3)) * 18 + cc);
      const int64_t r0 = tm * BM + q * 32 + (lane >> 3);
      for (int t = 0; t < a.nd; ++t) {
        const OzDest dd = a.d[t];
        double* base = a.C + (r0 + dd.row) * a.ldc + dd.col + col;
        const bool vec = col + 1 < a.N && ((reinterpret_cast<uintptr_t>(base) | (uintptr_t)(a.ldc * 8)) & 15) == 0;
        if (vec && dd.accumulate) {
          double2 c[8];
#pragma unroll
          for (int i = 0; i < 8; ++i)
            if (r0 + 4 * i < a.M) c[i] = *reinterpret_cast<const double2*>(base + 4 * i * a.ldc);
#pragma unroll
          for (int i = 0; i < 8; ++i)
            if (r0 + 4 * i < a.M)
              *reinterpret_cast<double2*>(base + 4 * i * a.ldc) =
                  make_double2(fma(dd.sign, v[i].x, c[i].x), fma(dd.sign, v[i].y, c[i].y));
        } else if (vec) {
#pragma unroll
          for (int i = 0; i < 8; ++i)
            if (r0 + 4 * i < a.M)
              *reinterpret_cast<double2*>(base + 4 * i * a.ldc) = make_double2(dd.sign * v[i].x, dd.sign * v[i].y);
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            if (r0 + 4 * i >= a.M) continue;
            double* d0 = base + 4 * i * a.ldc;
            if (col < a.N) d0[0] = dd.accumulate ? fma(dd.sign, v[i].x, d0[0]) : dd.sign * v[i].x;
            if (col + 1 < a.N) d0[1] = dd.accumulate ? fma(dd.sign, v[i].y, d0[1]) : dd.sign * v[i].y;
          }
        }
      }
      __syncwarp();
      if (tr && warp == 2 && lane == 0 && c0 == 0) tr[9] = gtimer();
    }
  }
  if (tr && warp == 2 && lane == 0) tr[5] = gtimer();
  tmem_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 512);
  if (tr && threadIdx.x == 0) tr[6] = gtimer();
}

// ---------------------------------------------------------------------------------------------
// Persistent variant: one CTA per SM walks tiles t = blockIdx.x, += gridDim.x. The TMA warp
// streams k-stages across tile boundaries (the next tile's first stages land during the
// epilogue); the epilogue warps drain TMEM into FP64 registers, release it (tmem_empty) so the
// next tile's MMAs start, and only then write C -- the stores overlap the next main loop.
// ---------------------------------------------------------------------------------------------
constexpr int PT_THREADS = 320;  // warp 0 TMA, warp 1 MMA issuer + TMEM owner, warps 2-9 epilogue

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t* v) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(taddr)
               : "memory");
}

__device__ __forceinline__ void map_tile(const Args& a, int t, int& tm, int& tn) {
  const int tiles_m = (a.M + BM - 1) / BM, g = MK_OZ_GROUP;
  const int per_group = g * a.tiles_n, grp = t / per_group, first = grp * g;
  const int rows = min(g, tiles_m - first), local = t - grp * per_group;
  tm = first + local % rows;
  tn = local / rows;
}

// Item lookup for the batched form: the tiles of item i are [tile_start[i], tile_start[i+1]).
__device__ __forceinline__ int find_item(const int* __restrict__ tile_start, int nitems, int t) {
  int lo = 0, hi = nitems - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (__ldg(tile_start + mid) <= t) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// BATCH: the tiles of several products (one colour group of leaves: disjoint destinations) in
// one launch, each product's Args in global memory; otherwise one product, Args by value.
template <int S, bool BATCH>
__global__ void __launch_bounds__(PT_THREADS, 1)
    ozaki_persistent_kernel(const __grid_constant__ Args a0, const Args* __restrict__ items,
                            const int* __restrict__ tile_start, int nitems, int tiles) {
  constexpr int A_TILE = BM * BK;
  constexpr int B_TILE = BN * BK;
  constexpr int STAGE_BYTES = S * (A_TILE + B_TILE);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tmem_full = empty + STAGES;
  uint64_t* tmem_empty = tmem_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 1);

  // (item args, tile index inside the item) of global tile t
  auto item_of = [&](int t, int& lt) -> const Args& {
    if (!BATCH) {
      lt = t;
      return a0;
    }
    const int i = find_item(tile_start, nitems, t);
    lt = t - __ldg(tile_start + i);
    return items[i];
  };

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(tmem_full, 1);
    mbar_init(tmem_empty, 8);  // one arrival per epilogue warp
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int it = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
        int lt;
        const Args& a = item_of(t, lt);
        int tm, tn;
        map_tile(a, lt, tm, tn);
        const int nkb = (a.K + BK - 1) / BK;
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int st = it % STAGES;
          if (it >= STAGES) mbar_wait(&empty[st], ((it / STAGES) - 1) & 1);
          uint8_t* sa = smem + st * STAGE_BYTES;
          mbar_arrive_expect_tx(&full[st], STAGE_BYTES);
          bulk_load(sa, a.px + ((int64_t)tm * nkb + kb) * (S * A_TILE), S * A_TILE, &full[st]);
          bulk_load(sa + S * A_TILE, a.py + ((int64_t)tn * nkb + kb) * (S * B_TILE), S * B_TILE, &full[st]);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      int it = 0, ti = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++ti) {
        int lt;
        const Args& a = item_of(t, lt);
        const int nkb = (a.K + BK - 1) / BK;
        if (ti > 0) {  // the epilogue has drained the previous tile's accumulators
          mbar_wait(tmem_empty, (ti - 1) & 1);
          tmem_fence_after();
        }
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int st = it % STAGES;
          mbar_wait(&full[st], (it / STAGES) & 1);
          tmem_fence_after();
          const uint8_t* sa = smem + st * STAGE_BYTES;
          const uint8_t* sb = sa + S * A_TILE;
#pragma unroll
          for (int s = 0; s < S; ++s) {
            const uint64_t da = smem_desc_sw32(sa + s * A_TILE);
            const uint32_t acc = (kb > 0 || s > 0) ? 1u : 0u;
#pragma unroll
            for (int t0 = 0; t0 < S - s; t0 += 4) {
              const int cnt = (S - s - t0) < 4 ? (S - s - t0) : 4;
              mma_i8(tmem + (uint32_t)((s + t0) * BN), da, smem_desc_sw32(sb + t0 * B_TILE),
                     idesc_i8(cnt * BN, s == 0, false), acc);
            }
          }
          mma_commit(&empty[st]);
        }
        mma_commit(tmem_full);
      }
    }
  } else {
    // epilogue warps 2..9: lane quarter q = warp % 4 (TMEM lanes 32q..), column half = (warp-2)/4
    const int q = warp & 3, half = (warp - 2) >> 2;
    int ti = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++ti) {
      int lt;
      const Args& a = item_of(t, lt);
      int tm, tn;
      map_tile(a, lt, tm, tn);
      const int row = tm * BM + q * 32 + lane;
      const bool row_ok = row < a.M;
      const int e = row_ok ? a.ex[row] : 0;
      long long chi = 0, clo = 0;
#pragma unroll
      for (int d = 0; d < S; ++d) {
        const long long c = row_ok ? 128ll * a.rs[(int64_t)d * a.M + row] : 0ll;
        if (d < 4) chi += c << (8 * (3 - d));
        else clo += c << (8 * (7 - d));
      }
      const bool e_fast = e > -900 && e < 900;
      const double escale = e_fast ? __longlong_as_double((long long)(e - 7 - 24 + 1023) << 52) : 0.0;
      const int col0 = tn * BN + half * (BN / 2);
      const int fl = col0 + lane < a.N ? a.fy[col0 + lane] : 0;
      mbar_wait_sleep(tmem_full, ti & 1);
      tmem_fence_after();
      const uint32_t tl = tmem + ((uint32_t)(q * 32) << 16);
      double p[BN / 2];
#pragma unroll
      for (int c8 = 0; c8 < BN / 2; c8 += 8) {
        long long hi[8], lo[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) hi[j] = lo[j] = 0;
#pragma unroll
        for (int d0 = 0; d0 < S; d0 += 2) {
          uint32_t r[2][8];
          tmem_ld8(tl + (uint32_t)(d0 * BN + half * (BN / 2) + c8), r[0]);
          if (d0 + 1 < S) tmem_ld8(tl + (uint32_t)((d0 + 1) * BN + half * (BN / 2) + c8), r[1]);
          tmem_wait_ld();
#pragma unroll
          for (int dd = 0; dd < 2; ++dd) {
            const int d = d0 + dd;
            if (d >= S) break;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const long long x = (long long)(int32_t)r[dd][j];
              if (d < 4) hi[j] += x << (8 * (3 - d));
              else lo[j] += x << (8 * (7 - d));
            }
          }
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const double v = fma((double)(lo[j] - clo), 2.3283064365386963e-10, (double)(hi[j] - chi));
          const int f = __shfl_sync(0xffffffffu, fl, c8 + j);
          const bool fast = e_fast && f > -900 && f < 900;
          double pj = (v * escale) * __longlong_as_double((long long)((fast ? f : 0) - 7 + 1023) << 52);
          if (!fast)
            pj = (e == EXP_NONFINITE || f == EXP_NONFINITE) ? __longlong_as_double(0x7ff8000000000000ll)
                                                            : ldexp(v, e + f - 38);
          p[c8 + j] = pj;
        }
      }
      tmem_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tmem_empty);  // accumulators free: the next tile's MMAs may start
      // write back (overlaps the next tile's main loop): this thread's row, 32 columns
      if (row_ok && a.slabs.n > 0) {  // fused reduce-scatter: owner slab rows, atomic adds (RED.ADD.F64)
        for (int d = 0; d < a.nd; ++d) {
          const OzDest dd = a.d[d];
          const int64_t R = dd.row + row, o = R / a.slabs.rows;
          double* dst = a.slabs.p[o] + (R - o * a.slabs.rows) * a.ldc + dd.col + col0;
#pragma unroll
          for (int j = 0; j < BN / 2; ++j)
            if (col0 + j < a.N) atomicAdd(dst + j, dd.sign * p[j]);
        }
      } else if (row_ok) {
        double* crow = a.C + (int64_t)row * a.ldc;
        for (int d = 0; d < a.nd; ++d) {
          const OzDest dd = a.d[d];
          double* dst = crow + dd.row * a.ldc + dd.col + col0;
          const bool vec = col0 + BN / 2 <= a.N && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0);
          if (vec) {
#pragma unroll
            for (int j = 0; j < BN / 2; j += 2) {
              double2* p2 = reinterpret_cast<double2*>(dst + j);
              double2 o = make_double2(dd.sign * p[j], dd.sign * p[j + 1]);
              if (dd.accumulate) {
                const double2 c = *p2;
                o = make_double2(fma(dd.sign, p[j], c.x), fma(dd.sign, p[j + 1], c.y));
              }
              *p2 = o;
            }
          } else {
#pragma unroll
            for (int j = 0; j < BN / 2; ++j)
              if (col0 + j < a.N) dst[j] = dd.accumulate ? fma(dd.sign, p[j], dst[j]) : dd.sign * p[j];
          }
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

// x * 2^-e = y in (-1, 1) is written as 2^-7 * sum_s d_s 2^(-8s): d_0 = floor(128 y) in
// [-128, 127] (signed plane), then d_s in [0, 255] the floor digits of the remainder (unsigned
// planes): 7 + 8 (S - 1) bits. These are exactly the bytes of the two's-complement integer
// floor(y * 2^63) (|y * 2^63| < 2^63; the power-of-two scaling is exact; truncating the low
// bytes is the floor at S digits), so one floor conversion per element yields all S digits.
// scale = 2^(63 - e). OFFSET: plane 0 stored as d_0 + 128 (top bit flipped) for the Y side.
// dsum (may be null): per-plane sums of the 4 digits (signed plane 0), for the row sums.
// scale = s1 * s2 (two factors: 2^(63 - e) overflows a double for row maxima below 2^-960;
// each product stays exact).
template <int S, bool OFFSET>
__device__ __forceinline__ void digits4(const double x[4], double s1, double s2, uint32_t out[S], int* dsum) {
  unsigned long long v[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) v[i] = (unsigned long long)__double2ll_rd((x[i] * s1) * s2);
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const int sh = 8 * (7 - s);
    uint32_t w = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) w |= (uint32_t)((v[i] >> sh) & 0xff) << (8 * i);
    if (dsum) {
      if (s == 0)
        dsum[0] += (int)(int8_t)(w & 0xff) + (int)(int8_t)((w >> 8) & 0xff) + (int)(int8_t)((w >> 16) & 0xff) +
                   (int)(int8_t)(w >> 24);
      else
        dsum[s] += (int)(w & 0xff) + (int)((w >> 8) & 0xff) + (int)((w >> 16) & 0xff) + (int)(w >> 24);
    }
    out[s] = (OFFSET && s == 0) ? (w ^ 0x80808080u) : w;
  }
}

// Operand value at (r, c): the signed sum of up to 4 blocks of one base (the Strassen / Winograd
// pre-addition, formed on load instead of materialised), in table order.
// NT = o.n as a template parameter: the term loop unrolls, so unrolled element loops keep several
// independent loads in flight.
template <int NT>
__device__ __forceinline__ double term_sum(const OzOperand& o, int64_t r, int64_t c) {
  const int64_t off = r * o.ld + c;
  double v = o.s[0] * o.p[0][off];
#pragma unroll
  for (int i = 1; i < NT; ++i) v = fma(o.s[i], o.p[i][off], v);
  return v;
}

// Row maxima of X as IEEE bit patterns (monotone for |x|; inf / nan -> +inf): one warp per
// (row, 1024-wide k chunk), 8 independent loads in flight per lane, one atomicMax per warp.
template <int NT>
__device__ __forceinline__ void rowmax_body(const OzOperand& X, int rows, int K, unsigned long long* __restrict__ rmax) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= rows) return;
  const int k0 = blockIdx.y * 1024, k1 = min(K, k0 + 1024);
  double m[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) m[i] = 0.0;
  bool bad = false;
  for (int k = k0 + lane; k < k1; k += 256) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int kk = k + 32 * i;
      const double v = kk < k1 ? fabs(term_sum<NT>(X, warp, kk)) : 0.0;
      bad |= !(v <= 1.7976931348623157e308);
      m[i] = fmax(m[i], v);
    }
  }
  double mx = fmax(fmax(fmax(m[0], m[1]), fmax(m[2], m[3])), fmax(fmax(m[4], m[5]), fmax(m[6], m[7])));
#pragma unroll
  for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  bad = __any_sync(0xffffffffu, bad);
  if (lane == 0)
    atomicMax(&rmax[warp], bad ? 0x7ff0000000000000ull : (unsigned long long)__double_as_longlong(mx));
}

// X rows -> exponents, digit row sums and S digit planes in the product kernel's tile images
// ([tile_m][kb][S][128 x 32 B], swizzled): one warp per row (rows up to the padded tile edge
// write zeros), each lane 4 consecutive k per step, 4 steps in flight.
template <int S, int NT>
__device__ __forceinline__ void split_rows_body(const OzOperand& X, int rows, int rows_pad, int K, int nkb,
                                  const unsigned long long* __restrict__ rmax, int32_t* __restrict__ ex,
                                  int32_t* __restrict__ rs, uint8_t* __restrict__ planes) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= rows_pad) return;
  const bool live = warp < rows;
  const int e = live ? row_exponent(__longlong_as_double((long long)rmax[warp])) : 0;
  if (lane == 0 && live) ex[warp] = e;
  const int sh = 63 - e, sh1 = sh < 1000 ? sh : 1000;
  const double scale = (e == EXP_NONFINITE) ? 0.0 : ldexp(1.0, sh1), scale2 = ldexp(1.0, sh - sh1);
  const bool load = live && e != EXP_NONFINITE;
  const int tmi = warp / BM, r = warp % BM;
  uint8_t* base = planes + (int64_t)tmi * nkb * (S * BM * BK);
  int dsum[S];
#pragma unroll
  for (int s = 0; s < S; ++s) dsum[s] = 0;
  const int kp = nkb * BK;
#pragma unroll 4
  for (int k0 = 4 * lane; k0 < kp; k0 += 128) {
    double x[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) x[i] = (load && k0 + i < K) ? term_sum<NT>(X, warp, k0 + i) : 0.0;
    uint32_t w[S];
    digits4<S, false>(x, scale, scale2, w, dsum);
    uint8_t* t = base + (int64_t)(k0 / BK) * (S * BM * BK) + swz32(r, k0 % BK);
#pragma unroll
    for (int s = 0; s < S; ++s) *reinterpret_cast<uint32_t*>(t + s * (BM * BK)) = w[s];
  }
#pragma unroll
  for (int s = 0; s < S; ++s) {
    int v = dsum[s];  // |sum| <= K * 255 < 2^31
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0 && live) rs[(int64_t)s * rows + warp] = v;
  }
}

// Column maxima of Y (k x n) as IEEE bit patterns (monotone for |y|): grid (n/256, k/64).
template <int NT>
__device__ __forceinline__ void colmax_body(const OzOperand& Y, int K, int N, unsigned long long* __restrict__ cmax) {
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= N) return;
  const int k0 = blockIdx.y * 64, k1 = min(K, k0 + 64);
  double mx = 0.0, m2 = 0.0;
  bool bad = false;
  int k = k0;
#pragma unroll 4
  for (; k + 1 < k1; k += 2) {
    const double y1 = fabs(term_sum<NT>(Y, k, col)), y2 = fabs(term_sum<NT>(Y, k + 1, col));
    bad |= !(y1 <= 1.7976931348623157e308) | !(y2 <= 1.7976931348623157e308);
    mx = fmax(mx, y1);
    m2 = fmax(m2, y2);
  }
  if (k < k1) {
    const double y = fabs(term_sum<NT>(Y, k, col));
    bad |= !(y <= 1.7976931348623157e308);
    mx = fmax(mx, y);
  }
  mx = fmax(mx, m2);
  const unsigned long long bits = bad ? 0x7ff0000000000000ull : (unsigned long long)__double_as_longlong(mx);
  atomicMax(&cmax[col], bits);
}

__device__ __forceinline__ void colexp_body(const unsigned long long* __restrict__ cmax, int N, int32_t* __restrict__ fy) {
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= N) return;
  fy[col] = row_exponent(__longlong_as_double((long long)cmax[col]));
}

// Y (k x n, row-major) -> S digit planes of Y^T in the product kernel's tile images
// ([tile_n][kb][S][64 x 32 B], swizzled; K-major for the B operand), 32 x 32 tiles through shared
// memory. Block (32, 8); the grid covers the padded tile edges (zeros).
template <int S, int NT>
__device__ __forceinline__ void split_cols_body(const OzOperand& Y, int K, int N, int nkb, const int32_t* __restrict__ fy,
                                  uint8_t* __restrict__ planes) {
  __shared__ uint32_t sm[S][32][9];  // [plane][col][k/4] (+1 pad)
  const int n0 = blockIdx.x * 32, k0 = blockIdx.y * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int col = n0 + tx;
  const int f = col < N ? fy[col] : 0;
  const int sh = 63 - f, sh1 = sh < 1000 ? sh : 1000;
  const double scale = (col < N && f != EXP_NONFINITE) ? ldexp(1.0, sh1) : 0.0, scale2 = ldexp(1.0, sh - sh1);
  // thread (tx, ty) converts k = k0 + 4*ty .. +3 of column col
  double x[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int k = k0 + 4 * ty + i;
    x[i] = (col < N && k < K && scale != 0.0) ? term_sum<NT>(Y, k, col) : 0.0;
  }
  uint32_t w[S];
  digits4<S, true>(x, scale, scale2, w, nullptr);
  if (col >= N) {  // padded columns: zero digits (not the +128 offset)
#pragma unroll
    for (int s = 0; s < S; ++s) w[s] = 0;
  }
#pragma unroll
  for (int s = 0; s < S; ++s) sm[s][tx][ty] = w[s];
  __syncthreads();
  // write: 32 rows (n) x 8 words (k) of each plane; 256 threads, one word each
  const int t = ty * 32 + tx;
  const int r = t >> 3, wi = t & 7;
  const int n = n0 + r;
  uint8_t* dst = planes + ((int64_t)(n / BN) * nkb + k0 / BK) * (S * BN * BK) + swz32(n % BN, 4 * wi);
#pragma unroll
  for (int s = 0; s < S; ++s) *reinterpret_cast<uint32_t*>(dst + s * (BN * BK)) = sm[s][r][wi];
}

// Kernels: one product's operands (grid-constant parameters), or a batch of equally shaped
// products (one job per blockIdx.z) -- the leaves of a breadth-first level split with one launch
// per kernel instead of one per leaf.
struct SplitJob {
  OzOperand X, Y;
  unsigned long long *rmax, *cmax;
  int32_t *ex, *fy, *rs;
  uint8_t *px, *py;
};

template <int NT>
__global__ void rowmax_kernel(const OzOperand X, int rows, int K, unsigned long long* __restrict__ rmax) {
  rowmax_body<NT>(X, rows, K, rmax);
}
template <int S, int NT>
__global__ void split_rows_kernel(const OzOperand X, int rows, int rows_pad, int K, int nkb,
                                  const unsigned long long* __restrict__ rmax, int32_t* __restrict__ ex,
                                  int32_t* __restrict__ rs, uint8_t* __restrict__ planes) {
  split_rows_body<S, NT>(X, rows, rows_pad, K, nkb, rmax, ex, rs, planes);
}
template <int NT>
__global__ void colmax_kernel(const OzOperand Y, int K, int N, unsigned long long* __restrict__ cmax) {
  colmax_body<NT>(Y, K, N, cmax);
}
__global__ void colexp_kernel(const unsigned long long* __restrict__ cmax, int N, int32_t* __restrict__ fy) {
  colexp_body(cmax, N, fy);
}
template <int S, int NT>
__global__ void split_cols_kernel(const OzOperand Y, int K, int N, int nkb, const int32_t* __restrict__ fy,
                                  uint8_t* __restrict__ planes) {
  split_cols_body<S, NT>(Y, K, N, nkb, fy, planes);
}

__global__ void zero_max_batch(const SplitJob* __restrict__ jobs, int rows, int cols) {
  const SplitJob& j = jobs[blockIdx.y];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < rows || i < cols; i += gridDim.x * blockDim.x) {
    if (i < rows) j.rmax[i] = 0;
    if (i < cols) j.cmax[i] = 0;
  }
}
template <int NT>
__global__ void rowmax_batch(const SplitJob* __restrict__ jobs, int rows, int K) {
  const SplitJob& j = jobs[blockIdx.z];
  rowmax_body<NT>(j.X, rows, K, j.rmax);
}
template <int S, int NT>
__global__ void split_rows_batch(const SplitJob* __restrict__ jobs, int rows, int rows_pad, int K, int nkb) {
  const SplitJob& j = jobs[blockIdx.z];
  split_rows_body<S, NT>(j.X, rows, rows_pad, K, nkb, j.rmax, j.ex, j.rs, j.px);
}
template <int NT>
__global__ void colmax_batch(const SplitJob* __restrict__ jobs, int K, int N) {
  const SplitJob& j = jobs[blockIdx.z];
  colmax_body<NT>(j.Y, K, N, j.cmax);
}
__global__ void colexp_batch(const SplitJob* __restrict__ jobs, int N) {
  const SplitJob& j = jobs[blockIdx.z];
  colexp_body(j.cmax, N, j.fy);
}
template <int S, int NT>
__global__ void split_cols_batch(const SplitJob* __restrict__ jobs, int K, int N, int nkb) {
  const SplitJob& j = jobs[blockIdx.z];
  split_cols_body<S, NT>(j.Y, K, N, nkb, j.fy, j.py);
}

// ---------------------------------------------------------------------------------------------
// Host side
// ---------------------------------------------------------------------------------------------
static int64_t kpad(int64_t k) { return (k + KPAD - 1) / KPAD * KPAD; }
static size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

struct Layout {
  size_t planes_x, planes_y, ex, fy, cmax, rs, rmax, total;
};
static Layout layout(int64_t m, int64_t n, int64_t k, int S) {
  Layout L;
  const int64_t kp = kpad(k);
  const int64_t mp = (m + BM - 1) / BM * BM, np = (n + BN - 1) / BN * BN;
  L.planes_x = 0;
  L.planes_y = align256(L.planes_x + (size_t)S * mp * kp);
  L.ex = align256(L.planes_y + (size_t)S * np * kp);
  L.fy = align256(L.ex + 4 * (size_t)m);
  L.cmax = align256(L.fy + 4 * (size_t)n);
  L.rs = align256(L.cmax + 8 * (size_t)n);
  L.rmax = align256(L.rs + 4 * (size_t)S * m);
  L.total = align256(L.rmax + 8 * (size_t)m);
  return L;
}

// K per call: the whole K when it fits the exact int32 accumulation, else equal chunks
static int64_t chunk_k(int64_t k, int S) {
  const int64_t mx = ozaki_max_k(S) / KPAD * KPAD;
  const int64_t nc = (k + mx - 1) / mx;
  return std::min(mx, kpad((k + nc - 1) / nc));
}

template <int S>
static size_t smem_bytes() {
  return STAGES * S * (BM + BN) * BK + 1024 /*align*/ + 256 /*barriers*/;
}

// One K chunk, phase 1: split both operands into the digit planes / exponents / row sums of ws.
template <int S>
static void split_phase(const OzOperand& X, const OzOperand& Y, int64_t m, int64_t n, int64_t k, uint8_t* ws,
                        cudaStream_t st) {
  const Layout L = layout(m, n, k, S);
  const int64_t kp = kpad(k), nkb = kp / BK;
  const int64_t tiles_m = (m + BM - 1) / BM, tiles_n = (n + BN - 1) / BN;
  uint8_t* px = ws + L.planes_x;
  uint8_t* py = ws + L.planes_y;
  int32_t* ex = reinterpret_cast<int32_t*>(ws + L.ex);
  int32_t* fy = reinterpret_cast<int32_t*>(ws + L.fy);
  auto* cmax = reinterpret_cast<unsigned long long*>(ws + L.cmax);
  int32_t* rs = reinterpret_cast<int32_t*>(ws + L.rs);

  auto* rmax = reinterpret_cast<unsigned long long*>(ws + L.rmax);
  cudaMemsetAsync(rmax, 0, 8 * (size_t)m, st);
  auto x_side = [&](auto nt) {
    constexpr int NT = decltype(nt)::value;
    // 128-thread blocks: they fit in the registers a resident product CTA leaves free, so the
    // splitting of the next leaf can run beside the current product kernel (ozaki_product_batch)
    rowmax_kernel<NT><<<dim3((unsigned)((m * 32 + 127) / 128), (unsigned)((k + 1023) / 1024)), 128, 0, st>>>(
        X, (int)m, (int)k, rmax);
    split_rows_kernel<S, NT><<<(unsigned)((tiles_m * BM * 32 + 127) / 128), 128, 0, st>>>(
        X, (int)m, (int)(tiles_m * BM), (int)k, (int)nkb, rmax, ex, rs, px);
  };
  auto y_side = [&](auto nt) {
    constexpr int NT = decltype(nt)::value;
    colmax_kernel<NT><<<dim3((unsigned)((n + 127) / 128), (unsigned)((k + 63) / 64)), 128, 0, st>>>(Y, (int)k,
                                                                                                  (int)n, cmax);
    colexp_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(cmax, (int)n, fy);
    split_cols_kernel<S, NT><<<dim3((unsigned)(tiles_n * BN / 32), (unsigned)nkb), dim3(32, 8), 0, st>>>(
        Y, (int)k, (int)n, (int)nkb, fy, py);
  };
  switch (X.n) {
    case 1: x_side(std::integral_constant<int, 1>{}); break;
    case 2: x_side(std::integral_constant<int, 2>{}); break;
    case 3: x_side(std::integral_constant<int, 3>{}); break;
    default: x_side(std::integral_constant<int, 4>{}); break;
  }
  cudaMemsetAsync(cmax, 0, 8 * (size_t)n, st);
  switch (Y.n) {
    case 1: y_side(std::integral_constant<int, 1>{}); break;
    case 2: y_side(std::integral_constant<int, 2>{}); break;
    case 3: y_side(std::integral_constant<int, 3>{}); break;
    default: y_side(std::integral_constant<int, 4>{}); break;
  }
}

// Kernel arguments of one product whose digit planes / exponents / row sums live in ws.
static Args make_args(int S, double* C, int64_t ldc, int64_t m, int64_t n, int64_t k, const OzDest* d, int nd,
                      uint8_t* ws, const OzSlabs* slabs) {
  const Layout L = layout(m, n, k, S);
  Args a{};
  a.px = ws + L.planes_x;
  a.py = ws + L.planes_y;
  a.ex = reinterpret_cast<int32_t*>(ws + L.ex);
  a.fy = reinterpret_cast<int32_t*>(ws + L.fy);
  a.rs = reinterpret_cast<int32_t*>(ws + L.rs);
  a.C = C;
  a.ldc = ldc;
  a.M = (int)m;
  a.N = (int)n;
  a.K = (int)k;
  a.tiles_n = (int)((n + BN - 1) / BN);
  a.nd = nd;
  a.pad_ = 0;
  for (int i = 0; i < nd; ++i) a.d[i] = d[i];
  a.slabs = slabs ? *slabs : OzSlabs{0, 1, {nullptr}};
  a.trace = nullptr;
  return a;
}

// Several products (disjoint destinations: one colour group of leaves) in one persistent launch;
// args_dev / tile_start_dev already on the device.
template <int S>
static int product_batch_launch(const Args* args_dev, const int* tile_start_dev, int nitems, int tiles,
                                cudaStream_t st, std::string* err) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const size_t psmem = smem_bytes<S>() + 8;
  cudaError_t e = cudaFuncSetAttribute(ozaki_persistent_kernel<S, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)psmem);
  if (e == cudaSuccess) {
    Args dummy{};
    ozaki_persistent_kernel<S, true><<<std::min(tiles, sms), PT_THREADS, psmem, st>>>(dummy, args_dev, tile_start_dev,
                                                                                       nitems, tiles);
    e = cudaGetLastError();
  }
  if (e != cudaSuccess) {
    *err = std::string("ozaki_persistent_kernel (batch) launch: ") + cudaGetErrorString(e);
    return MK_ERR_CUDA;
  }
  return MK_OK;
}

// One K chunk, phase 2: the product kernel from ws's digit planes into every destination.
template <int S>
static int product_phase(double* C, int64_t ldc, int64_t m, int64_t n, int64_t k, const OzDest* d, int nd,
                         uint8_t* ws, cudaStream_t st, std::string* err, const OzSlabs* slabs = nullptr) {
  Args a = make_args(S, C, ldc, m, n, k, d, nd, ws, slabs);
  const int tiles = (int)((m + BM - 1) / BM) * a.tiles_n;
  const size_t smem = smem_bytes<S>();
  // per launch (the attribute is per device; the call is cheap next to a leaf product)
  cudaError_t ae = cudaFuncSetAttribute(ozaki_product_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (ae != cudaSuccess) {
    *err = std::string("ozaki_product_kernel smem attribute: ") + cudaGetErrorString(ae);
    return MK_ERR_CUDA;
  }
  static const bool trace = getenv("MK_OZ_TRACE") && getenv("MK_OZ_TRACE")[0] == '1';
  a.trace = nullptr;
  static const bool persistent = !(getenv("MK_OZ_PERSISTENT") && getenv("MK_OZ_PERSISTENT")[0] == '0');
  if ((persistent && !trace) || a.slabs.n > 0) {  // slab routing lives in the persistent kernel
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const size_t psmem = smem + 8;
    cudaError_t pe = cudaFuncSetAttribute(ozaki_persistent_kernel<S, false>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)psmem);
    if (pe != cudaSuccess) {
      *err = std::string("ozaki_persistent_kernel smem attribute: ") + cudaGetErrorString(pe);
      return MK_ERR_CUDA;
    }
    ozaki_persistent_kernel<S, false><<<std::min(tiles, sms), PT_THREADS, psmem, st>>>(a, nullptr, nullptr, 1, tiles);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
      *err = std::string("ozaki_persistent_kernel launch: ") + cudaGetErrorString(e);
      return MK_ERR_CUDA;
    }
    return MK_OK;
  }
  if (trace) cudaMalloc(&a.trace, 10 * sizeof(unsigned long long) * tiles);
  ozaki_product_kernel<S><<<tiles, NTHREADS, smem, st>>>(a);
  if (trace) {  // debug: per-phase medians over the tiles, stderr
    std::vector<unsigned long long> h(10 * (size_t)tiles);
    cudaMemcpyAsync(h.data(), a.trace, h.size() * 8, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    cudaFree(a.trace);
    const char* names[6] = {"alloc", "fill", "mainloop", "mma_drain", "epilogue", "teardown"};
    unsigned long long t0 = ~0ull, t1 = 0;
    for (int t = 0; t < tiles; ++t) { t0 = std::min(t0, h[10 * t]); t1 = std::max(t1, h[10 * t + 6]); }
    fprintf(stderr, "ozaki trace S=%d M=%lld N=%lld K=%lld tiles=%d span=%.1f us:", S, (long long)m, (long long)n,
            (long long)k, tiles, (t1 - t0) / 1e3);
    for (int ph = 0; ph < 6; ++ph) {
      std::vector<long long> d(tiles);
      for (int t = 0; t < tiles; ++t) d[t] = ph < 6 ? (long long)h[10 * t + ph + 1] - (long long)h[10 * t + ph] : (long long)h[10 * t + ph + 1] - (long long)h[10 * t + ph];
      std::sort(d.begin(), d.end());
      fprintf(stderr, " %s %.2f", names[ph], d[tiles / 2] / 1e3);
    }
    {
      const char* sub[3] = {"c0_tmem_ld", "c0_compute", "c0_store"};
      const int from[3] = {4, 7, 8};
      for (int ph = 0; ph < 3; ++ph) {
        std::vector<long long> d(tiles);
        for (int t = 0; t < tiles; ++t) d[t] = (long long)h[10 * t + from[ph] + (ph == 0 ? 3 : 1)] - (long long)h[10 * t + from[ph]];
        std::sort(d.begin(), d.end());
        fprintf(stderr, " %s %.2f", sub[ph], d[tiles / 2] / 1e3);
      }
    }
    fprintf(stderr, " (us, medians)\n");
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    *err = std::string("ozaki_product_kernel launch: ") + cudaGetErrorString(e);
    return MK_ERR_CUDA;
  }
  return MK_OK;
}

template <int S>
static int run(const OzOperand& X, const OzOperand& Y, double* C, int64_t ldc, int64_t m, int64_t n, int64_t k,
               const OzDest* d, int nd, uint8_t* ws, cudaStream_t st, std::string* err,
               const OzSlabs* slabs = nullptr) {
  split_phase<S>(X, Y, m, n, k, ws, st);
  return product_phase<S>(C, ldc, m, n, k, d, nd, ws, st, err, slabs);
}

static void split_any(int S, const OzOperand& X, const OzOperand& Y, int64_t m, int64_t n, int64_t k, uint8_t* ws,
                      cudaStream_t st) {
  switch (S) {
    case 4: split_phase<4>(X, Y, m, n, k, ws, st); break;
    case 5: split_phase<5>(X, Y, m, n, k, ws, st); break;
    case 6: split_phase<6>(X, Y, m, n, k, ws, st); break;
    case 7: split_phase<7>(X, Y, m, n, k, ws, st); break;
    default: split_phase<8>(X, Y, m, n, k, ws, st); break;
  }
}
// Digit splitting of `nitems` equally shaped single-term products in one launch per kernel.
template <int S>
static void split_batch_phase(const SplitJob* jobs, int64_t m, int64_t n, int64_t k, int nitems, cudaStream_t st) {
  const int64_t kp = kpad(k), nkb = kp / BK;
  const int64_t tiles_m = (m + BM - 1) / BM, tiles_n = (n + BN - 1) / BN;
  const unsigned z = (unsigned)nitems;
  zero_max_batch<<<dim3((unsigned)((std::max(m, n) + 255) / 256), z), 256, 0, st>>>(jobs, (int)m, (int)n);
  rowmax_batch<1><<<dim3((unsigned)((m * 32 + 127) / 128), (unsigned)((k + 1023) / 1024), z), 128, 0, st>>>(
      jobs, (int)m, (int)k);
  split_rows_batch<S, 1><<<dim3((unsigned)((tiles_m * BM * 32 + 127) / 128), 1, z), 128, 0, st>>>(
      jobs, (int)m, (int)(tiles_m * BM), (int)k, (int)nkb);
  colmax_batch<1><<<dim3((unsigned)((n + 127) / 128), (unsigned)((k + 63) / 64), z), 128, 0, st>>>(jobs, (int)k,
                                                                                                    (int)n);
  colexp_batch<<<dim3((unsigned)((n + 255) / 256), 1, z), 256, 0, st>>>(jobs, (int)n);
  split_cols_batch<S, 1><<<dim3((unsigned)(tiles_n * BN / 32), (unsigned)nkb, z), dim3(32, 8), 0, st>>>(
      jobs, (int)k, (int)n, (int)nkb);
}
static void split_batch_any(int S, const SplitJob* jobs, int64_t m, int64_t n, int64_t k, int nitems,
                            cudaStream_t st) {
  switch (S) {
    case 4: split_batch_phase<4>(jobs, m, n, k, nitems, st); break;
    case 5: split_batch_phase<5>(jobs, m, n, k, nitems, st); break;
    case 6: split_batch_phase<6>(jobs, m, n, k, nitems, st); break;
    case 7: split_batch_phase<7>(jobs, m, n, k, nitems, st); break;
    default: split_batch_phase<8>(jobs, m, n, k, nitems, st); break;
  }
}
static SplitJob split_job(int S, const OzOperand& X, const OzOperand& Y, int64_t m, int64_t n, int64_t k,
                          uint8_t* ws) {
  const Layout L = layout(m, n, k, S);
  SplitJob j;
  j.X = X;
  j.Y = Y;
  j.rmax = reinterpret_cast<unsigned long long*>(ws + L.rmax);
  j.cmax = reinterpret_cast<unsigned long long*>(ws + L.cmax);
  j.ex = reinterpret_cast<int32_t*>(ws + L.ex);
  j.fy = reinterpret_cast<int32_t*>(ws + L.fy);
  j.rs = reinterpret_cast<int32_t*>(ws + L.rs);
  j.px = ws + L.planes_x;
  j.py = ws + L.planes_y;
  return j;
}

static int batch_launch_any(int S, const Args* args_dev, const int* tile_start_dev, int nitems, int tiles,
                            cudaStream_t st, std::string* err) {
  switch (S) {
    case 4: return product_batch_launch<4>(args_dev, tile_start_dev, nitems, tiles, st, err);
    case 5: return product_batch_launch<5>(args_dev, tile_start_dev, nitems, tiles, st, err);
    case 6: return product_batch_launch<6>(args_dev, tile_start_dev, nitems, tiles, st, err);
    case 7: return product_batch_launch<7>(args_dev, tile_start_dev, nitems, tiles, st, err);
    default: return product_batch_launch<8>(args_dev, tile_start_dev, nitems, tiles, st, err);
  }
}
static int product_any(int S, double* C, int64_t ldc, int64_t m, int64_t n, int64_t k, const OzDest* d, int nd,
                       uint8_t* ws, cudaStream_t st, std::string* err) {
  switch (S) {
    case 4: return product_phase<4>(C, ldc, m, n, k, d, nd, ws, st, err);
    case 5: return product_phase<5>(C, ldc, m, n, k, d, nd, ws, st, err);
    case 6: return product_phase<6>(C, ldc, m, n, k, d, nd, ws, st, err);
    case 7: return product_phase<7>(C, ldc, m, n, k, d, nd, ws, st, err);
    default: return product_phase<8>(C, ldc, m, n, k, d, nd, ws, st, err);
  }
}

// Whole product: K in chunks of chunk_k (later chunks accumulate into every destination).
static int product_chunks(const OzOperand& X, const OzOperand& Y, double* C, int64_t ldc, int64_t m, int64_t n,
                          int64_t k, int S, const OzDest* d, int nd, uint8_t* ws, cudaStream_t st, std::string* err,
                          const OzSlabs* slabs = nullptr) {
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
      case 4: rc = run<4>(Xc, Yc, C, ldc, m, n, kk, dd, nd, ws, st, err, slabs); break;
      case 5: rc = run<5>(Xc, Yc, C, ldc, m, n, kk, dd, nd, ws, st, err, slabs); break;
      case 6: rc = run<6>(Xc, Yc, C, ldc, m, n, kk, dd, nd, ws, st, err, slabs); break;
      case 7: rc = run<7>(Xc, Yc, C, ldc, m, n, kk, dd, nd, ws, st, err, slabs); break;
      default: rc = run<8>(Xc, Yc, C, ldc, m, n, kk, dd, nd, ws, st, err, slabs); break;
    }
    if (rc != MK_OK) return rc;
    for (int i = 0; i < nd; ++i) dd[i].accumulate = 1;
  }
  return MK_OK;
}

}  // namespace oz

int64_t ozaki_max_k(int slices) {
  // anti-diagonal d = S-1 sums per k one signed x unsigned pair (|.| <= 128 * 255) and S-1
  // unsigned x unsigned pairs (<= 255^2, Y's plane 0 offset included); the int32 accumulator
  // must hold K of them
  const int64_t worst = 128 * 255 + (int64_t)(slices - 1) * 255 * 255;
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

// Per thread and device: the side stream the digit splitting runs on beside the product kernels.
static cudaStream_t side_stream(int dev) {
  static thread_local std::map<int, cudaStream_t> side_streams;
  auto itx = side_streams.find(dev);
  if (itx == side_streams.end()) {
    cudaStream_t s2;
    if (cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking) != cudaSuccess) {
      cudaGetLastError();
      s2 = nullptr;
    }
    itx = side_streams.emplace(dev, s2).first;
  }
  return itx->second;
}

static void keep_pool_memory() {  // freed leaf workspaces stay in the stream-ordered pool
  static thread_local int pool_dev = -1;
  int dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess && dev != pool_dev) {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    pool_dev = dev;
  }
}

// Grouped form of ozaki_product_batch (every item one K chunk): the items of a launch group (equal
// OzItem::group, disjoint destinations) are split into one workspace and multiplied by ONE
// persistent launch over all their tiles -- small leaves fill the GPU together; the next group's
// splitting runs on the side stream meanwhile (two group workspaces).
static int batch_grouped(const OzItem* items, int count, int slices, cudaStream_t st, cudaStream_t side,
                         std::string* err) {
  constexpr size_t kMaxGroupBytes = size_t(4) << 30;
  struct Grp {
    int b, e;
    size_t bytes;
  };
  std::vector<Grp> groups;
  for (int i = 0; i < count; ++i) {
    const size_t wb = oz::align256(ozaki_workspace_bytes(items[i].m, items[i].n, items[i].k, slices));
    if (groups.empty() || items[i].group != items[groups.back().b].group || groups.back().bytes + wb > kMaxGroupBytes)
      groups.push_back(Grp{i, i, 0});
    groups.back().e = i + 1;
    groups.back().bytes += wb;
  }
  size_t maxb = 0;
  for (const Grp& g : groups) maxb = std::max(maxb, g.bytes);
  const int nbuf = (groups.size() > 1 && side) ? 2 : 1;
  uint8_t* ws[2] = {nullptr, nullptr};
  for (int b = 0; b < nbuf; ++b) {
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&ws[b]), maxb, st);
    if (e != cudaSuccess) {
      cudaGetLastError();
      for (int j = 0; j < b; ++j) cudaFreeAsync(ws[j], st);
      *err = std::string("Ozaki batch workspace: ") + cudaGetErrorString(e);
      return e == cudaErrorMemoryAllocation ? MK_ERR_WORKSPACE : MK_ERR_CUDA;
    }
  }
  cudaEvent_t start = nullptr, split_ev[2] = {nullptr, nullptr}, prod_ev[2] = {nullptr, nullptr};
  auto mkev = [](cudaEvent_t* e) { return cudaEventCreateWithFlags(e, cudaEventDisableTiming); };
  if (nbuf == 2) {
    if (mkev(&start) || mkev(&split_ev[0]) || mkev(&split_ev[1]) || mkev(&prod_ev[0]) || mkev(&prod_ev[1])) {
      cudaGetLastError();
      side = nullptr;
    } else {
      cudaEventRecord(start, st);
      cudaStreamWaitEvent(side, start, 0);
    }
  }
  const bool use_side = nbuf == 2 && side;
  int rc = MK_OK;
  for (size_t gi = 0; gi < groups.size() && rc == MK_OK; ++gi) {
    const Grp& g = groups[gi];
    const int b = (int)(gi % nbuf);
    cudaStream_t ss = use_side ? side : st;
    if (use_side && gi >= 2) cudaStreamWaitEvent(side, prod_ev[b], 0);
    std::vector<oz::Args> args(g.e - g.b);
    std::vector<int> tstart(g.e - g.b + 1, 0);
    std::vector<oz::SplitJob> jobs;
    bool uniform = true;  // equal shapes, single-term operands: one split launch per kernel
    for (int i = g.b; i < g.e; ++i)
      uniform = uniform && items[i].m == items[g.b].m && items[i].n == items[g.b].n && items[i].k == items[g.b].k &&
                items[i].X.n == 1 && items[i].Y.n == 1;
    size_t off = 0;
    for (int i = g.b; i < g.e; ++i) {
      const OzItem& it = items[i];
      uint8_t* w = ws[b] + off;
      off += oz::align256(ozaki_workspace_bytes(it.m, it.n, it.k, slices));
      if (uniform)
        jobs.push_back(oz::split_job(slices, it.X, it.Y, it.m, it.n, it.k, w));
      else
        oz::split_any(slices, it.X, it.Y, it.m, it.n, it.k, w, ss);
      args[i - g.b] = oz::make_args(slices, it.C, it.ldc, it.m, it.n, it.k, it.d, it.nd, w, nullptr);
      const int tiles_i = (int)((it.m + oz::BM - 1) / oz::BM) * args[i - g.b].tiles_n;
      tstart[i - g.b + 1] = tstart[i - g.b] + tiles_i;
    }
    if (uniform) {
      void* jd = nullptr;
      cudaError_t je = cudaMallocAsync(&jd, sizeof(oz::SplitJob) * jobs.size(), ss);
      if (je == cudaSuccess)
        je = cudaMemcpyAsync(jd, jobs.data(), sizeof(oz::SplitJob) * jobs.size(), cudaMemcpyHostToDevice, ss);
      if (je != cudaSuccess) {
        *err = std::string("Ozaki split jobs: ") + cudaGetErrorString(je);
        rc = MK_ERR_CUDA;
        break;
      }
      oz::split_batch_any(slices, static_cast<const oz::SplitJob*>(jd), items[g.b].m, items[g.b].n, items[g.b].k,
                          (int)jobs.size(), ss);
      cudaFreeAsync(jd, ss);
    }
    if (use_side) {
      cudaEventRecord(split_ev[b], side);
      cudaStreamWaitEvent(st, split_ev[b], 0);
    }
    const int n_it = g.e - g.b, tiles = tstart[n_it];
    void* dev = nullptr;
    const size_t abytes = sizeof(oz::Args) * n_it, tbytes = sizeof(int) * (n_it + 1);
    cudaError_t e = cudaMallocAsync(&dev, abytes + tbytes + 256, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(dev, args.data(), abytes, cudaMemcpyHostToDevice, st);
    int* tdev = reinterpret_cast<int*>(static_cast<char*>(dev) + ((abytes + 255) / 256) * 256);
    if (e == cudaSuccess) e = cudaMemcpyAsync(tdev, tstart.data(), tbytes, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) {
      *err = std::string("Ozaki batch arguments: ") + cudaGetErrorString(e);
      rc = MK_ERR_CUDA;
      break;
    }
    rc = oz::batch_launch_any(slices, static_cast<const oz::Args*>(dev), tdev, n_it, tiles, st, err);
    cudaFreeAsync(dev, st);
    if (use_side) cudaEventRecord(prod_ev[b], st);
  }
  for (int b = 0; b < nbuf; ++b) cudaFreeAsync(ws[b], st);
  for (cudaEvent_t ev : {start, split_ev[0], split_ev[1], prod_ev[0], prod_ev[1]})
    if (ev) cudaEventDestroy(ev);
  return rc;
}

int ozaki_product_batch(const OzItem* items, int count, int slices, cudaStream_t st, std::string* err) {
  if (count <= 0) return MK_OK;
  struct Sub {
    const OzItem* it;
    int64_t k0, kk;
    bool first;
  };
  std::vector<Sub> subs;
  size_t wsb = 0;
  bool one_chunk = true;
  for (int i = 0; i < count; ++i) {
    const OzItem& it = items[i];
    if (int rc = check_args(it.m, it.n, slices, it.nd, err)) return rc;
    if (it.X.n < 1 || it.X.n > kOzMaxTerms || it.Y.n < 1 || it.Y.n > kOzMaxTerms) {
      *err = "internal: operand term count out of range";
      return MK_ERR_ARG;
    }
    one_chunk = one_chunk && it.k <= oz::chunk_k(it.k, slices);
  }
  // Grouped launches pay off for small and medium leaves (fewer, fuller launches); for big leaves
  // (>= 2^34 work, e.g. the bench's 4096^3) the per-item pipeline overlaps splitting better.
  static const int grouped_mode = getenv("MK_OZ_GROUPED") ? atoi(getenv("MK_OZ_GROUPED")) : -1;  // -1 auto
  bool small = true;
  for (int i = 0; i < count; ++i) small = small && (double)items[i].m * items[i].n * items[i].k < 17179869184.0;
  const bool grouped = grouped_mode == 1 || (grouped_mode < 0 && small);
  if (grouped && one_chunk && count > 1) {
    keep_pool_memory();
    int dev = 0;
    cudaGetDevice(&dev);
    return batch_grouped(items, count, slices, st, side_stream(dev), err);
  }
  for (int i = 0; i < count; ++i) {
    const OzItem& it = items[i];
    const int64_t kc = oz::chunk_k(it.k, slices);
    for (int64_t k0 = 0; k0 < it.k; k0 += kc) subs.push_back(Sub{&it, k0, std::min(kc, it.k - k0), k0 == 0});
    wsb = std::max(wsb, ozaki_workspace_bytes(it.m, it.n, it.k, slices));
  }
  keep_pool_memory();
  const int nbuf = subs.size() > 1 ? 2 : 1;
  uint8_t* ws[2] = {nullptr, nullptr};
  for (int b = 0; b < nbuf; ++b) {
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&ws[b]), wsb, st);
    if (e != cudaSuccess) {
      cudaGetLastError();
      for (int j = 0; j < b; ++j) cudaFreeAsync(ws[j], st);
      *err = std::string("Ozaki leaf workspace: ") + cudaGetErrorString(e);
      return e == cudaErrorMemoryAllocation ? MK_ERR_WORKSPACE : MK_ERR_CUDA;
    }
  }
  // Splitting (HBM bound) of item i+1 runs on a side stream while the product kernel of item i
  // (tensor bound) runs on st: two workspaces, events in both directions.
  int dev = 0;
  cudaGetDevice(&dev);
  cudaStream_t side = nbuf == 2 ? side_stream(dev) : nullptr;
  cudaEvent_t start = nullptr, split_ev[2] = {nullptr, nullptr}, prod_ev[2] = {nullptr, nullptr};
  auto mkev = [](cudaEvent_t* e) { return cudaEventCreateWithFlags(e, cudaEventDisableTiming); };
  if (side) {
    if (mkev(&start) || mkev(&split_ev[0]) || mkev(&split_ev[1]) || mkev(&prod_ev[0]) || mkev(&prod_ev[1])) {
      cudaGetLastError();
      side = nullptr;
    } else {
      cudaEventRecord(start, st);
      cudaStreamWaitEvent(side, start, 0);  // operands produced earlier on st
    }
  }
  int rc = MK_OK;
  for (size_t i = 0; i < subs.size() && rc == MK_OK; ++i) {
    const Sub& sb = subs[i];
    const OzItem& it = *sb.it;
    const int b = (int)(i % nbuf);
    OzOperand Xc = it.X, Yc = it.Y;
    for (int t = 0; t < Xc.n; ++t) Xc.p[t] = it.X.p[t] + sb.k0;
    for (int t = 0; t < Yc.n; ++t) Yc.p[t] = it.Y.p[t] + sb.k0 * it.Y.ld;
    OzDest dd[kOzMaxDests];
    for (int t = 0; t < it.nd; ++t) {
      dd[t] = it.d[t];
      if (!sb.first) dd[t].accumulate = 1;
    }
    if (side) {
      if (i >= 2) cudaStreamWaitEvent(side, prod_ev[b], 0);  // product i-2 is done with ws[b]
      oz::split_any(slices, Xc, Yc, it.m, it.n, sb.kk, ws[b], side);
      cudaEventRecord(split_ev[b], side);
      cudaStreamWaitEvent(st, split_ev[b], 0);
      rc = oz::product_any(slices, it.C, it.ldc, it.m, it.n, sb.kk, dd, it.nd, ws[b], st, err);
      cudaEventRecord(prod_ev[b], st);
    } else {
      oz::split_any(slices, Xc, Yc, it.m, it.n, sb.kk, ws[b], st);
      rc = oz::product_any(slices, it.C, it.ldc, it.m, it.n, sb.kk, dd, it.nd, ws[b], st, err);
    }
  }
  for (int b = 0; b < nbuf; ++b) cudaFreeAsync(ws[b], st);  // after every product (and so every split)
  for (cudaEvent_t e : {start, split_ev[0], split_ev[1], prod_ev[0], prod_ev[1]})
    if (e) cudaEventDestroy(e);
  cudaError_t e = cudaGetLastError();
  if (rc == MK_OK && e != cudaSuccess) {
    *err = std::string("Ozaki batch: ") + cudaGetErrorString(e);
    rc = MK_ERR_CUDA;
  }
  return rc;
}

int ozaki_product_multi(const OzOperand& X, const OzOperand& Y, double* C, int64_t ldc, int64_t m, int64_t n,
                        int64_t k, int slices, const OzDest* d, int nd, cudaStream_t st, std::string* err,
                        const OzSlabs* slabs) {
  if (int rc = check_args(m, n, slices, nd, err)) return rc;
  if (X.n < 1 || X.n > kOzMaxTerms || Y.n < 1 || Y.n > kOzMaxTerms) {
    *err = "internal: operand term count out of range";
    return MK_ERR_ARG;
  }
  const size_t wsb = ozaki_workspace_bytes(m, n, k, slices);
  keep_pool_memory();
  void* ws = nullptr;
  cudaError_t e = cudaMallocAsync(&ws, wsb, st);
  if (e != cudaSuccess) {
    cudaGetLastError();
    *err = std::string("Ozaki leaf workspace: ") + cudaGetErrorString(e);
    return e == cudaErrorMemoryAllocation ? MK_ERR_WORKSPACE : MK_ERR_CUDA;
  }
  int rc = oz::product_chunks(X, Y, C, ldc, m, n, k, slices, d, nd, static_cast<uint8_t*>(ws), st, err, slabs);
  e = cudaFreeAsync(ws, st);
  if (rc == MK_OK && e != cudaSuccess) {
    *err = std::string("Ozaki leaf workspace free: ") + cudaGetErrorString(e);
    rc = MK_ERR_CUDA;
  }
  return rc;
}

}  // namespace mk
