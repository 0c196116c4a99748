// K1+K2+K3: the fused Strassen/Winograd leaf product for sm_100a.
//
//   K1  FP64 tensor-core GEMM: TMA (128B swizzle) -> smem ring (mbarrier full/empty)
//       -> conflict-free LDS.128 fragments -> mma.sync f64 (SASS DMMA.8x8x4),
//       128x128 CTA tile, 8 consumer warps of 64x32 + 1 TMA producer warp.
//   K2  operand pre-additions: every term tile of  sum_i s_i * A_i  is staged by TMA
//       into the same ring stage and summed in registers as the fragments are read,
//       so S1..S4 / T1..T4 (reference kernels.py:96-104) never exist in HBM.
//   K3  post-additions: the accumulator tile is added with its sign into every C
//       quadrant the product feeds (reference kernels.py:112-118) in one epilogue,
//       with 256-bit coalesced read-modify-writes and no P_i temporaries.
//
// Fragment layouts (PTX m8n8k4.f64): A lane=(row g=lane>>2, k=lane&3),
// B lane=(k=lane&3, col g), C lane=(row g, cols 2*(lane&3)+{0,1}).
// Smem layouts: A term tile = [128 rows][16 k] doubles, 128B-swizzled (chunk ^= row&7).
//               B term tile = 8 boxes of [16 k][16 n], each 128B-swizzled.
// A lane reads one 16B chunk of A holding k = 2c, 2c+1 (two k-steps per LDS.128); to make the
// 8 lanes of each quarter-warp hit 8 distinct chunks, fragment row g maps to smem row
// (g>>1) + 4*(g&1).  A lane reads one 16B chunk of a B row holding columns 2g, 2g+1, which
// feeds two n-fragments per LDS.128; the k order (2q+8t+e) matches A's.
#include <cuda_runtime.h>
#include <type_traits>
#include "mk_device.cuh"
#include "mk_plan.h"

namespace mk {

template <int MAXT>
__global__ void __launch_bounds__(MK_THREADS, 1)
fused_product_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const MkGemmArgs args, const __grid_constant__ MkProduct prod) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[16];
  __shared__ __align__(8) uint64_t empty_bar[16];

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int na = prod.na, nb = prod.nb;
  const int S = args.stages;
  const uint32_t stage_bytes = (uint32_t)(na + nb) * MK_TILE_BYTES;
  const uint32_t smem_base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  uint8_t* smem_gen = smem_raw + (smem_base - smem_u32(smem_raw));

  // ---- rasterised tile coordinates (group_m tile-rows walked column-major) ----
  int tm, tn;
  {
    const int bid = blockIdx.x;
    const int per_group = args.group_m * args.tiles_n;
    const int g = bid / per_group;
    const int first_m = g * args.group_m;
    const int gsz = min(args.tiles_m - first_m, args.group_m);
    const int r = bid - g * per_group;
    tm = first_m + r % gsz;
    tn = r / gsz;
  }
  const int m0 = tm * MK_BM, n0 = tn * MK_BN;
  const int KT = (args.K + MK_BK - 1) / MK_BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], MK_CONSUMER_WARPS);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp < 4) {
    // ============ producer warpgroup: frees its registers, one lane drives TMA ============
    asm volatile("setmaxnreg.dec.sync.aligned.u32 40;\n");
    if (warp == 0 && lane == 0) {
      tma_prefetch_desc(&tmA);
      tma_prefetch_desc(&tmB);
      for (int kt = 0; kt < KT; ++kt) {
        const int s = kt % S;
        if (kt >= S) mbar_wait(&empty_bar[s], ((kt / S) - 1) & 1);
        mbar_arrive_expect_tx(&full_bar[s], stage_bytes);
        uint8_t* sA = smem_gen + (size_t)s * stage_bytes;
        uint8_t* sB = sA + (size_t)na * MK_TILE_BYTES;
        const int k0 = kt * MK_BK;
        for (int t = 0; t < na; ++t)
          tma_load_2d(sA + t * MK_TILE_BYTES, &tmA, k0 + prod.a[t].col, m0 + prod.a[t].row, &full_bar[s]);
        for (int t = 0; t < nb; ++t) {
#pragma unroll
          for (int bj = 0; bj < 8; ++bj)
            tma_load_2d(sB + t * MK_TILE_BYTES + bj * 2048, &tmB, n0 + prod.b[t].col + bj * 16,
                        k0 + prod.b[t].row, &full_bar[s]);
        }
      }
    }
    return;
  }

  // ================== DMMA consumers (2 warpgroups = 8 warps) ==================
  asm volatile("setmaxnreg.inc.sync.aligned.u32 232;\n");
  const int cw = warp - 4;
  const int warp_m = cw >> 2;  // 0..1 -> 64-row half
  const int warp_n = cw & 3;   // 0..3 -> 32-col quarter
  const int q = lane & 3, g = lane >> 2;
  const int prow = (g >> 1) + 4 * (g & 1);

  // A: row (warp_m*64 + 8i + prow), chunk (q + 4t) ^ prow
  const uint32_t a_lane = (uint32_t)(warp_m * 64 + prow) * 128u;
  const uint32_t a_chunk0 = (uint32_t)(((q + 0) ^ prow) << 4);
  const uint32_t a_chunk1 = (uint32_t)(((q + 4) ^ prow) << 4);
  // B: box (warp_n*2 + j), row k = 2q + 8t + e, chunk g ^ ((2q + e) & 7)
  const uint32_t b_lane = (uint32_t)(warp_n * 2) * 2048u;
  uint32_t b_off[2][2];
#pragma unroll
  for (int t = 0; t < 2; ++t)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int k = 2 * q + 8 * t + e;
      b_off[t][e] = b_lane + (uint32_t)k * 128u + (uint32_t)((g ^ ((2 * q + e) & 7)) << 4);
    }

  double sa[MAXT], sb[MAXT];
#pragma unroll
  for (int t = 0; t < MAXT; ++t) {
    sa[t] = t < na ? prod.a[t].sign : 0.0;
    sb[t] = t < nb ? prod.b[t].sign : 0.0;
  }
  // Fold the first term's sign into the result so term 0 is loaded unscaled.
  double out_sign = sa[0] * sb[0];

  double acc[8][4][2];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int f = 0; f < 4; ++f) acc[i][f][0] = acc[i][f][1] = 0.0;

  // One ring stage: 4 k-steps of 8x4 m-frags x 4 n-frags per warp. With TAIL, k >= krem
  // (past the leaf's K extent, possibly a neighbour quadrant's data) is zeroed on both sides.
  auto stage = [&](const uint32_t sA, const uint32_t sB, const int krem, auto tail_tag) {
    constexpr bool TAIL = decltype(tail_tag)::value;
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const uint32_t a_chunk = t ? a_chunk1 : a_chunk0;
      double a0[8], a1[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) lds128(a0[i], a1[i], sA + a_lane + i * 1024u + a_chunk);
#pragma unroll
      for (int tt = 1; tt < MAXT; ++tt) {
        if (tt < na) {
          const double sg = sa[tt] * sa[0];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            double x, y;
            lds128(x, y, sA + tt * MK_TILE_BYTES + a_lane + i * 1024u + a_chunk);
            a0[i] = fma(sg, x, a0[i]);
            a1[i] = fma(sg, y, a1[i]);
          }
        }
      }
      if (TAIL) {
        const int k0 = 2 * q + 8 * t;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          a0[i] = k0 < krem ? a0[i] : 0.0;
          a1[i] = k0 + 1 < krem ? a1[i] : 0.0;
        }
      }
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        double b[4];
        lds128(b[0], b[1], sB + b_off[t][e]);
        lds128(b[2], b[3], sB + b_off[t][e] + 2048u);
#pragma unroll
        for (int tt = 1; tt < MAXT; ++tt) {
          if (tt < nb) {
            const double sg = sb[tt] * sb[0];
            double x0, x1, x2, x3;
            lds128(x0, x1, sB + tt * MK_TILE_BYTES + b_off[t][e]);
            lds128(x2, x3, sB + tt * MK_TILE_BYTES + b_off[t][e] + 2048u);
            b[0] = fma(sg, x0, b[0]);
            b[1] = fma(sg, x1, b[1]);
            b[2] = fma(sg, x2, b[2]);
            b[3] = fma(sg, x3, b[3]);
          }
        }
        if (TAIL) {
          const bool live = 2 * q + 8 * t + e < krem;
#pragma unroll
          for (int f = 0; f < 4; ++f) b[f] = live ? b[f] : 0.0;
        }
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int f = 0; f < 4; ++f) dmma(acc[i][f][0], acc[i][f][1], e ? a1[i] : a0[i], b[f]);
      }
    }
  };

  const int krem_last = args.K - (KT - 1) * MK_BK;  // 1..16
  for (int kt = 0; kt < KT; ++kt) {
    const int s = kt % S;
    mbar_wait(&full_bar[s], (kt / S) & 1);
    const uint32_t sA = smem_base + (uint32_t)s * stage_bytes;
    const uint32_t sB = sA + (uint32_t)na * MK_TILE_BYTES;
    if (kt == KT - 1 && krem_last < MK_BK)
      stage(sA, sB, krem_last, std::true_type{});
    else
      stage(sA, sB, MK_BK, std::false_type{});
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty_bar[s]);
  }

  // ============================ multi-destination epilogue ============================
  // Lane owns, per (i, j): row m0 + warp_m*64 + 8i + prow, cols n0 + warp_n*32 + 16j + 4q .. +3
  // holding {acc[i][2j][0], acc[i][2j+1][0], acc[i][2j][1], acc[i][2j+1][1]}.
  const int nd = prod.nd;
  for (int d = 0; d < nd; ++d) {
    const MkDest dst = prod.d[d];
    const double sg = dst.sign * out_sign;
    double* Cd = args.C + dst.row * args.ldc + dst.col;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int row = m0 + warp_m * 64 + 8 * i + prow;
      if (row >= args.M) continue;
      double* crow = Cd + (int64_t)row * args.ldc;
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int col = n0 + warp_n * 32 + 16 * j + 4 * q;
        const double v0 = acc[i][2 * j][0], v1 = acc[i][2 * j + 1][0];
        const double v2 = acc[i][2 * j][1], v3 = acc[i][2 * j + 1][1];
        if (args.vec_ok) {
          if (col >= args.N) continue;
          double* p = crow + col;
          if (dst.accumulate) {
            double c0, c1, c2, c3;
            ldg256(p, c0, c1, c2, c3);
            stg256(p, fma(sg, v0, c0), fma(sg, v1, c1), fma(sg, v2, c2), fma(sg, v3, c3));
          } else {
            stg256(p, sg * v0, sg * v1, sg * v2, sg * v3);
          }
        } else {
          const double v[4] = {v0, v1, v2, v3};
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            if (col + u < args.N) {
              double* p = crow + col + u;
              *p = dst.accumulate ? fma(sg, v[u], *p) : sg * v[u];
            }
          }
        }
      }
    }
  }
}

// ------------------------------------------------------------------------------------
// Host-side launcher (called by the planner).
// ------------------------------------------------------------------------------------
cudaError_t launch_fused_product(const CUtensorMap& tmA, const CUtensorMap& tmB, const MkGemmArgs& args_in,
                                 const MkProduct& prod, cudaStream_t stream) {
  MkGemmArgs args = args_in;
  const int maxt = prod.na > prod.nb ? prod.na : prod.nb;
  const uint32_t stage_bytes = (uint32_t)(prod.na + prod.nb) * MK_TILE_BYTES;
  int stages = (int)(MK_SMEM_BUDGET / stage_bytes);
  if (stages > 8) stages = 8;
  if (stages < 2) return cudaErrorInvalidValue;
  args.stages = stages;
  const size_t smem = (size_t)stages * stage_bytes + 1024;
  const int grid = args.tiles_m * args.tiles_n;
  if (grid == 0) return cudaSuccess;
  cudaError_t err;
#define MK_LAUNCH(T)                                                                              \
  do {                                                                                            \
    err = cudaFuncSetAttribute(fused_product_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                               (int)smem);                                                        \
    if (err != cudaSuccess) return err;                                                           \
    fused_product_kernel<T><<<grid, MK_THREADS, smem, stream>>>(tmA, tmB, args, prod);            \
  } while (0)
  if (maxt <= 1)
    MK_LAUNCH(1);
  else if (maxt <= 2)
    MK_LAUNCH(2);
  else
    MK_LAUNCH(4);
#undef MK_LAUNCH
  return cudaGetLastError();
}

}  // namespace mk
