// K1+K2+K3: the fused Strassen/Winograd leaf product for sm_100a.
//
//   K1  FP64 tensor-core GEMM: TMA (128B swizzle) -> smem operand ring (mbarrier full/empty)
//       -> conflict-free LDS.128 fragments -> mma.sync f64 (SASS DMMA.8x8x4), 128x128 CTA
//       tile, two consumer warpgroups (8 warps of 64x32) with register accumulators
//       (tcgen05 has no f64 kind, so there is no TMEM path for FP64).
//   K2  operand pre-additions: the producer warpgroup is a *combiner*. TMA lands the raw
//       term tiles of  sum_i s_i * A_i  (e.g. S4 = A11 + A12 - A21 - A22) in a raw ring; the
//       128 producer threads sum them once per CTA into the swizzled operand stage (layout
//       preserving, sign applied as a sign-bit flip + DADD). S1..S4 / T1..T4 (reference
//       kernels.py:96-104) never exist in HBM, and the DMMA warps run the plain GEMM loop.
//       Single-term sides are TMA'd straight into the operand stage.
//   K3  post-additions: the accumulator tile is added with its sign into every C block the
//       product feeds (reference kernels.py:112-118) in one epilogue, with 256-bit coalesced
//       read-modify-writes and no P_i temporaries.
//
// Fragment layouts (PTX m8n8k4.f64): A lane=(row g=lane>>2, k=lane&3),
// B lane=(k=lane&3, col g), C lane=(row g, cols 2*(lane&3)+{0,1}).
// Smem layouts: A tile = [128 rows][16 k] doubles, 128B-swizzled (16B chunk ^= row&7).
//               B tile = 8 boxes of [16 k][16 n], each 128B-swizzled.
// A lane reads one 16B chunk of A holding k = 2c, 2c+1 (two k-steps per LDS.128); to make the
// 8 lanes of each quarter-warp hit 8 distinct chunks, fragment row g maps to smem row
// (g>>1) + 4*(g&1).  A lane reads one 16B chunk of a B row holding columns 2g, 2g+1, which
// feeds two n-fragments per LDS.128; the k order (2q+8t+e) matches A's.
#include <cuda_runtime.h>
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <map>
#include <mutex>
#include <type_traits>
#include <vector>
#include "mk_device.cuh"
#include "mk_plan.h"
#include "mk_blockops.h"
#include "mk_xform.cuh"

namespace mk {

// Row-slab routing of the fused multi-GPU reduce-scatter (MkGemmArgs::nslab > 0): C row R goes to
// its owner's slab (a local buffer or a peer's, IPC-mapped over NVLink).
__device__ __forceinline__ double* slab_row(const MkGemmArgs& a, int64_t R, int64_t ldc) {
  const int64_t o = R / a.slab_rows;
  return a.slab[o] + (R - o * a.slab_rows) * ldc;
}


constexpr int kOpStageBytes = 2 * MK_TILE_BYTES;  // summed A tile + summed B tile
constexpr int kMaxStages = 8;

// x with its sign bit flipped by `m` (0 or 0x80000000): one LOP3 on the integer pipe.
__device__ __forceinline__ double flip(double x, uint32_t m) {
  return __hiloint2double(__double2hiint(x) ^ (int)m, __double2loint(x));
}

// Sum `nt` raw term tiles (16 KiB each, identical swizzled layout) into dst; thread `tid` of
// 128 handles 16-byte chunks tid, tid+128, ... (conflict-free, coalesced in smem).
__device__ __forceinline__ void combine_tile(uint8_t* dst, const uint8_t* raw, int nt, uint32_t negmask,
                                             int tid) {
#pragma unroll 1
  for (int c = tid; c < MK_TILE_BYTES / 16; c += 128 * 4) {
    double2 acc[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) acc[u] = *reinterpret_cast<const double2*>(raw + (c + u * 128) * 16);
    for (int t = 1; t < nt; ++t) {
      const uint8_t* src = raw + t * MK_TILE_BYTES;
      const uint32_t m = ((negmask >> t) & 1u) << 31;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double2 v = *reinterpret_cast<const double2*>(src + (c + u * 128) * 16);
        acc[u].x += flip(v.x, m);
        acc[u].y += flip(v.y, m);
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) *reinterpret_cast<double2*>(dst + (c + u * 128) * 16) = acc[u];
  }
}

__device__ __forceinline__ void named_bar_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// Consumer layouts: MT = m-fragments (8 rows each) per warp.
//   MT = 8: 8 consumer warps of 64x32 (2 per SMSP), 384 threads, 224 registers per consumer.
//   MT = 4: 16 consumer warps of 32x32 (4 per SMSP), 640 threads, 104-112 registers per
//           consumer: twice the warps to hide LDS / dependency latency behind DMMA.
template <int MT>
struct Layout {
  static constexpr int kConsumerWarps = 4 * (16 / MT);
  static constexpr int kThreads = 128 + 32 * kConsumerWarps;
};

// Register budgets (setmaxnreg immediates). The CTA is launched with floor(65536/threads)
// rounded down to 8 registers per thread; producer decrease + consumer increase must fit it.
template <int MT, bool COMBINE>
struct Regs;
template <bool C>
struct Regs<8, C> {  // 384 x 168 = 64512 = 128 x 56 + 256 x 224
  static constexpr int kProducer = 56, kConsumer = 224;
};
template <>
struct Regs<4, false> {  // 640 x 96 = 61440 = 128 x 32 + 512 x 112
  static constexpr int kProducer = 32, kConsumer = 112;
};
template <>
struct Regs<4, true> {  // 61440 >= 128 x 40 + 512 x 104
  static constexpr int kProducer = 40, kConsumer = 104;
};

#ifdef MK_TRACE
// Per-CTA timeline (trace builds only, tools/tile_trace.py): smid, entry, first stage ready,
// main loop done, epilogue done (%globaltimer ns), stamped by consumer warp 0.
__device__ unsigned long long mk_trace_buf[5 * 65536];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define MK_STAMP(slot)                                                                  \
  do {                                                                                  \
    if (warp == 4 && lane == 0 && blockIdx.x < 65536) mk_trace_buf[5 * blockIdx.x + (slot)] = gtimer(); \
  } while (0)
#else
#define MK_STAMP(slot) \
  do {                 \
  } while (0)
#endif

// CA / CB: the A / B operand has more than one term and goes through the combiner.
template <bool CA, bool CB, int MT>
__global__ void __launch_bounds__(Layout<MT>::kThreads, 1)
fused_product_kernel(const __grid_constant__ CUtensorMap tmA_param, const __grid_constant__ CUtensorMap tmB_param,
                     const __grid_constant__ CUtensorMap tmC_param, const MkGemmArgs args,
                     const __grid_constant__ MkProduct prod_param) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[kMaxStages];
  __shared__ __align__(8) uint64_t empty_bar[kMaxStages];
  __shared__ __align__(8) uint64_t raw_bar[2];
  __shared__ uint32_t tmem_base_sh;

  // Single product: maps and descriptor are kernel parameters. Batched launch: CTA blockIdx.x
  // works on tile (blockIdx.x % tiles_per_prod) of product (blockIdx.x / tiles_per_prod), whose
  // tensor maps (64-byte aligned, written before launch) and descriptor live in global memory.
  const MkBatchEntry* ent = args.batch ? args.batch + blockIdx.x / args.tiles_per_prod : nullptr;
  const MkProduct& prod = ent ? ent->prod : prod_param;
  const CUtensorMap* tmA = ent ? &ent->tmA : &tmA_param;
  const CUtensorMap* tmB = ent ? &ent->tmB : &tmB_param;
  const CUtensorMap* tmC = ent ? &ent->tmC : &tmC_param;
  double* const Cbase = ent ? ent->C : args.C;
  const int64_t ldc = ent ? ent->ldc : args.ldc;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
#ifdef MK_TRACE
  if (warp == 4 && lane == 0 && blockIdx.x < 65536) {
    unsigned smid;
    asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
    mk_trace_buf[5 * blockIdx.x] = smid;
    mk_trace_buf[5 * blockIdx.x + 1] = gtimer();
  }
#endif
  const int na = prod.na, nb = prod.nb;
  const int S = args.stages;    // operand stages
  const int D = args.raw_sets;  // raw term sets in flight (0 when nothing is combined)
  const uint32_t smem_base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  uint8_t* smem_gen = smem_raw + (smem_base - smem_u32(smem_raw));
  uint8_t* raw_base = smem_gen + (size_t)S * kOpStageBytes;
  const int raw_tiles = (CA ? na : 0) + (CB ? nb : 0);
  const uint32_t raw_set_bytes = (uint32_t)raw_tiles * MK_TILE_BYTES;
  const uint32_t direct_bytes = (CA ? 0u : (uint32_t)MK_TILE_BYTES) + (CB ? 0u : (uint32_t)MK_TILE_BYTES);

  // ---- rasterised tile coordinates (group_m tile-rows walked column-major) ----
  int tm, tn;
  {
    const int bid = ent ? (int)(blockIdx.x % args.tiles_per_prod) : (int)blockIdx.x;
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
      // one arrive.expect_tx from the TMA thread, plus one arrive per combiner thread
      mbar_init(&full_bar[s], (CA || CB) ? 1 + 128 : 1);
      mbar_init(&empty_bar[s], Layout<MT>::kConsumerWarps);
    }
    for (int d = 0; d < D; ++d) mbar_init(&raw_bar[d], 1);
    fence_barrier_init();
  }
  __syncthreads();

  if (warp < 4) {
    // ================= producer / combiner warpgroup (128 threads) =================
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(Regs<MT, CA || CB>::kProducer));
    const int tid = threadIdx.x;
    if (!(CA || CB) && tid != 0) return;  // plain GEMM: one thread drives TMA, the rest idle
    uint32_t fa = 0, fb = 0;  // bit t set: term t enters with the opposite sign of term 0
    for (int t = 1; t < na; ++t) fa |= (prod.a[t].sign * prod.a[0].sign < 0 ? 1u : 0u) << t;
    for (int t = 1; t < nb; ++t) fb |= (prod.b[t].sign * prod.b[0].sign < 0 ? 1u : 0u) << t;
    auto issue_raw = [&](int k) {  // thread 0 only: all raw term tiles of k-step k
      const int d = k % D;
      uint8_t* dst = raw_base + (size_t)d * raw_set_bytes;
      mbar_arrive_expect_tx(&raw_bar[d], raw_set_bytes);
      const int k0 = k * MK_BK;
      if (CA)
        for (int t = 0; t < na; ++t, dst += MK_TILE_BYTES)
          tma_load_2d(dst, tmA, k0 + prod.a[t].col, m0 + prod.a[t].row, &raw_bar[d]);
      if (CB)
        for (int t = 0; t < nb; ++t, dst += MK_TILE_BYTES)
#pragma unroll
          for (int bj = 0; bj < 8; ++bj)
            tma_load_2d(dst + bj * 2048, tmB, n0 + prod.b[t].col + bj * 16, k0 + prod.b[t].row, &raw_bar[d]);
    };
    if (tid == 0) {
      tma_prefetch_desc(tmA);
      tma_prefetch_desc(tmB);
      if (CA || CB)
        for (int k = 0; k < D && k < KT; ++k) issue_raw(k);
    }
    for (int k = 0; k < KT; ++k) {
      const int s = k % S;
      if (k >= S) mbar_wait(&empty_bar[s], ((k / S) - 1) & 1);
      uint8_t* opA = smem_gen + (size_t)s * kOpStageBytes;
      uint8_t* opB = opA + MK_TILE_BYTES;
      const int k0 = k * MK_BK;
      if (tid == 0) {
        mbar_arrive_expect_tx(&full_bar[s], direct_bytes);
        if (!CA) tma_load_2d(opA, tmA, k0 + prod.a[0].col, m0 + prod.a[0].row, &full_bar[s]);
        if (!CB)
#pragma unroll
          for (int bj = 0; bj < 8; ++bj)
            tma_load_2d(opB + bj * 2048, tmB, n0 + prod.b[0].col + bj * 16, k0 + prod.b[0].row, &full_bar[s]);
      }
      if (CA || CB) {
        const int d = k % D;
        mbar_wait(&raw_bar[d], (k / D) & 1);
        const uint8_t* raw = raw_base + (size_t)d * raw_set_bytes;
        if (CA) {
          combine_tile(opA, raw, na, fa, tid);
          raw += (size_t)na * MK_TILE_BYTES;
        }
        if (CB) combine_tile(opB, raw, nb, fb, tid);
        mbar_arrive(&full_bar[s]);
        named_bar_sync(1, 128);  // every combiner thread is done reading raw set d
        if (tid == 0 && k + D < KT) issue_raw(k + D);
      }
    }
    return;
  }

  // ================== DMMA consumers (2 warpgroups = 8 warps) ==================
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(Regs<MT, CA || CB>::kConsumer));
  const int cw = warp - 4;
  const int warp_m = cw >> 2;  // 64-row (MT=8) or 32-row (MT=4) slab
  const int warp_n = cw & 3;   // 32-col quarter
  const int q = lane & 3, g = lane >> 2;
  const int prow = (g >> 1) + 4 * (g & 1);

  // A: row (warp_m*64 + 8i + prow), chunk (q + 4t) ^ prow
  const uint32_t a_lane = (uint32_t)(warp_m * (8 * MT) + prow) * 128u;
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
  // Term 0 of each side is summed unscaled; its sign is folded into the epilogue.
  const double out_sign = prod.a[0].sign * prod.b[0].sign;

  double acc[MT][4][2];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int f = 0; f < 4; ++f) acc[i][f][0] = acc[i][f][1] = 0.0;

  // One operand stage: 4 k-steps of 8x4 m-frags x 4 n-frags per warp. With TAIL, k >= krem
  // (past the leaf's K extent, possibly a neighbour quadrant's data) is zeroed on both sides.
  auto stage = [&](const uint8_t* sA, const uint8_t* sB, const int krem, auto tail_tag) {
    constexpr bool TAIL = decltype(tail_tag)::value;
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const uint32_t a_chunk = t ? a_chunk1 : a_chunk0;
      double a0[MT], a1[MT];
#pragma unroll
      for (int i = 0; i < MT; ++i) lds128(a0[i], a1[i], sA + a_lane + i * 1024u + a_chunk);
      if (TAIL) {
        const int kk = 2 * q + 8 * t;
#pragma unroll
        for (int i = 0; i < MT; ++i) {
          a0[i] = kk < krem ? a0[i] : 0.0;
          a1[i] = kk + 1 < krem ? a1[i] : 0.0;
        }
      }
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        double b[4];
        lds128(b[0], b[1], sB + b_off[t][e]);
        lds128(b[2], b[3], sB + b_off[t][e] + 2048u);
        if (TAIL) {
          const bool live = 2 * q + 8 * t + e < krem;
#pragma unroll
          for (int f = 0; f < 4; ++f) b[f] = live ? b[f] : 0.0;
        }
#pragma unroll
        for (int i = 0; i < MT; ++i)
#pragma unroll
          for (int f = 0; f < 4; ++f) dmma(acc[i][f][0], acc[i][f][1], e ? a1[i] : a0[i], b[f]);
      }
    }
  };

  // Two-level accumulation: every `chunk` stages the register partial sums are added into a
  // master copy kept in tensor memory (this warp's 32 TMEM lanes x 16*MT columns) and reset,
  // so each output is a short register sum of <= 16*chunk products plus a sum of K/(16*chunk)
  // chunk totals -- the error growth of OpenBLAS-style K blocking, with the DMMA pipe idle for
  // only ~0.2% of the time. Disabled (chunk = 0) when K fits in one chunk.
  // leaves with K <= 512 keep a single register sum (<= 512 terms): folding them buys little
  const int chunk = (args.chunk_stages > 0 && KT > 32 && KT > args.chunk_stages) ? args.chunk_stages : 0;
  constexpr int kWords = 16 * MT;  // 32-bit words of accumulator per thread
  uint32_t taddr = 0;
  if (chunk) {
    if (cw == 0) tmem_alloc(&tmem_base_sh, 256);
    tmem_fence_before();
    named_bar_sync(3, 32 * Layout<MT>::kConsumerWarps);
    tmem_fence_after();
    taddr = tmem_base_sh + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((cw >> 2) * kWords);
  }
  // Fold: master (+)= registers, registers = 0, two 8-double pieces (2 x 16 TMEM columns) per
  // tcgen05.ld round trip. All warps fold at the same k-step (measured cheaper than staggering or
  // rotating single pieces: every tcgen05.wait is costly).
  constexpr int kPieces = kWords / 16;
  bool master_live = false;
  auto fold_to_tmem = [&]() {
#pragma unroll
    for (int pc = 0; pc < kPieces; pc += 2) {
      uint32_t w[2][16];
      if (master_live) {
        tmem_ld16(taddr + pc * 16, w[0]);
        tmem_ld16(taddr + pc * 16 + 16, w[1]);
        tmem_wait_ld();
      }
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int e = (pc + h) * 8 + u;  // flat index into acc[MT][4][2]
          double& a = acc[e >> 3][(e >> 1) & 3][e & 1];
          const double m = master_live ? __hiloint2double((int)w[h][2 * u + 1], (int)w[h][2 * u]) + a : a;
          w[h][2 * u] = (uint32_t)__double2loint(m);
          w[h][2 * u + 1] = (uint32_t)__double2hiint(m);
          a = 0.0;
        }
      tmem_st16(taddr + pc * 16, w[0]);
      tmem_st16(taddr + pc * 16 + 16, w[1]);
    }
    tmem_wait_st();
    master_live = true;
  };

  const int krem_last = args.K - (KT - 1) * MK_BK;  // 1..16
  for (int kt = 0; kt < KT; ++kt) {
    const int s = kt % S;
    mbar_wait(&full_bar[s], (kt / S) & 1);
    if (kt == 0) MK_STAMP(2);
    const uint8_t* sA = smem_gen + (size_t)s * kOpStageBytes;
    const uint8_t* sB = sA + MK_TILE_BYTES;
    if (kt == KT - 1 && krem_last < MK_BK)
      stage(sA, sB, krem_last, std::true_type{});
    else
      stage(sA, sB, MK_BK, std::false_type{});
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty_bar[s]);
    if (chunk && (kt + 1) % chunk == 0 && kt + 1 < KT) fold_to_tmem();
  }
  if (chunk) {
    if (master_live) {  // acc += master
#pragma unroll
      for (int pc = 0; pc < kPieces; ++pc) {
        uint32_t w[16];
        tmem_ld16(taddr + pc * 16, w);
        tmem_wait_ld();
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int e = pc * 8 + u;
          double& a = acc[e >> 3][(e >> 1) & 3][e & 1];
          a = __hiloint2double((int)w[2 * u + 1], (int)w[2 * u]) + a;
        }
      }
    }
    tmem_fence_before();
    named_bar_sync(3, 32 * Layout<MT>::kConsumerWarps);
    tmem_fence_after();
    if (cw == 0) tmem_dealloc(tmem_base_sh, 256);
  }

  MK_STAMP(3);
  // ============================ multi-destination epilogue ============================
  // Lane owns, per (i, j): row m0 + warp_m*8*MT + 8i + prow, cols n0 + warp_n*32 + 16j + 4q .. +3
  // holding {acc[i][2j][0], acc[i][2j+1][0], acc[i][2j][1], acc[i][2j+1][1]}.
  const int nd = prod.nd;
  if (args.async_epi) {
    // Asynchronous epilogue: the warp stages its (8*MT) x 32 fragment as two TMA boxes of
    // [8*MT rows][16 cols] (128B swizzle) in the now idle operand ring, then one lane issues,
    // per destination, a TMA store (first writer) or a TMA reduce-add (accumulate); the adds
    // run at L2. Positive-signed destinations go first; the tile is negated in place for the rest.
    named_bar_sync(2, 32 * Layout<MT>::kConsumerWarps);  // every consumer is done with the ring
    constexpr int kBoxRows = 8 * MT;
    uint8_t* stg = smem_gen + (size_t)cw * (2 * kBoxRows * 128);
    const int c_first = (g & 1) ? 1 : 0;  // store order making each quarter-warp conflict-free
    auto stage_out = [&](double sgn) {
#pragma unroll
      for (int i = 0; i < MT; ++i) {
        const int r = 8 * i + prow;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          uint8_t* rowp = stg + j * (kBoxRows * 128) + r * 128;
          const double v0 = sgn * acc[i][2 * j][0], v1 = sgn * acc[i][2 * j + 1][0];
          const double v2 = sgn * acc[i][2 * j][1], v3 = sgn * acc[i][2 * j + 1][1];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int c = 2 * q + (h ^ c_first);  // logical 16B chunk: cols 2c, 2c+1 of the box
            double2 v = (c & 1) ? make_double2(v2, v3) : make_double2(v0, v1);
            *reinterpret_cast<double2*>(rowp + ((c ^ prow) << 4)) = v;
          }
        }
      }
      fence_proxy_async();
      __syncwarp();
    };
    const int row0 = m0 + warp_m * kBoxRows;
    const int col0 = n0 + warp_n * 32;
    const bool slab_live = row0 < args.M && col0 < args.N;
    int issued = 0;
    for (int pass = 0; pass < 2; ++pass) {
      const double want = pass == 0 ? 1.0 : -1.0;
      bool any = false;
      for (int d = 0; d < nd; ++d) any |= (prod.d[d].sign * out_sign) == want;
      if (!any) continue;
      if (issued) {  // the previous pass's TMA reads of the staging must be done
        if (lane == 0) bulk_wait_read_all();
        __syncwarp();
      }
      stage_out(want);
      if (lane == 0 && slab_live) {
        for (int d = 0; d < nd; ++d) {
          const MkDest dst = prod.d[d];
          if ((dst.sign * out_sign) != want) continue;
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const int cc = (int)dst.col + col0 + 16 * j, rr = (int)dst.row + row0;
            if (col0 + 16 * j >= args.N) continue;
            if (dst.accumulate)
              tma_reduce_add_2d(tmC, cc, rr, stg + j * (kBoxRows * 128));
            else
              tma_store_2d(tmC, cc, rr, stg + j * (kBoxRows * 128));
          }
        }
        bulk_commit();
      }
      issued = 1;
    }
    if (lane == 0) bulk_wait_read_all();  // smem must stay valid until the TMA unit has read it
    __syncwarp();
    MK_STAMP(4);
    return;
  }
  for (int d = 0; d < nd; ++d) {
    const MkDest dst = prod.d[d];
    const double sg = dst.sign * out_sign;
    double* Cd = Cbase + dst.row * ldc + dst.col;
#pragma unroll
    for (int i = 0; i < MT; ++i) {
      const int row = m0 + warp_m * (8 * MT) + 8 * i + prow;
      if (row >= args.M) continue;
      double* crow = args.nslab ? slab_row(args, dst.row + row, ldc) + dst.col : Cd + (int64_t)row * ldc;
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int col = n0 + warp_n * 32 + 16 * j + 4 * q;
        const double v0 = acc[i][2 * j][0], v1 = acc[i][2 * j + 1][0];
        const double v2 = acc[i][2 * j][1], v3 = acc[i][2 * j + 1][1];
        if (args.vec_ok) {
          if (col >= args.N) continue;
          double* p = crow + col;
          if (dst.accumulate) {  // one contribution per element per launch: deterministic
            red_add(p, sg * v0);
            red_add(p + 1, sg * v1);
            red_add(p + 2, sg * v2);
            red_add(p + 3, sg * v3);
          } else {
            stg256(p, sg * v0, sg * v1, sg * v2, sg * v3);
          }
        } else {
          const double v[4] = {v0, v1, v2, v3};
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            if (col + u < args.N) {
              double* p = crow + col + u;
              if (dst.accumulate)
                red_add(p, sg * v[u]);
              else
                *p = sg * v[u];
            }
          }
        }
      }
    }
  }
}


// =====================================================================================
// Persistent plain product (single-term operands on both sides -- every leaf of the
// materialised plans and mk_dgemm). One CTA per SM walks the launch's tiles
// t = blockIdx.x + i*gridDim.x (product-major over a batch, rasterised as above). The TMA
// thread streams k-stages across tile boundaries, so the next tile's first stages land while
// the consumers run the current tile's epilogue; the epilogue stages each warp's fragment one
// 16-column box at a time in a dedicated area (not the ring), and the TMA unit's reads of the
// last box overlap the next tile's main loop. Removes the per-tile pipeline fill, CTA launch
// gap and epilogue drain (~5 us per tile measured by tools/tile_trace.py).
// =====================================================================================
// Persistent layouts: MT m-fragments (8 rows each) per warp, BN tile columns; warps of
// 8*MT x 32 cover the 128 x BN tile. (8, 128): 8 warps of 64x32 (default); (4, 128): 16 warps of
// 32x32 (MK_CONSUMER_WARPS=16); (4, 64): 8 warps of 32x32 for narrow leaves (BN = 64 halves the
// column padding of leaves whose width is not a multiple of 128, e.g. cfg5's 316).
#ifndef MK_EPI_BUFS_NARROW
#define MK_EPI_BUFS_NARROW 1
#endif
#ifndef MK_EPI_SLOTS
#define MK_EPI_SLOTS 1
#endif
#ifndef MK_TAIL_SKIP
#define MK_TAIL_SKIP 1
#endif
template <int MT, int BN, bool SW = false>
struct PLayout {
  static constexpr int kWarpsN = BN / 32;
  static constexpr int kConsumerWarps = (MK_BM / (8 * MT)) * kWarpsN;
  // SW (narrow tiles only): the launch carries side work (below); a second non-DMMA warpgroup
  // joins the producer's, so 7 side warps stream the transforms (3 are latency-bound at ~1 TB/s).
  // Launches without side work run the 384-thread layout (its consumers keep 224 registers).
  static constexpr bool kSideWork = SW;
  static constexpr int kLeadWarps = kSideWork ? 8 : 4;  // warps before the first DMMA consumer
  static constexpr int kSideThreads = kSideWork ? 32 * (kLeadWarps - 1) : 0;
  static constexpr int kThreads = 32 * kLeadWarps + 32 * kConsumerWarps;
  static constexpr int kStageBytes = MK_TILE_BYTES + BN * MK_BK * 8;
  // epilogue boxes per warp (MK_EPI_BUFS_NARROW > 1 lets a narrow-tile warp fill its next box while
  // the TMA unit still reads the last: measured no faster on cfg5, so one by default)
  static constexpr int kEpiBufs = BN == 64 ? MK_EPI_BUFS_NARROW : 1;
  static constexpr int kBoxBytes = kEpiBufs * kConsumerWarps * 8 * MT * 128;  // 16-column boxes
  // Narrow tiles: the producer stages each tile's destination list (count, sign and store/add
  // masks, offsets) in a 16-slot shared ring, so the epilogue reads it from shared memory instead
  // of waiting on L2 for the product descriptor (short-K tiles: a visible share of the tile).
  // Slots of 96 bytes: count, masks and the first 8 destinations (more -- depth-first plans only
  // -- are read from the descriptor), in the slack between the ring and the 227 KiB opt-in limit
  // (the ring keeps its 8 stages). Side layout only: there it takes cfg5 69.9 -> 68.3 ms; in the
  // 384-thread layout the same ring made every launch slower, batched or not (cfg5 sequential
  // 73.6 -> 75.2 ms, in-place n = 8192 L = 3 34.5 -> 38.0 ms, reproducibly, cause not found).
  static constexpr int kEpiSlots = (BN == 64 && SW && MK_EPI_SLOTS) ? 8 : 0;
  static constexpr int kEpiSlotInts = 24;
  static constexpr int kEpiSlotDests = 8;
  static constexpr int kEpiSlotBytes = kEpiSlots * kEpiSlotInts * 4;
  // Register split (setmaxnreg): the wide layout's 64 x 32 consumers take 224, its producer 56.
  // The side-work layout (512 threads, 128 each at launch): the two lead warpgroups drop to 104
  // (the two-level operand transform at 16-byte width needs 92; the post-addition runs at 8-byte
  // width there, 64) and the 32 x 32 consumer warps rise to 152 (at 128 they reload loop state
  // from local memory every k-stage: main loop -2.4%).
  static constexpr int kProducerRegs = kSideWork ? 104 : (kThreads == 384 ? 56 : 32);
  static constexpr int kConsumerRegs = kSideWork ? 152 : (kThreads == 384 ? 224 : 112);
};

// Side work: every task of the launch in order. A task's jobs are spread over groups of CTAs
// (enough CTAs per job for >= 4 element groups per thread); within a group the NT side threads
// of each CTA grid-stride over the job's element groups (row, W columns). The job's 49-64 block
// pointers are staged in shared memory once per job (the stand-alone kernels do the same) --
// read per element group from global memory, the pointer loads serialise every store behind an
// L1 round trip. Kinds 2 and 3 only: the one-level transform's runtime source/destination loops
// spill in the producer's register budget, so the launcher runs kind-1 tasks as their own launches.
template <int NT>
__device__ __forceinline__ void side_bar() { asm volatile("bar.sync 5, %0;" ::"n"(NT) : "memory"); }
template <int NT, int W, typename Stage, typename F>
__device__ __forceinline__ void side_loop(const MkSideTask& tk, uint32_t tid, uint32_t cta, uint32_t ncta, Stage&& stage,
                                          F&& f) {
  const uint32_t cv = (uint32_t)(tk.cols / W);
  const uint32_t per = (uint32_t)tk.rows * cv;
  uint32_t G = per / (NT * 4u);  // CTAs per job
  G = G < 1 ? 1 : (G > ncta ? ncta : G);
  const uint32_t ngroups = ncta / G;
  const uint32_t grp = cta / G, sub = cta - grp * G;
  if (grp >= ngroups) return;  // the CTAs past the last whole group sit this task out
  for (uint32_t j = grp; j < (uint32_t)tk.njobs; j += ngroups) {
    side_bar<NT>();  // the previous job's pointers are no longer read
    stage(j);
    side_bar<NT>();
    for (uint32_t e = sub * NT + tid; e < per; e += G * NT) {
      const uint32_t r = e / cv;
      f(j, r, (int64_t)(e - r * cv) * W);
    }
  }
}
template <int NT, int TAB, int SIDE, int W>
__device__ __forceinline__ void side_xform2(const MkSideTask& tk, uint32_t tid, uint32_t cta, uint32_t ncta,
                                            double** ptr_sh) {
  constexpr int NP = X2Tab<TAB, SIDE>::np;
  const MkXform2Job* jobs = static_cast<const MkXform2Job*>(tk.jobs);
  side_loop<NT, W>(
      tk, tid, cta, ncta,
      [&](uint32_t j) {
        if (tid < NP * NP) ptr_sh[tid] = jobs[j].dst[tid];
      },
      [&](uint32_t j, uint32_t r, int64_t c) {
        const MkXform2Job& jb = jobs[j];
        xform2_elem<TAB, SIDE, W>(jb.src, jb.lds, static_cast<double* const*>(ptr_sh), jb.ldd, tk.rows, tk.cols, r, c);
      });
}
template <int NT, int TAB, int SIDE, int W>
__device__ __forceinline__ void side_xform1(const MkSideTask& tk, uint32_t tid, uint32_t cta, uint32_t ncta,
                                            double** ptr_sh) {
  constexpr int NP = X2Tab<TAB, SIDE>::np;
  const MkXform2Job* jobs = static_cast<const MkXform2Job*>(tk.jobs);
  side_loop<NT, W>(
      tk, tid, cta, ncta,
      [&](uint32_t j) {
        if (tid < NP) ptr_sh[tid] = jobs[j].dst[tid];
      },
      [&](uint32_t j, uint32_t r, int64_t c) {
        const MkXform2Job& jb = jobs[j];
        xform1_elem<TAB, SIDE, W>(jb.src, jb.lds, static_cast<double* const*>(ptr_sh), jb.ldd, tk.rows, tk.cols, r, c);
      });
}
template <int NT, int TAB, int W>
__device__ __forceinline__ void side_xpost1(const MkSideTask& tk, uint32_t tid, uint32_t cta, uint32_t ncta,
                                            double** ptr_sh) {
  constexpr int NP = XCTab<TAB>::np;
  const MkXpost2Job* jobs = static_cast<const MkXpost2Job*>(tk.jobs);
  side_loop<NT, W>(
      tk, tid, cta, ncta,
      [&](uint32_t j) {
        if (tid < NP) ptr_sh[tid] = const_cast<double*>(jobs[j].src[tid]);
      },
      [&](uint32_t j, uint32_t r, int64_t c) {
        const MkXpost2Job& jb = jobs[j];
        xpost1_elem<TAB, W>(static_cast<const double* const*>(ptr_sh), jb.lds, jb.dst, jb.ldd, jb.acc_mask, tk.rows,
                            tk.cols, r, c);
      });
}
template <int NT, int TAB, int W>
__device__ __forceinline__ void side_xpost2(const MkSideTask& tk, uint32_t tid, uint32_t cta, uint32_t ncta,
                                            double** ptr_sh) {
  constexpr int NP = XCTab<TAB>::np;
  const MkXpost2Job* jobs = static_cast<const MkXpost2Job*>(tk.jobs);
  side_loop<NT, W>(
      tk, tid, cta, ncta,
      [&](uint32_t j) {
        if (tid < NP * NP) ptr_sh[tid] = const_cast<double*>(jobs[j].src[tid]);
      },
      [&](uint32_t j, uint32_t r, int64_t c) {
        const MkXpost2Job& jb = jobs[j];
        xpost2_elem<TAB, W>(static_cast<const double* const*>(ptr_sh), jb.lds, jb.dst, jb.ldd, jb.acc_mask, tk.rows,
                            tk.cols, r, c);
      });
}
template <int NT>
__device__ __forceinline__ void side_work(const MkGemmArgs& a, uint32_t tid, uint32_t cta, uint32_t ncta, double** ptr_sh) {
  for (int t = 0; t < a.nside; ++t) {
    const MkSideTask& tk = a.side[t];
#ifdef MK_SIDE_W1
    const bool w2 = false;
#else
    const bool w2 = tk.width == 2;
#endif
    if (tk.kind == 2) {
      switch (tk.table * 4 + tk.side * 2 + (w2 ? 1 : 0)) {
        case 0: side_xform2<NT, 0, 0, 1>(tk, tid, cta, ncta, ptr_sh); break;
        case 1: side_xform2<NT, 0, 0, 2>(tk, tid, cta, ncta, ptr_sh); break;
        case 2: side_xform2<NT, 0, 1, 1>(tk, tid, cta, ncta, ptr_sh); break;
        case 3: side_xform2<NT, 0, 1, 2>(tk, tid, cta, ncta, ptr_sh); break;
        case 4: side_xform2<NT, 1, 0, 1>(tk, tid, cta, ncta, ptr_sh); break;
        case 5: side_xform2<NT, 1, 0, 2>(tk, tid, cta, ncta, ptr_sh); break;
        case 6: side_xform2<NT, 1, 1, 1>(tk, tid, cta, ncta, ptr_sh); break;
        case 7: side_xform2<NT, 1, 1, 2>(tk, tid, cta, ncta, ptr_sh); break;
        case 8: side_xform2<NT, 2, 0, 1>(tk, tid, cta, ncta, ptr_sh); break;
        case 9: side_xform2<NT, 2, 0, 2>(tk, tid, cta, ncta, ptr_sh); break;
        case 10: side_xform2<NT, 2, 1, 1>(tk, tid, cta, ncta, ptr_sh); break;
        case 11: side_xform2<NT, 2, 1, 2>(tk, tid, cta, ncta, ptr_sh); break;
        case 12: side_xform2<NT, 3, 0, 1>(tk, tid, cta, ncta, ptr_sh); break;
        case 13: side_xform2<NT, 3, 0, 2>(tk, tid, cta, ncta, ptr_sh); break;
        case 14: side_xform2<NT, 3, 1, 1>(tk, tid, cta, ncta, ptr_sh); break;
        default: side_xform2<NT, 3, 1, 2>(tk, tid, cta, ncta, ptr_sh); break;
      }
    } else if (tk.kind == 3) {
      switch (tk.table * 2 + (w2 ? 1 : 0)) {
        case 0: side_xpost2<NT, 0, 1>(tk, tid, cta, ncta, ptr_sh); break;
        case 1: side_xpost2<NT, 0, 1>(tk, tid, cta, ncta, ptr_sh); break;
        case 2: side_xpost2<NT, 1, 1>(tk, tid, cta, ncta, ptr_sh); break;
        case 3: side_xpost2<NT, 1, 1>(tk, tid, cta, ncta, ptr_sh); break;
        case 4: side_xpost2<NT, 2, 1>(tk, tid, cta, ncta, ptr_sh); break;
        case 5: side_xpost2<NT, 2, 1>(tk, tid, cta, ncta, ptr_sh); break;
        case 6: side_xpost2<NT, 3, 1>(tk, tid, cta, ncta, ptr_sh); break;
        default: side_xpost2<NT, 3, 1>(tk, tid, cta, ncta, ptr_sh); break;
      }
    } else if (tk.kind == 5) {
      switch (tk.table * 4 + tk.side * 2 + (w2 ? 1 : 0)) {
        case 0: side_xform1<NT, 0, 0, 1>(tk, tid, cta, ncta, ptr_sh); break;
        case 1: side_xform1<NT, 0, 0, 2>(tk, tid, cta, ncta, ptr_sh); break;
        case 2: side_xform1<NT, 0, 1, 1>(tk, tid, cta, ncta, ptr_sh); break;
        case 3: side_xform1<NT, 0, 1, 2>(tk, tid, cta, ncta, ptr_sh); break;
        case 4: side_xform1<NT, 1, 0, 1>(tk, tid, cta, ncta, ptr_sh); break;
        case 5: side_xform1<NT, 1, 0, 2>(tk, tid, cta, ncta, ptr_sh); break;
        case 6: side_xform1<NT, 1, 1, 1>(tk, tid, cta, ncta, ptr_sh); break;
        case 7: side_xform1<NT, 1, 1, 2>(tk, tid, cta, ncta, ptr_sh); break;
        case 8: side_xform1<NT, 2, 0, 1>(tk, tid, cta, ncta, ptr_sh); break;
        case 9: side_xform1<NT, 2, 0, 2>(tk, tid, cta, ncta, ptr_sh); break;
        case 10: side_xform1<NT, 2, 1, 1>(tk, tid, cta, ncta, ptr_sh); break;
        case 11: side_xform1<NT, 2, 1, 2>(tk, tid, cta, ncta, ptr_sh); break;
        case 12: side_xform1<NT, 3, 0, 1>(tk, tid, cta, ncta, ptr_sh); break;
        case 13: side_xform1<NT, 3, 0, 2>(tk, tid, cta, ncta, ptr_sh); break;
        case 14: side_xform1<NT, 3, 1, 1>(tk, tid, cta, ncta, ptr_sh); break;
        default: side_xform1<NT, 3, 1, 2>(tk, tid, cta, ncta, ptr_sh); break;
      }
    } else if (tk.kind == 4) {
      switch (tk.table * 2 + (w2 ? 1 : 0)) {
        case 0: side_xpost1<NT, 0, 1>(tk, tid, cta, ncta, ptr_sh); break;
        case 1: side_xpost1<NT, 0, 2>(tk, tid, cta, ncta, ptr_sh); break;
        case 2: side_xpost1<NT, 1, 1>(tk, tid, cta, ncta, ptr_sh); break;
        case 3: side_xpost1<NT, 1, 2>(tk, tid, cta, ncta, ptr_sh); break;
        case 4: side_xpost1<NT, 2, 1>(tk, tid, cta, ncta, ptr_sh); break;
        case 5: side_xpost1<NT, 2, 2>(tk, tid, cta, ncta, ptr_sh); break;
        case 6: side_xpost1<NT, 3, 1>(tk, tid, cta, ncta, ptr_sh); break;
        default: side_xpost1<NT, 3, 2>(tk, tid, cta, ncta, ptr_sh); break;
      }
    }
  }
}

// Work units of one persistent CTA: its data-parallel tiles (t = b, b + G, ... < sk_tile0, whole
// K), then its share [lo(b), lo(b + 1)) of the stream-K iterations (tile-major, k-minor) of the
// tiles from sk_tile0 on, as segments (tile, [kb, ke)). Producer and consumers walk the same
// sequence. The launcher guarantees (total - sk_tile0) * KT * G < 2^31.
__device__ __forceinline__ int sk_total(const MkGemmArgs& a) { return a.tiles_per_prod * (a.batch ? a.nprod : 1); }
__device__ __forceinline__ int sk_kt(const MkGemmArgs& a) { return (a.K + MK_BK - 1) / MK_BK; }
__device__ __forceinline__ int sk_tile0(const MkGemmArgs& a) { return min(a.sk_tile0, sk_total(a)); }
__device__ __forceinline__ int sk_lo(const MkGemmArgs& a, int c) {
  return (sk_total(a) - sk_tile0(a)) * sk_kt(a) * c / (int)gridDim.x;
}
__device__ __forceinline__ bool sk_unit(const MkGemmArgs& a, int it, int& t, int& kb, int& ke) {
  const int hi = sk_lo(a, (int)blockIdx.x + 1);
  if (it >= hi) return false;
  const int KT = sk_kt(a);
  const int tr = it / KT;
  t = sk_tile0(a) + tr;
  kb = it - tr * KT;
  ke = min(KT, kb + (hi - it));
  return true;
}
template <int MT, int BN, bool SK, bool SW = false>
__global__ void __launch_bounds__(PLayout<MT, BN, SW>::kThreads, 1)
persistent_product_kernel(const __grid_constant__ CUtensorMap tmA_param, const __grid_constant__ CUtensorMap tmB_param,
                          const __grid_constant__ CUtensorMap tmC_param, const __grid_constant__ MkGemmArgs args,
                          const __grid_constant__ MkProduct prod_param) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[kMaxStages];
  __shared__ __align__(8) uint64_t empty_bar[kMaxStages];
  __shared__ uint32_t tmem_base_sh;
  __shared__ double* side_ptr_sh[SW ? MK_XFORM2_MAX : 1];  // side work: a job's pointers

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int S = args.stages;
  const uint32_t smem_base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  uint8_t* smem_gen = smem_raw + (smem_base - smem_u32(smem_raw));
  using PL = PLayout<MT, BN, SW>;
  uint8_t* box_area = smem_gen + (size_t)S * PL::kStageBytes;  // epilogue boxes, one per consumer warp
  // epilogue descriptor ring (narrow data-parallel tiles): int32 [0] count, [1] pass-0 mask (the
  // destination's sign times the product's is +1), [2] accumulate mask, [4 + d] row, [12 + d] col
  int32_t* const slot_area = reinterpret_cast<int32_t*>(box_area + PL::kBoxBytes);
  const int tiles_per = args.tiles_m * args.tiles_n;
  const int total = tiles_per * (args.batch ? args.nprod : 1);
  const int KT = (args.K + MK_BK - 1) / MK_BK;
  // Slot reuse is safe while the producer, at most S stages ahead of the consumers' releases,
  // cannot reach the slot of a tile whose epilogue may still run: kEpiSlots >= ceil(S / KT) + 2.
  const bool use_slots = PL::kEpiSlots > 0 && !SK && args.batch != nullptr &&
                         PL::kEpiSlots >= (S + KT - 1) / KT + 2;

  auto tile_of = [&](int t, int& pi, int& m0, int& n0) {
    pi = t / tiles_per;
    const int bid = t - pi * tiles_per;
    const int per_group = args.group_m * args.tiles_n;
    const int g = bid / per_group;
    const int first_m = g * args.group_m;
    const int gsz = min(args.tiles_m - first_m, args.group_m);
    const int r = bid - g * per_group;
    m0 = (first_m + r % gsz) * MK_BM;
    n0 = (r / gsz) * BN;
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], PL::kConsumerWarps);
    }
    fence_barrier_init();
  }
  __syncthreads();
  // launched as a programmatic dependent (MK_PDL), the CTA may be resident before the previous
  // kernel of the stream has finished: everything above touches only shared memory
  pdl_wait();

  if (warp < PL::kLeadWarps) {
    // ============================ TMA producer (one thread) ============================
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(PL::kProducerRegs));
    if constexpr (PL::kSideWork) {  // warps 1..7: the launch's side work
      if (warp >= 1) {
        if (!SK && args.nside > 0) side_work<PL::kSideThreads>(args, threadIdx.x - 32u, blockIdx.x, gridDim.x, side_ptr_sh);
        return;
      }
    }
    if (threadIdx.x != 0) return;
    int s = 0;            // ring slot of the next stage (carried across tiles)
    uint32_t eph = 0;     // parity of the empty-barrier phase to wait for (first lap: no wait)
    bool first_lap = true;
    int tseq = 0;  // tiles issued (epilogue descriptor ring slot)
    auto unit = [&](const int t, const int kb, const int ke) {
      int pi, m0, n0;
      tile_of(t, pi, m0, n0);
      const MkBatchEntry* ent = args.batch ? args.batch + pi : nullptr;
      const MkProduct& prod = ent ? ent->prod : prod_param;
      const CUtensorMap* tmA = ent ? &ent->tmA : &tmA_param;
      const CUtensorMap* tmB = ent ? &ent->tmB : &tmB_param;
      const int ar = m0 + prod.a[0].row, ac = prod.a[0].col;
      const int br = prod.b[0].row, bc = n0 + prod.b[0].col;
      if (use_slots) {
        // Written before the tile's first stage is armed (mbarrier arrive: release; the consumers'
        // wait on it: acquire). Reuse (see use_slots): writing tile T + R's slot needs the
        // consumers to have released every stage up to S stages before it, i.e. to be past
        // tile T's main loop and, warp by warp, its epilogue.
        int32_t* sl = slot_area + (tseq & (PL::kEpiSlots - 1)) * PL::kEpiSlotInts;
        const double osg = prod.a[0].sign * prod.b[0].sign;
        uint32_t pos = 0, accm = 0;
        for (int d = 0; d < prod.nd; ++d) {
          const MkDest& dd = prod.d[d];
          if (dd.sign * osg > 0.0) pos |= 1u << d;
          if (dd.accumulate) accm |= 1u << d;
          if (d < PL::kEpiSlotDests) {
            sl[4 + d] = (int32_t)dd.row;
            sl[12 + d] = (int32_t)dd.col;
          }
        }
        sl[0] = prod.nd;
        sl[1] = (int32_t)pos;
        sl[2] = (int32_t)accm;
        ++tseq;
      }
      for (int k = kb; k < ke; ++k) {
        if (!first_lap) mbar_wait(&empty_bar[s], eph);
        uint8_t* opA = smem_gen + (size_t)s * PL::kStageBytes;
        uint8_t* opB = opA + MK_TILE_BYTES;
        const int k0 = k * MK_BK;
        mbar_arrive_expect_tx(&full_bar[s], PL::kStageBytes);
        tma_load_2d(opA, tmA, k0 + ac, ar, &full_bar[s]);
#pragma unroll
        for (int bj = 0; bj < BN / 16; ++bj) tma_load_2d(opB + bj * 2048, tmB, bc + bj * 16, k0 + br, &full_bar[s]);
        if (++s == S) {
          s = 0;
          if (first_lap)
            first_lap = false;
          else
            eph ^= 1u;
        }
      }
    };
    if constexpr (!SK) {  // data-parallel tiles [0, min(total, sk_tile0))
      const int lim = min(total, args.sk_tile0);
      for (int t = blockIdx.x; t < lim; t += gridDim.x) unit(t, 0, KT);
    } else {  // stream-K segments of tiles [sk_tile0, total)
      const int tile0 = sk_tile0(args);
      int t, kb, ke;
      for (bool live = sk_unit(args, sk_lo(args, blockIdx.x), t, kb, ke); live;
           live = sk_unit(args, (t - tile0) * KT + ke, t, kb, ke))
        unit(t, kb, ke);
    }
    // every load of this CTA is issued: its consumers are at most S stages and one epilogue from
    // the end, so the stream's next kernel may start taking the SMs that fall idle
    pdl_trigger();
    return;
  }

  // ================================ DMMA consumers ================================
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(PL::kConsumerRegs));
  const int cw = warp - PL::kLeadWarps;
  const int warp_m = cw / PL::kWarpsN;
  const int warp_n = cw % PL::kWarpsN;
  const int q = lane & 3, g = lane >> 2;
  const int prow = (g >> 1) + 4 * (g & 1);
  const uint32_t a_lane = (uint32_t)(warp_m * (8 * MT) + prow) * 128u;
  const uint32_t a_chunk0 = (uint32_t)(((q + 0) ^ prow) << 4);
  const uint32_t a_chunk1 = (uint32_t)(((q + 4) ^ prow) << 4);
  const uint32_t b_lane = (uint32_t)(warp_n * 2) * 2048u;
  uint32_t b_off[2][2];
#pragma unroll
  for (int t = 0; t < 2; ++t)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int k = 2 * q + 8 * t + e;
      b_off[t][e] = b_lane + (uint32_t)k * 128u + (uint32_t)((g ^ ((2 * q + e) & 7)) << 4);
    }

  double acc[MT][4][2];
  auto stage = [&](const uint8_t* sA, const uint8_t* sB, const int krem, auto tail_tag) {
    constexpr bool TAIL = decltype(tail_tag)::value;
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      // last k-stage: k-steps 8t.. past the end of K hold only zero padding; skip their DMMAs
      // (they would add exact zeros: the accumulators are unchanged bit for bit)
      if (TAIL && MK_TAIL_SKIP && 8 * t >= krem) break;
      const uint32_t a_chunk = t ? a_chunk1 : a_chunk0;
      double a0[MT], a1[MT];
#pragma unroll
      for (int i = 0; i < MT; ++i) lds128(a0[i], a1[i], sA + a_lane + i * 1024u + a_chunk);
      if (TAIL) {
        const int kk = 2 * q + 8 * t;
#pragma unroll
        for (int i = 0; i < MT; ++i) {
          a0[i] = kk < krem ? a0[i] : 0.0;
          a1[i] = kk + 1 < krem ? a1[i] : 0.0;
        }
      }
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        double b[4];
        lds128(b[0], b[1], sB + b_off[t][e]);
        lds128(b[2], b[3], sB + b_off[t][e] + 2048u);
        if (TAIL) {
          const bool live = 2 * q + 8 * t + e < krem;
#pragma unroll
          for (int f = 0; f < 4; ++f) b[f] = live ? b[f] : 0.0;
        }
#pragma unroll
        for (int i = 0; i < MT; ++i)
#pragma unroll
          for (int f = 0; f < 4; ++f) dmma(acc[i][f][0], acc[i][f][1], e ? a1[i] : a0[i], b[f]);
      }
    }
  };

  // two-level accumulation (see fused_product_kernel); TMEM is allocated once per CTA
  // leaves with K <= 512 keep a single register sum (<= 512 terms): folding them buys little
  const int chunk = (args.chunk_stages > 0 && KT > 32 && KT > args.chunk_stages) ? args.chunk_stages : 0;
  constexpr int kWords = 16 * MT;
  constexpr int kPieces = kWords / 16;
  uint32_t taddr = 0;
  if (chunk) {
    if (cw == 0) tmem_alloc(&tmem_base_sh, 256);
    tmem_fence_before();
    named_bar_sync(3, 32 * PL::kConsumerWarps);
    tmem_fence_after();
    taddr = tmem_base_sh + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((cw >> 2) * kWords);
  }
  bool master_live = false;
  auto fold_to_tmem = [&]() {
#ifndef MK_FOLD_GROUP
#define MK_FOLD_GROUP 2
#endif
    constexpr int kGrp = MK_FOLD_GROUP < kPieces ? MK_FOLD_GROUP : kPieces;  // pieces per tcgen05.ld round trip
#pragma unroll
    for (int pc = 0; pc < kPieces; pc += kGrp) {
      uint32_t w[kGrp][16];
      if (master_live) {
#pragma unroll
        for (int h = 0; h < kGrp; ++h) tmem_ld16(taddr + (pc + h) * 16, w[h]);
        tmem_wait_ld();
      }
#pragma unroll
      for (int h = 0; h < kGrp; ++h)
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int e = (pc + h) * 8 + u;
          double& a = acc[e >> 3][(e >> 1) & 3][e & 1];
          const double m = master_live ? __hiloint2double((int)w[h][2 * u + 1], (int)w[h][2 * u]) + a : a;
          w[h][2 * u] = (uint32_t)__double2loint(m);
          w[h][2 * u + 1] = (uint32_t)__double2hiint(m);
          a = 0.0;
        }
#pragma unroll
      for (int h = 0; h < kGrp; ++h) tmem_st16(taddr + (pc + h) * 16, w[h]);
    }
    tmem_wait_st();
    master_live = true;
  };

  constexpr int kBoxRows = 8 * MT;
  uint8_t* const box0 = box_area + (size_t)cw * (kBoxRows * 128);
  int ebuf = 0;  // next epilogue box of this warp (carried across tiles)
  const int c_first = (g & 1) ? 1 : 0;
  bool reads_pending = false;  // TMA reads of this warp's box still in flight
  const int krem_last = args.K - (KT - 1) * MK_BK;
  int rs = 0;         // ring slot of the next stage (carried across tiles)
  uint32_t fph = 0;   // parity of the full-barrier phase to wait for
  int tseq = 0;       // tiles done (epilogue descriptor ring slot)

  // One unit: tile t, k-stages [kb, ke). Instantiated twice below -- data-parallel tiles (kb = 0,
  // ke = KT: the original loop, no extra live registers next to the 128-register accumulator)
  // and stream-K segments.
  auto unit = [&](const int t, const int kb, const int ke) {
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
      for (int f = 0; f < 4; ++f) acc[i][f][0] = acc[i][f][1] = 0.0;
    master_live = false;
    for (int kt = kb; kt < ke; ++kt) {
      mbar_wait(&full_bar[rs], fph);
      const uint8_t* sA = smem_gen + (size_t)rs * PL::kStageBytes;
      const uint8_t* sB = sA + MK_TILE_BYTES;
      if (kt == KT - 1 && krem_last < MK_BK)
        stage(sA, sB, krem_last, std::true_type{});
      else
        stage(sA, sB, MK_BK, std::false_type{});
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty_bar[rs]);
      if (++rs == S) {
        rs = 0;
        fph ^= 1u;
      }
      if (chunk && (kt + 1 - kb) % chunk == 0 && kt + 1 < ke) fold_to_tmem();
    }
    int pi, m0, n0;
    tile_of(t, pi, m0, n0);
    const MkBatchEntry* ent = args.batch ? args.batch + pi : nullptr;
    const MkProduct& prod = ent ? ent->prod : prod_param;
    if (chunk && master_live) {
#pragma unroll
      for (int pc = 0; pc < kPieces; ++pc) {
        uint32_t w[16];
        tmem_ld16(taddr + pc * 16, w);
        tmem_wait_ld();
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int e = pc * 8 + u;
          double& a = acc[e >> 3][(e >> 1) & 3][e & 1];
          a = __hiloint2double((int)w[2 * u + 1], (int)w[2 * u]) + a;
        }
      }
    }

    // ---- stream-K: a tile split over several CTAs is finished by whichever segment arrives last
    // (per warp: each warp's 64 x 32 piece is independent). Every segment publishes its partial
    // sum in its own slot (2 per CTA: its head segment and its other one) and counts up the
    // tile's flag; the last arriver adds all slots in k order -- deterministic, and nobody waits.
    if (SK && (kb > 0 || ke < KT)) {
      // slot layout [e/2][lane] of double2: every access is one 512-byte warp transaction
      constexpr int kPairs = MT * 4;  // accumulator double pairs per thread
      const size_t slot_pairs = (size_t)PL::kConsumerWarps * kPairs * 32;
      double2* const base2 = reinterpret_cast<double2*>(args.sk_partial);
      auto slot_of = [&](int cta, bool head) {
        return base2 + (size_t)(2 * cta + (head ? 1 : 0)) * slot_pairs + (size_t)cw * kPairs * 32 + lane;
      };
      {
        double2* mine = slot_of(blockIdx.x, kb == 0);
#pragma unroll
        for (int e2 = 0; e2 < kPairs; ++e2) {
          const int e = 2 * e2;
          __stcg(mine + e2 * 32, make_double2(acc[e >> 3][(e >> 1) & 3][e & 1], acc[e >> 3][(e >> 1) & 3][(e & 1) + 1]));
        }
      }
      // CTAs holding the tile's segments: b0 (head) .. b1
      const int G = gridDim.x, tile0 = sk_tile0(args);
      const int tile_begin = (t - tile0) * KT, tile_end = tile_begin + KT;
      int b0 = (int)((long long)tile_begin * G / ((long long)(total - tile0) * KT));
      while (b0 > 0 && sk_lo(args, b0) > tile_begin) --b0;
      while (b0 + 1 < G && sk_lo(args, b0 + 1) <= tile_begin) ++b0;
      int b1 = b0, nseg = 1;  // CTAs with a non-empty share of the tile: b0 and the non-empty ones up to b1
      while (b1 + 1 < G && sk_lo(args, b1 + 1) < tile_end) {
        ++b1;
        if (sk_lo(args, b1) < sk_lo(args, b1 + 1)) ++nseg;
      }
      int32_t* flag = args.sk_flags + (size_t)(t - tile0) * PL::kConsumerWarps + cw;
      __syncwarp();  // the warp's partial stores precede lane 0's release below
      int old = 0;
      if (lane == 0)
        asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;" : "=r"(old) : "l"(flag) : "memory");
      old = __shfl_sync(0xffffffffu, old, 0);
      if (old != nseg - 1) return;  // another segment finishes this piece
      // last arriver: sum the segments in k order (head first) -- deterministic. A head that
      // arrives last (the usual case: heads close their CTA's range) keeps its own sum in registers.
      auto add_slot = [&](const double2* sl) {
#pragma unroll
        for (int e2 = 0; e2 < kPairs; ++e2) {
          const double2 v = __ldcg(sl + e2 * 32);
          const int e = 2 * e2;
          acc[e >> 3][(e >> 1) & 3][e & 1] += v.x;
          acc[e >> 3][(e >> 1) & 3][(e & 1) + 1] += v.y;
          if ((e2 & 15) == 15) asm volatile("" ::: "memory");  // <= 16 loads in flight (registers)
        }
      };
      if (kb != 0) {  // reload the head's sum
        const double2* hs = slot_of(b0, true);
#pragma unroll
        for (int e2 = 0; e2 < kPairs; ++e2) {
          const double2 v = __ldcg(hs + e2 * 32);
          const int e = 2 * e2;
          acc[e >> 3][(e >> 1) & 3][e & 1] = v.x;
          acc[e >> 3][(e >> 1) & 3][(e & 1) + 1] = v.y;
          if ((e2 & 15) == 15) asm volatile("" ::: "memory");
        }
      }
      for (int c = b0 + 1; c <= b1; ++c)
        if (sk_lo(args, c) < sk_lo(args, c + 1)) add_slot(slot_of(c, false));
      if (lane == 0) *flag = 0;  // ready for the next launch on this stream
    }

    // ---- epilogue: every destination of the product, signs grouped into two passes ----
    if (args.async_epi) {
      const CUtensorMap* tmC = ent ? &ent->tmC : &tmC_param;
      const int row0 = m0 + warp_m * kBoxRows;
      const int col0 = n0 + warp_n * 32;
      const bool slab_live = row0 < args.M && col0 < args.N;
      const int32_t* const sl = use_slots ? slot_area + (tseq & (PL::kEpiSlots - 1)) * PL::kEpiSlotInts : nullptr;
      uint32_t pos_mask = 0, all_mask = 0, acc_mask = 0;
      if (use_slots) {
        const int nds = sl[0];
        all_mask = nds >= 32 ? 0xffffffffu : (1u << nds) - 1u;
        pos_mask = (uint32_t)sl[1];
        acc_mask = (uint32_t)sl[2];
      } else {
        const double out_sign = prod.a[0].sign * prod.b[0].sign;
        for (int d = 0; d < prod.nd; ++d) {
          all_mask |= 1u << d;
          if (prod.d[d].sign * out_sign > 0.0) pos_mask |= 1u << d;
          if (prod.d[d].accumulate) acc_mask |= 1u << d;
        }
      }
      for (int pass = 0; pass < 2; ++pass) {
        const uint32_t pass_mask = pass == 0 ? pos_mask : (all_mask & ~pos_mask);
        if (!pass_mask) continue;
        // the pass's sign is a sign-bit flip of the accumulators (integer pipe, not a DMUL)
        const long long flip = pass == 0 ? 0ll : (long long)0x8000000000000000ull;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          uint8_t* const box = box0 + (size_t)ebuf * (PL::kConsumerWarps * kBoxRows * 128);
          if (reads_pending) {  // the box's previous contents must have been read by the TMA unit
            // one bulk group per box fill: the group that used this box is kEpiBufs fills old
            if (lane == 0) bulk_wait_read<PL::kEpiBufs - 1>();
            __syncwarp();
          }
#pragma unroll
          for (int i = 0; i < MT; ++i) {
            const int r = 8 * i + prow;
            uint8_t* rowp = box + r * 128;
            auto sg = [&](double x) { return __longlong_as_double(__double_as_longlong(x) ^ flip); };
            const double v0 = sg(acc[i][2 * j][0]), v1 = sg(acc[i][2 * j + 1][0]);
            const double v2 = sg(acc[i][2 * j][1]), v3 = sg(acc[i][2 * j + 1][1]);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int c = 2 * q + (h ^ c_first);
              double2 v = (c & 1) ? make_double2(v2, v3) : make_double2(v0, v1);
              *reinterpret_cast<double2*>(rowp + ((c ^ prow) << 4)) = v;
            }
          }
          fence_proxy_async();
          __syncwarp();
          if (lane == 0) {
            if (slab_live && col0 + 16 * j < args.N) {
              for (uint32_t m = pass_mask; m; m &= m - 1) {
                const int d = __ffs(m) - 1;
                const bool in_slot = use_slots && d < PL::kEpiSlotDests;
                const int drow = in_slot ? sl[4 + d] : (int)prod.d[d].row;
                const int dcol = in_slot ? sl[12 + d] : (int)prod.d[d].col;
                const int cc = dcol + col0 + 16 * j, rr = drow + row0;
                if (acc_mask & (1u << d))
                  tma_reduce_add_2d(tmC, cc, rr, box);
                else
                  tma_store_2d(tmC, cc, rr, box);
              }
            }
            bulk_commit();  // (possibly empty) group per box fill, so wait_group counts box fills
          }
          reads_pending = true;
          if (++ebuf == PL::kEpiBufs) ebuf = 0;
        }
      }
    } else {
      const double out_sign = prod.a[0].sign * prod.b[0].sign;
      const int nd = prod.nd;
      double* const Cbase = ent ? ent->C : args.C;
      const int64_t ldc = ent ? ent->ldc : args.ldc;
      for (int d = 0; d < nd; ++d) {
        const MkDest dst = prod.d[d];
        const double sg = dst.sign * out_sign;
        double* Cd = Cbase + dst.row * ldc + dst.col;
#pragma unroll
        for (int i = 0; i < MT; ++i) {
          const int row = m0 + warp_m * (8 * MT) + 8 * i + prow;
          if (row >= args.M) continue;
          double* crow = args.nslab ? slab_row(args, dst.row + row, ldc) + dst.col : Cd + (int64_t)row * ldc;
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const int col = n0 + warp_n * 32 + 16 * j + 4 * q;
            const double v[4] = {acc[i][2 * j][0], acc[i][2 * j + 1][0], acc[i][2 * j][1], acc[i][2 * j + 1][1]};
            if (args.vec_ok) {
              if (col >= args.N) continue;
              double* p = crow + col;
              if (dst.accumulate) {
#pragma unroll
                for (int u = 0; u < 4; ++u) red_add(p + u, sg * v[u]);
              } else {
                stg256(p, sg * v[0], sg * v[1], sg * v[2], sg * v[3]);
              }
            } else {
#pragma unroll
              for (int u = 0; u < 4; ++u)
                if (col + u < args.N) {
                  if (dst.accumulate)
                    red_add(crow + col + u, sg * v[u]);
                  else
                    crow[col + u] = sg * v[u];
                }
            }
          }
        }
      }
    }
  };
  if constexpr (!SK) {
    const int lim = min(total, args.sk_tile0);
    for (int t = blockIdx.x; t < lim; t += gridDim.x) {
      unit(t, 0, KT);
      ++tseq;
    }
  } else {
    const int tile0 = sk_tile0(args);
    int t, kb, ke;
    for (bool live = sk_unit(args, sk_lo(args, blockIdx.x), t, kb, ke); live;
         live = sk_unit(args, (t - tile0) * KT + ke, t, kb, ke))
      unit(t, kb, ke);
  }
  if (lane == 0) bulk_wait_read_all();  // the boxes must stay valid until the TMA unit has read them
  __syncwarp();
  if (chunk) {
    tmem_fence_before();
    named_bar_sync(3, 32 * PL::kConsumerWarps);
    tmem_fence_after();
    if (cw == 0) tmem_dealloc(tmem_base_sh, 256);
  }
}

#ifdef MK_TRACE
extern "C" __attribute__((visibility("default"))) int mk_trace_read(unsigned long long* out, int n) {
  return (int)cudaMemcpyFromSymbol(out, mk_trace_buf, sizeof(unsigned long long) * 5 * n);
}
#endif

// ------------------------------------------------------------------------------------
// Host-side launcher (called by the planner).
// ------------------------------------------------------------------------------------
// Consumer warps per CTA: 8 (MT=8, default) or 16 (MT=4); env MK_CONSUMER_WARPS overrides.
static std::atomic<int> g_consumer_layout{0};
int consumer_layout() {
  if (g_consumer_layout == 0) {
    const char* e = getenv("MK_CONSUMER_WARPS");
    g_consumer_layout = (e && atoi(e) == 16) ? 16 : 8;
  }
  return g_consumer_layout;
}
void set_consumer_layout(int warps) { g_consumer_layout = (warps == 8) ? 8 : 16; }

// Stages per register chunk of the two-level (register + TMEM) accumulation; 0 disables it.
// Default 16 stages = 256 k (errors below the reference CPU's on every config, for ~0.7% of the main
// loop; 32 stages: 1.3x the reference's errors). Env MK_ACC_CHUNK overrides (0 = single-level).
static std::atomic<int> g_chunk{-1};
int accumulate_chunk_stages() {
  if (g_chunk < 0) {
    const char* e = getenv("MK_ACC_CHUNK");
    g_chunk = e ? atoi(e) : 16;
    if (g_chunk < 0) g_chunk = 0;
  }
  return g_chunk;
}

// Persistent plain-product kernel (env MK_PERSISTENT=0 selects the one-CTA-per-tile kernel).
static std::atomic<int> g_persistent{-1};
bool persistent_enabled() {
  if (g_persistent < 0) {
    const char* e = getenv("MK_PERSISTENT");
    g_persistent = (e && e[0] == '0') ? 0 : 1;
  }
  return g_persistent == 1;
}
static int sm_count() {
  static std::atomic<int> cache[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  if (cache[dev] == 0) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
    cache[dev] = n;
  }
  return cache[dev];
}
// Stream-K tail of the persistent kernel (default on; env MK_STREAMK=0 disables): launches
// whose tiles leave the last wave partial split the k-iterations of the tail over every SM.
static std::atomic<int> g_streamk{-1};
bool streamk_enabled() {
  if (g_streamk < 0) {
    const char* e = getenv("MK_STREAMK");
    g_streamk = (e && e[0] == '0') ? 0 : 1;
  }
  return g_streamk == 1;
}

// Per (device, stream) stream-K scratch: two partial-tile slots per CTA and one flag per
// (stream-K tile, consumer warp). Flags start at zero and every owner resets the ones it used,
// so launches on one stream reuse them; launches on different streams never share them.
struct SkScratch {
  double* partial = nullptr;
  int32_t* flags = nullptr;
  size_t partial_bytes = 0, flag_count = 0;
};
static cudaError_t sk_scratch(cudaStream_t stream, int ctas, int warps, int acc_per_thread, int sk_tiles,
                              SkScratch** out) {
  static std::mutex mu;
  static std::map<std::pair<int, cudaStream_t>, SkScratch> cache;
  int dev = 0;
  cudaError_t err = cudaGetDevice(&dev);
  if (err != cudaSuccess) return err;
  std::lock_guard<std::mutex> lock(mu);
  SkScratch& sc = cache[{dev, stream}];
  const size_t pbytes = (size_t)2 * ctas * warps * acc_per_thread * 32 * sizeof(double);
  const size_t nflags = (size_t)sk_tiles * warps;
  if (sc.partial_bytes < pbytes) {
    if (sc.partial) cudaFree(sc.partial);
    sc.partial = nullptr;
    sc.partial_bytes = 0;
    err = cudaMalloc(&sc.partial, pbytes);
    if (err != cudaSuccess) return err;
    sc.partial_bytes = pbytes;
  }
  if (sc.flag_count < nflags) {
    if (sc.flags) cudaFree(sc.flags);
    sc.flags = nullptr;
    sc.flag_count = 0;
    const size_t want = nflags < 4096 ? 4096 : nflags;
    err = cudaMalloc(&sc.flags, want * sizeof(int32_t));
    if (err != cudaSuccess) return err;
    err = cudaMemsetAsync(sc.flags, 0, want * sizeof(int32_t), stream);
    if (err != cudaSuccess) return err;
    sc.flag_count = want;
  }
  *out = &sc;
  return cudaSuccess;
}

// Tile width of the persistent kernel: 64 when it cuts the column padding of the leaf by more
// than 10% (e.g. cfg5's 320-column leaves: 5 tiles instead of 3 x 128 with 17% padding), else
// 128. Env MK_NARROW=0 disables narrow tiles. Also narrow when 128-column tiles would leave most
// SMs idle (fewer than 60% of the SM count in tiles, e.g. one 1024^2 leaf of a literal schedule). Narrow tiles run 8 warps
// of 32 x 32, so their TMA epilogue boxes are 32 rows (the planner builds the C maps to match:
// epilogue_box_rows).
static int sm_count();
int persistent_tile_n(int64_t tiles_m, int64_t N, int nprod) {
  static std::atomic<int> narrow{-1};
  if (narrow < 0) {
    const char* e = getenv("MK_NARROW");
    narrow = (e && e[0] == '0') ? 0 : (e && e[0] == '2') ? 2 : 1;  // 2: always narrow (studies)
  }
  if (!narrow) return 128;
  if (narrow == 2) return 64;
  const int64_t tiles128 = tiles_m * ((N + 127) / 128) * nprod;
  if (tiles128 * 10 < (int64_t)sm_count() * 6) return 64;
  const int64_t w128 = (N + 127) / 128 * 128, w64 = (N + 63) / 64 * 64;
  return (w64 * 10 < w128 * 9) ? 64 : 128;
}
int epilogue_box_rows(int64_t M, int64_t N, int nprod, bool single_terms) {
  // multi-term operands run the one-CTA-per-tile combiner kernel (128-column tiles)
  if (single_terms && persistent_enabled() && persistent_tile_n((M + MK_BM - 1) / MK_BM, N, nprod) == 64) return 32;
  return consumer_layout() == 16 ? 32 : 64;
}
static int persistent_bn(const MkGemmArgs& a, int nprod) { return persistent_tile_n(a.tiles_m, a.N, nprod); }

// One CTA per SM over the launch's tiles; the ring keeps S = (budget - boxes) / stage stages.
template <int MT, int BN>
static cudaError_t launch_persistent_t(const CUtensorMap& tmA, const CUtensorMap& tmB, const CUtensorMap& tmC,
                                       MkGemmArgs args, const MkProduct& prod, int nprod, cudaStream_t stream) {
  using PL = PLayout<MT, BN>;
  args.tiles_n = (args.N + BN - 1) / BN;
  const int tiles = args.tiles_m * args.tiles_n;
  // side work rides on the data-parallel launch of a narrow-tile kernel; otherwise (or when
  // this launch has no data-parallel part) it runs as stand-alone launches after the leaves
  static const bool attach = [] {  // env MK_SIDE_ATTACH=0: side tasks always as their own launches
    const char* e = getenv("MK_SIDE_ATTACH");
    return !(e && e[0] == '0');
  }();
  MkSideTask carry[MK_SIDE_MAX];  // the tasks this kernel can carry (kinds 2, 3; see side_work)
  int ncarry = 0;
  std::vector<MkSideTask> own;   // the rest: stand-alone launches
  for (int t = 0; t < args.nside; ++t) {
    const MkSideTask& tk = args.side[t];
    const int64_t groups = tk.rows * (tk.cols / (tk.width > 0 ? tk.width : 1)) * tk.njobs;
    if (attach && BN == 64 && (tk.kind >= 2 && tk.kind <= 5) && (tk.width == 1 || tk.width == 2) && tk.cols % tk.width == 0 &&
        groups < ((int64_t)1 << 32))
      carry[ncarry++] = tk;
    else
      own.push_back(tk);
  }
  args.nside = 0;
  for (const MkSideTask& tk : own) {  // independent of the leaves and of the other tasks: any order
    const cudaError_t e = launch_side_task(tk, stream);
    if (e != cudaSuccess) return e;
  }
  auto side_after = [&](cudaError_t e) {
    for (int t = 0; e == cudaSuccess && t < ncarry; ++t) e = launch_side_task(carry[t], stream);
    return e;
  };
  if (tiles == 0) return side_after(cudaSuccess);
  if ((int64_t)tiles * nprod > 0x7fffffff) return cudaErrorInvalidValue;
  args.tiles_per_prod = tiles;
  args.nprod = nprod;
  args.stages = (int)((MK_SMEM_BUDGET - PL::kBoxBytes) / PL::kStageBytes);
  if (args.stages > kMaxStages) args.stages = kMaxStages;
  args.raw_sets = 0;
  args.chunk_stages = accumulate_chunk_stages();
  const size_t smem = (size_t)args.stages * PL::kStageBytes + PL::kBoxBytes + PL::kEpiSlotBytes + 1024;
  cudaError_t err = cudaSuccess;
  const int total = tiles * nprod;
  int grid = total < sm_count() ? total : sm_count();
  args.sk_tile0 = total;
  args.sk_partial = nullptr;
  args.sk_flags = nullptr;
  const int G = sm_count();
  const int KT = (args.K + MK_BK - 1) / MK_BK;
  const int rem = total % G;
  auto dp = persistent_product_kernel<MT, BN, false>;
  err = cudaFuncSetAttribute(dp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (err != cudaSuccess) return err;
  // the data-parallel launch with the side work it carries (512-thread layout, same smem plan)
  auto launch_dp_side = [&](int g) {
    using PW = PLayout<MT, BN, BN == 64>;
    static_assert(PW::kStageBytes == PL::kStageBytes && PW::kBoxBytes == PL::kBoxBytes, "side layout smem plan");
    const size_t smem_w = (size_t)args.stages * PW::kStageBytes + PW::kBoxBytes + PW::kEpiSlotBytes + 1024;
    auto dw = persistent_product_kernel<MT, BN, false, BN == 64>;
    cudaError_t e2 = cudaFuncSetAttribute(dw, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_w);
    if (e2 != cudaSuccess) return e2;
    MkGemmArgs dargs = args;
    dargs.nside = ncarry;
    for (int t = 0; t < ncarry; ++t) dargs.side[t] = carry[t];
    dw<<<g, PW::kThreads, smem_w, stream>>>(tmA, tmB, tmC, dargs, prod);
    return cudaGetLastError();
  };
  // only when the last wave is less than 3/4 full: a nearly full last wave loses less than the
  // stream-K launch costs (measured on 1024-tile launches: 6.92 waves)
  if (streamk_enabled() && total > G && rem != 0 && rem * 4 < G * 3 && KT >= 8 &&
      (int64_t)(rem + G) * KT * G < ((int64_t)1 << 31)) {
    // Data-parallel waves, then stream-K over the partial last wave plus one full wave (every
    // CTA's share is one to two tiles of k-iterations), as two launches: the stream-K kernel's
    // extra state would cost the data-parallel main loop registers. Launches of less than one
    // wave stay data-parallel (narrow tiles fill the SMs there; measured faster at 1024^2).
    const int tile0 = (total / G - 1) * G;
    SkScratch* sc = nullptr;
    err = sk_scratch(stream, G, PL::kConsumerWarps, MT * 8, total - tile0, &sc);
    if (err != cudaSuccess) return err;
    args.sk_tile0 = tile0;
    args.sk_partial = sc->partial;
    args.sk_flags = sc->flags;
    bool side_done = false;
    if (tile0 > 0) {
      if (ncarry > 0) {
        err = launch_dp_side(G);
        side_done = true;
      } else {
        err = launch_dep(false, dp, dim3(G), dim3(PL::kThreads), smem, stream, tmA, tmB, tmC, args, prod);
      }
      if (err != cudaSuccess) return err;
    }
    auto sk = persistent_product_kernel<MT, BN, true>;
    err = cudaFuncSetAttribute(sk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (err != cudaSuccess) return err;
    err = launch_dep(false, sk, dim3(G), dim3(PL::kThreads), smem, stream, tmA, tmB, tmC, args, prod);
    return side_done ? err : side_after(err);
  }
  if (ncarry > 0) return launch_dp_side(grid);
  return side_after(launch_dep(total <= G, dp, dim3(grid), dim3(PL::kThreads), smem, stream, tmA, tmB, tmC, args, prod));
}

static cudaError_t launch_persistent(const CUtensorMap& tmA, const CUtensorMap& tmB, const CUtensorMap& tmC,
                                     MkGemmArgs args, const MkProduct& prod, int nprod, cudaStream_t stream) {
  if (persistent_bn(args, nprod) == 64)  // async epilogue: tmC has 32-row boxes (epilogue_box_rows)
    return launch_persistent_t<4, 64>(tmA, tmB, tmC, args, prod, nprod, stream);
  if (consumer_layout() == 16) return launch_persistent_t<4, 128>(tmA, tmB, tmC, args, prod, nprod, stream);
  return launch_persistent_t<8, 128>(tmA, tmB, tmC, args, prod, nprod, stream);
}

cudaError_t launch_fused_product(const CUtensorMap& tmA, const CUtensorMap& tmB, const CUtensorMap& tmC,
                                 const MkGemmArgs& args_in, const MkProduct& prod, cudaStream_t stream) {
  if (prod.na < 1 || prod.na > MK_MAX_TERMS || prod.nb < 1 || prod.nb > MK_MAX_TERMS) return cudaErrorInvalidValue;
  MkGemmArgs args = args_in;
  const bool ca = prod.na > 1, cb = prod.nb > 1;
  if (!ca && !cb && persistent_enabled()) {
    args.batch = nullptr;
    return launch_persistent(tmA, tmB, tmC, args, prod, 1, stream);
  }
  const int raw_tiles = (ca ? prod.na : 0) + (cb ? prod.nb : 0);
  const size_t raw_set = (size_t)raw_tiles * MK_TILE_BYTES;
  const size_t budget = MK_SMEM_BUDGET;
  int stages, sets = 0;
  if (raw_tiles == 0) {
    stages = (int)(budget / kOpStageBytes);
  } else {
    // two raw sets when they fit next to >= 2 operand stages, else one
    sets = (budget >= 2 * raw_set + 2 * kOpStageBytes) ? 2 : 1;
    stages = (int)((budget - (size_t)sets * raw_set) / kOpStageBytes);
    if (stages < 2) return cudaErrorInvalidValue;
  }
  if (stages > kMaxStages) stages = kMaxStages;
  args.stages = stages;
  args.raw_sets = sets;
  args.chunk_stages = accumulate_chunk_stages();
  const size_t smem = (size_t)stages * kOpStageBytes + (size_t)sets * raw_set + 1024;
  const int grid = args.tiles_m * args.tiles_n;
  if (grid == 0) return cudaSuccess;
  using KernelFn = void (*)(const CUtensorMap, const CUtensorMap, const CUtensorMap, const MkGemmArgs,
                            const MkProduct);
  static const KernelFn table[2][2][2] = {
      {{fused_product_kernel<false, false, 8>, fused_product_kernel<false, true, 8>},
       {fused_product_kernel<true, false, 8>, fused_product_kernel<true, true, 8>}},
      {{fused_product_kernel<false, false, 4>, fused_product_kernel<false, true, 4>},
       {fused_product_kernel<true, false, 4>, fused_product_kernel<true, true, 4>}},
  };
  const int wide = consumer_layout() == 16 ? 1 : 0;
  KernelFn fn = table[wide][ca ? 1 : 0][cb ? 1 : 0];
  const int threads = wide ? Layout<4>::kThreads : Layout<8>::kThreads;
  cudaError_t err = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (err != cudaSuccess) return err;
  fn<<<grid, threads, smem, stream>>>(tmA, tmB, tmC, args, prod);
  return cudaGetLastError();
}

cudaError_t launch_product_batch(const MkBatchEntry* entries_dev, int nprod, const MkGemmArgs& args_in,
                                 cudaStream_t stream) {
  MkGemmArgs args = args_in;
  const int tiles = args.tiles_m * args.tiles_n;
  if (nprod <= 0 || tiles == 0) {  // no leaves: only the side work
    cudaError_t err = cudaSuccess;
    for (int t = 0; err == cudaSuccess && t < args.nside; ++t) err = launch_side_task(args.side[t], stream);
    return err;
  }
  if ((int64_t)tiles * nprod > 0x7fffffff) return cudaErrorInvalidValue;
  args.stages = (int)(MK_SMEM_BUDGET / kOpStageBytes);
  if (args.stages > kMaxStages) args.stages = kMaxStages;
  args.raw_sets = 0;
  args.chunk_stages = accumulate_chunk_stages();
  args.tiles_per_prod = tiles;
  args.batch = entries_dev;
  args.nprod = nprod;
  if (persistent_enabled()) {
    CUtensorMap z{};
    MkProduct zp{};
    zp.na = zp.nb = 1;
    return launch_persistent(z, z, z, args, zp, nprod, stream);
  }
  const size_t smem = (size_t)args.stages * kOpStageBytes + 1024;
  const bool wide = consumer_layout() == 16;
  auto fn = wide ? fused_product_kernel<false, false, 4> : fused_product_kernel<false, false, 8>;
  const int threads = wide ? Layout<4>::kThreads : Layout<8>::kThreads;
  cudaError_t err = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (err != cudaSuccess) return err;
  // parameter copies are unused in batched mode; pass the first entry's maps by value is not
  // possible from the host (device memory), so hand over zeroed placeholders
  CUtensorMap z{};
  MkProduct zp{};
  zp.na = zp.nb = 1;
  MkGemmArgs largs = args;
  largs.nside = 0;
  fn<<<(unsigned)(tiles * nprod), threads, smem, stream>>>(z, z, z, largs, zp);
  err = cudaGetLastError();
  for (int t = 0; err == cudaSuccess && t < args.nside; ++t) err = launch_side_task(args.side[t], stream);
  return err;
}

}  // namespace mk
