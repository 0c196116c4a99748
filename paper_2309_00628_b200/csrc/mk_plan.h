// Plan structures shared by the host planner and the sm_100a kernels.
//
// A "product" is one leaf multiplication of the Strassen/Winograd recursion:
//     P = (sum_i sa_i * A[rows ra_i.., cols ca_i..]) x (sum_j sb_j * B[rb_j.., cb_j..])
// with P accumulated as  C[rd_k.., cd_k..] (+)= sd_k * P  for every destination k.
// The pre-additions (reference: kernels.py:66-160 block sums, e.g. S4 = A12 - S2)
// are formed in registers from TMA-staged tiles; the post-additions (reference
// kernels.py:112-118, U2..U7) are the multi-destination epilogue.
#pragma once
#include <cstdint>

#define MK_MAX_TERMS 4   // operand terms per side fused into one product
#define MK_MAX_DESTS 16  // C destinations one product's epilogue writes
#define MK_BM 128
#define MK_BN 128
#define MK_BK 16
// CTA = warpgroup 0 (TMA producer / pre-add combiner) + 2 or 4 DMMA consumer warpgroups
#define MK_TILE_BYTES (MK_BM * MK_BK * 8)  // 16 KiB: one operand term tile per stage
#ifndef MK_SMEM_BUDGET
#define MK_SMEM_BUDGET (224 * 1024)
#endif
#define MK_MIN_LEAF 32    // smallest leaf order the level policy recurses to
#define MK_MAX_LEVELS 5   // deepest recursion the level policy plans (7^5 leaves)
#define MK_MAX_SLABS 8    // output row slabs (ranks) of the fused multi-GPU reduce-scatter

struct MkTerm {
  int32_t row, col;  // offset of the term block inside the operand base matrix
  double sign;       // +1 / -1
};

struct MkDest {
  int64_t row, col;  // offset of the destination block inside C
  double sign;       // +1 / -1
  int32_t accumulate;  // 0: first writer (store), 1: read-modify-write
  int32_t pad_;
};

struct MkProduct {
  int32_t na, nb, nd, pad_;
  MkTerm a[MK_MAX_TERMS];
  MkTerm b[MK_MAX_TERMS];
  MkDest d[MK_MAX_DESTS];
};


struct MkBatchEntry;

// HBM-bound side work for the persistent leaf kernel: its producer warpgroup has one TMA thread,
// so warps 1-3 (96 threads per CTA) stream block transforms that are independent of the launch's
// leaves -- the next breadth-first pass's operand sums and the previous pass's post-additions --
// while the DMMA warps run (the FP64 tensor pipe leaves HBM ~80% idle). Same element code as the
// stand-alone kernels (mk_xform.cuh): results are bit-identical whichever kernel runs a task.
#define MK_SIDE_MAX 8
struct MkSideTask {
  const void* jobs;  // device array of njobs jobs: MkXformJob / MkXform2Job / MkXpost2Job
  int64_t rows, cols;
  int32_t njobs;
  int8_t kind;       // 1 one-level transform, 2 two-level operand transform, 3 two-level post-addition,
                     // 4 one-level post-addition, 5 one-level operand transform (compiled tables)
  int8_t table;      // kinds 2, 3: 0 Strassen, 1 Winograd block, 2 Winograd Knuth, 3 Knuth 8-call
  int8_t side;       // kind 2: 0 A, 1 B
  int8_t width;      // doubles per access: 1, 2 (or 4 for kind 1)
  int64_t bytes;     // HBM bytes the task moves (host-side estimate for balancing; unused on the device)
};

struct MkGemmArgs {
  double* C;
  int64_t ldc;
  int32_t M, N, K;       // leaf product extents (K % 16 == 0 unless single full-matrix terms)
  int32_t tiles_m, tiles_n;
  int32_t stages;        // operand ring depth (set by the launcher)
  int32_t raw_sets;      // raw term sets in flight for the combiner (set by the launcher)
  int32_t group_m;       // rasterisation group height (tiles)
  int32_t vec_ok;        // 32B-vector epilogue allowed
  int32_t async_epi;     // TMA store / reduce-add epilogue (tile-aligned leaf, tmC valid)
  int32_t chunk_stages;               // >0: two-level accumulation, flush registers to TMEM every N stages
  int32_t tiles_per_prod;             // batched launch: CTAs per product
  int32_t nprod;                      // batched launch: products in the batch (persistent kernel)
  const MkBatchEntry* batch;          // batched launch: per-product maps/descriptors (nullptr: single)
  // Row-slab output (fused multi-GPU reduce-scatter, mk_strassen_partial_slabs): nslab > 0 routes
  // C row R (relative to C's base) to slab[R / slab_rows] + (R % slab_rows) * ldc -- each slab
  // owned by one rank, peers' slabs mapped over NVLink -- with the synchronous REDG.ADD epilogue.
  int32_t nslab, pad_slab;
  int64_t slab_rows;
  double* slab[MK_MAX_SLABS];
  // Stream-K tail (persistent kernel): tiles [0, sk_tile0) run whole, one CTA each (data-parallel
  // waves); the k-iterations of tiles [sk_tile0, total) are split evenly over the grid. A tile's
  // head segment (k from 0) owns it: the CTAs holding its later k-segments write their partial
  // accumulators to sk_partial (one slot per CTA) and count up sk_flags[tile][warp]; the owner
  // adds them in k order (deterministic) and runs the epilogue. sk_tile0 >= total: no stream-K.
  int32_t sk_tile0, pad_sk;
  double* sk_partial;
  int32_t* sk_flags;
  // side work (persistent kernel, data-parallel launches): tasks run in order by every CTA's
  // warps 1-3; the tasks of one launch must be independent of each other and of its leaves
  int32_t nside, pad_side;
  MkSideTask side[MK_SIDE_MAX];
};
