// Element functions of the HBM-bound block transforms (breadth-first plan), shared by the
// stand-alone kernels (mk_blockops.cu) and the side-work warps of the persistent leaf kernel
// (mk_fused_gemm.cu), which run the next pass's operand transforms and the previous pass's
// post-additions while the DMMA warps compute the current pass's leaves. One call = one element
// group (W consecutive doubles) of one job; the same code in both places keeps the results
// bit-identical whichever kernel runs a transform.
#pragma once
#include <cstdint>
#include "mk_blockops.h"

namespace mk {

// W consecutive doubles: 8, 16 or 32-byte accesses.
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

// ---- one-level batched quadrant transform: dst_j = sum_i coef[j][i] * src_i ----------------
template <int W>
__device__ __forceinline__ void xform_elem(const MkXformJob& jb, uint32_t r, int64_t c) {
  const int ns = jb.nsrc, nd = jb.ndst;
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
      const int32_t cr = jb.clip_rows[j], cc = jb.clip_cols[j];
      if ((cr == 0 || (int64_t)r < cr) && (cc == 0 || c < cc)) st_vec<W>(jb.dst[j] + r * jb.ldd[j] + c, acc);
    }
  }
}

// ---- two-level operand transform (K2'') ------------------------------------------------------
// One job = one recursion node's operand block X (4 x 4 sub-blocks of rows x cols: sub-block
// (q1, q2) is sub-quadrant q2 of quadrant q1) -> all its grandchildren's operands
//     G(p, p2) = sum_q2 c[p2][q2] * ( sum_q1 c[p][q1] * X(q1, q2) )
// in one pass: the children's sums T(p, .) stay in registers, so two depths of the recursion
// cost one read of X and one write of the grandchildren instead of writing and re-reading the
// children. The coefficient tables are compile-time constants (every zero term is skipped at
// compile time, so the kernel stays memory-bound; the round-1 runtime-table version was
// instruction-bound); sums run in quadrant order from zero, exactly as two one-level passes
// would compute them (bit-identical results). Tables: reference kernels.py:66-160.
template <int TAB, int SIDE>
struct X2Tab;
// quadrant order 11, 12, 21, 22; [product][quadrant]
template <> struct X2Tab<0, 0> {  // Strassen, A side
  static constexpr int np = 7;
  __host__ __device__ static constexpr int cf(int p, int q) {
    constexpr int8_t c[8][4] = {{1, 0, 0, 1}, {0, 0, 1, 1}, {1, 0, 0, 0}, {0, 0, 0, 1},
                                     {1, 1, 0, 0}, {-1, 0, 1, 0}, {0, 1, 0, -1}, {0, 0, 0, 0}};
    return c[p][q];
  }
};
template <> struct X2Tab<0, 1> {  // Strassen, B side
  static constexpr int np = 7;
  __host__ __device__ static constexpr int cf(int p, int q) {
    constexpr int8_t c[8][4] = {{1, 0, 0, 1}, {1, 0, 0, 0}, {0, 1, 0, -1}, {-1, 0, 1, 0},
                                     {0, 0, 0, 1}, {1, 1, 0, 0}, {0, 0, 1, 1}, {0, 0, 0, 0}};
    return c[p][q];
  }
};
template <> struct X2Tab<1, 0> {  // Winograd block, A side
  static constexpr int np = 7;
  __host__ __device__ static constexpr int cf(int p, int q) {
    constexpr int8_t c[8][4] = {{1, 0, 0, 0}, {0, 1, 0, 0}, {1, 1, -1, -1}, {0, 0, 0, 1},
                                     {0, 0, 1, 1}, {-1, 0, 1, 1}, {1, 0, -1, 0}, {0, 0, 0, 0}};
    return c[p][q];
  }
};
template <> struct X2Tab<1, 1> {  // Winograd block, B side
  static constexpr int np = 7;
  __host__ __device__ static constexpr int cf(int p, int q) {
    constexpr int8_t c[8][4] = {{1, 0, 0, 0}, {0, 0, 1, 0}, {0, 0, 0, 1}, {1, -1, -1, 1},
                                     {-1, 1, 0, 0}, {1, -1, 0, 1}, {0, -1, 0, 1}, {0, 0, 0, 0}};
    return c[p][q];
  }
};
template <> struct X2Tab<2, 0> {  // Winograd Knuth, A side
  static constexpr int np = 7;
  __host__ __device__ static constexpr int cf(int p, int q) {
    constexpr int8_t c[8][4] = {{1, 0, 0, 0}, {0, 1, 0, 0}, {-1, 0, 1, 0}, {0, 0, 1, 1},
                                     {-1, 0, 1, 1}, {1, 1, -1, -1}, {0, 0, 0, 1}, {0, 0, 0, 0}};
    return c[p][q];
  }
};
template <> struct X2Tab<2, 1> {  // Winograd Knuth, B side
  static constexpr int np = 7;
  __host__ __device__ static constexpr int cf(int p, int q) {
    constexpr int8_t c[8][4] = {{1, 0, 0, 0}, {0, 0, 1, 0}, {0, 1, 0, -1}, {-1, 1, 0, 0},
                                     {1, -1, 0, 1}, {0, 0, 0, 1}, {-1, 1, 1, -1}, {0, 0, 0, 0}};
    return c[p][q];
  }
};
template <> struct X2Tab<3, 0> {  // Winograd Knuth, 8 calls (first product recomputed), A side
  static constexpr int np = 8;
  __host__ __device__ static constexpr int cf(int p, int q) {
    constexpr int8_t c[8][4] = {{1, 0, 0, 0}, {0, 1, 0, 0}, {-1, 0, 1, 0}, {0, 0, 1, 1},
                                     {-1, 0, 1, 1}, {1, 1, -1, -1}, {0, 0, 0, 1}, {1, 0, 0, 0}};
    return c[p][q];
  }
};
template <> struct X2Tab<3, 1> {  // Winograd Knuth, 8 calls, B side
  static constexpr int np = 8;
  __host__ __device__ static constexpr int cf(int p, int q) {
    constexpr int8_t c[8][4] = {{1, 0, 0, 0}, {0, 0, 1, 0}, {0, 1, 0, -1}, {-1, 1, 0, 0},
                                     {1, -1, 0, 1}, {0, 0, 0, 1}, {-1, 1, 1, -1}, {1, 0, 0, 0}};
    return c[p][q];
  }
};

// dst: the job's NP * NP destination pointers (shared memory in the stand-alone kernel, the job
// itself in global memory for side work); nullptr = not written.
template <int TAB, int SIDE, int W, typename DstPtrs>
__device__ __forceinline__ void xform2_elem(const double* src, int64_t lds, DstPtrs dst, int64_t ldd, int64_t rows,
                                            int64_t cols, uint32_t r, int64_t c) {
  using T = X2Tab<TAB, SIDE>;
  constexpr int NP = T::np;
  Vec<W> x[4][4];
#pragma unroll
  for (int q1 = 0; q1 < 4; ++q1)
#pragma unroll
    for (int q2 = 0; q2 < 4; ++q2) {
      const int64_t rr = ((q1 >> 1) * 2 + (q2 >> 1)) * rows + r;
      const int64_t cc = ((q1 & 1) * 2 + (q2 & 1)) * cols + c;
      x[q1][q2] = ld_vec<W>(src + rr * lds + cc);
    }
  const int64_t off = (int64_t)r * ldd + c;
#pragma unroll
  for (int p = 0; p < NP; ++p) {
    bool any = false;
#pragma unroll
    for (int p2 = 0; p2 < NP; ++p2) any = any || dst[p * NP + p2] != nullptr;
    if (!any) continue;  // job-uniform: this child is not in the pass, or all its grandchildren are views
    Vec<W> t[4];
#pragma unroll
    for (int q2 = 0; q2 < 4; ++q2) {
#pragma unroll
      for (int u = 0; u < W; ++u) t[q2].v[u] = 0.0;
#pragma unroll
      for (int q1 = 0; q1 < 4; ++q1) {
        const int cf = T::cf(p, q1);
        if (cf > 0) {
#pragma unroll
          for (int u = 0; u < W; ++u) t[q2].v[u] += x[q1][q2].v[u];
        } else if (cf < 0) {
#pragma unroll
          for (int u = 0; u < W; ++u) t[q2].v[u] -= x[q1][q2].v[u];
        }
      }
    }
#pragma unroll
    for (int p2 = 0; p2 < NP; ++p2) {
      double* d = dst[p * NP + p2];
      if (!d) continue;
      Vec<W> o;
#pragma unroll
      for (int u = 0; u < W; ++u) o.v[u] = 0.0;
#pragma unroll
      for (int q2 = 0; q2 < 4; ++q2) {
        const int cf = T::cf(p2, q2);
        if (cf > 0) {
#pragma unroll
          for (int u = 0; u < W; ++u) o.v[u] += t[q2].v[u];
        } else if (cf < 0) {
#pragma unroll
          for (int u = 0; u < W; ++u) o.v[u] -= t[q2].v[u];
        }
      }
      st_vec<W>(d + off, o);
    }
  }
}

// ---- two-level post-addition -----------------------------------------------------------------
// One job = one recursion node at depth d - 2: its grandchildren's outputs G(p, p2) (depth d,
// rows x cols each) -> the node's output block, 4 x 4 sub-blocks:
//     out(q1, q2) = sum_p c[q1][p] * ( sum_p2 c[q2][p2] * G(p, p2) )
// the children's outputs never touch memory. Sums run from zero in product order, exactly as
// two one-level passes (bit-identical). C tables: reference kernels.py:66-160 post-additions.
template <int TAB>
struct XCTab;
template <> struct XCTab<0> {  // Strassen
  static constexpr int np = 7;
  __host__ __device__ static constexpr int cf(int q, int p) {
    constexpr int8_t c[4][8] = {{1, 0, 0, 1, -1, 0, 1, 0}, {0, 0, 1, 0, 1, 0, 0, 0},
                                {0, 1, 0, 1, 0, 0, 0, 0}, {1, -1, 1, 0, 0, 1, 0, 0}};
    return c[q][p];
  }
};
template <> struct XCTab<1> {  // Winograd block
  static constexpr int np = 7;
  __host__ __device__ static constexpr int cf(int q, int p) {
    constexpr int8_t c[4][8] = {{1, 1, 0, 0, 0, 0, 0, 0}, {1, 0, 1, 0, 1, 1, 0, 0},
                                {1, 0, 0, -1, 0, 1, 1, 0}, {1, 0, 0, 0, 1, 1, 1, 0}};
    return c[q][p];
  }
};
template <> struct XCTab<2> {  // Winograd Knuth
  static constexpr int np = 7;
  __host__ __device__ static constexpr int cf(int q, int p) {
    constexpr int8_t c[4][8] = {{1, 1, 0, 0, 0, 0, 0, 0}, {1, 0, 0, 1, 1, 1, 0, 0},
                                {1, 0, 1, 0, 1, 0, 1, 0}, {1, 0, 1, 1, 1, 0, 0, 0}};
    return c[q][p];
  }
};
template <> struct XCTab<3> {  // Winograd Knuth, 8 calls
  static constexpr int np = 8;
  __host__ __device__ static constexpr int cf(int q, int p) {
    constexpr int8_t c[4][8] = {{0, 1, 0, 0, 0, 0, 0, 1}, {1, 0, 0, 1, 1, 1, 0, 0},
                                {1, 0, 1, 0, 1, 0, 1, 0}, {1, 0, 1, 1, 1, 0, 0, 0}};
    return c[q][p];
  }
};

template <int TAB, int W, typename SrcPtrs>
__device__ __forceinline__ void xpost2_elem(SrcPtrs src, int64_t lds, double* dst, int64_t ldd, uint32_t acc_mask,
                                            int64_t rows, int64_t cols, uint32_t r, int64_t c) {
  using T = XCTab<TAB>;
  constexpr int NP = T::np;
  const int64_t soff = (int64_t)r * lds + c;
  Vec<W> out[16];
#pragma unroll
  for (int o = 0; o < 16; ++o)
#pragma unroll
    for (int u = 0; u < W; ++u) out[o].v[u] = 0.0;
#pragma unroll
  for (int p = 0; p < NP; ++p) {
    if (!src[p * NP]) continue;  // job-uniform: product outside this pass
    Vec<W> t[4];
#pragma unroll
    for (int q2 = 0; q2 < 4; ++q2)
#pragma unroll
      for (int u = 0; u < W; ++u) t[q2].v[u] = 0.0;
#pragma unroll
    for (int p2 = 0; p2 < NP; ++p2) {
      const Vec<W> g = ld_vec<W>(src[p * NP + p2] + soff);
#pragma unroll
      for (int q2 = 0; q2 < 4; ++q2) {
        const int cf = T::cf(q2, p2);
        if (cf > 0) {
#pragma unroll
          for (int u = 0; u < W; ++u) t[q2].v[u] += g.v[u];
        } else if (cf < 0) {
#pragma unroll
          for (int u = 0; u < W; ++u) t[q2].v[u] -= g.v[u];
        }
      }
    }
#pragma unroll
    for (int q1 = 0; q1 < 4; ++q1) {
      const int cf = T::cf(q1, p);
#pragma unroll
      for (int q2 = 0; q2 < 4; ++q2) {
        if (cf > 0) {
#pragma unroll
          for (int u = 0; u < W; ++u) out[q1 * 4 + q2].v[u] += t[q2].v[u];
        } else if (cf < 0) {
#pragma unroll
          for (int u = 0; u < W; ++u) out[q1 * 4 + q2].v[u] -= t[q2].v[u];
        }
      }
    }
  }
#pragma unroll
  for (int q1 = 0; q1 < 4; ++q1)
#pragma unroll
    for (int q2 = 0; q2 < 4; ++q2) {
      const int64_t rr = ((q1 >> 1) * 2 + (q2 >> 1)) * rows + r;
      const int64_t cc = ((q1 & 1) * 2 + (q2 & 1)) * cols + c;
      if (acc_mask & (1u << (q1 * 4 + q2))) {
        const Vec<W> old = ld_vec<W>(dst + rr * ldd + cc);
#pragma unroll
        for (int u = 0; u < W; ++u) out[q1 * 4 + q2].v[u] += old.v[u];
      }
      st_vec<W>(dst + rr * ldd + cc, out[q1 * 4 + q2]);
    }
}

// ---- one-level operand transform (side work of the pipelined plan) -----------------------------
// One job = one node: its operand block (2 x 2 quadrants of rows x cols at src, leading dimension
// lds) -> the children's operands G(p) = sum_q c[p][q] X(q) for every p with dst[p] set (others:
// views or not in the pass), summed from zero in quadrant order as the generic transform job does
// (bit-identical). Reuses MkXform2Job (dst[0 .. np-1]).
template <int TAB, int SIDE, int W, typename DstPtrs>
__device__ __forceinline__ void xform1_elem(const double* src, int64_t lds, DstPtrs dst, int64_t ldd, int64_t rows,
                                            int64_t cols, uint32_t r, int64_t c) {
  using T = X2Tab<TAB, SIDE>;
  constexpr int NP = T::np;
  Vec<W> x[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) x[q] = ld_vec<W>(src + ((q >> 1) * rows + r) * lds + (q & 1) * cols + c);
  const int64_t off = (int64_t)r * ldd + c;
#pragma unroll
  for (int p = 0; p < NP; ++p) {
    double* d = dst[p];
    if (!d) continue;
    Vec<W> o;
#pragma unroll
    for (int u = 0; u < W; ++u) o.v[u] = 0.0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int cf = T::cf(p, q);
      if (cf > 0) {
#pragma unroll
        for (int u = 0; u < W; ++u) o.v[u] += x[q].v[u];
      } else if (cf < 0) {
#pragma unroll
        for (int u = 0; u < W; ++u) o.v[u] -= x[q].v[u];
      }
    }
    st_vec<W>(d + off, o);
  }
}

// ---- one-level post-addition (side work of the pipelined plan) -------------------------------
// One job = one node: its children's outputs (src[p], common leading dimension lds, rows x cols)
// -> the node's four quadrants (dst, 2 x 2 blocks of rows x cols, leading dimension ldd):
//     out(q) = sum_p c[q][p] * G(p)   (+ the quadrant's previous contents when bit q of acc_mask)
// summed from zero in product order, as the generic transform job does (bit-identical). Reuses
// MkXpost2Job (src[0 .. np-1]).
template <int TAB, int W, typename SrcPtrs>
__device__ __forceinline__ void xpost1_elem(SrcPtrs src, int64_t lds, double* dst, int64_t ldd, uint32_t acc_mask,
                                            int64_t rows, int64_t cols, uint32_t r, int64_t c) {
  using T = XCTab<TAB>;
  constexpr int NP = T::np;
  const int64_t soff = (int64_t)r * lds + c;
  Vec<W> g[NP];
#pragma unroll
  for (int p = 0; p < NP; ++p) g[p] = ld_vec<W>(src[p] + soff);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    Vec<W> o;
#pragma unroll
    for (int u = 0; u < W; ++u) o.v[u] = 0.0;
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      const int cf = T::cf(q, p);
      if (cf > 0) {
#pragma unroll
        for (int u = 0; u < W; ++u) o.v[u] += g[p].v[u];
      } else if (cf < 0) {
#pragma unroll
        for (int u = 0; u < W; ++u) o.v[u] -= g[p].v[u];
      }
    }
    double* d = dst + ((q >> 1) * rows + r) * ldd + (q & 1) * cols + c;
    if (acc_mask & (1u << q)) {
      const Vec<W> old = ld_vec<W>(d);
#pragma unroll
      for (int u = 0; u < W; ++u) o.v[u] += old.v[u];
    }
    st_vec<W>(d, o);
  }
}

}  // namespace mk
