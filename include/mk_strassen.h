/*
 * mk_strassen.h -- C ABI of the B200-native Strassen / Strassen-Winograd engine
 * (libmk_strassen.so). Plain pointers, sizes and a cudaStream_t passed as void*;
 * every matrix is row-major FP64 in device memory with an explicit leading
 * dimension (elements). No torch or numpy types cross this boundary.
 *
 * The reference (`matmulkit`, /root/reference/pkg/src/matmulkit) is pure Python
 * with no FFI; each entry point below replaces the reference function cited next
 * to it, and the Python package paper_2309_00628_b200 binds them with ctypes
 * (see INTEGRATION.md for the binding a matmulkit maintainer would add).
 *
 * Status codes (mirroring the reference's exception types):
 *   MK_OK 0, MK_ERR_DIMENSION 1 (DimensionError, core.py:18), MK_ERR_ALIAS 2
 *   (AliasError, core.py:22), MK_ERR_CUDA 3, MK_ERR_WORKSPACE 4, MK_ERR_ARG 5
 *   (ValueError), MK_ERR_INEXACT 6 (integer operands not exactly representable).
 * mk_last_error() returns a thread-local message for the last non-zero status.
 */
#ifndef MK_STRASSEN_H
#define MK_STRASSEN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

enum mk_status {
  MK_OK = 0,
  MK_ERR_DIMENSION = 1,
  MK_ERR_ALIAS = 2,
  MK_ERR_CUDA = 3,
  MK_ERR_WORKSPACE = 4,
  MK_ERR_ARG = 5,
  MK_ERR_INEXACT = 6
};

/* Algorithm ids: the reference's kernel names (hybrid.py:28, kernels.py:188-193). */
enum mk_algo {
  MK_ALGO_NAIVE = 0,                /* naive_mul            kernels.py:350 */
  MK_ALGO_STRASSEN = 1,             /* strassen_mul         kernels.py:370 */
  MK_ALGO_WINOGRAD_BLOCK = 2,       /* winograd_block_mul   kernels.py:378 */
  MK_ALGO_WINOGRAD_KNUTH = 3,       /* winograd_knuth_mul   kernels.py:386 */
  MK_ALGO_WINOGRAD_KNUTH_8CALL = 4, /* ..., recompute_first_product=True  kernels.py:396 */
  MK_ALGO_TWO_TEMP = 5,             /* two_temp_winograd    schedules.py:332 */
  MK_ALGO_IN_PLACE = 6              /* in_place_winograd    schedules.py:344 */
};

/* Engine version: (major << 16) | minor. */
int mk_version(void);

/* Engine options (process-wide).
 * MK_OPT_FUSE_PREADDS: 1 = form the last level's operand sums inside the DMMA kernel (K2
 *   combiner), 0 = materialise them with HBM-bound block kernels first (default; measured
 *   faster on B200).
 * MK_OPT_PLAN (strassen / winograd kinds, L >= 2): 0 = breadth-first (default: batched leaves,
 *   fastest, largest workspace), 1 = depth-first (workspace-minimal: operand sums only, P_i
 *   accumulated straight into C by the epilogue), 2 = hybrid (top level depth-first, each
 *   top-level product breadth-first below it: about 1/7 of the breadth-first workspace).
 * MK_OPT_LITERAL_TAIL (two-temp): 0 = the literal Table-2 schedule down to the leaves (default:
 *   two (n/2^(l+1))^2 scratch blocks per level, the paper's memory bound), 1 = the last two levels
 *   breadth-first under the literal levels (faster at >= 3 levels, more scratch).
 * MK_OPT_LEAF_SLICES: 0 = leaf products on the FP64 tensor cores (DMMA, default); 4..8 = on the
 *   INT8 tensor cores (tcgen05 kind::i8, Ozaki scheme I) with that many digit slices per operand
 *   (see mk_ozaki_dgemm; 8 is more accurate than the DMMA leaf, fewer trade accuracy for speed).
 *   Applies to every leaf product of the engine with m*n*k >= 2^MK_OPT_LEAF_MIN_LOG2.
 * MK_OPT_LEAF_MIN_LOG2: the INT8 leaf's size threshold, log2 of m*n*k (default 29, about 812^3):
 *   smaller leaves stay on DMMA (the per-leaf INT8 kernels are launch- and wave-bound there).
 * MK_OPT_BFS_GROUP (breadth-first plan, L >= 2): top-level products per pass. 0 = auto (4: two
 *   passes over the 7 products, each keeping only its own operand sums and outputs -- about half
 *   the single-pass workspace; one pass for products of at most 4096 in every extent); 7 or 8 = one pass (largest workspace); 1 = one top-level subtree
 *   at a time (smallest). Results differ only in the order C's partial sums are added.
 * MK_OPT_LITERAL_STREAMS (two-temp / in-place): 1 = block additions the next product does not
 *   depend on are issued on internal side streams, ordered by block-level hazard tracking, and
 *   run beside the leaf products (default); 0 = every step on the caller's stream. Same steps,
 *   same operands, bit-identical results either way; the side streams are joined into `stream`
 *   before the call returns.
 * MK_OPT_HOST_GROUP (mk_strassen_host, 2 levels, DMMA leaves): the top-level products between the
 *   first few and the last run as one grouped breadth-first pass once every upload has landed
 *   (instead of child by child behind the sub-block uploads). -1 = auto (the pass starts after as
 *   many products as outlast the uploads: 3 at n = 16384, none at n <= 8192), 0 = off, k in 1..6 =
 *   start after k products. Results differ only in the order C's partial sums are added.
 * MK_OPT_PDL: 1 = sub-wave leaf launches and small block additions (the one-at-a-time launch
 *   chains of the two-temp / in-place schedules) are launched as programmatic dependents
 *   (cudaLaunchAttributeProgrammaticStreamSerialization): the next kernel of a stream is resident
 *   and past its shared-memory prologue when the previous one ends, and touches global memory only
 *   after griddepcontrol.wait (default); 0 = plain stream-ordered launches. Same kernels, same
 *   order, bit-identical results.
 * MK_OPT_PIPELINE (breadth-first plan, L >= 2, narrow-tile leaves): the pipelined plan -- one pass
 *   per top-level product, each pass's transforms carried as side work by its neighbours' leaf
 *   launches. 1 = when the leaves are long enough to hide transforms under (leaf volume >= 2^24
 *   and 7^L leaves >= 2^36; default: smaller calls are launch-bound and take the grouped plan),
 *   0 = never, 2 = for every call with narrow-tile leaves. Integer results are identical; real
 *   results differ only in the order C's partial sums are added. */
enum mk_option { MK_OPT_FUSE_PREADDS = 1, MK_OPT_PLAN = 2, MK_OPT_LITERAL_TAIL = 3, MK_OPT_LEAF_SLICES = 4,
                 MK_OPT_LEAF_MIN_LOG2 = 5, MK_OPT_BFS_GROUP = 6, MK_OPT_LITERAL_STREAMS = 7, MK_OPT_HOST_GROUP = 8,
                 MK_OPT_PDL = 9, MK_OPT_PIPELINE = 10 };
int mk_set_option(int key, int value);
int mk_get_option(int key, int* value);
/* Calling-thread override of MK_OPT_PLAN / MK_OPT_LITERAL_TAIL (value -1 removes it). Applies to
 * every later sizing (mk_*_workspace_bytes) and launch made from this thread, so a workspace sized
 * under an override always fits the launch that follows, whatever other threads set meanwhile.
 * mk_get_option reports the effective value for the calling thread. */
int mk_set_thread_option(int key, int value);

/* Instrumentation (bench.py). mk_launch_count: kernels this thread has launched so far.
 * mk_timing_begin / mk_timing_end: bracket engine calls; every leaf-product (DMMA) launch in
 * between is timed with CUDA events on its own stream; _end synchronises and returns the
 * summed kernel time, the number of product launches and their algorithmic flops (2mnk).
 * mk_fp64_peak: DMMA-only microbenchmark on all SMs (the FP64 tensor roofline), TFLOP/s. */
long long mk_launch_count(void);
int mk_timing_begin(void);
int mk_timing_end(double* kernel_ms, int* launches, double* flops);
int mk_fp64_peak(double* tflops, void* stream);

/* Thread-local description of the last failing call ("" if none). */
const char* mk_last_error(void);

/* C[m x n] = A[m x k] * B[k x n] on the fused DMMA kernel (single-term products).
 * Replaces naive_mul kernels.py:350-367 / _naive_arrays kernels.py:258-266
 * (np.matmul -> OpenBLAS dgemm). lda/ldb must be even and A/B 16-byte aligned
 * (TMA); C may have any ld. C must not overlap A or B (MK_ERR_ALIAS). */
int mk_dgemm(const double* A, int64_t lda, const double* B, int64_t ldb, double* C, int64_t ldc,
             int64_t m, int64_t n, int64_t k, void* stream);

/* C[m x n] = A[m x k] * B[k x n] with FP64 operands multiplied on the INT8 tensor cores
 * (Ozaki scheme I: each row of A / column of B scaled by a power of two and split into `slices`
 * digit planes -- a signed 7-bit leading digit and unsigned 8-bit digits, 7 + 8 (slices - 1) bits,
 * the floor digits of the value; the slices*(slices+1)/2 digit-pair products accumulated exactly in
 * int32 TMEM accumulators by tcgen05.mma kind::i8 (pairs on one anti-diagonal share one), the
 * diagonal sums recombined exactly in int64 and rounded once to FP64). Same operand/alias rules
 * as mk_dgemm; the opt-in alternative to the DMMA leaf (mk_set_option(MK_OPT_LEAF_SLICES, s)).
 * slices in [4, 8]; any k (k > 4402 at 8 slices runs in K chunks that accumulate). ws:
 * mk_ozaki_workspace_bytes(m, n, k, slices) bytes of device memory, 256-byte aligned.
 * Integer-valued data that fits the digits (|x| < 2^56 at 8 slices) is reproduced exactly; at 8
 * slices real data is more accurate than the FP64 tensor-core product (K5).
 * A non-finite entry makes its whole row (of A) / column (of B) of C NaN.
 * Replaces the same call sites as mk_dgemm (kernels.py:258-266). */
size_t mk_ozaki_workspace_bytes(int64_t m, int64_t n, int64_t k, int slices);
int mk_ozaki_dgemm(const double* A, int64_t lda, const double* B, int64_t ldb, double* C, int64_t ldc,
                   int64_t m, int64_t n, int64_t k, int slices, void* ws, size_t ws_bytes, void* stream);

/* Levels the engine runs for an order-n problem under the reference's base policy
 * (BasePolicy kernels.py:26-57): kind 0 = "scalar", 1 = "unrolled" (param = order),
 * 2 = "naive-cutoff" (param = threshold). naive-cutoff is honoured exactly
 * (leaf when n <= threshold, kernels.py:276) down to the engine's limits: leaf order >= 32
 * and at most 5 levels (7^5 leaves); deeper recursion (scalar / unrolled policies, tiny
 * thresholds) is clamped -- results identical for integer data, within tolerance otherwise. */
int mk_levels_for_policy(int64_t n, int kind, int64_t param, int algo, int* levels_out);

/* Device workspace bytes mk_strassen needs for (algo, n, levels). 0 for the fully
 * fused single-level plan and for the in-place schedule. */
size_t mk_workspace_bytes(int algo, int64_t n, int levels);

/* Square power-of-two product C = A * B (order n) with `levels` recursion levels.
 * Replaces _run_dc kernels.py:335-347 (strassen / winograd-block / knuth) and
 * _run_schedule schedules.py:300-329 (two-temp / in-place). A and B are read-only
 * except for MK_ALGO_IN_PLACE, which, like schedules.py:344-353, stores intermediates
 * in quadrants of A, B and C and leaves A/B unspecified. ws/ws_bytes: caller-owned
 * device workspace of at least mk_workspace_bytes(). Asynchronous on `stream`. */
int mk_strassen(int algo, double* A, int64_t lda, double* B, int64_t ldb, double* C, int64_t ldc,
                int64_t n, int levels, void* ws, size_t ws_bytes, void* stream);

/* Rectangular driver (hybrid.py:105-146 multiply): C[m x n] = A[m x k] * B[k x n]
 * with `levels` Strassen-Winograd levels on zero-padded operands whose extents are
 * rounded up to multiples of 2^(levels+1) (m, k) and 2^(levels+2) (n) -- not the
 * reference's square 2^j order.
 * Padding is staged in ws (size from mk_rect_workspace_bytes). */
size_t mk_rect_workspace_bytes(int algo, int64_t m, int64_t n, int64_t k, int levels);
int mk_multiply_rect(int algo, const double* A, int64_t lda, const double* B, int64_t ldb, double* C,
                     int64_t ldc, int64_t m, int64_t n, int64_t k, int levels, void* ws, size_t ws_bytes,
                     void* stream);

/* Synchronous block copies of 8-byte elements (rows x cols, leading dimensions in elements)
 * between host and device, ordered after prior work on `stream`. Pageable host memory is
 * staged through pinned bounce slots with parallel host copies on two streams (several times
 * the driver's pageable path); pinned memory is copied directly. */
int mk_copy_to_device(double* dst, int64_t ldd, const double* src, int64_t lds, int64_t rows, int64_t cols,
                      void* stream);
int mk_copy_to_host(double* dst, int64_t ldd, const double* src, int64_t lds, int64_t rows, int64_t cols,
                    void* stream);

/* Workspace bytes mk_strassen_host needs for (algo, n, levels) (0 on invalid input): the
 * depth-first plan's for L <= 2, a breadth-first plan per top-level product for L >= 3. */
size_t mk_host_workspace_bytes(int algo, int64_t n, int levels);

/* End-to-end product for HOST operands with transfers overlapped with compute (fused
 * algorithms, levels >= 1). hA/hB/hC: host matrices (pinned for asynchronous DMA); dA/dB/dC:
 * caller-owned device buffers of order n with even leading dimension ldd. Operands are
 * uploaded on `copy_stream` (quadrants for L = 1; for L = 2, quarter-quadrant sub-blocks in the
 * order the compute first needs them, each top-level product running child by child and
 * waiting only for the sub-blocks it reads), the top-level products run on `stream` in the
 * order mk_overlap_order reports, and every C quadrant is downloaded as soon as its last
 * contributor finishes (the last one by sub-blocks). Synchronous: returns when hC holds the
 * result. Workspace from mk_host_workspace_bytes. */
int mk_strassen_host(int algo, const double* hA, int64_t lda, const double* hB, int64_t ldb, double* hC, int64_t ldc,
                     int64_t n, int levels, double* dA, double* dB, double* dC, int64_t ldd, void* ws,
                     size_t ws_bytes, void* stream, void* copy_stream);
/* Top-level product order (order_out[nprod]) and quadrant upload order (uploads_out[8]: A11..A22
 * = 0..3, B11..B22 = 4..7) of the overlapped host path; returns nprod. */
int mk_overlap_order(int algo, int* order_out, int* uploads_out);

/* dst = sum_i sign[i] * src_i over a rows x cols block (nsrc <= 8); dst may alias a
 * source exactly. Replaces block_add core.py:153-169 (np.add / np.subtract). */
int mk_block_combine(double* dst, int64_t ldd, const double* const* src, const int64_t* lds,
                     const double* sign, int nsrc, int64_t rows, int64_t cols, void* stream);

/* Integer operand support (reference tests run int64, conftest.py:29-30). */
int mk_i64_to_f64(const int64_t* src, int64_t lds, double* dst, int64_t ldd, int64_t rows, int64_t cols,
                  void* stream);
int mk_f64_to_i64(const double* src, int64_t lds, int64_t* dst, int64_t ldd, int64_t rows, int64_t cols,
                  void* stream);
/* max |x| of a block, synchronous (returns through *out). */
int mk_absmax_f64(const double* src, int64_t lds, int64_t rows, int64_t cols, double* out, void* stream);
int mk_absmax_i64(const int64_t* src, int64_t lds, int64_t rows, int64_t cols, double* out, void* stream);

/* Multi-GPU sharding. mk_product_count: leaf products of (algo, levels). A partial product
 * computes shard units [first, first+count), where unit u is row panel (u mod panels) of leaf
 * (u div panels) -- leaves split into `panels` equal row panels so ranks get equal work -- and
 * accumulates them into C (zero-initialised by the caller); the caller sum-reduces the partials
 * (NCCL). Workspace from mk_partial_workspace_bytes. */
int mk_product_count(int algo, int levels);
size_t mk_partial_workspace_bytes(int algo, int64_t n, int levels);
int mk_strassen_partial(int algo, const double* A, int64_t lda, const double* B, int64_t ldb, double* C,
                        int64_t ldc, int64_t n, int levels, int first, int count, int panels, void* ws,
                        size_t ws_bytes, void* stream);

/* Sharded form of mk_multiply_rect (BASELINE cfg5 on N GPUs): this rank's leaf row-panel units
 * [first, first+count) of the padded rectangular product (panels per leaf; mk_product_count(algo,
 * levels) * panels units in all), written to C (m x n) as a partial -- C is overwritten with this
 * rank's contribution; the ranks' partials sum to A*B (e.g. one NCCL reduce). Replaces
 * hybrid.multiply (hybrid.py:105-146) with its products sharded. */
size_t mk_rect_partial_workspace_bytes(int algo, int64_t m, int64_t n, int64_t k, int levels, int panels);
int mk_multiply_rect_partial(int algo, const double* A, int64_t lda, const double* B, int64_t ldb, double* C,
                             int64_t ldc, int64_t m, int64_t n, int64_t k, int levels, int first, int count,
                             int panels, void* ws, size_t ws_bytes, void* stream);

/* Multi-GPU product in ONE process (the single-process counterpart of the torch.distributed
 * path; SURVEY.md 8(b) "mk_multi_gpu_winograd"): C = A B, algo as mk_strassen (fused kinds),
 * square order n = 2^j, `levels` >= 1. A, B and C are device memory of devices[0]. The 7^L leaf
 * products, split into 8 row panels each, are dealt out to the ngpu devices in contiguous
 * level-major ranges (balanced to one panel); rank r >= 1 receives by peer copies (NVLink) only
 * the top-level operand quadrants its panels read, accumulates its partial C locally, and
 * device 0 adds the partials into C in rank order, reading them over peer memory. ws[r] /
 * ws_bytes[r]: workspace on devices[r] of mk_multi_gpu_workspace_bytes(algo, n, levels, r, ngpu)
 * bytes; streams[r]: a stream of devices[r]. Work is enqueued asynchronously (ordered by events);
 * synchronise streams[0] before reading C. A device may appear more than once (ranks sharing a
 * GPU: the same code path on one device). Peer access between devices[0] and the others is
 * enabled on the way. */
size_t mk_multi_gpu_workspace_bytes(int algo, int64_t n, int levels, int rank, int ngpu);
int mk_multi_gpu_winograd(int algo, int ngpu, const int* devices, const double* A, int64_t lda, const double* B,
                          int64_t ldb, double* C, int64_t ldc, int64_t n, int levels, void* const* ws,
                          const size_t* ws_bytes, void* const* streams);

/* Enable NVLink peer access from the current device to peer_device (idempotent). */
int mk_enable_peer_access(int peer_device);

/* Fused multi-GPU reduce-scatter form of mk_strassen_partial: the
 * leaf epilogue adds this rank's contributions straight into the C row slab of the rank that owns
 * each row -- slabs[r] is rank r's (slab_rows x n, leading dimension ldc) buffer, its own one local
 * and the others peer (IPC-mapped, NVLink) addresses -- with REDG.ADD.F64, so the partial-C buffer
 * and the separate reduce collective disappear. Every slab must be zeroed before any rank starts
 * (barrier), and read after every rank has finished (device sync + barrier). nslabs * slab_rows
 * == n; levels <= 2 (every leaf contribution then lands in the epilogue); the leaves run on the
 * DMMA kernel or, with MK_OPT_LEAF_SLICES set, the INT8 (Ozaki) kernel, whose write-back then uses
 * atomic adds. FP64 summation order at a row follows arrival order (integer data stays exact). */
int mk_strassen_partial_slabs(int algo, const double* A, int64_t lda, const double* B, int64_t ldb,
                              double* const* slabs, int nslabs, int64_t slab_rows, int64_t ldc, int64_t n,
                              int levels, int first, int count, int panels, void* ws, size_t ws_bytes,
                              void* stream);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif

#ifdef __cplusplus
}
#endif
#endif /* MK_STRASSEN_H */
