// Probe: does TMA tensor reduce-add (cp.reduce.async.bulk.tensor ... .add) work for FP64 tensor
// maps with 128B swizzle on sm_100a? Also the non-tensor bulk reduce (.add.f64).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tma_reduce_probe tma_reduce_probe.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

typedef CUresult (*PFN_encode)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                               const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                               CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__global__ void k_tensor(const __grid_constant__ CUtensorMap tm, int mode) {
  extern __shared__ __align__(1024) unsigned char smem[];
  double* s = reinterpret_cast<double*>(smem);
  // box {16 cols, 64 rows} swizzled 128B: logical (r, c) at row r, chunk (c/2) ^ (r & 7)
  for (int idx = threadIdx.x; idx < 64 * 16; idx += blockDim.x) {
    int r = idx / 16, c = idx % 16;
    int chunk = (c / 2) ^ (r & 7);
    s[r * 16 + chunk * 2 + (c & 1)] = (double)(r * 100 + c);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
    if (mode == 0)
      asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%1, %2}], [%3];"
                   ::"l"(&tm), "r"(16), "r"(64), "r"(sa) : "memory");
    else
      asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];"
                   ::"l"(&tm), "r"(16), "r"(64), "r"(sa) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

__global__ void k_flat(double* g) {
  __shared__ __align__(128) double s[32];
  if (threadIdx.x < 32) s[threadIdx.x] = 1.5 * threadIdx.x;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t sa = (uint32_t)__cvta_generic_to_shared(s);
    asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f64 [%0], [%1], 256;" ::"l"(g), "r"(sa)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

int main() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  PFN_encode enc = (PFN_encode)p;
  const int R = 256, C = 64;
  std::vector<double> h(R * C, 1.0);
  double* d;
  cudaMalloc(&d, R * C * 8);
  cudaMemcpy(d, h.data(), R * C * 8, cudaMemcpyHostToDevice);
  CUtensorMap tm;
  cuuint64_t dims[2] = {C, R}, str[1] = {C * 8};
  cuuint32_t box[2] = {16, 64}, es[2] = {1, 1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode=%d\n", (int)r);
  for (int mode = 0; mode < 2; ++mode) {
    cudaMemcpy(d, h.data(), R * C * 8, cudaMemcpyHostToDevice);
    k_tensor<<<1, 128, 64 * 16 * 8>>>(tm, mode);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<double> o(R * C);
    cudaMemcpy(o.data(), d, R * C * 8, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int rr = 0; rr < R; ++rr)
      for (int cc = 0; cc < C; ++cc) {
        double want = 1.0;
        if (rr >= 64 && rr < 128 && cc >= 16 && cc < 32)
          want = (mode == 0 ? 1.0 : 0.0) + (double)((rr - 64) * 100 + (cc - 16));
        if (o[rr * C + cc] != want) ++bad;
      }
    printf("{\"probe\": \"tensor_%s_f64_swizzle128\", \"err\": \"%s\", \"bad\": %d, \"sample\": %.1f}\n",
           mode == 0 ? "reduce_add" : "store", cudaGetErrorString(e), bad, o[70 * C + 20]);
  }
  {
    double* g;
    cudaMalloc(&g, 32 * 8);
    std::vector<double> one(32, 2.0);
    cudaMemcpy(g, one.data(), 256, cudaMemcpyHostToDevice);
    k_flat<<<1, 32>>>(g);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(one.data(), g, 256, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int i = 0; i < 32; ++i) bad += one[i] != 2.0 + 1.5 * i;
    printf("{\"probe\": \"flat_reduce_add_f64\", \"err\": \"%s\", \"bad\": %d}\n", cudaGetErrorString(e), bad);
  }
  return 0;
}
