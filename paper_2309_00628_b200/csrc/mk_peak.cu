// FP64 tensor-pipe roofline probe: every SM issues independent DMMA.8x8x4 chains (no memory
// traffic). Its TFLOP/s is the denominator bench.py reports roofline fractions against,
// measured on the same GPU in the same run (MEASURED_PEAKS.json carries no FP64 figure).
#include <cuda_runtime.h>
#include "mk_device.cuh"

namespace mk {

__global__ void __launch_bounds__(256) dmma_peak_kernel(double* sink, int iters, double seed) {
  const double a = seed + threadIdx.x * 1e-3, b = seed * 0.5 + threadIdx.x * 1e-4;
  double acc[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(acc[i][0]), "+d"(acc[i][1])
                   : "d"(a), "d"(b));
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
  if (s == 1234.5) sink[threadIdx.x] = s;  // keep the chains alive
}

cudaError_t measure_dmma_peak(double* tflops_out, cudaStream_t st) {
  int dev = 0, sms = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return e;
  double* sink = nullptr;
  e = cudaMallocAsync(&sink, 256 * sizeof(double), st);
  if (e != cudaSuccess) return e;
  const int blocks = sms * 2, threads = 256, iters = 4000;
  const double flops = (double)blocks * (threads / 32) * iters * 8 * 512.0;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 2; ++w) dmma_peak_kernel<<<blocks, threads, 0, st>>>(sink, iters, 1.0);
  const int reps = 5;
  cudaEventRecord(e0, st);
  for (int r = 0; r < reps; ++r) dmma_peak_kernel<<<blocks, threads, 0, st>>>(sink, iters, 1.0);
  cudaEventRecord(e1, st);
  e = cudaEventSynchronize(e1);
  float ms = 0.f;
  if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFreeAsync(sink, st);
  if (e != cudaSuccess) return e;
  *tflops_out = flops * reps / (ms * 1e-3) / 1e12;
  return cudaGetLastError();
}

}  // namespace mk
