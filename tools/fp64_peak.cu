// FP64 pipe microbenchmark for sm_100a: DMMA (mma.sync f64) vs DFMA vs both.
// Measures the FP64 tensor-core roofline used as the denominator in bench.py.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

// Each warp: NACC independent 8x8x4 DMMA accumulators, ITERS rounds.
template <int NACC>
__global__ void dmma_loop(double* out, int iters, double seed) {
  double a = seed + threadIdx.x * 1e-3, b = seed * 0.5 + threadIdx.x * 1e-4;
  double acc[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { acc[i][0] = 0.0; acc[i][1] = 0.0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += acc[i][0] + acc[i][1];
  if (s == 1234.5) out[threadIdx.x] = s;
}

template <int NACC>
__global__ void dfma_loop(double* out, int iters, double seed) {
  double a = seed + threadIdx.x * 1e-3, b = 0.999999;
  double acc[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) acc[i] = i * 1e-7;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
#pragma unroll
      for (int i = 0; i < NACC; ++i) acc[i] = fma(acc[i], b, a);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += acc[i];
  if (s == 1234.5) out[threadIdx.x] = s;
}

// Mixed: half of the warps run DMMA, half run DFMA (warp-level split).
template <int NACC>
__global__ void mixed_loop(double* out, int iters, int dfma_iters, double seed) {
  int warp = threadIdx.x / 32;
  if (warp & 1) {
    double a = seed + threadIdx.x * 1e-3, b = 0.999999;
    double acc[NACC];
#pragma unroll
    for (int i = 0; i < NACC; ++i) acc[i] = i * 1e-7;
    for (int it = 0; it < dfma_iters; ++it) {
#pragma unroll
      for (int r = 0; r < 8; ++r) {
#pragma unroll
        for (int i = 0; i < NACC; ++i) acc[i] = fma(acc[i], b, a);
      }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < NACC; ++i) s += acc[i];
    if (s == 1234.5) out[threadIdx.x] = s;
  } else {
    double a = seed + threadIdx.x * 1e-3, b = seed * 0.5 + threadIdx.x * 1e-4;
    double acc[NACC][2];
#pragma unroll
    for (int i = 0; i < NACC; ++i) { acc[i][0] = 0.0; acc[i][1] = 0.0; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < NACC; ++i) {
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(a), "d"(b));
      }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < NACC; ++i) s += acc[i][0] + acc[i][1];
    if (s == 1234.5) out[threadIdx.x] = s;
  }
}

// DMMA latency: a single dependent chain in one warp.
__global__ void dmma_latency(double* out, int iters, long long* cyc) {
  double a = 1.0 + threadIdx.x, b = 0.5;
  double c0 = 0, c1 = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
  long long t1 = clock64();
  if (threadIdx.x == 0) *cyc = t1 - t0;
  if (c0 + c1 == 1234.5) out[0] = c0;
}

int main() {
  int dev = 0;
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int sms = p.multiProcessorCount;
  int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"clock_khz_attr\": %d}\n", p.name, sms, clk_khz);
  double* out; CK(cudaMalloc(&out, 1 << 20));
  long long* cyc; CK(cudaMalloc(&cyc, 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);

  dmma_latency<<<1, 32>>>(out, 10000, cyc); CK(cudaDeviceSynchronize());
  long long hc; CK(cudaMemcpy(&hc, cyc, 8, cudaMemcpyDeviceToHost));
  printf("{\"dmma_dep_latency_cyc\": %.2f}\n", hc / 10000.0);

  auto run = [&](const char* name, auto launch, double flops_per_launch) {
    for (int w = 0; w < 3; ++w) launch();
    CK(cudaDeviceSynchronize());
    const int reps = 10;
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) launch();
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double tf = flops_per_launch * reps / (ms * 1e-3) / 1e12;
    printf("{\"test\": \"%s\", \"ms_per_launch\": %.3f, \"tflops\": %.3f}\n", name, ms / reps, tf);
    return tf;
  };
  const int iters = 4000;
  for (int warps : {4, 8, 16}) {
    int threads = warps * 32;
    for (int bps : {1, 2}) {
      int blocks = sms * bps;
      double flops = (double)blocks * warps * iters * 8 /*NACC*/ * 512.0;
      char nm[64]; snprintf(nm, 64, "dmma_w%d_b%d", warps, bps);
      run(nm, [&] { dmma_loop<8><<<blocks, threads>>>(out, iters, 1.0); }, flops);
    }
  }
  for (int warps : {8, 16, 32}) {
    int threads = warps * 32;
    int blocks = sms;
    double flops = (double)blocks * threads * iters * 8 * 8 * 2.0;
    char nm[64]; snprintf(nm, 64, "dfma_w%d", warps);
    run(nm, [&] { dfma_loop<8><<<blocks, threads>>>(out, iters, 1.0); }, flops);
  }
  // Mixed: 16 warps, 8 DMMA + 8 DFMA; DFMA iterations sized to equal time if separate pipes.
  {
    int warps = 16, threads = warps * 32, blocks = sms;
    int dfma_iters = iters / 2;  // 64 DFMA*32 lanes per iter-unit vs 8 DMMA = 2048 FMA
    double f_dmma = (double)blocks * (warps / 2) * iters * 8 * 512.0;
    double f_dfma = (double)blocks * (warps / 2) * 32 * dfma_iters * 64 * 2.0;
    run("mixed_total", [&] { mixed_loop<8><<<blocks, threads>>>(out, iters, dfma_iters, 1.0); },
        f_dmma + f_dfma);
  }
  return 0;
}
